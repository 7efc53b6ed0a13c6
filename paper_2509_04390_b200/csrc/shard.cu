// shard.cu -- loudspeaker-channel sharding of an auralizer across GPUs
// (DESIGN.md section 6): the exchange buffers, their CUDA IPC
// wiring (aura_b200_shard_*), and the NCCL transport kept as the ablation.
// The exchange kernels themselves (k_afc_finish / k_afc_apply) are launched
// by the block graph (engine.cu).
#include "engine.hpp"

extern "C" {

namespace {

void shard_alloc(aura_b200_engine* e, int world, int rank) {
  if (!e->aur)
    fail(AURA_B200_E_INVALID_ARGUMENT,
         "only a feedback canceller exchanges data between shards (convolver shards are independent)");
  if (world < 2 || world > kMaxShards || rank < 0 || rank >= world)
    fail(AURA_B200_E_INVALID_ARGUMENT, "shard world must be 2..8 and 0 <= rank < world");
  if (e->xbuf || e->args.xchg) fail(AURA_B200_E_INVALID_ARGUMENT, "engine is already sharded");
  if (e->blocks) fail(AURA_B200_E_INVALID_ARGUMENT, "shard before the first block");
  CK(cudaSetDevice(e->device));
  const size_t S = e->P * e->N + 2 * e->N;
  e->xbuf_bytes = kXFlagBytes + 2 * (size_t)world * S * sizeof(float);
  e->xbuf = reinterpret_cast<char*>(dalloc<float>(e->xbuf_bytes / sizeof(float), e->dmem));
  CK(cudaMemset(e->xbuf, 0, e->xbuf_bytes));
  e->args.xmine = dalloc<float>(S, e->dmem);
  CK(cudaMemset(e->args.xmine, 0, S * sizeof(float)));
  e->G = world;
  e->grank = rank;
}

// NCCL exchange: the exchange buffers, the communicator (one per engine,
// ranks = shards), then the graphs with the all-reduce captured in them.
void nccl_connect(aura_b200_engine* e, int world, int rank, const void* id) {
  if (!e->aur)
    fail(AURA_B200_E_INVALID_ARGUMENT,
         "only a feedback canceller exchanges data between shards (convolver shards are independent)");
  if (world < 1 || world > kMaxShards || rank < 0 || rank >= world)
    fail(AURA_B200_E_INVALID_ARGUMENT, "shard world must be 1..8 and 0 <= rank < world");
  if (e->args.xchg) fail(AURA_B200_E_INVALID_ARGUMENT, "engine is already sharded");
  if (e->blocks) fail(AURA_B200_E_INVALID_ARGUMENT, "shard before the first block");
  NcclApi& api = nccl_api();
  CK(cudaSetDevice(e->device));
  const size_t S = e->P * e->N + 2 * e->N;
  e->args.xmine = dalloc<float>(S, e->dmem);
  e->args.xsum = dalloc<float>(S, e->dmem);
  CK(cudaMemset(e->args.xmine, 0, S * sizeof(float)));
  CK(cudaMemset(e->args.xsum, 0, S * sizeof(float)));
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  nccl_check(api.init_rank(&e->nccl, world, uid, rank), "ncclCommInitRank");
  e->G = world;
  e->grank = rank;
  BlockArgs& a = e->args;
  a.G = world;
  a.grank = rank;
  a.xchg = 2;
  set_advance_total(e);
  CK(cudaStreamSynchronize(e->stream));
  e->rebuild_graphs();
  BlockArgs d = a;
  d.out = e->d_out;
  d.in = e->d_in_pool;
  d.out_flag = nullptr;
  e->dev_args = d;
}

void shard_finalize(aura_b200_engine* e, char* const* peers) {
  CK(cudaSetDevice(e->device));
  BlockArgs& a = e->args;
  a.G = e->G;
  a.grank = e->grank;
  a.xchg = 1;
  for (int g = 0; g < kMaxShards; ++g) a.xpeer[g] = g < e->G ? peers[g] : nullptr;
  set_advance_total(e);
  CK(cudaStreamSynchronize(e->stream));
  e->rebuild_graphs();
  BlockArgs d = a;
  d.out = e->d_out;
  d.in = e->d_in_pool;
  d.out_flag = nullptr;
  e->dev_args = d;
}

}  // namespace

int aura_b200_shard_export(aura_b200_engine* e, int world, int rank, void* handle) {
  return guarded([&] {
    if (!e || !handle) fail(AURA_B200_E_INVALID_ARGUMENT, "null argument");
    shard_alloc(e, world, rank);
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, e->xbuf));
    static_assert(sizeof(h) == AURA_B200_SHARD_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle, &h, sizeof h);
  });
}

int aura_b200_shard_connect(aura_b200_engine* e, const void* handles) {
  return guarded([&] {
    if (!e || !handles) fail(AURA_B200_E_INVALID_ARGUMENT, "null argument");
    if (!e->xbuf) fail(AURA_B200_E_INVALID_ARGUMENT, "call aura_b200_shard_export first");
    CK(cudaSetDevice(e->device));
    std::vector<char*> peers(e->G, nullptr);
    for (int g = 0; g < e->G; ++g) {
      if (g == e->grank) {
        peers[g] = e->xbuf;
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, static_cast<const char*>(handles) + (size_t)g * sizeof h, sizeof h);
      void* p = nullptr;
      CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
      e->ipc_opened.push_back(p);
      peers[g] = static_cast<char*>(p);
    }
    shard_finalize(e, peers.data());
  });
}

int aura_b200_shard_connect_local(aura_b200_engine* const* engines, int world) {
  return guarded([&] {
    if (!engines) fail(AURA_B200_E_INVALID_ARGUMENT, "null argument");
    for (int g = 0; g < world; ++g)
      if (!engines[g]) fail(AURA_B200_E_INVALID_ARGUMENT, "null engine");
    for (int g = 0; g < world; ++g) shard_alloc(engines[g], world, g);
    // engines on different devices of one process reach each other by P2P
    for (int g = 0; g < world; ++g)
      for (int h = 0; h < world; ++h) {
        const int dg = engines[g]->device, dh = engines[h]->device;
        if (dg == dh) continue;
        int ok = 0;
        CK(cudaDeviceCanAccessPeer(&ok, dg, dh));
        if (!ok) fail(AURA_B200_E_BACKEND_UNAVAILABLE, "devices cannot access each other (no P2P)");
        CK(cudaSetDevice(dg));
        const cudaError_t r = cudaDeviceEnablePeerAccess(dh, 0);
        if (r != cudaErrorPeerAccessAlreadyEnabled) ck(r, "cudaDeviceEnablePeerAccess");
        cudaGetLastError();
      }
    std::vector<char*> peers(world);
    for (int g = 0; g < world; ++g) peers[g] = engines[g]->xbuf;
    for (int g = 0; g < world; ++g) shard_finalize(engines[g], peers.data());
  });
}

int aura_b200_nccl_unique_id(void* id) {
  return guarded([&] {
    if (!id) fail(AURA_B200_E_INVALID_ARGUMENT, "null argument");
    ncclUniqueId uid;
    nccl_check(nccl_api().get_unique_id(&uid), "ncclGetUniqueId");
    std::memcpy(id, &uid, sizeof uid);
  });
}

int aura_b200_shard_connect_nccl(aura_b200_engine* e, int world, int rank, const void* id) {
  return guarded([&] {
    if (!e || !id) fail(AURA_B200_E_INVALID_ARGUMENT, "null argument");
    nccl_connect(e, world, rank, id);
  });
}

int aura_b200_shard_info(const aura_b200_engine* e, int* world, int* rank) {
  return guarded([&] {
    if (!e || !world || !rank) fail(AURA_B200_E_INVALID_ARGUMENT, "null argument");
    *world = e->G;
    *rank = e->grank;
  });
}

}  // extern "C"
