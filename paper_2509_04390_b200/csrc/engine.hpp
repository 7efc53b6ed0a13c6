// engine.hpp -- the host side of libaura_b200.so shared by its three
// translation units: engine.cu (construction, the work planner, the block
// loop and the reference-replacing C-ABI of include/aura_b200.h -- the only
// unit that contains the kernels), shard.cu (multi-GPU loudspeaker
// sharding) and diag.cu (the measurement / diagnostics C-ABI of
// include/aura_b200_diag.h). Internal: not installed, not part of the ABI.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include "../../include/aura_b200_diag.h"
#include "args.cuh"

using namespace aura_b200;

extern thread_local std::string g_err;  // aura_b200_last_error() (engine.cu)

struct Fail {
  int code;
  std::string msg;
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Fail{code, msg}; }

inline void ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  cudaGetLastError();
  if (e == cudaErrorMemoryAllocation)
    fail(AURA_B200_E_OUT_OF_MEMORY, std::string(what) + ": " + cudaGetErrorString(e));
  fail(AURA_B200_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CK(x) ck((x), #x)

// Raise a kernel's dynamic shared-memory limit on the current device, never
// lower it: the attribute is per function, so engines of different shapes in
// one process must not undo each other's (a smaller engine created after a
// larger one would otherwise make the larger one's launches invalid).
template <typename Fn>
void raise_smem_limit(Fn fn, size_t bytes) {
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  cudaFuncAttributes fa{};
  CK(cudaFuncGetAttributes(&fa, (const void*)fn));
  if ((size_t)fa.maxDynamicSharedSizeBytes < bytes)
    CK(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return AURA_B200_OK;
  } catch (const Fail& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return AURA_B200_E_OUT_OF_MEMORY;
  }
}

inline bool is_pow2(size_t v) { return v && !(v & (v - 1)); }
inline int ilog2(size_t v) {
  int r = 0;
  while ((size_t(1) << r) < v) ++r;
  return r;
}

// engine.hpp:74-94 (validate_config), same codes and precedence. MIMO (an
// extension) lifts only the C_in in {1, C_out} rule.
inline void validate(const aura_b200_config* c, bool mimo) {
  if (!c) fail(AURA_B200_E_INVALID_ARGUMENT, "config is null");
  if (c->sample_rate_hz == 0) fail(AURA_B200_E_ZERO_SAMPLE_RATE, "sample rate must be positive");
  if (!is_pow2(c->block_size) || c->block_size < 16 || c->block_size > 8192)
    fail(AURA_B200_E_NON_POWER_OF_TWO_BLOCK,
         "block size must be a power of two in [16, 8192], got " + std::to_string(c->block_size));
  if (c->fft_size != 2 * c->block_size)
    fail(AURA_B200_E_FFT_SIZE_MISMATCH, "fft size must be 2 * block size");
  if (c->outputs == 0 || c->inputs == 0 ||
      (!mimo && c->inputs != 1 && c->inputs != c->outputs))
    fail(AURA_B200_E_BAD_CHANNEL_COMBINATION,
         "input channels must be 1 or equal to output channels");
}

// NLMS regulariser default: SURVEY Appendix A's delta = 1e-6 N (DESIGN.md
// section 4: at this value the GPU's W error against a float64 run is within
// 1.5x of the fp32 C oracle's own).
constexpr float kDefaultDeltaPerN = 1e-6f;

template <class T>
T* dalloc(size_t count, std::vector<void*>& owned) {
  void* p = nullptr;
  if (count == 0) count = 1;
  CK(cudaMalloc(&p, count * sizeof(T)));
  owned.push_back(p);
  return static_cast<T*>(p);
}

// NCCL, loaded on first use (dlopen): only the NCCL exchange ablation needs
// it, so the library loads and runs without NCCL installed.
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allreduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string why;
};
inline NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.init_rank = reinterpret_cast<decltype(api.init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.allreduce = reinterpret_cast<decltype(api.allreduce)>(dlsym(h, "ncclAllReduce"));
    api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(h, "ncclCommDestroy"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!api.get_unique_id || !api.init_rank || !api.allreduce || !api.destroy || !api.error_string)
      api.why = "libnccl.so.2 lacks the NCCL 2 API";
  });
  if (!api.why.empty()) fail(AURA_B200_E_BACKEND_UNAVAILABLE, "NCCL exchange unavailable: " + api.why);
  return api;
}
inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(AURA_B200_E_CUDA, std::string(what) + ": " + nccl_api().error_string(r));
}


enum Phase { PH_FRONT = 0, PH_BACK_HEAD, PH_BACK, PH_REDUCE, PH_AFC_FINISH, PH_ADVANCE, PH_COUNT };
static const char* kPhaseNames[PH_COUNT] = {"k_front",  "k_back_head",  "k_back",
                                            "k_reduce", "k_afc_finish", "k_advance"};

using BackFn = void (*)(BlockArgs);

// Poll until the stream has drained (true) or `seconds` pass (false).
inline bool wait_stream_idle(cudaStream_t s, double seconds) {
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = cudaStreamQuery(s);
    if (q != cudaErrorNotReady) {
      cudaGetLastError();
      return true;
    }
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > seconds) return false;
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

struct aura_b200_engine {
  int device = 0;
  int sms = 148;
  bool aur = false;
  int mode = 0;
  size_t N = 0, Q = 1, L = 1, P = 0, K = 0, KF = 0, n_h = 0, n_hf = 0;
  int Qx = 1;  // FDL channels
  int LT = 1, PT = 0;
  uint64_t blocks = 0;
  cudaStream_t stream = nullptr;  // the engine's stream
  cudaEvent_t ev_front = nullptr;  // output ready (only without output words, OUTFLAG=0)
  std::vector<void*> dmem;
  float4* W0 = nullptr;  // initial canceller spectra (reset of NLMS)
  size_t w_elems = 0;
  float* h_in = nullptr;    // mapped pinned
  // failure detection: process() / process_io() latency vs the budget N / f_s
  double budget_us = 0.0, max_us = 0.0, last_us = 0.0;
  uint64_t deadline_misses = 0;
  float* h_out = nullptr;   // mapped pinned
  float* d_in_pool = nullptr;
  size_t pool_blocks = 0;
  float* d_out = nullptr;
  BlockArgs args{};
  BlockArgs dev_args{};
  struct BlockGraph {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ex = nullptr;
    cudaGraphNode_t out_node = nullptr;  // external event-record node (output ready)
    cudaGraphNode_t end_node = nullptr;  // event-record node after the block's last kernel
    void destroy() {
      if (ex) cudaGraphExecDestroy(ex);
      if (g) cudaGraphDestroy(g);
      ex = nullptr;
      g = nullptr;
    }
  };
  BlockGraph g_block;
  // streaming kernel k_back
  BackFn back_fn = nullptr;
  bool pdl_off = false;  // measurement: serialise k_back / k_reduce launches
  int launch_mode = 0;   // 0: one CUDA graph per block; 1: the same kernels launched on the stream
  unsigned long long* h_outflag = nullptr;  // mapped: k_front CTA b writes block + 1 in [b] when done
  size_t n_outflags = 0;    // = k_front's grid (every CTA that reads the mapped input)
  bool use_outflag = true;
  std::string knobs;        // non-default AURA_B200_* tuning knobs in effect (describe())
  uint64_t block_base = 0;  // device number of host block 0 (aura_b200_seek_block; else 0)
  int back_ctas = 0;
  size_t smem_back = 0, smem_reduce = 0;
  size_t n_syn_segs = 0, n_afc_segs = 0;
  size_t n_afc_seq = 0;  // words of args.afc_seq (early canceller reduction)
  std::vector<int4> h_chunks;  // host copy of the k_back work queue (diagnostics)
  // sharding: shard grank of G; xbuf = own exchange buffer
  int G = 1, grank = 0;
  char* xbuf = nullptr;
  size_t xbuf_bytes = 0;
  std::vector<void*> ipc_opened;  // peer buffers opened through CUDA IPC
  ncclComm_t nccl = nullptr;      // NCCL exchange (xchg 2)
  unsigned* h_status = nullptr;   // mapped pinned; set by k_afc_finish on timeout
  size_t smem_front = 0, smem_head = 0;
  size_t smem_cons = 0;  // k_afc_constrain (constrained NLMS gradient)
  int cons_ctas = 0, cons_warps = 0;
  bool cons8 = false;  // k_afc_constrain8 (N = 64)

  ~aura_b200_engine() {
    cudaSetDevice(device);
    // wedged (a shard peer that never arrives is bounded in-kernel, but be
    // safe): leak rather than block, the frees below would synchronise
    if (stream && !wait_stream_idle(stream, 10.0)) return;
    g_block.destroy();
    for (void* p : dmem) cudaFree(p);
    if (h_in) cudaFreeHost(h_in);
    if (h_out) cudaFreeHost(h_out);
    if (h_status) cudaFreeHost(h_status);
    if (h_outflag) cudaFreeHost(h_outflag);
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    if (nccl) nccl_api().destroy(nccl);
    if (ev_front) cudaEventDestroy(ev_front);
    if (stream) cudaStreamDestroy(stream);
  }

  bool has_syn() const { return K > 1; }
  bool has_back() const { return has_syn() || aur; }
  bool front_head = true;  // k_front runs the canceller head; k_back is its PDL dependent
  bool has_head() const { return !front_head && (aur || mode != AURA_B200_ELEMENTWISE); }
  int front_grid(const BlockArgs& a) const {
    return (int)((L + a.cpb - 1) / a.cpb) + ((front_head && aur && a.nlms) ? (int)P : 0);
  }
  bool sharded() const { return aur && args.xchg != 0; }

  // k_back after k_back_head is a programmatic dependent launch: it starts
  // while k_back_head runs and waits for it (griddepcontrol.wait) only where
  // it reads k_back_head's outputs.
  template <typename Kern>
  void launch_pdl(Kern kern, unsigned grid, unsigned threads, size_t smem, bool pdl, const BlockArgs& a,
                  cudaStream_t s) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    CK(cudaLaunchKernelEx(&cfg, kern, a));
  }

  // launch one phase kernel of a block (engine.cu: the only translation
  // unit with the kernels)
  void launch_phase(int ph, const BlockArgs& a, cudaStream_t s);

  // kernels launched per block
  int launches_per_block() const {
    return 1 + (has_head() ? 1 : 0) + (has_back() ? 2 : 0) + (sharded() ? 1 : 0) +  // (+ NCCL's own)
           (has_back() ? 0 : 1) + (args.afc_cons ? 1 : 0);
  }

  // One graph per block: k_front, an external event node the host waits on
  // (output ready), then k_back_head -> k_back (PDL) [-> k_afc_finish].
  // end_event (measurement): an event-record node after the block's last
  // kernel, re-pointed per launch -- per-block device times without an
  // extra operation in the stream between two block graphs
  BlockGraph capture_block(const BlockArgs& a, cudaEvent_t out_event, cudaEvent_t end_event = nullptr) {
    BlockGraph bg;
    CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
    launch_phase(PH_FRONT, a, stream);
    if (out_event) CK(cudaEventRecordWithFlags(out_event, stream, cudaEventRecordExternal));
    for (int ph = PH_BACK_HEAD; ph < PH_COUNT; ++ph) launch_phase(ph, a, stream);
    if (end_event) CK(cudaEventRecordWithFlags(end_event, stream, cudaEventRecordExternal));
    CK(cudaStreamEndCapture(stream, &bg.g));
    if (out_event || end_event) {
      size_t n = 0;
      CK(cudaGraphGetNodes(bg.g, nullptr, &n));
      std::vector<cudaGraphNode_t> nodes(n);
      CK(cudaGraphGetNodes(bg.g, nodes.data(), &n));
      for (auto nd : nodes) {
        cudaGraphNodeType t;
        CK(cudaGraphNodeGetType(nd, &t));
        if (t != cudaGraphNodeTypeEventRecord) continue;
        cudaEvent_t ev = nullptr;
        CK(cudaGraphEventRecordNodeGetEvent(nd, &ev));
        if (ev == out_event) bg.out_node = nd;
        if (ev == end_event) bg.end_node = nd;
      }
    }
    CK(cudaGraphInstantiate(&bg.ex, bg.g, 0));
    return bg;
  }

  // Enqueue one block on the stream: the graph, or (launch_mode 1) the same
  // kernels launched directly (PDL edges included); out_event is recorded
  // after k_front.
  void enqueue_block(const BlockGraph& g, const BlockArgs& a, cudaEvent_t out_event) {
    if (launch_mode == 0) {
      CK(cudaGraphLaunch(g.ex, stream));
      return;
    }
    launch_phase(PH_FRONT, a, stream);
    if (out_event) CK(cudaEventRecord(out_event, stream));
    for (int ph = PH_BACK_HEAD; ph < PH_COUNT; ++ph) launch_phase(ph, a, stream);
  }

  void rebuild_graphs() {
    g_block.destroy();
    // no event node after k_front unless the host waits on it: a node
    // between k_front and k_back would stand in their programmatic edge
    g_block = capture_block(args, use_outflag ? nullptr : ev_front);
  }

  // Every device buffer a block writes (measurement calls that relaunch
  // kernels snapshot and restore them): {pointer, bytes}
  std::vector<std::pair<void*, size_t>> mutable_state() const {
    const size_t NF = N / 2, f4 = sizeof(float4), fl = sizeof(float);
    const BlockArgs& a = args;
    std::vector<std::pair<void*, size_t>> v = {
        {a.st, sizeof(DevState)},
        {a.prev_in, fl * Qx * N},
        {a.hist1, fl * Qx * N},
        {a.cur_mt, fl * std::max<size_t>(1, Q) * N},
        {a.X, f4 * Qx * K * NF},
        {a.S, f4 * L * NF},
        {a.part_syn, f4 * std::max<size_t>(1, n_syn_segs * LT * a.CT)},
        {a.front_seq, 2 * sizeof(unsigned long long)},
        {a.tick, 6 * sizeof(unsigned)}};
    if (a.afc_seq) v.push_back({a.afc_seq, n_afc_seq * sizeof(blk_t)});
    if (aur) {
      v.push_back({a.prev_spk, fl * L * N});
      v.push_back({a.spk, fl * L * N});
      v.push_back({a.XA, f4 * L * (KF + 1) * NF});
      v.push_back({a.W, f4 * w_elems});
      v.push_back({a.pw, sizeof(float2) * N});
      v.push_back({a.E, f4 * Q * NF});
      v.push_back({a.fhat, fl * P * N});
      v.push_back({a.part_afc, f4 * std::max<size_t>(1, n_afc_segs * (P + 1) * a.CT)});
      v.push_back({a.yhat, f4 * (P + 1) * NF});
      if (a.xmine) v.push_back({a.xmine, fl * (P * N + 2 * N)});
    }
    return v;
  }

  // algorithmic HBM bytes per block: 8N per packed partition
  double phase_bytes(int ph) const {
    const double row = 8.0 * (double)N;  // one packed partition
    const double Qh = mode == AURA_B200_MIMO ? (double)Q : 1.0;
    switch (ph) {
      case PH_FRONT:  // inputs, X push, H[.][.][0], S, outputs
        return 4.0 * N * Qx + row * Qx + row * (double)L * Qh + row * L + 4.0 * N * L;
      case PH_BACK: {
        double b = has_syn() ? row * ((double)L * Qh * (K - 1) + (double)Qx * (K - 1)) : 0.0;
        if (aur) b += row * ((double)P * L * KF * (1.0 + (args.nlms ? 1.0 : 0.0)) + (double)L * KF);
        return b;
      }
      case PH_REDUCE: {  // the split-K partials, read once
        const double E = (double)LT * args.CT * 16.0;
        return (double)n_syn_segs * E + (double)n_afc_segs * args.red_afc_rows * args.CT * 16.0;
      }
      case PH_AFC_FINISH:  // push P*N + 2N floats to G shards, read G slots
        return sharded() ? 2.0 * G * 4.0 * (double)(P * N + 2 * N) : 0.0;
      case PH_BACK_HEAD: return aur ? (row + 8.0 * N) * L + row * P : 4.0 * N * Qx;
    }
    return 0.0;
  }
};

// CTAs that tick the block ticket in retire_block: only the sharded
// canceller's k_afc_finish (k_back retires a block itself).
inline void set_advance_total(aura_b200_engine* e) { e->args.advance_total = e->sharded() ? 1 : 0; }

// The device block number the next graph launch will process: the host
// counts blocks; measurement calls advance host and device together.
inline uint64_t device_block_hint(aura_b200_engine* e) { return e->blocks + e->block_base; }

// A shard peer missed the canceller exchange deadline (k_afc_finish): the
// engine's f^ stopped tracking the other shards', so every call fails until
// a coordinated reset of all shards.
inline void check_shard_status(aura_b200_engine* e) {
  if (e->h_status && *reinterpret_cast<volatile unsigned*>(e->h_status))
    fail(AURA_B200_E_TIMEOUT, *reinterpret_cast<volatile unsigned*>(e->h_status) == 2u
                                  ? "the canceller reduction timed out waiting for its partials (reset)"
                                  : "a shard peer missed the canceller exchange deadline (reset every shard)");
}

// Spin until every k_front CTA has published `target` in its mapped word.
inline void wait_flag(aura_b200_engine* e, unsigned long long target, const char* what) {
  volatile unsigned long long* f = e->h_outflag;
  uint64_t spins = 0;
  const auto t0 = std::chrono::steady_clock::now();
  size_t i = 0;
  for (;;) {
    while (i < e->n_outflags && f[i] >= target) ++i;
    if (i == e->n_outflags) break;
#if defined(__x86_64__)
    _mm_pause();
#endif
    if ((++spins & 0xFFFF) == 0) {
      const cudaError_t q = cudaStreamQuery(e->stream);
      if (q != cudaErrorNotReady && q != cudaSuccess) ck(q, what);
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(20))
        fail(AURA_B200_E_TIMEOUT, std::string(what) + ": not complete within 20 s");
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
}

// Spin until `ev` (recorded on the engine stream; null: the whole stream)
// has completed; kernel completion makes the block's writes visible.
inline void wait_event(aura_b200_engine* e, cudaEvent_t ev, const char* what) {
  uint64_t spins = 0;
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t q = ev ? cudaEventQuery(ev) : cudaStreamQuery(e->stream);
    if (q == cudaSuccess) break;
    if (q != cudaErrorNotReady) ck(q, what);
#if defined(__x86_64__)
    _mm_pause();
#endif
    if ((++spins & 0xFFF) == 0 &&
        std::chrono::steady_clock::now() - t0 > std::chrono::seconds(20))
      fail(AURA_B200_E_TIMEOUT, std::string(what) + ": not complete within 20 s");
  }
  std::atomic_thread_fence(std::memory_order_acquire);
}

