// args.cuh -- what the host planner and the kernels share: launch
// constants, the block-loop state and argument structs, and the
// shared-memory size formulas of the kernels (sm_100a). No __global__
// code: every translation unit of libaura_b200.so may include it; the
// kernels themselves are only in the one that launches them (engine.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft.cuh"

namespace aura_b200 {

constexpr int kMacThreads = 256;
constexpr int kTailThreads = 256;
constexpr int kFrontThreads = 256;

// Block numbers are 64-bit: a 32-bit counter wraps after 2^32 blocks (16.6
// days at N = 16, 48 kHz) and, as 2^32 is no multiple of K, would reorder
// the delay-line rings (slot = block mod K) at the wrap.
typedef unsigned long long blk_t;

// Device-resident stream state: index of the block in flight. Every kernel
// of block n (front and background) reads it; the last CTA of the
// background's tail kernels (ticket) moves it to n + 1.
struct DevState {
  blk_t block;
  uint32_t ticket;
  uint32_t pad;
};

// Optional timeline trace (%globaltimer, ns): per traced block slot and
// kernel, the earliest CTA start and the latest CTA end.
constexpr int kTraceBlocks = 64;
constexpr int kTraceKernels = 13;  // the last slot carries the next block's front start (cycle)
enum TraceId {
  TR_FRONT = 0, TR_BACK_HEAD, TR_BACK, TR_REDUCE, TR_AFC_DONE, TR_AFC_FINISH, TR_OUTPUT,
  TR_AFC_SUMMED,  // k_reduce: the canceller's split-K sums are in (the CTA that runs the c2r)
  TR_AFC_C2R,     // k_reduce: f^ written (before the power update)
  TR_FRONT_X,     // k_front: this block's input spectra computed and pushed (per front CTA)
  TR_AFC_WAIT,    // k_reduce's early canceller CTA: {resident, partials published}
  TR_AFC_CONS     // k_afc_constrain (constrained NLMS gradient)
};

// Loudspeaker-channel sharding: at most kMaxShards engines
// (one per GPU, or virtual shards on one GPU) exchange their canceller
// partials every block. Each engine owns an exchange buffer: kMaxShards
// u64 flags (flag g = 1 + last block whose partial shard g delivered),
// padded to kXFlagBytes, then slots[2 parities][G][P*N + 2N] floats.
constexpr int kMaxShards = 8;
constexpr size_t kXFlagBytes = 256;
constexpr unsigned long long kShardTimeoutNs = 5ull * 1000 * 1000 * 1000;

struct BlockArgs {
  // geometry
  int N, logN, NF;   // NF = N/2 float4 columns per packed spectrum
  int Q, L, P;       // inputs, outputs, mics (auralizer: P = Q)
  int K, KF;         // synth partitions, canceller partitions
  int mode;          // 0 broadcast, 1 elementwise, 2 mimo
  int is_aur, nlms;
  int afc_cons;      // constrained NLMS gradient (k_afc_constrain updates W; k_back only filters)
  int cons_prefetch; // k_afc_constrain: register prefetch of the next unit (N = 64, 128)
  int cons_tables;   // k_afc_constrain: DftPlan tables staged in shared memory (all but the largest N)
  float gain, mu, lambda, delta;
  int cpb;           // output channels per front CTA
  int front_pre;     // k_front stages its first channel's S and H0 up front
  int smem_tables;   // k_front / k_back_head stage the DftPlan tables in shared memory
  int advance_total; // CTAs that retire the block (k_afc_finish only; k_back counts its own)
  unsigned long long* trace;  // [kTraceBlocks][kTraceKernels][2] or null
  // streaming kernel k_back (stream.cuh): tiling, pipeline, host-planned work
  int CT, CTn;       // float4 columns per column tile, column tiles
  int sp, spa;       // synthesis taps / canceller units per pipeline stage
  int stages;        // shared-memory ring depth
  int slot_f4;       // float4 per ring slot
  int red_f4;        // float4 of reduction (and c2r) scratch
  int n_syn_tiles;   // (L/LT) * CTn
  int h_in_l2;       // spectra fit in L2: stream them with evict_normal
  int w_in_l2;       // canceller W + delay lines fit in L2: keep W there (evict_last)
  const int4* chunks;   // work items {kind | tile << 1, b, e, partial index}:
                        //   [n_static] per-CTA static pieces, then [n_chunks - n_static] queue
  int n_chunks, n_static;
  const int4* cta_first;  // [plan_ctas][2]: {first static item, end, 0, 0}, that item's record
  int plan_ctas;        // CTAs the static pieces were planned for (a larger grid: queue only)
  const int4* tinfo;    // per tile (synthesis, then canceller column tiles):
                        //   {first partial, partials, first group, groups}
  unsigned* tick;       // k_reduce tickets [0] canceller CTAs, [1] all CTAs; [tick_queue] work queue, [+1] k_back exits
  int tick_queue;
  int LTr;              // channels per synthesis tile
  int red_syn_ctas, red_syn_cpt;  // k_reduce: synthesis CTAs, CTAs per tile
  int red_afc_ctas, red_afc_cpt;  // canceller CTAs, CTAs per column tile
  int red_afc_rows;               // canceller partial rows: P (+1 power row with NLMS)
  // single-CTA canceller reduction that starts before k_back ends: per
  // canceller partial, (block + 1) once k_back has published it; k_reduce's
  // canceller CTA (index 0) waits on these words instead of on all of k_back
  blk_t* afc_seq;
  float* hist1;                 // second window-history buffer (the first is prev_in)
  // front CTA b publishes (block + 1) in out_flag[b] (mapped host memory)
  // once it is done with the block's input and its outputs are written --
  // the host polls these words instead of an event; one system-scope
  // release store per CTA (every k_front CTA, the error-spectrum CTAs too,
  // so no CTA still reads the mapped input when process() returns)
  unsigned long long* out_flag;
  // fused head: k_front also runs the canceller head (and, on P extra CTAs,
  // the NLMS error spectra) and k_back is its programmatic dependent; the
  // window history then alternates prev_in / hist1 by block parity
  int front_head;
  unsigned long long* front_seq;  // fused head: [block & 1] front CTAs done (k_reduce clears the slot)
  int front_hold;                 // ... and k_back's producers wait for all of them before streaming
  int front_ctas;                 // k_front CTAs that write outputs
  int front_warps;                // > 0: k_front runs one output channel per warp (front_warps_body)
  unsigned long long* seg_trace;  // diagnostics: [chunks] x {end, cta}, then [ctas] x {start, first data, exit}
  // tables
  const float2* tw;     // N/2, e^{-2 pi i j / N}
  const float2* split;  // N/2+1, e^{-2 pi i k / (2N)}
  // state
  DevState* st;
  float* prev_in;       // Qx x N    previous input block (after g m - f^)
  float* cur_mt;        // Q x N     this block's m~ (front -> background)
  float4* X;            // input FDL (tiled, see above)
  const float4* Ht;     // spectra, partitions >= 1 (tiled)
  const float4* H0;     // partition 0 of every row, contiguous [L][Qh][NF]
  float4* S;            // [L][NF]   precomputed partitions >= 1 for next block
  float4* part_syn;     // split-K partials [slot][LT][CT] (one per chunk)
  float* prev_spk;      // L x N     previous loudspeaker block
  float* spk;           // L x N     l_n (device copy for the canceller stage)
  float4* XA;           // canceller FDL (tiled)
  float4* W;            // canceller spectra (tiled)
  float2* pw;           // [N]       smoothed power (packed: bin0 = DC,Nyq)
  float4* E;            // [P][NF]   error spectra
  float4* part_afc;     // split-K partials [slot][P + nlms][CT] (row P: loudspeaker power)
  float4* yhat;         // [P+1][NF]  reduced canceller spectra (+ power row)
  float* fhat;          // P x N     feedback estimate for the next block
  // sharding: this engine is shard `grank` of G; xchg = how the canceller
  // partials are exchanged: 0 none (unsharded), 1 P2P stores + flags
  // (k_afc_finish), 2 NCCL all-reduce into xsum (+ k_afc_apply)
  int G, grank, xchg;
  float* xmine;                 // [P*N + 2N] this shard's partial f^ and power sum
  float* xsum;                  // [P*N + 2N] the all-reduced sum (xchg 2)
  char* xpeer[kMaxShards];      // every shard's exchange buffer (xpeer[grank] = own)
  unsigned* status_host;        // mapped; nonzero when a peer missed the deadline
  // I/O (device pointers; may alias pinned mapped host memory)
  const float* in;      // Qx x N
  float* out;           // L x N
};

// ---- k_front
// Shared-memory float2 count of the front's work area for Qs shared inputs
// (tables and the first channel's staged S/H0 come on top, see finish_init).
__host__ __device__ inline size_t front_work_f2(int N, int Qs) { return (size_t)N * (Qs + 2); }

// Shared-memory float2 count of front_warps_body for Qs shared inputs and
// W warps: input spectra + window/scratch + tables, then per warp the
// channel's S and H0 (1 + Qs) N, its accumulator and c2r scratch 2N.
__host__ __device__ inline size_t front_warps_f2(int N, int Qs, int W) {
  return (size_t)N * (Qs + 2) + table_f2(N) + (size_t)W * N * (3 + Qs);
}

// ---- k_back (stream.cuh)
constexpr int kConsumers = 256;                 // 8 consumer warps
constexpr int kBackThreads = kConsumers + 64;   // + the producer warp + the signal warp
constexpr int kSigSlots = 4;                    // consumers -> signal warp hand-off ring
constexpr int kMaxStages = 8;
constexpr int kBackBarrierBytes = 512;          // mbarriers + stage metadata at the start of smem

// ---- k_afc_constrain (kernels.cuh): one warp per canceller unit (p, l, k)
constexpr int kConsThreads = 64;  // small CTAs: three fit beside a k_back CTA (registers)
// Shared-memory bytes per warp: the gradient spectrum (N float2), the 2N
// window and the FFT scratch (N float2).
__host__ __device__ inline size_t cons_smem_per_warp(int N) { return (size_t)N * 24; }
// ... after the CTA's copy of the DftPlan tables (16-byte aligned)
__host__ __device__ inline size_t cons_smem_tables(int N) { return ((size_t)table_f2(N) * 8 + 15) / 16 * 16; }

// ---- k_reduce (stream.cuh)
constexpr int kReduceThreads = 256;

// Shared-memory float4 count of k_reduce's scratch: the combine buffer, and
// for the canceller the c2r scratch (N float2), the DftPlan tables and the
// smoothed power (N float2).
// Canceller sums kept in shared memory by the single-CTA path (one column
// tile, N <= 64): (P + 1) rows of NF float4.
__host__ __device__ inline size_t afc_ys_f4(int N, int P) { return N <= 64 ? (size_t)(P + 1) * (N / 2) : 0; }
__host__ __device__ inline size_t reduce_smem_f4(int N, bool aur, int P = 1) {
  // c2r scratch: one N-float2 area per mic when the mics' c2r run on separate warps
  const size_t scratch = (N <= 1024 ? (size_t)P : 1) * N;
  return kReduceThreads + (aur ? afc_ys_f4(N, P) + (scratch + N + table_f2(N) + 1) / 2 : 0);
}

// ---- k_partition
// Where k_partition scatters row r's partition spectra (see kernels.cuh).
struct PartOut {
  float4* dst;
  float4* dst0;
  long long kstride, cstride;
  int CT;
};

}  // namespace aura_b200
