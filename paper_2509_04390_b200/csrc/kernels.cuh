// kernels.cuh -- the per-block UPOLS + feedback-canceller kernels (sm_100a).
//
// Block n runs as two CUDA graphs on one stream; completion is observed by
// the host through stream events (no system-scope fences inside kernels).
//
//  FRONT (the latency-critical path, one kernel):
//   k_front       m~ = g m - f^ (auralizer.hpp:73-76), window + r2c of every
//                 input (convolver.hpp:180-191), FDL push, then per output
//                 channel  Y_l = S_l + sum_q X_q,n (.) H_{l,q}[0],  c2r +
//                 overlap-save straight into the (mapped) output buffer.
//
//  BACK (off the critical path; two concurrent branches, then k_advance):
//   branch 1: k_mac_pre
//                 S_l for block n+1 = sum_{j=0}^{K-2} X(age j) (.) H_l[j+1]:
//                 every partition but the first depends only on inputs <= n.
//   branch 2: k_back_head -> k_mac_afc [-> k_afc_finish when sharded]
//                 canceller stage 1 on l_n (r2c, FDL push), NLMS error
//                 spectra, canceller MAC with the fused NLMS update and the
//                 loudspeaker power, one c2r per mic -> f^ for block n+1.
//   Both MACs end with a fused split-K reduction (split_k_reduce): the last
//   CTA of each group of chunks sums that group, the last group-reducer sums
//   the groups -- no separate reduction kernel. The CTAs that finish a
//   reduction tree tick the block ticket; the last one advances the block
//   counter (k_advance only when a block has no MAC).
//
// So the output of block n is c2r(X_n H_0 + sum_{k>=1} X_{n-k} H_k), exactly
// the reference's accumulator (backend.hpp:212-235) with the partition sum
// split in two; the work per block is unchanged, only its position in time.
// All reductions run in a fixed order -- split-K partials are summed chunk
// by chunk, then group by group, whichever CTA happens to arrive last -- so
// results are bit-reproducible run to run (test_convolver.cpp:172-193).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cooperative_groups.h>

#include "fft.cuh"

namespace aura_b200 {

constexpr int kMacThreads = 256;
constexpr int kTailThreads = 256;
constexpr int kFrontThreads = 256;

// Device-resident stream state: index of the block in flight. Every kernel
// of block n (front and background) reads it; the last CTA of the
// background's tail kernels (ticket) moves it to n + 1.
struct DevState {
  uint32_t block;
  uint32_t ticket;
  uint32_t pad[2];
};

// Optional timeline trace (%globaltimer, ns): per traced block slot and
// kernel, the earliest CTA start and the latest CTA end.
constexpr int kTraceBlocks = 64;
constexpr int kTraceKernels = 8;
enum TraceId {
  TR_FRONT = 0, TR_MAC_PRE, TR_TAIL_PRE, TR_BACK_HEAD, TR_MAC_AFC, TR_TAIL_AFC, TR_AFC_FINISH
};

// Loudspeaker-channel sharding: at most kMaxShards engines
// (one per GPU, or virtual shards on one GPU) exchange their canceller
// partials every block. Each engine owns an exchange buffer: kMaxShards
// uint32 flags (flag g = 1 + last block whose partial shard g delivered),
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
  float gain, mu, lambda, delta;
  int cpb;           // output channels per front CTA
  int advance_total; // CTAs of the tail kernels that retire the block (ticket)
  unsigned long long* trace;  // [kTraceBlocks][kTraceKernels][2] or null
  // split-K geometry
  int syn_chunks, syn_tc, syn_nft, syn_tiles, syn_g1;  // g1: chunks per level-1 reducer
  int afc_chunks, afc_uc, afc_nft, afc_tiles, afc_g1;
  // tables
  const float2* tw;     // N/2, e^{-2 pi i j / N}
  const float2* split;  // N/2+1, e^{-2 pi i k / (2N)}
  // state
  DevState* st;
  float* prev_in;       // Qx x N    previous input block (after g m - f^)
  float* cur_mt;        // Q x N     this block's m~ (front -> background)
  float4* X;            // input FDL [Qx][K][NF]
  const float4* H;      // spectra   [L][Qh][K][NF] (Qh = Q for mimo, else 1)
  const float4* H0;     // partition 0 of every row, contiguous [L][Qh][NF]
  float4* S;            // [L][NF]   precomputed partitions >= 1 for next block
  float4* part_syn;     // [syn_chunks][L][NF]   split-K partials
  float4* part_syn2;    // [ceil(syn_chunks/8)][L][NF] level-2 partials
  unsigned* tick_syn;   // [L/LT][syn_tiles][ceil(syn_chunks/8) + 1] reduction tickets
  float* prev_spk;      // L x N     previous loudspeaker block
  float* spk;           // L x N     l_n (device copy for the canceller stage)
  float4* XA;           // canceller FDL [L][KF+1][NF]
  float4* W;            // canceller spectra [P][L][KF][NF]
  float2* pw;           // [N]       smoothed power (packed: bin0 = DC,Nyq)
  float4* E;            // [P][NF]   error spectra
  float4* part_afc;     // [afc_chunks][P+1][NF] (row P: loudspeaker power)
  float4* part_afc2;    // [ceil(afc_chunks/8)][P+1][NF]
  float4* yhat;         // [P+1][NF]  reduced canceller spectra (+ power row)
  unsigned* tick_afc;   // [afc_tiles][ceil(afc_chunks/8) + 1] + 1 (tiles)
  float* fhat;          // P x N     feedback estimate for the next block
  float* fhat_host;     // P x N     same, mapped pinned host copy
  // sharding (G > 1): this engine is shard `grank` of G
  int G, grank;
  float* xmine;                 // [P*N + 2N] this shard's partial f^ and power sum
  char* xpeer[kMaxShards];      // every shard's exchange buffer (xpeer[grank] = own)
  unsigned* status_host;        // mapped; nonzero when a peer missed the deadline
  // I/O (device pointers; may alias pinned mapped host memory)
  const float* in;      // Qx x N
  float* out;           // L x N
};

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ float4 ld_stream(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}

// Packed-spectrum complex MAC over one float4 (two bins). For column 0 the
// first pair is (DC, Nyquist), both real: acc.x += x.x*h.x, acc.y +=
// x.y*h.y. xr0/xi0 are x.x/x.y with the cross terms zeroed on that lane.
struct XPack {
  float4 v;
  float xr0, xi0;
};
__device__ __forceinline__ XPack xpack(float4 x, bool dc) {
  XPack p;
  p.v = x;
  p.xr0 = dc ? 0.0f : x.x;
  p.xi0 = dc ? 0.0f : x.y;
  return p;
}
__device__ __forceinline__ void cmac(float4& acc, const XPack& x, float4 h, bool dc) {
  const float hr0 = dc ? h.y : h.x;
  acc.x = fmaf(x.v.x, h.x, acc.x);
  acc.x = fmaf(-x.xi0, h.y, acc.x);
  acc.y = fmaf(x.xr0, h.y, acc.y);
  acc.y = fmaf(x.v.y, hr0, acc.y);
  acc.z = fmaf(x.v.z, h.z, acc.z);
  acc.z = fmaf(-x.v.w, h.w, acc.z);
  acc.w = fmaf(x.v.z, h.w, acc.w);
  acc.w = fmaf(x.v.w, h.z, acc.w);
}
// same on one packed complex bin j (float2 granularity)
__device__ __forceinline__ float2 cmac2(float2 acc, float2 x, float2 h, bool dc) {
  if (dc) return make_float2(fmaf(x.x, h.x, acc.x), fmaf(x.y, h.y, acc.y));
  acc.x = fmaf(x.x, h.x, acc.x);
  acc.x = fmaf(-x.y, h.y, acc.x);
  acc.y = fmaf(x.x, h.y, acc.y);
  acc.y = fmaf(x.y, h.x, acc.y);
  return acc;
}
__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

__device__ __forceinline__ int ring(int v, int cap) {
  v %= cap;
  return v < 0 ? v + cap : v;
}

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_begin(const BlockArgs& a, int id, uint32_t n) {
  if (a.trace && threadIdx.x == 0)
    atomicMin(&a.trace[((n % kTraceBlocks) * kTraceKernels + id) * 2], globaltimer());
}
__device__ __forceinline__ void trace_end(const BlockArgs& a, int id, uint32_t n) {
  if (a.trace) {
    __syncthreads();
    if (threadIdx.x == 0)
      atomicMax(&a.trace[((n % kTraceBlocks) * kTraceKernels + id) * 2 + 1], globaltimer());
  }
}
// Last CTA of the background's tail kernels advances the block counter.
// Device scope suffices: every reader of st->block for block n has read it
// before its CTA reached this point, and the next block's front is
// stream-ordered after the whole background graph.
__device__ void retire_block(const BlockArgs& a, uint32_t n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(&a.st->ticket, 1u) == (uint32_t)a.advance_total - 1) {
      a.st->ticket = 0;
      a.st->block = n + 1;
    }
  }
}

// Sum cnt partial rows src[i*stride] (i = 0..cnt-1) for E elements with the
// whole CTA. Each element gets `sub` threads; thread j of an element sums a
// fixed contiguous range of rows in order with 8 loads in flight, and the
// sub-sums are then added in j order through shared `red` (>= blockDim
// float4). Fixed association => deterministic. Ends with a barrier.
template <typename Src, typename Dst>
__device__ void ordered_sum(int E, int cnt, size_t stride, Src src, Dst dst, float4* red) {
  const int T = blockDim.x;
  int sub = E >= T ? 1 : min(T / E, (cnt + 3) / 4);
  sub = max(sub, 1);
  const int per = (cnt + sub - 1) / sub;
  const int active = E * sub;
  for (int base = 0; base < E * sub; base += T) {
    const int t = base + threadIdx.x;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (t < active) {
      const int e = t % E, j = t / E;
      const int i0 = j * per, i1 = min(cnt, i0 + per);
      const float4* p = src(e);
      int i = i0;
      if (i < i1) v = __ldcg(p + (size_t)i * stride);
      ++i;
      for (; i + 8 <= i1; i += 8) {
        float4 b[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) b[u] = __ldcg(p + (size_t)(i + u) * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) v = f4add(v, b[u]);
      }
      for (; i < i1; ++i) v = f4add(v, __ldcg(p + (size_t)i * stride));
      if (sub == 1) dst(e, v);
    }
    if (sub > 1) {
      red[threadIdx.x] = v;
      __syncthreads();
      // T is a multiple of E*sub here (E*sub <= T), so base == 0
      if (threadIdx.x < E) {
        float4 w = red[threadIdx.x];
        for (int j = 1; j < sub; ++j) w = f4add(w, red[j * E + threadIdx.x]);
        dst(threadIdx.x, w);
      }
    }
  }
  __syncthreads();
}

// Fused, deterministic split-K reduction (the epilogue of both MACs).
// Chunk `chunk` of `nchunks` has just written its partial: R rows x columns
// [c0, c0 + nc) at part + chunk*cs + r*rs + c. Level 1: the last CTA to
// arrive in each group of `gsz` consecutive chunks sums the group in chunk
// order (into part2, or straight into out when there is one group); level
// 2: the last level-1 reducer sums the groups in group order into
// out + r*os + c. Which CTA arrives last never changes the association, so
// the result is bit-reproducible. Tickets t1[group] and *t2 start at 0 and
// are reset by their reducer. red: >= blockDim float4 of shared scratch.
// Returns true in exactly one CTA: the one holding the final result.
__device__ __noinline__ bool split_k_reduce(const float4* part, float4* part2, size_t cs, size_t rs, int R,
                               int c0, int nc, int chunk, int nchunks, int gsz, unsigned* t1,
                               unsigned* t2, float4* out, size_t os, float4* red) {
  __shared__ unsigned s_last;
  const int g = chunk / gsz;
  const int n1 = (nchunks + gsz - 1) / gsz;
  const int gsize = min(gsz, nchunks - g * gsz);
  const int E = R * nc;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&t1[g], 1u) == (unsigned)gsize - 1u;
  __syncthreads();
  if (!s_last) return false;
  if (threadIdx.x == 0) t1[g] = 0u;
  __threadfence();
  const float4* src0 = part + (size_t)g * gsz * cs;
  auto at = [&](int e) { return (size_t)(e / nc) * rs + c0 + (e % nc); };
  auto oat = [&](int e) { return (size_t)(e / nc) * os + c0 + (e % nc); };
  if (n1 == 1) {
    ordered_sum(E, gsize, cs, [&](int e) { return src0 + at(e); },
                [&](int e, float4 v) { __stcg(out + oat(e), v); }, red);
  } else {
    ordered_sum(E, gsize, cs, [&](int e) { return src0 + at(e); },
                [&](int e, float4 v) { __stcg(part2 + (size_t)g * cs + at(e), v); }, red);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(t2, 1u) == (unsigned)n1 - 1u;
    __syncthreads();
    if (!s_last) return false;
    if (threadIdx.x == 0) *t2 = 0u;
    __threadfence();
    ordered_sum(E, n1, cs, [&](int e) { return (const float4*)part2 + at(e); },
                [&](int e, float4 v) { __stcg(out + oat(e), v); }, red);
  }
  __threadfence();
  __syncthreads();
  return true;
}

// ------------------------------------------------------------- k_front
// grid = ceil(L / cpb), 256 threads; elementwise CTAs also own their
// channels' inputs. Shared: Qs input spectra (N float2 each), FFT scratch z
// (N float2), window/accumulator (2N floats).
__global__ void __launch_bounds__(kFrontThreads) k_front(BlockArgs a) {
  extern __shared__ float4 smem4[];
  const int N = a.N, NF = a.NF;
  const bool elem = a.mode == 1;
  const int Qs = elem ? 1 : a.Q;
  float2* Xs = reinterpret_cast<float2*>(smem4);          // Qs x N
  float2* z = Xs + (size_t)Qs * N;                        // N
  float* wa = reinterpret_cast<float*>(z + N);            // 2N (window / acc)
  float2* acc = reinterpret_cast<float2*>(wa);

  const uint32_t n = a.st->block;
  trace_begin(a, TR_FRONT, n);
  const int c0 = blockIdx.x * a.cpb;
  const int c1 = min(c0 + a.cpb, a.L);
  const int Qh = a.mode == 2 ? a.Q : 1;

  // ---- stage 1 for the shared inputs (broadcast / mimo)
  if (!elem) {
    for (int q = 0; q < Qs; ++q) {
      const float* in = a.in + (size_t)q * N;
      const float* prev = a.prev_in + (size_t)q * N;
      for (int i = threadIdx.x; i < N; i += blockDim.x) {
        float v = in[i];
        if (a.is_aur) v = __fsub_rn(__fmul_rn(a.gain, v), a.fhat[(size_t)q * N + i]);
        if (blockIdx.x == 0) a.cur_mt[(size_t)q * N + i] = v;
        wa[i] = prev[i];
        wa[N + i] = v;
      }
      __syncthreads();
      rfft_packed(wa, z, Xs + (size_t)q * N, N, a.logN, a.tw, a.split);
      if (blockIdx.x == 0) {
        float2* dst = reinterpret_cast<float2*>(a.X + ((size_t)q * a.K + n % (uint32_t)a.K) * NF);
        for (int j = threadIdx.x; j < N; j += blockDim.x) dst[j] = Xs[(size_t)q * N + j];
      }
    }
  }

  // ---- per output channel: Y = S + sum_q X_q H_q[0], c2r, overlap-save
  for (int l = c0; l < c1; ++l) {
    if (elem) {
      const float* in = a.in + (size_t)l * N;
      float* prev = a.prev_in + (size_t)l * N;
      for (int i = threadIdx.x; i < N; i += blockDim.x) {
        wa[i] = prev[i];
        wa[N + i] = in[i];
      }
      __syncthreads();
      for (int i = threadIdx.x; i < N; i += blockDim.x) prev[i] = wa[N + i];
      rfft_packed(wa, z, Xs, N, a.logN, a.tw, a.split);
      float2* dst = reinterpret_cast<float2*>(a.X + ((size_t)l * a.K + n % (uint32_t)a.K) * NF);
      for (int j = threadIdx.x; j < N; j += blockDim.x) dst[j] = Xs[j];
    }
    const float2* Sl = reinterpret_cast<const float2*>(a.S + (size_t)l * NF);
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
      float2 y = Sl[j];
      for (int q = 0; q < Qs; ++q) {
        const float2 h = reinterpret_cast<const float2*>(a.H0 + ((size_t)l * Qh + q) * NF)[j];
        y = cmac2(y, Xs[(size_t)q * N + j], h, j == 0);
      }
      acc[j] = y;
    }
    __syncthreads();
    float* out = a.out + (size_t)l * N;
    float* sp = a.spk + (size_t)l * N;
    const bool keep = a.is_aur;
    irfft_packed_tail(acc, z, N, a.logN, a.tw, a.split, [&](int i, float v) {
      out[i] = v;
      if (keep) sp[i] = v;
    });
  }
  trace_end(a, TR_FRONT, n);
}

// ---------------------------------------------------------- k_back_head
// Background of block n, canceller branch head. CTA l < L (auralizer):
// canceller stage 1 on l_n (convolver.hpp:180-191 on fc_); CTAs [Lb, Lb + P): NLMS error spectra E_p = r2c([0_N,
// m~_p]) (Appendix A step 2). CTA 0 also moves this block's m~ into the
// input window history (broadcast / mimo).
__global__ void __launch_bounds__(kFrontThreads) k_back_head(BlockArgs a) {
  extern __shared__ float4 smem4[];
  const int N = a.N, NF = a.NF;
  float2* z = reinterpret_cast<float2*>(smem4);  // N
  float* wa = reinterpret_cast<float*>(z + N);   // 2N
  const uint32_t n = a.st->block;
  trace_begin(a, TR_BACK_HEAD, n);
  const int Lb = a.is_aur ? a.L : 1;
  const int b = blockIdx.x;
  if (b == 0 && a.mode != 1)
    for (int i = threadIdx.x; i < a.Q * N; i += blockDim.x) a.prev_in[i] = a.cur_mt[i];
  if (!a.is_aur) {
    trace_end(a, TR_BACK_HEAD, n);
    return;
  }
  if (b < Lb) {
    const int l = b;
    float* prev = a.prev_spk + (size_t)l * N;
    const float* sp = a.spk + (size_t)l * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      wa[i] = prev[i];
      wa[N + i] = sp[i];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < N; i += blockDim.x) prev[i] = wa[N + i];
    float2* xnew = reinterpret_cast<float2*>(
        a.XA + ((size_t)l * (a.KF + 1) + n % (uint32_t)(a.KF + 1)) * NF);
    rfft_packed(wa, z, xnew, N, a.logN, a.tw, a.split);
  } else {
    const int p = b - Lb;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      wa[i] = 0.0f;
      wa[N + i] = a.cur_mt[(size_t)p * N + i];
    }
    __syncthreads();
    rfft_packed(wa, z, reinterpret_cast<float2*>(a.E + (size_t)p * NF), N, a.logN, a.tw,
                a.split);
  }
  trace_end(a, TR_BACK_HEAD, n);
}

// ------------------------------------------------------------ k_advance
__global__ void k_advance(DevState* st) { st->block += 1u; }  // blocks without tails

// ------------------------------------------------------------ k_mac_pre
// Split-K partials of S_l(n+1) = sum_q sum_{j=0}^{K-2} X_q(age j) H_{l,q}[j+1]
// (backend.hpp:212-235 over every partition but the first).
// grid = (syn_chunks, L/LT, syn_tiles), 256 threads; thread (kp, f): column
// f of the tile, tap phase kp. LT channels share every X load (broadcast /
// mimo): X comes from L2, H streams from HBM with 128-bit no-L1 loads.
// ELEM: channel l reads FDL channel l.
template <int LT, bool ELEM>
__global__ void __launch_bounds__(kMacThreads, 2) k_mac_pre(BlockArgs a) {
  __shared__ float4 red[kMacThreads * LT];
  const int nft = a.syn_nft;
  const int KP = kMacThreads / nft;
  const int fl = threadIdx.x & (nft - 1);
  const int kp = threadIdx.x / nft;
  const int f = blockIdx.z * nft + fl;
  const int l0 = blockIdx.y * LT;
  const int K = a.K;
  const int Kt = K - 1;                      // taps per input
  const int Qh = ELEM ? 1 : a.Q;
  const int T = Qh * Kt;
  const int t0 = blockIdx.x * a.syn_tc;
  const int t1 = min(t0 + a.syn_tc, T);
  const uint32_t n = a.st->block;
  trace_begin(a, TR_MAC_PRE, n);
  const int nk = (int)(n % (uint32_t)K);
  const bool dc = (f == 0);
  const int NF = a.NF;

  float4 acc[LT];
#pragma unroll
  for (int i = 0; i < LT; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);

  int t = t0 + kp;
  int q = t / Kt;
  int j = t - q * Kt;
#pragma unroll 2
  for (; t < t1; t += KP) {
    int slot = nk - j;
    if (slot < 0) slot += K;
    const size_t hrow = (size_t)q * K + j + 1;  // partition j+1 of input q
    if (ELEM) {
#pragma unroll
      for (int i = 0; i < LT; ++i) {
        const float4 xv = a.X[((size_t)(l0 + i) * K + slot) * NF + f];
        const float4 h = ld_stream(a.H + ((size_t)(l0 + i) * K + j + 1) * NF + f);
        cmac(acc[i], xpack(xv, dc), h, dc);
      }
    } else {
      const XPack x = xpack(a.X[((size_t)q * K + slot) * NF + f], dc);
      float4 h[LT];
#pragma unroll
      for (int i = 0; i < LT; ++i)
        h[i] = ld_stream(a.H + ((size_t)(l0 + i) * Qh * K + hrow) * NF + f);
#pragma unroll
      for (int i = 0; i < LT; ++i) cmac(acc[i], x, h[i], dc);
    }
    j += KP;
    while (j >= Kt) {
      j -= Kt;
      ++q;
    }
  }
#pragma unroll
  for (int i = 0; i < LT; ++i) red[(kp * LT + i) * nft + fl] = acc[i];
  __syncthreads();
  for (int e = threadIdx.x; e < LT * nft; e += kMacThreads) {
    const int i = e / nft, c = e - i * nft;
    float4 s = red[i * nft + c];
    for (int p = 1; p < KP; ++p) s = f4add(s, red[(p * LT + i) * nft + c]);
    __stcg(a.part_syn + ((size_t)blockIdx.x * a.L + l0 + i) * NF + blockIdx.z * nft + c, s);
  }
  // fused split-K reduction -> S for this CTA's LT channels x nft columns
  __syncthreads();  // red is reused as reduction scratch
  const int n1 = (a.syn_chunks + a.syn_g1 - 1) / a.syn_g1;
  unsigned* tk = a.tick_syn + ((size_t)blockIdx.y * gridDim.z + blockIdx.z) * (n1 + 1);
  const bool fin = split_k_reduce(a.part_syn + (size_t)l0 * NF, a.part_syn2 + (size_t)l0 * NF,
                                  (size_t)a.L * NF, NF, LT, blockIdx.z * nft, nft, blockIdx.x,
                                  a.syn_chunks, a.syn_g1, tk, tk + n1, a.S + (size_t)l0 * NF, NF,
                                  red);
  trace_end(a, TR_MAC_PRE, n);
  if (fin) retire_block(a, n);
}

// ----------------------------------------------------------- k_mac_afc
// Canceller MAC over units u = (l, k), all P mics per unit (X_l shared):
//   NLMS (Appendix A step 2): W += mu/(P+delta) * conj(X_l(pre-push age k)) E_p
//   filter (step 4):          Yhat_p += W * X_l(post-push age k)
//   power (step 5):           row P += |X_l(age 0)|^2 on the units k = 0
// Pre-push age k is post-push age k+1: the canceller FDL keeps KF+1 slots.
// grid = (afc_chunks, 1, afc_tiles), 256 threads. Epilogue: fused split-K
// reduction per column tile into yhat; the last tile-finisher then does one
// c2r per mic (the sum over l and k is done in the frequency domain -- one
// c2r per mic instead of the reference's L, auralizer.hpp:81-86) -> f^ for
// the next block, and smooths the power (or, sharded, leaves both partials
// in xmine for k_afc_finish). Dynamic shared memory: N float2 (c2r scratch).
template <int PT>
__global__ void __launch_bounds__(kMacThreads, (PT <= 2 ? 4 : 2)) k_mac_afc(BlockArgs a) {
  __shared__ float4 red[kMacThreads * (PT + 1)];
  extern __shared__ float4 afc_dyn[];
  __shared__ unsigned s_last_tile;
  const int nft = a.afc_nft;
  const int KP = kMacThreads / nft;
  const int fl = threadIdx.x & (nft - 1);
  const int kp = threadIdx.x / nft;
  const int f = blockIdx.z * nft + fl;
  const int N = a.N, NF = a.NF, KF = a.KF, L = a.L, P = a.P;
  const int cap = KF + 1;
  const int U = L * KF;
  const int u0 = blockIdx.x * a.afc_uc;
  const int u1 = min(u0 + a.afc_uc, U);
  const uint32_t n = a.st->block;
  trace_begin(a, TR_MAC_AFC, n);
  const int nk = (int)(n % (uint32_t)cap);
  const bool dc = (f == 0);
  const int R = P + (a.nlms ? 1 : 0);  // partial rows (row P: power)

  float4 acc[PT];
  float4 e[PT];
  float4 pacc = make_float4(0.f, 0.f, 0.f, 0.f);
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int p = 0; p < PT; ++p) {
    acc[p] = make_float4(0.f, 0.f, 0.f, 0.f);
    e[p] = (a.nlms && p < P) ? a.E[(size_t)p * NF + f] : acc[p];
  }
  if (a.nlms) {
    const float2 p0 = a.pw[2 * f], p1 = a.pw[2 * f + 1];
    s = make_float4(__fdiv_rn(a.mu, __fadd_rn(p0.x, a.delta)),
                    __fdiv_rn(a.mu, __fadd_rn(p0.y, a.delta)),
                    __fdiv_rn(a.mu, __fadd_rn(p1.x, a.delta)),
                    __fdiv_rn(a.mu, __fadd_rn(p1.y, a.delta)));
  }

  int u = u0 + kp;
  int l = u / KF;
  int k = u - l * KF;
  for (; u < u1; u += KP) {
    const float4* xl = a.XA + (size_t)l * cap * NF;
    const float4 xv = xl[(size_t)ring(nk - k, cap) * NF + f];
    const XPack x0 = xpack(xv, dc);
    float4 x1 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (a.nlms) {
      x1 = xl[(size_t)ring(nk - k - 1, cap) * NF + f];
      if (k == 0) {  // packed |X_l(age 0)|^2 (bin 0: DC^2, Nyquist^2), rounded as the oracle
        if (dc) {
          pacc.x = __fadd_rn(pacc.x, __fmul_rn(xv.x, xv.x));
          pacc.y = __fadd_rn(pacc.y, __fmul_rn(xv.y, xv.y));
        } else {
          const float m = __fadd_rn(__fmul_rn(xv.x, xv.x), __fmul_rn(xv.y, xv.y));
          pacc.x = __fadd_rn(pacc.x, m);
          pacc.y = __fadd_rn(pacc.y, m);
        }
        const float m2 = __fadd_rn(__fmul_rn(xv.z, xv.z), __fmul_rn(xv.w, xv.w));
        pacc.z = __fadd_rn(pacc.z, m2);
        pacc.w = __fadd_rn(pacc.w, m2);
      }
    }
#pragma unroll
    for (int p = 0; p < PT; ++p) {
      if (p >= P) break;
      float4* wp = a.W + (((size_t)p * L + l) * KF + k) * NF + f;
      float4 w = *wp;
      if (a.nlms) {
        // g = conj(x1) * E_p ; packed bin 0 is (DC, Nyquist) real products.
        // Rounded exactly as the oracle (aura_oracle.c nlms_update): no FMA.
        float4 g;
        if (dc) {
          g.x = __fmul_rn(x1.x, e[p].x);
          g.y = __fmul_rn(x1.y, e[p].y);
        } else {
          g.x = __fadd_rn(__fmul_rn(x1.x, e[p].x), __fmul_rn(x1.y, e[p].y));
          g.y = __fsub_rn(__fmul_rn(x1.x, e[p].y), __fmul_rn(x1.y, e[p].x));
        }
        g.z = __fadd_rn(__fmul_rn(x1.z, e[p].z), __fmul_rn(x1.w, e[p].w));
        g.w = __fsub_rn(__fmul_rn(x1.z, e[p].w), __fmul_rn(x1.w, e[p].z));
        w.x = __fadd_rn(w.x, __fmul_rn(s.x, g.x));
        w.y = __fadd_rn(w.y, __fmul_rn(s.y, g.y));
        w.z = __fadd_rn(w.z, __fmul_rn(s.z, g.z));
        w.w = __fadd_rn(w.w, __fmul_rn(s.w, g.w));
        *wp = w;
      }
      cmac(acc[p], x0, w, dc);
    }
    k += KP;
    while (k >= KF) {
      k -= KF;
      ++l;
    }
  }
#pragma unroll
  for (int p = 0; p < PT; ++p) red[(kp * (PT + 1) + p) * nft + fl] = acc[p];
  red[(kp * (PT + 1) + PT) * nft + fl] = pacc;
  __syncthreads();
  const size_t rows = (size_t)P + 1;
  for (int e2 = threadIdx.x; e2 < R * nft; e2 += kMacThreads) {
    const int r = e2 / nft, c = e2 - r * nft;
    const int rr = r < P ? r : PT;  // power row
    float4 t = red[rr * nft + c];
    for (int q = 1; q < KP; ++q) t = f4add(t, red[(q * (PT + 1) + rr) * nft + c]);
    __stcg(a.part_afc + ((size_t)blockIdx.x * rows + r) * NF + blockIdx.z * nft + c, t);
  }
  const int n1 = (a.afc_chunks + a.afc_g1 - 1) / a.afc_g1;
  unsigned* tk = a.tick_afc + (size_t)blockIdx.z * (n1 + 1);
  __syncthreads();  // red is reused as reduction scratch
  const bool fin = split_k_reduce(a.part_afc, a.part_afc2, rows * NF, NF, R, blockIdx.z * nft, nft,
                                  blockIdx.x, a.afc_chunks, a.afc_g1, tk, tk + n1, a.yhat, NF,
                                  red);
  if (!fin) {
    trace_end(a, TR_MAC_AFC, n);
    return;
  }
  // last of the column tiles finishes the block's canceller
  if (gridDim.z > 1) {
    if (threadIdx.x == 0) {
      unsigned* tt = a.tick_afc + (size_t)gridDim.z * (n1 + 1);
      s_last_tile = atomicAdd(tt, 1u) == gridDim.z - 1u;
      if (s_last_tile) *tt = 0u;
    }
    __syncthreads();
    if (!s_last_tile) {
      trace_end(a, TR_MAC_AFC, n);
      return;
    }
    __threadfence();
  }
  const bool sharded = a.G > 1;
  float2* z = reinterpret_cast<float2*>(afc_dyn);
  for (int p = 0; p < P; ++p) {
    // sharded: this shard's partial f^_p (c2r is linear), summed by k_afc_finish
    float* fh = sharded ? a.xmine + (size_t)p * N : a.fhat + (size_t)p * N;
    float* fhh = a.fhat_host + (size_t)p * N;
    irfft_packed_tail(reinterpret_cast<const float2*>(a.yhat + (size_t)p * NF), z, N, a.logN, a.tw,
                      a.split, [&](int i, float v) {
                        fh[i] = v;
                        if (!sharded) fhh[i] = v;
                      });
  }
  if (a.nlms) {
    const float2* sum = reinterpret_cast<const float2*>(a.yhat + (size_t)P * NF);
    const float oml = __fsub_rn(1.0f, a.lambda);
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
      const float2 v = __ldcg(sum + j);
      if (sharded) {  // partial power of this shard's loudspeakers
        reinterpret_cast<float2*>(a.xmine + (size_t)P * N)[j] = v;
        continue;
      }
      // Appendix A step 5: lambda P + (1 - lambda) sum_l |X_l|^2
      float2 w = a.pw[j];
      w.x = __fadd_rn(__fmul_rn(a.lambda, w.x), __fmul_rn(oml, v.x));
      w.y = __fadd_rn(__fmul_rn(a.lambda, w.y), __fmul_rn(oml, v.y));
      a.pw[j] = w;
    }
  }
  trace_end(a, TR_MAC_AFC, n);
  if (!sharded) retire_block(a, n);
}

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ------------------------------------------------------- k_afc_finish
// Sharded canceller (G > 1), one CTA per shard and block: push this shard's
// partial (P*N f^ samples + 2N packed power values) into slot [n&1][grank]
// of every shard's exchange buffer over NVLink (P2P stores; same-device
// stores for virtual shards), publish flag[grank] = n+1 with a system-scope
// release, wait for every shard's flag, then sum the G slots in rank order.
// Every shard sums the same values in the same order, so all shards hold a
// bit-identical f^ and power. Two parities suffice: a shard can only write
// block n+1's partial after finishing block n, which needed every shard's
// block-n partial, and each shard consumes its block-n slots before it
// produces block n+1 (stream order). The wait is bounded (kShardTimeoutNs):
// a missing peer sets status_host instead of hanging the GPU.
__global__ void __launch_bounds__(kTailThreads) k_afc_finish(BlockArgs a) {
  const uint32_t n = a.st->block;
  trace_begin(a, TR_AFC_FINISH, n);
  const int N = a.N, P = a.P, G = a.G;
  const size_t S = (size_t)P * N + 2 * (size_t)N;
  const int par = (int)(n & 1u);
  for (int g = 0; g < G; ++g) {
    float* dst = reinterpret_cast<float*>(a.xpeer[g] + kXFlagBytes) + ((size_t)par * G + a.grank) * S;
    for (size_t i = threadIdx.x; i < S; i += blockDim.x) dst[i] = __ldcg(a.xmine + i);
  }
  __syncthreads();
  __shared__ int timed_out;
  if (threadIdx.x == 0) {
    timed_out = 0;
    __threadfence_system();
    for (int g = 0; g < G; ++g) st_release_sys(reinterpret_cast<unsigned*>(a.xpeer[g]) + a.grank, n + 1);
    const unsigned* flags = reinterpret_cast<const unsigned*>(a.xpeer[a.grank]);
    const unsigned long long t0 = globaltimer();
    for (int g = 0; g < G && !timed_out; ++g)
      while (ld_acquire_sys(flags + g) < n + 1) {
        if (globaltimer() - t0 > kShardTimeoutNs) {
          timed_out = 1;
          *reinterpret_cast<volatile unsigned*>(a.status_host) = 1u;
          break;
        }
        __nanosleep(64);
      }
  }
  __syncthreads();
  const float* slots = reinterpret_cast<const float*>(a.xpeer[a.grank] + kXFlagBytes) + (size_t)par * G * S;
  for (int i = threadIdx.x; i < P * N; i += blockDim.x) {
    float v = __ldcg(slots + i);
    for (int g = 1; g < G; ++g) v = __fadd_rn(v, __ldcg(slots + (size_t)g * S + i));
    a.fhat[i] = v;
    a.fhat_host[i] = v;
  }
  if (a.nlms) {
    const float oml = __fsub_rn(1.0f, a.lambda);
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
      const float* b = slots + (size_t)P * N + 2 * j;
      float2 sum = make_float2(__ldcg(b), __ldcg(b + 1));
      for (int g = 1; g < G; ++g) {
        sum.x = __fadd_rn(sum.x, __ldcg(b + (size_t)g * S));
        sum.y = __fadd_rn(sum.y, __ldcg(b + (size_t)g * S + 1));
      }
      float2 w = a.pw[j];
      w.x = __fadd_rn(__fmul_rn(a.lambda, w.x), __fmul_rn(oml, sum.x));
      w.y = __fadd_rn(__fmul_rn(a.lambda, w.y), __fmul_rn(oml, sum.y));
      a.pw[j] = w;
    }
  }
  trace_end(a, TR_AFC_FINISH, n);
  retire_block(a, n);
}

// ------------------------------------------------------ k_partition
// Setup (make_partitioned_filters, convolver.hpp:19-46) on the GPU: CTA
// (k, r) transforms taps[r][kN .. kN+N) zero-padded to 2N into the packed
// spectrum dst + row_off[r] + k*NF. taps rows are n_h long.
__global__ void __launch_bounds__(256) k_partition(
    const float* __restrict__ taps, size_t n_h, int rows, int K, int N, int logN,
    const float2* tw, const float2* split, float4* dst, const size_t* __restrict__ row_off) {
  extern __shared__ float smem[];
  float* win = smem;
  float2* z = reinterpret_cast<float2*>(win + 2 * N);
  const int k = blockIdx.x;
  const int r = blockIdx.y;
  const size_t begin = (size_t)k * N;
  const float* src = taps + (size_t)r * n_h;
  for (int i = threadIdx.x; i < 2 * N; i += blockDim.x) {
    const size_t t = begin + i;
    win[i] = (i < N && t < n_h) ? src[t] : 0.0f;
  }
  __syncthreads();
  float2* out = reinterpret_cast<float2*>(dst + row_off[r] + (size_t)k * (N / 2));
  rfft_packed(win, z, out, N, logN, tw, split);
}

}  // namespace aura_b200
