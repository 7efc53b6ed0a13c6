// kernels.cuh -- the small per-block kernels of the UPOLS + feedback-
// canceller block loop (sm_100a); the streaming MACs are in stream.cuh.
//
// Block n is ONE CUDA graph on the engine stream:
//
//   k_front       m~ = g m - f^ (auralizer.hpp:73-76), window + r2c of every
//                 input (convolver.hpp:180-191), FDL push, then per output
//                 channel  Y_l = S_l + sum_q X_q,n (.) H_{l,q}[0],  c2r +
//                 overlap-save straight into the (mapped) output buffer; each
//                 CTA publishes an output word the host polls (process()
//                 returns here); then canceller stage 1 on l_n (r2c, FDL
//                 push) and, on P extra CTAs, the NLMS error spectra. It
//                 triggers its dependent launch at once, so
//   [k_afc_constrain  the constrained NLMS gradient, optional]
//   k_back        (stream.cuh, programmatic dependent launch) starts its
//                 synthesis stream during the front: S_l for block n+1
//                 (every partition but the first -- they depend only on
//                 inputs <= n) and the canceller MAC + NLMS;
//   k_reduce      (stream.cuh) the fixed-order split-K sums -> S, f^ for n+1;
//   k_afc_finish  only when the loudspeakers are sharded over GPUs.
// (k_back_head, the separate canceller stage 1, remains for
// AURA_B200_FRONT_HEAD=0.)
//
// So the output of block n is c2r(X_n H_0 + sum_{k>=1} X_{n-k} H_k), exactly
// the reference's accumulator (backend.hpp:212-235) with the partition sum
// split in two; the work per block is unchanged, only its position in time.
// All reductions run in a fixed order, so results are bit-reproducible run to
// run (test_convolver.cpp:172-193).
//
// Device layouts (N = block size, NF = N/2 float4 per packed spectrum, CT =
// min(NF, 32) float4 columns per column tile, CTn = NF / CT):
//   input FDL X       [Qx][CTn][K][CT]         ring slot = block mod K
//   canceller FDL XA  [L][CTn][KF+1][CT]       ring slot = block mod (KF+1)
//   spectra H (k>=1)  [L/LT][CTn][Qh*(K-1)][LT][CT]   tap t = q (K-1) + k - 1
//   partition 0  H0   [L][Qh][NF]
//   canceller W       [CTn][L*KF][P][CT]       unit u = l KF + k
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cooperative_groups.h>

#include <type_traits>

#include "args.cuh"

namespace aura_b200 {

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
__device__ __forceinline__ void trace_begin(const BlockArgs& a, int id, blk_t n) {
  if (a.trace && threadIdx.x == 0)
    atomicMin(&a.trace[((n % kTraceBlocks) * kTraceKernels + id) * 2], globaltimer());
}
__device__ __forceinline__ void trace_end(const BlockArgs& a, int id, blk_t n) {
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
__device__ void retire_block(const BlockArgs& a, blk_t n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(&a.st->ticket, 1u) == (uint32_t)a.advance_total - 1) {
      a.st->ticket = 0;
      a.st->block = n + 1;
    }
  }
}

// Store the packed spectrum spec (N float2, shared) as ring slot `slot` of
// delay-line channel ch, tiled [ch][CTn][cap][CT] float4 (see above).
template <typename Team = Cta>
__device__ __forceinline__ void push_tiled(const BlockArgs& a, float4* fdl, int ch, int cap, int slot,
                                           const float2* spec, Team tm = Team()) {
  const int CT = a.CT;
  float2* d = reinterpret_cast<float2*>(fdl);
  for (int j = tm.tid(); j < a.N; j += tm.size()) {
    const int f = j >> 1;
    const size_t i4 = (((size_t)ch * a.CTn + f / CT) * cap + slot) * CT + (f % CT);
    d[2 * i4 + (j & 1)] = spec[j];
  }
}

// ------------------------------------------------------------- k_front

// The front of block n for output channels [c0, c1) with a team of threads:
// m~ = g m - f^ (auralizer.hpp:73-76), window + r2c of every input
// (convolver.hpp:180-191; the leader also pushes it into the FDL and writes
// this block's m~ to cur_out), then per channel Y_l = S_l + sum_q X_q H0_l,q,
// c2r + overlap-save into the output (and, for the canceller, into spk).
// on_x() runs on the whole team once the leader has pushed the input
// spectra. smem: front_work_f2 float2, then the tables (a.smem_tables) and
// the staged S/H0 (a.front_pre).
// Issue every load of a window before its stores: a store in between may
// alias the later loads as far as the compiler knows, which serialises the
// load rounds -- one dependent memory round trip per round (profiles/
// r1s5_stream.md: +2.5 us on a warp front). U rounds per batch.
template <int U, typename Ld, typename St>
__device__ __forceinline__ void batched(int tid, int nt, int n, Ld ld, St st) {
  for (int i0 = tid; i0 < n; i0 += U * nt) {
    decltype(ld(0)) v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * nt;
      if (i < n) v[u] = ld(i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * nt;
      if (i < n) st(i, v[u]);
    }
  }
}

struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

template <typename Team, typename OnX = NoHook>
__device__ void front_body(const BlockArgs& a, blk_t n, int c0, int c1, float2* Xs, const float* in,
                           const float* prev_in, float* cur_out, bool leader, Team tm, OnX on_x = OnX()) {
  const int N = a.N, NF = a.NF;
  const int tid = tm.tid(), nt = tm.size();
  const bool elem = a.mode == 1;
  const int Qs = elem ? 1 : a.Q;
  const int Qh = a.mode == 2 ? a.Q : 1;
  float2* z = Xs + (size_t)Qs * N;                        // N
  float* wa = reinterpret_cast<float*>(z + N);            // 2N (window / acc)
  float2* acc = reinterpret_cast<float2*>(wa);
  float2* stw = reinterpret_cast<float2*>(wa + 2 * N);    // DftPlan tables (if staged)
  float2* pre = stw + (a.smem_tables ? table_f2(N) : 0);  // [S_l, H0_l,q] of the first channel
  const float2* tw = a.smem_tables ? stw : a.tw;
  const float2* split = a.smem_tables ? stw + N / 2 : a.split;

  // ---- one round of independent loads: tables, input windows, and the
  // first channel's precomputed S_l and partition-0 spectra (front_pre)
  if (a.smem_tables) stage_tables(stw, stw + N / 2, a.tw, a.split, N, tm);
  if (a.front_pre) {
    const float2* Sl = reinterpret_cast<const float2*>(a.S + (size_t)c0 * NF);
    const float2* H0 = reinterpret_cast<const float2*>(a.H0 + (size_t)c0 * Qh * NF);
    for (int j = tid; j < N; j += nt) pre[j] = Sl[j];
    for (int j = tid; j < Qs * N; j += nt) pre[N + j] = H0[j];
  }

  // ---- stage 1 for the shared inputs (broadcast / mimo)
  if (!elem) {
    for (int q = 0; q < Qs; ++q) {
      const float* inq = in + (size_t)q * N;
      const float* prev = prev_in + (size_t)q * N;
      const float* fq = a.fhat + (size_t)q * N;
      batched<4>(tid, nt, N,
                 [&](int i) { return make_float3(inq[i], a.is_aur ? fq[i] : 0.f, prev[i]); },
                 [&](int i, float3 x) {
                   const float v = a.is_aur ? __fsub_rn(__fmul_rn(a.gain, x.x), x.y) : x.x;
                   if (leader) cur_out[(size_t)q * N + i] = v;
                   wa[i] = x.z;
                   wa[N + i] = v;
                 });
      tm.sync();
      rfft_packed(wa, z, Xs + (size_t)q * N, N, a.logN, tw, split, tm);
      if (leader) push_tiled(a, a.X, q, a.K, (int)(n % (blk_t)a.K), Xs + (size_t)q * N, tm);
    }
    on_x();
  }

  // ---- per output channel: Y = S + sum_q X_q H_q[0], c2r, overlap-save
  for (int l = c0; l < c1; ++l) {
    if (elem) {
      const float* inl = in + (size_t)l * N;
      float* prev = a.prev_in + (size_t)l * N;
      batched<4>(tid, nt, N, [&](int i) { return make_float2(prev[i], inl[i]); },
                 [&](int i, float2 x) {
                   wa[i] = x.x;
                   wa[N + i] = x.y;
                 });
      tm.sync();
      for (int i = tid; i < N; i += nt) prev[i] = wa[N + i];
      rfft_packed(wa, z, Xs, N, a.logN, tw, split, tm);
      push_tiled(a, a.X, l, a.K, (int)(n % (blk_t)a.K), Xs, tm);
      if (l + 1 == c1) on_x();
    }
    const bool staged = a.front_pre && l == c0;
    const float2* Sl = staged ? pre : reinterpret_cast<const float2*>(a.S + (size_t)l * NF);
    const float2* H0 = staged ? pre + N : reinterpret_cast<const float2*>(a.H0 + (size_t)l * Qh * NF);
    for (int j = tid; j < N; j += nt) {
      float2 y = Sl[j];
      for (int q = 0; q < Qs; ++q) y = cmac2(y, Xs[(size_t)q * N + j], H0[(size_t)q * N + j], j == 0);
      acc[j] = y;
    }
    tm.sync();
    float* out = a.out + (size_t)l * N;
    float* sp = a.spk + (size_t)l * N;
    const bool keep = a.is_aur;
    irfft_packed_tail(acc, z, N, a.logN, tw, split, [&](int i, float v) {
      out[i] = v;
      if (keep) sp[i] = v;
    }, tm);
  }
}

// Canceller stage 1 (convolver.hpp:180-191 on fc_) for loudspeakers
// [c0, c1): r2c of [l_{n-1}, l_n] into the canceller FDL. Team-generic
// (k_front's fused head and k_back_head). smem: 3N float2 + tables.
template <typename Team>
__device__ void head_channels(const BlockArgs& a, blk_t n, int c0, int c1, float2* z, const float2* tw,
                              const float2* split, Team tm) {
  const int N = a.N;
  float* wa = reinterpret_cast<float*>(z + N);         // 2N
  float2* sp = reinterpret_cast<float2*>(wa + 2 * N);  // N (spectrum)
  for (int l = c0; l < c1; ++l) {
    float* prev = a.prev_spk + (size_t)l * N;
    const float* spk = a.spk + (size_t)l * N;
    batched<4>(tm.tid(), tm.size(), N, [&](int i) { return make_float2(prev[i], spk[i]); },
               [&](int i, float2 x) {
                 wa[i] = x.x;
                 wa[N + i] = x.y;
               });
    tm.sync();
    for (int i = tm.tid(); i < N; i += tm.size()) prev[i] = wa[N + i];
    if constexpr (std::is_same<Team, Warp>::value) rfft_warp_any(wa, z, sp, N, a.logN, tw, split);
    else rfft_packed(wa, z, sp, N, a.logN, tw, split, tm);
    push_tiled(a, a.XA, l, a.KF + 1, (int)(n % (blk_t)(a.KF + 1)), sp, tm);
    tm.sync();
  }
}

// NLMS error spectrum E_p = r2c([0_N, m~_p]) (Appendix A step 2) from the
// raw input: m~_p = g m_p - f^_p. Team-generic. smem: 3N float2.
template <typename Team>
__device__ void error_spectrum(const BlockArgs& a, int p, const float* in, float2* z, const float2* tw,
                               const float2* split, Team tm) {
  const int N = a.N;
  float* wa = reinterpret_cast<float*>(z + N);
  batched<4>(tm.tid(), tm.size(), N,
             [&](int i) { return make_float2(in[(size_t)p * N + i], a.fhat[(size_t)p * N + i]); },
             [&](int i, float2 x) {
               wa[i] = 0.0f;
               wa[N + i] = __fsub_rn(__fmul_rn(a.gain, x.x), x.y);
             });
  tm.sync();
  rfft_packed(wa, z, reinterpret_cast<float2*>(a.E + (size_t)p * a.NF), N, a.logN, tw, split, tm);
}


// The front with one output channel per warp (channels c0 + w, c0 + w + W,
// ... for warp w): the shared input stage runs on the whole CTA, then each
// warp does its channels' MAC and c2r with __syncwarp only -- a 64-point
// transform has too little work for 256 threads and a CTA barrier per stage.
// Same floating-point operations as front_body (bit-identical). Tables are
// always staged. After every warp's outputs: publish (as k_front), then the
// fused canceller head per channel on the same warps.
template <typename OnX = NoHook>
__device__ void front_warps_body(const BlockArgs& a, blk_t n, int c0, int c1, float2* sm,
                                 const float* in, const float* prev_in, float* cur_out, bool leader,
                                 OnX on_x = OnX()) {
  const int N = a.N, NF = a.NF;
  const int Qs = a.mode == 1 ? 1 : a.Q;
  const int Qh = a.mode == 2 ? a.Q : 1;
  const int W = a.front_warps, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Cta cta;
  const Warp wt;
  float2* Xs = sm;                                     // Qs x N
  float2* z = Xs + (size_t)Qs * N;                     // N
  float* wa = reinterpret_cast<float*>(z + N);         // 2N
  float2* tw = reinterpret_cast<float2*>(wa + 2 * N);  // tables
  float2* split = tw + N / 2;
  float2* mine = tw + table_f2(N) + (size_t)w * N * (3 + Qs);  // this warp's area
  float2* pS = mine;                                   // S_l, then H0_l,q (first channel)
  float2* acc = mine + (size_t)N * (1 + Qs);           // N
  float2* wz = acc + N;                                // N
  stage_tables(tw, split, a.tw, a.split, N, cta);
  const int l0 = c0 + w;
  if (w < W && l0 < c1) {  // this warp's first channel: S and H0 in one round of loads
    const float2* Sl = reinterpret_cast<const float2*>(a.S + (size_t)l0 * NF);
    const float2* H0 = reinterpret_cast<const float2*>(a.H0 + (size_t)l0 * Qh * NF);
    for (int j = lane; j < N; j += 32) pS[j] = Sl[j];
    for (int j = lane; j < Qs * N; j += 32) pS[N + j] = H0[j];
  }
  // ---- stage 1 for the shared inputs (broadcast / mimo): input q's window,
  // r2c and FDL push on warp q in its own area, warp-synchronous (the same
  // operations as the CTA transform, so the same bits), one CTA barrier
  // after instead of one per butterfly stage
  (void)z;
  (void)wa;
  __syncthreads();  // the staged tables
  if (w < W) {
    for (int q = w; q < Qs; q += W) {
      const float* inq = in + (size_t)q * N;
      const float* prev = prev_in + (size_t)q * N;
      float* wq = reinterpret_cast<float*>(acc);  // 2N floats
      const float* fq = a.fhat + (size_t)q * N;
      batched<4>(lane, 32, N,
                 [&](int i) { return make_float3(inq[i], a.is_aur ? fq[i] : 0.f, prev[i]); },
                 [&](int i, float3 x) {
                   const float v = a.is_aur ? __fsub_rn(__fmul_rn(a.gain, x.x), x.y) : x.x;
                   if (leader) cur_out[(size_t)q * N + i] = v;
                   wq[i] = x.z;
                   wq[N + i] = v;
                 });
      __syncwarp();
      rfft_warp_any(wq, wz, Xs + (size_t)q * N, N, a.logN, tw, split);
      if (leader) push_tiled(a, a.X, q, a.K, (int)(n % (blk_t)a.K), Xs + (size_t)q * N, wt);
    }
  }
  __syncthreads();  // every input spectrum
  on_x();
  // ---- per output channel (one warp each): Y = S + sum_q X_q H_q[0], c2r
  if (w < W) {
    for (int l = l0; l < c1; l += W) {
      const bool staged = l == l0;
      const float2* Sl = staged ? pS : reinterpret_cast<const float2*>(a.S + (size_t)l * NF);
      const float2* H0 = staged ? pS + N : reinterpret_cast<const float2*>(a.H0 + (size_t)l * Qh * NF);
      for (int j = lane; j < N; j += 32) {
        float2 y = Sl[j];
        for (int q = 0; q < Qs; ++q) y = cmac2(y, Xs[(size_t)q * N + j], H0[(size_t)q * N + j], j == 0);
        acc[j] = y;
      }
      __syncwarp();
      float* out = a.out + (size_t)l * N;
      float* sp = a.spk + (size_t)l * N;
      const bool keep = a.is_aur;
      irfft_warp_any(acc, wz, N, a.logN, tw, split, [&](int i, float v) {
        out[i] = v;
        if (keep) sp[i] = v;
      });
    }
  }
}

__global__ void __launch_bounds__(kFrontThreads) k_front(BlockArgs a) {
  extern __shared__ float4 smem4[];
  if (a.front_head) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const blk_t n = a.st->block;
  trace_begin(a, TR_FRONT, n);
  const int nerr = (a.front_head && a.is_aur && a.nlms) ? a.P : 0;
  const int nfront = (int)gridDim.x - nerr;
  float2* work = reinterpret_cast<float2*>(smem4);
  if ((int)blockIdx.x >= nfront) {  // NLMS error spectrum E_p (fused-head mode)
    error_spectrum(a, (int)blockIdx.x - nfront, a.in, work, a.tw, a.split, Cta());
    if (a.out_flag) {  // done with the mapped input: the host may refill it
      __syncthreads();
      if (threadIdx.x == 0)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a.out_flag + blockIdx.x), "l"(n + 1)
                     : "memory");
    }
    trace_end(a, TR_FRONT, n);
    return;
  }
  const int c0 = blockIdx.x * a.cpb;
  const int c1 = min(c0 + a.cpb, a.L);
  const float* prev = a.prev_in;
  float* cur = a.cur_mt;
  if (a.front_head) {
    prev = (n & 1u) ? a.hist1 : a.prev_in;
    cur = (n & 1u) ? a.prev_in : a.hist1;
  }
  // front_hold 2: k_back's producers wait until every front CTA has its
  // inputs in (its loads are the part a saturated memory system slows down)
  auto inputs_in = [&] {
    if (a.trace) {
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned long long now = globaltimer();
        atomicMin(&a.trace[((n % kTraceBlocks) * kTraceKernels + TR_FRONT_X) * 2], now);
        atomicMax(&a.trace[((n % kTraceBlocks) * kTraceKernels + TR_FRONT_X) * 2 + 1], now);
      }
    }
    if (a.front_head && a.front_hold == 2) {
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(a.front_seq + (n & 1u), 1ull);
      }
    }
  };
  if (a.front_warps)
    front_warps_body(a, n, c0, c1, work, a.in, prev, cur, blockIdx.x == 0, inputs_in);
  else
    front_body(a, n, c0, c1, work, a.in, prev, cur, blockIdx.x == 0, Cta(), inputs_in);
  if (a.out_flag || a.front_head) {  // outputs written: tell the host (and k_back)
    __syncthreads();  // every thread's output stores precede thread 0's release
    if (threadIdx.x == 0) {
      if (a.out_flag)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a.out_flag + blockIdx.x), "l"(n + 1)
                     : "memory");
      if (a.front_head && a.front_hold != 2) {
        __threadfence();
        atomicAdd(a.front_seq + (n & 1u), 1ull);
      }
      if (a.trace) {  // the moment this CTA's outputs are published (max over CTAs)
        const unsigned long long now = globaltimer();
        atomicMin(&a.trace[((n % kTraceBlocks) * kTraceKernels + TR_OUTPUT) * 2], now);
        atomicMax(&a.trace[((n % kTraceBlocks) * kTraceKernels + TR_OUTPUT) * 2 + 1], now);
      }
    }
  }
  if (a.front_head && a.is_aur) {  // canceller stage 1 on the loudspeakers just produced
    const int N = a.N, Qs = a.mode == 1 ? 1 : a.Q;
    __syncthreads();
    if (a.front_warps) {  // per warp, in the warp's own area (3N float2 from its S/H0 slot)
      const int W = a.front_warps, w = threadIdx.x >> 5;
      const float2* tw = work + (size_t)N * (Qs + 2);
      if (w < W) {
        float2* mine = const_cast<float2*>(tw) + table_f2(N) + (size_t)w * N * (3 + Qs);
        for (int l = c0 + w; l < c1; l += W) head_channels(a, n, l, l + 1, mine, tw, tw + N / 2, Warp());
      }
    } else {
      const float2* tw = a.smem_tables ? work + front_work_f2(N, Qs) : a.tw;
      const float2* split = a.smem_tables ? tw + N / 2 : a.split;
      head_channels(a, n, c0, c1, work, tw, split, Cta());
    }
  }
  trace_end(a, TR_FRONT, n);
}

// ---------------------------------------------------------- k_back_head
// Canceller branch head of block n. CTA l < L (auralizer): canceller stage 1
// on l_n (convolver.hpp:180-191 on fc_): r2c([l_{n-1}, l_n]), FDL push; CTAs
// [L, L + P): NLMS error spectra E_p = r2c([0_N, m~_p]) (Appendix A step 2).
// CTA 0 also moves this block's m~ into the input window history
// (broadcast / mimo). It lets k_back launch at once (PDL): k_back's
// canceller work waits for this grid with griddepcontrol.wait.
__global__ void __launch_bounds__(kFrontThreads) k_back_head(BlockArgs a) {
  extern __shared__ float4 smem4[];
  const int N = a.N;
  float2* z = reinterpret_cast<float2*>(smem4);  // 3N float2 work area
  float2* stw = z + 3 * N;                       // DftPlan tables (if staged)
  const float2* tw = a.smem_tables ? stw : a.tw;
  const float2* split = a.smem_tables ? stw + N / 2 : a.split;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (a.smem_tables) stage_tables(stw, stw + N / 2, a.tw, a.split, N);
  const blk_t n = a.st->block;
  trace_begin(a, TR_BACK_HEAD, n);
  const int Lb = a.is_aur ? a.L : 1;
  const int b = blockIdx.x;
  if (b == 0 && a.mode != 1)
    for (int i = threadIdx.x; i < a.Q * N; i += blockDim.x) a.prev_in[i] = a.cur_mt[i];
  if (!a.is_aur) {
    trace_end(a, TR_BACK_HEAD, n);
    return;
  }
  __syncthreads();
  if (b < Lb) {
    head_channels(a, n, b, b + 1, z, tw, split, Cta());
  } else {
    // E_p = r2c([0_N, m~_p]) from the m~ the front saved
    const int p = b - Lb;
    float* wa = reinterpret_cast<float*>(z + N);
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      wa[i] = 0.0f;
      wa[N + i] = a.cur_mt[(size_t)p * N + i];
    }
    __syncthreads();
    rfft_packed(wa, z, reinterpret_cast<float2*>(a.E + (size_t)p * a.NF), N, a.logN, tw, split);
  }
  trace_end(a, TR_BACK_HEAD, n);
}

// ------------------------------------------------------------ k_advance
__global__ void k_advance(DevState* st) { st->block += 1u; }  // blocks without k_back

__device__ __forceinline__ void st_release_sys(blk_t* p, blk_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ blk_t ld_acquire_sys(const blk_t* p) {
  blk_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
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
// a missing peer sets status_host (the host fails the next call on this
// engine until a coordinated reset) and the block keeps the previous f^ and
// power instead of summing stale slots; the block still retires, so the
// device block counter stays in step with the host's.
__global__ void __launch_bounds__(kTailThreads) k_afc_finish(BlockArgs a) {
  const blk_t n = a.st->block;
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
    for (int g = 0; g < G; ++g) st_release_sys(reinterpret_cast<blk_t*>(a.xpeer[g]) + a.grank, n + 1);
    const blk_t* flags = reinterpret_cast<const blk_t*>(a.xpeer[a.grank]);
    const unsigned long long t0 = globaltimer();
    for (int g = 0; g < G && !timed_out; ++g)
      while (ld_acquire_sys(flags + g) < n + 1) {
        if (globaltimer() - t0 > kShardTimeoutNs) {
          timed_out = 1;
          *reinterpret_cast<volatile unsigned*>(a.status_host) = 1u;
          __threadfence_system();
          break;
        }
        __nanosleep(64);
      }
  }
  __syncthreads();
  if (!timed_out) {
    const float* slots = reinterpret_cast<const float*>(a.xpeer[a.grank] + kXFlagBytes) + (size_t)par * G * S;
    for (int i = threadIdx.x; i < P * N; i += blockDim.x) {
      float v = __ldcg(slots + i);
      for (int g = 1; g < G; ++g) v = __fadd_rn(v, __ldcg(slots + (size_t)g * S + i));
      a.fhat[i] = v;
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
  }
  trace_end(a, TR_AFC_FINISH, n);
  retire_block(a, n);
}

// -------------------------------------------------------- k_afc_apply
// NCCL exchange (xchg 2): after ncclAllReduce(xmine -> xsum) on the engine
// stream, install the summed f^ and smooth the summed power exactly as
// k_afc_finish does, then retire the block. Every rank receives the same
// reduced values from NCCL (reduce-scatter + all-gather), so every shard
// holds the same f^ and power; the summation order is NCCL's (pinned by
// NCCL_ALGO / NCCL_PROTO), not rank order.
__global__ void __launch_bounds__(kTailThreads) k_afc_apply(BlockArgs a) {
  const blk_t n = a.st->block;
  trace_begin(a, TR_AFC_FINISH, n);
  const int N = a.N, P = a.P;
  for (int i = threadIdx.x; i < P * N; i += blockDim.x) {
    a.fhat[i] = __ldcg(a.xsum + i);
  }
  if (a.nlms) {
    const float oml = __fsub_rn(1.0f, a.lambda);
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
      const float2 sum = make_float2(__ldcg(a.xsum + (size_t)P * N + 2 * j), __ldcg(a.xsum + (size_t)P * N + 2 * j + 1));
      float2 w = a.pw[j];
      w.x = __fadd_rn(__fmul_rn(a.lambda, w.x), __fmul_rn(oml, sum.x));
      w.y = __fadd_rn(__fmul_rn(a.lambda, w.y), __fmul_rn(oml, sum.y));
      a.pw[j] = w;
    }
  }
  trace_end(a, TR_AFC_FINISH, n);
  retire_block(a, n);
}

// -------------------------------------------------- k_afc_constrain
// SURVEY Appendix A step 2, constrained variant (AfcParams.constrained): per
// canceller unit (p, l, k) the NLMS gradient G = mu/(P + delta) (.) conj(X_l
// (pre-push age k)) E_p -- rounded exactly as k_back's fused update and the
// oracle (aura_oracle.c constrained_step) -- goes to the time domain (c2r),
// its last N samples are dropped (a partition's taps are the first N of its
// 2N window), and the r2c of [g, 0_N] is added to W. The transforms are the
// bit-exact DftPlan ones (fft.cuh), one warp per unit. Runs after the front
// (E_p, the pushed canceller FDL row) and before k_back, whose canceller
// items then only filter with the updated W: k_front -PDL-> k_afc_constrain
// -PDL-> k_back, so the synthesis stream starts while this kernel runs.
// grid-stride over units; up to kConsThreads threads (fewer warps for large
// N); dynamic smem: the tables (cons_smem_tables), then per warp
// cons_smem_per_warp(N).
// The inputs of one unit as one lane holds them (PL float4 columns: NF = 32 PL).
template <int PL>
struct ConsIn {
  float4 x1[PL], ep[PL], pw[PL], w[PL];
};

// Units u, u + stride, ... of one warp. PL > 0 (N = 64, 128): the next
// unit's loads -- W included -- are issued before this unit's transforms, so
// a warp waits on memory once per unit at most; PL = 0: any N, no prefetch.
template <int PL>
__device__ __forceinline__ void cons_units(const BlockArgs& a, int u, int stride, int nka,
                                           float2* spec, float* win, float2* z, const float2* tw,
                                           const float2* split) {
  const int N = a.N, NF = a.NF, CT = a.CT, CTn = a.CTn, KF = a.KF, P = a.P;
  const int lane = threadIdx.x & 31, cap = KF + 1;
  // 32-bit unit arithmetic (the planner keeps P L K_f < 2^30): a 64-bit
  // division is ~100 instructions, as many as a butterfly stage
  const int U = a.L * KF, units = P * U;
  const float4* pw4 = reinterpret_cast<const float4*>(a.pw);
  float4* spec4 = reinterpret_cast<float4*>(spec);
  constexpr int PLm = PL > 0 ? PL : 1;
  // unit u -> mic p, unit within the mic ul = l KF + k, canceller FDL slot of
  // the pre-push age k (= post-push age k + 1)
  auto decode = [&](int v, int& p, int& ul, int& slot) {
    p = v / U;
    ul = v - p * U;
    const int l = ul / KF, k = ul - l * KF;
    slot = nka - k - 1;
    if (slot < 0) slot += cap;
    return l;
  };
  auto xa_at = [&](int l, int slot, int fg) -> const float4* {
    const int c = fg / CT, f = fg - c * CT;
    return a.XA + ((size_t)(l * CTn + c) * cap + slot) * CT + f;
  };
  auto w_at = [&](int p, int ul, int fg) -> float4* {
    const int c = fg / CT, f = fg - c * CT;
    return a.W + ((size_t)c * U + ul) * P * CT + (size_t)p * CT + f;
  };
  auto load = [&](int v, ConsIn<PLm>& in) {
    int p, slot, ul;
    const int l = decode(v, p, ul, slot);
#pragma unroll
    for (int r = 0; r < PLm; ++r) {
      const int fg = lane + 32 * r;
      in.x1[r] = *xa_at(l, slot, fg);
      in.ep[r] = a.E[(size_t)p * NF + fg];
      in.pw[r] = pw4[fg];
      in.w[r] = *w_at(p, ul, fg);
    }
  };
  // G = mu / (P + delta) (.) conj(x1) E, rounded as k_back's fused update
  auto grad = [&](float4 x1, float4 ep, float4 pw, int fg) {
    const bool dc = fg == 0;
    const float4 st = make_float4(__fdiv_rn(a.mu, __fadd_rn(pw.x, a.delta)), __fdiv_rn(a.mu, __fadd_rn(pw.y, a.delta)),
                                  __fdiv_rn(a.mu, __fadd_rn(pw.z, a.delta)), __fdiv_rn(a.mu, __fadd_rn(pw.w, a.delta)));
    const float px = __fmul_rn(x1.x, ep.x), py = __fmul_rn(x1.y, ep.y);
    float4 gr;
    gr.x = dc ? px : __fadd_rn(px, py);
    gr.y = dc ? py : __fsub_rn(__fmul_rn(x1.x, ep.y), __fmul_rn(x1.y, ep.x));
    gr.z = __fadd_rn(__fmul_rn(x1.z, ep.z), __fmul_rn(x1.w, ep.w));
    gr.w = __fsub_rn(__fmul_rn(x1.z, ep.w), __fmul_rn(x1.w, ep.z));
    spec4[fg] = make_float4(__fmul_rn(st.x, gr.x), __fmul_rn(st.y, gr.y), __fmul_rn(st.z, gr.z),
                            __fmul_rn(st.w, gr.w));
  };
  auto add = [](float4 w, float4 g) {
    return make_float4(__fadd_rn(w.x, g.x), __fadd_rn(w.y, g.y), __fadd_rn(w.z, g.z), __fadd_rn(w.w, g.w));
  };
  // c2r, keep the first N samples, r2c of [g, 0_N] (spec -> spec)
  auto project = [&]() {
    __syncwarp();
    irfft_warp_head(spec, z, N, a.logN, tw, split, [&](int i, float x) { win[i] = x; });
    for (int i = lane; i < N; i += 32) win[N + i] = 0.0f;
    __syncwarp();
    rfft_warp_any(win, z, spec, N, a.logN, tw, split);
  };
  if constexpr (PL > 0) {
    ConsIn<PL> cur, nxt;
    if (u < units) load(u, cur);
    for (; u < units; u += stride) {
#pragma unroll
      for (int r = 0; r < PL; ++r) grad(cur.x1[r], cur.ep[r], cur.pw[r], lane + 32 * r);
      if (u + stride < units) load(u + stride, nxt);
      project();
      int p, slot, ul;
      decode(u, p, ul, slot);
#pragma unroll
      for (int r = 0; r < PL; ++r) *w_at(p, ul, lane + 32 * r) = add(cur.w[r], spec4[lane + 32 * r]);
      __syncwarp();  // spec is reused by the next unit
      cur = nxt;
    }
  } else {
    for (; u < units; u += stride) {
      int p, slot, ul;
      const int l = decode(u, p, ul, slot);
      for (int fg = lane; fg < NF; fg += 32) grad(*xa_at(l, slot, fg), a.E[(size_t)p * NF + fg], pw4[fg], fg);
      project();
      for (int fg = lane; fg < NF; fg += 32) {
        float4* wp = w_at(p, ul, fg);
        *wp = add(*wp, spec4[fg]);
      }
      __syncwarp();
    }
  }
}

__global__ void __launch_bounds__(kConsThreads, 16) k_afc_constrain(const __grid_constant__ BlockArgs a) {
  extern __shared__ float4 csm4[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int N = a.N;
  const int warp = threadIdx.x >> 5;
  // the DftPlan tables (shared by the CTA's warps), then per warp its scratch
  const float2* stw = a.tw;
  const float2* ssplit = a.split;
  float2* spec = reinterpret_cast<float2*>(reinterpret_cast<char*>(csm4) + (a.cons_tables ? cons_smem_tables(N) : 0) +
                                           (size_t)warp * cons_smem_per_warp(N));
  float* win = reinterpret_cast<float*>(spec + N);
  float2* z = reinterpret_cast<float2*>(win + 2 * N);
  if (a.cons_tables) {
    float2* t = reinterpret_cast<float2*>(csm4);
    stage_tables(t, t + N / 2, a.tw, a.split, N);
    stw = t;
    ssplit = t + N / 2;
  }
  __syncthreads();
  asm volatile("griddepcontrol.wait;" ::: "memory");  // E_p and this block's canceller FDL row
  const blk_t n = a.st->block;
  trace_begin(a, TR_AFC_CONS, n);
  const int nka = (int)(n % (blk_t)(a.KF + 1));
  const int warps = (int)(blockDim.x >> 5);
  const int u0 = (int)blockIdx.x * warps + warp, stride = (int)gridDim.x * warps;
  if (a.NF == 32 && a.cons_prefetch) cons_units<1>(a, u0, stride, nka, spec, win, z, stw, ssplit);
  else if (a.NF == 64 && a.cons_prefetch) cons_units<2>(a, u0, stride, nka, spec, win, z, stw, ssplit);
  else cons_units<0>(a, u0, stride, nka, spec, win, z, stw, ssplit);
  trace_end(a, TR_AFC_CONS, n);
}

// ------------------------------------------------- k_afc_constrain8
// k_afc_constrain for N = 64 (c3's block size) with eight threads per unit
// and eight points per thread: the 64-point transforms run their first three
// radix-2 stages inside each thread (contiguous points), a shared-memory
// transpose, and the last three inside each thread again (strided points) --
// every butterfly computed once, by one thread, with no shuffles -- where the
// one-warp-per-unit kernel computes each butterfly on both lanes of a pair.
// Same butterflies, twiddles and association as DftPlan (fft.cuh), so the
// same bits as k_afc_constrain. Four units per warp; grid-stride over units.
// Dynamic smem: the DftPlan tables, E_p and the power of the CTA's block,
// then per warp four units x {spectrum, exchange buffer} (64 float2 each).
constexpr int kCons8Threads = 128;
__host__ __device__ inline size_t cons8_smem(int P) {
  return 16 * (size_t)(34 + 32 * (P + 1)) + (size_t)(kCons8Threads / 32) * 4 * 2 * 64 * 8;
}

__device__ __forceinline__ int bitrev6(int m) { return (int)(__brev((unsigned)m) >> 26); }

// radix-2 DIT butterfly on (u, v) with twiddle w: u + v w, u - v w (v w
// rounded as cmul_rn), the same operations as fft_dit_smem / fft_dit_warp
__device__ __forceinline__ void bfly(float2& u, float2& v, float2 w) {
  const float2 wv = cmul_rn(v, w);
  const float2 a = cadd_rn(u, wv);
  v = csub_rn(u, wv);
  u = a;
}

// 64-point DIT on the 8 points of thread t (of 8) held contiguously
// (z[8t + r], bit-reversed input order); returns them strided (z[t + 8r]).
// buf: the unit's 64-float2 exchange buffer; tw: e^{-2 pi i j / 64}, j < 32.
__device__ __forceinline__ void fft64_oct(float2 (&z)[8], int t, float2* buf, const float2* tw) {
#pragma unroll
  for (int h = 1; h < 8; h <<= 1) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if ((r & h) == 0) bfly(z[r], z[r + h], tw[(r & (h - 1)) * (32 / h)]);
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) buf[8 * t + r] = z[r];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 8; ++r) z[r] = buf[t + 8 * r];
  __syncwarp();
#pragma unroll
  for (int hh = 1; hh < 8; hh <<= 1) {  // h = 8 hh: pairs (r, r + hh) of the strided points
    const int h = 8 * hh;
#pragma unroll
    for (int r = 0; r < 8; ++r)
      if ((r & hh) == 0) bfly(z[r], z[r + hh], tw[(t + 8 * (r & (hh - 1))) * (32 / h)]);
  }
}

__global__ void __launch_bounds__(kCons8Threads, 8) k_afc_constrain8(const __grid_constant__ BlockArgs a) {
  extern __shared__ float4 c8sm[];
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  constexpr int N = 64, NF = 32, H = 32;
  const int P = a.P, KF = a.KF, L = a.L;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane >> 3, t = lane & 7;  // unit within the warp, thread within the unit
  float2* stw = reinterpret_cast<float2*>(c8sm);  // 32 + 33 float2 (34 float4)
  float2* ssplit = stw + N / 2;
  float4* sE = c8sm + 34;                         // [P][NF]
  float4* spw = sE + (size_t)P * NF;              // [NF]
  float2* ubase = reinterpret_cast<float2*>(spw + NF) + (size_t)(warp * 4 + sub) * 2 * 64;
  float2* spec = ubase;       // the unit's packed spectrum (64 float2)
  float2* buf = ubase + 64;   // its exchange buffer
  float4* spec4 = reinterpret_cast<float4*>(spec);
  stage_tables(stw, ssplit, a.tw, a.split, N);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // E_p from the front
  for (int i = threadIdx.x; i < P * NF; i += blockDim.x) sE[i] = a.E[i];
  for (int i = threadIdx.x; i < NF; i += blockDim.x) spw[i] = reinterpret_cast<const float4*>(a.pw)[i];
  __syncthreads();
  const blk_t n = a.st->block;
  trace_begin(a, TR_AFC_CONS, n);
  const int cap = KF + 1;
  const int nka = (int)(n % (blk_t)cap);
  const int U = L * KF, units = P * U;
  const int per_pass = (int)gridDim.x * (kCons8Threads / 32) * 4;
  const float scale = 1.0f / (float)N;
  for (int base = ((int)blockIdx.x * (kCons8Threads / 32) + warp) * 4; base < units; base += per_pass) {
    const int u = base + sub;
    const bool ok = u < units;
    int p = 0, ul = 0, slot = 0, l = 0;
    if (ok) {
      p = u / U;
      ul = u - p * U;
      l = ul / KF;
      const int k = ul - l * KF;
      slot = nka - k - 1;  // pre-push age k
      if (slot < 0) slot += cap;
    }
    // (1) the gradient G = mu / (P + delta) (.) conj(x1) E_p -> spec, four
    // float4 columns per thread, rounded as k_back's fused update
    float4 wv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int fg = t + 8 * j;
      if (!ok) {
        wv[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        continue;
      }
      const bool dc = fg == 0;
      const float4 x1 = a.XA[((size_t)l * cap + slot) * NF + fg];
      wv[j] = a.W[((size_t)ul) * P * NF + (size_t)p * NF + fg];
      const float4 ep = sE[(size_t)p * NF + fg];
      const float4 pw = spw[fg];
      const float4 st = make_float4(__fdiv_rn(a.mu, __fadd_rn(pw.x, a.delta)), __fdiv_rn(a.mu, __fadd_rn(pw.y, a.delta)),
                                    __fdiv_rn(a.mu, __fadd_rn(pw.z, a.delta)), __fdiv_rn(a.mu, __fadd_rn(pw.w, a.delta)));
      const float px = __fmul_rn(x1.x, ep.x), py = __fmul_rn(x1.y, ep.y);
      float4 gr;
      gr.x = dc ? px : __fadd_rn(px, py);
      gr.y = dc ? py : __fsub_rn(__fmul_rn(x1.x, ep.y), __fmul_rn(x1.y, ep.x));
      gr.z = __fadd_rn(__fmul_rn(x1.z, ep.z), __fmul_rn(x1.w, ep.w));
      gr.w = __fsub_rn(__fmul_rn(x1.z, ep.w), __fmul_rn(x1.w, ep.z));
      spec4[fg] = make_float4(__fmul_rn(st.x, gr.x), __fmul_rn(st.y, gr.y), __fmul_rn(st.z, gr.z),
                              __fmul_rn(st.w, gr.w));
    }
    __syncwarp();
    // (2) c2r: merge into the half-size spectrum (dft.hpp:130-146, as
    // irfft_packed_tail), bit-reversed into this thread's 8 contiguous points
    float2 z[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int k = bitrev6(8 * t + r);
      float2 zk;
      if (k == 0) {
        const float2 s0 = spec[0];  // (DC, Nyquist)
        const float xe = __fmul_rn(0.5f, __fadd_rn(s0.x, s0.y));
        const float xo = __fmul_rn(0.5f, __fsub_rn(s0.x, s0.y));
        zk = make_float2(xe, -xo);
      } else {
        const float2 av = spec[k];
        const float2 bv = conjf2(spec[N - k]);
        const float2 even = half_of(cadd_rn(av, bv));
        float2 tw2;
        if (k <= H) {
          tw2 = ssplit[k];
        } else {
          const float2 q = conjf2(ssplit[N - k]);
          tw2 = make_float2(-q.x, -q.y);
        }
        const float2 odd = cmul_rn(conjf2(tw2), half_of(csub_rn(av, bv)));
        const float2 iodd = cmul_rn(make_float2(0.0f, 1.0f), odd);
        zk = conjf2(cadd_rn(even, iodd));
      }
      z[r] = zk;
    }
    fft64_oct(z, t, buf, stw);  // now z[r] = point t + 8 r
    // (3) the first N samples x[2m], x[2m+1] = (z[m].x, -z[m].y) / N for
    // m < 32 (r < 4); the window's second half is zero. r2c input: point
    // bitrev(m) = (x[2m], x[2m+1]), via the exchange buffer
#pragma unroll
    for (int r = 0; r < 4; ++r)
      buf[t + 8 * r] = make_float2(__fmul_rn(z[r].x, scale), __fmul_rn(-z[r].y, scale));
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int m = bitrev6(8 * t + r);
      z[r] = m < 32 ? buf[m] : make_float2(0.0f, 0.0f);
    }
    __syncwarp();
    fft64_oct(z, t, buf, stw);
    // (4) split (dft.hpp:88-100, as rfft_packed) -> spec, then W += spec
#pragma unroll
    for (int r = 0; r < 8; ++r) buf[t + 8 * r] = z[r];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      const int k = t + 8 * j;
      if (k > H) break;
      if (k == 0) {
        const float2 z0 = buf[0];
        spec[0] = make_float2(__fadd_rn(z0.x, z0.y), __fsub_rn(z0.x, z0.y));
        continue;
      }
      const float2 av = buf[k];
      const float2 bv = conjf2(buf[N - k]);
      const float2 even = half_of(cadd_rn(av, bv));
      const float2 d = csub_rn(av, bv);
      const float2 odd = cmul_rn(make_float2(0.0f, -0.5f), d);
      const float2 rot = cmul_rn(ssplit[k], odd);
      const float2 lo = cadd_rn(even, rot);
      const float2 hi = conjf2(csub_rn(even, rot));
      if (k != H) spec[k] = lo;  // at k = N/2 the reference's second store wins
      spec[N - k] = hi;
    }
    __syncwarp();
    if (ok) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int fg = t + 8 * j;
        const float4 g = spec4[fg];
        float4 w = wv[j];
        w.x = __fadd_rn(w.x, g.x);
        w.y = __fadd_rn(w.y, g.y);
        w.z = __fadd_rn(w.z, g.z);
        w.w = __fadd_rn(w.w, g.w);
        a.W[((size_t)ul) * P * NF + (size_t)p * NF + fg] = w;
      }
    }
    __syncwarp();  // spec and buf are reused by the next unit
  }
  trace_end(a, TR_AFC_CONS, n);
}

// ------------------------------------------------------ k_partition
// Setup (make_partitioned_filters, convolver.hpp:19-46) on the GPU: CTA
// (k, r) transforms taps[r][kN .. kN+N) zero-padded to 2N and scatters the
// packed spectrum into the device layout: column f of partition k of row r
// goes to dst[base[r] + k*kstride + (f/CT)*cstride + f%CT], except partition
// 0 when dst0 is set (-> dst0[base0[r] + f]). taps rows are n_h long.
__global__ void __launch_bounds__(256) k_partition(
    const float* __restrict__ taps, size_t n_h, int K, int N, int logN, const float2* tw,
    const float2* split, PartOut o, const long long* __restrict__ base,
    const long long* __restrict__ base0) {
  extern __shared__ float smem[];
  float* win = smem;                                   // 2N floats, then the spectrum
  float2* z = reinterpret_cast<float2*>(win + 2 * N);  // N
  float2* stw = z + N;                                 // DftPlan tables
  float2* ssplit = stw + N / 2;
  stage_tables(stw, ssplit, tw, split, N);
  const int k = blockIdx.x;
  const int r = blockIdx.y;
  const size_t begin = (size_t)k * N;
  const float* src = taps + (size_t)r * n_h;
  for (int i = threadIdx.x; i < 2 * N; i += blockDim.x) {
    const size_t t = begin + i;
    win[i] = (i < N && t < n_h) ? src[t] : 0.0f;
  }
  __syncthreads();
  float2* spec = reinterpret_cast<float2*>(win);  // rfft reads win before it writes spec
  rfft_packed(win, z, spec, N, logN, stw, ssplit);
  if (k == 0 && o.dst0) {
    float2* d = reinterpret_cast<float2*>(o.dst0 + base0[r]);
    for (int j = threadIdx.x; j < N; j += blockDim.x) d[j] = spec[j];
    return;
  }
  float2* d = reinterpret_cast<float2*>(o.dst);
  const long long b = base[r] + (long long)k * o.kstride;
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    const int f = j >> 1;
    const long long i4 = b + (long long)(f / o.CT) * o.cstride + (f % o.CT);
    d[2 * i4 + (j & 1)] = spec[j];
  }
}

}  // namespace aura_b200
