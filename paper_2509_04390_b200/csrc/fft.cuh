// fft.cuh -- block-level real FFTs for the UPOLS block loop (sm_100a).
//
// The reference computes an n_f-point real transform as an n_f/2-point
// complex radix-2 DIT FFT of the even/odd-interleaved samples plus a split
// step (dft.hpp:69-101 forward, dft.hpp:124-153 inverse; forward
// unnormalised, inverse scaled by 1/n_f). The device transforms here
// perform the SAME floating-point operations in the same association
// (products rounded separately via __fmul_rn -- no FMA contraction -- and
// twiddle tables built on the host exactly as DftPlan builds them), so the
// spectra are bit-identical to the reference's. That pins the partition
// spectra of make_partitioned_filters, the FDL contents and the canceller's
// error spectra exactly; only the MAC's summation order differs.
//
// Layout differs from the reference: spectra are PACKED -- N = n_f/2
// complex values, bin 0 holds DC in .x and Nyquist in .y (both exactly real)
// -- so every partition is 8N bytes, 16-byte aligned for the streaming MAC.
// The butterflies run in shared memory with all threads of the CTA.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace aura_b200 {

// The threads that run a transform together: the whole CTA (Cta), or the
// 256 consumer threads of the warp-specialised streaming kernel (named
// barrier 1, so its producer warp never has to join).
struct Cta {
  __device__ __forceinline__ int tid() const { return threadIdx.x; }
  __device__ __forceinline__ int size() const { return blockDim.x; }
  __device__ __forceinline__ void sync() const { __syncthreads(); }
};
// One warp (independent of the rest of its CTA): __syncwarp between stages.
struct Warp {
  __device__ __forceinline__ int tid() const { return threadIdx.x & 31; }
  __device__ __forceinline__ int size() const { return 32; }
  __device__ __forceinline__ void sync() const { __syncwarp(); }
};
template <int NT>
struct Consumers {
  __device__ __forceinline__ int tid() const { return threadIdx.x; }
  __device__ __forceinline__ int size() const { return NT; }
  __device__ __forceinline__ void sync() const { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); }
};

// (a.x c - a.y d, a.x d + a.y c), each product rounded (= libstdc++
// complex<float> multiply on x86-64 without FMA).
__device__ __forceinline__ float2 cmul_rn(float2 a, float2 b) {
  return make_float2(__fsub_rn(__fmul_rn(a.x, b.x), __fmul_rn(a.y, b.y)),
                     __fadd_rn(__fmul_rn(a.x, b.y), __fmul_rn(a.y, b.x)));
}
__device__ __forceinline__ float2 cadd_rn(float2 a, float2 b) {
  return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
}
__device__ __forceinline__ float2 csub_rn(float2 a, float2 b) {
  return make_float2(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y));
}
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 half_of(float2 a) {
  return make_float2(__fmul_rn(0.5f, a.x), __fmul_rn(0.5f, a.y));
}

// In-place radix-2 DIT FFT of size M on shared z (input already in
// bit-reversed order), butterflies as dft.hpp:163-176. tw[j] =
// e^{-2 pi i j / M}, j < M/2. Ends with a barrier.
template <typename Team = Cta>
__device__ void fft_dit_smem(float2* z, int M, const float2* __restrict__ tw, Team tm = Team()) {
  for (int len = 2; len <= M; len <<= 1) {
    const int h = len >> 1;
    const int stride = M / len;
    for (int b = tm.tid(); b < (M >> 1); b += tm.size()) {
      const int pos = b & (h - 1);
      const int i0 = ((b - pos) << 1) + pos;  // base + k
      const int i1 = i0 + h;
      const float2 w = tw[pos * stride];
      const float2 u = z[i0];
      const float2 v = cmul_rn(z[i1], w);
      z[i0] = cadd_rn(u, v);
      z[i1] = csub_rn(u, v);
    }
    tm.sync();
  }
}

// Stage the DftPlan tables in shared memory (tw: N/2, split: N/2 + 1 float2)
// so the butterfly stages read them at shared-memory latency instead of one
// dependent L2 round trip per stage. No barrier: the caller syncs.
template <typename Team = Cta>
__device__ __forceinline__ void stage_tables(float2* s_tw, float2* s_split, const float2* __restrict__ tw,
                                             const float2* __restrict__ split, int N, Team tm = Team()) {
  for (int j = tm.tid(); j < N / 2; j += tm.size()) s_tw[j] = __ldg(tw + j);
  for (int j = tm.tid(); j <= N / 2; j += tm.size()) s_split[j] = __ldg(split + j);
}
// shared-memory float2 count of the staged tables
__host__ __device__ constexpr int table_f2(int N) { return N + 2; }

__device__ __forceinline__ int bitrev(int m, int logM) {
  return (int)(__brev((unsigned)m) >> (32 - logM));
}

// r2c of the 2N-sample real window `win` (shared) into the packed spectrum
// `spec` (N complex; shared or global). z: N float2 shared scratch.
// split[k] = e^{-2 pi i k / (2N)}, k <= N/2. dft.hpp:69-101. Ends with a
// barrier.
template <typename Team = Cta>
__device__ void rfft_packed(const float* win, float2* z, float2* spec, int N,
                            int logN, const float2* __restrict__ tw,
                            const float2* __restrict__ split, Team tm = Team()) {
  for (int m = tm.tid(); m < N; m += tm.size())
    z[bitrev(m, logN)] = make_float2(win[2 * m], win[2 * m + 1]);
  tm.sync();
  fft_dit_smem(z, N, tw, tm);
  const int H = N >> 1;
  for (int k = tm.tid(); k <= H; k += tm.size()) {
    if (k == 0) {
      const float2 z0 = z[0];
      spec[0] = make_float2(__fadd_rn(z0.x, z0.y), __fsub_rn(z0.x, z0.y));
      continue;
    }
    const float2 a = z[k];
    const float2 b = conjf2(z[N - k]);
    const float2 even = half_of(cadd_rn(a, b));
    // odd = (0, -0.5) * (a - b), evaluated as the complex product
    const float2 d = csub_rn(a, b);
    const float2 odd = cmul_rn(make_float2(0.0f, -0.5f), d);
    const float2 rot = cmul_rn(split[k], odd);
    const float2 lo = cadd_rn(even, rot);
    const float2 hi = conjf2(csub_rn(even, rot));
    if (k != H) spec[k] = lo;  // at k = N/2 the reference's second store wins
    spec[N - k] = hi;
  }
  tm.sync();
}

// c2r of the packed spectrum `spec` (shared, N complex) into the LAST N
// samples of the 2N-point inverse (overlap-save keeps only those,
// convolver.hpp:202-205), scaled by 1/(2N): store(i, x[N + i]).
// dft.hpp:124-153 (merge, conj -> forward FFT -> conj, scale 1/half).
// z: N float2 shared scratch. Ends with a barrier.
// kHead: the FIRST N samples instead, store(i, x[i]) (the constrained
// canceller gradient keeps those).
template <typename Store, typename Team = Cta, bool kHead = false>
__device__ void irfft_packed_tail(const float2* spec, float2* z, int N,
                                  int logN, const float2* __restrict__ tw,
                                  const float2* __restrict__ split,
                                  Store store, Team tm = Team()) {
  const int H = N >> 1;
  for (int k = tm.tid(); k < N; k += tm.size()) {
    float2 zk;
    if (k == 0) {
      const float2 s = spec[0];  // (DC, Nyquist)
      const float xe = __fmul_rn(0.5f, __fadd_rn(s.x, s.y));
      const float xo = __fmul_rn(0.5f, __fsub_rn(s.x, s.y));
      zk = make_float2(xe, -xo);
    } else {
      const float2 a = spec[k];
      const float2 b = conjf2(spec[N - k]);
      const float2 even = half_of(cadd_rn(a, b));
      float2 tw2;
      if (k <= H) {
        tw2 = split[k];
      } else {
        const float2 s = conjf2(split[N - k]);
        tw2 = make_float2(-s.x, -s.y);
      }
      const float2 odd = cmul_rn(conjf2(tw2), half_of(csub_rn(a, b)));
      const float2 iodd = cmul_rn(make_float2(0.0f, 1.0f), odd);
      zk = conjf2(cadd_rn(even, iodd));
    }
    z[bitrev(k, logN)] = zk;
  }
  tm.sync();
  fft_dit_smem(z, N, tw, tm);
  const float scale = 1.0f / (float)N;
  // samples N .. 2N-1 are z[m] for m in [N/2, N) (samples 0 .. N-1: m < N/2)
  for (int m = tm.tid(); m < H; m += tm.size()) {
    const float2 v = z[kHead ? m : H + m];
    store(2 * m, __fmul_rn(v.x, scale));
    store(2 * m + 1, __fmul_rn(-v.y, scale));
  }
  tm.sync();
}

// ------------------------------------------------ register-resident warp FFTs
// One warp, M = 32 * PER points, element i in lane i % 32, register i / 32.
// The SAME radix-2 DIT butterflies as fft_dit_smem (pairs (i0, i0 + h), twiddle
// tw[(i0 mod h) * M / 2h], u + w v and u - w v with w v = cmul_rn(v, w), each
// product rounded), so the same bits; partners h < 32 apart are exchanged with
// shuffles, no shared memory and no barriers between stages. Measured
// (tools/c2r_probe.cu): the shared-memory warp transform of N = 64 takes ~2460
// cycles, the latency of the LDS -> math -> STS -> __syncwarp chain per stage.
template <int PER>
__device__ __forceinline__ void fft_dit_warp(float2 (&v)[PER], const float2* __restrict__ tw, int lane) {
  constexpr int M = 32 * PER;
#pragma unroll
  for (int h = 1; h < M; h <<= 1) {
    const int stride = M / (2 * h);
    float2 nv[PER];
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int i = lane + 32 * r;
      const float2 x = v[r];
      float2 y;
      if (h < 32) {
        y.x = __shfl_xor_sync(0xffffffffu, x.x, h);
        y.y = __shfl_xor_sync(0xffffffffu, x.y, h);
      } else {
        y = v[r ^ (h >> 5)];
      }
      const bool lo = (i & h) == 0;
      const float2 w = tw[(i & (h - 1)) * stride];
      const float2 wv = cmul_rn(lo ? y : x, w);
      const float2 u = lo ? x : y;
      nv[r] = lo ? cadd_rn(u, wv) : csub_rn(u, wv);
    }
#pragma unroll
    for (int r = 0; r < PER; ++r) v[r] = nv[r];
  }
}

// irfft_packed_tail on one warp with the transform in registers (N = 32 PER).
template <int PER, typename Store, bool kHead = false>
__device__ __forceinline__ void irfft_packed_tail_reg(const float2* spec, int logN, const float2* __restrict__ tw,
                                                      const float2* __restrict__ split, Store store) {
  constexpr int N = 32 * PER, H = N / 2;
  const int lane = threadIdx.x & 31;
  float2 v[PER];
  float4 sv[PER];
#pragma unroll
  for (int r = 0; r < PER; ++r) {  // every load first
    const int k = bitrev(lane + 32 * r, logN);
    const float2 s0 = spec[k], s1 = spec[(N - k) & (N - 1)];
    sv[r] = make_float4(s0.x, s0.y, s1.x, s1.y);
  }
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    const int k = bitrev(lane + 32 * r, logN);
    float2 zk;
    if (k == 0) {
      const float xe = __fmul_rn(0.5f, __fadd_rn(sv[r].x, sv[r].y));
      const float xo = __fmul_rn(0.5f, __fsub_rn(sv[r].x, sv[r].y));
      zk = make_float2(xe, -xo);
    } else {
      const float2 a = make_float2(sv[r].x, sv[r].y);
      const float2 b = conjf2(make_float2(sv[r].z, sv[r].w));
      const float2 even = half_of(cadd_rn(a, b));
      float2 tw2;
      if (k <= H) {
        tw2 = split[k];
      } else {
        const float2 q = conjf2(split[N - k]);
        tw2 = make_float2(-q.x, -q.y);
      }
      const float2 odd = cmul_rn(conjf2(tw2), half_of(csub_rn(a, b)));
      const float2 iodd = cmul_rn(make_float2(0.0f, 1.0f), odd);
      zk = conjf2(cadd_rn(even, iodd));
    }
    v[r] = zk;
  }
  fft_dit_warp<PER>(v, tw, lane);
  const float scale = 1.0f / (float)N;
#pragma unroll
  for (int r = kHead ? 0 : PER / 2; r < (kHead ? PER / 2 : PER); ++r) {  // z[m], m in [N/2, N): samples N .. 2N-1
    const int m = lane + 32 * r - (kHead ? 0 : H);
    store(2 * m, __fmul_rn(v[r].x, scale));
    store(2 * m + 1, __fmul_rn(-v[r].y, scale));
  }
  __syncwarp();  // the caller may overwrite `spec` next
}

// rfft_packed on one warp with the transform in registers (N = 32 PER); z:
// N float2 shared scratch for the split step. Ends with __syncwarp.
template <int PER>
__device__ __forceinline__ void rfft_packed_reg(const float* win, float2* z, float2* spec, int logN,
                                                const float2* __restrict__ tw, const float2* __restrict__ split) {
  constexpr int N = 32 * PER, H = N / 2;
  const int lane = threadIdx.x & 31;
  float2 v[PER];
#pragma unroll
  for (int r = 0; r < PER; ++r) {
    const int m = bitrev(lane + 32 * r, logN);
    v[r] = make_float2(win[2 * m], win[2 * m + 1]);
  }
  fft_dit_warp<PER>(v, tw, lane);
#pragma unroll
  for (int r = 0; r < PER; ++r) z[lane + 32 * r] = v[r];
  __syncwarp();
  for (int k = lane; k <= H; k += 32) {
    if (k == 0) {
      const float2 z0 = z[0];
      spec[0] = make_float2(__fadd_rn(z0.x, z0.y), __fsub_rn(z0.x, z0.y));
      continue;
    }
    const float2 a = z[k];
    const float2 b = conjf2(z[N - k]);
    const float2 even = half_of(cadd_rn(a, b));
    const float2 d = csub_rn(a, b);
    const float2 odd = cmul_rn(make_float2(0.0f, -0.5f), d);
    const float2 rot = cmul_rn(split[k], odd);
    const float2 lo = cadd_rn(even, rot);
    const float2 hi = conjf2(csub_rn(even, rot));
    if (k != H) spec[k] = lo;  // at k = N/2 the reference's second store wins
    spec[N - k] = hi;
  }
  __syncwarp();
}

// One warp's c2r / r2c: registers for N = 64 and 128, shared memory otherwise.
template <typename Store>
__device__ __forceinline__ void irfft_warp_any(const float2* spec, float2* z, int N, int logN,
                                               const float2* __restrict__ tw, const float2* __restrict__ split,
                                               Store store) {
  if (N == 64) irfft_packed_tail_reg<2>(spec, logN, tw, split, store);
  else if (N == 128) irfft_packed_tail_reg<4>(spec, logN, tw, split, store);
  else irfft_packed_tail(spec, z, N, logN, tw, split, store, Warp());
}
// The first N samples of one warp's c2r (irfft_warp_any's head).
template <typename Store>
__device__ __forceinline__ void irfft_warp_head(const float2* spec, float2* z, int N, int logN,
                                                const float2* __restrict__ tw, const float2* __restrict__ split,
                                                Store store) {
  if (N == 64) irfft_packed_tail_reg<2, Store, true>(spec, logN, tw, split, store);
  else if (N == 128) irfft_packed_tail_reg<4, Store, true>(spec, logN, tw, split, store);
  else irfft_packed_tail<Store, Warp, true>(spec, z, N, logN, tw, split, store, Warp());
}
__device__ __forceinline__ void rfft_warp_any(const float* win, float2* z, float2* spec, int N, int logN,
                                              const float2* __restrict__ tw, const float2* __restrict__ split) {
  if (N == 64) rfft_packed_reg<2>(win, z, spec, logN, tw, split);
  else if (N == 128) rfft_packed_reg<4>(win, z, spec, logN, tw, split);
  else rfft_packed(win, z, spec, N, logN, tw, split, Warp());
}

}  // namespace aura_b200
