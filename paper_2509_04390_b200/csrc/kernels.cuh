// kernels.cuh -- the per-block UPOLS + feedback-canceller kernels (sm_100a).
//
// One block of audio = one CUDA-graph launch of these kernels, in order:
//   k_input      m~ = g m - f^, window, r2c, FDL push; NLMS error spectra
//   k_mac_synth  streaming FDL x filter-spectra MAC, split over partitions
//   k_tail_synth fixed-order split-K reduce, c2r, overlap-save output,
//                feedback-canceller r2c + FDL push, power partials
//   k_mac_afc    feedback-canceller MAC with the fused NLMS update of W
//   k_tail_afc   fixed-order reduce, one c2r per mic -> f^ for next block
// (a Convolver launches only the first three.)
//
// Reference anchors: convolver.hpp:150-206 (stages 1-3), backend.hpp:212-235
// (spectral_mac_channel), auralizer.hpp:61-87 (AFC pipeline), SURVEY.md
// Appendix A/B (NLMS, MIMO). All reductions run in a fixed order, so
// results are bit-reproducible run to run (test_convolver.cpp:172-193).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fft.cuh"

namespace aura_b200 {

constexpr int kMacThreads = 256;
constexpr int kTailThreads = 512;

// Device-resident stream state. `block` is the index of the block being
// processed; it advances when the last CTA of the last kernel retires.
struct DevState {
  uint32_t block;
  uint32_t ticket;
};

struct BlockArgs {
  // geometry
  int N, logN, NF;   // NF = N/2 float4 columns per packed spectrum
  int Q, L, P;       // inputs, outputs (local), mics (auralizer: P = Q)
  int K, KF;         // synth partitions, canceller partitions
  int mode;          // 0 broadcast, 1 elementwise, 2 mimo
  int is_aur, nlms;
  float gain, mu, lambda, delta;
  // split-K geometry
  int syn_chunks, syn_tc, syn_nft, syn_tiles;
  int afc_chunks, afc_uc, afc_nft, afc_tiles;
  // tables
  const float2* tw;     // N/2, e^{-2 pi i j / N}
  const float2* split;  // N,   e^{-i pi k / N}
  // state
  DevState* st;
  float* prev_in;       // Q x N (elementwise: L x N)  previous input block
  float4* X;            // input FDL   [Qx][K][NF]
  const float4* H;      // spectra     [L][Q][K][NF] (bcast/elem Q = 1)
  float4* part_syn;     // [syn_chunks][L][NF]
  float* prev_spk;      // L x N previous loudspeaker block
  float4* XA;           // canceller FDL [L][KF+1][NF]
  float4* W;            // canceller spectra [P][L][KF][NF]
  float2* pw_part;      // [L][N]   packed |X_l|^2 of the newest spectrum
  float2* pw;           // [N]      smoothed power (packed: bin0 = DC,Nyq)
  float4* E;            // [P][NF]  error spectra
  float4* part_afc;     // [afc_chunks][P][NF]
  float* fhat;          // P x N    feedback estimate for the next block
  // I/O (device pointers; may alias pinned mapped host memory)
  const float* in;      // inputs x N
  float* out;           // L x N
  volatile uint32_t* done;  // mapped host word: block sequence when done
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
  float xr0, xi0;  // cross-term operands for the first pair
};
__device__ __forceinline__ XPack xpack(float4 x, bool dc) {
  XPack p;
  p.v = x;
  p.xr0 = dc ? 0.0f : x.x;
  p.xi0 = dc ? 0.0f : x.y;
  return p;
}
__device__ __forceinline__ void cmac(float4& acc, const XPack& x, float4 h,
                                     bool dc) {
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
__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

__device__ __forceinline__ int ring(int v, int cap) {
  v %= cap;
  return v < 0 ? v + cap : v;
}

// Sum `nc` partial rows part[c*stride + col] for every column of an NF-wide
// float4 row, in a fixed order, into out[col] (shared). Uses all threads.
// red: blockDim float4 shared scratch.
__device__ void reduce_partials(const float4* __restrict__ part, int nc,
                                size_t stride, int NF, float4* red,
                                float4* out) {
  const int T = blockDim.x;
  if (NF >= T) {
    for (int f = threadIdx.x; f < NF; f += T) {
      float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int c = 0; c < nc; ++c) s = f4add(s, part[(size_t)c * stride + f]);
      out[f] = s;
    }
    __syncthreads();
    return;
  }
  const int R = T / NF;
  const int f = threadIdx.x % NF;
  const int r = threadIdx.x / NF;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int c = r; c < nc; c += R) s = f4add(s, part[(size_t)c * stride + f]);
  red[threadIdx.x] = s;
  __syncthreads();
  if (r == 0) {
    float4 t = red[f];
    for (int rr = 1; rr < R; ++rr) t = f4add(t, red[rr * NF + f]);
    out[f] = t;
  }
  __syncthreads();
}

// Retire one CTA of the last kernel of a block; the last one advances the
// block counter and publishes the host-visible done word.
__device__ void retire_block(const BlockArgs& a, uint32_t n) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const uint32_t total = gridDim.x * gridDim.y * gridDim.z;
    const uint32_t t = atomicAdd(&a.st->ticket, 1u);
    if (t == total - 1) {
      a.st->ticket = 0;
      a.st->block = n + 1;
      __threadfence_system();
      *a.done = n + 1;
    }
  }
}

// ------------------------------------------------------------ k_input
// Stage 1 (convolver.hpp:180-191) for every input channel, with the
// auralizer's m~ = g*m - f^ (auralizer.hpp:73-76) fused in. CTAs
// [Qx, Qx + P) build the NLMS error spectra E_p = r2c([0_N, m~_p])
// (Appendix A step 2). Shared: 2N floats window + N float2 FFT scratch.
__global__ void __launch_bounds__(256) k_input(BlockArgs a) {
  extern __shared__ float smem[];
  float* win = smem;                           // 2N
  float2* z = reinterpret_cast<float2*>(win + 2 * a.N);  // N
  const int N = a.N;
  const uint32_t n = a.st->block;
  const int Qx = a.mode == 1 ? a.L : a.Q;  // FDL channels
  const int ch = blockIdx.x;
  const bool err_cta = ch >= Qx;
  const int q = err_cta ? ch - Qx : ch;
  const float* in = a.in + (size_t)q * N;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    float v = in[i];
    if (a.is_aur) v = __fsub_rn(__fmul_rn(a.gain, v), a.fhat[(size_t)q * N + i]);
    if (err_cta) {
      win[i] = 0.0f;
      win[N + i] = v;
    } else {
      float* prev = a.prev_in + (size_t)q * N;
      win[i] = prev[i];
      win[N + i] = v;
    }
  }
  __syncthreads();
  if (!err_cta) {
    float* prev = a.prev_in + (size_t)q * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) prev[i] = win[N + i];
  }
  float2* dst = err_cta
                    ? reinterpret_cast<float2*>(a.E + (size_t)q * a.NF)
                    : reinterpret_cast<float2*>(
                          a.X + ((size_t)q * a.K + (n % (uint32_t)a.K)) * a.NF);
  rfft_packed(win, z, dst, N, a.logN, a.tw, a.split);
}

// --------------------------------------------------------- k_mac_synth
// out[l][j] += sum_{taps t in chunk} X[q(t)][age k(t)][j] * H[l][t][j]
// (backend.hpp:212-235). grid = (syn_chunks, L/LT, syn_tiles), 256 threads.
// Thread (kp, f): column f of the tile, tap phase kp; LT channels share
// each X load (broadcast / MIMO) -- X is read from L2, H streamed from HBM
// with 128-bit no-L1-allocate loads. ELEM: channel l reads FDL channel l.
template <int LT, bool ELEM>
__global__ void __launch_bounds__(kMacThreads, 2) k_mac_synth(BlockArgs a) {
  __shared__ float4 red[kMacThreads * LT];
  const int nft = a.syn_nft;
  const int KP = kMacThreads / nft;
  const int fl = threadIdx.x & (nft - 1);
  const int kp = threadIdx.x / nft;
  const int f = blockIdx.z * nft + fl;
  const int l0 = blockIdx.y * LT;
  const int K = a.K;
  const int T = ELEM ? K : a.Q * K;
  const int t0 = blockIdx.x * a.syn_tc;
  const int t1 = min(t0 + a.syn_tc, T);
  const int nk = (int)(a.st->block % (uint32_t)K);
  const bool dc = (f == 0);
  const int NF = a.NF;

  float4 acc[LT];
#pragma unroll
  for (int i = 0; i < LT; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);

  int t = t0 + kp;
  int q = t / K;
  int k = t - q * K;
#pragma unroll 2
  for (; t < t1; t += KP) {
    int slot = nk - k;
    if (slot < 0) slot += K;
    if (ELEM) {
#pragma unroll
      for (int i = 0; i < LT; ++i) {
        const float4 xv = a.X[((size_t)(l0 + i) * K + slot) * NF + f];
        const float4 h = ld_stream(a.H + ((size_t)(l0 + i) * T + t) * NF + f);
        cmac(acc[i], xpack(xv, dc), h, dc);
      }
    } else {
      const XPack x = xpack(a.X[((size_t)q * K + slot) * NF + f], dc);
      float4 h[LT];
#pragma unroll
      for (int i = 0; i < LT; ++i)
        h[i] = ld_stream(a.H + ((size_t)(l0 + i) * T + t) * NF + f);
#pragma unroll
      for (int i = 0; i < LT; ++i) cmac(acc[i], x, h[i], dc);
    }
    k += KP;
    while (k >= K) {
      k -= K;
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
    a.part_syn[((size_t)blockIdx.x * a.L + l0 + i) * NF + blockIdx.z * nft + c] = s;
  }
}

// -------------------------------------------------------- k_tail_synth
// One CTA per output channel l: fixed-order reduction of the split-K
// partials, c2r + overlap-save (convolver.hpp:202-205) straight into the
// output; for the auralizer also the canceller's stage 1 on l_n
// (convolver.hpp:180-191 on fc_) and the packed power |X_l|^2.
__global__ void __launch_bounds__(kTailThreads) k_tail_synth(BlockArgs a) {
  extern __shared__ float4 sm4[];
  const int N = a.N, NF = a.NF;
  float4* red = sm4;                                        // blockDim
  float4* acc = red + blockDim.x;                           // NF
  float2* z = reinterpret_cast<float2*>(acc + NF);          // N
  float* win = reinterpret_cast<float*>(z + N);             // 2N
  const int l = blockIdx.x;
  const uint32_t n = a.st->block;

  reduce_partials(a.part_syn + (size_t)l * NF, a.syn_chunks, (size_t)a.L * NF,
                  NF, red, acc);
  float* out = a.out + (size_t)l * N;
  float* tailw = win + N;
  irfft_packed_tail(reinterpret_cast<const float2*>(acc), z, N, a.logN, a.tw,
                    a.split, [&](int i, float v) {
                      out[i] = v;
                      tailw[i] = v;
                    });
  if (!a.is_aur) {
    retire_block(a, n);
    return;
  }
  float* prev = a.prev_spk + (size_t)l * N;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    win[i] = prev[i];
    prev[i] = tailw[i];
  }
  __syncthreads();
  float2* xnew = reinterpret_cast<float2*>(
      a.XA + ((size_t)l * (a.KF + 1) + (n % (uint32_t)(a.KF + 1))) * NF);
  float2* xs = reinterpret_cast<float2*>(acc);  // reuse: spectrum in smem
  rfft_packed(win, z, xs, N, a.logN, a.tw, a.split);
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    const float2 v = xs[j];
    xnew[j] = v;
    if (a.nlms) {
      float2 p;
      if (j == 0) p = make_float2(v.x * v.x, v.y * v.y);
      else {
        const float m = v.x * v.x + v.y * v.y;
        p = make_float2(m, m);
      }
      a.pw_part[(size_t)l * N + j] = p;
    }
  }
  __threadfence_system();
}

// ----------------------------------------------------------- k_mac_afc
// Canceller MAC over units u = (l, k), all P mics per unit (X_l shared):
//   NLMS (Appendix A step 2): W += mu/(P+delta) * conj(X_l(pre-push age k)) E_p
//   filter (step 4):          Yhat_p += W * X_l(post-push age k)
// Pre-push age k is post-push age k+1: the canceller FDL keeps KF+1 slots.
// grid = (afc_chunks, 1, afc_tiles), 256 threads.
template <int PT>
__global__ void __launch_bounds__(kMacThreads, 2) k_mac_afc(BlockArgs a) {
  __shared__ float4 red[kMacThreads * PT];
  const int nft = a.afc_nft;
  const int KP = kMacThreads / nft;
  const int fl = threadIdx.x & (nft - 1);
  const int kp = threadIdx.x / nft;
  const int f = blockIdx.z * nft + fl;
  const int NF = a.NF, KF = a.KF, L = a.L, P = a.P;
  const int cap = KF + 1;
  const int U = L * KF;
  const int u0 = blockIdx.x * a.afc_uc;
  const int u1 = min(u0 + a.afc_uc, U);
  const int nk = (int)(a.st->block % (uint32_t)cap);
  const bool dc = (f == 0);

  float4 acc[PT];
  float4 e[PT];
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int p = 0; p < PT; ++p) {
    acc[p] = make_float4(0.f, 0.f, 0.f, 0.f);
    e[p] = (a.nlms && p < P) ? a.E[(size_t)p * NF + f] : acc[p];
  }
  if (a.nlms) {
    const float2 p0 = a.pw[2 * f], p1 = a.pw[2 * f + 1];
    s = make_float4(a.mu / (p0.x + a.delta), a.mu / (p0.y + a.delta),
                    a.mu / (p1.x + a.delta), a.mu / (p1.y + a.delta));
  }

  int u = u0 + kp;
  int l = u / KF;
  int k = u - l * KF;
  for (; u < u1; u += KP) {
    const float4* xl = a.XA + (size_t)l * cap * NF;
    const XPack x0 = xpack(xl[(size_t)ring(nk - k, cap) * NF + f], dc);
    float4 x1 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (a.nlms) x1 = xl[(size_t)ring(nk - k - 1, cap) * NF + f];
#pragma unroll
    for (int p = 0; p < PT; ++p) {
      if (p >= P) break;
      float4* wp = a.W + (((size_t)p * L + l) * KF + k) * NF + f;
      float4 w = *wp;
      if (a.nlms) {
        // g = conj(x1) * E_p ; packed bin 0 is (DC, Nyquist) real products
        float4 g;
        if (dc) {
          g.x = x1.x * e[p].x;
          g.y = x1.y * e[p].y;
        } else {
          g.x = x1.x * e[p].x + x1.y * e[p].y;
          g.y = x1.x * e[p].y - x1.y * e[p].x;
        }
        g.z = x1.z * e[p].z + x1.w * e[p].w;
        g.w = x1.z * e[p].w - x1.w * e[p].z;
        w.x = fmaf(s.x, g.x, w.x);
        w.y = fmaf(s.y, g.y, w.y);
        w.z = fmaf(s.z, g.z, w.z);
        w.w = fmaf(s.w, g.w, w.w);
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
  for (int p = 0; p < PT; ++p) red[(kp * PT + p) * nft + fl] = acc[p];
  __syncthreads();
  for (int e2 = threadIdx.x; e2 < P * nft; e2 += kMacThreads) {
    const int p = e2 / nft, c = e2 - p * nft;
    float4 t = red[p * nft + c];
    for (int r = 1; r < KP; ++r) t = f4add(t, red[(r * PT + p) * nft + c]);
    a.part_afc[((size_t)blockIdx.x * P + p) * NF + blockIdx.z * nft + c] = t;
  }
}

// ---------------------------------------------------------- k_tail_afc
// One CTA per mic p: fixed-order reduce over chunks (the sum over l and k is
// done in the frequency domain -- one c2r per mic instead of the
// reference's L, auralizer.hpp:81-86), c2r -> f^_p for the next block.
// CTA 0 also advances the NLMS power (Appendix A step 5).
__global__ void __launch_bounds__(kTailThreads) k_tail_afc(BlockArgs a) {
  extern __shared__ float4 sm4[];
  const int N = a.N, NF = a.NF;
  float4* red = sm4;
  float4* acc = red + blockDim.x;
  float2* z = reinterpret_cast<float2*>(acc + NF);
  const int p = blockIdx.x;
  const uint32_t n = a.st->block;
  reduce_partials(a.part_afc + (size_t)p * NF, a.afc_chunks, (size_t)a.P * NF,
                  NF, red, acc);
  float* fh = a.fhat + (size_t)p * N;
  irfft_packed_tail(reinterpret_cast<const float2*>(acc), z, N, a.logN, a.tw,
                    a.split, [&](int i, float v) { fh[i] = v; });
  if (a.nlms && p == 0) {
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
      float2 sum = make_float2(0.f, 0.f);
      for (int ll = 0; ll < a.L; ++ll) {
        const float2 v = a.pw_part[(size_t)ll * N + j];
        sum.x += v.x;
        sum.y += v.y;
      }
      float2 w = a.pw[j];
      w.x = a.lambda * w.x + (1.0f - a.lambda) * sum.x;
      w.y = a.lambda * w.y + (1.0f - a.lambda) * sum.y;
      a.pw[j] = w;
    }
  }
  retire_block(a, n);
}

// ------------------------------------------------------ k_partition
// Setup (make_partitioned_filters, convolver.hpp:19-46) on the GPU: CTA
// (k, r) transforms taps[r][kN .. kN+N) zero-padded to 2N into the packed
// spectrum dst + row_off[r] + k*NF. taps rows are n_h long.
__global__ void __launch_bounds__(256) k_partition(
    const float* __restrict__ taps, size_t n_h, int rows, int K, int N,
    int logN, const float2* tw, const float2* split, float4* dst,
    const size_t* __restrict__ row_off) {
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
