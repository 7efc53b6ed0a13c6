// fft.cuh -- block-level real FFTs for the UPOLS block loop (sm_100a).
//
// The reference computes an n_f-point real transform as an n_f/2-point
// complex radix-2 FFT of the even/odd-interleaved samples plus a split step
// (dft.hpp:69-101 forward, dft.hpp:124-153 inverse; forward unnormalised,
// inverse scaled by 1/n_f). We compute the same transforms, but:
//   * spectra are PACKED: N = n_f/2 complex values, bin 0 holds DC in .x and
//     Nyquist in .y (both are exactly real), so every partition is exactly
//     8N bytes and 16-byte aligned for the streaming MAC;
//   * the complex FFT runs in shared memory with all threads of the CTA,
//     twiddles come from per-engine tables computed in double on the host.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace aura_b200 {

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
  return make_float2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
  return make_float2(a.x - b.x, a.y - b.y);
}

// In-place radix-2 DIT FFT of size M (power of two) on shared memory z that
// already holds its input in bit-reversed order. tw[j] = e^{-2 pi i j / M},
// j < M/2. INV selects the conjugate twiddles (unscaled inverse).
template <bool INV>
__device__ void fft_dit_smem(float2* z, int M, const float2* __restrict__ tw) {
  for (int len = 2; len <= M; len <<= 1) {
    const int h = len >> 1;
    const int stride = M / len;
    for (int b = threadIdx.x; b < (M >> 1); b += blockDim.x) {
      const int pos = b & (h - 1);
      const int i0 = ((b - pos) << 1) + pos;  // group*len + pos
      const int i1 = i0 + h;
      float2 w = __ldg(&tw[pos * stride]);
      if (INV) w.y = -w.y;
      const float2 u = z[i0];
      const float2 v = cmul(z[i1], w);
      z[i0] = cadd(u, v);
      z[i1] = csub(u, v);
    }
    __syncthreads();
  }
}

__device__ __forceinline__ int bitrev(int m, int logM) {
  return (int)(__brev((unsigned)m) >> (32 - logM));
}

// r2c of the 2N-sample real window `win` (shared) into the packed spectrum
// `spec` (N complex, any address space the caller can write). z: N float2 of
// shared scratch. split[k] = e^{-i pi k / N}, k < N. Ends with a barrier.
__device__ void rfft_packed(const float* win, float2* z, float2* spec, int N,
                            int logN, const float2* __restrict__ tw,
                            const float2* __restrict__ split) {
  for (int m = threadIdx.x; m < N; m += blockDim.x)
    z[bitrev(m, logN)] = make_float2(win[2 * m], win[2 * m + 1]);
  __syncthreads();
  fft_dit_smem<false>(z, N, tw);
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const float2 a = z[k];
    if (k == 0) {
      spec[0] = make_float2(a.x + a.y, a.x - a.y);
      continue;
    }
    const float2 zb = z[N - k];
    const float2 b = make_float2(zb.x, -zb.y);  // conj(Z[N-k])
    const float2 even = make_float2(0.5f * (a.x + b.x), 0.5f * (a.y + b.y));
    // odd = (a - b) / (2i)
    const float2 odd = make_float2(0.5f * (a.y - b.y), -0.5f * (a.x - b.x));
    const float2 rot = cmul(__ldg(&split[k]), odd);
    spec[k] = cadd(even, rot);
  }
  __syncthreads();
}

// c2r of packed spectrum `spec` (shared or global, N complex) into the LAST
// N samples of the 2N-point inverse (overlap-save keeps only those,
// convolver.hpp:202-205), scaled by 1/(2N). out[i] = x[N + i].
// z: N float2 of shared scratch. Ends with a barrier.
template <typename Store>
__device__ void irfft_packed_tail(const float2* spec, float2* z, int N,
                                  int logN, const float2* __restrict__ tw,
                                  const float2* __restrict__ split,
                                  Store store) {
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    float2 zk;
    if (k == 0) {
      const float2 s = spec[0];  // (DC, Nyquist)
      zk = make_float2(0.5f * (s.x + s.y), 0.5f * (s.x - s.y));
    } else {
      const float2 a = spec[k];
      const float2 sb = spec[N - k];
      const float2 b = make_float2(sb.x, -sb.y);
      const float2 A = make_float2(0.5f * (a.x + b.x), 0.5f * (a.y + b.y));
      const float2 D = make_float2(0.5f * (a.x - b.x), 0.5f * (a.y - b.y));
      const float2 w = __ldg(&split[k]);
      const float2 B = cmul(make_float2(w.x, -w.y), D);  // e^{+i pi k/N} D
      zk = make_float2(A.x - B.y, A.y + B.x);           // A + iB
    }
    z[bitrev(k, logN)] = zk;
  }
  __syncthreads();
  fft_dit_smem<true>(z, N, tw);
  const float scale = 1.0f / (float)N;
  // samples N .. 2N-1 are z[m] for m in [N/2, N)
  for (int m = threadIdx.x; m < (N >> 1); m += blockDim.x) {
    const float2 v = z[(N >> 1) + m];
    store(2 * m, v.x * scale);
    store(2 * m + 1, v.y * scale);
  }
  __syncthreads();
}

}  // namespace aura_b200
