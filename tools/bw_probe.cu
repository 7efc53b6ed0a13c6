// bw_probe.cu -- read-bandwidth probe for the streaming MAC's memory path on
// one B200: (a) plain 128-bit loads, (b) a cp.async.bulk + mbarrier ring
// with one producer lane and 8 consumer warps (the k_back structure), over
// stage sizes, ring depths and CTAs per SM. Prints one JSON line per case.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_bw_probe tools/bw_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("err %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// L2-resident read: the same `n` float4 every launch, cached at L2 (.cg)
__global__ void k_ldg_l2(const float4* __restrict__ p, size_t n, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    float4 a = __ldcg(p + i), b = __ldcg(p + i + stride), c = __ldcg(p + i + 2 * stride), d = __ldcg(p + i + 3 * stride);
    acc.x += a.x + b.x + c.x + d.x; acc.y += a.y + b.y + c.y + d.y;
    acc.z += a.z + b.z + c.z + d.z; acc.w += a.w + b.w + c.w + d.w;
  }
  for (; i < n; i += stride) { float4 a = __ldcg(p + i); acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w; }
  if (acc.x == 123.f) out[0] = acc.y + acc.z + acc.w;
}

__global__ void k_ldg(const float4* __restrict__ p, size_t n, float* out) {
  float4 acc = make_float4(0, 0, 0, 0);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    float4 a = __ldcs(p + i), b = __ldcs(p + i + stride), c = __ldcs(p + i + 2 * stride), d = __ldcs(p + i + 3 * stride);
    acc.x += a.x + b.x + c.x + d.x; acc.y += a.y + b.y + c.y + d.y;
    acc.z += a.z + b.z + c.z + d.z; acc.w += a.w + b.w + c.w + d.w;
  }
  for (; i < n; i += stride) { float4 a = __ldcs(p + i); acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w; }
  if (acc.x == 123.f) out[0] = acc.y + acc.z + acc.w;
}

// each CTA streams a contiguous range [cta*per, (cta+1)*per) bytes in stage-sized copies
__global__ void __launch_bounds__(288) k_bulk(const char* __restrict__ src, size_t per, int stage, int S,
                                              int copies, float* out, int l2_normal = 0) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm;
  uint64_t* empty = full + 16;
  float4* slots = (float4*)(sm + 256);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(full + s)), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(empty + s)), "r"(8));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const char* base = src + (size_t)blockIdx.x * per;
  const int nst = (int)(per / stage);
  if (warp == 8) {
    if (lane != 0) return;
    uint64_t pol;
    if (l2_normal) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    else asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int q = 0; q < nst; ++q) {
      const int s = q % S;
      const uint32_t par = ((q / S) & 1) ^ 1;
      asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(empty + s)), "r"(par) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)), "r"(stage) : "memory");
      const int cb = stage / copies;
      for (int c = 0; c < copies; ++c)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                     ::"r"(su32((char*)slots + (size_t)s * stage + c * cb)), "l"(base + (size_t)q * stage + c * cb), "r"(cb), "r"(su32(full + s)), "l"(pol) : "memory");
    }
    return;
  }
  float4 acc = make_float4(0, 0, 0, 0);
  for (int q = 0; q < nst; ++q) {
    const int s = q % S;
    const uint32_t par = (q / S) & 1;
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(full + s)), "r"(par) : "memory");
    const float4* v = (const float4*)((const char*)slots + (size_t)s * stage);
    for (int i = threadIdx.x; i < stage / 16; i += 256) { float4 a = v[i]; acc.x += a.x; acc.y += a.y; acc.z += a.z; acc.w += a.w; }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(empty + s)) : "memory");
  }
  if (acc.x == 123.f) out[0] = acc.y + acc.z + acc.w;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const size_t bytes = size_t(4) << 30;  // 4 GiB (>> L2)
  char* buf;
  float* out;
  CK(cudaMalloc(&buf, bytes));
  CK(cudaMalloc(&out, 16));
  CK(cudaMemset(buf, 1, bytes));
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  auto timeit = [&](auto launch, int reps) {
    launch();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(t0);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(t1);
    CK(cudaEventSynchronize(t1));
    float ms;
    cudaEventElapsedTime(&ms, t0, t1);
    return ms / reps;
  };
  if (getenv("BW_L2")) {  // L2-resident read bandwidth at a footprint (same bytes every launch)
    int l2 = 0;
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
    printf("{\"kind\": \"l2_size\", \"bytes\": %d}\n", l2);
    CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    for (double mb : {4.0, 8.0, 16.0, 24.0, 32.0, 48.0, 64.0, 80.0, 100.0, 126.0, 160.0, 256.0}) {
      const size_t fb = (size_t)(mb * 1e6) / 65536 * 65536;
      for (int per_sm : {2, 4}) {
        const int grid = sms * per_sm;
        float ms = timeit([&] { k_ldg_l2<<<grid, 512>>>((const float4*)buf, fb / 16, out); }, 50);
        printf("{\"kind\": \"l2_ldg\", \"footprint_mb\": %.1f, \"ctas\": %d, \"GBps\": %.1f, \"us\": %.2f}\n",
               fb / 1e6, grid, fb / ms / 1e6, ms * 1e3);
      }
      for (int stage : {16384, 32768}) {
        const int S = 4;
        const size_t smem = 256 + (size_t)S * stage;
        size_t per = fb / sms;
        per -= per % stage;
        if (per == 0) continue;
        float ms = timeit([&] { k_bulk<<<sms, 288, smem>>>(buf, per, stage, S, 1, out, 1); }, 50);
        printf("{\"kind\": \"l2_bulk\", \"footprint_mb\": %.1f, \"stage\": %d, \"GBps\": %.1f, \"us\": %.2f}\n",
               per * sms / 1e6, stage, (double)per * sms / ms / 1e6, ms * 1e3);
      }
    }
    return 0;
  }
  if (getenv("BW_PER_SM")) {  // per-SM ceiling: fewer CTAs than SMs
    CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    for (int grid : {16, 32, 64, 96, 148}) {
      for (int stage : {16384, 32768, 49152}) {
        for (int S : {3, 4, 6}) {
          const size_t smem = 256 + (size_t)S * stage;
          if (smem > 220 * 1024) continue;
          for (int copies : {1, 4}) {
            size_t per = bytes / 148;
            per -= per % stage;
            float ms = timeit([&] { k_bulk<<<grid, 288, smem>>>(buf, per, stage, S, copies, out); }, 5);
            printf("{\"kind\": \"bulk\", \"ctas\": %d, \"stage\": %d, \"stages\": %d, \"copies\": %d, \"GBps\": %.1f, \"per_sm\": %.1f}\n",
                   grid, stage, S, copies, (double)per * grid / ms / 1e6, (double)per / ms / 1e6);
          }
        }
      }
      for (int thr : {512, 1024}) {
        float ms = timeit([&] { k_ldg<<<grid, thr>>>((const float4*)buf, bytes / 16 / 148 * grid, out); }, 5);
        printf("{\"kind\": \"ldg128\", \"ctas\": %d, \"threads\": %d, \"per_sm\": %.1f}\n", grid, thr,
               (double)(bytes / 148) / ms / 1e6);
      }
    }
    return 0;
  }
  for (int per_sm : {2, 4, 8}) {
    const int grid = sms * per_sm;
    float ms = timeit([&] { k_ldg<<<grid, 512>>>((const float4*)buf, bytes / 16, out); }, 10);
    printf("{\"kind\": \"ldg128\", \"ctas\": %d, \"threads\": 512, \"GBps\": %.1f}\n", grid, bytes / ms / 1e6);
  }
  CK(cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  for (int cps : {1, 2}) {
    for (int stage : {8192, 16384, 32768, 65536}) {
      for (int S : {2, 3, 4, 6, 8}) {
        const size_t smem = 256 + (size_t)S * stage;
        if (smem * cps > 225 * 1024 || S > 16) continue;
        for (int copies : {1, 4}) {
          const int grid = sms * cps;
          size_t per = bytes / grid;
          per -= per % stage;
          float ms = timeit([&] { k_bulk<<<grid, 288, smem>>>(buf, per, stage, S, copies, out); }, 10);
          printf("{\"kind\": \"bulk\", \"ctas_per_sm\": %d, \"stage\": %d, \"stages\": %d, \"copies\": %d, \"GBps\": %.1f}\n",
                 cps, stage, S, copies, (double)per * grid / ms / 1e6);
        }
      }
    }
  }
  return 0;
}
