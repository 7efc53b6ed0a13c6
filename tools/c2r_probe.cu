// c2r_probe.cu -- time one warp's packed c2r / r2c (N = 64) inside a kernel
// with clock64(), cold and warm: the shared-memory warp transforms
// (irfft_packed_tail / rfft_packed with a Warp team) against the
// register-resident ones (irfft_packed_tail_reg / rfft_packed_reg).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2509_04390_b200/csrc -o tools/_c2r_probe tools/c2r_probe.cu
#include <cstdio>
#include <cmath>
#include <vector>
#include "fft.cuh"
using namespace aura_b200;

__global__ void k_probe(const float2* tw_g, const float2* split_g, float* out, long long* cyc, int N, int logN) {
  __shared__ float2 tw[64], split[65], spec[128], z[128];
  __shared__ float win[256];
  const Warp wt;
  const int lane = threadIdx.x & 31;
  for (int j = lane; j < N / 2; j += 32) tw[j] = tw_g[j];
  for (int j = lane; j <= N / 2; j += 32) split[j] = split_g[j];
  for (int j = lane; j < N; j += 32) spec[j] = make_float2(1.0f / (j + 1), 0.5f / (j + 2));
  for (int j = lane; j < 2 * N; j += 32) win[j] = 1.0f / (j + 3);
  __syncwarp();
  for (int rep = 0; rep < 3; ++rep) {
    long long t0 = clock64();
    irfft_packed_tail(spec, z, N, logN, tw, split, [&](int i, float v) { out[i] = v; }, wt);
    long long t1 = clock64();
    rfft_packed(win, z, spec, N, logN, tw, split, wt);
    long long t2 = clock64();
    long long t3 = clock64();
    irfft_packed_tail_reg<2>(spec, logN, tw, split, [&](int i, float v) { out[128 + i] = v; });
    long long t4 = clock64();
    rfft_packed_reg<2>(win, z, spec, logN, tw, split);
    long long t5 = clock64();
    if (lane == 0) {
      cyc[rep * 4] = t1 - t0;
      cyc[rep * 4 + 1] = t2 - t1;
      cyc[rep * 4 + 2] = t4 - t3;
      cyc[rep * 4 + 3] = t5 - t4;
    }
    __syncwarp();
  }
}

int main() {
  const int N = 64, logN = 6;
  std::vector<float2> tw(N / 2), split(N / 2 + 1);
  for (int j = 0; j < N / 2; ++j) tw[j] = make_float2((float)cos(-2 * M_PI * j / N), (float)sin(-2 * M_PI * j / N));
  for (int j = 0; j <= N / 2; ++j) split[j] = make_float2((float)cos(-M_PI * j / N), (float)sin(-M_PI * j / N));
  float2 *dtw, *dsp;
  float* dout;
  long long* dcyc;
  cudaMalloc(&dtw, sizeof(float2) * N / 2);
  cudaMalloc(&dsp, sizeof(float2) * (N / 2 + 1));
  cudaMalloc(&dout, sizeof(float) * 4 * N);
  cudaMalloc(&dcyc, sizeof(long long) * 12);
  cudaMemcpy(dtw, tw.data(), sizeof(float2) * N / 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dsp, split.data(), sizeof(float2) * (N / 2 + 1), cudaMemcpyHostToDevice);
  for (int launch = 0; launch < 2; ++launch) {
    k_probe<<<1, 32>>>(dtw, dsp, dout, dcyc, N, logN);
    cudaDeviceSynchronize();
    long long c[12];
    cudaMemcpy(c, dcyc, sizeof(c), cudaMemcpyDeviceToHost);
    printf("{\"launch\": %d, \"smem_c2r\": [%lld, %lld, %lld], \"smem_r2c\": [%lld, %lld, %lld], \"reg_c2r\": [%lld, %lld, %lld], \"reg_r2c\": [%lld, %lld, %lld]}\n",
           launch, c[0], c[4], c[8], c[1], c[5], c[9], c[2], c[6], c[10], c[3], c[7], c[11]);
  }
  return 0;
}
