// FP64 FMA throughput vs resident warps per SM (one CTA per SM, CH independent
// chains per thread): is 2 warps/SMSP enough to keep the FP64 pipe busy?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbo microbench_fp64_occ.cu
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048
template <int CH>
__global__ void k(double* out, double seed) {
  double d[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c] = seed + c + threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[c]) : "d"(1.0000001), "d"(1e-9));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int CH>
void run(int sms, int threads, double* out) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a); k<CH><<<sms, threads>>>(out, 1.0); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  double ops = (double)sms * threads * ITERS * CH;
  printf("warps/SM %3d chains %2d: %6.1f DFMA/clk/SM (1.965 GHz)\n", threads / 32, CH, ops / (best * 1e-3) / sms / 1.965e9);
}
int main() {
  double* out; cudaMalloc(&out, 1 << 24);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int t : {128, 256, 512, 1024}) { run<4>(sms, t, out); run<8>(sms, t, out); run<16>(sms, t, out); }
  return 0;
}
