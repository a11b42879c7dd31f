// Throughput microbenchmark of the arithmetic pipes the PSN kernels lean on
// (f64 add/mul/fma, f32<->f64 conversions, f32 fma, int add) on sm_100a.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CHAINS 8
#define ITERS 4096

template <int OP>
__global__ void kern(float* out, float seed) {
  double d[CHAINS];
  float f[CHAINS];
  int i32[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) {
    d[c] = seed + c + threadIdx.x;
    f[c] = seed * c + threadIdx.x;
    i32[c] = threadIdx.x + c;
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (OP == 0) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[c]) : "d"(1.0000001));
      if (OP == 1) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(d[c]) : "d"(1.0000001));
      if (OP == 2) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d[c]) : "d"(1.0000001), "d"(0.5));
      if (OP == 3) { double t; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(f[c])); asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f[c]) : "d"(t)); }
      if (OP == 4) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f[c]) : "f"(1.0000001f), "f"(0.5f));
      if (OP == 5) asm volatile("add.s32 %0, %0, %1;" : "+r"(i32[c]) : "r"(7));
      if (OP == 6) { double t; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(f[c])); asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[c]) : "d"(t)); }
    }
  }
  double s = 0; float sf = 0; int si = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { s += d[c]; sf += f[c]; si += i32[c]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s + sf + (float)si;
}

int main() {
  float* out;
  cudaMalloc(&out, 64 << 20);
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  const char* names[] = {"DADD", "DMUL", "DFMA", "F2F f32->f64->f32 (2 cvt)", "FFMA", "IADD", "F2F f32->f64 + DADD"};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  for (int op = 0; op < 7; ++op) {
    int blocks = sms * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      switch (op) {
        case 0: kern<0><<<blocks, threads>>>(out, 1.f); break;
        case 1: kern<1><<<blocks, threads>>>(out, 1.f); break;
        case 2: kern<2><<<blocks, threads>>>(out, 1.f); break;
        case 3: kern<3><<<blocks, threads>>>(out, 1.f); break;
        case 4: kern<4><<<blocks, threads>>>(out, 1.f); break;
        case 5: kern<5><<<blocks, threads>>>(out, 1.f); break;
        case 6: kern<6><<<blocks, threads>>>(out, 1.f); break;
      }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      double ops = (double)blocks * threads * ITERS * CHAINS;
      if (rep == 1)
        printf("%-28s %8.3f ms  %8.2f Gop/s  %6.1f op/clk/SM (at %d MHz nominal)\n", names[op], ms,
               ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk_khz * 1e3), clk_khz / 1000);
    }
  }
  return 0;
}
