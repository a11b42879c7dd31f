// Dependent-chain latency of the instructions the PSN kernels lean on, on
// sm_100a: one warp per SM walks a chain of N dependent ops; cycles/op = latency.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbl microbench_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

#define N 4096

template <int OP>
__global__ void lat(float* out, long long* cyc, float seed) {
  __shared__ float sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = (float)((i * 7 + 1) & 1023);
  __syncthreads();
  double d = seed + threadIdx.x;
  float f = seed * 0.5f + threadIdx.x;
  unsigned u = threadIdx.x;
  long long t0 = clock64();
#pragma unroll 16
  for (int it = 0; it < N; ++it) {
    if (OP == 0) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d) : "d"(1.0000001), "d"(1e-9));
    if (OP == 1) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d) : "d"(1e-9));
    if (OP == 2) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(f) : "f"(1.0000001f), "f"(1e-9f));
    if (OP == 3) { asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(f)); asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f) : "d"(d)); }
    if (OP == 4) { float v; asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"((unsigned)__cvta_generic_to_shared(sm) + (u & 1023) * 4)); u = (unsigned)v; }
    if (OP == 5) asm volatile("rcp.approx.ftz.f64 %0, %0;" : "+d"(d));
    if (OP == 6) asm volatile("rcp.approx.ftz.f32 %0, %0;" : "+f"(f));
    if (OP == 7) { double t; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(t) : "f"(f)); asm volatile("add.rn.f64 %0, %1, %1;" : "=d"(d) : "d"(t)); asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f) : "d"(d)); }
    if (OP == 8) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(u) : "r"(3u), "r"(1u));
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)d + f + (float)u;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float* out; long long* cyc; long long h;
  cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8);
  const char* names[] = {"DFMA", "DADD", "FFMA", "F2F f32->f64->f32 (2 ops)", "LDS (addr dep)", "MUFU.RCP64H", "MUFU.RCP", "F2F->DADD->F2F (3 ops)", "IMAD"};
  for (int op = 0; op < 9; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      switch (op) {
        case 0: lat<0><<<1, 32>>>(out, cyc, 1.f); break;
        case 1: lat<1><<<1, 32>>>(out, cyc, 1.f); break;
        case 2: lat<2><<<1, 32>>>(out, cyc, 1.f); break;
        case 3: lat<3><<<1, 32>>>(out, cyc, 1.f); break;
        case 4: lat<4><<<1, 32>>>(out, cyc, 1.f); break;
        case 5: lat<5><<<1, 32>>>(out, cyc, 1.f); break;
        case 6: lat<6><<<1, 32>>>(out, cyc, 1.f); break;
        case 7: lat<7><<<1, 32>>>(out, cyc, 1.f); break;
        case 8: lat<8><<<1, 32>>>(out, cyc, 1.f); break;
      }
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("%-28s %6.1f cycles per chain step\n", names[op], (double)h / N);
  }
  return 0;
}
