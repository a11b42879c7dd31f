// Compute rate of the forward pass-1 row loop (h1 = f32(sum_i W_i x), shifted
// moments in f64) in isolation: data resident in shared memory, one CTA per SM,
// W warps, each thread walking S streams with row blocks of U.  Reports
// elements/s per GPU and the equivalent time for the metric tensor (33.5M elements).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbr microbench_rows.cu
#include <cstdio>
#include <cuda_runtime.h>
#define K 4
#define ROWS 16
__device__ __forceinline__ double round_f32(double h) {
  unsigned ex = (unsigned)__double2hiint(h) & 0x7ff00000u;
  ex = ex < 0x38100000u ? 0x38100000u : ex;
  const double M = __hiloint2double((int)(ex + (29u << 20) + 0x00080000u), 0);
  return __dsub_rn(__dadd_rn(h, M), M);
}
template <int U, int S, int MODE>
__global__ void rows_kernel(int reps, double* out) {
  __shared__ float xs[ROWS * 16 * 32];
  for (int i = threadIdx.x; i < ROWS * 16 * 32; i += blockDim.x) xs[i] = (float)((i * 37) % 101) * 0.01f - 0.5f;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) & 7;
  double w[K] = {0.3, -0.2, 0.7, 0.11}, sh = 0.01;
  double acc1 = 0, acc2 = 0;
  for (int rep = 0; rep < reps; ++rep) {
    double xw[S][K - 1 + U];
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
      for (int j = 0; j < K - 1 + U; ++j) xw[s][j] = 0.0;
    double S1[S], S2[S];
#pragma unroll
    for (int s = 0; s < S; ++s) S1[s] = S2[s] = 0.0;
#pragma unroll 1
    for (int r0 = 0; r0 < ROWS; r0 += U) {
#pragma unroll
      for (int s = 0; s < S; ++s)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float v;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"((unsigned)__cvta_generic_to_shared(xs + ((r0 + u) * 16 + warp + 8 * s) * 32 + lane)));
          xw[s][K - 1 + u] = (double)v;
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int s = 0; s < S; ++s) {
          double h = w[0] * xw[s][u];
#pragma unroll
          for (int i = 1; i < K; ++i) h = fma(w[i], xw[s][u + i], h);
          double hc;
          if (MODE == 0) hc = round_f32(h) - sh;
          else hc = h - sh;  // no rounding (bound on the round's cost)
          S1[s] += hc;
          S2[s] = fma(hc, hc, S2[s]);
        }
#pragma unroll
      for (int s = 0; s < S; ++s)
#pragma unroll
        for (int j = 0; j < K - 1; ++j) xw[s][j] = xw[s][j + U];
    }
#pragma unroll
    for (int s = 0; s < S; ++s) {
      acc1 += S1[s];
      acc2 += S2[s];
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc1 + acc2;
}
template <int U, int S, int MODE>
void run(int sms, int warps, double* out) {
  const int reps = 200;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a); rows_kernel<U, S, MODE><<<sms, warps * 32>>>(reps, out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  const double el = (double)sms * warps * 32 * S * ROWS * reps;
  printf("U=%d streams=%d warps=%2d %s: %7.1f Gel/s -> %6.1f us per 33.5M elements\n", U, S, warps,
         MODE ? "no-round" : "round   ", el / (best * 1e-3) / 1e9, 33554432.0 / (el / (best * 1e-3)) * 1e6);
}
int main() {
  double* out; cudaMalloc(&out, 1 << 24);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4, 1, 0>(sms, 8, out); run<8, 1, 0>(sms, 8, out); run<4, 2, 0>(sms, 8, out); run<8, 2, 0>(sms, 8, out);
  run<4, 1, 1>(sms, 8, out); run<4, 2, 1>(sms, 8, out);
  run<4, 1, 0>(sms, 16, out); run<4, 2, 0>(sms, 16, out); run<4, 1, 0>(sms, 32, out);
  return 0;
}
