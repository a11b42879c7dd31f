// Compute rate of the backward pass-1 row loop in isolation (data in shared
// memory): exact f64 h2 (f32-rounded), f64 arctan surrogate, f64 db / dw_q
// sums, f32 BN-term sums.  Variants: streams per thread S, row block U, warps.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbb microbench_bwd1.cu
#include <cstdio>
#include <cuda_runtime.h>
#define K 4
#define ROWS 8
__device__ __forceinline__ double round_f32(double h) {
  unsigned ex = (unsigned)__double2hiint(h) & 0x7ff00000u;
  ex = ex < 0x38100000u ? 0x38100000u : ex;
  const double M = __hiloint2double((int)(ex + (29u << 20) + 0x00080000u), 0);
  return __dsub_rn(__dadd_rn(h, M), M);
}
__device__ __forceinline__ double rcp_f64(double v) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v));
  const double e = fma(-v, r, 1.0);
  return fma(r, e, r);
}
template <int U, int S, int MODE>
__global__ void bwd1(int reps, double* out) {
  __shared__ float xs[ROWS * 16 * 32], ys[ROWS * 16 * 32];
  for (int i = threadIdx.x; i < ROWS * 16 * 32; i += blockDim.x) {
    xs[i] = (float)((i * 37) % 101) * 0.01f - 0.5f;
    ys[i] = (float)((i * 53) % 97) * 0.01f - 0.5f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) & 7;
  const double wq[K] = {0.25, -0.125, 0.5, 1.0}, bf = -0.3, sc = 3.14159;
  const float w[K] = {0.3f, -0.2f, 0.7f, 0.11f}, mu = 0.01f;
  double acc[1 + K] = {0, 0, 0, 0, 0};
  float fsx[K] = {0, 0, 0, 0}, fsc[K] = {0, 0, 0, 0};
  for (int rep = 0; rep < reps; ++rep) {
    double xd[S][K - 1 + U];
    float xf[S][K - 1 + U];
#pragma unroll
    for (int s = 0; s < S; ++s)
#pragma unroll
      for (int j = 0; j < K - 1 + U; ++j) { xd[s][j] = 0.0; xf[s][j] = 0.f; }
#pragma unroll 1
    for (int r0 = 0; r0 < ROWS; r0 += U) {
      double yv[S][U];
#pragma unroll
      for (int s = 0; s < S; ++s)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          float v, y;
          const unsigned off = ((r0 + u) * 16 + warp + 8 * s) * 32 + lane;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"((unsigned)__cvta_generic_to_shared(xs + off)));
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(y) : "r"((unsigned)__cvta_generic_to_shared(ys + off)));
          xf[s][K - 1 + u] = v;
          xd[s][K - 1 + u] = (double)v;
          yv[s][u] = (double)y;
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int s = 0; s < S; ++s) {
          double h = wq[0] * xd[s][u];
#pragma unroll
          for (int i = 1; i < K; ++i) h = fma(wq[i], xd[s][u + i], h);
          double dh;
          if (MODE == 0) {
            h = round_f32(__dadd_rn(h, bf));
            const double q = sc * h;
            dh = yv[s][u] * rcp_f64(fma(q, q, 1.0));
          } else {  // f32 surrogate (precision-insufficient variant, for the cost comparison)
            const float hf = (float)__dadd_rn(h, bf);
            const float q = 3.14159f * hf;
            dh = yv[s][u] * (double)__fdividef(1.f, fmaf(q, q, 1.f));
          }
          acc[0] += dh;
#pragma unroll
          for (int i = 0; i < K; ++i) acc[1 + i] = fma(xd[s][u + i], dh, acc[1 + i]);
          float h1 = w[0] * xf[s][u];
#pragma unroll
          for (int i = 1; i < K; ++i) h1 = fmaf(w[i], xf[s][u + i], h1);
          const float hc = h1 - mu;
#pragma unroll
          for (int i = 0; i < K; ++i) {
            fsx[i] += xf[s][u + i];
            fsc[i] = fmaf(xf[s][u + i], hc, fsc[i]);
          }
        }
#pragma unroll
      for (int s = 0; s < S; ++s)
#pragma unroll
        for (int j = 0; j < K - 1; ++j) { xd[s][j] = xd[s][j + U]; xf[s][j] = xf[s][j + U]; }
    }
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i <= K; ++i) t += acc[i];
#pragma unroll
  for (int i = 0; i < K; ++i) t += fsx[i] + fsc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int U, int S, int MODE>
void run(int sms, int warps, double* out) {
  const int reps = 400;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(a); bwd1<U, S, MODE><<<sms, warps * 32>>>(reps, out); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  const double el = (double)sms * warps * 32 * S * ROWS * reps;
  printf("bwd1 U=%d streams=%d warps=%2d %s: %7.1f Gel/s -> %6.1f us per 33.5M elements\n", U, S, warps,
         MODE ? "f32 sur " : "f64 sur ", el / (best * 1e-3) / 1e9, 33554432.0 / (el / (best * 1e-3)) * 1e6);
}
int main() {
  double* out; cudaMalloc(&out, 1 << 24);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<2, 1, 0>(sms, 8, out); run<4, 1, 0>(sms, 8, out); run<2, 2, 0>(sms, 8, out); run<4, 2, 0>(sms, 8, out);
  run<2, 1, 0>(sms, 16, out); run<2, 2, 0>(sms, 16, out); run<4, 1, 0>(sms, 16, out);
  run<2, 1, 1>(sms, 8, out); run<2, 2, 1>(sms, 16, out);
  return 0;
}
