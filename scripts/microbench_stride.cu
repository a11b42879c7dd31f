// HBM read throughput of a time-major [R = T*N rows, C] f32 tensor read as
// channel groups of W columns (W*4-byte runs per row), group after group --
// the access pattern of a channel-grouped two-pass kernel.  Two readers:
//   LDG: 8 warps per CTA, float4 per lane, 8 loads in flight per thread;
//   TMA: one producer lane, S-stage ring of 2-D boxes [W cols x BR rows].
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbs microbench_stride.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__global__ void ldg_groups(const float4* __restrict__ x, int R, int C4, int W4, float* out) {
  // global thread id walks (group, row, col4) in row-major order within a group
  const long long per_group = (long long)R * W4;
  const long long total = per_group * (C4 / W4);
  float acc = 0.f;
  const long long nthr = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 7 * nthr < total; i += 8 * nthr) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const long long e = i + u * nthr;
      const long long g = e / per_group, rem = e % per_group;
      const long long r = rem / W4, c = g * W4 + rem % W4;
      v[u] = __ldg(x + r * C4 + c);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 123.456f) out[0] = acc;
}

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(288, 1) tma_groups(const __grid_constant__ CUtensorMap map, int R, int C, int W,
                                                     int BR, int S, int stage_bytes, float* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = (uint64_t*)(sm + S * stage_bytes);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(full + s)), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(empty + s)), "r"(8));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int groups = C / W, rb = (R + BR - 1) / BR;
  const long long ntiles = (long long)groups * rb;
  // contiguous ranges of tiles per CTA *within each group* (like the PSN kernel)
  int q = 0;
  float acc = 0.f;
  for (int g = 0; g < groups; ++g) {
    const int a = (int)((long long)blockIdx.x * rb / gridDim.x), b = (int)((long long)(blockIdx.x + 1) * rb / gridDim.x);
    for (int t = a; t < b; ++t, ++q) {
      const int s = q % S;
      if (warp == 8) {
        if (lane == 0) {
          if (q >= S) {
            unsigned ok = 0;
            while (!ok)
              asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                           : "=r"(ok) : "r"(su32(empty + s)), "r"(((q / S) - 1) & 1) : "memory");
          }
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)),
                       "r"(W * BR * 4) : "memory");
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                       ::"r"(su32(sm + s * stage_bytes)), "l"((unsigned long long)&map), "r"(g * W), "r"(t * BR),
                       "r"(su32(full + s)) : "memory");
        }
      } else {
        unsigned ok = 0;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(su32(full + s)), "r"((q / S) & 1) : "memory");
        acc += ((float*)(sm + s * stage_bytes))[threadIdx.x];
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(empty + s)) : "memory");
      }
    }
  }
  if (acc == 123.456f) out[0] = acc;
}

__global__ void __launch_bounds__(288, 1) tma3_groups(const __grid_constant__ CUtensorMap map, int T, int N, int C,
                                                      int BT, int S, int stage_bytes, int twopass, int lag,
                                                      float* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = (uint64_t*)(sm + S * stage_bytes);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(full + s)), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(empty + s)), "r"(8));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint64_t pol_keep, pol_drop;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_keep));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_drop));
  const int G = C / 32, nbk = N / 8, ttl = T / BT, tpg = nbk * ttl;
  const int P = tpg < (int)gridDim.x ? tpg : gridDim.x;
  int q = 0;
  float acc = 0.f;
  const int iters = twopass ? G + lag : G;
  for (int it = 0; it < iters; ++it) {
    for (int pass = 0; pass < (twopass ? 2 : 1); ++pass) {
      const int g = pass == 0 ? it : it - lag;
      if (g < 0 || g >= G) continue;
      const int rot = (g * 61 + pass * 29) % gridDim.x;
      const int v = ((int)blockIdx.x - rot + gridDim.x) % gridDim.x;
      if (v >= P) continue;
      const int a = (int)((long long)v * tpg / P), b = (int)((long long)(v + 1) * tpg / P);
      for (int t = a; t < b; ++t, ++q) {
        const int s = q % S;
        const int nbi = t / ttl, tt = t % ttl;
        if (warp == 8) {
          if (lane == 0) {
            if (q >= S) {
              unsigned ok = 0;
              while (!ok)
                asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                             : "=r"(ok) : "r"(su32(empty + s)), "r"(((q / S) - 1) & 1) : "memory");
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(full + s)),
                         "r"(32 * 8 * BT * 4) : "memory");
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;"
                         ::"r"(su32(sm + s * stage_bytes)), "l"((unsigned long long)&map), "r"(g * 32), "r"(nbi * 8),
                         "r"(tt * BT), "r"(su32(full + s)), "l"(pass == 0 ? pol_keep : pol_drop) : "memory");
          }
        } else {
          unsigned ok = 0;
          while (!ok)
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                         : "=r"(ok) : "r"(su32(full + s)), "r"((q / S) & 1) : "memory");
          acc += ((float*)(sm + s * stage_bytes))[threadIdx.x];
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(empty + s)) : "memory");
        }
      }
    }
  }
  if (acc == 123.456f) out[0] = acc;
}

int main() {
  const int T = 1024, N = 64, C = 512, R = T * N;
  float* x; float* out;
  cudaMalloc(&x, (size_t)R * C * 4); cudaMalloc(&out, 64);
  cudaMemset(x, 0, (size_t)R * C * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const double bytes = (double)R * C * 4;
  // flush buffer > L2
  char* fl; cudaMalloc(&fl, 256 << 20);
  int Ws[] = {32, 64, 128, 256, 512};
  for (int W : Ws) {
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(e0);
      ldg_groups<<<sms * 4, 256>>>((const float4*)x, R, C / 4, W / 4, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("LDG  W=%4d (%5d B runs): %8.1f GB/s\n", W, W * 4, bytes / (best * 1e-3) / 1e9);
  }
  PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
  int Wt[] = {32, 64, 128, 256};
  for (int W : Wt) {
    for (int S : {4, 6}) {
      const int stage = 32768, BR = stage / (W * 4);
      if (BR > 256) continue;
      CUtensorMap map;
      cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R}, strides[1] = {(cuuint64_t)C * 4};
      cuuint32_t box[2] = {(cuuint32_t)W, (cuuint32_t)BR}, es[2] = {1, 1};
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r) { printf("encode failed %d\n", r); continue; }
      const int smem = S * stage + 1024;
      cudaFuncSetAttribute(tma_groups, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      float best = 1e9;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        tma_groups<<<sms, 288, smem>>>(map, R, C, W, BR, S, stage, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      cudaError_t e = cudaGetLastError();
      printf("TMA  W=%4d (%5d B runs) box rows %3d S=%d: %8.1f GB/s %s\n", W, W * 4, BR, S, bytes / (best * 1e-3) / 1e9,
             e ? cudaGetErrorString(e) : "");
    }
  }

  // 3-D boxes [32 cols][8 batch][BT time] over [C, N, T]: the PSN stream kernel's pattern
  for (int twopass = 0; twopass < 2; ++twopass)
    for (int BT : {16, 32, 64}) {
      const int S = BT == 64 ? 3 : 6, stage = 32 * 8 * BT * 4;
      CUtensorMap map;
      cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)N, (cuuint64_t)T};
      cuuint64_t strides[2] = {(cuuint64_t)C * 4, (cuuint64_t)C * N * 4};
      cuuint32_t box[3] = {32, 8, (cuuint32_t)BT}, es[3] = {1, 1, 1};
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r) { printf("encode3 failed %d\n", r); continue; }
      const int smem = S * stage + 1024;
      cudaFuncSetAttribute(tma3_groups, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      float best = 1e9;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        tma3_groups<<<sms, 288, smem>>>(map, T, N, C, BT, S, stage, twopass, 2, out);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      cudaError_t e = cudaGetLastError();
      printf("TMA3 box [32,8,%2d] S=%d %s: %7.1f us, %8.1f GB/s of HBM-algorithmic reads %s\n", BT, S,
             twopass ? "two-pass lag2" : "one pass     ", best * 1e3, bytes / (best * 1e-3) / 1e9, e ? cudaGetErrorString(e) : "");
    }
  return 0;
}
