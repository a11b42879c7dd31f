// psn_readout.cu — the readout's leaky accumulator (reference network.py:365-436)
// as a weighted time reduction on sm_100a.
//
// The reference runs v = (1 - inv) v + inv cur[t] over t with
// cur[t] = x[t] W^T + b, so the logits are
//     v_T = sum_t w_t cur[t],  w_t = inv (1 - inv)^(T-1-t),  inv = 1 / tau.
// The map x -> cur is linear, so the reduction runs on x first:
//     logits = xbar W^T + b sum_t w_t,   xbar[n, c] = sum_t w_t x[t, n, c]
// (psn_readout_reduce; the small xbar W^T product is a library GEMM), and the
// backward's dcur[t] = w_t dlogits gives
//     dx[t, n, c] = w_t (dlogits W)[n, c]
// (psn_readout_expand), a rank-one-in-time broadcast.  Both kernels stream the
// [T, N, C] tensor once (HBM-bound); one thread owns one (n, c) column, walks t
// from the newest step down (w_{T-1} = inv, w_{t-1} = (1 - inv) w_t) and
// accumulates in f64.  Deterministic: each column's sum has one fixed order.
#include "psn_common.cuh"

namespace psn {

int fail(int code, const char* msg);
int cuda_check(const char* where);

namespace {

constexpr int kRoThreads = 256;

template <typename IO>
__global__ void __launch_bounds__(kRoThreads) readout_reduce_kernel(int64_t T, int64_t cols, double inv,
                                                                    const IO* __restrict__ x,
                                                                    double* __restrict__ xbar) {
  const int64_t j = (int64_t)blockIdx.x * kRoThreads + threadIdx.x;
  if (j >= cols) return;
  const double keep = 1.0 - inv;
  double w = inv, acc = 0.0;
  const IO* p = x + (T - 1) * cols + j;
  int64_t t = T - 1;
  // 4 loads in flight per thread
  for (; t >= 3; t -= 4, p -= 4 * cols) {
    const double x0 = load_wide(p), x1 = load_wide(p - cols), x2 = load_wide(p - 2 * cols),
                 x3 = load_wide(p - 3 * cols);
    acc = fma(w, x0, acc);
    w *= keep;
    acc = fma(w, x1, acc);
    w *= keep;
    acc = fma(w, x2, acc);
    w *= keep;
    acc = fma(w, x3, acc);
    w *= keep;
  }
  for (; t >= 0; --t, p -= cols) {
    acc = fma(w, load_wide(p), acc);
    w *= keep;
  }
  xbar[j] = acc;
}

template <typename IO>
__global__ void __launch_bounds__(kRoThreads) readout_expand_kernel(int64_t T, int64_t cols, double inv,
                                                                    const double* __restrict__ g,
                                                                    IO* __restrict__ dx) {
  const int64_t j = (int64_t)blockIdx.x * kRoThreads + threadIdx.x;
  if (j >= cols) return;
  const double keep = 1.0 - inv;
  const double gj = g[j];
  double w = inv;
  IO* p = dx + (T - 1) * cols + j;
  for (int64_t t = T - 1; t >= 0; --t, p -= cols) {
    Carrier<IO>::store(p, w * gj);
    w *= keep;
  }
}

int readout_args(int64_t T, int64_t N, int64_t C, int32_t dtype, double tau, const void* a, const void* b) {
  if (T < 1 || N < 1 || C < 1) return fail(PSN_ERR_INVALID, "readout: T, N and C must be >= 1");
  if (!(tau > 1.0)) return fail(PSN_ERR_INVALID, "readout: tau must be > 1 (network.py:374-375)");
  if (dtype != PSN_F32 && dtype != PSN_F64 && dtype != PSN_BF16)
    return fail(PSN_ERR_DTYPE, "readout: carrier must be f32, bf16 or f64");
  if (!a || !b) return fail(PSN_ERR_INVALID, "readout: null pointer");
  return PSN_OK;
}

}  // namespace
}  // namespace psn

using namespace psn;

extern "C" {

int psn_readout_reduce(int64_t T, int64_t N, int64_t C, int32_t dtype, double tau, const void* x, double* xbar,
                       psn_stream_t stream) {
  int rc = readout_args(T, N, C, dtype, tau, x, xbar);
  if (rc) return rc;
  const int64_t cols = N * C;
  const dim3 grid((unsigned)((cols + kRoThreads - 1) / kRoThreads));
  cudaStream_t st = (cudaStream_t)stream;
  const double inv = 1.0 / tau;
  if (dtype == PSN_F32)
    readout_reduce_kernel<float><<<grid, kRoThreads, 0, st>>>(T, cols, inv, (const float*)x, xbar);
  else if (dtype == PSN_F64)
    readout_reduce_kernel<double><<<grid, kRoThreads, 0, st>>>(T, cols, inv, (const double*)x, xbar);
  else
    readout_reduce_kernel<__nv_bfloat16><<<grid, kRoThreads, 0, st>>>(T, cols, inv, (const __nv_bfloat16*)x, xbar);
  return cuda_check("psn_readout_reduce");
}

int psn_readout_expand(int64_t T, int64_t N, int64_t C, int32_t dtype, double tau, const double* g, void* dx,
                       psn_stream_t stream) {
  int rc = readout_args(T, N, C, dtype, tau, g, dx);
  if (rc) return rc;
  const int64_t cols = N * C;
  const dim3 grid((unsigned)((cols + kRoThreads - 1) / kRoThreads));
  cudaStream_t st = (cudaStream_t)stream;
  const double inv = 1.0 / tau;
  if (dtype == PSN_F32)
    readout_expand_kernel<float><<<grid, kRoThreads, 0, st>>>(T, cols, inv, g, (float*)dx);
  else if (dtype == PSN_F64)
    readout_expand_kernel<double><<<grid, kRoThreads, 0, st>>>(T, cols, inv, g, (double*)dx);
  else
    readout_expand_kernel<__nv_bfloat16><<<grid, kRoThreads, 0, st>>>(T, cols, inv, g, (__nv_bfloat16*)dx);
  return cuda_check("psn_readout_expand");
}

}  // extern "C"
