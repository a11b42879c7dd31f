// psn_optim.cu — the reference's Adam update (train.py:147-172) for every
// parameter tensor of a network in ONE launch.
//
// The module-level optimizer issued ~6 element-wise torch kernels per
// parameter tensor (about 100 launches of 1-2 us each for the SHD-shaped net,
// ~0.4 ms of a 1.6 ms training step even inside a CUDA graph).  Here the host
// describes the tensors once as chunks (pointer table in device memory) and one
// block updates one chunk.  The arithmetic is the reference's, operation by
// operation, with explicitly rounded intrinsics (no FMA contraction), so the
// result is bit-identical to the element-wise formulation:
//   m = m*b1 + (1-b1)*g;  v = v*b2 + ((1-b2)*g)*g;
//   p = p - (lr * (m / c1)) / (sqrt(v / c2) + eps),  c_i = 1 - b_i^t.
// The bias corrections come from the host (c1, c2) or, for a captured step,
// from the device step count t (1 - pow(b, t), the same libdevice pow the
// element-wise capturable formulation uses).
#include "psn_common.cuh"

namespace psn {

int fail(int code, const char* msg);
int cuda_check(const char* where);

namespace {

constexpr int kAdamThreads = 256;

__global__ void __launch_bounds__(kAdamThreads) adam_kernel(const psn_adam_chunk_t* __restrict__ chunks,
                                                            double lr, double b1, double b2, double eps,
                                                            double c1h, double c2h,
                                                            const double* __restrict__ t_dev) {
  const psn_adam_chunk_t ch = chunks[blockIdx.x];
  double c1 = c1h, c2 = c2h;
  if (t_dev) {
    const double t = *t_dev;
    c1 = __dsub_rn(1.0, pow(b1, t));
    c2 = __dsub_rn(1.0, pow(b2, t));
  }
  const double a1 = __dsub_rn(1.0, b1), a2 = __dsub_rn(1.0, b2);
  for (int64_t i = threadIdx.x; i < ch.n; i += kAdamThreads) {
    const double g = ch.grad[i];
    const double m = __dadd_rn(__dmul_rn(ch.m[i], b1), __dmul_rn(a1, g));
    const double v = __dadd_rn(__dmul_rn(ch.v[i], b2), __dmul_rn(__dmul_rn(a2, g), g));
    const double mh = __ddiv_rn(m, c1), vh = __ddiv_rn(v, c2);
    const double upd = __ddiv_rn(__dmul_rn(lr, mh), __dadd_rn(__dsqrt_rn(vh), eps));
    ch.m[i] = m;
    ch.v[i] = v;
    ch.param[i] = __dsub_rn(ch.param[i], upd);
  }
}

}  // namespace
}  // namespace psn

using namespace psn;

extern "C" {

int psn_adam_step(const psn_adam_chunk_t* chunks, int64_t n_chunks, double lr, double beta1, double beta2,
                  double eps, double c1, double c2, const double* t_dev, psn_stream_t stream) {
  if (n_chunks < 0 || n_chunks > 0x7fffffff) return fail(PSN_ERR_INVALID, "adam: bad chunk count");
  if (n_chunks == 0) return PSN_OK;
  if (!chunks) return fail(PSN_ERR_INVALID, "adam: null chunk table");
  if (((uintptr_t)chunks) % 8) return fail(PSN_ERR_ALIGN, "adam: misaligned chunk table");
  if (!(lr >= 0.0) || !(eps > 0.0) || !(beta1 >= 0.0 && beta1 < 1.0) || !(beta2 >= 0.0 && beta2 < 1.0))
    return fail(PSN_ERR_INVALID, "adam: lr >= 0, eps > 0 and beta in [0, 1) required");
  adam_kernel<<<(unsigned)n_chunks, kAdamThreads, 0, (cudaStream_t)stream>>>(chunks, lr, beta1, beta2, eps, c1,
                                                                              c2, t_dev);
  return cuda_check("psn_adam_step");
}

}  // extern "C"
