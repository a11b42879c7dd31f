// psn_stream_dispatch.h — entry points of the per-(carrier, direction)
// instantiation units of the streamed PSN kernels (psn_stream_inst.cuh).
#pragma once
#include "psn_stream.cuh"

namespace psn {
namespace stream {

int run_f32_fwd(int k, int d, const Args& a, const void* x, const void* dy, cudaStream_t st);
int run_f32_bwd(int k, int d, const Args& a, const void* x, const void* dy, cudaStream_t st);
int run_bf16_fwd(int k, int d, const Args& a, const void* x, const void* dy, cudaStream_t st);
int run_bf16_bwd(int k, int d, const Args& a, const void* x, const void* dy, cudaStream_t st);

bool eligible(const psn_desc_t* desc);        // shape_eligible and not PSN_FORCE_GENERIC
bool shape_eligible(const psn_desc_t* desc);  // the shape / carrier alone (no run-time knobs)
bool aligned_for_tma(const void* x, const void* dy);
bool make_plan(const psn_desc_t* desc, bool bwd, Plan& p, bool for_sizing = false);
size_t workspace_bytes(const psn_desc_t* desc);
int forward(const psn_desc_t* desc, const Plan& p, const void* x, const double* W, const double* gamma,
            const double* beta, double* rm, double* rv, void* out, double* fold, void* ws, cudaStream_t st);
int backward(const psn_desc_t* desc, const Plan& p, const void* x, const void* dy, const double* W,
             const double* gamma, const double* fold, void* dx, double* dW, double* dgamma, double* dbeta,
             void* ws, cudaStream_t st);

}  // namespace stream
}  // namespace psn
