// psn_engines.cu — the reference's engine-level operators on sm_100a
// (engines.py:117-138, 258-325, 350-431; quant.py:111-139).
//
// These are the building blocks the reference's SpikingLayer composes; they
// are exposed through the C ABI so every engine KAT of the reference test
// suite can run against the GPU.  Convolutions accumulate in f64 in the
// reference's tap order (mul, then add), so DIRECT / shift / backward-input
// results are bit-identical to the reference; weight/bias gradients are f64
// reductions in a fixed (but different) order.
#include <string>

#include "psn_common.cuh"

namespace psn {

// forward conv with float weights (SHIFT=false) or sign/exponent weights;
// SPIKE: the ShiftLayer's Heaviside fused on the carrier-rounded membrane
// (network.py:352-362: spikes = (f32(h) >= 0), no h written).  Streams x through
// the per-warp shared-memory ring (psn_common.cuh stream_any).
template <int K, typename IO, bool SHIFT, bool SPIKE = false>
__global__ void __launch_bounds__(kThreads, 2) eng_fwd_kernel(Geom g, const IO* __restrict__ x,
                                                           const double* __restrict__ w,
                                                           const int8_t* __restrict__ sgn,
                                                           const int8_t* __restrict__ ex,
                                                           int64_t w_rows, const double* __restrict__ bias,
                                                           IO* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const bool jv = j < g.J;
  const int64_t c = jv ? j / g.Q : 0;
  const int64_t row = (w_rows == 1) ? 0 : c;
  double wv[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    if (!jv)
      wv[i] = 0.0;
    else if (SHIFT)
      wv[i] = ldexp((double)sgn[row * K + i], (int)ex[row * K + i]);
    else
      wv[i] = w[row * K + i];
  }
  const bool hb = bias != nullptr;
  const double b = (jv && hb) ? bias[c] : 0.0;
  const int64_t step = (int64_t)g.d * g.row;
  extern __shared__ __align__(16) unsigned char psn_dsm[];
  IO* ring = reinterpret_cast<IO*>(psn_dsm) + warp * kRingSteps * 32;
  const ColTile ct = col_tile<IO>(g, x, x);
  for (int64_t seg = (int64_t)blockIdx.y * kWarps + warp; seg < g.nseg; seg += (int64_t)gridDim.y * kWarps) {
    Seg s;
    if (!decode_seg(g, seg, s)) continue;
    const int64_t off = (int64_t)s.r * g.row + s.n * g.J + j;
    double xw[K];
#pragma unroll
    for (int m = 1; m < K; ++m) {
      const int64_t sp = s.s0 - K + m;
      xw[m] = (jv && sp >= 0) ? load_wide(x + off + sp * step) : 0.0;
    }
    const IO* p = x + off + s.s0 * step;
    IO* o = out + off + s.s0 * step;
    stream_any<(K > 8 ? 4 : 8), false>(ring, ct, p, p, x, x, step, s.s0, s.s1, s.s1, [&](IO xv, IO, int64_t, int64_t eo) {
#pragma unroll
      for (int i = 0; i < K - 1; ++i) xw[i] = xw[i + 1];
      xw[K - 1] = wide(xv);
      double h = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) h = __dadd_rn(h, __dmul_rn(wv[i], xw[i]));
      if (hb) h = __dadd_rn(h, b);
      if (jv) {
        if (SPIKE)
          Carrier<IO>::storef(o + eo, Carrier<IO>::round(h) >= 0.0 ? 1.0f : 0.0f);
        else
          Carrier<IO>::store(o + eo, h);
      }
    });
  }
}

// int32 fixed-point shift engine (engines.py:297-325)
template <int K>
__global__ void __launch_bounds__(kThreads) eng_shift_int_kernel(Geom g, const int32_t* __restrict__ x,
                                                                 const int8_t* __restrict__ sgn,
                                                                 const int8_t* __restrict__ ex, int64_t w_rows,
                                                                 const double* __restrict__ bias,
                                                                 int32_t* __restrict__ out,
                                                                 unsigned long long* __restrict__ sat) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const bool jv = j < g.J;
  const int64_t c = jv ? j / g.Q : 0;
  const int64_t row = (w_rows == 1) ? 0 : c;
  int sv[K], ev[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    sv[i] = jv ? (int)sgn[row * K + i] : 0;
    ev[i] = jv ? (int)ex[row * K + i] : 0;
  }
  const bool hb = bias != nullptr;
  const long long b = (jv && hb) ? (long long)bias[c] : 0;  // numpy astype(int64): trunc toward 0
  const int64_t step = (int64_t)g.d * g.row;
  unsigned long long nsat = 0;
  for (int64_t seg = (int64_t)blockIdx.y * kWarps + warp; seg < g.nseg; seg += (int64_t)gridDim.y * kWarps) {
    Seg s;
    if (!decode_seg(g, seg, s)) continue;
    const int64_t off = (int64_t)s.r * g.row + s.n * g.J + j;
    long long xw[K];
#pragma unroll
    for (int m = 1; m < K; ++m) {
      const int64_t sp = s.s0 - K + m;
      xw[m] = (jv && sp >= 0) ? (long long)__ldg(x + off + sp * step) : 0;
    }
    const int32_t* p = x + off + s.s0 * step;
    int32_t* o = out + off + s.s0 * step;
    for (int64_t t = s.s0; t < s.s1; ++t) {
#pragma unroll
      for (int i = 0; i < K - 1; ++i) xw[i] = xw[i + 1];
      xw[K - 1] = jv ? (long long)__ldg(p) : 0;
      long long acc = 0;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const long long v = ev[i] >= 0 ? (xw[i] << ev[i]) : (xw[i] >> (-ev[i]));
        acc += (long long)sv[i] * v;
      }
      acc += b;
      long long cl = acc;
      if (cl > 2147483647LL) cl = 2147483647LL;
      if (cl < -2147483648LL) cl = -2147483648LL;
      if (jv) {
        nsat += (cl != acc);
        *o = (int32_t)cl;
      }
      p += step;
      o += step;
    }
  }
#pragma unroll
  for (int off2 = 16; off2 > 0; off2 >>= 1) nsat += __shfl_xor_sync(0xffffffffu, nsat, off2);
  if (lane == 0 && nsat) atomicAdd(sat, nsat);
}

// backward-input: out[s] = sum_i w_i dh[s + (K-1-i)] in reference tap order;
// ywin[m] holds dh at subsequence step s + m.
template <int K, typename IO>
__global__ void __launch_bounds__(kThreads) eng_bwd_in_kernel(Geom g, const IO* __restrict__ dh,
                                                              const double* __restrict__ w, int64_t w_rows,
                                                              IO* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const bool jv = j < g.J;
  const int64_t c = jv ? j / g.Q : 0;
  const int64_t row = (w_rows == 1) ? 0 : c;
  double wv[K];
#pragma unroll
  for (int i = 0; i < K; ++i) wv[i] = jv ? w[row * K + i] : 0.0;
  const int64_t step = (int64_t)g.d * g.row;
  for (int64_t seg = (int64_t)blockIdx.y * kWarps + warp; seg < g.nseg; seg += (int64_t)gridDim.y * kWarps) {
    Seg s;
    if (!decode_seg(g, seg, s)) continue;
    const int64_t off = (int64_t)s.r * g.row + s.n * g.J + j;
    double yw[K];
#pragma unroll
    for (int m = 1; m < K; ++m) {
      const int64_t sp = s.s0 + m - 1;
      yw[m] = (jv && sp < s.Sr) ? load_wide(dh + off + sp * step) : 0.0;
    }
    IO* o = out + off + s.s0 * step;
    const IO* p = dh + off + (s.s0 + K - 1) * step;
    for (int64_t t = s.s0; t < s.s1; ++t) {
#pragma unroll
      for (int i = 0; i < K - 1; ++i) yw[i] = yw[i + 1];
      yw[K - 1] = (jv && t + K - 1 < s.Sr) ? load_wide(p) : 0.0;
      double h = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) h = __dadd_rn(h, __dmul_rn(wv[i], yw[K - 1 - i]));
      if (jv) Carrier<IO>::store(o, h);
      p += step;
      o += step;
    }
  }
}

// per-column correlations: part[row][0] = sum dh, part[row][1+i] = sum x[t-off_i] dh[t]
template <int K, typename IO>
__global__ void __launch_bounds__(kThreads) eng_corr_kernel(Geom g, const IO* __restrict__ x,
                                                            const IO* __restrict__ dh,
                                                            double* __restrict__ part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const bool jv = j < g.J;
  const int64_t step = (int64_t)g.d * g.row;
  double db = 0.0, dw[K];
#pragma unroll
  for (int i = 0; i < K; ++i) dw[i] = 0.0;
  for (int sp = 0; sp < g.spw; ++sp) {
    const int64_t seg = ((int64_t)blockIdx.y * g.spw + sp) * kWarps + warp;
    if (seg >= g.nseg) break;
    Seg s;
    if (!decode_seg(g, seg, s)) continue;
    const int64_t off = (int64_t)s.r * g.row + s.n * g.J + j;
    double xw[K];
#pragma unroll
    for (int m = 1; m < K; ++m) {
      const int64_t sp2 = s.s0 - K + m;
      xw[m] = (jv && sp2 >= 0 && x) ? load_wide(x + off + sp2 * step) : 0.0;
    }
    for (int64_t t = s.s0; t < s.s1; ++t) {
#pragma unroll
      for (int i = 0; i < K - 1; ++i) xw[i] = xw[i + 1];
      xw[K - 1] = (jv && x) ? load_wide(x + off + t * step) : 0.0;
      const double v = jv ? load_wide(dh + off + t * step) : 0.0;
      db += v;
#pragma unroll
      for (int i = 0; i < K; ++i) dw[i] = fma(xw[i], v, dw[i]);
    }
  }
  constexpr int NV = K + 1;
  __shared__ double sh[kWarps][32];
  double* o = part + (int64_t)blockIdx.y * NV * g.J + j;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double val = (v == 0) ? db : 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i)
      if (v == 1 + i) val = dw[i];
    sh[warp][lane] = val;
    __syncthreads();
    if (warp == 0) {
      double t = sh[0][lane];
#pragma unroll
      for (int w2 = 1; w2 < kWarps; ++w2) t += sh[w2][lane];
      if (jv) o[(int64_t)v * g.J] = t;
    }
    __syncthreads();
  }
}

// per-channel fold of eng_corr partials: WHICH=0 -> bias grad [C], 1 -> weight grad [C,K]
__global__ void eng_corr_fold_kernel(Geom g, const double* __restrict__ part, int which, double* __restrict__ outp) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (c >= g.C) return;
  const int K = g.k, NV = K + 1;
  const int64_t total = g.rows * g.Q;
  const int v0 = which ? 1 : 0, v1 = which ? NV : 1;
  for (int v = v0; v < v1; ++v) {
    double acc = 0.0;
    for (int64_t idx = lane; idx < total; idx += 32) {
      const int64_t r = idx / g.Q, q = idx % g.Q;
      acc += part[(r * NV + v) * g.J + c * g.Q + q];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, acc, off);
      acc = (lane & off) ? o + acc : acc + o;
    }
    if (lane == 0) {
      if (which) outp[c * K + (v - 1)] = acc;
      else outp[c] = acc;
    }
  }
}

__global__ void eng_rowsum_kernel(const double* __restrict__ in, int64_t C, int K, double* __restrict__ out) {
  const int i = threadIdx.x;
  if (i >= K) return;
  double acc = 0.0;
  for (int64_t c = 0; c < C; ++c) acc += in[c * K + i];
  out[i] = acc;
}

__global__ void eng_quant_kernel(const double* __restrict__ w, int64_t n, int8_t* __restrict__ sgn,
                                 int8_t* __restrict__ ex) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int s, e;
  quantize_pow2(w[i], s, e);
  sgn[i] = (int8_t)s;
  ex[i] = (int8_t)e;
}

static inline dim3 grid_map(const Geom& g) {
  int64_t y = (g.nseg + kWarps - 1) / kWarps;
  if (y > 65535) y = 65535;
  return dim3((unsigned)g.ctiles, (unsigned)y);
}

#define PSN_K_SWITCH(k, CALL)          \
  switch (k) {                         \
    case 1: { constexpr int K = 1; CALL; break; }   \
    case 2: { constexpr int K = 2; CALL; break; }   \
    case 3: { constexpr int K = 3; CALL; break; }   \
    case 4: { constexpr int K = 4; CALL; break; }   \
    case 5: { constexpr int K = 5; CALL; break; }   \
    case 6: { constexpr int K = 6; CALL; break; }   \
    case 7: { constexpr int K = 7; CALL; break; }   \
    case 8: { constexpr int K = 8; CALL; break; }   \
    case 9: { constexpr int K = 9; CALL; break; }   \
    case 10: { constexpr int K = 10; CALL; break; } \
    case 11: { constexpr int K = 11; CALL; break; } \
    case 12: { constexpr int K = 12; CALL; break; } \
    case 13: { constexpr int K = 13; CALL; break; } \
    case 14: { constexpr int K = 14; CALL; break; } \
    case 15: { constexpr int K = 15; CALL; break; } \
    case 16: { constexpr int K = 16; CALL; break; } \
    default: return fail(PSN_ERR_ORDER, "order out of range"); \
  }

static int check_float_carrier(const psn_desc_t* desc) {
  if (desc->dtype != PSN_F32 && desc->dtype != PSN_F64)
    return fail(PSN_ERR_DTYPE, "engine operators take f32 or f64 carriers");
  return PSN_OK;
}

static int check_rows(const psn_desc_t* desc, int64_t w_rows) {
  if (w_rows != 1 && w_rows != desc->C) return fail(PSN_ERR_INVALID, "weight rows do not match channels");
  return PSN_OK;
}

}  // namespace psn

using namespace psn;

extern "C" {

int psn_conv_forward(const psn_desc_t* desc, const void* x, const double* w, int64_t w_rows,
                     const double* bias, void* out, psn_stream_t stream) {
  int rc;
  if ((rc = validate(desc, false)) || (rc = check_float_carrier(desc)) || (rc = check_rows(desc, w_rows))) return rc;
  const size_t es = dtype_size(desc->dtype);
  if ((rc = check_ptr(x, es, "x")) || (rc = check_ptr(out, es, "out")) || (rc = check_ptr(w, 8, "w"))) return rc;
  const Geom g = plan(desc);
  cudaStream_t st = (cudaStream_t)stream;
  if (desc->dtype == PSN_F32) {
    PSN_K_SWITCH(desc->k, (eng_fwd_kernel<K, float, false><<<grid_map(g), kThreads, ring_bytes<float>(1), st>>>(
                              g, (const float*)x, w, nullptr, nullptr, w_rows, bias, (float*)out)));
  } else {
    PSN_K_SWITCH(desc->k, (rc = smem_optin(eng_fwd_kernel<K, double, false>, ring_bytes<double>(1))));
    if (rc) return rc;
    PSN_K_SWITCH(desc->k, (eng_fwd_kernel<K, double, false><<<grid_map(g), kThreads, ring_bytes<double>(1), st>>>(
                              g, (const double*)x, w, nullptr, nullptr, w_rows, bias, (double*)out)));
  }
  return cuda_check("psn_conv_forward");
}

int psn_conv_forward_shift(const psn_desc_t* desc, const void* x, const int8_t* sign, const int8_t* exponent,
                           int64_t w_rows, const double* bias, void* out, psn_stream_t stream) {
  int rc;
  if ((rc = validate(desc, false)) || (rc = check_float_carrier(desc)) || (rc = check_rows(desc, w_rows))) return rc;
  const size_t es = dtype_size(desc->dtype);
  if ((rc = check_ptr(x, es, "x")) || (rc = check_ptr(out, es, "out")) || (rc = check_ptr(sign, 1, "sign")) ||
      (rc = check_ptr(exponent, 1, "exponent")))
    return rc;
  const Geom g = plan(desc);
  cudaStream_t st = (cudaStream_t)stream;
  if (desc->dtype == PSN_F32) {
    PSN_K_SWITCH(desc->k, (eng_fwd_kernel<K, float, true><<<grid_map(g), kThreads, ring_bytes<float>(1), st>>>(
                              g, (const float*)x, nullptr, sign, exponent, w_rows, bias, (float*)out)));
  } else {
    PSN_K_SWITCH(desc->k, (rc = smem_optin(eng_fwd_kernel<K, double, true>, ring_bytes<double>(1))));
    if (rc) return rc;
    PSN_K_SWITCH(desc->k, (eng_fwd_kernel<K, double, true><<<grid_map(g), kThreads, ring_bytes<double>(1), st>>>(
                              g, (const double*)x, nullptr, sign, exponent, w_rows, bias, (double*)out)));
  }
  return cuda_check("psn_conv_forward_shift");
}

int psn_shift_spike_forward(const psn_desc_t* desc, const void* x, const int8_t* sign, const int8_t* exponent,
                            int64_t w_rows, const double* bias, void* out, psn_stream_t stream) {
  int rc;
  if ((rc = validate(desc, false)) || (rc = check_float_carrier(desc)) || (rc = check_rows(desc, w_rows))) return rc;
  const size_t es = dtype_size(desc->dtype);
  if ((rc = check_ptr(x, es, "x")) || (rc = check_ptr(out, es, "out")) || (rc = check_ptr(sign, 1, "sign")) ||
      (rc = check_ptr(exponent, 1, "exponent")))
    return rc;
  const Geom g = plan(desc);
  cudaStream_t st = (cudaStream_t)stream;
  if (desc->dtype == PSN_F32) {
    PSN_K_SWITCH(desc->k,
                 (eng_fwd_kernel<K, float, true, true><<<grid_map(g), kThreads, ring_bytes<float>(1), st>>>(
                     g, (const float*)x, nullptr, sign, exponent, w_rows, bias, (float*)out)));
  } else {
    PSN_K_SWITCH(desc->k, (rc = smem_optin(eng_fwd_kernel<K, double, true, true>, ring_bytes<double>(1))));
    if (rc) return rc;
    PSN_K_SWITCH(desc->k,
                 (eng_fwd_kernel<K, double, true, true><<<grid_map(g), kThreads, ring_bytes<double>(1), st>>>(
                     g, (const double*)x, nullptr, sign, exponent, w_rows, bias, (double*)out)));
  }
  return cuda_check("psn_shift_spike_forward");
}

int psn_conv_forward_shift_int(const psn_desc_t* desc, const int32_t* x, const int8_t* sign,
                               const int8_t* exponent, int64_t w_rows, const double* bias, int32_t* out,
                               unsigned long long* saturations, psn_stream_t stream) {
  int rc;
  if ((rc = validate(desc, true)) || (rc = check_rows(desc, w_rows))) return rc;
  if (desc->dtype != PSN_I32) return fail(PSN_ERR_DTYPE, "shift_int takes an int32 carrier");
  if ((rc = check_ptr(x, 4, "x")) || (rc = check_ptr(out, 4, "out")) || (rc = check_ptr(sign, 1, "sign")) ||
      (rc = check_ptr(exponent, 1, "exponent")) || (rc = check_ptr(saturations, 8, "saturations")))
    return rc;
  const Geom g = plan(desc);
  cudaStream_t st = (cudaStream_t)stream;
  PSN_K_SWITCH(desc->k, (eng_shift_int_kernel<K><<<grid_map(g), kThreads, 0, st>>>(g, x, sign, exponent, w_rows,
                                                                                  bias, out, saturations)));
  return cuda_check("psn_conv_forward_shift_int");
}

int psn_conv_backward_input(const psn_desc_t* desc, const void* dh, const double* w, int64_t w_rows, void* out,
                            psn_stream_t stream) {
  int rc;
  if ((rc = validate(desc, false)) || (rc = check_float_carrier(desc)) || (rc = check_rows(desc, w_rows))) return rc;
  const size_t es = dtype_size(desc->dtype);
  if ((rc = check_ptr(dh, es, "dh")) || (rc = check_ptr(out, es, "out")) || (rc = check_ptr(w, 8, "w"))) return rc;
  const Geom g = plan(desc);
  cudaStream_t st = (cudaStream_t)stream;
  if (desc->dtype == PSN_F32) {
    PSN_K_SWITCH(desc->k, (eng_bwd_in_kernel<K, float><<<grid_map(g), kThreads, 0, st>>>(
                              g, (const float*)dh, w, w_rows, (float*)out)));
  } else {
    PSN_K_SWITCH(desc->k, (eng_bwd_in_kernel<K, double><<<grid_map(g), kThreads, 0, st>>>(
                              g, (const double*)dh, w, w_rows, (double*)out)));
  }
  return cuda_check("psn_conv_backward_input");
}

static int corr_common(const psn_desc_t* desc, const void* x, const void* dh, int which, int shared, double* grad,
                       void* workspace, psn_stream_t stream) {
  const Geom g = plan(desc);
  cudaStream_t st = (cudaStream_t)stream;
  double* part = (double*)((char*)workspace + workspace_part3_offset(desc));
  const dim3 grid((unsigned)g.ctiles, (unsigned)g.rows);
  if (desc->dtype == PSN_F32) {
    PSN_K_SWITCH(desc->k, (eng_corr_kernel<K, float><<<grid, kThreads, 0, st>>>(g, (const float*)x,
                                                                               (const float*)dh, part)));
  } else {
    PSN_K_SWITCH(desc->k, (eng_corr_kernel<K, double><<<grid, kThreads, 0, st>>>(g, (const double*)x,
                                                                                (const double*)dh, part)));
  }
  const unsigned fb = (unsigned)((g.C + kWarps - 1) / kWarps);
  if (which == 1 && shared) {
    // per-channel grads into the workspace's first region, then the row sum
    double* tmp = (double*)((char*)workspace + workspace_dwtmp_offset(desc));
    eng_corr_fold_kernel<<<fb, kThreads, 0, st>>>(g, part, 1, tmp);
    eng_rowsum_kernel<<<1, 32, 0, st>>>(tmp, g.C, g.k, grad);
  } else {
    eng_corr_fold_kernel<<<fb, kThreads, 0, st>>>(g, part, which, grad);
  }
  return cuda_check("psn_conv_backward_weight/bias");
}

int psn_conv_backward_weight(const psn_desc_t* desc, const void* x, const void* dh, int shared, double* grad,
                             void* workspace, psn_stream_t stream) {
  int rc;
  if ((rc = validate(desc, false)) || (rc = check_float_carrier(desc))) return rc;
  const size_t es = dtype_size(desc->dtype);
  if ((rc = check_ptr(x, es, "x")) || (rc = check_ptr(dh, es, "dh")) || (rc = check_ptr(grad, 8, "grad")) ||
      (rc = check_ptr(workspace, 256, "workspace")))
    return rc;
  return corr_common(desc, x, dh, 1, shared, grad, workspace, stream);
}

int psn_conv_backward_bias(const psn_desc_t* desc, const void* dh, double* grad, void* workspace,
                           psn_stream_t stream) {
  int rc;
  if ((rc = validate(desc, false)) || (rc = check_float_carrier(desc))) return rc;
  const size_t es = dtype_size(desc->dtype);
  if ((rc = check_ptr(dh, es, "dh")) || (rc = check_ptr(grad, 8, "grad")) ||
      (rc = check_ptr(workspace, 256, "workspace")))
    return rc;
  return corr_common(desc, nullptr, dh, 0, 0, grad, workspace, stream);
}

int psn_quantize_pow2(const double* w, int64_t n, int8_t* sign, int8_t* exponent, psn_stream_t stream) {
  int rc;
  if (n < 0) return fail(PSN_ERR_INVALID, "negative length");
  if (n == 0) return PSN_OK;
  if ((rc = check_ptr(w, 8, "w")) || (rc = check_ptr(sign, 1, "sign")) || (rc = check_ptr(exponent, 1, "exponent")))
    return rc;
  eng_quant_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(w, n, sign, exponent);
  return cuda_check("psn_quantize_pow2");
}

}  // extern "C"
