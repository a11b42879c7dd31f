// psn_layer.cu — sm_100a kernels for SpikingLayer TRAIN/SMOOTH forward,
// backward and EVAL forward (reference network.py:213-318), plus the C ABI.
//
// Pass structure (BN batch statistics force one global reduction barrier in
// each direction, reference network.py:239-259 and :291-315):
//   forward : fwd_stats  (h1 = conv(x, W) on the fly; per-column Chan moments)
//             fwd_fold   (merge moments per channel; running update; BN fold;
//                         exact pow2 quantization)               [1 warp/channel]
//             fwd_spike  (h2 = sum_i w_q,i * x[t-off_i] + b_f in f64 tap order;
//                         Heaviside or spike_primitive; writes spikes only)
//   backward: bwd_reduce (recompute h1, h2; dh2 = dy*sigma'(h2); per-column
//                         sums db, dw_q[i], Sx[i], Sxc[i] = sum x[t-off_i](h1-mu))
//             bwd_fold   (STE, dW, dgamma, dbeta, BN-through-stats scalars)
//             bwd_dx     (recompute dh2, dh1 = alpha1 + beta1 (h1 - mu); the
//                         time-reversed conv accumulated in a k-slot register ring)
// h1 and h2 are never stored: 20 B/elem of algorithmic HBM traffic for f32 I/O.
#include <stdio.h>
#include <string.h>

#include <string>
#include <type_traits>

#include "psn_common.cuh"
#include "psn_stream_dispatch.h"

namespace psn {

thread_local std::string g_last_error;

int fail(int code, const char* msg) {
  g_last_error = msg;
  return code;
}

int cuda_check(const char* where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[256];
    snprintf(buf, sizeof(buf), "%s: %s", where, cudaGetErrorString(e));
    g_last_error = buf;
    return PSN_ERR_CUDA;
  }
  return PSN_OK;
}

// ------------------------------------------------------------------------------
// planning
// ------------------------------------------------------------------------------
Geom plan(const psn_desc_t* desc) {
  Geom g;
  g.T = desc->T;
  g.N = desc->N;
  g.C = desc->C;
  g.Q = desc->Q;
  g.J = g.C * g.Q;
  g.row = g.N * g.J;
  g.d = desc->d;
  g.k = desc->k;
  g.S = (g.T + g.d - 1) / g.d;
  g.ctiles = (g.J + 31) / 32;
  const int64_t target_warps = 148 * 32;
  int64_t L = 256;
  while (L > 16 && g.ctiles * g.N * g.d * ((g.S + L - 1) / L) < target_warps) L >>= 1;
  if (L > g.S) L = g.S;
  if (L < 1) L = 1;
  g.nch = (g.S + L - 1) / L;
  g.L = (g.S + g.nch - 1) / g.nch;  // equal chunks: a warp's segments are all about as long
  g.nseg = g.N * g.d * g.nch;
  int spw = 1;
  while (spw < 64 && g.ctiles * ((g.nseg + kWarps * spw * 2 - 1) / (kWarps * spw * 2)) * kWarps >= target_warps)
    spw *= 2;
  // keep gridDim.y within limits
  while ((g.nseg + (int64_t)kWarps * spw - 1) / ((int64_t)kWarps * spw) > 65535) spw *= 2;
  g.spw = spw;
  g.rows = (g.nseg + (int64_t)kWarps * spw - 1) / ((int64_t)kWarps * spw);
  return g;
}

struct WsLayout {
  size_t part1, part3, bfold, dwtmp, evalfold, fused, dhm, dhm_bytes, total;
};

static size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

WsLayout ws_layout(const psn_desc_t* desc) {
  const Geom g = plan(desc);
  WsLayout w;
  size_t off = 0;
  w.part1 = off;
  off = align256(off + sizeof(double) * 3 * (size_t)g.rows * g.J);
  w.part3 = off;
  off = align256(off + sizeof(double) * (3 * (size_t)g.k + 1) * (size_t)g.rows * g.J);
  w.bfold = off;
  off = align256(off + sizeof(double) * 2 * (size_t)g.C);
  w.dwtmp = off;
  off = align256(off + sizeof(double) * (size_t)g.k * g.C);
  w.evalfold = off;
  off = align256(off + sizeof(double) * PSN_FOLD_STRIDE((size_t)g.k) * g.C);
  w.fused = off;
  off = align256(off + stream::workspace_bytes(desc));
  // generic backward of a 4 / 2 B carrier: dh2 and h1 - mu materialised as f32
  // by bwd_reduce for an FP32-only bwd_dx_mat.  Sized from the shape alone (never
  // from run-time knobs): a streamable shape that still takes the generic path
  // recomputes them instead (bwd_dx_kernel).
  w.dhm = off;
  w.dhm_bytes = (desc->dtype != PSN_F64 && !stream::shape_eligible(desc))
                    ? 2 * sizeof(float) * (size_t)desc->T * desc->N * desc->C * desc->Q : 0;
  off = align256(off + w.dhm_bytes);
  w.total = off;
  return w;
}

size_t workspace_part3_offset(const psn_desc_t* desc) { return ws_layout(desc).part3; }
size_t workspace_dwtmp_offset(const psn_desc_t* desc) { return ws_layout(desc).dwtmp; }

int validate(const psn_desc_t* d, bool allow_i32) {
  if (!d) return fail(PSN_ERR_INVALID, "null descriptor");
  if (d->T < 1 || d->N < 1 || d->C < 1 || d->Q < 1)
    return fail(PSN_ERR_INVALID, "T, N, C and Q must all be >= 1");
  if (d->d < 1) return fail(PSN_ERR_INVALID, "dilation must be >= 1");
  if (d->k < 1) return fail(PSN_ERR_INVALID, "order must be >= 1");
  if (d->k > PSN_MAX_ORDER) return fail(PSN_ERR_ORDER, "order above PSN_MAX_ORDER (16)");
  if (d->dtype != PSN_F32 && d->dtype != PSN_BF16 && d->dtype != PSN_F64 &&
      !(allow_i32 && d->dtype == PSN_I32))
    return fail(PSN_ERR_DTYPE, "unsupported carrier dtype");
  if (d->surrogate != PSN_ARCTAN && d->surrogate != PSN_RATIONAL)
    return fail(PSN_ERR_INVALID, "unknown surrogate kind");
  if (!(d->alpha > 0.0)) return fail(PSN_ERR_INVALID, "alpha must be positive");
  if (!(d->eps > 0.0)) return fail(PSN_ERR_INVALID, "eps must be positive");
  if (!(d->momentum > 0.0 && d->momentum < 1.0))
    return fail(PSN_ERR_INVALID, "momentum must be in (0, 1)");
  const double elems = (double)d->T * (double)d->N * (double)d->C * (double)d->Q;
  if (elems > 9.0e18) return fail(PSN_ERR_INVALID, "tensor too large");
  return PSN_OK;
}

int check_ptr(const void* p, size_t align, const char* what) {
  if (!p) {
    g_last_error = std::string("null pointer: ") + what;
    return PSN_ERR_INVALID;
  }
  if (((uintptr_t)p) % align) {
    g_last_error = std::string("misaligned pointer: ") + what;
    return PSN_ERR_ALIGN;
  }
  return PSN_OK;
}

size_t dtype_size(int dt) {
  return dt == PSN_F64 ? 8 : (dt == PSN_BF16 ? 2 : 4);
}

Surrogate make_surrogate(const psn_desc_t* d) {
  Surrogate s;
  s.kind = d->surrogate;
  if (d->surrogate == PSN_ARCTAN) {
    s.c = (float)(0.5 * 3.141592653589793 * d->alpha);
    s.scale = (float)(d->alpha / 2.0);
  } else {
    s.c = (float)d->alpha;
    s.scale = 1.0f;
  }
  return s;
}

// ------------------------------------------------------------------------------
// window helpers
// ------------------------------------------------------------------------------
// xw[i] holds the input seen by tap i: x at subsequence step s-(K-1-i).
template <int K, typename IO>
__device__ __forceinline__ void prime_window(double (&xw)[K], const IO* base, int64_t step,
                                             int64_t s0, bool jv) {
#pragma unroll
  for (int m = 1; m < K; ++m) {
    const int64_t sp = s0 - K + m;
    xw[m] = (jv && sp >= 0) ? load_wide(base + sp * step) : 0.0;
  }
}

template <int K>
__device__ __forceinline__ void push(double (&xw)[K], double v) {
#pragma unroll
  for (int i = 0; i < K - 1; ++i) xw[i] = xw[i + 1];
  xw[K - 1] = v;
}

// reference tap order (oldest tap first) with fused multiply-adds: for the
// power-of-two w_q every product is exact, so the DFMA chain equals the
// reference's mul-then-add bit for bit; for float W it differs by at most an
// f64 ulp before the carrier rounding (the streamed kernels do the same).  The
// engine-level operators (psn_engines.cu) keep the separate mul and add.
template <int K>
__device__ __forceinline__ double conv_taps(const double (&w)[K], const double (&xw)[K]) {
  double h = w[0] * xw[0];
#pragma unroll
  for (int i = 1; i < K; ++i) h = fma(w[i], xw[i], h);
  return h;
}

// the same sum as two interleaved half chains (even / odd taps) for the
// quantities only compared under a tolerance (h1 for the statistics, h1 / h2
// in the backward): half the dependent-DFMA latency per step, a different
// rounding order (~1 f64 ulp) than the reference's tap order
template <int K>
__device__ __forceinline__ double conv_taps2(const double (&w)[K], const double (&xw)[K]) {
  if constexpr (K < 4) {
    return conv_taps<K>(w, xw);
  } else {
    double a = w[0] * xw[0], b = w[1] * xw[1];
#pragma unroll
    for (int i = 2; i + 1 < K; i += 2) {
      a = fma(w[i], xw[i], a);
      b = fma(w[i + 1], xw[i + 1], b);
    }
    if (K & 1) a = fma(w[K - 1], xw[K - 1], a);
    return a + b;
  }
}

// ------------------------------------------------------------------------------
// forward pass 1: statistics of h1 = conv(x, W)
// ------------------------------------------------------------------------------
template <int K, typename IO>
__global__ void __launch_bounds__(kThreads, (K > 8 ? 1 : 2)) fwd_stats_kernel(Geom g, const IO* __restrict__ x,
                                                             const double* __restrict__ W,
                                                             int shared,
                                                             double* __restrict__ part) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const bool jv = j < g.J;
  const int64_t c = jv ? j / g.Q : 0;
  double w[K];
#pragma unroll
  for (int i = 0; i < K; ++i) w[i] = jv ? W[(shared ? 0 : c) * K + i] : 0.0;
  const int64_t step = (int64_t)g.d * g.row;
  extern __shared__ __align__(16) unsigned char psn_dsm[];
  IO* ring = reinterpret_cast<IO*>(psn_dsm) + warp * kRingSteps * 32;
  const ColTile ct = col_tile<IO>(g, x, x);
  Moments acc{0.0, 0.0, 0.0};
  for (int sp = 0; sp < g.spw; ++sp) {
    const int64_t seg = ((int64_t)blockIdx.y * g.spw + sp) * kWarps + warp;
    if (seg >= g.nseg) break;
    Seg s;
    if (!decode_seg(g, seg, s)) continue;
    const IO* base = x + (int64_t)s.r * g.row + s.n * g.J + j;
    double xw[K];
    prime_window<K>(xw, base, step, s.s0, jv);
    const IO* p = base + s.s0 * step;
    double k0 = 0.0, s1 = 0.0, s2 = 0.0;  // k0: the segment's first h1, shift for the moments
    stream_any<8, false>(ring, ct, p, p, x, x, step, s.s0, s.s1, s.s1, [&](IO xv, IO, int64_t t, int64_t) {
      push<K>(xw, wide(xv));
      const double h1 = Carrier<IO>::round(conv_taps2<K>(w, xw));
      if (t == s.s0) k0 = h1;
      const double dl = h1 - k0;
      s1 += dl;
      s2 = fma(dl, dl, s2);
    });
    const double n = (double)(s.s1 - s.s0);
    Moments m{n, k0 + s1 / n, fmax(s2 - s1 * s1 / n, 0.0)};
    acc = merge(acc, m);
  }
  __shared__ double sh[3][kWarps][32];
  sh[0][warp][lane] = acc.n;
  sh[1][warp][lane] = acc.mean;
  sh[2][warp][lane] = acc.m2;
  __syncthreads();
  if (warp == 0) {
    Moments t{sh[0][0][lane], sh[1][0][lane], sh[2][0][lane]};
#pragma unroll
    for (int w2 = 1; w2 < kWarps; ++w2) t = merge(t, Moments{sh[0][w2][lane], sh[1][w2][lane], sh[2][w2][lane]});
    if (jv) {
      double* o = part + (int64_t)blockIdx.y * 3 * g.J + j;
      o[0] = t.n;
      o[g.J] = t.mean;
      o[2 * g.J] = t.m2;
    }
  }
}

// (partial row, spatial column) of flat index idx = r Q + q, advanced by 32 per
// lane step without a division in the loop (the folds walk rows * Q partials)
struct RowCol {
  int64_t r;
  int q, Q, dr, dq;
  __device__ RowCol(int lane, int Q_) : r(lane / Q_), q(lane % Q_), Q(Q_), dr(32 / Q_), dq(32 % Q_) {}
  __device__ void next() {
    r += dr;
    q += dq;
    if (q >= Q) {
      q -= Q;
      ++r;
    }
  }
};

// ------------------------------------------------------------------------------
// forward fold: one warp per channel (deterministic merge order)
// ------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) fwd_fold_kernel(Geom g, const double* __restrict__ part,
                                                            const double* __restrict__ W, int flags,
                                                            const double* __restrict__ gamma,
                                                            const double* __restrict__ beta,
                                                            double* __restrict__ running_mean,
                                                            double* __restrict__ running_var,
                                                            double eps, double momentum,
                                                            double* __restrict__ fold) {
  const int lane = threadIdx.x & 31;
  const int64_t c = (int64_t)blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (c >= g.C) return;
  const int K = g.k;
  Moments acc{0.0, 0.0, 0.0};
  const int64_t total = g.rows * g.Q;
  RowCol rq(lane, (int)g.Q);
  for (int64_t idx = lane; idx < total; idx += 32, rq.next()) {
    const double* p = part + rq.r * 3 * g.J + c * g.Q + rq.q;
    acc = merge(acc, Moments{p[0], p[g.J], p[2 * g.J]});
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    Moments o{__shfl_xor_sync(0xffffffffu, acc.n, off), __shfl_xor_sync(0xffffffffu, acc.mean, off),
              __shfl_xor_sync(0xffffffffu, acc.m2, off)};
    acc = (lane & off) ? merge(o, acc) : merge(acc, o);  // lower lane first on both sides
  }
  if (lane != 0) return;
  const bool smooth = flags & PSN_SMOOTH;
  const bool use_batch = flags & PSN_USE_BATCH_STATS;
  const bool quantize = (flags & PSN_QUANTIZED) && (!smooth || (flags & PSN_QUANTIZE_IN_SMOOTH));
  const double m = (double)(g.T * g.N * g.Q);
  const double mu_b = acc.mean;
  const double var_b = acc.m2 / m;
  const double rm_prev = running_mean[c], rv_prev = running_var[c];
  if (!smooth) {  // network.py:241-248
    const double unbiased = m > 1.0 ? var_b * (m / (m - 1.0)) : var_b;
    double rm = rm_prev * (1.0 - momentum);
    rm = rm + momentum * mu_b;
    double rv = rv_prev * (1.0 - momentum);
    rv = rv + momentum * unbiased;
    running_mean[c] = rm;
    running_var[c] = rv;
  }
  const double mu = use_batch ? mu_b : rm_prev;  // network.py:250-255
  const double var = use_batch ? var_b : rv_prev;
  const double s = sqrt(var + eps);
  const double a = gamma[c] / s;
  const double b_f = beta[c] - a * mu;
  const double* Wc = W + ((flags & PSN_SHARED) ? 0 : c * K);
  double* f = fold + c * PSN_FOLD_STRIDE(K);
  f[0] = mu;
  f[1] = s;
  f[2] = a;
  f[3] = b_f;
  f[4] = mu_b;
  f[5] = var_b;
  f[6] = 0.0;  // no BN-term data sums (the generic backward forms its own)
  for (int i = 0; i < K; ++i) {
    const double wf = a * Wc[i];
    f[PSN_FOLD_HDR + i] = wf;
    double wq = wf;
    if (quantize) {
      int sg, e;
      quantize_pow2(wf, sg, e);
      wq = ldexp((double)sg, e);
    }
    f[PSN_FOLD_HDR + K + i] = wq;
  }
}

// EVAL fold: running statistics (neuron.py:228-244, network.py:203-209, 219-234)
__global__ void eval_fold_kernel(Geom g, const double* __restrict__ W, int flags,
                                 const double* __restrict__ gamma, const double* __restrict__ beta,
                                 const double* __restrict__ running_mean,
                                 const double* __restrict__ running_var, double eps,
                                 double* __restrict__ fold) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= g.C) return;
  const int K = g.k;
  const double scale = gamma[c] / sqrt(running_var[c] + eps);
  const double b_f = beta[c] - scale * running_mean[c];
  const double* Wc = W + ((flags & PSN_SHARED) ? 0 : c * K);
  double* f = fold + c * PSN_FOLD_STRIDE(K);
  f[0] = running_mean[c];
  f[1] = 0.0;
  f[2] = scale;
  f[3] = (double)(float)b_f;  // the f32 bias a saved model carries
  f[4] = 0.0;
  f[5] = 0.0;
  for (int i = 0; i < K; ++i) {
    const double wf = Wc[i] * scale;
    f[PSN_FOLD_HDR + i] = wf;
    double wq;
    if (flags & PSN_QUANTIZED) {
      int sg, e;
      quantize_pow2(wf, sg, e);
      wq = ldexp((double)sg, e);
    } else {
      wq = (double)(float)wf;
    }
    f[PSN_FOLD_HDR + K + i] = wq;
  }
}

// ------------------------------------------------------------------------------
// forward pass 2: spikes
// MODE 0 = TRAIN (Heaviside), 1 = SMOOTH (spike_primitive), 2 = EVAL (x and h
// rounded to f32 like the reference's float32 deployment path)
// ------------------------------------------------------------------------------
template <int K, typename IO, int MODE>
__global__ void __launch_bounds__(kThreads, (K > 8 ? 1 : 2)) fwd_spike_kernel(Geom g, const IO* __restrict__ x,
                                                             const double* __restrict__ fold,
                                                             int skind, double alpha,
                                                             IO* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const bool jv = j < g.J;
  const int64_t c = jv ? j / g.Q : 0;
  const double* f = fold + c * PSN_FOLD_STRIDE(K);
  double wq[K];
#pragma unroll
  for (int i = 0; i < K; ++i) wq[i] = jv ? f[PSN_FOLD_HDR + K + i] : 0.0;
  const double bf = jv ? f[3] : 0.0;
  const int64_t step = (int64_t)g.d * g.row;
  extern __shared__ __align__(16) unsigned char psn_dsm[];
  IO* ring = reinterpret_cast<IO*>(psn_dsm) + warp * kRingSteps * 32;
  const ColTile ct = col_tile<IO>(g, x, x);
  for (int64_t seg = (int64_t)blockIdx.y * kWarps + warp; seg < g.nseg;
       seg += (int64_t)gridDim.y * kWarps) {
    Seg s;
    if (!decode_seg(g, seg, s)) continue;
    const int64_t off = (int64_t)s.r * g.row + s.n * g.J + j;
    const IO* base = x + off;
    double xw[K];
    if (MODE == 2) {
#pragma unroll
      for (int m = 1; m < K; ++m) {
        const int64_t sp = s.s0 - K + m;
        xw[m] = (jv && sp >= 0) ? Carrier<IO>::to_f32(load_wide(base + sp * step)) : 0.0;
      }
    } else {
      prime_window<K>(xw, base, step, s.s0, jv);
    }
    const IO* p = base + s.s0 * step;
    IO* o = out + off + s.s0 * step;
    stream_any<8, false>(ring, ct, p, p, x, x, step, s.s0, s.s1, s.s1, [&](IO xv, IO, int64_t, int64_t eo) {
      double v = wide(xv);
      if (MODE == 2) v = Carrier<IO>::to_f32(v);
      push<K>(xw, v);
      double h = __dadd_rn(conv_taps<K>(wq, xw), bf);
      h = (MODE == 2) ? (double)(float)h : Carrier<IO>::round(h);
      if (jv) {
        IO* ot = o + eo;
        if (MODE == 1)
          Carrier<IO>::store(ot, surrogate_primitive(skind, alpha, h));
        else
          Carrier<IO>::storef(ot, h >= 0.0 ? 1.0f : 0.0f);
      }
    });
  }
}

// ------------------------------------------------------------------------------
// backward pass 1: per-column reductions
// part3 layout: [rows][3K+1][J]: db, dwq[0..K), sx[0..K), sxc[0..K)
// ------------------------------------------------------------------------------
// dh2 = dy * sigma'(h2) on a prefetched dy element, in f64 like the reference
// (surrogate.py:36-38): the float64 carrier with the reference's own
// expressions, the f32 / bf16 carriers with a 2^-44-accurate reciprocal (an f32
// sigma' is off by up to an ulp per element, and the per-channel sums of
// 10^5..10^7 such terms drift by ~1e-5 relative)
template <typename IO>
__device__ __forceinline__ double dh2_val(const Surrogate& sur, int skind, double alpha, double h2, IO dyr) {
  if constexpr (std::is_same<IO, double>::value) {
    double sg;
    if (skind == PSN_ARCTAN) {
      const double u = 0.5 * 3.141592653589793 * alpha * h2;
      sg = alpha / (2.0 * (1.0 + u * u));
    } else {
      sg = 1.0 / (1.0 + alpha * h2 * h2);
    }
    return dyr * sg;
  } else {
    if (skind == PSN_ARCTAN) {
      const double u = (0.5 * 3.141592653589793 * alpha) * h2;
      return wide(dyr) * (0.5 * alpha) * rcp_f64(fma(u, u, 1.0));
    }
    return wide(dyr) * rcp_f64(fma(alpha * h2, h2, 1.0));
  }
}

template <int K, typename IO>
__global__ void __launch_bounds__(kThreads) bwd_reduce_kernel(Geom g, const IO* __restrict__ x,
                                                              const IO* __restrict__ dy,
                                                              const double* __restrict__ W,
                                                              int shared,
                                                              const double* __restrict__ fold,
                                                              Surrogate sur, int skind, double alpha,
                                                              double* __restrict__ part,
                                                              float* __restrict__ dhm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const bool jv = j < g.J;
  const int64_t c = jv ? j / g.Q : 0;
  const double* f = fold + c * PSN_FOLD_STRIDE(K);
  double w[K], wq[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    w[i] = jv ? W[(shared ? 0 : c) * K + i] : 0.0;
    wq[i] = jv ? f[PSN_FOLD_HDR + K + i] : 0.0;
  }
  const double bf = jv ? f[3] : 0.0;
  const double mu = jv ? f[0] : 0.0;
  const int64_t step = (int64_t)g.d * g.row;
  // sx[i] = sum_t x[t - (K-1-i)] is not accumulated per step: it is the
  // column's total minus, for every residue subsequence, its last K-1-i
  // values (taken from the window at the subsequence's end, kept in shared
  // memory; x before the stream start is zero).
  __shared__ double tails[K > 1 ? K - 1 : 1][kWarps][32];
  extern __shared__ __align__(16) unsigned char psn_dsm[];
  IO* ring = reinterpret_cast<IO*>(psn_dsm) + warp * 2 * kRingSteps * 32;
  const ColTile ct = col_tile<IO>(g, x, dy);
  const int64_t nel = g.T * g.row;
#pragma unroll
  for (int i = 0; i < K - 1; ++i) tails[i][warp][lane] = 0.0;
  double db = 0.0, xsum = 0.0, dwq[K], sxc[K];
#pragma unroll
  for (int i = 0; i < K; ++i) dwq[i] = sxc[i] = 0.0;
  for (int sp = 0; sp < g.spw; ++sp) {
    const int64_t seg = ((int64_t)blockIdx.y * g.spw + sp) * kWarps + warp;
    if (seg >= g.nseg) break;
    Seg s;
    if (!decode_seg(g, seg, s)) continue;
    const int64_t off = (int64_t)s.r * g.row + s.n * g.J + j;
    double xw[K];
    prime_window<K>(xw, x + off, step, s.s0, jv);
    const IO* p = x + off + s.s0 * step;
    const IO* q = dy + off + s.s0 * step;
    float* dm = dhm ? dhm + off + s.s0 * step : nullptr;  // materialised dh2 | h1 - mu for bwd_dx_mat
    stream_any<8, true>(ring, ct, p, q, x, dy, step, s.s0, s.s1, s.s1, [&](IO xv, IO dv, int64_t, int64_t eo) {
      const double v = wide(xv);
      push<K>(xw, v);
      xsum += v;
      const double h1 = Carrier<IO>::round(conv_taps2<K>(w, xw));
      const double h2 = Carrier<IO>::round(__dadd_rn(conv_taps2<K>(wq, xw), bf));
      const double dh2 = jv ? dh2_val<IO>(sur, skind, alpha, h2, dv) : 0.0;
      const double hc = h1 - mu;
      if (dm && jv) {
        dm[eo] = (float)dh2;
        dm[nel + eo] = (float)hc;
      }
      db += dh2;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        dwq[i] = fma(xw[i], dh2, dwq[i]);
        sxc[i] = fma(xw[i], hc, sxc[i]);
      }
    });
    if (s.s1 == s.Sr) {
      double run = 0.0;
#pragma unroll
      for (int i = K - 2; i >= 0; --i) {
        run += xw[i + 1];
        tails[i][warp][lane] += run;
      }
    }
  }
  // block reduction over warps in fixed order, 8 values per round
  constexpr int NV = 3 * K + 1;
  __shared__ double sh[kWarps][8][32];
  double* o = part + (int64_t)blockIdx.y * NV * g.J + j;
#pragma unroll
  for (int v0 = 0; v0 < NV; v0 += 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int v = v0 + u;
      double val = 0.0;
      if (v == 0) val = db;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (v == 1 + i) val = dwq[i];
        if (v == 1 + K + i) val = (i < K - 1) ? xsum - tails[i < K - 1 ? i : 0][warp][lane] : xsum;
        if (v == 1 + 2 * K + i) val = sxc[i];
      }
      sh[warp][u][lane] = val;
    }
    __syncthreads();
    if (warp < 8) {
      const int v = v0 + warp;  // each warp finalises one value
      if (v < NV) {
        double t = sh[0][warp][lane];
#pragma unroll
        for (int w2 = 1; w2 < kWarps; ++w2) t += sh[w2][warp][lane];
        if (jv) o[(int64_t)v * g.J] = t;
      }
    }
    __syncthreads();
  }
}

// backward fold: one block per channel, each warp sums some of the 3K+1
// values over the partial rows (lanes over rows, fixed-order shuffle tree),
// then one thread writes dW (per channel into dwtmp when shared), dgamma,
// dbeta and the BN-through-stats scalars (alpha1, beta1).
__global__ void __launch_bounds__(kThreads) bwd_fold_kernel(Geom g, const double* __restrict__ part,
                                                            const double* __restrict__ W, int flags,
                                                            const double* __restrict__ gamma,
                                                            const double* __restrict__ fold,
                                                            double* __restrict__ dW,
                                                            double* __restrict__ dgamma,
                                                            double* __restrict__ dbeta,
                                                            double* __restrict__ bfold) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c = blockIdx.x;
  const int K = g.k;
  const int NV = 3 * K + 1;
  __shared__ double tot[3 * PSN_MAX_ORDER + 1];
  const int64_t total = g.rows * g.Q;
  for (int v = warp; v < NV; v += kWarps) {
    double acc = 0.0;
    RowCol rq(lane, (int)g.Q);
    for (int64_t idx = lane; idx < total; idx += 32, rq.next())
      acc += part[(rq.r * NV + v) * g.J + c * g.Q + rq.q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double o = __shfl_xor_sync(0xffffffffu, acc, off);
      acc = (lane & off) ? o + acc : acc + o;
    }
    if (lane == 0) tot[v] = acc;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const double* f = fold + c * PSN_FOLD_STRIDE(K);
  const double mu = f[0], s = f[1], a = f[2];
  const bool quantized = (flags & PSN_QUANTIZED) &&
                         (!(flags & PSN_SMOOTH) || (flags & PSN_QUANTIZE_IN_SMOOTH));
  const double* Wc = W + ((flags & PSN_SHARED) ? 0 : c * K);
  const double db_f = tot[0];
  double da = 0.0;
  double dwf[PSN_MAX_ORDER];
  for (int i = 0; i < K; ++i) {
    double g1 = tot[1 + i];
    if (quantized && (flags & PSN_ROUND_STE)) {  // quant.py:194-216
      const double wf = f[PSN_FOLD_HDR + i], wq = f[PSN_FOLD_HDR + K + i];
      g1 = (wf != 0.0) ? g1 * (fabs(wq) / fabs(wf)) : 0.0;
    }
    dwf[i] = g1;
    da = da + dwf[i] * Wc[i];
  }
  da = da - db_f * mu;  // network.py:293
  double alpha1 = 0.0, beta1 = 0.0;
  if (flags & PSN_USE_BATCH_STATS) {  // network.py:298-315
    const double m = (double)(g.T * g.N * g.Q);
    const double ds = -da * gamma[c] / (s * s);
    const double dvar = ds / (2.0 * s);
    const double dmu = -db_f * a;
    alpha1 = dmu / m;
    beta1 = (2.0 / m) * dvar;
  }
  for (int i = 0; i < K; ++i) {
    double dw = a * dwf[i];
    if (flags & PSN_USE_BATCH_STATS) dw += alpha1 * tot[1 + K + i] + beta1 * tot[1 + 2 * K + i];
    dW[c * K + i] = dw;
  }
  dbeta[c] = db_f;
  dgamma[c] = da / s;
  bfold[2 * c] = alpha1;
  bfold[2 * c + 1] = beta1;
}

// shared-weight row sum over channels in fixed order (network.py:317)
__global__ void shared_rowsum_kernel(const double* __restrict__ dwtmp, int64_t C, int K,
                                     double* __restrict__ dW) {
  const int i = threadIdx.x;
  if (i >= K) return;
  double acc = 0.0;
  for (int64_t c = 0; c < C; ++c) acc += dwtmp[c * K + i];
  dW[i] = acc;
}

// ------------------------------------------------------------------------------
// backward pass 2: dx = sum_i w_q,i dh2[t+off_i] + W_i dh1[t+off_i]
// ------------------------------------------------------------------------------
template <int K, typename IO>
__global__ void __launch_bounds__(kThreads) bwd_dx_kernel(Geom g, const IO* __restrict__ x,
                                                          const IO* __restrict__ dy,
                                                          const double* __restrict__ W, int shared,
                                                          const double* __restrict__ fold,
                                                          const double* __restrict__ bfold,
                                                          Surrogate sur, int skind, double alpha,
                                                          IO* __restrict__ dx) {
  using Acc = typename std::conditional<std::is_same<IO, double>::value, double, float>::type;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const bool jv = j < g.J;
  const int64_t c = jv ? j / g.Q : 0;
  const double* f = fold + c * PSN_FOLD_STRIDE(K);
  double w[K], wq[K];
  Acc wa[K], wqa[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    w[i] = jv ? W[(shared ? 0 : c) * K + i] : 0.0;
    wq[i] = jv ? f[PSN_FOLD_HDR + K + i] : 0.0;
    wa[i] = (Acc)w[i];
    wqa[i] = (Acc)wq[i];
  }
  const double bf = jv ? f[3] : 0.0;
  const double mu = jv ? f[0] : 0.0;
  const double alpha1 = jv ? bfold[2 * c] : 0.0;
  const double beta1 = jv ? bfold[2 * c + 1] : 0.0;
  const int64_t step = (int64_t)g.d * g.row;
  extern __shared__ __align__(16) unsigned char psn_dsm[];
  IO* ring = reinterpret_cast<IO*>(psn_dsm) + warp * 2 * kRingSteps * 32;
  const ColTile ct = col_tile<IO>(g, x, dy);
  for (int64_t seg = (int64_t)blockIdx.y * kWarps + warp; seg < g.nseg;
       seg += (int64_t)gridDim.y * kWarps) {
    Seg s;
    if (!decode_seg(g, seg, s)) continue;
    const int64_t off = (int64_t)s.r * g.row + s.n * g.J + j;
    double xw[K];
    prime_window<K>(xw, x + off, step, s.s0, jv);
    Acc pacc[K];
#pragma unroll
    for (int i = 0; i < K; ++i) pacc[i] = (Acc)0;
    const IO* p = x + off + s.s0 * step;
    const IO* q = dy + off + s.s0 * step;
    IO* o = dx + off + (s.s0 - (K - 1)) * step;
    const int64_t tend = s.s1 + K - 1;
    const int64_t lim = tend < s.Sr ? tend : s.Sr;
    stream_any<8, true>(ring, ct, p, q, x, dy, step, s.s0, tend, lim, [&](IO xv, IO dv, int64_t t, int64_t eo) {
      Acc dh2 = (Acc)0, dh1 = (Acc)0;
      if (t < s.Sr) {
        push<K>(xw, wide(xv));
        const double h1 = Carrier<IO>::round(conv_taps2<K>(w, xw));
        const double h2 = Carrier<IO>::round(__dadd_rn(conv_taps2<K>(wq, xw), bf));
        dh2 = jv ? (Acc)dh2_val<IO>(sur, skind, alpha, h2, dv) : (Acc)0;
        dh1 = (Acc)(alpha1 + beta1 * (h1 - mu));
      }
#pragma unroll
      for (int i = 0; i < K; ++i) {
        pacc[i] = fma(wqa[i], dh2, pacc[i]);
        pacc[i] = fma(wa[i], dh1, pacc[i]);
      }
      if (t - (K - 1) >= s.s0 && jv) Carrier<IO>::store(o + eo, (double)pacc[0]);
#pragma unroll
      for (int i = 0; i < K - 1; ++i) pacc[i] = pacc[i + 1];
      pacc[K - 1] = (Acc)0;
    });
  }
}

// backward pass 2 from dh2 and h1 - mu materialised (f32) by bwd_reduce:
// dx[t] = sum_i w_q,i dh2[t+off_i] + W_i dh1[t+off_i], dh1 = alpha1 + beta1 (h1 - mu),
// FP32 only (the recomputing bwd_dx_kernel spends 2k DFMA per element on h1, h2)
template <int K, typename IO>
__global__ void __launch_bounds__(kThreads, 2) bwd_dx_mat_kernel(Geom g, const float* __restrict__ dhm,
                                                                 const double* __restrict__ W, int shared,
                                                                 const double* __restrict__ fold,
                                                                 const double* __restrict__ bfold,
                                                                 IO* __restrict__ dx) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const bool jv = j < g.J;
  const int64_t c = jv ? j / g.Q : 0;
  const double* f = fold + c * PSN_FOLD_STRIDE(K);
  float wa[K], wqa[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    wa[i] = jv ? (float)W[(shared ? 0 : c) * K + i] : 0.0f;
    wqa[i] = jv ? (float)f[PSN_FOLD_HDR + K + i] : 0.0f;
  }
  const float a1 = jv ? (float)bfold[2 * c] : 0.0f;
  const float b1 = jv ? (float)bfold[2 * c + 1] : 0.0f;
  const int64_t step = (int64_t)g.d * g.row;
  const int64_t nel = g.T * g.row;
  extern __shared__ __align__(16) unsigned char psn_dsm[];
  float* ring = reinterpret_cast<float*>(psn_dsm) + warp * 2 * kRingSteps * 32;
  const ColTile ct = col_tile<float>(g, dhm, dhm + nel);
  for (int64_t seg = (int64_t)blockIdx.y * kWarps + warp; seg < g.nseg;
       seg += (int64_t)gridDim.y * kWarps) {
    Seg s;
    if (!decode_seg(g, seg, s)) continue;
    const int64_t off = (int64_t)s.r * g.row + s.n * g.J + j;
    float pacc[K];
#pragma unroll
    for (int i = 0; i < K; ++i) pacc[i] = 0.0f;
    const float* p = dhm + off + s.s0 * step;
    IO* o = dx + off + (s.s0 - (K - 1)) * step;
    const int64_t tend = s.s1 + K - 1;
    const int64_t lim = tend < s.Sr ? tend : s.Sr;
    stream_any<8, true>(ring, ct, p, p + nel, dhm, dhm, step, s.s0, tend, lim,
                     [&](float d2, float hc, int64_t t, int64_t eo) {
      const float dh1 = (t < s.Sr) ? fmaf(b1, hc, a1) : 0.0f;  // d2 reads 0 there
#pragma unroll
      for (int i = 0; i < K; ++i) {
        pacc[i] = fmaf(wqa[i], d2, pacc[i]);
        pacc[i] = fmaf(wa[i], dh1, pacc[i]);
      }
      if (t - (K - 1) >= s.s0 && jv) Carrier<IO>::storef(o + eo, pacc[0]);
#pragma unroll
      for (int i = 0; i < K - 1; ++i) pacc[i] = pacc[i + 1];
      pacc[K - 1] = 0.0f;
    });
  }
}

// ------------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------------
inline dim3 grid_red(const Geom& g) { return dim3((unsigned)g.ctiles, (unsigned)g.rows); }
inline dim3 grid_map(const Geom& g) {
  int64_t y = (g.nseg + kWarps - 1) / kWarps;
  if (y > 65535) y = 65535;
  return dim3((unsigned)g.ctiles, (unsigned)y);
}

template <int K, typename IO>
int launch_forward(const psn_desc_t* desc, const Geom& g, const void* x, const double* W,
                   const double* gamma, const double* beta, double* rm, double* rv, void* out,
                   double* fold, char* ws, const WsLayout& L, cudaStream_t st) {
  double* part1 = (double*)(ws + L.part1);
  const int shared = (desc->flags & PSN_SHARED) ? 1 : 0;
  const size_t sm1 = ring_bytes<IO>(1);
  int rc;
  if ((rc = smem_optin(fwd_stats_kernel<K, IO>, sm1)) || (rc = smem_optin(fwd_spike_kernel<K, IO, 0>, sm1)) ||
      (rc = smem_optin(fwd_spike_kernel<K, IO, 1>, sm1)))
    return rc;
  fwd_stats_kernel<K, IO><<<grid_red(g), kThreads, sm1, st>>>(g, (const IO*)x, W, shared, part1);
  fwd_fold_kernel<<<(unsigned)((g.C + kWarps - 1) / kWarps), kThreads, 0, st>>>(
      g, part1, W, desc->flags, gamma, beta, rm, rv, desc->eps, desc->momentum, fold);
  if (desc->flags & PSN_SMOOTH)
    fwd_spike_kernel<K, IO, 1><<<grid_map(g), kThreads, sm1, st>>>(g, (const IO*)x, fold, desc->surrogate,
                                                                     desc->alpha, (IO*)out);
  else
    fwd_spike_kernel<K, IO, 0><<<grid_map(g), kThreads, sm1, st>>>(g, (const IO*)x, fold, desc->surrogate,
                                                                     desc->alpha, (IO*)out);
  return cuda_check("psn_forward_train");
}

template <int K, typename IO>
int launch_backward(const psn_desc_t* desc, const Geom& g, const void* x, const void* dy,
                    const double* W, const double* gamma, const double* fold, void* dx, double* dW,
                    double* dgamma, double* dbeta, char* ws, const WsLayout& L, cudaStream_t st) {
  double* part3 = (double*)(ws + L.part3);
  double* bfold = (double*)(ws + L.bfold);
  double* dwtmp = (double*)(ws + L.dwtmp);
  const int shared = (desc->flags & PSN_SHARED) ? 1 : 0;
  const Surrogate sur = make_surrogate(desc);
  float* dhm = L.dhm_bytes ? (float*)(ws + L.dhm) : nullptr;
  const size_t sm2 = ring_bytes<IO>(2), smf = ring_bytes<float>(2);
  int rc;
  if ((rc = smem_optin(bwd_reduce_kernel<K, IO>, sm2)) || (rc = smem_optin(bwd_dx_kernel<K, IO>, sm2)) ||
      (rc = smem_optin(bwd_dx_mat_kernel<K, IO>, smf)))
    return rc;
  bwd_reduce_kernel<K, IO><<<grid_red(g), kThreads, sm2, st>>>(g, (const IO*)x, (const IO*)dy, W, shared, fold,
                                                               sur, desc->surrogate, desc->alpha, part3, dhm);
  bwd_fold_kernel<<<(unsigned)g.C, kThreads, 0, st>>>(
      g, part3, W, desc->flags, gamma, fold, shared ? dwtmp : dW, dgamma, dbeta, bfold);
  if (shared) shared_rowsum_kernel<<<1, 32, 0, st>>>(dwtmp, g.C, K, dW);
  if (dhm)
    bwd_dx_mat_kernel<K, IO><<<grid_map(g), kThreads, smf, st>>>(g, dhm, W, shared, fold, bfold, (IO*)dx);
  else
    bwd_dx_kernel<K, IO><<<grid_map(g), kThreads, sm2, st>>>(g, (const IO*)x, (const IO*)dy, W, shared, fold,
                                                             bfold, sur, desc->surrogate, desc->alpha, (IO*)dx);
  return cuda_check("psn_backward");
}

template <int K, typename IO>
int launch_eval(const psn_desc_t* desc, const Geom& g, const void* x, const double* W,
                const double* gamma, const double* beta, const double* rm, const double* rv,
                void* out, double* fold, cudaStream_t st) {
  eval_fold_kernel<<<(unsigned)((g.C + 127) / 128), 128, 0, st>>>(g, W, desc->flags, gamma, beta, rm, rv,
                                                                   desc->eps, fold);
  const size_t sm1 = ring_bytes<IO>(1);
  if (int rc = smem_optin(fwd_spike_kernel<K, IO, 2>, sm1)) return rc;
  fwd_spike_kernel<K, IO, 2><<<grid_map(g), kThreads, sm1, st>>>(g, (const IO*)x, fold, desc->surrogate,
                                                                   desc->alpha, (IO*)out);
  return cuda_check("psn_forward_eval");
}

#define PSN_K_CASES(M) \
  M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15) M(16)

struct FwdOp {
  template <int K, typename IO, typename... A>
  static int run(A&&... a) { return launch_forward<K, IO>(a...); }
};
struct BwdOp {
  template <int K, typename IO, typename... A>
  static int run(A&&... a) { return launch_backward<K, IO>(a...); }
};
struct EvalOp {
  template <int K, typename IO, typename... A>
  static int run(A&&... a) { return launch_eval<K, IO>(a...); }
};

template <typename Op, typename IO, typename... A>
int by_k(int k, A&&... a) {
  switch (k) {
#define PSN_CASE(KK) \
  case KK:           \
    return Op::template run<KK, IO>(a...);
    PSN_K_CASES(PSN_CASE)
#undef PSN_CASE
  }
  return fail(PSN_ERR_ORDER, "order out of range");
}

template <typename Op, typename... A>
int by_dtype_k(const psn_desc_t* desc, A&&... a) {
  switch (desc->dtype) {
    case PSN_F32:
      return by_k<Op, float>(desc->k, a...);
    case PSN_BF16:
      return by_k<Op, __nv_bfloat16>(desc->k, a...);
    case PSN_F64:
      return by_k<Op, double>(desc->k, a...);
  }
  return fail(PSN_ERR_DTYPE, "unsupported carrier dtype");
}

}  // namespace psn

using namespace psn;

extern "C" {

const char* psn_last_error(void) { return g_last_error.c_str(); }
int psn_abi_version(void) { return PSN_ABI_VERSION; }
int psn_max_order(void) { return PSN_MAX_ORDER; }

size_t psn_fold_doubles(const psn_desc_t* desc) {
  if (!desc) return 0;
  return (size_t)desc->C * PSN_FOLD_STRIDE((size_t)desc->k);
}

size_t psn_workspace_bytes(const psn_desc_t* desc) {
  if (validate(desc, true) != PSN_OK) return 0;
  return ws_layout(desc).total;
}

int psn_forward_train(const psn_desc_t* desc, const void* x, const double* W, const double* gamma,
                      const double* beta, double* running_mean, double* running_var, void* out,
                      double* fold, void* workspace, psn_stream_t stream) {
  int rc = validate(desc, false);
  if (rc) return rc;
  const size_t es = dtype_size(desc->dtype);
  if ((rc = check_ptr(x, es, "x")) || (rc = check_ptr(out, es, "out")) || (rc = check_ptr(W, 8, "W")) ||
      (rc = check_ptr(gamma, 8, "gamma")) || (rc = check_ptr(beta, 8, "beta")) ||
      (rc = check_ptr(running_mean, 8, "running_mean")) || (rc = check_ptr(running_var, 8, "running_var")) ||
      (rc = check_ptr(fold, 8, "fold")) || (rc = check_ptr(workspace, 256, "workspace")))
    return rc;
  const Geom g = plan(desc);
  const WsLayout L = ws_layout(desc);
  stream::Plan P;
  if (stream::aligned_for_tma(x, out) && stream::make_plan(desc, false, P)) {
    rc = stream::forward(desc, P, x, W, gamma, beta, running_mean, running_var, out, fold,
                         (char*)workspace + L.fused, (cudaStream_t)stream);
    if (rc != stream::kFallback) return rc ? rc : cuda_check("psn_forward_train (stream)");
  }
  return by_dtype_k<FwdOp>(desc, desc, g, x, W, gamma, beta, running_mean, running_var, out, fold,
                           (char*)workspace, L, (cudaStream_t)stream);
}

int psn_backward(const psn_desc_t* desc, const void* x, const void* dy, const double* W,
                 const double* gamma, const double* fold, void* dx, double* dW, double* dgamma,
                 double* dbeta, void* workspace, psn_stream_t stream) {
  int rc = validate(desc, false);
  if (rc) return rc;
  const size_t es = dtype_size(desc->dtype);
  if ((rc = check_ptr(x, es, "x")) || (rc = check_ptr(dy, es, "dy")) || (rc = check_ptr(dx, es, "dx")) ||
      (rc = check_ptr(W, 8, "W")) || (rc = check_ptr(gamma, 8, "gamma")) || (rc = check_ptr(fold, 8, "fold")) ||
      (rc = check_ptr(dW, 8, "dW")) || (rc = check_ptr(dgamma, 8, "dgamma")) ||
      (rc = check_ptr(dbeta, 8, "dbeta")) || (rc = check_ptr(workspace, 256, "workspace")))
    return rc;
  const Geom g = plan(desc);
  const WsLayout L = ws_layout(desc);
  stream::Plan P;
  if (stream::aligned_for_tma(x, dy) && stream::make_plan(desc, true, P)) {
    double* dwtmp = (double*)((char*)workspace + L.dwtmp);
    const bool shared = desc->flags & PSN_SHARED;
    rc = stream::backward(desc, P, x, dy, W, gamma, fold, dx, shared ? dwtmp : dW, dgamma, dbeta,
                          (char*)workspace + L.fused, (cudaStream_t)stream);
    if (rc != stream::kFallback) {
      if (rc) return rc;
      if (shared) shared_rowsum_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(dwtmp, desc->C, desc->k, dW);
      return cuda_check("psn_backward (stream)");
    }
  }
  return by_dtype_k<BwdOp>(desc, desc, g, x, dy, W, gamma, fold, dx, dW, dgamma, dbeta, (char*)workspace, L,
                           (cudaStream_t)stream);
}

int psn_forward_eval(const psn_desc_t* desc, const void* x, const double* W, const double* gamma,
                     const double* beta, const double* running_mean, const double* running_var, void* out,
                     void* workspace, psn_stream_t stream) {
  int rc = validate(desc, false);
  if (rc) return rc;
  const size_t es = dtype_size(desc->dtype);
  if ((rc = check_ptr(x, es, "x")) || (rc = check_ptr(out, es, "out")) || (rc = check_ptr(W, 8, "W")) ||
      (rc = check_ptr(gamma, 8, "gamma")) || (rc = check_ptr(beta, 8, "beta")) ||
      (rc = check_ptr(running_mean, 8, "running_mean")) || (rc = check_ptr(running_var, 8, "running_var")) ||
      (rc = check_ptr(workspace, 256, "workspace")))
    return rc;
  const Geom g = plan(desc);
  double* fold = (double*)((char*)workspace + ws_layout(desc).evalfold);
  return by_dtype_k<EvalOp>(desc, desc, g, x, W, gamma, beta, running_mean, running_var, out, fold,
                            (cudaStream_t)stream);
}

// Execution plan of psn_forward_train (backward = 0) / psn_backward (1):
// info = {streamed (1) or generic (0), CTAs, groups, tiles per group, stages,
//         kernel launches per call (memsets included)}.
int psn_plan_info(const psn_desc_t* desc, int backward, int64_t* info, int n) {
  if (!desc || !info || n <= 0 || validate(desc, false) != PSN_OK) return 0;
  int64_t v[8] = {0, 0, 0, 0, 0, 3, 0, 0};
  const int rowsum = (backward && (desc->flags & PSN_SHARED)) ? 1 : 0;
  stream::Plan P;
  if (stream::make_plan(desc, backward != 0, P)) {
    v[0] = 1;
    v[1] = P.nCTA;
    v[2] = P.G;
    v[3] = P.tpg;
    v[4] = P.S;
    v[5] = 2 + rowsum;
    v[6] = P.nT;
    v[7] = P.lag;
  } else {
    v[5] = 3 + rowsum;
  }
  const int m = n < 8 ? n : 8;
  for (int i = 0; i < m; ++i) info[i] = v[i];
  return m;
}

}  // extern "C"
