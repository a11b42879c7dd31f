/*
 * psn_b200.h — C ABI of the B200-native mul-free channel-wise Parallel Spiking
 * Neuron (arXiv 2501.14490), the drop-in for the reference's hot path.
 *
 * Plain C: caller-owned device pointers, sizes, an explicit CUDA stream and an
 * int status.  No torch types, no C++ exceptions cross this boundary, no
 * allocation or global mutable state inside (re-entrant per stream).
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/shiftsnn/):
 *   psn_forward_train   SpikingLayer.forward(x, Mode.TRAIN|SMOOTH)   network.py:213-217, 236-268
 *                        (conv_forward x2, batch_stats, running update, BN fold,
 *                         quantize_pow2, Heaviside / spike_primitive)
 *   psn_backward        SpikingLayer.backward(dy)                     network.py:272-318
 *                        (spike_backward, conv_backward_{bias,weight,input} x2,
 *                         quantize_backward, BN-through-stats terms)
 *   psn_forward_eval    SpikingLayer._forward_eval / ShiftLayer.forward network.py:219-234, 351-359
 *   psn_conv_forward    engines.conv_forward(engine=DIRECT)            engines.py:117-138, 336-347
 *   psn_conv_forward_shift      engines.conv_forward_shift (float)    engines.py:258-294
 *   psn_shift_spike_forward     ShiftLayer.forward (shift conv + spike) network.py:352-362
 *   psn_conv_forward_shift_int  engines.conv_forward_shift (int32)    engines.py:297-325
 *   psn_conv_backward_input     engines.conv_backward_input           engines.py:350-377
 *   psn_conv_backward_weight    engines.conv_backward_weight          engines.py:402-425
 *   psn_conv_backward_bias      engines.conv_backward_bias            engines.py:428-431
 *   psn_quantize_pow2           quant.quantize_pow2                   quant.py:111-139
 *   psn_readout_reduce  ReadoutLayer.forward (leaky accumulator)      network.py:399-419
 *   psn_readout_expand  ReadoutLayer.backward (dcur -> dx)            network.py:421-436
 *   psn_adam_step       Adam.step over all parameter tensors           train.py:147-172
 *
 * Tensor layout: time-first, contiguous [T, N, C, Q] where Q is the product of
 * the spatial axes (1 for rank-3 [T, N, C]); reference tensor.py:71-81.
 * Per-channel parameters and statistics are float64 like the reference's.
 */
#ifndef PSN_B200_H
#define PSN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define PSN_API __attribute__((visibility("default")))
#else
#define PSN_API
#endif

/* == cudaStream_t; declared opaquely so this header needs no CUDA headers */
typedef struct CUstream_st *psn_stream_t;

#define PSN_ABI_VERSION 2
#define PSN_MAX_ORDER 16

typedef enum {
  PSN_OK = 0,
  PSN_ERR_INVALID = 1,     /* bad descriptor / shape / pointer  (ValueError) */
  PSN_ERR_DTYPE = 2,       /* unsupported carrier dtype         (TypeError)  */
  PSN_ERR_ORDER = 3,       /* order k above PSN_MAX_ORDER       (ValueError) */
  PSN_ERR_CUDA = 4,        /* CUDA launch / runtime failure     (RuntimeError) */
  PSN_ERR_ALIGN = 5        /* pointer misaligned for its dtype  (ValueError) */
} psn_status_t;

typedef enum { PSN_F32 = 0, PSN_BF16 = 1, PSN_F64 = 2, PSN_I32 = 3 } psn_dtype_t;

typedef enum { PSN_ARCTAN = 0, PSN_RATIONAL = 1 } psn_surrogate_t;   /* surrogate.py:17-19 */

typedef enum {
  PSN_QUANTIZED = 1,               /* NeuronConfig.quantized                       */
  PSN_SHARED = 2,                  /* WeightSharing.SHARED: W is [1, k]            */
  PSN_USE_BATCH_STATS = 4,         /* SpikingLayer.fuse_from_batch_stats           */
  PSN_SMOOTH = 8,                  /* Mode.SMOOTH: primitive output, stats frozen  */
  PSN_QUANTIZE_IN_SMOOTH = 16,     /* SpikingLayer.quantize_in_smooth_mode         */
  PSN_ROUND_STE = 32,              /* QuantGradMode.ROUND_STE (else WHOLE_STE)     */
  PSN_GENERIC = 64,                /* force the three-launch kernels (no streamed  */
                                   /* kernel); part of the descriptor so that the  */
                                   /* workspace size and the call agree            */
  PSN_STREAM = 128                 /* streamed kernels whenever the shape allows   */
                                   /* them (skip the small-size / wide-window      */
                                   /* preference for the three-launch kernels)     */
} psn_flag_t;

typedef struct {
  int64_t T, N, C, Q;   /* x is [T, N, C, Q], time-major, contiguous          */
  int32_t k;            /* order (taps), 1..PSN_MAX_ORDER                     */
  int32_t d;            /* dilation >= 1                                      */
  int32_t dtype;        /* psn_dtype_t of x / dy / spikes / dx                */
  int32_t flags;        /* OR of psn_flag_t                                    */
  int32_t surrogate;    /* psn_surrogate_t                                     */
  int32_t reserved;
  double alpha;         /* surrogate sharpness (SurrogateConfig.alpha)        */
  double eps;           /* BN epsilon (ThresholdParams.eps, 1e-5)             */
  double momentum;      /* BN momentum (ThresholdParams.momentum, 0.1)        */
} psn_desc_t;

/* Per-channel forward state ("fold") the backward consumes; float64,
 * psn_fold_doubles(desc) values = C * PSN_FOLD_STRIDE(k), row c:
 *   [mu*, s, a, b_f, mu_batch, var_batch, bn_sums, w_f[0..k), w_q[0..k),
 *    Sx[0..k), Cx[0..k)]
 * Sx[i] = sum_(t,n,q) x[t-off_i] and Cx[i] = sum x[t-off_i] (h1[t] - mu_batch)
 * are the data terms of the BN-through-statistics weight gradient
 * (network.py:298-315); the streamed forward writes them (bn_sums = 1) and the
 * streamed backward requires them (it traps if bn_sums != 1).                  */
#define PSN_FOLD_HDR 7
#define PSN_FOLD_STRIDE(k) (PSN_FOLD_HDR + 4 * (k))

PSN_API const char *psn_last_error(void);          /* thread-local message of last failure */
PSN_API int psn_abi_version(void);
PSN_API int psn_max_order(void);

PSN_API size_t psn_fold_doubles(const psn_desc_t *desc);
PSN_API size_t psn_workspace_bytes(const psn_desc_t *desc);

/* TRAIN (or SMOOTH when desc->flags has PSN_SMOOTH) forward.
 *   x            [T,N,C,Q] carrier dtype
 *   W            [C,k] or [1,k] (PSN_SHARED) f64
 *   gamma, beta  [C] f64
 *   running_mean, running_var  [C] f64, updated in place in TRAIN mode
 *   out          [T,N,C,Q] carrier dtype: spikes (0/1) or spike_primitive(h2)
 *   fold         psn_fold_doubles(desc) f64, written (consumed by psn_backward)
 *   workspace    psn_workspace_bytes(desc) bytes, scratch                        */
PSN_API int psn_forward_train(const psn_desc_t *desc, const void *x, const double *W,
                      const double *gamma, const double *beta,
                      double *running_mean, double *running_var,
                      void *out, double *fold, void *workspace, psn_stream_t stream);

/* Backward of the last psn_forward_train with the same x / fold.
 *   dy           [T,N,C,Q] carrier dtype
 *   dx           [T,N,C,Q] carrier dtype (written)
 *   dW           [C,k] or [1,k] f64 (written, not accumulated)
 *   dgamma, dbeta [C] f64 (written)                                              */
PSN_API int psn_backward(const psn_desc_t *desc, const void *x, const void *dy,
                 const double *W, const double *gamma, const double *fold,
                 void *dx, double *dW, double *dgamma, double *dbeta,
                 void *workspace, psn_stream_t stream);

/* EVAL forward: running statistics folded into the weights, pow2-quantized and
 * shift-executed when PSN_QUANTIZED; x is rounded to f32 like the reference.    */
PSN_API int psn_forward_eval(const psn_desc_t *desc, const void *x, const double *W,
                     const double *gamma, const double *beta,
                     const double *running_mean, const double *running_var,
                     void *out, void *workspace, psn_stream_t stream);

/* Execution plan of psn_forward_train (backward = 0) / psn_backward (1):
 * info[0] = 1 if the persistent fused kernel runs (else the generic 3-kernel path),
 * info[1] = CTAs, info[2] = channel groups, info[3] = 32-column tiles per group,
 * info[4] = pipeline stages, info[5] = kernel launches per call (memsets included),
 * info[6] = CTA teams (groups streamed concurrently), info[7] = pass-2 lag in groups.
 * Returns the number of entries written (<= n).                                  */
PSN_API int psn_plan_info(const psn_desc_t *desc, int backward, int64_t *info, int n);

/* ---- engine-level operators (the reference's plugin functions) ---------- */
/* w: [w_rows, k] f64 with w_rows in {1, C}; bias: [C] f64 or NULL.
 * Carrier dtype F32 or F64; accumulation f64 in reference tap order.         */
PSN_API int psn_conv_forward(const psn_desc_t *desc, const void *x, const double *w,
                     int64_t w_rows, const double *bias, void *out, psn_stream_t stream);
/* sign/exponent: [w_rows, k] int8 (ShiftWeights); float carrier (ldexp).     */
PSN_API int psn_conv_forward_shift(const psn_desc_t *desc, const void *x, const int8_t *sign,
                           const int8_t *exponent, int64_t w_rows, const double *bias,
                           void *out, psn_stream_t stream);
/* the same membrane, thresholded in the same pass: out = (carrier(h) >= 0) as
 * 0 / 1 in the carrier dtype (the deserialised quantized model's layer).      */
PSN_API int psn_shift_spike_forward(const psn_desc_t *desc, const void *x, const int8_t *sign,
                            const int8_t *exponent, int64_t w_rows, const double *bias,
                            void *out, psn_stream_t stream);
/* int32 carrier: arithmetic shifts, int64 accumulation, bias truncated to
 * int64, clip to int32; *saturations (device u64) incremented per clip.      */
PSN_API int psn_conv_forward_shift_int(const psn_desc_t *desc, const int32_t *x, const int8_t *sign,
                               const int8_t *exponent, int64_t w_rows, const double *bias,
                               int32_t *out, unsigned long long *saturations,
                               psn_stream_t stream);
PSN_API int psn_conv_backward_input(const psn_desc_t *desc, const void *dh, const double *w,
                            int64_t w_rows, void *out, psn_stream_t stream);
/* grad: [C, k] f64, or [1, k] when shared != 0; workspace >= psn_workspace_bytes */
PSN_API int psn_conv_backward_weight(const psn_desc_t *desc, const void *x, const void *dh,
                             int shared, double *grad, void *workspace, psn_stream_t stream);
/* grad: [C] f64 */
PSN_API int psn_conv_backward_bias(const psn_desc_t *desc, const void *dh, double *grad,
                           void *workspace, psn_stream_t stream);
/* n float64 weights -> int8 sign / exponent (exact nearest pow2, clamp [-16, 15]) */
PSN_API int psn_quantize_pow2(const double *w, int64_t n, int8_t *sign, int8_t *exponent,
                      psn_stream_t stream);

/* ---- readout leaky accumulator (network.py:365-436) --------------------- */
/* The readout's v = (1 - 1/tau) v + (1/tau) cur[t] over t, with the linear
 * cur[t] = x[t] W^T + b, equals xbar W^T + b sum_t w_t with
 *   xbar[n, c] = sum_t w_t x[t, n, c],  w_t = (1/tau) (1 - 1/tau)^(T-1-t).
 * psn_readout_reduce: x [T, N, C] (dtype f32 / bf16 / f64) -> xbar [N, C] f64.
 * psn_readout_expand: backward, dx[t, n, c] = w_t g[n, c] for g = dlogits W
 *   ([N, C] f64) -> dx [T, N, C] in dtype.  tau > 1 (else PSN_ERR_INVALID).  */
PSN_API int psn_readout_reduce(int64_t T, int64_t N, int64_t C, int32_t dtype, double tau,
                               const void *x, double *xbar, psn_stream_t stream);
PSN_API int psn_readout_expand(int64_t T, int64_t N, int64_t C, int32_t dtype, double tau,
                               const double *g, void *dx, psn_stream_t stream);

/* ---- Adam (train.py:147-172) -------------------------------------------- */
/* One chunk = n contiguous float64 elements of a parameter, its gradient and
 * its two moment buffers.  The table lives in device memory (one block per
 * chunk).  The update is the reference's element-wise sequence, bitwise:
 *   m = m b1 + (1-b1) g;  v = v b2 + ((1-b2) g) g;
 *   p -= (lr (m / c1)) / (sqrt(v / c2) + eps)
 * with c1, c2 = 1 - beta^t from the host, or, when t_dev is non-null, from
 * the device step count *t_dev (for a step captured in a CUDA graph).      */
typedef struct {
  double *param;
  const double *grad;
  double *m;
  double *v;
  int64_t n;
} psn_adam_chunk_t;
PSN_API int psn_adam_step(const psn_adam_chunk_t *chunks, int64_t n_chunks, double lr, double beta1,
                          double beta2, double eps, double c1, double c2, const double *t_dev,
                          psn_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* PSN_B200_H */
