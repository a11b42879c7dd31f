// psn_common.cuh — shared device/host helpers for the sm_100a PSN kernels.
//
// Data view used by every kernel: x is time-first [T, N, J] with J = C*Q
// columns (Q = product of spatial axes) and channel(j) = j / Q.  A "stream"
// is one (n, j) column walked along t.  Dilation d splits each stream into d
// residue subsequences t = r + s*d (r in [0, d)); inside a subsequence the
// dilated causal conv of order k is an UNdilated k-tap conv, so one register
// window of k values serves any dilation (reference engines.py:127-132 offset
// rule off_i = (k-1-i)*d becomes "tap i looks back k-1-i subsequence steps").
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/psn_b200.h"

namespace psn {

constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;

// ---- geometry ---------------------------------------------------------------
struct Geom {
  int64_t T, N, C, Q, J;  // J = C*Q columns
  int64_t row;            // elements per time step = N*J
  int d, k;
  int64_t S;              // ceil(T/d): length of the longest residue subsequence
  int64_t L;              // chunk length in subsequence steps
  int64_t nch;            // chunks per residue subsequence
  int64_t nseg;           // segments per column tile = N * d * nch
  int spw;                // segments per warp (reduction passes)
  int64_t rows;           // partial rows (gridDim.y) of reduction passes
  int64_t ctiles;         // column tiles of 32
};

struct Seg {
  int64_t n, s0, s1, Sr;
  int r;
};

// segment id -> (n, residue r, chunk); adjacent ids are adjacent time chunks
// of the same stream so their halos overlap in L1/L2.
__device__ __forceinline__ bool decode_seg(const Geom& g, int64_t seg, Seg& o) {
  const int64_t ch = seg % g.nch;
  const int64_t tmp = seg / g.nch;
  o.r = (int)(tmp % g.d);
  o.n = tmp / g.d;
  o.Sr = (o.r < g.T) ? (g.T - o.r + g.d - 1) / g.d : 0;
  o.s0 = ch * g.L;
  o.s1 = o.s0 + g.L < o.Sr ? o.s0 + g.L : o.Sr;
  return o.s0 < o.s1;
}

// ---- carrier dtypes -----------------------------------------------------------
// "round" is the reference's cast of the float64 accumulator back to the
// carrier (engines.py:104-106).  bf16 I/O computes with an f32 carrier: x is
// widened exactly, internal h1/h2 are f32-rounded, outputs are rounded to bf16.
template <typename IO>
struct Carrier;

template <>
struct Carrier<float> {
  static constexpr int kDtype = PSN_F32;
  __device__ __forceinline__ static float loadf(const float* p) { return __ldg(p); }
  __device__ __forceinline__ static double round(double h) { return (double)(float)h; }
  __device__ __forceinline__ static void store(float* p, double v) { *p = (float)v; }
  __device__ __forceinline__ static void storef(float* p, float v) { *p = v; }
  __device__ __forceinline__ static double to_f32(double v) { return v; }
};

template <>
struct Carrier<double> {
  static constexpr int kDtype = PSN_F64;
  __device__ __forceinline__ static double loadd(const double* p) { return __ldg(p); }
  __device__ __forceinline__ static double round(double h) { return h; }
  __device__ __forceinline__ static void store(double* p, double v) { *p = v; }
  __device__ __forceinline__ static void storef(double* p, float v) { *p = (double)v; }
  __device__ __forceinline__ static double to_f32(double v) { return (double)(float)v; }
};

template <>
struct Carrier<__nv_bfloat16> {
  static constexpr int kDtype = PSN_BF16;
  __device__ __forceinline__ static float loadf(const __nv_bfloat16* p) {
    return __bfloat162float(__ldg(p));
  }
  __device__ __forceinline__ static double round(double h) { return (double)(float)h; }
  __device__ __forceinline__ static void store(__nv_bfloat16* p, double v) {
    *p = __float2bfloat16_rn((float)v);
  }
  __device__ __forceinline__ static void storef(__nv_bfloat16* p, float v) {
    *p = __float2bfloat16_rn(v);
  }
  __device__ __forceinline__ static double to_f32(double v) { return v; }
};

// load one carrier element widened to f64 (exact for all carriers)
__device__ __forceinline__ double load_wide(const float* p) { return (double)__ldg(p); }
__device__ __forceinline__ double load_wide(const double* p) { return __ldg(p); }
__device__ __forceinline__ double load_wide(const __nv_bfloat16* p) {
  return (double)__bfloat162float(__ldg(p));
}
__device__ __forceinline__ float load_f(const float* p) { return __ldg(p); }
__device__ __forceinline__ float load_f(const double* p) { return (float)__ldg(p); }
__device__ __forceinline__ float load_f(const __nv_bfloat16* p) {
  return __bfloat162float(__ldg(p));
}

// ---- statistics merge (Chan et al.) --------------------------------------------
struct Moments {
  double n, mean, m2;
};

__device__ __forceinline__ Moments merge(const Moments& a, const Moments& b) {
  if (a.n == 0.0) return b;
  if (b.n == 0.0) return a;
  Moments o;
  o.n = a.n + b.n;
  const double delta = b.mean - a.mean;
  o.mean = a.mean + delta * (b.n / o.n);
  o.m2 = a.m2 + b.m2 + delta * delta * (a.n * b.n / o.n);
  return o;
}

// ---- exact power-of-two quantizer (reference quant.py:111-139) ----------------
// |w| = m * 2^q with m in [0.5, 1): nearest exponent is q-1 below sqrt(1/2) and
// q at or above it; 0x3FE6A09E667F3BCD is the smallest double >= sqrt(1/2).
__device__ __forceinline__ void quantize_pow2(double w, int& sgn, int& e) {
  if (w == 0.0) {
    sgn = 0;
    e = 0;
    return;
  }
  sgn = w > 0.0 ? 1 : -1;
  int q;
  const double m = frexp(fabs(w), &q);
  e = q - 1 + (m >= __longlong_as_double(0x3FE6A09E667F3BCDLL) ? 1 : 0);
  e = e < -16 ? -16 : (e > 15 ? 15 : e);
}

// ---- surrogate derivative (reference surrogate.py:32-39), f32 -------------------
struct Surrogate {
  int kind;       // PSN_ARCTAN / PSN_RATIONAL
  float c;        // arctan: pi*alpha/2 ; rational: alpha
  float scale;    // arctan: alpha/2    ; rational: 1
};

__device__ __forceinline__ float rcp_approx(float v) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ float surrogate_grad(const Surrogate& s, float h) {
  const float t = s.c * h;
  return s.scale * rcp_approx(fmaf(t, s.kind == PSN_ARCTAN ? t : h, 1.0f));
}

// spike_primitive (surrogate.py:42-54) in f64 for SMOOTH mode
__device__ __forceinline__ double surrogate_primitive(int kind, double alpha, double h) {
  const double pi = 3.141592653589793;
  if (kind == PSN_ARCTAN) return atan(0.5 * pi * alpha * h) / pi + 0.5;
  const double r = sqrt(alpha);
  return atan(r * h) / r + 0.5;
}

// ---- host-side helpers shared by the translation units (psn_layer.cu) ----------
int fail(int code, const char* msg);
int cuda_check(const char* where);
Geom plan(const psn_desc_t* desc);
int validate(const psn_desc_t* d, bool allow_i32);
int check_ptr(const void* p, size_t align, const char* what);
size_t dtype_size(int dt);
size_t workspace_part3_offset(const psn_desc_t* desc);
size_t workspace_dwtmp_offset(const psn_desc_t* desc);

}  // namespace psn
