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
// the same on register values (prefetched raw carrier elements)
__device__ __forceinline__ double wide(float v) { return (double)v; }
__device__ __forceinline__ double wide(double v) { return v; }
__device__ __forceinline__ double wide(__nv_bfloat16 v) { return (double)__bfloat162float(v); }
__device__ __forceinline__ float as_f(float v) { return v; }
__device__ __forceinline__ float as_f(double v) { return (float)v; }
__device__ __forceinline__ float as_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename IO>
__device__ __forceinline__ IO io_zero() { return IO(0); }
template <>
__device__ __forceinline__ __nv_bfloat16 io_zero<__nv_bfloat16>() { return __float2bfloat16_rn(0.0f); }

// Walk one column of x (and dy when DY) over subsequence steps [t0, t1) with
// U loads of each stream in flight: f(xv, dyv, t, eo) runs for every step in
// order, eo = (t - t0) * step the step's element offset from px; steps at or
// beyond `lim` (or an invalid column) read as zero.  px / pq point at step t0,
// consecutive steps are `step` elements apart.  The U-deep register prefetch
// keeps enough bytes in flight per SM for HBM (a load consumed by the next
// instruction stalls the warp for the full memory latency); full chunks of U
// steps call f unconditionally so the callers' shifting register windows are
// renamed rather than moved.
template <int U, bool DY, typename IO, typename F>
__device__ __forceinline__ void stream_col(const IO* px, const IO* pq, int64_t step, int64_t t0,
                                           int64_t t1, int64_t lim, bool jv, F&& f) {
  IO bx[U], bq[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const bool ok = jv && t0 + u < lim;
    bx[u] = ok ? __ldg(px + u * step) : io_zero<IO>();
    bq[u] = (DY && ok) ? __ldg(pq + u * step) : io_zero<IO>();
  }
  const int64_t ustep = (int64_t)U * step;
  int64_t t = t0, eo = 0;
  for (; t + U <= t1; t += U) {
    IO cx[U], cq[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      cx[u] = bx[u];
      cq[u] = bq[u];
    }
    const IO* nx = px + eo + ustep;
    const IO* nq = pq + eo + ustep;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = jv && t + U + u < lim;
      bx[u] = ok ? __ldg(nx + u * step) : io_zero<IO>();
      bq[u] = (DY && ok) ? __ldg(nq + u * step) : io_zero<IO>();
    }
#pragma unroll
    for (int u = 0; u < U; ++u) f(cx[u], cq[u], t + u, eo + u * step);
    eo += ustep;
  }
  // tail (< U steps): already in bx / bq
#pragma unroll
  for (int u = 0; u < U - 1; ++u)
    if (t + u < t1) f(bx[u], bq[u], t + u, eo + u * step);
}

// ---- per-warp shared-memory ring (cp.async) -------------------------------------
// Each lane copies ITS OWN column element of every step into the warp's ring
// and later reads it back itself, so no lane-to-lane synchronisation is needed
// (cp.async.wait_group is per thread).  CH steps per commit group (also the
// compute unroll), kRingSteps / CH groups in the ring, all but one in flight:
// kRingSteps - CH steps of every stream in flight per warp without holding
// registers.
constexpr int kRingSteps = 32;

// per-lane copies need a 4 / 8 B element (cp.async has no 2-byte form); bf16
// rings run in the 16-byte-piece mode only
template <typename IO>
__host__ __device__ constexpr bool ring_scalar_ok() { return sizeof(IO) >= 4; }
template <typename IO>
__host__ __device__ constexpr size_t ring_bytes(int streams) {  // dynamic shared memory of one block
  return (size_t)streams * kWarps * kRingSteps * 32 * sizeof(IO);
}

template <int BYTES>
__device__ __forceinline__ void cp_async_elem(void* sdst, const void* gsrc, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  const int n = ok ? BYTES : 0;  // 0 source bytes: the destination is zero-filled
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(sa), "l"(gsrc), "n"(BYTES), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// A lane's view of its 32-column tile: its lane index, whether its own column
// exists, how many columns of the tile exist, and whether the tile's rows may
// be moved as 16-byte pieces (every stream 16-B aligned, J a multiple of the
// elements per piece, so a piece is wholly inside or outside the tile).
struct ColTile {
  int lane, nvalid;
  bool jv, vec;
};
template <typename IO>
__device__ __forceinline__ ColTile col_tile(const Geom& g, const void* a, const void* b) {
  ColTile t;
  t.lane = threadIdx.x & 31;
  const int64_t j0 = (int64_t)blockIdx.x * 32;
  t.nvalid = (int)(g.J - j0 < 32 ? g.J - j0 : 32);
  t.jv = t.lane < t.nvalid;
  t.vec = (g.J % (16 / (int)sizeof(IO)) == 0) && ((((uintptr_t)a) | ((uintptr_t)b)) & 15) == 0;
  return t;
}

// stream_col through the ring: rx / rq are this warp's rings ([kRingSteps][32]
// elements each), gx / gq any valid global address (source of the zero-byte
// copies for steps that read as zero).  Scalar mode: every lane copies its own
// column (no lane-to-lane hand-off).  Vector mode: 16-B pieces, 32 / (16 / es)
// lanes per step row, lanes read rows other lanes copied, so the warp
// synchronises after each wait and before each refill.
template <int kRingCH, bool DY, typename IO, typename F>
__device__ __forceinline__ void stream_ring(IO* rx, IO* rq, const ColTile& ct, const IO* px, const IO* pq,
                                            const IO* gx, const IO* gq, int64_t step, int64_t t0,
                                            int64_t t1, int64_t lim, F&& f) {
  constexpr int kRingN = kRingSteps / kRingCH;
  constexpr int EPP = 16 / (int)sizeof(IO);  // elements per 16-B piece
  constexpr int LPS = 32 / EPP;              // lanes per step row
  constexpr int SPI = 32 / LPS;              // step rows per warp-wide copy
  static_assert(kRingCH % SPI == 0, "chunk must be a multiple of the rows per copy");
  const int lane = ct.lane;
  const int nchunks = (int)((t1 - t0 + kRingCH - 1) / kRingCH);
  const int64_t cstep = (int64_t)kRingCH * step;
  // vector mode: this lane copies piece pc of rows su, su + SPI, ...
  const int su = lane / LPS, pc = lane % LPS;
  const bool pok = pc * EPP < ct.nvalid;
  const IO* vx = px - lane + pc * EPP;  // tile start + piece
  const IO* vq = pq - lane + pc * EPP;
  int64_t ie = 0;  // element offset (from px) of the next chunk to issue
  int ic = 0;      // next chunk to issue
  auto issue = [&]() {
    if (ic < nchunks) {
      const int base = (ic & (kRingN - 1)) * kRingCH;
      const int64_t tb = t0 + (int64_t)ic * kRingCH;
      if (ct.vec) {
#pragma unroll
        for (int u0 = 0; u0 < kRingCH; u0 += SPI) {
          const int u = u0 + su;
          const bool ok = pok && tb + u < lim;
          const int64_t e = ie + u * step;
          cp_async_elem<16>(rx + (base + u) * 32 + pc * EPP, ok ? vx + e : gx, ok);
          if (DY) cp_async_elem<16>(rq + (base + u) * 32 + pc * EPP, ok ? vq + e : gq, ok);
        }
      } else if constexpr (ring_scalar_ok<IO>()) {
#pragma unroll
        for (int u = 0; u < kRingCH; ++u) {
          const bool ok = ct.jv && tb + u < lim;
          const int64_t e = ie + u * step;
          cp_async_elem<sizeof(IO)>(rx + (base + u) * 32 + lane, ok ? px + e : gx, ok);
          if (DY) cp_async_elem<sizeof(IO)>(rq + (base + u) * 32 + lane, ok ? pq + e : gq, ok);
        }
      }
    }
    cp_async_commit();
    ++ic;
    ie += cstep;
  };
#pragma unroll
  for (int c = 0; c < kRingN - 1; ++c) issue();
  int64_t eo = 0;
  for (int c = 0; c < nchunks; ++c) {
    if (ct.vec) __syncwarp();  // every lane is done with the slot about to be refilled
    issue();
    cp_async_wait<kRingN - 1>();
    if (ct.vec) __syncwarp();  // rows copied by other lanes are visible
    const int base = (c & (kRingN - 1)) * kRingCH;
    const int64_t tc = t0 + (int64_t)c * kRingCH;
    const IO* sx = rx + base * 32 + lane;
    const IO* sq = rq + base * 32 + lane;
    if (tc + kRingCH <= t1) {
#pragma unroll
      for (int u = 0; u < kRingCH; ++u) f(sx[u * 32], DY ? sq[u * 32] : io_zero<IO>(), tc + u, eo + u * step);
    } else {
#pragma unroll
      for (int u = 0; u < kRingCH; ++u)
        if (tc + u < t1) f(sx[u * 32], DY ? sq[u * 32] : io_zero<IO>(), tc + u, eo + u * step);
    }
    eo += cstep;
  }
  cp_async_wait<0>();
  if (ct.vec) __syncwarp();  // the ring is reused by the warp's next segment
}

// the streaming loop of the generic kernels: the shared-memory ring for 4 / 8 B
// carriers, and for bf16 tiles that move as 16-byte pieces (8 rows per warp
// copy, so chunks of 8); the register prefetch for the other bf16 tiles.
// `ring` is this warp's slice of the block's dynamic shared memory (2
// streams when DY).  CH: steps per chunk (unrolled; 8 at every order: at
// k = 16 the longer unroll beats the lower register pressure of 4,
// k = 16 d = 3 f32 0.81 -> 0.77 ms).
template <int CH, bool DY, typename IO, typename F>
__device__ __forceinline__ void stream_any(IO* ring, const ColTile& ct, const IO* px, const IO* pq, const IO* gx,
                                           const IO* gq, int64_t step, int64_t t0, int64_t t1, int64_t lim,
                                           F&& f) {
  if constexpr (ring_scalar_ok<IO>()) {
    stream_ring<CH, DY>(ring, ring + kRingSteps * 32, ct, px, pq, gx, gq, step, t0, t1, lim, f);
  } else if constexpr (CH % 8 == 0) {
    if (ct.vec)
      stream_ring<CH, DY>(ring, ring + kRingSteps * 32, ct, px, pq, gx, gq, step, t0, t1, lim, f);
    else
      stream_col<4, DY>(px, pq, step, t0, t1, lim, ct.jv, f);
  } else {
    stream_col<4, DY>(px, pq, step, t0, t1, lim, ct.jv, f);
  }
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
// 1/v to ~2^-44 relative: MUFU.RCP64H seed (~2^-22) and one Newton step
__device__ __forceinline__ double rcp_f64(double v) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v));
  const double e = fma(-v, r, 1.0);
  return fma(r, e, r);
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

// static + dynamic shared memory above the 48 KB default needs the per-kernel
// opt-in (the rings add to kernels that also hold static reduction buffers)
template <typename Kern>
int smem_optin(Kern* kern, size_t bytes) {
  if (bytes == 0) return PSN_OK;
  if (cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) !=
      cudaSuccess)
    return fail(PSN_ERR_CUDA, "cudaFuncSetAttribute (generic kernel smem) failed");
  return PSN_OK;
}
size_t workspace_dwtmp_offset(const psn_desc_t* desc);

}  // namespace psn
