// psn_stream.cuh — TMA-staged, persistent sm_100a kernels for the PSN TRAIN
// forward and backward (reference network.py:236-318).  Included by the
// psn_stream_*.cu instantiation units; host planning lives in psn_stream.cu.
//
// Why this shape.  The BN batch statistics put a per-channel reduction over
// ALL (t, n) between the two halves of each direction (forward: stats of h1
// -> spikes from h2; backward: db/dw sums -> dx).  Streaming x (and dy) twice
// from HBM costs 32 B/elem against the 20 B/elem algorithmic minimum (f32).
// So the channels are cut into groups of 32 columns (one 128-byte row segment
// per (t, n)), small enough that a group's x (+dy) stays in the 126 MB L2
// between its two passes, and the passes are software-pipelined over groups
// inside one cooperative launch (one CTA per SM):
//
//     iteration it:  pass1(it)  |  fold(it-1) on its folder CTAs  |  pass2(it-LAG)
//
// pass1 streams group `it` from HBM (TMA, L2 evict_last) and publishes per-CTA
// partial sums; fold(g) (tiny, fixed-order f64 sums over the per-CTA slots)
// runs on F statically chosen folder CTAs one iteration later; pass2 re-reads
// group it-LAG from L2 (TMA, evict_first) and writes spikes / dx.
//
// Inside a CTA: warp 8 is the TMA producer (one elected lane issues
// cp.async.bulk.tensor into a ring of S stages guarded by full/empty
// mbarriers; the warp also gathers each segment's per-channel parameters into
// the stage), warps 0..7 consume.  A tile is a TMA box [32 columns][8 batch
// rows][TB time steps] of the time-major tensor; lane = column (channel),
// warp = batch row, and each thread walks its (n, c) stream down the tile
// with a register window of the last H = (K-1)*D inputs, so every element is
// read from shared memory once and the dilated taps are register renames.  A
// thread keeps its window across consecutive tiles of its tile range; where a
// range starts mid-stream a HEAD item (H rows before the tile) primes it, and
// where the backward's dx range ends mid-stream a TAIL item (H rows after)
// supplies the future dh the time-reversed conv needs.
//
// Work is assigned statically (contiguous tile ranges per CTA, rotated per
// group so remainders spread), so every per-channel sum is formed in a fixed
// order: results are bit-reproducible run to run.
#pragma once

#include <cuda.h>
#include <stdio.h>

#include <type_traits>

#include "psn_common.cuh"

namespace psn {
namespace stream {

constexpr int kConsumerWarps = 8;
constexpr int kThreads = (kConsumerWarps + 1) * 32;
constexpr int kCols = 32;                        // columns per tile (lanes)
constexpr int kRedBytes = 8 * kConsumerWarps * 32 * (int)sizeof(double);  // 16 KB
constexpr int kMaxH = 24;                        // largest (k-1)*d on this path

#ifndef PSN_WAIT_LIMIT_NS
#define PSN_WAIT_LIMIT_NS 4000000000ull
#endif

// -------------------------------------------------------------------------
// plan + arguments (plain data, passed by value)
// -------------------------------------------------------------------------
struct Plan {
  int T, N, J, C;  // J = C (Q == 1 on this path)
  int k, d, H;
  int TB;          // time rows per tile
  int G;           // groups of 32 columns
  int nbk;         // ceil(N / 8)
  int ttl;         // ceil(T / TB)
  int tpg;         // tiles per group = nbk * ttl
  int P;           // workers per (pass, group) = min(nCTA, tpg)
  int F;           // folder CTAs per group
  int nCTA;
  int lag;         // pass2 runs `lag` iterations behind pass1 (>= 1)
  int S;           // pipeline stages
  int stage_bytes;
};

struct Args {
  Plan p;
  void* out;              // spikes (forward) or dx (backward), carrier dtype
  const double* W;        // [C,k] or [1,k]
  const double* gamma;
  const double* beta;
  double* rm;             // running mean / var (forward, updated by the fold)
  double* rv;
  double* fold;           // [C][PSN_FOLD_HDR + 2k] (written by forward, read by backward)
  double* dW;             // [C,k] (or per-channel scratch when shared)
  double* dgamma;
  double* dbeta;
  double* bfold;          // [C][2] backward BN-through-stats scalars (alpha1, beta1)
  double* part;           // [G][NV][32][P] per-CTA partial sums
  unsigned* cnt;          // [G] pass-1 arrivals
  unsigned* fdone;        // [G] folder completions
  int flags;
  int shared;
  double eps, momentum;
  Surrogate sur;    // f32 surrogate (dx pass)
  double sc, sscale; // f64 surrogate: arctan c = pi*alpha/2, scale = alpha/2; rational c = alpha, scale = 1
  int skind;
};

// -------------------------------------------------------------------------
// PTX helpers
// -------------------------------------------------------------------------
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
static __device__ __noinline__ void expired(const char* what, int a, int b) {
  printf("psn stream kernel: wait '%s' expired (block %d thread %d, %d/%d)\n", what, (int)blockIdx.x,
         (int)threadIdx.x, a, b);
  __trap();
}

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, unsigned bytes) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(su32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(su32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  if (mbar_try(b, parity)) return;
  const unsigned long long t0 = gtimer();
  while (!mbar_try(b, parity))
    if (gtimer() - t0 > PSN_WAIT_LIMIT_NS) expired("mbarrier", (int)parity, 0);
}

__device__ __forceinline__ uint64_t pol_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 3-D tiled TMA load (coordinates innermost first) completing on `bar`
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(su32(dst)),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void red_release(unsigned* a, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(a), "r"(v) : "memory");
}
// one thread waits for a grid counter (co-residency is guaranteed by the
// cooperative launch); callers publish the result with a CTA barrier
__device__ __forceinline__ void wait_counter(const unsigned* a, unsigned target, const char* what) {
  if (ld_acquire(a) >= target) return;
  const unsigned long long t0 = gtimer();
  unsigned v;
  while ((v = ld_acquire(a)) < target) {
    __nanosleep(64);
    if (gtimer() - t0 > PSN_WAIT_LIMIT_NS) expired(what, (int)v, (int)target);
  }
}

__device__ __forceinline__ void consumer_sync() {  // named barrier over the 8 consumer warps
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
}

// streaming stores of the outputs (L2 evict_first: keep the resident groups)
__device__ __forceinline__ void st_out(float* a, float v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_out(__nv_bfloat16* a, float v, uint64_t pol) {
  const __nv_bfloat16 b = __float2bfloat16_rn(v);
  const unsigned short u = *reinterpret_cast<const unsigned short*>(&b);
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.u16 [%0], %1, %2;" ::"l"(a), "h"(u), "l"(pol) : "memory");
}

__device__ __forceinline__ float lds(const float* p) { return *p; }
__device__ __forceinline__ float lds(const __nv_bfloat16* p) { return __bfloat162float(*p); }

// exact (double)(float)h with two DADDs (F2F.F32.F64 issues at ~8/clk/SM on
// B200, DADD at 64): adding M = 1.5 * 2^(E+29) puts the rounding point of the
// sum at ulp_f32(h); ties-to-even is preserved, f32 denormals included
__device__ __forceinline__ double round_f32(double h) {
  unsigned ex = (unsigned)__double2hiint(h) & 0x7ff00000u;
  ex = ex < 0x38100000u ? 0x38100000u : ex;
  const double M = __hiloint2double((int)(ex + (29u << 20) + 0x00080000u), 0);
  return __dsub_rn(__dadd_rn(h, M), M);
}

// 1/v to ~2^-44 relative: MUFU.RCP64H seed (~2^-22) and one Newton step
__device__ __forceinline__ double rcp_f64(double v) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v));
  const double e = fma(-v, r, 1.0);
  return fma(r, e, r);
}

// -------------------------------------------------------------------------
// configuration per (order, dilation, carrier, direction)
// -------------------------------------------------------------------------
template <int K, int D, typename IO, bool BWD>
struct Cfg {
  static constexpr int H = (K - 1) * D;
  static constexpr int NV = BWD ? 3 * K + 1 : 2;
  static constexpr int ES = (int)sizeof(IO);
  static constexpr int TB = BWD ? (ES == 4 ? 16 : 32) : (ES == 4 ? 32 : 64);
  static constexpr int XROWS = TB > H ? TB : H;
  static constexpr int ROWB = kConsumerWarps * kCols * ES;  // bytes of one time row of a box
  static constexpr int XBYTES = XROWS * ROWB;
  static constexpr int DBYTES = BWD ? XROWS * ROWB : 0;
  // per-lane parameter bytes: fwd f64 {w or w_q}[K] + {shift or b_f}; bwd f64 w_q[K], b_f + f32 W[K], mu, a1, b1
  static constexpr int PSTRIDE = BWD ? (8 * (K + 1) + 4 * (K + 3) + 15) / 16 * 16 : 8 * (K + 1);
  static constexpr int PBYTES = kCols * PSTRIDE;
  static constexpr int STAGE = ((XBYTES + DBYTES + PBYTES) + 1023) / 1024 * 1024;
  static_assert(H <= kMaxH, "window above the streamed-path limit");
};

// tap i reads x[t - (K-1-i)*D] = window slot H - (K-1-i)*D
template <int K, int D>
__device__ __forceinline__ constexpr int slot(int i) {
  return (K - 1) * D - (K - 1 - i) * D;
}

// -------------------------------------------------------------------------
// static schedule, shared by the producer and the consumers
// -------------------------------------------------------------------------
__device__ __forceinline__ int worker_of(const Plan& p, int g, int pass) {
  const int rot = (int)(((long long)g * 61 + pass * 29) % p.nCTA);
  return ((int)blockIdx.x - rot + p.nCTA) % p.nCTA;
}
__device__ __forceinline__ int folder_of(const Plan& p, int g, int f) {
  return (int)(((long long)g * p.F + f) % p.nCTA);
}

enum ItemKind { kHead = 0, kTile = 1, kTail = 2 };

// -------------------------------------------------------------------------
// the kernel
// -------------------------------------------------------------------------
template <int K, int D, typename IO, bool BWD>
__global__ void __launch_bounds__(kThreads, 1)
    psn_stream_kernel(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap mxh,
                      const __grid_constant__ CUtensorMap my, const __grid_constant__ CUtensorMap myh,
                      const Args a) {
  using C_ = Cfg<K, D, IO, BWD>;
  constexpr int H = C_::H, NV = C_::NV, TB = C_::TB;
  const Plan& p = a.p;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  double* red = (double*)(smem + (size_t)p.S * C_::STAGE);
  uint64_t* full = (uint64_t*)(smem + (size_t)p.S * C_::STAGE + kRedBytes);
  uint64_t* empty = full + p.S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int iters = p.G + p.lag;

  if (warp == kConsumerWarps) {
    // ======================= producer warp =======================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mx) : "memory");
      if (H > 0) asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mxh) : "memory");
      if (BWD) asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&my) : "memory");
      if (BWD && H > 0) asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&myh) : "memory");
    }
    const uint64_t pol_keep = pol_evict_last(), pol_drop = pol_evict_first(), pol_norm = pol_evict_normal();
    int q = 0;
    auto issue = [&](int kind, int pass, int g, int nbi, int trow, bool params) {
      const int s = q % p.S;
      if (q >= p.S) {
        if (lane == 0) mbar_wait(empty + s, (unsigned)(((q / p.S) - 1) & 1));
        __syncwarp();
      }
      unsigned char* st = smem + (size_t)s * C_::STAGE;
      if (params) {
        // per-channel parameters of this segment, one lane per column
        const int c = g * kCols + lane;
        const bool cv = c < p.C;
        const int cc = cv ? c : 0;
        const int wr = a.shared ? 0 : cc;
        unsigned char* pr = st + C_::XBYTES + C_::DBYTES + lane * C_::PSTRIDE;
        const double* f = a.fold + (size_t)cc * (PSN_FOLD_HDR + 2 * K);
        if (!BWD) {
          double* pd = (double*)pr;
          if (pass == 0) {
#pragma unroll
            for (int i = 0; i < K; ++i) pd[i] = cv ? __ldg(a.W + (size_t)wr * K + i) : 0.0;
            pd[K] = cv ? __ldcg(a.rm + cc) : 0.0;  // shift of the pass-1 moments
          } else {
#pragma unroll
            for (int i = 0; i < K; ++i) pd[i] = cv ? __ldcg(f + PSN_FOLD_HDR + K + i) : 0.0;
            pd[K] = cv ? __ldcg(f + 3) : 0.0;
          }
        } else {
          double* pd = (double*)pr;
          float* pf = (float*)(pr + 8 * (K + 1));
#pragma unroll
          for (int i = 0; i < K; ++i) {
            pd[i] = cv ? __ldg(f + PSN_FOLD_HDR + K + i) : 0.0;  // w_q
            pf[i] = cv ? (float)__ldg(a.W + (size_t)wr * K + i) : 0.0f;
          }
          pd[K] = cv ? __ldg(f + 3) : 0.0;                  // b_f
          pf[K] = cv ? (float)__ldg(f + 0) : 0.0f;          // mu*
          pf[K + 1] = (cv && pass == 1) ? (float)__ldcg(a.bfold + 2 * (size_t)cc) : 0.0f;
          pf[K + 2] = (cv && pass == 1) ? (float)__ldcg(a.bfold + 2 * (size_t)cc + 1) : 0.0f;
        }
        __syncwarp();
      }
      if (lane == 0) {
        const uint64_t pol = (kind == kTile) ? (pass == 0 ? pol_keep : pol_drop) : (pass == 0 ? pol_keep : pol_norm);
        const int c0 = g * kCols, n0 = nbi * kConsumerWarps;
        if (kind == kTile) {
          mbar_arrive_tx(full + s, (unsigned)(TB * C_::ROWB * (BWD ? 2 : 1)));
          tma_load3(st, &mx, c0, n0, trow, full + s, pol);
          if (BWD) tma_load3(st + C_::XBYTES, &my, c0, n0, trow, full + s, pol);
        } else if (kind == kHead) {
          mbar_arrive_tx(full + s, (unsigned)(H * C_::ROWB));
          tma_load3(st, &mxh, c0, n0, trow, full + s, pol);
        } else {
          mbar_arrive_tx(full + s, (unsigned)(2 * H * C_::ROWB));
          tma_load3(st, &mxh, c0, n0, trow, full + s, pol);
          tma_load3(st + C_::XBYTES, &myh, c0, n0, trow, full + s, pol);
        }
      }
      __syncwarp();
      ++q;
    };
    for (int it = 0; it < iters; ++it) {
      for (int pass = 0; pass < 2; ++pass) {
        const int g = pass == 0 ? it : it - p.lag;
        if (g < 0 || g >= p.G) continue;
        const int v = worker_of(p, g, pass);
        if (v >= p.P) continue;
        if (pass == 1) {  // the fold of group g must be complete before its parameters are read
          if (lane == 0) wait_counter(a.fdone + g, (unsigned)p.F, "fold done");
          __syncwarp();
        }
        const int t_a = (int)((long long)v * p.tpg / p.P), t_b = (int)((long long)(v + 1) * p.tpg / p.P);
        bool params = true;
        for (int tile = t_a; tile < t_b; ++tile) {
          const int nbi = tile / p.ttl, tt = tile % p.ttl, t0 = tt * TB;
          if constexpr (H > 0) if (tile == t_a && t0 > 0) {
            issue(kHead, pass, g, nbi, t0 - H, params);
            params = false;
          }
          issue(kTile, pass, g, nbi, t0, params);
          params = false;
          if (BWD && H > 0 && pass == 1 && tile == t_b - 1 && t0 + TB < p.T) issue(kTail, pass, g, nbi, t0 + TB, false);
        }
      }
    }
    return;
  }

  // ======================= consumer warps =======================
  const int n_in = warp;  // batch row within the tile
  const uint64_t pol_out = pol_evict_first();
  int q = 0;
  auto wait_item = [&]() -> unsigned char* {
    const int s = q % p.S;
    mbar_wait(full + s, (unsigned)((q / p.S) & 1));
    return smem + (size_t)s * C_::STAGE;
  };
  auto release_item = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + (q % p.S));
    ++q;
  };
  const size_t rowstride = (size_t)p.N * p.J;
  const unsigned mN = (unsigned)p.N;

  for (int it = 0; it < iters; ++it) {
    // ------------------------------------------------------------- pass 1
    if (it < p.G) {
      const int g = it;
      const int v = worker_of(p, g, 0);
      if (v < p.P) {
        const int col = g * kCols + lane;
        const int t_a = (int)((long long)v * p.tpg / p.P), t_b = (int)((long long)(v + 1) * p.tpg / p.P);
        double acc[NV];
#pragma unroll
        for (int u = 0; u < NV; ++u) acc[u] = 0.0;
        if constexpr (!BWD) {
          double w[K], sh = 0.0, xw[H + 1];
          for (int tile = t_a; tile < t_b; ++tile) {
            const int nbi = tile / p.ttl, tt = tile % p.ttl, t0 = tt * TB;
            const bool lv = (unsigned)(nbi * kConsumerWarps + n_in) < mN && col < p.J;
            if (tile == t_a || tt == 0) {
#pragma unroll
              for (int j = 0; j <= H; ++j) xw[j] = 0.0;
            }
            if constexpr (H > 0) if (tile == t_a && t0 > 0) {
              const unsigned char* st = wait_item();
              if (tile == t_a) {
                const double* pd = (const double*)(st + C_::XBYTES + C_::DBYTES + lane * C_::PSTRIDE);
#pragma unroll
                for (int i = 0; i < K; ++i) w[i] = pd[i];
                sh = pd[K];
              }
              const IO* xs = (const IO*)st + n_in * kCols + lane;
#pragma unroll
              for (int r = 0; r < H; ++r) {
#pragma unroll
                for (int j = 0; j < H; ++j) xw[j] = xw[j + 1];
                xw[H - 1] = (double)lds(xs + r * kConsumerWarps * kCols);
              }
              release_item();
            }
            const unsigned char* st = wait_item();
            if (tile == t_a && !(H > 0 && t0 > 0)) {
              const double* pd = (const double*)(st + C_::XBYTES + C_::DBYTES + lane * C_::PSTRIDE);
#pragma unroll
              for (int i = 0; i < K; ++i) w[i] = pd[i];
              sh = pd[K];
            }
            const IO* xs = (const IO*)st + n_in * kCols + lane;
            const int nvalid = lv ? min(TB, p.T - t0) : 0;
            double S1 = 0.0, S2 = 0.0;
#pragma unroll
            for (int r = 0; r < TB; ++r) {
              xw[H] = (double)lds(xs + r * kConsumerWarps * kCols);
              double h = 0.0;
#pragma unroll
              for (int i = 0; i < K; ++i) h = fma(w[i], xw[slot<K, D>(i)], h);
              const double h1 = round_f32(h);
              const double hc = (r < nvalid) ? h1 - sh : 0.0;
              S1 += hc;
              S2 = fma(hc, hc, S2);
#pragma unroll
              for (int j = 0; j < H; ++j) xw[j] = xw[j + 1];
            }
            acc[0] += S1;
            acc[1] += S2;
            release_item();
          }
        } else {
          // db, dw_q: f64 end to end (h2 exact and f32-rounded like the reference's
          // carrier, sigma' and dh2 in f64) -- f32 per-element errors (~1e-7)
          // would grow to ~sqrt(m)*1e-7 in these m-term sums, above the 1e-5
          // absolute bound on small dW entries; the BN-term sums sx, sxc reach dW
          // through 1/m-scaled factors and use f32 within a tile.
          float w[K], mu = 0.f, xw[H + 1];
          double wq[K], bf = 0.0, xd[H + 1];
          for (int tile = t_a; tile < t_b; ++tile) {
            const int nbi = tile / p.ttl, tt = tile % p.ttl, t0 = tt * TB;
            if (tile == t_a || tt == 0) {
#pragma unroll
              for (int j = 0; j <= H; ++j) {
                xw[j] = 0.f;
                xd[j] = 0.0;
              }
            }
            auto load_params = [&](const unsigned char* st) {
              const unsigned char* pr = st + C_::XBYTES + C_::DBYTES + lane * C_::PSTRIDE;
              const double* pd = (const double*)pr;
              const float* pf = (const float*)(pr + 8 * (K + 1));
#pragma unroll
              for (int i = 0; i < K; ++i) {
                wq[i] = pd[i];
                w[i] = pf[i];
              }
              bf = pd[K];
              mu = pf[K];
            };
            if constexpr (H > 0) if (tile == t_a && t0 > 0) {
              const unsigned char* st = wait_item();
              load_params(st);
              const IO* xs = (const IO*)st + n_in * kCols + lane;
#pragma unroll
              for (int r = 0; r < H; ++r) {
#pragma unroll
                for (int j = 0; j < H; ++j) {
                  xw[j] = xw[j + 1];
                  xd[j] = xd[j + 1];
                }
                xw[H - 1] = lds(xs + r * kConsumerWarps * kCols);
                xd[H - 1] = (double)xw[H - 1];
              }
              release_item();
            }
            const unsigned char* st = wait_item();
            if (tile == t_a && !(H > 0 && t0 > 0)) load_params(st);
            const IO* xs = (const IO*)st + n_in * kCols + lane;
            const IO* ys = (const IO*)(st + C_::XBYTES) + n_in * kCols + lane;
            const int nvalid = min(TB, p.T - t0);
            float fsx[K], fsc[K];
#pragma unroll
            for (int i = 0; i < K; ++i) fsx[i] = fsc[i] = 0.f;
#pragma unroll
            for (int r = 0; r < TB; ++r) {
              xw[H] = lds(xs + r * kConsumerWarps * kCols);
              xd[H] = (double)xw[H];
              const bool ok = r < nvalid;
              const double yv = ok ? (double)lds(ys + r * kConsumerWarps * kCols) : 0.0;
              double h2 = 0.0;  // exact: power-of-two products
#pragma unroll
              for (int i = 0; i < K; ++i) h2 = fma(wq[i], xd[slot<K, D>(i)], h2);
              h2 = round_f32(__dadd_rn(h2, bf));
              const double tq = a.sc * h2;
              const double den = fma(tq, a.skind == PSN_ARCTAN ? tq : h2, 1.0);
              const double dh = yv * rcp_f64(den);  // dh2 / scale (scale applied in the fold)
              acc[0] += dh;
#pragma unroll
              for (int i = 0; i < K; ++i) acc[1 + i] = fma(xd[slot<K, D>(i)], dh, acc[1 + i]);
              float h1 = 0.f;
#pragma unroll
              for (int i = 0; i < K; ++i) h1 = fmaf(w[i], xw[slot<K, D>(i)], h1);
              const float hc = ok ? h1 - mu : 0.f;
              const float okf = ok ? 1.f : 0.f;
#pragma unroll
              for (int i = 0; i < K; ++i) {
                const float xi = xw[slot<K, D>(i)];
                fsx[i] = fmaf(xi, okf, fsx[i]);
                fsc[i] = fmaf(xi, hc, fsc[i]);
              }
#pragma unroll
              for (int j = 0; j < H; ++j) {
                xw[j] = xw[j + 1];
                xd[j] = xd[j + 1];
              }
            }
#pragma unroll
            for (int i = 0; i < K; ++i) {
              acc[1 + K + i] += (double)fsx[i];
              acc[1 + 2 * K + i] += (double)fsc[i];
            }
            release_item();
          }
        }
        // ---- CTA reduction over the 8 batch rows, fixed order; one slot per worker
#pragma unroll
        for (int v0 = 0; v0 < NV; v0 += 8) {
          consumer_sync();
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (v0 + u < NV) red[(warp * 8 + u) * 32 + lane] = acc[v0 + u];
          consumer_sync();
          if (v0 + warp < NV) {
            double t = red[(0 * 8 + warp) * 32 + lane];
#pragma unroll
            for (int w2 = 1; w2 < kConsumerWarps; ++w2) t += red[(w2 * 8 + warp) * 32 + lane];
            a.part[(((size_t)g * NV + v0 + warp) * kCols + lane) * p.P + v] = t;
          }
        }
        consumer_sync();
        if (threadIdx.x == 0) red_release(a.cnt + g, 1u);
      }
    }
    // ------------------------------------------------------------- fold of group it-1
    if (it >= 1 && it - 1 < p.G) {
      const int g = it - 1;
      for (int f = 0; f < p.F; ++f) {
        if (folder_of(p, g, f) != (int)blockIdx.x) continue;
        consumer_sync();  // `red` is free
        if (threadIdx.x == 0) wait_counter(a.cnt + g, (unsigned)p.P, "pass-1 partials");
        consumer_sync();
        const int cpf = kCols / p.F;
        const int ntask = cpf * NV;
        const int qn = (p.P + 31) / 32;
        double* tot = red;  // [cpf][NV]
        for (int tb = warp * 4; tb < ntask; tb += kConsumerWarps * 4) {
          double sums[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int task = tb + u;
            double s = 0.0;
            if (task < ntask) {
              const int chl = f * cpf + task / NV, val = task % NV;
              const double* src = a.part + (((size_t)g * NV + val) * kCols + chl) * p.P;
              double vals[5];
#pragma unroll
              for (int j = 0; j < 5; ++j) {
                const int vv = lane + 32 * j;
                vals[j] = (j < qn && vv < p.P) ? __ldcg(src + vv) : 0.0;
              }
#pragma unroll
              for (int j = 0; j < 5; ++j) s += vals[j];
            }
            sums[u] = s;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
              const double o = __shfl_xor_sync(0xffffffffu, sums[u], off);
              sums[u] = (lane & off) ? o + sums[u] : sums[u] + o;
            }
            if (lane == 0 && tb + u < ntask) tot[tb + u] = sums[u];
          }
        }
        consumer_sync();
        if ((int)threadIdx.x < cpf) {
          const int c = g * kCols + f * cpf + threadIdx.x;
          if (c < p.C) {
            const double* tt = tot + threadIdx.x * NV;
            const double* Wc = a.W + (a.shared ? 0 : (size_t)c * K);
            double* fr = a.fold + (size_t)c * (PSN_FOLD_HDR + 2 * K);
            const int flags = a.flags;
            const double m = (double)p.T * (double)p.N;
            if constexpr (!BWD) {
              const bool smooth = flags & PSN_SMOOTH;
              const bool use_batch = flags & PSN_USE_BATCH_STATS;
              const bool quantize = (flags & PSN_QUANTIZED) && (!smooth || (flags & PSN_QUANTIZE_IN_SMOOTH));
              const double rm_prev = a.rm[c], rv_prev = a.rv[c];
              const double dmean = tt[0] / m;
              const double mu_b = rm_prev + dmean;  // the pass-1 shift was running_mean (pre-update)
              double var_b = tt[1] / m - dmean * dmean;
              var_b = var_b < 0.0 ? 0.0 : var_b;
              if (!smooth) {  // network.py:241-248
                const double unbiased = m > 1.0 ? var_b * (m / (m - 1.0)) : var_b;
                double r1 = rm_prev * (1.0 - a.momentum);
                r1 = r1 + a.momentum * mu_b;
                double r2 = rv_prev * (1.0 - a.momentum);
                r2 = r2 + a.momentum * unbiased;
                a.rm[c] = r1;
                a.rv[c] = r2;
              }
              const double mu = use_batch ? mu_b : rm_prev;  // network.py:250-255
              const double var = use_batch ? var_b : rv_prev;
              const double s = sqrt(var + a.eps);
              const double aa = a.gamma[c] / s;
              fr[0] = mu;
              fr[1] = s;
              fr[2] = aa;
              fr[3] = a.beta[c] - aa * mu;
              fr[4] = mu_b;
              fr[5] = var_b;
              for (int i = 0; i < K; ++i) {
                const double wf = aa * Wc[i];
                fr[PSN_FOLD_HDR + i] = wf;
                double wq = wf;
                if (quantize) {
                  int sg, e;
                  quantize_pow2(wf, sg, e);
                  wq = ldexp((double)sg, e);
                }
                fr[PSN_FOLD_HDR + K + i] = wq;
              }
            } else {
              const double mu = fr[0], s = fr[1], aa = fr[2];
              const bool quantized =
                  (flags & PSN_QUANTIZED) && (!(flags & PSN_SMOOTH) || (flags & PSN_QUANTIZE_IN_SMOOTH));
              const double db_f = tt[0] * a.sscale;
              double da = 0.0, dwf[K];
              for (int i = 0; i < K; ++i) {  // quantize_backward, quant.py:194-216
                double g1 = tt[1 + i] * a.sscale;
                if (quantized && (flags & PSN_ROUND_STE)) {
                  const double wf = fr[PSN_FOLD_HDR + i], wq = fr[PSN_FOLD_HDR + K + i];
                  g1 = (wf != 0.0) ? g1 * (fabs(wq) / fabs(wf)) : 0.0;
                }
                dwf[i] = g1;
                da = da + dwf[i] * Wc[i];
              }
              da = da - db_f * mu;  // network.py:291-296
              double alpha1 = 0.0, beta1 = 0.0;
              if (flags & PSN_USE_BATCH_STATS) {  // network.py:298-315
                const double ds = -da * a.gamma[c] / (s * s);
                const double dvar = ds / (2.0 * s);
                const double dmu = -db_f * aa;
                alpha1 = dmu / m;
                beta1 = (2.0 / m) * dvar;
              }
              for (int i = 0; i < K; ++i) {
                double dw = aa * dwf[i];
                if (flags & PSN_USE_BATCH_STATS) dw += alpha1 * tt[1 + K + i] + beta1 * tt[1 + 2 * K + i];
                a.dW[(size_t)c * K + i] = dw;
              }
              a.dbeta[c] = db_f;
              a.dgamma[c] = da / s;
              a.bfold[2 * (size_t)c] = alpha1;
              a.bfold[2 * (size_t)c + 1] = beta1;
            }
          }
        }
        consumer_sync();
        if (threadIdx.x == 0) red_release(a.fdone + g, 1u);
      }
    }
    // ------------------------------------------------------------- pass 2
    if (it >= p.lag && it - p.lag < p.G) {
      const int g = it - p.lag;
      const int v = worker_of(p, g, 1);
      if (v < p.P) {
        const int col = g * kCols + lane;
        const int t_a = (int)((long long)v * p.tpg / p.P), t_b = (int)((long long)(v + 1) * p.tpg / p.P);
        IO* out = (IO*)a.out;
        if constexpr (!BWD) {
          double wq[K], bf = 0.0, xw[H + 1];
          for (int tile = t_a; tile < t_b; ++tile) {
            const int nbi = tile / p.ttl, tt = tile % p.ttl, t0 = tt * TB;
            const int n = nbi * kConsumerWarps + n_in;
            const bool lv = (unsigned)n < mN && col < p.J;
            if (tile == t_a || tt == 0) {
#pragma unroll
              for (int j = 0; j <= H; ++j) xw[j] = 0.0;
            }
            auto load_params = [&](const unsigned char* st) {
              const double* pd = (const double*)(st + C_::XBYTES + C_::DBYTES + lane * C_::PSTRIDE);
#pragma unroll
              for (int i = 0; i < K; ++i) wq[i] = pd[i];
              bf = pd[K];
            };
            if constexpr (H > 0) if (tile == t_a && t0 > 0) {
              const unsigned char* st = wait_item();
              load_params(st);
              const IO* xs = (const IO*)st + n_in * kCols + lane;
#pragma unroll
              for (int r = 0; r < H; ++r) {
#pragma unroll
                for (int j = 0; j < H; ++j) xw[j] = xw[j + 1];
                xw[H - 1] = (double)lds(xs + r * kConsumerWarps * kCols);
              }
              release_item();
            }
            const unsigned char* st = wait_item();
            if (tile == t_a && !(H > 0 && t0 > 0)) load_params(st);
            const IO* xs = (const IO*)st + n_in * kCols + lane;
            const int nvalid = lv ? min(TB, p.T - t0) : 0;
            IO* o = out + ((size_t)t0 * mN + (lv ? n : 0)) * p.J + (lv ? col : 0);
#pragma unroll
            for (int r = 0; r < TB; ++r) {
              xw[H] = (double)lds(xs + r * kConsumerWarps * kCols);
              double h = 0.0;  // power-of-two products are exact: DFMA == the reference's mul-then-add
#pragma unroll
              for (int i = 0; i < K; ++i) h = fma(wq[i], xw[slot<K, D>(i)], h);
              h = __dadd_rn(h, bf);
              // Heaviside on the f32-rounded membrane: f32(h) >= 0  <=>  h >= -2^-150
              const float sp = h >= -0x1p-150 ? 1.0f : 0.0f;
              if (r < nvalid) st_out(o + (size_t)r * rowstride, sp, pol_out);
#pragma unroll
              for (int j = 0; j < H; ++j) xw[j] = xw[j + 1];
            }
            release_item();
          }
        } else {
          float w[K], wq[K], bf = 0.f, mu = 0.f, a1 = 0.f, b1 = 0.f, xw[H + 1], pacc[H + 1];
          int run_t0 = 0;
          bool lv = false;
          IO* obase = out;
          // one time step of the transposed conv: scatter this step's dh into the
          // H+1-slot ring, then emit dx for the step H behind (now complete)
          auto step = [&](float xv, float yv, bool ok, int tcur) {
            xw[H] = xv;
            float h1 = 0.f, h2 = 0.f;
#pragma unroll
            for (int i = 0; i < K; ++i) {
              h1 = fmaf(w[i], xw[slot<K, D>(i)], h1);
              h2 = fmaf(wq[i], xw[slot<K, D>(i)], h2);
            }
            h2 += bf;
            const float dh2 = ok ? yv * surrogate_grad(a.sur, h2) : 0.f;
            const float dh1 = ok ? fmaf(b1, h1 - mu, a1) : 0.f;
#pragma unroll
            for (int i = 0; i < K; ++i) {
              pacc[slot<K, D>(i)] = fmaf(wq[i], dh2, pacc[slot<K, D>(i)]);
              pacc[slot<K, D>(i)] = fmaf(w[i], dh1, pacc[slot<K, D>(i)]);
            }
            const int od = tcur - H;
            if (lv && od >= run_t0 && od < p.T) st_out(obase + (size_t)od * rowstride, pacc[0], pol_out);
#pragma unroll
            for (int j = 0; j < H; ++j) {
              pacc[j] = pacc[j + 1];
              xw[j] = xw[j + 1];
            }
            pacc[H] = 0.f;
          };
          auto drain = [&](int tnext) {  // the stream ended at T: flush the ring
#pragma unroll
            for (int s2 = 0; s2 < H; ++s2) {
              const int od = tnext + s2 - H;
              if (lv && od >= run_t0 && od < p.T) st_out(obase + (size_t)od * rowstride, pacc[0], pol_out);
#pragma unroll
              for (int j = 0; j < H; ++j) pacc[j] = pacc[j + 1];
              pacc[H] = 0.f;
            }
          };
          auto load_params = [&](const unsigned char* st) {
            const unsigned char* pr = st + C_::XBYTES + C_::DBYTES + lane * C_::PSTRIDE;
            const double* pd = (const double*)pr;
            const float* pf = (const float*)(pr + 8 * (K + 1));
#pragma unroll
            for (int i = 0; i < K; ++i) {
              wq[i] = (float)pd[i];
              w[i] = pf[i];
            }
            bf = (float)pd[K];
            mu = pf[K];
            a1 = pf[K + 1];
            b1 = pf[K + 2];
          };
          for (int tile = t_a; tile < t_b; ++tile) {
            const int nbi = tile / p.ttl, tt = tile % p.ttl, t0 = tt * TB;
            if (tile == t_a || tt == 0) {
              const int n = nbi * kConsumerWarps + n_in;
              lv = (unsigned)n < mN && col < p.J;
              obase = out + (size_t)(lv ? n : 0) * p.J + (lv ? col : 0);
              run_t0 = t0;
#pragma unroll
              for (int j = 0; j <= H; ++j) xw[j] = pacc[j] = 0.f;
            }
            if constexpr (H > 0) if (tile == t_a && t0 > 0) {
              const unsigned char* st = wait_item();
              load_params(st);
              const IO* xs = (const IO*)st + n_in * kCols + lane;
#pragma unroll
              for (int r = 0; r < H; ++r) {
#pragma unroll
                for (int j = 0; j < H; ++j) xw[j] = xw[j + 1];
                xw[H - 1] = lds(xs + r * kConsumerWarps * kCols);
              }
              release_item();
            }
            const unsigned char* st = wait_item();
            if (tile == t_a && !(H > 0 && t0 > 0)) load_params(st);
            {
              const IO* xs = (const IO*)st + n_in * kCols + lane;
              const IO* ys = (const IO*)(st + C_::XBYTES) + n_in * kCols + lane;
              const int nvalid = min(TB, p.T - t0);
#pragma unroll
              for (int r = 0; r < TB; ++r)
                step(lds(xs + r * kConsumerWarps * kCols), lds(ys + r * kConsumerWarps * kCols), r < nvalid, t0 + r);
            }
            release_item();
            if constexpr (H > 0) {
              if (t0 + TB >= p.T) {
                drain(t0 + TB);
              } else if (tile == t_b - 1) {  // range ends mid-stream: future dh from the TAIL rows
                const unsigned char* st2 = wait_item();
                const IO* xs = (const IO*)st2 + n_in * kCols + lane;
                const IO* ys = (const IO*)(st2 + C_::XBYTES) + n_in * kCols + lane;
                const int te = t0 + TB;
                const int nvalid = min(H, p.T - te);
#pragma unroll
                for (int r = 0; r < H; ++r)
                  step(lds(xs + r * kConsumerWarps * kCols), lds(ys + r * kConsumerWarps * kCols), r < nvalid, te + r);
                release_item();
              }
            }
          }
        }
      }
    }
  }
}

// -------------------------------------------------------------------------
// host launcher (instantiated per configuration in psn_stream_*.cu)
// -------------------------------------------------------------------------
int stream_encode_maps(const Plan& p, int es, bool bwd, const void* x, const void* dy, CUtensorMap* maps);

template <int K, int D, typename IO, bool BWD>
int stream_launch(const Args& args, const void* x, const void* dy, cudaStream_t st) {
  using C_ = Cfg<K, D, IO, BWD>;
  CUtensorMap maps[4];
  int rc = stream_encode_maps(args.p, (int)sizeof(IO), BWD, x, dy, maps);
  if (rc) return rc;
  const size_t smem = (size_t)args.p.S * C_::STAGE + kRedBytes + 16 * (size_t)args.p.S + 1024;
  auto kern = psn_stream_kernel<K, D, IO, BWD>;
  cudaError_t e = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return fail(PSN_ERR_CUDA, "cudaFuncSetAttribute (stream kernel smem) failed");
  Args a = args;
  void* kargs[] = {(void*)&maps[0], (void*)&maps[1], (void*)&maps[2], (void*)&maps[3], (void*)&a};
  e = cudaLaunchCooperativeKernel((const void*)kern, dim3(args.p.nCTA), dim3(kThreads), kargs, smem, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    char buf[256];
    snprintf(buf, sizeof(buf), "stream kernel launch failed: %s", cudaGetErrorString(e));
    return fail(PSN_ERR_CUDA, buf);
  }
  return PSN_OK;
}

template <int K, int D, typename IO, bool BWD>
constexpr int stage_bytes() {
  return Cfg<K, D, IO, BWD>::STAGE;
}

}  // namespace stream
}  // namespace psn
