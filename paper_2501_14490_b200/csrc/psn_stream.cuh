// psn_stream.cuh — TMA-staged, persistent sm_100a kernels for the PSN TRAIN
// forward and backward (reference network.py:236-318).  Included by the
// psn_stream_*.cu instantiation units; host planning lives in psn_stream.cu.
//
// Why this shape.  The BN batch statistics put a per-channel reduction over
// ALL (t, n) between the two halves of each direction (forward: stats of h1
// -> spikes from h2; backward: db/dw sums -> dx).  Streaming x (and dy) twice
// from HBM costs 32 B/elem against the 20 B/elem algorithmic minimum (f32).
// So the channels are cut into groups of 32 columns (one 128-byte row segment
// per (t, n)) and the two passes are software-pipelined over groups inside one
// cooperative launch (one CTA per SM):
//
//     iteration it:  pass1(it)  |  fold(it-1) on the folder warp  |  pass2(it-LAG)
//
// pass1 streams group `it` (TMA, L2 evict_last) and publishes per-CTA partial
// sums (f64 red.add per channel + an arrival counter); every CTA of the team
// folds the group once all members arrived; pass2 re-reads the group (TMA,
// evict_first) and writes spikes / dx.  The CTAs form nT teams (CTA b is in
// team b % nT) that stream different groups concurrently, so that each CTA's
// share of a group spans several tiles.
//
// Inside a CTA: warp 16 is the TMA producer (one elected lane issues
// cp.async.bulk.tensor into a ring of S stages guarded by full/empty
// mbarriers), warp 17 publishes the consumers' sums, warp 18 folds, warps
// 0..15 consume.  A tile is a TMA box [32 columns][16 batch rows][TB time
// steps] of the time-major tensor; lane = column (channel), warp = batch row,
// and each thread walks its (n, c) stream down the tile with a register window
// of the last H = (K-1)*D inputs, so every element is read from shared memory
// once and the dilated taps are register renames.  A thread keeps its window
// across consecutive tiles of its tile range; where a range starts mid-stream
// a HEAD item (H rows before the tile) primes it, and where the backward's dx
// range ends mid-stream a TAIL item (H rows after) supplies the future dh the
// time-reversed conv needs.
//
// Work is assigned statically (contiguous tile ranges per CTA, rotated per
// group so remainders spread).  Every CTA reduces its sums in a fixed order;
// across CTAs the partials are added EXACTLY (publish_exact), so the totals do
// not depend on the order the CTAs arrive in: results are bitwise reproducible
// run to run (the reference is, tests/test_train.py:70-82).
#pragma once

#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>

#include <type_traits>

#include "psn_common.cuh"

namespace psn {
namespace stream {

constexpr int kConsumerWarps = 16;
constexpr int kThreads = (kConsumerWarps + 3) * 32;  // + TMA producer, publisher and folder warps
constexpr int kCols = 32;                        // columns per tile (lanes)
constexpr int kBoxN = kConsumerWarps;            // batch rows per tile: consumer warp w owns row w
constexpr int kMaxH = 24;                        // largest (k-1)*d on this path
constexpr int kRowBlock = 4;                     // time rows a consumer thread advances at once (ILP)
// ... per pass (forward pass 1 / 2, backward pass 1 / 2); each must divide the tile rows
#ifndef PSN_U_F1
#define PSN_U_F1 2  // round 2: 2 (fewer live registers beside the f32 data-sum window; fwd -2.3 us)
#endif
#ifndef PSN_U_F2
#define PSN_U_F2 4
#endif
#ifndef PSN_U_B1
#define PSN_U_B1 4
#endif
#ifndef PSN_U_B2
#define PSN_U_B2 4
#endif

#ifndef PSN_F2_FILTER
#define PSN_F2_FILTER 1  // forward pass 2 decides spikes in f32 outside the tie band (exact f64 inside)
#endif

#ifndef PSN_B1_ALT
#define PSN_B1_ALT 1  // backward pass 1: alternate rows between two f64 accumulator sets (ILP)
#endif

#ifndef PSN_TB_FWD
#define PSN_TB_FWD 32  // f32 time rows per forward tile (bf16: twice)
#endif
#ifndef PSN_TB_BWD
#define PSN_TB_BWD 16  // f32 time rows per backward tile (x + dy)
#endif

#ifndef PSN_TRACE_BUILD
#define PSN_TRACE_BUILD 0  // 1: per-CTA wait/compute breakdown (PSN_TRACE=1 at run time)
#endif


// -------------------------------------------------------------------------
// plan + arguments (plain data, passed by value)
// -------------------------------------------------------------------------
struct Plan {
  int T, N, J, C, Q;  // J = C * Q columns; channel(j) = j / Q
  int k, d, H;
  int TB;          // time rows per tile
  int G;           // groups of nch whole channels
  int nch;         // channels per group (<= 32: one fold lane per channel)
  int ncol;        // 32-column tiles per group = ceil(nch * Q / 32)
  int nbk;         // ceil(N / kBoxN)
  int ttl;         // ceil(T / TB)
  int tpg;         // tiles per group = ncol * nbk * ttl (time fastest, then batch block, then column tile)
  int nCTA;
  int nT;          // CTA teams: team q = CTAs b with b % nT == q streams groups g with g % nT == q
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
  double* fold;           // [C][PSN_FOLD_STRIDE(k)] (written by forward, read by backward)
  double* dW;             // [C,k] (or per-channel scratch when shared)
  double* dgamma;
  double* dbeta;
  double* acc;            // [G][NV][32] per-channel pass-1 sums (exact adds, publish_exact)
  unsigned* emax;         // [G][NV][32] largest biased exponent of the CTA partials, + 1 (0: none)
  unsigned* cnt;          // [G] pass-1 arrivals (every CTA arrives once per group)
  unsigned* cntA;         // [G] exponent-agreement arrivals (all four zeroed per launch)
  const void* x;          // the input (forward: one sample per channel sets the moment shift)
  unsigned long long wait_ns;  // watchdog of every wait (0: off); PSN_WAIT_LIMIT_MS at run time
  int flags;
  int shared;
  double eps, momentum;
  Surrogate sur;    // f32 surrogate (dx pass)
  int ablate;        // PSN_ABLATE (benchmarking only): 1 no row math, 2 no cross-CTA wait, 4 no TMA,
                     // 16 no pass-2 deposit, 64 no L2 evict_last/evict_first hints
  int trace;         // PSN_TRACE: print per-CTA wait/compute breakdown at kernel end
  double scc, sscale;  // f64 surrogate sigma'(h) = sscale / (1 + scc h^2): arctan scc = (pi alpha / 2)^2,
                       // sscale = alpha / 2; rational scc = alpha, sscale = 1 (surrogate.py)
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
// try_wait with a suspend-time hint: the waiting warp is parked by the hardware
// until the phase completes (or the hint expires), so waiting warps do not
// steal issue slots from the warps doing arithmetic; the watchdog clock is
// read only once per 64 unsuccessful polls
__device__ __forceinline__ bool mbar_try_hint(uint64_t* b, unsigned parity, unsigned hint_ns) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(su32(b)), "r"(parity), "r"(hint_ns)
      : "memory");
  return ok != 0;
}
// `lim` (ns, 0 = no watchdog) turns a hang into a trap with a message
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity, unsigned long long lim) {
  if (mbar_try(b, parity)) return;
  const unsigned long long t0 = gtimer();
  for (unsigned n = 1;; ++n) {
    if (mbar_try_hint(b, parity, 20000u)) return;
    if ((n & 63u) == 0 && lim && gtimer() - t0 > lim) expired("mbarrier", (int)parity, 0);
  }
}

// keep an incrementally updated loop counter opaque, so the compiler does not
// rematerialise it as a per-iteration integer division
__device__ __forceinline__ void opaque(int& v) { asm volatile("" : "+r"(v)); }

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

#ifndef PSN_RED_RELEASE
#define PSN_RED_RELEASE 1  // 0: fence.acq_rel.gpu + relaxed red (round-1 form, A/B)
#endif
// arrival on a grid counter that releases this thread's prior writes (and,
// through the preceding __syncwarp, its warp's)
__device__ __forceinline__ void arrive_release(unsigned* a) {
  if (PSN_RED_RELEASE) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a) : "memory");
  } else {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(a) : "memory");
  }
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* a) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
  return v;
}
// one thread waits for a grid counter (co-residency is guaranteed by the
// cooperative launch); callers publish the result with a CTA barrier
__device__ __forceinline__ void wait_counter(const unsigned* a, unsigned target, const char* what,
                                             unsigned long long lim) {
  if (ld_acquire(a) >= target) return;
  const unsigned long long t0 = gtimer();
  for (;;) {  // bursts of cheap polls (this wait is on the critical path of every group's fold),
              // the watchdog clock read once per burst
#pragma unroll 1
    for (int n = 0; n < 64; ++n) {
      if (ld_acquire(a) >= target) return;
      __nanosleep(256);
    }
    if (lim && gtimer() - t0 > lim) expired(what, (int)ld_acquire(a), (int)target);
  }
}

// streaming stores of the outputs (L2 evict_first: keep the resident groups)
__device__ __forceinline__ void st_out(float* a, float v, uint64_t) { __stcs(a, v); }
__device__ __forceinline__ void st_out(__nv_bfloat16* a, float v, uint64_t) { __stcs(a, __float2bfloat16_rn(v)); }

// shared-space loads from 32-bit shared-window addresses (no generic pointer,
// no per-load address-space conversion)
template <typename IO>
__device__ __forceinline__ float ldsx(uint32_t a);
template <>
__device__ __forceinline__ float ldsx<float>(uint32_t a) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
template <>
__device__ __forceinline__ float ldsx<__nv_bfloat16>(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return __uint_as_float(((unsigned)v) << 16);
}
__device__ __forceinline__ double ldsd(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(su32(p)));
  return v;
}
__device__ __forceinline__ float ldsf(const float* p) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(su32(p)));
  return v;
}

// (double)(float)h on the integer pipe (F2F.F32.F64 issues at only ~8/clk/SM,
// profiles/r1_microbench_pipes.txt): round the f64 pattern to 24 significant
// bits (ties to even) by a 64-bit add and mask.  Exact wherever f32(h) is
// normal.  In the f32 denormal range (|h| < 2^-126) it keeps extra bits: that
// cannot change sigma'(h) = 1 / (1 + c h^2) (1.0 exactly there), and moves a
// moment sum by < 2^-149 per element.
#ifndef PSN_ROUND_CVT
#define PSN_ROUND_CVT 0  // 1: round with F2F.F32.F64 + F2F.F64.F32 instead (A/B experiment)
#endif
__device__ __forceinline__ double round_f32_sg(double h) {
  if (PSN_ROUND_CVT) return (double)__double2float_rn(h);
  const unsigned long long b = (unsigned long long)__double_as_longlong(h);
  const unsigned long long r = (b + 0x0FFFFFFFull + ((b >> 29) & 1ull)) & ~0x1FFFFFFFull;
  return __longlong_as_double((long long)r);
}


// -------------------------------------------------------------------------
// shared-memory layout per (order, dilation, carrier size, direction); host
// planning (stage count) and the kernel both use it
// -------------------------------------------------------------------------
struct Layout {
  int H, NV, NV2, TB, rowb, xbytes, dbytes, pstride, pbytes, stage, dep, tot, fixed;
};
__host__ __device__ constexpr int tile_rows(int es, bool bwd) { return bwd ? (es == 4 ? PSN_TB_BWD : 2 * PSN_TB_BWD) : (es == 4 ? PSN_TB_FWD : 2 * PSN_TB_FWD); }
__host__ __device__ constexpr Layout layout_of(int k, int d, int es, bool bwd) {
  Layout L{};
  L.H = (k - 1) * d;
  L.NV = bwd ? 1 + k : 2 + 2 * k;  // pass-1 sums: fwd S1, S2, P[k], Sx[k]; bwd db, dw_q[k]
  L.NV2 = 0;
  L.TB = tile_rows(es, bwd);
  L.rowb = kBoxN * kCols * es;  // bytes of one time row of a box
  const int xrows = L.TB > L.H ? L.TB : L.H;
  L.xbytes = xrows * L.rowb;
  L.dbytes = bwd ? xrows * L.rowb : 0;
  // per-lane parameters: fwd f64 {W or w_q}[k] + {shift or b_f}; bwd f64 w_q[k], b_f + f32 W[k], mu, a1, b1, c
  // per-lane pass-2 parameters: fwd f64 w_q[k], b_f; bwd f64 w_q[k], b_f' + f32 W[k], mu', a1, b1, c
  L.pstride = bwd ? (8 * (k + 1) + 4 * (k + 4) + 15) / 16 * 16 : 8 * (k + 2);
  L.pbytes = (kCols * L.pstride + 127) / 128 * 128;
  L.stage = (L.xbytes + L.dbytes + 1023) / 1024 * 1024;
  L.dep = 8 * L.NV * kCols * 8;  // per-warp-pair partial sums handed to the publisher
  L.tot = 8 * 2 * kCols * 8;                  // publisher ring: pre-update running stats of 8 groups
  L.fixed = L.dep + 4 * L.pbytes + L.tot + 512;
  return L;
}

template <int K, int D, typename IO, bool BWD>
struct Cfg {
  static constexpr Layout L = layout_of(K, D, (int)sizeof(IO), BWD);
  static constexpr int H = L.H, NV = L.NV, TB = L.TB;
  static constexpr int XBYTES = L.xbytes, PSTRIDE = L.pstride, PBYTES = L.pbytes, STAGE = L.stage;
  static constexpr int ROWB = L.rowb;
  static_assert(H <= kMaxH, "window above the streamed-path limit");
  static_assert(TB % kRowBlock == 0, "tile rows must be a multiple of the row block");
};

// tap i reads x[t - (K-1-i)*D] = window slot H - (K-1-i)*D
template <int K, int D>
__device__ __forceinline__ constexpr int slot(int i) {
  return (K - 1) * D - (K - 1 - i) * D;
}

// -------------------------------------------------------------------------
// static schedule, shared by the three warp roles
// -------------------------------------------------------------------------
// 32-bit schedule arithmetic only (a 64-bit divide is a ~100-instruction
// subroutine, and every warp evaluates these once per segment); the planner
// guarantees tpg * nCTA < 2^32
// This CTA's team: member m of sz CTAs, streaming the team's ng groups
// g = q + j * nT (j = the team-local group index); P = workers per group.
struct Team {
  int q, m, sz, ng, P;
};
__device__ __forceinline__ Team team_of(const Plan& p) {
  Team t;
  const unsigned nT = (unsigned)p.nT;
  t.q = (int)(blockIdx.x % nT);
  t.m = (int)(blockIdx.x / nT);
  t.sz = (int)(((unsigned)p.nCTA - (unsigned)t.q + nT - 1u) / nT);
  t.ng = p.G > t.q ? (int)(((unsigned)(p.G - t.q) + nT - 1u) / nT) : 0;
  t.P = p.tpg < t.sz ? p.tpg : t.sz;
  return t;
}
// worker index of this CTA for local group j (rotated per group and pass, so
// the idle members and the short ranges move around the team)
__device__ __forceinline__ int worker_of_member(const Team& t, int mm, int j, int pass) {
  const unsigned n = (unsigned)t.sz;
  const unsigned rot = ((unsigned)j * 61u + (unsigned)pass * 29u) % n;
  return (int)(((unsigned)mm + n - rot) % n);
}
__device__ __forceinline__ int worker_of(const Team& t, int j, int pass) { return worker_of_member(t, t.m, j, pass); }
__device__ __forceinline__ void tile_range(const Plan& p, const Team& t, int v, int& ta, int& tb) {
  ta = (int)((unsigned)v * (unsigned)p.tpg / (unsigned)t.P);
  tb = (int)((unsigned)(v + 1) * (unsigned)p.tpg / (unsigned)t.P);
}


// A group's tiles run time-fastest, then batch block, then 32-column tile:
// stream block sb = tile / ttl is (column tile ct = sb / nbk, batch block nb).
__device__ __forceinline__ void split_sb(const Plan& p, int sb, int& ct, int& nb) {
  ct = (int)((unsigned)sb / (unsigned)p.nbk);
  nb = sb - ct * p.nbk;
}
__device__ __forceinline__ int gcol0(const Plan& p, int g) { return g * p.nch * p.Q; }  // first column of group g
__device__ __forceinline__ int gcolend(const Plan& p, int g) {
  const long long e = (long long)(g + 1) * p.nch * p.Q;
  return e < p.J ? (int)e : p.J;
}

enum ItemKind { kHead = 0, kTile = 1, kTail = 2 };

// -------------------------------------------------------------------------
// fold of channel c from its per-channel pass-1 sums, one publisher lane per
// channel (forward: network.py:239-258; backward: network.py:279-317).  Every
// CTA folds the 32 channels of the group it is about to stream in pass 2 and
// writes the pass-2 parameters straight into its shared-memory slot; only the
// group's designated CTA (`store`) writes the layer outputs to global memory.
// -------------------------------------------------------------------------
// static per-channel inputs of a fold (loaded by the folder warp before it
// waits for the group's sums, so their latency hides behind that wait)
template <int K, bool BWD>
struct FoldIn {
  double W[K], gamma, beta;
  double mu, s, aa, bf, wf[BWD ? K : 1], wq[BWD ? K : 1];  // the forward's fold row (backward only)
  double sx[BWD ? K : 1], cx[BWD ? K : 1], bn;               // ... and its BN-term data sums
};
template <int K, bool BWD>
__device__ __forceinline__ void load_fold_in(const Args& a, int c, FoldIn<K, BWD>& in) {
  const double* Wc = a.W + (a.shared ? 0 : (size_t)c * K);
#pragma unroll
  for (int i = 0; i < K; ++i) in.W[i] = __ldg(Wc + i);
  in.gamma = __ldg(a.gamma + c);
  if constexpr (!BWD) {
    in.beta = __ldg(a.beta + c);
  } else {
    const double* fr = a.fold + (size_t)c * PSN_FOLD_STRIDE(K);
    in.mu = __ldg(fr + 0);
    in.s = __ldg(fr + 1);
    in.aa = __ldg(fr + 2);
    in.bf = __ldg(fr + 3);
    in.bn = __ldg(fr + 6);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      in.wf[i] = __ldg(fr + PSN_FOLD_HDR + i);
      in.wq[i] = __ldg(fr + PSN_FOLD_HDR + K + i);
      in.sx[i] = __ldg(fr + PSN_FOLD_HDR + 2 * K + i);
      in.cx[i] = __ldg(fr + PSN_FOLD_HDR + 3 * K + i);
    }
  }
}

// -------------------------------------------------------------------------
// fold of channel c from its per-channel pass-1 sums, one folder lane per
// channel (forward: network.py:239-258; backward: network.py:279-317).  Every
// CTA folds the 32 channels of the group it is about to stream in pass 2 and
// writes the pass-2 parameters straight into its shared-memory slot; only the
// group's designated CTA (`store`) writes the layer outputs to global memory.
// -------------------------------------------------------------------------
template <int K, bool BWD>
__device__ __forceinline__ void fold_channel(const Args& a, int c, const FoldIn<K, BWD>& in, const double* tt,
                                             double rm_prev, double rv_prev, double sh, double cxs, bool store,
                                             unsigned char* prow) {
  const Plan& p = a.p;
  double* fr = a.fold + (size_t)c * PSN_FOLD_STRIDE(K);
  double* pd = (double*)prow;
  const int flags = a.flags;
  const double m = (double)p.T * (double)p.N * (double)p.Q;  // elements per channel
  if constexpr (!BWD) {
    const bool smooth = flags & PSN_SMOOTH;
    const bool use_batch = flags & PSN_USE_BATCH_STATS;
    const bool quantize = (flags & PSN_QUANTIZED) && (!smooth || (flags & PSN_QUANTIZE_IN_SMOOTH));
    const double dmean = tt[0] / m;
    const double mu_b = sh + dmean;  // pass-1 moments are shifted by one h1 sample of the channel
    double var_b = tt[1] / m - dmean * dmean;
    var_b = var_b < 0.0 ? 0.0 : var_b;
    const double mu = use_batch ? mu_b : rm_prev;  // network.py:250-255
    const double var = use_batch ? var_b : rv_prev;
    const double s = sqrt(var + a.eps);
    const double aa = in.gamma / s;
    const double bf = in.beta - aa * mu;
    if (store) {
      if (!smooth) {  // network.py:241-248
        const double unbiased = m > 1.0 ? var_b * (m / (m - 1.0)) : var_b;
        double r1 = rm_prev * (1.0 - a.momentum);
        r1 = r1 + a.momentum * mu_b;
        double r2 = rv_prev * (1.0 - a.momentum);
        r2 = r2 + a.momentum * unbiased;
        a.rm[c] = r1;
        a.rv[c] = r2;
      }
      fr[0] = mu;
      fr[1] = s;
      fr[2] = aa;
      fr[3] = bf;
      fr[4] = mu_b;
      fr[5] = var_b;
      fr[6] = 1.0;  // BN-term data sums present
      // data terms of the BN-through-statistics dW (network.py:298-315):
      // Sx_i = sum x[t-off_i] and Cx_i = sum x[t-off_i] (h1[t] - mu_b).  Pass 1
      // summed the centred D_i = sum (x[t-off_i] - cx) (x = 0 before the stream
      // start) and P_i = sum (x[t-off_i] - cx)(h1[t] - shift); since
      // sum_t (h1[t] - mu_b) = 0, Cx_i = P_i - (mu_b - shift) D_i exactly.
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const double di = tt[2 + K + i];
        fr[PSN_FOLD_HDR + 2 * K + i] = di + cxs * m;
        fr[PSN_FOLD_HDR + 3 * K + i] = tt[2 + i] - (mu_b - sh) * di;
      }
    }
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const double wf = aa * in.W[i];
      double wq = wf;
      if (quantize) {  // quant.py:111-139
        int sg, e;
        quantize_pow2(wf, sg, e);
        wq = ldexp((double)sg, e);
      }
      if (store) {
        fr[PSN_FOLD_HDR + i] = wf;
        fr[PSN_FOLD_HDR + K + i] = wq;
      }
      pd[i] = wq;
    }
    pd[K] = bf;
  } else {
    float* pf = (float*)(prow + 8 * (K + 1));
    const double mu = in.mu, s = in.s, aa = in.aa;
    const bool quantized = (flags & PSN_QUANTIZED) && (!(flags & PSN_SMOOTH) || (flags & PSN_QUANTIZE_IN_SMOOTH));
    const double db_f = tt[0] * a.sscale;
    double da = 0.0, dwf[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {  // quantize_backward, quant.py:194-216
      double g1 = tt[1 + i] * a.sscale;
      if (quantized && (flags & PSN_ROUND_STE)) {
        const double wf = in.wf[i], wq = in.wq[i];
        g1 = (wf != 0.0) ? g1 * (fabs(wq) / fabs(wf)) : 0.0;
      }
      dwf[i] = g1;
      da = da + dwf[i] * in.W[i];
    }
    da = da - db_f * mu;  // network.py:291-296
    double alpha1 = 0.0, beta1 = 0.0;
    if (flags & PSN_USE_BATCH_STATS) {  // network.py:298-315
      const double ds = -da * in.gamma / (s * s);
      const double dvar = ds / (2.0 * s);
      const double dmu = -db_f * aa;
      alpha1 = dmu / m;
      beta1 = (2.0 / m) * dvar;
    }
    if (store) {
      a.dbeta[c] = db_f;
      a.dgamma[c] = da / s;
      // dW = a dw_f + sum_t x[t-off_i] dh1[t] with dh1 = alpha1 + beta1 (h1 - mu):
      // the BN term from the forward's exact data sums (network.py:298-315)
      const bool bnt = flags & PSN_USE_BATCH_STATS;
      if (bnt && in.bn != 1.0) {
        printf("psn stream backward: the fold has no BN-term sums (forward not run by the streamed kernel)\n");
        __trap();
      }
#pragma unroll
      for (int i = 0; i < K; ++i)
        a.dW[(size_t)c * K + i] = aa * dwf[i] + (bnt ? alpha1 * in.sx[i] + beta1 * in.cx[i] : 0.0);
    }
    // pass 2 runs in f32 on centred inputs x - c (c: the channel's mean input,
    // from the forward's data sums): h1 - mu and h2 then carry no large common
    // offset the f32 arithmetic would have to cancel (inputs like x + 50);
    // masked taps hold -c so that x = 0 there, as the reference skips them
    const double cx = in.bn == 1.0 ? (double)(float)(in.sx[K - 1] / m) : 0.0;
    double sw = 0.0, swq = 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      pd[i] = in.wq[i];
      pf[i] = (float)in.W[i];
      sw += in.W[i];
      swq += in.wq[i];
    }
    pd[K] = in.bf + cx * swq;
    pf[K] = (float)(mu - cx * sw);
    pf[K + 1] = (float)alpha1;
    pf[K + 2] = (float)beta1;
    pf[K + 3] = (float)cx;
  }
}

// the team member that writes the layer outputs of local group j
__device__ __forceinline__ bool designated(const Team& t, int j) {
  return (int)(((unsigned)j * 37u + 11u) % (unsigned)t.sz) == t.m;
}

// Exact, order-independent sum of one value over the team's CTAs (phase B of
// the publisher): every partial is rounded to the grid 2^q with
// q = E + ceil(log2 P) - 53, where 2^E bounds the largest |partial| of the
// value (agreed in phase A by an integer atomicMax on the exponents).  All
// partials and all their partial sums are then integer multiples of 2^q below
// 2^(q+53), so every f64 addition is exact and the total is the same whatever
// order the atomic adds land in.  The rounding moves a partial by at most
// 2^(q-1) = 2^-54 * P * 2^E (relative 1e-15 of the largest partial).
__device__ __forceinline__ unsigned exp_key(double v) {  // biased exponent + 1 (>= 2 for v != 0)
  const unsigned be = (unsigned)((__double_as_longlong(v) >> 52) & 0x7FF);
  return (be > 1u ? be : 1u) + 1u;
}
__device__ __forceinline__ double round_to_agreed_grid(double v, unsigned key, int lgP) {
  const int E = (int)key - 1 - 1022;  // |partial| < 2^E for every partial of the value
  int q = E + lgP - 53;
  q = q < -1074 ? -1074 : q;
  return ldexp(rint(ldexp(v, -q)), q);
}
__device__ __forceinline__ void red_add_f64(double* a, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(a), "d"(v) : "memory");
}

__device__ __forceinline__ float ld_io(const float* p) { return __ldg(p); }
__device__ __forceinline__ float ld_io(const __nv_bfloat16* p) { return __bfloat162float(__ldg(p)); }

// Shift of the forward's pass-1 moments for channel c: h1 of stream (n = 0,
// first column of c) at t = T - 1, computed like the consumers compute h1.  One sample of the
// channel's own distribution lies within a few standard deviations of its
// mean, so the one-pass moments sum (h1 - shift) without the cancellation a
// far-away shift (e.g. a stale running mean) would cause.  Every CTA derives
// the same value from the same data.
// The same stream's newest sample x[T - 1] is the centring value `cx` of the
// forward's f32 BN-term data sums (pass 1).
template <int K, int D, typename IO>
__device__ __forceinline__ double group_shift(const Args& a, const double* w, int c, double& cx) {
  const Plan& p = a.p;
  const IO* x = (const IO*)a.x;
  const int ts = p.T - 1;
  double h = 0.0, xv = 0.0;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const int t = ts - (K - 1 - i) * D;
    xv = t >= 0 ? (double)ld_io(x + ((size_t)t * p.N) * p.J + (size_t)c * p.Q) : 0.0;
    h = i == 0 ? w[0] * xv : fma(w[i], xv, h);
  }
  cx = xv;
  return round_f32_sg(h);
}

// -------------------------------------------------------------------------
// the kernel: warps 0..15 consume tiles, warp 16 issues TMA, warp 17
// publishes the per-group sums, warp 18 folds (see the file header)
// -------------------------------------------------------------------------
template <int K, int D, typename IO, bool BWD, bool SP>
__global__ void __launch_bounds__(kThreads, 1)
    psn_stream_kernel(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap mxh,
                      const __grid_constant__ CUtensorMap my, const __grid_constant__ CUtensorMap myh,
                      const Args a) {
  // SP: spatial inputs (Q > 1, groups of several 32-column tiles); false: one
  // column tile per group, lane = channel (the channel sums need no merge)
  using C_ = Cfg<K, D, IO, BWD>;
  constexpr Layout LY = C_::L;
  constexpr int H = C_::H, NV = C_::NV, TB = C_::TB;
  constexpr int kMaxNV = C_::L.NV > C_::L.NV2 ? C_::L.NV : C_::L.NV2;  // deposit slot stride
  const Plan& p = a.p;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = (unsigned char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  double* dep = (double*)(smem + (size_t)p.S * C_::STAGE);
  unsigned char* p1s = (unsigned char*)dep + LY.dep;
  unsigned char* p2s = p1s + 2 * LY.pbytes;
  double* tot = (double*)(p2s + 2 * LY.pbytes);
  uint64_t* full = (uint64_t*)((unsigned char*)tot + LY.tot);
  uint64_t* empty = full + p.S;
  uint64_t* depf = empty + p.S;
  uint64_t* depe = depf + 1;
  uint64_t* p1f = depe + 1;
  uint64_t* p1e = p1f + 2;
  uint64_t* p2f = p1e + 2;
  uint64_t* p2e = p2f + 2;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kConsumerWarps);
    }
    // shared-memory hand-offs between warps (deposits, parameter slots): every
    // thread arrives, so each one releases its own accesses (a per-thread
    // release-acquire pair per access, as compute-sanitizer racecheck models it)
    mbar_init(depf, kConsumerWarps * 32);
    mbar_init(depe, 32);
    for (int i = 0; i < 2; ++i) {
      mbar_init(p1f + i, 32);
      mbar_init(p1e + i, kConsumerWarps * 32);
      mbar_init(p2f + i, 32);
      mbar_init(p2e + i, kConsumerWarps * 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const Team tm = team_of(p);
  auto sbsplit = [&](int sb, int& ct, int& nb) {
    if constexpr (SP) {
      split_sb(p, sb, ct, nb);
    } else {
      ct = 0;
      nb = sb;
    }
  };
  const int iters = tm.ng > 0 ? tm.ng + p.lag : 0;
  auto gid = [&](int j) { return tm.q + j * p.nT; };  // team-local group index -> group

  if (warp == kConsumerWarps) {
    // ======================= producer warp: TMA only =======================
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mx) : "memory");
      if (H > 0) asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mxh) : "memory");
      if (BWD) asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&my) : "memory");
      if (BWD && H > 0) asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&myh) : "memory");
      const uint64_t pol_keep = pol_evict_last(), pol_drop = pol_evict_first(), pol_norm = pol_evict_normal();
      unsigned long long tr_start = gtimer(), tr_empty = 0;
      int q = 0, s = 0;
      unsigned ph = 0;  // parity of the current pass over the ring
      auto issue = [&](int kind, int pass, int g, int nbi, int trow) {
        if (q >= p.S) {
          const unsigned long long t0 = (PSN_TRACE_BUILD && a.trace) ? gtimer() : 0;
          mbar_wait(empty + s, ph ^ 1u, a.wait_ns);
          if (PSN_TRACE_BUILD && a.trace) tr_empty += gtimer() - t0;
        }
        unsigned char* st = smem + (size_t)s * C_::STAGE;
        uint64_t pol = (kind == kTile) ? (pass == 0 ? pol_keep : pol_drop) : (pass == 0 ? pol_keep : pol_norm);
        if (a.ablate & 64) pol = pol_norm;  // experiment: no L2 residency hints
        int ct, nb;
        sbsplit(nbi, ct, nb);
        const int c0 = gcol0(p, g) + ct * kCols, n0 = nb * kBoxN;
        if (a.ablate & 4) {
          mbar_arrive(full + s);
        } else if (kind == kTile) {
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
        ++q;
        if (++s == p.S) {
          s = 0;
          ph ^= 1u;
        }
      };
      for (int it = 0; it < iters; ++it) {
        for (int pass = 0; pass < 2; ++pass) {
          const int j = pass == 0 ? it : it - p.lag;
          if (j < 0 || j >= tm.ng) continue;
          const int g = gid(j);
          const int v = worker_of(tm, j, pass);
          if (v >= tm.P) continue;
          int t_a, t_b;
          tile_range(p, tm, v, t_a, t_b);
          int nbi = t_a / p.ttl, tt = t_a - nbi * p.ttl;
        opaque(nbi);
        opaque(tt);
          for (int tile = t_a; tile < t_b; ++tile) {
            const int t0 = tt * TB;
            if (H > 0 && tile == t_a && t0 > 0) issue(kHead, pass, g, nbi, t0 - H);
            issue(kTile, pass, g, nbi, t0);
            if (BWD && H > 0 && pass == 1 && tile == t_b - 1 && t0 + TB < p.T) issue(kTail, pass, g, nbi, t0 + TB);
            if (++tt == p.ttl) {
              tt = 0;
              ++nbi;
            }
            opaque(tt);
            opaque(nbi);
          }
        }
      }
      if (PSN_TRACE_BUILD && a.trace)
        printf("PSNTRACE %s prod cta %d total %llu empty %llu items %d\n", BWD ? "bwd" : "fwd", (int)blockIdx.x,
               gtimer() - tr_start, tr_empty, q);
    }
    return;
  }

  double* prev = tot;  // [8][2][32] ring: pre-update running mean / var per group (forward only)
  if (warp == kConsumerWarps + 1) {
    // ======================= publisher warp =======================
    // per group `it`: snapshot the pre-update running statistics the fold will
    // use (prefetched one group ahead), hand this CTA's pass-1 sums to the grid
    // (fixed-order reduction over the consumer-pair slots, then f64 atomic adds
    // into the group's per-channel accumulators) and arrive on the group
    // counter -- every CTA arrives, workers or not.
    unsigned long long tp_start = gtimer(), tp_dep = 0;
    int nd = 0;
    double nrm = 0.0, nrv = 0.0;
    auto prefetch_stats = [&](int g) {  // lane = channel of the group
      const int c = g * p.nch + lane;
      const bool cv = lane < p.nch && c < p.C;
      nrm = cv ? __ldcg(a.rm + c) : 0.0;
      nrv = cv ? __ldcg(a.rv + c) : 0.0;
    };
    if (!BWD && tm.ng > 0) prefetch_stats(gid(0));
    // pass-1 parameters for local group j into slot j & 1 (freed by the
    // consumers' done_p1(j - 2))
    auto stage_p1 = [&](int j) {
      if (j >= 2) {
        mbar_wait(p1e + (j & 1), (unsigned)(((j >> 1) - 1) & 1), a.wait_ns);
        __syncwarp();
      }
      const int c = gid(j) * p.nch + lane;  // lane = channel of the group
      const bool cv = lane < p.nch && c < p.C;
      const int cc = cv ? c : 0;
      double* d = (double*)(p1s + (j & 1) * LY.pbytes) + lane * (K + 2);
      if constexpr (!BWD) {
        const double* Wc = a.W + (size_t)(a.shared ? 0 : cc) * K;
        double wl[K];
#pragma unroll
        for (int i = 0; i < K; ++i) {
          wl[i] = cv ? __ldg(Wc + i) : 0.0;
          d[i] = wl[i];
        }
        double cxs = 0.0;
        d[K] = cv ? group_shift<K, D, IO>(a, wl, cc, cxs) : 0.0;  // shift of the pass-1 moments
        d[K + 1] = cxs;                                           // centring of the BN-term data sums
      } else {
        const double* f = a.fold + (size_t)cc * PSN_FOLD_STRIDE(K);
#pragma unroll
        for (int i = 0; i < K; ++i) d[i] = cv ? __ldg(f + PSN_FOLD_HDR + K + i) : 0.0;  // w_q
        d[K] = cv ? __ldg(f + 3) : 0.0;                                                // b_f
      }
      __syncwarp();
      mbar_arrive(p1f + (j & 1));
    };
    if (tm.ng > 0) stage_p1(0);
    // fixed-order sum over the 8 consumer-pair slots (the deposit of this CTA's
    // consumers is complete: the caller saw depf's phase)
    auto take_deposit = [&](int nv, double* t) {
#pragma unroll
      for (int val = 0; val < kMaxNV; ++val) {
        if (val < nv) {
          double s = dep[(0 * kMaxNV + val) * kCols + lane];
#pragma unroll
          for (int w2 = 1; w2 < 8; ++w2) s += dep[(w2 * kMaxNV + val) * kCols + lane];
          t[val] = s;
        }
      }
      __syncwarp();
      mbar_arrive(depe);
      ++nd;
    };
    // Event loop (one warp, uniform control flow): the team-wide exponent
    // agreement of group j (phase A -> every member arrived -> phase B) must
    // not hold up this CTA's own pipeline, so the publisher stages the next
    // groups' pass-1 parameters as soon as their slot is free and takes the next
    // deposit while up to two groups wait for their phase B.
    int jA = 0, jB = 0, jS = 1;
    double tP0[kMaxNV], tP1[kMaxNV];  // partials of the groups awaiting phase B (by parity)
    auto phaseA = [&](int j, double* t) {
      const int g = gid(j);
      if constexpr (!BWD) {
        prev[((j & 7) * 2 + 0) * kCols + lane] = nrm;  // pre-update running stats of group j
        prev[((j & 7) * 2 + 1) * kCols + lane] = nrv;
        if (j + 1 < tm.ng) prefetch_stats(gid(j + 1));
      }
      if (worker_of(tm, j, 0) < tm.P) {
        take_deposit(NV, t);
        unsigned* em = a.emax + (size_t)g * NV * kCols + lane;
#pragma unroll
        for (int val = 0; val < NV; ++val)
          if (t[val] != 0.0) atomicMax(em + val * kCols, exp_key(t[val]));
      }
      __syncwarp();
      if (lane == 0) arrive_release(a.cntA + g);
    };
    auto phaseB = [&](int j, const double* t) {
      const int g = gid(j);
      if (worker_of(tm, j, 0) < tm.P) {
        const unsigned* em = a.emax + (size_t)g * NV * kCols + lane;
        const int lgP = tm.P > 1 ? 32 - __clz(tm.P - 1) : 0;
#pragma unroll
        for (int val = 0; val < NV; ++val) {
          const unsigned key = __ldcg(em + val * kCols);
          if (t[val] != 0.0)
            red_add_f64(a.acc + ((size_t)g * NV + val) * kCols + lane, round_to_agreed_grid(t[val], key, lgP));
        }
      }
      __syncwarp();
      if (lane == 0) arrive_release(a.cnt + g);  // releases this group's adds
    };
    unsigned long long tl0 = 0;  // start of the current idle stretch (watchdog)
    unsigned idle = 0;
    while (jB < tm.ng) {
      bool prog = false;
      // (1) pass-1 parameters of group jS once the consumers released its slot (group jS - 2)
      if (jS < tm.ng && jS <= jA + 1) {
        const bool fr = jS < 2 || __all_sync(0xffffffffu, mbar_try(p1e + (jS & 1), (unsigned)(((jS >> 1) - 1) & 1)));
        if (fr) {
          stage_p1(jS);
          ++jS;
          prog = true;
        }
      }
      // (2) phase A of group jA: its deposit is in (or this CTA has no tiles of it)
      if (jA < tm.ng && jA < jB + 2) {
        const bool wk = worker_of(tm, jA, 0) < tm.P;
        const bool in = !wk || __all_sync(0xffffffffu, mbar_try(depf, (unsigned)(nd & 1)));
        if (in) {
          if (jA & 1) phaseA(jA, tP1); else phaseA(jA, tP0);
          ++jA;
          prog = true;
        }
      }
      // (3) phase B of group jB once every member arrived in its phase A
      if (jB < jA) {
        unsigned v = 0;
        if (lane == 0) v = ld_acquire(a.cntA + gid(jB));
        v = __shfl_sync(0xffffffffu, v, 0);
        if (v >= (unsigned)tm.sz) {
          if (jB & 1) phaseB(jB, tP1); else phaseB(jB, tP0);
          ++jB;
          prog = true;
        }
      }
      if (prog) {
        idle = 0;
      } else {
        if (idle++ == 0) tl0 = gtimer();
        __nanosleep(64);
        if ((idle & 4095u) == 0 && a.wait_ns && gtimer() - tl0 > a.wait_ns) expired("publisher", jA, jB);
      }
    }
    if (PSN_TRACE_BUILD && a.trace && lane == 0)
      printf("PSNTRACE %s publ cta %d total %llu dep %llu\n", BWD ? "bwd" : "fwd", (int)blockIdx.x,
             gtimer() - tp_start, tp_dep);
    return;
  }

  if (warp == kConsumerWarps + 2) {
    // ======================= folder warp =======================
    // per group g, in order: load the static fold inputs, wait until every CTA
    // arrived on the group counter, fold the group's 32 channels (lane =
    // channel) into the pass-2 parameter slot the consumers read.
    unsigned long long tf_start = gtimer(), tf_cnt = 0, tf_fold = 0;
    for (int j = 0; j < tm.ng; ++j) {
      const int g = gid(j);
      const int sl = j & 1;
      const int c = g * p.nch + lane;  // lane = channel of the group
      const bool cv = lane < p.nch && c < p.C;
      FoldIn<K, BWD> in;
      double sh = 0.0, cxs = 0.0;  // static fold inputs: loaded before the wait hides their latency
      if (cv) {
        load_fold_in<K, BWD>(a, c, in);
        if constexpr (!BWD) sh = group_shift<K, D, IO>(a, in.W, c, cxs);
      }
      unsigned long long t0 = (PSN_TRACE_BUILD && a.trace) ? gtimer() : 0;
      if (lane == 0 && !(a.ablate & 2)) wait_counter(a.cnt + g, (unsigned)tm.sz, "pass-1 sums", a.wait_ns);
      __syncwarp();
      if (PSN_TRACE_BUILD && a.trace) {
        const unsigned long long t1 = gtimer();
        tf_cnt += t1 - t0;
        t0 = t1;
      }
      if (j >= 2) {
        mbar_wait(p2e + sl, (unsigned)(((j >> 1) - 1) & 1), a.wait_ns);
        __syncwarp();
      }
      if (cv) {
        double tt[NV];
#pragma unroll
        for (int val = 0; val < NV; ++val) tt[val] = __ldcg(a.acc + ((size_t)g * NV + val) * kCols + lane);
        const double rmp = BWD ? 0.0 : prev[((j & 7) * 2 + 0) * kCols + lane];
        const double rvp = BWD ? 0.0 : prev[((j & 7) * 2 + 1) * kCols + lane];
        fold_channel<K, BWD>(a, c, in, tt, rmp, rvp, sh, cxs, designated(tm, j),
                             p2s + sl * LY.pbytes + lane * LY.pstride);
      } else {
        double* pd = (double*)(p2s + sl * LY.pbytes + lane * LY.pstride);
#pragma unroll
        for (int i = 0; i < LY.pstride / 8; ++i) pd[i] = 0.0;
      }
      __syncwarp();
      mbar_arrive(p2f + sl);
      if (PSN_TRACE_BUILD && a.trace) tf_fold += gtimer() - t0;
    }
    if (PSN_TRACE_BUILD && a.trace && lane == 0)
      printf("PSNTRACE %s fold cta %d total %llu cnt %llu fold %llu\n", BWD ? "bwd" : "fwd", (int)blockIdx.x,
             gtimer() - tf_start, tf_cnt, tf_fold);
    return;
  }

  // ======================= consumer warps =======================
  constexpr int U = kRowBlock;
  constexpr int RS = kBoxN * kCols;  // elements between consecutive time rows of a box
  constexpr uint32_t RSB = RS * sizeof(IO);  // ... in bytes
  const int n_in = warp;                      // batch row within the tile
  const uint64_t pol_out = pol_evict_first();
  int q = 0, nd = 0, cs = 0;
  unsigned cph = 0;  // parity of the current pass over the ring
  unsigned long long tc_start = gtimer(), tc_full = 0, tc_param = 0, tc_dep = 0;
  unsigned long long tc_pass[2] = {0, 0}, tc_fullp[2] = {0, 0}, tc_t = 0;
  int tc_cur = 0;
  const uint32_t sbase = su32(smem) + (uint32_t)((n_in * kCols + lane) * sizeof(IO));  // this thread's column
  auto wait_item = [&]() -> uint32_t {
    const unsigned long long t0 = (PSN_TRACE_BUILD && a.trace) ? gtimer() : 0;
    mbar_wait(full + cs, cph, a.wait_ns);
    if (PSN_TRACE_BUILD && a.trace) {
      const unsigned long long dt = gtimer() - t0;
      tc_full += dt;
      tc_fullp[tc_cur] += dt;
    }
    return sbase + (uint32_t)(cs * C_::STAGE);
  };
  auto release_item = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + cs);
    ++q;
    if (++cs == p.S) {
      cs = 0;
      cph ^= 1u;
    }
  };
  auto take_params = [&](int j) -> const unsigned char* {  // j: team-local group index
    const int sl = j & 1;
    const unsigned long long t0 = (PSN_TRACE_BUILD && a.trace) ? gtimer() : 0;
    mbar_wait(p2f + sl, (unsigned)((j >> 1) & 1), a.wait_ns);
    if (PSN_TRACE_BUILD && a.trace) tc_param += gtimer() - t0;
    return p2s + sl * LY.pbytes;  // the slot; channel chl's row at chl * pstride
  };
  auto done_params = [&](int j) {
    __syncwarp();
    mbar_arrive(p2e + (j & 1));
  };
  // Per-warp pass-1 sums handed to the publisher through the warp pair's
  // channel-indexed slot (warps w and w + 8 share slot w).  A flush turns the
  // lanes' column sums into channel sums: a channel's columns are a contiguous
  // run of lanes (Q > 1), and an inclusive segmented scan in fixed order leaves
  // the run's sum in its last lane (`tail`), which adds it at the channel's
  // slot entry `chl`.  The low warp writes first (zeroing the slot at the
  // range's first flush, once the publisher took the previous range's sums),
  // then the high warp adds; end_deposit hands the slot over.
  auto flush = [&](double* accv, int nv, int chl, int seg0, bool tail, bool first) {
    if (first) {
      const unsigned long long t0 = (PSN_TRACE_BUILD && a.trace) ? gtimer() : 0;
      if (nd >= 1) mbar_wait(depe, (unsigned)((nd - 1) & 1), a.wait_ns);
      if (PSN_TRACE_BUILD && a.trace) tc_dep += gtimer() - t0;
    }
    if constexpr (SP) {
#pragma unroll
      for (int val = 0; val < kMaxNV; ++val) {
        if (val < nv) {
          double v = accv[val];
#pragma unroll
          for (int off = 1; off < 32; off <<= 1) {
            const double u = __shfl_up_sync(0xffffffffu, v, off);
            if (lane - off >= seg0) v += u;
          }
          accv[val] = v;
        }
      }
    }
    const int sw = warp & 7;
    double* slot = dep + sw * kMaxNV * kCols;
    if (warp < 8) {
      if (first) {
#pragma unroll
        for (int val = 0; val < kMaxNV; ++val)
          if (val < nv) slot[val * kCols + lane] = 0.0;
        __syncwarp();
      }
      if (tail) {
#pragma unroll
        for (int val = 0; val < kMaxNV; ++val)
          if (val < nv) slot[val * kCols + chl] += accv[val];
      }
    }
    asm volatile("bar.sync %0, 64;" ::"r"(2 + sw) : "memory");  // pair barrier (warps sw, sw + 8)
    if (warp >= 8 && tail) {
#pragma unroll
      for (int val = 0; val < kMaxNV; ++val)
        if (val < nv) slot[val * kCols + chl] += accv[val];
    }
    asm volatile("bar.sync %0, 64;" ::"r"(2 + sw) : "memory");
#pragma unroll
    for (int val = 0; val < kMaxNV; ++val)
      if (val < nv) accv[val] = 0.0;
  };
  auto end_deposit = [&]() {
    __syncwarp();
    mbar_arrive(depf);
    ++nd;
  };
  // column -> (its channel's slot in the group, first lane of the channel's run
  // in this 32-column tile, whether this lane ends the run)
  struct ColInfo {
    int col, chl, seg0;
    bool valid, tail;
  };
  auto col_info = [&](int g, int ct) {
    ColInfo ci;
    const int gc0 = gcol0(p, g), gce = gcolend(p, g);
    ci.col = gc0 + ct * kCols + lane;
    ci.valid = ci.col < gce;
    const int cq = ci.valid ? (int)((unsigned)ci.col / (unsigned)p.Q) : g * p.nch;
    ci.chl = cq - g * p.nch;
    const int inq = ci.valid ? ci.col - cq * p.Q : 0;
    ci.seg0 = lane - (lane < inq ? lane : inq);
    ci.tail = ci.valid && (lane == kCols - 1 || ci.col + 1 >= gce || inq == p.Q - 1);
    return ci;
  };
  const size_t rowstride = (size_t)p.N * p.J;
  const uint32_t rs32 = (uint32_t)rowstride;  // the planner guarantees T*N*C < 2^32
  const unsigned mN = (unsigned)p.N;
  // pass-1 parameters of local group j (W and the moment shift, or the
  // forward's w_q and b_f): staged in shared memory by the publisher warp
  auto take_p1 = [&](int j) -> const double* {  // the slot; channel chl's row at chl * (K + 2)
    mbar_wait(p1f + (j & 1), (unsigned)((j >> 1) & 1), a.wait_ns);
    return (const double*)(p1s + (j & 1) * LY.pbytes);
  };
  auto done_p1 = [&](int j) {
    __syncwarp();
    mbar_arrive(p1e + (j & 1));
  };

  for (int it = 0; it < iters; ++it) {
    // ------------------------------------------------------------- pass 1
    if (it < tm.ng) {
      if (PSN_TRACE_BUILD && a.trace) {
        tc_cur = 0;
        tc_t = gtimer();
      }
      const int g = gid(it);
      const int v = worker_of(tm, it, 0);
      int t_a, t_b;
      tile_range(p, tm, v, t_a, t_b);
      if (v >= tm.P) t_a = t_b = 0;
      double acc[NV];
#pragma unroll
      for (int u = 0; u < NV; ++u) acc[u] = 0.0;
      const double* p1b = take_p1(it);
      int cur_ct = -1;  // the 32-column tile the lane's parameters / sums belong to
      bool first_flush = true;
      ColInfo ci{};
      if constexpr (!BWD) {
        // ---- forward pass 1: shifted moments of h1 = f32(sum_i W_i x[t-off_i]) (f64 taps, f64
        // moments) and the BN-term data sums of the backward's dW on the FP32 pipe (the FP64
        // pipe bounds this pass): P_i = sum (x[t-off_i] - cx)(h1[t] - shift) and
        // D_i = sum (x[t-off_i] - cx), centred by a sample cx of the channel so the f32
        // products carry no common offset; f32 over 16 rows, f64 beyond (fold_channel)
        constexpr int U = PSN_U_F1;
        constexpr int FR = 16;  // rows per f32 partial of the data sums
        double w[K], xw[H + U], sh = 0.0;
        float xt[H + U], pf[K], sxf = 0.f, shf = 0.f, cxf = 0.f;
#pragma unroll
        for (int i = 0; i < K; ++i) pf[i] = 0.f;
        auto flush_f = [&]() {  // column sums -> channel sums
          const ColInfo cf = SP ? ci : col_info(g, 0);  // (non-spatial: recomputed, not kept live)
          flush(acc, NV, cf.chl, cf.seg0, cf.tail, first_flush);
          first_flush = false;
        };
        int nbi = t_a / p.ttl, tt = t_a - nbi * p.ttl;
        int ct, nb;
        sbsplit(nbi, ct, nb);
        opaque(nbi);
        opaque(tt);
        auto params_f = [&]() {
          const double* pp = p1b + ci.chl * (K + 2);
#pragma unroll
          for (int i = 0; i < K; ++i) w[i] = ldsd(pp + i);
          sh = ldsd(pp + K);
          shf = (float)sh;  // exact: the shift is an f32-rounded membrane
          cxf = (float)ldsd(pp + K + 1);  // exact: a sample of x
        };
        if constexpr (!SP) {
          ci = col_info(g, 0);
          params_f();
        }
        for (int tile = t_a; tile < t_b; ++tile) {
          const int t0 = tt * TB;
          // warps whose batch row is padding (N not a multiple of 16) skip the row math
          const bool rowv = (unsigned)(nb * kBoxN + n_in) < mN;
          if constexpr (SP) {
            if (ct != cur_ct) {
              if (tile != t_a) flush_f();
              ci = col_info(g, ct);
              cur_ct = ct;
              params_f();
            }
          }
          const int col = ci.col;
          const bool lv = (unsigned)(nb * kBoxN + n_in) < mN && ci.valid;
          if (tile == t_a || tt == 0) {
#pragma unroll
            for (int j = 0; j < H + U; ++j) {
              xw[j] = 0.0;
              xt[j] = -cxf;  // before the stream start: x = 0
            }
          }
          if constexpr (H > 0) if (tile == t_a && t0 > 0) {
            const uint32_t st = wait_item();
            const uint32_t xs = st;
#pragma unroll
            for (int r = 0; r < H; ++r) {
              const float xv = ldsx<IO>(xs + (r) * RSB);
              xw[r] = (double)xv;
              xt[r] = xv - cxf;
            }
            release_item();
          }
          const uint32_t st = wait_item();
          const uint32_t xs = st;
          const int nvalid = min(TB, p.T - t0);
          double S1[U], S2[U];
#pragma unroll
          for (int u = 0; u < U; ++u) S1[u] = S2[u] = 0.0;
          // full tiles (every row < T) run without per-row predicates
          auto rows = [&](auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
            for (int r0 = 0; r0 < TB; r0 += U) {
#pragma unroll
              for (int u = 0; u < U; ++u) {
                const float xv = ldsx<IO>(xs + (r0 + u) * RSB);
                xw[H + u] = (double)xv;
                xt[H + u] = xv - cxf;
              }
              double h[U];
#pragma unroll
              for (int u = 0; u < U; ++u) h[u] = w[0] * xw[u + slot<K, D>(0)];
#pragma unroll
              for (int i = 1; i < K; ++i)
#pragma unroll
                for (int u = 0; u < U; ++u) h[u] = fma(w[i], xw[u + slot<K, D>(i)], h[u]);
#pragma unroll
              for (int u = 0; u < U; ++u) {
                const float hr32 = __double2float_rn(h[u]);  // the reference's f32 membrane (F2F, XU pipe)
                const bool ok = FULL || r0 + u < nvalid;
                const double hc = ok ? (double)hr32 - sh : 0.0;
                const float hcf = ok ? hr32 - shf : 0.f;
                S1[u] += hc;
                S2[u] = fma(hc, hc, S2[u]);
#pragma unroll
                for (int i = 0; i < K; ++i) pf[i] = fmaf(xt[u + slot<K, D>(i)], hcf, pf[i]);
                sxf += ok ? xt[H + u] : 0.f;
              }
              if ((r0 + U) % FR == 0 || r0 + U == TB) {  // f32 partials -> f64 (padding lanes dropped)
#pragma unroll
                for (int i = 0; i < K; ++i) {
                  if (lv) acc[2 + i] += (double)pf[i];
                  pf[i] = 0.f;
                }
                if (lv) {
#pragma unroll
                  for (int i = 0; i < K; ++i) acc[2 + K + i] += (double)sxf;
                }
                sxf = 0.f;
              }
#pragma unroll
              for (int j = 0; j < H; ++j) {
                xw[j] = xw[j + U];
                xt[j] = xt[j + U];
              }
            }
          };
          if ((a.ablate & 1) || !rowv) {} else if (nvalid == TB) rows(std::true_type{}); else rows(std::false_type{});
          if (lv) {  // padding lanes (n >= N or column >= C) saw TMA zero fill; drop them
#pragma unroll
            for (int u = 0; u < U; ++u) {
              acc[0] += S1[u];
              acc[1] += S2[u];
            }
          }
          release_item();
          if constexpr (H > 0) {
            // end of the stream: D_i = sum_{t < T} (x[t] - cx) - sum_{t >= T - off_i} x[t]
            // (the cx of the last off_i samples and of the off_i window samples before
            // the stream start cancel); the tail is loaded from global, H values per stream
            if (tt == p.ttl - 1 && lv) {
              const IO* xp = (const IO*)a.x + (size_t)(nb * kBoxN + n_in) * p.J + col;
#pragma unroll
              for (int r = 0; r < H; ++r) {
                const int t = p.T - 1 - r;
                const double v = t >= 0 ? (double)ld_io(xp + (size_t)t * rowstride) : 0.0;
#pragma unroll
                for (int i = 0; i < K; ++i)
                  if (r < (K - 1 - i) * D) acc[2 + K + i] -= v;
              }
            }
          }
          if (++tt == p.ttl) {
            tt = 0;
            ++nbi;
            sbsplit(nbi, ct, nb);
          }
          opaque(tt);
          opaque(nbi);
        }
        if (t_b > t_a) flush_f();
      } else {
        // ---- backward pass 1: db, dw_q -- f64 end to end (h2 exact and f32-rounded like the
        // reference's carrier, sigma' and dh2 in f64): f32 per-element errors (~1e-7) would
        // grow to ~sqrt(m)*1e-7 in these m-term sums, above the 1e-5 bound on small dW
        // entries.  (The BN term of dW comes from the forward's data sums.)  Rows
        // alternate between two f64 accumulator sets (ILP).
        constexpr int U = PSN_U_B1;
        double wq[K], xd[H + U], acc2[1 + K], bf = 0.0;
#pragma unroll
        for (int i = 0; i <= K; ++i) acc2[i] = 0.0;
        auto flush_b = [&]() {  // column sums -> channel sums
#pragma unroll
          for (int i = 0; i <= K; ++i) {
            acc[i] += acc2[i];
            acc2[i] = 0.0;
          }
          const ColInfo cf = SP ? ci : col_info(g, 0);
          flush(acc, NV, cf.chl, cf.seg0, cf.tail, first_flush);
          first_flush = false;
        };
        const double scc = a.scc;
        int nbi = t_a / p.ttl, tt = t_a - nbi * p.ttl;
        int ct, nb;
        sbsplit(nbi, ct, nb);
        opaque(nbi);
        opaque(tt);
        auto params_b = [&]() {
          const double* pp = p1b + ci.chl * (K + 2);
#pragma unroll
          for (int i = 0; i < K; ++i) wq[i] = ldsd(pp + i);
          bf = ldsd(pp + K);
        };
        if constexpr (!SP) {
          ci = col_info(g, 0);
          params_b();
        }
        for (int tile = t_a; tile < t_b; ++tile) {
          const int t0 = tt * TB;
          // warps whose batch row is padding (N not a multiple of 16) skip the row math
          const bool rowv = (unsigned)(nb * kBoxN + n_in) < mN;
          if constexpr (SP) {
            if (ct != cur_ct) {
              if (tile != t_a) flush_b();
              ci = col_info(g, ct);
              cur_ct = ct;
              params_b();
            }
          }
          if (tile == t_a || tt == 0) {
#pragma unroll
            for (int j = 0; j < H + U; ++j) xd[j] = 0.0;
          }
          if constexpr (H > 0) if (tile == t_a && t0 > 0) {
            const uint32_t st = wait_item();
            const uint32_t xs = st;
#pragma unroll
            for (int r = 0; r < H; ++r) xd[r] = (double)ldsx<IO>(xs + (r) * RSB);
            release_item();
          }
          const uint32_t st = wait_item();
          const uint32_t xs = st;
          const uint32_t ys = st + C_::XBYTES;
          auto rows = [&]() {
#pragma unroll
            for (int r0 = 0; r0 < TB; r0 += U) {
              double yv[U], h2[U], dh[U];
#pragma unroll
              for (int u = 0; u < U; ++u) {
                xd[H + u] = (double)ldsx<IO>(xs + ((r0 + u)) * RSB);
                yv[u] = (double)ldsx<IO>(ys + ((r0 + u)) * RSB);  // rows >= T: TMA zero fill -> dh2 = 0
              }
#pragma unroll
              for (int u = 0; u < U; ++u) h2[u] = fma(wq[0], xd[u + slot<K, D>(0)], bf);
#pragma unroll
              for (int i = 1; i < K; ++i)
#pragma unroll
                for (int u = 0; u < U; ++u) h2[u] = fma(wq[i], xd[u + slot<K, D>(i)], h2[u]);
#pragma unroll
              for (int u = 0; u < U; ++u) {
                // the f32 membrane of the reference's carrier (b_f enters the f64 sum first
                // here: with probability ~2^-29 the f32 rounding then differs by one ulp,
                // which moves that element's sigma' by ~1e-7 relative)
                const double h = round_f32_sg(h2[u]);
                const double den = fma(scc * h, h, 1.0);
                dh[u] = yv[u] * rcp_f64(den);  // dh2 / scale (scale applied in the fold)
              }
#pragma unroll
              for (int u = 0; u < U; ++u) {
                double* A = (PSN_B1_ALT && (u & 1)) ? acc2 : acc;
                A[0] += dh[u];
#pragma unroll
                for (int i = 0; i < K; ++i) A[1 + i] = fma(xd[u + slot<K, D>(i)], dh[u], A[1 + i]);
              }
#pragma unroll
              for (int j = 0; j < H; ++j) xd[j] = xd[j + U];
            }
          };
          if (!(a.ablate & 1) && rowv) rows();
          release_item();
          if (++tt == p.ttl) {
            tt = 0;
            ++nbi;
            sbsplit(nbi, ct, nb);
          }
          opaque(tt);
          opaque(nbi);
        }
        if (t_b > t_a) flush_b();
      }
      done_p1(it);
      if (v < tm.P) end_deposit();  // CTA reduction + publication happen on the publisher warp
      if (PSN_TRACE_BUILD && a.trace) tc_pass[0] += gtimer() - tc_t;
    }
    // ------------------------------------------------------------- pass 2
    if (it >= p.lag && it - p.lag < tm.ng) {
      if (PSN_TRACE_BUILD && a.trace) {
        tc_cur = 1;
        tc_t = gtimer();
      }
      const int j = it - p.lag;
      const int g = gid(j);
      const int v = worker_of(tm, j, 1);
      const unsigned char* p2b = take_params(j);
      int cur_ct = -1;
      ColInfo ci{};
      int t_a, t_b;
      tile_range(p, tm, v, t_a, t_b);
      if (v >= tm.P) t_a = t_b = 0;
      IO* out = (IO*)a.out;
      if constexpr (!BWD) {
        // ---- forward pass 2: spikes = [f32(sum_i w_q,i x[t-off_i] + b_f) >= 0]
        // The sign is decided in f32 (the FP64 pipe bounds this pass otherwise):
        // with power-of-two taps every product is exact, so the f32 chain hf is
        // within (K+1) 2^-24 (|b_f| + sum |w_q x|) of the exact membrane h; where
        // |hf| exceeds 4x that bound, sign(hf) = sign(h) = the reference's spike.
        // Rows inside the bound (a threshold tie band, ~1e-6 of random rows) take
        // the exact f64 chain -- warp-uniformly, for the rows that need it.
        constexpr int U = PSN_U_F2;
        double wq[K], bf = 0.0;
        float wqf[K], wqa[K], bff = 0.f, bfa = 0.f, xf[H + U];
        int nbi = t_a / p.ttl, tt = t_a - nbi * p.ttl;
        int ct, nb;
        sbsplit(nbi, ct, nb);
        opaque(nbi);
        opaque(tt);
        auto params_f2 = [&]() {  // the lane's channel parameters for this column tile
          const double* pd = (const double*)(p2b + ci.chl * LY.pstride);
#pragma unroll
          for (int i = 0; i < K; ++i) {
            wq[i] = ldsd(pd + i);
            wqf[i] = (float)wq[i];  // exact: a power of two in [2^-16, 2^15] (or a float weight: rounded,
            wqa[i] = fabsf(wqf[i]);  // its error is inside the bound's factor-4 margin only if quantized)
          }
          bf = ldsd(pd + K);
          bff = (float)bf;
          bfa = fabsf(bff);
        };
        // the filter's error bound assumes exact products: power-of-two taps only
        const bool filt = PSN_F2_FILTER && (a.flags & PSN_QUANTIZED);
        if constexpr (!SP) {
          ci = col_info(g, 0);
          params_f2();
        }
        for (int tile = t_a; tile < t_b; ++tile) {
          const int t0 = tt * TB;
          // warps whose batch row is padding (N not a multiple of 16) skip the row math
          const bool rowv = (unsigned)(nb * kBoxN + n_in) < mN;
          if constexpr (SP) {
            if (ct != cur_ct) {
              ci = col_info(g, ct);
              cur_ct = ct;
              params_f2();
            }
          }
          const int col = ci.col;
          const int n = nb * kBoxN + n_in;
          const bool lv = (unsigned)n < mN && ci.valid;
          if (tile == t_a || tt == 0) {
#pragma unroll
            for (int j = 0; j < H + U; ++j) xf[j] = 0.f;
          }
          if constexpr (H > 0) if (tile == t_a && t0 > 0) {
            const uint32_t st = wait_item();
            const uint32_t xs = st;
#pragma unroll
            for (int r = 0; r < H; ++r) xf[r] = ldsx<IO>(xs + (r) * RSB);
            release_item();
          }
          const uint32_t st = wait_item();
          const uint32_t xs = st;
          const int nvalid = min(TB, p.T - t0);
          uint32_t ooff = ((uint32_t)t0 * mN + (uint32_t)(lv ? n : 0)) * (uint32_t)p.J + (uint32_t)(lv ? col : 0);
          auto rows = [&](auto full_tag) {
            constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
            for (int r0 = 0; r0 < TB; r0 += U) {
#pragma unroll
              for (int u = 0; u < U; ++u) xf[H + u] = ldsx<IO>(xs + ((r0 + u)) * RSB);
              float sp[U];
              bool need = false, nd_u[U];
#pragma unroll
              for (int u = 0; u < U; ++u) {
                float hf = bff, sf = bfa;
#pragma unroll
                for (int i = 0; i < K; ++i) {
                  hf = fmaf(wqf[i], xf[u + slot<K, D>(i)], hf);
                  sf = fmaf(wqa[i], fabsf(xf[u + slot<K, D>(i)]), sf);
                }
                nd_u[u] = !filt || !(fabsf(hf) > fmaf(sf, (float)(4 * (K + 1)) * 0x1p-24f, 0x1p-126f));
                need |= nd_u[u];
                sp[u] = hf >= 0.f ? 1.0f : 0.0f;
              }
              if (__any_sync(0xffffffffu, need)) {  // exact membrane for the rows inside the tie band
#pragma unroll
                for (int u = 0; u < U; ++u) {
                  if (nd_u[u]) {  // power-of-two products are exact: DFMA == the reference's mul-then-add
                    double h = wq[0] * (double)xf[u + slot<K, D>(0)];
#pragma unroll
                    for (int i = 1; i < K; ++i) h = fma(wq[i], (double)xf[u + slot<K, D>(i)], h);
                    // Heaviside on the f32-rounded membrane: f32(h) >= 0  <=>  h >= -2^-150
                    sp[u] = __dadd_rn(h, bf) >= -0x1p-150 ? 1.0f : 0.0f;
                  }
                }
              }
#pragma unroll
              for (int u = 0; u < U; ++u) {
                if (lv && (FULL || r0 + u < nvalid)) st_out(out + ooff, sp[u], pol_out);
                ooff += rs32;
              }
#pragma unroll
              for (int j = 0; j < H; ++j) xf[j] = xf[j + U];
            }
          };
          if ((a.ablate & 1) || !rowv) {} else if (nvalid == TB) rows(std::true_type{}); else rows(std::false_type{});
          release_item();
          if (++tt == p.ttl) {
            tt = 0;
            ++nbi;
            sbsplit(nbi, ct, nb);
          }
          opaque(tt);
          opaque(nbi);
        }
        done_params(j);
      } else {
        // ---- backward pass 2: dx[t] = sum_i w_q,i dh2[t+off_i] + W_i dh1[t+off_i]
        // (time-reversed conv as a scatter into an (H+U)-slot ring: slot j holds the
        // partial dx of row t_blk - H + j; after a block of U rows the first U slots
        // are complete).  The BN term of dW comes from the forward's exact data
        // sums (fold_channel), so this pass only writes dx.
        constexpr int U = PSN_U_B2;
        float w[K], wq[K], wqs[K], xw[H + U], pacc[H + U];
        // surrogate.py: sigma'(h) = scale / (1 + cc h^2), cc = (pi alpha / 2)^2 (arctan) or
        // alpha (rational); the scale is folded into the w_q taps of the scatter
        const float cc = a.sur.kind == PSN_ARCTAN ? a.sur.c * a.sur.c : a.sur.c;
        float bf = 0.f, mu = 0.f, a1 = 0.f, b1 = 0.f, cx = 0.f;
        auto load_params = [&]() {  // the lane's channel parameters (fold_channel) for this column tile
          const unsigned char* pr = p2b + ci.chl * LY.pstride;
          const double* pd = (const double*)pr;
          const float* pf = (const float*)(pr + 8 * (K + 1));
#pragma unroll
          for (int i = 0; i < K; ++i) {
            wq[i] = (float)ldsd(pd + i);
            w[i] = ldsf(pf + i);
            wqs[i] = wq[i] * a.sur.scale;
          }
          bf = (float)ldsd(pd + K);  // b_f + c sum w_q   (centred inputs)
          mu = ldsf(pf + K);         // mu - c sum W
          a1 = ldsf(pf + K + 1);
          b1 = ldsf(pf + K + 2);
          cx = ldsf(pf + K + 3);
        };
        int run_t0 = 0;
        bool lv = false;
        uint32_t obase = 0;
        auto emit = [&](int od, float val) {
          if (lv && od >= run_t0 && od < p.T) st_out(out + (obase + (uint32_t)od * rs32), val, pol_out);
        };
        // dh2 / scale and dh1 of row u of the window (rows with !ok contribute nothing)
        auto dh_row = [&](int u, float yv, bool ok, float& dh2, float& dh1) {
          float h1c = fmaf(w[0], xw[u + slot<K, D>(0)], -mu), h2 = fmaf(wq[0], xw[u + slot<K, D>(0)], bf);
#pragma unroll
          for (int i = 1; i < K; ++i) {
            h1c = fmaf(w[i], xw[u + slot<K, D>(i)], h1c);
            h2 = fmaf(wq[i], xw[u + slot<K, D>(i)], h2);
          }
          const float r = rcp_approx(fmaf(cc * h2, h2, 1.0f));
          dh2 = ok ? yv * r : 0.f;
          dh1 = ok ? fmaf(b1, h1c, a1) : 0.f;
        };
        auto scatter = [&](int u, float dh2, float dh1) {
#pragma unroll
          for (int i = 0; i < K; ++i) {
            pacc[u + slot<K, D>(i)] = fmaf(wqs[i], dh2, pacc[u + slot<K, D>(i)]);
            pacc[u + slot<K, D>(i)] = fmaf(w[i], dh1, pacc[u + slot<K, D>(i)]);
          }
        };
        // single-row step (TAIL rows): scatter, emit the row H behind, shift by one
        auto step1 = [&](float xv, float yv, bool ok, int tcur) {
          xw[H] = xv - cx;
          float dh2, dh1;
          dh_row(0, yv, ok, dh2, dh1);
          scatter(0, dh2, dh1);
          emit(tcur - H, pacc[0]);
#pragma unroll
          for (int j = 0; j < H + U - 1; ++j) pacc[j] = pacc[j + 1];
          pacc[H + U - 1] = 0.f;
#pragma unroll
          for (int j = 0; j < H; ++j) xw[j] = xw[j + 1];
        };
        auto drain = [&](int tnext) {  // the stream ended at T: flush the ring
#pragma unroll
          for (int s2 = 0; s2 < H; ++s2) {
            emit(tnext + s2 - H, pacc[0]);
#pragma unroll
            for (int j = 0; j < H + U - 1; ++j) pacc[j] = pacc[j + 1];
            pacc[H + U - 1] = 0.f;
          }
        };
        int nbi = t_a / p.ttl, tt = t_a - nbi * p.ttl;
        int ct, nb;
        sbsplit(nbi, ct, nb);
        opaque(nbi);
        opaque(tt);
        if constexpr (!SP) {
          ci = col_info(g, 0);
          load_params();
        }
        for (int tile = t_a; tile < t_b; ++tile) {
          const int t0 = tt * TB;
          // warps whose batch row is padding (N not a multiple of 16) skip the row math
          const bool rowv = (unsigned)(nb * kBoxN + n_in) < mN;
          if constexpr (SP) {
            if (ct != cur_ct) {
              ci = col_info(g, ct);
              cur_ct = ct;
              load_params();
            }
          }
          if (tile == t_a || tt == 0) {
            const int n = nb * kBoxN + n_in;
            lv = (unsigned)n < mN && ci.valid;
            obase = (uint32_t)(lv ? n : 0) * (uint32_t)p.J + (uint32_t)(lv ? ci.col : 0);
            run_t0 = t0;
#pragma unroll
            for (int j = 0; j < H + U; ++j) {
              xw[j] = -cx;  // before the stream start: x = 0
              pacc[j] = 0.f;
            }
          }
          if constexpr (H > 0) if (tile == t_a && t0 > 0) {
            const uint32_t st = wait_item();
            const uint32_t xs = st;
#pragma unroll
            for (int r = 0; r < H; ++r) xw[r] = ldsx<IO>(xs + (r) * RSB) - cx;
            release_item();
          }
          const uint32_t st = wait_item();
          {
            const uint32_t xs = st;
            const uint32_t ys = st + C_::XBYTES;
            const int nvalid = min(TB, p.T - t0);
            auto rows = [&](auto full_tag) {
              constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
              for (int r0 = 0; r0 < TB; r0 += U) {
                float dh2[U], dh1[U];
#pragma unroll
                for (int u = 0; u < U; ++u) xw[H + u] = ldsx<IO>(xs + ((r0 + u)) * RSB) - cx;
#pragma unroll
                for (int u = 0; u < U; ++u)
                  dh_row(u, ldsx<IO>(ys + ((r0 + u)) * RSB), FULL || r0 + u < nvalid, dh2[u], dh1[u]);
#pragma unroll
                for (int u = 0; u < U; ++u) scatter(u, dh2[u], dh1[u]);
                const int od0 = t0 + r0 - H;  // rows od0 .. od0+U-1 are complete now
                if (FULL && lv && od0 >= run_t0) {  // the common case: no per-row predicate
                  uint32_t oo = obase + (uint32_t)od0 * rs32;  // 32-bit element offsets: one wide
#pragma unroll                                                // multiply-add per store address
                  for (int u = 0; u < U; ++u) {
                    st_out(out + oo, pacc[u], pol_out);
                    oo += rs32;
                  }
                } else {
#pragma unroll
                  for (int u = 0; u < U; ++u) {
                    const int od = od0 + u;
                    const bool ok = lv && od >= run_t0 && (FULL || od < p.T);  // rows < run_t0: previous range
                    if (ok) st_out(out + (obase + (uint32_t)od * rs32), pacc[u], pol_out);
                  }
                }
#pragma unroll
                for (int j = 0; j < H; ++j) {
                  pacc[j] = pacc[j + U];
                  xw[j] = xw[j + U];
                }
#pragma unroll
                for (int j = H; j < H + U; ++j) pacc[j] = 0.f;
              }
            };
            if ((a.ablate & 1) || !rowv) {} else if (nvalid == TB) rows(std::true_type{}); else rows(std::false_type{});
          }
          release_item();
          if constexpr (H > 0) {
            if (t0 + TB >= p.T) {
              drain(t0 + TB);
            } else if (tile == t_b - 1) {  // range ends mid-stream: future dh from the TAIL rows
              const uint32_t st2 = wait_item();
              const uint32_t xs = st2;
              const uint32_t ys = st2 + C_::XBYTES;
              const int te = t0 + TB;
              const int nvalid = min(H, p.T - te);
#pragma unroll
              for (int r = 0; r < H; ++r) step1(ldsx<IO>(xs + (r) * RSB), ldsx<IO>(ys + (r) * RSB), r < nvalid, te + r);
              release_item();
            }
          }
          if (++tt == p.ttl) {
            tt = 0;
            ++nbi;
            sbsplit(nbi, ct, nb);
          }
          opaque(tt);
          opaque(nbi);
        }
        done_params(j);
      }
      if (PSN_TRACE_BUILD && a.trace) tc_pass[1] += gtimer() - tc_t;
    }
  }
  if (PSN_TRACE_BUILD && a.trace && threadIdx.x == 0)
    printf("PSNTRACE %s cons cta %d total %llu full %llu param %llu dep %llu pass1 %llu pass2 %llu full1 %llu full2 %llu items %d\n",
           BWD ? "bwd" : "fwd", (int)blockIdx.x, gtimer() - tc_start, tc_full, tc_param, tc_dep, tc_pass[0], tc_pass[1],
           tc_fullp[0], tc_fullp[1], q);
}

// -------------------------------------------------------------------------
// host launcher (instantiated per configuration in psn_stream_*.cu)
// -------------------------------------------------------------------------
int stream_encode_maps(const Plan& p, int es, bool bwd, const void* x, const void* dy, CUtensorMap* maps);

// stream_launch result: the persistent kernel cannot be co-resident on this
// device / context (occupancy, MPS or partition limits) -- run the generic path
constexpr int kFallback = -1;

template <int K, int D, typename IO, bool BWD, bool SP>
int stream_launch(const Args& args, const void* x, const void* dy, cudaStream_t st) {
  using C_ = Cfg<K, D, IO, BWD>;
  CUtensorMap maps[4];
  int rc = stream_encode_maps(args.p, (int)sizeof(IO), BWD, x, dy, maps);
  if (rc) return rc;
  const size_t smem = (size_t)args.p.S * C_::STAGE + C_::L.fixed + 16 * (size_t)args.p.S + 1024;
  auto kern = psn_stream_kernel<K, D, IO, BWD, SP>;
  cudaError_t e = cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return fail(PSN_ERR_CUDA, "cudaFuncSetAttribute (stream kernel smem) failed");
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kThreads, smem) != cudaSuccess || occ < 1) {
    cudaGetLastError();
    return kFallback;
  }
  Args a = args;
  void* kargs[] = {(void*)&maps[0], (void*)&maps[1], (void*)&maps[2], (void*)&maps[3], (void*)&a};
  e = cudaLaunchCooperativeKernel((const void*)kern, dim3(args.p.nCTA), dim3(kThreads), kargs, smem, st);
  if (e == cudaErrorCooperativeLaunchTooLarge) {
    cudaGetLastError();
    return kFallback;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    char buf[256];
    snprintf(buf, sizeof(buf), "stream kernel launch failed: %s", cudaGetErrorString(e));
    return fail(PSN_ERR_CUDA, buf);
  }
  return PSN_OK;
}

}  // namespace stream
}  // namespace psn
