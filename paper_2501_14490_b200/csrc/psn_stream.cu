// psn_stream.cu — host side of the TMA-staged persistent PSN kernels
// (psn_stream.cuh): eligibility, planning, workspace, tensor-map encoding and
// the (order, dilation, carrier) dispatch.
#include <cudaTypedefs.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "psn_stream.cuh"
#include "psn_stream_dispatch.h"

namespace psn {
namespace stream {

// Device attributes are looked up per device (the current device of the
// calling thread, which the caller sets to the device of its pointers), once
// per device.
constexpr int kMaxDevices = 64;
struct DevAttr {
  int sms = 0, smem_optin = 0, coop = 0;
};
static DevAttr g_dev[kMaxDevices];
static std::once_flag g_dev_once[kMaxDevices];
static std::once_flag g_encode_once;
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static void encode_init() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  cudaGetLastError();
}

static const DevAttr* dev_attr() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
    cudaGetLastError();
    return nullptr;
  }
  std::call_once(g_dev_once[dev], [dev] {
    DevAttr& a = g_dev[dev];
    cudaDeviceGetAttribute(&a.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&a.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&a.coop, cudaDevAttrCooperativeLaunch, dev);
    cudaGetLastError();
  });
  std::call_once(g_encode_once, encode_init);
  return &g_dev[dev];
}

bool aligned_for_tma(const void* x, const void* dy) {
  return (((uintptr_t)x | (uintptr_t)dy) & 15u) == 0;  // TMA global addresses are 16-byte aligned
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// watchdog of the in-kernel waits: PSN_WAIT_LIMIT_MS (default 4000 ms; 0 turns
// it off, e.g. under compute-sanitizer or a debugger)
static unsigned long long wait_limit_ns() {
  const char* e = getenv("PSN_WAIT_LIMIT_MS");
  const long long ms = e ? atoll(e) : 4000;
  return ms > 0 ? (unsigned long long)ms * 1000000ull : 0ull;
}

bool eligible(const psn_desc_t* desc) {
  if (env_int("PSN_FORCE_GENERIC", 0)) return false;
  return shape_eligible(desc);
}

// Routing between the streamed kernel and the three generic launches, measured
// on B200 (profiles/r2_route.txt, CUDA-graph replay of fwd+bwd): below ~1.5M
// elements the streamed kernel's cross-CTA synchronisation skeleton costs more
// than the whole generic pass (BASELINE config 1, 1.0M elements: 0.049 vs
// 0.039 ms), and the widest windows ((k-1) d > 16: k = 8, d = 3) spill
// registers in the streamed kernels (f32 0.72 vs 0.51 ms, bf16 0.60 vs 0.53 ms
// at T=1024, B=64, C=512).  PSN_STREAM in the descriptor skips this preference.
bool prefer_generic(const psn_desc_t* desc) {
  if (desc->flags & PSN_STREAM) return false;
  if ((double)desc->T * desc->N * desc->C * desc->Q < 1.5e6) return true;
  return (desc->k - 1) * desc->d > 16;
}

bool shape_eligible(const psn_desc_t* desc) {
  if (desc->flags & PSN_GENERIC) return false;
  if (prefer_generic(desc)) return false;
  if (desc->dtype != PSN_F32 && desc->dtype != PSN_BF16) return false;
  if (desc->k > 8 || desc->d > 3) return false;   // instantiated orders / sawtooth dilations
  // spatial inputs (Q > 1): the per-channel sums of a group are merged from its
  // column sums in shared memory; the forward's 2 + 2k sums must fit the deposit
  if (desc->Q > 1 && desc->k > 4) return false;
  if ((desc->k - 1) * desc->d > kMaxH) return false;
  if (desc->flags & PSN_SMOOTH) return false;     // SMOOTH (finite-difference checks): generic path
  const int es = (int)dtype_size(desc->dtype);
  if ((desc->C * desc->Q * es) % 16 != 0) return false;  // TMA row stride must be a multiple of 16 B
  if (desc->T > (1 << 30) || desc->N > (1 << 30) || desc->C > (1 << 30) || desc->Q > (1 << 20)) return false;
  return true;
}

bool make_plan(const psn_desc_t* desc, bool bwd, Plan& p, bool for_sizing) {
  // workspace sizing ignores PSN_FORCE_GENERIC: a workspace sized while the
  // knob was set must still fit a later streamed call
  if (!(for_sizing ? shape_eligible(desc) : eligible(desc))) return false;
  const DevAttr* da = dev_attr();
  if (!da || !g_encode || da->sms <= 0 || !da->coop) return false;
  const int g_sms = da->sms, g_smem_optin = da->smem_optin;
  const int es = (int)dtype_size(desc->dtype);
  if (desc->T > (1 << 24) || desc->C > (1 << 24)) return false;  // group / iteration indices stay small
  if ((double)desc->T * desc->N * desc->C * desc->Q >= 4294967296.0) return false;  // 32-bit element offsets
  p.T = (int)desc->T;
  p.N = (int)desc->N;
  p.C = (int)desc->C;
  p.Q = (int)desc->Q;
  p.J = p.C * p.Q;
  // channel groups: whole channels, at most 32 (one fold lane each), their
  // columns a multiple of 32 where the channel count allows (so no 32-column
  // tile straddles two groups), and >= 256 columns when that is cheap
  if (p.Q == 1) {
    p.nch = kCols;
  } else {
    int g = p.Q, b = kCols;
    while (b) {  // gcd(Q, 32)
      const int t = g % b;
      g = b;
      b = t;
    }
    p.nch = kCols / g;
    while (p.nch * 2 <= kCols && (long long)p.nch * p.Q < 256) p.nch *= 2;
  }
  if (p.nch > p.C) p.nch = p.C;
  p.ncol = (int)(((long long)p.nch * p.Q + kCols - 1) / kCols);
  p.k = desc->k;
  p.d = desc->d;
  p.H = (p.k - 1) * p.d;
  const Layout L = layout_of(p.k, p.d, es, bwd);
  p.TB = L.TB;
  p.G = (p.C + p.nch - 1) / p.nch;
  p.nbk = (p.N + kBoxN - 1) / kBoxN;
  p.ttl = (p.T + p.TB - 1) / p.TB;
  const long long tpg = (long long)p.ncol * p.nbk * p.ttl;
  if (tpg * (long long)(g_sms + 1) >= (1LL << 32)) return false;  // 32-bit schedule arithmetic
  p.tpg = (int)tpg;
  p.nCTA = g_sms;
  p.lag = env_int(bwd ? "PSN_LAG_BWD" : "PSN_LAG_FWD", env_int("PSN_LAG", 2));
  if (p.lag < 1) p.lag = 1;
  if (p.lag > 6) p.lag = 6;  // the publisher's ring of pre-update running statistics holds 8 groups
  // CTA teams: nT teams stream nT groups concurrently, so each CTA's range of a
  // group spans several tiles and the per-range costs (HEAD rows, schedule,
  // deposit, parameter hand-off) amortise.  Aim at >= 6 tiles per range and
  // give every team the same number of groups (nT divides G, or nT = G).
  // Measured at the metric shape: flat from 4 to 16 teams when balanced, 25%
  // slower with 1 team or an unbalanced split (profiles/r1_sweep_teams.txt).
  // Round 2: at most 2 groups per team when G allows (a balanced split): longer
  // ranges measured faster than more pipelining depth (backward at the metric
  // shape 4 -> 8 teams: 132 -> 129 us; profiles/r2_sweep_plan.txt).
  {
    int nT = (int)((6LL * p.nCTA + p.tpg - 1) / p.tpg);
    if (nT < 1) nT = 1;
    if (nT < p.G / 2) nT = p.G / 2;
    while (nT < p.G && p.G % nT != 0) ++nT;
    if (nT > p.G) nT = p.G;
    nT = env_int(bwd ? "PSN_TEAMS_BWD" : "PSN_TEAMS_FWD", env_int("PSN_TEAMS", nT));
    if (nT < 1) nT = 1;
    if (nT > p.G) nT = p.G;
    if (nT > p.nCTA) nT = p.nCTA;
    p.nT = nT;
  }
  p.stage_bytes = L.stage;
  const int budget = (g_smem_optin > 0 ? g_smem_optin : 232448) - L.fixed - 2048;
  int S = budget / p.stage_bytes;
  const int smax = env_int("PSN_STAGES", 8);
  if (S > smax) S = smax;
  if (S < 2) return false;
  p.S = S;
  return true;
}

static size_t a256(size_t v) { return (v + 255) & ~(size_t)255; }

// workspace, all zeroed per launch: group counters cnt[G], cntA[G] | exponent
// keys emax[G][NV][32] (u32) | per-channel sums acc[G][NV][32] (f64)
static size_t counter_bytes(const Plan& p) { return a256(2 * sizeof(unsigned) * p.G); }
static size_t emax_bytes(const Plan& p, bool bwd) {
  return a256(sizeof(unsigned) * (size_t)p.G * layout_of(p.k, p.d, 4, bwd).NV * kCols);
}
static size_t zeroed_bytes(const Plan& p, bool bwd) {
  return counter_bytes(p) + emax_bytes(p, bwd) + sizeof(double) * (size_t)p.G * layout_of(p.k, p.d, 4, bwd).NV * kCols;
}

size_t workspace_bytes(const psn_desc_t* desc) {
  size_t need = 0;
  for (int b = 0; b < 2; ++b) {
    Plan p;
    if (!make_plan(desc, b == 1, p, true)) continue;
    const size_t bytes = a256(zeroed_bytes(p, b == 1));
    if (bytes > need) need = bytes;
  }
  return need;
}

int stream_encode_maps(const Plan& p, int es, bool bwd, const void* x, const void* dy, CUtensorMap* maps) {
  memset(maps, 0, 4 * sizeof(CUtensorMap));
  const CUtensorMapDataType dt = es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const cuuint64_t dims[3] = {(cuuint64_t)p.J, (cuuint64_t)p.N, (cuuint64_t)p.T};
  const cuuint64_t strides[2] = {(cuuint64_t)p.J * es, (cuuint64_t)p.J * p.N * es};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapL2promotion prom = es == 4 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
  for (int m = 0; m < 4; ++m) {
    const bool is_dy = m >= 2, halo = m & 1;
    if (is_dy && !bwd) continue;
    if (halo && p.H == 0) continue;
    const cuuint32_t box[3] = {(cuuint32_t)kCols, (cuuint32_t)kBoxN, (cuuint32_t)(halo ? p.H : p.TB)};
    CUresult r = g_encode(&maps[m], dt, 3, const_cast<void*>(is_dy ? dy : x), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, prom,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(PSN_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  }
  return PSN_OK;
}

struct Ws {
  unsigned* cnt;
  unsigned* cntA;
  unsigned* emax;
  double* acc;
};

static Ws carve(void* ws, const Plan& p, bool bwd) {
  Ws w;
  w.cnt = (unsigned*)ws;
  w.cntA = w.cnt + p.G;
  w.emax = (unsigned*)((char*)ws + counter_bytes(p));
  w.acc = (double*)((char*)ws + counter_bytes(p) + emax_bytes(p, bwd));
  return w;
}

static int dispatch(const psn_desc_t* desc, bool bwd, const Args& a, const void* x, const void* dy, cudaStream_t st) {
  const int k = desc->k, d = desc->d;
  if (desc->dtype == PSN_F32)
    return bwd ? run_f32_bwd(k, d, a, x, dy, st) : run_f32_fwd(k, d, a, x, dy, st);
  return bwd ? run_bf16_bwd(k, d, a, x, dy, st) : run_bf16_fwd(k, d, a, x, dy, st);
}

int forward(const psn_desc_t* desc, const Plan& p, const void* x, const double* W, const double* gamma,
            const double* beta, double* rm, double* rv, void* out, double* fold, void* ws, cudaStream_t st) {
  Ws w = carve(ws, p, false);
  if (cudaMemsetAsync(ws, 0, zeroed_bytes(p, false), st) != cudaSuccess)
    return fail(PSN_ERR_CUDA, "memset of stream counters failed");
  Args a;
  memset(&a, 0, sizeof(a));
  a.p = p;
  a.out = out;
  a.W = W;
  a.gamma = gamma;
  a.beta = beta;
  a.rm = rm;
  a.rv = rv;
  a.fold = fold;
  a.cnt = w.cnt;
  a.cntA = w.cntA;
  a.emax = w.emax;
  a.acc = w.acc;
  a.flags = desc->flags;
  a.shared = (desc->flags & PSN_SHARED) ? 1 : 0;
  a.eps = desc->eps;
  a.momentum = desc->momentum;
  a.x = x;
  a.wait_ns = wait_limit_ns();
  a.trace = env_int("PSN_TRACE", 0);
  a.ablate = env_int("PSN_ABLATE", 0);
  return dispatch(desc, false, a, x, nullptr, st);
}

int backward(const psn_desc_t* desc, const Plan& p, const void* x, const void* dy, const double* W,
             const double* gamma, const double* fold, void* dx, double* dW, double* dgamma, double* dbeta,
             void* ws, cudaStream_t st) {
  Ws w = carve(ws, p, true);
  if (cudaMemsetAsync(ws, 0, zeroed_bytes(p, true), st) != cudaSuccess)
    return fail(PSN_ERR_CUDA, "memset of stream counters failed");
  Args a;
  memset(&a, 0, sizeof(a));
  a.p = p;
  a.out = dx;
  a.W = W;
  a.gamma = gamma;
  a.fold = const_cast<double*>(fold);
  a.dW = dW;
  a.dgamma = dgamma;
  a.dbeta = dbeta;
  a.cnt = w.cnt;
  a.cntA = w.cntA;
  a.emax = w.emax;
  a.acc = w.acc;
  a.flags = desc->flags;
  a.shared = (desc->flags & PSN_SHARED) ? 1 : 0;
  a.eps = desc->eps;
  a.momentum = desc->momentum;
  a.x = x;
  a.wait_ns = wait_limit_ns();
  a.trace = env_int("PSN_TRACE", 0);
  a.ablate = env_int("PSN_ABLATE", 0);
  Surrogate s;
  s.kind = desc->surrogate;
  if (desc->surrogate == PSN_ARCTAN) {
    s.c = (float)(0.5 * 3.141592653589793 * desc->alpha);
    s.scale = (float)(desc->alpha / 2.0);
  } else {
    s.c = (float)desc->alpha;
    s.scale = 1.0f;
  }
  a.sur = s;
  {
    const double c = desc->surrogate == PSN_ARCTAN ? 0.5 * 3.141592653589793 * desc->alpha : desc->alpha;
    a.scc = desc->surrogate == PSN_ARCTAN ? c * c : c;
  }
  a.sscale = desc->surrogate == PSN_ARCTAN ? desc->alpha / 2.0 : 1.0;
  return dispatch(desc, true, a, x, dy, st);
}

}  // namespace stream
}  // namespace psn
