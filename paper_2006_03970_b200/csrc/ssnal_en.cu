// ssnal_en.cu — C ABI + solver driver for the B200 SsNAL-EN hot path.
//
// The driver enqueues the kernels of k_aty.cuh / k_newton.cuh on the handle's stream
// and runs Algorithm 1 with the readings of DESIGN.md.  Control
// decisions (inner stop, branch on r, Armijo) read one small EvalOut record back per
// ψ evaluation; all vector arithmetic stays on the device.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <stdarg.h>

#include <algorithm>
#include <chrono>
#include <string>
#include <vector>

#include "k_aty.cuh"
#include "k_ctl.cuh"
#include "k_newton.cuh"
#include "k_chol_dsm.cuh"
#include "k_chol_d2.cuh"
#include "k_small.cuh"
#include "k_small_cl.cuh"
#include "k_peer.cuh"
#include "ssnal_en.h"

using namespace ssn;

namespace {

thread_local std::string g_err;

void set_err(const char* fmt, ...) __attribute__((format(printf, 1, 2)));
void set_err(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
}

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      set_err("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_));       \
      return SSNAL_ECUDA;                                                                \
    }                                                                                    \
  } while (0)

#define CKL()                                                                            \
  do {                                                                                   \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess) {                                                             \
      set_err("%s:%d launch: %s", __FILE__, __LINE__, cudaGetErrorString(e_));           \
      return SSNAL_ECUDA;                                                                \
    }                                                                                    \
  } while (0)

constexpr double kEps = 2.220446049250313e-16;

Scal make_scal(double sigma, double l1, double l2) {
  // Same operation order as the oracle (plain IEEE double, no contraction on x86-64).
  Scal s;
  s.sigma = sigma;
  s.l1 = l1;
  s.l2 = l2;
  s.thr = sigma * l1;
  s.den = 1.0 + sigma * l2;
  s.cpsi = (1.0 + sigma * l2) / (2.0 * sigma);
  s.kappa = sigma / (1.0 + sigma * l2);
  return s;
}

int mr_bucket(int64_t m) {
  if (m <= 32) return 1;
  if (m <= 64) return 2;
  if (m <= 128) return 4;
  if (m <= 256) return 8;
  if (m <= 512) return 16;
  if (m <= 800) return 25;
  return 32;
}

typedef void (*k1_fn)(const K1Params);

template <bool R>
k1_fn k1_for_r(int mr) {
  switch (mr) {
    case 1: return k1_aty_fused<1, R>;
    case 2: return k1_aty_fused<2, R>;
    case 4: return k1_aty_fused<4, R>;
    case 8: return k1_aty_fused<8, R>;
    case 16: return k1_aty_fused<16, R>;
    case 25: return k1_aty_fused<25, R>;
    default: return k1_aty_fused<32, R>;
  }
}
// reuse: the instantiation that checks y == −b and serves Aᵀy from the kept Aᵀb (R40)
k1_fn k1_for(int mr, bool reuse = false) { return reuse ? k1_for_r<true>(mr) : k1_for_r<false>(mr); }
k1_fn k1g_for(int tw, bool reuse = false) {
  if (reuse) return tw <= 1 ? k1g_aty_fused<1, true> : k1g_aty_fused<2, true>;
  return tw <= 1 ? k1g_aty_fused<1> : k1g_aty_fused<2>;
}

// Kernels that read individual columns are templated on the column accessor (AccA: fp64 design,
// AccG: packed genotype codes, §8(f4)); these tables pick the register-tile variant.
template <class Acc>
using gax_fn = void (*)(const Acc, int64_t, const int32_t*, const double*, int64_t, const int64_t*, double*, int*,
                        const int*);
template <class Acc>
gax_fn<Acc> gax_for(int mr) {
  switch (mr) {
    case 1: return k_gather_axpy<Acc, 1>;
    case 2: return k_gather_axpy<Acc, 2>;
    case 4: return k_gather_axpy<Acc, 4>;
    case 8: return k_gather_axpy<Acc, 8>;
    case 16: return k_gather_axpy<Acc, 16>;
    case 25: return k_gather_axpy<Acc, 25>;
    default: return k_gather_axpy<Acc, 32>;
  }
}
template <class Acc>
using cg_fn = void (*)(const CgParams, const Acc);
template <class Acc>
cg_fn<Acc> cg_for(int mr) {
  switch (mr) {
    case 1: return k_cg_newton<Acc, 1>;
    case 2: return k_cg_newton<Acc, 2>;
    case 4: return k_cg_newton<Acc, 4>;
    case 8: return k_cg_newton<Acc, 8>;
    case 16: return k_cg_newton<Acc, 16>;
    case 25: return k_cg_newton<Acc, 25>;
    default: return k_cg_newton<Acc, 32>;
  }
}

// Packed genotype validation: one warp per column; flag[0] = codes of value 3 or non-finite
// table entries, flag[1] = columns whose decoded entries are all zero.
__global__ void k_validate_geno(const uint8_t* codes, int64_t cs, const double* tab, int64_t m, int64_t n,
                                const double* b, int* flag) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const AccG acc{codes, cs, tab};
  for (int64_t i = wid; i < n; i += nw) {
    int bad = 0, nz = 0;
    for (int64_t k = lane; k < m; k += 32) {
      const unsigned g = (codes[i * cs + (k >> 2)] >> (2 * (int)(k & 3))) & 3u;
      if (g == 3u) bad = 1;
      const double v = acc.ld(i, k);
      if (!isfinite(v)) bad = 1;
      if (v != 0.0) nz = 1;
    }
    bad = __any_sync(0xffffffffu, bad);
    nz = __any_sync(0xffffffffu, nz);
    if (lane == 0) {
      if (bad) atomicAdd(&flag[0], 1);
      if (!nz) atomicAdd(&flag[1], 1);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    int bad = 0;
    for (int64_t k = threadIdx.x; k < m; k += 32)
      if (!isfinite(b[k])) bad = 1;
    bad = __any_sync(0xffffffffu, bad);
    if (threadIdx.x == 0 && bad) atomicAdd(&flag[0], 1);
  }
}

// Validation of A on the device: one warp per column; flag[0] = non-finite count,
// flag[1] = zero-column count.
__global__ void k_validate(const double* A, int64_t m, int64_t n, const double* b, int* flag) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = wid; i < n; i += nw) {
    const double* col = A + i * m;
    int bad = 0, nz = 0;
    for (int64_t k = lane; k < m; k += 32) {
      const double v = col[k];
      if (!isfinite(v)) bad = 1;
      if (v != 0.0) nz = 1;
    }
    bad = __any_sync(0xffffffffu, bad);
    nz = __any_sync(0xffffffffu, nz);
    if (lane == 0) {
      if (bad) atomicAdd(&flag[0], 1);
      if (!nz) atomicAdd(&flag[1], 1);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    int bad = 0;
    for (int64_t k = threadIdx.x; k < m; k += 32)
      if (!isfinite(b[k])) bad = 1;
    bad = __any_sync(0xffffffffu, bad);
    if (threadIdx.x == 0 && bad) atomicAdd(&flag[0], 1);
  }
}

// Primal objective pieces at x (support Jx, Px, rx) with resid = A x − b:
// out[0] = ½‖resid‖², out[1] = Σ|x|, out[2] = Σ x², out[3] = nnz
__global__ void k_objective(int64_t m, const double* resid, const double* Px, const int64_t* rx, double* out) {
  __shared__ double red[3][32];
  const int tid = threadIdx.x;
  double a = 0, l1 = 0, q = 0;
  for (int64_t k = tid; k < m; k += blockDim.x) a += resid[k] * resid[k];
  const int64_t r = *rx;
  for (int64_t i = tid; i < r; i += blockDim.x) {
    l1 += fabs(Px[i]);
    q += Px[i] * Px[i];
  }
  a = warp_allsum(a);
  l1 = warp_allsum(l1);
  q = warp_allsum(q);
  if ((tid & 31) == 0) {
    red[0][tid >> 5] = a;
    red[1][tid >> 5] = l1;
    red[2][tid >> 5] = q;
  }
  __syncthreads();
  if (tid == 0) {
    double s[3] = {0, 0, 0};
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
      for (int j = 0; j < 3; ++j) s[j] += red[j][w];
    out[0] = 0.5 * s[0];
    out[1] = s[1];
    out[2] = s[2];
    out[3] = (double)r;
  }
}

// KKT certificate: with w = Aᵀ(Ax − b), c_i = −w_i − λ2 x_i and
// v_i = |c_i − λ1 sign x_i| (x_i ≠ 0) or (|c_i| − λ1)₊; per-block max → out[blockIdx] (max is exact).
__global__ void __launch_bounds__(256) k_kkt_viol(int64_t n, const double* __restrict__ w, const double* __restrict__ x,
                                                  double l1, double l2, double* out) {
  __shared__ double red[8];
  double v = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = x[i];
    const double c = -w[i] - l2 * xi;
    const double vi = xi > 0.0 ? fabs(c - l1) : (xi < 0.0 ? fabs(c + l1) : fmax(fabs(c) - l1, 0.0));
    v = fmax(v, vi);
  }
  v = warp_allmax(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = red[0];
    for (int q = 1; q < 8; ++q) m = fmax(m, red[q]);
    out[blockIdx.x] = m;
  }
}

__global__ void k_max_reduce(const double* in, int cnt, double* out) {
  double v = 0.0;
  for (int q = threadIdx.x; q < cnt; q += 32) v = fmax(v, in[q]);
  v = warp_allmax(v);
  if (threadIdx.x == 0) *out = v;
}

}  // namespace

// λ path results, one pinned (mapped) slot per point: written by the host-side copies of a point solved
// by its own graph launch, or directly by k_path_end in the device-resident path graph.
struct PathSlot {
  DevCtl ctl;
  EvalOut ev;
  double scratch[64];
  double l1, l2;
  int warm_pass, pad;
  int64_t launches;
  unsigned long long t0, t1;  // path graph: %globaltimer at the point's begin / end
};
// device state of the path graph (ssnal_en_solve_path_device, points 1 … npts − 1 in one launch)
struct PathDev {
  const double* l1s;
  const double* l2s;
  double* xout;          // the caller's x_out (npts × n)
  long long i, npts;     // current point, point count
  int carry_sigma, pad;
  unsigned long long t0;
  DevCtl tmpl;           // the solve settings (σ0 in tmpl.sigma), copied into the control block per point
};

namespace {
// point i > 0 begins (reading R38/R39: from the previous point's final x, y, w and — with
// carry_sigma — σ, all still in the handle): its settings and λ into the control block, |supp x0|
// for the stats, and the outer loop armed
__global__ void k_path_begin(DevCtl* C, PathDev* pd, int64_t* r_dev, cudaGraphConditionalHandle h_outer) {
  const long long i = pd->i;
  const double sig = pd->carry_sigma ? C->sigma_final : pd->tmpl.sigma;
  DevCtl c = pd->tmpl;
  c.l1 = pd->l1s[i];
  c.l2 = pd->l2s[i];
  c.sigma = sig;
  *C = c;
  r_dev[4] = r_dev[2];
  pd->t0 = global_ns();
  cudaGraphSetConditional(h_outer, 1);
}
__global__ void k_path_copy_x(const double* __restrict__ x, const PathDev* pd, int64_t n) {
  double* dst = pd->xout + pd->i * n;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    dst[k] = x[k];
}
// point i ends: its control block, final evaluation record and objective pieces into its (mapped
// pinned) slot, the next point or the end of the path
__global__ void k_path_end(const DevCtl* C, const EvalOut* ev, const double* scratch, const int64_t* r_dev,
                           PathSlot* slots, PathDev* pd, cudaGraphConditionalHandle h_path) {
  const long long i = pd->i;
  PathSlot* sl = slots + i;
  sl->ctl = *C;
  sl->ev = ev[0];
  for (int j = 16; j < 20; ++j) sl->scratch[j] = scratch[j];
  *reinterpret_cast<long long*>(sl->scratch + 20) = r_dev[4];
  sl->t0 = pd->t0;
  sl->t1 = global_ns();
  __threadfence_system();
  pd->i = i + 1;
  cudaGraphSetConditional(h_path, i + 1 < pd->npts);
}
}  // namespace

// ===========================================================================
struct ssnal_en_problem {
  int64_t m = 0, n = 0;
  int dev = 0, nsm = 0;
  const double* A = nullptr;
  const double* b = nullptr;
  double* A_own = nullptr;
  // packed genotype storage (§8(f4)); fmt = 1 when A is given as codes + tables
  int fmt = 0;
  const uint8_t* codes = nullptr;
  const double* tab = nullptr;
  int64_t cstride = 0;
  uint8_t* codes_own = nullptr;
  double* tab_own = nullptr;
  int TW = 1;
  double* b_own = nullptr;
  cudaStream_t st = nullptr;
  // K1 configuration
  int MR = 0, C = 0, S = 0, G = 0;
  int64_t T = 0;
  size_t k1_smem = 0;
  uint32_t k1_bfr_off = 0;  // K1g: offset of the shared B-fragment table
  uint32_t stage_elems = 0, xstage_elems = 0;
  int cluster = 16;
  size_t chol_smem = 0;
  int use_dsm = 1;   // option chol_dsm: DSMEM-resident K4 for N ≤ 512 when schedulable
  int dsm_ok = 0;    // … schedulable on this device
  int chol_dsm = 0;  // use_dsm && dsm_ok
  int use_d2 = 1;    // option chol_d2: split-ownership DSMEM K4 (k_chol_d2) for 96 < N ≤ 512
  int d2_ok = 0;     // … schedulable on this device
  int gax_grid = 0;
  int use_gram_sk = 1;  // option gram_sk: K3 as one cooperative round of (tile, K-slice) items (k_gram_sk)
  int gsk_grid = 0;     // its grid: SMs × co-resident CTAs per SM (≤ 2)
  int gsk_minch = 1;    // option gram_sk_minch: ≥ this many 32-wide reduction chunks per (tile, slice) item
  double* gsk_part = nullptr;  // its partial tiles (max(grid, tiles) × 64 × 64)
  unsigned* gsk_cnt = nullptr;  // its per-tile arrival / finish counters
  // device buffers
  double* w[3] = {nullptr, nullptr, nullptr};  // current / trial / backtrack
  double* x = nullptr;
  int32_t* seg_idx = nullptr;
  double* seg_P = nullptr;
  uint8_t* mask = nullptr;
  int* cta_cnt = nullptr;
  double* part_scal = nullptr;
  double* part_vec = nullptr;
  int32_t* J[2] = {nullptr, nullptr};
  double* PJ[2] = {nullptr, nullptr};
  int64_t* r_dev = nullptr;  // [0], [1]: J sets; [2]: support of x
  int32_t* Jx = nullptr;
  double* Px = nullptr;
  double* y[2] = {nullptr, nullptr};
  double* g[2] = {nullptr, nullptr};
  double* d = nullptr;
  double* u = nullptr;
  double* tmpm = nullptr;
  double* Mmat = nullptr;
  double* Msel = nullptr;  // model selection: (2m) × m with appended rows (allocated on first use)
  double* Winv = nullptr;  // inverses of the 32 × 32 diagonal blocks of L
  double* W = nullptr;
  int W_splits = 0;
  int* info = nullptr;
  int* kflag = nullptr;  // K4 W-ready flags (one per panel)
  EvalOut* ev_dev = nullptr;   // slots
  EvalOut* ev_host = nullptr;  // mapped pinned mirror (GPU writes it directly)
  EvalOut* ev_host_dev = nullptr;  // device alias of ev_host
  unsigned long long ev_seq = 0;
  double* scratch = nullptr;   // small device scratch (objective, λmax)
  double* scratch_host = nullptr;
  int* flags = nullptr;
  double* blk = nullptr;       // eval-reduce per-CTA partials
  int* gax_valid = nullptr;    // device-r gather: CTA had columns
  double* cg_res = nullptr;    // K6: residual (m), per-CTA partials (nsm × m), scalars (2 nsm)
  double* cg_parts = nullptr;
  double* cg_scal = nullptr;
  size_t cg_smem_bytes = 0;
  unsigned* ticket = nullptr;  // eval-reduce last-block counter
  // state
  double lambda_max = 0, nb = 0;
  // options
  double sigma_factor = 5.0, sigma_max = 1e8, mu = 0.2, beta = 0.5;
  int max_outer = 100, max_inner = 100, max_bt = 50, init_mode = 1, time_k1 = 0, certify = 0;
  double cg_ratio = 0.0, cg_threshold = 1e4, cg_tol = 1e-10;  // Newton strategy (R32)
  int cg_maxit = 1000;
  // §8(f3) column sharding: this handle holds one block of columns; every cross-column sum goes
  // through the caller's all-reduce (host-driven control, identical decisions on every rank)
  ssnal_en_allreduce_fn comm_fn = nullptr;
  void* comm_ctx = nullptr;
  int comm_rank = 0, comm_size = 0;  // comm_size > 0: sharded
  double* xbuf = nullptr;            // exchange buffer, m² + 2m + 64 doubles (device)
  int64_t* rg_dev = nullptr;         // global r for the eval record
  int32_t* iota = nullptr;           // 0 … m−1: indices of the gathered active columns
  double* comm_host = nullptr;       // pinned staging (nranks + 8 doubles)
  // §8(f3) device-resident exchanges over peer memory (k_peer.cuh; ssnal_en_peer_export / _attach):
  // the exchanges are kernels, so sharded solves keep the graph's device-resident control
  int peer = 0;                                     // 1: attached (comm_fn unused)
  char* peer_region = nullptr;                      // this rank's region (cudaMalloc: IPC-exportable)
  int peer_nranks = 0;                              // ranks the region was sized for
  char* peer_open[kPeerMaxRanks] = {};              // the peers' regions mapped by cudaIpcOpenMemHandle
  PeerComm pc = {};
  unsigned long long* peer_epoch = nullptr;         // [0] epoch; then ticket (unsigned), err (int)
  int32_t* peer_idx = nullptr;                      // gathered-column index list (SMW all-gather)
  CholArgs* chol_args = nullptr;  // graph mode: K4 outputs per exact branch (device, 2 entries)
  int inner_tol_mode = 0;  // 1: tol_in = max(tol, 0.1 res3 at the outer start) (R37)
  int inject_fail = 0;    // test hook: the next N factorisations of a solve report failure
  double jitter = 1e-10;  // factor retry M_ii ← M_ii (1 + jitter) after a non-positive pivot (R36)
  // counters for the current call
  int64_t launches = 0;
  void* arena = nullptr;    // all device buffers above (one allocation)
  void* arena_h = nullptr;  // mapped pinned host buffers (one allocation)
  double stat_l1 = 0, stat_l2 = 0;
  bool stat_warm_pass = false;
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;  // solve timing (persistent)
  std::vector<cudaEvent_t> ev_pool;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> k1_pending;
  double k1_time = 0;
  int k1_count = 0;
  // graph mode (device-resident control, k_ctl.cuh)
  int use_graph = 1;
  int use_small = 1;
  int use_small_cl = 1;  // option small_cluster: the 16-CTA cluster version of the small-problem solve
  int small_cl_ok = 0;   // … schedulable on this device
  int eval16_ok = 0;  // the 16-CTA-cluster evaluation kernels are schedulable (m ≤ 512)  // option small: one-CTA solve (k_small_solve) for m ≤ 64, n ≤ 1024
  ssn::DevCtl* ctl = nullptr;       // device control block
  ssn::DevCtl* ctl_host = nullptr;  // pinned staging (inputs in, results back)
  EvalOut* ev_out_host = nullptr;   // pinned: final EvalOut of the current point
  bool capturing = false;
  int cap_depth = 0;
  cudaStream_t cap[3] = {nullptr, nullptr, nullptr};
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  int seg_kernels[5] = {0, 0, 0, 0, 0};
  int seg_kernels_r[5] = {0, 0, 0, 0, 0};  // the reuse graph's (its inner body carries the redo nodes)
  bool stat_graph_r = false;               // the pending solve ran the reuse graph
  bool graph_pending = false;
  // λ-path call (ssnal_en_solve_path_device): per-point pinned result slots and timing events
  void* path_slots = nullptr;
  int64_t path_cap = 0;
  std::vector<cudaEvent_t> path_ev;
  // option carry_sigma (reading R38): path point i starts at point i − 1's final σ
  int carry_sigma = 1;
  // option carry_dual (reading R39): path point i > 0 also starts at point i − 1's final dual
  // iterate y (and its w = Aᵀy), so the warm start costs no Aᵀ pass; option warm_dual: the same for
  // a single warm-started solve (the handle's y, w from its previous solve instead of y0 = A x0 − b)
  int carry_dual = 1;
  int warm_dual = 0;
  // option reuse_atb (reading R40): create keeps Aᵀb (the λmax pass) in atb; the first Newton step of a
  // cold start (x0 = 0 ⇒ y0 = 0, d = −b exactly) takes Aᵀ(y0 + d) = −Aᵀb from it — bitwise what the
  // streaming K1 / K1g launch writes — instead of a pass over A.
  int reuse_atb = 1;
  double* atb = nullptr;
  unsigned long long* gate_cnt = nullptr;  // k_atb_gate scratch (count, ticket), kept zero
  int* gate_flag_host = nullptr;           // mapped pinned: the gate's decision (host-driven control, statistics)
  int* gate_flag_dev = nullptr;            // its device alias
  int reuse_psi_only = 1;                  // above reuse_frac: serve ψ only, redo streamed if s = 1 is accepted
  int64_t reuse_min_bytes = 2ll << 30;     // no gate for designs below 2 GB: its synchronisation (and the REUSE
                                           // instantiation's slower small-n launch) cost cfg2 (0.4 GB) +0.25 ms per path
  bool prepared = false;                   // create_prepare ran (configure + allocate)
  bool capture_reuse = false;              // capture_graph: the trial K1 node is the REUSE instantiation
  cudaGraph_t graph_r = nullptr;           // second solve graph (REUSE trial K1), built on first use
  cudaGraphExec_t gexec_r = nullptr;
  double reuse_frac = 0.3;                 // gate: reuse while #{|Aᵀb|_i > λ1} ≤ reuse_frac · n (the gather of those
                                           // columns runs at ~4 TB/s against 7.1 for the stream: break-even near n/2)
  int64_t atb_reuses = 0;  // cold solves started with the first trial served from atb (get_info "atb_reuses")
  // device-resident λ path (option path_graph): points 1 … npts − 1 of ssnal_en_solve_path_device
  // in ONE launch of a graph whose WHILE loop runs the solve graph's body once per point
  int use_path_graph = 1;
  cudaStream_t cap_path = nullptr;
  cudaGraph_t pgraph = nullptr;
  cudaGraphExec_t pgexec = nullptr;
  PathDev* pdev = nullptr;       // device
  PathDev* pdev_host = nullptr;  // pinned staging
  double* path_l = nullptr;      // device λ1[path_lcap], λ2[path_lcap]
  int64_t path_lcap = 0;
  int pgraph_fixed = 0;          // kernel nodes per point outside the solve's segments
  // small-problem cluster path: the caller's device x buffer the kernel writes directly (no copy)
  double* direct_xout = nullptr;
  bool xout_done = false;
};

namespace {

// Large per-handle allocations (the owned copy of A, the buffer arena) come from the device's
// stream-ordered memory pool with an unlimited release threshold: destroy returns them to the
// pool and the next create reuses them without mapping / unmapping device memory.
void* pool_alloc(size_t bytes) {
  static bool init = false;
  if (!init) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    init = true;
  }
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes, 0) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (cudaStreamSynchronize(0) != cudaSuccess) return nullptr;
  return p;
}
void pool_free(void* p) {
  if (p) {
    cudaFreeAsync(p, 0);
    cudaStreamSynchronize(0);
  }
}

int alloc(void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes > 0 ? bytes : 16);
  if (e != cudaSuccess) {
    set_err("cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
    return SSNAL_ECUDA;
  }
  return SSNAL_OK;
}

#define AL(ptr, bytes)                                            \
  do {                                                            \
    int rc_ = alloc((void**)&(ptr), (bytes));                     \
    if (rc_) return rc_;                                          \
  } while (0)

// Largest k_chol_cluster cluster size ≤ want (halving) that the occupancy calculator can schedule.
int chol_cluster_fit(ssnal_en_problem* P, int want) {
  for (; want > 1; want /= 2) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(want);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = P->chol_smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = want;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclus = 0;
    if (cudaOccupancyMaxActiveClusters(&nclus, k_chol_cluster, &cfg) == cudaSuccess && nclus >= 1) break;
    cudaGetLastError();
  }
  return want < 1 ? 1 : want;
}

int configure(ssnal_en_problem* P) {
  const int64_t m = P->m, n = P->n;
  P->MR = mr_bucket(m);
  // bytes of A per column in a K1 stage: fp64 (8m) or packed codes + table (cstride + 24)
  const int64_t bytes_col = P->fmt ? P->cstride + 24 : 8 * m;
  // ~32 KB of A per tile (fp64); packed codes: ~16 KB, so ≥ 2 tiles per consumer warp fit the ring
  // (K1g is issue-bound, so a consumer must find its next tile loaded when it finishes one)
  int k = (int)((P->fmt ? 16384 : 32768) / (K1_GRP * bytes_col));
  if (k < 1) k = 1;
  if (k > 32) k = 32;  // ≤ 256 columns per tile
  {  // small n: smaller tiles, so the pass spreads over the SMs and their consumer warps (a warp
     // owns whole tiles; cfg1 with 32 KB tiles ran 13 tiles on 13 warps, 14.6 µs per pass)
    const int64_t kmax = (n + (int64_t)K1_GRP * P->nsm * K1_NWC - 1) / ((int64_t)K1_GRP * P->nsm * K1_NWC);
    if (k > kmax) k = (int)(kmax < 1 ? 1 : kmax);
  }
  P->C = K1_GRP * k;   // multiple of 8: one mask byte per 8 columns, 16-B aligned tiles
  if (P->fmt) {
    P->TW = (int)((P->cstride / 4 + 31) / 32);
    const int64_t code_elems = (P->cstride * P->C + 7) / 8;  // = cstride·C/8 (cstride % 16 == 0)
    P->stage_elems = (uint32_t)((code_elems + 3 * P->C + 15) / 16 * 16);
  } else {
    P->stage_elems = (uint32_t)(((int64_t)P->C * m + 15) / 16 * 16);
  }
  P->xstage_elems = (uint32_t)((P->C + 15) / 16 * 16);
  const size_t per_stage = (size_t)(P->stage_elems + P->xstage_elems) * 8;
  // ring depth: as many stages as fit ~224 KB, at most 6 (measured at n = 1e7 / 1e6, r ≈ 1e-4 n:
  // m = 500 (32 KB stages) 5 / 6 / 7 stages 7.15 / 7.13 / 6.74 TB/s; m = 800 (51 KB stages) 3 / 4
  // stages 6.78 / 7.12 TB/s — profiles/r2_k1_stages_sweep.jsonl, r2_k1_stages_m800.jsonl)
  // (packed genotypes keep a 200 KB ring of ≤ 14 stages: 13 → 14 stages was 1% slower at cfg4)
  int S = (int)(((P->fmt ? 200 : 224) * 1024) / per_stage);
  if (S > (P->fmt ? 2 * K1_NWC : 6)) S = P->fmt ? 2 * K1_NWC : 6;
  if (S < 2) S = 2;
  while ((size_t)S * P->stage_elems < (size_t)K1_NWC * m + K1_NWC * 4 + K1_NWC) ++S;
  P->S = S;
  P->k1_smem = (size_t)S * per_stage + 2 * S * 8 + 64 + 4 * S + 16;
  if (P->fmt) {  // K1g: shared B-fragment table after the ring and barriers (32 × 32 × 8 B)
    P->k1_bfr_off = (uint32_t)((P->k1_smem + 15) / 16 * 16);
    P->k1_smem = P->k1_bfr_off + 32 * 32 * 8;
  }
  P->T = (n + P->C - 1) / P->C;
  P->G = (int)(P->T < P->nsm ? P->T : P->nsm);
  P->gax_grid = P->nsm;
  if (P->k1_smem > 227 * 1024) {
    set_err("K1 shared memory %zu exceeds 227 KB (m=%lld)", P->k1_smem, (long long)m);
    return SSNAL_EINVAL;
  }
  // the attribute is per function and process-wide: always the device maximum, so that a later handle with a
  // smaller ring (same MR bucket) cannot lower the cap under a live handle with a larger one
  CK(cudaFuncSetAttribute(P->fmt ? k1g_for(P->TW) : k1_for(P->MR), cudaFuncAttributeMaxDynamicSharedMemorySize,
                          227 * 1024));
  CK(cudaFuncSetAttribute(P->fmt ? k1g_for(P->TW, true) : k1_for(P->MR, true),
                          cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  P->cg_smem_bytes = cg_smem(m);
  // per-function caps at the size of the largest supported m (1024), not this handle's (see above)
  const int gsm_cap = 8 * 1024 * 8, cg_cap = (int)cg_smem(1024);
  if (P->fmt) {
    CK(cudaFuncSetAttribute(gax_for<AccG>(P->MR), cudaFuncAttributeMaxDynamicSharedMemorySize, gsm_cap));
    CK(cudaFuncSetAttribute(cg_for<AccG>(P->MR), cudaFuncAttributeMaxDynamicSharedMemorySize, cg_cap));
  } else {
    CK(cudaFuncSetAttribute(gax_for<AccA>(P->MR), cudaFuncAttributeMaxDynamicSharedMemorySize, gsm_cap));
    CK(cudaFuncSetAttribute(cg_for<AccA>(P->MR), cudaFuncAttributeMaxDynamicSharedMemorySize, cg_cap));
  }
  P->chol_smem = kCholSmem;
  CK(cudaFuncSetAttribute(k_chol_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->chol_smem));
  CK(cudaFuncSetAttribute(k_chol_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  // cluster size: 16 (non-portable) when schedulable, else 8
  P->cluster = chol_cluster_fit(P, P->cluster > 0 ? P->cluster : 16);
  // DSMEM-resident K4 (N ≤ 512): needs a schedulable 16-CTA cluster with ~175 KB smem per CTA
  P->dsm_ok = 0;
  {
    CK(cudaFuncSetAttribute(k_chol_dsm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDsmSmem));
    CK(cudaFuncSetAttribute(k_chol_dsm, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kDsmCS);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = kDsmSmem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kDsmCS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclus = 0;
    if (cudaOccupancyMaxActiveClusters(&nclus, k_chol_dsm, &cfg) == cudaSuccess && nclus >= 1) P->dsm_ok = 1;
    cudaGetLastError();
  }
  P->chol_dsm = P->use_dsm && P->dsm_ok;
  P->d2_ok = 0;
  if (P->dsm_ok) {
    CK(cudaFuncSetAttribute(k_chol_d2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kD2Smem));
    CK(cudaFuncSetAttribute(k_chol_d2, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kDsmCS);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = kD2Smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kDsmCS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nclus = 0;
    if (cudaOccupancyMaxActiveClusters(&nclus, k_chol_d2, &cfg) == cudaSuccess && nclus >= 1) P->d2_ok = 1;
    cudaGetLastError();
  }
  if (P->d2_ok) {
    CK(cudaFuncSetAttribute(k_chol_dsm_any, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kD2Smem));
    CK(cudaFuncSetAttribute(k_chol_dsm_any, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  }
  {  // k_gram_sk: co-resident CTAs per SM for its cooperative launch (both accessors: the sharded SMW
     // form reads gathered fp64 columns even on a genotype handle)
    int oa = 0, og = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oa, k_gram_sk<AccA>, 256, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&og, k_gram_sk<AccG>, 256, 0));
    int occ = std::min(std::min(oa, og), 2);
    P->gsk_grid = P->nsm * std::max(occ, 1);
    if (occ < 1) P->use_gram_sk = 0;
  }
  P->eval16_ok = 0;
  if (P->m <= 32 * kEval16) {
    CK(cudaFuncSetAttribute(k_eval_reduce16, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(k_eval_ctl16<kHookInnerBegin>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(k_eval_ctl16<kHookArmijo>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(k_eval_ctl16<kHookArmijoRedo>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(k_eval_ctl16<kHookBacktrack>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(k_eval_ctl16<kHookInnerEnd>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kEval16);
    cfg.blockDim = dim3(K5_THREADS);
    int nclus = 0;
    if (cudaOccupancyMaxActiveClusters(&nclus, k_eval_reduce16, &cfg) == cudaSuccess && nclus >= 1) P->eval16_ok = 1;
    cudaGetLastError();
  }
  P->small_cl_ok = 0;
  if (P->m <= kSmallMaxM && P->n <= kSmallMaxN) {
    CK(cudaFuncSetAttribute(k_small_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmallSmem));
    CK(cudaFuncSetAttribute(k_small_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kClSmem));
    CK(cudaFuncSetAttribute(k_small_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kClCtas);
    cfg.blockDim = dim3(kClThreads);
    cfg.dynamicSmemBytes = kClSmem;
    int nclus = 0;
    if (cudaOccupancyMaxActiveClusters(&nclus, k_small_cl, &cfg) == cudaSuccess && nclus >= 1) P->small_cl_ok = 1;
    cudaGetLastError();
  }
  return SSNAL_OK;
}

// All per-handle buffers live in one device arena and one mapped pinned host arena: create and
// destroy cost two allocations instead of ~40 (cudaFree / cudaFreeHost synchronise the device).
struct Arena {
  std::vector<std::pair<void**, size_t>> req;
  size_t total = 0;
  void add(void** p, size_t bytes) {
    req.push_back({p, total});
    total += (bytes + 255) / 256 * 256;
  }
  void assign(char* base) {
    for (auto& r : req) *r.first = base + r.second;
  }
};

int allocate(ssnal_en_problem* P) {
  const int64_t m = P->m, n = P->n;
  Arena d;
  for (int i = 0; i < 3; ++i) d.add((void**)&P->w[i], n * 8);
  d.add((void**)&P->atb, n * 8);
  d.add((void**)&P->gate_cnt, 64);
  d.add((void**)&P->x, n * 8);
  d.add((void**)&P->seg_idx, n * 4);
  d.add((void**)&P->mask, n / 8 + 64);
  d.add((void**)&P->seg_P, n * 8);
  d.add((void**)&P->cta_cnt, (size_t)P->nsm * 4 + 64);
  d.add((void**)&P->part_scal, (size_t)P->nsm * 4 * 8 + 64);
  d.add((void**)&P->part_vec, (size_t)P->nsm * m * 8);
  for (int i = 0; i < 2; ++i) {
    d.add((void**)&P->J[i], n * 4);
    d.add((void**)&P->PJ[i], n * 8);
    d.add((void**)&P->y[i], m * 8);
    d.add((void**)&P->g[i], m * 8);
  }
  d.add((void**)&P->r_dev, 8 * 8);
  d.add((void**)&P->Jx, n * 4);
  d.add((void**)&P->Px, n * 8);
  d.add((void**)&P->d, m * 8);
  d.add((void**)&P->u, m * 8);
  d.add((void**)&P->tmpm, m * 8);
  d.add((void**)&P->Mmat, (size_t)(m + 1) * (m + 1) * 8);
  d.add((void**)&P->Winv, (size_t)((m + 31) / 32) * 33 * 32 * 8);  // block inverses
  P->W_splits = 16;
  d.add((void**)&P->W, (size_t)P->W_splits * m * m * 8);
  d.add((void**)&P->info, 64);
  d.add((void**)&P->ev_dev, sizeof(EvalOut) * 4);
  d.add((void**)&P->scratch, 64 * 8);
  d.add((void**)&P->flags, 64);
  d.add((void**)&P->blk, (size_t)((m + 31) / 32) * 3 * 8 + 64);
  d.add((void**)&P->ticket, 64);
  d.add((void**)&P->chol_args, 2 * sizeof(CholArgs));
  d.add((void**)&P->gax_valid, 4 * 256);
  d.add((void**)&P->cg_res, m * 8);
  d.add((void**)&P->cg_parts, (size_t)P->nsm * m * 8);
  d.add((void**)&P->cg_scal, (size_t)P->nsm * 2 * 8 + 64);
  d.add((void**)&P->ctl, sizeof(DevCtl));
  d.add((void**)&P->kflag, 256 * sizeof(int));
  const int gsk_tiles = gram_tiles(m + 1);
  d.add((void**)&P->gsk_part, (size_t)std::max(P->gsk_grid, gsk_tiles) * GT * GT * 8);
  d.add((void**)&P->gsk_cnt, (size_t)(2 * gsk_tiles + 64) * 4);
  P->arena = pool_alloc(d.total);
  if (!P->arena) {
    set_err("device allocation of %zu bytes failed", d.total);
    return SSNAL_ECUDA;
  }
  d.assign((char*)P->arena);
  CK(cudaMemset(P->ticket, 0, 64));
  CK(cudaMemset(P->gate_cnt, 0, 64));
  {  // K4 outputs per exact branch for the graph's branch-agnostic launch (k_chol_* with want < 0):
     // [0] SMW v → u; [1] m × m d = −M⁻¹g, gᵀd = scratch[0], y[1] = y[0] + d.  Uploaded here, before the
     // caller's A is enqueued: a synchronous copy in build_graph would wait for that upload and serialise
     // the graph capture behind it.
    const CholArgs ca[2] = {{P->u, 1.0, nullptr, nullptr, nullptr, nullptr},
                            {P->d, -1.0, P->g[0], P->scratch, P->y[0], P->y[1]}};
    CK(cudaMemcpy(P->chol_args, ca, sizeof(ca), cudaMemcpyHostToDevice));
  }
  CK(cudaMemset(P->gsk_cnt, 0, (size_t)(2 * gsk_tiles + 64) * 4));
  Arena h;
  h.add((void**)&P->ev_host, sizeof(EvalOut) * 4);
  h.add((void**)&P->scratch_host, 64 * 8);
  h.add((void**)&P->ctl_host, sizeof(DevCtl));
  h.add((void**)&P->ev_out_host, sizeof(EvalOut));
  h.add((void**)&P->gate_flag_host, 64);
  CK(cudaHostAlloc(&P->arena_h, h.total, cudaHostAllocMapped));
  memset(P->arena_h, 0, h.total);
  h.assign((char*)P->arena_h);
  CK(cudaHostGetDevicePointer((void**)&P->ev_host_dev, P->ev_host, 0));
  CK(cudaHostGetDevicePointer((void**)&P->gate_flag_dev, P->gate_flag_host, 0));
  return SSNAL_OK;
}

// ---------------- launch wrappers ----------------

// Calls f(acc) with the handle's column accessor (fp64 design or packed genotype codes).
template <class F>
int with_acc(ssnal_en_problem* P, F&& f) {
  if (P->fmt) return f(AccG{P->codes, P->cstride, P->tab});
  return f(AccA{P->A, P->m});
}

cudaEvent_t take_event(ssnal_en_problem* P) {
  if (!P->ev_pool.empty()) {
    cudaEvent_t e = P->ev_pool.back();
    P->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void harvest_k1(ssnal_en_problem* P) {  // call after a stream sync
  for (auto& pr : P->k1_pending) {
    cudaEventSynchronize(pr.second);
    float ms = 0;
    cudaEventElapsedTime(&ms, pr.first, pr.second);
    P->k1_time += ms * 1e-3;
    P->k1_count++;
    P->ev_pool.push_back(pr.first);
    P->ev_pool.push_back(pr.second);
  }
  P->k1_pending.clear();
}

// K1 at y (device, m).  fused=0: plain w = Aᵀy into w_out (+ per-CTA max|w|).
int launch_k1(ssnal_en_problem* P, const double* y, const double* x, const Scal& sc, int fused, double* w_out,
              const Scal* scp = nullptr, unsigned long long* tstamp = nullptr, int reuse = 0, int notime = 0,
              const int* pred = nullptr, int force_stream = 0) {
  // reuse: 0 plain instantiation; 1 / 2 the REUSE instantiation with that K1Params::rmode; −1 the REUSE
  // instantiation with the mode, the ψ-only flag and (pred) the redo predicate in the control block (graph)
  K1Params k;
  k.A = P->A;
  k.m = P->m;
  k.n = P->n;
  k.y = y;
  k.x = x;
  k.w_out = w_out;
  k.seg_idx = P->seg_idx;
  k.seg_P = P->seg_P;
  k.mask = P->mask;
  k.cta_cnt = P->cta_cnt;
  k.part_scal = P->part_scal;
  k.part_vec = fused ? P->part_vec : nullptr;
  k.sc = sc;
  k.scp = scp;
  k.tstamp = tstamp;
  k.C = P->C;
  k.T = P->T;
  k.stages = P->S;
  k.fused = fused;
  k.stage_elems = P->stage_elems;
  k.xstage_elems = P->xstage_elems;
  k.codes = P->codes;
  k.tab = P->tab;
  k.cstride = P->cstride;
  k.bfr_off = P->k1_bfr_off;
  const bool use_r = reuse && fused && P->atb;  // R40: the launch may be served from the kept Aᵀb
  k.atb = use_r ? P->atb : nullptr;
  k.bvec = P->b;
  k.rmode = reuse > 0 ? reuse : 0;
  k.rmodep = (use_r && reuse < 0) ? &P->ctl->reuse_mode : nullptr;
  k.pred = use_r ? pred : nullptr;
  k.force_stream = force_stream;
  k.gmiss = !use_r ? nullptr : (reuse < 0 ? &P->ctl->gmiss : P->gate_flag_dev + 1);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  const bool ev_time = P->time_k1 && !P->capturing && !notime;  // notime: may be served from Aᵀb (not a pass over A)
  if (ev_time) {
    e0 = take_event(P);
    e1 = take_event(P);
    cudaEventRecord(e0, P->st);
  }
  (P->fmt ? k1g_for(P->TW, use_r) : k1_for(P->MR, use_r))<<<P->G, K1_THREADS, P->k1_smem, P->st>>>(k);
  P->launches++;
  if (ev_time) {
    cudaEventRecord(e1, P->st);
    P->k1_pending.push_back({e0, e1});
  }
  CKL();
  return SSNAL_OK;
}

int launch_k1e(ssnal_en_problem* P, const double* w0, const double* w1, double s, const double* x, const Scal& sc,
               double* w_out, const Scal* scp = nullptr, const double* sp = nullptr) {
  K1eParams k;
  k.n = P->n;
  k.w0 = w0;
  k.w1 = w1;
  k.s = s;
  k.x = x;
  k.w_out = w_out;
  k.seg_idx = P->seg_idx;
  k.seg_P = P->seg_P;
  k.cta_cnt = P->cta_cnt;
  k.part_scal = P->part_scal;
  k.sc = sc;
  k.scp = scp;
  k.sp = sp;
  k.C = P->C;
  k.T = P->T;
  k1e_epilogue<<<P->G, K1E_THREADS, 0, P->st>>>(k);
  P->launches++;
  CKL();
  return SSNAL_OK;
}

int launch_finalize(ssnal_en_problem* P, int32_t* J, double* PJ, int64_t* r_dev, const int* pred = nullptr) {
  k1_finalize<<<P->G, 256, 0, P->st>>>(P->seg_idx, P->seg_P, P->cta_cnt, P->G, P->T, P->C, P->n, J, PJ, r_dev, pred);
  P->launches++;
  CKL();
  return SSNAL_OK;
}

// parts (P->part_vec, `grid` rows) = Σ coef_a A[:, J_a] over r (host-known) columns
int launch_gather(ssnal_en_problem* P, const int32_t* J, const double* coef, int64_t r, int* grid_out) {
  int grid = (int)((r + 63) / 64);
  if (grid > P->gax_grid) grid = P->gax_grid;
  if (grid < 1) grid = 1;
  with_acc(P, [&](auto acc) {
    gax_for<decltype(acc)>(P->MR)<<<grid, 256, (size_t)8 * P->m * 8, P->st>>>(acc, P->m, J, coef, r, nullptr,
                                                                               P->part_vec, nullptr, nullptr);
    return 0;
  });
  P->launches++;
  *grid_out = grid;
  CKL();
  return SSNAL_OK;
}

// The hot gathers: row-block clusters (k_gather_rows), grid ⌈m/32⌉ × 8 whatever r is.
unsigned gather_rows_grid(const ssnal_en_problem* P) { return (unsigned)((P->m + 31) / 32) * kGatherCS; }

// part_vec row 0 = A_J coef with r on the device (∇ψ, Eq. (15)); consumed by launch_eval with
// nparts = 1 and no validity flags.
int launch_gather_vec(ssnal_en_problem* P, const int32_t* J, const double* coef, const int64_t* r_dev,
                      const int* pred = nullptr) {
  with_acc(P, [&](auto acc) {
    k_gather_rows<<<gather_rows_grid(P), 256, 0, P->st>>>(acc, P->m, J, coef, -1, r_dev, pred, nullptr, kGatherVec,
                                                           P->part_vec, nullptr, nullptr, nullptr, nullptr, nullptr,
                                                           nullptr);
    return 0;
  });
  P->launches++;
  CKL();
  return SSNAL_OK;
}

// Same with r resident on the device (no host round trip): fixed grid, validity flags in gax_valid.
constexpr int kGatherDevGrid = 128;
int launch_gather_dev(ssnal_en_problem* P, const int32_t* J, const double* coef, const int64_t* r_dev,
                      const int* pred = nullptr) {
  with_acc(P, [&](auto acc) {
    gax_for<decltype(acc)>(P->MR)<<<kGatherDevGrid, 256, (size_t)8 * P->m * 8, P->st>>>(
        acc, P->m, J, coef, -1, r_dev, P->part_vec, P->gax_valid, pred);
    return 0;
  });
  P->launches++;
  CKL();
  return SSNAL_OK;
}

int launch_eval(ssnal_en_problem* P, const double* y, const Scal& sc, int with_grad, const int* valid, int nparts,
                double* g_out, const int64_t* r_dev, int slot, const double* gd_src = nullptr,
                const int* info_src = nullptr, const Scal* scp = nullptr, const int* pred = nullptr,
                const double* vec = nullptr, const double* scal = nullptr, int nscal = 0, int hook = 0,
                const CtlHook* hk = nullptr) {
  const unsigned nblk = (unsigned)((P->m + 31) / 32);
  if (!P->capturing) ++P->ev_seq;
  if (!vec) vec = P->part_vec;
  if (!scal) {
    scal = P->part_scal;
    nscal = P->G;
  }
  EvalOut* hout = P->capturing ? nullptr : P->ev_host_dev + slot;  // graph mode: decisions on the device
  const double* nbp = P->capturing ? &P->ctl->nb : nullptr;
  const dim3 grid(nblk * kEvalCS);
#define SSN_EVAL_ARGS                                                                                              \
  P->m, y, P->b, vec, valid, nparts, scal, nscal, sc, P->nb, with_grad, g_out, r_dev, P->ev_dev + slot, P->blk,   \
      P->ticket, gd_src, info_src, hout, P->ev_seq, scp, pred, nbp
  if (nblk <= (unsigned)kEval16 && P->eval16_ok) {  // m ≤ 512: one 16-CTA cluster
    const dim3 g16(kEval16);
    switch (hook) {
      case kHookInnerBegin: k_eval_ctl16<kHookInnerBegin><<<g16, K5_THREADS, 0, P->st>>>(SSN_EVAL_ARGS, *hk); break;
      case kHookArmijo: k_eval_ctl16<kHookArmijo><<<g16, K5_THREADS, 0, P->st>>>(SSN_EVAL_ARGS, *hk); break;
      case kHookArmijoRedo: k_eval_ctl16<kHookArmijoRedo><<<g16, K5_THREADS, 0, P->st>>>(SSN_EVAL_ARGS, *hk); break;
      case kHookBacktrack: k_eval_ctl16<kHookBacktrack><<<g16, K5_THREADS, 0, P->st>>>(SSN_EVAL_ARGS, *hk); break;
      case kHookInnerEnd: k_eval_ctl16<kHookInnerEnd><<<g16, K5_THREADS, 0, P->st>>>(SSN_EVAL_ARGS, *hk); break;
      default: k_eval_reduce16<<<g16, K5_THREADS, 0, P->st>>>(SSN_EVAL_ARGS);
    }
    P->launches++;
    CKL();
    return SSNAL_OK;
  }
  switch (hook) {  // graph mode: the control decision that consumes this evaluation, in the same launch
    case kHookInnerBegin: k_eval_ctl<kHookInnerBegin><<<grid, K5_THREADS, 0, P->st>>>(SSN_EVAL_ARGS, *hk); break;
    case kHookArmijo: k_eval_ctl<kHookArmijo><<<grid, K5_THREADS, 0, P->st>>>(SSN_EVAL_ARGS, *hk); break;
    case kHookArmijoRedo: k_eval_ctl<kHookArmijoRedo><<<grid, K5_THREADS, 0, P->st>>>(SSN_EVAL_ARGS, *hk); break;
    case kHookBacktrack: k_eval_ctl<kHookBacktrack><<<grid, K5_THREADS, 0, P->st>>>(SSN_EVAL_ARGS, *hk); break;
    case kHookInnerEnd: k_eval_ctl<kHookInnerEnd><<<grid, K5_THREADS, 0, P->st>>>(SSN_EVAL_ARGS, *hk); break;
    default: k_eval_reduce<<<grid, K5_THREADS, 0, P->st>>>(SSN_EVAL_ARGS);
  }
#undef SSN_EVAL_ARGS
  P->launches++;
  CKL();
  return SSNAL_OK;
}

// ---- §8(f3) column sharding: exchanges through the caller's all-reduce ----
bool sharded(const ssnal_en_problem* P) { return P->comm_size > 0; }

unsigned reduce_grid(ssnal_en_problem* P, int64_t tot);
// Peer-memory all-reduce (k_peer.cuh): one CTA through the double-buffered small slots, or a
// multi-CTA deposit into the big slots followed by a waiting rank-ordered reduction.
int peer_allreduce(ssnal_en_problem* P, double* buf, int64_t count, int op) {
  if (count <= P->pc.ss) {
    k_peer_allreduce<<<1, 1024, 0, P->st>>>(P->pc, buf, count, op);
    P->launches++;
  } else {
    if (count > P->pc.sb) {
      set_err("peer all-reduce of %lld doubles exceeds the exchange slot (%lld)", (long long)count,
              (long long)P->pc.sb);
      return SSNAL_EINVAL;
    }
    const unsigned grid = reduce_grid(P, count);
    k_peer_put_big<<<grid, 256, 0, P->st>>>(P->pc, buf, count);
    k_peer_reduce_big<<<grid, 256, 0, P->st>>>(P->pc, buf, count, op);
    P->launches += 2;
  }
  CKL();
  return SSNAL_OK;
}

// After a stream synchronisation: a peer exchange that timed out or saw inconsistent counts leaves
// an error code in device memory (k_peer.cuh) — the call fails instead of returning bad results.
int peer_check(ssnal_en_problem* P) {
  int v[2] = {0, 0};  // ticket, err
  CK(cudaMemcpy(v, P->peer_epoch + 1, 8, cudaMemcpyDeviceToHost));
  if (v[1] == 1) {
    set_err("peer exchange timed out (a rank stopped participating)");
    return SSNAL_ECUDA;
  }
  if (v[1] != 0) {
    set_err("peer exchange: gathered active counts disagree with the global r (code %d)", v[1]);
    return SSNAL_ECUDA;
  }
  return SSNAL_OK;
}

int comm_allreduce(ssnal_en_problem* P, double* buf, int64_t count, int op) {
  CKL();
  if (P->peer) return peer_allreduce(P, buf, count, op);
  const int rc = P->comm_fn(P->comm_ctx, buf, count, op, (void*)P->st);
  if (rc) {
    set_err("all-reduce callback failed (%d)", rc);
    return SSNAL_ECUDA;
  }
  return SSNAL_OK;
}

// xbuf = [Σ local partial vectors (m) | Σ local scalar partials (4) | local r] summed over the ranks;
// rg_dev = the global r.  vec/nparts/valid: the partial m-vectors (nparts = 0: none).
int exchange_eval(ssnal_en_problem* P, const double* vec, const int* valid, int nparts, const double* scal, int nscal,
                  const int64_t* r_local) {
  if (P->peer) {  // record + deposit + wait + rank-ordered sum in one kernel
    k_peer_eval<<<kRecCS, 256, 0, P->st>>>(P->pc, P->m, vec, valid, nparts, scal, nscal, r_local, P->xbuf,
                                           P->rg_dev, nullptr);
    P->launches++;
    CKL();
    return SSNAL_OK;
  }
  k_prereduce16<<<kRecCS, 256, 0, P->st>>>(P->m, vec, valid, nparts, scal, nscal, r_local, P->xbuf);
  P->launches++;
  int rc = comm_allreduce(P, P->xbuf, P->m + 5, 0);
  if (rc) return rc;
  k_to_i64<<<1, 1, 0, P->st>>>(P->xbuf + P->m + 4, P->rg_dev);
  P->launches++;
  CKL();
  return SSNAL_OK;
}

// launch_eval on the global sums when sharded (partial vectors: part_vec rows, `valid` flags)
int eval_g(ssnal_en_problem* P, const double* y, const Scal& sc, int with_grad, const int* valid, int nparts,
           double* g_out, const int64_t* r_dev, int slot, const double* gd_src = nullptr,
           const int* info_src = nullptr) {
  if (!sharded(P)) return launch_eval(P, y, sc, with_grad, valid, nparts, g_out, r_dev, slot, gd_src, info_src);
  int rc = exchange_eval(P, nparts ? P->part_vec : nullptr, valid, nparts, P->part_scal, P->G, r_dev);
  if (rc) return rc;
  return launch_eval(P, y, sc, with_grad, nullptr, nparts ? 1 : 0, g_out, P->rg_dev, slot, gd_src, info_src, nullptr,
                     nullptr, P->xbuf, P->xbuf + P->m, 1);
}

// Wait for the EvalOut of the most recent launch_eval on `slot`: spin on the mapped host copy's
// sequence number (no stream synchronisation); poll the stream for errors now and then.
int fetch_eval(ssnal_en_problem* P, int slot, EvalOut* out) {
  volatile EvalOut* h = P->ev_host + slot;
  const unsigned long long want = P->ev_seq;
  for (uint64_t spin = 0; h->seq != want; ++spin) {
    if ((spin & 0xFFFF) == 0xFFFF) {
      cudaError_t e = cudaStreamQuery(P->st);
      if (e != cudaSuccess && e != cudaErrorNotReady) {
        set_err("stream error while waiting for an evaluation: %s", cudaGetErrorString(e));
        return SSNAL_ECUDA;
      }
      if (e == cudaSuccess && h->seq != want) {
        __sync_synchronize();
        if (h->seq != want) {
          set_err("evaluation record not delivered (seq %llu, want %llu)", (unsigned long long)h->seq, want);
          return SSNAL_ECUDA;
        }
      }
    }
  }
  __sync_synchronize();
  out->psi = h->psi; out->psimag = h->psimag; out->res1 = h->res1; out->yy = h->yy; out->by = h->by; out->gg = h->gg;
  for (int j = 0; j < 4; ++j) out->s[j] = h->s[j];
  out->gd = h->gd; out->r = h->r; out->info = h->info; out->seq = h->seq; out->pad = 0;
  return SSNAL_OK;
}

// Cluster Cholesky of the N × N lower part of M with NR − N appended rows (ld ≥ NR); with `out`
// the first appended row is the right-hand side and the solve (L Lᵀ)⁻¹ rhs is written to out.
int launch_chol_ex(ssnal_en_problem* P, double* M, int N, int NR, int ld, double* out, double scale,
                   const double* dotv, double* dot_out, const double* ybase, double* yt, int* info) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P->cluster);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = P->chol_smem;
  cfg.stream = P->st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P->cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const DirGeo* nog = nullptr;
  CK(cudaLaunchKernelEx(&cfg, k_chol_cluster, M, N, NR, ld, out, scale, dotv, dot_out, P->Winv, info, ybase, yt, nog,
                        0, P->kflag, 0, (const CholArgs*)nullptr));
  P->launches++;
  return SSNAL_OK;
}

// DSMEM-resident K4 (k_chol_dsm.cuh): same contract as the k_chol_cluster launch below.  Used for
// N ≤ kDsmUseMax, where it is faster than k_chol_d2 (and than k_chol_cluster: N = 100 35 vs 47 µs; N = 500
// takes ~300 vs ~211 µs: its per-owner update load is uneven).
int launch_chol_dsm(ssnal_en_problem* P, double* M, int N, double* out, double scale, const double* dotv,
                    double* dot_out, const double* ybase, double* yt, const DirGeo* geo, int want) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kDsmCS);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = kDsmSmem;
  cfg.stream = P->st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kDsmCS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const CholArgs* ca = want < 0 ? P->chol_args : nullptr;
  CK(cudaLaunchKernelEx(&cfg, k_chol_dsm, (const double*)M, N, N + 1, out, scale, dotv, dot_out, P->info, ybase, yt,
                        geo, want, kDsmUseMax, ca));
  P->launches++;
  return SSNAL_OK;
}

// Split-ownership DSMEM K4 (k_chol_d2.cuh) for kDsmUseMax < N ≤ kDsmMaxN: same contract.
int launch_chol_d2(ssnal_en_problem* P, double* M, int N, double* out, double scale, const double* dotv,
                   double* dot_out, const double* ybase, double* yt, const DirGeo* geo, int want) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kDsmCS);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = kD2Smem;
  cfg.stream = P->st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kDsmCS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const CholArgs* ca = want < 0 ? P->chol_args : nullptr;
  CK(cudaLaunchKernelEx(&cfg, k_chol_d2, (const double*)M, N, N + 1, out, scale, dotv, dot_out, P->info, ybase, yt,
                        geo, want, kDsmUseMax + 1, kDsmMaxN, ca));
  P->launches++;
  return SSNAL_OK;
}

// Cluster Cholesky + both triangular solves: M holds the matrix (ld = N+1) and the rhs in row N.
// Host mode: k_chol_dsm for N ≤ 96, k_chol_d2 for 96 < N ≤ 512, else k_chol_cluster.  Graph
// mode (geo): each kernel that can occur for this m, predicated on its N range.
int launch_chol(ssnal_en_problem* P, double* M, int N, double* out, double scale, const double* dotv,
                double* dot_out, const double* ybase = nullptr, double* yt = nullptr, const DirGeo* geo = nullptr,
                int want = 0) {
  int nmin = 0;
  if (geo && P->chol_dsm && P->use_d2 && P->d2_ok && P->m > kDsmUseMax) {  // one node for both DSMEM kernels
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(kDsmCS);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = kD2Smem;
    cfg.stream = P->st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kDsmCS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const CholArgs* ca = want < 0 ? P->chol_args : nullptr;
    CK(cudaLaunchKernelEx(&cfg, k_chol_dsm_any, (const double*)M, out, scale, dotv, dot_out, P->info, ybase, yt, geo,
                          want, ca));
    P->launches++;
    if (P->m <= kDsmMaxN) return SSNAL_OK;
    nmin = kDsmMaxN + 1;
  } else if (P->chol_dsm) {
    if (geo || N <= kDsmUseMax) {
      int rc = launch_chol_dsm(P, M, N, out, scale, dotv, dot_out, ybase, yt, geo, want);
      if (rc) return rc;
    }
    if (geo ? P->m <= kDsmUseMax : N <= kDsmUseMax) return SSNAL_OK;
    nmin = kDsmUseMax + 1;
    if (P->use_d2 && P->d2_ok) {
      if (geo || N <= kDsmMaxN) {
        int rc = launch_chol_d2(P, M, N, out, scale, dotv, dot_out, ybase, yt, geo, want);
        if (rc) return rc;
      }
      if (geo ? P->m <= kDsmMaxN : N <= kDsmMaxN) return SSNAL_OK;
      nmin = kDsmMaxN + 1;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P->cluster);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = P->chol_smem;
  cfg.stream = P->st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P->cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const CholArgs* ca = want < 0 ? P->chol_args : nullptr;
  CK(cudaLaunchKernelEx(&cfg, k_chol_cluster, M, N, N + 1, N + 1, out, scale, dotv, dot_out, P->Winv, P->info,
                        ybase, yt, geo, want, P->kflag, nmin, ca));
  P->launches++;
  return SSNAL_OK;
}

// K6: CG Newton direction, one cooperative launch (nsm CTAs, grid barriers); host values or geo.
int launch_cg(ssnal_en_problem* P, const int32_t* J, int64_t r, const double* g, double kappa, double* d,
              double* gd_dev, const double* y, double* yt, const DirGeo* geo) {
  CgParams c;
  c.m = P->m;
  c.J = J;
  c.r = r;
  c.g = g;
  c.kappa = kappa;
  c.tol = P->cg_tol;
  c.maxit = P->cg_maxit;
  c.y = y;
  c.d = d;
  c.yt = yt;
  c.gd_out = gd_dev;
  c.res = P->cg_res;
  c.parts = P->cg_parts;
  c.scal = P->cg_scal;
  c.iters_out = &P->ctl->cg_iters;
  c.geo = geo;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P->nsm);
  cfg.blockDim = dim3(K6_THREADS);
  cfg.dynamicSmemBytes = P->cg_smem_bytes;
  cfg.stream = P->st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaError_t e = (cudaError_t)with_acc(P, [&](auto acc) {
    return (int)cudaLaunchKernelEx(&cfg, cg_for<decltype(acc)>(P->MR), c, acc);
  });
  CK(e);
  P->launches++;
  return SSNAL_OK;
}

// Gram / reduce grids: persistent CTAs (results do not depend on the grid; DirGeo fixes the work)
int gram_grid(ssnal_en_problem* P, int items) { return items < 2 * P->nsm ? (items < 1 ? 1 : items) : 2 * P->nsm; }
// k_gram_fused: one 8-CTA cluster per tile, at most ~2 CTAs per SM (clusters stride over tiles)
unsigned gram_fused_grid(ssnal_en_problem* P, int tiles) {
  int ncl = (2 * P->nsm) / kGramCS;
  if (tiles < ncl) ncl = tiles;
  if (ncl < 1) ncl = 1;
  return (unsigned)(ncl * kGramCS);
}

// §8(f3): a sharded rank's raw local partial Gram A_J A_Jᵀ (m × m, ld = m, lower) into out by k_gram_sk;
// graph mode: predicated on the global branch 2, the local r from r_loc.
template <class Acc>
int launch_gram_raw(ssnal_en_problem* P, const Acc& acc, const int32_t* J, int64_t r_host, const int64_t* r_loc,
                    double* out, const DirGeo* geo) {
  const int64_t m = P->m;
  const GramFusedArgs gfa{2, r_host, m, m, gram_tiles(m), (int)m, 0.0, 1.0, 0.0};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P->gsk_grid);
  cfg.blockDim = dim3(256);
  cfg.stream = P->st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_gram_sk<Acc>, acc, m, J, out, (const double*)nullptr, gfa, geo, 2, P->gsk_part,
                        P->gsk_cnt, P->gsk_minch, r_loc, 1));
  P->launches++;
  CKL();
  return SSNAL_OK;
}

// K3 of the Newton systems (Eq. (18)/(19)): k_gram_sk (one cooperative round over the whole GPU) or,
// with option gram_sk = 0, k_gram_fused (8-CTA clusters per tile).  geo: graph mode (worst-case
// grid); only > 0: one branch alone.
template <class Acc>
int launch_gram_one(ssnal_en_problem* P, const Acc& acc, const int32_t* J, const double* g, const GramFusedArgs& gfa,
                    const DirGeo* geo, int only, bool sk) {
  if (only < 0) return SSNAL_OK;
  if (!sk) {
    k_gram_fused<<<gram_fused_grid(P, geo ? gram_tiles(P->m) : gfa.tiles), 256, 0, P->st>>>(acc, P->m, J, P->Mmat, g,
                                                                                           gfa, geo, only);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P->gsk_grid);
    cfg.blockDim = dim3(256);
    cfg.stream = P->st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_gram_sk<Acc>, acc, P->m, J, P->Mmat, g, gfa, geo, only, P->gsk_part, P->gsk_cnt,
                          P->gsk_minch, (const int64_t*)nullptr, 0));
  }
  P->launches++;
  CKL();
  return SSNAL_OK;
}

template <class Acc>
int launch_gram(ssnal_en_problem* P, const Acc& acc, const int32_t* J, const double* g, const GramFusedArgs& gfa,
                const DirGeo* geo, int only = 0) {
  // option gram_sk: 0 = k_gram_fused for both branches; 1 (default) = k_gram_fused for the SMW branch
  // (few tiles, K = m: its DSMEM reduction beats the L2 round trip of the partials and the launch of a
  // full-GPU grid) and k_gram_sk for m × m (36 tiles at m = 500, K = r large); 2 = k_gram_sk for both.
  // Graph mode with option 1: one node of each, predicated on its branch.
  if (P->use_gram_sk == 1) {
    if (geo) {
      int rc = launch_gram_one(P, acc, J, g, gfa, geo, only == 2 ? -1 : 1, 0);
      if (rc) return rc;
      return only == 1 ? SSNAL_OK : launch_gram_one(P, acc, J, g, gfa, geo, 2, 1);
    }
    return launch_gram_one(P, acc, J, g, gfa, nullptr, only, gfa.branch == 2);
  }
  return launch_gram_one(P, acc, J, g, gfa, geo, only, P->use_gram_sk == 2);
}
unsigned reduce_grid(ssnal_en_problem* P, int64_t tot) {
  int64_t g = (tot + 255) / 256;
  if (g > 4 * P->nsm) g = 4 * P->nsm;
  return (unsigned)(g < 1 ? 1 : g);
}

// Newton direction for (J, r) at gradient g: d ← solution, *gd_dev ← gᵀd (Eq. (18)/(19)); if yt,
// also the Armijo trial y_t = y + d (fused into the last kernel of each branch).
// §8(f3): the Newton direction of a sharded handle from the global r.  0 < r < m: the ranks' active
// columns are all-gathered (each placed at its prefix offset of an r × m buffer, summed) and the
// SMW form Eq. (19) runs on them; r ≥ m: the partial Grams A_J A_Jᵀ are summed (Eq. (18)).
int newton_direction_sharded(ssnal_en_problem* P, const int32_t* J, int64_t rg, const int64_t* r_loc_dev,
                             const double* g, double kappa, double* d, double* gd_dev, int* branch, const double* y,
                             double* yt, double jit) {
  const int64_t m = P->m;
  int rc;
  if (rg == 0) {
    *branch = 0;
    k_neg_copy<<<1, 1024, 0, P->st>>>(m, g, d, g, gd_dev, y, yt, nullptr);
    P->launches++;
    CKL();
    return SSNAL_OK;
  }
  CK(cudaMemcpyAsync(P->comm_host, r_loc_dev, 8, cudaMemcpyDeviceToHost, P->st));
  CK(cudaStreamSynchronize(P->st));
  int64_t rl;
  memcpy(&rl, P->comm_host, 8);
  CK(cudaMemsetAsync(P->info, 0, sizeof(int), P->st));
  if (rg < m) {
    *branch = 1;
    const int R = P->comm_size;
    CK(cudaMemsetAsync(P->xbuf, 0, (size_t)R * 8, P->st));
    P->comm_host[0] = (double)rl;
    CK(cudaMemcpyAsync(P->xbuf + P->comm_rank, P->comm_host, 8, cudaMemcpyHostToDevice, P->st));
    if ((rc = comm_allreduce(P, P->xbuf, R, 0))) return rc;
    CK(cudaMemcpyAsync(P->comm_host + 8, P->xbuf, (size_t)R * 8, cudaMemcpyDeviceToHost, P->st));
    CK(cudaStreamSynchronize(P->st));
    int64_t off = 0, tot = 0;
    for (int q = 0; q < R; ++q) {
      const int64_t c = (int64_t)P->comm_host[8 + q];
      if (q < P->comm_rank) off += c;
      tot += c;
    }
    if (tot != rg) {
      set_err("sharded active counts disagree (%lld vs %lld)", (long long)tot, (long long)rg);
      return SSNAL_ECUDA;
    }
    double* GA = P->xbuf;  // gathered A_J, column-major m × rg
    CK(cudaMemsetAsync(GA, 0, (size_t)rg * m * 8, P->st));
    if (rl > 0) {
      with_acc(P, [&](auto acc) {
        k_pack_cols<<<(unsigned)(rl < 2 * P->nsm ? rl : 2 * P->nsm), 256, 0, P->st>>>(acc, m, J, rl, GA + off * m);
        return 0;
      });
      P->launches++;
    }
    if ((rc = comm_allreduce(P, GA, rg * m, 0))) return rc;
    DirGeo geo = make_geo(rg, m, P->nsm, P->W_splits, kappa, 1.0 / kappa, 0.0, INFINITY);
    geo.jit = jit;
    const AccA ga{GA, m};
    const GramFusedArgs gfa{1, rg, geo.nout, geo.nmat, geo.tiles, geo.ld, geo.diag, geo.mult, geo.jit};
    if ((rc = launch_gram(P, ga, P->iota, g, gfa, nullptr))) return rc;
    CKL();
    if ((rc = launch_chol(P, P->Mmat, geo.N, P->u, 1.0, nullptr, nullptr))) return rc;
    k_gather_rows<<<gather_rows_grid(P), 256, 0, P->st>>>(ga, m, P->iota, P->u, rg, nullptr, nullptr, nullptr,
                                                           kGatherSmw, d, g, y ? y : g, yt ? yt : P->tmpm, gd_dev, P->blk,
                                                           P->ticket);
    P->launches++;
    CKL();
    return SSNAL_OK;
  }
  *branch = 2;
  CK(cudaMemsetAsync(P->xbuf, 0, (size_t)m * m * 8, P->st));
  // the raw local partial Gram (k_gram_sk: one cooperative round) straight into the exchange buffer
  if ((rc = with_acc(P, [&](auto acc) { return launch_gram_raw(P, acc, J, rl, nullptr, P->xbuf, nullptr); })))
    return rc;
  if ((rc = comm_allreduce(P, P->xbuf, m * m, 0))) return rc;
  k_gram_reduce<<<reduce_grid(P, m * m), 256, 0, P->st>>>(P->xbuf, 1, m, m, 1.0, kappa, P->Mmat, m + 1, g, nullptr, 0,
                                                          jit);
  P->launches++;
  CKL();
  return launch_chol(P, P->Mmat, (int)m, d, -1.0, g, gd_dev, y, yt);
}

int newton_direction(ssnal_en_problem* P, const int32_t* J, int64_t r, const double* g, double kappa, double* d,
                     double* gd_dev, int* branch, const double* y = nullptr, double* yt = nullptr,
                     double jit = 0.0, const int64_t* r_loc_dev = nullptr) {
  if (sharded(P)) return newton_direction_sharded(P, J, r, r_loc_dev, g, kappa, d, gd_dev, branch, y, yt, jit);
  const int64_t m = P->m;
  DirGeo geo = make_geo(r, m, P->nsm, P->W_splits, kappa, 1.0 / kappa, P->cg_ratio, P->cg_threshold);
  geo.jit = jit;
  *branch = geo.branch;
  if (geo.branch == 3)  // K6: conjugate gradient (R32)
    return launch_cg(P, J, r, g, kappa, d, gd_dev, y, yt, nullptr);
  if (geo.branch == 0) {  // d = −g, gᵀd, y + d: the SMW back-substitution kernel with no columns
    with_acc(P, [&](auto acc) {
      k_gather_rows<<<gather_rows_grid(P), 256, 0, P->st>>>(acc, m, J, g, 0, nullptr, nullptr, nullptr, kGatherSmw, d,
                                                             g, y ? y : g, yt ? yt : P->tmpm, gd_dev, P->blk,
                                                             P->ticket);
      return 0;
    });
    P->launches++;
    CKL();
    return SSNAL_OK;
  }
  CK(cudaMemsetAsync(P->info, 0, sizeof(int), P->st));
  const GramFusedArgs gfa{geo.branch, r, geo.nout, geo.nmat, geo.tiles, geo.ld, geo.diag, geo.mult, geo.jit};
  if (geo.branch == 1) {  // Sherman–Morrison–Woodbury, Eq. (19): factor κ⁻¹I_r + A_JᵀA_J (R13)
    int rc = with_acc(P, [&](auto acc) { return launch_gram(P, acc, J, g, gfa, nullptr); });
    if (rc) return rc;
    rc = launch_chol(P, P->Mmat, geo.N, P->u, 1.0, nullptr, nullptr);  // v = (κ⁻¹I + G)⁻¹ u
    if (rc) return rc;
    // d = −g + A_J v, gᵀd, y_t = y + d (last-CTA finalisation)
    with_acc(P, [&](auto acc) {
      k_gather_rows<<<gather_rows_grid(P), 256, 0, P->st>>>(acc, m, J, P->u, r, nullptr, nullptr, nullptr, kGatherSmw,
                                                             d, g, y ? y : g, yt ? yt : P->tmpm, gd_dev, P->blk,
                                                             P->ticket);
      return 0;
    });
    P->launches++;
    CKL();
    return SSNAL_OK;
  }
  // r ≥ m: Eq. (18), M = I_m + κ A_J A_Jᵀ; the fused reduce also writes g into the rhs row
  if (int rc = with_acc(P, [&](auto acc) { return launch_gram(P, acc, J, g, gfa, nullptr); })) return rc;
  return launch_chol(P, P->Mmat, (int)m, d, -1.0, g, gd_dev, y, yt);  // d = −M⁻¹ g, gd = gᵀd
}

// Graph mode: every branch's kernels, predicated on the device geometry C->geo (computed by the
// control kernels from r); worst-case grids, surplus CTAs exit.  Same work decomposition as
// newton_direction for the same r.  Reads J[0], g[0], y[0]; writes d, y[1], gᵀd → scratch[0].
// Graph mode on a peer-attached sharded handle (§8(f3)): the same branch kernels as the
// host-driven sharded direction, with the exchanges fused into them over peer memory (k_peer.cuh) —
//   0 < r < m: k_peer_dir1 writes the local A_J into every rank's big slot (the all-gather),
//              k_peer_dir2 orders the gathered columns by rank, SMW Eq. (19) reads them in place;
//   r ≥ m:     k_peer_dir1 forms the local partial Gram, k_peer_dir2 deposits it into every rank and
//              k_peer_gram_sum forms I_m + κ Σ_q in rank order (Eq. (18)).
// Every kernel is predicated on the global branch (geo from the global r); worst-case grids.
int newton_direction_graph_peer(ssnal_en_problem* P) {
  const int64_t m = P->m;
  const DirGeo* geo = &P->ctl->geo;
  const AccA ga{(const double*)(P->pc.base[P->pc.rank] + peer_big_off(P->pc.size, P->pc.ss)), m};
  const unsigned gsm = 2 * P->nsm;
  int rc = with_acc(P, [&](auto acc) {
    k_peer_dir1<<<gsm, 256, 0, P->st>>>(P->pc, acc, m, P->J[0], P->r_dev + 0, geo);  // SMW: the all-gather
    P->launches++;
    return launch_gram_raw(P, acc, P->J[0], 0, P->r_dev + 0, P->W, geo);  // m × m: the local partial Gram
  });
  if (rc) return rc;
  k_peer_dir2<<<reduce_grid(P, m * m), 256, 0, P->st>>>(P->pc, P->W, m, geo, P->peer_idx);
  P->launches++;
  // SMW on the gathered columns (the K3 launch of the unsharded graph, restricted to branch 1)
  rc = launch_gram(P, ga, P->peer_idx, P->g[0], GramFusedArgs{}, geo, 1);
  if (rc) return rc;
  k_peer_gram_sum<<<reduce_grid(P, m * m), 256, 0, P->st>>>(P->pc, m, P->Mmat, P->g[0], geo, 0.0, 0, 0.0);
  P->launches++;
  CKL();
  rc = launch_chol(P, P->Mmat, 0, nullptr, 0.0, nullptr, nullptr, nullptr, nullptr, geo, -1);
  if (rc) return rc;
  k_gather_rows<<<gather_rows_grid(P), 256, 0, P->st>>>(ga, m, P->peer_idx, P->u, 0, nullptr, nullptr, geo, kGatherSmw,
                                                         P->d, P->g[0], P->y[0], P->y[1], P->scratch, P->blk,
                                                         P->ticket);
  P->launches++;
  CKL();
  return SSNAL_OK;
}

int newton_direction_graph(ssnal_en_problem* P) {
  if (P->peer) return newton_direction_graph_peer(P);
  const int64_t m = P->m;
  const DirGeo* geo = &P->ctl->geo;
  const int32_t* J = P->J[0];
  const double* g = P->g[0];
  double* gd = P->scratch;
  // K3 (worst-case grid: the m × m tiles; the SMW tiles for r < m are fewer)
  int rc = with_acc(P, [&](auto acc) { return launch_gram(P, acc, J, g, GramFusedArgs{}, geo); });
  if (rc) return rc;
  rc = launch_chol(P, P->Mmat, 0, nullptr, 0.0, nullptr, nullptr, nullptr, nullptr, geo, -1);
  if (rc) return rc;
  with_acc(P, [&](auto acc) {  // SMW back-substitution, or d = −g when r = 0
    k_gather_rows<<<gather_rows_grid(P), 256, 0, P->st>>>(acc, m, J, P->u, 0, nullptr, nullptr, geo, kGatherSmw, P->d,
                                                           g, P->y[0], P->y[1], gd, P->blk, P->ticket);
    return 0;
  });
  P->launches++;
  CKL();
  // K6 only when the strategy can select it (the options drop the graph when they change)
  if (!(P->cg_ratio > 0.0) && !((double)std::min<int64_t>(m, P->n) > P->cg_threshold)) return SSNAL_OK;
  return launch_cg(P, J, 0, g, 0.0, P->d, gd, P->y[0], P->y[1], geo);  // predicated on branch 3
}

int check_args(ssnal_en_problem* P, double l1, double l2, double sigma0, double tol) {
  if (!P) {
    set_err("null handle");
    return SSNAL_EINVAL;
  }
  if (!(l1 >= 0) || !(l2 >= 0) || (l1 == 0 && l2 == 0) || !isfinite(l1) || !isfinite(l2)) {
    set_err("invalid lambda (l1=%g, l2=%g)", l1, l2);
    return SSNAL_EINVAL;
  }
  if (!(sigma0 > 0) || !isfinite(sigma0)) {
    set_err("invalid sigma0 %g", sigma0);
    return SSNAL_EINVAL;
  }
  if (!(tol > 0)) {
    set_err("invalid tol %g", tol);
    return SSNAL_EINVAL;
  }
  return SSNAL_OK;
}

// ---------------- Algorithm 1 ----------------
// Start point (both modes).  x (P->x) holds x0 on entry (device).  Writes the support of x
// (Jx, Px, r_dev[2]), y0 into y[0] and w0 = Aᵀy0 into w[0].  *rx = host-known |supp x| (0 cold,
// −1 = on the device only).
int init_point(ssnal_en_problem* P, int have_x0, ssnal_en_stats* S, int64_t* rx, bool keep_dual = false,
               bool support_current = false) {
  const int64_t m = P->m, n = P->n;
  int rc;
  if (keep_dual && support_current && have_x0) {
    // a path point continuing from the previous solve on this handle: x, its support (Jx, Px, r_dev[2])
    // and the dual iterate (y[0], w[0]) are all that solve's final state — nothing to recompute
    CK(cudaMemcpyAsync(P->r_dev + 4, P->r_dev + 2, 8, cudaMemcpyDeviceToDevice, P->st));  // |supp x0| for stats
    *rx = -1;
    return SSNAL_OK;
  }
  // Support of x (Jx, Px, rx): K1e with w = 0, σ = 1, λ = 0 selects x ≠ 0 and P = x.
  *rx = 0;
  if (have_x0) {
    CK(cudaMemsetAsync(P->w[2], 0, n * 8, P->st));
    const Scal s0 = make_scal(1.0, 0.0, 0.0);
    if ((rc = launch_k1e(P, P->w[2], nullptr, 0.0, P->x, s0, nullptr))) return rc;
    if ((rc = launch_finalize(P, P->Jx, P->Px, P->r_dev + 2))) return rc;
    CK(cudaMemcpyAsync(P->r_dev + 4, P->r_dev + 2, 8, cudaMemcpyDeviceToDevice, P->st));  // |supp x0| for stats
    *rx = -1;
  } else {
    CK(cudaMemsetAsync(P->x, 0, n * 8, P->st));
    CK(cudaMemsetAsync(P->r_dev + 2, 0, 8, P->st));
    CK(cudaMemsetAsync(P->r_dev + 4, 0, 8, P->st));
  }
  // keep_dual (reading R39, a warm-started path point): y[0] and w[0] = Aᵀy[0] still hold the
  // previous solve's final dual iterate — the start of this one, no Aᵀ pass
  if (keep_dual) return SSNAL_OK;
  // Initial y, w (P:242 silent; reading R8): y0 = A x0 − b if x0 ≠ 0, else 0 (decided on the device)
  if (have_x0 && P->init_mode == 1) {
    // unsharded: the row-block cluster gather leaves the finished A_S x0_S in part_vec row 0
    if ((rc = sharded(P) ? launch_gather_dev(P, P->Jx, P->Px, P->r_dev + 2)
                         : launch_gather_vec(P, P->Jx, P->Px, P->r_dev + 2)))
      return rc;
    if (sharded(P)) {  // y0 = Σ_ranks A_S x0_S − b; warm iff the global support is non-empty
      if ((rc = exchange_eval(P, P->part_vec, P->gax_valid, kGatherDevGrid, nullptr, 0, P->r_dev + 2))) return rc;
      k_init_y<<<1, 1024, 0, P->st>>>(m, P->b, P->xbuf, nullptr, 1, P->rg_dev, P->y[0]);
      CK(cudaMemcpyAsync(P->r_dev + 4, P->rg_dev, 8, cudaMemcpyDeviceToDevice, P->st));
    } else {
      k_init_y<<<1, 1024, 0, P->st>>>(m, P->b, P->part_vec, nullptr, 1, P->r_dev + 2, P->y[0]);
    }
    P->launches++;
    CKL();
    if ((rc = launch_k1(P, P->y[0], nullptr, make_scal(1.0, 0.0, 0.0), 0, P->w[0]))) return rc;
    S->aty_passes++;  // corrected at the end if x0 turned out to be zero (cold start, no pass)
  } else {
    CK(cudaMemsetAsync(P->y[0], 0, m * 8, P->st));
    CK(cudaMemsetAsync(P->w[0], 0, n * 8, P->st));
  }
  return SSNAL_OK;
}

// Objective pieces at the final x (both modes): resid = A x − b from the support (Jx, Px, r_dev[2])
// → scratch_host[16..19] = [½‖resid‖², Σ|x|, Σx², nnz], scratch_host[20] = |supp x0| (after a sync).
// The objective pieces' kernels (and, sharded, their exchanges) without the host copies: also
// captured into the path graph.
int objective_kernels(ssnal_en_problem* P) {
  int rc;
  if ((rc = sharded(P) ? launch_gather_dev(P, P->Jx, P->Px, P->r_dev + 2)
                       : launch_gather_vec(P, P->Jx, P->Px, P->r_dev + 2)))
    return rc;
  if (sharded(P)) {  // resid = Σ_ranks A_S x_S − b; Σ|x|, Σx², nnz summed over the ranks
    if ((rc = exchange_eval(P, P->part_vec, P->gax_valid, kGatherDevGrid, nullptr, 0, P->r_dev + 2))) return rc;
    k_combine<<<1, 1024, 0, P->st>>>(P->m, P->b, -1.0, P->xbuf, 1, P->tmpm, nullptr, nullptr, nullptr);
    k_objective<<<1, 1024, 0, P->st>>>(P->m, P->tmpm, P->Px, P->r_dev + 2, P->scratch + 16);
    P->launches += 2;
    CKL();
    CK(cudaMemcpyAsync(P->xbuf, P->scratch + 17, 3 * 8, cudaMemcpyDeviceToDevice, P->st));
    if ((rc = comm_allreduce(P, P->xbuf, 3, 0))) return rc;
    CK(cudaMemcpyAsync(P->scratch + 17, P->xbuf, 3 * 8, cudaMemcpyDeviceToDevice, P->st));
  } else {
    k_combine<<<1, 1024, 0, P->st>>>(P->m, P->b, -1.0, P->part_vec, 1, P->tmpm, nullptr, nullptr, nullptr);
    P->launches++;
    CKL();
    k_objective<<<1, 1024, 0, P->st>>>(P->m, P->tmpm, P->Px, P->r_dev + 2, P->scratch + 16);
    P->launches++;
    CKL();
  }
  return SSNAL_OK;
}

int launch_objective(ssnal_en_problem* P) {
  int rc = objective_kernels(P);
  if (rc) return rc;
  CK(cudaMemcpyAsync(P->scratch_host + 16, P->scratch + 16, 4 * 8, cudaMemcpyDeviceToHost, P->st));
  CK(cudaMemcpyAsync(P->scratch_host + 20, P->r_dev + 4, 8, cudaMemcpyDeviceToHost, P->st));
  return SSNAL_OK;
}

// Host-driven mode: control decisions on the CPU from the EvalOut records (mapped memory).
// R40 gate for a cold solve (x0 = 0, y0 = 0): may this solve's trial K1 launches serve y == −b from the
// Aᵀb kept by create?  Yes while the active set at y = −b, #{|Aᵀb|_i > λ1}, is at most reuse_frac·n
// (those columns are gathered from global memory for the ∇ψ rows).  One small kernel and one stream
// synchronisation, only for cold solves on designs of at least reuse_min_bytes (2 GB).
int reuse_gate(ssnal_en_problem* P, double l1, int have_x0, bool keep_dual, int* allow) {
  *allow = 0;  // → K1Params::rmode: 1 with the ∇ψ rows (small active set at −b), 2 ψ only (large; unsharded handles)
  if (have_x0 || keep_dual || !P->atb || !P->reuse_atb) return SSNAL_OK;
  if ((int64_t)8 * P->m * P->n < P->reuse_min_bytes) return SSNAL_OK;
  k_atb_gate<<<2 * P->nsm, 256, 0, P->st>>>(P->atb, P->n, l1, (int64_t)(P->reuse_frac * (double)P->n), P->gate_cnt,
                                             P->gate_flag_dev, nullptr);
  P->launches++;
  CKL();
  CK(cudaStreamSynchronize(P->st));
  *allow = *(volatile int*)P->gate_flag_host ? 1 : ((P->reuse_psi_only && !sharded(P)) ? 2 : 0);
  P->atb_reuses += *allow != 0;
  return SSNAL_OK;
}

int solve_core(ssnal_en_problem* P, double l1, double l2, double sigma0, double tol, int have_x0,
               ssnal_en_stats* S, bool keep_dual = false) {
  const int64_t m = P->m;
  memset(S, 0, sizeof(*S));
  int rc;
  int cur = 0;  // index of current J/PJ/y/g
  int wcur = 0; // index of current w buffer (0..2)
  EvalOut ev, evt;
  int64_t rx = 0;
  CK(cudaMemsetAsync(&P->ctl->cg_iters, 0, sizeof(int), P->st));
  if ((rc = init_point(P, have_x0, S, &rx, keep_dual))) return rc;
  int reuse_first = 0;  // R40: trials at y == −b from the kept Aᵀb while its active set is small
  if ((rc = reuse_gate(P, l1, have_x0, keep_dual, &reuse_first))) return rc;

  double sigma = sigma0;
  int converged = 0, numeric = 0, k;
  int inject = P->inject_fail;
  for (k = 0; k < P->max_outer && !numeric; ++k) {
    const Scal sc = make_scal(sigma, l1, l2);
    // EVAL(y, w) with the new (x, σ): K1e + finalize + gather (∇ψ) + reduce
    if ((rc = launch_k1e(P, P->w[wcur], nullptr, 0.0, P->x, sc, nullptr))) return rc;
    // partial scalars of K1e are in part_scal; they are reduced by the eval kernel
    if ((rc = launch_finalize(P, P->J[cur], P->PJ[cur], P->r_dev + cur))) return rc;
    // ∇ψ needs A_J P_J for the re-thresholded J: gather with r read on the device
    if ((rc = launch_gather_vec(P, P->J[cur], P->PJ[cur], P->r_dev + cur))) return rc;
    // K1e wrote G scalar partials; the gather wrote the finished vector A_J P_J (part_vec row 0)
    if ((rc = eval_g(P, P->y[cur], sc, 1, nullptr, 1, P->g[cur], P->r_dev + cur, 0))) return rc;
    if ((rc = fetch_eval(P, 0, &ev))) return rc;
    S->psi_evals++;

    double tol_in = tol;  // inner stop (R6); adaptive schedule (R37)
    if (P->inner_tol_mode) {
      const double res3_0 = (sqrt(ev.s[1]) / sigma) / (1.0 + sqrt(ev.yy) + sqrt(ev.s[2]));
      tol_in = fmax(tol, 0.1 * res3_0);
    }
    int retry = 0;  // the current step's factor failed once: recompute it with the jitter (R36)
    for (int j = 0; j < P->max_inner; ++j) {
      if (ev.res1 <= tol_in) break;  // inner stop, Eq. (20) res(kkt1) (R6)
      int br = 0;
      double* gd_dev = P->scratch;
      // trial s = 1: y_t = y + d (written by the direction's last kernel); K1 fused at y_t
      const int tr = 1 - cur;
      const int wtr = (wcur + 1) % 3, wbt = (wcur + 2) % 3;
      if ((rc = newton_direction(P, P->J[cur], ev.r, P->g[cur], sc.kappa, P->d, gd_dev, &br, P->y[cur], P->y[tr],
                                 retry ? P->jitter : 0.0, P->r_dev + cur)))
        return rc;
      S->branch_steps[br]++;
      // R40: while J = ∅ after a cold start the trial is at y = −b: K1 checks and takes w = −Aᵀb kept by create
      if ((rc = launch_k1(P, P->y[tr], P->x, sc, 1, P->w[wtr], nullptr, nullptr, reuse_first,
                          reuse_first && ev.r == 0)))
        return rc;
      S->aty_passes++;
      if ((rc = launch_finalize(P, P->J[tr], P->PJ[tr], P->r_dev + tr))) return rc;
      if ((rc = eval_g(P, P->y[tr], sc, 1, P->cta_cnt, P->G, P->g[tr], P->r_dev + tr, 1, gd_dev,
                            (br == 1 || br == 2) ? P->info : nullptr)))
        return rc;
      if ((rc = fetch_eval(P, 1, &evt))) return rc;
      S->psi_evals++;
      if (reuse_first == 2 && ((volatile int*)P->gate_flag_host)[1] && isfinite(evt.psi) && isfinite(evt.gd) &&
          evt.psi - ev.psi <= P->mu * evt.gd + 10.0 * kEps * ev.psimag) {
        // R40: s = 1 accepted on a ψ-only trial — the same trial streamed (bitwise the same ψ, with its ∇ψ)
        if ((rc = launch_k1(P, P->y[tr], P->x, sc, 1, P->w[wtr]))) return rc;
        if ((rc = launch_finalize(P, P->J[tr], P->PJ[tr], P->r_dev + tr))) return rc;
        if ((rc = eval_g(P, P->y[tr], sc, 1, P->cta_cnt, P->G, P->g[tr], P->r_dev + tr, 1, gd_dev, nullptr))) return rc;
        if ((rc = fetch_eval(P, 1, &evt))) return rc;
      }
      if ((br == 1 || br == 2) && inject > 0) {
        inject--;
        evt.info = 1;
      }
      if ((br == 1 || br == 2) && evt.info != 0 && !retry && P->jitter > 0.0) {
        retry = 1;  // same y, same step index: redo the direction with the jittered factor
        S->jitter_retries++;
        --j;
        continue;
      }
      if ((br == 1 || br == 2) && evt.info != 0) {
        numeric = 1;
        set_err("Cholesky pivot not positive (branch %d, r=%lld)", br, (long long)ev.r);
        break;
      }
      const double gd = evt.gd;
      if (!isfinite(evt.psi) || !isfinite(gd)) {
        numeric = 1;
        set_err("non-finite psi/gd");
        break;
      }
      // Armijo, Eq. (13) with μ, halving (R5), roundoff guard (R29)
      double s = 1.0;
      int nbt = 0;
      bool ok = evt.psi - ev.psi <= P->mu * s * gd + 10.0 * kEps * ev.psimag;
      while (!ok) {
        if (nbt >= P->max_bt) {
          S->line_search_stalled = 1;  // R30: accept the last s
          break;
        }
        s *= P->beta;
        nbt++;
        // trial y + s d; w_s = w + s (w1 − w) (linearity of Aᵀ, R14)
        k_axpy_m<<<(unsigned)((m + 255) / 256), 256, 0, P->st>>>(m, P->y[cur], s, P->d, P->y[tr], nullptr);
        P->launches++;
        CKL();
        if ((rc = launch_k1e(P, P->w[wcur], P->w[wtr], s, P->x, sc, P->w[wbt]))) return rc;
        if ((rc = launch_finalize(P, P->J[tr], P->PJ[tr], P->r_dev + tr))) return rc;
        if ((rc = eval_g(P, P->y[tr], sc, 0, nullptr, 0, nullptr, P->r_dev + tr, 2))) return rc;
        EvalOut eb;
        if ((rc = fetch_eval(P, 2, &eb))) return rc;
        S->psi_evals++;
        evt = eb;
        ok = evt.psi - ev.psi <= P->mu * s * gd + 10.0 * kEps * ev.psimag;
      }
      S->backtracks += nbt;
      // accept: y ← y + s d (Algorithm 1 step (3)); z implicit via P (step (4))
      if (nbt == 0) {
        cur = tr;
        wcur = wtr;
        ev = evt;
      } else {
        cur = tr;
        wcur = wbt;  // materialised w + s (w1 − w)
        // ∇ψ at the accepted point needs A_J P_J for the re-thresholded J (K2)
        if ((rc = launch_gather_vec(P, P->J[cur], P->PJ[cur], P->r_dev + cur))) return rc;
        // scalar partials in part_scal still belong to the accepted K1e launch
        if ((rc = eval_g(P, P->y[cur], sc, 1, nullptr, 1, P->g[cur], P->r_dev + cur, 0)))
          return rc;
        if ((rc = fetch_eval(P, 0, &ev))) return rc;
      }
      S->newton_iters++;
      retry = 0;
    }
    if (numeric) break;
    // Multiplier update Eq. (10): x ← x − σ(Aᵀy + z̄) = P (Moreau); res(kkt3) Eq. (20)
    const double res3 = (sqrt(ev.s[1]) / sigma) / (1.0 + sqrt(ev.yy) + sqrt(ev.s[2]));
    S->res_kkt3 = res3;
    S->res_kkt1 = ev.res1;
    if (rx > 0) {
      k_zero_at<<<(unsigned)((rx + 255) / 256), 256, 0, P->st>>>(P->Jx, rx, nullptr, P->x, nullptr);
      P->launches++;
      CKL();
    } else if (rx < 0) {  // warm start: count on the device
      k_zero_at<<<2 * P->nsm, 256, 0, P->st>>>(P->Jx, -1, P->r_dev + 2, P->x, nullptr);
      P->launches++;
      CKL();
    }
    if (sharded(P)) {  // ev.r is the global count: the local support lives on the device only
      k_zero_at<<<2 * P->nsm, 256, 0, P->st>>>(P->Jx, -1, P->r_dev + 2, P->x, nullptr);
      k_scatter_dev<<<2 * P->nsm, 256, 0, P->st>>>(P->J[cur], P->PJ[cur], P->r_dev + cur, P->x, P->Jx, P->Px,
                                                    P->r_dev + 2);
      P->launches += 2;
      CKL();
      rx = -1;
      if (res3 <= tol && ev.res1 <= tol) {
        converged = 1;
        k++;
        break;
      }
      sigma = fmin(P->sigma_factor * sigma, P->sigma_max);
      continue;
    }
    const int64_t rnew = ev.r;
    if (rnew > 0) {
      k_scatter<<<(unsigned)((rnew + 255) / 256), 256, 0, P->st>>>(P->J[cur], P->PJ[cur], rnew, P->x);
      P->launches++;
      CKL();
      CK(cudaMemcpyAsync(P->Jx, P->J[cur], rnew * 4, cudaMemcpyDeviceToDevice, P->st));
      CK(cudaMemcpyAsync(P->Px, P->PJ[cur], rnew * 8, cudaMemcpyDeviceToDevice, P->st));
    }
    CK(cudaMemcpyAsync(P->r_dev + 2, P->r_dev + cur, 8, cudaMemcpyDeviceToDevice, P->st));
    rx = rnew;
    if (res3 <= tol && ev.res1 <= tol) {  // R7
      converged = 1;
      k++;
      break;
    }
    sigma = fmin(P->sigma_factor * sigma, P->sigma_max);  // P:497, R9
  }
  S->outer_iters = k;
  S->sigma_final = sigma;
  S->status = numeric ? SSNAL_ENUMERIC : (converged ? SSNAL_OK : SSNAL_NOT_CONVERGED);
  // the final dual iterate into the fixed slots y[0], w[0], as graph mode leaves it, so that the next
  // solve of a path can start there (reading R39, option warm_dual / carry_dual)
  if (cur != 0) CK(cudaMemcpyAsync(P->y[0], P->y[cur], P->m * 8, cudaMemcpyDeviceToDevice, P->st));
  if (wcur != 0) CK(cudaMemcpyAsync(P->w[0], P->w[wcur], P->n * 8, cudaMemcpyDeviceToDevice, P->st));
  // Stats: F(x) (Eq. (1)) via resid = A x − b; D(y) = −½yᵀy − bᵀy − Σ(|w|−λ1)²₊/(2λ2)
  if ((rc = launch_objective(P))) return rc;
  S->dual_obj = (l2 > 0) ? (-(0.5 * ev.yy + ev.by) - ev.s[3] / (2.0 * l2)) : NAN;
  CK(cudaMemcpyAsync(P->scratch_host + 40, &P->ctl->cg_iters, sizeof(int), cudaMemcpyDeviceToHost, P->st));
  P->stat_l1 = l1;
  P->stat_l2 = l2;
  P->stat_warm_pass = (have_x0 && P->init_mode == 1 && !keep_dual);
  P->graph_pending = false;
  return S->status;
}

// ---------------- graph mode ----------------
// Append a conditional WHILE node (handle h) to the graph being captured on st; returns its body.
int add_while(cudaStream_t st, cudaGraphConditionalHandle h, cudaGraph_t* body) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, deps, nd, &cp));
  CK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
  *body = cp.conditional.phGraph_out[0];
  return SSNAL_OK;
}

// Captures the three loop levels into the bodies of nested WHILE nodes (see k_ctl.cuh).
// body_pre / h_pre (path graph): capture the solve into an existing outer-loop body whose WHILE node
// (handle h_pre) the caller has added; otherwise the outer WHILE node is added at the root of G.
int capture_graph(ssnal_en_problem* P, cudaGraph_t G, cudaGraph_t body_pre = nullptr,
                  cudaGraphConditionalHandle h_pre = 0) {
  const int64_t m = P->m, n = P->n;
  DevCtl* C = P->ctl;
  const Scal none = make_scal(1.0, 0.0, 0.0);  // placeholder: every kernel reads C->sc
  int rc;
  cudaGraphConditionalHandle h_outer, h_inner, h_bt;
  // ψ evaluation + the control decision that consumes it; on a peer-attached sharded handle the
  // evaluation record is first summed over the ranks by k_peer_eval (same predicate on every rank)
  auto eval_at = [&](const double* y, int with_grad, const int* valid, int nparts, double* g_out, int64_t* r_loc,
                     int slot, const double* gd_src, const int* info_src, const int* pred, int hook,
                     const CtlHook* hk) -> int {
    if (!P->peer)
      return launch_eval(P, y, none, with_grad, valid, nparts, g_out, r_loc, slot, gd_src, info_src, &C->sc, pred,
                         nullptr, nullptr, 0, hook, hk);
    k_peer_eval<<<kRecCS, 256, 0, P->st>>>(P->pc, m, nparts ? P->part_vec : nullptr, valid, nparts, P->part_scal,
                                           P->G, r_loc, P->xbuf, P->rg_dev, pred);
    P->launches++;
    return launch_eval(P, y, none, with_grad, nullptr, nparts ? 1 : 0, g_out, P->rg_dev, slot, gd_src, info_src, &C->sc,
                       pred, P->xbuf, P->xbuf + m, 1, hook, hk);
  };
  cudaGraph_t body_o, body_i, body_b;
  if (body_pre) {
    h_outer = h_pre;
    body_o = body_pre;
  } else {
    CK(cudaGraphConditionalHandleCreate(&h_outer, G, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h_outer;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, G, nullptr, 0, &cp));
    body_o = cp.conditional.phGraph_out[0];
  }
  // ---- outer body: σ-scalars, EVAL(y, x), first inner test ----
  CK(cudaStreamBeginCaptureToGraph(P->cap[0], body_o, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  P->cap_depth = 1;
  P->st = P->cap[0];
  CK(cudaGraphConditionalHandleCreate(&h_inner, body_o, 0, 0));
  int64_t L = P->launches;
  k_ctl_outer_begin<<<1, 1, 0, P->st>>>(C);
  P->launches++;
  if ((rc = launch_k1e(P, P->w[0], nullptr, 0.0, P->x, none, nullptr, &C->sc, nullptr))) return rc;
  if ((rc = launch_finalize(P, P->J[0], P->PJ[0], P->r_dev + 0))) return rc;
  if ((rc = launch_gather_vec(P, P->J[0], P->PJ[0], P->r_dev + 0))) return rc;
  CtlHook hk{C, P->ev_dev + 0, nullptr, m, P->nsm, P->W_splits, P->info, h_inner};
  if ((rc = eval_at(P->y[0], 1, nullptr, 1, P->g[0], P->r_dev + 0, 0, nullptr, nullptr, nullptr, kHookInnerBegin, &hk)))
    return rc;
  (P->capture_reuse ? P->seg_kernels_r : P->seg_kernels)[0] = (int)(P->launches - L);
  if ((rc = add_while(P->cap[0], h_inner, &body_i))) return rc;
  {
    // ---- inner body: direction, trial K1 at y + d, Armijo ----
    CK(cudaStreamBeginCaptureToGraph(P->cap[1], body_i, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    P->cap_depth = 2;
    P->st = P->cap[1];
    CK(cudaGraphConditionalHandleCreate(&h_bt, body_i, 0, 0));
    L = P->launches;
    if ((rc = newton_direction_graph(P))) return rc;
    if ((rc = launch_k1(P, P->y[1], P->x, none, 1, P->w[1], &C->sc, C->tstamp, P->capture_reuse ? -1 : 0))) return rc;
    if ((rc = launch_finalize(P, P->J[1], P->PJ[1], P->r_dev + 1))) return rc;
    CtlHook ha{C, P->ev_dev + 0, P->ev_dev + 1, m, P->nsm, P->W_splits, P->info, h_bt};
    if ((rc = eval_at(P->y[1], 1, P->cta_cnt, P->G, P->g[1], P->r_dev + 1, 1, P->scratch, P->info, nullptr, kHookArmijo,
                      &ha)))
      return rc;
    if (P->capture_reuse) {  // R40 redo (predicated on C->redo): a ψ-only trial whose s = 1 Armijo accepted, streamed
      if ((rc = launch_k1(P, P->y[1], P->x, none, 1, P->w[1], &C->sc, C->tstamp, -1, 0, &C->redo, 1))) return rc;
      if ((rc = launch_finalize(P, P->J[1], P->PJ[1], P->r_dev + 1, &C->redo))) return rc;
      if ((rc = eval_at(P->y[1], 1, P->cta_cnt, P->G, P->g[1], P->r_dev + 1, 1, P->scratch, nullptr, &C->redo,
                        kHookArmijoRedo, &ha)))
        return rc;
    }
    (P->capture_reuse ? P->seg_kernels_r : P->seg_kernels)[1] = (int)(P->launches - L);
    if ((rc = add_while(P->cap[1], h_bt, &body_b))) return rc;
    {
      // ---- backtrack body: y + s d, K1e from w + s (w1 − w), Armijo ----
      CK(cudaStreamBeginCaptureToGraph(P->cap[2], body_b, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
      P->cap_depth = 3;
      P->st = P->cap[2];
      L = P->launches;
      k_axpy_m<<<(unsigned)((m + 255) / 256), 256, 0, P->st>>>(m, P->y[0], 0.0, P->d, P->y[1], &C->s);
      P->launches++;
      if ((rc = launch_k1e(P, P->w[0], P->w[1], 0.0, P->x, none, P->w[2], &C->sc, &C->s))) return rc;
      if ((rc = launch_finalize(P, P->J[1], P->PJ[1], P->r_dev + 1))) return rc;
      CtlHook hb{C, P->ev_dev + 0, P->ev_dev + 2, m, P->nsm, P->W_splits, P->info, h_bt};
      if ((rc = eval_at(P->y[1], 0, nullptr, 0, nullptr, P->r_dev + 1, 2, nullptr, nullptr, nullptr, kHookBacktrack,
                        &hb)))
        return rc;
      (P->capture_reuse ? P->seg_kernels_r : P->seg_kernels)[2] = (int)(P->launches - L);
      cudaGraph_t tmp;
      CK(cudaStreamEndCapture(P->cap[2], &tmp));
      P->cap_depth = 2;
      P->st = P->cap[1];
    }
    // ---- accept (trial → current), gradient after a backtrack, next inner test ----
    L = P->launches;
    k_accept<<<2 * P->nsm, 256, 0, P->st>>>(C, m, n, P->y[0], P->y[1], P->g[0], P->g[1], P->J[0], P->J[1],
                                              P->PJ[0], P->PJ[1], P->r_dev, P->w[0], P->w[1], P->w[2], P->ev_dev);
    P->launches++;
    if ((rc = launch_gather_vec(P, P->J[0], P->PJ[0], P->r_dev + 0, &C->need_grad))) return rc;
    CtlHook he{C, P->ev_dev + 0, nullptr, m, P->nsm, P->W_splits, P->info, h_inner};
    if ((rc = eval_at(P->y[0], 1, nullptr, 1, P->g[0], P->r_dev + 0, 0, nullptr, nullptr, &C->need_grad, kHookInnerEnd,
                      &he)))
      return rc;
    (P->capture_reuse ? P->seg_kernels_r : P->seg_kernels)[3] = (int)(P->launches - L);
    cudaGraph_t tmp;
    CK(cudaStreamEndCapture(P->cap[1], &tmp));
    P->cap_depth = 1;
    P->st = P->cap[0];
  }
  // ---- multiplier update x ← P, KKT stop, σ update ----
  L = P->launches;
  k_zero_at<<<2 * P->nsm, 256, 0, P->st>>>(P->Jx, -1, P->r_dev + 2, P->x, &C->numeric);
  k_xupdate<<<2 * P->nsm, 256, 0, P->st>>>(C, P->J[0], P->PJ[0], P->r_dev, P->x, P->Jx, P->Px);
  k_ctl_outer_end<<<1, 1, 0, P->st>>>(C, P->ev_dev + 0, h_outer);
  P->launches += 3;
  CKL();
  (P->capture_reuse ? P->seg_kernels_r : P->seg_kernels)[4] = (int)(P->launches - L);
  cudaGraph_t tmp;
  CK(cudaStreamEndCapture(P->cap[0], &tmp));
  P->cap_depth = 0;
  return SSNAL_OK;
}

int build_graph(ssnal_en_problem* P, bool reuse = false) {
  cudaGraphExec_t& gexec = reuse ? P->gexec_r : P->gexec;
  cudaGraph_t& graph = reuse ? P->graph_r : P->graph;
  if (gexec) return SSNAL_OK;
  for (int i = 0; i < 3; ++i)
    if (!P->cap[i]) CK(cudaStreamCreateWithFlags(&P->cap[i], cudaStreamNonBlocking));
  cudaGraph_t G;
  CK(cudaGraphCreate(&G, 0));
  cudaStream_t saved = P->st;
  const int64_t L0 = P->launches;
  P->capturing = true;
  P->capture_reuse = reuse;
  int rc = capture_graph(P, G);
  P->capture_reuse = false;
  // unwind any capture left open by a failure
  for (int d = P->cap_depth; d > 0; --d) {
    cudaGraph_t tmp;
    cudaStreamEndCapture(P->cap[d - 1], &tmp);
  }
  P->cap_depth = 0;
  P->capturing = false;
  P->st = saved;
  P->launches = L0;
  if (rc == SSNAL_OK) {
    cudaError_t e = cudaGraphInstantiate(&gexec, G, 0);
    if (e != cudaSuccess) {
      set_err("cudaGraphInstantiate: %s", cudaGetErrorString(e));
      rc = SSNAL_ECUDA;
      gexec = nullptr;
    } else if ((e = cudaGraphUpload(gexec, P->st)) != cudaSuccess) {  // device-side setup off the first solve
      set_err("cudaGraphUpload: %s", cudaGetErrorString(e));
      rc = SSNAL_ECUDA;
    }
  }
  if (rc) {
    cudaGetLastError();
    cudaGraphDestroy(G);
    return rc;
  }
  graph = G;
  return SSNAL_OK;
}

void drop_path_graph(ssnal_en_problem* P) {
  if (P->pgexec) cudaGraphExecDestroy(P->pgexec);
  if (P->pgraph) cudaGraphDestroy(P->pgraph);
  P->pgexec = nullptr;
  P->pgraph = nullptr;
}

void drop_graph(ssnal_en_problem* P) {
  if (P->gexec) cudaGraphExecDestroy(P->gexec);
  if (P->graph) cudaGraphDestroy(P->graph);
  if (P->gexec_r) cudaGraphExecDestroy(P->gexec_r);
  if (P->graph_r) cudaGraphDestroy(P->graph_r);
  P->gexec = P->gexec_r = nullptr;
  P->graph = P->graph_r = nullptr;
  drop_path_graph(P);  // it embeds the same solve body
}

// The device-resident λ path: WHILE (point < npts) { k_path_begin; the solve (the solve graph's
// nested WHILE loops, captured again into this body); the objective pieces; x → x_out[point];
// k_path_end } — points 1 … npts − 1 of a warm-started path in one launch, no host round trip
// between points (the host only reads the per-point slots after the path).  Multi-kernel graph mode
// (unsharded or peer-sharded), the dual and x carried (reading R39).
int build_path_graph(ssnal_en_problem* P, PathSlot* slots_dev) {
  if (P->pgexec) return SSNAL_OK;
  int rc;
  if (!P->pdev) {
    if ((rc = alloc((void**)&P->pdev, sizeof(PathDev)))) return rc;
    CK(cudaHostAlloc((void**)&P->pdev_host, sizeof(PathDev), cudaHostAllocDefault));
  }
  for (int i = 0; i < 3; ++i)
    if (!P->cap[i]) CK(cudaStreamCreateWithFlags(&P->cap[i], cudaStreamNonBlocking));
  if (!P->cap_path) CK(cudaStreamCreateWithFlags(&P->cap_path, cudaStreamNonBlocking));
  cudaGraph_t G;
  CK(cudaGraphCreate(&G, 0));
  cudaGraphConditionalHandle h_path;
  CK(cudaGraphConditionalHandleCreate(&h_path, G, 1, cudaGraphCondAssignDefault));
  cudaGraph_t body_p;
  {
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h_path;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    CK(cudaGraphAddNode(&node, G, nullptr, 0, &cp));
    body_p = cp.conditional.phGraph_out[0];
  }
  cudaStream_t saved = P->st;
  const int64_t L0 = P->launches;
  P->capturing = true;
  bool cap_open = false;
  rc = SSNAL_OK;
  do {
    cudaError_t e = cudaStreamBeginCaptureToGraph(P->cap_path, body_p, nullptr, nullptr, 0,
                                                  cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
      set_err("path graph capture: %s", cudaGetErrorString(e));
      rc = SSNAL_ECUDA;
      break;
    }
    cap_open = true;
    P->st = P->cap_path;
    cudaGraphConditionalHandle h_outer;
    if ((e = cudaGraphConditionalHandleCreate(&h_outer, body_p, 0, 0)) != cudaSuccess) {
      set_err("path graph handle: %s", cudaGetErrorString(e));
      rc = SSNAL_ECUDA;
      break;
    }
    k_path_begin<<<1, 1, 0, P->st>>>(P->ctl, P->pdev, P->r_dev, h_outer);
    cudaGraph_t body_o;
    if ((rc = add_while(P->cap_path, h_outer, &body_o))) break;
    if ((rc = capture_graph(P, G, body_o, h_outer))) break;  // the solve, on cap[0..2]
    P->st = P->cap_path;
    // the objective pieces of the final x (launch_objective without its host copies; peer-sharded:
    // with its exchanges, all kernels)
    const int64_t L1 = P->launches;
    if ((rc = objective_kernels(P))) break;
    const int nobj = (int)(P->launches - L1);
    k_path_copy_x<<<2 * P->nsm, 256, 0, P->st>>>(P->x, P->pdev, P->n);
    k_path_end<<<1, 1, 0, P->st>>>(P->ctl, P->ev_dev, P->scratch, P->r_dev, slots_dev, P->pdev, h_path);
    if ((e = cudaGetLastError()) != cudaSuccess) {
      set_err("path graph capture launch: %s", cudaGetErrorString(e));
      rc = SSNAL_ECUDA;
      break;
    }
    P->pgraph_fixed = 3 + nobj;  // begin, the objective's kernels, copy, end
  } while (false);
  for (int d = P->cap_depth; d > 0; --d) {  // a capture left open inside capture_graph by a failure
    cudaGraph_t tmp;
    cudaStreamEndCapture(P->cap[d - 1], &tmp);
  }
  P->cap_depth = 0;
  if (cap_open) {
    cudaGraph_t tmp;
    cudaError_t e = cudaStreamEndCapture(P->cap_path, &tmp);
    if (e != cudaSuccess && rc == SSNAL_OK) {
      set_err("path graph end capture: %s", cudaGetErrorString(e));
      rc = SSNAL_ECUDA;
    }
  }
  P->capturing = false;
  P->st = saved;
  P->launches = L0;
  if (rc == SSNAL_OK) {
    cudaError_t e = cudaGraphInstantiate(&P->pgexec, G, 0);
    if (e != cudaSuccess) {
      set_err("path graph instantiate: %s", cudaGetErrorString(e));
      P->pgexec = nullptr;
      rc = SSNAL_ECUDA;
    } else if ((e = cudaGraphUpload(P->pgexec, P->st)) != cudaSuccess) {
      set_err("path graph upload: %s", cudaGetErrorString(e));
      rc = SSNAL_ECUDA;
    }
  }
  if (rc) {
    cudaGetLastError();
    cudaGraphDestroy(G);
    drop_path_graph(P);
    return rc;
  }
  P->pgraph = G;
  return SSNAL_OK;
}

// Graph mode: the whole Algorithm 1 loop nest is one graph launch; stats are read back with the
// objective after the caller's synchronisation (finish_stats).
// Small problems (k_small.cuh): the whole loop nest in one CTA.  Same statistics path as graph mode
// (device control block + final EvalOut, finish_stats).
bool small_eligible(const ssnal_en_problem* P) {
  return P->use_small && !sharded(P) && !P->fmt && P->m <= kSmallMaxM && P->n <= kSmallMaxN &&
         !(P->cg_ratio > 0.0) && !((double)P->m > P->cg_threshold);  // time_k1: no K1 launches to time
}

int solve_small_core(ssnal_en_problem* P, double l1, double l2, double sigma0, double tol, int have_x0,
                     ssnal_en_stats* S, const double* sigma_dev = nullptr, bool keep_dual = false,
                     bool support_current = false) {
  memset(S, 0, sizeof(*S));
  int rc;
  int64_t rx = 0;
  const bool cl = P->use_small_cl && P->small_cl_ok;
  // the cluster kernel initialises a cold start itself (no memsets) and computes the objective
  if ((!cl || have_x0) && (rc = init_point(P, have_x0, S, &rx, keep_dual, support_current))) return rc;
  if (cl && !have_x0) S->aty_passes = 0;
  DevCtl* h = P->ctl_host;
  memset(h, 0, sizeof(DevCtl));
  h->l1 = l1;
  h->l2 = l2;
  h->tol = tol;
  h->sigma = sigma0;
  h->sigma_factor = P->sigma_factor;
  h->sigma_max = P->sigma_max;
  h->mu = P->mu;
  h->beta = P->beta;
  h->max_outer = P->max_outer;
  h->max_inner = P->max_inner;
  h->max_bt = P->max_bt;
  h->nb = P->nb;
  h->jitter = P->jitter;
  h->inject = P->inject_fail;
  h->inner_tol_mode = P->inner_tol_mode;
  SmallParams sp;
  memset(&sp, 0, sizeof(sp));
  if (cl) {  // settings by value, results straight into the mapped host mirrors (no copies)
    sp.use_cin = 1;
    sp.cin = *h;
    sp.sigma_in = sigma_dev;
    CK(cudaHostGetDevicePointer((void**)&sp.cout_host, h, 0));
    CK(cudaHostGetDevicePointer((void**)&sp.ev_host, P->ev_out_host, 0));
    double* sh_dev = nullptr;
    CK(cudaHostGetDevicePointer((void**)&sh_dev, P->scratch_host, 0));
    sp.obj = sh_dev + 16;
    sp.rx0_host = sh_dev + 20;
    sp.xout = P->direct_xout;
    P->xout_done = P->direct_xout != nullptr;
  } else {
    CK(cudaMemcpyAsync(P->ctl, h, sizeof(DevCtl), cudaMemcpyHostToDevice, P->st));
    if (sigma_dev)  // σ0 carried on the device from the previous path point (R38)
      CK(cudaMemcpyAsync(&P->ctl->sigma, sigma_dev, 8, cudaMemcpyDeviceToDevice, P->st));
  }
  sp.cold = (cl && !have_x0) ? 1 : 0;
  sp.rx0 = P->r_dev + 4;
  sp.resid = cl ? P->tmpm : nullptr;
  sp.A = P->A;
  sp.b = P->b;
  sp.m = (int)P->m;
  sp.n = (int)P->n;
  sp.x = P->x;
  sp.y0 = P->y[0];
  sp.w0 = P->w[0];
  sp.Jx = P->Jx;
  sp.Px = P->Px;
  sp.rx = P->r_dev + 2;
  sp.C = P->ctl;
  sp.ev = P->ev_dev;
  if (cl)  // A resident in the cluster's shared memory (k_small_cl.cuh); objective included
    k_small_cl<<<kClCtas, kClThreads, kClSmem, P->st>>>(sp);
  else
    k_small_solve<<<1, kSmallThreads, kSmallSmem, P->st>>>(sp);
  P->launches++;
  CKL();
  if (!cl) {
    if ((rc = launch_objective(P))) return rc;
    CK(cudaMemcpyAsync(h, P->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, P->st));
    CK(cudaMemcpyAsync(P->ev_out_host, P->ev_dev, sizeof(EvalOut), cudaMemcpyDeviceToHost, P->st));
  } else if (have_x0) {  // warm start: |supp x0| was counted by init_point on the device
    CK(cudaMemcpyAsync(P->scratch_host + 20, P->r_dev + 4, 8, cudaMemcpyDeviceToHost, P->st));
  }
  P->stat_l1 = l1;
  P->stat_l2 = l2;
  P->stat_warm_pass = (have_x0 && P->init_mode == 1 && !keep_dual);
  P->graph_pending = true;
  return SSNAL_OK;
}

int solve_graph_core(ssnal_en_problem* P, double l1, double l2, double sigma0, double tol, int have_x0,
                     ssnal_en_stats* S, const double* sigma_dev = nullptr, bool keep_dual = false,
                     bool support_current = false) {
  memset(S, 0, sizeof(*S));
  int rc;
  if ((rc = build_graph(P))) return rc;
  int64_t rx = 0;
  if ((rc = init_point(P, have_x0, S, &rx, keep_dual, support_current))) return rc;
  DevCtl* h = P->ctl_host;
  memset(h, 0, sizeof(DevCtl));
  h->l1 = l1;
  h->l2 = l2;
  h->tol = tol;
  h->sigma = sigma0;
  h->sigma_factor = P->sigma_factor;
  h->sigma_max = P->sigma_max;
  h->mu = P->mu;
  h->beta = P->beta;
  h->max_outer = P->max_outer;
  h->max_inner = P->max_inner;
  h->max_bt = P->max_bt;
  h->cg_ratio = sharded(P) ? 0.0 : P->cg_ratio;  // sharded: exact branches only (as host-driven)
  h->cg_threshold = sharded(P) ? INFINITY : P->cg_threshold;
  h->nb = P->nb;
  h->jitter = P->jitter;
  h->inject = P->inject_fail;
  h->inner_tol_mode = P->inner_tol_mode;
  h->tstamp[0] = ~0ull;
  h->tstamp[1] = 0ull;
  int reuse = 0;  // R40: the solve graph whose trial K1 may serve y == −b from the kept Aᵀb (mode 1 / 2)
  if ((rc = reuse_gate(P, l1, have_x0, keep_dual, &reuse))) return rc;
  if (reuse && (rc = build_graph(P, true))) return rc;
  h->reuse_mode = reuse;
  CK(cudaMemcpyAsync(P->ctl, h, sizeof(DevCtl), cudaMemcpyHostToDevice, P->st));
  if (sigma_dev)  // σ0 carried on the device from the previous path point (R38)
    CK(cudaMemcpyAsync(&P->ctl->sigma, sigma_dev, 8, cudaMemcpyDeviceToDevice, P->st));
  CK(cudaGraphLaunch(reuse ? P->gexec_r : P->gexec, P->st));
  P->stat_graph_r = reuse != 0;
  if ((rc = launch_objective(P))) return rc;
  CK(cudaMemcpyAsync(h, P->ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, P->st));
  CK(cudaMemcpyAsync(P->ev_out_host, P->ev_dev, sizeof(EvalOut), cudaMemcpyDeviceToHost, P->st));
  P->stat_l1 = l1;
  P->stat_l2 = l2;
  P->stat_warm_pass = (have_x0 && P->init_mode == 1 && !keep_dual);
  P->graph_pending = true;
  return SSNAL_OK;
}

// Complete the stats from the objective pieces copied by solve_core (after a stream sync).
void finish_stats(ssnal_en_problem* P, ssnal_en_stats* S) {
  if (P->graph_pending) {  // graph mode: counters and decisions from the device control block
    const DevCtl* C = P->ctl_host;
    const EvalOut* ev = P->ev_out_host;
    S->outer_iters = C->outer_iters;
    S->newton_iters = C->newton_iters;
    S->psi_evals = C->psi_evals;
    S->backtracks = C->backtracks;
    S->aty_passes += C->aty_passes;
    for (int b = 0; b < 4; ++b) S->branch_steps[b] = C->branch_steps[b];
    S->cg_iters = C->cg_iters;
    S->jitter_retries = C->jitter_retries;
    S->line_search_stalled = C->stalled;
    S->res_kkt1 = C->res1;
    S->res_kkt3 = C->res3;
    S->sigma_final = C->sigma_final;
    S->status = C->numeric ? SSNAL_ENUMERIC : (C->converged ? SSNAL_OK : SSNAL_NOT_CONVERGED);
    if (C->numeric && C->numeric_kind == 1) set_err("Cholesky pivot not positive (r=%lld)", (long long)C->numeric_r);
    else if (C->numeric) set_err("non-finite psi/gd");
    const double l2 = P->stat_l2;
    S->dual_obj = (l2 > 0) ? (-(0.5 * ev->yy + ev->by) - ev->s[3] / (2.0 * l2)) : NAN;
    const int* sk = P->stat_graph_r ? P->seg_kernels_r : P->seg_kernels;
    P->launches += (int64_t)C->seg_outer * (sk[0] + sk[4]) + (int64_t)C->seg_inner * (sk[1] + sk[3]) +
                   (int64_t)C->seg_bt * sk[2];
    P->stat_graph_r = false;
    if (P->time_k1) {  // in-kernel globaltimer stamps (events cannot sit inside conditional bodies)
      P->k1_time += C->k1_ns * 1e-9;
      P->k1_count += C->k1_cnt;
    }
    P->graph_pending = false;
  } else {
    int it = 0;
    memcpy(&it, P->scratch_host + 40, sizeof(int));
    S->cg_iters = it;
  }
  const double* o = P->scratch_host + 16;
  S->primal_obj = o[0] + P->stat_l1 * o[1] + 0.5 * P->stat_l2 * o[2];
  S->active = (int64_t)o[3];
  S->gap = S->primal_obj - S->dual_obj;
  int64_t rx0;
  memcpy(&rx0, P->scratch_host + 20, 8);
  if (P->stat_warm_pass && rx0 == 0) S->aty_passes--;  // x0 was all zero: cold start, no pass (R8)
}

}  // namespace

// ===========================================================================
extern "C" {

const char* ssnal_en_last_error(void) { return g_err.c_str(); }

const char* ssnal_en_version(void) { return "ssnal_en_b200 0.2 (sm_100a, fp64)"; }

// Device query, launch configuration and every allocation of the handle.  The host-memory creates call it
// BEFORE they enqueue the upload of A: the pool allocations synchronise the default stream, and behind
// the upload they would wait for it (cfg2: 7.3 ms) and push the graph capture after it instead of under it.
static int create_prepare(ssnal_en_problem* P) {
  if (P->prepared) return SSNAL_OK;
  CK(cudaGetDevice(&P->dev));
  CK(cudaDeviceGetAttribute(&P->nsm, cudaDevAttrMultiProcessorCount, P->dev));
  int rc = configure(P);
  if (rc) return rc;
  rc = allocate(P);
  if (rc) return rc;
  P->prepared = true;
  return SSNAL_OK;
}

static int create_common(ssnal_en_problem* P) {
  int rc = create_prepare(P);
  if (rc) return rc;
  // Capture + instantiate the solve graph now: host work that overlaps the asynchronous upload of A
  // (ssnal_en_create with pinned input) instead of delaying the first solve.
  // (not for handles the one-launch small path serves: their solves never launch it; a later set_option
  // that makes the handle ineligible builds it on the first solve)
  if (P->use_graph && !small_eligible(P) && (rc = build_graph(P))) return rc;
  if (P->use_graph && P->atb && P->reuse_atb && (int64_t)8 * P->m * P->n >= P->reuse_min_bytes &&
      (rc = build_graph(P, true)))  // R40: the cold-solve graph with the REUSE trial K1
    return rc;
  // validate inputs on the device
  CK(cudaMemsetAsync(P->flags, 0, 8, P->st));
  if (P->fmt)
    k_validate_geno<<<4 * P->nsm, 256, 0, P->st>>>(P->codes, P->cstride, P->tab, P->m, P->n, P->b, P->flags);
  else
    k_validate<<<4 * P->nsm, 256, 0, P->st>>>(P->A, P->m, P->n, P->b, P->flags);
  CKL();
  int hf[2] = {0, 0};
  CK(cudaMemcpyAsync(P->scratch_host, P->flags, 8, cudaMemcpyDeviceToHost, P->st));
  CK(cudaStreamSynchronize(P->st));
  memcpy(hf, P->scratch_host, 8);
  if (hf[0]) {
    set_err(P->fmt ? "invalid genotype codes / table or non-finite b (%d columns)" : "A or b contains NaN/Inf (%d columns)",
            hf[0]);
    return SSNAL_EINVAL;
  }
  if (hf[1]) {
    set_err("A has %d all-zero columns", hf[1]);
    return SSNAL_EINVAL;
  }
  // λmax = ‖Aᵀb‖∞ (plain K1 pass) and ‖b‖
  rc = launch_k1(P, P->b, nullptr, make_scal(1.0, 0.0, 0.0), 0, P->atb ? P->atb : P->w[0]);  // kept: R40
  if (rc) return rc;
  k_max_partials<<<1, 32, 0, P->st>>>(P->part_scal, P->G, P->scratch);
  CKL();
  CK(cudaMemcpyAsync(P->scratch_host, P->scratch, 8, cudaMemcpyDeviceToHost, P->st));
  std::vector<double> hb(P->m);
  CK(cudaMemcpyAsync(hb.data(), P->b, P->m * 8, cudaMemcpyDeviceToHost, P->st));
  CK(cudaStreamSynchronize(P->st));
  P->lambda_max = P->scratch_host[0];
  double nb = 0;
  for (int64_t k = 0; k < P->m; ++k) nb += hb[k] * hb[k];
  P->nb = sqrt(nb);
  P->k1_pending.clear();
  return SSNAL_OK;
}

// §8(f3) peer exchange state: close the peers' IPC mappings, free this rank's region
static void peer_release(ssnal_en_problem* P) {
  for (int q = 0; q < kPeerMaxRanks; ++q)
    if (P->peer_open[q]) {
      cudaIpcCloseMemHandle(P->peer_open[q]);
      P->peer_open[q] = nullptr;
    }
  cudaFree(P->peer_region);
  cudaFree(P->peer_epoch);
  cudaFree(P->peer_idx);
  P->peer_region = nullptr;
  P->peer_epoch = nullptr;
  P->peer_idx = nullptr;
  P->peer = 0;
  P->peer_nranks = 0;
}

static void destroy_bufs(ssnal_en_problem* P) {
  if (!P) return;
  if (P->path_slots) cudaFreeHost(P->path_slots);
  for (auto e : P->path_ev) cudaEventDestroy(e);
  pool_free(P->arena);
  cudaFree(P->Msel);
  if (P->arena_h) cudaFreeHost(P->arena_h);
  drop_graph(P);
  for (int i = 0; i < 3; ++i)
    if (P->cap[i]) cudaStreamDestroy(P->cap[i]);
  for (auto e : P->ev_pool) cudaEventDestroy(e);
  if (P->ev_t0) cudaEventDestroy(P->ev_t0);
  if (P->ev_t1) cudaEventDestroy(P->ev_t1);
  for (auto& pr : P->k1_pending) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  cudaFree(P->xbuf);
  cudaFree(P->rg_dev);
  cudaFree(P->iota);
  if (P->comm_host) cudaFreeHost(P->comm_host);
  peer_release(P);
  drop_path_graph(P);
  if (P->cap_path) cudaStreamDestroy(P->cap_path);
  cudaFree(P->pdev);
  cudaFree(P->path_l);
  if (P->pdev_host) cudaFreeHost(P->pdev_host);
  pool_free(P->A_own);
  pool_free(P->codes_own);
  pool_free(P->tab_own);
  pool_free(P->b_own);
}

static int check_dims(int64_t m, int64_t n) {
  if (m < 2 || m > 1024 || n < 1 || n >= ((int64_t)1 << 31)) {
    set_err("unsupported size m=%lld n=%lld (need 2<=m<=1024, 1<=n<2^31)", (long long)m, (long long)n);
    return SSNAL_EINVAL;
  }
  return SSNAL_OK;
}

int ssnal_en_create(const double* A_colmajor, const double* b, int64_t m, int64_t n, ssnal_en_problem** out) {
  if (!out || !A_colmajor || !b) {
    set_err("null argument");
    return SSNAL_EINVAL;
  }
  *out = nullptr;
  int rc = check_dims(m, n);
  if (rc) return rc;
  ssnal_en_problem* P = new ssnal_en_problem();
  P->m = m;
  P->n = n;
  P->A_own = (double*)pool_alloc((size_t)m * n * 8 + 64);
  P->b_own = (double*)pool_alloc((size_t)m * 8 + 64);
  if (!P->A_own || !P->b_own) {
    set_err("cudaMalloc for A (%zu bytes) failed", (size_t)m * n * 8);
    destroy_bufs(P);
    delete P;
    return SSNAL_ECUDA;
  }
  P->st = nullptr;
  if ((rc = create_prepare(P))) {
    destroy_bufs(P);
    delete P;
    return rc;
  }
  // asynchronous for pinned input (overlaps the graph build in create_common); staged otherwise
  if (cudaMemcpyAsync(P->A_own, A_colmajor, (size_t)m * n * 8, cudaMemcpyHostToDevice, 0) != cudaSuccess ||
      cudaMemcpyAsync(P->b_own, b, (size_t)m * 8, cudaMemcpyHostToDevice, 0) != cudaSuccess) {
    set_err("H2D copy failed");
    destroy_bufs(P);
    delete P;
    return SSNAL_ECUDA;
  }
  P->A = P->A_own;
  P->b = P->b_own;
  P->st = nullptr;
  rc = create_common(P);
  if (rc) {
    destroy_bufs(P);
    delete P;
    return rc;
  }
  *out = P;
  return SSNAL_OK;
}

int ssnal_en_create_device(const double* dA, const double* db, int64_t m, int64_t n, void* cuda_stream,
                           ssnal_en_problem** out) {
  if (!out || !dA || !db) {
    set_err("null argument");
    return SSNAL_EINVAL;
  }
  *out = nullptr;
  int rc = check_dims(m, n);
  if (rc) return rc;
  if (((uintptr_t)dA & 15) != 0) {
    set_err("dA must be 16-byte aligned");
    return SSNAL_EINVAL;
  }
  ssnal_en_problem* P = new ssnal_en_problem();
  P->m = m;
  P->n = n;
  P->A = dA;
  P->b = db;
  P->st = (cudaStream_t)cuda_stream;
  rc = create_common(P);
  if (rc) {
    destroy_bufs(P);
    delete P;
    return rc;
  }
  *out = P;
  return SSNAL_OK;
}

static int geno_common(ssnal_en_problem* P, int64_t stride) {
  if (stride < (P->m + 3) / 4 || stride % 16 != 0) {
    set_err("genotype stride %lld must be a multiple of 16 and >= ceil(m/4)", (long long)stride);
    return SSNAL_EINVAL;
  }
  P->fmt = 1;
  P->cstride = stride;
  return SSNAL_OK;
}

int ssnal_en_create_geno_device(const uint8_t* codes, int64_t stride, const double* tab, const double* db, int64_t m,
                                int64_t n, void* cuda_stream, ssnal_en_problem** out) {
  if (!out || !codes || !tab || !db) {
    set_err("null argument");
    return SSNAL_EINVAL;
  }
  *out = nullptr;
  int rc = check_dims(m, n);
  if (rc) return rc;
  if (((uintptr_t)codes & 15) != 0 || ((uintptr_t)tab & 15) != 0) {
    set_err("codes and tab must be 16-byte aligned");
    return SSNAL_EINVAL;
  }
  ssnal_en_problem* P = new ssnal_en_problem();
  P->m = m;
  P->n = n;
  P->codes = codes;
  P->tab = tab;
  P->b = db;
  P->st = (cudaStream_t)cuda_stream;
  rc = geno_common(P, stride);
  if (!rc) rc = create_common(P);
  if (rc) {
    destroy_bufs(P);
    delete P;
    return rc;
  }
  *out = P;
  return SSNAL_OK;
}

int ssnal_en_create_geno(const uint8_t* codes, int64_t stride, const double* tab, const double* b, int64_t m,
                         int64_t n, ssnal_en_problem** out) {
  if (!out || !codes || !tab || !b) {
    set_err("null argument");
    return SSNAL_EINVAL;
  }
  *out = nullptr;
  int rc = check_dims(m, n);
  if (rc) return rc;
  ssnal_en_problem* P = new ssnal_en_problem();
  P->m = m;
  P->n = n;
  rc = geno_common(P, stride);
  if (rc) {
    delete P;
    return rc;
  }
  P->codes_own = (uint8_t*)pool_alloc((size_t)n * stride + 64);
  P->tab_own = (double*)pool_alloc((size_t)n * 3 * 8 + 64);
  P->b_own = (double*)pool_alloc((size_t)m * 8 + 64);
  if (!P->codes_own || !P->tab_own || !P->b_own) {
    set_err("cudaMalloc for genotype codes failed");
    destroy_bufs(P);
    delete P;
    return SSNAL_ECUDA;
  }
  P->st = nullptr;
  if ((rc = create_prepare(P))) {  // before the upload is enqueued (see create_prepare)
    destroy_bufs(P);
    delete P;
    return rc;
  }
  if (cudaMemcpyAsync(P->codes_own, codes, (size_t)n * stride, cudaMemcpyHostToDevice, 0) != cudaSuccess ||
      cudaMemcpyAsync(P->tab_own, tab, (size_t)n * 3 * 8, cudaMemcpyHostToDevice, 0) != cudaSuccess ||
      cudaMemcpyAsync(P->b_own, b, (size_t)m * 8, cudaMemcpyHostToDevice, 0) != cudaSuccess) {
    set_err("H2D copy failed");
    destroy_bufs(P);
    delete P;
    return SSNAL_ECUDA;
  }
  P->codes = P->codes_own;
  P->tab = P->tab_own;
  P->b = P->b_own;
  P->st = nullptr;
  rc = create_common(P);
  if (rc) {
    destroy_bufs(P);
    delete P;
    return rc;
  }
  *out = P;
  return SSNAL_OK;
}

double ssnal_en_lambda_max_l1(const ssnal_en_problem* p) { return p ? p->lambda_max : NAN; }

int ssnal_en_set_option(ssnal_en_problem* P, const char* key, double v) {
  if (!P || !key) {
    set_err("null argument");
    return SSNAL_EINVAL;
  }
  std::string k(key);
  if (k == "sigma_factor" && v > 1) P->sigma_factor = v;
  else if (k == "sigma_max" && v > 0) P->sigma_max = v;
  else if (k == "mu" && v > 0 && v < 0.5) P->mu = v;
  else if (k == "beta" && v > 0 && v < 1) P->beta = v;
  else if (k == "max_outer" && v >= 1) P->max_outer = (int)v;
  else if (k == "max_inner" && v >= 1) P->max_inner = (int)v;
  else if (k == "max_backtracks" && v >= 0) P->max_bt = (int)v;
  else if (k == "init_mode" && (v == 0 || v == 1)) P->init_mode = (int)v;
  else if (k == "time_k1") {  // also resets the K1 timing accumulators read by get_info("k1_time_s")
    P->time_k1 = v != 0;
    P->k1_time = 0;
    P->k1_count = 0;
  }
  else if (k == "certify" && (v == 0 || v == 1)) P->certify = (int)v;
  else if (k == "graph" && (v == 0 || v == 1)) P->use_graph = (int)v;
  else if (k == "cg_ratio" && v >= 0) {
    if ((v > 0) != (P->cg_ratio > 0)) drop_graph(P);  // the graph holds K6 only when CG can be chosen
    P->cg_ratio = v;
  } else if (k == "cg_threshold" && v >= 0) {
    P->cg_threshold = v;
    drop_graph(P);
  }
  else if (k == "jitter" && v >= 0 && v < 1) P->jitter = v;
  else if (k == "test_fail_factor" && v >= 0) P->inject_fail = (int)v;
  else if (k == "inner_tol_mode" && (v == 0 || v == 1)) P->inner_tol_mode = (int)v;
  else if (k == "carry_sigma" && (v == 0 || v == 1)) P->carry_sigma = (int)v;
  else if (k == "carry_dual" && (v == 0 || v == 1)) P->carry_dual = (int)v;
  else if (k == "reuse_atb" && (v == 0 || v == 1)) P->reuse_atb = (int)v;
  else if (k == "reuse_frac" && v >= 0 && v <= 1) P->reuse_frac = v;
  else if (k == "reuse_psi_only" && (v == 0 || v == 1)) P->reuse_psi_only = (int)v;
  else if (k == "reuse_min_bytes" && v >= 0) P->reuse_min_bytes = (int64_t)v;
  else if (k == "path_graph" && (v == 0 || v == 1)) P->use_path_graph = (int)v;
  else if (k == "warm_dual" && (v == 0 || v == 1)) P->warm_dual = (int)v;
  else if (k == "cg_tol" && v > 0 && v < 1) {
    P->cg_tol = v;
    drop_graph(P);  // baked into the captured CG launch
  } else if (k == "cg_maxit" && v >= 1) {
    P->cg_maxit = (int)v;
    drop_graph(P);
  }
  else if (k == "k1_stages" && v >= 2 && v <= 16 && !P->fmt) {
    // depth of K1's bulk-copy ring (default: as many ~32 KB stages as fit 200 KB, ≤ 8)
    const int S = (int)v;
    const size_t per_stage = (size_t)(P->stage_elems + P->xstage_elems) * 8;
    const size_t smem = (size_t)S * per_stage + 2 * S * 8 + 64 + 4 * S + 16;
    if ((size_t)S * P->stage_elems < (size_t)K1_NWC * P->m + K1_NWC * 4 + K1_NWC || smem > 227 * 1024) {
      set_err("k1_stages=%d does not fit (m=%lld)", S, (long long)P->m);
      return SSNAL_EINVAL;
    }
    P->S = S;
    P->k1_smem = smem;
    drop_graph(P);  // the K1 launch configuration is baked into the graph
  }
  else if (k == "gram_sk_minch" && v >= 1 && v <= 64) {
    P->gsk_minch = (int)v;
    drop_graph(P);
  }
  else if (k == "gram_sk" && (v == 0 || v == 1 || v == 2)) {
    P->use_gram_sk = (int)v;
    drop_graph(P);  // the K3 launch is baked into the graph
  }
  else if (k == "small" && (v == 0 || v == 1))
    P->use_small = (int)v;
  else if (k == "small_cluster" && (v == 0 || v == 1))
    P->use_small_cl = (int)v;
  else if (k == "chol_d2" && (v == 0 || v == 1)) {
    P->use_d2 = (int)v;
    drop_graph(P);  // the K4 variant is baked into the graph
  }
  else if (k == "chol_dsm" && (v == 0 || v == 1)) {
    P->use_dsm = (int)v;
    P->chol_dsm = P->use_dsm && P->dsm_ok;
    drop_graph(P);  // the K4 variant is baked into the graph
  } else if (k == "cluster_size" && (v == 0 || v == 1 || v == 2 || v == 4 || v == 8 || v == 16)) {
    // 0 = auto (16 if schedulable, else the largest smaller power of two); an explicit size the
    // device cannot schedule is refused rather than failing mid-solve
    const int want = v == 0 ? 16 : (int)v;
    const int fit = chol_cluster_fit(P, want);
    if (v != 0 && fit != want) {
      set_err("cluster_size=%g is not schedulable on this device (largest: %d)", v, fit);
      return SSNAL_EINVAL;
    }
    P->cluster = fit;
    drop_graph(P);  // the cluster launch configuration is baked into the graph
  } else {
    set_err("unknown option or bad value: %s=%g", key, v);
    return SSNAL_EINVAL;
  }
  return SSNAL_OK;
}

double ssnal_en_get_info(const ssnal_en_problem* P, const char* key) {
  if (!P || !key) return NAN;
  std::string k(key);
  if (k == "m") return (double)P->m;
  if (k == "n") return (double)P->n;
  if (k == "k1_cols") return P->C;
  if (k == "k1_stages") return P->S;
  if (k == "gram_sk") return P->use_gram_sk;
  if (k == "gram_sk_grid") return P->gsk_grid;
  if (k == "k1_grid") return P->G;
  if (k == "k1_smem") return (double)P->k1_smem;
  if (k == "cluster_size") return P->cluster;
  if (k == "chol_dsm") return P->chol_dsm;
  if (k == "small") return small_eligible(P) ? 1 : 0;
  if (k == "small_cluster") return (small_eligible(P) && P->use_small_cl && P->small_cl_ok) ? 1 : 0;
  if (k == "chol_d2") return P->chol_dsm && P->use_d2 && P->d2_ok;
  if (k == "num_sms") return P->nsm;
  if (k == "graph") return P->use_graph;
  if (k == "format") return P->fmt;
  if (k == "cg_ratio") return P->cg_ratio;
  if (k == "cg_threshold") return P->cg_threshold;
  if (k == "carry_sigma") return P->carry_sigma;
  if (k == "carry_dual") return P->carry_dual;
  if (k == "reuse_atb") return (P->atb && P->reuse_atb) ? 1 : 0;
  if (k == "atb_reuses") return (double)P->atb_reuses;  // cold-start first trials served from Aᵀb (R40)
  if (k == "path_graph") return P->use_path_graph;
  if (k == "warm_dual") return P->warm_dual;
  if (k == "k1_time_s") return P->k1_time;       // Σ K1 launch times timed by the hook calls (option time_k1)
  if (k == "k1_launches") return P->k1_count;
  return NAN;
}

static int solve_wrapped(ssnal_en_problem* P, double l1, double l2, double sigma0, double tol, const double* x0,
                         int x0_dev, double* x_out, int xout_dev, ssnal_en_stats* stats) {
  int rc = check_args(P, l1, l2, sigma0, tol);
  if (rc) return rc;
  auto t0 = std::chrono::steady_clock::now();
  P->launches = 0;
  P->k1_time = 0;
  P->k1_count = 0;
  if (!P->ev_t0) {
    CK(cudaEventCreate(&P->ev_t0));
    CK(cudaEventCreate(&P->ev_t1));
  }
  cudaEvent_t e0 = P->ev_t0, e1 = P->ev_t1;
  CK(cudaEventRecord(e0, P->st));
  if (x0) {
    CK(cudaMemcpyAsync(P->x, x0, P->n * 8, x0_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, P->st));
  }
  int have_x0 = x0 != nullptr;
  if (sharded(P)) {  // warm start iff any rank has an x0 slice (the others count as zero)
    P->comm_host[0] = have_x0;
    CK(cudaMemcpyAsync(P->xbuf, P->comm_host, 8, cudaMemcpyHostToDevice, P->st));
    if ((rc = comm_allreduce(P, P->xbuf, 1, 0))) return rc;
    CK(cudaMemcpyAsync(P->comm_host + 1, P->xbuf, 8, cudaMemcpyDeviceToHost, P->st));
    CK(cudaStreamSynchronize(P->st));
    if (P->comm_host[1] > 0 && !have_x0) CK(cudaMemsetAsync(P->x, 0, P->n * 8, P->st));
    have_x0 = P->comm_host[1] > 0;
  }
  ssnal_en_stats S;
  P->direct_xout = (x_out && xout_dev && x_out != x0) ? x_out : nullptr;
  P->xout_done = false;
  const bool keep = P->warm_dual && have_x0;  // R39: start from the handle's previous (y, w)
  rc = small_eligible(P)                ? solve_small_core(P, l1, l2, sigma0, tol, have_x0, &S, nullptr, keep)
       : (P->use_graph && (!sharded(P) || P->peer)) ? solve_graph_core(P, l1, l2, sigma0, tol, have_x0, &S, nullptr, keep)
                                       : solve_core(P, l1, l2, sigma0, tol, have_x0, &S, keep);
  if (rc == SSNAL_ECUDA || rc == SSNAL_EINVAL) return rc;
  if (x_out && !P->xout_done) {
    CK(cudaMemcpyAsync(x_out, P->x, P->n * 8, xout_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, P->st));
  }
  P->direct_xout = nullptr;
  P->xout_done = false;
  CK(cudaEventRecord(e1, P->st));
  CK(cudaStreamSynchronize(P->st));
  harvest_k1(P);
  if (P->peer && (rc = peer_check(P))) return rc;
  finish_stats(P, &S);
  S.primal_viol = NAN;
  if (P->certify) {  // one extra Aᵀ pass at Ax − b (tmpm holds it from the objective), outside TTS
    const int keep = P->time_k1;
    P->time_k1 = 0;
    rc = launch_k1(P, P->tmpm, nullptr, make_scal(1.0, 0.0, 0.0), 0, P->w[2]);
    P->time_k1 = keep;
    if (rc) return rc;
    const int nb = 2 * P->nsm;  // block maxima into cg_scal (2·nsm + 8 doubles)
    k_kkt_viol<<<nb, 256, 0, P->st>>>(P->n, P->w[2], P->x, P->stat_l1, P->stat_l2, P->cg_scal);
    k_max_reduce<<<1, 32, 0, P->st>>>(P->cg_scal, nb, P->scratch + 40);
    CKL();
    if (sharded(P) && (rc = comm_allreduce(P, P->scratch + 40, 1, 1))) return rc;
    CK(cudaMemcpyAsync(P->scratch_host + 42, P->scratch + 40, 8, cudaMemcpyDeviceToHost, P->st));
    CK(cudaStreamSynchronize(P->st));
    S.primal_viol = P->scratch_host[42];
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  S.time_device_s = ms * 1e-3;
  S.time_total_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  S.kernel_launches = P->launches;
  S.k1_time_s = P->k1_time;
  S.k1_launches = P->k1_count;
  if (stats) *stats = S;
  return S.status;
}

#ifdef SMALL_PROF
int ssnal_en_small_prof(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, ssn::g_small_prof, 8 * sizeof(unsigned long long));
  if (reset) {
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(ssn::g_small_prof, z, sizeof(z));
  }
  return 0;
}
#endif

int ssnal_en_solve(ssnal_en_problem* P, double l1, double l2, double sigma0, double tol, const double* x0,
                   double* x_out, ssnal_en_stats* stats) {
  return solve_wrapped(P, l1, l2, sigma0, tol, x0, 0, x_out, 0, stats);
}

// A warm-started λ path on device buffers: point i starts from point i − 1's solution
// and, with option carry_sigma (default; reading R38), from point i − 1's final σ, so that a nearby
// warm start "usually converges in just one iteration".
// Device-resident control (graph or one-CTA path): every point is enqueued before ONE stream
// synchronisation — per-point results land in pinned slots and are completed afterwards; the
// carried σ moves on the device (ctl.sigma_final → scratch[60] → the next point's ctl.sigma).  Other
// modes (host-driven control, sharded handles, certify) loop over ssnal_en_solve_device.

int ssnal_en_solve_path_device(ssnal_en_problem* P, int64_t npts, const double* lambda1, const double* lambda2,
                               double sigma0, double tol, const double* x0, double* x_out, ssnal_en_stats* stats) {
  if (!P || npts < 1 || !lambda1 || !lambda2 || !x_out) {
    set_err("solve_path: bad arguments");
    return SSNAL_EINVAL;
  }
  const int64_t n = P->n;
  int worst = SSNAL_OK;
  auto fold = [&](int rc) {
    if (rc != SSNAL_OK && worst == SSNAL_OK) worst = rc;
  };
  // peer-attached sharded handles keep the deferred path (their exchanges are kernels); host-callback
  // providers need host-driven control
  const bool deferred = (!sharded(P) || P->peer) && !P->certify && (small_eligible(P) || P->use_graph);
  if (!deferred) {
    double sig = sigma0;
    for (int64_t i = 0; i < npts; ++i) {
      const double* xi = i == 0 ? x0 : x_out + (i - 1) * n;
      ssnal_en_stats st;
      const int keep_wd = P->warm_dual;
      P->warm_dual = (P->carry_dual && i > 0) ? 1 : keep_wd;  // R39 along the path
      const int rc = solve_wrapped(P, lambda1[i], lambda2[i], sig, tol, xi, 1, x_out + i * n, 1, &st);
      P->warm_dual = keep_wd;
      if (rc == SSNAL_EINVAL || rc == SSNAL_ECUDA) return rc;
      if (stats) stats[i] = st;
      fold(rc);
      if (P->carry_sigma) sig = st.sigma_final;
    }
    return worst;
  }
  for (int64_t i = 0; i < npts; ++i) {
    int rc = check_args(P, lambda1[i], lambda2[i], sigma0, tol);
    if (rc) return rc;
  }
  if (P->path_cap < npts) {
    drop_path_graph(P);  // it writes into the slots
    if (P->path_slots) cudaFreeHost(P->path_slots);
    P->path_slots = nullptr;
    P->path_cap = 0;
    CK(cudaHostAlloc(&P->path_slots, sizeof(PathSlot) * npts, cudaHostAllocMapped));  // kernels write results here
    P->path_cap = npts;
  }
  // points 1 … npts − 1 in one launch of the device-resident path graph (unsharded graph mode, the
  // dual carried — reading R39); point 0 runs as a single solve first
  const bool pg = P->use_path_graph && npts > 1 && P->carry_dual && !small_eligible(P) && P->use_graph &&
                  (!sharded(P) || P->peer);
  if (pg) {
    int rc0;
    if ((rc0 = build_graph(P))) return rc0;  // also uploads the K4 output table both graphs read
    PathSlot* slots_dev = nullptr;
    CK(cudaHostGetDevicePointer((void**)&slots_dev, P->path_slots, 0));
    if ((rc0 = build_path_graph(P, slots_dev))) return rc0;
    if (P->path_lcap < npts) {
      cudaFree(P->path_l);
      P->path_l = nullptr;
      P->path_lcap = 0;
      if ((rc0 = alloc((void**)&P->path_l, (size_t)2 * npts * 8))) return rc0;
      P->path_lcap = npts;
    }
  }
  while ((int64_t)P->path_ev.size() < 2 * npts) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    P->path_ev.push_back(e);
  }
  PathSlot* slot = (PathSlot*)P->path_slots;
  DevCtl* ctl0 = P->ctl_host;
  EvalOut* ev0 = P->ev_out_host;
  double* sh0 = P->scratch_host;
  auto t0 = std::chrono::steady_clock::now();
  std::vector<ssnal_en_stats> S(npts);
  std::vector<size_t> k1_beg(npts + 1, 0);  // K1 event pairs (warm-start passes with time_k1) per point
  double* sigma_carry = P->scratch + 60;
  int rc = SSNAL_OK;
  int have0 = x0 != nullptr;
  if (sharded(P)) {  // point 0: warm iff any rank has an x0 slice (the others count as zero)
    P->comm_host[0] = have0;
    CK(cudaMemcpyAsync(P->xbuf, P->comm_host, 8, cudaMemcpyHostToDevice, P->st));
    if ((rc = comm_allreduce(P, P->xbuf, 1, 0))) return rc;
    CK(cudaMemcpyAsync(P->comm_host + 1, P->xbuf, 8, cudaMemcpyDeviceToHost, P->st));
    CK(cudaStreamSynchronize(P->st));
    have0 = P->comm_host[1] > 0;
  }
  for (int64_t i = 0; i < npts && rc == SSNAL_OK; ++i) {  // enqueue every point
    if (pg && i == 1) {  // the rest of the path: one graph launch
      CK(cudaMemcpyAsync(P->path_l, lambda1, npts * 8, cudaMemcpyHostToDevice, P->st));
      CK(cudaMemcpyAsync(P->path_l + P->path_lcap, lambda2, npts * 8, cudaMemcpyHostToDevice, P->st));
      PathDev* pd = P->pdev_host;
      pd->l1s = P->path_l;
      pd->l2s = P->path_l + P->path_lcap;
      pd->xout = x_out;
      pd->i = 1;
      pd->npts = npts;
      pd->carry_sigma = P->carry_sigma;
      pd->t0 = 0;
      DevCtl* h = &pd->tmpl;  // the settings, as solve_graph_core fills them
      memset(h, 0, sizeof(DevCtl));
      h->tol = tol;
      h->sigma = sigma0;
      h->sigma_factor = P->sigma_factor;
      h->sigma_max = P->sigma_max;
      h->mu = P->mu;
      h->beta = P->beta;
      h->max_outer = P->max_outer;
      h->max_inner = P->max_inner;
      h->max_bt = P->max_bt;
      h->cg_ratio = P->cg_ratio;
      h->cg_threshold = P->cg_threshold;
      h->nb = P->nb;
      h->jitter = P->jitter;
      h->inject = P->inject_fail;
      h->inner_tol_mode = P->inner_tol_mode;
      h->tstamp[0] = ~0ull;
      h->tstamp[1] = 0ull;
      CK(cudaMemcpyAsync(P->pdev, pd, sizeof(PathDev), cudaMemcpyHostToDevice, P->st));
      CK(cudaGraphLaunch(P->pgexec, P->st));
      for (int64_t q = 1; q < npts; ++q) {
        slot[q].l1 = lambda1[q];
        slot[q].l2 = lambda2[q];
        slot[q].warm_pass = 0;  // R39: no warm-start pass
        slot[q].pad = 0;        // the path graph embeds the plain solve body
        slot[q].launches = P->pgraph_fixed;
        k1_beg[q] = P->k1_pending.size();
      }
      break;
    }
    P->ctl_host = &slot[i].ctl;
    P->ev_out_host = &slot[i].ev;
    P->scratch_host = slot[i].scratch;
    P->launches = 0;
    k1_beg[i] = P->k1_pending.size();
    CK(cudaEventRecord(P->path_ev[2 * i], P->st));
    const double* xi = i == 0 ? x0 : x_out + (i - 1) * n;
    const bool keep = P->carry_dual && i > 0;  // R39: the previous point's final (x, y, w) and support
    if (xi && !keep) CK(cudaMemcpyAsync(P->x, xi, n * 8, cudaMemcpyDeviceToDevice, P->st));
    else if (i == 0 && have0 && !xi) CK(cudaMemsetAsync(P->x, 0, n * 8, P->st));  // sharded: no slice here
    const int warm = i == 0 ? have0 : 1;
    const double* sig_in = (P->carry_sigma && i > 0) ? sigma_carry : nullptr;
    P->direct_xout = x_out + i * n;
    P->xout_done = false;
    rc = small_eligible(P) ? solve_small_core(P, lambda1[i], lambda2[i], sigma0, tol, warm, &S[i], sig_in, keep, keep)
                           : solve_graph_core(P, lambda1[i], lambda2[i], sigma0, tol, warm, &S[i], sig_in, keep, keep);
    if (rc == SSNAL_OK && P->carry_sigma)
      CK(cudaMemcpyAsync(sigma_carry, &P->ctl->sigma_final, 8, cudaMemcpyDeviceToDevice, P->st));
    if (rc == SSNAL_OK && !P->xout_done) CK(cudaMemcpyAsync(x_out + i * n, P->x, n * 8, cudaMemcpyDeviceToDevice, P->st));
    P->direct_xout = nullptr;
    P->xout_done = false;
    CK(cudaEventRecord(P->path_ev[2 * i + 1], P->st));
    slot[i].l1 = P->stat_l1;
    slot[i].l2 = P->stat_l2;
    slot[i].warm_pass = P->stat_warm_pass;
    slot[i].pad = P->stat_graph_r ? 1 : 0;
    slot[i].launches = P->launches;
  }
  k1_beg[npts] = P->k1_pending.size();
  P->ctl_host = ctl0;
  P->ev_out_host = ev0;
  P->scratch_host = sh0;
  CK(cudaStreamSynchronize(P->st));
  // K1 launches timed by events (the warm-start passes) belong to the point that enqueued them
  std::vector<double> k1_t(npts, 0.0);
  std::vector<int> k1_c(npts, 0);
  for (int64_t i = 0; i < npts; ++i)
    for (size_t q = k1_beg[i]; q < k1_beg[i + 1] && q < P->k1_pending.size(); ++q) {
      float ms = 0;
      cudaEventElapsedTime(&ms, P->k1_pending[q].first, P->k1_pending[q].second);
      k1_t[i] += ms * 1e-3;
      k1_c[i]++;
    }
  for (auto& pr : P->k1_pending) {
    P->ev_pool.push_back(pr.first);
    P->ev_pool.push_back(pr.second);
  }
  P->k1_pending.clear();
  if (rc != SSNAL_OK) return rc;
  if (P->peer && (rc = peer_check(P))) return rc;
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (int64_t i = 0; i < npts; ++i) {  // complete the statistics point by point
    P->ctl_host = &slot[i].ctl;
    P->ev_out_host = &slot[i].ev;
    P->scratch_host = slot[i].scratch;
    P->stat_l1 = slot[i].l1;
    P->stat_l2 = slot[i].l2;
    P->stat_warm_pass = slot[i].warm_pass;
    P->stat_graph_r = slot[i].pad != 0;
    P->launches = slot[i].launches;
    P->k1_time = k1_t[i];
    P->k1_count = k1_c[i];
    P->graph_pending = true;
    finish_stats(P, &S[i]);
    S[i].primal_viol = NAN;
    float ms = 0;
    if (pg && i > 0) {  // in-kernel stamps of the path graph (events cannot sit inside its loop)
      ms = (float)((double)(slot[i].t1 - slot[i].t0) * 1e-6);
    } else {
      cudaEventElapsedTime(&ms, P->path_ev[2 * i], P->path_ev[2 * i + 1]);
    }
    S[i].time_device_s = ms * 1e-3;
    S[i].time_total_s = wall / npts;  // the host time of the whole path, shared evenly
    S[i].kernel_launches = P->launches;
    S[i].k1_time_s = P->k1_time;
    S[i].k1_launches = P->k1_count;
    if (stats) stats[i] = S[i];
    fold(S[i].status);
  }
  P->ctl_host = ctl0;
  P->ev_out_host = ev0;
  P->scratch_host = sh0;
  return worst;
}

int ssnal_en_solve_device(ssnal_en_problem* P, double l1, double l2, double sigma0, double tol, const double* x0,
                          double* x_out, ssnal_en_stats* stats) {
  return solve_wrapped(P, l1, l2, sigma0, tol, x0, 1, x_out, 1, stats);
}

int ssnal_en_aty_fused(ssnal_en_problem* P, const double* y, const double* x, double sigma, double l1, double l2,
                       double* w_out, int32_t* J_out, double* PJ_out, int64_t* r_out, double partials_out[4],
                       double* grad_out) {
  if (!P || !y || !x || !w_out || !J_out || !PJ_out || !(sigma > 0)) {
    set_err("invalid argument");
    return SSNAL_EINVAL;
  }
  P->launches = 0;
  const Scal sc = make_scal(sigma, l1, l2);
  int rc = launch_k1(P, y, x, sc, 1, w_out);
  if (rc) return rc;
  rc = launch_finalize(P, J_out, PJ_out, P->r_dev + 3);
  if (rc) return rc;
  rc = launch_eval(P, y, sc, grad_out != nullptr, P->cta_cnt, P->G, grad_out ? grad_out : P->tmpm, P->r_dev + 3, 3);
  if (rc) return rc;
  EvalOut e;
  rc = fetch_eval(P, 3, &e);
  if (rc) return rc;
  harvest_k1(P);  // option time_k1: the K1 launch's own event time (get_info "k1_time_s")
  if (r_out) *r_out = e.r;
  if (partials_out)
    for (int j = 0; j < 4; ++j) partials_out[j] = e.s[j];
  return SSNAL_OK;
}

int ssnal_en_epilogue(ssnal_en_problem* P, const double* w0, const double* w1, double s, const double* x,
                      double sigma, double l1, double l2, double* w_out, int32_t* J_out, double* PJ_out,
                      int64_t* r_out, double partials_out[4]) {
  if (!P || !w0 || !x || !J_out || !PJ_out || !(sigma > 0)) {
    set_err("invalid argument");
    return SSNAL_EINVAL;
  }
  const Scal sc = make_scal(sigma, l1, l2);
  int rc = launch_k1e(P, w0, w1, s, x, sc, w_out);
  if (rc) return rc;
  rc = launch_finalize(P, J_out, PJ_out, P->r_dev + 3);
  if (rc) return rc;
  rc = launch_eval(P, P->b, sc, 0, nullptr, 0, nullptr, P->r_dev + 3, 3);
  if (rc) return rc;
  EvalOut e;
  rc = fetch_eval(P, 3, &e);
  if (rc) return rc;
  if (r_out) *r_out = e.r;
  if (partials_out)
    for (int j = 0; j < 4; ++j) partials_out[j] = e.s[j];
  return SSNAL_OK;
}

int ssnal_en_newton_direction(ssnal_en_problem* P, const int32_t* J, int64_t r, const double* g, double kappa,
                              double* d_out, double* gd_out, int32_t* branch_out) {
  if (P && sharded(P)) {
    set_err("not available on a column-sharded handle");
    return SSNAL_EINVAL;
  }
  if (!P || (r > 0 && !J) || !g || !d_out || !(kappa > 0) || r < 0 || r > P->n) {
    set_err("invalid argument");
    return SSNAL_EINVAL;
  }
  int br = 0, info = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {  // a failed factor is retried once with the jitter (R36)
    int rc = newton_direction(P, J, r, g, kappa, d_out, P->scratch, &br, nullptr, nullptr, attempt ? P->jitter : 0.0);
    if (rc) return rc;
    CK(cudaMemcpyAsync(P->scratch_host, P->scratch, 8, cudaMemcpyDeviceToHost, P->st));
    CK(cudaMemcpyAsync(P->scratch_host + 1, P->info, 4, cudaMemcpyDeviceToHost, P->st));
    CK(cudaStreamSynchronize(P->st));
    memcpy(&info, P->scratch_host + 1, 4);
    if (!((br == 1 || br == 2) && info) || !(P->jitter > 0.0)) break;
  }
  if (gd_out) *gd_out = P->scratch_host[0];
  if (branch_out) *branch_out = br;
  if ((br == 1 || br == 2) && info) {
    set_err("Cholesky pivot not positive");
    return SSNAL_ENUMERIC;
  }
  return SSNAL_OK;
}

// Section 3.3: ν, OLS de-biasing, rss, GCV, e-BIC for the latest solution.
int ssnal_en_model_select(ssnal_en_problem* P, double l2, double* xdb_out, ssnal_en_criteria* out) {
  if (P && sharded(P)) {
    set_err("not available on a column-sharded handle");
    return SSNAL_EINVAL;
  }
  if (!P || !out || !(l2 >= 0)) {
    set_err("invalid argument");
    return SSNAL_EINVAL;
  }
  const int64_t m = P->m, n = P->n;
  CK(cudaMemcpyAsync(P->scratch_host, P->r_dev + 2, 8, cudaMemcpyDeviceToHost, P->st));
  CK(cudaStreamSynchronize(P->st));
  int64_t r;
  memcpy(&r, P->scratch_host, 8);
  if (!P->Msel) {
    int rc = alloc((void**)&P->Msel, (size_t)2 * m * m * 8 + 64);
    if (rc) return rc;
  }
  auto splits = [&](int tiles, int64_t K) { return gram_splits(P->nsm, tiles, K, P->W_splits); };
  int* info_nu = P->info + 2;
  int* info_ols = P->info + 3;
  CK(cudaMemsetAsync(P->info + 2, 0, 2 * sizeof(int), P->st));
  double* frob = P->scratch + 24;
  double* crit = P->scratch + 28;
  const int32_t* J = P->Jx;
  int rc;
  int ident = 0;
  bool ols_possible = false;
  if (r == 0) {
    CK(cudaMemsetAsync(frob, 0, 8, P->st));
  } else if (r < m) {
    // ν: factor A_JᵀA_J + λ2 I with A_J appended as m rows: ν = ‖A_J L⁻ᵀ‖_F²
    const int N = (int)r, NR = (int)(r + m);
    const int tiles = gram_tiles(N), ns = splits(tiles, m);
    with_acc(P, [&](auto acc) {
      k_gram<true><<<gram_grid(P, tiles * ns), 256, 0, P->st>>>(acc, m, J, r, P->W, nullptr, tiles, ns, nullptr);
      return 0;
    });
    k_gram_reduce<<<reduce_grid(P, r * r), 256, 0, P->st>>>(P->W, ns, r, r, l2, 1.0, P->Msel, NR, nullptr, nullptr, 0, 0.0);
    with_acc(P, [&](auto acc) {
      k_fill_rows<<<(unsigned)((m * r + 255) / 256), 256, 0, P->st>>>(P->Msel, NR, r, acc, m, J, r, 0);
      return 0;
    });
    P->launches += 3;
    CKL();
    if ((rc = launch_chol_ex(P, P->Msel, N, NR, NR, nullptr, 1.0, nullptr, nullptr, nullptr, nullptr, info_nu)))
      return rc;
    k_frob<<<1, 1024, 0, P->st>>>(P->Msel, NR, r, m, r, frob);
    // OLS de-biasing: factor A_JᵀA_J with rhs row A_Jᵀb; v → P->u
    const int64_t nout = r + 1;
    const int tiles2 = gram_tiles(nout), ns2 = splits(tiles2, m);
    with_acc(P, [&](auto acc) {
      k_gram<true><<<gram_grid(P, tiles2 * ns2), 256, 0, P->st>>>(acc, m, J, r, P->W, P->b, tiles2, ns2, nullptr);
      return 0;
    });
    k_gram_reduce<<<reduce_grid(P, nout * nout), 256, 0, P->st>>>(P->W, ns2, nout, r, 0.0, 1.0, P->Mmat, N + 1, nullptr,
                                                                  nullptr, 0, 0.0);
    P->launches += 3;
    CKL();
    if ((rc = launch_chol_ex(P, P->Mmat, N, N + 1, N + 1, P->u, 1.0, nullptr, nullptr, nullptr, nullptr, info_ols)))
      return rc;
    int grid = 0;
    if ((rc = launch_gather(P, J, P->u, r, &grid))) return rc;
    k_combine<<<1, 1024, 0, P->st>>>(m, P->b, -1.0, P->part_vec, grid, P->tmpm, nullptr, nullptr,
                                     nullptr);  // A_J v − b
    P->launches++;
    CKL();
    ols_possible = true;
  } else {
    // r ≥ m: ν = tr(K (K + λ2 I)⁻¹), K = A_J A_Jᵀ, = m − λ2 ‖L⁻¹‖_F² with I_m appended
    const int N = (int)m, NR = (int)(2 * m);
    const int tiles = gram_tiles(m), ns = splits(tiles, r);
    with_acc(P, [&](auto acc) {
      k_gram<false><<<gram_grid(P, tiles * ns), 256, 0, P->st>>>(acc, m, J, r, P->W, nullptr, tiles, ns, nullptr);
      return 0;
    });
    k_gram_reduce<<<reduce_grid(P, m * m), 256, 0, P->st>>>(P->W, ns, m, m, l2, 1.0, P->Msel, NR, nullptr, nullptr, 0, 0.0);
    with_acc(P, [&](auto acc) {
      k_fill_rows<<<(unsigned)((m * m + 255) / 256), 256, 0, P->st>>>(P->Msel, NR, m, acc, m, J, m, 1);
      return 0;
    });
    P->launches += 3;
    CKL();
    if ((rc = launch_chol_ex(P, P->Msel, N, NR, NR, nullptr, 1.0, nullptr, nullptr, nullptr, nullptr, info_nu)))
      return rc;
    k_frob<<<1, 1024, 0, P->st>>>(P->Msel, NR, m, m, m, frob);
    ident = 1;
  }
  if (r == 0) {  // x_ols = 0: residual = −b
    k_combine<<<1, 1024, 0, P->st>>>(m, P->b, -1.0, P->part_vec, 0, P->tmpm, nullptr, nullptr, nullptr);
    CK(cudaMemsetAsync(info_ols, 0, sizeof(int), P->st));
    ols_possible = true;
  }
  k_criteria<<<1, 1024, 0, P->st>>>(frob, ident, l2, P->tmpm, m, n, ols_possible ? info_ols : nullptr, crit);
  P->launches += 2;
  CKL();
  CK(cudaMemcpyAsync(P->scratch_host + 28, crit, 4 * 8, cudaMemcpyDeviceToHost, P->st));
  CK(cudaMemcpyAsync(P->scratch_host + 32, P->info + 2, 2 * sizeof(int), cudaMemcpyDeviceToHost, P->st));
  if (xdb_out) {
    CK(cudaMemsetAsync(P->w[2], 0, n * 8, P->st));
    if (ols_possible && r > 0) {
      k_scatter<<<(unsigned)((r + 255) / 256), 256, 0, P->st>>>(J, P->u, r, P->w[2]);
      CKL();
    }
    CK(cudaMemcpyAsync(xdb_out, P->w[2], n * 8, cudaMemcpyDeviceToHost, P->st));
  }
  CK(cudaStreamSynchronize(P->st));
  const double* c = P->scratch_host + 28;
  int infos[2];
  memcpy(infos, P->scratch_host + 32, 8);
  out->active = r;
  out->nu = c[0];
  out->rss = c[1];
  out->gcv = c[2];
  out->ebic = c[3];
  out->ols_ok = (ols_possible && infos[1] == 0) ? 1 : 0;
  out->reserved = 0;
  if (infos[0] != 0) {
    set_err("degrees-of-freedom factorisation not positive definite");
    return SSNAL_ENUMERIC;
  }
  return SSNAL_OK;
}

// ‖A x − b‖² for an external x: support of x by K1e (w = 0, σ = 1, λ = 0 selects x ≠ 0 with P = x)
// into the trial set (J[1], PJ[1], r_dev[3]) — free outside a solve — then K2 + combine + norm.
static int residual_impl(ssnal_en_problem* P, const double* x, int x_dev, double* rss_out) {
  if (P && sharded(P)) {
    set_err("not available on a column-sharded handle");
    return SSNAL_EINVAL;
  }
  if (!P || !x || !rss_out) {
    set_err("null argument");
    return SSNAL_EINVAL;
  }
  const int64_t n = P->n;
  int rc;
  CK(cudaMemcpyAsync(P->w[1], x, n * 8, x_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, P->st));
  CK(cudaMemsetAsync(P->w[2], 0, n * 8, P->st));
  if ((rc = launch_k1e(P, P->w[2], nullptr, 0.0, P->w[1], make_scal(1.0, 0.0, 0.0), nullptr))) return rc;
  if ((rc = launch_finalize(P, P->J[1], P->PJ[1], P->r_dev + 3))) return rc;
  if ((rc = launch_gather_dev(P, P->J[1], P->PJ[1], P->r_dev + 3))) return rc;
  k_combine<<<1, 1024, 0, P->st>>>(P->m, P->b, -1.0, P->part_vec, kGatherDevGrid, P->tmpm, nullptr, nullptr,
                                   P->gax_valid);
  k_objective<<<1, 1024, 0, P->st>>>(P->m, P->tmpm, P->PJ[1], P->r_dev + 3, P->scratch + 36);
  CKL();
  CK(cudaMemcpyAsync(P->scratch_host + 36, P->scratch + 36, 8, cudaMemcpyDeviceToHost, P->st));
  CK(cudaStreamSynchronize(P->st));
  *rss_out = 2.0 * P->scratch_host[36];  // k_objective reports ½‖resid‖²
  return SSNAL_OK;
}

int ssnal_en_residual(ssnal_en_problem* P, const double* x, double* rss_out) { return residual_impl(P, x, 0, rss_out); }

int ssnal_en_residual_device(ssnal_en_problem* P, const double* x, double* rss_out) {
  return residual_impl(P, x, 1, rss_out);
}

// Buffers of a sharded handle and the rank bookkeeping (both exchange providers)
static int comm_setup(ssnal_en_problem* P, int rank, int nranks) {
  const int64_t m = P->m;
  if (!P->xbuf) {
    int rc;
    if ((rc = alloc((void**)&P->xbuf, (size_t)(m * m + 2 * m + 64 + nranks) * 8))) return rc;
    if ((rc = alloc((void**)&P->rg_dev, 64))) return rc;
    if ((rc = alloc((void**)&P->iota, (size_t)(m + 1) * 4))) return rc;
  }
  if (P->comm_host) cudaFreeHost(P->comm_host);
  P->comm_host = nullptr;
  CK(cudaHostAlloc((void**)&P->comm_host, (size_t)(nranks + 16) * 8, cudaHostAllocDefault));
  P->comm_rank = rank;
  P->comm_size = nranks;
  CK(cudaFuncSetAttribute(k_prereduce16, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));  // 16-CTA clusters
  CK(cudaFuncSetAttribute(k_peer_eval, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  k_iota<<<1, 1024, 0, P->st>>>(P->iota, m);
  CKL();
  drop_graph(P);  // the graph's evaluations and directions depend on the exchange provider
  return SSNAL_OK;
}

// λmax = max over the ranks of the local ‖A_qᵀb‖∞ (the first exchange of a sharded handle)
static int comm_lambda_max(ssnal_en_problem* P) {
  P->comm_host[0] = P->lambda_max;
  CK(cudaMemcpyAsync(P->xbuf, P->comm_host, 8, cudaMemcpyHostToDevice, P->st));
  int rc = comm_allreduce(P, P->xbuf, 1, 1);
  if (rc) return rc;
  CK(cudaMemcpyAsync(P->comm_host + 1, P->xbuf, 8, cudaMemcpyDeviceToHost, P->st));
  CK(cudaStreamSynchronize(P->st));
  if (P->peer && (rc = peer_check(P))) return rc;
  P->lambda_max = P->comm_host[1];
  return SSNAL_OK;
}

int ssnal_en_peer_export(ssnal_en_problem* P, int nranks, void* handle_out) {
  if (!P || !handle_out || nranks < 1 || nranks > kPeerMaxRanks) {
    set_err("invalid argument (nranks must be in [1, %d])", kPeerMaxRanks);
    return SSNAL_EINVAL;
  }
  peer_release(P);
  const int64_t m = P->m;
  const int64_t ss = (m + 16 + kPeerMaxRanks + 31) / 32 * 32;  // an evaluation record, counts, scalars
  const int64_t ccap = m < 8 ? 8 : m;                           // gathered columns per rank (r_q < m)
  const int64_t sb = ccap * m;                                  // ≥ m² (partial Gram)
  const size_t bytes = (size_t)peer_region_bytes(nranks, ss, sb);
  CK(cudaMalloc((void**)&P->peer_region, bytes));  // not the stream-ordered pool: IPC-exportable
  CK(cudaMemset(P->peer_region, 0, bytes));        // flags = 0 before any peer can write
  CK(cudaMalloc((void**)&P->peer_epoch, 64));
  CK(cudaMemset(P->peer_epoch, 0, 64));
  CK(cudaMalloc((void**)&P->peer_idx, (size_t)(m + 1) * 4));
  CK(cudaDeviceSynchronize());
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, P->peer_region));
  static_assert(sizeof(cudaIpcMemHandle_t) == SSNAL_EN_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof(h));
  P->peer_nranks = nranks;
  P->pc = PeerComm{};
  P->pc.size = nranks;
  P->pc.ss = ss;
  P->pc.sb = sb;
  P->pc.ccap = ccap;
  return SSNAL_OK;
}

int ssnal_en_peer_attach(ssnal_en_problem* P, int rank, int nranks, const void* handles) {
  if (!P || !handles || !P->peer_region || nranks != P->peer_nranks || rank < 0 || rank >= nranks) {
    set_err("invalid argument (call ssnal_en_peer_export with the same nranks first)");
    return SSNAL_EINVAL;
  }
  const char* hb = (const char*)handles;
  for (int q = 0; q < nranks; ++q) {
    if (q == rank) {
      P->pc.base[q] = P->peer_region;
      continue;
    }
    if (P->peer_open[q]) {
      cudaIpcCloseMemHandle(P->peer_open[q]);
      P->peer_open[q] = nullptr;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, hb + (size_t)q * SSNAL_EN_IPC_HANDLE_BYTES, sizeof(h));
    void* ptr = nullptr;
    CK(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    P->peer_open[q] = (char*)ptr;
    P->pc.base[q] = (char*)ptr;
  }
  P->pc.rank = rank;
  P->pc.epoch = P->peer_epoch;
  P->pc.ticket = (unsigned*)(P->peer_epoch + 1);
  P->pc.err = (int*)(P->peer_epoch + 1) + 1;
  int rc = comm_setup(P, rank, nranks);
  if (rc) return rc;
  P->comm_fn = nullptr;
  P->comm_ctx = nullptr;
  P->peer = 1;
  return comm_lambda_max(P);
}

int ssnal_en_peer_selftest(int nranks, int iters, int64_t count, int64_t* mismatch_out, double* small_out,
                           double* big_out) {
  if (nranks < 1 || nranks > kPeerMaxRanks || iters < 1 || count < 1 || count > 65536 || !mismatch_out) {
    set_err("invalid argument");
    return SSNAL_EINVAL;
  }
  const int64_t ss = (count + 31) / 32 * 32;
  const size_t rb = ((size_t)peer_region_bytes(nranks, ss, ss) + 255) / 256 * 256;
  char* all = nullptr;
  char** bases = nullptr;
  unsigned long long* ep = nullptr;
  int *errs = nullptr, *mis = nullptr;
  double *ls = nullptr, *lb = nullptr;
  int rc = SSNAL_OK;
  auto fail = [&](const char* what, cudaError_t e) {
    set_err("peer selftest: %s: %s", what, cudaGetErrorString(e));
    rc = SSNAL_ECUDA;
  };
  cudaError_t e;
  if ((e = cudaMalloc((void**)&all, rb * nranks)) != cudaSuccess) fail("alloc", e);
  if (!rc && (e = cudaMalloc((void**)&bases, kPeerMaxRanks * sizeof(char*))) != cudaSuccess) fail("alloc", e);
  if (!rc && (e = cudaMalloc((void**)&ep, kPeerMaxRanks * 8 + 2 * kPeerMaxRanks * 4 + 64)) != cudaSuccess)
    fail("alloc", e);
  if (!rc && (e = cudaMalloc((void**)&ls, (size_t)2 * nranks * count * 8)) != cudaSuccess) fail("alloc", e);
  if (!rc) {
    errs = (int*)(ep + kPeerMaxRanks);
    mis = errs + kPeerMaxRanks;
    lb = ls + (size_t)nranks * count;
    std::vector<char*> hb(kPeerMaxRanks, nullptr);
    for (int q = 0; q < nranks; ++q) hb[q] = all + (size_t)q * rb;
    cudaMemset(all, 0, rb * nranks);
    cudaMemset(ep, 0, kPeerMaxRanks * 8 + 2 * kPeerMaxRanks * 4 + 64);
    cudaMemcpy(bases, hb.data(), kPeerMaxRanks * sizeof(char*), cudaMemcpyHostToDevice);
    PeerComm proto{};
    proto.size = nranks;
    proto.ss = ss;
    proto.sb = ss;
    proto.ccap = 1;
    char* const* cb = bases;
    void* args[] = {&proto, (void*)&cb, &iters, &count, &ep, &errs, &mis, &ls, &lb};
    if ((e = cudaLaunchCooperativeKernel((const void*)k_peer_emulate, dim3(nranks), dim3(256), args, 0, 0)) !=
        cudaSuccess)
      fail("launch", e);
    else if ((e = cudaDeviceSynchronize()) != cudaSuccess)
      fail("run", e);
  }
  if (!rc) {
    int herr[kPeerMaxRanks + 1];
    cudaMemcpy(herr, errs, (kPeerMaxRanks + 1) * 4, cudaMemcpyDeviceToHost);
    *mismatch_out = herr[kPeerMaxRanks];
    for (int q = 0; q < nranks; ++q)
      if (herr[q]) {
        set_err("peer selftest: rank %d timed out", q);
        rc = SSNAL_ECUDA;
      }
    if (small_out) cudaMemcpy(small_out, ls, (size_t)nranks * count * 8, cudaMemcpyDeviceToHost);
    if (big_out) cudaMemcpy(big_out, lb, (size_t)nranks * count * 8, cudaMemcpyDeviceToHost);
  }
  cudaFree(all);
  cudaFree(bases);
  cudaFree(ep);
  cudaFree(ls);
  return rc;
}

int ssnal_en_set_comm(ssnal_en_problem* P, ssnal_en_allreduce_fn fn, void* ctx, int rank, int nranks) {
  if (!P || !fn || nranks < 1 || rank < 0 || rank >= nranks) {
    set_err("invalid argument");
    return SSNAL_EINVAL;
  }
  peer_release(P);
  int rc = comm_setup(P, rank, nranks);
  if (rc) return rc;
  P->comm_fn = fn;
  P->comm_ctx = ctx;
  return comm_lambda_max(P);
}

void ssnal_en_destroy(ssnal_en_problem* P) {
  if (!P) return;
  if (P->st) cudaStreamSynchronize(P->st);
  else cudaDeviceSynchronize();
  destroy_bufs(P);
  delete P;
}

}  // extern "C"
