/*
 * ssnal_en.h — C ABI of the B200 (sm_100a) SsNAL-EN hot path.
 *
 * Solves the Elastic Net  min_x ½‖Ax − b‖² + λ1‖x‖₁ + (λ2/2)‖x‖²   (Eq. (1))
 * with the Semi-smooth Newton Augmented Lagrangian method of arXiv 2006.03970:
 * Algorithm 1, ψ from Prop. 2, ∇ψ Eq. (15),
 * the generalized Hessian V = I + κ A_J A_Jᵀ Eq. (16)-(18), the
 * Sherman–Morrison–Woodbury form Eq. (19), Armijo line search Eq. (13)
 * (μ = 0.2 at P:497), KKT residuals Eq. (20), σ ← 5σ.
 * Readings of garbled / silent passages are listed in DESIGN.md ("Readings").
 * A is either fp64 column-major (ssnal_en_create*) or packed 2-bit genotype codes with
 * per-column tables (ssnal_en_create_geno*).
 *
 * Conventions (all entry points):
 *   - fp64 throughout; A is column-major m × n with lda = m (column i = A + i*m).
 *   - "host" pointers are ordinary CPU memory; "device" pointers are CUDA device memory
 *     on the handle's device (e.g. torch.Tensor.data_ptr()).
 *   - Functions return an SSNAL_* status; on failure a thread-local message is
 *     available from ssnal_en_last_error().  No function falls back to the CPU.
 *   - One solve in flight per handle; different handles are independent.
 *   - Limits of this build: 2 ≤ m ≤ 1024, 1 ≤ n < 2^31.
 */
#ifndef SSNAL_EN_H
#define SSNAL_EN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SSNAL_OK = 0,            /* converged (solve) / success                               */
  SSNAL_NOT_CONVERGED = 1, /* iteration cap hit; x_out and stats are still written      */
  SSNAL_EINVAL = 2,        /* bad argument (sizes, NaN/Inf, zero column, λ, σ0, tol …)   */
  SSNAL_ECUDA = 3,         /* CUDA error or out of device memory                        */
  SSNAL_ENUMERIC = 4       /* non-positive Cholesky pivot or NaN in an iterate          */
};

typedef struct ssnal_en_problem ssnal_en_problem; /* opaque handle */

/* Bytes of one exported exchange-region handle (a cudaIpcMemHandle_t), ssnal_en_peer_export. */
#define SSNAL_EN_IPC_HANDLE_BYTES 64

/* Caller-supplied all-reduce for column-sharded handles (see ssnal_en_set_comm). */
typedef int (*ssnal_en_allreduce_fn)(void* ctx, double* buf, int64_t count, int op, void* stream);

typedef struct {
  int32_t status;          /* SSNAL_OK / SSNAL_NOT_CONVERGED / SSNAL_ENUMERIC            */
  int32_t outer_iters;     /* augmented-Lagrangian iterations (the paper's "(k)", R23)   */
  int32_t newton_iters;    /* semi-smooth Newton steps, summed over outer iterations      */
  int32_t psi_evals;       /* ψ evaluations (Armijo trials incl. backtracks)              */
  int32_t backtracks;      /* step halvings                                               */
  int32_t aty_passes;      /* Aᵀy products at new points (K1 launches); with reuse_atb=1 a cold
                              solve's trials at y = −b read Aᵀb kept by create instead of A */
  int32_t branch_steps[4]; /* Newton steps with r = 0, 0 < r < m (Eq. 19), r ≥ m (Eq. 18), CG (R32) */
  int32_t line_search_stalled; /* max_backtracks reached at least once (R30)              */
  int32_t cg_iters;        /* conjugate-gradient iterations, summed over CG steps             */
  int64_t active;          /* nnz(x) at return                                            */
  double res_kkt1;         /* ‖y + b − Ax‖/(1 + ‖b‖) at the last evaluation, Eq. (20)    */
  double res_kkt3;         /* ‖Aᵀy + z‖/(1 + ‖y‖ + ‖z‖) at the last outer step, Eq. (20) */
  double primal_obj;       /* F(x), Eq. (1)                                               */
  double dual_obj;         /* −h*(y) − p*(Aᵀy) at the final y (NaN if λ2 = 0)             */
  double gap;              /* primal_obj − dual_obj ≥ 0                                   */
  double sigma_final;      /* σ of the last inner solve                                   */
  double time_device_s;    /* CUDA-event time of the solve on the handle's stream         */
  double time_total_s;     /* host wall time of the call, copies included                 */
  int64_t kernel_launches; /* kernels launched by this call                              */
  double k1_time_s;        /* Σ device time of K1 launches (option time_k1 = 1), else 0   */
  int32_t k1_launches;     /* K1 launches timed                                           */
  int32_t jitter_retries;  /* Newton steps whose factor was redone with the jitter (R36) */
  double primal_viol;      /* option certify=1: max_i v_i of the KKT inclusion c = Aᵀ(b − Ax) − λ2x ∈
                              λ1∂‖x‖₁ over ALL n columns (v_i = |c_i − λ1 sign x_i| on the support, else
                              (|c_i| − λ1)₊); one extra Aᵀ pass after the solve, outside time_device_s.
                              NaN when certify = 0. */
} ssnal_en_stats;

/* Copy A (host, column-major m × n) and b (host, m) to the current device; the handle owns
 * the copies (caller may free its buffers).  Also computes λmax = ‖Aᵀb‖∞
 * with one fused pass.  EINVAL: m < 2, m > 1024, n < 1, NaN/Inf or an all-zero column. */
int ssnal_en_create(const double* A_colmajor, const double* b, int64_t m, int64_t n, ssnal_en_problem** out);

/* Borrow device buffers dA (column-major, 16-byte aligned) and db; the caller keeps them
 * alive until ssnal_en_destroy.  cuda_stream (cudaStream_t, may be NULL = legacy default)
 * is used for every launch.  Inputs are validated on the device (NaN/Inf, zero columns). */
int ssnal_en_create_device(const double* dA, const double* db, int64_t m, int64_t n, void* cuda_stream,
                           ssnal_en_problem** out);

/* Compressed genotype storage (not in the paper): A given as 2-bit codes
 * g ∈ {0, 1, 2} with a per-column table, a_kj = tab[3j + g_kj] (e.g. the standardised value
 * (g − mean_j)/sd_j, which synth/ computes bit-exactly with its fp64 design).  Column j is
 * `stride` bytes at codes + j·stride (stride a multiple of 16, ≥ ceil(m/4)); row k lives in
 * bits 2(k mod 4)..2(k mod 4)+1 of byte k/4, padding bits zero.  K1 streams 32× fewer bytes
 * than fp64; every other kernel decodes the columns it touches.  Everything else (options,
 * solve, hooks, model selection) is as for the fp64 handle.
 *   _device: codes, tab, db are device pointers borrowed until destroy (codes 16-B aligned).
 *   host:    copies codes (n·stride bytes), tab (3n doubles) and b to the device.
 * EINVAL: bad sizes/stride, a code of value 3, a non-finite table entry or b, or a column
 * whose decoded entries are all zero. */
int ssnal_en_create_geno_device(const uint8_t* codes, int64_t stride, const double* tab, const double* db, int64_t m,
                                int64_t n, void* cuda_stream, ssnal_en_problem** out);
int ssnal_en_create_geno(const uint8_t* codes, int64_t stride, const double* tab, const double* b, int64_t m,
                         int64_t n, ssnal_en_problem** out);

/* ‖Aᵀb‖∞ computed at create (plain K1 pass).  λ1 ≥ this value gives x = 0. */
double ssnal_en_lambda_max_l1(const ssnal_en_problem* p);

/* Options (defaults from P:497 and DESIGN.md readings):
 *   sigma_factor=5, sigma_max=1e8, mu=0.2, beta=0.5, max_outer=100, max_inner=100,
 *   max_backtracks=50, init_mode=1 (y0 = A x0 − b when x0 ≠ 0, else y0 = 0; 0: always y0 = 0),
 *   time_k1=0 (1: time every K1 launch → stats.k1_time_s; CUDA events in host-driven mode,
 *     in-kernel %globaltimer stamps inside the graph),
 *   cluster_size=0 (auto: 16 if the device allows, else the largest schedulable power of two; an
 *     explicit 1/2/4/8/16 the device cannot schedule for k_chol_cluster is refused with EINVAL),
 *   carry_sigma=1 (ssnal_en_solve_path_device: point i > 0 starts at point i − 1's sigma_final
 *     instead of σ0 — reading R38 of P:411 "usually SsNAL-EN converges in just one iteration";
 *     0: every point restarts at σ0),
 *   reuse_atb=1 (both storage formats; reading R40: create keeps the product Aᵀb of its λmax pass, 8n bytes.
 *     After a cold start (x0 = NULL ⇒ x = 0, y0 = 0) the active set is empty for the first Newton
 *     step(s), so g = y + b, d = −g and the trial point y + d is −b: K1 compares its y with −b bit
 *     for bit and, if equal, takes Aᵀy = −Aᵀb from the kept product — bitwise what the streaming pass
 *     computes — instead of reading A once more.  While the active set at y = −b,
 *     #{i : |Aᵀb|_i > λ1}, is at most reuse_frac·n (=0.3) its columns are gathered for ∇ψ; above
 *     (reuse_psi_only=1, unsharded handles) the trial is served ψ-only — Armijo usually rejects
 *     s = 1 there and the gradient is rebuilt at the accepted step; if it accepts, the same trial is
 *     redone streamed — so the iterates stay bitwise those of the streamed solve either way.  Only
 *     for designs of at least reuse_min_bytes (=2 GB: the gate costs one small kernel and a stream
 *     synchronisation per cold solve); ssnal_en_get_info "atb_reuses" counts the solves that
 *     were allowed; 0: always stream A),
 *   small=1 (m ≤ 64 and n ≤ 1024, fp64 storage, unsharded, no CG strategy: the whole solve is ONE
 *     kernel launch — same iteration and statistics, reduction orders differ; 0: the multi-kernel
 *     graph / host paths), small_cluster=1 (that launch is k_small_cl, one 16-CTA cluster with A
 *     resident in distributed shared memory, when such a cluster is schedulable; 0: k_small_solve,
 *     one 512-thread CTA streaming A from L2),
 *   K4 variants (identical contract, results equal up to rounding): chol_dsm=1 (DSMEM-resident
 *     16-CTA cluster Cholesky for N ≤ 96; 0: the L2-tiled k_chol_cluster for every N), chol_d2=1
 *     (split-ownership DSMEM Cholesky k_chol_d2 for 96 < N ≤ 512; needs chol_dsm=1),
 *   certify=0 (1: after each solve compute stats.primal_viol with one extra Aᵀ pass),
 *   graph=1 (Algorithm 1 control on the device, the whole solve one CUDA graph; 0: host-driven
 *     control with one evaluation record read per ψ evaluation — identical results),
 *   Newton-system strategy (Algorithm 1 step (1); reading R32): conjugate gradient
 *     when r > cg_ratio·m (cg_ratio=0: off) or min(m, r) > cg_threshold (=1e4), else the
 *     exact branches; cg_tol=1e-10 (stop at ‖V d + ∇ψ‖ ≤ cg_tol‖∇ψ‖), cg_maxit=1000.
 *   jitter=1e-10 (R36): a non-positive Cholesky pivot redoes that Newton step once from
 *     the same y with the factored matrix's diagonal scaled by (1 + jitter) — the step is not
 *     counted, stats.jitter_retries is; a second failure returns SSNAL_ENUMERIC.  0: no retry.
 *   inner_tol_mode=0 (inner stop res1 ≤ tol, R6; 1: res1 ≤ max(tol, 0.1·res3) with res3 of Eq. (20)
 *     at the point each outer iteration starts from — SPEC's schedule, reading R37),
 *   test_fail_factor=0 (test hook: each solve treats its first N Cholesky factorisations as
 *     failed, to exercise the retry and SSNAL_ENUMERIC paths),
 *   EINVAL for unknown keys. */
int ssnal_en_set_option(ssnal_en_problem* p, const char* key, double value);

/* Read-only introspection: "m", "n", "k1_cols", "k1_stages", "k1_grid", "k1_smem",
 * "cluster_size", "num_sms", "graph", "format", "cg_ratio", "cg_threshold", "carry_sigma", "k1_time_s" /
 * "k1_launches" (Σ device time and count of the K1 launches of ssnal_en_aty_fused calls since option time_k1
 * was last set; CUDA events around the K1 launch alone), and which kernels a
 * solve on this handle uses: "small" (1: the single-launch small-problem path), "small_cluster" (1: that
 * path runs k_small_cl, 0: k_small_solve), "chol_dsm" (1: k_chol_dsm
 * for N ≤ 96), "chol_d2" (1: k_chol_d2 for 96 < N ≤ 512).  Returns NaN for unknown keys. */
double ssnal_en_get_info(const ssnal_en_problem* p, const char* key);

/* Solve Algorithm 1 for (λ1, λ2) in the paper's unnormalised units.
 * σ0 > 0 is the initial augmented-Lagrangian parameter (5e-3 in P:497); tol > 0 the
 * KKT tolerance: stop when res_kkt3 ≤ tol and res_kkt1 ≤ tol (Eq. (20), R7).
 * x0 (host, n; NULL = cold start y0 = 0) warm-starts the multiplier.
 * x_out (host, n, caller-owned) receives x, exactly zero off the active set.
 * stats may be NULL.  Returns SSNAL_OK, SSNAL_NOT_CONVERGED, SSNAL_EINVAL (λ1 < 0, λ2 < 0,
 * both zero, σ0 ≤ 0, tol ≤ 0), SSNAL_ENUMERIC or SSNAL_ECUDA. */
int ssnal_en_solve(ssnal_en_problem* p, double lambda1, double lambda2, double sigma0, double tol,
                   const double* x0, double* x_out, ssnal_en_stats* stats);

/* As ssnal_en_solve with x0 / x_out as DEVICE pointers (x0 may be NULL; x0 == x_out allowed). */
int ssnal_en_solve_device(ssnal_en_problem* p, double lambda1, double lambda2, double sigma0, double tol,
                          const double* x0_dev, double* x_out_dev, ssnal_en_stats* stats);

/* A warm-started λ path on DEVICE buffers (the path protocol of Table D.4 / BASELINE
 * configs[1]): point i solves (lambda1[i], lambda2[i]) starting from point i − 1's solution (point 0
 * from x0, nullable = cold) and, with option carry_sigma = 1 (default, reading R38), from point
 * i − 1's sigma_final instead of sigma0 (point 0 uses sigma0; the carried σ stays on the device).  x_out: device, npts × n (row i = point i's x).  stats: host, npts
 * entries (nullable).  With device-resident control (graph mode or the one-CTA path) every point is
 * enqueued before a single stream synchronisation; otherwise (host-driven control, sharded handles,
 * certify) it is a loop over ssnal_en_solve_device.  Same results and statistics as that loop;
 * time_total_s is the path's host time shared evenly.  Returns SSNAL_OK, or the first non-OK
 * status of a point (all stats are still written); EINVAL/ECUDA abort the path. */
int ssnal_en_solve_path_device(ssnal_en_problem* p, int64_t npts, const double* lambda1, const double* lambda2,
                               double sigma0, double tol, const double* x0, double* x_out, ssnal_en_stats* stats);

/* K1 hook (tests / bandwidth sweep).  All vector arguments are DEVICE pointers.
 * One fused pass at y (m) with multiplier x (n) and (σ, λ1, λ2):
 *   w_out (n) = Aᵀy; J_out (int32, capacity n) = {i : |x_i − σ w_i| > σλ1} ascending (Eq. (17));
 *   PJ_out (capacity n) = prox_{σp}(x − σw)_J (Eq. (6)); *r_out (host) = |J|;
 *   partials_out (host, 4) = [Σ P², Σ (x − P)², Σ z², Σ ((|w| − λ1)_+)²] with z = (x − P)/σ − w;
 *   grad_out (device m, nullable) = y + b − A_J P_J (Eq. (15)).
 * Synchronises the handle's stream before returning. */
int ssnal_en_aty_fused(ssnal_en_problem* p, const double* y, const double* x, double sigma, double lambda1,
                       double lambda2, double* w_out, int32_t* J_out, double* PJ_out, int64_t* r_out,
                       double partials_out[4], double* grad_out);

/* K1e hook: the K1 epilogue from a stored w0 (device, n) — or from w0 + s (w1 − w0) when
 * w1 != NULL (Armijo backtrack by linearity) — without touching A.  Same outputs as
 * ssnal_en_aty_fused except the gradient; w_out (nullable) receives the effective w. */
int ssnal_en_epilogue(ssnal_en_problem* p, const double* w0, const double* w1, double s, const double* x,
                      double sigma, double lambda1, double lambda2, double* w_out, int32_t* J_out,
                      double* PJ_out, int64_t* r_out, double partials_out[4]);

/* K2–K4/K6 hook: the Newton direction d (device, m) solving (I_m + κ A_J A_Jᵀ) d = −g for the
 * active set J (device int32, r entries, ascending) and g (device, m): r = 0 → d = −g;
 * 0 < r < m → SMW Eq. (19); r ≥ m → m × m Cholesky Eq. (18); CG (K6) when the cg_* options
 * select it.  *gd_out (host) = gᵀd, *branch_out (host) ∈ {0, 1, 2, 3}.  A non-positive Cholesky
 * pivot is retried once with the factored matrix's diagonal scaled by (1 + jitter) (option
 * "jitter", R36); SSNAL_ENUMERIC if the retry fails too (or jitter = 0). */
int ssnal_en_newton_direction(ssnal_en_problem* p, const int32_t* J, int64_t r, const double* g, double kappa,
                              double* d_out, double* gd_out, int32_t* branch_out);

/* Model-selection quantities of the solution of the most recent ssnal_en_solve / _solve_device
 * on this handle (Section 3.3):
 *   active = r = |supp x|;
 *   nu   = tr(A_J (A_JᵀA_J + λ2 I)⁻¹ A_Jᵀ), the Elastic Net degrees of freedom;
 *   rss  = ‖b − A_J x_ols‖² after de-biasing by least squares on the selected features;
 *   gcv  = m⁻¹ rss / (1 − ν/m)²,  ebic = log(rss/m) + (ν/m)(log m + log n)   (Eq. (21)).
 * ols_ok = 0 (and rss, gcv, ebic = NaN) when A_JᵀA_J is not positive definite (r ≥ m or collinear
 * columns).  xdb_out (host, n, nullable) receives the de-biased coefficients (zero off supp x).
 * λ2 must equal the one the solution was computed with. */
typedef struct {
  int64_t active;
  double nu, rss, gcv, ebic;
  int32_t ols_ok;
  int32_t reserved;
} ssnal_en_criteria;

int ssnal_en_model_select(ssnal_en_problem* p, double lambda2, double* xdb_out, ssnal_en_criteria* out);

/* Held-out residual for cross-validation (Section 3.3): *rss_out = ‖A x − b‖²
 * for this handle's A and b (e.g. the test rows of a fold) and a given x (n; host for
 * ssnal_en_residual, device for _device).  Uses only the support of x (gathered columns).  Does not
 * touch the handle's last solution.  EINVAL for null arguments. */
int ssnal_en_residual(ssnal_en_problem* p, const double* x, double* rss_out);
int ssnal_en_residual_device(ssnal_en_problem* p, const double* x_dev, double* rss_out);

/* Column-sharded solves ("the path shards naturally by column blocks of A").
 * Rank q of nranks owns a contiguous block of columns; its handle is created on that block alone
 * (n = the block's column count, any create call).  Every cross-column quantity of Algorithm 1 is
 * a sum over the blocks and goes through the caller's all-reduce, called on the handle's stream
 * order: per ψ evaluation the partial m-vector A_J P_J, four scalar partial sums and |J| (m + 5
 * doubles); per Newton step either the active columns (0 < r < m: each rank's A_J placed at its
 * prefix offset of an r × m buffer, so the sum is an all-gather; SMW Eq. (19) on the result) or
 * the partial m × m Gram A_J A_Jᵀ (r ≥ m, Eq. (18)); plus the warm-start A x0, the objective and
 * λmax.  All ranks therefore hold identical reduced values and take identical control decisions;
 * solves run host-driven (a host callback cannot sit inside the graph; see ssnal_en_peer_attach
 * for the device-resident provider) and the CG strategy is not used on a sharded handle.
 *   fn(ctx, buf, count, op, stream): all-reduce count doubles at the DEVICE pointer buf in place,
 *     op 0 = sum, 1 = max, ordered after the work already queued on `stream` (cudaStream_t) and
 *     complete before work queued after the call; return 0 on success.  Called only from inside
 *     this library's calls, on the calling thread.
 *   Each rank must call ssnal_en_solve* with the same λ1, λ2, σ0, tol and options; x0 / x_out are
 *   the rank's slices (x0 may be NULL on some ranks: missing slices count as zero).
 * set_comm exchanges λmax (lambda_max_l1 becomes the global value).  rank ∈ [0, nranks).  Stats:
 * active, primal_obj, gap, res_kkt* are global.  Returns SSNAL_EINVAL for bad arguments. */
int ssnal_en_set_comm(ssnal_en_problem* p, ssnal_en_allreduce_fn fn, void* ctx, int rank, int nranks);

/* Column-sharded solves with DEVICE-RESIDENT exchanges over peer memory ("a few
 * µs with … symmetric memory"; one process per GPU, NVLink / NVSwitch peers).  The same exchange
 * points and the same rank-ordered sums as ssnal_en_set_comm, but every exchange is a kernel of this
 * library — each rank writes its contribution straight into a slot of EVERY rank's exchange region
 * (P2P stores), raises a flag per region, and sums the G slots of its own region in rank order
 * 0 … G−1 once all flags reached the exchange's epoch — so the solve keeps its device-resident
 * control (one CUDA graph with conditional nodes per solve; option graph = 1, the default) and no
 * host callback runs inside a solve.  The compute and the collective are fused where one follows
 * the other: the gather of the active columns writes them into the peers (the all-gather of the SMW
 * branch, Eq. (19)), and the split-K reduction of the local partial Gram deposits it into the peers
 * (Eq. (18)).  Waits give up after 20 s (the call then returns SSNAL_ECUDA).
 *   1. ssnal_en_peer_export(p, nranks, handle_out): allocates this rank's exchange region (about
 *      8·nranks·max(m, 8)·m bytes + 2 evaluation records per rank) and writes its CUDA IPC handle
 *      (SSNAL_EN_IPC_HANDLE_BYTES bytes, host memory) to handle_out.  1 ≤ nranks ≤ 16.
 *   2. The caller all-gathers the handles (any transport, e.g. torch.distributed.all_gather_object).
 *   3. ssnal_en_peer_attach(p, rank, nranks, handles): handles = nranks × SSNAL_EN_IPC_HANDLE_BYTES
 *      bytes in rank order (host); maps the peers' regions (cudaIpcOpenMemHandle; the own one is used
 *      directly) and exchanges λmax (a collective call: every rank must call it).  Replaces a
 *      set_comm provider.  SSNAL_EINVAL if export was not called with the same nranks.
 * Solve calls follow the rules of ssnal_en_set_comm (same arguments and options on every rank,
 * x0 / x_out are the rank's slices).  The exchange region is freed by destroy or a new export. */
int ssnal_en_peer_export(ssnal_en_problem* p, int nranks, void* handle_out);
int ssnal_en_peer_attach(ssnal_en_problem* p, int rank, int nranks, const void* handles);

/* Test hook for the exchange protocol of ssnal_en_peer_attach on ONE device: nranks ranks are
 * emulated by nranks CTAs of one cooperative launch (co-resident, so their waits on one another
 * cannot deadlock), each with its own region inside one allocation, running `iters` exchanges (two
 * small ones, then a big one, repeated) of `count` doubles through the same deposit / flag / epoch /
 * rank-ordered-sum code as the solve's exchanges.  Every sum is checked in the kernel against its
 * closed form; *mismatch_out = number of wrong elements over all ranks and exchanges.  small_out /
 * big_out (host, nranks × count, nullable) receive each rank's last small / big sum.
 * 1 ≤ nranks ≤ 16, 1 ≤ count ≤ 65536.  SSNAL_ECUDA if a wait timed out. */
int ssnal_en_peer_selftest(int nranks, int iters, int64_t count, int64_t* mismatch_out, double* small_out,
                           double* big_out);

void ssnal_en_destroy(ssnal_en_problem* p);

/* Thread-local message of the last failure on this thread ("" if none). */
const char* ssnal_en_last_error(void);

/* Build identification string (arch, version). */
const char* ssnal_en_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SSNAL_EN_H */
