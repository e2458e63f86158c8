/*
 * sunfold.h — C-ABI of the B200 (sm_100a) SU(N) unfold of the GKSL master equation.
 *
 * Paper: "Unfolding quantum master equation into a system of real-valued equations:
 * computationally effective expansion over the basis of SU(N) generators",
 * arXiv:1812.11626.  Citations P:n are PAPER.md line numbers.
 *
 * What the library computes (Eq. 1, Eq. 5, Eq. 6 P:171-174,
 * Eq. 9, Eqs. 10-11; Table I Step 2 P:287):
 *
 *   Given H(t) = H0 + eps(t) H1 and dissipators {L_p, gamma_p}, p = 1..P, the GKSL generator
 *     L(t) rho = -i[H(t), rho] + sum_p gamma_p (L_p rho L_p^+ - 1/2 {L_p^+ L_p, rho})
 *   is unfolded over the SU(N) generators F_1..F_M (M = N^2 - 1; basis P:135-144, DESIGN.md
 *   readings R4/R5) into the real system
 *     dv/dt = (Q0 + eps(t) Q1) v + K,      rho = I/N + sum_j v_j F_j,
 *   with  Q0_sm = Tr(F_s L0(F_m)),  Q1_sm = Tr(F_s (-i[H1, F_m])),  K_s = Tr(F_s L0(I/N)),
 *   where L0 is L with H = H0.  Q0 contains both the paper's Q (Eq. 6, from H0) and R
 *   (Eq. 10); K is Eq. 11 (with gamma_p, R2).  A trace of L_p is allowed (R3).
 *
 * Generator order (part of the ABI, R5), 0-based, a < b, l = 1..N-1:
 *   idx(S_ab) = p(a,b), idx(J_ab) = N(N-1)/2 + p(a,b), idx(D^l) = N(N-1) + l - 1,
 *   p(a,b) = a(2N-a-1)/2 + (b-a-1).
 *
 * Stored pattern (R6): an entry q is stored iff |q| > tau, with
 *   tau(Q0) = 1e-14 (||H0||_F + sum_p gamma_p ||L_p||_F^2),  tau(Q1) = 1e-14 ||H1||_F.
 * Columns ascend within each row.  Results are bitwise deterministic.
 *
 * Memory ownership: every array argument is a DEVICE pointer owned by the caller (the
 * Python binding allocates with torch); the library never allocates device memory.
 * `stream` is a cudaStream_t passed as void*.  A plan is bound to one stream and is not
 * thread-safe.  Nothing throws across the ABI: every call returns a sun_status.
 *
 * Call sequence (the paper's two-step CRS fill: "the number of nonzero elements
 * in each row is computed. Next, the elements are calculated and indexes are written"):
 *   sun_workspace_bytes(n, P) -> caller allocates the device workspace
 *   sun_plan_create  -> validate + analyse the operator patterns (one small readback)
 *   sun_count        -> expand (a1), count pass (a3), prefix scan (a4)          [async]
 *   sun_plan_nnz     -> synchronises; nnz of Q0 / Q1 (16-byte readback)
 *   caller allocates Q0 / Q1 CSR (row_ptr int64[M+1], col int32[nnz], val double[nnz]), K
 *   sun_unfold       -> fill pass with fused K (a5), Q1 (a6)                     [async]
 *   sun_apply        -> dv/dt = Q0 v + eps Q1 v + K (a7)                         [async]
 * or, without the host round trip between the passes:
 *   sun_run          -> count + scan + fill into outputs of a given capacity      [async]
 *   sun_plan_nnz     -> nnz (SUN_ERR_CAPACITY: refill with sun_unfold)
 */
#ifndef SUNFOLD_H_
#define SUNFOLD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SUN_OK = 0,
  SUN_ERR_ARG = 1,           /* null / inconsistent pointers or sizes, malformed CSR        */
  SUN_ERR_DIM = 2,           /* N < 2, N > 46340 (M must fit int32), operators of other N   */
  SUN_ERR_NOT_HERMITIAN = 3, /* max|H - H^+| > 1e-12 ||H||_F for H0 or H1    */
  SUN_ERR_RATE = 4,          /* gamma_p < 0 or non-finite                   */
  SUN_ERR_CAPACITY = 5,      /* an output CSR capacity is below the required nnz            */
  SUN_ERR_CUDA = 6,          /* CUDA runtime error; sun_status_string() reports it          */
  SUN_ERR_UNSUPPORTED = 7,   /* operation not available for this plan: the matrix-free RK4 /
                                apply on a general-pattern (mode 3) plan; a single output row
                                with >= 2^32 candidate terms                                 */
  SUN_ERR_STATE = 8          /* call out of sequence (e.g. sun_unfold before sun_count), or
                                operator values outside the pattern fixed by the plan       */
} sun_status;

/* N x N complex operator, CSR, device memory.  row_ptr int64[n+1]; col int32[nnz], strictly
 * ascending within a row, in [0, n); val = interleaved (re, im) float64[2*nnz]. */
typedef struct {
  int32_t n;
  int64_t nnz;
  const int64_t* row_ptr;
  const int32_t* col;
  const double* val;
} sun_zcsr;

/* M x M real output, CSR, device memory.  `nnz` is the CAPACITY of col/val on input.
 * row_ptr int64[m+1]; col int32[capacity]; val float64[capacity]. */
typedef struct {
  int64_t m;
  int64_t nnz;
  int64_t* row_ptr;
  int32_t* col;
  double* val;
} sun_dcsr;

typedef struct sun_plan_s* sun_plan;

/* Plan diagnostics (host struct filled by sun_plan_info). */
typedef struct {
  int32_t n, P;
  int32_t w_h0, w_h1, w_l, w_k; /* half-bandwidths: H0, H1, max_p L_p, K = H0 + i/2 sum gamma L^+L */
  double tau_q0, tau_q1;        /* drop thresholds (R6) */
  int32_t mode_q0, mode_q1;     /* 0: thread-per-pair far tiles (compile-time widths); 1: warp-per-pair,
                                   runtime widths; 2: warp-per-pair far path, compile-time widths;
                                   3: general pattern (candidate merge, sunfold_general.cu) */
  int32_t pairs_per_tile_q0, pairs_per_tile_q1;
  int64_t tiles_q0, tiles_q1;   /* scan slots (S tiles, J tiles, D slots) */
  int32_t has_h1;
  int32_t npos_far_q0, npos_far_q1; /* candidate positions per far pair */
  int32_t launches_count;       /* kernels enqueued by sun_count (expand, count, scan) */
  int32_t launches_fill;        /* kernels enqueued by sun_unfold (sun_run = both) */
} sun_plan_info_t;

/* Bytes of device workspace a plan for dimension n with P dissipators needs when its operators
 * are banded (0 if n or P is out of range): the band-expanded operators, the per-row counts
 * (2 x 4 bytes per output row) and the tile offsets; 256-byte aligned.  Operators of any other
 * pattern need sun_workspace_bytes_ops. */
size_t sun_workspace_bytes(int32_t n, int32_t P);

/* Bytes of device workspace that suffice for these operators whatever their pattern (host-only:
 * reads the n and nnz fields): sun_workspace_bytes(n, P) plus, for the general-pattern mode,
 * column access to every L_p (8 bytes per nonzero, 8 bytes per column) and the heavy-row lists
 * (8 bytes per generator pair).  0 for invalid arguments. */
size_t sun_workspace_bytes_ops(const sun_zcsr* H0, const sun_zcsr* H1, const sun_zcsr* const* L, int32_t P);

/* Validate the inputs and analyse their patterns (half-bandwidths, Frobenius norms) on the
 * device, then build the plan.  Operators of ANY pattern are accepted ("any complex N x N matrix
 * could be chosen as an operator L_p"): banded ones (max(w_H0, 2 w_L) <= 15, w_L <= 7,
 * w_H1 <= 15) take the band kernels (modes 0-2), every other pattern the general mode (mode 3,
 * candidate terms merged per row by a sort and a segmented reduction).
 *   H0: required.  H1: NULL if there is no periodic drive (then Q1 is not produced).
 *   L: array of P pointers to operators (may be NULL if P == 0); gamma: HOST array of P rates.
 *   workspace: device, >= sun_workspace_bytes(H0->n, P); owned by the caller, bound to the
 *   plan until sun_plan_destroy.
 * Runs one kernel on `stream` and synchronises on a small readback.  The input operators
 * must stay valid until sun_count has completed on the stream (their values are read there;
 * their patterns, i.e. bandwidths, are fixed by the plan).  Errors: SUN_ERR_DIM, _ARG (also
 * malformed CSR: unsorted/out-of-range columns), _RATE, _CAPACITY (a general-pattern plan with a
 * workspace smaller than sun_workspace_bytes_ops), _CUDA; *out is NULL then. */
int sun_plan_create(sun_plan* out, const sun_zcsr* H0, const sun_zcsr* H1, const sun_zcsr* const* L,
                    const double* gamma, int32_t P, void* workspace, size_t workspace_bytes, void* stream);

/* sun_plan_create with options.  flags: SUN_PLAN_GENERAL = take the general mode even for banded
 * operators (cross-checks); SUN_PLAN_SMALLCAP = general mode with a 16-candidate merge buffer
 * (tests: forces the key-range chunks and the single-key reduction at small N; slow);
 * 0 = sun_plan_create. */
#define SUN_PLAN_GENERAL 1
#define SUN_PLAN_SMALLCAP 2
int sun_plan_create_ex(sun_plan* out, const sun_zcsr* H0, const sun_zcsr* H1, const sun_zcsr* const* L,
                       const double* gamma, int32_t P, int32_t flags, void* workspace, size_t workspace_bytes,
                       void* stream);

/* Expand H0/H1/L_p into band storage, form K = H0 + (i/2) sum_p gamma_p L_p^+ L_p and the drop
 * thresholds from the operators' current values, run the count pass and the prefix scan for
 * Q0 (and Q1).  Asynchronous on `stream`.  May be called again (with changed operator values,
 * same patterns) to re-unfold with the same plan. */
int sun_count(sun_plan plan, void* stream);

/* Synchronise the sun_count stream and return nnz(Q0) and nnz(Q1) (0 if no drive); reports
 * SUN_ERR_NOT_HERMITIAN / SUN_ERR_ARG found by the device-side validation,
 * SUN_ERR_STATE if an operator's values now exceed the half-bandwidth fixed by a banded plan, and
 * SUN_ERR_UNSUPPORTED for a row with >= 2^32 candidate terms (general mode). */
int sun_plan_nnz(sun_plan plan, int64_t* nnz_q0, int64_t* nnz_q1);

/* Fill pass: write Q0 (CSR), K (float64[M]) and, if the plan has H1, Q1.  Q1 may be NULL
 * only if the plan has no H1.  Capacities (nnz fields) must be >= sun_plan_nnz's values.
 * Asynchronous on `stream`. */
int sun_unfold(sun_plan plan, sun_dcsr* Q0, sun_dcsr* Q1, double* K, void* stream);

/* Single-pass enqueue of the whole unfold (expand, count, scan, fill + K, Q1) into outputs of
 * the given capacities, with no host synchronisation between the passes.  Use capacities
 * from sun_nnz_bound (always sufficient) or from a previous sun_plan_nnz.  Afterwards call
 * sun_plan_nnz: it returns the nnz and SUN_ERR_CAPACITY if an output was too small (then no
 * entry at or beyond the capacity was written; allocate nnz entries and call sun_unfold,
 * which refills from the counts already computed).  Asynchronous on `stream`. */
int sun_run(sun_plan plan, sun_dcsr* Q0, sun_dcsr* Q1, double* K, void* stream);

/* Structural upper bound on nnz(Q0) (which = 0) or nnz(Q1) (which = 1) for this plan's
 * patterns (independent of values); -1 for an invalid request. */
int64_t sun_nnz_bound(sun_plan plan, int32_t which);

/* dv/dt = Q0 v + eps Q1 v + K  (Eq. 9).  Q1 may be NULL; K may be NULL (= 0).
 * v, dvdt: float64[M], must not alias.  Asynchronous on `stream`. */
int sun_apply(const sun_dcsr* Q0, const sun_dcsr* Q1, double eps, const double* K, const double* v,
              double* dvdt, void* stream);

/* ---- Propagation (PAPER.md Step 3) and states (Step 2.6 P:456-457, Eq. 5) ---- */

/* v(0): the coherence vector of an N x N operator rho (Eq. 5):
 *   v_s = Re Tr(F_s rho),  s = 0 .. M-1 (generator order R5); for S_ab / J_ab only the
 *   entries (a, b) and (b, a) contribute, for D^l the diagonal prefix (sum_{c<l} rho_cc -
 *   l rho_ll) / sqrt(l(l+1)).  rho: CSR (device), any entries; v: device float64[M], written
 *   (fully overwritten).  Asynchronous on `stream`.  Errors: SUN_ERR_ARG, SUN_ERR_DIM, _CUDA. */
int sun_expand_state(const sun_zcsr* rho, double* v, void* stream);

/* Populations of the state with coherence vector v (inverse of Eq. 5 on the diagonal):
 *   diag[a] = <a|rho|a> = 1/N + sum_l v_{D^l} delta_l(a),  delta_l(a) = (D^l)_aa,
 * i.e. the bifurcation-diagram observable p_n.  v: device float64[N^2 - 1];
 * diag: device float64[N].  Asynchronous.  Errors: SUN_ERR_ARG, SUN_ERR_DIM, _CUDA. */
int sun_state_diag(const double* v, int32_t n, double* diag, void* stream);

/* rho(T) from its coherence vector (Step 3.2; Eq. 5): rho = I/N + sum_j v_j F_j,
 * written as a dense complex N x N array (row-major, interleaved re, im; all 2 N^2 doubles
 * written).  Off-diagonal entries from the S_ab / J_ab coefficients, the diagonal as in
 * sun_state_diag.  v: device float64[N^2 - 1]; rho: device float64[2 N^2].  Asynchronous.
 * Errors: SUN_ERR_ARG, SUN_ERR_DIM, SUN_ERR_CUDA. */
int sun_state_reconstruct(const double* v, int32_t n, double* rho, void* stream);

/* Fixed-step classic fourth-order Runge-Kutta (the paper's integrator, Step 3.1 P:464-470) of
 *   dv/dt = (Q0 + eps(t) Q1) v + K,   eps(t) = eps0 + eps1 sin(omega t)   (Eq. 9, reading R10)
 * from t0 over nsteps steps of size h:
 *   k1 = f(t, v), k2 = f(t + h/2, v + h/2 k1), k3 = f(t + h/2, v + h/2 k2), k4 = f(t + h, v + h k3),
 *   v <- v + h/6 (k1 + 2 k2 + 2 k3 + k4).
 * One fused SpMV kernel per stage (the stage input v + c k is formed in the gather; the RK4
 * sum is accumulated in the epilogue; the stage vectors k are double-buffered).  Q1 may be NULL (no drive); K may be NULL (= 0).
 * v: device float64[M], in/out.  work: device scratch of sun_rk4_work_bytes(M) bytes owned by
 * the caller (8-byte aligned).  Rows of Q0 with more than 64 entries are processed by a warp
 * each (their list is built at the start of the call: one 4-byte readback, i.e. the call
 * synchronises once); all else is asynchronous on `stream`.
 * Errors: SUN_ERR_ARG, SUN_ERR_DIM (M = 0 or M > 2^31 - 1), SUN_ERR_CUDA. */
int sun_rk4(const sun_dcsr* Q0, const sun_dcsr* Q1, const double* K, double eps0, double eps1, double omega,
            double t0, double h, int64_t nsteps, double* v, void* work, void* stream);

/* Bytes of scratch sun_rk4 needs for an M-row system (4 M doubles + M + 2 ints); 0 if M <= 0. */
size_t sun_rk4_work_bytes(int64_t m);

/* F1, matrix-free: the same fixed-step RK4 as sun_rk4 on the system of a counted plan (after
 * sun_count or sun_run on the current operator values), without reading Q0 / Q1: every stage
 * regenerates the far-pair entries from the plan's band storage with the count/fill
 * expressions and tau masks, takes the near and D rows from the count pass's side buffer
 * (chain tails in O(1) from a per-stage prefix over the D coefficients), K from the same data.
 * Supported: mode-0 plans and mode-2 plans (sun_plan_info mode_q0 = 0 or 2) without a drive or
 * with a diagonal H1; else SUN_ERR_UNSUPPORTED.  v: device float64[M], in/out.  work: device scratch of
 * sun_rk4_plan_work_bytes(plan) bytes (4 M + N doubles).  Asynchronous on `stream`.
 * Errors: SUN_ERR_ARG, SUN_ERR_STATE (plan not counted), SUN_ERR_UNSUPPORTED, SUN_ERR_CAPACITY,
 * SUN_ERR_CUDA. */
int sun_rk4_plan(sun_plan plan, double eps0, double eps1, double omega, double t0, double h, int64_t nsteps,
                 double* v, void* work, size_t work_bytes, void* stream);
size_t sun_rk4_plan_work_bytes(sun_plan plan);

/* dv/dt = (Q0 + eps Q1) v + K matrix-free (the stage of sun_rk4_plan with a plain output): the
 * same support and state requirements as sun_rk4_plan.  v, dvdt: device float64[M] (distinct).
 * work: device scratch of >= N doubles.  Asynchronous.  Errors: as sun_rk4_plan. */
int sun_apply_plan(sun_plan plan, double eps, const double* v, double* dvdt, void* work, size_t work_bytes,
                   void* stream);

/* Enable (1, the default) or disable (0) CUDA-graph replay of this plan's enqueue sequences.
 * With graphs, sun_count / sun_unfold / sun_run capture their launches once per distinct
 * output buffer set and replay the graph (one launch); without, every kernel is launched
 * directly (used to time a kernel alone).  The environment variable SUNFOLD_NO_GRAPHS=1
 * sets the default to 0.  Errors: SUN_ERR_ARG. */
int sun_plan_set_graphs(sun_plan plan, int32_t enable);

/* Light-row stash of a general-pattern plan (mode 3).  The count pass assembles
 * every row from its candidate terms (gather, sort by key, segmented reduction); with a stash,
 * it also writes each light pair's two assembled rows (<= GW_CAP candidates, at most
 * sun_plan_stash_bytes' per-row capacity of entries) into the stash, and the fill pass copies
 * them to their CSR offsets instead of assembling them a second time (bit-identical output:
 * the stash is written by the same operations in the same order as the fill's own writing
 * pass).  sun_plan_stash_bytes: bytes the stash needs (0 for banded plans, whose fill does
 * not assemble rows).  sun_plan_set_stash: `buf` = device memory of at least that many bytes,
 * 256-byte aligned, caller-owned, kept until the plan is destroyed or the stash is changed;
 * buf = NULL switches the stash off (the default).  Changing it drops the plan's cached
 * graphs and requires a new count pass before the next fill (SUN_ERR_STATE otherwise).
 * Errors: SUN_ERR_ARG (null plan; buffer too small or misaligned; a banded plan). */
size_t sun_plan_stash_bytes(sun_plan plan);
int sun_plan_set_stash(sun_plan plan, void* buf, size_t bytes);

/* Phase timing (SURVEY §5 tracing; bench.py's roofline): with enable = 1, every sun_run /
 * sun_count / sun_unfold sequence of this plan records CUDA events (event-record nodes of its
 * graph) before the count pass (expand + count + scan), between count and fill, and after the
 * fill; sun_plan_phase_ms then returns the device time of the last sequence's phases in ms
 * (count_ms: expand + count + scan, fill_ms: the fill pass incl. K and Q1; -1 for a phase the
 * sequence did not run).  sun_plan_phase_ms waits for the last sequence to complete.  Toggling
 * drops the plan's cached graphs.  Errors: SUN_ERR_ARG, SUN_ERR_STATE (no timed sequence yet),
 * SUN_ERR_CUDA. */
int sun_plan_set_timing(sun_plan plan, int32_t enable);
int sun_plan_phase_ms(sun_plan plan, float* count_ms, float* fill_ms);

/* ---- Dense unfold of a generator given by a rate matrix A -----------
 * PAPER.md Eq. 7 writes the dissipator with a positive semidefinite M x M rate
 * matrix A over the basis; P:568-570 samples "a 'dense', randomly generated, rate matrix A"
 * at N = 100 over > 10^3 realisations.  For each realisation r of a batch:
 *   L(X) = -i[H, X] + sum_jk a_jk (F_j X F_k - 1/2 {F_k F_j, X})      (F_k^+ = F_k)
 *   Q_sm = Tr(F_s L(F_m)),  K_s = Tr(F_s L(I/N))       (dense; generator order R5)
 * n: N, 2 <= N <= 1024.  batch: number of realisations (>= 0; 0 is a no-op).
 * H: device double[batch][N][N][2]: complex Hermitian H (row-major, interleaved re, im; the
 *    Hermiticity is not checked here).
 * A: device double[batch][M][M][2]: complex Hermitian rate matrix in the F basis (row-major),
 *    or NULL: no dissipator (Q = Q_H, K = 0).
 * Q: device double[batch][M][M] (row-major, all M^2 entries written; real because L
 *    preserves Hermiticity).  K: device double[batch][M], or NULL: not written.
 * work: device scratch owned by the caller, >= sun_dense_work_bytes(n, 1) bytes (256-byte
 *    aligned); realisations are processed floor(work_bytes / sun_dense_work_bytes(n, 1)) at a
 *    time.  Asynchronous on `stream`; deterministic.
 * Errors: SUN_ERR_DIM (N out of range), SUN_ERR_ARG (batch < 0; null H, Q or work),
 *    SUN_ERR_CAPACITY (work too small), SUN_ERR_CUDA. */
int sun_unfold_dense(int32_t n, int32_t batch, const double* H, const double* A, double* Q, double* K, void* work,
                     size_t work_bytes, void* stream);

/* Scratch bytes for `chunk` realisations at once (16 N^4 + 16 (N-1) N^2 + 16 N^2 each, each
 * part 256-byte aligned); 0 if N is out of range or chunk < 1. */
size_t sun_dense_work_bytes(int32_t n, int32_t chunk);

/* Kernel launches sun_unfold_dense makes for these arguments (0 if it would fail). */
int sun_dense_launches(int32_t n, int32_t batch, int32_t has_a, size_t work_bytes);

/* ---- Structure constants (Step 2.2; Eqs. 2-4) ----
 * The nonzero f_mns (which = 0) or d_mns (which = 1) of SU(N) over the basis F (generator order
 * R5), every ordered triple (f totally antisymmetric, d totally symmetric), generated on
 * the device from the closed-form classes (triangle, pair, DDD).  Counts:
 * NZ_F = 5N^3 - 9N^2 - 2N + 6, NZ_D = 6N^3 - N(21N+7)/2 + 1.  The unfold itself never
 * stores them.  Deterministic order (by index pair, then class).
 * n: 2 <= N <= 1024.  idx: device int32[cap][3] (m, n, s) and val: device double[cap], or both
 * NULL with cap = 0 (count only).  nnz: host int64*, the total (written; the call synchronises
 * `stream`).  work: device scratch of sun_sc_work_bytes(n) bytes.
 * Errors: SUN_ERR_DIM, SUN_ERR_ARG, SUN_ERR_CAPACITY (work too small, or cap < nnz: entries
 * beyond cap are not written), SUN_ERR_CUDA. */
int sun_structure_constants(int32_t n, int32_t which, int32_t* idx, double* val, int64_t cap, int64_t* nnz,
                            void* work, size_t work_bytes, void* stream);
size_t sun_sc_work_bytes(int32_t n);

/* Fill a diagnostics struct for the plan. */
int sun_plan_info(sun_plan plan, sun_plan_info_t* info);

/* Free the host-side plan (it owns no device memory). */
void sun_plan_destroy(sun_plan plan);

/* Human-readable status (includes the last CUDA error text for SUN_ERR_CUDA). */
const char* sun_status_string(int status);

/* Canonical generator index (host helper, R5): kind 0 = S_ab, 1 = J_ab (a < b),
 * 2 = D^l (a = l in [1, n-1], b ignored).  Returns -1 for invalid arguments. */
int64_t sun_gen_index(int32_t n, int32_t kind, int32_t a, int32_t b);

/* Library version string. */
const char* sun_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SUNFOLD_H_ */
