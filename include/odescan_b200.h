/*
 * odescan_b200.h — C ABI of the B200-native parallel-in-time Newton solver.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `odescan` (arXiv 2511.01465).  Every entry point below replaces one
 * reference interface; the citation after each declaration is the
 * reference file:line (relative to /root/reference/pkg/src/odescan/) whose
 * behaviour it reproduces.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers (cudaMalloc / torch tensors),
 *    fp64, C-contiguous, caller-owned.  Scalars are passed by value; small
 *    descriptor structs (problem / stepper / config) are HOST pointers and are
 *    copied by value into kernel parameters, so they may be freed on return.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Every call only enqueues work on that stream and returns immediately;
 *    no call synchronises the device.
 *  - Return value: ODX_OK (0) or a negative ODX_E* code.  No exception ever
 *    crosses the ABI; odx_last_error() returns a thread-local message.
 *  - The library keeps no global mutable state other than cached device
 *    properties, so calls on different streams/devices may run concurrently.
 *  - There is no CPU fallback: every compute entry point runs CUDA kernels
 *    built for sm_100a, or fails with ODX_ECUDA / ODX_EUNSUPPORTED.
 */
#ifndef ODESCAN_B200_H
#define ODESCAN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ODX_ABI_VERSION 1

/* ---- return codes ------------------------------------------------------ */
#define ODX_OK            0
#define ODX_EINVAL       (-1)  /* bad argument (ValueError on the Python side) */
#define ODX_EUNSUPPORTED (-2)  /* no device functor / unsupported dim or stepper */
#define ODX_ECUDA        (-3)  /* CUDA runtime error */
#define ODX_EWORKSPACE   (-4)  /* workspace too small */

/* ---- per-trajectory solve status (int32 status[b]) --------------------- */
#define ODX_ST_MAXITER    0  /* ran max_iters updates (the reference's normal exit) */
#define ODX_ST_CONVERGED  1  /* residual_tol or step_tol rule fired               */
#define ODX_ST_NONFINITE  2  /* ||h||_inf = +-inf at iteration status_index
                                (newton_pint.py:381-383, NonFiniteError)          */
#define ODX_ST_SINGULAR   3  /* pivot < 1e-300 in block status_index
                                (newton_pint.py:378-380, SingularDiagonalBlockError) */

/* ---- ODE problems (device functors) ------------------------------------ */
/* Reference plug-in type: OdeProblem(f_into, jac_into) problems.py:36-65.
 * numba dispatchers cannot run on the GPU, so a problem crosses the ABI as
 * (problem_id, dim, params) selecting a compiled device functor.            */
#define ODX_PROB_LOGISTIC     0  /* params: r, K              problems.py:88-114  */
#define ODX_PROB_VDP          1  /* params: mu                problems.py:117-147 */
#define ODX_PROB_CARTPOLE     2  /* params: g, l, m_c, m_p    problems.py:162-194 */
#define ODX_PROB_CARTPOLE_SQ  3  /* centripetal variant       problems.py:197-226 */
#define ODX_PROB_DAHLQUIST    4  /* params: lambda            problems.py:248-272 */
#define ODX_PROB_ROBERTSON    5  /* params: k1, k2, k3        problems.py:275-318 */
#define ODX_PROB_LORENZ63     6  /* params: sigma, rho, beta  (BASELINE cfg 1/3)  */
#define ODX_PROB_ALLEN_CAHN   7  /* params: eps, dx; dim = grid points (cfg 4)    */
#define ODX_PROB_EXP_GROWTH   8  /* dy/dt = exp(y)  tests/test_newton_pint.py:28-46 */
#define ODX_PROB_SQUARE       9  /* dy/dt = y^2     tests/test_newton_pint.py:49-68 */
#define ODX_PROB_LINEAR      10  /* dx/dt = A x; params: A row-major (dim<=8)      */
#define ODX_NUM_PROBLEMS     11

/* initial-guess policies (newton_pint.initial_guess, newton_pint.py:174-207) */
#define ODX_GUESS_ONES         0
#define ODX_GUESS_ZEROS        1
#define ODX_GUESS_REPLICATE_X0 2
#define ODX_GUESS_COARSE_EULER 3

#define ODX_MAX_PARAMS 64

typedef struct odx_problem {
    int32_t problem_id;
    int32_t dim;
    int32_t n_params;
    int32_t reserved;
    double  params[ODX_MAX_PARAMS];
} odx_problem;

/* ---- step maps ---------------------------------------------------------- */
/* Reference: StepperIncrement{kind, tableau | weights} steppers.py:80-99.    */
#define ODX_STEP_EXPLICIT_RK        0  /* tableau a (s x s, strictly lower), b (s) */
#define ODX_STEP_IMPLICIT_WEIGHTED  1  /* g = dt (w_prev f(prev) + w_next f(next)) */
#define ODX_MAX_STAGES 4

typedef struct odx_stepper {
    int32_t kind;
    int32_t stages;                              /* explicit only, 1..4 */
    double  a[ODX_MAX_STAGES * ODX_MAX_STAGES];  /* row-major s x s    */
    double  b[ODX_MAX_STAGES];
    double  w_prev, w_next;                      /* implicit only      */
} odx_stepper;

/* ---- Newton controls ---------------------------------------------------- */
/* Reference: NewtonConfig(max_iters, residual_tol, record_residuals)
 * newton_pint.py:119-138, plus the BASELINE step rule (step_tol) and a
 * non-aborting fixed-iteration mode used for timing.      */
typedef struct odx_newton_cfg {
    int32_t max_iters;        /* >= 1                                        */
    int32_t abort_nonfinite;  /* 1: stop with NONFINITE like solve(); 0: keep going */
    double  residual_tol;     /* 0 disables; stop when ||h||_inf <= tol      */
    double  step_tol;         /* 0 disables; stop when max|dx| of the last update < tol */
} odx_newton_cfg;

/* ---- library info -------------------------------------------------------- */
int         odx_abi_version(void);
const char* odx_last_error(void);
/* 1 if (problem, stepper) has a compiled device path, else 0. */
int         odx_supported(const odx_problem* P, const odx_stepper* S);
/* Number of CUDA kernels this library has launched in this process (a
 * monotone counter, used to report `gpu_launches` in bench.py).            */
int64_t     odx_launch_count(void);
/* Name of the device path (kernel family) the last odx_solve / odx_solve_host
 * on this host thread launched ("" before any): diagnostics and bench labels. */
const char* odx_last_route(void);

/* ---- the solver ------------------------------------------------------------
 * Replaces odescan.solve()  newton_pint.py:326-406 (batched over B
 * independent trajectories).  X holds the initial guess on entry
 * and the final iterate on exit (the guess policy is built by the caller,
 * newton_pint.py:352-355).  For every trajectory b:
 *   hist[b*(max_iters+1)+it]        = ||h(xi^(it))||_inf   (NaN-ignoring, _kernels.py:84-95)
 *   scaled_hist[b*(max_iters+1)+it] = max|ce| (implicit) or == hist (explicit)
 *   iters[b]   = iterations_run, status[b] = ODX_ST_*, status_index[b] = the
 *   iteration (NONFINITE) or block index (SINGULAR), -1 otherwise.
 * hist / scaled_hist may be NULL.  Workspace: odx_solve_workspace_bytes().
 * Trajectories of up to 2048 steps (1024 for d = 4) run one CTA each in one
 * launch; longer ones (and d = 64) run one after another on the stream.      */
size_t odx_solve_workspace_bytes(const odx_problem* P, const odx_stepper* S,
                                 int64_t B, int64_t N, const odx_newton_cfg* C);
int odx_solve(const odx_problem* P, const odx_stepper* S,
              const double* x0, double* X, int64_t B, int64_t N, double dt,
              const odx_newton_cfg* C,
              double* hist, double* scaled_hist,
              int32_t* iters, int32_t* status, int64_t* status_index,
              void* workspace, size_t workspace_bytes, void* stream);

/* The same solve with HOST buffers (numpy-in / numpy-out, as the reference's
 * solve() is called): x0 (B*d), X_guess (B*N*d) in; X_out (may alias
 * X_guess), hist / scaled_hist (B*(max_iters+1), entries past the iterations
 * run set to NaN; may be NULL), iters, status, status_index (B) out.  One H2D
 * and one D2H through cached pinned staging (a large batch of resident
 * trajectories is cut into up to 8 batch chunks whose copies and solves
 * overlap on internal streams, forked from and joined back into `stream`);
 * blocks until the result is on the host.  Device buffers and workspace are
 * cached per device (grow-only). */
int odx_solve_host(const odx_problem* P, const odx_stepper* S,
                   const double* x0, const double* X_guess, double* X_out,
                   int64_t B, int64_t N, double dt, const odx_newton_cfg* C,
                   double* hist, double* scaled_hist,
                   int32_t* iters, int32_t* status, int64_t* status_index, void* stream);

/* Host staging-copy threads of odx_solve_host — the counterpart of
 * odescan.threads (threads.py:17-32: max_threads / set_threads).  The pool is
 * sized once (ODX_HOST_THREADS, default min(8, cores/2)); set clamps n into
 * [1, max] and returns the count now used.                                  */
int odx_host_threads_max(void);
int odx_set_host_threads(int n);

/* The starting iterate built on the device (newton_pint.initial_guess
 * :174-207): X (B x N x d, device) from x0 (B x d, device) by an
 * ODX_GUESS_* policy; dt = (tf - t0) / N as the reference computes it
 * (coarse_euler: stride max(1, N/100), v += (stride*dt) f(v), each coarse
 * value held over the next stride rows).                                    */
int odx_initial_guess(const odx_problem* P, int32_t policy, const double* x0, double* X,
                      int64_t B, int64_t N, double dt, void* stream);

/* Sequential marchers (baselines.solve_sequential_*), one GPU thread per
 * trajectory, d <= 4.  Explicit stepper: _kernels.seq_explicit :345-360,
 * X[b,k] = state after k+1 steps.  Implicit: _kernels.seq_implicit :467-526,
 * a per-step Newton solve (tol, max_inner); status[b] (device int64) = -1,
 * -(k+2) for a singular step-k system, or k when step k did not converge
 * (X rows from that step on are left unwritten).                            */
int odx_seq_march(const odx_problem* P, const odx_stepper* S, const double* x0, double* X,
                  int64_t B, int64_t N, double dt, double tol, int32_t max_inner,
                  int64_t* status, void* stream);

/* Parareal's sequential coarse sweep (baselines.solve_parareal :164-227) on
 * the device: mode 0 nodes[0..m] = x0, G(x0), G(G(x0)), ... and g_prev = the
 * G values; mode 1 nodes[k+1] = G(nodes[k]) + fine[k, sub-1] - g_prev[k]
 * (g_prev updated).  G = one step of the explicit S_coarse of dt_coarse.
 * The fine passes are odx_seq_march over the m start nodes.               */
int odx_parareal_coarse(const odx_problem* P, const odx_stepper* S_coarse, const double* x0,
                        double* nodes, double* g_prev, const double* fine, int32_t m,
                        int64_t sub, double dt_coarse, int32_t mode, void* stream);

/* ---- piecewise ops mirroring the reference's compiled loops ---------------- */
/* _kernels.build_explicit  _kernels.py:299-342 (+ _rk_increment_with_jac :261-296) */
int odx_build_explicit(const odx_problem* P, const odx_stepper* S,
                       const double* x0, const double* X, int64_t N, double dt,
                       double* Fe, double* ce, double* h, void* stream);
/* _kernels.build_implicit  _kernels.py:393-464; *first_bad (device int64) = -1 or k */
int odx_build_implicit(const odx_problem* P, const odx_stepper* S,
                       const double* x0, const double* X, int64_t N, double dt,
                       double* Fe, double* ce, double* h, int64_t* first_bad,
                       void* stream);
/* _kernels.scan_affine  _kernels.py:116-233 (inclusive scan, Fp may be NULL) */
size_t odx_scan_affine_workspace_bytes(int64_t N, int32_t d);
int odx_scan_affine(const double* Fin, const double* cin, int64_t N, int32_t d,
                    double* Fp, double* cp, void* workspace,
                    size_t workspace_bytes, void* stream);
/* _kernels.max_abs  _kernels.py:84-95 (NaN-ignoring); *out is a device double */
int odx_max_abs(const double* A, int64_t n, int32_t d, double* out, void* stream);
/* _kernels.add_inplace  _kernels.py:98-103 */
int odx_add_inplace(double* X, const double* U, int64_t n, int32_t d, void* stream);

/* ---- time-sharded solve (one rank per GPU) ----------------------
 * Rank r owns steps [offset, offset+N_local) of one trajectory; `halo` is the
 * state before its first step (x0 on rank 0, the last state of rank r-1
 * otherwise).  d <= 4 problems run every entry point below; the d = 64
 * Allen-Cahn path (cfg4) runs odx_shard_local, odx_shard_decide_step,
 * odx_shard_fixup and odx_solve_sharded (its record carries the 64 x 64 rank
 * aggregate).  Per Newton iteration of the reference loop
 * (newton_pint.py:366-396):
 *   odx_shard_local  builds the local elements (_kernels.py:299-342 /
 *                    :393-464; F is zeroed only at the global step 0), scans
 *                    them into the workspace and writes a record of
 *                    ODX_SHARD_REC(d) doubles:
 *                    [F_agg (d*d) | c_agg (d) | x_last (d) | rn | sc | step_prev | bad]
 *                    (step_prev is NaN; the caller stores the previous step there)
 *   (caller)         all-gathers the records (NCCL) and takes solve()'s decision
 *   odx_shard_fixup  folds the carry of ranks < r from the gathered records,
 *                    X_local += Fp_k z + cp_k, *step_out = max|dx| (NaN-ignoring),
 *                    and halo += carry (rank r-1's last dx, bit-identical), so
 *                    the halo needs no second exchange.
 *   odx_shard_step   odx_shard_fixup of iteration it fused with
 *                    odx_shard_local of iteration it+1: one pass over the
 *                    rank's steps applies the update and builds the next
 *                    elements while the new rows are in registers.  The
 *                    record's step_prev slot is filled (this rank's max|dx|).
 *                    Protocol: local once, then per continuing iteration:
 *                    all-gather, decide, step.  Requires a preceding local or
 *                    step on the same workspace.
 *   odx_shard_decide_step  the same step preceded by solve()'s decision for
 *                    iteration `it`, taken ON THE DEVICE from the gathered
 *                    records (identical on every rank): hist / scaled_hist
 *                    [it] are written, state = {stopped, status, iterations,
 *                    status_index} (int64, device) is set when the solve
 *                    stops, and every later call is a no-op.  The host
 *                    enqueues local, then per it = 0..max_iters: all-gather,
 *                    decide_step — no host round trip per iteration; it reads
 *                    state when it chooses to (e.g. every few iterations).
 * The workspace must be the same buffer for all calls of a solve; X_local
 * must be 16-byte aligned (it is streamed with TMA bulk copies).             */
#define ODX_SHARD_REC(d) ((d) * (d) + 2 * (d) + 4)
size_t odx_shard_workspace_bytes(const odx_problem* P, const odx_stepper* S,
                                 int64_t N_local);
int odx_shard_local(const odx_problem* P, const odx_stepper* S,
                    const double* halo, const double* X_local, int64_t N_local,
                    int64_t offset, double dt, double* record,
                    void* workspace, size_t workspace_bytes, void* stream);
int odx_shard_fixup(const odx_problem* P, const double* records, int32_t rank,
                    int32_t nranks, double* X_local, int64_t N_local, double* halo,
                    double* step_out, void* workspace, size_t workspace_bytes,
                    void* stream);
int odx_shard_step(const odx_problem* P, const odx_stepper* S, const double* records,
                   int32_t rank, int32_t nranks, double* halo, double* X_local,
                   int64_t N_local, int64_t offset, double dt, double* record,
                   void* workspace, size_t workspace_bytes, void* stream);
int odx_shard_decide_step(const odx_problem* P, const odx_stepper* S,
                          const odx_newton_cfg* C, const double* records, int32_t rank,
                          int32_t nranks, int32_t it, double* halo, double* X_local,
                          int64_t N_local, int64_t offset, double dt, double* record,
                          double* hist, double* scaled_hist, int64_t* state,
                          void* workspace, size_t workspace_bytes, void* stream);

/* ---- the whole time-sharded solve natively (SURVEY §8b odx_solve_sharded) ----
 * One call per rank runs odx_shard_local, then per iteration it = 0..max_iters
 * ncclAllGather(record -> records) + odx_shard_decide_step, everything on
 * `stream` (no host round trip).  comm is an ncclComm_t of the process's
 * libnccl.so.2 (odx_nccl_comm_init makes one; a communicator created by the
 * caller with the same library works too).  halo: device, d doubles (x0 on rank
 * 0, else rank r-1's last guess row; not modified).  state: device int64[4]
 * {stopped, status, iterations, status_index}; hist / scaled_hist: device,
 * max_iters + 1 (entries past the stop untouched; may be NULL).  poll > 0:
 * read the stop flag every `poll` iterations (a stream sync) and stop
 * enqueuing once stopped — identical on every rank; poll = 0: fully
 * asynchronous (iterations after the stop are no-ops).                        */
int    odx_nccl_available(void);
int    odx_nccl_unique_id(void* id /* 128 bytes */);
int    odx_nccl_comm_init(void** comm, int32_t nranks, const void* id, int32_t rank);
int    odx_nccl_comm_destroy(void* comm);
size_t odx_solve_sharded_workspace_bytes(const odx_problem* P, const odx_stepper* S,
                                         int64_t N_local, int32_t nranks);
int    odx_solve_sharded(const odx_problem* P, const odx_stepper* S, const odx_newton_cfg* C,
                         void* comm, int32_t rank, int32_t nranks, const double* halo,
                         double* X_local, int64_t N_local, int64_t offset, double dt,
                         double* hist, double* scaled_hist, int64_t* state, int32_t poll,
                         void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ODESCAN_B200_H */
