// abi.cu — the extern "C" boundary (include/odescan_b200.h).  Validates
// descriptors, converts them to kernel parameters and dispatches to the
// templated device paths.  No exception crosses this boundary; errors are
// negative codes plus a thread-local message (odx_last_error).
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "common.cuh"
#include "dispatch.cuh"
#include "solve_small.cuh"

namespace odx {

extern thread_local std::string g_err;
extern std::atomic<long long> g_launches;
extern thread_local const char* g_route;

template <class P, int KIND, int S>
int solve_small(SolveParams& p, void* ws, size_t ws_bytes, cudaStream_t st, bool query,
                size_t* need);
template <class P, int KIND, int S>
int build_op(const ProbParams& pp, const StepCoefs& sc, const double* x0, const double* X,
             long long N, double* Fe, double* ce, double* h, long long* first_bad,
             cudaStream_t st, long long offset);
template <class P, int KIND, int S>
int seq_march(const ProbParams& pp, const StepCoefs& sc, double tol, int max_inner,
              const double* x0, double* X, long long B, long long N, long long* status,
              cudaStream_t st);
template <class P, int KIND, int S>
int parareal_coarse(const ProbParams& pp, const StepCoefs& sc, const double* x0, double* nodes,
                    double* g_prev, const double* fine, int m, long long sub, int mode,
                    cudaStream_t st);
template <class P, int KIND, int S>
int shard_tiled_local(const ProbParams& pp, const StepCoefs& sc, const double* halo,
                      const double* X_local, long long n, long long offset, double* record,
                      void* ws, size_t ws_bytes, cudaStream_t st, int fused);
int scan_op(const double* F, const double* c, long long N, int d, double* Fp, double* cp,
            void* ws, size_t ws_bytes, cudaStream_t st);
size_t scan_op_ws(long long N, int d);
int max_abs_op(const double* A, long long n, int d, double* out, cudaStream_t st);
int add_op(double* X, const double* U, long long n, int d, cudaStream_t st);

// d = 64 dense path (solve_dense.cu)
int dense_supported(const odx_problem* P, const odx_stepper* S);
int dense_shard_local(const ProbParams& pp, const StepCoefs& sc, const double* halo,
                      const double* X_local, long long n, long long offset, double* record,
                      void* ws, size_t ws_bytes, cudaStream_t st, bool device_decided);
int dense_shard_decide_step(const double* records, int rank, int nranks, int it, int max_iters,
                            int abort_nonfinite, double rtol, double stol, double* hist,
                            double* shist, long long* state, const ProbParams& pp,
                            const StepCoefs& sc, double* halo, double* X_local, long long n,
                            long long offset, double* record, void* ws, size_t ws_bytes,
                            cudaStream_t st);
int dense_solve(const odx_problem* P, const odx_stepper* S, SolveParams& p, void* ws,
                size_t ws_bytes, cudaStream_t st, bool query, size_t* need);
int dense_build_op(const odx_problem* P, const odx_stepper* S, const StepCoefs& sc,
                   const double* x0, const double* X, long long N, double* Fe, double* ce,
                   double* h, long long* first_bad, cudaStream_t st);
int dense_scan_op(const double* F, const double* c, long long N, int d, double* Fp, double* cp,
                  void* ws, size_t ws_bytes, cudaStream_t st);
size_t dense_scan_op_ws(long long N, int d);

// Stage-count / kind dispatch for a fixed problem type.
template <class P, class Fn>
int with_stepper(const odx_stepper* S, Fn&& fn) {
    if (S->kind == ODX_STEP_IMPLICIT_WEIGHTED) return fn.template operator()<P, 1, 1>();
    switch (S->stages) {
    case 1: return fn.template operator()<P, 0, 1>();
    case 2: return fn.template operator()<P, 0, 2>();
    case 3: return fn.template operator()<P, 0, 3>();
    case 4: return fn.template operator()<P, 0, 4>();
    default: return ODX_EUNSUPPORTED;
    }
}

struct ProbeFn {
    const odx_stepper* S;
    template <class PP>
    int operator()() {
        return with_stepper<PP>(S, [&]<class Q, int K, int SS>() { return 1; }) == 1 ? 1 : 0;
    }
};

struct SolveFn {
    const odx_stepper* S;
    SolveParams* p;
    void* ws;
    size_t ws_bytes;
    cudaStream_t st;
    bool query;
    size_t* need;
    template <class PP>
    int operator()() {
        return with_stepper<PP>(S, [&]<class Q, int K, int SS>() {
            return solve_small<Q, K, SS>(*p, ws, ws_bytes, st, query, need);
        });
    }
};

struct BuildFn {
    const odx_stepper* S;
    const ProbParams* pp;
    const StepCoefs* sc;
    const double *x0, *X;
    long long N;
    double *Fe, *ce, *h;
    long long* fb;
    cudaStream_t st;
    long long offset = 0;
    template <class PP>
    int operator()() {
        return with_stepper<PP>(S, [&]<class Q, int K, int SS>() {
            return build_op<Q, K, SS>(*pp, *sc, x0, X, N, Fe, ce, h, fb, st, offset);
        });
    }
};

struct SeqFn {
    const odx_stepper* S;
    const ProbParams* pp;
    const StepCoefs* sc;
    double tol;
    int max_inner;
    const double* x0;
    double* X;
    long long B, N;
    long long* status;
    cudaStream_t st;
    template <class PP>
    int operator()() {
        return with_stepper<PP>(S, [&]<class Q, int K, int SS>() {
            return seq_march<Q, K, SS>(*pp, *sc, tol, max_inner, x0, X, B, N, status, st);
        });
    }
};

struct PararealFn {
    const odx_stepper* S;
    const ProbParams* pp;
    const StepCoefs* sc;
    const double* x0;
    double *nodes, *g_prev;
    const double* fine;
    int m;
    long long sub;
    int mode;
    cudaStream_t st;
    template <class PP>
    int operator()() {
        return with_stepper<PP>(S, [&]<class Q, int K, int SS>() {
            return parareal_coarse<Q, K, SS>(*pp, *sc, x0, nodes, g_prev, fine, m, sub, mode, st);
        });
    }
};

struct ShardLocalFn {
    const odx_stepper* S;
    const ProbParams* pp;
    const StepCoefs* sc;
    const double *halo, *X;
    long long n, offset;
    double* record;
    void* ws;
    size_t ws_bytes;
    cudaStream_t st;
    int fused;
    template <class PP>
    int operator()() {
        return with_stepper<PP>(S, [&]<class Q, int K, int SS>() {
            return shard_tiled_local<Q, K, SS>(*pp, *sc, halo, X, n, offset, record, ws, ws_bytes, st,
                                               fused);
        });
    }
};

static int check_problem(const odx_problem* P, const odx_stepper* S) {
    if (!P || !S) return fail(ODX_EINVAL, "null problem or stepper descriptor");
    if (P->dim < 1 || P->dim > 64) return fail(ODX_EINVAL, "dim must be in [1, 64]");
    if (P->problem_id < 0 || P->problem_id >= ODX_NUM_PROBLEMS)
        return fail(ODX_EUNSUPPORTED, "unknown problem id (no device functor)");
    return ODX_OK;
}

}  // namespace odx

using namespace odx;

extern "C" {

int odx_abi_version(void) { return ODX_ABI_VERSION; }

const char* odx_last_error(void) { return g_err.c_str(); }

int64_t odx_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* odx_last_route(void) { return g_route; }

int odx_supported(const odx_problem* P, const odx_stepper* S) {
    if (check_problem(P, S) != ODX_OK) return 0;
    StepCoefs sc;
    if (!fill_coefs(S, 1.0, sc)) return 0;
    if (dense_supported(P, S)) return 1;
    int r = with_small_problem(P->problem_id, P->dim, ProbeFn{S});
    return r == 1 ? 1 : 0;
}

static int make_solve_params(const odx_problem* P, const odx_stepper* S, const double* x0,
                             double* X, int64_t B, int64_t N, double dt, const odx_newton_cfg* C,
                             double* hist, double* shist, int32_t* iters, int32_t* status,
                             int64_t* sidx, SolveParams& p) {
    int rc = check_problem(P, S);
    if (rc) return rc;
    if (!C || C->max_iters < 1) return fail(ODX_EINVAL, "max_iters must be at least 1");
    if (C->residual_tol < 0.0 || C->step_tol < 0.0) return fail(ODX_EINVAL, "negative tolerance");
    if (B < 1 || N < 1) return fail(ODX_EINVAL, "need B >= 1 and N >= 1");
    if (!(dt > 0.0)) return fail(ODX_EINVAL, "dt must be positive");
    std::memset(&p, 0, sizeof(p));
    if (!fill_params(P, p.prob)) return fail(ODX_EINVAL, "bad problem parameters");
    if (!fill_coefs(S, dt, p.sc)) return fail(ODX_EINVAL, "bad stepper descriptor");
    p.x0 = x0;
    p.X = X;
    p.B = B;
    p.N = N;
    p.max_iters = C->max_iters;
    p.abort_nonfinite = C->abort_nonfinite;
    p.rtol = C->residual_tol;
    p.stol = C->step_tol;
    p.hist = hist;
    p.shist = shist;
    p.iters = iters;
    p.status = status;
    p.sidx = reinterpret_cast<long long*>(sidx);
    return ODX_OK;
}

static int solve_impl(const odx_problem* P, const odx_stepper* S, SolveParams& p, void* ws,
                      size_t ws_bytes, cudaStream_t st, bool query, size_t* need);

// B > 1 trajectories longer than the batched kernel takes (and the d = 64
// path, one trajectory per launch): the single-trajectory solve per
// trajectory, back to back on the stream, sharing the workspace.  A
// trajectory whose rows are not 16-byte aligned (odd N * d) is staged through
// an aligned copy at the front of the workspace (the streaming kernels move
// rows with TMA).
static int solve_each(const odx_problem* P, const odx_stepper* S, SolveParams& p, void* ws,
                      size_t ws_bytes, cudaStream_t st, bool query, size_t* need) {
    const long long d = P->dim;
    const size_t xbytes = (size_t)p.N * (size_t)d * 8;
    const size_t stage = align_up(xbytes, 256) + 256;
    SolveParams q = p;
    q.B = 1;
    size_t one = 0;
    if (int rc = solve_impl(P, S, q, nullptr, 0, st, true, &one)) return rc;
    if (query) {
        *need = stage + one;
        return ODX_OK;
    }
    if (!ws || ws_bytes < stage + one) return fail(ODX_EWORKSPACE, "workspace too small");
    char* base = reinterpret_cast<char*>(align_up(reinterpret_cast<size_t>(ws), 256));
    double* scratch = reinterpret_cast<double*>(base);
    void* ws1 = base + stage - 256;
    const size_t ws1_bytes = ws_bytes - (size_t)(static_cast<char*>(ws1) - static_cast<char*>(ws));
    const long long H = p.max_iters + 1;
    for (long long b = 0; b < p.B; b++) {
        double* Xb = p.X + b * p.N * d;
        const bool aligned = (reinterpret_cast<uintptr_t>(Xb) & 15) == 0;
        q.x0 = p.x0 + b * d;
        q.X = aligned ? Xb : scratch;
        q.hist = p.hist ? p.hist + b * H : nullptr;
        q.shist = p.shist ? p.shist + b * H : nullptr;
        q.iters = p.iters + b;
        q.status = p.status + b;
        q.sidx = p.sidx + b;
        if (!aligned) ODX_CUDA(cudaMemcpyAsync(scratch, Xb, xbytes, cudaMemcpyDeviceToDevice, st));
        if (int rc = solve_impl(P, S, q, ws1, ws1_bytes, st, false, nullptr)) return rc;
        if (!aligned) ODX_CUDA(cudaMemcpyAsync(Xb, scratch, xbytes, cudaMemcpyDeviceToDevice, st));
    }
    return ODX_OK;
}

static int solve_impl(const odx_problem* P, const odx_stepper* S, SolveParams& p, void* ws,
                      size_t ws_bytes, cudaStream_t st, bool query, size_t* need) {
    const bool long_traj = dense_supported(P, S) || p.N > resident_max_steps(P->dim);
    if (long_traj && p.B > 1) return solve_each(P, S, p, ws, ws_bytes, st, query, need);
    if (long_traj && !query && (reinterpret_cast<uintptr_t>(p.X) & 15) != 0) {
        // one misaligned trajectory: staged when the workspace has room for the
        // copy (a B > 1 query's size), else the kernels report the alignment
        size_t each = 0;
        if (solve_each(P, S, p, nullptr, 0, st, true, &each) == ODX_OK && ws_bytes >= each)
            return solve_each(P, S, p, ws, ws_bytes, st, false, nullptr);
    }
    if (dense_supported(P, S)) return dense_solve(P, S, p, ws, ws_bytes, st, query, need);
    int rc = with_small_problem(P->problem_id, P->dim, SolveFn{S, &p, ws, ws_bytes, st, query, need});
    if (rc == ODX_EUNSUPPORTED && odx_last_error()[0] == 0)
        set_error("no device path for problem %d with dim %d", P->problem_id, P->dim);
    if (rc == ODX_EINVAL) set_error("problem %d does not have dim %d", P->problem_id, P->dim);
    return rc;
}

size_t odx_solve_workspace_bytes(const odx_problem* P, const odx_stepper* S, int64_t B,
                                 int64_t N, const odx_newton_cfg* C) {
    SolveParams p;
    if (make_solve_params(P, S, nullptr, nullptr, B, N, 1.0, C, nullptr, nullptr, nullptr,
                          nullptr, nullptr, p) != ODX_OK)
        return 0;
    size_t need = 0;
    if (solve_impl(P, S, p, nullptr, 0, nullptr, true, &need) != ODX_OK) return 0;
    return need;
}

int odx_solve(const odx_problem* P, const odx_stepper* S, const double* x0, double* X, int64_t B,
              int64_t N, double dt, const odx_newton_cfg* C, double* hist, double* scaled_hist,
              int32_t* iters, int32_t* status, int64_t* status_index, void* workspace,
              size_t workspace_bytes, void* stream) {
    g_err.clear();
    g_route = "";
    SolveParams p;
    int rc = make_solve_params(P, S, x0, X, B, N, dt, C, hist, scaled_hist, iters, status,
                               status_index, p);
    if (rc) return rc;
    if (!x0 || !X || !iters || !status || !status_index)
        return fail(ODX_EINVAL, "null device buffer");
    return solve_impl(P, S, p, workspace, workspace_bytes, (cudaStream_t)stream, false, nullptr);
}

}  // extern "C"

namespace odx {
int build_common_offset(const odx_problem* P, const odx_stepper* S, int kind, const double* x0,
                        const double* X, int64_t N, double dt, double* Fe, double* ce, double* h,
                        int64_t* first_bad, void* stream, long long offset);
}

extern "C" {

static int build_common(const odx_problem* P, const odx_stepper* S, int kind, const double* x0,
                        const double* X, int64_t N, double dt, double* Fe, double* ce, double* h,
                        int64_t* first_bad, void* stream) {
    return odx::build_common_offset(P, S, kind, x0, X, N, dt, Fe, ce, h, first_bad, stream, 0);
}

}  // extern "C"

namespace odx {
int build_common_offset(const odx_problem* P, const odx_stepper* S, int kind, const double* x0,
                        const double* X, int64_t N, double dt, double* Fe, double* ce, double* h,
                        int64_t* first_bad, void* stream, long long offset) {
    g_err.clear();
    int rc = check_problem(P, S);
    if (rc) return rc;
    if (S->kind != kind) return fail(ODX_EINVAL, "stepper kind does not match the build op");
    if (N < 0) return fail(ODX_EINVAL, "N must be >= 0");
    ProbParams pp;
    StepCoefs sc;
    if (!fill_params(P, pp)) return fail(ODX_EINVAL, "bad problem parameters");
    if (!fill_coefs(S, dt, sc)) return fail(ODX_EINVAL, "bad stepper descriptor");
    if (kind == ODX_STEP_IMPLICIT_WEIGHTED && !first_bad)
        return fail(ODX_EINVAL, "first_bad must be a device int64 pointer");
    cudaStream_t st = (cudaStream_t)stream;
    if (dense_supported(P, S))
        return dense_build_op(P, S, sc, x0, X, N, Fe, ce, h,
                              reinterpret_cast<long long*>(first_bad), st);
    BuildFn fn{S, &pp, &sc, x0, X, N, Fe, ce, h, reinterpret_cast<long long*>(first_bad), st};
    fn.offset = offset;
    return with_small_problem(P->problem_id, P->dim, fn);
}

// the d = 64 shard's device-decided step (shard.cu validates)
int shard_dense_decide_dispatch(const odx_problem* P, const odx_stepper* S, double dt,
                                const odx_newton_cfg* C, const double* records, int rank,
                                int nranks, int it, double* halo, double* X_local, long long n,
                                long long offset, double* record, double* hist, double* shist,
                                long long* state, void* ws, size_t ws_bytes, cudaStream_t st) {
    ProbParams pp;
    StepCoefs sc;
    if (!fill_params(P, pp)) return fail(ODX_EINVAL, "bad problem parameters");
    if (!fill_coefs(S, dt, sc)) return fail(ODX_EINVAL, "bad stepper descriptor");
    return dense_shard_decide_step(records, rank, nranks, it, C->max_iters, C->abort_nonfinite,
                                   C->residual_tol, C->step_tol, hist, shist, state, pp, sc, halo,
                                   X_local, n, offset, record, ws, ws_bytes, st);
}

// one rank's local pass of the time-sharded iteration (shard.cu validates)
int shard_local_dispatch(const odx_problem* P, const odx_stepper* S, double dt,
                         const double* halo, const double* X_local, long long n, long long offset,
                         double* record, void* ws, size_t ws_bytes, cudaStream_t st, int fused) {
    ProbParams pp;
    StepCoefs sc;
    if (!fill_params(P, pp)) return fail(ODX_EINVAL, "bad problem parameters");
    if (!fill_coefs(S, dt, sc)) return fail(ODX_EINVAL, "bad stepper descriptor");
    if (dense_supported(P, S)) {
        if (fused) return fail(ODX_EUNSUPPORTED, "the d = 64 shard runs the two-pass protocol");
        return dense_shard_local(pp, sc, halo, X_local, n, offset, record, ws, ws_bytes, st, false);
    }
    ShardLocalFn fn{S, &pp, &sc, halo, X_local, n, offset, record, ws, ws_bytes, st, fused};
    return with_small_problem(P->problem_id, P->dim, fn);
}
}  // namespace odx

extern "C" {

int odx_seq_march(const odx_problem* P, const odx_stepper* S, const double* x0, double* X,
                  int64_t B, int64_t N, double dt, double tol, int32_t max_inner,
                  int64_t* status, void* stream) {
    g_err.clear();
    int rc = check_problem(P, S);
    if (rc) return rc;
    if (P->dim > 4) return fail(ODX_EUNSUPPORTED, "sequential marchers support d <= 4");
    if (!x0 || !X || B < 1 || N < 0) return fail(ODX_EINVAL, "bad buffers or extents");
    if (S->kind == ODX_STEP_IMPLICIT_WEIGHTED && (!status || max_inner < 1 || !(tol >= 0.0)))
        return fail(ODX_EINVAL, "implicit march needs status, max_inner >= 1 and tol >= 0");
    ProbParams pp;
    StepCoefs sc;
    if (!fill_params(P, pp)) return fail(ODX_EINVAL, "bad problem parameters");
    if (!fill_coefs(S, dt, sc)) return fail(ODX_EINVAL, "bad stepper descriptor");
    if (N == 0) return ODX_OK;
    SeqFn fn{S, &pp, &sc, tol, max_inner, x0, X, B, N, reinterpret_cast<long long*>(status),
             (cudaStream_t)stream};
    return with_small_problem(P->problem_id, P->dim, fn);
}

int odx_parareal_coarse(const odx_problem* P, const odx_stepper* S_coarse, const double* x0,
                        double* nodes, double* g_prev, const double* fine, int32_t m,
                        int64_t sub, double dt_coarse, int32_t mode, void* stream) {
    g_err.clear();
    int rc = check_problem(P, S_coarse);
    if (rc) return rc;
    if (P->dim > 4) return fail(ODX_EUNSUPPORTED, "parareal supports d <= 4");
    if (S_coarse->kind != ODX_STEP_EXPLICIT_RK) return fail(ODX_EINVAL, "coarse stepper must be explicit");
    if (!x0 || !nodes || !g_prev || m < 1 || (mode == 1 && (!fine || sub < 1)) || mode < 0 || mode > 1)
        return fail(ODX_EINVAL, "bad parareal buffers or extents");
    ProbParams pp;
    StepCoefs sc;
    if (!fill_params(P, pp)) return fail(ODX_EINVAL, "bad problem parameters");
    if (!fill_coefs(S_coarse, dt_coarse, sc)) return fail(ODX_EINVAL, "bad stepper descriptor");
    PararealFn fn{S_coarse, &pp, &sc, x0, nodes, g_prev, fine, m, sub, mode, (cudaStream_t)stream};
    return with_small_problem(P->problem_id, P->dim, fn);
}

int odx_build_explicit(const odx_problem* P, const odx_stepper* S, const double* x0,
                       const double* X, int64_t N, double dt, double* Fe, double* ce, double* h,
                       void* stream) {
    return build_common(P, S, ODX_STEP_EXPLICIT_RK, x0, X, N, dt, Fe, ce, h, nullptr, stream);
}

int odx_build_implicit(const odx_problem* P, const odx_stepper* S, const double* x0,
                       const double* X, int64_t N, double dt, double* Fe, double* ce, double* h,
                       int64_t* first_bad, void* stream) {
    return build_common(P, S, ODX_STEP_IMPLICIT_WEIGHTED, x0, X, N, dt, Fe, ce, h, first_bad,
                        stream);
}

size_t odx_scan_affine_workspace_bytes(int64_t N, int32_t d) {
    if (N < 0 || d < 1 || d > 64) return 0;
    if (d > 4) return dense_scan_op_ws(N, d);
    return scan_op_ws(N, d);
}

int odx_scan_affine(const double* Fin, const double* cin, int64_t N, int32_t d, double* Fp,
                    double* cp, void* workspace, size_t workspace_bytes, void* stream) {
    g_err.clear();
    if (N < 0 || d < 1 || d > 64) return fail(ODX_EINVAL, "bad N or d");
    if (d > 4)
        return dense_scan_op(Fin, cin, N, d, Fp, cp, workspace, workspace_bytes,
                             (cudaStream_t)stream);
    return scan_op(Fin, cin, N, d, Fp, cp, workspace, workspace_bytes, (cudaStream_t)stream);
}

int odx_max_abs(const double* A, int64_t n, int32_t d, double* out, void* stream) {
    g_err.clear();
    if (n < 0 || d < 1 || !out) return fail(ODX_EINVAL, "bad max_abs arguments");
    return max_abs_op(A, n, d, out, (cudaStream_t)stream);
}

int odx_add_inplace(double* X, const double* U, int64_t n, int32_t d, void* stream) {
    g_err.clear();
    if (n < 0 || d < 1) return fail(ODX_EINVAL, "bad add_inplace arguments");
    return add_op(X, U, n, d, (cudaStream_t)stream);
}

}  // extern "C"
