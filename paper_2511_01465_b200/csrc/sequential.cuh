// sequential.cuh — the reference's sequential marchers on the GPU, one thread
// per trajectory: the same-box sequential comparison for
// the parallel Newton solve and a converged-solution reference at large N.
//
//   seq_explicit_kernel  _kernels.seq_explicit :345-360 (+ _rk_increment
//                        :243-258): x <- x + dt sum_i b_i kappa_i
//   seq_implicit_kernel  _kernels.seq_implicit :467-526: per step a Newton
//                        solve of x - x_prev - dt (w_p f(x_prev) + w_n f(x)) = 0
//                        warm-started at x_prev, pivoted LU, tol / max_inner;
//                        status -1, -(k+2) singular at k, or k (no convergence)
#pragma once

#include "common.cuh"
#include "elements.cuh"

namespace odx {

template <class P, int S>
__global__ void seq_explicit_kernel(ProbParams pp, StepCoefs sc, const double* x0, double* X,
                                    long long B, long long N) {
    constexpr int D = P::D;
    const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const P prob(pp);
    double x[D];
#pragma unroll
    for (int r = 0; r < D; r++) x[r] = x0[b * D + r];
    double* Xb = X + b * N * D;
    for (long long k = 0; k < N; k++) {
        double kap[S][D];
#pragma unroll
        for (int i = 0; i < S; i++) {
            double xs[D];
#pragma unroll
            for (int r = 0; r < D; r++) {
                double acc = x[r];
#pragma unroll
                for (int j = 0; j < i; j++) acc += sc.dta[i * S + j] * kap[j][r];
                xs[r] = acc;
            }
            prob.f(xs, kap[i]);
        }
#pragma unroll
        for (int r = 0; r < D; r++) {
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < S; i++) acc += sc.b[i] * kap[i][r];
            x[r] = x[r] + sc.dt * acc;
            Xb[k * D + r] = x[r];
        }
    }
}

template <class P>
__global__ void seq_implicit_kernel(ProbParams pp, StepCoefs sc, double tol, int max_inner,
                                    const double* x0, double* X, long long B, long long N,
                                    long long* status) {
    constexpr int D = P::D;
    const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const P prob(pp);
    double xprev[D], x[D], fp[D], fx[D], r[D];
#pragma unroll
    for (int i = 0; i < D; i++) xprev[i] = x0[b * D + i];
    double* Xb = X + b * N * D;
    long long st = -1;
    for (long long k = 0; k < N && st == -1; k++) {
        prob.f(xprev, fp);
#pragma unroll
        for (int i = 0; i < D; i++) x[i] = xprev[i];
        bool converged = false;
        for (int it = 0; it < max_inner; it++) {
            prob.f(x, fx);
            double rn = 0.0;
#pragma unroll
            for (int i = 0; i < D; i++) {
                r[i] = x[i] - xprev[i] - sc.dt * (sc.w_prev * fp[i] + sc.w_next * fx[i]);
                const double av = fabs(r[i]);
                if (av > rn) rn = av;
            }
            if (rn <= tol) {
                converged = true;
                break;
            }
            double A[D * D];
            prob.jac(x, A);
#pragma unroll
            for (int i = 0; i < D; i++)
#pragma unroll
                for (int j = 0; j < D; j++)
                    A[i * D + j] = __dsub_rn((i == j) ? 1.0 : 0.0, __dmul_rn(sc.dt_wnext, A[i * D + j]));
            int piv[D];
            double rinv[D];
            if (lu_factor_reg<D>(A, piv, rinv) >= 0) {
                st = -(k + 2);
                break;
            }
            lu_solve_reg<D>(A, piv, rinv, r);
#pragma unroll
            for (int i = 0; i < D; i++) x[i] -= r[i];
        }
        if (st != -1) break;
        if (!converged) {  // the last update was never checked
            prob.f(x, fx);
            double rn = 0.0;
#pragma unroll
            for (int i = 0; i < D; i++) {
                const double rv = x[i] - xprev[i] - sc.dt * (sc.w_prev * fp[i] + sc.w_next * fx[i]);
                const double av = fabs(rv);
                if (av > rn) rn = av;
            }
            if (rn > tol) {
                st = k;
                break;
            }
        }
#pragma unroll
        for (int i = 0; i < D; i++) {
            Xb[k * D + i] = x[i];
            xprev[i] = x[i];
        }
    }
    status[b] = st;
}

// Parareal's sequential coarse sweep (baselines.solve_parareal :164-227), one
// thread: mode 0 initialises the nodes with the coarse propagator G (one
// explicit step of dt_coarse per interval); mode 1 applies the correction
//   nodes[k+1] <- G(nodes[k]^new) + F(nodes[k]^old) - G(nodes[k]^old)
// with F = the last state of interval k's fine pass (fine: m x sub x d).
template <class P, int S>
__global__ void parareal_coarse_kernel(ProbParams pp, StepCoefs sc, const double* x0,
                                       double* nodes, double* g_prev, const double* fine, int m,
                                       long long sub, int mode) {
    constexpr int D = P::D;
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const P prob(pp);
    double x[D];
#pragma unroll
    for (int r = 0; r < D; r++) {
        x[r] = x0[r];
        nodes[r] = x0[r];
    }
    for (int k = 0; k < m; k++) {
        double kap[S][D];
#pragma unroll
        for (int i = 0; i < S; i++) {
            double xs[D];
#pragma unroll
            for (int r = 0; r < D; r++) {
                double acc = x[r];
#pragma unroll
                for (int j = 0; j < i; j++) acc += sc.dta[i * S + j] * kap[j][r];
                xs[r] = acc;
            }
            prob.f(xs, kap[i]);
        }
#pragma unroll
        for (int r = 0; r < D; r++) {
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < S; i++) acc += sc.b[i] * kap[i][r];
            const double g = x[r] + sc.dt * acc;  // G(x) = x + coarse increment
            double nxt;
            if (mode == 0) {
                nxt = g;
            } else {
                const double fe = fine[((long long)k * sub + (sub - 1)) * D + r];
                nxt = g + fe - g_prev[k * D + r];
            }
            g_prev[k * D + r] = g;
            nodes[(k + 1) * D + r] = nxt;
            x[r] = nxt;
        }
    }
}

template <class P, int KIND, int S>
int parareal_coarse(const ProbParams& pp, const StepCoefs& sc, const double* x0, double* nodes,
                    double* g_prev, const double* fine, int m, long long sub, int mode,
                    cudaStream_t st) {
    if constexpr (KIND != 0) {
        return fail(ODX_EINVAL, "parareal needs an explicit coarse stepper");
    } else {
        parareal_coarse_kernel<P, S><<<1, 32, 0, st>>>(pp, sc, x0, nodes, g_prev, fine, m, sub, mode);
        ODX_CUDA(cudaGetLastError());
        count_launch(1);
        return ODX_OK;
    }
}

template <class P, int KIND, int S>
int seq_march(const ProbParams& pp, const StepCoefs& sc, double tol, int max_inner,
              const double* x0, double* X, long long B, long long N, long long* status,
              cudaStream_t st) {
    const unsigned blocks = (unsigned)((B + 63) / 64);
    if constexpr (KIND == 0) {
        seq_explicit_kernel<P, S><<<blocks, 64, 0, st>>>(pp, sc, x0, X, B, N);
    } else {
        seq_implicit_kernel<P><<<blocks, 64, 0, st>>>(pp, sc, tol, max_inner, x0, X, B, N, status);
    }
    ODX_CUDA(cudaGetLastError());
    count_launch(1);
    return ODX_OK;
}

}  // namespace odx
