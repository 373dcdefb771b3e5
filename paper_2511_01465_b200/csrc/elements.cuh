// elements.cuh — per-step residual / scan-element construction in registers,
// the affine element algebra, and the NaN-ignoring max-abs row rule.
//
// Reference: _kernels.py:261-342 (explicit RK elements with chain-ruled
// tangents), :393-464 (implicit weighted elements with a pivoted LU per block),
// :28-77 (LU), :84-95 (max_abs), affine_scan.py:64-78 (combine).
#pragma once

#include <cstdint>

#include "problems.cuh"

namespace odx {

// ---------------------------------------------------------------------------
// Step-map coefficients, precomputed on the host.  dta[i*S+j] = dt*a[i][j] is
// the same double the reference forms inline (`dt * a[i, j] * kap`,
// _kernels.py:271), so precomputing it changes no bits.
// ---------------------------------------------------------------------------
struct StepCoefs {
    double dta[ODX_MAX_STAGES * ODX_MAX_STAGES];
    double b[ODX_MAX_STAGES];
    double dt;
    double dt_wprev;  // dt * w_prev  (_kernels.py:455)
    double dt_wnext;  // dt * w_next  (_kernels.py:430)
    double w_prev, w_next;
    int stages;
};

template <int D>
struct Elem {
    double F[D * D];
    double c[D];
};

// combine(earlier e, later l) = (Fl Fe, Fl ce + cl)   affine_scan.py:64-78
template <int D>
__device__ __forceinline__ void compose(const Elem<D>& e, const Elem<D>& l, Elem<D>& o) {
    Elem<D> t;
#pragma unroll
    for (int r = 0; r < D; r++) {
        double acc = l.c[r];
#pragma unroll
        for (int q = 0; q < D; q++) acc += l.F[r * D + q] * e.c[q];
        t.c[r] = acc;
    }
#pragma unroll
    for (int r = 0; r < D; r++)
#pragma unroll
        for (int s = 0; s < D; s++) {
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < D; q++) acc += l.F[r * D + q] * e.F[q * D + s];
            t.F[r * D + s] = acc;
        }
    o = t;
}

// y = F z + c  (apply an element to a state offset)
template <int D>
__device__ __forceinline__ void apply(const Elem<D>& e, const double* z, double* y) {
    double t[D];
#pragma unroll
    for (int r = 0; r < D; r++) {
        double acc = e.c[r];
#pragma unroll
        for (int q = 0; q < D; q++) acc += e.F[r * D + q] * z[q];
        t[r] = acc;
    }
#pragma unroll
    for (int r = 0; r < D; r++) y[r] = t[r];
}

template <int D>
__device__ __forceinline__ void set_identity(Elem<D>& e) {
#pragma unroll
    for (int r = 0; r < D; r++) {
        e.c[r] = 0.0;
#pragma unroll
        for (int s = 0; s < D; s++) e.F[r * D + s] = (r == s) ? 1.0 : 0.0;
    }
}

// Row rule of _kernels.max_abs (:84-95): loc takes v whenever !(v <= loc), so a
// NaN replaces loc and is replaced again by the next entry; a row whose loc
// ends NaN is dropped by the cross-row max (fmax drops NaN, like numba's
// max(out, nan)).  Results are >= 0 or +inf, so their bit patterns order as
// unsigned integers (atomicMax on the bits).
template <int D>
__device__ __forceinline__ double row_max_abs(const double* v) {
    double loc = 0.0;
#pragma unroll
    for (int j = 0; j < D; j++) {
        double a = fabs(v[j]);
        if (!(a <= loc)) loc = a;
    }
    return loc;
}

__device__ __forceinline__ double nan_drop_max(double acc, double loc) {
    return fmax(acc, loc);  // fmax(acc, NaN) = acc
}

// ---------------------------------------------------------------------------
// Explicit RK element for one step (_kernels.py:261-342).
// prev = x0 (k == 0) or X[k-1]; xk = X[k].  Outputs element (F, c) with
// F = I + dg/dx (0 for k == 0), c = -h, and the residual row h.
// The stage loops run over every j < i including zero tableau entries, as the
// reference does, so non-finite stages propagate identically.
// ---------------------------------------------------------------------------
template <class P, int S>
__device__ __forceinline__ void build_explicit_step(const P& prob, const StepCoefs& sc,
                                                    const double* prev, const double* xk,
                                                    bool first, Elem<P::D>& el, double* h) {
    constexpr int D = P::D;
    double kap[S][D];
    double dkap[S][D * D];
#pragma unroll
    for (int i = 0; i < S; i++) {
        double xs[D];
#pragma unroll
        for (int r = 0; r < D; r++) {
            double acc = prev[r];
#pragma unroll
            for (int j = 0; j < i; j++) acc += sc.dta[i * S + j] * kap[j][r];
            xs[r] = acc;
        }
        prob.f(xs, kap[i]);
        double Js[D * D];
        prob.jac(xs, Js);
        double M[D * D];
#pragma unroll
        for (int r = 0; r < D; r++)
#pragma unroll
            for (int c = 0; c < D; c++) {
                double m = (r == c) ? 1.0 : 0.0;
#pragma unroll
                for (int j = 0; j < i; j++) m += sc.dta[i * S + j] * dkap[j][r * D + c];
                M[r * D + c] = m;
            }
#pragma unroll
        for (int r = 0; r < D; r++)
#pragma unroll
            for (int c = 0; c < D; c++) {
                double acc = 0.0;
#pragma unroll
                for (int q = 0; q < D; q++) acc += Js[r * D + q] * M[q * D + c];
                dkap[i][r * D + c] = acc;
            }
    }
#pragma unroll
    for (int r = 0; r < D; r++) {
        double acc = 0.0;
#pragma unroll
        for (int i = 0; i < S; i++) acc += sc.b[i] * kap[i][r];
        double g = sc.dt * acc;
        double hv = xk[r] - prev[r] - g;
        h[r] = hv;
        el.c[r] = -hv;
    }
#pragma unroll
    for (int r = 0; r < D; r++)
#pragma unroll
        for (int c = 0; c < D; c++) {
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < S; i++) acc += sc.b[i] * dkap[i][r * D + c];
            double jg = sc.dt * acc;
            el.F[r * D + c] = first ? 0.0 : jg + ((r == c) ? 1.0 : 0.0);
        }
}

// NI independent steps built together, stage by stage (the loops over items
// are innermost), so the scheduler sees NI independent dependency chains at
// every point of the RK stage sequence.  Same arithmetic, per item, as
// build_explicit_step.
template <class P, int S, int NI>
__device__ __forceinline__ void build_explicit_multi(const P& prob, const StepCoefs& sc,
                                                     const double (&prev)[NI][P::D],
                                                     const double (&xk)[NI][P::D],
                                                     const bool (&first)[NI], Elem<P::D> (&el)[NI],
                                                     double (&h)[NI][P::D]) {
    constexpr int D = P::D;
    double kap[S][NI][D];
    double dkap[S][NI][D * D];
#pragma unroll
    for (int i = 0; i < S; i++) {
        double xs[NI][D];
#pragma unroll
        for (int n = 0; n < NI; n++)
#pragma unroll
            for (int r = 0; r < D; r++) {
                double acc = prev[n][r];
#pragma unroll
                for (int j = 0; j < i; j++) acc += sc.dta[i * S + j] * kap[j][n][r];
                xs[n][r] = acc;
            }
        double Js[NI][D * D];
#pragma unroll
        for (int n = 0; n < NI; n++) {
            prob.f(xs[n], kap[i][n]);
            prob.jac(xs[n], Js[n]);
        }
#pragma unroll
        for (int n = 0; n < NI; n++) {
            double M[D * D];
#pragma unroll
            for (int r = 0; r < D; r++)
#pragma unroll
                for (int c = 0; c < D; c++) {
                    double m = (r == c) ? 1.0 : 0.0;
#pragma unroll
                    for (int j = 0; j < i; j++) m += sc.dta[i * S + j] * dkap[j][n][r * D + c];
                    M[r * D + c] = m;
                }
#pragma unroll
            for (int r = 0; r < D; r++)
#pragma unroll
                for (int c = 0; c < D; c++) {
                    double acc = 0.0;
#pragma unroll
                    for (int q = 0; q < D; q++) acc += Js[n][r * D + q] * M[q * D + c];
                    dkap[i][n][r * D + c] = acc;
                }
        }
    }
#pragma unroll
    for (int n = 0; n < NI; n++) {
#pragma unroll
        for (int r = 0; r < D; r++) {
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < S; i++) acc += sc.b[i] * kap[i][n][r];
            const double g = sc.dt * acc;
            const double hv = xk[n][r] - prev[n][r] - g;
            h[n][r] = hv;
            el[n].c[r] = -hv;
        }
#pragma unroll
        for (int r = 0; r < D; r++)
#pragma unroll
            for (int c = 0; c < D; c++) {
                double acc = 0.0;
#pragma unroll
                for (int i = 0; i < S; i++) acc += sc.b[i] * dkap[i][n][r * D + c];
                const double jg = sc.dt * acc;
                el[n].F[r * D + c] = first[n] ? 0.0 : jg + ((r == c) ? 1.0 : 0.0);
            }
    }
}

// ---------------------------------------------------------------------------
// Register LU with partial pivoting (_kernels.py:28-77).  Row swaps are
// expressed as predicated moves over compile-time indices so A stays in
// registers.  Returns -1 or the first pivot index below the 1e-300 floor.
// The elimination uses non-contracted products (__dmul_rn / __dsub_rn): the
// singular-block test compares pivots against 1e-300, and an FMA would turn
// the reference's exact cancellations (e.g. 1 - 0.1*10 = 0) into tiny
// non-zero pivots.  With identical A the factorisation is bit-identical to
// the reference's.
// ---------------------------------------------------------------------------
// IEEE-754 a / b.  The hardware division sequence sends non-finite operands
// and zero divisors down a slow subroutine; diverging trajectories (NaN/inf
// rows) hit that on every step.  Here the division always runs on safe
// operands and the special cases (results 0, inf or NaN with the IEEE sign
// rules) are selected afterwards — branch-free, so the unrolled items of a
// thread keep their instruction-level parallelism.
__device__ __forceinline__ double div_rn(double a, double b) {
    const bool fa = isfinite(a), fb = isfinite(b);
    const bool safe = fa && fb && b != 0.0;
    double as = safe ? a : 1.0, bs = safe ? b : 1.0;
    // opaque to the optimiser, which would otherwise fold the selects past
    // the division (safe ? a / b : 1.0) and divide the raw operands again
    asm("mov.b64 %0, %0;" : "+d"(as));
    asm("mov.b64 %0, %0;" : "+d"(bs));
    const double q = as / bs;
    const long long sgn = (__double_as_longlong(a) ^ __double_as_longlong(b)) & (long long)0x8000000000000000ull;
    const double inf = __longlong_as_double(0x7ff0000000000000ll | sgn);
    const double zero = __longlong_as_double(sgn);
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    const bool ia = isinf(a), ib = isinf(b);
    const bool is_nan = isnan(a) || isnan(b) || (ia && ib) || (a == 0.0 && b == 0.0);
    const bool is_inf = ia || (b == 0.0);  // (NaN cases already taken)
    const double sp = is_nan ? nan : (is_inf ? inf : zero);  // zero: finite / inf
    return safe ? q : sp;
}

// rinv[k] = 1 / U[k][k] (div_rn); the triangular solve multiplies by it
// instead of dividing (x / d vs x * (1/d): <= 1 ulp apart for finite values,
// the same 0 / inf / NaN class and sign otherwise, |d| >= 1e-300 by the
// pivot floor) — D divisions per block instead of D per right-hand side.
template <int D>
__device__ __forceinline__ int lu_factor_reg(double* A, int* piv, double* rinv) {
#pragma unroll
    for (int k = 0; k < D; k++) {
        int p = k;
        double best = fabs(A[k * D + k]);
#pragma unroll
        for (int i = k + 1; i < D; i++) {
            double v = fabs(A[i * D + k]);
            if (v > best) { best = v; p = i; }
        }
        if (best < 1e-300) return k;
        piv[k] = p;
#pragma unroll
        for (int i = k + 1; i < D; i++) {
            if (p == i) {
#pragma unroll
                for (int j = 0; j < D; j++) {
                    double t = A[k * D + j];
                    A[k * D + j] = A[i * D + j];
                    A[i * D + j] = t;
                }
            }
        }
        const double inv = div_rn(1.0, A[k * D + k]);
        rinv[k] = inv;
#pragma unroll
        for (int i = k + 1; i < D; i++) {
            double m = A[i * D + k] * inv;
            A[i * D + k] = m;
#pragma unroll
            for (int j = k + 1; j < D; j++) A[i * D + j] = __dsub_rn(A[i * D + j], __dmul_rn(m, A[k * D + j]));
        }
    }
    return -1;
}

template <int D>
__device__ __forceinline__ void lu_solve_reg(const double* A, const int* piv, const double* rinv,
                                             double* x) {
#pragma unroll
    for (int k = 0; k < D; k++) {
#pragma unroll
        for (int i = k + 1; i < D; i++) {
            if (piv[k] == i) { double t = x[k]; x[k] = x[i]; x[i] = t; }
        }
#pragma unroll
        for (int i = k + 1; i < D; i++) x[i] = __dsub_rn(x[i], __dmul_rn(A[i * D + k], x[k]));
    }
#pragma unroll
    for (int i = D - 1; i >= 0; i--) {
        double acc = x[i];
#pragma unroll
        for (int j = i + 1; j < D; j++) acc = __dsub_rn(acc, __dmul_rn(A[i * D + j], x[j]));
        x[i] = acc * rinv[i];
    }
}

// ---------------------------------------------------------------------------
// Implicit weighted element (_kernels.py:393-464):
//   h = X[k] - prev - dt (w_p f(prev) + w_n f(X[k]))
//   A = I - dt w_n J(X[k]);  c = A^{-1}(-h);  F = A^{-1}(I + dt w_p J(prev)), 0 at k=0
// f and J are evaluated at prev even when w_prev = 0.  A singular
// block gives F = c = 0 and returns true.
// ---------------------------------------------------------------------------
template <class P>
__device__ __forceinline__ bool build_implicit_step(const P& prob, const StepCoefs& sc,
                                                   const double* prev, const double* xk,
                                                   bool first, Elem<P::D>& el, double* h) {
    constexpr int D = P::D;
    double fprev[D], fnext[D], Jp[D * D], A[D * D];
    prob.f(prev, fprev);
    prob.f(xk, fnext);
    prob.jac(prev, Jp);
    prob.jac(xk, A);
#pragma unroll
    for (int r = 0; r < D; r++)
        h[r] = xk[r] - prev[r] - sc.dt * (sc.w_prev * fprev[r] + sc.w_next * fnext[r]);
#pragma unroll
    for (int r = 0; r < D; r++)
#pragma unroll
        for (int c = 0; c < D; c++)
            A[r * D + c] = __dsub_rn((r == c) ? 1.0 : 0.0, __dmul_rn(sc.dt_wnext, A[r * D + c]));
    int piv[D];
    double rinv[D];
    int st = lu_factor_reg<D>(A, piv, rinv);
    if (st >= 0) {
#pragma unroll
        for (int r = 0; r < D; r++) {
            el.c[r] = 0.0;
#pragma unroll
            for (int c = 0; c < D; c++) el.F[r * D + c] = 0.0;
        }
        return true;
    }
    double col[D];
#pragma unroll
    for (int r = 0; r < D; r++) col[r] = -h[r];
    lu_solve_reg<D>(A, piv, rinv, col);
#pragma unroll
    for (int r = 0; r < D; r++) el.c[r] = col[r];
    if (first) {
#pragma unroll
        for (int i = 0; i < D * D; i++) el.F[i] = 0.0;
    } else {
#pragma unroll
        for (int c = 0; c < D; c++) {
#pragma unroll
            for (int r = 0; r < D; r++)
                col[r] = __dadd_rn(__dmul_rn(sc.dt_wprev, Jp[r * D + c]), (r == c) ? 1.0 : 0.0);
            lu_solve_reg<D>(A, piv, rinv, col);
#pragma unroll
            for (int r = 0; r < D; r++) el.F[r * D + c] = col[r];
        }
    }
    return false;
}

// Branch-free form of lu_factor_reg + build_implicit_step (same arithmetic
// for every non-singular block; a singular block still yields F = c = 0 and
// true): no early exits, so two items' builds written back to back can be
// interleaved by the compiler (the grid-resident kernel's latency-bound build).
template <int D>
__device__ __forceinline__ int lu_factor_reg_bf(double* A, int* piv, double* rinv) {
    int st = -1;
#pragma unroll
    for (int k = 0; k < D; k++) {
        int p = k;
        double best = fabs(A[k * D + k]);
#pragma unroll
        for (int i = k + 1; i < D; i++) {
            double v = fabs(A[i * D + k]);
            if (v > best) { best = v; p = i; }
        }
        if (best < 1e-300 && st < 0) st = k;
        piv[k] = p;
#pragma unroll
        for (int i = k + 1; i < D; i++) {
            if (p == i) {
#pragma unroll
                for (int j = 0; j < D; j++) {
                    double t = A[k * D + j];
                    A[k * D + j] = A[i * D + j];
                    A[i * D + j] = t;
                }
            }
        }
        const double inv = div_rn(1.0, A[k * D + k]);
        rinv[k] = inv;
#pragma unroll
        for (int i = k + 1; i < D; i++) {
            double m = A[i * D + k] * inv;
            A[i * D + k] = m;
#pragma unroll
            for (int j = k + 1; j < D; j++) A[i * D + j] = __dsub_rn(A[i * D + j], __dmul_rn(m, A[k * D + j]));
        }
    }
    return st;
}

template <class P>
__device__ __forceinline__ bool build_implicit_step_bf(const P& prob, const StepCoefs& sc,
                                                      const double* prev, const double* xk,
                                                      bool first, Elem<P::D>& el, double* h) {
    constexpr int D = P::D;
    double fprev[D], fnext[D], Jp[D * D], A[D * D];
    prob.f(prev, fprev);
    prob.f(xk, fnext);
    prob.jac(prev, Jp);
    prob.jac(xk, A);
#pragma unroll
    for (int r = 0; r < D; r++)
        h[r] = xk[r] - prev[r] - sc.dt * (sc.w_prev * fprev[r] + sc.w_next * fnext[r]);
#pragma unroll
    for (int r = 0; r < D; r++)
#pragma unroll
        for (int c = 0; c < D; c++)
            A[r * D + c] = __dsub_rn((r == c) ? 1.0 : 0.0, __dmul_rn(sc.dt_wnext, A[r * D + c]));
    int piv[D];
    double rinv[D];
    const bool sing = lu_factor_reg_bf<D>(A, piv, rinv) >= 0;
    double col[D];
#pragma unroll
    for (int r = 0; r < D; r++) col[r] = -h[r];
    lu_solve_reg<D>(A, piv, rinv, col);
#pragma unroll
    for (int r = 0; r < D; r++) el.c[r] = sing ? 0.0 : col[r];
#pragma unroll
    for (int c = 0; c < D; c++) {
#pragma unroll
        for (int r = 0; r < D; r++)
            col[r] = __dadd_rn(__dmul_rn(sc.dt_wprev, Jp[r * D + c]), (r == c) ? 1.0 : 0.0);
        lu_solve_reg<D>(A, piv, rinv, col);
#pragma unroll
        for (int r = 0; r < D; r++) el.F[r * D + c] = (sing || first) ? 0.0 : col[r];
    }
    return sing;
}

// Uniform entry used by the fused kernels: KIND 0 = explicit RK with S stages,
// KIND 1 = implicit weighted.  Returns true for a singular implicit block.
template <class P, int KIND, int S>
__device__ __forceinline__ bool build_step(const P& prob, const StepCoefs& sc, const double* prev,
                                           const double* xk, bool first, Elem<P::D>& el,
                                           double* h) {
    if constexpr (KIND == 0) {
        build_explicit_step<P, S>(prob, sc, prev, xk, first, el, h);
        return false;
    } else {
        return build_implicit_step<P>(prob, sc, prev, xk, first, el, h);
    }
}

}  // namespace odx
