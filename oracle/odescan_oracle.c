/*
 * odescan_oracle.c — CPU ORACLE for the parallel-in-time Newton hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is a plain-C restatement of the
 * reference package's compiled loops (numba, /root/reference/pkg/src/odescan/
 * _kernels.py) and of the solve() control flow (newton_pint.py:326-406).  It is
 * imported only by tests/, by __graft_entry__.smoke() and by bench.py's CPU
 * baseline leg, always as the checker / the timed CPU reference, never as the
 * product path.  The product path (paper_2511_01465_b200) never links it.
 *
 * Arithmetic follows the reference operation by operation (same association,
 * same accumulation order, same zero-tableau / zero-weight terms, no FMA:
 * build with -ffp-contract=off), so on finite AND non-finite data it is
 * bit-identical to the numba reference.  That claim is pinned by
 * tests/test_oracle_golden.py against vectors produced by the reference itself
 * (tests/golden/make_golden.py).  Loops over independent elements are
 * OpenMP-parallel like the reference's prange; every result is independent of
 * the thread count (each element is computed by exactly one thread and the
 * max-reduction is exact).
 *
 * Problems without a reference implementation (Lorenz-63, Allen-Cahn, the
 * parametrised van der Pol) are defined here, in tests/golden/make_golden.py
 * (numba, plugged into the reference as OdeProblem(f_into, jac_into)) and in
 * the CUDA functors with the same expression order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/odescan_b200.h"

#define PIVOT_FLOOR 1e-300 /* _kernels.py:21 */
#define MAXD 64

typedef struct {
    int id, dim;
    const double* p; /* params */
} prob_t;

/* ------------------------------------------------------------------------ */
/* Problem right-hand sides.  Expression trees mirror problems.py exactly.  */
/* ------------------------------------------------------------------------ */

static void prob_f(const prob_t* P, const double* x, double* out) {
    const double* p = P->p;
    switch (P->id) {
    case ODX_PROB_LOGISTIC: /* problems.py:92-94 */
        out[0] = p[0] * x[0] * (1.0 - x[0] / p[1]);
        break;
    case ODX_PROB_VDP: /* problems.py:123-126, mu as a parameter */
        out[0] = x[1];
        out[1] = p[0] * (1.0 - x[0] * x[0]) * x[1] - x[0];
        break;
    case ODX_PROB_CARTPOLE:
    case ODX_PROB_CARTPOLE_SQ: { /* problems.py:162-171, 197-206 */
        const double G = p[0], L = p[1], MC = p[2], MP = p[3];
        double s = sin(x[2]), c = cos(x[2]), w = x[3];
        double den = MC + MP * s * s;
        out[0] = x[1];
        if (P->id == ODX_PROB_CARTPOLE)
            out[1] = MP * s * (L * w + G * c) / den;
        else
            out[1] = MP * s * (L * w * w + G * c) / den;
        out[2] = w;
        out[3] = (-MP * L * w * w * c * s - (MC + MP) * G * s) / (L * den);
        break;
    }
    case ODX_PROB_DAHLQUIST: /* problems.py:252-254 */
        out[0] = p[0] * x[0];
        break;
    case ODX_PROB_ROBERTSON: /* problems.py:280-284 */
        out[0] = -p[0] * x[0] + p[2] * x[1] * x[2];
        out[1] = p[0] * x[0] - p[1] * x[1] * x[1] - p[2] * x[1] * x[2];
        out[2] = p[1] * x[1] * x[1];
        break;
    case ODX_PROB_LORENZ63: /* BASELINE cfg 1/3: sigma, rho, beta */
        out[0] = p[0] * (x[1] - x[0]);
        out[1] = x[0] * (p[1] - x[2]) - x[1];
        out[2] = x[0] * x[1] - p[2] * x[2];
        break;
    case ODX_PROB_ALLEN_CAHN: { /* BASELINE cfg 4: u_t = eps u_xx + u - u^3, periodic */
        const int n = P->dim;
        const double cdiff = p[0] / (p[1] * p[1]);
        for (int i = 0; i < n; i++) {
            double um = x[(i + n - 1) % n], ui = x[i], up = x[(i + 1) % n];
            out[i] = cdiff * ((um - 2.0 * ui) + up) + (ui - ui * ui * ui);
        }
        break;
    }
    case ODX_PROB_EXP_GROWTH: /* tests/test_newton_pint.py:28-30 */
        out[0] = exp(x[0]);
        break;
    case ODX_PROB_SQUARE: /* tests/test_newton_pint.py:49-51 */
        out[0] = x[0] * x[0];
        break;
    case ODX_PROB_LINEAR: {
        const int n = P->dim;
        for (int r = 0; r < n; r++) {
            double acc = 0.0;
            for (int q = 0; q < n; q++) acc += p[r * n + q] * x[q];
            out[r] = acc;
        }
        break;
    }
    default:
        break;
    }
}

static void prob_jac(const prob_t* P, const double* x, double* J) {
    const double* p = P->p;
    const int n = P->dim;
    switch (P->id) {
    case ODX_PROB_LOGISTIC: /* problems.py:97-99 */
        J[0] = p[0] * (1.0 - 2.0 * x[0] / p[1]);
        break;
    case ODX_PROB_VDP: /* problems.py:129-134 */
        J[0] = 0.0;
        J[1] = 1.0;
        J[2] = -2.0 * p[0] * x[0] * x[1] - 1.0;
        J[3] = p[0] * (1.0 - x[0] * x[0]);
        break;
    case ODX_PROB_CARTPOLE:
    case ODX_PROB_CARTPOLE_SQ: { /* problems.py:174-194, 209-226 */
        const double G = p[0], L = p[1], MC = p[2], MP = p[3];
        double s = sin(x[2]), c = cos(x[2]), w = x[3];
        double den = MC + MP * s * s;
        double dden = 2.0 * MP * s * c;
        for (int i = 0; i < 16; i++) J[i] = 0.0;
        J[0 * 4 + 1] = 1.0;
        J[2 * 4 + 3] = 1.0;
        double num1, dnum1;
        if (P->id == ODX_PROB_CARTPOLE) {
            num1 = MP * s * (L * w + G * c);
            dnum1 = MP * c * (L * w + G * c) + MP * s * (-G * s);
        } else {
            num1 = MP * s * (L * w * w + G * c);
            dnum1 = MP * c * (L * w * w + G * c) + MP * s * (-G * s);
        }
        J[1 * 4 + 2] = dnum1 / den - num1 * dden / (den * den);
        if (P->id == ODX_PROB_CARTPOLE)
            J[1 * 4 + 3] = MP * s * L / den;
        else
            J[1 * 4 + 3] = 2.0 * MP * s * L * w / den;
        double num3 = -MP * L * w * w * c * s - (MC + MP) * G * s;
        double dnum3 = -MP * L * w * w * (c * c - s * s) - (MC + MP) * G * c;
        J[3 * 4 + 2] = dnum3 / (L * den) - num3 * dden / (L * den * den);
        J[3 * 4 + 3] = -2.0 * MP * L * w * c * s / (L * den);
        break;
    }
    case ODX_PROB_DAHLQUIST:
        J[0] = p[0];
        break;
    case ODX_PROB_ROBERTSON: /* problems.py:287-297 */
        J[0] = -p[0];
        J[1] = p[2] * x[2];
        J[2] = p[2] * x[1];
        J[3] = p[0];
        J[4] = -2.0 * p[1] * x[1] - p[2] * x[2];
        J[5] = -p[2] * x[1];
        J[6] = 0.0;
        J[7] = 2.0 * p[1] * x[1];
        J[8] = 0.0;
        break;
    case ODX_PROB_LORENZ63:
        J[0] = -p[0]; J[1] = p[0];  J[2] = 0.0;
        J[3] = p[1] - x[2]; J[4] = -1.0; J[5] = -x[0];
        J[6] = x[1]; J[7] = x[0]; J[8] = -p[2];
        break;
    case ODX_PROB_ALLEN_CAHN: {
        const double cdiff = p[0] / (p[1] * p[1]);
        for (int i = 0; i < n * n; i++) J[i] = 0.0;
        for (int i = 0; i < n; i++) {
            J[i * n + i] = -2.0 * cdiff + (1.0 - 3.0 * (x[i] * x[i]));
            J[i * n + (i + n - 1) % n] += cdiff;
            J[i * n + (i + 1) % n] += cdiff;
        }
        break;
    }
    case ODX_PROB_EXP_GROWTH:
        J[0] = exp(x[0]);
        break;
    case ODX_PROB_SQUARE:
        J[0] = 2.0 * x[0];
        break;
    case ODX_PROB_LINEAR:
        for (int i = 0; i < n * n; i++) J[i] = p[i];
        break;
    default:
        break;
    }
}

/* ------------------------------------------------------------------------ */
/* Tiny LU, partial pivoting: _kernels.py:28-77                              */
/* ------------------------------------------------------------------------ */

static int lu_factor(double* A, int64_t* piv, int n) { /* _kernels.py:28-57 */
    for (int k = 0; k < n; k++) {
        int p = k;
        double best = fabs(A[k * n + k]);
        for (int i = k + 1; i < n; i++) {
            double v = fabs(A[i * n + k]);
            if (v > best) { best = v; p = i; }
        }
        if (best < PIVOT_FLOOR) return k;
        piv[k] = p;
        if (p != k) {
            for (int j = 0; j < n; j++) {
                double t = A[k * n + j];
                A[k * n + j] = A[p * n + j];
                A[p * n + j] = t;
            }
        }
        double inv = 1.0 / A[k * n + k];
        for (int i = k + 1; i < n; i++) {
            double m = A[i * n + k] * inv;
            A[i * n + k] = m;
            for (int j = k + 1; j < n; j++) A[i * n + j] -= m * A[k * n + j];
        }
    }
    return -1;
}

static void lu_solve(const double* A, const int64_t* piv, double* x, int n) { /* :60-77 */
    for (int k = 0; k < n; k++) {
        int64_t p = piv[k];
        if (p != k) { double t = x[k]; x[k] = x[p]; x[p] = t; }
        for (int i = k + 1; i < n; i++) x[i] -= A[i * n + k] * x[k];
    }
    for (int i = n - 1; i >= 0; i--) {
        double acc = x[i];
        for (int j = i + 1; j < n; j++) acc -= A[i * n + j] * x[j];
        x[i] = acc / A[i * n + i];
    }
}

int orc_lu_factor(double* A, int64_t* piv, int n) { return lu_factor(A, piv, n); }
void orc_lu_solve(const double* A, const int64_t* piv, double* x, int n) { lu_solve(A, piv, x, n); }

/* ------------------------------------------------------------------------ */
/* Reductions: _kernels.py:84-103                                            */
/* ------------------------------------------------------------------------ */

/* Row rule: loc takes v whenever !(v <= loc) (so a NaN replaces loc and is
 * then replaced by the next entry); rows whose loc ends NaN are skipped by
 * the cross-row max (numba's max(out, nan) keeps out).  All-NaN -> 0.0.    */
double orc_max_abs(const double* A, int64_t n, int d) {
    double out = 0.0;
#pragma omp parallel for reduction(max : out) schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double loc = 0.0;
        for (int j = 0; j < d; j++) {
            double v = fabs(A[i * d + j]);
            if (!(v <= loc)) loc = v;
        }
        if (loc > out) out = loc; /* NaN loc never wins */
    }
    return out;
}

void orc_add_inplace(double* X, const double* U, int64_t n, int d) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n * d; i++) X[i] += U[i];
}

/* ------------------------------------------------------------------------ */
/* Blelloch affine scan: _kernels.py:116-233                                  */
/* combine(earlier e, later l) = (Fl Fe, Fl ce + cl)                          */
/* ------------------------------------------------------------------------ */

static void pair_into(const double* Fl, const double* cl, const double* Fe, const double* ce,
                      double* Fo, double* co, int d) {
    /* later = (Fl, cl) applied after earlier = (Fe, ce); Fo/co must not alias inputs */
    for (int r = 0; r < d; r++) {
        double acc = cl[r];
        for (int q = 0; q < d; q++) acc += Fl[r * d + q] * ce[q];
        co[r] = acc;
    }
    for (int r = 0; r < d; r++)
        for (int s = 0; s < d; s++) {
            double acc = 0.0;
            for (int q = 0; q < d; q++) acc += Fl[r * d + q] * Fe[q * d + s];
            Fo[r * d + s] = acc;
        }
}

/* Fp may be NULL (solve() uses only cp, newton_pint.py:395). Returns 0 / -1 (alloc). */
int orc_scan_affine(const double* Fin, const double* cin, int64_t n, int d,
                    double* Fp, double* cp) {
    int64_t m = 1;
    while (m < n) m <<= 1;
    const int64_t dd = (int64_t)d * d;
    double* Fw = (double*)malloc(sizeof(double) * m * dd);
    double* cw = (double*)malloc(sizeof(double) * m * d);
    if (!Fw || !cw) { free(Fw); free(cw); return -1; }

#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < m; k++) {
        if (k < n) {
            memcpy(Fw + k * dd, Fin + k * dd, sizeof(double) * dd);
            memcpy(cw + k * d, cin + k * d, sizeof(double) * d);
        } else {
            for (int r = 0; r < d; r++) {
                for (int s = 0; s < d; s++) Fw[k * dd + r * d + s] = (r == s) ? 1.0 : 0.0;
                cw[k * d + r] = 0.0;
            }
        }
    }
    /* up-sweep :138-168 — node j (later) absorbs node j-step (earlier) */
    for (int64_t step = 1; step < m; step *= 2) {
        int64_t width = 2 * step, npairs = m / width;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < npairs; i++) {
            double tf[MAXD * MAXD], tc[MAXD];
            int64_t j = (i + 1) * width - 1, l = j - step;
            pair_into(Fw + j * dd, cw + j * d, Fw + l * dd, cw + l * d, tf, tc, d);
            memcpy(cw + j * d, tc, sizeof(double) * d);
            memcpy(Fw + j * dd, tf, sizeof(double) * dd);
        }
    }
    /* down-sweep :170-216 */
    for (int r = 0; r < d; r++) {
        for (int s = 0; s < d; s++) Fw[(m - 1) * dd + r * d + s] = (r == s) ? 1.0 : 0.0;
        cw[(m - 1) * d + r] = 0.0;
    }
    for (int64_t step = m >> 1; step >= 1; step >>= 1) {
        int64_t width = 2 * step, npairs = m / width;
#pragma omp parallel for schedule(static)
        for (int64_t i = 0; i < npairs; i++) {
            double lf[MAXD * MAXD], lc[MAXD], tf[MAXD * MAXD], tc[MAXD];
            int64_t j = (i + 1) * width - 1, l = j - step;
            memcpy(lf, Fw + l * dd, sizeof(double) * dd);
            memcpy(lc, cw + l * d, sizeof(double) * d);
            memcpy(Fw + l * dd, Fw + j * dd, sizeof(double) * dd);
            memcpy(cw + l * d, cw + j * d, sizeof(double) * d);
            /* node prefix (earlier) then old left subtotal (later) */
            pair_into(lf, lc, Fw + j * dd, cw + j * d, tf, tc, d);
            memcpy(cw + j * d, tc, sizeof(double) * d);
            memcpy(Fw + j * dd, tf, sizeof(double) * dd);
        }
    }
    /* fold each input onto its exclusive prefix :218-233 */
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; k++) {
        const double* F = Fin + k * dd;
        for (int r = 0; r < d; r++) {
            double acc = cin[k * d + r];
            for (int q = 0; q < d; q++) acc += F[r * d + q] * cw[k * d + q];
            cp[k * d + r] = acc;
        }
        if (Fp) {
            for (int r = 0; r < d; r++)
                for (int s = 0; s < d; s++) {
                    double acc = 0.0;
                    for (int q = 0; q < d; q++) acc += F[r * d + q] * Fw[k * dd + q * d + s];
                    Fp[k * dd + r * d + s] = acc;
                }
        }
    }
    free(Fw);
    free(cw);
    return 0;
}

/* Offsets of affine_scan.scan_sequential (affine_scan.py:106-113) over
 * init_elements-style input (element 0's matrix part is zero, so every prefix
 * offset is the state, extract_states :153-160): cp_k = F_k cp_{k-1} + c_k,
 * accumulated as combine() does (:64-78, acc = c_l; acc += F_l[r,q] ce[q]).
 * The definitional left-to-right recursion; used by the tests to decide which
 * association is right where two scan trees overflow differently. */
void orc_scan_sequential(const double* Fin, const double* cin, int64_t n, int d, double* cp) {
    const int64_t dd = (int64_t)d * d;
    for (int r = 0; r < d; r++) cp[r] = cin[r];
    for (int64_t k = 1; k < n; k++) {
        const double* F = Fin + k * dd;
        for (int r = 0; r < d; r++) {
            double acc = cin[k * d + r];
            for (int q = 0; q < d; q++) acc += F[r * d + q] * cp[(k - 1) * d + q];
            cp[k * d + r] = acc;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Explicit RK elements: _kernels.py:261-342                                  */
/* ------------------------------------------------------------------------ */

static void rk_increment_with_jac(const prob_t* P, const double* a, const double* b, int s,
                                  const double* x, double dt, double* kap, double* dkap,
                                  double* g, double* Jg) {
    const int d = P->dim;
    double xs[MAXD], Js[MAXD * MAXD], M[MAXD * MAXD];
    for (int i = 0; i < s; i++) {
        for (int r = 0; r < d; r++) {
            double acc = x[r];
            for (int j = 0; j < i; j++) acc += dt * a[i * s + j] * kap[j * d + r];
            xs[r] = acc;
        }
        prob_f(P, xs, kap + i * d);
        prob_jac(P, xs, Js);
        for (int r = 0; r < d; r++)
            for (int c = 0; c < d; c++) {
                double m = (r == c) ? 1.0 : 0.0;
                for (int j = 0; j < i; j++) m += dt * a[i * s + j] * dkap[(j * d + r) * d + c];
                M[r * d + c] = m;
            }
        for (int r = 0; r < d; r++)
            for (int c = 0; c < d; c++) {
                double acc = 0.0;
                for (int q = 0; q < d; q++) acc += Js[r * d + q] * M[q * d + c];
                dkap[(i * d + r) * d + c] = acc;
            }
    }
    for (int r = 0; r < d; r++) {
        double acc = 0.0;
        for (int i = 0; i < s; i++) acc += b[i] * kap[i * d + r];
        g[r] = dt * acc;
    }
    for (int r = 0; r < d; r++)
        for (int c = 0; c < d; c++) {
            double acc = 0.0;
            for (int i = 0; i < s; i++) acc += b[i] * dkap[(i * d + r) * d + c];
            Jg[r * d + c] = dt * acc;
        }
}

static void rk_increment(const prob_t* P, const double* a, const double* b, int s,
                         const double* x, double dt, double* kap, double* g) { /* :240-258 */
    const int d = P->dim;
    double xs[MAXD];
    for (int i = 0; i < s; i++) {
        for (int r = 0; r < d; r++) {
            double acc = x[r];
            for (int j = 0; j < i; j++) acc += dt * a[i * s + j] * kap[j * d + r];
            xs[r] = acc;
        }
        prob_f(P, xs, kap + i * d);
    }
    for (int r = 0; r < d; r++) {
        double acc = 0.0;
        for (int i = 0; i < s; i++) acc += b[i] * kap[i * d + r];
        g[r] = dt * acc;
    }
}

/* Range variant used by the sharding tests: steps offset..offset+n-1 of a
 * trajectory, prev of the first local step = x0 (the halo), F zeroed only at
 * the global step 0.  offset = 0 is exactly _kernels.build_explicit. */
void orc_build_explicit_range(int pid, int d, const double* params, const double* a,
                              const double* b, int s, const double* x0, const double* X,
                              int64_t n, double dt, double* Fe, double* ce, double* h,
                              int64_t offset);
void orc_build_explicit(int pid, int d, const double* params, const double* a, const double* b,
                        int s, const double* x0, const double* X, int64_t n, double dt,
                        double* Fe, double* ce, double* h) {
    orc_build_explicit_range(pid, d, params, a, b, s, x0, X, n, dt, Fe, ce, h, 0);
}

void orc_build_explicit_range(int pid, int d, const double* params, const double* a,
                              const double* b, int s, const double* x0, const double* X,
                              int64_t n, double dt, double* Fe, double* ce, double* h,
                              int64_t offset) {
    prob_t P = {pid, d, params};
    const int64_t dd = (int64_t)d * d;
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; k++) {
        double kap[ODX_MAX_STAGES * MAXD], g[MAXD];
        double* dkap = (double*)malloc(sizeof(double) * s * dd);
        double* Jg = (double*)malloc(sizeof(double) * dd);
        const double* prev = (k == 0) ? x0 : X + (k - 1) * d;
        rk_increment_with_jac(&P, a, b, s, prev, dt, kap, dkap, g, Jg);
        for (int r = 0; r < d; r++) {
            double hv = X[k * d + r] - prev[r] - g[r];
            h[k * d + r] = hv;
            ce[k * d + r] = -hv;
        }
        for (int r = 0; r < d; r++)
            for (int c = 0; c < d; c++)
                Fe[k * dd + r * d + c] = (offset + k == 0) ? 0.0 : Jg[r * d + c] + ((r == c) ? 1.0 : 0.0);
        free(dkap);
        free(Jg);
    }
}

/* ------------------------------------------------------------------------ */
/* Implicit weighted elements: _kernels.py:393-464                            */
/* ------------------------------------------------------------------------ */

int64_t orc_build_implicit_range(int pid, int d, const double* params, double w_prev,
                                 double w_next, const double* x0, const double* X, int64_t n,
                                 double dt, double* Fe, double* ce, double* h, int64_t offset);
int64_t orc_build_implicit(int pid, int d, const double* params, double w_prev, double w_next,
                           const double* x0, const double* X, int64_t n, double dt,
                           double* Fe, double* ce, double* h) {
    return orc_build_implicit_range(pid, d, params, w_prev, w_next, x0, X, n, dt, Fe, ce, h, 0);
}

/* Range variant (see orc_build_explicit_range); returned bad index is global. */
int64_t orc_build_implicit_range(int pid, int d, const double* params, double w_prev,
                                 double w_next, const double* x0, const double* X, int64_t n,
                                 double dt, double* Fe, double* ce, double* h, int64_t offset) {
    prob_t P = {pid, d, params};
    const int64_t dd = (int64_t)d * d;
    int64_t worst = -1;
#pragma omp parallel
    {
        double* Jp = (double*)malloc(sizeof(double) * dd);
        double* Jn = (double*)malloc(sizeof(double) * dd);
        double* A = (double*)malloc(sizeof(double) * dd);
        int64_t local_bad = -1;
#pragma omp for schedule(static)
        for (int64_t k = 0; k < n; k++) {
            double fprev[MAXD], fnext[MAXD], col[MAXD];
            int64_t piv[MAXD];
            const double* prev = (k == 0) ? x0 : X + (k - 1) * d;
            const double* nxt = X + k * d;
            prob_f(&P, prev, fprev);
            prob_f(&P, nxt, fnext);
            prob_jac(&P, prev, Jp);
            prob_jac(&P, nxt, Jn);
            for (int r = 0; r < d; r++)
                h[k * d + r] = nxt[r] - prev[r] - dt * (w_prev * fprev[r] + w_next * fnext[r]);
            for (int r = 0; r < d; r++)
                for (int c = 0; c < d; c++)
                    A[r * d + c] = ((r == c) ? 1.0 : 0.0) - dt * w_next * Jn[r * d + c];
            int st = lu_factor(A, piv, d);
            if (st >= 0) {
                if (local_bad < 0 || offset + k < local_bad) local_bad = offset + k;
                for (int r = 0; r < d; r++) {
                    ce[k * d + r] = 0.0;
                    for (int c = 0; c < d; c++) Fe[k * dd + r * d + c] = 0.0;
                }
                continue;
            }
            for (int r = 0; r < d; r++) col[r] = -h[k * d + r];
            lu_solve(A, piv, col, d);
            for (int r = 0; r < d; r++) ce[k * d + r] = col[r];
            if (offset + k == 0) {
                for (int64_t i = 0; i < dd; i++) Fe[k * dd + i] = 0.0;
            } else {
                for (int c = 0; c < d; c++) {
                    for (int r = 0; r < d; r++)
                        col[r] = dt * w_prev * Jp[r * d + c] + ((r == c) ? 1.0 : 0.0);
                    lu_solve(A, piv, col, d);
                    for (int r = 0; r < d; r++) Fe[k * dd + r * d + c] = col[r];
                }
            }
        }
#pragma omp critical
        {
            if (local_bad >= 0 && (worst < 0 || local_bad < worst)) worst = local_bad;
        }
        free(Jp);
        free(Jn);
        free(A);
    }
    return worst;
}

/* ------------------------------------------------------------------------ */
/* Sequential marchers (converged-solution oracle): _kernels.py:345-360, 467-526 */
/* ------------------------------------------------------------------------ */

void orc_seq_explicit(int pid, int d, const double* params, const double* a, const double* b,
                      int s, const double* x0, double dt, int64_t n, double* X) {
    prob_t P = {pid, d, params};
    double kap[ODX_MAX_STAGES * MAXD], g[MAXD], x[MAXD];
    for (int r = 0; r < d; r++) x[r] = x0[r];
    for (int64_t k = 0; k < n; k++) {
        rk_increment(&P, a, b, s, x, dt, kap, g);
        for (int r = 0; r < d; r++) {
            x[r] = x[r] + g[r];
            X[k * d + r] = x[r];
        }
    }
}

int64_t orc_seq_implicit(int pid, int d, const double* params, double w_prev, double w_next,
                         const double* x0, double dt, int64_t n, double tol, int max_inner,
                         double* X) {
    prob_t P = {pid, d, params};
    double xprev[MAXD], x[MAXD], fp[MAXD], fx[MAXD], r[MAXD];
    int64_t piv[MAXD];
    double* J = (double*)malloc(sizeof(double) * d * d);
    double* A = (double*)malloc(sizeof(double) * d * d);
    int64_t ret = -1;
    for (int i = 0; i < d; i++) xprev[i] = x0[i];
    for (int64_t k = 0; k < n && ret == -1; k++) {
        prob_f(&P, xprev, fp);
        for (int i = 0; i < d; i++) x[i] = xprev[i];
        int converged = 0;
        for (int it = 0; it < max_inner; it++) {
            prob_f(&P, x, fx);
            double rn = 0.0;
            for (int i = 0; i < d; i++) {
                r[i] = x[i] - xprev[i] - dt * (w_prev * fp[i] + w_next * fx[i]);
                double av = fabs(r[i]);
                if (av > rn) rn = av;
            }
            if (rn <= tol) { converged = 1; break; }
            prob_jac(&P, x, J);
            for (int i = 0; i < d; i++)
                for (int j = 0; j < d; j++)
                    A[i * d + j] = ((i == j) ? 1.0 : 0.0) - dt * w_next * J[i * d + j];
            if (lu_factor(A, piv, d) >= 0) { ret = -(k + 2); break; }
            lu_solve(A, piv, r, d);
            for (int i = 0; i < d; i++) x[i] -= r[i];
        }
        if (ret != -1) break;
        if (!converged) {
            prob_f(&P, x, fx);
            double rn = 0.0;
            for (int i = 0; i < d; i++) {
                double rv = x[i] - xprev[i] - dt * (w_prev * fp[i] + w_next * fx[i]);
                double av = fabs(rv);
                if (av > rn) rn = av;
            }
            if (rn > tol) { ret = k; break; }
        }
        for (int i = 0; i < d; i++) { X[k * d + i] = x[i]; xprev[i] = x[i]; }
    }
    free(J);
    free(A);
    return ret;
}

/* ------------------------------------------------------------------------ */
/* The Newton driver: solve() newton_pint.py:326-406 + BASELINE step rule.  */
/* Per iteration it = 0..max_iters (identical control flow on the GPU):      */
/*   build -> SINGULAR(k) if a pivot fell below the floor (:378-380)          */
/*   rn = max_abs(h); sc = rn (explicit) or max_abs(ce) (:381-389)           */
/*   rn = +-inf and abort -> NONFINITE(it)                                    */
/*   conv = (residual_tol>0 && rn<=residual_tol) ||                          */
/*          (step_tol>0 && it>0 && max|dx of the previous update| < step_tol) */
/*   it >= max_iters -> CONVERGED if conv else MAXITER, iters = max_iters     */
/*   conv -> CONVERGED, iters = it                                            */
/*   scan, X += cp (:395-396)                                                 */
/* trace (optional) receives every iterate: trace[it*n*d ...].               */
/* ------------------------------------------------------------------------ */

int orc_solve(int pid, int d, const double* params, const odx_stepper* S, const double* x0,
              double* X, int64_t n, double dt, const odx_newton_cfg* C, double* hist,
              double* shist, int32_t* iters, int32_t* status, int64_t* status_index,
              double* trace) {
    const int64_t dd = (int64_t)d * d;
    double* Fe = (double*)malloc(sizeof(double) * n * dd);
    double* ce = (double*)malloc(sizeof(double) * n * d);
    double* h = (double*)malloc(sizeof(double) * n * d);
    double* cp = (double*)malloc(sizeof(double) * n * d);
    if (!Fe || !ce || !h || !cp) { free(Fe); free(ce); free(h); free(cp); return -1; }
    double step_prev = NAN;
    int rc = 0;
    *status_index = -1;
    for (int it = 0; it <= C->max_iters; it++) {
        if (trace) memcpy(trace + (int64_t)it * n * d, X, sizeof(double) * n * d);
        double rn, sc;
        if (S->kind == ODX_STEP_EXPLICIT_RK) {
            orc_build_explicit(pid, d, params, S->a, S->b, S->stages, x0, X, n, dt, Fe, ce, h);
            rn = orc_max_abs(h, n, d);
            sc = rn;
        } else {
            int64_t bad = orc_build_implicit(pid, d, params, S->w_prev, S->w_next, x0, X, n, dt,
                                             Fe, ce, h);
            if (bad >= 0) {
                *status = ODX_ST_SINGULAR; *status_index = bad; *iters = it;
                goto done;
            }
            rn = orc_max_abs(h, n, d);
            sc = orc_max_abs(ce, n, d);
        }
        if (hist) hist[it] = rn;
        if (shist) shist[it] = sc;
        if (isinf(rn) && C->abort_nonfinite) {
            *status = ODX_ST_NONFINITE; *status_index = it; *iters = it;
            goto done;
        }
        int conv = (C->residual_tol > 0.0 && rn <= C->residual_tol) ||
                   (C->step_tol > 0.0 && it > 0 && step_prev < C->step_tol);
        if (it >= C->max_iters) {
            *status = conv ? ODX_ST_CONVERGED : ODX_ST_MAXITER; *iters = C->max_iters;
            goto done;
        }
        if (conv) { *status = ODX_ST_CONVERGED; *iters = it; goto done; }
        if (orc_scan_affine(Fe, ce, n, d, NULL, cp) != 0) { rc = -1; goto done; }
        orc_add_inplace(X, cp, n, d);
        step_prev = orc_max_abs(cp, n, d);
    }
done:
    free(Fe); free(ce); free(h); free(cp);
    return rc;
}

int orc_abi_version(void) { return ODX_ABI_VERSION; }
