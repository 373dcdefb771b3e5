// dense_band.cuh — fast K1 for the d = 64 path when A = I - dt w_next Jn is
// periodic tridiagonal (Allen-Cahn, BASELINE cfg 4) and partial pivoting
// keeps every pivot on the diagonal.
//
// The reference's lu_factor / lu_solve (_kernels.py:28-77) applied to such an
// A touch, per pivot k, only rows k+1 and 63 ("arrow" row) and columns k+1 and
// 63 (fill-in column); every other update is x - 0*y or x - m*0 with finite
// operands, i.e. a no-op.  This kernel performs exactly the non-trivial
// operations, in the reference's order, non-contracted:
//
//   pivot k:  p from {k, k+1, 63} by the reference rule (strict >, first max)
//             inv = 1/A_kk;  m1 = A_k+1,k * inv;  m2 = A_63,k * inv
//             A_k+1,k+1 -= m1 A_k,k+1    A_k+1,63 -= m1 A_k,63
//             A_63,k+1  -= m2 A_k,k+1    A_63,63  -= m2 A_k,63
//   solve:    x_k+1 -= L_k+1,k x_k ; x_63 -= L_63,k x_k            (forward)
//             x_i = ((x_i - U_i,i+1 x_i+1) - U_i,63 x_63) / U_ii     (back)
//
// A step is handed to the general warp LU (dense_lu.cuh) — recorded in a
// list, rebuilt by a second kernel — whenever that argument does not hold:
// a pivot would leave the diagonal, or any factor / output is non-finite
// (then 0 * inf = NaN terms must not be skipped).  Singular steps (pivot
// below 1e-300 with no row swap) are resolved here, as the reference does.
//
// Work split: one warp per step.  The factorisation and the c = A^{-1}(-h)
// solve run redundantly in every lane (registers, fully unrolled); the 64
// columns of F = A^{-1} B are two passes of one column per lane, the column
// vector held in registers (static indices), B's column built from its three
// band entries.  Factors live in shared memory (2.5 KB per warp), so an SM
// keeps 12-16 warps in flight.
#pragma once

#include "common.cuh"
#include "dense_problems.cuh"

namespace odx {

constexpr int BAND_N = 64;
constexpr int BAND_WARPS = 4;

struct BandWarpSmem {
    double xk[BAND_N], xp[BAND_N];
    double Al[BAND_N], Ad[BAND_N], Au[BAND_N];  // A[i][i-1], A[i][i], A[i][i+1] (mod 64)
    double Bl[BAND_N], Bd[BAND_N], Bu[BAND_N];  // same for B = I + dt w_prev Jp
    double L1[BAND_N];                          // L[k+1][k]
    double Lr[BAND_N];                          // L[63][k]
    double Ud[BAND_N];                          // U[k][k]
    double Ur[BAND_N];                          // 1 / U[k][k] (div_rn)
    double Us[BAND_N];                          // U[k][63] (k <= 62)
    double c[BAND_N];
};

__device__ __forceinline__ double bsub(double a, double m, double u) {
    return __dsub_rn(a, __dmul_rn(m, u));
}

// Factorise the band matrix held in W (all lanes, identical values) and solve
// c = A^{-1}(-h) (W.c = -h on entry, the result on exit).  Returns 0 on success,
// 1 + k for a singular pivot k, -1 when a row swap would be needed.
__device__ __forceinline__ int band_factor_solve_c(BandWarpSmem& W) {
    const volatile BandWarpSmem& V = W;  // reads stay next to their use (see band_solve_col)
    double x[BAND_N];
    double chk = 0.0;  // becomes NaN if any factor entry is inf / NaN
#pragma unroll
    for (int i = 0; i < BAND_N; i++) x[i] = W.c[i];
    double d = V.Ad[0];        // running A[k][k]
    double s = V.Al[0];        // running A[k][63]  (row 0: periodic corner)
    double r = V.Au[63];       // running A[63][k]  (row 63: periodic corner)
    double r63 = V.Ad[63];     // running A[63][63]
    int status = 0;            // no early exits: the loop must unroll fully
#pragma unroll
    for (int k = 0; k < BAND_N - 1; k++) {
        if (status == 0) {
            // ---- pivot rule over the candidates {k, k+1, 63} ---------------
            const double akk = d;
            chk = fma(akk, 0.0, chk);
            double best = fabs(akk);
            int p = k;
            if (k < BAND_N - 2) {
                const double v1 = fabs(V.Al[k + 1]);
                if (v1 > best) {
                    best = v1;
                    p = k + 1;
                }
            }
            const double v2 = fabs(r);
            if (v2 > best) {
                best = v2;
                p = BAND_N - 1;
            }
            if (p != k) {
                status = -1;
            } else if (best < 1e-300) {
                status = 1 + k;
            } else {
                const double inv = 1.0 / akk;
                W.Ud[k] = akk;
                W.Ur[k] = inv;
                if (k < BAND_N - 2) {
                    const double m1 = V.Al[k + 1] * inv;
                    const double m2 = r * inv;
                    const double uk = V.Au[k];
                    W.L1[k] = m1;
                    W.Lr[k] = m2;
                    W.Us[k] = s;
                    chk = fma(m1, 0.0, chk);
                    chk = fma(m2, 0.0, chk);
                    chk = fma(s, 0.0, chk);
                    chk = fma(uk, 0.0, chk);
                    // row k+1: diagonal and column 63
                    const double dn = bsub(V.Ad[k + 1], m1, uk);
                    const double s_init = (k + 1 == BAND_N - 2) ? V.Au[BAND_N - 2] : 0.0;
                    const double sn = bsub(s_init, m1, s);
                    // row 63: column k+1 and column 63
                    const double r_init = (k + 1 == BAND_N - 2) ? V.Al[BAND_N - 1] : 0.0;
                    const double rn = bsub(r_init, m2, uk);
                    r63 = bsub(r63, m2, s);
                    // c: forward elimination with the same multipliers
                    x[k + 1] = bsub(x[k + 1], m1, x[k]);
                    x[BAND_N - 1] = bsub(x[BAND_N - 1], m2, x[k]);
                    d = dn;
                    s = sn;
                    r = rn;
                } else {
                    // k = 62: the only row below is 63 (its column-62 entry is r)
                    const double m2 = r * inv;
                    W.Lr[k] = m2;
                    W.Us[k] = s;  // A[62][63]
                    chk = fma(m2, 0.0, chk);
                    chk = fma(s, 0.0, chk);
                    r63 = bsub(r63, m2, s);
                    x[BAND_N - 1] = bsub(x[BAND_N - 1], m2, x[k]);
                    d = r63;
                }
            }
        }
    }
    if (status != 0) return status;
    // last pivot: no candidates below
    if (fabs(d) < 1e-300) return BAND_N;
    W.Ud[BAND_N - 1] = d;
    W.Ur[BAND_N - 1] = div_rn(1.0, d);
    if (isnan(fma(d, 0.0, chk))) return -1;  // non-finite factors: exact path
    // back substitution for c
    x[BAND_N - 1] = x[BAND_N - 1] * V.Ur[BAND_N - 1];
    x[BAND_N - 2] = bsub(x[BAND_N - 2], V.Us[BAND_N - 2], x[BAND_N - 1]) * V.Ur[BAND_N - 2];
#pragma unroll
    for (int i = BAND_N - 3; i >= 0; i--) {
        double acc = bsub(x[i], V.Au[i], x[i + 1]);
        acc = bsub(acc, V.Us[i], x[BAND_N - 1]);
        x[i] = acc * V.Ur[i];
    }
#pragma unroll
    for (int i = 0; i < BAND_N; i++) W.c[i] = x[i];
    return 0;
}

// x = A^{-1} x with the factors in W (one column per lane).  The back
// substitution multiplies by the pivot reciprocals (x / d and x * (1/d) are
// <= 1 ulp apart; 64 divisions per step instead of 64 per column).  The factor
// reads are volatile so they stay next to their use: hoisting all 320 of them
// ahead of the dependent chain would spill the register-resident column.
__device__ __forceinline__ void band_solve_col(const BandWarpSmem& Wn, double (&x)[BAND_N]) {
    const volatile BandWarpSmem& W = Wn;
#pragma unroll
    for (int k = 0; k < BAND_N - 2; k++) {
        x[k + 1] = bsub(x[k + 1], W.L1[k], x[k]);
        x[BAND_N - 1] = bsub(x[BAND_N - 1], W.Lr[k], x[k]);
    }
    x[BAND_N - 1] = bsub(x[BAND_N - 1], W.Lr[BAND_N - 2], x[BAND_N - 2]);
    x[BAND_N - 1] = x[BAND_N - 1] * W.Ur[BAND_N - 1];
    x[BAND_N - 2] = bsub(x[BAND_N - 2], W.Us[BAND_N - 2], x[BAND_N - 1]) * W.Ur[BAND_N - 2];
#pragma unroll
    for (int i = BAND_N - 3; i >= 0; i--) {
        double acc = bsub(x[i], W.Au[i], x[i + 1]);
        acc = bsub(acc, W.Us[i], x[BAND_N - 1]);
        x[i] = acc * W.Ur[i];
    }
}

}  // namespace odx
