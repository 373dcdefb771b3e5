// dense_lu.cuh — K1 of the d = 64 path: one WARP builds one step's element
// with the reference's own factorisation (_kernels.py:28-77, :393-464):
//
//   A = I - dt w_next Jn        pivoted LU, reference pivot rule, 1e-300 floor
//   c = A^{-1}(-h)              lu_solve
//   F = A^{-1}(I + dt w_prev Jp) lu_solve per column (0 at step 0)
//
// Same operations, same order, non-contracted products — except that a
// product that is an exact zero times a FINITE number is skipped: x - (+-0)
// is x for every x (up to the sign of a zero result), so skipping it never
// changes a non-zero value, a NaN or an infinity.  For the Allen-Cahn
// Jacobian (periodic tridiagonal) the factors stay O(1) per row/column:
// the elimination touches ~4 entries per pivot instead of ~4000, and each
// triangular solve ~3 per row.  Dense matrices take the same code at full
// cost (every entry non-zero => nothing skipped).
//
// Sparsity is discovered at run time from exact zeros (warp ballots), never
// assumed, so row swaps and fill-in are handled as they occur.  A pivot
// step whose multipliers or pivot row hold a non-finite value updates the
// full trailing block (0 * inf must give NaN, as in the reference).
//
// Layout (shared memory, per warp): A[64][65] (odd stride: row and column
// walks are both conflict-free), the right-hand sides X[64][64] (lane l owns
// columns l and l+32; c is a third column every lane carries redundantly),
// pivots and the per-row / per-column non-zero masks of U and L.
#pragma once

#include "common.cuh"
#include "dense_problems.cuh"
#include "scan.cuh"

namespace odx {

constexpr int LU_N = 64;
constexpr int LU_LD = 65;
constexpr int LU_WARPS = 3;  // warps (= steps in flight) per CTA; ~70 KB smem each

struct LuWarpSmem {
    double A[LU_N * LU_LD];
    double X[LU_N * LU_N];
    double cs[LU_N];
    double xk[LU_N];
    double xp[LU_N];
    unsigned long long Lmask[LU_N];  // rows i > k with L[i][k] != 0
    unsigned long long Umask[LU_N];  // cols j > i with U[i][j] != 0
    int piv[LU_N];
};

__device__ __forceinline__ double nc_sub_mul(double a, double m, double u) {
    return __dsub_rn(a, __dmul_rn(m, u));
}

// Pivoted LU of W.A in place (reference lu_factor).  Returns the first
// singular column or -1.  Warp-collective.
__device__ __forceinline__ int warp_lu_factor(LuWarpSmem& W, int lane) {
    double* A = W.A;
    for (int k = 0; k < LU_N; k++) {
        // ---- pivot: start from row k, a later row wins only if strictly
        // larger (first max); a NaN never wins; NaN at the diagonal stays
        // Only rows with a non-zero (or NaN) entry can win: walk them in order.
        const double d0 = fabs(A[k * LU_LD + k]);
        double bv = d0;
        int bi = k;
        unsigned long long cand =
            (unsigned long long)__ballot_sync(FULL, lane > k && A[lane * LU_LD + k] != 0.0) |
            ((unsigned long long)__ballot_sync(FULL, A[(lane + 32) * LU_LD + k] != 0.0 && lane + 32 > k)
             << 32);
        while (cand) {
            const int i = __ffsll((long long)cand) - 1;
            cand &= cand - 1;
            const double v = fabs(A[i * LU_LD + k]);
            if (v > bv) {
                bv = v;
                bi = i;
            }
        }
        if (bv < 1e-300) return k;
        if (lane == 0) W.piv[k] = bi;
        if (bi != k) {
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int j = lane + 32 * h;
                const double t = A[k * LU_LD + j];
                A[k * LU_LD + j] = A[bi * LU_LD + j];
                A[bi * LU_LD + j] = t;
            }
            __syncwarp();
        }
        const double inv = 1.0 / A[k * LU_LD + k];
        // ---- multipliers (rows below k) and the pivot row (cols right of k)
        double m[2], u[2];
        bool mz[2], mnf[2], uz[2], unf[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int i = lane + 32 * h;
            const bool below = i > k;
            m[h] = below ? A[i * LU_LD + k] * inv : 0.0;
            if (below) A[i * LU_LD + k] = m[h];
            mz[h] = below && m[h] != 0.0;  // NaN counts as non-zero
            mnf[h] = below && !isfinite(m[h]);
            u[h] = below ? A[k * LU_LD + i] : 0.0;
            uz[h] = below && u[h] != 0.0;
            unf[h] = below && !isfinite(u[h]);
        }
        const unsigned long long rmask =
            (unsigned long long)__ballot_sync(FULL, mz[0]) |
            ((unsigned long long)__ballot_sync(FULL, mz[1]) << 32);
        const unsigned long long cmask =
            (unsigned long long)__ballot_sync(FULL, uz[0]) |
            ((unsigned long long)__ballot_sync(FULL, uz[1]) << 32);
        const bool poisoned = __any_sync(FULL, mnf[0] || mnf[1] || unf[0] || unf[1]);
        __syncwarp();
        if (!poisoned) {
            // exact-zero products skipped: rows with m = 0 and columns with u = 0
            unsigned long long rm = rmask;
            const bool c0 = (cmask >> lane) & 1ull, c1 = (cmask >> (lane + 32)) & 1ull;
            while (rm) {
                const int i = __ffsll((long long)rm) - 1;
                rm &= rm - 1;
                const double mi = A[i * LU_LD + k];
                if (c0) A[i * LU_LD + lane] = nc_sub_mul(A[i * LU_LD + lane], mi, u[0]);
                if (c1) A[i * LU_LD + lane + 32] = nc_sub_mul(A[i * LU_LD + lane + 32], mi, u[1]);
            }
        } else {
            for (int i = k + 1; i < LU_N; i++) {
                const double mi = A[i * LU_LD + k];
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int j = lane + 32 * h;
                    if (j > k) A[i * LU_LD + j] = nc_sub_mul(A[i * LU_LD + j], mi, A[k * LU_LD + j]);
                }
            }
        }
        __syncwarp();
    }
    return -1;
}

// Non-zero structure of the finished factors (after all row swaps).
__device__ __forceinline__ void warp_lu_masks(LuWarpSmem& W, int lane) {
    const double* A = W.A;
    for (int r = 0; r < LU_N; r++) {
        // U row r: columns j > r; L column r: rows i > r
        const unsigned long long um =
            (unsigned long long)__ballot_sync(FULL, lane > r && A[r * LU_LD + lane] != 0.0) |
            ((unsigned long long)__ballot_sync(FULL, lane + 32 > r && A[r * LU_LD + lane + 32] != 0.0)
             << 32);
        const unsigned long long lm =
            (unsigned long long)__ballot_sync(FULL, lane > r && A[lane * LU_LD + r] != 0.0) |
            ((unsigned long long)__ballot_sync(FULL, lane + 32 > r && A[(lane + 32) * LU_LD + r] != 0.0)
             << 32);
        if (lane == 0) {
            W.Umask[r] = um;
            W.Lmask[r] = lm;
        }
    }
    __syncwarp();
}

// lu_solve (reference :60-77) on three right-hand sides at once: this lane's
// columns `lane` and `lane + 32` of X and the shared column cs (every lane
// carries it, writing identical values).  Exact-zero products are skipped only
// while every multiplied value in the warp is finite (warp-uniform branch).
__device__ __forceinline__ void warp_lu_solve3(LuWarpSmem& W, int lane, bool with_X) {
    const double* A = W.A;
    double* x0 = W.X + lane;
    double* x1 = W.X + lane + 32;
    double* x2 = W.cs;
    for (int k = 0; k < LU_N; k++) {
        const int p = W.piv[k];
        if (p != k) {
            double t;
            if (with_X) {
                t = x0[k * LU_N]; x0[k * LU_N] = x0[p * LU_N]; x0[p * LU_N] = t;
                t = x1[k * LU_N]; x1[k * LU_N] = x1[p * LU_N]; x1[p * LU_N] = t;
            }
            t = x2[k]; x2[k] = x2[p]; x2[p] = t;
        }
        const double a0 = with_X ? x0[k * LU_N] : 0.0, a1 = with_X ? x1[k * LU_N] : 0.0, a2 = x2[k];
        const bool fin = __all_sync(FULL, isfinite(a0) && isfinite(a1) && isfinite(a2));
        if (fin) {
            unsigned long long m = W.Lmask[k];
            while (m) {
                const int i = __ffsll((long long)m) - 1;
                m &= m - 1;
                const double l = A[i * LU_LD + k];
                if (with_X) {
                    x0[i * LU_N] = nc_sub_mul(x0[i * LU_N], l, a0);
                    x1[i * LU_N] = nc_sub_mul(x1[i * LU_N], l, a1);
                }
                x2[i] = nc_sub_mul(x2[i], l, a2);
            }
        } else {
            for (int i = k + 1; i < LU_N; i++) {
                const double l = A[i * LU_LD + k];
                if (with_X) {
                    x0[i * LU_N] = nc_sub_mul(x0[i * LU_N], l, a0);
                    x1[i * LU_N] = nc_sub_mul(x1[i * LU_N], l, a1);
                }
                x2[i] = nc_sub_mul(x2[i], l, a2);
            }
        }
    }
    bool nf = false;  // a non-finite x[j], j > i, forbids skipping U[i][j] == 0
    for (int i = LU_N - 1; i >= 0; i--) {
        double c0 = with_X ? x0[i * LU_N] : 0.0, c1 = with_X ? x1[i * LU_N] : 0.0, c2 = x2[i];
        if (!nf) {
            unsigned long long m = W.Umask[i];
            while (m) {
                const int j = __ffsll((long long)m) - 1;
                m &= m - 1;
                const double u = A[i * LU_LD + j];
                if (with_X) {
                    c0 = nc_sub_mul(c0, u, x0[j * LU_N]);
                    c1 = nc_sub_mul(c1, u, x1[j * LU_N]);
                }
                c2 = nc_sub_mul(c2, u, x2[j]);
            }
        } else {
            for (int j = i + 1; j < LU_N; j++) {
                const double u = A[i * LU_LD + j];
                if (with_X) {
                    c0 = nc_sub_mul(c0, u, x0[j * LU_N]);
                    c1 = nc_sub_mul(c1, u, x1[j * LU_N]);
                }
                c2 = nc_sub_mul(c2, u, x2[j]);
            }
        }
        const double dg = A[i * LU_LD + i];
        if (with_X) {
            c0 = c0 / dg;
            c1 = c1 / dg;
            x0[i * LU_N] = c0;
            x1[i * LU_N] = c1;
        }
        c2 = c2 / dg;
        x2[i] = c2;
        nf = __any_sync(FULL, nf || !isfinite(c0) || !isfinite(c1) || !isfinite(c2));
    }
}

}  // namespace odx
