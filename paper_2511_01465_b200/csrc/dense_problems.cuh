// dense_problems.cuh — row-parallel device functors for large state dims.
//
// For d = 64 a thread per state component evaluates f_i(x) and the i-th row
// of the (dense, zeros included) Jacobian — the same values the reference's
// jac_into writes (tests/golden/make_golden.py, oracle/odescan_oracle.c).
#pragma once

#include "problems.cuh"

namespace odx {

// Allen-Cahn method of lines, periodic (BASELINE cfg 4): params eps, dx.
// The dense path runs d = 64 only (dense_supported), so the periodic
// neighbours are masks.
struct AllenCahnRows {
    static constexpr int n = 64;
    double cdiff;
    __device__ __forceinline__ AllenCahnRows(const ProbParams& q, int dim)
        : cdiff(q.p[0] / (q.p[1] * q.p[1])) {
        (void)dim;
    }
    // non-contracted, as numpy evaluates it (problems.allen_cahn f_into)
    __device__ __forceinline__ double f(const double* x, int i) const {
        const double um = x[(i + n - 1) % n], ui = x[i], up = x[(i + 1) % n];
        const double lap = __dadd_rn(__dsub_rn(um, __dmul_rn(2.0, ui)), up);
        const double cub = __dsub_rn(ui, __dmul_rn(__dmul_rn(ui, ui), ui));
        return __dadd_rn(__dmul_rn(cdiff, lap), cub);
    }
    // Row i's entries that can be non-zero, as (column, value) pairs with the
    // same values jac(x, i, j) returns; every other entry of row i is 0.0.
    static constexpr int ROW_NZ = 3;
    __device__ __forceinline__ void jac_row(const double* x, int i, int* cols, double* vals) const {
        cols[0] = (i + n - 1) % n;
        cols[1] = i;
        cols[2] = (i + 1) % n;
#pragma unroll
        for (int q = 0; q < ROW_NZ; q++) vals[q] = jac(x, i, cols[q]);
    }
    // J[i][j] for j in [0, n)
    __device__ __forceinline__ double jac(const double* x, int i, int j) const {
        double v = 0.0;
        if (j == i) v = -2.0 * cdiff + (1.0 - 3.0 * (x[i] * x[i]));
        if (j == (i + n - 1) % n) v += cdiff;
        if (j == (i + 1) % n) v += cdiff;
        return v;
    }
};

}  // namespace odx
