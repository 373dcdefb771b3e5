// build_op.cuh — per-step build ops (one thread per step, dense outputs like
// the reference's build_explicit/_implicit, _kernels.py:299-342 / :393-464).
// Instantiated per problem by the generated translation units (csrc/gen/).
#pragma once
#include <climits>

#include "common.cuh"
#include "dispatch.cuh"

namespace odx {

// ---------------------------------------------------------------------------
// build ops: one thread per step, dense outputs like the reference.
// ---------------------------------------------------------------------------
template <class P, int KIND, int S>
__global__ void __launch_bounds__(128)
build_op_kernel(const ProbParams pp, const StepCoefs sc, const double* __restrict__ x0,
                const double* __restrict__ X, long long N, double* __restrict__ Fe,
                double* __restrict__ ce, double* __restrict__ h, long long* first_bad,
                long long offset) {
    constexpr int D = P::D;
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= N) return;
    const P prob(pp);
    double prev[D], xk[D], hh[D];
#pragma unroll
    for (int j = 0; j < D; j++) {
        prev[j] = (k == 0) ? x0[j] : X[(k - 1) * D + j];
        xk[j] = X[k * D + j];
    }
    Elem<D> el;
    // prev = x0 (the halo) for the first local step; F is zeroed only for the
    // trajectory's global first step (offset + k == 0)
    bool sing = build_step<P, KIND, S>(prob, sc, prev, xk, offset + k == 0, el, hh);
#pragma unroll
    for (int j = 0; j < D; j++) {
        h[k * D + j] = hh[j];
        ce[k * D + j] = el.c[j];
    }
#pragma unroll
    for (int j = 0; j < D * D; j++) Fe[k * D * D + j] = el.F[j];
    if (KIND == 1 && sing) atomicMin(first_bad, offset + k);
}

static __global__ void set_i64_kernel(long long* p, long long v) { *p = v; }
static __global__ void finalize_bad_kernel(long long* p) {
    if (*p == LLONG_MAX) *p = -1;
}

template <class P, int KIND, int S>
int build_op(const ProbParams& pp, const StepCoefs& sc, const double* x0, const double* X,
             long long N, double* Fe, double* ce, double* h, long long* first_bad,
             cudaStream_t st, long long offset) {
    if (KIND == 1) set_i64_kernel<<<1, 1, 0, st>>>(first_bad, LLONG_MAX);
    if (N > 0)
        build_op_kernel<P, KIND, S><<<(unsigned)((N + 127) / 128), 128, 0, st>>>(pp, sc, x0, X, N, Fe,
                                                                                 ce, h, first_bad, offset);
    if (KIND == 1) finalize_bad_kernel<<<1, 1, 0, st>>>(first_bad);
    ODX_CUDA(cudaGetLastError());
    count_launch((N > 0 ? 1 : 0) + (KIND == 1 ? 2 : 0));
    return ODX_OK;
}

}  // namespace odx
