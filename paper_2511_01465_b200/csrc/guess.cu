// guess.cu — the reference's initial-guess policies on the device
// (newton_pint.initial_guess, newton_pint.py:174-207): the O(N d) fill and
// the coarse explicit-Euler sweep happen where the solve runs, so a policy
// guess costs no host construction and no host-to-device copy.
#include "common.cuh"
#include "dense_problems.cuh"
#include "dispatch.cuh"

namespace odx {

__device__ __forceinline__ void fill_rows(double* Xb, const double* v, long long lo, long long hi,
                                          int d) {
    for (long long q = lo * d + threadIdx.x; q < hi * d; q += blockDim.x) Xb[q] = v[q % d];
}

// One CTA per trajectory.  Small-d problems: functor P (f(x, out)).
template <class P>
__global__ void guess_kernel(ProbParams pp, int policy, const double* x0, double* X, long long N,
                             double dt) {
    constexpr int D = P::D;
    const long long b = blockIdx.x;
    double* Xb = X + b * N * D;
    __shared__ double v[D];
    if (threadIdx.x == 0) {
#pragma unroll
        for (int j = 0; j < D; j++)
            v[j] = policy == ODX_GUESS_ONES ? 1.0 : policy == ODX_GUESS_ZEROS ? 0.0 : x0[b * D + j];
    }
    __syncthreads();
    if (policy != ODX_GUESS_COARSE_EULER) {
        fill_rows(Xb, v, 0, N, D);
        return;
    }
    const long long stride = N / 100 > 1 ? N / 100 : 1;
    const double dtc = (double)stride * dt;
    // thread 0 marches the coarse grid, writing each value at the head of its
    // stride; then every thread copies the heads across their strides
    if (threadIdx.x == 0) {
        const P prob(pp);
        double vv[D], f[D];
#pragma unroll
        for (int j = 0; j < D; j++) vv[j] = v[j];
        for (long long k = 0; k < N; k += stride) {
            prob.f(vv, f);
#pragma unroll
            for (int j = 0; j < D; j++) {
                vv[j] = __dadd_rn(vv[j], __dmul_rn(dtc, f[j]));  // v + dt_coarse * f(v)
                Xb[k * D + j] = vv[j];
            }
        }
    }
    __syncthreads();
    for (long long q = threadIdx.x; q < N * D; q += blockDim.x) {
        const long long k = q / D;
        const long long head = (k / stride) * stride;
        if (k != head) Xb[q] = Xb[head * D + (q % D)];
    }
}

// d = 64 Allen-Cahn: the coarse sweep evaluates f row by row.
__global__ void guess_dense_kernel(ProbParams pp, int policy, const double* x0, double* X,
                                   long long N, double dt) {
    constexpr int D = 64;
    const long long b = blockIdx.x;
    double* Xb = X + b * N * D;
    __shared__ double v[D], f[D];
    for (int j = threadIdx.x; j < D; j += blockDim.x)
        v[j] = policy == ODX_GUESS_ONES ? 1.0 : policy == ODX_GUESS_ZEROS ? 0.0 : x0[b * D + j];
    __syncthreads();
    if (policy != ODX_GUESS_COARSE_EULER) {
        fill_rows(Xb, v, 0, N, D);
        return;
    }
    const long long stride = N / 100 > 1 ? N / 100 : 1;
    const double dtc = (double)stride * dt;
    const AllenCahnRows prob(pp, D);
    for (long long k = 0; k < N; k += stride) {
        for (int j = threadIdx.x; j < D; j += blockDim.x) f[j] = prob.f(v, j);
        __syncthreads();
        for (int j = threadIdx.x; j < D; j += blockDim.x) {
            v[j] = __dadd_rn(v[j], __dmul_rn(dtc, f[j]));
            Xb[k * D + j] = v[j];
        }
        __syncthreads();
    }
    for (long long q = threadIdx.x; q < N * D; q += blockDim.x) {
        const long long k = q / D;
        const long long head = (k / stride) * stride;
        if (k != head) Xb[q] = Xb[head * D + (q % D)];
    }
}

struct GuessFn {
    ProbParams pp;
    int policy;
    const double* x0;
    double* X;
    long long B, N;
    double dt;
    cudaStream_t st;
    template <class P>
    int operator()() {
        guess_kernel<P><<<(unsigned)B, 256, 0, st>>>(pp, policy, x0, X, N, dt);
        ODX_CUDA(cudaGetLastError());
        count_launch(1);
        return ODX_OK;
    }
};

}  // namespace odx

using namespace odx;

extern "C" int odx_initial_guess(const odx_problem* P, int32_t policy, const double* x0, double* X,
                                 int64_t B, int64_t N, double dt, void* stream) {
    if (!P || !X || (!x0 && policy == ODX_GUESS_REPLICATE_X0) ||
        (!x0 && policy == ODX_GUESS_COARSE_EULER))
        return fail(ODX_EINVAL, "null descriptor or device buffer");
    if (policy < ODX_GUESS_ONES || policy > ODX_GUESS_COARSE_EULER)
        return fail(ODX_EINVAL, "unknown initial-guess policy");
    if (B < 1 || N < 1) return fail(ODX_EINVAL, "B and N must be >= 1");
    ProbParams pp;
    if (!fill_params(P, pp)) return fail(ODX_EINVAL, "bad problem parameters");
    cudaStream_t st = (cudaStream_t)stream;
    if (P->problem_id == ODX_PROB_ALLEN_CAHN && P->dim == 64) {
        guess_dense_kernel<<<(unsigned)B, 256, 0, st>>>(pp, policy, x0, X, N, dt);
        ODX_CUDA(cudaGetLastError());
        count_launch(1);
        return ODX_OK;
    }
    return with_small_problem(P->problem_id, P->dim, GuessFn{pp, policy, x0, X, B, N, dt, st});
}
