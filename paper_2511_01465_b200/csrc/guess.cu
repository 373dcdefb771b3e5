// guess.cu — the reference's initial-guess policies on the device
// (newton_pint.initial_guess, newton_pint.py:174-207): the O(N d) fill and
// the coarse explicit-Euler sweep happen where the solve runs, so a policy
// guess costs no host construction and no host-to-device copy.
#include "common.cuh"
#include "dense_problems.cuh"
#include "dispatch.cuh"

namespace odx {

// The policy's constant row (ones / zeros / x0 of trajectory b).
__device__ __forceinline__ double policy_value(int policy, const double* x0, long long b, int d,
                                              int j) {
    return policy == ODX_GUESS_ONES ? 1.0 : policy == ODX_GUESS_ZEROS ? 0.0 : x0[b * d + j];
}

// Fill: grid (chunks, B) — every CTA streams a slice of trajectory b
// (blockIdx.y), 16-byte stores when the row width allows.
__global__ void guess_fill_kernel(int policy, const double* x0, double* X, long long N, int d) {
    const long long b = blockIdx.y;
    double* Xb = X + b * N * d;
    const long long total = N * d;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (d == 2 && (reinterpret_cast<size_t>(Xb) & 15) == 0) {
        const double2 v = make_double2(policy_value(policy, x0, b, 2, 0),
                                       policy_value(policy, x0, b, 2, 1));
        double2* X2 = reinterpret_cast<double2*>(Xb);
        for (long long q = t0; q < N; q += stride) X2[q] = v;
        return;
    }
    for (long long q = t0; q < total; q += stride) Xb[q] = policy_value(policy, x0, b, d, (int)(q % d));
}

// coarse_euler (newton_pint.py:191-207): the coarse explicit-Euler march over
// every stride-th row, one thread per trajectory (small d), written at the
// head of each stride; guess_spread_kernel then copies the heads across.
template <class P>
__global__ void guess_coarse_kernel(ProbParams pp, const double* x0, double* X, long long B,
                                    long long N, double dt) {
    constexpr int D = P::D;
    const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    double* Xb = X + b * N * D;
    const long long stride = N / 100 > 1 ? N / 100 : 1;
    const double dtc = (double)stride * dt;
    const P prob(pp);
    double vv[D], f[D];
#pragma unroll
    for (int j = 0; j < D; j++) vv[j] = x0[b * D + j];
    for (long long k = 0; k < N; k += stride) {
        prob.f(vv, f);
#pragma unroll
        for (int j = 0; j < D; j++) {
            vv[j] = __dadd_rn(vv[j], __dmul_rn(dtc, f[j]));  // v + dt_coarse * f(v)
            Xb[k * D + j] = vv[j];
        }
    }
}

__global__ void guess_spread_kernel(double* X, long long N, int d) {
    const long long b = blockIdx.y;
    double* Xb = X + b * N * d;
    const long long stride = N / 100 > 1 ? N / 100 : 1;
    const long long st = (long long)gridDim.x * blockDim.x;
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < N * d; q += st) {
        const long long k = q / d;
        const long long head = (k / stride) * stride;
        if (k != head) Xb[q] = Xb[head * d + (q % d)];
    }
}

// d = 64 Allen-Cahn: the coarse sweep evaluates f row by row, one CTA per
// trajectory (heads only; guess_spread_kernel copies them across).
__global__ void guess_dense_coarse_kernel(ProbParams pp, const double* x0, double* X, long long N,
                                          double dt) {
    constexpr int D = 64;
    const long long b = blockIdx.x;
    double* Xb = X + b * N * D;
    __shared__ double v[D], f[D];
    for (int j = threadIdx.x; j < D; j += blockDim.x) v[j] = x0[b * D + j];
    __syncthreads();
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
}

// CTAs per trajectory for the streaming fill / spread: ~8 per SM over the batch
inline dim3 guess_grid(long long B, long long N, int d) {
    long long per = (8LL * num_sms() + B - 1) / B;
    const long long need = (N * d + 256 * 8 - 1) / (256 * 8);
    if (per > need) per = need;
    if (per < 1) per = 1;
    return dim3((unsigned)per, (unsigned)B);
}

// validation only: with_small_problem's id / dim checks
struct KnownProblem {
    template <class Q>
    int operator()() { return ODX_OK; }
};

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
        guess_coarse_kernel<P><<<(unsigned)((B + 127) / 128), 128, 0, st>>>(pp, x0, X, B, N, dt);
        guess_spread_kernel<<<guess_grid(B, N, P::D), 256, 0, st>>>(X, N, P::D);
        ODX_CUDA(cudaGetLastError());
        count_launch(2);
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
    if (B > 65535) return fail(ODX_EINVAL, "B must be <= 65535");
    const bool dense = P->problem_id == ODX_PROB_ALLEN_CAHN && P->dim == 64;
    if (!dense) {  // the same problem / dim validation as the solve
        if (int rc = with_small_problem(P->problem_id, P->dim, KnownProblem{}))
            return fail(rc, rc == ODX_EINVAL ? "problem does not have this dim"
                                             : "unknown problem id (no device functor)");
    }
    if (policy != ODX_GUESS_COARSE_EULER) {  // a constant row: one streaming fill
        guess_fill_kernel<<<guess_grid(B, N, P->dim), 256, 0, st>>>(policy, x0, X, N, P->dim);
        ODX_CUDA(cudaGetLastError());
        count_launch(1);
        return ODX_OK;
    }
    if (dense) {
        guess_dense_coarse_kernel<<<(unsigned)B, 64, 0, st>>>(pp, x0, X, N, dt);
        guess_spread_kernel<<<guess_grid(B, N, 64), 256, 0, st>>>(X, N, 64);
        ODX_CUDA(cudaGetLastError());
        count_launch(2);
        return ODX_OK;
    }
    return with_small_problem(P->problem_id, P->dim, GuessFn{pp, policy, x0, X, B, N, dt, st});
}
