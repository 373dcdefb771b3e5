// trace_ws.cu — standalone timeline trace of the warp-specialised persistent
// solve (VdP mu=1 RK4, BASELINE cfg 5 shape).  Build:
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -DODX_TRACE \
//        -I include -o tools/trace_ws tools/trace_ws.cu paper_2511_01465_b200/csrc/{host_util,ops}.cu
// Run: tools/trace_ws <N> <iters> > trace.bin  (8 u64 per tile of iteration 1)
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2511_01465_b200/csrc/solve_small_launch.cuh"

using namespace odx;

int main(int argc, char** argv) {
    long long N = argc > 1 ? atoll(argv[1]) : (1LL << 22);
    int iters = argc > 2 ? atoi(argv[2]) : 3;
    odx_problem P{};
    P.problem_id = ODX_PROB_VDP; P.dim = 2; P.n_params = 1; P.params[0] = 1.0;
    odx_stepper S{};
    S.kind = ODX_STEP_EXPLICIT_RK; S.stages = 4;
    S.a[4] = 0.5; S.a[9] = 0.5; S.a[14] = 1.0;
    S.b[0] = 1.0 / 6; S.b[1] = 1.0 / 3; S.b[2] = 1.0 / 3; S.b[3] = 1.0 / 6;
    odx_newton_cfg C{iters, 0, 0.0, 0.0};
    double *x0, *X, *hist, *shist; int *it, *st; long long* ix;
    cudaMalloc(&x0, 16); cudaMalloc(&X, N * 16); cudaMalloc(&hist, 8 * (iters + 1));
    cudaMalloc(&shist, 8 * (iters + 1)); cudaMalloc(&it, 4); cudaMalloc(&st, 4); cudaMalloc(&ix, 8);
    std::vector<double> h(2 * N);
    for (long long k = 0; k < N; k++) { h[2 * k] = 2.0; h[2 * k + 1] = 0.0; }
    cudaMemcpy(x0, h.data(), 16, cudaMemcpyHostToDevice);
    size_t ws_bytes = 0;
    {
        SolveParams q{};
        q.B = 1; q.N = N; q.max_iters = iters;
        solve_small<VanDerPol, 0, 4>(q, nullptr, 0, 0, true, &ws_bytes);
    }
    void* ws; cudaMalloc(&ws, ws_bytes);
    long long ntiles = (N + 255) / 256;
    unsigned long long* tr; cudaMalloc(&tr, ntiles * 128); cudaMemset(tr, 0, ntiles * 128);
    cudaMemcpyToSymbol(g_trace, &tr, sizeof(tr));
    for (int rep = 0; rep < 2; rep++) {
        cudaMemcpy(X, h.data(), N * 16, cudaMemcpyHostToDevice);
        SolveParams p{};
        fill_params(&P, p.prob); fill_coefs(&S, 1e-3, p.sc);
        p.x0 = x0; p.X = X; p.B = 1; p.N = N; p.max_iters = iters; p.abort_nonfinite = 0;
        p.hist = hist; p.shist = shist; p.iters = it; p.status = st; p.sidx = (long long*)ix;
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        int rc = solve_small<VanDerPol, 0, 4>(p, ws, ws_bytes, 0, false, nullptr);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        fprintf(stderr, "rc=%d %s  ms=%.3f  ntiles=%lld\n", rc, cudaGetErrorString(cudaGetLastError()), ms, ntiles);
    }
    std::vector<unsigned long long> ht(ntiles * 16);
    cudaMemcpy(ht.data(), tr, ntiles * 128, cudaMemcpyDeviceToHost);
    fwrite(ht.data(), 8, ht.size(), stdout);
    return 0;
}
