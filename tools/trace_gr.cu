// trace_gr.cu — per-phase %globaltimer stamps of the grid-resident solve
// (BASELINE cfg 2 shape: VdP mu=10, backward Euler, N=65536, 10 iterations).
// Build: nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -DODX_GR_TRACE \
//        -I include -o tools/trace_gr tools/trace_gr.cu paper_2511_01465_b200/csrc/{host_util,ops}.cu
#include <cstdio>
#include <vector>

#include "../paper_2511_01465_b200/csrc/solve_small_launch.cuh"

using namespace odx;

int main(int argc, char** argv) {
    const long long N = argc > 1 ? atoll(argv[1]) : 65536;
    const int iters = 10;
    odx_problem P{};
    P.problem_id = ODX_PROB_VDP; P.dim = 2; P.n_params = 1; P.params[0] = 10.0;
    odx_stepper S{};
    S.kind = ODX_STEP_IMPLICIT_WEIGHTED; S.stages = 1; S.w_prev = 0.0; S.w_next = 1.0;
    double *x0, *X, *hist, *shist; int *it, *st; long long* ix;
    cudaMalloc(&x0, 16); cudaMalloc(&X, N * 16); cudaMalloc(&hist, 8 * (iters + 1));
    cudaMalloc(&shist, 8 * (iters + 1)); cudaMalloc(&it, 4); cudaMalloc(&st, 4); cudaMalloc(&ix, 8);
    std::vector<double> h(2 * N);
    const bool nan_fill = argc > 2 && argv[2][0] == 'n';  // every row NaN (diverged data)
    for (long long k = 0; k < N; k++) { h[2 * k] = 2.0; h[2 * k + 1] = 0.0; }
    if (nan_fill)
        for (long long k = 1; k < N; k++) h[2 * k] = h[2 * k + 1] = __builtin_nan("");
    cudaMemcpy(x0, h.data(), 16, cudaMemcpyHostToDevice);
    size_t ws_bytes = 0;
    { SolveParams q{}; q.B = 1; q.N = N; q.max_iters = iters;
      solve_small<VanDerPol, 1, 1>(q, nullptr, 0, 0, true, &ws_bytes); }
    void* ws; cudaMalloc(&ws, ws_bytes);
    unsigned long long* tr; cudaMalloc(&tr, 3 * 64 * 16 * 8); cudaMemset(tr, 0, 3 * 64 * 16 * 8);
    cudaMemcpyToSymbol(g_gr_trace, &tr, sizeof(tr));
    for (int rep = 0; rep < 5; rep++) {
        cudaMemcpy(X, h.data(), N * 16, cudaMemcpyHostToDevice);
        SolveParams p{};
        fill_params(&P, p.prob); fill_coefs(&S, 1e-3, p.sc);
        p.x0 = x0; p.X = X; p.B = 1; p.N = N; p.max_iters = iters; p.abort_nonfinite = 0;
        p.hist = hist; p.shist = shist; p.iters = it; p.status = st; p.sidx = ix;
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        int rc = solve_small<VanDerPol, 1, 1>(p, ws, ws_bytes, 0, false, nullptr);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        fprintf(stderr, "rc=%d %s ms=%.4f\n", rc, cudaGetErrorString(cudaGetLastError()), ms);
    }
    std::vector<unsigned long long> ht(3 * 64 * 16);
    cudaMemcpy(ht.data(), tr, ht.size() * 8, cudaMemcpyDeviceToHost);
    const char* names[] = {"halo", "build", "scan", "agg+red", "barrier", "decide", "fold", "apply", "tail"};
    unsigned long long t0 = ht[0];
    for (int c = 0; c < 3; c++) {
        printf("CTA %s\n", c == 0 ? "0" : c == 1 ? "G/2" : "G-1");
        for (int i = 0; i <= iters; i++) {
            const unsigned long long* r = &ht[(c * 64 + i) * 16];
            printf("  it %2d start %7.2f us |", i, (r[0] - t0) / 1e3);
            for (int k = 1; k <= 9; k++)
                if (r[k]) printf(" %s %5.2f", names[k - 1], (r[k] - r[k - 1]) / 1e3);
            printf("\n");
        }
    }
    return 0;
}
