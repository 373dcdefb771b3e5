// solve_dense.cu — d = 64 dense path (Allen-Cahn, BASELINE cfg 4).  (stub)
#include "common.cuh"
#include "solve_small.cuh"

namespace odx {

int dense_supported(const odx_problem*, const odx_stepper*) { return 0; }
int dense_solve(const odx_problem*, const odx_stepper*, SolveParams&, void*, size_t, cudaStream_t,
                bool, size_t*) {
    return fail(ODX_EUNSUPPORTED, "dense path not built");
}
int dense_build_op(const odx_problem*, const odx_stepper*, const StepCoefs&, const double*,
                   const double*, long long, double*, double*, double*, long long*, cudaStream_t) {
    return fail(ODX_EUNSUPPORTED, "dense path not built");
}
int dense_scan_op(const double*, const double*, long long, int, double*, double*, void*, size_t,
                  cudaStream_t) {
    return fail(ODX_EUNSUPPORTED, "dense path not built");
}
size_t dense_scan_op_ws(long long, int) { return 0; }

}  // namespace odx

extern "C" {
size_t odx_shard_workspace_bytes(const odx_problem*, const odx_stepper*, int64_t) { return 0; }
int odx_shard_local(const odx_problem*, const odx_stepper*, const double*, const double*, int64_t,
                    int64_t, double, double*, void*, size_t, void*) {
    return ODX_EUNSUPPORTED;
}
int odx_shard_fixup(const odx_problem*, const double*, int32_t, int32_t, double*, int64_t, double*,
                    void*, size_t, void*) {
    return ODX_EUNSUPPORTED;
}
}
