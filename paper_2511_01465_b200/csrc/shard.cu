// shard.cu — time-sharded Newton iteration (one rank per GPU).
//
// Rank r owns steps [offset, offset + N_local) of one trajectory and, per
// Newton iteration of the reference loop (newton_pint.py:366-396):
//   odx_shard_local : elements of its steps from (halo, X_local) — the halo is
//                     the last state of rank r-1 (x0 on rank 0) — a local
//                     inclusive scan (kept in the workspace), and a summary
//                     record [F_agg | c_agg | x_last | rn | sc | step_prev | bad]
//   (caller)        : all-gather of the records (NCCL), identical decision on
//                     every rank
//   odx_shard_fixup : carry z_r = A_{r-1}(...A_0(0)) from the gathered
//                     aggregates, X_local += Fp_k z_r + cp_k, max|dx| -> step
// The next halo is halo + z_r (rank r-1's last dx IS z_r), so the halo needs
// no extra exchange.
#include <climits>
#include <cstring>

#include "common.cuh"
#include "scan.cuh"

namespace odx {

int build_common_offset(const odx_problem* P, const odx_stepper* S, int kind, const double* x0,
                        const double* X, int64_t N, double dt, double* Fe, double* ce, double* h,
                        int64_t* first_bad, void* stream, long long offset);
int scan_op(const double* F, const double* c, long long N, int d, double* Fp, double* cp,
            void* ws, size_t ws_bytes, cudaStream_t st);
size_t scan_op_ws(long long N, int d);
int max_abs_op(const double* A, long long n, int d, double* out, cudaStream_t st);
int dense_supported(const odx_problem* P, const odx_stepper* S);

struct ShardLayout {
    size_t Fe, ce, h, Fp, cp, scal, scanws, total;
    ShardLayout(long long n, int d) {
        size_t off = 0;
        auto at = [&](size_t bytes) { off = align_up(off, 256); size_t o = off; off += bytes; return o; };
        Fe = at((size_t)n * d * d * 8);
        ce = at((size_t)n * d * 8);
        h = at((size_t)n * d * 8);
        Fp = at((size_t)n * d * d * 8);
        cp = at((size_t)n * d * 8);
        scal = at(64);  // first_bad (i64), rn, sc, z[4]
        scanws = at(scan_op_ws(n, d));
        total = off + 256;
    }
};

__global__ void shard_record_kernel(const double* Fp, const double* cp, const double* X, long long n,
                                    int d, const double* scal, int explicit_kind, double* rec) {
    // scal: [first_bad (as i64), rn, sc]
    const int t = threadIdx.x;
    const int dd = d * d;
    if (t < dd) rec[t] = Fp[(n - 1) * dd + t];
    if (t < d) {
        rec[dd + t] = cp[(n - 1) * d + t];
        rec[dd + d + t] = X[(n - 1) * d + t];
    }
    if (t == 0) {
        const long long bad = reinterpret_cast<const long long*>(scal)[0];
        rec[dd + 2 * d + 0] = scal[1];
        rec[dd + 2 * d + 1] = explicit_kind ? scal[1] : scal[2];
        rec[dd + 2 * d + 2] = __longlong_as_double(0x7ff8000000000000ll);  // step_prev: caller
        rec[dd + 2 * d + 3] = (double)bad;
    }
}

// out = F z + c.  One non-inlined function for both the carry fold and the
// fix-up, so rank r's carry is bit-identical to rank r-1's last dx (the halo
// update relies on it).
__device__ __noinline__ void affine_apply(const double* F, const double* c, const double* z, int d,
                                          double* out) {
    for (int r = 0; r < d; r++) {
        double acc = c[r];
        for (int q = 0; q < d; q++) acc = __fma_rn(F[r * d + q], z[q], acc);
        out[r] = acc;
    }
}

// carry of `rank` from the gathered records; halo += carry (rank > 0)
__global__ void shard_carry_kernel(const double* recs, int rank, int d, double* z, double* halo) {
    if (threadIdx.x != 0) return;
    const int R = ODX_SHARD_REC(d);
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    for (int q = 0; q < rank; q++) {
        const double* F = recs + (long long)q * R;
        double t[4];
        affine_apply(F, F + d * d, v, d, t);
        for (int r = 0; r < d; r++) v[r] = t[r];
    }
    for (int r = 0; r < d; r++) z[r] = v[r];
    if (halo && rank > 0)
        for (int r = 0; r < d; r++) halo[r] = halo[r] + v[r];
}

__global__ void shard_apply_kernel(const double* Fp, const double* cp, const double* z, long long n,
                                   int d, double* X, double* dxbuf) {
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    double acc[4];
    affine_apply(Fp + k * d * d, cp + k * d, z, d, acc);
    for (int r = 0; r < d; r++) {
        X[k * d + r] = X[k * d + r] + acc[r];
        dxbuf[k * d + r] = acc[r];
    }
}

}  // namespace odx

using namespace odx;

extern "C" {

size_t odx_shard_workspace_bytes(const odx_problem* P, const odx_stepper* S, int64_t N_local) {
    if (!P || !S || P->dim < 1 || P->dim > 4 || N_local < 1 || dense_supported(P, S)) return 0;
    // + an n x d scratch for dx (the step reduction) reuses the h buffer
    return ShardLayout(N_local, P->dim).total;
}

int odx_shard_local(const odx_problem* P, const odx_stepper* S, const double* halo,
                    const double* X_local, int64_t N_local, int64_t offset, double dt,
                    double* record, void* workspace, size_t workspace_bytes, void* stream) {
    if (!P || !S || P->dim < 1 || P->dim > 4 || dense_supported(P, S))
        return fail(ODX_EUNSUPPORTED, "time sharding supports d <= 4");
    if (N_local < 1 || offset < 0) return fail(ODX_EINVAL, "bad shard extent");
    const int d = P->dim;
    const ShardLayout lay(N_local, d);
    if (!workspace || workspace_bytes < lay.total) return fail(ODX_EWORKSPACE, "shard workspace");
    char* base = reinterpret_cast<char*>(align_up(reinterpret_cast<size_t>(workspace), 256));
    double* Fe = reinterpret_cast<double*>(base + lay.Fe);
    double* ce = reinterpret_cast<double*>(base + lay.ce);
    double* h = reinterpret_cast<double*>(base + lay.h);
    double* Fp = reinterpret_cast<double*>(base + lay.Fp);
    double* cp = reinterpret_cast<double*>(base + lay.cp);
    double* scal = reinterpret_cast<double*>(base + lay.scal);
    cudaStream_t st = (cudaStream_t)stream;
    ODX_CUDA(cudaMemsetAsync(scal, 0, 64, st));
    const int kind = S->kind;
    int rc = build_common_offset(P, S, kind, halo, X_local, N_local, dt, Fe, ce, h,
                                 kind == ODX_STEP_IMPLICIT_WEIGHTED ? reinterpret_cast<int64_t*>(scal)
                                                                    : nullptr,
                                 stream, offset);
    if (rc) return rc;
    if (kind != ODX_STEP_IMPLICIT_WEIGHTED) {
        const long long m1 = -1;
        ODX_CUDA(cudaMemcpyAsync(scal, &m1, 8, cudaMemcpyHostToDevice, st));
    }
    rc = scan_op(Fe, ce, N_local, d, Fp, cp, base + lay.scanws, scan_op_ws(N_local, d), st);
    if (rc) return rc;
    rc = max_abs_op(h, N_local, d, scal + 1, st);
    if (rc) return rc;
    rc = max_abs_op(ce, N_local, d, scal + 2, st);
    if (rc) return rc;
    shard_record_kernel<<<1, 32, 0, st>>>(Fp, cp, X_local, N_local, d, scal,
                                          kind == ODX_STEP_EXPLICIT_RK, record);
    ODX_CUDA(cudaGetLastError());
    count_launch(1);
    return ODX_OK;
}

int odx_shard_fixup(const odx_problem* P, const double* records, int32_t rank, int32_t nranks,
                    double* X_local, int64_t N_local, double* halo, double* step_out,
                    void* workspace, size_t workspace_bytes, void* stream) {
    if (!P || P->dim < 1 || P->dim > 4) return fail(ODX_EUNSUPPORTED, "time sharding supports d <= 4");
    if (rank < 0 || rank >= nranks || N_local < 1) return fail(ODX_EINVAL, "bad rank / extent");
    const int d = P->dim;
    const ShardLayout lay(N_local, d);
    if (!workspace || workspace_bytes < lay.total) return fail(ODX_EWORKSPACE, "shard workspace");
    char* base = reinterpret_cast<char*>(align_up(reinterpret_cast<size_t>(workspace), 256));
    double* Fp = reinterpret_cast<double*>(base + lay.Fp);
    double* cp = reinterpret_cast<double*>(base + lay.cp);
    double* dx = reinterpret_cast<double*>(base + lay.h);
    double* z = reinterpret_cast<double*>(base + lay.scal) + 3;
    cudaStream_t st = (cudaStream_t)stream;
    shard_carry_kernel<<<1, 32, 0, st>>>(records, rank, d, z, halo);
    shard_apply_kernel<<<(unsigned)((N_local + 255) / 256), 256, 0, st>>>(Fp, cp, z, N_local, d,
                                                                         X_local, dx);
    ODX_CUDA(cudaGetLastError());
    count_launch(2);
    return max_abs_op(dx, N_local, d, step_out, st);
}

}  // extern "C"
