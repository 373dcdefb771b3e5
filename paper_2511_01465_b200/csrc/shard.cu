// shard.cu — time-sharded Newton iteration (one rank per GPU).
//
// Rank r owns steps [offset, offset + N_local) of one trajectory and, per
// Newton iteration of the reference loop (newton_pint.py:366-396):
//   odx_shard_local : its elements (halo = the last state of rank r-1, x0 on
//                     rank 0) built and kept in the workspace, their aggregate
//                     and the record [F_agg | c_agg | x_last | rn | sc |
//                     step_prev | bad]  (shard_tiled.cuh: tiled K1 + K2)
//   (caller)        : all-gather of the records (NCCL), identical decision on
//                     every rank
//   odx_shard_fixup : carry z_r = A_{r-1}(...A_0(0)) from the gathered
//                     aggregates, the tiled apply with that incoming state,
//                     max|dx| -> step; the last row is set to x_last + A_r(z_r)
//                     and halo += z_r, both from the same affine map, so the
//                     halo is bit-identical to rank r-1's new last row.
//   odx_solve_sharded: the whole loop on one rank natively — local, then per
//                     iteration ncclAllGather of the records + the
//                     device-decided step, all on the caller's stream (NCCL
//                     is resolved at run time from the process's libnccl.so.2,
//                     the one torch loaded when present).
//   odx_shard_step  : fixup + the next iteration's local in one pass over the
//                     rank's steps (shard_tiled.cuh: shard_fused_kernel); the
//                     carry pass below precomputes every chunk's incoming
//                     update state with the same affine map.
#include <dlfcn.h>
#include <nccl.h>

#include <climits>
#include <cstring>

#include "common.cuh"
#include "shard_tiled.cuh"

namespace odx {

int shard_local_dispatch(const odx_problem* P, const odx_stepper* S, double dt,
                         const double* halo, const double* X_local, long long n, long long offset,
                         double* record, void* ws, size_t ws_bytes, cudaStream_t st, int fused);
int dense_supported(const odx_problem* P, const odx_stepper* S);
size_t dense_shard_workspace(long long n);
int dense_shard_fixup(const double* records, int rank, double* X_local, long long n, double* halo,
                      double* step_out, void* ws, size_t ws_bytes, cudaStream_t st,
                      bool device_decided);
int shard_dense_decide_dispatch(const odx_problem* P, const odx_stepper* S, double dt,
                                const odx_newton_cfg* C, const double* records, int rank,
                                int nranks, int it, double* halo, double* X_local, long long n,
                                long long offset, double* record, double* hist, double* shist,
                                long long* state, void* ws, size_t ws_bytes, cudaStream_t st);
inline bool dense_problem(const odx_problem* P) {
    return P && P->problem_id == ODX_PROB_ALLEN_CAHN && P->dim == 64;
}

// carry z of `rank` and its exit state dlast = A_rank(z); halo += z (rank > 0);
// the step slot of the reduction quad is reset
__global__ void shard_carry_kernel(const double* recs, int rank, int d, double* z, double* dlast,
                                   double* halo, unsigned long long* red) {
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
    const double* Fr = recs + (long long)rank * R;
    double e[4];
    affine_apply(Fr, Fr + d * d, v, d, e);
    for (int r = 0; r < d; r++) dlast[r] = e[r];
    if (halo && rank > 0)
        for (int r = 0; r < d; r++) halo[r] = halo[r] + v[r];
    red[2] = 0ull;
}

// last row := x_last + dlast (x_last from this rank's record); step -> double
__global__ void shard_finish_kernel(const double* recs, int rank, int d, const double* dlast,
                                    double* X, long long n, const unsigned long long* red,
                                    double* step_out) {
    const int t = threadIdx.x;
    const double* xl = recs + (long long)rank * ODX_SHARD_REC(d) + d * d + d;
    if (t < d) X[(n - 1) * d + t] = xl[t] + dlast[t];
    if (t == 0 && step_out) *step_out = bitsd(red[2]);
}

template <int D>
int shard_step_d(const odx_problem* P, const odx_stepper* S, const double* records, int rank,
                 int nranks, int it, const ShardDecision* dec, double* halo, double* X_local,
                 long long n, long long offset, double dt, double* record, void* ws,
                 size_t ws_bytes, cudaStream_t st) {
    constexpr int THREADS = SHARD_THREADS, ITEMS = shard_items<D>();
    constexpr long long T = (long long)THREADS * ITEMS;
    const int nch_max = shard_chunks();
    const ShardTiledLayout<D> lay(n, nch_max);
    if (!ws || ws_bytes < lay.total) return fail(ODX_EWORKSPACE, "shard workspace");
    if (reinterpret_cast<uintptr_t>(X_local) & 15) return fail(ODX_EINVAL, "X_local must be 16-byte aligned");
    char* base = reinterpret_cast<char*>(align_up(reinterpret_cast<size_t>(ws), 256));
    const long long ntiles = (n + T - 1) / T;
    const int nch = (int)(ntiles < nch_max ? ntiles : nch_max);
    ShardDecision dd;
    std::memset(&dd, 0, sizeof(dd));
    if (dec) dd = *dec;
    shard_step_carry_kernel<D><<<1, 448, 0, st>>>(
        records, rank, nranks, it, dd, dec ? 1 : 0,
        reinterpret_cast<const double*>(base + lay.cpre), nch,
        reinterpret_cast<const double*>(base + lay.bnd), halo,
        reinterpret_cast<double*>(base + lay.zc), reinterpret_cast<double*>(base + lay.prevs),
        reinterpret_cast<unsigned long long*>(base + lay.red), reinterpret_cast<int*>(base + lay.stop));
    ODX_CUDA(cudaGetLastError());
    count_launch(1);
    // the pass builds iteration it+1's elements: never applied when it+1 is
    // the last iteration of the decision's budget
    const int mode = (dec && it + 1 == dec->max_iters) ? 2 : 1;
    return shard_local_dispatch(P, S, dt, halo, X_local, n, offset, record, ws, ws_bytes, st, mode);
}

template <int D>
int shard_fixup_d(const double* records, int rank, double* X_local, long long n, double* halo,
                  double* step_out, void* ws, size_t ws_bytes, cudaStream_t st) {
    constexpr int THREADS = SHARD_THREADS, ITEMS = shard_items<D>();
    constexpr long long T = (long long)THREADS * ITEMS;
    const int nch_max = shard_chunks();
    const ShardTiledLayout<D> lay(n, nch_max);
    if (!ws || ws_bytes < lay.total) return fail(ODX_EWORKSPACE, "shard workspace");
    char* base = reinterpret_cast<char*>(align_up(reinterpret_cast<size_t>(ws), 256));
    const long long ntiles = (n + T - 1) / T;
    const int nch = (int)(ntiles < nch_max ? ntiles : nch_max);
    TiledParams tp;
    std::memset(&tp, 0, sizeof(tp));
    tp.sp.X = X_local;
    tp.sp.B = 1;
    tp.sp.N = n;
    tp.sp.max_iters = 1;
    tp.sp.red = reinterpret_cast<unsigned long long*>(base + lay.red);
    tp.el = reinterpret_cast<double*>(base + lay.el);
    tp.cagg = reinterpret_cast<double*>(base + lay.cagg);
    tp.cpre = reinterpret_cast<double*>(base + lay.cpre);
    tp.stop = reinterpret_cast<int*>(base + lay.stop);
    tp.carry = reinterpret_cast<double*>(base + lay.z);
    tp.ntiles = ntiles;
    tp.nchunks = nch;
    double* dlast = reinterpret_cast<double*>(base + lay.dlast);
    shard_carry_kernel<<<1, 32, 0, st>>>(records, rank, D, const_cast<double*>(tp.carry), dlast,
                                         halo, tp.sp.red);
    const size_t smem = sizeof(TiledApplySmem<D, THREADS, ITEMS>);
    auto k3 = tiled_apply_kernel<D, THREADS, ITEMS>;
    int occ = 0;
    if (int rc = kernel_occupancy((const void*)k3, THREADS, smem, &occ)) return rc;
    k3<<<(unsigned)nch, THREADS, smem, st>>>(tp, 0);
    shard_finish_kernel<<<1, 32, 0, st>>>(records, rank, D, dlast, X_local, n, tp.sp.red,
                                          step_out);
    ODX_CUDA(cudaGetLastError());
    count_launch(3);
    return ODX_OK;
}

template <class Fn>
int with_dim(int d, Fn&& fn) {
    switch (d) {
    case 1: return fn.template operator()<1>();
    case 2: return fn.template operator()<2>();
    case 3: return fn.template operator()<3>();
    case 4: return fn.template operator()<4>();
    default: return ODX_EUNSUPPORTED;
    }
}

}  // namespace odx

using namespace odx;

extern "C" {

size_t odx_shard_workspace_bytes(const odx_problem* P, const odx_stepper* S, int64_t N_local) {
    if (P && S && N_local >= 1 && dense_supported(P, S)) return dense_shard_workspace(N_local);
    if (!P || !S || P->dim < 1 || P->dim > 4 || N_local < 1 || dense_supported(P, S)) return 0;
    size_t total = 0;
    with_dim(P->dim, [&]<int D>() {
        total = ShardTiledLayout<D>(N_local, shard_chunks()).total;
        return 0;
    });
    return total;
}

int odx_shard_local(const odx_problem* P, const odx_stepper* S, const double* halo,
                    const double* X_local, int64_t N_local, int64_t offset, double dt,
                    double* record, void* workspace, size_t workspace_bytes, void* stream) {
    if (!P || !S || ((P->dim < 1 || P->dim > 4) && !dense_supported(P, S)))
        return fail(ODX_EUNSUPPORTED, "time sharding supports d <= 4 and the d = 64 Allen-Cahn path");
    if (N_local < 1 || offset < 0) return fail(ODX_EINVAL, "bad shard extent");
    if (!halo || !X_local || !record) return fail(ODX_EINVAL, "null device buffer");
    if (reinterpret_cast<uintptr_t>(X_local) & 15) return fail(ODX_EINVAL, "X_local must be 16-byte aligned");
    return shard_local_dispatch(P, S, dt, halo, X_local, N_local, offset, record, workspace,
                                workspace_bytes, (cudaStream_t)stream, 0);
}

int odx_shard_step(const odx_problem* P, const odx_stepper* S, const double* records, int32_t rank,
                   int32_t nranks, double* halo, double* X_local, int64_t N_local, int64_t offset,
                   double dt, double* record, void* workspace, size_t workspace_bytes,
                   void* stream) {
    if (!P || !S || P->dim < 1 || P->dim > 4 || dense_supported(P, S))
        return fail(ODX_EUNSUPPORTED, "time sharding supports d <= 4");
    if (rank < 0 || rank >= nranks || N_local < 1 || offset < 0)
        return fail(ODX_EINVAL, "bad rank / extent");
    if (!records || !halo || !X_local || !record) return fail(ODX_EINVAL, "null device buffer");
    return with_dim(P->dim, [&]<int D>() {
        return shard_step_d<D>(P, S, records, rank, nranks, 0, nullptr, halo, X_local, N_local,
                               offset, dt, record, workspace, workspace_bytes, (cudaStream_t)stream);
    });
}

int odx_shard_decide_step(const odx_problem* P, const odx_stepper* S, const odx_newton_cfg* C,
                          const double* records, int32_t rank, int32_t nranks, int32_t it,
                          double* halo, double* X_local, int64_t N_local, int64_t offset,
                          double dt, double* record, double* hist, double* scaled_hist,
                          int64_t* state, void* workspace, size_t workspace_bytes,
                          void* stream) {
    if (P && S && C && dense_supported(P, S)) {
        if (C->max_iters < 1) return fail(ODX_EINVAL, "max_iters must be >= 1");
        if (rank < 0 || rank >= nranks || N_local < 1 || offset < 0 || it < 0 || it > C->max_iters)
            return fail(ODX_EINVAL, "bad rank / extent / iteration");
        if (!records || !halo || !X_local || !record || !state)
            return fail(ODX_EINVAL, "null device buffer");
        return shard_dense_decide_dispatch(P, S, dt, C, records, rank, nranks, it, halo, X_local,
                                           N_local, offset, record, hist, scaled_hist,
                                           reinterpret_cast<long long*>(state), workspace,
                                           workspace_bytes, (cudaStream_t)stream);
    }
    if (!P || !S || P->dim < 1 || P->dim > 4 || dense_supported(P, S))
        return fail(ODX_EUNSUPPORTED, "time sharding supports d <= 4");
    if (!C || C->max_iters < 1) return fail(ODX_EINVAL, "max_iters must be >= 1");
    if (rank < 0 || rank >= nranks || N_local < 1 || offset < 0 || it < 0 || it > C->max_iters)
        return fail(ODX_EINVAL, "bad rank / extent / iteration");
    if (!records || !halo || !X_local || !record || !state)
        return fail(ODX_EINVAL, "null device buffer");
    ShardDecision dec;
    dec.max_iters = C->max_iters;
    dec.abort_nonfinite = C->abort_nonfinite;
    dec.rtol = C->residual_tol;
    dec.stol = C->step_tol;
    dec.hist = hist;
    dec.shist = scaled_hist;
    dec.state = reinterpret_cast<long long*>(state);
    return with_dim(P->dim, [&]<int D>() {
        return shard_step_d<D>(P, S, records, rank, nranks, it, &dec, halo, X_local, N_local,
                               offset, dt, record, workspace, workspace_bytes, (cudaStream_t)stream);
    });
}

int odx_shard_fixup(const odx_problem* P, const double* records, int32_t rank, int32_t nranks,
                    double* X_local, int64_t N_local, double* halo, double* step_out,
                    void* workspace, size_t workspace_bytes, void* stream) {
    if (rank < 0 || rank >= nranks || N_local < 1) return fail(ODX_EINVAL, "bad rank / extent");
    if (!records || !X_local) return fail(ODX_EINVAL, "null device buffer");
    if (dense_problem(P))
        return dense_shard_fixup(records, rank, X_local, N_local, halo, step_out, workspace,
                                 workspace_bytes, (cudaStream_t)stream, false);
    if (!P || P->dim < 1 || P->dim > 4) return fail(ODX_EUNSUPPORTED, "time sharding supports d <= 4");
    return with_dim(P->dim, [&]<int D>() {
        return shard_fixup_d<D>(records, rank, X_local, N_local, halo, step_out, workspace,
                                workspace_bytes, (cudaStream_t)stream);
    });
}


}  // extern "C"

namespace odx {
namespace {
// NCCL entry points resolved at run time: the library torch already loaded
// (so communicators made by either side are the same library's), else the
// system libnccl.so.2.
struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
};
NcclApi& nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_gather;
        return a;
    }();
    return api;
}
int nccl_fail(ncclResult_t r, const char* what) {
    const NcclApi& a = nccl_api();
    std::string m = std::string(what) + ": " + (a.error_string ? a.error_string(r) : "NCCL error");
    return fail(ODX_ECUDA, m.c_str());
}
size_t al256s(size_t v) { return (v + 255) & ~size_t(255); }
}  // namespace
}  // namespace odx

extern "C" {

int odx_nccl_available(void) { return odx::nccl_api().ok ? 1 : 0; }

int odx_nccl_unique_id(void* id) {
    using namespace odx;
    if (!id) return fail(ODX_EINVAL, "null id buffer");
    if (!nccl_api().ok) return fail(ODX_EUNSUPPORTED, "libnccl.so.2 not found");
    ncclUniqueId u;
    if (ncclResult_t r = nccl_api().get_unique_id(&u)) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
    return ODX_OK;
}

int odx_nccl_comm_init(void** comm, int32_t nranks, const void* id, int32_t rank) {
    using namespace odx;
    if (!comm || !id || nranks < 1 || rank < 0 || rank >= nranks)
        return fail(ODX_EINVAL, "bad communicator arguments");
    if (!nccl_api().ok) return fail(ODX_EUNSUPPORTED, "libnccl.so.2 not found");
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    ncclComm_t c = nullptr;
    if (ncclResult_t r = nccl_api().comm_init_rank(&c, nranks, u, rank))
        return nccl_fail(r, "ncclCommInitRank");
    *comm = c;
    return ODX_OK;
}

int odx_nccl_comm_destroy(void* comm) {
    using namespace odx;
    if (!comm) return ODX_OK;
    if (!nccl_api().ok) return fail(ODX_EUNSUPPORTED, "libnccl.so.2 not found");
    if (ncclResult_t r = nccl_api().comm_destroy(static_cast<ncclComm_t>(comm)))
        return nccl_fail(r, "ncclCommDestroy");
    return ODX_OK;
}

size_t odx_solve_sharded_workspace_bytes(const odx_problem* P, const odx_stepper* S,
                                         int64_t N_local, int32_t nranks) {
    const size_t sh = odx_shard_workspace_bytes(P, S, N_local);
    if (sh == 0 || nranks < 1) return 0;
    const int R = ODX_SHARD_REC(P->dim);
    return odx::al256s(sh) + odx::al256s((size_t)R * 8) + odx::al256s((size_t)nranks * R * 8) +
           odx::al256s((size_t)P->dim * 8) + 256;
}

int odx_solve_sharded(const odx_problem* P, const odx_stepper* S, const odx_newton_cfg* C,
                      void* comm, int32_t rank, int32_t nranks, const double* halo,
                      double* X_local, int64_t N_local, int64_t offset, double dt, double* hist,
                      double* scaled_hist, int64_t* state, int32_t poll, void* workspace,
                      size_t workspace_bytes, void* stream) {
    using namespace odx;
    const bool dense = P && S && dense_supported(P, S);
    if (!P || !S || ((P->dim < 1 || P->dim > 4) && !dense))
        return fail(ODX_EUNSUPPORTED, "time sharding supports d <= 4 and the d = 64 Allen-Cahn path");
    if (!C || C->max_iters < 1) return fail(ODX_EINVAL, "max_iters must be >= 1");
    if (!comm) return fail(ODX_EINVAL, "null NCCL communicator");
    if (rank < 0 || rank >= nranks || N_local < 1 || offset < 0)
        return fail(ODX_EINVAL, "bad rank / extent");
    if (!halo || !X_local || !state) return fail(ODX_EINVAL, "null device buffer");
    if (!nccl_api().ok) return fail(ODX_EUNSUPPORTED, "libnccl.so.2 not found");
    const size_t need = odx_solve_sharded_workspace_bytes(P, S, N_local, nranks);
    if (!workspace || workspace_bytes < need) return fail(ODX_EWORKSPACE, "sharded workspace");
    const int d = P->dim, R = ODX_SHARD_REC(d);
    const size_t sh = odx_shard_workspace_bytes(P, S, N_local);
    char* base = reinterpret_cast<char*>(align_up(reinterpret_cast<size_t>(workspace), 256));
    char* w2 = base + al256s(sh);
    double* rec = reinterpret_cast<double*>(w2);
    double* recs = reinterpret_cast<double*>(w2 + al256s((size_t)R * 8));
    double* halo_w = reinterpret_cast<double*>(w2 + al256s((size_t)R * 8) +
                                               al256s((size_t)nranks * R * 8));
    cudaStream_t st = (cudaStream_t)stream;
    ncclComm_t cm = static_cast<ncclComm_t>(comm);
    ODX_CUDA(cudaMemcpyAsync(halo_w, halo, (size_t)d * 8, cudaMemcpyDeviceToDevice, st));
    if (int rc = odx_shard_local(P, S, halo_w, X_local, N_local, offset, dt, rec, base, sh, stream))
        return rc;
    ShardDecision dec;
    dec.max_iters = C->max_iters;
    dec.abort_nonfinite = C->abort_nonfinite;
    dec.rtol = C->residual_tol;
    dec.stol = C->step_tol;
    dec.hist = hist;
    dec.shist = scaled_hist;
    dec.state = reinterpret_cast<long long*>(state);
    for (int it = 0; it <= C->max_iters; it++) {
        if (ncclResult_t r = nccl_api().all_gather(rec, recs, (size_t)R, ncclDouble, cm, st))
            return nccl_fail(r, "ncclAllGather");
        const int rc =
            dense ? shard_dense_decide_dispatch(P, S, dt, C, recs, rank, nranks, it, halo_w,
                                                X_local, N_local, offset, rec, hist, scaled_hist,
                                                reinterpret_cast<long long*>(state), base, sh, st)
                  : with_dim(d, [&]<int D>() {
                        return shard_step_d<D>(P, S, recs, rank, nranks, it, &dec, halo_w,
                                               X_local, N_local, offset, dt, rec, base, sh, st);
                    });
        if (rc) return rc;
        if (poll > 0 && it < C->max_iters && (it + 1) % poll == 0) {
            long long stopped = 0;  // identical on every rank: all leave together
            ODX_CUDA(cudaMemcpyAsync(&stopped, state, 8, cudaMemcpyDeviceToHost, st));
            ODX_CUDA(cudaStreamSynchronize(st));
            if (stopped) break;
        }
    }
    return ODX_OK;
}

}  // extern "C"
