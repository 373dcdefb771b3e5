// shard_tiled.cuh — one rank's part of a time-sharded Newton iteration on the
// tiled kernels (solve_tiled.cuh), SURVEY §8(e):
//
//   local  : K1 build (elements stored, chunk aggregates, rn/sc/first bad)
//            + K2 chunk scan -> the range aggregate -> the rank's record
//            [F_agg | c_agg | x_last | rn | sc | step_prev | bad]
//   (caller all-gathers the records, takes the decision)
//   fixup  : carry z_r = A_{r-1}(...A_0(0)) and this rank's exit state
//            A_r(z_r) with ONE non-inlined affine map, K3 apply with the carry,
//            then the last row is set from the exit state — bit-identical to
//            what rank r+1 adds to its halo — and halo += z_r.
//
// The rank's elements stay in its workspace between the two calls: one build
// per iteration, no look-back, one collective.
#pragma once

#include "solve_tiled.cuh"

namespace odx {

inline int shard_chunks() { return 2 * num_sms(); }

template <int D>
struct ShardTiledLayout {
    static constexpr int E = D * D + D;
    static constexpr int T = 512;  // THREADS (128) x ITEMS (4) for d <= 2; d >= 3 uses 256
    size_t red, stop, z, dlast, el, cagg, cpre, total;
    ShardTiledLayout(long long n, int nch) {
        size_t off = 0;
        auto at = [&](size_t bytes) { off = align_up(off, 256); size_t o = off; off += bytes; return o; };
        red = at(4 * 8);  // first: init_ws sets its bad slot
        stop = at(8);
        z = at(4 * 8);
        dlast = at(4 * 8);
        el = at((size_t)n * E * 8);
        cagg = at((size_t)nch * E * 8);
        cpre = at(((size_t)nch + 1) * E * 8);
        total = off + 256;
    }
};

template <int D>
__global__ void shard_tiled_record_kernel(const double* cpre_range, const double* X, long long n,
                                          const unsigned long long* red, int explicit_kind,
                                          double* rec) {
    const int t = threadIdx.x;
    constexpr int dd = D * D;
    if (t < dd) rec[t] = cpre_range[t];
    if (t < D) {
        rec[dd + t] = cpre_range[dd + t];
        rec[dd + D + t] = X[(n - 1) * D + t];
    }
    if (t == 0) {
        const double rn = bitsd(red[0]);
        rec[dd + 2 * D + 0] = rn;
        rec[dd + 2 * D + 1] = explicit_kind ? rn : bitsd(red[1]);
        rec[dd + 2 * D + 2] = __longlong_as_double(0x7ff8000000000000ll);  // step_prev: caller
        rec[dd + 2 * D + 3] = (red[3] == ~0ull) ? -1.0 : (double)(long long)red[3];
    }
}

template <class P, int KIND, int S>
int shard_tiled_local(const ProbParams& pp, const StepCoefs& sc, const double* halo,
                      const double* X_local, long long n, long long offset, double* record,
                      void* ws, size_t ws_bytes, cudaStream_t st) {
    constexpr int D = P::D;
    constexpr int THREADS = 128, ITEMS = (D <= 2) ? 4 : 2;
    constexpr long long T = (long long)THREADS * ITEMS;
    const int nch_max = shard_chunks();
    const ShardTiledLayout<D> lay(n, nch_max);
    if (ws == nullptr || ws_bytes < lay.total) return fail(ODX_EWORKSPACE, "shard workspace");
    char* base = reinterpret_cast<char*>(align_up(reinterpret_cast<size_t>(ws), 256));
    const long long ntiles = (n + T - 1) / T;
    const int nch = (int)(ntiles < nch_max ? ntiles : nch_max);
    TiledParams tp;
    std::memset(&tp, 0, sizeof(tp));
    tp.sp.prob = pp;
    tp.sp.sc = sc;
    tp.sp.X = const_cast<double*>(X_local);
    tp.sp.B = 1;
    tp.sp.N = n;
    tp.sp.max_iters = 1;
    tp.sp.red = reinterpret_cast<unsigned long long*>(base + lay.red);
    tp.el = reinterpret_cast<double*>(base + lay.el);
    tp.cagg = reinterpret_cast<double*>(base + lay.cagg);
    tp.cpre = reinterpret_cast<double*>(base + lay.cpre);
    tp.stop = reinterpret_cast<int*>(base + lay.stop);
    tp.halo = halo;
    tp.carry = nullptr;
    tp.offset = offset;
    tp.ntiles = ntiles;
    tp.nchunks = nch;
    tp.decide_here = 0;
    tp.kind = KIND;
    init_ws(base, lay.stop + 8, 1, st);
    tiled_build_kernel<P, KIND, S, THREADS, ITEMS><<<(unsigned)nch, THREADS, 0, st>>>(tp, 0);
    tiled_scan_kernel<D><<<1, 32, 0, st>>>(tp, 0);
    shard_tiled_record_kernel<D><<<1, 32, 0, st>>>(tp.cpre + (long long)nch * (D * D + D), X_local,
                                                   n, tp.sp.red, KIND == 0, record);
    ODX_CUDA(cudaGetLastError());
    count_launch(4);
    return ODX_OK;
}

}  // namespace odx
