// solve_small_launch.cuh — host launchers of the fused small-d Newton solve
// kernels (resident and persistent).  Instantiated per problem by the generated
// translation units under csrc/gen/ (see paper_2511_01465_b200/build.py).
#pragma once
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "dispatch.cuh"
#include "solve_small.cuh"
#include "solve_tiled.cuh"
#include "shard_tiled.cuh"
#include "solve_ws.cuh"
#include "solve_chain.cuh"
#include "solve_chain2.cuh"

namespace odx {

namespace {

template <class P, int KIND, int S, int THREADS, int ITEMS>
int launch_resident(SolveParams& p, cudaStream_t st) {
    using E = SmallEngine<P, KIND, S, THREADS, ITEMS>;
    auto kern = resident_solve_kernel<P, KIND, S, THREADS, ITEMS>;
    const size_t smem = sizeof(typename E::Shared);
    int per_sm = 0;
    if (int rc = kernel_occupancy((const void*)kern, THREADS, smem, &per_sm)) return rc;
    kern<<<(unsigned)p.B, THREADS, smem, st>>>(p);
    ODX_CUDA(cudaGetLastError());
    count_launch(1);
    set_route("resident_solve_kernel (one CTA per trajectory, whole solve in one launch)");
    return ODX_OK;
}

template <int D>
struct WsLayout {
    size_t total = 0, zero_off = 0, zero_bytes = 0;
    size_t Xalt, recs, ctr, red, bar;
    long long ntiles = 0;
    WsLayout(long long N, long long T, int max_iters) {
        ntiles = (N + T - 1) / T;
        size_t off = 0;
        auto at = [&](size_t bytes) { off = align_up(off, 256); size_t o = off; off += bytes; return o; };
        Xalt = at((size_t)N * D * sizeof(double));
        zero_off = align_up(off, 256);
        recs = at((size_t)ntiles * sizeof(LbRecord<D>));
        ctr = at(((size_t)max_iters + 1) * 4);
        red = at(4 * ((size_t)max_iters + 1) * 8);
        bar = at(2 * 4);
        zero_bytes = off - zero_off;
        total = off + 256;
    }
};

template <class P, int KIND, int S, int NCW, int ITEMS>
int launch_ws(SolveParams& p, void* ws, size_t ws_bytes, cudaStream_t st) {
    using W = WsEngine<P, KIND, S, NCW, ITEMS>;
    constexpr int D = P::D;
    auto kern = persistent_ws_kernel<P, KIND, S, NCW, ITEMS>;
    const WsLayout<D> lay(p.N, (long long)W::T, p.max_iters);
    if (ws == nullptr || ws_bytes < lay.total)
        return fail(ODX_EWORKSPACE, "workspace too small for persistent solve");
    char* base = reinterpret_cast<char*>(align_up(reinterpret_cast<size_t>(ws), 256));
    WsParams wp;
    wp.sp = p;
    wp.sp.Xalt = reinterpret_cast<double*>(base + lay.Xalt);
    wp.sp.ctr = reinterpret_cast<uint32_t*>(base + lay.ctr);
    wp.sp.red = reinterpret_cast<unsigned long long*>(base + lay.red);
    wp.sp.bar = reinterpret_cast<unsigned*>(base + lay.bar);
    wp.sp.ntiles = lay.ntiles;
    wp.recs = base + lay.recs;
    ODX_CUDA(cudaMemsetAsync(base + lay.zero_off, 0, lay.zero_bytes, st));
    init_bad_slots(wp.sp.red, p.max_iters + 1, st);
    const size_t smem = sizeof(typename W::Shared);
    int per_sm = 0;
    if (int rc = kernel_occupancy((const void*)kern, W::NT, smem, &per_sm)) return rc;
    if (per_sm < 1) return fail(ODX_ECUDA, "persistent kernel cannot be resident");
    long long grid = (long long)per_sm * num_sms();
    if (grid > lay.ntiles) grid = lay.ntiles;
    if (getenv("ODX_VERBOSE"))
        fprintf(stderr, "launch_ws: T=%d smem=%zu per_sm=%d grid=%lld\n", W::T, smem, per_sm, grid);
    void* args[] = {&wp};
    ODX_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)grid), dim3(W::NT), args,
                                         smem, st));
    ODX_CUDA(cudaGetLastError());
    count_launch(2);  // init_bad_slots + the persistent solve
    set_route("persistent_ws_kernel (warp-specialised streaming look-back)");
    return ODX_OK;
}

// Grid-resident solve (one tile per CTA for the whole solve).  Returns
// ODX_EUNSUPPORTED (without launching) when the trajectory does not fit one
// co-resident wave of CTAs.
template <class P, int KIND, int S, int THREADS, int ITEMS>
int launch_grid_resident(SolveParams& p, void* ws, size_t ws_bytes, cudaStream_t st, bool query,
                         size_t* need) {
    using E = SmallEngine<P, KIND, S, THREADS, ITEMS>;
    constexpr int D = P::D;
    auto kern = grid_resident_kernel<P, KIND, S, THREADS, ITEMS>;
    const long long G = (p.N + E::T - 1) / E::T;
    const size_t smem = sizeof(typename E::Shared);
    int per_sm = 0;
    if (kernel_occupancy((const void*)kern, THREADS, smem, &per_sm) != ODX_OK) {
        (void)cudaGetLastError();
        return ODX_EUNSUPPORTED;
    }
    if (G > (long long)per_sm * num_sms()) return ODX_EUNSUPPORTED;
    size_t off = 0;
    auto at = [&](size_t bytes) { off = align_up(off, 256); size_t o = off; off += bytes; return o; };
    const size_t o_red = at(4 * ((size_t)p.max_iters + 1) * 8);
    const size_t o_bar = at(8);
    const size_t o_halo = at((size_t)G * 64);  // HaloRow
    const size_t zero_end = off;
    const size_t o_aggs = at(2 * (size_t)G * (D * D + D) * 8);  // by iteration parity
    const size_t total = off + 256;
    if (query) {
        *need = total;
        return ODX_OK;
    }
    if (ws == nullptr || ws_bytes < total) return fail(ODX_EWORKSPACE, "workspace too small");
    char* base = reinterpret_cast<char*>(align_up(reinterpret_cast<size_t>(ws), 256));
    GridResParams gp;
    gp.sp = p;
    gp.sp.red = reinterpret_cast<unsigned long long*>(base + o_red);
    gp.sp.bar = reinterpret_cast<unsigned*>(base + o_bar);
    gp.halos = base + o_halo;
    gp.aggs = reinterpret_cast<double*>(base + o_aggs);
    init_ws(base, zero_end, p.max_iters + 1, st);  // o_red == 0: the quads come first
    void* args[] = {&gp};
    ODX_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3((unsigned)G), dim3(THREADS), args,
                                         smem, st));
    ODX_CUDA(cudaGetLastError());
    count_launch(2);
    set_route("grid_resident_kernel (one co-resident wave of CTAs, whole solve in one launch)");
    return ODX_OK;
}


// Tiled two-pass solve (solve_tiled.cuh) of one trajectory: 3 kernels per
// Newton iteration, every iteration enqueued up front.
template <int D>
struct TiledLayout {
    size_t total = 0, el, cagg, cpre, red, stop;
    long long ntiles;
    TiledLayout(long long N, long long T, int max_iters, int nchunks) {
        ntiles = (N + T - 1) / T;
        constexpr int E = D * D + D;
        size_t off = 0;
        auto at = [&](size_t bytes) { off = align_up(off, 256); size_t o = off; off += bytes; return o; };
        red = at(4 * ((size_t)max_iters + 1) * 8);  // first: init_ws sets its bad slots
        stop = at(8);
        el = at((size_t)N * E * 8);
        cagg = at((size_t)nchunks * E * 8);
        cpre = at(((size_t)nchunks + 1) * E * 8);
        total = off + 256;
    }
};

template <class P, int KIND, int S, int THREADS, int ITEMS>
int launch_tiled(SolveParams& p, void* ws, size_t ws_bytes, cudaStream_t st, bool query,
                 size_t* need) {
    constexpr int D = P::D;
    constexpr long long T = (long long)THREADS * ITEMS;
    auto k1 = tiled_build_kernel<P, KIND, S, THREADS, ITEMS>;
    auto k3 = tiled_apply_kernel<D, THREADS, ITEMS>;
    auto k2 = tiled_scan_kernel<D>;
    const size_t smem3 = sizeof(TiledApplySmem<D, THREADS, ITEMS>);
    int o1 = 1, o3 = 1;
    if (!query) {
        if (int rc = kernel_occupancy((const void*)k1, THREADS, 0, &o1)) return rc;
        if (int rc = kernel_occupancy((const void*)k3, THREADS, smem3, &o3)) return rc;
    }
    const long long ntiles = (p.N + T - 1) / T;
    // one chunking for K1 and K3 (a chunk per resident CTA of the slower one)
    long long nch = (long long)(o1 < o3 ? o1 : o3) * num_sms();
    if (nch > 4LL * num_sms()) nch = 4LL * num_sms();  // the workspace query's bound
    if (nch < 1) nch = 1;
    if (nch > ntiles) nch = ntiles;
    const TiledLayout<D> lay(p.N, T, p.max_iters, query ? 4 * num_sms() : (int)nch);
    if (query) {
        *need = lay.total;
        return ODX_OK;
    }
    if (ws == nullptr || ws_bytes < lay.total) return fail(ODX_EWORKSPACE, "workspace too small");
    char* base = reinterpret_cast<char*>(align_up(reinterpret_cast<size_t>(ws), 256));
    TiledParams tp;
    tp.sp = p;
    tp.sp.red = reinterpret_cast<unsigned long long*>(base + lay.red);
    tp.el = reinterpret_cast<double*>(base + lay.el);
    tp.cagg = reinterpret_cast<double*>(base + lay.cagg);
    tp.cpre = reinterpret_cast<double*>(base + lay.cpre);
    tp.stop = reinterpret_cast<int*>(base + lay.stop);
    tp.halo = p.x0;
    tp.carry = nullptr;
    tp.offset = 0;
    tp.ntiles = lay.ntiles;
    tp.nchunks = (int)nch;
    tp.decide_here = 1;
    tp.kind = KIND;
    init_ws(base, lay.stop + 8, p.max_iters + 1, st);
    int launches = 1;
    for (int it = 0; it <= p.max_iters; it++) {
        k1<<<(unsigned)nch, THREADS, 0, st>>>(tp, it);
        k2<<<1, 32, 0, st>>>(tp, it);
        launches += 2;
        if (it < p.max_iters) {
            k3<<<(unsigned)nch, THREADS, smem3, st>>>(tp, it);
            launches += 1;
        }
    }
    ODX_CUDA(cudaGetLastError());
    count_launch(launches);
    set_route("tiled_build/scan/apply_kernel (two-pass tiled)");
    return ODX_OK;
}

inline bool use_tiled() {
    static const bool on = [] {
        const char* v = std::getenv("ODX_TILED");
        return v && std::strcmp(v, "1") == 0;
    }();
    return on;
}

// long single trajectories: the fused tiled passes (shard_tiled.cuh) unless
// ODX_FUSED_TILED=0 selects the streaming warp-specialised kernel
inline bool use_fused_tiled() {
    static const bool on = [] {
        const char* v = std::getenv("ODX_FUSED_TILED");
        return !(v && std::strcmp(v, "0") == 0);
    }();
    return on;
}

// long single trajectories (d <= 3): the single-pass chained kernel
// (solve_chain.cuh) unless ODX_CHAIN=0 selects the fused tiled passes
inline bool use_chain() {
    static const bool on = [] {
        const char* v = std::getenv("ODX_CHAIN");
        return !(v && std::strcmp(v, "0") == 0);
    }();
    return on;
}

inline bool use_grid_resident() {
    static const bool on = [] {
        const char* v = std::getenv("ODX_GRID_RESIDENT");
        return !(v && std::strcmp(v, "0") == 0);
    }();
    return on;
}


// compute warps per CTA of the large-N streaming kernel: d <= 2 runs 7 warps
// x 896-step tiles at one CTA per SM (8 warps per SM leave 255 registers per
// thread; fewer, larger tiles than 4-warp CTAs mean fewer look-backs); larger
// d keeps 4 warps (its elements would not fit shared memory)
template <int D>
constexpr int ws_ncw() { return D <= 2 ? 7 : 4; }
// items per compute thread of the warp-specialised kernel, by state dim
template <int D>
constexpr int ws_items() { return D == 1 ? 8 : (D == 2 ? 4 : 2); }

}  // namespace

// Resident path when the whole trajectory fits one CTA; grid-resident when one
// trajectory fits a co-resident wave of CTAs; the streaming warp-specialised
// kernel otherwise.
template <class P, int KIND, int S>
int solve_small(SolveParams& p, void* ws, size_t ws_bytes, cudaStream_t st, bool query,
                size_t* need) {
    constexpr int D = P::D;
    constexpr int RI = (D <= 3) ? 8 : 4;   // items per thread, resident
    static_assert(256LL * RI == resident_max_steps(D), "resident limit");
    const bool resident = p.N <= 256LL * RI;
    constexpr int WI = ws_items<D>();
    const bool small_ws = p.N < 128LL * WI * 296;  // keep >= 2 tiles per SM
    // one trajectory that fits one wave of CTAs: grid-resident solve
    if (!resident && p.B == 1 && use_grid_resident()) {
        constexpr int GI = (D <= 2) ? 4 : 2;
        int rc = ODX_EUNSUPPORTED;
        // one 2-item tile per SM when that covers N; else 4-item tiles
        // (measured: more, smaller CTAs lose more to the per-iteration sync
        // than they gain in build time)
        if (p.N <= 128LL * 2 * 148)
            rc = launch_grid_resident<P, KIND, S, 128, 2>(p, ws, ws_bytes, st, query, need);
        if (rc == ODX_EUNSUPPORTED)
            rc = launch_grid_resident<P, KIND, S, 128, GI>(p, ws, ws_bytes, st, query, need);
        if (rc != ODX_EUNSUPPORTED) return rc;
    }
    if constexpr (D <= 3) {
        if (!resident && p.B == 1 && !small_ws && use_chain())
            return chain_solve<P, KIND, S>(p, ws, ws_bytes, st, query, need);
    }
    if (!resident && p.B == 1 && !small_ws && use_fused_tiled())
        return fused_tiled_solve<P, KIND, S>(p, ws, ws_bytes, st, query, need);
    if (!resident && p.B == 1 && use_tiled())  // (static smem: T*E*8 <= 48 KB)
        return launch_tiled<P, KIND, S, 128, (D <= 2 ? 4 : 2)>(p, ws, ws_bytes, st, query, need);
    if (query) {
        *need = 0;
        if (!resident) {
            const long long T = small_ws ? 128 : 32LL * ws_ncw<D>() * WI;
            *need = WsLayout<D>(p.N, T, p.max_iters).total;
        }
        return ODX_OK;
    }
    if (resident) {
        // a few trajectories cannot fill the GPU: per-iteration latency rules,
        // so spread each one over 256 threads x 4 steps (measured on cfg1:
        // 0.072 ms vs 0.093 ms for 128 x 8; 512 x 2 spills at 128 registers)
        if constexpr (D <= 3) {
            if (p.B <= 16 && p.N <= 256LL * 4) return launch_resident<P, KIND, S, 256, 4>(p, st);
        }
        if (p.N <= 128LL * RI) return launch_resident<P, KIND, S, 128, RI>(p, st);
        return launch_resident<P, KIND, S, 256, RI>(p, st);
    }
    if (p.B != 1) return fail(ODX_EUNSUPPORTED, "batched solve needs N <= resident limit");
    if (small_ws) return launch_ws<P, KIND, S, 4, 1>(p, ws, ws_bytes, st);
    return launch_ws<P, KIND, S, ws_ncw<D>(), WI>(p, ws, ws_bytes, st);
}

}  // namespace odx
