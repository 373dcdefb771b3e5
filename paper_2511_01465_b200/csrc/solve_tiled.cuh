// solve_tiled.cuh — tiled two-pass Newton iteration for long trajectories
// (and for one rank's contiguous range of a time-sharded trajectory).
//
// Per Newton iteration of the reference loop (newton_pint.py:366-396):
//
//   K1 tiled_build   every tile (T = THREADS*ITEMS steps) in parallel: build
//                    the elements (_kernels.build_*), store them (E doubles per
//                    step), block-reduce them to the tile aggregate; residual
//                    norm / scaled norm / first singular step -> atomics
//   K2 tiled_scan    one CTA: solve()'s decision (stop flag, histories,
//                    status) and the exclusive scan of the tile aggregates
//                    -> each tile's incoming element (composition of the
//                    tiles before it); the range aggregate for sharding
//   K3 tiled_apply   every tile in parallel: incoming state = tile prefix
//                    applied to the range's incoming state, block scan of the
//                    stored elements, X += dx, max|dx| -> atomic
//
// No tile waits on another inside a kernel (no look-back): kernel boundaries
// are the only synchronisation, and every iteration is enqueued up front
// (kernels after the stop decision return at once).  Per step and iteration:
// 16*d bytes of X read by K1, E*8 written, E*8 + 16*d read and 8*d written by
// K3 — a bandwidth-for-latency trade against the single-pass streaming
// kernel (solve_ws.cuh).
#pragma once

#include "sm100.cuh"
#include "solve_small.cuh"

namespace odx {

struct TiledParams {
    SolveParams sp;       // X (in/out), N, coefficients, histories, red
    double* el;           // N x E elements
    double* cagg;         // nchunks x E chunk aggregates
    double* cpre;         // (nchunks + 1) x E exclusive chunk prefixes (+ range aggregate)
    int* stop;            // decision flag (device)
    const double* halo;   // the state before local step 0
    const double* carry;  // incoming state of the range's scan (null: zero)
    long long offset;     // global index of local step 0 (F = 0 only at global step 0)
    long long ntiles;
    int nchunks;          // = gridDim.x of K1 and K3: CTA c owns tiles [c*tpc, (c+1)*tpc)
    int decide_here;      // 1: K2 takes the decision (single-GPU solve)
    int kind;             // 1: implicit (scaled history = max|c|), 0: explicit
};

__device__ __forceinline__ void chunk_tiles(long long ntiles, int nchunks, int c, long long& t0,
                                            long long& t1) {
    const long long per = (ntiles + nchunks - 1) / nchunks;
    t0 = (long long)c * per;
    t1 = t0 + per < ntiles ? t0 + per : ntiles;
}

template <int D>
__device__ __forceinline__ void ld_elem(const double* src, Elem<D>& e) {
#pragma unroll
    for (int c = 0; c < D * D; c++) e.F[c] = src[c];
#pragma unroll
    for (int c = 0; c < D; c++) e.c[c] = src[D * D + c];
}
template <int D>
__device__ __forceinline__ void st_elem(double* dst, const Elem<D>& e) {
#pragma unroll
    for (int c = 0; c < D * D; c++) dst[c] = e.F[c];
#pragma unroll
    for (int c = 0; c < D; c++) dst[D * D + c] = e.c[c];
}

// K1: CTA c builds its contiguous chunk of tiles in order.  Elements are
// staged in shared memory and written as one contiguous block per tile
// (coalesced); the chunk aggregate is the in-order composition of the tile
// aggregates.
template <class P, int KIND, int S, int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS)
tiled_build_kernel(const TiledParams tp, int it) {
    constexpr int D = P::D, E = D * D + D, NW = THREADS / 32, T = THREADS * ITEMS;
    const SolveParams& p = tp.sp;
    if (*tp.stop) return;
    __shared__ __align__(16) double s_el[T * E];
    __shared__ double s_wt[NW][E];
    __shared__ int s_wh[NW];
    __shared__ double s_rd[2][NW];
    __shared__ unsigned long long s_rb[NW];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const P prob(p.prob);
    const long long N = p.N;
    const bool store = it < p.max_iters;
    double rn = 0.0, scn = 0.0;
    unsigned long long bad = ~0ull;
    long long t0, t1;
    chunk_tiles(tp.ntiles, tp.nchunks, blockIdx.x, t0, t1);
    Elem<D> chunk;
    bool chunk_has = false;
    for (long long t = t0; t < t1; t++) {
        const long long base = t * T;
        Elem<D> agg;
        bool has = false;
        auto take = [&](int q, long long k, const Elem<D>& e, const double* h, bool sing) {
            rn = nan_drop_max(rn, row_max_abs<D>(h));
            if (KIND == 1) scn = nan_drop_max(scn, row_max_abs<D>(e.c));
            if (sing && (unsigned long long)(tp.offset + k) < bad)
                bad = (unsigned long long)(tp.offset + k);
            if (store) {
                st_elem<D>(&s_el[(tid * ITEMS + q) * E], e);
                if (has)
                    compose<D>(agg, e, agg);
                else {
                    agg = e;
                    has = true;
                }
            }
        };
        const long long kb = base + (long long)tid * ITEMS;
        if (KIND == 0 && kb + ITEMS <= N) {
            // explicit, all items present: stage-interleaved build (ILP)
            double prev[ITEMS][D], xk[ITEMS][D], h[ITEMS][D];
            bool first[ITEMS];
            Elem<D> e[ITEMS];
#pragma unroll
            for (int j = 0; j < D; j++) prev[0][j] = (kb == 0) ? tp.halo[j] : p.X[(kb - 1) * D + j];
#pragma unroll
            for (int q = 0; q < ITEMS; q++) {
#pragma unroll
                for (int j = 0; j < D; j++) xk[q][j] = p.X[(kb + q) * D + j];
                if (q + 1 < ITEMS)
#pragma unroll
                    for (int j = 0; j < D; j++) prev[q + 1][j] = xk[q][j];
                first[q] = (tp.offset + kb + q == 0);
            }
            build_explicit_multi<P, S, ITEMS>(prob, p.sc, prev, xk, first, e, h);
#pragma unroll
            for (int q = 0; q < ITEMS; q++) take(q, kb + q, e[q], h[q], false);
        } else if (KIND == 1 && kb + ITEMS <= N) {
            // implicit, all items present: branch-free builds back to back
#pragma unroll
            for (int q = 0; q < ITEMS; q++) {
                const long long k = kb + q;
                double prev[D], xk[D], h[D];
#pragma unroll
                for (int j = 0; j < D; j++) {
                    prev[j] = (k == 0) ? tp.halo[j] : p.X[(k - 1) * D + j];
                    xk[j] = p.X[k * D + j];
                }
                Elem<D> e;
                const bool sing =
                    build_implicit_step_bf<P>(prob, p.sc, prev, xk, tp.offset + k == 0, e, h);
                take(q, k, e, h, sing);
            }
        } else {
#pragma unroll
            for (int q = 0; q < ITEMS; q++) {
                const long long k = kb + q;
                if (k < N) {
                    double prev[D], xk[D], h[D];
#pragma unroll
                    for (int j = 0; j < D; j++) {
                        prev[j] = (k == 0) ? tp.halo[j] : p.X[(k - 1) * D + j];
                        xk[j] = p.X[k * D + j];
                    }
                    Elem<D> e;
                    const bool sing =
                        build_step<P, KIND, S>(prob, p.sc, prev, xk, tp.offset + k == 0, e, h);
                    take(q, k, e, h, sing);
                }
            }
        }
        if (!store) continue;
        if (!has) set_identity<D>(agg);
        warp_reduce_earliest_first<D>(agg, has, lane);
        if (lane == 0) {
            st_elem<D>(s_wt[w], agg);
            s_wh[w] = has ? 1 : 0;
        }
        fence_proxy_async_smem();  // staged elements -> the bulk store (async proxy)
        __syncthreads();
        // the tile's elements: one bulk copy (rows*E*8 is a multiple of 16)
        const long long rows = (N - base) < T ? (N - base) : T;
        if (tid == 0) {
            tma_store_1d(tp.el + base * E, s_el, (uint32_t)(rows * E * 8));
            tma_store_commit();
            for (int q = 0; q < NW; q++) {
                if (!s_wh[q]) continue;
                Elem<D> a;
                ld_elem<D>(s_wt[q], a);
                if (chunk_has)
                    compose<D>(chunk, a, chunk);
                else {
                    chunk = a;
                    chunk_has = true;
                }
            }
            tma_store_wait_read();  // s_el is rewritten after the sync below
        }
        __syncthreads();
    }
    if (store && tid == 0) {
        tma_store_wait_all();
        if (!chunk_has) set_identity<D>(chunk);
        st_elem<D>(tp.cagg + (long long)blockIdx.x * E, chunk);
    }
    rn = warp_max_nan_drop(rn);
    scn = warp_max_nan_drop(scn);
    bad = warp_min_u64(bad);
    if (lane == 0) {
        s_rd[0][w] = rn;
        s_rd[1][w] = scn;
        s_rb[w] = bad;
    }
    __syncthreads();
    if (tid == 0) {
        double a = 0.0, c = 0.0;
        unsigned long long m = ~0ull;
        for (int q = 0; q < NW; q++) {
            a = fmax(a, s_rd[0][q]);
            c = fmax(c, s_rd[1][q]);
            m = s_rb[q] < m ? s_rb[q] : m;
        }
        unsigned long long* red = p.red + 4ll * it;
        if (a > 0.0) atomicMax(red + 0, dbits(a));
        if (c > 0.0) atomicMax(red + 1, dbits(c));
        if (m != ~0ull) atomicMin(red + 3, m);
    }
}

// K2: one warp.  Decision (single-GPU mode), then the exclusive scan of the
// nchunks chunk aggregates (lane l owns a contiguous run) -> cpre; the range
// aggregate goes to cpre[nchunks].
template <int D>
__global__ void __launch_bounds__(32) tiled_scan_kernel(const TiledParams tp, int it) {
    constexpr int E = D * D + D;
    const SolveParams& p = tp.sp;
    if (*tp.stop) return;
    const int lane = threadIdx.x;
    int stop = 0;
    if (lane == 0 && tp.decide_here) {
        const unsigned long long* red = p.red + 4ll * it;
        const double rn = bitsd(red[0]);
        const double sc = tp.kind ? bitsd(red[1]) : rn;
        const double step_prev = (it > 0) ? bitsd(red[-4 + 2]) : __longlong_as_double(0x7ff8000000000000ll);
        const Decision dd = decide(it, p, rn, red[3], step_prev);
        if (dd.status != ODX_ST_SINGULAR) {
            if (p.hist) p.hist[it] = rn;
            if (p.shist) p.shist[it] = sc;
        }
        if (dd.stop) {
            stop = 1;
            *tp.stop = 1;
            p.iters[0] = dd.iters;
            p.status[0] = dd.status;
            p.sidx[0] = dd.index;
        }
    }
    stop = __shfl_sync(FULL, stop, 0);
    if (stop || it >= p.max_iters) return;
    const int nc = tp.nchunks;
    const int per = (nc + 31) / 32;
    const int lo = lane * per, hi = (lo + per < nc) ? lo + per : nc;
    Elem<D> agg;
    bool has = false;
    for (int c = lo; c < hi; c++) {
        Elem<D> a;
        ld_elem<D>(tp.cagg + (long long)c * E, a);
        if (has)
            compose<D>(agg, a, agg);
        else {
            agg = a;
            has = true;
        }
    }
    Elem<D> inc = agg;
    bool ih = has;
    if (!ih) set_identity<D>(inc);
    warp_inclusive_scan<D>(inc, ih, lane);
    Elem<D> ex;
    shfl_up_elem<D>(inc, ex, 1);
    bool exh = __shfl_up_sync(FULL, ih, 1) && lane > 0;
    if (!exh) set_identity<D>(ex);
    for (int c = lo; c < hi; c++) {
        st_elem<D>(tp.cpre + (long long)c * E, ex);
        Elem<D> a;
        ld_elem<D>(tp.cagg + (long long)c * E, a);
        compose<D>(ex, a, ex);
    }
    if (lane == 31) st_elem<D>(tp.cpre + (long long)nc * E, inc);  // range aggregate
}

// K3: CTA c walks its chunk in order with the running state: incoming state
// of the chunk = its prefix applied to the range's incoming state.  Each
// tile's elements and old rows arrive by TMA bulk copies into a double buffer
// (the next tile streams in while this one is scanned); a block scan gives
// each thread its incoming state, X += dx.
template <int D, int THREADS, int ITEMS>
struct TiledApplySmem {
    static constexpr int E = D * D + D, T = THREADS * ITEMS;
    double el[2][T * E];
    double x[2][T * D];
    uint64_t bar[2];
};

template <int D, int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS) tiled_apply_kernel(const TiledParams tp, int it) {
    constexpr int E = D * D + D, NW = THREADS / 32, T = THREADS * ITEMS;
    using SM = TiledApplySmem<D, THREADS, ITEMS>;
    const SolveParams& p = tp.sp;
    if (*tp.stop) return;
    extern __shared__ __align__(16) unsigned char tiled_raw[];
    SM& sm = *reinterpret_cast<SM*>(tiled_raw);
    __shared__ double s_wt[NW][E];
    __shared__ int s_wh[NW];
    __shared__ double s_z[D];
    __shared__ double s_st[NW];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const long long N = p.N;
    long long t0, t1;
    chunk_tiles(tp.ntiles, tp.nchunks, blockIdx.x, t0, t1);
    // tile t -> buffer b: elements (rows*E doubles) and old rows (rows*D),
    // 16-byte multiples (E*8 and D*8 are multiples of 8; rows even except
    // possibly the last tile, whose odd tail is read directly)
    auto stage = [&](long long t, int b) {
        const long long base = t * T;
        const long long rows = (N - base) < T ? (N - base) : T;
        const uint32_t be = (uint32_t)(rows * E * 8) & ~15u, bx = (uint32_t)(rows * D * 8) & ~15u;
        mbar_arrive_expect_tx(&sm.bar[b], be + bx);
        if (be) tma_load_1d(sm.el[b], tp.el + base * E, be, &sm.bar[b]);
        if (bx) tma_load_1d(sm.x[b], p.X + base * D, bx, &sm.bar[b]);
    };
    if (tid == 0) {
        mbar_init(&sm.bar[0], 1);
        mbar_init(&sm.bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async_global();
        if (t0 < t1) stage(t0, 0);
        if (t0 + 1 < t1) stage(t0 + 1, 1);
        double zr[D];
#pragma unroll
        for (int j = 0; j < D; j++) zr[j] = tp.carry ? tp.carry[j] : 0.0;
        Elem<D> pre;
        ld_elem<D>(tp.cpre + (long long)blockIdx.x * E, pre);
        double z[D];
        apply<D>(pre, zr, z);
#pragma unroll
        for (int j = 0; j < D; j++) s_z[j] = z[j];
    }
    __syncthreads();
    uint32_t ph[2] = {0u, 0u};
    double step = 0.0;
    for (long long t = t0; t < t1; t++) {
        const int b = (int)((t - t0) & 1);
        const long long base = t * T;
        const long long rows = (N - base) < T ? (N - base) : T;
        mbar_wait(&sm.bar[b], ph[b]);
        ph[b] ^= 1u;
        Elem<D> el[ITEMS];
        double xo[ITEMS][D];
        Elem<D> agg;
        bool has = false;
        const uint32_t be = (uint32_t)(rows * E * 8) & ~15u, bx = (uint32_t)(rows * D * 8) & ~15u;
#pragma unroll
        for (int q = 0; q < ITEMS; q++) {
            const int r = tid * ITEMS + q;
            if (r < rows) {
                if ((uint32_t)(r + 1) * E * 8 <= be)
                    ld_elem<D>(&sm.el[b][r * E], el[q]);
                else
                    ld_elem<D>(tp.el + (base + r) * E, el[q]);
#pragma unroll
                for (int j = 0; j < D; j++)
                    xo[q][j] = ((uint32_t)(r * D + j + 1) * 8 <= bx) ? sm.x[b][r * D + j]
                                                                     : p.X[(base + r) * D + j];
                if (has)
                    compose<D>(agg, el[q], agg);
                else {
                    agg = el[q];
                    has = true;
                }
            }
        }
        Elem<D> inc = agg;
        bool ih = has;
        if (!ih) set_identity<D>(inc);
        warp_inclusive_scan<D>(inc, ih, lane);
        if (lane == 31) {
            st_elem<D>(s_wt[w], inc);
            s_wh[w] = ih ? 1 : 0;
        }
        __syncthreads();
        // buffer b fully read into registers: stream tile t+2 into it
        if (tid == 0 && t + 2 < t1) {
            fence_proxy_async_smem();
            stage(t + 2, b);
        }
        double z[D];
#pragma unroll
        for (int j = 0; j < D; j++) z[j] = s_z[j];
        for (int q = 0; q < w; q++) {
            if (!s_wh[q]) continue;
            Elem<D> a;
            ld_elem<D>(s_wt[q], a);
            apply<D>(a, z, z);
        }
        Elem<D> lx;
        shfl_up_elem<D>(inc, lx, 1);
        const bool lxh = __shfl_up_sync(FULL, ih, 1) && lane > 0;
        if (lxh) apply<D>(lx, z, z);
#pragma unroll
        for (int q = 0; q < ITEMS; q++) {
            const long long k = base + (long long)tid * ITEMS + q;
            if (k < N) {
                double dx[D];
                apply<D>(el[q], z, dx);
                step = nan_drop_max(step, row_max_abs<D>(dx));
#pragma unroll
                for (int j = 0; j < D; j++) {
                    z[j] = dx[j];
                    p.X[k * D + j] = xo[q][j] + dx[j];
                }
            }
        }
        __syncthreads();  // every thread has read s_z / s_wt
        if (tid == (int)((rows - 1) / ITEMS)) {  // the tile's last step: next tile's state
#pragma unroll
            for (int j = 0; j < D; j++) s_z[j] = z[j];
        }
        __syncthreads();
    }
    step = warp_max_nan_drop(step);
    if (lane == 0) s_st[w] = step;
    __syncthreads();
    if (tid == 0) {
        double s2 = 0.0;
        for (int q = 0; q < NW; q++) s2 = fmax(s2, s_st[q]);
        if (s2 > 0.0) atomicMax(p.red + 4ll * it + 2, dbits(s2));
    }
}

}  // namespace odx
