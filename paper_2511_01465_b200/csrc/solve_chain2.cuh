// solve_chain2.cuh — single-pass chained Newton iteration for long trajectories
// (cfg 5: one trajectory of N = 2^26 steps, d = 2).
//
// One launch per Newton iteration reads X_it once and writes X_it+1 once
// (16*d bytes per step, SURVEY §8(d)'s algorithmic traffic): the residual,
// the step-map Jacobian (_kernels.build_explicit :299-342 / build_implicit
// :393-464), the affine scan (_kernels.scan_affine :116-233) and the update
// (add_inplace :98-103) all happen while a tile's data is on chip.
//
// Each CTA (one per SM, 8 warps, 255 registers per thread) holds independent
// GROUPS of warps (four groups of two warps for heavy builds, two groups of four
// otherwise), each with its own tile stream, its own share of the shared memory
// and its own named barrier: while one group scans, waits at its barrier, polls
// its carry or applies, the others build (each scheduler holds warps of
// different groups).  There is no control warp: all eight warps build.  With
// the warps of a CTA in lockstep (the first cut of this kernel) the FP64 pipe
// idled through every scan / barrier / apply phase: build 2.2 us of a 4.5 us
// tile period.
//
//   group, iteration i (tile t_i claimed two iterations ahead):
//     top      issue the loads of the rows of t_{i+1}, of the old rows of
//              t_{i-LAG} and of the prefix chunk of tile t_{i-LAG}-1
//     build    t_i's elements (ITEMS consecutive steps per thread, pairs
//              interleaved), parked in shared-memory slot i % SL; thread fold;
//              warp scan; warp total to shared memory
//     barrier  ONE named barrier of the group per tile
//     compose  every warp folds the totals of the warps before it into its
//              threads' exclusive prefixes; the last warp publishes the tile
//              aggregate (E .b128 chunks)
//     apply    t_{i-LAG}: incoming state = the scanner's inclusive prefix of the
//              preceding tile (published LAG tile periods of slack earlier)
//              -> dx -> X_it+1 = X_it + dx
//   scanner (CTA 0, all 8 warps, its SM to itself): as in solve_chain.cuh —
//     32-tile windows round-robin over the warps.
//
// Reference functions replaced: _kernels.build_explicit :299-342 /
// build_implicit :393-464, scan_affine :116-233, add_inplace :98-103, and
// solve()'s per-iteration decision (newton_pint.py:373-394) — as solve_chain.cuh.
#pragma once

#include "solve_chain.cuh"

namespace odx {

// Warps per group.  Two-warp groups (four per CTA) overlap best when the build
// is heavy (d = 2, RK3 / RK4 or an implicit step: cfg5 12.8 ms against 13.5 ms
// with four-warp groups); their 384-step tiles double the scanner's load, and a
// cheap build (Euler, d = 1) or the small d = 3 tiles would run at the
// scanner's rate (one hand-off per 32 tiles, ~0.19 us) — those keep four warps.
#ifndef ODX_CHAIN2_WARPS
#define ODX_CHAIN2_WARPS 8   // warps per CTA (experiment: 16 at 128 registers)
#endif
template <int D, int KIND, int S>
constexpr int chain2_group_warps() {
    if (ODX_CHAIN2_WARPS != 8) return 4;
    return (D == 2 && (KIND == 1 || S >= 3)) ? 2 : 4;
}

template <int D, int NWV>
struct Chain2Cfg {
    static constexpr int NW = NWV;      // warps per group (all compute)
    static constexpr int GT = NW * 32;  // threads per group
    static constexpr int NG = ODX_CHAIN2_WARPS / NW;   // groups per CTA
    static constexpr int NT = NG * GT;
    static constexpr int NWS = NG * NW;  // scanner warps (CTA 0)
    static constexpr int ITEMS = D <= 2 ? (ODX_CHAIN2_WARPS == 16 ? 3 : ODX_CHAIN2_WARPS == 12 ? 4 : 6)
                                        : (ODX_CHAIN2_WARPS == 16 ? 1 : ODX_CHAIN2_WARPS == 12 ? 2 : 3);  // steps per thread
    static constexpr int T = GT * ITEMS;          // steps per tile
    static constexpr int LAG = 2;                 // tile i-LAG is applied in iteration i
    static constexpr int SL = LAG + 1;            // parked tiles
    static constexpr int E = D * D + D;
    static constexpr int NP = (D <= 2 && ODX_CHAIN2_WARPS != 16) ? 2 : 1;  // explicit steps built together
    // scanner: tiles per lane — 64-tile windows for the 384-step tiles of two-warp
    // groups, i.e. one hand-off per 24576 steps either way (with 32-tile windows
    // the hand-off chain took 84% of cfg5's pass; a cheaper build would wait on it)
    static constexpr int TPL = NWV == 2 ? 2 : 1;
    static constexpr int WIN = 32 * TPL;          // scanner: tiles per window
};

template <int D, int NWV>
struct Chain2Shared {
    using C = Chain2Cfg<D, NWV>;
    double els[C::NG][C::SL][C::E][C::T];  // [group][slot][component][item*GT + thread]
    double wt[C::NG][2][C::NW][C::E];      // warp totals of the tile being built
    int wthas[C::NG][2][C::NW];
    long long tile[C::NG][4];  // claimed tile ids, by i % 4
    double zr[16][D];          // scanner: running state after window j, by j % 16
    long long ztag[16];        // = j once zr[j % 16] holds the state after window j
    double redd[3][C::NWS];
    unsigned long long redb[C::NWS];
};

// Record layout: chunk c of tile t at [t / 32][c][t % 32], so that the
// scanner's warp-wide access to one component of a 32-tile window is 512
// contiguous bytes (4 lines instead of 32 requests: its polls are bound by the
// SM's L2 request rate otherwise).
template <int C>
__device__ __forceinline__ long long rec_idx(long long t, int c) {
    return (t >> 5) * (C * 32) + c * 32 + (t & 31);
}

template <class P, int KIND, int S>
__global__ void __launch_bounds__(ODX_CHAIN2_WARPS * 32, 1)
chain2_pass_kernel(const ChainParams cp, const int it) {
    constexpr int D = P::D;
    using C = Chain2Cfg<D, chain2_group_warps<D, KIND, S>()>;
    constexpr int NW = C::NW, GT = C::GT, NWS = C::NWS, ITEMS = C::ITEMS, T = C::T, SL = C::SL;
    constexpr int LAG = C::LAG, E = C::E, TPL = C::TPL, WIN = C::WIN;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Chain2Shared<D, NW>& sm = *reinterpret_cast<Chain2Shared<D, NW>*>(smem_raw);
    const SolveParams& p = cp.sp;
    if (*(volatile int*)cp.stop) return;

    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int g = w / NW;                 // group
    const int gw = w % NW;                // warp within the group
    const int tid = threadIdx.x % GT;     // thread within the group
    const long long N = p.N;
    const long long ntiles = (N + T - 1) / T;
    const bool do_scan = it < p.max_iters;
    const double* cur = (it & 1) ? p.Xalt : p.X;
    double* nxt = (it & 1) ? p.X : p.Xalt;
    const unsigned long long tagA = 2ull * (unsigned long long)(it + 1);
    const unsigned long long tagP = tagA + 1ull;
    unsigned long long* red = p.red + 4ll * it;

    double rn = 0.0, scn = 0.0, step = 0.0;
    unsigned long long bad = ~0ull;
    const P prob(p.prob);

    if (!do_scan) {
        // the last iterate's residual only: a grid-stride build
        for (long long t = (long long)blockIdx.x * C::NG + g; t < ntiles; t += (long long)gridDim.x * C::NG) {
            const long long r0 = t * T + (long long)tid * ITEMS;
            double rw[(ITEMS + 1) * D];
            load_rows<D, ITEMS>(cur, p.x0, N, r0, rw);
#pragma unroll
            for (int q = 0; q < ITEMS; q++) {
                const long long k = r0 + q;
                if (k < N) {
                    Elem<D> e;
                    double h[D];
                    const bool sing = build_step<P, KIND, S>(prob, p.sc, &rw[q * D], &rw[(q + 1) * D],
                                                             k == 0, e, h);
                    rn = nan_drop_max(rn, row_max_abs<D>(h));
                    if (KIND == 1) scn = nan_drop_max(scn, row_max_abs<D>(e.c));
                    if (sing && (unsigned long long)k < bad) bad = (unsigned long long)k;
                }
            }
        }
    } else if (blockIdx.x == 0) {
        // ------------------------------------------------------------ scanner --
        // WIN-tile windows, window j on warp j % NW; each lane composes its TPL
        // consecutive tile aggregates, the warp scans the lane composites
        // (independent of the running state), then takes the state after
        // window j-1 from shared memory, hands the state after window j on and
        // publishes every tile's inclusive prefix — a d-vector, because
        // element 0 has F = 0 (_kernels.py:333-336).
        const Chunk* recA = cp.recA;
        Chunk* recP = cp.recP;
        if (threadIdx.x < 16) ((volatile long long*)sm.ztag)[threadIdx.x] = -1;
        __syncthreads();
        // (Measured: prefetching a warp's next window while it scans the
        // current one loses 12% — the prefetched copy is always stale, because
        // the scanner runs at the aggregate frontier, and costs a second load.)
        auto load_window = [&](long long jw, Chunk (&ch)[TPL][E]) {
            const long long tw = jw * WIN + (long long)lane * TPL;
#pragma unroll
            for (int q = 0; q < TPL; q++)
                if (tw + q < ntiles) {
#pragma unroll
                    for (int c = 0; c < E; c++) ch[q][c] = ld_chunk(&recA[rec_idx<E>(tw + q, c)]);
                }
        };
        for (long long j = w; j * WIN < ntiles; j += NWS) {
            const long long t0 = j * WIN + (long long)lane * TPL;
            Chunk ch[TPL][E];
            if (lane == 0) CHAIN_TRACE(t0, 12, chain_now());
            load_window(j, ch);
            Elem<D> e[TPL];
            int spins = 0;
            while (true) {
                bool ok = true;
#pragma unroll
                for (int q = 0; q < TPL; q++)
                    if (t0 + q < ntiles) {
#pragma unroll
                        for (int c = 0; c < E; c++) ok &= (ch[q][c].tag == tagA);
                    }
                if (__all_sync(FULL, ok)) break;
                if (++spins > 1) __nanosleep(64);
                load_window(j, ch);
            }
            if (lane == 0) CHAIN_TRACE(t0, 13, chain_now());
#pragma unroll
            for (int q = 0; q < TPL; q++) {
#pragma unroll
                for (int c = 0; c < D * D; c++) e[q].F[c] = ch[q][c].v;
#pragma unroll
                for (int c = 0; c < D; c++) e[q].c[c] = ch[q][D * D + c].v;
            }
            Elem<D> a = e[0];
            bool has = t0 < ntiles;
#pragma unroll
            for (int q = 1; q < TPL; q++)
                if (t0 + q < ntiles) compose<D>(a, e[q], a);
            warp_inclusive_scan<D>(a, has, lane);
            Elem<D> ex;
            shfl_up_elem<D>(a, ex, 1);
            const bool exhas = lane > 0;  // (lanes below a valid lane are valid)
            double z[D] = {};
            const bool zh = j > 0;
            const long long left = ntiles - j * WIN;
            const int lv = (int)((left < WIN ? left - 1 : WIN - 1) / TPL);
            // The only serial step between windows, done by ONE lane (the last
            // valid one, which holds the window's composite): wait for the
            // state after window j-1, push it through the composite, hand the
            // state after window j on.  States live in a ring indexed by window
            // (a slot is rewritten 16 windows later, after this warp has long
            // finished this window); shared memory is accessed with volatile
            // operations and no fence (a membar would also wait for the warp's
            // outstanding global stores): one thread writes the state, then
            // its tag, and the SM's shared-memory pipe performs a thread's
            // accesses in program order.
            if (lane == lv) {
                double hz[D], ho[D];
                if (zh) {
                    // tag first, state second (performed in that order): a
                    // probe that sees the tag also has the state, in one
                    // shared-memory round trip
                    while (true) {
                        const long long tg = ((volatile long long*)sm.ztag)[(j - 1) & 15];
#pragma unroll
                        for (int k = 0; k < D; k++) hz[k] = ((volatile double*)sm.zr[(j - 1) & 15])[k];
                        if (tg == j - 1) break;
                    }
                    apply<D>(a, hz, ho);
                } else {
#pragma unroll
                    for (int k = 0; k < D; k++) ho[k] = a.c[k];
                }
#pragma unroll
                for (int k = 0; k < D; k++) ((volatile double*)sm.zr[j & 15])[k] = ho[k];
                ((volatile long long*)sm.ztag)[j & 15] = j;
            }
            __syncwarp();
            if (zh) {
#pragma unroll
                for (int k = 0; k < D; k++) z[k] = ((volatile double*)sm.zr[(j - 1) & 15])[k];
            }
            if (lane == 0) CHAIN_TRACE(t0, 14, chain_now());
            // the state after this lane's last tile
            double pl[D];
            if (zh)
                apply<D>(a, z, pl);
            else
#pragma unroll
                for (int k = 0; k < D; k++) pl[k] = a.c[k];
            // every tile's inclusive prefix: the lane's last valid tile gets
            // pl (what the next lane / window continues from), the ones before
            // it run through the tile aggregates from the lane's entry state
            double s[D];
            bool sh = zh;
#pragma unroll
            for (int k = 0; k < D; k++) s[k] = z[k];
            if (exhas) {
                if (zh)
                    apply<D>(ex, z, s);
                else
#pragma unroll
                    for (int k = 0; k < D; k++) s[k] = ex.c[k];
                sh = true;
            }
#pragma unroll
            for (int q = 0; q < TPL; q++) {
                if (t0 + q < ntiles) {
                    const bool lastq = (q == TPL - 1) || !(t0 + q + 1 < ntiles);
                    double pq[D];
                    if (lastq) {
#pragma unroll
                        for (int k = 0; k < D; k++) pq[k] = pl[k];
                    } else if (sh) {
                        apply<D>(e[q], s, pq);
                    } else {
#pragma unroll
                        for (int k = 0; k < D; k++) pq[k] = e[q].c[k];
                    }
#pragma unroll
                    for (int k = 0; k < D; k++) st_chunk(&recP[rec_idx<D>(t0 + q, k)], pq[k], tagP);
                    CHAIN_TRACE(t0 + q, 3, chain_now());
                    CHAIN_TRACE(t0 + q, 7, (unsigned long long)(spins + 1));
#pragma unroll
                    for (int k = 0; k < D; k++) s[k] = pq[k];
                    sh = true;
                }
            }
        }
    } else {
        // ------------------------------------------------------------ compute --
        auto group_sync = [&]() {
            if constexpr (NW == 1) {
                __syncwarp();
            } else {
                if (g == 0) named_sync<1, GT>();
                else if (g == 1) named_sync<2, GT>();
                else if (g == 2) named_sync<3, GT>();
                else named_sync<4, GT>();
            }
        };
        auto claim_now = [&]() -> long long {
            const unsigned t = atomicAdd(p.ctr + it, 1u);
            if ((long long)t < ntiles) CHAIN_TRACE((long long)t, 0, chain_now());
            return (long long)t < ntiles ? (long long)t : -1;
        };
        unsigned pend = 0;     // in-flight claim (thread 0)
        bool pending = false;
        if (tid == 0) {
            const long long c0 = claim_now();
            const long long c1 = c0 >= 0 ? claim_now() : -1;
            sm.tile[g][0] = c0;
            sm.tile[g][1] = c1;
            if (c1 >= 0) {
                pend = atomicAdd(p.ctr + it, 1u);
                pending = true;
            }
        }
        group_sync();
        long long tq[LAG + 1];  // tq[k] = t_{i-k}
#pragma unroll
        for (int k = 1; k <= LAG; k++) tq[k] = -1;
        tq[0] = sm.tile[g][0];
        const long long ti1 = sm.tile[g][1];
        double rw[(ITEMS + 1) * D];   // rows of t_i (row before the thread's first step first)
        double rwn[(ITEMS + 1) * D];  // rows of t_{i+1}, loading
        double xo[ITEMS * D];         // old rows of t_{i-LAG}, loading
        if (tq[0] >= 0) rows_issue<D, ITEMS>(cur, p.x0, N, tq[0] * T + (long long)tid * ITEMS, lane, rw);
        // the thread's exclusive prefix within its tile, tiles t_i .. t_{i-LAG}
        Elem<D> tin[LAG + 1];
        bool tinh[LAG + 1];
        unsigned nspin = 0, nlate = 0, napp = 0;  // diagnostics (ODX_CHAIN_KNOB & 4)
#pragma unroll
        for (int k = 0; k <= LAG; k++) tinh[k] = false;
        for (int i = 0;; i++) {
            bool any = false;
#pragma unroll
            for (int k = 0; k <= LAG; k++) any |= tq[k] >= 0;
            if (!any) break;
            const long long ti = tq[0], ta = tq[LAG];  // built / applied this iteration
            if (ti >= 0 && tid == 0) CHAIN_TRACE(ti, 8, chain_now());
            const long long tn = i > 0 ? sm.tile[g][(i + 1) & 3] : ti1;  // t_{i+1}
            // ---- build t_i
            const int s = i % SL;
            const int pb = i & 1;
            tinh[0] = false;
            if (ti >= 0) {
                if (tid == 0) CHAIN_TRACE(ti, 1, chain_now());
                const long long r0 = ti * T + (long long)tid * ITEMS;
                rows_halo<D, ITEMS>(N, r0, lane, rw);
                const bool full = (ti + 1) * T <= N;  // CTA-uniform
                Elem<D> agg;
                bool has = false;
                auto take = [&](int q, const Elem<D>& e, const double* h, bool sing) {
                    const long long k = r0 + q;
                    rn = nan_drop_max(rn, row_max_abs<D>(h));
                    if (KIND == 1) scn = nan_drop_max(scn, row_max_abs<D>(e.c));
                    if (sing && (unsigned long long)k < bad) bad = (unsigned long long)k;
#pragma unroll
                    for (int c = 0; c < D * D; c++) sm.els[g][s][c][q * GT + tid] = e.F[c];
#pragma unroll
                    for (int c = 0; c < D; c++) sm.els[g][s][D * D + c][q * GT + tid] = e.c[c];
                    if (has)
                        compose<D>(agg, e, agg);
                    else {
                        agg = e;
                        has = true;
                    }
                };
                constexpr int NP = (KIND == 0) ? C::NP : 1;
                if (NP > 1 && r0 + ITEMS <= N) {
#pragma unroll
                    for (int q0 = 0; q0 < ITEMS; q0 += NP) {
                        double prev[NP][D], xk[NP][D], h[NP][D];
                        bool first[NP];
                        Elem<D> e[NP];
#pragma unroll
                        for (int n = 0; n < NP; n++) {
#pragma unroll
                            for (int j = 0; j < D; j++) {
                                prev[n][j] = rw[(q0 + n) * D + j];
                                xk[n][j] = rw[(q0 + n + 1) * D + j];
                            }
                            first[n] = (r0 + q0 + n == 0);
                        }
                        build_explicit_multi<P, S, NP>(prob, p.sc, prev, xk, first, e, h);
#pragma unroll
                        for (int n = 0; n < NP; n++) take(q0 + n, e[n], h[n], false);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < ITEMS; q++) {
                        if (r0 + q < N) {
                            Elem<D> e;
                            double h[D];
                            const bool sing = build_step<P, KIND, S>(prob, p.sc, &rw[q * D],
                                                                     &rw[(q + 1) * D], r0 + q == 0, e, h);
                            take(q, e, h, sing);
                        }
                    }
                }
                if (tid == 0) CHAIN_TRACE(ti, 9, chain_now());
                // warp scan of the thread folds: exclusive prefix per thread,
                // warp total to shared memory
                bool ih = has;
                if (full) {
                    warp_inclusive_scan_full<D>(agg, lane);
                    ih = true;
                } else {
                    if (!has) set_identity<D>(agg);
                    warp_inclusive_scan<D>(agg, ih, lane);
                }
                shfl_up_elem<D>(agg, tin[0], 1);
                tinh[0] = __shfl_up_sync(FULL, ih, 1) && lane > 0;
                if (lane == 31) {
#pragma unroll
                    for (int k = 0; k < D * D; k++) sm.wt[g][pb][gw][k] = agg.F[k];
#pragma unroll
                    for (int k = 0; k < D; k++) sm.wt[g][pb][gw][D * D + k] = agg.c[k];
                    sm.wthas[g][pb][gw] = ih ? 1 : 0;
                }
                if (tid == 0) CHAIN_TRACE(ti, 10, chain_now());
            }
            // ---- loads: rows of t_{i+1}, old rows of t_{i-LAG}.  Issued AFTER
            //      the build, so their 52 registers are free while the pairs
            //      are built (the build's schedule is register-bound); they
            //      land during the barrier, the fold and the apply
            if (tn >= 0) rows_issue<D, ITEMS>(cur, p.x0, N, tn * T + (long long)tid * ITEMS, lane, rwn);
            if (ta >= 0) {
                const long long r0 = ta * T + (long long)tid * ITEMS;
                if (D == 2 && ITEMS % 2 == 0 && r0 + ITEMS <= N) {
#pragma unroll
                    for (int q = 0; q < ITEMS / 2; q++)
                        ld256_nc(cur + r0 * 2 + 4 * q, xo[4 * q], xo[4 * q + 1], xo[4 * q + 2],
                                 xo[4 * q + 3]);
                } else if (D == 2 && r0 + ITEMS <= N) {
#pragma unroll
                    for (int q = 0; q < ITEMS; q++) ld_row2_nc(cur + (r0 + q) * 2, xo[2 * q], xo[2 * q + 1]);
                } else if (D == 1 && ITEMS % 2 == 0 && r0 + ITEMS <= N) {
#pragma unroll
                    for (int q = 0; q < ITEMS / 2; q++)
                        ld_row2_nc(cur + r0 + 2 * q, xo[2 * q], xo[2 * q + 1]);
                } else {
#pragma unroll
                    for (int q = 0; q < ITEMS; q++)
                        if (r0 + q < N)
#pragma unroll
                            for (int k = 0; k < D; k++) xo[q * D + k] = __ldg(cur + (r0 + q) * D + k);
                }
            }
            // ---- the claim issued one iteration ago is t_{i+2}; issue t_{i+3}'s
            if (tid == 0) {
                long long t2 = -1;
                if (pending) {
                    t2 = (long long)pend < ntiles ? (long long)pend : -1;
                    if (t2 >= 0) {
                        CHAIN_TRACE(t2, 0, chain_now());
                        pend = atomicAdd(p.ctr + it, 1u);
                    } else {
                        pending = false;
                    }
                }
                sm.tile[g][(i + 2) & 3] = t2;
            }
            // the carry of t_{i-LAG}, sampled as late as possible: it lands
            // while the group waits at its barrier and folds the warp totals.
            // (Every lane loads, from a clamped address, so that the chunk's
            // registers are written by the load alone: a conditional load
            // merges with a default value through moves that wait for it.
            // Measured: sampled at the top of the iteration instead, without
            // waiting, 15.3 ms per cfg5 solve against 13.9 ms.)
            Chunk pch = ld_chunk(&cp.recP[rec_idx<D>(ta > 0 ? ta - 1 : 0, lane < D ? lane : 0)]);
            group_sync();
            // ---- fold the totals of the warps before this one into the
            //      threads' exclusive prefixes; the last warp publishes the
            //      tile aggregate
            if (ti >= 0) {
                Elem<D> ex;
                bool exh = false;
#pragma unroll
                for (int v = 0; v < NW - 1; v++) {
                    if (v < gw && sm.wthas[g][pb][v]) {
                        Elem<D> ev;
#pragma unroll
                        for (int k = 0; k < D * D; k++) ev.F[k] = sm.wt[g][pb][v][k];
#pragma unroll
                        for (int k = 0; k < D; k++) ev.c[k] = sm.wt[g][pb][v][D * D + k];
                        if (exh)
                            compose<D>(ex, ev, ex);
                        else {
                            ex = ev;
                            exh = true;
                        }
                    }
                }
                if (gw == NW - 1) {
                    Elem<D> tot;
                    bool toth = sm.wthas[g][pb][NW - 1] != 0;
#pragma unroll
                    for (int k = 0; k < D * D; k++) tot.F[k] = sm.wt[g][pb][NW - 1][k];
#pragma unroll
                    for (int k = 0; k < D; k++) tot.c[k] = sm.wt[g][pb][NW - 1][D * D + k];
                    if (exh) {
                        if (toth)
                            compose<D>(ex, tot, tot);
                        else
                            tot = ex;
                    }
                    double v = 0.0;
#pragma unroll
                    for (int k = 0; k < D * D; k++)
                        if (lane == k) v = tot.F[k];
#pragma unroll
                    for (int k = 0; k < D; k++)
                        if (lane == D * D + k) v = tot.c[k];
                    if (lane < E) st_chunk(&cp.recA[rec_idx<E>(ti, lane)], v, tagA);
                    if (lane == 0) {
                        CHAIN_TRACE(ti, 2, chain_now());
                        CHAIN_TRACE(ti, 6, (unsigned long long)(blockIdx.x * C::NG + g));
                    }
                }
                if (exh) {
                    if (tinh[0])
                        compose<D>(ex, tin[0], tin[0]);
                    else {
                        tin[0] = ex;
                        tinh[0] = true;
                    }
                }
            }
            // ---- apply t_{i-LAG}: dx_k = F_k dx_{k-1} + c_k from its incoming state
            if (ta >= 0) {
                const int s3 = (i + 1) % SL;  // == (i - LAG) % SL (SL = LAG + 1)
                double z[D];
                bool zh = ta > 0;
                if (zh) {
                    int spins = 0;
                    while (true) {
                        const bool okk = (lane >= D) || pch.tag == tagP;
                        if (__all_sync(FULL, okk)) break;
                        if (++spins > 2) __nanosleep(32);
                        if (lane < D) pch = ld_chunk(&cp.recP[rec_idx<D>(ta - 1, lane)]);
                    }
                    nspin += spins;
                    nlate += spins ? 1 : 0;
                    napp++;
#pragma unroll
                    for (int k = 0; k < D; k++) z[k] = __shfl_sync(FULL, pch.v, k);
                }
                if (tid == 0) CHAIN_TRACE(ta, 4, chain_now());
                if (tinh[LAG]) {
                    if (zh)
                        apply<D>(tin[LAG], z, z);
                    else {
#pragma unroll
                        for (int k = 0; k < D; k++) z[k] = tin[LAG].c[k];
                        zh = true;
                    }
                }
                const long long r0 = ta * T + (long long)tid * ITEMS;
                double xn[ITEMS * D];
                if (zh && r0 + ITEMS <= N) {
                    // full thread with an incoming state (every thread but the
                    // trajectory's first): branch-free — all parked elements
                    // loaded first, then the dependent chain; the row maxima
                    // are reduced apart from it
                    Elem<D> e[ITEMS];
#pragma unroll
                    for (int q = 0; q < ITEMS; q++) {
#pragma unroll
                        for (int c = 0; c < D * D; c++) e[q].F[c] = sm.els[g][s3][c][q * GT + tid];
#pragma unroll
                        for (int c = 0; c < D; c++) e[q].c[c] = sm.els[g][s3][D * D + c][q * GT + tid];
                    }
                    double rm[ITEMS];
#pragma unroll
                    for (int q = 0; q < ITEMS; q++) {
                        double dx[D];
                        apply<D>(e[q], z, dx);
                        rm[q] = row_max_abs<D>(dx);
#pragma unroll
                        for (int k = 0; k < D; k++) {
                            z[k] = dx[k];
                            xn[q * D + k] = xo[q * D + k] + dx[k];
                        }
                    }
#pragma unroll
                    for (int q = 0; q < ITEMS; q++) step = nan_drop_max(step, rm[q]);
                } else
#pragma unroll
                for (int q = 0; q < ITEMS; q++) {
                    if (r0 + q < N) {
                        Elem<D> e;
#pragma unroll
                        for (int c = 0; c < D * D; c++) e.F[c] = sm.els[g][s3][c][q * GT + tid];
#pragma unroll
                        for (int c = 0; c < D; c++) e.c[c] = sm.els[g][s3][D * D + c][q * GT + tid];
                        double dx[D];
                        if (zh)
                            apply<D>(e, z, dx);
                        else
#pragma unroll
                            for (int k = 0; k < D; k++) dx[k] = e.c[k];
                        zh = true;
                        step = nan_drop_max(step, row_max_abs<D>(dx));
#pragma unroll
                        for (int k = 0; k < D; k++) {
                            z[k] = dx[k];
                            xn[q * D + k] = xo[q * D + k] + dx[k];
                        }
                    }
                }
                double* dst = nxt + r0 * D;
                if constexpr (D == 2) {
                    if (r0 + ITEMS <= N) {
#pragma unroll
                        for (int q = 0; q < ITEMS; q++)
                            *reinterpret_cast<double2*>(dst + 2 * q) = make_double2(xn[2 * q], xn[2 * q + 1]);
                    } else {
#pragma unroll
                        for (int q = 0; q < ITEMS; q++)
                            if (r0 + q < N) {
                                dst[2 * q] = xn[2 * q];
                                dst[2 * q + 1] = xn[2 * q + 1];
                            }
                    }
                } else {
                    if (D == 1 && ITEMS % 2 == 0 && r0 + ITEMS <= N) {
#pragma unroll
                        for (int q = 0; q < ITEMS / 2; q++)
                            *reinterpret_cast<double2*>(dst + 2 * q) = make_double2(xn[2 * q], xn[2 * q + 1]);
                    } else {
#pragma unroll
                        for (int q = 0; q < ITEMS; q++)
                            if (r0 + q < N)
#pragma unroll
                                for (int k = 0; k < D; k++) dst[q * D + k] = xn[q * D + k];
                    }
                }
                if (tid == 0) CHAIN_TRACE(ta, 5, chain_now());
            }
            if (ti >= 0 && tid == 0) CHAIN_TRACE(ti, 11, chain_now());
#pragma unroll
            for (int j = 0; j < (ITEMS + 1) * D; j++) rw[j] = rwn[j];
#pragma unroll
            for (int k = LAG; k > 0; k--) {
                tin[k] = tin[k - 1];
                tinh[k] = tinh[k - 1];
                tq[k] = tq[k - 1];
            }
            tq[0] = tn;
        }
        if (cp.trace && (cp.knob & 4) && it == cp.trace_it && lane == 0) {
            atomicAdd(cp.trace + 0, (unsigned long long)nspin);
            atomicAdd(cp.trace + 1, (unsigned long long)nlate);
            atomicAdd(cp.trace + 2, (unsigned long long)napp);
        }

    }

    // ---------------------------------------------- reductions + decision --
    rn = warp_max_nan_drop(rn);
    scn = warp_max_nan_drop(scn);
    step = warp_max_nan_drop(step);
    bad = warp_min_u64(bad);
    if (lane == 0) {
        sm.redd[0][w] = rn;
        sm.redd[1][w] = scn;
        sm.redd[2][w] = step;
        sm.redb[w] = bad;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    double a = 0.0, c = 0.0, s = 0.0;
    unsigned long long m = ~0ull;
    for (int q = 0; q < NWS; q++) {
        a = fmax(a, sm.redd[0][q]);
        c = fmax(c, sm.redd[1][q]);
        s = fmax(s, sm.redd[2][q]);
        m = sm.redb[q] < m ? sm.redb[q] : m;
    }
    if (a > 0.0) atomicMax(red + 0, dbits(a));
    if (c > 0.0) atomicMax(red + 1, dbits(c));
    if (s > 0.0) atomicMax(red + 2, dbits(s));
    if (m != ~0ull) atomicMin(red + 3, m);
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(cp.done + it) : "memory");
    if (old != gridDim.x - 1) return;
    // last CTA: solve()'s decision for iteration `it`
    const double rnb = bitsd(__ldcg(red + 0));
    const double scb = (KIND == 0) ? rnb : bitsd(__ldcg(red + 1));
    const unsigned long long badb = __ldcg(red + 3);
    const double sprev = *cp.step_prev;
    const Decision dd = decide(it, p, rnb, badb, sprev);
    if (dd.status != ODX_ST_SINGULAR) {
        if (p.hist) p.hist[it] = rnb;
        if (p.shist) p.shist[it] = scb;
    }
    if (dd.stop) {
        *cp.stop = 1;
        *cp.final_alt = it & 1;
        p.iters[0] = dd.iters;
        p.status[0] = dd.status;
        p.sidx[0] = dd.index;
    } else {
        *cp.step_prev = bitsd(__ldcg(red + 2));
    }
}

// Host side: workspace layout, one cooperative launch per Newton iteration (all
// enqueued up front; passes after the device-side stop return at once), and
// the finish kernel.
template <class P, int KIND, int S>
int chain_solve(SolveParams& p, void* ws, size_t ws_bytes, cudaStream_t st, bool query,
                size_t* need) {
    constexpr int D = P::D;
    using C2 = Chain2Cfg<D, chain2_group_warps<D, KIND, S>()>;
    constexpr int T = C2::T;
    constexpr int NT = C2::NT;
    const ChainLayout<D> lay(p.N, p.max_iters, T);
    if (query) {
        *need = lay.total;
        return ODX_OK;
    }
    if (!ws || ws_bytes < lay.total) return fail(ODX_EWORKSPACE, "workspace too small");
    if (reinterpret_cast<uintptr_t>(p.X) & 15) return fail(ODX_EINVAL, "X must be 16-byte aligned");
    char* base = reinterpret_cast<char*>(align_up(reinterpret_cast<size_t>(ws), 256));
    ChainParams cp;
    cp.sp = p;
    cp.sp.red = reinterpret_cast<unsigned long long*>(base + lay.red);
    cp.sp.ctr = reinterpret_cast<uint32_t*>(base + lay.ctr);
    cp.sp.Xalt = reinterpret_cast<double*>(base + lay.Xalt);
    cp.sp.ntiles = lay.ntiles;
    cp.done = reinterpret_cast<unsigned*>(base + lay.done);
    cp.stop = reinterpret_cast<int*>(base + lay.flags);
    cp.final_alt = cp.stop + 1;
    cp.step_prev = reinterpret_cast<double*>(base + lay.flags + 8);
    cp.recA = reinterpret_cast<Chunk*>(base + lay.recA);
    cp.recP = reinterpret_cast<Chunk*>(base + lay.recP);
    init_ws(base, lay.zero_end, p.max_iters + 1, st);  // red first: bad slots = ~0
    cp.trace = nullptr;
    cp.trace_it = 1;
    cp.knob = getenv("ODX_CHAIN_KNOB") ? atoi(getenv("ODX_CHAIN_KNOB")) : 0;
    static unsigned long long* tbuf = nullptr;
    static size_t tbytes = 0;
    const char* tpath = getenv("ODX_CHAIN_TRACE");
    if (tpath) {
        const size_t need = (size_t)lay.ntiles * 16 * 8;
        if (tbytes < need) {
            if (tbuf) cudaFree(tbuf);
            ODX_CUDA(cudaMalloc(&tbuf, need));
            tbytes = need;
        }
        ODX_CUDA(cudaMemsetAsync(tbuf, 0, need, st));
        cp.trace = tbuf;
    }
    const void* kern = (const void*)chain2_pass_kernel<P, KIND, S>;
    const size_t smem = sizeof(Chain2Shared<D, C2::NW>);
    int per_sm = 0;
    if (int rc = kernel_occupancy(kern, NT, smem, &per_sm)) return rc;
    if (per_sm < 1) return fail(ODX_ECUDA, "chain kernel cannot be resident");
    // every CTA co-resident (the scanner in CTA 0 must run alongside every
    // compute CTA): one CTA per SM
    long long grid = (long long)num_sms();
    if (grid > lay.ntiles + 1) grid = lay.ntiles + 1;  // CTA 0 scans
    if (grid < 2) grid = 2;
    if (getenv("ODX_VERBOSE"))
        fprintf(stderr, "chain_solve: T=%d (%d-warp groups) smem=%zu per_sm=%d grid=%lld ntiles=%lld\n",
                T, C2::NW, smem, per_sm, grid, lay.ntiles);
    for (int it = 0; it <= p.max_iters; it++) {
        int itv = it;
        void* args[] = {&cp, &itv};
        ODX_CUDA(cudaLaunchCooperativeKernel(kern, dim3((unsigned)grid), dim3(NT), args, smem, st));
    }
    chain_finish_kernel<D><<<2 * num_sms(), 256, 0, st>>>(p.X, cp.sp.Xalt, p.N, cp.final_alt);
    ODX_CUDA(cudaGetLastError());
    if (tpath) {  // diagnostics only: synchronous dump of pass 1's stamps
        const size_t need = (size_t)lay.ntiles * 16 * 8;
        unsigned long long* h = (unsigned long long*)malloc(need);
        ODX_CUDA(cudaStreamSynchronize(st));
        ODX_CUDA(cudaMemcpy(h, tbuf, need, cudaMemcpyDeviceToHost));
        if (FILE* f = fopen(tpath, "wb")) {
            fwrite(h, 1, need, f);
            fclose(f);
        }
        free(h);
    }
    count_launch(p.max_iters + 3);  // init_ws + passes + finish
    set_route("chain2_pass_kernel (single pass per iteration: x read, x_new written; independent "
              "warp groups per CTA out of phase, scanner CTA)");
    return ODX_OK;
}

}  // namespace odx
