// solve_chain.cuh — single-pass chained Newton iteration for long trajectories
// (cfg 5: one trajectory of N = 2^26 steps, d = 2).
//
// One launch per Newton iteration reads X_it once and writes X_it+1 once
// (16*d bytes per step, SURVEY §8(d)'s algorithmic traffic): the residual,
// the step-map Jacobian (_kernels.build_explicit :299-342 / build_implicit
// :393-464), the affine scan (_kernels.scan_affine :116-233) and the update
// (add_inplace :98-103) all happen while a tile's data is on chip.
//
// One CTA per SM.  CTA 0 is the scanner; every other CTA has 8 compute warps
// and 1 control warp.
//
//   compute  tile t_i: build its 1024 elements (4 consecutive steps per
//            thread, pairs interleaved), park them with the old rows in one of
//            three shared-memory slots, fold per thread, warp scan; then APPLY
//            tile t_{i-2}: its incoming state (from the control warp) through
//            the warp / thread exclusive prefixes and the parked elements ->
//            dx -> X_it+1 = X_it + dx, stored.  Rows of t_{i+1} are loaded into
//            registers while t_i is built.
//   control  composes the 8 warp totals of t_i (the tile aggregate), publishes
//            it, claims tile t_{i+2}, and fetches the inclusive prefix of
//            tile t_{i-2}-1 (published by the scanner) for the compute warps.
//   scanner  (CTA 0) walks the tile aggregates IN ORDER in 32-tile windows,
//            one window per warp in flight (8 at a time): each window is
//            scanned independently, then chained through the running state,
//            and every tile's inclusive prefix is published — a d-vector,
//            because element 0 has F = 0 (_kernels.py:333-336) so every prefix
//            from the trajectory start is a pure state.
//
// A tile's carry is needed two tile-builds after its aggregate was published,
// so neither the compute warps nor the control warp normally wait on the
// scanner: there is no per-tile look-back.  Records are {value, tag} .b128
// chunks (sm100.cuh), tag = 2*(it+1) (+1 for prefixes), zeroed per solve.
//
// The pass of iteration `it` starts by checking the stop flag (passes after the
// stop return at once: all iterations are enqueued up front); the last CTA to
// finish takes solve()'s decision (newton_pint.py:373-394 + the BASELINE step
// rule, `decide`) from the pass's reductions.  Pass max_iters only builds
// (the residual of the last iterate).
#pragma once

#include "solve_small.cuh"

namespace odx {

template <int D>
struct ChainCfg {
    static constexpr int NCW = 7;                 // compute warps (+ control: 8 warps, 255 regs)
    static constexpr int NCT = NCW * 32;
    static constexpr int NT = NCT + 32;           // + control warp
    static constexpr int ITEMS = D <= 2 ? 6 : 2;  // consecutive steps per thread
    static constexpr int T = NCT * ITEMS;         // steps per tile
    static constexpr int LAG = D <= 2 ? 2 : 3;    // tile i-LAG is applied in iteration i
    static constexpr int SL = LAG + 1;            // parked tiles
    static constexpr int E = D * D + D;
    static constexpr int NP = D <= 2 ? 2 : 1;     // explicit steps built together
};

template <int D>
struct ChainShared {
    using C = ChainCfg<D>;
    double els[C::SL][C::E][C::T];   // [slot][component][item*NCT + thread]
    double wt[2][C::NCW][C::E];      // warp totals of the tile being built
    int wthas[2][C::NCW];
    double wex[C::SL][C::NCW][C::E];  // exclusive composition of warps 0..w-1
    int wexhas[C::SL][C::NCW];
    double z[2][D];   // incoming state of the tile being applied
    int zhas[2];
    long long tile[4];  // claimed tile ids, by i % 4
    double redd[3][C::NCW];
    unsigned long long redb[C::NCW];
};

struct ChainParams {
    SolveParams sp;    // X, Xalt, red, ctr (claims, per it), hist, ...
    Chunk* recA;       // [ntiles][E]
    Chunk* recP;       // [ntiles][D]
    unsigned* done;    // CTAs finished, per it
    int* stop;         // set by the deciding CTA
    int* final_alt;    // final iterate lives in Xalt
    double* step_prev; // max|dx| of the previous update (for the step rule)
    unsigned long long* trace;  // diagnostics (ODX_CHAIN_TRACE): [tile][16] stamps of one pass
    int trace_it;
    int knob;  // experiment switches (ODX_CHAIN_KNOB), 0 = product
};

__device__ __forceinline__ unsigned long long chain_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define CHAIN_TRACE(t_, k_, v_)                                           \
    do {                                                                  \
        if (cp.trace && !(cp.knob & 4) && it == cp.trace_it) cp.trace[(t_) * 16 + (k_)] = (v_); \
    } while (0)

enum : uint32_t { CB_BUILT = 1, CB_CARRY = 3, CB_CW = 5 };

// Prefetch loads: the "memory" clobber keeps the compiler from sinking them
// past the shared-memory stores of the build they are meant to overlap.
__device__ __forceinline__ void ld_row2_nc(const double* p, double& a, double& b) {
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "l"(p) : "memory");
}

__device__ __forceinline__ void ld256_nc(const double* p, double& a, double& b, double& c, double& d) {
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
                 : "l"(p)
                 : "memory");
}

// Issue the loads of rows r0-1 .. r0+ITEMS-1 (row -1 of the trajectory is x0).
// d = 2, 4 items: two 256-bit loads per thread (few scoreboard entries); the
// row before the thread's first step comes from the previous lane in
// rows_halo(), except on lane 0, which loads it.
template <int D, int ITEMS>
__device__ __forceinline__ void rows_issue(const double* X, const double* x0, long long N,
                                          long long r0, int lane, double (&rw)[(ITEMS + 1) * D]) {
    if (r0 >= N) return;
    if constexpr (D == 2 && ITEMS % 2 == 0) {
        if (r0 + ITEMS <= N) {
            const double* src = X + r0 * 2;
#pragma unroll
            for (int q = 0; q < ITEMS / 2; q++)
                ld256_nc(src + 4 * q, rw[2 + 4 * q], rw[3 + 4 * q], rw[4 + 4 * q], rw[5 + 4 * q]);
            if (lane == 0) {
                if (r0 == 0) {
                    rw[0] = x0[0];
                    rw[1] = x0[1];
                } else {
                    ld_row2_nc(src - 2, rw[0], rw[1]);
                }
            }
            return;
        }
    }
    if (r0 == 0)
#pragma unroll
        for (int j = 0; j < D; j++) rw[j] = x0[j];
    const double* src = X + (r0 - 1) * D;
#pragma unroll
    for (int q = 0; q <= ITEMS; q++)
        if ((q > 0 || r0 > 0) && r0 - 1 + q < N)
#pragma unroll
            for (int j = 0; j < D; j++) rw[q * D + j] = __ldg(src + q * D + j);
}
// completes rows_issue (all lanes of the warp call it)
template <int D, int ITEMS>
__device__ __forceinline__ void rows_halo(long long N, long long r0, int lane,
                                          double (&rw)[(ITEMS + 1) * D]) {
    if constexpr (D == 2 && ITEMS % 2 == 0) {
        const double h0 = __shfl_up_sync(FULL, rw[2 * ITEMS], 1);
        const double h1 = __shfl_up_sync(FULL, rw[2 * ITEMS + 1], 1);
        if (lane > 0 && r0 + ITEMS <= N) {
            rw[0] = h0;
            rw[1] = h1;
        }
    }
}

// Inclusive warp scan when every lane holds an element (full tiles): no
// validity bits, one predicated composition per level.
template <int D>
__device__ __forceinline__ void warp_inclusive_scan_full(Elem<D>& agg, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        Elem<D> o, t;
        shfl_up_elem<D>(agg, o, off);
        compose<D>(o, agg, t);
        if (lane >= off) agg = t;
    }
}

// rows r0-1 .. r0+ITEMS-1 of X (row -1 of the trajectory is x0)
template <int D, int ITEMS>
__device__ __forceinline__ void load_rows(const double* X, const double* x0, long long N,
                                          long long r0, double (&rw)[(ITEMS + 1) * D]) {
    if (r0 >= N) return;
    if (r0 == 0) {
#pragma unroll
        for (int j = 0; j < D; j++) rw[j] = x0[j];
    }
    const double* src = X + (r0 - 1) * D;
    if constexpr (D == 2) {
        if (r0 + ITEMS <= N) {
#pragma unroll
            for (int q = (0); q <= ITEMS; q++)
                if (q > 0 || r0 > 0) ld_row2_nc(src + 2 * q, rw[2 * q], rw[2 * q + 1]);
            return;
        }
    }
#pragma unroll
    for (int q = 0; q <= ITEMS; q++)
        if ((q > 0 || r0 > 0) && r0 - 1 + q < N)
#pragma unroll
            for (int j = 0; j < D; j++) rw[q * D + j] = __ldg(src + q * D + j);
}

template <class P, int KIND, int S>
__global__ void __launch_bounds__(ChainCfg<P::D>::NT, 1)
chain_pass_kernel(const ChainParams cp, const int it) {
    constexpr int D = P::D;
    using C = ChainCfg<D>;
    constexpr int NCW = C::NCW, NCT = C::NCT, ITEMS = C::ITEMS, T = C::T, SL = C::SL;
    constexpr int LAG = C::LAG;
    constexpr int E = C::E;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ChainShared<D>& sm = *reinterpret_cast<ChainShared<D>*>(smem_raw);
    const SolveParams& p = cp.sp;
    if (*(volatile int*)cp.stop) return;

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
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
        if (w >= NCW) return;
        for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
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
        // CTA 0 only scans.  32-tile windows, window j on warp j % NCW: each
        // warp polls its window's aggregates, scans them (independent of the
        // running state), then takes the state after window j-1 from shared
        // memory, publishes its 32 inclusive prefixes and hands the state on.
        // Only that hand-off is serial, so NCW windows are in flight at once.
        if (w >= NCW) return;
        const Chunk* recA = cp.recA;
        Chunk* recP = cp.recP;
        volatile long long* zwin = &sm.tile[0];  // last window whose state is in sm.z[0]
        if (tid == 0) *zwin = -1;
        named_sync<CB_CW, NCT>();
        for (long long j = w; j * 32 < ntiles; j += NCW) {
            const long long t = j * 32 + lane;
            Elem<D> a;
            int spins = 0;
            while (true) {
                bool ok = true;
                if (t < ntiles) {
                    Chunk ch[E];
#pragma unroll
                    for (int c = 0; c < E; c++) ch[c] = ld_chunk(&recA[t * E + c]);
#pragma unroll
                    for (int c = 0; c < E; c++) ok &= (ch[c].tag == tagA);
#pragma unroll
                    for (int c = 0; c < D * D; c++) a.F[c] = ch[c].v;
#pragma unroll
                    for (int c = 0; c < D; c++) a.c[c] = ch[D * D + c].v;
                }
                if (__all_sync(FULL, ok)) break;
                if (++spins > 1) __nanosleep(64);
            }
            const bool valid = t < ntiles;
            bool has = valid;  // (the scan sets it on every lane above a valid one)
            warp_inclusive_scan<D>(a, has, lane);
            double z[D];
            bool zh = j > 0;
            if (zh) {
                if (lane == 0)
                    while (*zwin != j - 1) { }
                __syncwarp();
                __threadfence_block();
#pragma unroll
                for (int k = 0; k < D; k++) z[k] = ((volatile double*)sm.z[0])[k];
            }
            double pz[D];
            if (zh)
                apply<D>(a, z, pz);
            else
#pragma unroll
                for (int k = 0; k < D; k++) pz[k] = a.c[k];
            const long long left = ntiles - j * 32;
            const int lv = left < 32 ? (int)left - 1 : 31;
#pragma unroll
            for (int k = 0; k < D; k++) z[k] = __shfl_sync(FULL, pz[k], lv);
            if (lane == 0) {
#pragma unroll
                for (int k = 0; k < D; k++) ((volatile double*)sm.z[0])[k] = z[k];
                __threadfence_block();
                *zwin = j;
            }
            if (valid) {
#pragma unroll
                for (int k = 0; k < D; k++) st_chunk(&recP[t * D + k], pz[k], tagP);
                CHAIN_TRACE(t, 3, chain_now());
                CHAIN_TRACE(t, 7, (unsigned long long)w);
            }
        }
    } else if (w == NCW) {
        // ------------------------------------------------------------ control --
        // Iteration i: wait for tile t_i's warp totals, compose and publish its
        // aggregate, hand the compute warps the incoming state of t_{i-2}
        // (which they apply at the start of iteration i+1) and the id of
        // t_{i+2} (whose rows they prefetch then).  The claim of t_{i+3} was
        // issued in iteration i-1 and the prefix of t_{i-2}-1 loaded then, so
        // no global round trip is waited on unless the scanner is behind.
        const Chunk* recP = cp.recP;
        auto claim = [&]() -> long long {
            unsigned t = 0;
            if (lane == 0) {
                t = atomicAdd(p.ctr + it, 1u);
                if ((long long)t < ntiles) CHAIN_TRACE((long long)t, 0, chain_now());
            }
            t = __shfl_sync(FULL, t, 0);
            return (long long)t < ntiles ? (long long)t : -1;
        };
        // tq[k] = t_{i-k}, k = 0..LAG (rotated each iteration); ti1, ti2 ahead
        long long tq[LAG + 1];
#pragma unroll
        for (int k = 1; k <= LAG; k++) tq[k] = -1;
        tq[0] = claim();
        long long ti1 = tq[0] >= 0 ? claim() : -1;
        long long ti2 = ti1 >= 0 ? claim() : -1;
        if (lane == 0) {
            sm.tile[0] = tq[0];
            sm.tile[1] = ti1;
        }
        __syncwarp();
        named_arrive<CB_CARRY, NCT + 32>();  // compute iteration 0's hand-off
        unsigned pend = 0;  // in-flight claim of t_{i+3} (lane 0)
        if (lane == 0 && ti2 >= 0) pend = atomicAdd(p.ctr + it, 1u);
        Chunk pch{0.0, 0ull};  // in-flight prefix of t_{i+1-LAG}-1 (lanes < D)
        for (int i = 0;; i++) {
            // compute runs iteration i iff one of t_i .. t_{i-LAG} exists
            bool any = false;
#pragma unroll
            for (int k = 0; k <= LAG; k++) any |= tq[k] >= 0;
            if (!any) break;
            // the prefix this iteration hands over (u-1, u = t_{i+1-LAG}):
            // loaded now, it lands while the compute warps build t_i
            {
                const long long u = tq[LAG - 1];
                if (u > 0 && lane < D) pch = ld_chunk(&recP[(u - 1) * D + lane]);
            }
            named_sync2<CB_BUILT, NCT + 32>(i & 1);
            auto handoff = [&]() {
                // does compute run iteration i+1 (t_{i+1} .. t_{i+1-LAG})?
                bool next = ti1 >= 0;
#pragma unroll
                for (int k = 0; k < LAG; k++) next |= tq[k] >= 0;
                if (next) {
                    const int nb = (i + 1) & 1;
                    // (2) incoming state of u = t_{i+1-LAG} (applied in compute
                    //     iteration i+1): the inclusive prefix of u-1
                    const long long u = tq[LAG - 1];
                    if (u >= 0) {
                        double zz = 0.0;
                        int zh = 0;
                        if (u > 0) {
                            zh = 1;
                            int spins = 0;
                            while (true) {
                                const bool okk = (lane >= D) || pch.tag == tagP;
                                if (__all_sync(FULL, okk)) break;
                                if (++spins > 2) __nanosleep(32);
                                if (lane < D) pch = ld_chunk(&recP[(u - 1) * D + lane]);
                            }
                            zz = pch.v;
                        }
                        if (lane < D) sm.z[nb][lane] = zz;
                        if (lane == 0) {
                            sm.zhas[nb] = zh;
                            CHAIN_TRACE(u, 4, chain_now());
                        }
                    }
                    // (3) t_{i+2}, whose rows compute prefetches in iteration i+1
                    if (lane == 0) sm.tile[(i + 2) & 3] = ti2;
                    __syncwarp();
                    named_arrive2<CB_CARRY, NCT + 32>(nb);
                }
            };
            auto publish = [&]() {
                // (1b) tile aggregate of t_i from the warp totals; publish it (the
                //      compute warps are already past the hand-off above)
                const long long ti = tq[0];
                if (ti >= 0) {
                    const int pb = i & 1;
                    Elem<D> a;
                    bool has = false;
                    if (lane < NCW) {
                        has = sm.wthas[pb][lane] != 0;
#pragma unroll
                        for (int k = 0; k < D * D; k++) a.F[k] = sm.wt[pb][lane][k];
#pragma unroll
                        for (int k = 0; k < D; k++) a.c[k] = sm.wt[pb][lane][D * D + k];
                    } else {
                        set_identity<D>(a);
                    }
                    warp_inclusive_scan<D>(a, has, lane);
                    Elem<D> ex;
                    shfl_up_elem<D>(a, ex, 1);
                    const bool exhas = __shfl_up_sync(FULL, has, 1) && lane > 0;
                    const int s = i % SL;
                    if (lane < NCW) {
                        sm.wexhas[s][lane] = exhas ? 1 : 0;
#pragma unroll
                        for (int k = 0; k < D * D; k++) sm.wex[s][lane][k] = ex.F[k];
#pragma unroll
                        for (int k = 0; k < D; k++) sm.wex[s][lane][D * D + k] = ex.c[k];
                    }
                    // lane NCW-1 holds the tile aggregate; lanes 0..E-1 publish it
                    double v = 0.0;
#pragma unroll
                    for (int k = 0; k < D * D; k++) {
                        const double o = __shfl_sync(FULL, a.F[k], NCW - 1);
                        if (lane == k) v = o;
                    }
#pragma unroll
                    for (int k = 0; k < D; k++) {
                        const double o = __shfl_sync(FULL, a.c[k], NCW - 1);
                        if (lane == D * D + k) v = o;
                    }
                    if (lane < E) st_chunk(&cp.recA[ti * E + lane], v, tagA);
                    if (lane == 0) {
                        CHAIN_TRACE(ti, 2, chain_now());
                        CHAIN_TRACE(ti, 6, (unsigned long long)blockIdx.x);
                    }
                }
            };
            if constexpr (LAG >= 2) {
                handoff();
                publish();
            } else {
                // LAG 1: the carry is the prefix of this tile's predecessor, so
                // this tile's aggregate must be out first (else the CTAs would
                // publish one after another, each waiting for the previous one)
                publish();
                handoff();
            }
            // (5) the claim issued last iteration is t_{i+3}; issue t_{i+4}'s
            long long ti3 = -1;
            if (ti2 >= 0) {
                const long long got = (long long)__shfl_sync(FULL, pend, 0);
                ti3 = got < ntiles ? got : -1;
                if (lane == 0 && ti3 >= 0) CHAIN_TRACE(ti3, 0, chain_now());
            }
            if (lane == 0 && ti3 >= 0) pend = atomicAdd(p.ctr + it, 1u);
#pragma unroll
            for (int k = LAG; k > 0; k--) tq[k] = tq[k - 1];
            tq[0] = ti1;
            ti1 = ti2;
            ti2 = ti3;
        }
        return;
    } else {
        // ------------------------------------------------------------ compute --
        // Iteration i: (after the hand-off barrier) issue the loads of the rows
        // of t_{i+1} and of the old rows of t_{i-LAG}, build t_i into slot
        // i % SL, then apply t_{i-LAG} with the incoming state the control
        // warp handed over in iteration i-1.  Loads are issued right after a
        // barrier and consumed before the next one (a barrier waits for the
        // thread's outstanding loads).
        named_sync2<CB_CARRY, NCT + 32>(0);
        long long tq[LAG + 1];  // tq[k] = t_{i-k}
#pragma unroll
        for (int k = 1; k <= LAG; k++) tq[k] = -1;
        tq[0] = sm.tile[0];
        const long long ti1 = sm.tile[1];
        double rw[(ITEMS + 1) * D];   // rows of t_i (row before the thread's first step first)
        double rwn[(ITEMS + 1) * D];  // rows of t_{i+1}, loading
        double xo[ITEMS * D];         // old rows of t_{i-LAG}, loading
        if (tq[0] >= 0) rows_issue<D, ITEMS>(cur, p.x0, N, tq[0] * T + (long long)tid * ITEMS, lane, rw);
        // the thread's exclusive prefix (within its warp) in tiles t_i .. t_{i-LAG}
        Elem<D> tin[LAG + 1];
        bool tinh[LAG + 1];
#pragma unroll
        for (int k = 0; k <= LAG; k++) tinh[k] = false;
        for (int i = 0;; i++) {
            bool any = false;
#pragma unroll
            for (int k = 0; k <= LAG; k++) any |= tq[k] >= 0;
            if (!any) break;
            const long long ti = tq[0], ta = tq[LAG];  // built / applied this iteration
            if (i > 0) named_sync2<CB_CARRY, NCT + 32>(i & 1);
            if (ti >= 0 && tid == 0) CHAIN_TRACE(ti, 8, chain_now());
            const long long tn = i > 0 ? sm.tile[(i + 1) & 3] : ti1;  // t_{i+1}
            // ---- loads: rows of t_{i+1}, old rows of t_{i-LAG}
            if (tn >= 0) rows_issue<D, ITEMS>(cur, p.x0, N, tn * T + (long long)tid * ITEMS, lane, rwn);
            if (ta >= 0) {
                const long long r0 = ta * T + (long long)tid * ITEMS;
                if (D == 2 && ITEMS % 2 == 0 && r0 + ITEMS <= N) {
#pragma unroll
                    for (int q = 0; q < ITEMS / 2; q++)
                        ld256_nc(cur + r0 * 2 + 4 * q, xo[4 * q], xo[4 * q + 1], xo[4 * q + 2],
                                 xo[4 * q + 3]);
                } else {
#pragma unroll
                    for (int q = 0; q < ITEMS; q++)
                        if (r0 + q < N)
#pragma unroll
                            for (int k = 0; k < D; k++) xo[q * D + k] = __ldg(cur + (r0 + q) * D + k);
                }
            }
            // ---- build t_i
            const int s = i % SL;
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
                    for (int c = 0; c < D * D; c++) sm.els[s][c][q * NCT + tid] = e.F[c];
#pragma unroll
                    for (int c = 0; c < D; c++) sm.els[s][D * D + c][q * NCT + tid] = e.c[c];
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
                // warp scan of the thread folds: exclusive prefix per thread,
                // warp total to the control warp
                if (tid == 0) CHAIN_TRACE(ti, 9, chain_now());
                if (tid == 96) CHAIN_TRACE(ti, 12, chain_now());
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
                    const int pb = i & 1;
#pragma unroll
                    for (int k = 0; k < D * D; k++) sm.wt[pb][w][k] = agg.F[k];
#pragma unroll
                    for (int k = 0; k < D; k++) sm.wt[pb][w][D * D + k] = agg.c[k];
                    sm.wthas[pb][w] = ih ? 1 : 0;
                }
                if (tid == 0) CHAIN_TRACE(ti, 10, chain_now());
            }
            // ---- apply t_{i-LAG}: dx_k = F_k dx_{k-1} + c_k from its incoming state
            if (ta >= 0) {
                const int s3 = (i + 1) % SL;  // == (i - LAG) % SL (SL = LAG + 1)
                const int pb = i & 1;
                double z[D];
                bool zh = sm.zhas[pb] != 0;
#pragma unroll
                for (int k = 0; k < D; k++) z[k] = sm.z[pb][k];
                auto through = [&](const Elem<D>& e, bool eh) {
                    if (!eh) return;
                    if (zh)
                        apply<D>(e, z, z);
                    else {
#pragma unroll
                        for (int k = 0; k < D; k++) z[k] = e.c[k];
                        zh = true;
                    }
                };
                if (sm.wexhas[s3][w]) {
                    Elem<D> e;
#pragma unroll
                    for (int k = 0; k < D * D; k++) e.F[k] = sm.wex[s3][w][k];
#pragma unroll
                    for (int k = 0; k < D; k++) e.c[k] = sm.wex[s3][w][D * D + k];
                    through(e, true);
                }
                through(tin[LAG], tinh[LAG]);
                const long long r0 = ta * T + (long long)tid * ITEMS;
                double xn[ITEMS * D];
#pragma unroll
                for (int q = 0; q < ITEMS; q++) {
                    if (r0 + q < N) {
                        Elem<D> e;
#pragma unroll
                        for (int c = 0; c < D * D; c++) e.F[c] = sm.els[s3][c][q * NCT + tid];
#pragma unroll
                        for (int c = 0; c < D; c++) e.c[c] = sm.els[s3][D * D + c][q * NCT + tid];
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
#pragma unroll
                    for (int q = 0; q < ITEMS; q++)
                        if (r0 + q < N)
#pragma unroll
                            for (int k = 0; k < D; k++) dst[q * D + k] = xn[q * D + k];
                }
                if (tid == 0) CHAIN_TRACE(ta, 5, chain_now());
            }
            if (ti >= 0 && tid == 0) CHAIN_TRACE(ti, 11, chain_now());
            if (ti >= 0 && tid == 96) CHAIN_TRACE(ti, 13, chain_now());
            named_arrive2<CB_BUILT, NCT + 32>(i & 1);
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
    }

    // ---------------------------------------------- reductions + decision --
    if (w >= NCW) return;  // (the build-only pass returned its extra warps above)
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
    named_sync<CB_CW, NCT>();
    if (tid != 0) return;
    double a = 0.0, c = 0.0, s = 0.0;
    unsigned long long m = ~0ull;
    for (int q = 0; q < NCW; q++) {
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

// the final iterate into the caller's X when it lives in the ping-pong copy
template <int D>
__global__ void chain_finish_kernel(double* X, const double* Xalt, long long n, const int* final_alt) {
    if (!*final_alt) return;
    const long long total = n * D;
    for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
         q += (long long)gridDim.x * blockDim.x)
        X[q] = __ldcg(Xalt + q);
}

template <int D>
struct ChainLayout {
    size_t red, ctr, done, flags, recA, recP, zero_end, Xalt, total;
    long long ntiles;
    ChainLayout(long long N, int max_iters, int T) {
        using C = ChainCfg<D>;
        ntiles = (N + T - 1) / T;
        size_t off = 0;
        auto at = [&](size_t bytes) { off = align_up(off, 256); size_t o = off; off += bytes; return o; };
        red = at(4 * ((size_t)max_iters + 1) * 8);  // first: init_ws sets its bad slots
        ctr = at(((size_t)max_iters + 1) * 4);
        done = at(((size_t)max_iters + 1) * 4);
        flags = at(4 * 8);  // stop, final_alt, step_prev
        const size_t nt32 = ((size_t)ntiles + 31) / 32 * 32;  // (solve_chain2.cuh: 32-tile blocks)
        recA = at(nt32 * C::E * sizeof(Chunk));
        recP = at(nt32 * D * sizeof(Chunk));
        zero_end = off;
        Xalt = at((size_t)N * D * 8);
        total = off + 256;
    }
};

}  // namespace odx
