// solve_ws.cuh — warp-specialised persistent Newton solve for long trajectories.
//
// Per CTA: NCW compute warps (CW) + 1 control warp (CTL).  Tiles of
// T = NCW*32*ITEMS consecutive steps are claimed in order from a per-iteration
// counter and flow through a two-buffer pipeline:
//
//   CTL: [wait AGG_b] decoupled look-back for the tile whose aggregate CW
//        just published, publish its inclusive prefix, hand the tile's
//        incoming state to CW [arrive PREF_b] -> only then claim the tile
//        after next and TMA-copy its rows into staging buffer b (mbarrier),
//        so no tile is ever claimed by a CTA that is blocked on a look-back
//   CW:  [wait mbarrier] build the tile's elements (residual + step-map
//        Jacobian, _kernels.py:299-342 / :393-464) in registers, keep its X
//        rows in registers, fold, warp scan, park elements in smem
//        [arrive AGG_b] -> apply the PREVIOUS tile's prefix [wait PREF_b']
//        -> X + dx into an output staging buffer -> TMA bulk store
//
// so the look-back of tile i (CTL) overlaps the build of tile i+1 (CW), and
// the HBM loads of tile i+2 overlap both.  Look-back records are
// self-validating 16-byte {value, tag} chunks (sm100.cuh): one L2 round trip
// per 32-tile window, no flag/fence handshake.  One grid barrier per Newton
// iteration; every CTA takes the same on-device decision afterwards
// (newton_pint.py:373-394 + the BASELINE step rule).
#pragma once

#include "sm100.cuh"
#include "solve_small.cuh"

namespace odx {

enum : uint32_t { BAR_AGG = 1, BAR_PREF = 3, BAR_CW = 5 };

// Optional pipeline trace (build with -DODX_TRACE): per tile of Newton
// iteration ODX_TRACE_IT, 8 %globaltimer stamps:
//   0 CW build start  1 CW aggregate published  2 CTL look-back start
//   3 CTL look-back end  4 CW apply start (prefix received)  5 CW apply end
//   6 CTL claim  7 CTA id
#ifdef ODX_TRACE
__device__ unsigned long long* g_trace = nullptr;
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TRACE(it_, t_, k_, v_)                                              \
    do {                                                                    \
        if (g_trace && (it_) == 1) g_trace[(t_) * 16 + (k_)] = (v_);        \
    } while (0)
#else
#define TRACE(it_, t_, k_, v_) do { } while (0)
__device__ __forceinline__ unsigned long long gtime() { return 0; }
#endif

// A tile's look-back record: aggregate (F, c) then inclusive prefix, one
// self-validating chunk per double.  The chunk count is padded to an odd number
// so that, with an odd number of tiles per lane (LBK), the lanes' shared-memory
// reads of a staged look-back window fall on distinct banks.
template <int D, bool PAD = ((D * D + 2 * D) % 2 == 0)>
struct LbRecord {
    Chunk agg[D * D + D];
    Chunk incl[D];
    Chunk pad;
};
template <int D>
struct LbRecord<D, false> {
    Chunk agg[D * D + D];
    Chunk incl[D];
};

struct WsParams {
    SolveParams sp;
    void* recs;   // LbRecord<D>[ntiles]
};

// Wide decoupled look-back: each lane covers LBK consecutive tiles (a round
// examines 32*LBK tiles).  The round's records ({value, tag} chunks, 16 B) are
// staged into shared memory by one TMA bulk copy, then validated from smem
// (self-validating tags); a round with unpublished tiles is fetched again.
// Returns the exclusive prefix state (lane 0).
constexpr int LBK = 5;  // odd: see LbRecord
// register budget per thread: a sub-partition (SMSP) holds 16K registers, so
// 3 warps on one SMSP cap a thread at 168 and 2 warps at 255.  4 compute warps
// + control run two CTAs per SM (10 warps: 168); 7 + control run one (8
// warps: the build can keep two items' RK stages in flight without spilling)
#define WS_MAXREG(ncw) ((ncw) <= 4 ? 168 : 255)
#ifndef WS_PAIR
#define WS_PAIR 2  // explicit steps built together per thread (see build_explicit_multi)
#endif

template <int D>
__device__ __forceinline__ void lookback_wide1(long long t, unsigned long long tagA,
                                               unsigned long long tagI, const LbRecord<D>* recs,
                                               Chunk* area /* [32*LBK][E + D] per warp */,
                                               uint64_t* lbbar, uint32_t& lbph,
                                               double* z, int lane, long long* stats = nullptr) {
    constexpr int E = D * D + D;
    constexpr int RCP = (int)(sizeof(LbRecord<D>) / sizeof(Chunk));  // padded record
    constexpr int WT = 32 * LBK;  // tiles per round
    long long n_rounds = 0, n_spins = 0, t_copy = 0, t_red = 0, t_tma = 0;
    Elem<D> R;
    bool R_has = false;
    long long pos = t - 1;  // round covers tiles pos, pos-1, ..., pos-WT+1
    while (true) {
        // lane owns round-relative tiles j = lane*LBK + k (k = 0..LBK-1)
        const long long hi = pos - (long long)lane * LBK;
        const int nreal = hi < 0 ? 0 : (hi + 1 < LBK ? (int)(hi + 1) : LBK);
        unsigned valid = 0, incl = 0;  // this lane's per-tile bits
        const unsigned need = (1u << nreal) - 1u;
        int spins = 0;
        long long tc0 = (long long)gtime();
        // The round's records are contiguous: one TMA bulk copy (off the LSU
        // path the compute warps keep busy) stages them; lane l's tiles sit at
        // an odd record stride, so its reads below hit distinct banks.
        const long long nround = pos + 1 < WT ? pos + 1 : WT;
        const long long lo = pos - nround + 1;
        const Chunk* my = area + (hi - lo) * RCP;  // this lane's newest tile
        while (true) {
            if (lane == 0) {
                const uint32_t bytes = (uint32_t)(nround * sizeof(LbRecord<D>));
                fence_proxy_async_smem();  // prior generic reads of the area
                mbar_arrive_expect_tx(lbbar, bytes);
                tma_load_1d(area, &recs[lo], bytes, lbbar);
            }
            mbar_wait(lbbar, lbph);
            lbph ^= 1u;
            if (n_spins == 0 && spins == 0) t_tma += (long long)gtime() - tc0;

#pragma unroll
            for (int k = 0; k < LBK; k++) {
                if (k < nreal && !((valid >> k) & 1u)) {
                    const Chunk* a = my - k * RCP;
                    bool iv = true, av = true;
#pragma unroll
                    for (int c = 0; c < D; c++) iv &= (a[E + c].tag == tagI);
#pragma unroll
                    for (int c = 0; c < E; c++) av &= (a[c].tag == tagA);
                    if (iv) {
                        valid |= 1u << k;
                        incl |= 1u << k;
                    } else if (av) {
                        valid |= 1u << k;
                    }
                }
            }
            if (__all_sync(FULL, (valid & need) == need)) break;
            if (++spins > 16) __nanosleep(16);
        }
        n_rounds++;
        n_spins += spins;
        long long tc1 = (long long)gtime();
        t_copy += tc1 - tc0;
        // newest inclusive prefix in this lane's range, or the start sentinel
        const int kstop = incl ? (__ffs(incl) - 1) : nreal;
        Elem<D> acc;
        bool acc_has = false;
#pragma unroll
        for (int k = 0; k < LBK; k++) {
            if (k < kstop) {
                Elem<D> e;
                const Chunk* a = my - k * RCP;
#pragma unroll
                for (int c = 0; c < D * D; c++) e.F[c] = a[c].v;
#pragma unroll
                for (int c = 0; c < D; c++) e.c[c] = a[D * D + c].v;
                if (acc_has)
                    compose<D>(e, acc, acc);
                else {
                    acc = e;
                    acc_has = true;
                }
            }
        }
        const bool found = kstop < LBK;
        if (found) {
            Elem<D> e;
#pragma unroll
            for (int c = 0; c < D * D; c++) e.F[c] = 0.0;
#pragma unroll
            for (int c = 0; c < D; c++)
                e.c[c] = (kstop < nreal) ? my[E + c - kstop * RCP].v : 0.0;
            if (acc_has)
                compose<D>(e, acc, acc);
            else {
                acc = e;
                acc_has = true;
            }
        }
        __syncwarp();  // the area is refilled in the next round
        const unsigned m = __ballot_sync(FULL, found);
        const int first = m ? (__ffs(m) - 1) : 32;
        bool has = lane <= first && acc_has;
        warp_reduce_latest_first<D>(acc, has, lane);
        if (lane == 0 && has) {
            if (R_has)
                compose<D>(acc, R, R);
            else {
                R = acc;
                R_has = true;
            }
        }
        t_red += (long long)gtime() - tc1;
        if (first < 32) {
            if (stats && lane == 0) {
                stats[0] = n_rounds;
                stats[1] = t_tma;
                stats[2] = t - (pos - (long long)first * LBK);
                stats[3] = t_copy;
                stats[4] = t_red;
            }
            break;
        }
        pos -= WT;
    }
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < D; k++) z[k] = R.c[k];
    }
}

template <class P, int KIND, int S, int NCW, int ITEMS>
struct WsEngine {
    static constexpr int D = P::D;
    static constexpr int E = D * D + D;
    static constexpr int NCT = NCW * 32;
    static constexpr int NT = NCT + 32;
    static constexpr int T = NCT * ITEMS;
    static constexpr int EST = ITEMS * E + (((ITEMS * E) & 1) ? 0 : 1);  // odd stride
    static constexpr int AGS = E + ((E & 1) ? 0 : 1);

    struct Shared {
        double xr[2][T * D];  // tile rows; first member => 16-byte aligned TMA target
        double xh[2][D];      // halo: the state before the tile's first step
        double els[2][NCT * EST];
        double tin[2][NCT * AGS];
        double wt[2][NCW][E];
        int thas[2][NCT];
        int wthas[2][NCW];
        double z[2][D];
        double A[2][D * D + D];  // tile aggregate (composed and published by CW thread 0)
        double wex[2][NCW][D * D + D];  // exclusive composition of warp totals 0..w-1
        int wexhas[2][NCW];
        long long tile[2];
        uint64_t mbar[2];
        uint64_t lbbar;  // control warp: look-back bulk copies
        double redd[3][NCW];
        unsigned long long redb[NCW];
        LbRecord<D> lb_area[32 * LBK];  // control-warp look-back staging
    };
};

__device__ __forceinline__ unsigned long long lb_tag(uint32_t epoch, uint32_t kind) {
    return ((unsigned long long)epoch << 2) | kind;
}

template <class P, int KIND, int S, int NCW, int ITEMS>
__global__ void __maxnreg__(WS_MAXREG(NCW))
persistent_ws_kernel(const WsParams wp) {
    using W = WsEngine<P, KIND, S, NCW, ITEMS>;
    constexpr int D = W::D, E = W::E, NCT = W::NCT, NT = W::NT, T = W::T;
    constexpr int EST = W::EST, AGS = W::AGS;
    using Rec = LbRecord<D>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    typename W::Shared& sm = *reinterpret_cast<typename W::Shared*>(smem_raw);

    const SolveParams& p = wp.sp;
    Rec* recs = reinterpret_cast<Rec*>(wp.recs);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const bool is_ctl = (w == NCW);
    const long long N = p.N;
    const unsigned nblocks = gridDim.x;

    if (tid == 0) {
        mbar_init(&sm.mbar[0], 2);  // TMA (expect_tx) + cp.async halo arrival
        mbar_init(&sm.mbar[1], 2);
        mbar_init(&sm.lbbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    double* cur = p.X;
    double* nxt = p.Xalt;
    double step_prev = __longlong_as_double(0x7ff8000000000000ll);
    Decision dd{0, -1, -1, 0};
    uint32_t ph0 = 0, ph1 = 0;  // CW: mbarrier phase parity per buffer
    uint32_t lbph = 0;          // CTL: look-back mbarrier phase parity

    for (int it = 0; it <= p.max_iters; it++) {
        const bool do_scan = it < p.max_iters;
        const uint32_t epoch = (uint32_t)it + 1u;
        const unsigned long long tagA = lb_tag(epoch, 1), tagI = lb_tag(epoch, 2);

        if (is_ctl) {
            // ------------------------------------------------ control warp --
            fence_proxy_async_global();
            auto claim = [&]() -> long long {
                long long t = 0;
                if (lane == 0) t = (long long)atomicAdd(p.ctr + it, 1u);
                t = __shfl_sync(FULL, t, 0);
                if (lane == 0 && t < p.ntiles) {
                    TRACE(it, t, 6, gtime());
                    TRACE(it, t, 7, (unsigned long long)blockIdx.x);
                }
                return t < p.ntiles ? t : -1;
            };
            // stage tile t into slot b: rows via TMA (expect_tx), the halo row
            // via cp.async (arrives on the same mbarrier when it lands), so the
            // control warp never blocks on a global load here
            auto issue = [&](int b, long long t) {
                if (lane == 0) {
                    sm.tile[b] = t;
                    if (t >= 0) {
                        const long long base = t * T;
                        const long long rows = (N - base) < T ? (N - base) : T;
                        if (base == 0) {
                            for (int q = 0; q < D; q++) sm.xh[b][q] = p.x0[q];
                        } else {
                            for (int q = 0; q < D; q++)
                                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                                                 smem_u32(&sm.xh[b][q])),
                                             "l"(cur + (base - 1) * D + q)
                                             : "memory");
                        }
                        uint32_t bytes = (uint32_t)(rows * D * 8);
                        uint32_t tma_bytes = bytes & ~15u;
                        for (uint32_t q = tma_bytes / 8; q < bytes / 8; q++)
                            sm.xr[b][q] = __ldcg(cur + base * D + q);
                        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                                         smem_u32(&sm.mbar[b]))
                                     : "memory");
                        if (tma_bytes) {
                            mbar_arrive_expect_tx(&sm.mbar[b], tma_bytes);
                            tma_load_1d(sm.xr[b], cur + base * D, tma_bytes, &sm.mbar[b]);
                        } else {
                            mbar_arrive(&sm.mbar[b]);
                        }
                    } else {
                        mbar_arrive(&sm.mbar[b]);
                        mbar_arrive(&sm.mbar[b]);
                    }
                }
                __syncwarp();
            };
            long long mt[2];
            mt[0] = claim();
            issue(0, mt[0]);
            mt[1] = -1;
            if (mt[0] >= 0) {
                mt[1] = claim();
                issue(1, mt[1]);
            }
            for (int i = 0;; i++) {
                const int b = i & 1;
                const long long t = mt[b];
                if (t < 0) break;
                named_sync2<BAR_AGG, NT>(b);
                if (lane == 0) TRACE(it, t, 2, gtime());
                if (do_scan) {
                    // the tile aggregate was composed and published by CW thread 0
                    Elem<D> A;
#pragma unroll
                    for (int k = 0; k < D * D; k++) A.F[k] = sm.A[b][k];
#pragma unroll
                    for (int k = 0; k < D; k++) A.c[k] = sm.A[b][D * D + k];
                    double z[D];
#pragma unroll
                    for (int k = 0; k < D; k++) z[k] = 0.0;
                    long long lbs[5] = {0, 0, 0, 0, 0};
                    if (t > 0) lookback_wide1<D>(t, tagA, tagI, recs, &sm.lb_area[0].agg[0], &sm.lbbar, lbph, z, lane, lbs);
                    if (lane == 0) {
                        TRACE(it, t, 11, (unsigned long long)lbs[0]);
                        TRACE(it, t, 12, (unsigned long long)lbs[1]);
                        TRACE(it, t, 13, (unsigned long long)lbs[2]);
                        TRACE(it, t, 14, (unsigned long long)lbs[3]);
                        TRACE(it, t, 15, (unsigned long long)lbs[4]);
                    }
                    if (lane == 0) {
                        double incl[D];
                        apply<D>(A, z, incl);
#pragma unroll
                        for (int k = 0; k < D; k++) st_chunk(&recs[t].incl[k], incl[k], tagI);
#pragma unroll
                        for (int k = 0; k < D; k++) sm.z[b][k] = z[k];
                    }
                }
                __syncwarp();
                if (lane == 0) TRACE(it, t, 3, gtime());
                named_arrive2<BAR_PREF, NT>(b);
                // Claim the tile after next only now: the compute warps will
                // build it right after applying this tile, so a claimed tile
                // never waits behind a look-back (no convoys).  Its rows land
                // in staging buffer b (consumed by this tile's build) while
                // the compute warps apply this tile.
                long long tn = -1;
                if (mt[b ^ 1] >= 0) {
                    tn = claim();
                    issue(b, tn);
                }
                mt[b] = tn;
            }
        } else {
            // ------------------------------------------------ compute warps --
            double rn = 0.0, scn = 0.0, step = 0.0;
            unsigned long long bad = ~0ull;
            const P prob(p.prob);
            auto row = [&](int b, int r, int j) -> double {
                return r < 0 ? sm.xh[b][j] : sm.xr[b][r * D + j];
            };
            // apply tile (buffer c, first step `base`, its X rows in xk)
            // the old rows are re-read from L2 (read-only this iteration, loaded
            // by this CTA a few microseconds ago) rather than kept in registers
            // across the next tile's build
            auto apply_tile = [&](int c, long long base) {
                // the old rows (L2) are requested before waiting for the prefix
                double xold[ITEMS * D];
                {
                    const long long r0 = base + (long long)tid * ITEMS;
                    const double* src = cur + r0 * D;
                    if (do_scan && r0 + ITEMS <= N && ((ITEMS * D) & 1) == 0 &&
                        (reinterpret_cast<size_t>(src) & 15) == 0) {
#pragma unroll
                        for (int q = 0; q < ITEMS * D; q += 2) {
                            const double2 v = __ldcg(reinterpret_cast<const double2*>(src + q));
                            xold[q] = v.x;
                            xold[q + 1] = v.y;
                        }
                    } else if (do_scan) {
#pragma unroll
                        for (int q = 0; q < ITEMS * D; q++)
                            xold[q] = (r0 * D + q < N * D) ? __ldcg(src + q) : 0.0;
                    }
                }
                named_sync2<BAR_PREF, NT>(c);
                if (tid == 0) TRACE(it, base / T, 4, gtime());
                if (!do_scan) return;
                double z[D];
#pragma unroll
                for (int k = 0; k < D; k++) z[k] = sm.z[c][k];
                if (sm.wexhas[c][w]) {
                    Elem<D> e;
#pragma unroll
                    for (int k = 0; k < D * D; k++) e.F[k] = sm.wex[c][w][k];
#pragma unroll
                    for (int k = 0; k < D; k++) e.c[k] = sm.wex[c][w][D * D + k];
                    apply<D>(e, z, z);
                }
                if (lane > 0 && sm.thas[c][tid - 1]) {
                    Elem<D> e;
                    const double* src = &sm.tin[c][(tid - 1) * AGS];
#pragma unroll
                    for (int k = 0; k < D * D; k++) e.F[k] = src[k];
#pragma unroll
                    for (int k = 0; k < D; k++) e.c[k] = src[D * D + k];
                    apply<D>(e, z, z);
                }
                // X + dx goes straight from registers to HBM: each thread owns
                // ITEMS*D consecutive doubles (whole 32-byte sectors), so the
                // warp's stores are fully coalesced without a staging buffer
                double xn[ITEMS * D];
#pragma unroll
                for (int i = 0; i < ITEMS; i++) {
                    const int r = tid * ITEMS + i;
                    if (base + r < N) {
                        Elem<D> e;
                        const double* src = &sm.els[c][tid * EST + i * E];
#pragma unroll
                        for (int k = 0; k < D * D; k++) e.F[k] = src[k];
#pragma unroll
                        for (int k = 0; k < D; k++) e.c[k] = src[D * D + k];
                        double dx[D];
                        apply<D>(e, z, dx);
                        step = nan_drop_max(step, row_max_abs<D>(dx));
#pragma unroll
                        for (int k = 0; k < D; k++) {
                            z[k] = dx[k];
                            xn[i * D + k] = xold[i * D + k] + dx[k];
                        }
                    }
                }
                double* dst = nxt + (base + (long long)tid * ITEMS) * D;
                if (base + (long long)(tid + 1) * ITEMS <= N && ((ITEMS * D) & 1) == 0 &&
                    (reinterpret_cast<size_t>(dst) & 15) == 0) {
#pragma unroll
                    for (int q = 0; q < ITEMS * D; q += 2)
                        *reinterpret_cast<double2*>(dst + q) = make_double2(xn[q], xn[q + 1]);
                } else {
#pragma unroll
                    for (int i = 0; i < ITEMS; i++)
                        if (base + tid * ITEMS + i < N)
#pragma unroll
                            for (int k = 0; k < D; k++) dst[i * D + k] = xn[i * D + k];
                }
                if (tid == 0) TRACE(it, base / T, 5, gtime());
            };
            long long basep = 0;
            int i = 0;
            for (;; i++) {
                const int b = i & 1;
                if (b == 0) {
                    mbar_wait(&sm.mbar[0], ph0);
                    ph0 ^= 1u;
                } else {
                    mbar_wait(&sm.mbar[1], ph1);
                    ph1 ^= 1u;
                }
                const long long t = sm.tile[b];
                if (t < 0) break;
                if (tid == 0) TRACE(it, t, 0, gtime());
                const long long base = t * T;
                // each item's element goes to shared memory (for the apply) and
                // into the thread's running fold as soon as it is built, so no
                // per-item element stays live in registers
                Elem<D> agg;
                bool has = false;
                // one item's element is staged to shared memory (for the apply)
                // and folded into the thread's running aggregate as soon as it
                // is built; explicit steps are built WS_PAIR at a time, stage by
                // stage, for instruction-level parallelism
                auto take = [&](int q, long long k, const Elem<D>& e, const double* h, bool sing) {
                    rn = nan_drop_max(rn, row_max_abs<D>(h));
                    if (KIND == 1) scn = nan_drop_max(scn, row_max_abs<D>(e.c));
                    if (sing && (unsigned long long)k < bad) bad = (unsigned long long)k;
                    if (do_scan) {
                        double* dst = &sm.els[b][tid * EST + q * E];
#pragma unroll
                        for (int kk = 0; kk < D * D; kk++) dst[kk] = e.F[kk];
#pragma unroll
                        for (int kk = 0; kk < D; kk++) dst[D * D + kk] = e.c[kk];
                        if (has)
                            compose<D>(agg, e, agg);
                        else {
                            agg = e;
                            has = true;
                        }
                    }
                };
                constexpr int NP = (KIND == 0 && ITEMS % WS_PAIR == 0) ? WS_PAIR : 1;
#pragma unroll
                for (int q0 = 0; q0 < ITEMS; q0 += NP) {
                    const long long k0 = base + tid * ITEMS + q0;
                    if constexpr (NP > 1) {
                        if (k0 + NP <= N) {
                            double prev[NP][D], xk[NP][D], h[NP][D];
                            bool first[NP];
                            Elem<D> e[NP];
#pragma unroll
                            for (int n = 0; n < NP; n++) {
                                const int r = tid * ITEMS + q0 + n;
#pragma unroll
                                for (int j = 0; j < D; j++) {
                                    prev[n][j] = row(b, r - 1, j);
                                    xk[n][j] = row(b, r, j);
                                }
                                first[n] = (k0 + n == 0);
                            }
                            build_explicit_multi<P, S, NP>(prob, p.sc, prev, xk, first, e, h);
#pragma unroll
                            for (int n = 0; n < NP; n++) take(q0 + n, k0 + n, e[n], h[n], false);
                            continue;
                        }
                    }
#pragma unroll
                    for (int n = 0; n < NP; n++) {
                        const int q = q0 + n;
                        const int r = tid * ITEMS + q;
                        const long long k = base + r;
                        if (k < N) {
                            double prev[D], xk[D], h[D];
#pragma unroll
                            for (int j = 0; j < D; j++) {
                                prev[j] = row(b, r - 1, j);
                                xk[j] = row(b, r, j);
                            }
                            Elem<D> e;
                            const bool sing = build_step<P, KIND, S>(prob, p.sc, prev, xk, k == 0, e, h);
                            take(q, k, e, h, sing);
                        }
                    }
                }
                if (do_scan) {
                    if (!has) set_identity<D>(agg);
                    warp_inclusive_scan<D>(agg, has, lane);
                    double* dst = &sm.tin[b][tid * AGS];
#pragma unroll
                    for (int k = 0; k < D * D; k++) dst[k] = agg.F[k];
#pragma unroll
                    for (int k = 0; k < D; k++) dst[D * D + k] = agg.c[k];
                    sm.thas[b][tid] = has ? 1 : 0;
                    if (lane == 31) {
#pragma unroll
                        for (int k = 0; k < D * D; k++) sm.wt[b][w][k] = agg.F[k];
#pragma unroll
                        for (int k = 0; k < D; k++) sm.wt[b][w][D * D + k] = agg.c[k];
                        sm.wthas[b][w] = has ? 1 : 0;
                    }
                    // publish this tile's aggregate now, not when the control
                    // warp gets to it: look-backs must never queue behind
                    // another tile's look-back
                    named_sync<BAR_CW, NCT>();
                    if (tid == 0) {
                        Elem<D> A;
                        bool A_has = false;
                        for (int q = 0; q < NCW; q++) {
                            if (A_has) {
#pragma unroll
                                for (int k = 0; k < D * D; k++) sm.wex[b][q][k] = A.F[k];
#pragma unroll
                                for (int k = 0; k < D; k++) sm.wex[b][q][D * D + k] = A.c[k];
                            }
                            sm.wexhas[b][q] = A_has ? 1 : 0;
                            if (!sm.wthas[b][q]) continue;
                            Elem<D> e;
#pragma unroll
                            for (int k = 0; k < D * D; k++) e.F[k] = sm.wt[b][q][k];
#pragma unroll
                            for (int k = 0; k < D; k++) e.c[k] = sm.wt[b][q][D * D + k];
                            if (A_has)
                                compose<D>(A, e, A);
                            else {
                                A = e;
                                A_has = true;
                            }
                        }
                        if (!A_has) set_identity<D>(A);
#pragma unroll
                        for (int k = 0; k < D * D; k++) st_chunk(&recs[t].agg[k], A.F[k], tagA);
#pragma unroll
                        for (int k = 0; k < D; k++) st_chunk(&recs[t].agg[D * D + k], A.c[k], tagA);
                        TRACE(it, t, 1, gtime());
#pragma unroll
                        for (int k = 0; k < D * D; k++) sm.A[b][k] = A.F[k];
#pragma unroll
                        for (int k = 0; k < D; k++) sm.A[b][D * D + k] = A.c[k];
                    }
                }
                named_arrive2<BAR_AGG, NT>(b);
                if (i > 0) apply_tile(b ^ 1, basep);
                basep = base;
            }
            if (i > 0) apply_tile((i - 1) & 1, basep);
            if (tid == 0) {
                tma_store_wait_all();
                fence_proxy_async_global();
            }
            // block reduction over the compute warps -> one atomic each
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
            named_sync<BAR_CW, NCT>();
            if (tid == 0) {
                double a = 0.0, c = 0.0, s = 0.0;
                unsigned long long m = ~0ull;
                for (int q = 0; q < NCW; q++) {
                    a = fmax(a, sm.redd[0][q]);
                    c = fmax(c, sm.redd[1][q]);
                    s = fmax(s, sm.redd[2][q]);
                    m = sm.redb[q] < m ? sm.redb[q] : m;
                }
                unsigned long long* red = p.red + 4ll * it;
                if (a > 0.0) atomicMax(red + 0, dbits(a));
                if (c > 0.0) atomicMax(red + 1, dbits(c));
                if (s > 0.0) atomicMax(red + 2, dbits(s));
                if (m != ~0ull) atomicMin(red + 3, m);
            }
        }
        grid_barrier(p.bar, p.bar + 1, nblocks);
        if (tid == 0) (void)ld_acquire_gpu_u32(p.bar + 1);
        __syncthreads();
        const unsigned long long* red = p.red + 4ll * it;
        const double rnb = bitsd(__ldcg(red + 0));
        const double scb = (KIND == 0) ? rnb : bitsd(__ldcg(red + 1));
        const unsigned long long badb = __ldcg(red + 3);
        dd = decide(it, p, rnb, badb, step_prev);
        if (blockIdx.x == 0 && tid == 0 && dd.status != ODX_ST_SINGULAR) {
            if (p.hist) p.hist[it] = rnb;
            if (p.shist) p.shist[it] = scb;
        }
        if (dd.stop) break;
        step_prev = bitsd(__ldcg(red + 2));
        double* t2 = cur;
        cur = nxt;
        nxt = t2;
    }
    if (cur != p.X) {
        const long long total = N * D;
        for (long long q = (long long)blockIdx.x * NT + tid; q < total; q += (long long)nblocks * NT)
            p.X[q] = __ldcg(cur + q);
    }
    if (blockIdx.x == 0 && tid == 0) {
        p.iters[0] = dd.iters;
        p.status[0] = dd.status;
        p.sidx[0] = dd.index;
    }
}

}  // namespace odx
