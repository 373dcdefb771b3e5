// solve_small.cuh — fused Newton-iteration kernels for small state dims (d <= 4).
//
// One Newton iteration of the reference (newton_pint.py:366-396) is
//   build (_kernels.build_*) -> max_abs(h) -> scan_affine -> add_inplace,
// four passes over HBM plus the scan's temporaries.  Here one pass does all
// of it: the tile of X is staged in shared memory, every thread builds the
// elements of ITEMS consecutive steps in registers, the block scans them, the
// tile chains to its predecessors through a decoupled look-back, and
// X_next = X + dx is written.  Only X is read and X_next written per
// iteration (16*d bytes per step).  The Newton loop itself runs on the device:
//
//  * resident_solve_kernel — one CTA per trajectory (N <= THREADS*ITEMS), the
//    whole solve in one launch with X resident in shared memory (BASELINE
//    cfg 1 and the batched cfg 3).
//  * grid_resident_kernel — one trajectory over a co-resident wave of CTAs
//    (cfg 2): each CTA keeps its tile of X in shared memory for the whole
//    solve; one grid barrier, one aggregate fold and an identical on-device
//    decision per iteration.
//  * persistent_ws_kernel (solve_ws.cuh) — the streaming kernel for
//    trajectories larger than one wave (cfg 5).
//
// The decision sequence is solve()'s (newton_pint.py:373-394) plus the
// BASELINE step rule, identical to oracle/odescan_oracle.c:orc_solve.
#pragma once

#include <cstdint>

#include "scan.cuh"
#include "sm100.cuh"

namespace odx {

struct SolveParams {
    ProbParams prob;
    StepCoefs sc;
    const double* x0;  // B x D
    double* X;         // B x N x D (guess in, final iterate out)
    long long B, N;
    int max_iters;
    int abort_nonfinite;
    double rtol, stol;
    double* hist;   // B x (max_iters+1) or null
    double* shist;  // B x (max_iters+1) or null
    int* iters;
    int* status;
    long long* sidx;
    // persistent-kernel workspace
    double* Xalt;
    uint32_t* flags;
    double* aggbuf;
    double* inclbuf;
    uint32_t* ctr;
    unsigned long long* red;  // 4 x (max_iters+1): rn, sc, step, bad
    unsigned* bar;            // count, gen
    long long ntiles;
};

struct Decision {
    int stop;
    int status;
    long long index;
    int iters;
};

// solve() decision sequence (newton_pint.py:373-394) + BASELINE step rule.
__device__ __forceinline__ Decision decide(int it, const SolveParams& p, double rn,
                                           unsigned long long bad, double step_prev) {
    Decision d{0, -1, -1, 0};
    if (bad != ~0ull) {
        d.stop = 1; d.status = ODX_ST_SINGULAR; d.index = (long long)bad; d.iters = it;
        return d;
    }
    if (isinf(rn) && p.abort_nonfinite) {
        d.stop = 1; d.status = ODX_ST_NONFINITE; d.index = it; d.iters = it;
        return d;
    }
    bool conv = (p.rtol > 0.0 && rn <= p.rtol) || (p.stol > 0.0 && it > 0 && step_prev < p.stol);
    if (it >= p.max_iters) {
        d.stop = 1; d.status = conv ? ODX_ST_CONVERGED : ODX_ST_MAXITER; d.iters = p.max_iters;
        return d;
    }
    if (conv) {
        d.stop = 1; d.status = ODX_ST_CONVERGED; d.iters = it;
    }
    return d;
}

// Shared-memory row staging with one pad double per ITEMS*D doubles, so that
// thread t's rows start at an odd multiple of 8 bytes (no bank conflicts when
// a warp reads its blocked rows).
template <int D, int ITEMS>
struct RowLayout {
    static constexpr int CH = ITEMS * D;  // doubles per thread chunk
    __device__ __forceinline__ static int idx(int linear) { return linear + linear / CH; }
    static constexpr int size(int rows) { return rows * D + (rows * D) / CH + 1; }
};

template <class P, int KIND, int S, int THREADS, int ITEMS>
struct SmallEngine {
    static constexpr int D = P::D;
    static constexpr int NW = THREADS / 32;
    static constexpr int T = THREADS * ITEMS;
    using L = RowLayout<D, ITEMS>;
    static constexpr int XS = L::size(T + 1);

    struct Shared {
        double xs[XS];
        double wtF[NW][D * D];
        double wtc[NW][D];
        int wthas[NW];
        double z[D];
        double redd[3][NW];
        unsigned long long redb[NW];
        long long tile;
    };

    // Build the ITEMS elements of this thread from rows staged in sm.xs
    // (row 0 = the state before step `base`).  Accumulates rn/sc/bad.
    __device__ __forceinline__ static void build_items(const P& prob, const StepCoefs& sc,
                                                       const Shared& sm, long long base,
                                                       long long N, Elem<D> (&el)[ITEMS],
                                                       double& rn, double& scn,
                                                       unsigned long long& bad) {
        const int tid = threadIdx.x;
#pragma unroll
        for (int i = 0; i < ITEMS; i++) {
            const int r = tid * ITEMS + i;
            const long long k = base + r;
            if (k < N) {
                double prev[D], xk[D], h[D];
#pragma unroll
                for (int j = 0; j < D; j++) {
                    prev[j] = sm.xs[L::idx(r * D + j)];
                    xk[j] = sm.xs[L::idx((r + 1) * D + j)];
                }
                bool sing = build_step<P, KIND, S>(prob, sc, prev, xk, k == 0, el[i], h);
                rn = nan_drop_max(rn, row_max_abs<D>(h));
                if (KIND == 1) scn = nan_drop_max(scn, row_max_abs<D>(el[i].c));
                if (sing && (unsigned long long)k < bad) bad = (unsigned long long)k;
            }
        }
    }

    // One item (step base + tid*ITEMS + i) of build_items.
    __device__ __forceinline__ static void build_item(const P& prob, const StepCoefs& sc,
                                                      const Shared& sm, long long base, long long N,
                                                      int i, Elem<D>& el, double& rn, double& scn,
                                                      unsigned long long& bad) {
        const int r = threadIdx.x * ITEMS + i;
        const long long k = base + r;
        if (k < N) {
            double prev[D], xk[D], h[D];
#pragma unroll
            for (int j = 0; j < D; j++) {
                prev[j] = sm.xs[L::idx(r * D + j)];
                xk[j] = sm.xs[L::idx((r + 1) * D + j)];
            }
            bool sing = build_step<P, KIND, S>(prob, sc, prev, xk, k == 0, el, h);
            rn = nan_drop_max(rn, row_max_abs<D>(h));
            if (KIND == 1) scn = nan_drop_max(scn, row_max_abs<D>(el.c));
            if (sing && (unsigned long long)k < bad) bad = (unsigned long long)k;
        }
    }

    // build_item for an item known to exist, branch-free for implicit steps
    // (two calls written back to back interleave)
    __device__ __forceinline__ static void build_item_bf(const P& prob, const StepCoefs& sc,
                                                         const Shared& sm, long long base, int i,
                                                         Elem<D>& el, double& rn, double& scn,
                                                         unsigned long long& bad) {
        const int r = threadIdx.x * ITEMS + i;
        const long long k = base + r;
        double prev[D], xk[D], h[D];
#pragma unroll
        for (int j = 0; j < D; j++) {
            prev[j] = sm.xs[L::idx(r * D + j)];
            xk[j] = sm.xs[L::idx((r + 1) * D + j)];
        }
        bool sing;
        if constexpr (KIND == 1)
            sing = build_implicit_step_bf<P>(prob, sc, prev, xk, k == 0, el, h);
        else
            sing = build_step<P, KIND, S>(prob, sc, prev, xk, k == 0, el, h);
        rn = nan_drop_max(rn, row_max_abs<D>(h));
        if (KIND == 1) scn = nan_drop_max(scn, row_max_abs<D>(el.c));
        if (sing && (unsigned long long)k < bad) bad = (unsigned long long)k;
    }

    // NI consecutive explicit items (i0 .. i0+NI-1, all present) built
    // stage-interleaved (build_explicit_multi)
    template <int NI>
    __device__ __forceinline__ static void build_items_multi(const P& prob, const StepCoefs& sc,
                                                             const Shared& sm, long long base,
                                                             int i0, Elem<D>* el, double& rn) {
        double prev[NI][D], xk[NI][D], h[NI][D];
        bool first[NI];
        Elem<D> e[NI];
#pragma unroll
        for (int n = 0; n < NI; n++) {
            const int r = threadIdx.x * ITEMS + i0 + n;
#pragma unroll
            for (int j = 0; j < D; j++) {
                prev[n][j] = sm.xs[L::idx(r * D + j)];
                xk[n][j] = sm.xs[L::idx((r + 1) * D + j)];
            }
            first[n] = (base + r == 0);
        }
        build_explicit_multi<P, S, NI>(prob, sc, prev, xk, first, e, h);
#pragma unroll
        for (int n = 0; n < NI; n++) {
            el[n] = e[n];
            rn = nan_drop_max(rn, row_max_abs<D>(h[n]));
        }
    }

    // Fold this thread's items, scan the block, and leave the warp totals in
    // shared memory.  Returns the thread inclusive aggregate (within its warp).
    __device__ __forceinline__ static void block_scan(Shared& sm, long long base, long long N,
                                                      const Elem<D> (&el)[ITEMS], Elem<D>& agg,
                                                      bool& has) {
        const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
        if (base + T <= N) {
            // full tile (CTA-uniform): the same compositions in the same
            // order without validity bits or branches
            agg = el[0];
#pragma unroll
            for (int i = 1; i < ITEMS; i++) compose<D>(agg, el[i], agg);
            has = true;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                Elem<D> o, t;
                shfl_up_elem<D>(agg, o, off);
                compose<D>(o, agg, t);
                if (lane >= off) agg = t;
            }
        } else {
        has = false;
#pragma unroll
        for (int i = 0; i < ITEMS; i++) {
            const long long k = base + tid * ITEMS + i;
            if (k < N) {
                if (has)
                    compose<D>(agg, el[i], agg);
                else {
                    agg = el[i];
                    has = true;
                }
            }
        }
        if (!has) set_identity<D>(agg);
        warp_inclusive_scan<D>(agg, has, lane);
        }
        if (lane == 31) {
#pragma unroll
            for (int i = 0; i < D * D; i++) sm.wtF[w][i] = agg.F[i];
#pragma unroll
            for (int i = 0; i < D; i++) sm.wtc[w][i] = agg.c[i];
            sm.wthas[w] = has ? 1 : 0;
        }
    }

    // Tile aggregate = warp totals composed in order (one thread).
    __device__ __forceinline__ static void tile_aggregate(const Shared& sm, Elem<D>& A, bool& A_has) {
        A_has = false;
#pragma unroll 1
        for (int w = 0; w < NW; w++) {
            if (!sm.wthas[w]) continue;
            Elem<D> e;
#pragma unroll
            for (int i = 0; i < D * D; i++) e.F[i] = sm.wtF[w][i];
#pragma unroll
            for (int i = 0; i < D; i++) e.c[i] = sm.wtc[w][i];
            if (A_has)
                compose<D>(A, e, A);
            else {
                A = e;
                A_has = true;
            }
        }
    }

    // Apply the scanned prefix: given the tile-exclusive state offset sm.z,
    // compute dx for every item, write X + dx into sm.xs rows 1..T, and
    // accumulate max|dx| (NaN-ignoring row rule).
    __device__ __forceinline__ static void apply_items(Shared& sm, long long base, long long N,
                                                       const Elem<D> (&el)[ITEMS],
                                                       const Elem<D>& agg, bool has,
                                                       double& step) {
        const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
        double z[D];
#pragma unroll
        for (int r = 0; r < D; r++) z[r] = sm.z[r];
        // warp-exclusive: warp totals 0..w-1 applied in order (full tiles:
        // unrolled, so the next total's loads overlap the current apply)
        if (base + T <= N) {
#pragma unroll
            for (int q = 0; q < NW - 1; q++) {
                if (q < w) {
                    Elem<D> e;
#pragma unroll
                    for (int i = 0; i < D * D; i++) e.F[i] = sm.wtF[q][i];
#pragma unroll
                    for (int i = 0; i < D; i++) e.c[i] = sm.wtc[q][i];
                    apply<D>(e, z, z);
                }
            }
        } else
#pragma unroll 1
        for (int q = 0; q < w; q++) {
            if (!sm.wthas[q]) continue;
            Elem<D> e;
#pragma unroll
            for (int i = 0; i < D * D; i++) e.F[i] = sm.wtF[q][i];
#pragma unroll
            for (int i = 0; i < D; i++) e.c[i] = sm.wtc[q][i];
            apply<D>(e, z, z);
        }
        // lane-exclusive within the warp
        Elem<D> ex;
        shfl_up_elem<D>(agg, ex, 1);
        bool exh = __shfl_up_sync(FULL, has, 1) && lane > 0;
        if (exh) apply<D>(ex, z, z);
        if (base + (long long)(tid + 1) * ITEMS <= N) {
            // full thread: the same operations in the same order, branch-free;
            // the row maxima are reduced apart from the dependent chain
            double rm[ITEMS];
#pragma unroll
            for (int i = 0; i < ITEMS; i++) {
                const int r = tid * ITEMS + i;
                double dx[D];
                apply<D>(el[i], z, dx);
                rm[i] = row_max_abs<D>(dx);
#pragma unroll
                for (int j = 0; j < D; j++) {
                    z[j] = dx[j];
                    sm.xs[L::idx((r + 1) * D + j)] += dx[j];
                }
            }
#pragma unroll
            for (int i = 0; i < ITEMS; i++) step = nan_drop_max(step, rm[i]);
            return;
        }
#pragma unroll
        for (int i = 0; i < ITEMS; i++) {
            const int r = tid * ITEMS + i;
            const long long k = base + r;
            if (k < N) {
                double dx[D];
                apply<D>(el[i], z, dx);
                step = nan_drop_max(step, row_max_abs<D>(dx));
#pragma unroll
                for (int j = 0; j < D; j++) {
                    z[j] = dx[j];
                    sm.xs[L::idx((r + 1) * D + j)] += dx[j];
                }
            }
        }
    }
};

// ---------------------------------------------------------------------------
// Resident solve: one CTA per trajectory, N <= THREADS*ITEMS, X in smem.
// ---------------------------------------------------------------------------
template <class P, int KIND, int S, int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS)
resident_solve_kernel(const SolveParams p) {
    using E = SmallEngine<P, KIND, S, THREADS, ITEMS>;
    constexpr int D = P::D;
    constexpr int NW = E::NW;
    using L = typename E::L;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    typename E::Shared& sm = *reinterpret_cast<typename E::Shared*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const long long b = blockIdx.x;
    const long long N = p.N;
    const P prob(p.prob);
    double* Xb = p.X + b * N * D;
    const int H = p.max_iters + 1;

    for (int i = tid; i < (int)((N + 1) * D); i += THREADS) {
        long long row = i / D - 1;
        sm.xs[L::idx(i)] = (row < 0) ? p.x0[b * D + i] : Xb[i - D];
    }
    if (tid < D) sm.z[tid] = 0.0;  // the trajectory starts in this tile: no incoming offset
    __syncthreads();

    double step_prev = __longlong_as_double(0x7ff8000000000000ll);  // NaN
    Decision dd{0, -1, -1, 0};
    for (int it = 0; it <= p.max_iters; it++) {
        Elem<D> el[ITEMS];
        double rn = 0.0, scn = 0.0;
        unsigned long long bad = ~0ull;
        if (KIND == 0 && ITEMS % 2 == 0 && N == E::T) {  // explicit, full tile: stage-interleaved pairs
#pragma unroll
            for (int i = 0; i < ITEMS; i += 2) E::template build_items_multi<2>(prob, p.sc, sm, 0, i, &el[i], rn);
        } else if (ITEMS % 2 == 0 && N == E::T) {  // full tile: items in interleavable pairs
#pragma unroll
            for (int i = 0; i < ITEMS; i += 2) {
                E::build_item_bf(prob, p.sc, sm, 0, i, el[i], rn, scn, bad);
                E::build_item_bf(prob, p.sc, sm, 0, i + 1, el[i + 1], rn, scn, bad);
            }
        } else {
            E::build_items(prob, p.sc, sm, 0, N, el, rn, scn, bad);
        }
        rn = warp_max_nan_drop(rn);
        scn = warp_max_nan_drop(scn);
        bad = warp_min_u64(bad);
        if (lane == 0) { sm.redd[0][w] = rn; sm.redd[1][w] = scn; sm.redb[w] = bad; }
        // The block scan does not depend on the decision (and changes no
        // state), so it runs before the iteration's first barrier; every
        // thread then reduces the warps' residuals itself (same order as a
        // single thread would) — two barriers per iteration instead of five.
        Elem<D> agg;
        bool has;
        E::block_scan(sm, 0, N, el, agg, has);
        __syncthreads();
        double rnb = 0.0, scb = 0.0;
        unsigned long long badb = ~0ull;
#pragma unroll
        for (int q = 0; q < NW; q++) {
            rnb = fmax(rnb, sm.redd[0][q]);
            scb = fmax(scb, sm.redd[1][q]);
            badb = sm.redb[q] < badb ? sm.redb[q] : badb;
        }
        if (KIND == 0) scb = rnb;
        dd = decide(it, p, rnb, badb, step_prev);
        if (tid == 0 && dd.status != ODX_ST_SINGULAR) {
            if (p.hist) p.hist[b * H + it] = rnb;
            if (p.shist) p.shist[b * H + it] = scb;
        }
        if (dd.stop) break;

        double step = 0.0;
        E::apply_items(sm, 0, N, el, agg, has, step);
        step = warp_max_nan_drop(step);
        if (lane == 0) sm.redd[2][w] = step;
        __syncthreads();
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < NW; q++) s = fmax(s, sm.redd[2][q]);
        step_prev = s;
    }
    for (int i = tid; i < (int)(N * D); i += THREADS) Xb[i] = sm.xs[L::idx(i + D)];
    if (tid == 0) {
        p.iters[b] = dd.iters;
        p.status[b] = dd.status;
        p.sidx[b] = dd.index;
    }
}

// ---------------------------------------------------------------------------
// Grid-resident solve: one trajectory with N <= G * THREADS * ITEMS, G CTAs
// co-resident (cooperative launch).  CTA g owns steps [g*T, g*T + T) for the
// whole solve: X rows stay in its shared memory and its elements in registers;
// per Newton iteration there is ONE grid barrier (after the tile aggregates and
// the residual reductions are published).  Each CTA then folds the aggregates
// of the CTAs before it (L2-resident, a warp-parallel ordered reduction) into
// its incoming state, applies it, and hands its new last row to CTA g+1
// through a tagged 16-byte chunk (no second barrier).  HBM is touched only by
// the initial load and the final store (BASELINE cfg 2: 1 MB of state).
// ---------------------------------------------------------------------------
struct GridResParams {
    SolveParams sp;
    double* aggs;      // 2 x G x (D*D + D): tile aggregates by iteration parity
    void* halos;       // G rows {tag, v[4]} (HaloRow)
};

template <int D>
__device__ __forceinline__ void warp_reduce_earliest_first(Elem<D>& e, bool& has, int lane) {
    // lower lanes are EARLIER in time; lane 0 ends with the composition of all
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        Elem<D> o;
        shfl_down_elem<D>(e, o, off);
        bool oh = __shfl_down_sync(FULL, has, off);
        if ((lane & (2 * off - 1)) == 0 && lane + off < 32 && oh) {
            if (has)
                compose<D>(e, o, e);  // o is later
            else {
                e = o;
                has = true;
            }
        }
    }
}

#ifdef ODX_GR_TRACE
__device__ unsigned long long* g_gr_trace = nullptr;  // [3 CTAs][iters][16]
#define GR_STAMP(slot_)                                                                  \
    do {                                                                                 \
        if (g_gr_trace && threadIdx.x == 0) {                                            \
            const int which_ = (g == 0) ? 0 : (g == G / 2) ? 1 : (g == G - 1) ? 2 : -1;  \
            if (which_ >= 0 && it < 64) {                                                \
                unsigned long long t_;                                                   \
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                   \
                g_gr_trace[(which_ * 64 + it) * 16 + (slot_)] = t_;                      \
            }                                                                            \
        }                                                                                \
    } while (0)
#else
#define GR_STAMP(slot_) do { } while (0)
#endif

template <class P, int KIND, int S, int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS)
grid_resident_kernel(const GridResParams gp) {
    using E = SmallEngine<P, KIND, S, THREADS, ITEMS>;
    constexpr int D = P::D;
    constexpr int NW = E::NW;
    constexpr int T = E::T;
    constexpr int EA = D * D + D;
    using L = typename E::L;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    typename E::Shared& sm = *reinterpret_cast<typename E::Shared*>(smem_raw);
    __shared__ double s_wagg[NW][EA];
    __shared__ int s_whas[NW];

    const SolveParams& p = gp.sp;
    // CTA g's last row for CTA g+1: one 16-byte {value, tag} chunk per
    // component (st_chunk / ld_chunk: ONE scalar .b128 memory operation, so
    // the PTX memory model guarantees a reader never pairs a new tag with an
    // old value — sm100.cuh), so the reader validates every
    // value by its own tag and the writer needs no release fence — a fence
    // here stalled the writing thread, and with it the next iteration's
    // entry barrier, by an L2 round trip
    struct alignas(64) HaloRow {
        Chunk c[4];
    };
    HaloRow* halos = reinterpret_cast<HaloRow*>(gp.halos);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const long long g = blockIdx.x;
    const unsigned G = gridDim.x;
    const long long N = p.N;
    const long long base = g * T;
    const long long rows = (N - base) < T ? (N - base) : T;
    const P prob(p.prob);

    // initial rows (row 0 = the state before step base)
    for (int i = tid; i < (int)((rows + 1) * D); i += THREADS) {
        const long long gi = (base - 1) * D + i;
        sm.xs[L::idx(i)] = (gi < 0) ? p.x0[i] : p.X[gi];
    }
    __syncthreads();

    Decision dd{0, -1, -1, 0};
    bool step_pending = false;
    for (int it = 0; it <= p.max_iters; it++) {
        GR_STAMP(0);
        __syncthreads();  // the last apply's rows are visible to every thread
        GR_STAMP(1);
        Elem<D> el[ITEMS];
        double rn = 0.0, scn = 0.0;
        unsigned long long bad = ~0ull;
        // items in the order 1..ITEMS-1, 0: thread 0's item 0 needs the halo
        // from CTA g-1 (its last row of the current iterate), whose arrival
        // then overlaps the thread's other items
        auto fetch_halo = [&]() {
            if (tid == 0 && it > 0 && g > 0) {
                const HaloRow* src = halos + (g - 1);
                const unsigned long long want = (unsigned long long)it;
                Chunk ch[D];
                int spins = 0;
                while (true) {
                    bool ok = true;
#pragma unroll
                    for (int k = 0; k < D; k++) {
                        ch[k] = ld_chunk(&src->c[k]);
                        ok = ok && ch[k].tag == want;
                    }
                    if (ok) break;
                    if (++spins > 8) __nanosleep(20);
                }
#pragma unroll
                for (int k = 0; k < D; k++) sm.xs[L::idx(k)] = ch[k].v;
            }
        };
        if (ITEMS % 2 == 0 && rows == T) {
            // full tile: pairs (1,2), (3,4), ..., (ITEMS-1, 0) built
            // back to back (branch-free: they interleave); the halo before the
            // pair that holds item 0
#pragma unroll
            for (int ii = 1; ii < ITEMS; ii += 2) {
                const int i0 = ii, i1 = (ii + 1) % ITEMS;
                if (i1 == 0) fetch_halo();
                E::build_item_bf(prob, p.sc, sm, base, i0, el[i0], rn, scn, bad);
                E::build_item_bf(prob, p.sc, sm, base, i1, el[i1], rn, scn, bad);
            }
        } else {
#pragma unroll
            for (int ii = 0; ii < ITEMS; ii++) {
                const int i = (ii + 1) % ITEMS;
                if (i == 0) fetch_halo();
                E::build_item(prob, p.sc, sm, base, N, i, el[i], rn, scn, bad);
            }
        }
        GR_STAMP(2);
        Elem<D> agg;
        bool has;
        const bool do_scan = it < p.max_iters;
        if (do_scan) E::block_scan(sm, base, N, el, agg, has);
        GR_STAMP(3);
        rn = warp_max_nan_drop(rn);
        scn = warp_max_nan_drop(scn);
        bad = warp_min_u64(bad);
        if (lane == 0) {
            sm.redd[0][w] = rn;
            sm.redd[1][w] = scn;
            sm.redb[w] = bad;
        }
        __syncthreads();
        if (tid == 0) {
            double a = 0.0, c = 0.0;
            unsigned long long m = ~0ull;
            for (int q = 0; q < NW; q++) {
                a = fmax(a, sm.redd[0][q]);
                c = fmax(c, sm.redd[1][q]);
                m = sm.redb[q] < m ? sm.redb[q] : m;
            }
            unsigned long long* red = p.red + 4ll * it;
            if (a > 0.0) atomicMax(red + 0, dbits(a));
            if (c > 0.0) atomicMax(red + 1, dbits(c));
            if (m != ~0ull) atomicMin(red + 3, m);
            if (step_pending) {  // max|dx| of iteration it-1
                double s2 = 0.0;
                for (int q = 0; q < NW; q++) s2 = fmax(s2, sm.redd[2][q]);
                if (s2 > 0.0) atomicMax(red - 4 + 2, dbits(s2));
            }
        }
        // the tile aggregate on another warp, alongside thread 0's reductions
        // (the barrier's opening __syncthreads orders both before the arrival)
        if (tid == (NW > 1 ? 32 : 0)) {
            if (do_scan) {
                Elem<D> A;
                bool A_has = false;
                E::tile_aggregate(sm, A, A_has);
                // double-buffered by iteration parity: a CTA that is already
                // publishing iteration it+1 must not overwrite aggregates a
                // slower CTA is still folding for iteration it
                double* dst = gp.aggs + ((long long)(it & 1) * G + g) * EA;
#pragma unroll
                for (int k = 0; k < D * D; k++) dst[k] = A.F[k];
#pragma unroll
                for (int k = 0; k < D; k++) dst[D * D + k] = A.c[k];
            }
        }
        GR_STAMP(4);
        grid_barrier_mono(p.bar, (unsigned)(it + 1) * G);
        GR_STAMP(5);
        // incoming state: ordered fold of the aggregates of CTAs 0..g-1 over the
        // whole block (its L2 loads overlap the decision's); thread t folds a
        // contiguous run, warps reduce earliest-first, warp 0 joins the warps
        const unsigned long long* red = p.red + 4ll * it;
        const unsigned long long r_rn = __ldcg(red + 0), r_sc = __ldcg(red + 1), r_bad = __ldcg(red + 3);
        const unsigned long long r_step = (it > 0) ? __ldcg(red - 4 + 2) : 0ull;
        Elem<D> fe;
        bool fh = false;
        {
            const long long per = (g + THREADS - 1) / THREADS;
            const long long lo = tid * per, hi = (lo + per < g) ? lo + per : g;
            for (long long q = lo; q < hi; q++) {
                Elem<D> a;
                const double* src = gp.aggs + ((long long)(it & 1) * G + q) * EA;
#pragma unroll
                for (int k = 0; k < D * D; k++) a.F[k] = __ldcg(src + k);
#pragma unroll
                for (int k = 0; k < D; k++) a.c[k] = __ldcg(src + D * D + k);
                if (fh)
                    compose<D>(fe, a, fe);
                else {
                    fe = a;
                    fh = true;
                }
            }
        }
        const double rnb = bitsd(r_rn);
        const double scb = (KIND == 0) ? rnb : bitsd(r_sc);
        // every CTA's step atomic of iteration it-1 precedes this barrier
        const double step_prev = (it > 0) ? bitsd(r_step) : __longlong_as_double(0x7ff8000000000000ll);
        dd = decide(it, p, rnb, r_bad, step_prev);
        if (g == 0 && tid == 0 && dd.status != ODX_ST_SINGULAR) {
            if (p.hist) p.hist[it] = rnb;
            if (p.shist) p.shist[it] = scb;
        }
        GR_STAMP(6);
        if (dd.stop) break;
        if (!fh) set_identity<D>(fe);
        warp_reduce_earliest_first<D>(fe, fh, lane);
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < D * D; k++) s_wagg[w][k] = fe.F[k];
#pragma unroll
            for (int k = 0; k < D; k++) s_wagg[w][D * D + k] = fe.c[k];
            s_whas[w] = fh ? 1 : 0;
        }
        __syncthreads();
        if (tid == 0) {
            Elem<D> e;
            bool eh = false;
            for (int q = 0; q < NW; q++) {
                if (!s_whas[q]) continue;
                Elem<D> a;
#pragma unroll
                for (int k = 0; k < D * D; k++) a.F[k] = s_wagg[q][k];
#pragma unroll
                for (int k = 0; k < D; k++) a.c[k] = s_wagg[q][D * D + k];
                if (eh)
                    compose<D>(e, a, e);
                else {
                    e = a;
                    eh = true;
                }
            }
#pragma unroll
            for (int k = 0; k < D; k++) sm.z[k] = eh ? e.c[k] : 0.0;
        }
        __syncthreads();
        GR_STAMP(7);
        double step = 0.0;
        E::apply_items(sm, base, N, el, agg, has, step);
        GR_STAMP(8);
        // the thread that owns the last row hands it to CTA g+1 (tag = next
        // iteration) as soon as it has written it
        if (g + 1 < G && tid == (int)((rows - 1) / ITEMS)) {
            HaloRow* dst = halos + g;
#pragma unroll
            for (int k = 0; k < D; k++)
                st_chunk(&dst->c[k], sm.xs[L::idx((int)rows * D + k)], (unsigned long long)(it + 1));
        }
        // max|dx|: warp maxima now; the block max and its atomic ride on the
        // next iteration's reduction (before that iteration's barrier)
        step = warp_max_nan_drop(step);
        if (lane == 0) sm.redd[2][w] = step;
        step_pending = true;
        GR_STAMP(9);
    }
    // final iterate back to global memory
    for (int i = tid; i < (int)(rows * D); i += THREADS) p.X[base * D + i] = sm.xs[L::idx(i + D)];
    if (g == 0 && tid == 0) {
        p.iters[0] = dd.iters;
        p.status[0] = dd.status;
        p.sidx[0] = dd.index;
    }
}

}  // namespace odx
