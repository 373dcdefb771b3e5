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
//   step   : fixup of iteration it fused with local of iteration it+1 in ONE
//            pass over the rank's steps (shard_fused_kernel): each tile's old
//            elements and rows are scanned into the new rows, which are built
//            into the new elements while still in registers; the elements and
//            rows cross HBM once per iteration instead of twice.
//
// The rank's elements stay in its workspace between the calls: one build per
// iteration, no look-back, one collective.
#pragma once

#include "solve_tiled.cuh"

namespace odx {

// contiguous chunks per rank = CTAs of the build / apply / fused kernels (each
// CTA walks its chunk's tiles in order): two per SM, the fused kernel's
// residency for d <= 2
inline int shard_chunks() { return 2 * num_sms(); }

// tile shape of the shard kernels: 128 threads x ITEMS consecutive steps each.
// ITEMS is odd for d <= 2 so a lane's items (ITEMS*E doubles apart in shared
// memory) fall on distinct bank pairs up to 2-way.  Measured for d = 2 (cfg5):
// 5 items (640-step tiles, two CTAs per SM at 253 registers, five builds
// interleaved) 1.678 ms per iteration; 3 items (three CTAs per SM at 168
// registers) 1.703 ms; 4 items 16-way bank conflicts.
constexpr int SHARD_THREADS = 128;
template <int D>
constexpr int shard_items() { return D <= 2 ? 5 : 2; }

template <int D>
struct ShardTiledLayout {
    static constexpr int E = D * D + D;
    size_t red, stop, z, dlast, el, cagg, cpre, zc, prevs, bnd, total;
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
        zc = at(((size_t)nch + 1) * D * 8);     // chunk incoming update states
        prevs = at(((size_t)nch + 1) * D * 8);  // new state before each chunk
        bnd = at(((size_t)nch + 1) * D * 8);    // [c] = row before chunk c
        total = off + 256;
    }
};

// K2 + record in one CTA (nch <= SHARD_SCAN_THREADS chunks, one per thread):
// block scan of the chunk aggregates -> exclusive prefixes cpre[c] and the
// range aggregate cpre[nch]; then the rank's record [range F | range c |
// x_last | rn | sc | step_prev | bad] — step_prev is this pass's max|dx| when
// it applied an update (fused), else NaN.  Non-fused passes also record the
// row before each chunk (bnd) for the next fused pass.
constexpr int SHARD_SCAN_THREADS = 512;

template <int D>
__global__ void __launch_bounds__(SHARD_SCAN_THREADS)
shard_scan_record_kernel(const double* cagg, double* cpre, int nch, const double* X, long long n,
                         const unsigned long long* red, const int* stop, int explicit_kind,
                         int fused, double* bnd, long long rows_per_chunk, double* rec) {
    constexpr int E = D * D + D, dd = D * D, NW = SHARD_SCAN_THREADS / 32;
    if (*stop) return;
    __shared__ double s_w[NW][E];
    __shared__ int s_wh[NW];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    Elem<D> a;
    const bool has = t < nch;
    if (has)
        ld_elem<D>(cagg + (long long)t * E, a);
    else
        set_identity<D>(a);
    Elem<D> inc = a;
    bool ih = has;
    warp_inclusive_scan<D>(inc, ih, lane);
    if (lane == 31) {
        st_elem<D>(s_w[w], inc);
        s_wh[w] = ih ? 1 : 0;
    }
    __syncthreads();
    Elem<D> ex;
    bool exh = false;
    for (int q = 0; q < w; q++) {
        if (!s_wh[q]) continue;
        Elem<D> b;
        ld_elem<D>(s_w[q], b);
        if (exh)
            compose<D>(ex, b, ex);
        else {
            ex = b;
            exh = true;
        }
    }
    Elem<D> lx;
    shfl_up_elem<D>(inc, lx, 1);
    const bool lxh = __shfl_up_sync(FULL, ih, 1) && lane > 0;
    if (lxh) {
        if (exh)
            compose<D>(ex, lx, ex);
        else {
            ex = lx;
            exh = true;
        }
    }
    if (!exh) set_identity<D>(ex);
    if (has) st_elem<D>(cpre + (long long)t * E, ex);
    if (t == nch - 1) {  // the range aggregate, straight into the record too
        Elem<D> r = a;
        if (exh) compose<D>(ex, a, r);
        st_elem<D>(cpre + (long long)nch * E, r);
        st_elem<D>(rec, r);
    }
    if (t < D) rec[dd + D + t] = X[(n - 1) * D + t];
    if (t == 0) {
        const double rn = bitsd(red[0]);
        rec[dd + 2 * D + 0] = rn;
        rec[dd + 2 * D + 1] = explicit_kind ? rn : bitsd(red[1]);
        rec[dd + 2 * D + 2] = fused ? bitsd(red[2]) : __longlong_as_double(0x7ff8000000000000ll);
        rec[dd + 2 * D + 3] = (red[3] == ~0ull) ? -1.0 : (double)(long long)red[3];
    }
    if (!fused && t >= 1 && t < nch) {
        const long long k0 = (long long)t * rows_per_chunk;
        if (k0 < n)
#pragma unroll
            for (int j = 0; j < D; j++) bnd[t * D + j] = X[(k0 - 1) * D + j];
    }
}

// out = F z + c.  One non-inlined function for the carry, the exit state and
// hence the halo update.
static __device__ __noinline__ void affine_apply(const double* F, const double* c, const double* z, int d,
                                          double* out) {
    for (int r = 0; r < d; r++) {
        double acc = c[r];
        for (int q = 0; q < d; q++) acc = __fma_rn(F[r * d + q], z[q], acc);
        out[r] = acc;
    }
}

// solve()'s decision on the device, from the gathered records (the same
// reductions and order as sharded.decide / ShardedNewton.run): every rank
// evaluates it on identical inputs, so all ranks agree without a host round
// trip.  state = {stopped, status, iterations, status_index}.
struct ShardDecision {
    int max_iters, abort_nonfinite;
    double rtol, stol;
    double* hist;     // max_iters + 1 (may be null)
    double* shist;
    long long* state;
};

// carry pass of a fused step (one CTA): [decision of iteration `it`], then the
// carry z of `rank` from the gathered records, halo += z, and per chunk c:
// zc[c] = A_cpre[c](z) (zc[nch] is the rank's exit state) and the new state
// before chunk c's first step: the new halo (c = 0) or bnd[c] + zc[c].
// Resets the pass's reductions; *stop = 1 skips the rest of the step.
template <int D>
__global__ void shard_step_carry_kernel(const double* recs, int rank, int nranks, int it,
                                        ShardDecision dec, int decide_here, const double* cpre,
                                        int nch, const double* bnd, double* halo, double* zc,
                                        double* prevs, unsigned long long* red, int* stop) {
    constexpr int E = D * D + D, R = ODX_SHARD_REC(D);
    __shared__ double s_z[4], s_h[4];
    __shared__ int s_go;
    if (threadIdx.x == 0) {
        int go = 1;
        if (decide_here) {
            if (it > 0 && dec.state[0]) {
                go = 0;  // stopped at an earlier iteration
            } else {
                constexpr int i_rn = D * D + 2 * D;
                double rn = 0.0, sc = 0.0, stp = 0.0;
                unsigned long long bad = ~0ull;
                for (int q = 0; q < nranks; q++) {
                    const double* r = recs + (long long)q * R;
                    rn = nan_drop_max(rn, r[i_rn]);
                    sc = nan_drop_max(sc, r[i_rn + 1]);
                    stp = nan_drop_max(stp, r[i_rn + 2]);
                    const double b = r[i_rn + 3];
                    if (b >= 0.0 && (unsigned long long)b < bad) bad = (unsigned long long)b;
                }
                SolveParams sp;
                memset(&sp, 0, sizeof(sp));
                sp.max_iters = dec.max_iters;
                sp.abort_nonfinite = dec.abort_nonfinite;
                sp.rtol = dec.rtol;
                sp.stol = dec.stol;
                const double step_prev = it > 0 ? stp : __longlong_as_double(0x7ff8000000000000ll);
                const Decision d = decide(it, sp, rn, bad, step_prev);
                if (d.status != ODX_ST_SINGULAR) {
                    if (dec.hist) dec.hist[it] = rn;
                    if (dec.shist) dec.shist[it] = sc;
                }
                if (d.stop) {
                    dec.state[0] = 1;
                    dec.state[1] = d.status;
                    dec.state[2] = d.iters;
                    dec.state[3] = d.index;
                    go = 0;
                } else {
                    dec.state[0] = 0;
                }
            }
        }
        s_go = go;
        *stop = go ? 0 : 1;
        if (go) {
            red[0] = red[1] = red[2] = 0ull;
            red[3] = ~0ull;
            double v[4] = {0.0, 0.0, 0.0, 0.0};
            for (int q = 0; q < rank; q++) {
                const double* F = recs + (long long)q * R;
                double t[4];
                affine_apply(F, F + D * D, v, D, t);
                for (int r = 0; r < D; r++) v[r] = t[r];
            }
            for (int r = 0; r < D; r++) {
                s_z[r] = v[r];
                double h = halo[r];
                if (rank > 0) {
                    h = h + v[r];
                    halo[r] = h;
                }
                s_h[r] = h;
            }
        }
    }
    __syncthreads();
    if (!s_go) return;
    for (int c = threadIdx.x; c <= nch; c += blockDim.x) {
        const double* A = cpre + (long long)c * E;
        double e[4];
        affine_apply(A, A + D * D, s_z, D, e);
        for (int j = 0; j < D; j++) {
            zc[c * D + j] = e[j];
            if (c < nch) prevs[c * D + j] = (c == 0) ? s_h[j] : bnd[c * D + j] + e[j];
        }
    }
}

// one row of X: 16-byte stores where the row allows (torch / cudaMalloc rows
// of d = 2, 4 doubles are 16-byte aligned)
template <int D>
__device__ __forceinline__ void st_row(double* dst, const double* v) {
    if constexpr (D % 2 == 0) {
#pragma unroll
        for (int j = 0; j < D; j += 2)
            *reinterpret_cast<double2*>(dst + j) = make_double2(v[j], v[j + 1]);
    } else {
#pragma unroll
        for (int j = 0; j < D; j++) dst[j] = v[j];
    }
}

struct ShardFusedParams {
    ProbParams prob;
    StepCoefs sc;
    double* X;             // n x d rows: old in, new out (in place)
    double* el;            // n x E elements: old in, new out (in place)
    double* cagg;          // nch x E new chunk aggregates
    const double* zc;      // (nch + 1) x d: update state entering chunk c (old scan)
    const double* prevs;   // nch x d: new state before chunk c's first step
    double* bnd;           // (nch + 1) x d: new last row of chunk c-1 at [c]
    unsigned long long* red;
    const int* stop;       // set by the carry / decision pass: skip the pass
    long long n, offset, ntiles;
    int nch;
    int store;             // 0: the built elements are never applied (last pass): not stored
};

template <int D, int THREADS, int ITEMS>
struct ShardFusedSmem {
    static constexpr int E = D * D + D, T = THREADS * ITEMS;
    double el[2][T * E];
    double x[2][T * D];
    double out[T * E];
    uint64_t bar[2];
};

// CTA c walks its chunk in order.  Per tile: old elements + old rows (TMA,
// double-buffered) -> block scan with the running update state -> new rows
// (X += dx, written in place); the chunk's last row is instead set to
// x_old + zc[c+1], the same value the next chunk's CTA derives for its first
// step's predecessor (prevs) — so every step is built against exactly the row
// stored.  The new rows are then built into the new elements (build_step),
// staged in smem, written over the old ones, and folded into the chunk
// aggregate; rn / sc / first singular step / max|dx| -> red.
template <class P, int KIND, int S, int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS, ITEMS <= 3 ? 3 : 2) shard_fused_kernel(const ShardFusedParams fp) {
    constexpr int D = P::D, E = D * D + D, NW = THREADS / 32, T = THREADS * ITEMS;
    using SM = ShardFusedSmem<D, THREADS, ITEMS>;
    extern __shared__ __align__(16) unsigned char fused_raw[];
    SM& sm = *reinterpret_cast<SM*>(fused_raw);
    __shared__ double s_wt[NW][E];
    __shared__ int s_wh[NW];
    __shared__ double s_nt[NW][E];
    __shared__ int s_nh[NW];
    __shared__ double s_z[D];
    __shared__ double s_prev[D];
    __shared__ double s_wl[NW][D];
    __shared__ double s_rd[3][NW];
    __shared__ unsigned long long s_rb[NW];
    if (*fp.stop) return;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const P prob(fp.prob);
    const long long N = fp.n;
    const int c = blockIdx.x;
    long long t0, t1;
    chunk_tiles(fp.ntiles, fp.nch, c, t0, t1);
    const long long klast = (t1 * T < N ? t1 * T : N) - 1;
    auto stage = [&](long long t, int b) {
        const long long base = t * T;
        const long long rows = (N - base) < T ? (N - base) : T;
        const uint32_t be = (uint32_t)(rows * E * 8) & ~15u, bx = (uint32_t)(rows * D * 8) & ~15u;
        mbar_arrive_expect_tx(&sm.bar[b], be + bx);
        if (be) tma_load_1d(sm.el[b], fp.el + base * E, be, &sm.bar[b]);
        if (bx) tma_load_1d(sm.x[b], fp.X + base * D, bx, &sm.bar[b]);
    };
    if (tid == 0) {
        mbar_init(&sm.bar[0], 1);
        mbar_init(&sm.bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_proxy_async_global();
        if (t0 < t1) stage(t0, 0);
        if (t0 + 1 < t1) stage(t0 + 1, 1);
#pragma unroll
        for (int j = 0; j < D; j++) {
            s_z[j] = fp.zc[c * D + j];
            s_prev[j] = fp.prevs[c * D + j];
        }
    }
    double zn[D];
#pragma unroll
    for (int j = 0; j < D; j++) zn[j] = fp.zc[(c + 1) * D + j];
    __syncthreads();
    uint32_t ph[2] = {0u, 0u};
    double step = 0.0, rn = 0.0, scn = 0.0;
    unsigned long long bad = ~0ull;
    Elem<D> chunk;
    bool chunk_has = false;
    for (long long t = t0; t < t1; t++) {
        const int b = (int)((t - t0) & 1);
        const long long base = t * T;
        const long long rows = (N - base) < T ? (N - base) : T;
        mbar_wait(&sm.bar[b], ph[b]);
        ph[b] ^= 1u;
        double xn[ITEMS][D], zt[D];
        {
            Elem<D> el[ITEMS];
            Elem<D> agg;
            bool has = false;
            // rows * E * 8 is a multiple of 16 (E = d(d+1) is even): the whole
            // tile's elements are in smem; an odd tail row of X (odd d) is not
            if (rows == T) {
#pragma unroll
                for (int q = 0; q < ITEMS; q++) {
                    const int r = tid * ITEMS + q;
                    ld_elem<D>(&sm.el[b][r * E], el[q]);
#pragma unroll
                    for (int j = 0; j < D; j++) xn[q][j] = sm.x[b][r * D + j];
                    if (q == 0)
                        agg = el[0];
                    else
                        compose<D>(agg, el[q], agg);
                }
                has = true;
            } else {
                const uint32_t bx = (uint32_t)(rows * D * 8) & ~15u;
#pragma unroll
                for (int q = 0; q < ITEMS; q++) {
                    const int r = tid * ITEMS + q;
                    if (r < rows) {
                        ld_elem<D>(&sm.el[b][r * E], el[q]);
#pragma unroll
                        for (int j = 0; j < D; j++)
                            xn[q][j] = ((uint32_t)(r * D + j + 1) * 8 <= bx)
                                           ? sm.x[b][r * D + j]
                                           : fp.X[(base + r) * D + j];
                        if (has)
                            compose<D>(agg, el[q], agg);
                        else {
                            agg = el[q];
                            has = true;
                        }
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
            if (t + 1 < t1) {  // a full tile without the chunk's last row
#pragma unroll
                for (int q = 0; q < ITEMS; q++) {
                    const long long k = base + (long long)tid * ITEMS + q;
                    double dx[D];
                    apply<D>(el[q], z, dx);
                    step = nan_drop_max(step, row_max_abs<D>(dx));
#pragma unroll
                    for (int j = 0; j < D; j++) {
                        z[j] = dx[j];
                        xn[q][j] = xn[q][j] + dx[j];
                    }
                    st_row<D>(fp.X + k * D, xn[q]);
                }
            } else {
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
                            xn[q][j] = xn[q][j] + (k == klast ? zn[j] : dx[j]);
                        }
                        st_row<D>(fp.X + k * D, xn[q]);
                        if (k == klast)
#pragma unroll
                            for (int j = 0; j < D; j++) fp.bnd[(c + 1) * D + j] = xn[q][j];
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < D; j++) zt[j] = z[j];
        }
        double pin[D];
#pragma unroll
        for (int j = 0; j < D; j++) pin[j] = s_prev[j];
        if (lane == 31)
#pragma unroll
            for (int j = 0; j < D; j++) s_wl[w][j] = xn[ITEMS - 1][j];
        if (tid == 0) tma_store_wait_read();  // the previous tile's bulk store left sm.out
        __syncthreads();  // (1) s_wl published, s_prev read, sm.out free
        double p0[D];
#pragma unroll
        for (int j = 0; j < D; j++) {
            const double up = __shfl_up_sync(FULL, xn[ITEMS - 1][j], 1);
            p0[j] = (tid == 0) ? pin[j] : (lane == 0 ? s_wl[w - 1][j] : up);
        }
        Elem<D> nagg;
        bool nh = false;
        auto take = [&](int q, long long k, const Elem<D>& e, const double* h, bool sing) {
            rn = nan_drop_max(rn, row_max_abs<D>(h));
            if (KIND == 1) scn = nan_drop_max(scn, row_max_abs<D>(e.c));
            if (sing && (unsigned long long)(fp.offset + k) < bad)
                bad = (unsigned long long)(fp.offset + k);
            if (fp.store) st_elem<D>(&sm.out[(tid * ITEMS + q) * E], e);
            if (nh)
                compose<D>(nagg, e, nagg);
            else {
                nagg = e;
                nh = true;
            }
        };
        const long long kb = base + (long long)tid * ITEMS;
        if (KIND == 0 && kb + ITEMS <= N) {
            // explicit, all items present: stage-interleaved build (ILP)
            double prev[ITEMS][D], h[ITEMS][D];
            bool first[ITEMS];
            Elem<D> e[ITEMS];
#pragma unroll
            for (int q = 0; q < ITEMS; q++) {
#pragma unroll
                for (int j = 0; j < D; j++) prev[q][j] = (q == 0) ? p0[j] : xn[q - 1][j];
                first[q] = (fp.offset + kb + q == 0);
            }
            build_explicit_multi<P, S, ITEMS>(prob, fp.sc, prev, xn, first, e, h);
#pragma unroll
            for (int q = 0; q < ITEMS; q++) take(q, kb + q, e[q], h[q], false);
        } else if (KIND == 1 && kb + ITEMS <= N) {
            // implicit, all items present: branch-free builds back to back
#pragma unroll
            for (int q = 0; q < ITEMS; q++) {
                const long long k = kb + q;
                double prev[D], h[D];
#pragma unroll
                for (int j = 0; j < D; j++) prev[j] = (q == 0) ? p0[j] : xn[q - 1][j];
                Elem<D> e;
                const bool sing =
                    build_implicit_step_bf<P>(prob, fp.sc, prev, xn[q], fp.offset + k == 0, e, h);
                take(q, k, e, h, sing);
            }
        } else {
#pragma unroll
            for (int q = 0; q < ITEMS; q++) {
                const long long k = kb + q;
                if (k < N) {
                    double prev[D], h[D];
#pragma unroll
                    for (int j = 0; j < D; j++) prev[j] = (q == 0) ? p0[j] : xn[q - 1][j];
                    Elem<D> e;
                    const bool sing =
                        build_step<P, KIND, S>(prob, fp.sc, prev, xn[q], fp.offset + k == 0, e, h);
                    take(q, k, e, h, sing);
                }
            }
        }
        if (!nh) set_identity<D>(nagg);
        warp_reduce_earliest_first<D>(nagg, nh, lane);
        if (lane == 0) {
            st_elem<D>(s_nt[w], nagg);
            s_nh[w] = nh ? 1 : 0;
        }
        if (tid == (int)((rows - 1) / ITEMS)) {  // the tile's last step: next tile's states
            const int ql = (int)((rows - 1) % ITEMS);
#pragma unroll
            for (int j = 0; j < D; j++) s_z[j] = zt[j];
#pragma unroll
            for (int q = 0; q < ITEMS; q++)
                if (q == ql)
#pragma unroll
                    for (int j = 0; j < D; j++) s_prev[j] = xn[q][j];
        }
        fence_proxy_async_smem();  // staged elements -> the bulk store (async proxy)
        __syncthreads();  // (2) new elements staged, tile aggregates published
        if (tid == 0) {
            if (fp.store) {
                tma_store_1d(fp.el + base * E, sm.out, (uint32_t)(rows * E * 8));
                tma_store_commit();
            }
            for (int q = 0; q < NW; q++) {
                if (!s_nh[q]) continue;
                Elem<D> a;
                ld_elem<D>(s_nt[q], a);
                if (chunk_has)
                    compose<D>(chunk, a, chunk);
                else {
                    chunk = a;
                    chunk_has = true;
                }
            }
        }
        // sm.out is rewritten after the next tile's sync (1), which thread 0
        // reaches only once the bulk store has read it
    }
    if (tid == 0) {
        tma_store_wait_all();
        if (!chunk_has) set_identity<D>(chunk);
        st_elem<D>(fp.cagg + (long long)c * E, chunk);
    }
    rn = warp_max_nan_drop(rn);
    scn = warp_max_nan_drop(scn);
    step = warp_max_nan_drop(step);
    bad = warp_min_u64(bad);
    if (lane == 0) {
        s_rd[0][w] = rn;
        s_rd[1][w] = scn;
        s_rd[2][w] = step;
        s_rb[w] = bad;
    }
    __syncthreads();
    if (tid == 0) {
        double a = 0.0, cc = 0.0, st2 = 0.0;
        unsigned long long m = ~0ull;
        for (int q = 0; q < NW; q++) {
            a = fmax(a, s_rd[0][q]);
            cc = fmax(cc, s_rd[1][q]);
            st2 = fmax(st2, s_rd[2][q]);
            m = s_rb[q] < m ? s_rb[q] : m;
        }
        if (a > 0.0) atomicMax(fp.red + 0, dbits(a));
        if (cc > 0.0) atomicMax(fp.red + 1, dbits(cc));
        if (st2 > 0.0) atomicMax(fp.red + 2, dbits(st2));
        if (m != ~0ull) atomicMin(fp.red + 3, m);
    }
}

template <class P, int KIND, int S>
int shard_tiled_local(const ProbParams& pp, const StepCoefs& sc, const double* halo,
                      const double* X_local, long long n, long long offset, double* record,
                      void* ws, size_t ws_bytes, cudaStream_t st, int fused) {
    constexpr int D = P::D;
    constexpr int THREADS = SHARD_THREADS, ITEMS = shard_items<D>();
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
    double* bnd = reinterpret_cast<double*>(base + lay.bnd);
    if (nch > SHARD_SCAN_THREADS) return fail(ODX_EUNSUPPORTED, "too many shard chunks");
    if (fused) {
        // the carry / decision pass (shard.cu) has reset red and stop and
        // filled zc / prevs from the gathered records and the previous
        // pass's chunk prefixes
        ShardFusedParams fp;
        fp.prob = pp;
        fp.sc = sc;
        fp.X = const_cast<double*>(X_local);
        fp.el = tp.el;
        fp.cagg = tp.cagg;
        fp.zc = reinterpret_cast<const double*>(base + lay.zc);
        fp.prevs = reinterpret_cast<const double*>(base + lay.prevs);
        fp.bnd = bnd;
        fp.red = tp.sp.red;
        fp.stop = tp.stop;
        fp.n = n;
        fp.offset = offset;
        fp.ntiles = ntiles;
        fp.nch = nch;
        fp.store = (fused == 1) ? 1 : 0;  // 2: the last pass of a fixed-length solve
        const size_t smem = sizeof(ShardFusedSmem<D, THREADS, ITEMS>);
        auto kf = shard_fused_kernel<P, KIND, S, THREADS, ITEMS>;
        int occ = 0;
        if (int rc = kernel_occupancy((const void*)kf, THREADS, smem, &occ)) return rc;
        kf<<<(unsigned)nch, THREADS, smem, st>>>(fp);
    } else {
        init_ws(base, lay.stop + 8, 1, st);
        tiled_build_kernel<P, KIND, S, THREADS, ITEMS><<<(unsigned)nch, THREADS, 0, st>>>(tp, 0);
    }
    const long long per = (ntiles + nch - 1) / nch;
    shard_scan_record_kernel<D><<<1, SHARD_SCAN_THREADS, 0, st>>>(
        tp.cagg, tp.cpre, nch, X_local, n, tp.sp.red, tp.stop, KIND == 0, fused, bnd, per * T, record);
    ODX_CUDA(cudaGetLastError());
    count_launch(fused ? 2 : 3);
    return ODX_OK;
}


// ---------------------------------------------------------------------------
// One long trajectory on one GPU through the same passes (a "single-rank time
// shard"): local once, then per iteration [device decision + carry, fused
// fix-up + build, chunk scan + record], every iteration enqueued up front —
// passes after the stop decision return at once.  The record of the rank is
// its own "gathered" record (nranks = 1).
static __global__ void fused_solve_finish_kernel(const long long* state, int* iters, int* status,
                                          long long* sidx) {
    iters[0] = (int)state[2];
    status[0] = (int)state[1];
    sidx[0] = state[3];
}

template <class P, int KIND, int S>
int fused_tiled_solve(const SolveParams& p, void* ws, size_t ws_bytes, cudaStream_t st, bool query,
                      size_t* need) {
    constexpr int D = P::D, R = ODX_SHARD_REC(D);
    constexpr long long T = (long long)SHARD_THREADS * shard_items<D>();
    const int nch_max = shard_chunks();
    const ShardTiledLayout<D> lay(p.N, nch_max);
    const size_t rec_off = align_up(lay.total, 256);
    const size_t state_off = align_up(rec_off + (size_t)R * 8, 256);
    const size_t total = state_off + 4 * 8 + 256;
    if (query) {
        *need = total;
        return ODX_OK;
    }
    if (!ws || ws_bytes < total) return fail(ODX_EWORKSPACE, "workspace too small");
    if (reinterpret_cast<uintptr_t>(p.X) & 15) return fail(ODX_EINVAL, "X must be 16-byte aligned");
    char* base = reinterpret_cast<char*>(align_up(reinterpret_cast<size_t>(ws), 256));
    double* rec = reinterpret_cast<double*>(base + rec_off);
    long long* state = reinterpret_cast<long long*>(base + state_off);
    const long long ntiles = (p.N + T - 1) / T;
    const int nch = (int)(ntiles < nch_max ? ntiles : nch_max);
    if (int rc = shard_tiled_local<P, KIND, S>(p.prob, p.sc, p.x0, p.X, p.N, 0, rec, ws, ws_bytes,
                                               st, 0))
        return rc;
    ShardDecision dec;
    dec.max_iters = p.max_iters;
    dec.abort_nonfinite = p.abort_nonfinite;
    dec.rtol = p.rtol;
    dec.stol = p.stol;
    dec.hist = p.hist;
    dec.shist = p.shist;
    dec.state = state;
    for (int it = 0; it <= p.max_iters; it++) {
        shard_step_carry_kernel<D><<<1, 448, 0, st>>>(
            rec, 0, 1, it, dec, 1, reinterpret_cast<const double*>(base + lay.cpre), nch,
            reinterpret_cast<const double*>(base + lay.bnd), const_cast<double*>(p.x0),
            reinterpret_cast<double*>(base + lay.zc), reinterpret_cast<double*>(base + lay.prevs),
            reinterpret_cast<unsigned long long*>(base + lay.red),
            reinterpret_cast<int*>(base + lay.stop));
        count_launch(1);
        // the pass of iteration it builds iteration it+1's elements; at
        // it+1 == max_iters they are never applied (only rn is needed)
        if (int rc = shard_tiled_local<P, KIND, S>(p.prob, p.sc, p.x0, p.X, p.N, 0, rec, ws,
                                                   ws_bytes, st, it + 1 == p.max_iters ? 2 : 1))
            return rc;
    }
    fused_solve_finish_kernel<<<1, 1, 0, st>>>(state, p.iters, p.status, p.sidx);
    ODX_CUDA(cudaGetLastError());
    count_launch(1);
    set_route("shard_fused_kernel (fused tiled passes, elements stored between passes)");
    return ODX_OK;
}

}  // namespace odx
