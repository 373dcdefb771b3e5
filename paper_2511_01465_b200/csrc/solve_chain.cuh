// solve_chain.cuh — shared pieces of the single-pass chained Newton iteration
// for long trajectories (cfg 5: one trajectory of N = 2^26 steps, d = 2): launch
// parameters, the per-tile trace, row loaders, the workspace layout and the
// finish kernel.  The pass kernel itself is in solve_chain2.cuh.
//
// (The first cut of the pass kernel lived here: one CTA per SM with seven
// compute warps in lockstep and a control warp, 16.1 ms per cfg5 solve.  It was
// replaced by solve_chain2.cuh's independent warp groups, 12.8 ms, and removed:
// with a cheap build — explicit Euler, d = 1 — its control-warp hand-off could
// deadlock at N = 2^25.)
#pragma once

#include "solve_small.cuh"

namespace odx {

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
    if constexpr (D == 2 && ITEMS % 2 == 1) {
        if (r0 + ITEMS <= N) {
            const double* src = X + r0 * 2;
#pragma unroll
            for (int q = 0; q < ITEMS; q++) ld_row2_nc(src + 2 * q, rw[2 + 2 * q], rw[3 + 2 * q]);
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
    if constexpr (D == 1 && ITEMS % 2 == 0) {
        // d = 1: the thread's ITEMS rows as 16-byte pairs (r0 is even)
        if (r0 + ITEMS <= N) {
#pragma unroll
            for (int q = 0; q < ITEMS / 2; q++) ld_row2_nc(X + r0 + 2 * q, rw[1 + 2 * q], rw[2 + 2 * q]);
            if (lane == 0) rw[0] = (r0 == 0) ? x0[0] : __ldg(X + r0 - 1);
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
    if constexpr (D == 2) {
        const double h0 = __shfl_up_sync(FULL, rw[2 * ITEMS], 1);
        const double h1 = __shfl_up_sync(FULL, rw[2 * ITEMS + 1], 1);
        if (lane > 0 && r0 + ITEMS <= N) {
            rw[0] = h0;
            rw[1] = h1;
        }
    }
    if constexpr (D == 1 && ITEMS % 2 == 0) {
        const double h0 = __shfl_up_sync(FULL, rw[ITEMS], 1);
        if (lane > 0 && r0 + ITEMS <= N) rw[0] = h0;
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
        constexpr int E = D * D + D;
        ntiles = (N + T - 1) / T;
        size_t off = 0;
        auto at = [&](size_t bytes) { off = align_up(off, 256); size_t o = off; off += bytes; return o; };
        red = at(4 * ((size_t)max_iters + 1) * 8);  // first: init_ws sets its bad slots
        ctr = at(((size_t)max_iters + 1) * 4);
        done = at(((size_t)max_iters + 1) * 4);
        flags = at(4 * 8);  // stop, final_alt, step_prev
        const size_t nt32 = ((size_t)ntiles + 31) / 32 * 32;  // (solve_chain2.cuh: 32-tile blocks)
        recA = at(nt32 * E * sizeof(Chunk));
        recP = at(nt32 * D * sizeof(Chunk));
        zero_end = off;
        Xalt = at((size_t)N * D * 8);
        total = off + 256;
    }
};

}  // namespace odx
