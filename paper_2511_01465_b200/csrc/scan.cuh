// scan.cuh — warp / block / grid scan primitives over affine elements.
//
// The reference computes the Newton step with a Blelloch up/down-sweep over
// padded arrays (_kernels.py:116-233, 3 full passes plus 4 temporaries).  On
// the GPU the scan is single pass: each thread folds its ITEMS consecutive
// elements in registers, warps combine with __shfl_up_sync (Kogge-Stone), the
// block combines warp totals through shared memory, and tiles chain through a
// decoupled look-back (aggregate / inclusive-prefix publication with
// release/acquire flags).  Because element 0 has F = 0 (_kernels.py:333-336),
// every inclusive prefix from the start of the trajectory has F = 0, so the
// inclusive payload a tile publishes is only the d-vector state offset.
//
// Elements carry a validity bit instead of being padded with identities, so no
// 0*inf products are introduced by padding.
#pragma once

#include <cstdint>

#include "elements.cuh"

namespace odx {

constexpr unsigned FULL = 0xffffffffu;

template <int D>
__device__ __forceinline__ void shfl_up_elem(const Elem<D>& in, Elem<D>& out, int off) {
#pragma unroll
    for (int i = 0; i < D * D; i++) out.F[i] = __shfl_up_sync(FULL, in.F[i], off);
#pragma unroll
    for (int i = 0; i < D; i++) out.c[i] = __shfl_up_sync(FULL, in.c[i], off);
}

template <int D>
__device__ __forceinline__ void shfl_down_elem(const Elem<D>& in, Elem<D>& out, int off) {
#pragma unroll
    for (int i = 0; i < D * D; i++) out.F[i] = __shfl_down_sync(FULL, in.F[i], off);
#pragma unroll
    for (int i = 0; i < D; i++) out.c[i] = __shfl_down_sync(FULL, in.c[i], off);
}

// Inclusive warp scan; lane L ends with elements of lanes 0..L composed in order.
template <int D>
__device__ __forceinline__ void warp_inclusive_scan(Elem<D>& agg, bool& has, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        Elem<D> o;
        shfl_up_elem<D>(agg, o, off);
        bool oh = __shfl_up_sync(FULL, has, off);
        if (lane >= off && oh) {
            if (has)
                compose<D>(o, agg, agg);
            else {
                agg = o;
                has = true;
            }
        }
    }
}

// Ordered warp reduction where LOWER lanes are LATER in time (look-back window).
// Lane 0 ends with the composition of all lanes that have an element.
template <int D>
__device__ __forceinline__ void warp_reduce_latest_first(Elem<D>& e, bool& has, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        Elem<D> o;
        shfl_down_elem<D>(e, o, off);
        bool oh = __shfl_down_sync(FULL, has, off);
        if ((lane & (2 * off - 1)) == 0 && lane + off < 32 && oh) {
            if (has)
                compose<D>(o, e, e);  // o is earlier
            else {
                e = o;
                has = true;
            }
        }
    }
}

// ---- memory-ordering helpers for the look-back flags -----------------------
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr uint32_t LB_AGG = 1u, LB_INCL = 2u;

__device__ __forceinline__ uint32_t lb_flag(uint32_t epoch, uint32_t kind) {
    return (epoch << 2) | kind;
}

// Spin until tile j's flag carries the current epoch; returns the kind.
__device__ __forceinline__ uint32_t lb_wait(const uint32_t* flags, long long j, uint32_t epoch) {
    uint32_t f = ld_acquire_u32(flags + j);
    int spins = 0;
    while ((f >> 2) != epoch) {
        if (++spins > 8) __nanosleep(32);
        f = ld_acquire_u32(flags + j);
    }
    return f & 3u;
}


// ---- block-wide reductions ---------------------------------------------------
__device__ __forceinline__ double warp_max_nan_drop(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, off));
    return v;
}
__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        unsigned long long o = __shfl_xor_sync(FULL, v, off);
        v = o < v ? o : v;
    }
    return v;
}

// Non-negative doubles (and +inf) order like their bit patterns.
__device__ __forceinline__ unsigned long long dbits(double v) {
    return (unsigned long long)__double_as_longlong(v);
}
__device__ __forceinline__ double bitsd(unsigned long long b) {
    return __longlong_as_double((long long)b);
}

// ---- grid barrier for cooperative (co-resident) launches --------------------
__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen, unsigned nblocks) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g = *(volatile unsigned*)gen;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *(volatile unsigned*)count = 0u;
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*(volatile unsigned*)gen == g) __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

// Grid barrier on a monotonically increasing arrival counter (zeroed once per
// launch): the caller's k-th barrier passes once count >= k * nblocks, i.e.
// `target`.  One acq_rel atomic per CTA; the last arriver never spins.
__device__ __forceinline__ void grid_barrier_mono(unsigned* count, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(count) : "memory");
        if ((int)(old + 1u - target) < 0) {
            unsigned v;
            do {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(count) : "memory");
            } while ((int)(v - target) < 0);
        }
    }
    __syncthreads();
}

}  // namespace odx
