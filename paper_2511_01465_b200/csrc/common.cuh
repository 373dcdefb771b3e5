// common.cuh — host-side helpers shared by the ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/odescan_b200.h"
#include "elements.cuh"

namespace odx {

void set_error(const char* fmt, ...);

inline int fail(int code, const char* msg) {
    set_error("%s", msg);
    return code;
}

#define ODX_CUDA(call)                                                              \
    do {                                                                            \
        cudaError_t _e = (call);                                                    \
        if (_e != cudaSuccess) {                                                    \
            ::odx::set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,             \
                             cudaGetErrorString(_e));                               \
            return ODX_ECUDA;                                                       \
        }                                                                           \
    } while (0)

int num_sms();
void count_launch(int n = 1);
// names the device path the last solve on this host thread took (odx_last_route)
void set_route(const char* route);

// Sets the kernel's dynamic shared-memory limit and returns its resident CTAs
// per SM, once per (kernel, block size, smem, device): both CUDA queries cost
// microseconds that would otherwise sit on every solve's launch path.
int kernel_occupancy(const void* kern, int threads, size_t smem, int* per_sm);

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// longest trajectory the batched (one CTA per trajectory) solve takes:
// 256 threads x (8 steps for d <= 3, 4 for d = 4) — solve_small_launch.cuh
constexpr long long resident_max_steps(int d) { return 256LL * (d <= 3 ? 8 : 4); }

// Carves a workspace into aligned sub-buffers (dry run when base is null).
struct Carver {
    char* base;
    size_t off = 0;
    template <class T>
    T* take(size_t count) {
        off = align_up(off, 256);
        T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
        off += count * sizeof(T);
        return p;
    }
};

bool fill_params(const odx_problem* P, ProbParams& pp);
bool fill_coefs(const odx_stepper* S, double dt, StepCoefs& sc);
void init_bad_slots(unsigned long long* red, int n, cudaStream_t st);
// zero [base, base+bytes) with the first n reduction quads' bad slots = ~0
// (base must be 8-byte aligned and start with those quads)
void init_ws(void* base, size_t bytes, int n, cudaStream_t st);

}  // namespace odx
