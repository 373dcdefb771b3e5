// host_solve.cu — odx_solve_host: the solver with HOST buffers on both sides
// (what the reference's numpy-in / numpy-out solve() hands over), one H2D and
// one D2H per call.  Replaces newton_pint.solve :326-406 for callers that hold
// their guess in host memory.
//
// Per device a grow-only cache keeps: the device region
//   x0 (B*d) | X (B*N*d) | outcome (hist | shist | sidx | iters | status)
// the solver workspace, and two pinned staging blocks (in: x0 | X, out: X |
// outcome).  A call packs the inputs into pinned memory, issues one H2D, the
// solve, one D2H, synchronises the stream and unpacks into the caller's
// buffers; caller buffers that are already page-locked skip the staging copy
// (DMA to / from them directly).  Calls are serialised by a mutex (the caches
// are shared).
//
// Large batches of resident trajectories (cfg 3: 4096 x 2048 x 3, 201 MB each
// way) are independent solves, so they run as a pipeline of up to 8 batch
// chunks, each on its own stream: the host packs chunk k+1 while chunk k is
// copied in, chunk k-1 is solved and chunk k-2 is copied out (PCIe is full
// duplex).  The caller's stream forks into the chunk streams after the x0 copy
// and joins them before the outcome copy, so it still orders the whole call.
#include <pthread.h>

#include <algorithm>
#include <atomic>
#include <emmintrin.h>
#include <chrono>
#include <condition_variable>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"

extern "C" {
size_t odx_solve_workspace_bytes(const odx_problem* P, const odx_stepper* S, int64_t B, int64_t N,
                                 const odx_newton_cfg* C);
int odx_solve(const odx_problem* P, const odx_stepper* S, const double* x0, double* X, int64_t B,
              int64_t N, double dt, const odx_newton_cfg* C, double* hist, double* scaled_hist,
              int32_t* iters, int32_t* status, int64_t* status_index, void* workspace,
              size_t workspace_bytes, void* stream);
}

namespace odx {
namespace {

struct HostCache {
    void* dregion = nullptr;
    size_t dbytes = 0;
    void* ws = nullptr;
    size_t wsbytes = 0;
    void* pin_in = nullptr;
    size_t in_bytes = 0;
    void* pin_out = nullptr;
    size_t out_bytes = 0;
    // batch pipeline (large resident batches): one stream + event per chunk
    static constexpr int MAXC = 8;
    cudaStream_t cs[MAXC] = {};
    cudaEvent_t ce[MAXC] = {};
    cudaEvent_t fork = nullptr;
};

std::mutex g_host_mu;
std::vector<HostCache> g_host_cache;

int grow_device(void** p, size_t* have, size_t need) {
    if (*have >= need) return ODX_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *have = 0;
    ODX_CUDA(cudaMalloc(p, need));
    *have = need;
    return ODX_OK;
}

int grow_pinned(void** p, size_t* have, size_t need) {
    if (*have >= need) return ODX_OK;
    if (*p) cudaFreeHost(*p);
    *p = nullptr;
    *have = 0;
    ODX_CUDA(cudaMallocHost(p, need));
    *have = need;
    return ODX_OK;
}

inline size_t al256(size_t v) { return (v + 255) & ~size_t(255); }

// Host memcpy of the staging path split over a small persistent worker pool
// (one core copies ~15-20 GB/s; the trajectory is MBs).  After a job the
// workers spin for a short while (back-to-back solves find them awake, no
// futex wake-up on the critical path), then sleep on a condition variable.
// ODX_HOST_THREADS sets the pool size (default: 8, at most half the cores;
// 0 or 1 = plain memcpy).
// Copy with non-temporal stores: the destination (pinned staging the DMA
// engine reads next, or the caller's result) does not linger dirty in this
// core's caches, so the device's reads of it need no cross-core snoops.
inline void nt_copy(char* dst, const char* src, size_t n) {
    size_t i = 0;
    if (((reinterpret_cast<size_t>(dst) | reinterpret_cast<size_t>(src)) & 15) == 0) {
        for (; i + 64 <= n; i += 64) {
            const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
            const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
            const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
            const __m128i d = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
            _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), d);
        }
        _mm_sfence();
    }
    if (i < n) std::memcpy(dst + i, src + i, n - i);
}

class CopyPool {
  public:
    static CopyPool& get() {
        // intentionally never destroyed: its threads simply end with the process
        static CopyPool* pool = new CopyPool();
        return *pool;
    }
    void copy(void* dst, const void* src, size_t n) {
        // a forked child has no worker threads (fork copies only the caller)
        int T = forked_.load(std::memory_order_relaxed) ? 0 : (int)workers_.size();
        const int act = active_.load(std::memory_order_relaxed) - 1;  // the caller copies too
        if (act < T) T = act < 0 ? 0 : act;
        if (T == 0 || n < (size_t(1) << 18)) {
            nt_copy(static_cast<char*>(dst), static_cast<const char*>(src), n);
            return;
        }
        const int parts = T + 1;
        const size_t chunk = ((n + parts - 1) / parts + 63) & ~size_t(63);
        dst_ = static_cast<char*>(dst);
        src_ = static_cast<const char*>(src);
        n_ = n;
        chunk_ = chunk;
        used_ = T;
        pending_.store(T, std::memory_order_relaxed);
        gen_.fetch_add(1, std::memory_order_seq_cst);  // publishes the job (release)
        if (sleepers_.load(std::memory_order_seq_cst) > 0) {
            std::lock_guard<std::mutex> lk(mu_);
            cv_.notify_all();
        }
        const size_t lo = (size_t)T * chunk;  // the caller copies the last part
        if (lo < n) nt_copy(dst_ + lo, src_ + lo, n - lo);
        while (pending_.load(std::memory_order_acquire) != 0) _mm_pause();
    }

    // threads.max_threads / set_threads (threads.py:17-32): the pool size is
    // fixed at first use; set_threads clamps into [1, max] and returns it
    int max_threads() const { return (int)workers_.size() + 1; }
    int set_threads(int n) {
        const int used = n < 1 ? 1 : (n > max_threads() ? max_threads() : n);
        active_.store(used, std::memory_order_relaxed);
        return used;
    }

  private:
    CopyPool() {
        pthread_atfork(nullptr, nullptr, [] { get().forked_.store(true); });
        const char* e = std::getenv("ODX_HOST_THREADS");
        const int hw = (int)std::thread::hardware_concurrency();
        int t = e ? std::atoi(e) : std::min(8, std::max(1, hw / 2));
        if (t > 1)
            for (int i = 0; i < t - 1; i++) workers_.emplace_back([this, i] { run(i); });
    }
    void run(int i) {
        unsigned long long seen = 0;
        while (true) {
            // spin ~0.5 ms for the next job, then sleep
            bool got = false;
            for (int k = 0; k < 20000 && !got; k++) {
                if (gen_.load(std::memory_order_acquire) != seen) got = true;
                else _mm_pause();
            }
            if (!got) {
                std::unique_lock<std::mutex> lk(mu_);
                sleepers_.fetch_add(1, std::memory_order_seq_cst);
                cv_.wait(lk, [&] { return gen_.load(std::memory_order_seq_cst) != seen; });
                sleepers_.fetch_sub(1, std::memory_order_relaxed);
            }
            seen = gen_.load(std::memory_order_acquire);
            if (i >= used_) continue;  // set_threads() left this worker out of the job
            const size_t lo = (size_t)i * chunk_;
            if (lo < n_) nt_copy(dst_ + lo, src_ + lo, (lo + chunk_ < n_ ? chunk_ : n_ - lo));
            pending_.fetch_sub(1, std::memory_order_release);
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::atomic<unsigned long long> gen_{0};
    std::atomic<int> sleepers_{0};
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t n_ = 0, chunk_ = 0;
    std::atomic<int> pending_{0};
    std::atomic<int> active_{1 << 20};
    int used_ = 0;
    std::atomic<bool> forked_{false};
};

// page-locked (cudaHostAlloc / registered) host memory can be a DMA endpoint
bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        (void)cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

}  // namespace
}  // namespace odx

extern "C" int odx_host_threads_max(void) { return odx::CopyPool::get().max_threads(); }
extern "C" int odx_set_host_threads(int n) { return odx::CopyPool::get().set_threads(n); }

extern "C" int odx_solve_host(const odx_problem* P, const odx_stepper* S, const double* x0,
                              const double* X_guess, double* X_out, int64_t B, int64_t N,
                              double dt, const odx_newton_cfg* C, double* hist,
                              double* scaled_hist, int32_t* iters, int32_t* status,
                              int64_t* status_index, void* stream) {
    using namespace odx;
    if (!P || !S || !C || !x0 || !X_guess || !X_out || !iters || !status || !status_index)
        return fail(ODX_EINVAL, "null host buffer");
    if (B < 1 || N < 1) return fail(ODX_EINVAL, "B and N must be >= 1");
    if (C->max_iters < 0) return fail(ODX_EINVAL, "max_iters must be >= 0");
    const int64_t d = P->dim;
    if (d < 1) return fail(ODX_EINVAL, "bad state dimension");
    // (invalid descriptors make the query return 0; odx_solve then reports them)
    size_t wsb = odx_solve_workspace_bytes(P, S, B, N, C);
    if (wsb < 256) wsb = 256;
    const int64_t H = (int64_t)C->max_iters + 1;
    const size_t nx0 = (size_t)(B * d) * 8, nX = (size_t)(B * N * d) * 8;
    const size_t o_X = al256(nx0), o_out = o_X + al256(nX);
    const size_t o_sh = (size_t)(B * H) * 8, o_sidx = 2 * o_sh, o_it = o_sidx + (size_t)B * 8,
                 o_st = o_it + (size_t)B * 4, out_bytes = o_st + (size_t)B * 4;
    int dev = 0;
    ODX_CUDA(cudaGetDevice(&dev));
    cudaStream_t st = (cudaStream_t)stream;

    std::lock_guard<std::mutex> lock(g_host_mu);
    if ((int)g_host_cache.size() <= dev) g_host_cache.resize(dev + 1);
    HostCache& hc = g_host_cache[dev];
    int rc;
    if ((rc = grow_device(&hc.dregion, &hc.dbytes, o_out + out_bytes))) return rc;
    if ((rc = grow_device(&hc.ws, &hc.wsbytes, wsb))) return rc;
    if ((rc = grow_pinned(&hc.pin_in, &hc.in_bytes, o_X + nX))) return rc;
    if ((rc = grow_pinned(&hc.pin_out, &hc.out_bytes, (o_out - o_X) + out_bytes))) return rc;

    static const bool timing = std::getenv("ODX_HOST_TIMING") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto t0 = now();
    char* din = static_cast<char*>(hc.dregion);
    char* pin = static_cast<char*>(hc.pin_in);
    char* pout = static_cast<char*>(hc.pin_out);
    // pinned caller buffers are DMA'd directly; pageable ones go through
    // the cached staging blocks
    const bool in_pinned = is_pinned(X_guess), out_pinned = is_pinned(X_out);
    std::memcpy(pin, x0, nx0);

    // ---- pipelined batch chunks (independent resident trajectories) ----------
    static const bool no_pipe = std::getenv("ODX_HOST_PIPELINE") &&
                                std::getenv("ODX_HOST_PIPELINE")[0] == '0';
    if (!no_pipe && B >= 64 && nX >= (size_t(32) << 20) && d <= 4 && N <= resident_max_steps((int)d)) {
        const int K = HostCache::MAXC;
        const int64_t Bc = (B + K - 1) / K;
        size_t wsc = odx_solve_workspace_bytes(P, S, Bc, N, C);
        wsc = al256(wsc < 256 ? 256 : wsc);
        if ((rc = grow_device(&hc.ws, &hc.wsbytes, wsc * K))) return rc;
        if (!hc.fork) {
            ODX_CUDA(cudaEventCreateWithFlags(&hc.fork, cudaEventDisableTiming));
            for (int k = 0; k < K; k++) {
                ODX_CUDA(cudaStreamCreateWithFlags(&hc.cs[k], cudaStreamNonBlocking));
                ODX_CUDA(cudaEventCreateWithFlags(&hc.ce[k], cudaEventDisableTiming));
            }
        }
        char* dout = din + o_out;
        ODX_CUDA(cudaMemcpyAsync(din, pin, nx0, cudaMemcpyHostToDevice, st));
        ODX_CUDA(cudaEventRecord(hc.fork, st));
        const size_t row = (size_t)(N * d) * 8;  // bytes of one trajectory
        for (int k = 0; k < K; k++) {
            const int64_t b0 = (int64_t)k * Bc;
            if (b0 >= B) break;
            const int64_t bn = (b0 + Bc <= B) ? Bc : B - b0;
            const size_t off = (size_t)b0 * row, len = (size_t)bn * row;
            cudaStream_t sk = hc.cs[k];
            ODX_CUDA(cudaStreamWaitEvent(sk, hc.fork, 0));
            const char* src = reinterpret_cast<const char*>(X_guess) + off;
            if (!in_pinned) {
                CopyPool::get().copy(pin + o_X + off, src, len);
                src = pin + o_X + off;
            }
            ODX_CUDA(cudaMemcpyAsync(din + o_X + off, src, len, cudaMemcpyHostToDevice, sk));
            rc = odx_solve(P, S, reinterpret_cast<const double*>(din) + b0 * d,
                           reinterpret_cast<double*>(din + o_X + off), bn, N, dt, C,
                           reinterpret_cast<double*>(dout) + b0 * H,
                           reinterpret_cast<double*>(dout + o_sh) + b0 * H,
                           reinterpret_cast<int32_t*>(dout + o_it) + b0,
                           reinterpret_cast<int32_t*>(dout + o_st) + b0,
                           reinterpret_cast<int64_t*>(dout + o_sidx) + b0,
                           static_cast<char*>(hc.ws) + (size_t)k * wsc, wsc, (void*)sk);
            if (rc) return rc;
            char* dst = out_pinned ? reinterpret_cast<char*>(X_out) + off : pout + off;
            ODX_CUDA(cudaMemcpyAsync(dst, din + o_X + off, len, cudaMemcpyDeviceToHost, sk));
            ODX_CUDA(cudaEventRecord(hc.ce[k], sk));
            ODX_CUDA(cudaStreamWaitEvent(st, hc.ce[k], 0));
        }
        ODX_CUDA(cudaMemcpyAsync(pout + (o_out - o_X), din + o_out, out_bytes, cudaMemcpyDeviceToHost, st));
        auto t4 = now();
        ODX_CUDA(cudaStreamSynchronize(st));
        auto t5 = now();
        if (!out_pinned) CopyPool::get().copy(X_out, pout, nX);
        if (timing) {
            auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
            std::fprintf(stderr, "odx_solve_host (pipelined x%d) us: enqueue+pack %.1f sync %.1f unpack %.1f\n", K,
                         us(t0, t4), us(t4, t5), us(t5, now()));
        }
    } else {

    if (!in_pinned) CopyPool::get().copy(pin + o_X, X_guess, nX);
    auto t1 = now();
    if (in_pinned) {
        ODX_CUDA(cudaMemcpyAsync(din, pin, nx0, cudaMemcpyHostToDevice, st));
        ODX_CUDA(cudaMemcpyAsync(din + o_X, X_guess, nX, cudaMemcpyHostToDevice, st));
    } else {
        ODX_CUDA(cudaMemcpyAsync(din, pin, o_X + nX, cudaMemcpyHostToDevice, st));
    }
    auto t2 = now();
    char* dout = din + o_out;
    rc = odx_solve(P, S, reinterpret_cast<const double*>(din), reinterpret_cast<double*>(din + o_X),
                   B, N, dt, C, reinterpret_cast<double*>(dout),
                   reinterpret_cast<double*>(dout + o_sh), reinterpret_cast<int32_t*>(dout + o_it),
                   reinterpret_cast<int32_t*>(dout + o_st), reinterpret_cast<int64_t*>(dout + o_sidx),
                   hc.ws, hc.wsbytes, stream);
    if (rc) return rc;
    auto t3 = now();
    if (out_pinned) {
        ODX_CUDA(cudaMemcpyAsync(X_out, din + o_X, nX, cudaMemcpyDeviceToHost, st));
        ODX_CUDA(cudaMemcpyAsync(pout + (o_out - o_X), din + o_out, out_bytes,
                                 cudaMemcpyDeviceToHost, st));
    } else {
        ODX_CUDA(cudaMemcpyAsync(pout, din + o_X, (o_out - o_X) + out_bytes,
                                 cudaMemcpyDeviceToHost, st));
    }
    auto t4 = now();
    ODX_CUDA(cudaStreamSynchronize(st));
    auto t5 = now();

    if (!out_pinned) CopyPool::get().copy(X_out, pout, nX);
    if (timing) {
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        std::fprintf(stderr, "odx_solve_host us: pack %.1f h2d-enq %.1f solve-enq %.1f d2h-enq %.1f sync %.1f unpack %.1f\n",
                     us(t0, t1), us(t1, t2), us(t2, t3), us(t3, t4), us(t4, t5), us(t5, now()));
    }
    }
    const char* ob = pout + (o_out - o_X);
    std::memcpy(status_index, ob + o_sidx, (size_t)B * 8);
    std::memcpy(iters, ob + o_it, (size_t)B * 4);
    std::memcpy(status, ob + o_st, (size_t)B * 4);
    // history entries past the iterations run are not written by the device
    // loop: report them as NaN (a singular block stops before recording)
    const double qnan = std::nan("");
    for (int64_t b = 0; b < B; b++) {
        const int64_t last = (status[b] == ODX_ST_SINGULAR) ? (int64_t)iters[b] - 1 : iters[b];
        const double* hs = reinterpret_cast<const double*>(ob) + b * H;
        const double* ss = reinterpret_cast<const double*>(ob + o_sh) + b * H;
        for (int64_t i = 0; i < H; i++) {
            if (hist) hist[b * H + i] = (i <= last) ? hs[i] : qnan;
            if (scaled_hist) scaled_hist[b * H + i] = (i <= last) ? ss[i] : qnan;
        }
    }
    return ODX_OK;
}
