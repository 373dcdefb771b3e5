// host_util.cu — host helpers shared by every translation unit: error
// reporting, device-property cache, launch counter, descriptor conversion.
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "common.cuh"

namespace odx {

thread_local std::string g_err;


void set_error(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
}

thread_local const char* g_route = "";
void set_route(const char* route) { g_route = route; }

std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int num_sms() {
    static std::mutex mu;
    static std::unordered_map<int, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
    cache[dev] = n;
    return n;
}

bool fill_params(const odx_problem* P, ProbParams& pp) {
    if (!P || P->n_params < 0 || P->n_params > ODX_MAX_PARAMS) return false;
    std::memset(&pp, 0, sizeof(pp));
    for (int i = 0; i < P->n_params; i++) pp.p[i] = P->params[i];
    return true;
}

bool fill_coefs(const odx_stepper* S, double dt, StepCoefs& sc) {
    if (!S) return false;
    std::memset(&sc, 0, sizeof(sc));
    sc.dt = dt;
    if (S->kind == ODX_STEP_EXPLICIT_RK) {
        const int s = S->stages;
        if (s < 1 || s > ODX_MAX_STAGES) return false;
        for (int i = 0; i < s; i++) {
            for (int j = 0; j < s; j++) {
                if (j >= i && S->a[i * s + j] != 0.0) return false;  // explicit only
                sc.dta[i * s + j] = dt * S->a[i * s + j];
            }
            sc.b[i] = S->b[i];
        }
        sc.stages = s;
        return true;
    }
    if (S->kind == ODX_STEP_IMPLICIT_WEIGHTED) {
        sc.w_prev = S->w_prev;
        sc.w_next = S->w_next;
        sc.dt_wprev = dt * S->w_prev;
        sc.dt_wnext = dt * S->w_next;
        sc.stages = 1;
        return true;
    }
    return false;
}

}  // namespace odx

namespace odx {
int kernel_occupancy(const void* kern, int threads, size_t smem, int* per_sm) {
    struct Key {
        const void* k;
        int t, dev;
        size_t s;
        bool operator==(const Key& o) const { return k == o.k && t == o.t && dev == o.dev && s == o.s; }
    };
    struct Hash {
        size_t operator()(const Key& q) const {
            return std::hash<const void*>()(q.k) ^ (size_t(q.t) << 20) ^ (q.s << 1) ^ size_t(q.dev);
        }
    };
    static std::mutex mu;
    static std::unordered_map<Key, int, Hash> cache;
    int dev = 0;
    ODX_CUDA(cudaGetDevice(&dev));
    const Key key{kern, threads, dev, smem};
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find(key);
        if (it != cache.end()) {
            *per_sm = it->second;
            return ODX_OK;
        }
    }
    ODX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int v = 0;
    ODX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, threads, smem));
    std::lock_guard<std::mutex> lock(mu);
    cache[key] = v;
    *per_sm = v;
    return ODX_OK;
}
}  // namespace odx
