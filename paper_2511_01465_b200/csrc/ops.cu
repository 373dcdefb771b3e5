// ops.cu — piecewise device ops mirroring the reference's compiled loops one to
// one (used for parity bisection and by callers that drive their own loop):
//   build_explicit (_kernels.py:299-342), build_implicit (:393-464),
//   scan_affine (:116-233, here single-pass decoupled look-back with full
//   (F, c) inclusive prefixes), max_abs (:84-95), add_inplace (:98-103).
#include <climits>

#include "common.cuh"
#include "dispatch.cuh"
#include "scan.cuh"

namespace odx {

__global__ void init_bad_slots_kernel(unsigned long long* red, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) red[4 * i + 3] = ~0ull;
}

// Zero `words` 8-byte words at base, except the "bad" slot (4th) of each of
// the first n reduction quads, which starts at all-ones: one launch instead of
// a memset plus init_bad_slots.
__global__ void init_ws_kernel(unsigned long long* base, long long words, int n) {
    for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < words;
         w += (long long)gridDim.x * blockDim.x)
        base[w] = (w < 4LL * n && (w & 3) == 3) ? ~0ull : 0ull;
}

void init_ws(void* base, size_t bytes, int n, cudaStream_t st) {
    const long long words = (long long)((bytes + 7) / 8);
    long long blocks = (words + 255) / 256;
    if (blocks > 4LL * num_sms()) blocks = 4LL * num_sms();
    if (blocks < 1) blocks = 1;
    init_ws_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<unsigned long long*>(base),
                                                      words, n);
}

void init_bad_slots(unsigned long long* red, int n, cudaStream_t st) {
    init_bad_slots_kernel<<<(n + 127) / 128, 128, 0, st>>>(red, n);
}

// ---------------------------------------------------------------------------
// scan_affine op: single-pass decoupled look-back over given elements, full
// inclusive prefixes (F and c) since element 0 need not have F = 0 here.
// ---------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ void lookback_full(long long t, const Elem<D>& A, uint32_t* flags,
                                              double* aggbuf, double* inclbuf, Elem<D>& Pex,
                                              bool& Pex_has, int lane) {
    constexpr int E = D * D + D;
    const uint32_t epoch = 1u;
    if (t == 0) {
        if (lane == 0) {
            double* dst = inclbuf;
#pragma unroll
            for (int i = 0; i < D * D; i++) dst[i] = A.F[i];
#pragma unroll
            for (int i = 0; i < D; i++) dst[D * D + i] = A.c[i];
            st_release_u32(flags, lb_flag(epoch, LB_INCL));
        }
        Pex_has = false;
        __syncwarp();
        return;
    }
    if (lane == 0) {
        double* dst = aggbuf + t * E;
#pragma unroll
        for (int i = 0; i < D * D; i++) dst[i] = A.F[i];
#pragma unroll
        for (int i = 0; i < D; i++) dst[D * D + i] = A.c[i];
        st_release_u32(flags + t, lb_flag(epoch, LB_AGG));
    }
    Elem<D> R;
    bool R_has = false;
    long long pos = t - 1;
    while (true) {
        long long j = pos - lane;
        uint32_t kind = (j >= 0) ? lb_wait(flags, j, epoch) : LB_INCL;
        unsigned incl_mask = __ballot_sync(FULL, kind == LB_INCL);
        int first = incl_mask ? (__ffs(incl_mask) - 1) : 32;
        Elem<D> e;
        bool has = lane <= first && j >= 0;
        if (has) {
            const double* src = (lane < first ? aggbuf : inclbuf) + j * E;
#pragma unroll
            for (int i = 0; i < D * D; i++) e.F[i] = __ldcg(src + i);
#pragma unroll
            for (int i = 0; i < D; i++) e.c[i] = __ldcg(src + D * D + i);
        } else {
            set_identity<D>(e);
        }
        warp_reduce_latest_first<D>(e, has, lane);
        if (lane == 0 && has) {
            if (R_has)
                compose<D>(e, R, R);
            else {
                R = e;
                R_has = true;
            }
        }
        if (first < 32) break;
        pos -= 32;
    }
    if (lane == 0) {
        Elem<D> incl;
        compose<D>(R, A, incl);
        double* dst = inclbuf + t * E;
#pragma unroll
        for (int i = 0; i < D * D; i++) dst[i] = incl.F[i];
#pragma unroll
        for (int i = 0; i < D; i++) dst[D * D + i] = incl.c[i];
        st_release_u32(flags + t, lb_flag(epoch, LB_INCL));
        Pex = R;
    }
    Pex_has = true;
    __syncwarp();
}

template <int D, int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS)
scan_op_kernel(const double* __restrict__ Fin, const double* __restrict__ cin, long long N,
               double* __restrict__ Fp, double* __restrict__ cp, uint32_t* ctr, uint32_t* flags,
               double* aggbuf, double* inclbuf) {
    constexpr int NW = THREADS / 32;
    constexpr int T = THREADS * ITEMS;
    __shared__ double wtF[NW][D * D], wtc[NW][D];
    __shared__ int wthas[NW];
    __shared__ double PF[D * D], Pc[D];
    __shared__ int Phas;
    __shared__ long long tile_s;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) tile_s = (long long)atomicAdd(ctr, 1u);
    __syncthreads();
    const long long t = tile_s;
    const long long base = t * T;
    Elem<D> el[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        long long k = base + tid * ITEMS + i;
        if (k < N) {
#pragma unroll
            for (int q = 0; q < D * D; q++) el[i].F[q] = Fin[k * D * D + q];
#pragma unroll
            for (int q = 0; q < D; q++) el[i].c[q] = cin[k * D + q];
        }
    }
    Elem<D> agg;
    bool has = false;
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        if (base + tid * ITEMS + i < N) {
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
    if (lane == 31) {
#pragma unroll
        for (int i = 0; i < D * D; i++) wtF[w][i] = agg.F[i];
#pragma unroll
        for (int i = 0; i < D; i++) wtc[w][i] = agg.c[i];
        wthas[w] = has;
    }
    __syncthreads();
    if (w == 0) {
        Elem<D> A;
        bool A_has = false;
        if (lane == 0) {
            for (int q = 0; q < NW; q++) {
                if (!wthas[q]) continue;
                Elem<D> e;
#pragma unroll
                for (int i = 0; i < D * D; i++) e.F[i] = wtF[q][i];
#pragma unroll
                for (int i = 0; i < D; i++) e.c[i] = wtc[q][i];
                if (A_has)
                    compose<D>(A, e, A);
                else {
                    A = e;
                    A_has = true;
                }
            }
        }
        Elem<D> Pex;
        bool Pex_has = false;
        lookback_full<D>(t, A, flags, aggbuf, inclbuf, Pex, Pex_has, lane);
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < D * D; i++) PF[i] = Pex.F[i];
#pragma unroll
            for (int i = 0; i < D; i++) Pc[i] = Pex.c[i];
            Phas = Pex_has;
        }
    }
    __syncthreads();
    Elem<D> Z;
    bool zh = Phas != 0;
    if (zh) {
#pragma unroll
        for (int i = 0; i < D * D; i++) Z.F[i] = PF[i];
#pragma unroll
        for (int i = 0; i < D; i++) Z.c[i] = Pc[i];
    }
    for (int q = 0; q < w; q++) {
        if (!wthas[q]) continue;
        Elem<D> e;
#pragma unroll
        for (int i = 0; i < D * D; i++) e.F[i] = wtF[q][i];
#pragma unroll
        for (int i = 0; i < D; i++) e.c[i] = wtc[q][i];
        if (zh)
            compose<D>(Z, e, Z);
        else {
            Z = e;
            zh = true;
        }
    }
    Elem<D> ex;
    shfl_up_elem<D>(agg, ex, 1);
    bool exh = __shfl_up_sync(FULL, has, 1) && lane > 0;
    if (exh) {
        if (zh)
            compose<D>(Z, ex, Z);
        else {
            Z = ex;
            zh = true;
        }
    }
#pragma unroll
    for (int i = 0; i < ITEMS; i++) {
        long long k = base + tid * ITEMS + i;
        if (k < N) {
            if (zh)
                compose<D>(Z, el[i], Z);
            else {
                Z = el[i];
                zh = true;
            }
            if (Fp) {
#pragma unroll
                for (int q = 0; q < D * D; q++) Fp[k * D * D + q] = Z.F[q];
            }
#pragma unroll
            for (int q = 0; q < D; q++) cp[k * D + q] = Z.c[q];
        }
    }
}

static constexpr int SCAN_THREADS = 128, SCAN_ITEMS = 2;

size_t scan_op_ws(long long N, int d) {
    const long long T = SCAN_THREADS * SCAN_ITEMS;
    const long long nt = (N + T - 1) / T;
    return align_up(8 + (size_t)nt * 4, 256) + 2 * (size_t)nt * (d * d + d) * 8 + 512;
}

template <int D>
int scan_op_d(const double* F, const double* c, long long N, double* Fp, double* cp, void* ws,
              cudaStream_t st) {
    const long long T = SCAN_THREADS * SCAN_ITEMS;
    const long long nt = (N + T - 1) / T;
    char* base = reinterpret_cast<char*>(align_up(reinterpret_cast<size_t>(ws), 256));
    uint32_t* ctr = reinterpret_cast<uint32_t*>(base);
    uint32_t* flags = ctr + 2;
    size_t off = align_up(8 + (size_t)nt * 4, 256);
    double* aggbuf = reinterpret_cast<double*>(base + off);
    double* inclbuf = aggbuf + nt * (D * D + D);
    ODX_CUDA(cudaMemsetAsync(base, 0, 8 + (size_t)nt * 4, st));
    scan_op_kernel<D, SCAN_THREADS, SCAN_ITEMS><<<(unsigned)nt, SCAN_THREADS, 0, st>>>(
        F, c, N, Fp, cp, ctr, flags, aggbuf, inclbuf);
    ODX_CUDA(cudaGetLastError());
    count_launch(1);
    return ODX_OK;
}

int scan_op(const double* F, const double* c, long long N, int d, double* Fp, double* cp,
            void* ws, size_t ws_bytes, cudaStream_t st) {
    if (N <= 0) return ODX_OK;
    if (ws == nullptr || ws_bytes < scan_op_ws(N, d))
        return fail(ODX_EWORKSPACE, "scan_affine workspace too small");
    switch (d) {
    case 1: return scan_op_d<1>(F, c, N, Fp, cp, ws, st);
    case 2: return scan_op_d<2>(F, c, N, Fp, cp, ws, st);
    case 3: return scan_op_d<3>(F, c, N, Fp, cp, ws, st);
    case 4: return scan_op_d<4>(F, c, N, Fp, cp, ws, st);
    default: return fail(ODX_EUNSUPPORTED, "scan_affine op supports d <= 4 (d=64: dense path)");
    }
}

// ---------------------------------------------------------------------------
// max_abs / add_inplace
// ---------------------------------------------------------------------------
__global__ void max_abs_kernel(const double* __restrict__ A, long long n, int d,
                               unsigned long long* out) {
    double acc = 0.0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double loc = 0.0;
        for (int j = 0; j < d; j++) {
            double v = fabs(A[i * d + j]);
            if (!(v <= loc)) loc = v;
        }
        acc = fmax(acc, loc);
    }
    acc = warp_max_nan_drop(acc);
    __shared__ double sm[32];
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int q = 0; q < (int)(blockDim.x >> 5); q++) a = fmax(a, sm[q]);
        if (a > 0.0) atomicMax(out, dbits(a));
    }
}

int max_abs_op(const double* A, long long n, int d, double* out, cudaStream_t st) {
    ODX_CUDA(cudaMemsetAsync(out, 0, sizeof(double), st));
    if (n <= 0) return ODX_OK;
    long long blocks = (n + 255) / 256;
    if (blocks > 4LL * num_sms()) blocks = 4LL * num_sms();
    max_abs_kernel<<<(unsigned)blocks, 256, 0, st>>>(A, n, d,
                                                     reinterpret_cast<unsigned long long*>(out));
    ODX_CUDA(cudaGetLastError());
    count_launch(1);
    return ODX_OK;
}

__global__ void add_kernel(double* __restrict__ X, const double* __restrict__ U, long long m) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += (long long)gridDim.x * blockDim.x)
        X[i] += U[i];
}

int add_op(double* X, const double* U, long long n, int d, cudaStream_t st) {
    const long long m = n * d;
    if (m <= 0) return ODX_OK;
    long long blocks = (m + 255) / 256;
    if (blocks > 8LL * num_sms()) blocks = 8LL * num_sms();
    add_kernel<<<(unsigned)blocks, 256, 0, st>>>(X, U, m);
    ODX_CUDA(cudaGetLastError());
    count_launch(1);
    return ODX_OK;
}

}  // namespace odx
