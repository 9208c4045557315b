// runtime.cu — library plumbing plus the small data-model kernels:
// A1 row norms, f64 column mean, medoid, frontier top-k decode.
#include <cstdarg>
#include <cstring>
#include "common.cuh"
#include <map>
#include <mutex>
#include "runtime.cuh"

namespace jb {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int grow_smem_attr(const void* func, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> set;
    int dev = 0;
    JB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    int& cur = set[{func, dev}];
    if (cur < bytes) {
        JB_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        cur = bytes;
    }
    return JB_OK;
}

int sm_count_current() {
    static thread_local int cached_dev = -1, cached_n = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cached_n;
    if (dev != cached_dev) {
        cudaDeviceGetAttribute(&cached_n, cudaDevAttrMultiProcessorCount, dev);
        cached_dev = dev;
    }
    return cached_n;
}

void retain_pool_memory() {
    static thread_local int done_dev = -1;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done_dev = dev;
}

// ---- row norms (search.py:101, 113; build.py:120) ----------------------
__global__ void row_sq_norms_kernel(const float* __restrict__ x, int64_t n, int D, float* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* r = x + i * D;
    out[i] = a1_dot<false>(r, r, D);
}

// ---- f64 column sum, sequential over rows (numpy mean(axis=0), A3) ------
// numpy reduces axis 0 of a C-contiguous array row by row (acc[:] += row), so
// each column's f64 sum is one sequential chain over the rows and the result
// is bit-exact only in that order. The chain cannot be split; what limits it is
// feeding it. One block per group of 8 columns (one 32 B sector per row): warps
// 1..8 stream tiles of CS_ROWS rows x 8 columns into smem (double-buffered) while
// lanes 0..7 of warp 0 run the 8 chains from smem. (A single block of one thread
// per column, loading its own operands, ran at ~4 GB/s: 84 ms of a 1M x 128
// build; now the chains' DADD latency is the bound.)
constexpr int CS_ROWS = 512;
constexpr int CS_LOADERS = 256;                 // warps 1..8: 16 loads in flight per thread per tile
constexpr int CS_THREADS = 32 + CS_LOADERS;
constexpr int CS_PER = CS_ROWS * 8 / CS_LOADERS;

__global__ void __launch_bounds__(CS_THREADS)
column_sum_f64_kernel(const float* __restrict__ x, int64_t n, int D, double* __restrict__ out) {
    __shared__ float tile[2][CS_ROWS][8];
    const int c0 = blockIdx.x * 8;
    const int nc = min(8, D - c0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntiles = (n + CS_ROWS - 1) / CS_ROWS;
    auto fill = [&](int64_t t, int buf) {  // all loads issued before any store
        const int64_t r0 = t * CS_ROWS;
        const int rows = (int)(n - r0 < CS_ROWS ? n - r0 : CS_ROWS);
        const int t0 = threadIdx.x - 32;
        float v[CS_PER];
#pragma unroll
        for (int u = 0; u < CS_PER; ++u) {
            const int idx = t0 + u * CS_LOADERS, r = idx >> 3, j = idx & 7;
            v[u] = (r < rows && j < nc) ? __ldg(x + (r0 + r) * D + c0 + j) : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < CS_PER; ++u) {
            const int idx = t0 + u * CS_LOADERS;
            tile[buf][idx >> 3][idx & 7] = v[u];
        }
    };
    if (warp > 0 && ntiles > 0) fill(0, 0);
    __syncthreads();
    double s = 0.0;
    for (int64_t t = 0; t < ntiles; ++t) {
        const int buf = (int)(t & 1);
        if (warp > 0) {
            if (t + 1 < ntiles) fill(t + 1, buf ^ 1);
        } else if (lane < nc) {
            const int rows = (int)(n - t * CS_ROWS < CS_ROWS ? n - t * CS_ROWS : CS_ROWS);
            int r = 0;
            for (; r + 16 <= rows; r += 16) {
                float v[16];
#pragma unroll
                for (int u = 0; u < 16; ++u) v[u] = tile[buf][r + u][lane];
#pragma unroll
                for (int u = 0; u < 16; ++u) s = __dadd_rn(s, (double)v[u]);
            }
            for (; r < rows; ++r) s = __dadd_rn(s, (double)tile[buf][r][lane]);
        }
        __syncthreads();
    }
    if (warp == 0 && lane < nc) out[c0 + lane] = s;
}

__global__ void mean_finish_kernel(const double* __restrict__ sum, int64_t n, int D, double* __restrict__ mean64,
                                   float* __restrict__ mean32) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= D) return;
    double m = __ddiv_rn(sum[c], (double)n);
    if (mean64) mean64[c] = m;
    if (mean32) mean32[c] = __double2float_rn(m);
}

// medoid distance: diff = f64(x) - center; einsum('nd,nd->n') f64 2-lane order
// (graph.py:167-171), then argmin with the lowest id on ties.
__device__ __forceinline__ double medoid_dist(const float* __restrict__ r, const double* __restrict__ c, int D) {
    Acc2d acc; acc.zero();
    int e = 0;
    for (; e + 8 <= D; e += 8) {
#pragma unroll
        for (int i = 3; i >= 0; --i) {
            double d0 = __dsub_rn((double)r[e + 2 * i], c[e + 2 * i]);
            double d1 = __dsub_rn((double)r[e + 2 * i + 1], c[e + 2 * i + 1]);
            acc.l0 = __dadd_rn(__dmul_rn(d0, d0), acc.l0);
            acc.l1 = __dadd_rn(__dmul_rn(d1, d1), acc.l1);
        }
    }
    for (; e < D; ++e) {
        double d0 = __dsub_rn((double)r[e], c[e]);
        if (e & 1) acc.l1 = __dadd_rn(__dmul_rn(d0, d0), acc.l1);
        else acc.l0 = __dadd_rn(__dmul_rn(d0, d0), acc.l0);
    }
    return acc.reduce();
}

struct DI { double d; int64_t i; };
__device__ __forceinline__ DI di_min(DI a, DI b) {
    if (b.d < a.d || (b.d == a.d && b.i < a.i)) return b;
    return a;
}

__global__ void medoid_partial_kernel(const float* __restrict__ x, int64_t n, int D, const double* __restrict__ center,
                                      DI* __restrict__ partial) {
    extern __shared__ double csh[];
    for (int c = threadIdx.x; c < D; c += blockDim.x) csh[c] = center[c];
    __syncthreads();
    DI best{__longlong_as_double(0x7FF0000000000000ll), INT64_MAX};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        DI cur{medoid_dist(x + i * D, csh, D), i};
        best = di_min(best, cur);
    }
    // warp reduce then block reduce
    for (int o = 16; o > 0; o >>= 1) {
        DI other{__shfl_down_sync(0xFFFFFFFFu, best.d, o), __shfl_down_sync(0xFFFFFFFFu, best.i, o)};
        best = di_min(best, other);
    }
    __shared__ DI wbest[32];
    if ((threadIdx.x & 31) == 0) wbest[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        DI b = wbest[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) b = di_min(b, wbest[w]);
        partial[blockIdx.x] = b;
    }
}

__global__ void medoid_final_kernel(const DI* __restrict__ partial, int np, int64_t* __restrict__ out) {
    DI b{__longlong_as_double(0x7FF0000000000000ll), INT64_MAX};
    for (int i = 0; i < np; ++i) b = di_min(b, partial[i]);
    *out = b.i;
}

// ---- frontier -> top-k (search.py:375-382, exact source) -----------------
__global__ void frontier_topk_kernel(const uint64_t* __restrict__ keys, int64_t nq, int L, int k,
                                     int32_t* __restrict__ ids, double* __restrict__ dists, bool integer) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nq * k) return;
    int64_t q = t / k;
    int j = (int)(t % k);
    uint64_t key = keys[q * L + j];
    if (key == UMAX) {
        ids[t] = -1;
        dists[t] = __longlong_as_double(0x7FF0000000000000ll);
    } else {
        ids[t] = (int32_t)(key & 0xFFFFFFFFull);
        const uint32_t w = (uint32_t)(key >> 32);
        dists[t] = integer ? (double)w : (double)__uint_as_float(w);  // _decode_keys (search.py:148-153)
    }
}

// u8 rows: integer norms sum(x*x) (row_sq_norms, core.py:162-166) and exact f32 copies
__global__ void row_sq_norms_u8_kernel(const uint8_t* __restrict__ x, int64_t n, int D, uint32_t* __restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint8_t* r = x + i * D;
    uint32_t s = 0;
    for (int e = 0; e < D; ++e) s += (uint32_t)r[e] * (uint32_t)r[e];
    out[i] = s;
}

__global__ void u8_to_f32_kernel(const uint8_t* __restrict__ x, int64_t count, float* __restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (float)x[i];
}

}  // namespace jb

using namespace jb;

extern "C" {

const char* jb_last_error(void) { return g_err; }
int jb_abi_version(void) { return 1; }

int jb_sm_count(int device, int32_t* out) {
    int n = 0;
    JB_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device));
    *out = n;
    return JB_OK;
}

int jb_row_sq_norms(const float* x, int64_t n, int32_t dims, float* out, void* stream) {
    JB_CHECK_ARG(dims >= 1 && n >= 0, "jb_row_sq_norms: bad shape");
    if (n == 0) return JB_OK;
    int threads = 256;
    row_sq_norms_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, as_stream(stream)>>>(x, n, dims, out);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

int jb_column_mean_f32(const float* x, int64_t n, int32_t dims, float* out, void* stream) {
    JB_CHECK_ARG(dims >= 1 && n >= 1, "jb_column_mean_f32: bad shape");
    cudaStream_t st = as_stream(stream);
    Scratch sum;
    JB_CUDA(sum.alloc(sizeof(double) * dims, st));
    int threads = 128, blocks = (dims + threads - 1) / threads;
    column_sum_f64_kernel<<<(dims + 7) / 8, CS_THREADS, 0, st>>>(x, n, dims, sum.as<double>());
    mean_finish_kernel<<<blocks, threads, 0, st>>>(sum.as<double>(), n, dims, nullptr, out);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

int jb_medoid(const float* x, int64_t n, int32_t dims, int64_t* out_host, void* stream) {
    JB_CHECK_ARG(n >= 1, "medoid of an empty dataset");
    JB_CHECK_ARG(dims >= 1, "jb_medoid: bad dims");
    cudaStream_t st = as_stream(stream);
    int nb = std::min<int64_t>((n + 255) / 256, 4 * sm_count_current());
    Scratch buf;
    size_t off_center = sizeof(double) * dims;
    size_t off_part = off_center * 2;
    size_t off_out = off_part + sizeof(DI) * nb;
    JB_CUDA(buf.alloc(off_out + 16, st));
    char* b = buf.as<char>();
    double* sum = reinterpret_cast<double*>(b);
    double* center = reinterpret_cast<double*>(b + off_center);
    DI* part = reinterpret_cast<DI*>(b + off_part);
    int64_t* dout = reinterpret_cast<int64_t*>(b + off_out);
    int threads = 128, blocks = (dims + threads - 1) / threads;
    column_sum_f64_kernel<<<(dims + 7) / 8, CS_THREADS, 0, st>>>(x, n, dims, sum);
    mean_finish_kernel<<<blocks, threads, 0, st>>>(sum, n, dims, center, nullptr);
    JB_CUDA_RC(grow_smem(medoid_partial_kernel, (int)(sizeof(double) * dims)));
    medoid_partial_kernel<<<nb, 256, sizeof(double) * dims, st>>>(x, n, dims, center, part);
    medoid_final_kernel<<<1, 1, 0, st>>>(part, nb, dout);
    JB_LAUNCH_CHECK();
    JB_CUDA(cudaMemcpyAsync(out_host, dout, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    JB_CUDA(cudaStreamSynchronize(st));
    return JB_OK;
}

int jb_frontier_topk(const uint64_t* frontier_keys, int64_t nq, int32_t beam_width, int32_t k,
                     int32_t* out_ids, double* out_dists, void* stream) {
    JB_CHECK_ARG(k >= 1 && k <= beam_width, "k must satisfy 1 <= k <= beam_width");
    if (nq == 0) return JB_OK;
    int64_t total = nq * k;
    int threads = 256;
    frontier_topk_kernel<<<(unsigned)((total + threads - 1) / threads), threads, 0, as_stream(stream)>>>(
        frontier_keys, nq, beam_width, k, out_ids, out_dists, false);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

int jb_frontier_topk_u8(const uint64_t* frontier_keys, int64_t nq, int32_t beam_width, int32_t k, int32_t* out_ids,
                        double* out_dists, void* stream) {
    JB_CHECK_ARG(k >= 1 && k <= beam_width, "k must satisfy 1 <= k <= beam_width");
    if (nq == 0) return JB_OK;
    int64_t total = nq * k;
    int threads = 256;
    frontier_topk_kernel<<<(unsigned)((total + threads - 1) / threads), threads, 0, as_stream(stream)>>>(
        frontier_keys, nq, beam_width, k, out_ids, out_dists, true);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

int jb_row_sq_norms_u8(const uint8_t* x, int64_t n, int32_t dims, uint32_t* out, void* stream) {
    JB_CHECK_ARG(dims >= 1 && n >= 0, "jb_row_sq_norms_u8: bad shape");
    JB_CHECK_ARG((int64_t)dims * 255 * 255 < (1ll << 32), "u8 dims too large for 32-bit packed distances");
    if (n == 0) return JB_OK;
    row_sq_norms_u8_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(x, n, dims, out);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

int jb_u8_to_f32(const uint8_t* x, int64_t count, float* out, void* stream) {
    JB_CHECK_ARG(count >= 0, "jb_u8_to_f32: bad count");
    if (count == 0) return JB_OK;
    const int blocks = (int)std::min<int64_t>((count + 255) / 256, 16 * sm_count_current());
    u8_to_f32_kernel<<<blocks, 256, 0, as_stream(stream)>>>(x, count, out);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

int jb_medoid_u8(const uint8_t* x, int64_t n, int32_t dims, int64_t* out_host, void* stream) {
    JB_CHECK_ARG(n >= 1, "medoid of an empty dataset");
    JB_CHECK_ARG(dims >= 1, "jb_medoid: bad dims");
    cudaStream_t st = as_stream(stream);
    Scratch f;
    JB_CUDA(f.alloc(sizeof(float) * (size_t)n * dims, st));
    int rc = jb_u8_to_f32(x, n * dims, f.as<float>(), stream);
    if (rc) return rc;
    return jb_medoid(f.as<float>(), n, dims, out_host, stream);
}

}  // extern "C"
