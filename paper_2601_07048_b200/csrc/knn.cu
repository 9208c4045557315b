// knn.cu — exact brute-force top-k in f64 (ground truth), sm_100a.
//
// Replaces `exact_knn` (oracle.py:20-62): scores = (xn - 2 q.x) + qn in f64,
// clamped at 0 (squared Euclidean), or -(q.x) (inner product, oracle.py:53-54),
// ranked by (score, id) ascending (numpy's stable argsort), the first k written
// as int32 ids and f32 distances.
//
// Layout: queries are processed in blocks of QB (a multiple of 64 sized so the
// f64 score block QB x n stays ~2 GB in HBM).
//   1. knn_norms_kernel      xn (f64, once) and qn per block
//   2. knn_scores_kernel     64x64 tiles of the f64 score block, SIMT DFMA from
//                            smem-staged f64 tiles (4x4 outputs per thread)
//   3. knn_select_kernel     one CTA per query: MSD radix select on the score
//                            bits (f64 >= 0 orders like its u64 pattern), 12-bit
//                            digits, until the k-th bucket holds <= CAND_CAP
//                            scores; then everything below the bucket plus the
//                            bucket is collected and sorted by (score, id).
// Summation order differs from OpenBLAS dgemm, so scores agree with the
// reference to f64 rounding (a few ulp); ids agree except between scores equal
// to within that rounding (tests compare with that tolerance).
#include <algorithm>
#include <cub/block/block_scan.cuh>
#include "common.cuh"
#include "runtime.cuh"

namespace jb {

constexpr int KNN_TILE = 64;       // queries x rows per score tile
constexpr int KNN_KC = 16;         // K chunk staged in smem
constexpr int SEL_THREADS = 1024;
constexpr int SEL_BITS = 12;
constexpr int SEL_BINS = 1 << SEL_BITS;
constexpr int CAND_CAP = 2048;     // bucket size at which the select stops refining
constexpr int KNN_MAX_K = 1024;
constexpr int SORT_N = 4096;       // >= KNN_MAX_K + CAND_CAP, power of two
constexpr int SEL_SMEM = SORT_N * 12 + SEL_BINS * 4;

__global__ void knn_norms_kernel(const float* __restrict__ x, int64_t n, int D, double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* r = x + i * D;
    double s = 0.0;
    for (int e = 0; e < D; ++e) {
        const double v = (double)r[e];
        s = fma(v, v, s);
    }
    out[i] = s;
}

// S[q, i] = max((xn[i] - 2 * <q, x_i>) + qn[q], 0) for q in [0, nqb), i in [0, n).
__global__ void __launch_bounds__(256)
knn_scores_kernel(const float* __restrict__ x, int64_t n, int D, const float* __restrict__ q, int64_t nqb,
                  const double* __restrict__ xn, const double* __restrict__ qn, double* __restrict__ S, bool ip) {
    __shared__ double qs[KNN_KC][KNN_TILE + 2];
    __shared__ double xs[KNN_KC][KNN_TILE + 2];
    const int tid = threadIdx.x;
    const int tq = tid >> 4, tx = tid & 15;  // 16 x 16 threads, 4 x 4 outputs each
    const int64_t q0 = (int64_t)blockIdx.y * KNN_TILE;
    const int64_t x0 = (int64_t)blockIdx.x * KNN_TILE;
    double acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    for (int k0 = 0; k0 < D; k0 += KNN_KC) {
        // stage 64 x 16 of each operand (k-major), zero padded
        for (int t = tid; t < KNN_TILE * KNN_KC; t += 256) {
            const int r = t / KNN_KC, c = t % KNN_KC;
            const int kk = k0 + c;
            const int64_t qi = q0 + r, xi = x0 + r;
            qs[c][r] = (qi < nqb && kk < D) ? (double)q[qi * D + kk] : 0.0;
            xs[c][r] = (xi < n && kk < D) ? (double)x[xi * D + kk] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < KNN_KC; ++c) {
            double av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) av[a] = qs[c][tq + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; ++b) bv[b] = xs[c][tx + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int64_t qi = q0 + tq + 16 * a;
        if (qi >= nqb) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t xi = x0 + tx + 16 * b;
            if (xi >= n) continue;
            if (ip) {
                S[qi * n + xi] = 0.0 - acc[a][b];  // -(q @ x.T); 0 - 0 = +0, so no -0 patterns
            } else {
                double s = (xn[xi] - 2.0 * acc[a][b]) + qn[qi];
                S[qi * n + xi] = s > 0.0 ? s : 0.0;
            }
        }
    }
}

// f64 -> u64 with the same order (negative scores appear in inner-product mode)
__device__ __forceinline__ uint64_t dbits(double v) {
    const uint64_t b = (uint64_t)__double_as_longlong(v);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dval(uint64_t k) {
    return __longlong_as_double((long long)((k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k));
}

__global__ void __launch_bounds__(SEL_THREADS)
knn_select_kernel(const double* __restrict__ S, int64_t n, int k, int32_t* __restrict__ out_ids,
                  float* __restrict__ out_d) {
    using Scan = cub::BlockScan<int, SEL_THREADS>;
    __shared__ typename Scan::TempStorage scan_tmp;
    extern __shared__ __align__(16) unsigned char dsm[];  // SEL_SMEM bytes
    uint64_t* skey = reinterpret_cast<uint64_t*>(dsm);
    int32_t* sid = reinterpret_cast<int32_t*>(dsm + SORT_N * 8);
    int* hist = reinterpret_cast<int*>(dsm + SORT_N * 12);
    __shared__ int s_bucket, s_below, s_count, s_ncand;
    const int tid = threadIdx.x;
    const double* row = S + (int64_t)blockIdx.x * n;

    // MSD radix select: find the bucket (prefix over the bits decided so far)
    // holding the k-th smallest score and the rank within it.
    uint64_t prefix = 0, pmask = 0;  // decided bits and their mask
    int krem = k;                    // 1-based rank of the target inside the current bucket
    int shift = 64;
    for (;;) {
        const int width = shift >= SEL_BITS ? SEL_BITS : shift;
        shift -= width;
        const uint64_t dmask = (((uint64_t)1 << width) - 1) << shift;
        for (int b = tid; b < SEL_BINS; b += SEL_THREADS) hist[b] = 0;
        __syncthreads();
        for (int64_t i = tid; i < n; i += SEL_THREADS) {
            const uint64_t v = dbits(row[i]);
            if ((v & pmask) == prefix) atomicAdd(&hist[(v & dmask) >> shift], 1);
        }
        __syncthreads();
        int c[SEL_BINS / SEL_THREADS], tot = 0;
#pragma unroll
        for (int j = 0; j < SEL_BINS / SEL_THREADS; ++j) { c[j] = hist[tid * (SEL_BINS / SEL_THREADS) + j]; tot += c[j]; }
        int before;
        Scan(scan_tmp).ExclusiveSum(tot, before);
#pragma unroll
        for (int j = 0; j < SEL_BINS / SEL_THREADS; ++j) {
            if (before < krem && krem <= before + c[j]) {
                s_bucket = tid * (SEL_BINS / SEL_THREADS) + j;
                s_below = before;
                s_count = c[j];
            }
            before += c[j];
        }
        __syncthreads();
        prefix |= (uint64_t)s_bucket << shift;
        pmask |= dmask;
        krem -= s_below;
        const int cnt = s_count;
        __syncthreads();
        if (cnt <= CAND_CAP || shift == 0) break;
    }

    // Collect every score strictly below the bucket (all in the top k: fewer
    // than k of them) and the bucket itself (capped; when shift reached 0 the
    // bucket is one exact value and only its smallest ids can matter).
    if (tid == 0) s_ncand = 0;
    __syncthreads();
    const uint64_t lo = prefix;  // smallest pattern in the bucket
    for (int64_t i = tid; i < n; i += SEL_THREADS) {
        const uint64_t v = dbits(row[i]);
        const bool take = v < lo || (v & pmask) == prefix;
        if (take) {
            const int p = atomicAdd(&s_ncand, 1);
            if (p < SORT_N) { skey[p] = v; sid[p] = (int32_t)i; }
        }
    }
    __syncthreads();
    int m = min(s_ncand, SORT_N);
    for (int p = m + tid; p < SORT_N; p += SEL_THREADS) { skey[p] = ~0ull; sid[p] = 0x7FFFFFFF; }
    __syncthreads();
    // bitonic sort of (key, id) pairs, ascending
    for (int kk = 2; kk <= SORT_N; kk <<= 1) {
        for (int j = kk >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < SORT_N; i += SEL_THREADS) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const uint64_t a = skey[i], b = skey[ixj];
                    const int32_t ia = sid[i], ib = sid[ixj];
                    const bool gt = a > b || (a == b && ia > ib);
                    if (gt == ((i & kk) == 0)) { skey[i] = b; skey[ixj] = a; sid[i] = ib; sid[ixj] = ia; }
                }
            }
            __syncthreads();
        }
    }
    for (int j = tid; j < k; j += SEL_THREADS) {
        out_ids[(int64_t)blockIdx.x * k + j] = sid[j];
        out_d[(int64_t)blockIdx.x * k + j] = (float)dval(skey[j]);
    }
}

}  // namespace jb

using namespace jb;

extern "C" int jb_exact_knn_kind(const float* data, int64_t n, int32_t dims, const float* queries, int64_t nq,
                                 int32_t k, int32_t inner_product, int32_t* out_ids, float* out_dists, void* stream) {
    JB_CHECK_ARG(dims >= 1, "dims must be >= 1");
    JB_CHECK_ARG(n >= 1 && n < (1ll << 31), "exact_knn: n must be in [1, 2^31)");
    JB_CHECK_ARG(k >= 1 && k <= n, "k must be in [1, %lld]", (long long)n);
    JB_CHECK_ARG(k <= KNN_MAX_K, "exact_knn: k must be <= %d", KNN_MAX_K);
    if (nq == 0) return JB_OK;
    cudaStream_t st = as_stream(stream);
    // query block: multiple of 64 with a ~2 GB f64 score block
    int64_t qb = ((int64_t)1 << 28) / n;
    qb = std::max<int64_t>(KNN_TILE, (qb / KNN_TILE) * KNN_TILE);
    qb = std::min<int64_t>(qb, ((nq + KNN_TILE - 1) / KNN_TILE) * KNN_TILE);
    Scratch xn, qn, sc;
    JB_CUDA(xn.alloc(sizeof(double) * n, st));
    JB_CUDA(qn.alloc(sizeof(double) * qb, st));
    JB_CUDA(sc.alloc(sizeof(double) * qb * n, st));
    JB_CUDA_RC(grow_smem(knn_select_kernel, SEL_SMEM));
    knn_norms_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(data, n, dims, xn.as<double>());
    JB_LAUNCH_CHECK();
    for (int64_t q0 = 0; q0 < nq; q0 += qb) {
        const int64_t m = std::min<int64_t>(qb, nq - q0);
        const float* qp = queries + q0 * dims;
        knn_norms_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(qp, m, dims, qn.as<double>());
        dim3 grid((unsigned)((n + KNN_TILE - 1) / KNN_TILE), (unsigned)((m + KNN_TILE - 1) / KNN_TILE));
        knn_scores_kernel<<<grid, 256, 0, st>>>(data, n, dims, qp, m, xn.as<double>(), qn.as<double>(),
                                                sc.as<double>(), inner_product != 0);
        knn_select_kernel<<<(unsigned)m, SEL_THREADS, SEL_SMEM, st>>>(sc.as<double>(), n, k, out_ids + q0 * k,
                                                               out_dists + q0 * k);
        JB_LAUNCH_CHECK();
    }
    return JB_OK;
}

extern "C" int jb_exact_knn(const float* data, int64_t n, int32_t dims, const float* queries, int64_t nq, int32_t k,
                            int32_t* out_ids, float* out_dists, void* stream) {
    return jb_exact_knn_kind(data, n, dims, queries, nq, k, 0, out_ids, out_dists, stream);
}
