// distances.cu — bound distance sources and the matrix form of robust prune.
//
// The reference's search engine and builder talk to distance sources through a
// small protocol: `bind_distance_source(source, queries)` (search.py:159-168)
// returns an object whose `distances(qrows, ids)` evaluates the source for
// (query row, vector id) pairs (ExactDistances search.py:82-130, _BoundQuantized
// rabitq.py:225-244), and `robust_prune` (graph.py:174-228) takes any
// `dist_fn(pivot, ids)`. The build and search kernels evaluate their sources
// inline; these entry points serve that public protocol on the device:
//   jb_bound_distances      one thread per (qrow, id) pair, the same rounding as
//                           the search kernel (A1 f32 / exact u32 / reference
//                           RaBitQ estimator)
//   jb_robust_prune_matrix  one warp: the reference prune over a candidate set
//                           given d(c_i, c_j) as a matrix (any dist_fn, e.g. the
//                           reference's own _PairwiseDistances or a user callable)
#include "common.cuh"
#include "metric.cuh"
#include "runtime.cuh"

namespace jb {

// Query rows are read at `qs` elements apart: the RaBitQ estimator reads the rotated
// query with 16-byte vector loads and the u8 dot reads 16-byte words, so the host
// pads those rows (qs = dims rounded up to 4 floats / 16 bytes).
template <int SRC, int BITS>
__global__ void bound_distances_kernel(jb_search_args a, int64_t qs, const int64_t* __restrict__ qrows,
                                       const int64_t* __restrict__ ids, int64_t n, void* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t q = qrows[i], v = ids[i];
    const int D = a.dims;
    if (SRC == JB_SRC_EXACT) {
        const float dot = a1_dot<false>(a.data + v * D, a.queries + q * qs, D);
        reinterpret_cast<float*>(out)[i] = exact_from_dot(a.data_norms[v], dot, a.query_add[q]);
    } else if (SRC == JB_SRC_EXACT_U8) {
        const uint8_t* x = a.data_u8 + v * D;
        const uint8_t* y = a.queries_u8 + q * qs;
        uint32_t dot = 0;
        if ((reinterpret_cast<uintptr_t>(x) & 3) == 0) {
            dot = u8_dot(x, y, D);  // y is 16 B aligned (padded stride)
        } else {
            for (int e = 0; e < D; ++e) dot += (uint32_t)x[e] * (uint32_t)y[e];
        }
        reinterpret_cast<uint32_t*>(out)[i] = u8_dist(a.norms_u32[v], dot, a.query_norms_u32[q]);
    } else {
        const int meta_off = ((((D * BITS) + 7) / 8 + 15) / 16) * 16;
        reinterpret_cast<float*>(out)[i] = rabitq_estimate<BITS>(a.records + v * a.record_bytes, a.queries + q * qs,
                                                                 D, meta_off, a.query_add[q], a.query_sumq[q]);
    }
}

// (d, id) lexicographic minimum across the warp
__device__ __forceinline__ void warp_min_pair(double& d, int64_t& id) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double od = __shfl_xor_sync(0xFFFFFFFFu, d, o);
        const int64_t oi = __shfl_xor_sync(0xFFFFFFFFu, id, o);
        if (od < d || (od == d && oi < id)) { d = od; id = oi; }
    }
}

// graph.py:174-228 with dist_fn(star, ids)[j] = dmat[star_pos * n + j]: take the
// closest remaining candidate by (dist, id), keep p' iff alpha^2 * d(star, p') > d(p, p')
// (f64), until degree_cap are kept. `alive` is per-candidate scratch.
__global__ void prune_matrix_kernel(const double* __restrict__ dmat, const int64_t* __restrict__ ids,
                                    const double* __restrict__ dists, int n, double alpha2, int R,
                                    uint8_t* __restrict__ alive, int32_t* __restrict__ out_pos,
                                    int32_t* __restrict__ out_n) {
    const int lane = threadIdx.x;
    for (int j = lane; j < n; j += 32) alive[j] = 1;
    __syncwarp();
    int kept = 0;
    while (kept < R) {
        double bd = __longlong_as_double(0x7FF0000000000000ll);
        int64_t bid = INT64_MAX;
        int bpos = -1;
        for (int j = lane; j < n; j += 32) {
            if (!alive[j]) continue;
            const double d = dists[j];
            if (bpos < 0 || d < bd || (d == bd && ids[j] < bid)) { bd = d; bid = ids[j]; bpos = j; }
        }
        // lanes without a live candidate hold (+inf, INT64_MAX) and lose every comparison
        double md = bd;
        int64_t mid = bid;
        warp_min_pair(md, mid);
        const unsigned any = __ballot_sync(0xFFFFFFFFu, bpos >= 0);
        if (!any) break;
        // the winning lane owns the star's position
        const unsigned win = __ballot_sync(0xFFFFFFFFu, bpos >= 0 && bid == mid && bd == md);
        const int star = __shfl_sync(0xFFFFFFFFu, bpos, __ffs(win) - 1);
        if (lane == 0) out_pos[kept] = star;
        ++kept;
        if (lane == 0) alive[star] = 0;
        __syncwarp();
        if (kept >= R) break;
        for (int j = lane; j < n; j += 32)
            if (alive[j] && !(alpha2 * dmat[(int64_t)star * n + j] > dists[j])) alive[j] = 0;
        __syncwarp();
    }
    if (lane == 0) *out_n = kept;
}

template <int SRC, int BITS>
static int launch_bound(const jb_search_args& a, int64_t qs, const int64_t* qrows, const int64_t* ids, int64_t n,
                        void* out, cudaStream_t st) {
    bound_distances_kernel<SRC, BITS><<<(unsigned)((n + 127) / 128), 128, 0, st>>>(a, qs, qrows, ids, n, out);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

}  // namespace jb

using namespace jb;

extern "C" int jb_bound_distances(const jb_search_args* args, int64_t query_stride, const int64_t* qrows,
                                  const int64_t* ids, int64_t n, void* out, void* stream) {
    JB_CHECK_ARG(args != nullptr, "jb_bound_distances: null args");
    const jb_search_args& a = *args;
    JB_CHECK_ARG(a.dims >= 1, "dims must be >= 1");
    const int64_t qs = query_stride > 0 ? query_stride : a.dims;
    JB_CHECK_ARG(qs >= a.dims, "query_stride below dims");
    if (n == 0) return JB_OK;
    cudaStream_t st = as_stream(stream);
    switch (a.source) {
        case JB_SRC_EXACT:
            JB_CHECK_ARG(a.data && a.data_norms && a.queries && a.query_add, "exact source: missing arrays");
            return launch_bound<JB_SRC_EXACT, 1>(a, qs, qrows, ids, n, out, st);
        case JB_SRC_EXACT_U8:
            JB_CHECK_ARG(a.data_u8 && a.norms_u32 && a.queries_u8 && a.query_norms_u32, "u8 source: missing arrays");
            JB_CHECK_ARG(qs % 16 == 0 && (reinterpret_cast<uintptr_t>(a.queries_u8) & 15) == 0,
                         "u8 bound queries need a 16-byte row stride");
            return launch_bound<JB_SRC_EXACT_U8, 1>(a, qs, qrows, ids, n, out, st);
        case JB_SRC_RABITQ:
            JB_CHECK_ARG(a.records && a.queries && a.query_add && a.query_sumq, "rabitq source: missing arrays");
            JB_CHECK_ARG(a.record_bytes == jb_rabitq_record_bytes(a.dims, a.bits), "rabitq: record_bytes mismatch");
            JB_CHECK_ARG(qs % 4 == 0 && (reinterpret_cast<uintptr_t>(a.queries) & 15) == 0,
                         "rabitq bound queries need a 16-byte row stride");
            switch (a.bits) {
                case 1: return launch_bound<JB_SRC_RABITQ, 1>(a, qs, qrows, ids, n, out, st);
                case 2: return launch_bound<JB_SRC_RABITQ, 2>(a, qs, qrows, ids, n, out, st);
                case 4: return launch_bound<JB_SRC_RABITQ, 4>(a, qs, qrows, ids, n, out, st);
                case 8: return launch_bound<JB_SRC_RABITQ, 8>(a, qs, qrows, ids, n, out, st);
                default: JB_CHECK_ARG(false, "bits must be one of (1, 2, 4, 8)");
            }
        default: JB_CHECK_ARG(false, "bound distances: unsupported source %d", a.source);
    }
}

extern "C" int jb_robust_prune_matrix(const double* dmat, const int64_t* ids, const double* dists, int32_t n,
                                      double alpha, int32_t degree_cap, int32_t* out_pos, int32_t* out_count,
                                      void* stream) {
    JB_CHECK_ARG(alpha >= 1.0, "alpha must be >= 1");
    JB_CHECK_ARG(degree_cap >= 1, "degree_cap must be >= 1");
    JB_CHECK_ARG(n >= 0, "n must be >= 0");
    cudaStream_t st = as_stream(stream);
    Scratch alive;
    JB_CUDA(alive.alloc((size_t)(n > 0 ? n : 1), st));
    prune_matrix_kernel<<<1, 32, 0, st>>>(dmat, ids, dists, n, alpha * alpha, degree_cap, alive.as<uint8_t>(),
                                          out_pos, out_count);
    JB_LAUNCH_CHECK();
    return JB_OK;
}
