// metric.cuh — distance policies of the construction kernels (build.cu).
//
// A construction kernel needs three things from its distance source: prepare a
// pivot (the vertex whose neighbours are being chosen) in per-warp smem,
// evaluate d(pivot, row) with the row in the data role and the pivot's norm
// added last (build.py:105-134), and turn the 32-bit key word of a distance
// back into the f64 value the prune compares (graph.py:218, build.py:134).
// Keys everywhere are (dist_bits << 32) | id, ordered as unsigned integers,
// which orders non-negative f32 distances and u32 integer distances alike.
//
//   F32Metric  exact f32 rows, numpy einsum rounding (A1)     search.py:82-130
//   U8Metric   exact u8 rows, integer distances               search.py:92-99
//
// Candidate rows can also be staged in smem (`stage`/`dist_staged`) when a
// prune's candidate set fits; both policies stage 16-byte-aligned rows.
#pragma once
#include "common.cuh"

namespace jb {

struct F32Metric {
    const float* data;
    const float* norms;
    int D;
    static constexpr bool kInt = false;

    __host__ __device__ int row_bytes() const { return D * 4; }
    // smem words of one staged row (16 B skew keeps per-lane float4 reads conflict free)
    __host__ __device__ int stage_stride_words() const { return ((D + 3) & ~3) + 4; }
    __host__ __device__ int pivot_words() const { return ((D + 3) & ~3) + 4; }
    __device__ static double value(uint32_t bits) { return (double)__uint_as_float(bits); }

    // warp: pivot row + its norm into smem
    __device__ void load_pivot(uint32_t* pv, uint32_t v) const {
        const int lane = lane_id();
        const float* r = data + (size_t)v * D;
        float* f = reinterpret_cast<float*>(pv);
        for (int e = lane; e < D; e += 32) f[e] = r[e];
        if (lane == 0) f[((D + 3) & ~3)] = norms[v];
        __syncwarp();
    }
    // d(pivot, row): max((xn[row] - 2*dot(x[row], pivot)) + xn[pivot], 0)
    __device__ uint32_t dist(const uint32_t* pv, uint32_t row) const {
        const float* f = reinterpret_cast<const float*>(pv);
        const float dot = a1_dot<false>(data + (size_t)row * D, f, D);
        return __float_as_uint(exact_from_dot(__ldg(norms + row), dot, f[((D + 3) & ~3)]));
    }
    // stage n candidate rows (ids in the low words of keys) + their norms
    __device__ void stage(uint32_t* rows, uint32_t* cn, const uint64_t* keys, int n) const {
        const int lane = lane_id();
        const int rs = stage_stride_words();
        if ((D & 3) == 0) {
            const int nv = D >> 2;
            for (int j = 0; j < n; ++j) {
                const float* src = data + (size_t)(uint32_t)(keys[j] & 0xFFFFFFFFull) * D;
                for (int f = lane; f < nv; f += 32) cp_async16(rows + (size_t)j * rs + 4 * f, src + 4 * f);
            }
        } else {
            for (int j = 0; j < n; ++j) {
                const float* src = data + (size_t)(uint32_t)(keys[j] & 0xFFFFFFFFull) * D;
                for (int f = lane; f < D; f += 32) cp_async4(rows + (size_t)j * rs + f, src + f);
            }
        }
        for (int j = lane; j < n; j += 32)
            cn[j] = __float_as_uint(__ldg(norms + (uint32_t)(keys[j] & 0xFFFFFFFFull)));
        cp_async_wait_all();
        __syncwarp();
    }
    // d(staged pivot p, staged row i)
    __device__ uint32_t dist_staged(const uint32_t* rows, const uint32_t* cn, int i, int p) const {
        const int rs = stage_stride_words();
        const float* a = reinterpret_cast<const float*>(rows + (size_t)i * rs);
        const float* b = reinterpret_cast<const float*>(rows + (size_t)p * rs);
        Acc4 acc; acc.zero();
        if ((D & 3) == 0) a1_range<true, false>(acc, a, b, 0, D);
        else a1_range<false, false>(acc, a, b, 0, D);
        return __float_as_uint(exact_from_dot(__uint_as_float(cn[i]), acc.reduce(), __uint_as_float(cn[p])));
    }
};

// <a, b> of two u8 rows; a in global or smem, b in smem (16 B aligned). Exact.
__device__ __forceinline__ uint32_t u8_dot(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int D) {
    uint32_t acc = 0;
    int e = 0;
    if ((reinterpret_cast<uintptr_t>(a) & 15) == 0) {
        for (; e + 16 <= D; e += 16) {
            const uint4 x = *reinterpret_cast<const uint4*>(a + e);
            const uint4 y = *reinterpret_cast<const uint4*>(b + e);
            acc = __dp4a(x.x, y.x, acc);
            acc = __dp4a(x.y, y.y, acc);
            acc = __dp4a(x.z, y.z, acc);
            acc = __dp4a(x.w, y.w, acc);
        }
    } else if ((reinterpret_cast<uintptr_t>(a) & 3) == 0) {
        for (; e + 4 <= D; e += 4)
            acc = __dp4a(*reinterpret_cast<const uint32_t*>(a + e), *reinterpret_cast<const uint32_t*>(b + e), acc);
    }
    for (; e < D; ++e) acc += (uint32_t)a[e] * (uint32_t)b[e];
    return acc;
}

// ||x||^2 - 2<x, q> + ||q||^2, exact (the caller bounds D * 255^2 < 2^32)
__device__ __forceinline__ uint32_t u8_dist(uint32_t xn, uint32_t dot, uint32_t qn) {
    return (uint32_t)((uint64_t)xn + (uint64_t)qn - 2ull * (uint64_t)dot);
}

struct U8Metric {
    const uint8_t* data;
    const uint32_t* norms;
    int D;
    static constexpr bool kInt = true;

    __host__ __device__ int row_bytes() const { return D; }
    __host__ __device__ int stage_stride_words() const { return ((D + 15) & ~15) / 4 + 4; }
    __host__ __device__ int pivot_words() const { return ((D + 15) & ~15) / 4 + 4; }
    __device__ static double value(uint32_t bits) { return (double)bits; }

    __device__ void load_pivot(uint32_t* pv, uint32_t v) const {
        const int lane = lane_id();
        const uint8_t* r = data + (size_t)v * D;
        uint8_t* b = reinterpret_cast<uint8_t*>(pv);
        for (int e = lane; e < D; e += 32) b[e] = r[e];
        if (lane == 0) pv[((D + 15) & ~15) / 4] = norms[v];
        __syncwarp();
    }
    __device__ uint32_t dist(const uint32_t* pv, uint32_t row) const {
        const uint32_t dot = u8_dot(data + (size_t)row * D, reinterpret_cast<const uint8_t*>(pv), D);
        return u8_dist(__ldg(norms + row), dot, pv[((D + 15) & ~15) / 4]);
    }
    __device__ void stage(uint32_t* rows, uint32_t* cn, const uint64_t* keys, int n) const {
        const int lane = lane_id();
        const int rs = stage_stride_words();
        if ((D & 15) == 0) {
            const int nv = D >> 4;
            for (int j = 0; j < n; ++j) {
                const uint8_t* src = data + (size_t)(uint32_t)(keys[j] & 0xFFFFFFFFull) * D;
                for (int f = lane; f < nv; f += 32) cp_async16(rows + (size_t)j * rs + 4 * f, src + 16 * f);
            }
            cp_async_wait_all();
        } else {
            for (int j = 0; j < n; ++j) {
                const uint8_t* src = data + (size_t)(uint32_t)(keys[j] & 0xFFFFFFFFull) * D;
                uint8_t* dst = reinterpret_cast<uint8_t*>(rows + (size_t)j * rs);
                for (int f = lane; f < D; f += 32) dst[f] = src[f];
            }
        }
        for (int j = lane; j < n; j += 32) cn[j] = __ldg(norms + (uint32_t)(keys[j] & 0xFFFFFFFFull));
        __syncwarp();
    }
    __device__ uint32_t dist_staged(const uint32_t* rows, const uint32_t* cn, int i, int p) const {
        const int rs = stage_stride_words();
        const uint8_t* a = reinterpret_cast<const uint8_t*>(rows + (size_t)i * rs);
        const uint8_t* b = reinterpret_cast<const uint8_t*>(rows + (size_t)p * rs);
        return u8_dist(cn[i], u8_dot(a, b, D), cn[p]);
    }
};

}  // namespace jb
