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
//   F32Metric     exact f32 rows, numpy einsum rounding (A1)   search.py:82-130
//   U8Metric      exact u8 rows, integer distances             search.py:92-99
//   RabitqMetric  RaBitQ estimates (quantized construction)    build.py:124-129
//
// Candidate rows can also be staged in smem (`stage`/`dist_staged`) when a
// prune's candidate set fits (kStage); the exact policies stage 16-byte-aligned rows.
#pragma once
#include "common.cuh"

namespace jb {

struct F32Metric {
    const float* data;
    const float* norms;
    int D;
    static constexpr bool kInt = false;
    static constexpr bool kStage = true;
    // Staged rows of D % 16 == 0 are stored 4x4-transposed inside every 16-element
    // block (word 16b + 4k + v holds element 16b + 4v + k): the four elements that
    // A1 accumulator lane k adds in one block are one float4, so 1, 2 or 4 threads
    // can share a distance with the reference's rounding (dot2_split).
    // Opt-in per launch (split_prune() in build.cu): it pays in phase 2 / refine,
    // where many candidates are pruned per round, not in the owner merge.
    static constexpr bool kSplit = true;
    bool split = false;
    // Gram-screened staged prune (warp_prune_gram, build.cu) for <= 64 candidates;
    // JB_GRAM=0 turns it off (A/B). Requires D % 8 == 0.
    bool gram = false;
    __host__ __device__ bool gram_ok(int n, int nmax = 64) const { return gram && (D & 7) == 0 && n <= nmax; }
    // Prune closure per vertex (build.cu, owner merge): closure[v] = alpha^2 of the
    // robust prune that last wrote v's row, 0 after any other write (append, bridge).
    // A row closed at alpha_a^2 <= the current alpha^2 has no member pruning a later
    // one, so a merge only needs the pairs involving the fresh sources. nullptr: off.
    double* closure = nullptr;
    __device__ void close_row(uint32_t v, double alpha2) const { if (closure) closure[v] = alpha2; }
    __device__ void open_row(uint32_t v) const { if (closure) closure[v] = 0.0; }
    __device__ bool row_closed(uint32_t v, double alpha2) const {
        if (!closure) return false;
        const double c = closure[v];
        return c > 0.0 && c <= alpha2;
    }
#ifdef JB_NO_SPLIT
    __host__ __device__ bool split_ok() const { return false; }  // dev A/B: natural layout, flat prune
#else
    __host__ __device__ bool split_ok() const { return split && (D & 15) == 0; }
#endif

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
    // as load_pivot, but the row copy is left in flight (cp.async): the caller's next
    // cp_async_wait_all + __syncwarp (e.g. the one closing stage()) completes it
    __device__ void load_pivot_async(uint32_t* pv, uint32_t v) const {
        const int lane = lane_id();
        const float* r = data + (size_t)v * D;
        if ((D & 3) == 0) {
            for (int f = lane; f < (D >> 2); f += 32) cp_async16(pv + 4 * f, r + 4 * f);
        } else {
            for (int e = lane; e < D; e += 32) cp_async4(pv + e, r + e);
        }
        if (lane == 0) pv[((D + 3) & ~3)] = __float_as_uint(norms[v]);
    }
    // d(pivot, row): max((xn[row] - 2*dot(x[row], pivot)) + xn[pivot], 0)
    __device__ uint32_t dist(const uint32_t* pv, uint32_t row) const {
        const float* f = reinterpret_cast<const float*>(pv);
        const float dot = a1_dot<false>(data + (size_t)row * D, f, D);
        return __float_as_uint(exact_from_dot(__ldg(norms + row), dot, f[((D + 3) & ~3)]));
    }
    // stage n candidate rows (ids in the low words of keys) + their norms; with a
    // per-warp mbarrier (bar, its phase) the rows go through cp.async.bulk, one
    // copy-engine instruction per row instead of a warp-wide 16 B cp.async loop
    __device__ void stage(uint32_t* rows, uint32_t* cn, const uint64_t* keys, int n, uint64_t* bar = nullptr,
                          uint32_t* phase = nullptr) const {
        const int lane = lane_id();
        const int rs = stage_stride_words();
        if (bar && (D & 3) == 0) {
            wbar_expect(bar, (uint32_t)n * (uint32_t)D * 4u);
            for (int j = lane; j < n; j += 32)
                bulk_row(rows + (size_t)j * rs, data + (size_t)(uint32_t)(keys[j] & 0xFFFFFFFFull) * D, (uint32_t)D * 4u,
                         bar);
        } else if ((D & 3) == 0) {
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
        cp_async_wait_all();  // (also the caller's cp.async pivot copy, load_pivot_async)
        if (bar && (D & 3) == 0) wbar_wait(bar, *phase);
        __syncwarp();
        if (split_ok()) {  // 4x4-transpose every 16-element block in place (one block per lane)
            const int nb = D >> 4;
            for (int t = lane; t < n * nb; t += 32) {
                float4* blk = reinterpret_cast<float4*>(rows + (size_t)(t / nb) * rs + 16 * (t % nb));
                const float4 v0 = blk[0], v1 = blk[1], v2 = blk[2], v3 = blk[3];
                blk[0] = make_float4(v0.x, v1.x, v2.x, v3.x);
                blk[1] = make_float4(v0.y, v1.y, v2.y, v3.y);
                blk[2] = make_float4(v0.z, v1.z, v2.z, v3.z);
                blk[3] = make_float4(v0.w, v1.w, v2.w, v3.w);
            }
            __syncwarp();
        }
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
    // d(pivot in pv, staged row i): same operation order as dist() on the global row
    __device__ uint32_t dist_pivot_staged(const uint32_t* pv, const uint32_t* rows, const uint32_t* cn, int i) const {
        const float* f = reinterpret_cast<const float*>(pv);
        const float* a = reinterpret_cast<const float*>(rows + (size_t)i * stage_stride_words());
        Acc4 acc; acc.zero();
        if (split_ok()) {  // natural pivot, transposed row
            const float4* P = reinterpret_cast<const float4*>(f);
            const float4* T = reinterpret_cast<const float4*>(a);
            for (int b = 0; b < (D >> 2); b += 4) {
                const float4 t0 = T[b], t1 = T[b + 1], t2 = T[b + 2], t3 = T[b + 3];
                const float4 p3 = P[b + 3], p2 = P[b + 2], p1 = P[b + 1], p0 = P[b];
                acc.madd(make_float4(t0.w, t1.w, t2.w, t3.w), p3);
                acc.madd(make_float4(t0.z, t1.z, t2.z, t3.z), p2);
                acc.madd(make_float4(t0.y, t1.y, t2.y, t3.y), p1);
                acc.madd(make_float4(t0.x, t1.x, t2.x, t3.x), p0);
            }
        } else if ((D & 3) == 0) a1_range<true, false>(acc, a, f, 0, D);
        else a1_range<false, false>(acc, a, f, 0, D);
        return __float_as_uint(exact_from_dot(__uint_as_float(cn[i]), acc.reduce(), f[((D + 3) & ~3)]));
    }
    // two rows against one pivot: the pivot's vectors are read once, the two A1
    // chains interleave (same per-row order, twice the independent work per lane)
    __device__ void dist_staged2(const uint32_t* rows, const uint32_t* cn, int i0, int i1, int p, uint32_t& d0,
                                 uint32_t& d1) const {
        if ((D & 15) != 0) {
            d0 = dist_staged(rows, cn, i0, p);
            d1 = dist_staged(rows, cn, i1, p);
            return;
        }
        const int rs = stage_stride_words();
        const float4* a0 = reinterpret_cast<const float4*>(rows + (size_t)i0 * rs);
        const float4* a1 = reinterpret_cast<const float4*>(rows + (size_t)i1 * rs);
        const float4* b = reinterpret_cast<const float4*>(rows + (size_t)p * rs);
        Acc4 x0, x1;
        x0.zero();
        x1.zero();
        for (int v = 0; v < (D >> 2); v += 4) {
#pragma unroll
            for (int i = 3; i >= 0; --i) {
                const float4 bv = b[v + i];
                x0.madd(a0[v + i], bv);
                x1.madd(a1[v + i], bv);
            }
        }
        const float pn = __uint_as_float(cn[p]);
        d0 = __float_as_uint(exact_from_dot(__uint_as_float(cn[i0]), x0.reduce(), pn));
        d1 = __float_as_uint(exact_from_dot(__uint_as_float(cn[i1]), x1.reduce(), pn));
    }
    // A1 dots of transposed staged rows i0 and i1 against staged row p, F threads per
    // row pair: thread `sub` runs accumulator lanes [sub*4/F, (sub+1)*4/F); the lanes
    // are combined as (l0 + l1) + (l2 + l3), so every F gives the same bits. The full
    // dots are valid in sub == 0 threads; all 32 lanes must call (shuffles).
    template <int F>
    __device__ void dot2_split(const uint32_t* rows, int i0, int i1, int p, int sub, float& d0, float& d1) const {
        constexpr int NK = 4 / F;
        const int rs = stage_stride_words();
        const float4* a0 = reinterpret_cast<const float4*>(rows + (size_t)i0 * rs) + sub * NK;
        const float4* a1 = reinterpret_cast<const float4*>(rows + (size_t)i1 * rs) + sub * NK;
        const float4* b = reinterpret_cast<const float4*>(rows + (size_t)p * rs) + sub * NK;
        float x0[NK], x1[NK];
#pragma unroll
        for (int t = 0; t < NK; ++t) x0[t] = x1[t] = 0.0f;
        for (int v = 0; v < (D >> 2); v += 4) {
#pragma unroll
            for (int t = 0; t < NK; ++t) {
                const float4 bv = b[v + t], u = a0[v + t], w = a1[v + t];
                x0[t] = __fadd_rn(__fmul_rn(u.w, bv.w), x0[t]);
                x1[t] = __fadd_rn(__fmul_rn(w.w, bv.w), x1[t]);
                x0[t] = __fadd_rn(__fmul_rn(u.z, bv.z), x0[t]);
                x1[t] = __fadd_rn(__fmul_rn(w.z, bv.z), x1[t]);
                x0[t] = __fadd_rn(__fmul_rn(u.y, bv.y), x0[t]);
                x1[t] = __fadd_rn(__fmul_rn(w.y, bv.y), x1[t]);
                x0[t] = __fadd_rn(__fmul_rn(u.x, bv.x), x0[t]);
                x1[t] = __fadd_rn(__fmul_rn(w.x, bv.x), x1[t]);
            }
        }
        const unsigned FULL = 0xFFFFFFFFu;
        if (F == 1) {
            d0 = __fadd_rn(__fadd_rn(x0[0], x0[NK > 1 ? 1 : 0]), __fadd_rn(x0[NK > 2 ? 2 : 0], x0[NK > 3 ? 3 : 0]));
            d1 = __fadd_rn(__fadd_rn(x1[0], x1[NK > 1 ? 1 : 0]), __fadd_rn(x1[NK > 2 ? 2 : 0], x1[NK > 3 ? 3 : 0]));
        } else if (F == 2) {  // thread 0: l0 + l1, thread 1: l2 + l3
            const float h0 = __fadd_rn(x0[0], x0[NK > 1 ? 1 : 0]), h1 = __fadd_rn(x1[0], x1[NK > 1 ? 1 : 0]);
            d0 = __fadd_rn(h0, __shfl_down_sync(FULL, h0, 1));
            d1 = __fadd_rn(h1, __shfl_down_sync(FULL, h1, 1));
        } else {  // thread k holds l_k
            const float q0 = __fadd_rn(x0[0], __shfl_down_sync(FULL, x0[0], 1));
            const float q1 = __fadd_rn(x1[0], __shfl_down_sync(FULL, x1[0], 1));
            d0 = __fadd_rn(q0, __shfl_down_sync(FULL, q0, 2));
            d1 = __fadd_rn(q1, __shfl_down_sync(FULL, q1, 2));
        }
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
    static constexpr bool kStage = true;
    __device__ void close_row(uint32_t, double) const {}
    __device__ void open_row(uint32_t) const {}
    __device__ bool row_closed(uint32_t, double) const { return false; }
    static constexpr bool kSplit = false;

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
    __device__ void load_pivot_async(uint32_t* pv, uint32_t v) const { load_pivot(pv, v); }
    __device__ uint32_t dist(const uint32_t* pv, uint32_t row) const {
        const uint32_t dot = u8_dot(data + (size_t)row * D, reinterpret_cast<const uint8_t*>(pv), D);
        return u8_dist(__ldg(norms + row), dot, pv[((D + 15) & ~15) / 4]);
    }
    __device__ void stage(uint32_t* rows, uint32_t* cn, const uint64_t* keys, int n, uint64_t* = nullptr,
                          uint32_t* = nullptr) const {
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
    __device__ void dist_staged2(const uint32_t* rows, const uint32_t* cn, int i0, int i1, int p, uint32_t& d0,
                                 uint32_t& d1) const {
        d0 = dist_staged(rows, cn, i0, p);
        d1 = dist_staged(rows, cn, i1, p);
    }
    __device__ uint32_t dist_pivot_staged(const uint32_t* pv, const uint32_t* rows, const uint32_t* cn, int i) const {
        const uint8_t* a = reinterpret_cast<const uint8_t*>(rows + (size_t)i * stage_stride_words());
        return u8_dist(cn[i], u8_dot(a, reinterpret_cast<const uint8_t*>(pv), D), pv[((D + 15) & ~15) / 4]);
    }
};

// ---- RaBitQ estimator (shared by the search kernel and RabitqMetric) --------
// RaBitQ estimator for one packed record (rabitq.py:235-244):
//   dd  = A1 dot(f32(u), rotated)           (einsum 'md,md->m')
//   est = max((qadd + data_add) + data_rescale * (dd - qsumq), 0)
// Full 16 B pieces are unrolled with compile-time bit positions. For m = 1,
// u*q is exactly q or +-0 and adding +-0 to an accumulator is a no-op, so the
// product/add pair becomes one predicated add with identical rounding.
template <int BITS>
__device__ __forceinline__ void rq_piece_full(Acc4& acc, const uint4 w4, const float* __restrict__ qv, int e0) {
    constexpr int PER16 = 128 / BITS;
    constexpr uint32_t MASK = (1u << BITS) - 1u;
    const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
    for (int blk = 0; blk < PER16 / 16; ++blk) {
#pragma unroll
        for (int i = 3; i >= 0; --i) {
            const float4 q4 = *reinterpret_cast<const float4*>(qv + e0 + blk * 16 + 4 * i);
            const float qq[4] = {q4.x, q4.y, q4.z, q4.w};
            float* lanes[4] = {&acc.l0, &acc.l1, &acc.l2, &acc.l3};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                constexpr int dummy = 0;
                (void)dummy;
                const int off = (blk * 16 + 4 * i + j) * BITS;
                const uint32_t code = (w[off >> 5] >> (off & 31)) & MASK;
                if (BITS == 1) {
                    if (code) *lanes[j] = __fadd_rn(qq[j], *lanes[j]);
                } else {
                    *lanes[j] = __fadd_rn(__fmul_rn((float)code, qq[j]), *lanes[j]);
                }
            }
        }
    }
}

// 16 B load from a global record (read-only path) or a smem-staged one
template <bool GL>
__device__ __forceinline__ uint4 ld16(const uint8_t* p) {
    if (GL) return __ldg(reinterpret_cast<const uint4*>(p));
    return *reinterpret_cast<const uint4*>(p);
}

// The record's last, partial code piece (D not a multiple of 128 / BITS): A1 order
// over 16-element blocks (vectors 3..0), then the tail forward.
template <int BITS>
__device__ __forceinline__ void rq_piece_partial(Acc4& acc, const uint4 w4, const float* __restrict__ qv, int e0,
                                                 int D) {
    constexpr uint32_t MASK = (1u << BITS) - 1u;
    const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
    int b = e0;
    for (; b + 16 <= D; b += 16) {
        for (int i = 3; i >= 0; --i) {
            for (int j = 0; j < 4; ++j) {
                const int off = (b - e0 + 4 * i + j) * BITS;
                acc.madd1(j, (float)((w[off >> 5] >> (off & 31)) & MASK), qv[b + 4 * i + j]);
            }
        }
    }
    for (; b < D; ++b) {
        const int off = (b - e0) * BITS;
        acc.madd1(b & 3, (float)((w[off >> 5] >> (off & 31)) & MASK), qv[b]);
    }
}

// 32 B load from global through the read-only path: one 256-bit LDG (sm_100), so a
// 32 B record (or half of a 64 B one) is one L1 request instead of two 16 B ones
// that both miss while the first is in flight (C5 ncu: 2x the L2 lookups of the
// sectors delivered). `p` must be 32 B aligned.
__device__ __forceinline__ void ldg32(const uint8_t* p, uint4& lo, uint4& hi) {
    asm volatile("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                 : "l"(p));
}

// <u, q> for one record whose first 16-byte code piece is already in registers
// (GL: the record is in global memory; else staged in smem).
template <int BITS, bool GL = true>
__device__ __forceinline__ float rabitq_dd(const uint8_t* __restrict__ rec, uint4 first, const float* __restrict__ qv,
                                           int D) {
    constexpr int PER16 = 128 / BITS;  // elements per 16-byte piece
    constexpr uint32_t MASK = (1u << BITS) - 1u;
    Acc4 acc; acc.zero();
    int e0 = 0;
    // the next piece's load is issued before this piece's adds (long records, e.g.
    // 480 B of 4-bit codes at D = 960, otherwise wait out one load latency per piece)
    uint4 cur = first;
    for (; e0 + PER16 <= D; e0 += PER16) {
        uint4 nxt = make_uint4(0, 0, 0, 0);
        if (e0 + PER16 < D) nxt = ld16<GL>(rec + ((e0 + PER16) * BITS) / 8);
        rq_piece_full<BITS>(acc, cur, qv, e0);
        cur = nxt;
    }
    if (e0 < D) rq_piece_partial<BITS>(acc, cur, qv, e0, D);  // last partial piece (rare shapes)
    return acc.reduce();
}

// rabitq_dd for a record held in registers as four 16 B pieces (64 B records: code
// of at most 48 B, so at most 3 code pieces); same accumulation order.
template <int BITS>
__device__ __forceinline__ float rabitq_dd_regs(const uint4 p0, const uint4 p1, const uint4 p2,
                                                const float* __restrict__ qv, int D) {
    constexpr int PER16 = 128 / BITS;
    Acc4 acc; acc.zero();
    int e0 = 0;
    if (e0 + PER16 <= D) { rq_piece_full<BITS>(acc, p0, qv, e0); e0 += PER16; }
    if (e0 + PER16 <= D) { rq_piece_full<BITS>(acc, p1, qv, e0); e0 += PER16; }
    if (e0 + PER16 <= D) { rq_piece_full<BITS>(acc, p2, qv, e0); e0 += PER16; }
    if (e0 < D) rq_piece_partial<BITS>(acc, e0 == 0 ? p0 : (e0 == PER16 ? p1 : p2), qv, e0, D);
    return acc.reduce();
}

// est = max((qadd + data_add) + data_rescale * (dd - qsumq), 0) in the reference's order
__device__ __forceinline__ float rabitq_finish(float dd, float2 m, float qadd, float qsumq) {
    const float est = __fadd_rn(__fadd_rn(qadd, m.x), __fmul_rn(m.y, __fsub_rn(dd, qsumq)));
    return est > 0.0f ? est : 0.0f;
}

template <int BITS>
__device__ __forceinline__ float rabitq_estimate(const uint8_t* __restrict__ rec, const float* __restrict__ qv,
                                                 int D, int meta_off, float qadd, float qsumq) {
    const uint4 first = __ldg(reinterpret_cast<const uint4*>(rec));
    const float dd = rabitq_dd<BITS>(rec, first, qv, D);
    return rabitq_finish(dd, __ldg(reinterpret_cast<const float2*>(rec + meta_off)), qadd, qsumq);
}


// Quantized construction (build.py:105-111, 124-129): every d(pivot, row) is the
// RaBitQ estimate of the row's code against the pivot's own row bound as a query
// (RaBitQIndex.bind(x[pivot]), rabitq.py:170-181). The bound rows (rotated f32,
// query_add, query_sumq) are computed once for the dataset by jb_rabitq_bind.
// No smem staging: candidates are 16-32 B records read in place.
template <int BITS>
struct RabitqMetric {
    const uint8_t* records;
    int record_bytes;
    const float* rotated;   // [count, D] bound rows
    const float* qadd;      // [count]
    const float* qsumq;     // [count]
    int D;
    static constexpr bool kInt = false;
    static constexpr bool kStage = false;
    __device__ void close_row(uint32_t, double) const {}
    __device__ void open_row(uint32_t) const {}
    __device__ bool row_closed(uint32_t, double) const { return false; }
    static constexpr bool kSplit = false;

    __host__ __device__ int meta_off() const { return ((((D * BITS) + 7) / 8 + 15) / 16) * 16; }
    __host__ __device__ int row_bytes() const { return record_bytes; }
    __host__ __device__ int stage_stride_words() const { return 4; }
    __host__ __device__ int pivot_words() const { return ((D + 3) & ~3) + 4; }
    __device__ static double value(uint32_t bits) { return (double)__uint_as_float(bits); }

    __device__ void load_pivot(uint32_t* pv, uint32_t v) const {
        const int lane = lane_id();
        const float* r = rotated + (size_t)v * D;
        float* f = reinterpret_cast<float*>(pv);
        for (int e = lane; e < D; e += 32) f[e] = r[e];
        if (lane == 0) {
            f[((D + 3) & ~3)] = qadd[v];
            f[((D + 3) & ~3) + 1] = qsumq[v];
        }
        __syncwarp();
    }
    __device__ void load_pivot_async(uint32_t* pv, uint32_t v) const { load_pivot(pv, v); }
    __device__ uint32_t dist(const uint32_t* pv, uint32_t row) const {
        const float* f = reinterpret_cast<const float*>(pv);
        const float est = rabitq_estimate<BITS>(records + (size_t)row * record_bytes, f, D, meta_off(),
                                                f[((D + 3) & ~3)], f[((D + 3) & ~3) + 1]);
        return __float_as_uint(est);
    }
    // never staged (the host passes crows = 0); present for the shared kernel bodies
    __device__ void stage(uint32_t*, uint32_t*, const uint64_t*, int, uint64_t* = nullptr, uint32_t* = nullptr) const {
        __trap();
    }
    __device__ uint32_t dist_staged(const uint32_t*, const uint32_t*, int, int) const { __trap(); return 0; }
    __device__ void dist_staged2(const uint32_t*, const uint32_t*, int, int, int, uint32_t&, uint32_t&) const {
        __trap();
    }
    __device__ uint32_t dist_pivot_staged(const uint32_t*, const uint32_t*, const uint32_t*, int) const {
        __trap();
        return 0;
    }
};

}  // namespace jb
