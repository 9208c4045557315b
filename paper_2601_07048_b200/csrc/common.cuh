// common.cuh — shared device helpers for the jasper_b200 kernels (sm_100a).
//
// The "A1" helpers reproduce numpy 2.x einsum('md,md->m') for f32 bit-exactly:
// 4 accumulator lanes (element e feeds lane e % 4), separate multiply and add
// (no FMA), full 16-element blocks visited as 4-wide vectors 3,2,1,0, the tail
// forward, and the final reduce (l0 + l1) + (l2 + l3). The f64 variant uses 2
// lanes, 8-element blocks, vectors 3,2,1,0. Verified against numpy for
// D in {1..1536} (re-probed in this repo's tests).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace jb {

constexpr uint64_t UMAX = 0xFFFFFFFFFFFFFFFFull;
constexpr uint64_t EXPANDED = 0x80000000ull;       // low-word bit 31: device-only flag
constexpr uint32_t EMPTY_SLOT = 0xFFFFFFFFu;

__device__ __forceinline__ uint64_t key_mask(uint64_t k) { return k & ~EXPANDED; }
__device__ __forceinline__ uint32_t key_id(uint64_t k) { return (uint32_t)(k & 0x7FFFFFFFull); }
__device__ __forceinline__ float key_dist(uint64_t k) { return __uint_as_float((uint32_t)(k >> 32)); }

// search.py:139-145 (_pack_keys, float branch): hi = bits(max(d, 0)).
__device__ __forceinline__ uint64_t pack_key(float d, uint32_t id) {
    d = d > 0.0f ? d : 0.0f;  // np.maximum(d, 0) (d is never NaN for finite data)
    return ((uint64_t)__float_as_uint(d) << 32) | (uint64_t)id;
}

struct Acc4 {
    float l0, l1, l2, l3;
    __device__ __forceinline__ void zero() { l0 = l1 = l2 = l3 = 0.0f; }
    __device__ __forceinline__ float reduce() const {
        return __fadd_rn(__fadd_rn(l0, l1), __fadd_rn(l2, l3));
    }
    // acc[j] = a[j]*b[j] + acc[j]  (numpy SSE: mul then add, no contraction)
    __device__ __forceinline__ void madd(const float4 a, const float4 b) {
        l0 = __fadd_rn(__fmul_rn(a.x, b.x), l0);
        l1 = __fadd_rn(__fmul_rn(a.y, b.y), l1);
        l2 = __fadd_rn(__fmul_rn(a.z, b.z), l2);
        l3 = __fadd_rn(__fmul_rn(a.w, b.w), l3);
    }
    // diff-square: (a-b)^2 per lane, used by the exact rerank (search.py:318-320)
    __device__ __forceinline__ void dsq(const float4 a, const float4 b) {
        float x = __fsub_rn(a.x, b.x), y = __fsub_rn(a.y, b.y);
        float z = __fsub_rn(a.z, b.z), w = __fsub_rn(a.w, b.w);
        l0 = __fadd_rn(__fmul_rn(x, x), l0);
        l1 = __fadd_rn(__fmul_rn(y, y), l1);
        l2 = __fadd_rn(__fmul_rn(z, z), l2);
        l3 = __fadd_rn(__fmul_rn(w, w), l3);
    }
    __device__ __forceinline__ void madd1(int lane, float a, float b) {
        float p = __fmul_rn(a, b);
        if (lane == 0) l0 = __fadd_rn(p, l0);
        else if (lane == 1) l1 = __fadd_rn(p, l1);
        else if (lane == 2) l2 = __fadd_rn(p, l2);
        else l3 = __fadd_rn(p, l3);
    }
    __device__ __forceinline__ void dsq1(int lane, float a, float b) {
        float d = __fsub_rn(a, b);
        madd1(lane, d, d);
    }
};

// A1 dot over elements [e0, e1) of two rows; e0 must be a multiple of 16 and
// e1 either a multiple of 16 or the row end D. Pointers address element 0.
// Both rows must be 16-byte aligned when ALIGNED (D % 4 == 0 rows).
template <bool ALIGNED, bool DIFF>
__device__ __forceinline__ void a1_range(Acc4& acc, const float* __restrict__ a,
                                         const float* __restrict__ b, int e0, int e1) {
    int e = e0;
    if (ALIGNED) {
        for (; e + 16 <= e1; e += 16) {
            const float4* av = reinterpret_cast<const float4*>(a + e);
            const float4* bv = reinterpret_cast<const float4*>(b + e);
            float4 a3 = av[3], a2 = av[2], a1 = av[1], a0 = av[0];
            float4 b3 = bv[3], b2 = bv[2], b1 = bv[1], b0 = bv[0];
            if (DIFF) { acc.dsq(a3, b3); acc.dsq(a2, b2); acc.dsq(a1, b1); acc.dsq(a0, b0); }
            else { acc.madd(a3, b3); acc.madd(a2, b2); acc.madd(a1, b1); acc.madd(a0, b0); }
        }
    } else {
        for (; e + 16 <= e1; e += 16) {
#pragma unroll
            for (int i = 3; i >= 0; --i) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (DIFF) acc.dsq1(j, a[e + 4 * i + j], b[e + 4 * i + j]);
                    else acc.madd1(j, a[e + 4 * i + j], b[e + 4 * i + j]);
                }
            }
        }
    }
    // tail: forward, groups of 4, zero fill (zero products are no-op adds)
    for (; e < e1; ++e) {
        if (DIFF) acc.dsq1(e & 3, a[e], b[e]);
        else acc.madd1(e & 3, a[e], b[e]);
    }
}

// Full-row A1 dot (einsum 'md,md->m' for one row pair).
template <bool DIFF = false>
__device__ __forceinline__ float a1_dot(const float* a, const float* b, int D) {
    Acc4 acc; acc.zero();
    if ((D & 3) == 0 && ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0)
        a1_range<true, DIFF>(acc, a, b, 0, D);
    else
        a1_range<false, DIFF>(acc, a, b, 0, D);
    return acc.reduce();
}

// The reference's exact distance with rows in the data role and the pivot /
// query norm added last: max((xn - 2*dot) + qn, 0) (search.py:126-130,
// build.py:130-134).
__device__ __forceinline__ float exact_from_dot(float xn, float dot, float qn) {
    float d = __fadd_rn(__fsub_rn(xn, __fmul_rn(2.0f, dot)), qn);
    return d > 0.0f ? d : 0.0f;
}

// f64 2-lane einsum order ('nd,nd->n' on f64).
struct Acc2d {
    double l0, l1;
    __device__ __forceinline__ void zero() { l0 = l1 = 0.0; }
    __device__ __forceinline__ double reduce() const { return __dadd_rn(l0, l1); }
};

// ---- warp helpers ------------------------------------------------------
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m;
}

__device__ __forceinline__ uint64_t shfl_xor_u64(uint64_t v, int m) {
    return __shfl_xor_sync(0xFFFFFFFFu, v, m);
}
__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
    return __shfl_sync(0xFFFFFFFFu, v, src);
}

// Ascending bitonic sort of one u64 per lane across the warp.
__device__ __forceinline__ uint64_t warp_sort_u64(uint64_t v) {
    const int lane = lane_id();
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            uint64_t o = shfl_xor_u64(v, j);
            bool up = (lane & k) == 0;
            bool lower = (lane & j) == 0;
            bool take_min = (lower == up);
            v = take_min ? (o < v ? o : v) : (o > v ? o : v);
        }
    }
    return v;
}

// Sort n (power of two, >= 32) u64 keys in shared memory, ascending, by one warp.
__device__ __forceinline__ void warp_bitonic_sort_smem(uint64_t* s, int n) {
    const int lane = lane_id();
    for (int k = 2; k <= n; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < n; i += 32) {
                int ixj = i ^ j;
                if (ixj > i) {
                    uint64_t a = s[i], b = s[ixj];
                    bool up = (i & k) == 0;
                    if ((a > b) == up) { s[i] = b; s[ixj] = a; }
                }
            }
            __syncwarp();
        }
    }
}

// lower_bound over a sorted u64 array (masked compare). Branch-free halving: the
// trip count depends on n only, so the lanes of a warp (same n) stay converged.
__device__ __forceinline__ int lower_bound_masked(const uint64_t* a, int n, uint64_t key) {
    int base = 0, len = n;
    while (len > 1) {
        const int half = len >> 1;
        base += (key_mask(a[base + half - 1]) < key) ? half : 0;
        len -= half;
    }
    return base + ((len == 1 && key_mask(a[base]) < key) ? 1 : 0);
}

// cp.async helpers (LDGSTS on sm_100a)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// ---- per-warp bulk row staging (the copy engine's cp.async.bulk, sm_90+) -----
// One lane per row issues one bulk copy (16 B multiples, 16 B aligned); completion
// is counted in bytes on a per-warp mbarrier (count 1: lane 0's expect_tx arrive).
// Replaces a warp-wide loop of 16 B cp.async per row: one instruction per row.
__device__ __forceinline__ void wbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// lane 0 announces `bytes`, then each lane with a row issues its copy; every lane
// must have finished reading the destination rows (generic proxy) before: the
// proxy fence + __syncwarp order those reads before the async writes
__device__ __forceinline__ void wbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if ((threadIdx.x & 31) == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(bar)),
                     "r"(bytes)
                     : "memory");
    __syncwarp();
}
__device__ __forceinline__ void bulk_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
                 : "memory");
}
__device__ __forceinline__ void wbar_wait(uint64_t* bar, uint32_t& phase) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(phase)
            : "memory");
    }
    phase ^= 1;
}

}  // namespace jb
