// build.cu — batch-parallel, lock-free construction and streaming insertion.
//
// Replaces the reference's build.py:
//   batch_insert          build.py:296-348  (jb_batch_insert: three phases + repair)
//   _seed_batch           build.py:246-266  (seed_prune_kernel)
//   robust_prune          graph.py:174-228  (warp_prune, one warp per pivot)
//   EdgeBuffer + _merge_reverse_edges  build.py:65-102, 269-293
//                         (per-source triple slots, two stable radix sorts giving
//                          (target, dist, source) order, one owner warp per target)
//   _repair_connectivity  build.py:137-224  (GPU BFS, tiled nearest-donor scan,
//                          ordered sequential attach on one warp)
//
// Lock-freedom: phase 2 writes only the new vertex's own row; phase 3 groups the
// reverse triples by target so exactly one warp owns each written row. Results do
// not depend on scheduling: triple order is fixed by the sort keys, not by atomics.
//
// Robust prune without a sort: the reference sorts candidates by (dist, id) and
// repeatedly takes the first survivor. Taking the minimum (dist, id) key among
// survivors each round extracts the same sequence, and the alpha filter is
// element-wise, so the kept list is identical.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>
#include <cub/cub.cuh>
#include "common.cuh"
#include "metric.cuh"
#include "runtime.cuh"
#include "donor_tc.cuh"

namespace jb {

constexpr int BW = 4;  // warps per block in the per-vertex kernels
#ifndef JB_OWNER_BW
#define JB_OWNER_BW 3  // 9 warps/SM instead of 8 at ~24 KB per warp: merge 29.9 -> 29.1 ms per batch at 3M
#endif
#ifndef JB_P2_BW
#define JB_P2_BW 1
#endif
#ifndef JB_P2_ROWS_OVER_L
#define JB_P2_ROWS_OVER_L 16  // phase-2 staged trace rows = L_build + this (traces average ~70 candidates at
                              // L_build = 64; at 3M x 96: 68 rows 16.3 ms, 76 rows 7.0 ms, 84 rows 7.6 ms)
#endif
constexpr int P2_BW = JB_P2_BW;  // warps per block of phase 2 (smem-bound by the staged traces)
constexpr int OWNER_BW = JB_OWNER_BW;  // warps per block of the deferred owner pass (smem-bound)
#ifndef JB_STAGE_KB
#define JB_STAGE_KB 26     // per-warp smem budget for staged candidate rows
#endif
#ifndef JB_P2_KB
#define JB_P2_KB 100  // phase-2 (new vertex) prune staging budget per warp (cap; the rows set the size)
#endif
#ifndef JB_OWNER_EXTRA
#define JB_OWNER_EXTRA 16  // owner-merge staging: up to R + this many candidate rows
#endif
constexpr uint32_t NO_TARGET = 0xFFFFFFFFu;

// d(pivot, row) with the row in the data role and the pivot norm added last
// (build.py:130-134): max((xn[row] - 2*dot(x[row], x[pivot])) + xn[pivot], 0).
// f32 only: the standalone robust_prune entry point (jb_robust_prune).
__device__ __forceinline__ float pair_dist(const float* __restrict__ data, const float* __restrict__ norms, int D,
                                           const float* __restrict__ pivot_row, float pivot_norm, uint32_t row) {
    const float dot = a1_dot<false>(data + (size_t)row * D, pivot_row, D);
    return exact_from_dot(__ldg(norms + row), dot, pivot_norm);
}

__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint64_t w = shfl_xor_u64(v, o);
        v = w < v ? w : v;
    }
    return v;
}

__device__ __forceinline__ uint64_t key_of(uint32_t bits, uint32_t id) { return ((uint64_t)bits << 32) | id; }

// Warp-cooperative robust prune over n candidate keys (dist_bits << 32 | id) in
// `cand` (modified in place). Writes kept ids / dist bits (extraction order) and
// returns how many were kept. `pv` is per-warp smem for the star (M::pivot_words).
template <class M>
__device__ int warp_prune(uint64_t* cand, int n, double alpha2, int R, const M& m, uint32_t* pv, int32_t* out_ids,
                          uint32_t* out_d) {
    const int lane = lane_id();
    int kept = 0;
    while (kept < R) {
        uint64_t mk = UMAX;
        for (int i = lane; i < n; i += 32) { uint64_t c = cand[i]; mk = c < mk ? c : mk; }
        mk = warp_min_u64(mk);
        if (mk == UMAX) break;
        const uint32_t star = (uint32_t)(mk & 0xFFFFFFFFull);
        if (lane == 0) {
            out_ids[kept] = (int32_t)star;
            out_d[kept] = (uint32_t)(mk >> 32);
        }
        for (int i = lane; i < n; i += 32)
            if (cand[i] == mk) cand[i] = UMAX;
        ++kept;
        if (kept >= R) break;
        // keep p' iff alpha^2 * d(star, p') > d(p, p')   (graph.py:218, f64)
        __syncwarp();
        m.load_pivot(pv, star);
        for (int i = lane; i < n; i += 32) {
            const uint64_t c = cand[i];
            if (c == UMAX) continue;
            const uint32_t dsp = m.dist(pv, (uint32_t)(c & 0xFFFFFFFFull));
            if (!(__dmul_rn(alpha2, M::value(dsp)) > M::value((uint32_t)(c >> 32)))) cand[i] = UMAX;
        }
        __syncwarp();
    }
    __syncwarp();
    return kept;
}

// Robust prune with every candidate row already staged in smem (rows[i] <-> cand[i]):
// same extraction sequence as warp_prune, no global traffic in the rounds.
// One prune round over the survivor list (star excluded, marked UMAX), F threads
// per pair of survivors: with few survivors left, the lanes share each distance
// instead of idling (F = 4 below 16 survivors, 2 below 32).
template <int F, class M>
__device__ __forceinline__ void split_round(uint64_t* cand, const uint16_t* lst, int s, int p, double alpha2,
                                            const M& m, const uint32_t* rows, const uint32_t* cn) {
    constexpr int G = 32 / F;
    const int lane = lane_id(), g = lane / F, sub = lane % F;
    const float pn = __uint_as_float(cn[p]);
    for (int base = 0; base < s; base += 2 * G) {
        const int j0 = base + g, j1 = base + G + g;
        const int i0 = j0 < s ? lst[j0] : p, i1 = j1 < s ? lst[j1] : p;
        const uint64_t c0 = j0 < s ? cand[i0] : UMAX, c1 = j1 < s ? cand[i1] : UMAX;
        if (!__any_sync(0xFFFFFFFFu, c0 != UMAX || c1 != UMAX)) continue;
        float t0, t1;
        m.template dot2_split<F>(rows, i0, i1, p, sub, t0, t1);
        if (sub == 0) {
            if (c0 != UMAX) {
                const float d0 = exact_from_dot(__uint_as_float(cn[i0]), t0, pn);
                if (!(__dmul_rn(alpha2, (double)d0) > M::value((uint32_t)(c0 >> 32)))) cand[i0] = UMAX;
            }
            if (c1 != UMAX) {
                const float d1 = exact_from_dot(__uint_as_float(cn[i1]), t1, pn);
                if (!(__dmul_rn(alpha2, (double)d1) > M::value((uint32_t)(c1 >> 32)))) cand[i1] = UMAX;
            }
        }
    }
}

// Staged prune over a compacted survivor list (u16 indices into cand/rows): the
// same extraction sequence as warp_prune; each round's argmin and distance pass
// touch only the survivors, and the distance pass picks F by their count.
template <class M>
__device__ int warp_prune_split(uint64_t* cand, int n, double alpha2, int R, const M& m, const uint32_t* rows,
                                const uint32_t* cn, uint16_t* lst, int32_t* out_ids, uint32_t* out_d) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = lane_id();
    for (int j = lane; j < n; j += 32) lst[j] = (uint16_t)j;
    __syncwarp();
    int s = n, kept = 0;
    while (kept < R && s > 0) {
        uint64_t mk = UMAX;
        int mi = -1;
        for (int j = lane; j < s; j += 32) {
            const int i = lst[j];
            const uint64_t c = cand[i];
            if (c < mk) { mk = c; mi = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t om = shfl_xor_u64(mk, o);
            const int oi = __shfl_xor_sync(FULL, mi, o);
            if (om < mk) { mk = om; mi = oi; }
        }
        if (mk == UMAX) break;
        __syncwarp();  // every lane's argmin reads of cand precede lane 0's write (WAR)
        if (lane == 0) {
            out_ids[kept] = (int32_t)(mk & 0xFFFFFFFFull);
            out_d[kept] = (uint32_t)(mk >> 32);
            cand[mi] = UMAX;
        }
        ++kept;
        __syncwarp();
        if (kept >= R) break;
        if (s <= 16) split_round<4>(cand, lst, s, mi, alpha2, m, rows, cn);
        else if (s <= 32) split_round<2>(cand, lst, s, mi, alpha2, m, rows, cn);
        else split_round<1>(cand, lst, s, mi, alpha2, m, rows, cn);
        __syncwarp();
        int ns = 0;  // compact: entries only move down, within the chunk being read
        for (int b = 0; b < s; b += 32) {
            const int j = b + lane;
            int i = 0;
            bool live = false;
            if (j < s) { i = lst[j]; live = cand[i] != UMAX; }
            const unsigned msk = __ballot_sync(FULL, live);
            __syncwarp();  // every lane's read of this chunk precedes the writes below (WAR)
            if (live) lst[ns + __popc(msk & lanemask_lt())] = (uint16_t)i;
            ns += __popc(msk);
            __syncwarp();
        }
        s = ns;
    }
    __syncwarp();
    return kept;
}

// the metric as passed to the kernels that take the split staged prune
template <class M>
static M split_prune(M m) {
    if constexpr (M::kSplit) m.split = true;
    return m;
}

template <class M>
__device__ int warp_prune_staged(uint64_t* cand, int n, double alpha2, int R, const M& m, const uint32_t* rows,
                                 const uint32_t* cn, uint16_t* lst, int32_t* out_ids, uint32_t* out_d) {
    if constexpr (M::kSplit) {
        if (m.split_ok()) return warp_prune_split(cand, n, alpha2, R, m, rows, cn, lst, out_ids, out_d);
    }
    (void)lst;
    const int lane = lane_id();
    int kept = 0;
    while (kept < R) {
        uint64_t mk = UMAX;
        int mi = -1;
        for (int i = lane; i < n; i += 32) {
            const uint64_t c = cand[i];
            if (c < mk) { mk = c; mi = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t om = shfl_xor_u64(mk, o);
            const int oi = __shfl_xor_sync(0xFFFFFFFFu, mi, o);
            if (om < mk) { mk = om; mi = oi; }
        }
        if (mk == UMAX) break;
        __syncwarp();  // every lane's argmin reads of cand precede lane 0's write (WAR)
        if (lane == 0) {
            out_ids[kept] = (int32_t)(mk & 0xFFFFFFFFull);
            out_d[kept] = (uint32_t)(mk >> 32);
            cand[mi] = UMAX;
        }
        ++kept;
        __syncwarp();
        if (kept >= R) break;
        // survivors two per lane per step (the second slot is i + 32), sharing the star's reads
        for (int i = lane; i < n; i += 64) {
            const int i2 = i + 32;
            const uint64_t c = cand[i];
            const uint64_t c2 = i2 < n ? cand[i2] : UMAX;
            const bool pair = c != UMAX && c2 != UMAX;
            if (__any_sync(__activemask(), pair)) {
                // one code path for the warp: single-survivor lanes run the pair routine
                // with their row twice instead of diverging into the single routine
                if (c != UMAX || c2 != UMAX) {
                    const int ia = c != UMAX ? i : i2;
                    const int ib = pair ? i2 : ia;
                    uint32_t d0, d1;
                    m.dist_staged2(rows, cn, ia, ib, mi, d0, d1);
                    const uint64_t ca = c != UMAX ? c : c2;
                    if (!(__dmul_rn(alpha2, M::value(d0)) > M::value((uint32_t)(ca >> 32)))) cand[ia] = UMAX;
                    if (pair && !(__dmul_rn(alpha2, M::value(d1)) > M::value((uint32_t)(c2 >> 32)))) cand[i2] = UMAX;
                }
            } else if (c != UMAX || c2 != UMAX) {
                const int ii = c != UMAX ? i : i2;
                const uint64_t cc = c != UMAX ? c : c2;
                const uint32_t dsp = m.dist_staged(rows, cn, ii, mi);
                if (!(__dmul_rn(alpha2, M::value(dsp)) > M::value((uint32_t)(cc >> 32)))) cand[ii] = UMAX;
            }
        }
        __syncwarp();
    }
    __syncwarp();
    return kept;
}

// ---- Gram-screened robust prune (f32 rows, staged, n <= GP_MAX) ---------------
// Same extraction sequence and result as warp_prune_staged. The candidates are
// ranked once by key (the extraction order of the reference's argmin loop,
// graph.py:205-226: keys are distinct), and each round's alpha test
//   remove c  iff  alpha^2 * d(p, c) <= d(t, c)          (graph.py:218, f64)
// is first decided from a tensor-core Gram block: G[p][c] = <x_p, x_c> on tf32
// mma.sync (m16n8k8, f32 accumulate) for the 16 ranked candidates of p's block
// against all n. With d~ = |p|^2 + |c|^2 - 2 G and |d~ - d_A1(p, c)| <= E (|p|^2 + |c|^2)
// (E = 2^-8: tf32 operands carry 2^-10 relative error, 2x margin as in donor_tc.cu),
// the test is certain when alpha^2 (d~ - err) > d(t, c) (keep) or alpha^2 (d~ + err)
// <= d(t, c) (remove); only the rest get the exact A1 distance. Per warp smem:
// ranked index list (GP_MAX bytes) + one Gram block (16 x GP_MAX f32).
// (A warp-level product: tcgen05's 128-row tiles and per-CTA issue do not fit a
// per-warp 48 x 48 x D Gram; the exact A1 rounds it replaces were ~45% of the
// owner merge's instructions.)
#ifndef JB_GP_MAX
#define JB_GP_MAX 48  // = the owner staging limit at R = 32 (R + 16); 64 cost occupancy: merge 32.4 vs 29.6 ms per batch at 3M
#endif
constexpr int GP_MAX = JB_GP_MAX;  // candidates per Gram-screened prune (multiple of 16, <= 64)
// Gram block | ranked norms | ranks | closed-row prune: 16 x 2 domination masks + 16 fresh positions
constexpr int GP_BYTES = ((16 * GP_MAX * 4 + GP_MAX * 4 + GP_MAX + 7) & ~7) + 16 * 8 * 2 + 32;

__device__ __forceinline__ void mma_tf32_16x8x8(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                                uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
        "{%0, %1, %2, %3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Gram block of ranked positions [16 b, 16 b + 16) x [16 b, n): gb[i][c] (row stride GP_MAX).
// Rows are staged with stride rs (natural or block-transposed: the same element
// permutation in every row leaves dot products unchanged). D % 8 == 0.
__device__ __forceinline__ void gram_block(const uint32_t* __restrict__ rows, int rs, int D, const uint8_t* rk, int n,
                                           int b, float* __restrict__ gb) {
    const int lane = lane_id(), g = lane >> 2, t = lane & 3;
    const int r0 = 16 * b + g, r1 = r0 + 8;
    const uint32_t* pa0 = rows + (size_t)rk[r0 < n ? r0 : 0] * rs + t;
    const uint32_t* pa1 = rows + (size_t)rk[r1 < n ? r1 : 0] * rs + t;
    const int j0 = 2 * b, nj = (n + 7) >> 3;  // column blocks of 8 (positions < 16 b are never tested)
    float acc[GP_MAX / 8][4];
    const uint32_t* pb[GP_MAX / 8];
#pragma unroll
    for (int j = 0; j < GP_MAX / 8; ++j) {
        acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
        const int c = 8 * j + g;
        pb[j] = rows + (size_t)rk[c < n ? c : 0] * rs + t;
    }
    for (int k = 0; k < D; k += 8) {
        const uint32_t a0 = pa0[k], a1 = pa1[k], a2 = pa0[k + 4], a3 = pa1[k + 4];
#pragma unroll
        for (int j = 0; j < GP_MAX / 8; ++j)
            if (j >= j0 && j < nj) mma_tf32_16x8x8(acc[j], a0, a1, a2, a3, pb[j][k], pb[j][k + 4]);
    }
#pragma unroll
    for (int j = 0; j < GP_MAX / 8; ++j) {
        if (j >= j0 && j < nj) {
            *reinterpret_cast<float2*>(gb + g * GP_MAX + 8 * j + 2 * t) = make_float2(acc[j][0], acc[j][1]);
            *reinterpret_cast<float2*>(gb + (g + 8) * GP_MAX + 8 * j + 2 * t) = make_float2(acc[j][2], acc[j][3]);
        }
    }
}

// Gram rows of an explicit candidate list (arow[0 .. na), na <= 16) against every
// ranked position: gb[i][c] = <x_arow[i], x_rk[c]> for c < n (row stride GP_MAX).
__device__ __forceinline__ void gram_rows(const uint32_t* __restrict__ rows, int rs, int D, const uint8_t* arow, int na,
                                          const uint8_t* rk, int n, float* __restrict__ gb) {
    const int lane = lane_id(), g = lane >> 2, t = lane & 3;
    const uint32_t* pa0 = rows + (size_t)arow[g < na ? g : 0] * rs + t;
    const uint32_t* pa1 = rows + (size_t)arow[g + 8 < na ? g + 8 : 0] * rs + t;
    const int nj = (n + 7) >> 3;
    float acc[GP_MAX / 8][4];
    const uint32_t* pb[GP_MAX / 8];
#pragma unroll
    for (int j = 0; j < GP_MAX / 8; ++j) {
        acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
        const int c = 8 * j + g;
        pb[j] = rows + (size_t)rk[c < n ? c : 0] * rs + t;
    }
    for (int k = 0; k < D; k += 8) {
        const uint32_t a0 = pa0[k], a1 = pa1[k], a2 = pa0[k + 4], a3 = pa1[k + 4];
#pragma unroll
        for (int j = 0; j < GP_MAX / 8; ++j)
            if (j < nj) mma_tf32_16x8x8(acc[j], a0, a1, a2, a3, pb[j][k], pb[j][k + 4]);
    }
#pragma unroll
    for (int j = 0; j < GP_MAX / 8; ++j) {
        if (j < nj) {
            *reinterpret_cast<float2*>(gb + g * GP_MAX + 8 * j + 2 * t) = make_float2(acc[j][0], acc[j][1]);
            if (na > 8)
                *reinterpret_cast<float2*>(gb + (g + 8) * GP_MAX + 8 * j + 2 * t) = make_float2(acc[j][2], acc[j][3]);
        }
    }
}

// exact A1 dot of staged rows i and p (per lane; natural or block-transposed layout)
__device__ __forceinline__ float staged_dot(const F32Metric& m, const uint32_t* rows, int i, int p) {
    const int rs = m.stage_stride_words();
    if (m.split_ok()) {  // transposed 16-blocks: float4 k of a block holds chain k's 4 elements, vectors 3..0 in .w..x
        const float4* a = reinterpret_cast<const float4*>(rows + (size_t)i * rs);
        const float4* b = reinterpret_cast<const float4*>(rows + (size_t)p * rs);
        Acc4 acc; acc.zero();
        float* l[4] = {&acc.l0, &acc.l1, &acc.l2, &acc.l3};
        for (int v = 0; v < (m.D >> 2); v += 4) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float4 u = a[v + k], w = b[v + k];
                *l[k] = __fadd_rn(__fmul_rn(u.w, w.w), *l[k]);
                *l[k] = __fadd_rn(__fmul_rn(u.z, w.z), *l[k]);
                *l[k] = __fadd_rn(__fmul_rn(u.y, w.y), *l[k]);
                *l[k] = __fadd_rn(__fmul_rn(u.x, w.x), *l[k]);
            }
        }
        return acc.reduce();
    }
    const float* a = reinterpret_cast<const float*>(rows + (size_t)i * rs);
    const float* b = reinterpret_cast<const float*>(rows + (size_t)p * rs);
    Acc4 acc; acc.zero();
    a1_range<true, false>(acc, a, b, 0, m.D);
    return acc.reduce();
}

__device__ int warp_prune_gram(uint64_t* cand, int n, double alpha2, int R, const F32Metric& m, const uint32_t* rows,
                               const uint32_t* cn, uint8_t* rk, float* gb, int32_t* out_ids, uint32_t* out_d,
                               int hd_closed = -1) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = lane_id();
    const int rs = m.stage_stride_words();
    float* snorm = gb + 16 * GP_MAX;  // |x|^2 of ranked positions
    // rank by key: rk[rank] = candidate index
    {
        const uint64_t k0 = lane < n ? cand[lane] : UMAX, k1 = lane + 32 < n ? cand[lane + 32] : UMAX;
        int c0 = 0, c1 = 0;
        for (int j = 0; j < n; ++j) {
            const uint64_t kj = cand[j];
            c0 += kj < k0;
            c1 += kj < k1;
        }
        if (lane < n) { rk[c0] = (uint8_t)lane; snorm[c0] = __uint_as_float(cn[lane]); }
        if (lane + 32 < n) { rk[c1] = (uint8_t)(lane + 32); snorm[c1] = __uint_as_float(cn[lane + 32]); }
        __syncwarp();
    }
    // this lane tests ranked positions lane and lane + 32
    const int i0 = lane < n ? rk[lane] : 0, i1 = lane + 32 < n ? rk[lane + 32] : 0;
    const uint64_t key0 = cand[i0], key1 = cand[i1];
    const float dt0 = __uint_as_float((uint32_t)(key0 >> 32)), dt1 = __uint_as_float((uint32_t)(key1 >> 32));
    const float n0 = __uint_as_float(cn[i0]), n1 = __uint_as_float(cn[i1]);
    // f32 screen with directed margins: a2lo <= alpha^2 <= a2hi; the (2^-8)(|p|^2 + |c|^2)
    // bound absorbs the screen's own f32 roundings (relative 2^-23 each) many times over
    const float a2lo = (float)alpha2 * (1.0f - 0x1p-20f), a2hi = (float)alpha2 * (1.0f + 0x1p-20f);
    const float E = 0x1p-8f;
    // one pair test, screened: does ranked position `s` (as the star) prune ranked `c`?
    // (alpha^2 d(s, c) <= d(t, c); d symmetric bit for bit, so one Gram entry serves both roles)
    auto prunes = [&](float g, float ns, float nc, float dtc, int is, int ic) -> bool {
        const float nn = ns + nc;
        const float dd = fmaf(-2.0f, g, nn);
        const float err = E * nn;
        if (a2lo * (dd - err) > dtc) return false;
        if (a2hi * (dd + err) < dtc) return true;
        const float d = exact_from_dot(__uint_as_float(cn[ic]), staged_dot(m, rows, ic, is), __uint_as_float(cn[is]));
        return !(__dmul_rn(alpha2, (double)d) > (double)dtc);
    };
    if (hd_closed >= 0 && n - hd_closed >= 1 && n - hd_closed <= 16) {
        // Closed row (its hd_closed existing members came out of a robust prune at
        // alpha_a^2 <= alpha^2, so none of them prunes another): only pairs with a
        // fresh source (candidate index >= hd_closed) can prune. Per fresh f:
        // doms[f] = ranked candidates after f that f prunes, domby[f] = ranked
        // candidates before f that prune f; one scan in rank order then keeps c iff
        // no kept candidate before it prunes it — the reference's extraction result.
        uint64_t* fdoms = reinterpret_cast<uint64_t*>(rk + GP_MAX);
        uint64_t* fdomby = fdoms + 16;
        uint8_t* fpos = reinterpret_cast<uint8_t*>(fdomby + 16);
        const bool fr0 = lane < n && i0 >= hd_closed, fr1 = lane + 32 < n && i1 >= hd_closed;
        const uint32_t fm0 = __ballot_sync(FULL, fr0), fm1 = __ballot_sync(FULL, fr1);
        const int nf = __popc(fm0) + __popc(fm1);
        if (fr0) fpos[__popc(fm0 & lanemask_lt())] = (uint8_t)lane;
        if (fr1) fpos[__popc(fm0) + __popc(fm1 & lanemask_lt())] = (uint8_t)(lane + 32);
        __syncwarp();
        uint8_t* arow = fpos + 16;  // candidate indices of the fresh rows (the Gram's A operand)
        if (lane < nf) arow[lane] = rk[fpos[lane]];
        __syncwarp();
        gram_rows(rows, rs, m.D, arow, nf, rk, n, gb);
        __syncwarp();
        for (int f = 0; f < nf; ++f) {
            const int pf = fpos[f];
            const int ifr = rk[pf];
            const float nfr = snorm[pf];
            const float dtf = __uint_as_float((uint32_t)(cand[ifr] >> 32));
            const float* grow = gb + f * GP_MAX;
            bool d0 = false, b0 = false, d1 = false, b1 = false;
            if (lane < n && lane != pf) {
                const float g = grow[lane];
                if (lane > pf) d0 = prunes(g, nfr, n0, dt0, ifr, i0);
                else b0 = prunes(g, n0, nfr, dtf, i0, ifr);
            }
            if (lane + 32 < n && lane + 32 != pf) {
                const float g = grow[lane + 32];
                if (lane + 32 > pf) d1 = prunes(g, nfr, n1, dt1, ifr, i1);
                else b1 = prunes(g, n1, nfr, dtf, i1, ifr);
            }
            const uint64_t dm = (uint64_t)__ballot_sync(FULL, d0) | ((uint64_t)__ballot_sync(FULL, d1) << 32);
            const uint64_t bm = (uint64_t)__ballot_sync(FULL, b0) | ((uint64_t)__ballot_sync(FULL, b1) << 32);
            if (lane == 0) { fdoms[f] = dm; fdomby[f] = bm; }
        }
        __syncwarp();
        const uint64_t fmask = (uint64_t)fm0 | ((uint64_t)fm1 << 32);
        uint64_t kept_mask = 0, kdoms = 0;
        int kept = 0, f = 0;
        for (int c = 0; c < n && kept < R; ++c) {
            bool dominated;
            const bool isf = (fmask >> c) & 1ull;
            if (isf) dominated = (fdomby[f] & kept_mask) != 0;
            else dominated = ((kdoms >> c) & 1ull) != 0;
            if (!dominated) {
                kept_mask |= 1ull << c;
                if (isf) kdoms |= fdoms[f];
                if (lane == 0) {
                    const uint64_t kc = cand[rk[c]];
                    out_ids[kept] = (int32_t)(kc & 0xFFFFFFFFull);
                    out_d[kept] = (uint32_t)(kc >> 32);
                }
                ++kept;
            }
            if (isf) ++f;
        }
        __syncwarp();
        return kept;
    }
    uint32_t alive0 = __ballot_sync(FULL, lane < n), alive1 = __ballot_sync(FULL, lane + 32 < n);
    int kept = 0, blk = -1;
    while (kept < R && (alive0 | alive1)) {
        const int p = alive0 ? __ffs(alive0) - 1 : 32 + __ffs(alive1) - 1;
        if (lane == 0) {
            const uint64_t kp = cand[rk[p]];
            out_ids[kept] = (int32_t)(kp & 0xFFFFFFFFull);
            out_d[kept] = (uint32_t)(kp >> 32);
        }
        if (p < 32) alive0 &= ~(1u << p); else alive1 &= ~(1u << (p - 32));
        ++kept;
        if (kept >= R || !(alive0 | alive1)) break;
        if ((p >> 4) != blk) {
            blk = p >> 4;
            __syncwarp();
            gram_block(rows, rs, m.D, rk, n, blk, gb);
            __syncwarp();
        }
        const float np = snorm[p];
        const float* grow = gb + (p & 15) * GP_MAX;
        bool rm0 = false, rm1 = false;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const bool live = ((h ? alive1 : alive0) >> lane) & 1u;
            if (!live) continue;
            const float nc = h ? n1 : n0, dtc = h ? dt1 : dt0;
            const float nn = np + nc;
            const float dd = fmaf(-2.0f, grow[lane + 32 * h], nn);
            const float err = E * nn;
            bool rm;
            if (a2lo * (dd - err) > dtc) rm = false;         // certainly kept
            else if (a2hi * (dd + err) < dtc) rm = true;     // certainly pruned
            else {                                           // exact A1 distance, f64 test as the reference
                const int ic = h ? i1 : i0, ip = rk[p];
                const float d = exact_from_dot(__uint_as_float(cn[ic]), staged_dot(m, rows, ic, ip),
                                               __uint_as_float(cn[ip]));
                rm = !(__dmul_rn(alpha2, (double)d) > (double)dtc);
            }
            if (h) rm1 = rm; else rm0 = rm;
        }
        alive0 &= ~__ballot_sync(FULL, rm0);
        alive1 &= ~__ballot_sync(FULL, rm1);
    }
    __syncwarp();
    return kept;
}

// Every row written here is the output of a robust prune at alpha2: the row is
// recorded as closed at alpha2 (F32 builds with closure tracking; else a no-op).
template <class M>
__device__ __forceinline__ void write_row(const M& m, double alpha2, int32_t* __restrict__ adj,
                                          int32_t* __restrict__ deg, int R, uint32_t v, const int32_t* ids, int n) {
    const int lane = lane_id();
    for (int j = lane; j < R; j += 32) adj[(size_t)v * R + j] = j < n ? ids[j] : -1;
    if (lane == 0) {
        deg[v] = n;
        m.close_row(v, alpha2);
    }
}

// Per-warp smem of the per-vertex kernels:
// pivot | staged rows (crows) | their norms | u16 survivor list (split prune)
template <class M>
__host__ __device__ inline int vertex_warp_words(const M& m, int crows) {
    return m.pivot_words() + crows * m.stage_stride_words() + ((crows + 3) & ~3) + ((crows + 7) & ~7) / 2 + 4;
}
// per-warp mbarrier of the bulk row staging (after the survivor list; 16 B aligned)
__device__ __forceinline__ uint64_t* stage_bar(uint32_t* cn, int crows) {
    return reinterpret_cast<uint64_t*>(cn + ((crows + 3) & ~3) + ((crows + 7) & ~7) / 2);
}
// lane 0 initialises the warp's staging barrier (once per kernel, before any stage())
__device__ __forceinline__ uint64_t* init_stage_bar(uint32_t* cn, int crows) {
    uint64_t* b = stage_bar(cn, crows);
    if (crows > 0 && lane_id() == 0) wbar_init(b);
    __syncwarp();
    return b;
}
__device__ __forceinline__ uint16_t* stage_list(uint32_t* cn, int crows) {
    return reinterpret_cast<uint16_t*>(cn + ((crows + 3) & ~3));
}

// ---- seed batch (build.py:246-266) ------------------------------------------
template <class M>
__global__ void __launch_bounds__(BW * 32)
seed_prune_kernel(const M m, int64_t start, int64_t stop, int64_t xi0, int64_t xi1, double alpha2, int R,
                  uint64_t* __restrict__ cand_all, int32_t* __restrict__ kept_ids, uint32_t* __restrict__ kept_d,
                  int32_t* __restrict__ adj, int32_t* __restrict__ deg) {
    extern __shared__ __align__(16) uint32_t shw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* pv = shw + warp * m.pivot_words();
    const int64_t n = stop - start;
    const int64_t xi = xi0 + (int64_t)blockIdx.x * BW + warp;  // pivots [xi0, xi1) of this tile
    if (xi >= xi1) return;
    const uint32_t x = (uint32_t)(start + xi);
    uint64_t* cand = cand_all + (xi - xi0) * (n - 1);
    // candidate dists d(x, others) with x as the pivot
    m.load_pivot(pv, x);
    for (int64_t j = lane; j < n - 1; j += 32) {
        const uint32_t o = (uint32_t)(start + (j < xi ? j : j + 1));
        cand[j] = key_of(m.dist(pv, o), o);
    }
    __syncwarp();
    int32_t* ki = kept_ids + (xi - xi0) * R;
    uint32_t* kd = kept_d + (xi - xi0) * R;
    const int k = warp_prune(cand, (int)(n - 1), alpha2, R, m, pv, ki, kd);
    write_row(m, alpha2, adj, deg, R, x, ki, k);
}

// ---- int8-screened staged prune (phase 2 with screen records, f32 rows) ------
// The extraction sequence of warp_prune_split (argmin over the survivors, then the
// star's pair test against each survivor c: remove c iff !(alpha^2 d(p, c) > d(t, c)),
// graph.py:218), with the pair test decided from the staged int8 screen records
// (screen.cu) when the bound is certain: |p - c| lies within |p~ - c~| -/+ (eps_p +
// eps_c), |p~ - c~|^2 = s_p^2|b_p|^2 + s_c^2|b_c|^2 - 2 s_p s_c <b_p, b_c> (exact
// integer dot, f64 evaluation with 2^-40 slacks), and the f32 distance the reference
// compares differs from |p - c|^2 by at most M = (D + 32) 2^-24 (|p|^2 + |c|^2). Only
// undecided pairs read the two f32 rows (global, A1 order, the staged path's operand
// roles). Records are ~3.5x smaller than f32 rows, so ~3x more warps stage a trace.
__device__ int warp_prune_screen(uint64_t* cand, int n, double alpha2, int R, const F32Metric& m,
                                 const unsigned char* recs, int rb, uint16_t* lst, int32_t* out_ids, uint32_t* out_d) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = lane_id();
    const int dp = rb - 16;
    const double Mk = (double)(m.D + 32) * 0x1p-24;
    for (int j = lane; j < n; j += 32) lst[j] = (uint16_t)j;
    __syncwarp();
    int s = n, kept = 0;
    while (kept < R && s > 0) {
        uint64_t mk = UMAX;
        int mi = -1;
        for (int j = lane; j < s; j += 32) {
            const int i = lst[j];
            const uint64_t c = cand[i];
            if (c < mk) { mk = c; mi = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t om = shfl_xor_u64(mk, o);
            const int oi = __shfl_xor_sync(FULL, mi, o);
            if (om < mk) { mk = om; mi = oi; }
        }
        if (mk == UMAX) break;
        __syncwarp();  // every lane's argmin reads of cand precede lane 0's write (WAR)
        if (lane == 0) {
            out_ids[kept] = (int32_t)(mk & 0xFFFFFFFFull);
            out_d[kept] = (uint32_t)(mk >> 32);
            cand[mi] = UMAX;
        }
        ++kept;
        __syncwarp();
        if (kept >= R) break;
        const unsigned char* rp = recs + (size_t)mi * rb;
        const float4 mp = *reinterpret_cast<const float4*>(rp + dp);  // s, |b|^2, eps, |x|^2
        const uint32_t idp = (uint32_t)(mk & 0xFFFFFFFFull);
        for (int j = lane; j < s; j += 32) {
            const int i = lst[j];
            const uint64_t c = cand[i];
            if (c == UMAX) continue;
            const unsigned char* rc = recs + (size_t)i * rb;
            int dot = 0;
            for (int w = 0; w < dp; w += 16) {
                const uint4 a = *reinterpret_cast<const uint4*>(rc + w);
                const uint4 b = *reinterpret_cast<const uint4*>(rp + w);
                dot = __dp4a((int)a.x, (int)b.x, dot);
                dot = __dp4a((int)a.y, (int)b.y, dot);
                dot = __dp4a((int)a.z, (int)b.z, dot);
                dot = __dp4a((int)a.w, (int)b.w, dot);
            }
            const float4 mc = *reinterpret_cast<const float4*>(rc + dp);
            const double A = (double)mp.x * mp.x * mp.y, B = (double)mc.x * mc.x * mc.y;
            const double dd = (A + B) - 2.0 * (double)mp.x * (double)mc.x * (double)dot;
            const double sl = 0x1p-40 * (A + B);
            const double e = (double)mp.z + (double)mc.z;
            const double lo = fmax(sqrt(fmax(dd - sl, 0.0)) * (1.0 - 0x1p-40) - e, 0.0);
            const double hi = sqrt(dd + sl) * (1.0 + 0x1p-40) + e;
            const double M = Mk * ((double)mp.w + (double)mc.w);
            const double dlo = lo * lo * (1.0 - 0x1p-40) - M, dhi = hi * hi * (1.0 + 0x1p-40) + M;
            const double dtc = (double)__uint_as_float((uint32_t)(c >> 32));
            bool remove;
            if (alpha2 * dlo * (1.0 - 0x1p-40) > dtc) remove = false;
            else if (alpha2 * dhi * (1.0 + 0x1p-40) <= dtc) remove = true;
            else {  // undecided: the exact A1 distance (c in the data role, the star as the pivot)
                const uint32_t idc = (uint32_t)(c & 0xFFFFFFFFull);
                const float d = exact_from_dot(mc.w, a1_dot<false>(m.data + (size_t)idc * m.D, m.data + (size_t)idp * m.D,
                                                                  m.D), mp.w);
                remove = !(__dmul_rn(alpha2, (double)d) > dtc);
            }
            if (remove) cand[i] = UMAX;
        }
        __syncwarp();
        int ns = 0;  // compact: entries only move down, within the chunk being read
        for (int b = 0; b < s; b += 32) {
            const int j = b + lane;
            int i = 0;
            bool live = false;
            if (j < s) { i = lst[j]; live = cand[i] != UMAX; }
            const unsigned msk = __ballot_sync(FULL, live);
            __syncwarp();  // every lane's read of this chunk precedes the writes below (WAR)
            if (live) lst[ns + __popc(msk & lanemask_lt())] = (uint16_t)i;
            ns += __popc(msk);
            __syncwarp();
        }
        s = ns;
    }
    __syncwarp();
    return kept;
}

// phase 2 with screen records: per warp (1-warp blocks) srows staged records |
// u16 survivor list | staging mbarrier | pivot row (global-row prune of longer traces)
__host__ __device__ inline int p2s_warp_bytes(int srows, int rb, int D) {
    return ((srows * rb + srows * 2 + 15) & ~15) + 16 + ((((D + 3) & ~3) + 4) * 4);
}

__global__ void __launch_bounds__(32)
phase2_screen_kernel(const F32Metric m, const uint8_t* __restrict__ screen, int rb, int srows, int64_t start,
                     int64_t nb, double alpha2, int R, const int32_t* __restrict__ hops,
                     const int32_t* __restrict__ tids, const uint32_t* __restrict__ tdst, int cap, int reverse_all,
                     uint64_t* __restrict__ cand_all, int32_t* __restrict__ kept_ids, uint32_t* __restrict__ kept_d,
                     int32_t* __restrict__ adj, int32_t* __restrict__ deg, uint32_t* __restrict__ tri_target,
                     uint64_t* __restrict__ tri_key, int W) {
    extern __shared__ __align__(16) unsigned char shs[];
    const int lane = threadIdx.x & 31;
    unsigned char* recs = shs;
    uint16_t* lst = reinterpret_cast<uint16_t*>(shs + (size_t)srows * rb);
    uint64_t* bar = reinterpret_cast<uint64_t*>(shs + (((size_t)srows * rb + srows * 2 + 15) & ~(size_t)15));
    uint32_t* pv = reinterpret_cast<uint32_t*>(reinterpret_cast<unsigned char*>(bar) + 16);
    const int64_t xi = blockIdx.x;
    if (xi >= nb) return;
    if (lane == 0) wbar_init(bar);
    __syncwarp();
    uint32_t sph = 0;
    const uint32_t x = (uint32_t)(start + xi);
    const int h = min(hops[xi], cap);
    uint64_t* cand = cand_all + xi * cap;
    const int32_t* ti = tids + xi * cap;
    const uint32_t* td = tdst + xi * cap;
    for (int j = lane; j < h; j += 32) cand[j] = key_of(td[j], (uint32_t)ti[j]);
    __syncwarp();
    int32_t* ki = kept_ids + xi * R;
    uint32_t* kd = kept_d + xi * R;
    int k;
    if (h <= srows) {
        wbar_expect(bar, (uint32_t)h * (uint32_t)rb);
        for (int j = lane; j < h; j += 32)
            bulk_row(recs + (size_t)j * rb, screen + (size_t)(uint32_t)ti[j] * rb, (uint32_t)rb, bar);
        wbar_wait(bar, sph);
        __syncwarp();
        k = warp_prune_screen(cand, h, alpha2, R, m, recs, rb, lst, ki, kd);
    } else {
        k = warp_prune(cand, h, alpha2, R, m, pv, ki, kd);
    }
    write_row(m, alpha2, adj, deg, R, x, ki, k);
    uint32_t* tt = tri_target + xi * W;
    uint64_t* tk = tri_key + xi * W;
    const int ne = reverse_all ? h : k;
    for (int j = lane; j < W; j += 32) {
        if (j < ne) {
            tt[j] = reverse_all ? (uint32_t)ti[j] : (uint32_t)ki[j];
            tk[j] = key_of(reverse_all ? td[j] : kd[j], x);
        } else {
            tt[j] = NO_TARGET;
            tk[j] = UMAX;
        }
    }
}

// ---- phase 2: prune each new vertex's visited trace, emit reverse triples ----
// Trace distances are the search keys' 32-bit words (tdst holds their bits).
template <class M>
__global__ void __launch_bounds__(BW * 32)
phase2_kernel(const M m, int64_t start, int64_t nb, double alpha2, int R, const int32_t* __restrict__ hops,
              const int32_t* __restrict__ tids, const uint32_t* __restrict__ tdst, int cap, int reverse_all,
              uint64_t* __restrict__ cand_all, int32_t* __restrict__ kept_ids, uint32_t* __restrict__ kept_d,
              int32_t* __restrict__ adj, int32_t* __restrict__ deg, uint32_t* __restrict__ tri_target,
              uint64_t* __restrict__ tri_key, int W, int crows) {
    extern __shared__ __align__(16) uint32_t shw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* pv = shw + (size_t)warp * vertex_warp_words(m, crows);
    uint32_t* rows = pv + m.pivot_words();
    uint32_t* cn = rows + (size_t)crows * m.stage_stride_words();
    const int64_t xi = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;  // P2_BW-warp blocks
    if (xi >= nb) return;
    const uint32_t x = (uint32_t)(start + xi);
    const int h = min(hops[xi], cap);
    uint64_t* cand = cand_all + xi * cap;
    const int32_t* ti = tids + xi * cap;
    const uint32_t* td = tdst + xi * cap;
    for (int j = lane; j < h; j += 32) cand[j] = key_of(td[j], (uint32_t)ti[j]);
    __syncwarp();
    int32_t* ki = kept_ids + xi * R;
    uint32_t* kd = kept_d + xi * R;
    int k;
    if (h <= crows) {
        // (the Gram-screened prune measured no faster here: 17.9 vs 16.8 ms per 100K batch at
        // 3M, its extra smem costing what the screen saves; phase 2 is latency-bound)
        uint32_t sph = 0;
        m.stage(rows, cn, cand, h, init_stage_bar(cn, crows), &sph);
        k = warp_prune_staged(cand, h, alpha2, R, m, rows, cn, stage_list(cn, crows), ki, kd);
    } else {
        k = warp_prune(cand, h, alpha2, R, m, pv, ki, kd);
    }
    write_row(m, alpha2, adj, deg, R, x, ki, k);
    // reverse triples (target, source=x, dist): kept edges, or the whole trace
    uint32_t* tt = tri_target + xi * W;
    uint64_t* tk = tri_key + xi * W;
    const int ne = reverse_all ? h : k;
    for (int j = lane; j < W; j += 32) {
        if (j < ne) {
            tt[j] = reverse_all ? (uint32_t)ti[j] : (uint32_t)ki[j];
            tk[j] = key_of(reverse_all ? td[j] : kd[j], x);
        } else {
            tt[j] = NO_TARGET;
            tk[j] = UMAX;
        }
    }
}

// Block (256 threads) A1 dot matrix of N <= 128 f32 rows ids[0..N): 64 x 64 tile
// pairs (tI <= tJ; both orientations written, dot(a, b) == dot(b, a) bit for bit),
// 4 x 4 pairs per thread, k-steps of 16 elements in A1 order (vectors 3,2,1,0,
// then the tail forward), the next k-step prefetched into registers. S holds two
// 64 x 17 slices. Ends with __syncthreads().
__device__ void block_dot_matrix(const float* __restrict__ data, int D, const int32_t* ids, int N, float* S,
                                 float* dotm, int ld) {
    constexpr int KB = 16;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int srow = tid / KB, scol = tid % KB;
    const int nt = (N + 63) / 64;
    for (int tI = 0; tI < nt; ++tI) {
        for (int tJ = tI; tJ < nt; ++tJ) {
            const int nA = min(64, N - tI * 64), nB = min(64, N - tJ * 64);
            const bool same = tI == tJ;
            float* SA = S;
            float* SB = same ? S : S + 64 * 17;
            const bool live = ty * 4 < nA && tx * 4 < nB;
            float pa[4], pb[4];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const int r = srow + 16 * h;
                pa[h] = (r < nA && scol < D) ? __ldg(data + (size_t)ids[tI * 64 + r] * D + scol) : 0.0f;
                pb[h] = (!same && r < nB && scol < D) ? __ldg(data + (size_t)ids[tJ * 64 + r] * D + scol) : 0.0f;
            }
            Acc4 acc[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b].zero();
            for (int k0 = 0; k0 < D; k0 += KB) {
                const int kl = min(KB, D - k0);
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    SA[(srow + 16 * h) * 17 + scol] = pa[h];
                    if (!same) SB[(srow + 16 * h) * 17 + scol] = pb[h];
                }
                __syncthreads();
                if (k0 + KB < D) {
                    const int e = k0 + KB + scol;
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const int r = srow + 16 * h;
                        pa[h] = (r < nA && e < D) ? __ldg(data + (size_t)ids[tI * 64 + r] * D + e) : 0.0f;
                        pb[h] = (!same && r < nB && e < D) ? __ldg(data + (size_t)ids[tJ * 64 + r] * D + e) : 0.0f;
                    }
                }
                if (!live) {
                } else if (kl == KB) {
#pragma unroll
                    for (int v = 3; v >= 0; --v) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            float av[4], bv[4];
#pragma unroll
                            for (int a = 0; a < 4; ++a) av[a] = SA[(ty * 4 + a) * 17 + 4 * v + j];
#pragma unroll
                            for (int b = 0; b < 4; ++b) bv[b] = SB[(tx * 4 + b) * 17 + 4 * v + j];
#pragma unroll
                            for (int a = 0; a < 4; ++a)
#pragma unroll
                                for (int b = 0; b < 4; ++b) {
                                    const float p = __fmul_rn(bv[b], av[a]);
                                    if (j == 0) acc[a][b].l0 = __fadd_rn(p, acc[a][b].l0);
                                    else if (j == 1) acc[a][b].l1 = __fadd_rn(p, acc[a][b].l1);
                                    else if (j == 2) acc[a][b].l2 = __fadd_rn(p, acc[a][b].l2);
                                    else acc[a][b].l3 = __fadd_rn(p, acc[a][b].l3);
                                }
                        }
                    }
                } else {
                    for (int e = 0; e < kl; ++e) {  // tail: forward
                        float av[4], bv[4];
#pragma unroll
                        for (int a = 0; a < 4; ++a) av[a] = SA[(ty * 4 + a) * 17 + e];
#pragma unroll
                        for (int b = 0; b < 4; ++b) bv[b] = SB[(tx * 4 + b) * 17 + e];
#pragma unroll
                        for (int a = 0; a < 4; ++a)
#pragma unroll
                            for (int b = 0; b < 4; ++b) acc[a][b].madd1((k0 + e) & 3, bv[b], av[a]);
                    }
                }
                __syncthreads();
            }
            if (live) {
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const int i = tI * 64 + ty * 4 + a, j = tJ * 64 + tx * 4 + b;
                        if (ty * 4 + a < nA && tx * 4 + b < nB) {
                            const float dv = acc[a][b].reduce();
                            dotm[i * ld + j] = dv;
                            if (!same) dotm[j * ld + i] = dv;
                        }
                    }
            }
        }
    }
    __syncthreads();
}

// Phase 2 for f32 rows too large to stage per warp: one block per new vertex,
// the trace's dot matrix (N <= 128) once, then warp 0 prunes from it (same
// extraction sequence as warp_prune) and emits the row and reverse triples.
// Longer traces fall back to the global-row prune on warp 0.
constexpr int MX2 = 128;
__global__ void __launch_bounds__(256, 2)
phase2_matrix_kernel(const F32Metric m, int64_t start, int64_t nb, double alpha2, int R,
                     const int32_t* __restrict__ hops, const int32_t* __restrict__ tids,
                     const uint32_t* __restrict__ tdst, int cap, int reverse_all, uint64_t* __restrict__ cand_all,
                     int32_t* __restrict__ kept_ids, uint32_t* __restrict__ kept_d, int32_t* __restrict__ adj,
                     int32_t* __restrict__ deg, uint32_t* __restrict__ tri_target, uint64_t* __restrict__ tri_key,
                     int W) {
    extern __shared__ __align__(16) unsigned char shp[];
    float* dotm = reinterpret_cast<float*>(shp);                 // [MX2][MX2 + 1]
    float* S = dotm + MX2 * (MX2 + 1);                           // [2][64][17]
    float* nrm = S + 2 * 64 * 17;                                // [MX2]
    int32_t* ids = reinterpret_cast<int32_t*>(nrm + MX2);        // [MX2]
    uint32_t* pv = reinterpret_cast<uint32_t*>(ids + MX2);       // fallback pivot row (16 B aligned)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t xi = blockIdx.x;
    const uint32_t x = (uint32_t)(start + xi);
    const int h = min(hops[xi], cap);
    uint64_t* cand = cand_all + xi * cap;
    const int32_t* ti = tids + xi * cap;
    const uint32_t* td = tdst + xi * cap;
    int32_t* ki = kept_ids + xi * R;
    uint32_t* kd = kept_d + xi * R;
    const bool mat = h <= MX2;
    if (mat) {
        for (int j = tid; j < h; j += 256) {
            ids[j] = ti[j];
            nrm[j] = __ldg(m.norms + ti[j]);
        }
        __syncthreads();
        block_dot_matrix(m.data, m.D, ids, h, S, dotm, MX2 + 1);
    }
    if (warp != 0) return;
    for (int j = lane; j < h; j += 32) cand[j] = key_of(td[j], (uint32_t)ti[j]);
    __syncwarp();
    int k;
    if (!mat) {
        k = warp_prune(cand, h, alpha2, R, m, pv, ki, kd);
    } else {
        k = 0;
        while (k < R) {
            uint64_t mk = UMAX;
            int mi = -1;
            for (int i = lane; i < h; i += 32) {
                const uint64_t c = cand[i];
                if (c < mk) { mk = c; mi = i; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const uint64_t om = shfl_xor_u64(mk, o);
                const int oi = __shfl_xor_sync(0xFFFFFFFFu, mi, o);
                if (om < mk) { mk = om; mi = oi; }
            }
            if (mk == UMAX) break;
            if (lane == 0) {
                ki[k] = (int32_t)(mk & 0xFFFFFFFFull);
                kd[k] = (uint32_t)(mk >> 32);
                cand[mi] = UMAX;
            }
            ++k;
            __syncwarp();
            if (k >= R) break;
            for (int i = lane; i < h; i += 32) {
                const uint64_t c = cand[i];
                if (c == UMAX) continue;
                const float dsp = exact_from_dot(nrm[i], dotm[i * (MX2 + 1) + mi], nrm[mi]);
                if (!(__dmul_rn(alpha2, (double)dsp) > (double)__uint_as_float((uint32_t)(c >> 32)))) cand[i] = UMAX;
            }
            __syncwarp();
        }
        __syncwarp();
    }
    write_row(m, alpha2, adj, deg, R, x, ki, k);
    uint32_t* tt = tri_target + xi * W;
    uint64_t* tk = tri_key + xi * W;
    const int ne = reverse_all ? h : k;
    for (int j = lane; j < W; j += 32) {
        if (j < ne) {
            tt[j] = reverse_all ? (uint32_t)ti[j] : (uint32_t)ki[j];
            tk[j] = key_of(reverse_all ? td[j] : kd[j], x);
        } else {
            tt[j] = NO_TARGET;
            tk[j] = UMAX;
        }
    }
}

// ---- two_pass refinement prune (build.py:362-381) --------------------------
// Per vertex x of the batch: candidates = its visited trace without x itself, plus
// its current neighbours missing from the trace (distances d(x, e) with x as the
// pivot); robust prune at the final alpha; rewrite x's row; reverse triples for
// the kept edges. Only warp x reads or writes row x, so the batch is parallel.
template <class M>
__global__ void __launch_bounds__(BW * 32)
refine_prune_kernel(const M m, int64_t start, int64_t nb, double alpha2, int R, const int32_t* __restrict__ hops,
                    const int32_t* __restrict__ tids, const uint32_t* __restrict__ tdst, int cap,
                    uint64_t* __restrict__ cand_all, int32_t* __restrict__ kept_ids, uint32_t* __restrict__ kept_d,
                    int32_t* __restrict__ adj, int32_t* __restrict__ deg, uint32_t* __restrict__ tri_target,
                    uint64_t* __restrict__ tri_key, int crows, int32_t* __restrict__ ncand) {
    extern __shared__ __align__(16) uint32_t shw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* pv = shw + (size_t)warp * vertex_warp_words(m, crows);
    uint32_t* rows = pv + m.pivot_words();
    uint32_t* cn = rows + (size_t)crows * m.stage_stride_words();
    const int64_t xi = (int64_t)blockIdx.x * BW + warp;
    if (xi >= nb) return;
    const uint32_t x = (uint32_t)(start + xi);
    const int h = min(hops[xi], cap);
    uint64_t* cand = cand_all + xi * (int64_t)(cap + R);
    const int32_t* ti = tids + xi * (int64_t)cap;
    const uint32_t* td = tdst + xi * (int64_t)cap;
    m.load_pivot(pv, x);
    int n = 0;
    for (int b = 0; b < h; b += 32) {  // the visited trace, x excluded (keep = cand_ids != x)
        const int j = b + lane;
        const bool ok = j < h && (uint32_t)ti[j] != x;
        const uint32_t msk = __ballot_sync(0xFFFFFFFFu, ok);
        if (ok) cand[n + __popc(msk & lanemask_lt())] = key_of(td[j], (uint32_t)ti[j]);
        n += __popc(msk);
    }
    __syncwarp();
    const int hd = deg[x];
    for (int b = 0; b < hd; b += 32) {  // extra = current[~isin(current, visited)]
        const int e = b + lane;
        bool extra = false;
        int32_t id = -1;
        if (e < hd) {
            id = adj[(size_t)x * R + e];
            extra = true;
            for (int j = 0; j < h; ++j) extra &= (ti[j] != id);
        }
        const uint32_t msk = __ballot_sync(0xFFFFFFFFu, extra);
        if (extra) cand[n + __popc(msk & lanemask_lt())] = key_of(m.dist(pv, (uint32_t)id), (uint32_t)id);
        n += __popc(msk);
    }
    __syncwarp();
    if (lane == 0) ncand[xi] = n;
    int32_t* ki = kept_ids + xi * R;
    uint32_t* kd = kept_d + xi * R;
    int k;
    if (n <= crows) {
        uint32_t sph = 0;
        m.stage(rows, cn, cand, n, init_stage_bar(cn, crows), &sph);
        k = warp_prune_staged(cand, n, alpha2, R, m, rows, cn, stage_list(cn, crows), ki, kd);
    } else {
        k = warp_prune(cand, n, alpha2, R, m, pv, ki, kd);
    }
    __syncwarp();
    write_row(m, alpha2, adj, deg, R, x, ki, k);
    uint32_t* tt = tri_target + xi * R;
    uint64_t* tk = tri_key + xi * R;
    for (int j = lane; j < R; j += 32) {
        tt[j] = j < k ? (uint32_t)ki[j] : NO_TARGET;
        tk[j] = j < k ? key_of(kd[j], x) : UMAX;
    }
}

// ---- batched standalone robust prune (graph.py:174-228), f32 rows ------------
__global__ void __launch_bounds__(BW * 32)
prune_batch_kernel(const F32Metric m, const int64_t* __restrict__ pivots, int64_t count,
                   const int64_t* __restrict__ offsets, const int32_t* __restrict__ cids, const float* __restrict__ cd,
                   double alpha2, int R, uint64_t* __restrict__ cand_all, int32_t* __restrict__ out_ids,
                   float* __restrict__ out_d, int32_t* __restrict__ out_n) {
    extern __shared__ __align__(16) uint32_t shw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* pv = shw + warp * m.pivot_words();
    const int64_t i = (int64_t)blockIdx.x * BW + warp;
    if (i >= count) return;
    const int64_t o0 = offsets[i], o1 = offsets[i + 1];
    const int n = (int)(o1 - o0);
    uint64_t* cand = cand_all + o0;
    for (int j = lane; j < n; j += 32) cand[j] = pack_key(cd[o0 + j], (uint32_t)cids[o0 + j]);
    __syncwarp();
    const int k = warp_prune(cand, n, alpha2, R, m, pv, out_ids + i * R, reinterpret_cast<uint32_t*>(out_d + i * R));
    if (lane == 0) out_n[i] = k;
    (void)pivots;
}

// ---- phase 3: group heads, owner merge (build.py:269-293) ------------------
__global__ void seg_head_kernel(const uint32_t* __restrict__ t, int64_t n, uint8_t* __restrict__ flag) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    flag[i] = (t[i] != NO_TARGET) && (i == 0 || t[i] != t[i - 1]);
}

#ifndef JB_OWNER_SC
#define JB_OWNER_SC 64
#endif
constexpr int OWNER_SC = JB_OWNER_SC;  // smem candidate slots per owner warp (larger groups use the global pool)
// per-warp bytes: keys | vertex words (pivot, staged rows, norms) | have, kid, kd
__host__ __device__ inline int owner_light_per_warp(int R) { return ((OWNER_SC * 8 + R * 4 * 3) + 15) & ~15; }
template <class M>
__host__ __device__ inline int owner_per_warp(const M& m, int R, int crows) {
    const int gram = std::is_same<M, F32Metric>::value ? GP_BYTES : 0;  // warp_prune_gram scratch
    return ((OWNER_SC * 8 + vertex_warp_words(m, crows) * 4 + R * 4 * 3 + gram) + 15) & ~15;
}

#ifdef JB_OWNER_STATS
__device__ unsigned long long g_owner_stats[16];
extern "C" int jb_debug_owner_stats(unsigned long long* out) {
    JB_CUDA(cudaMemcpyFromSymbol(out, g_owner_stats, sizeof(unsigned long long) * 16));
    static const unsigned long long zero[16] = {};
    JB_CUDA(cudaMemcpyToSymbol(g_owner_stats, zero, sizeof(zero)));
    return JB_OK;
}
#endif

// Closed-row prune for candidate sets too large to stage (rows read from global
// memory, e.g. R = 64): the same fresh-pair masks as warp_prune_gram's closed path,
// exact A1 distances (one dot per (fresh, candidate) pair serves both roles), up to
// 128 candidates (4 ranked positions per lane, 128-bit masks). `pv` is free scratch
// for one pivot row; `scr` >= 16 x 32 + 160 bytes.
__device__ int prune_closed_global(uint64_t* cand, int n, int hd, double alpha2, int R, const F32Metric& m, uint32_t* pv,
                                   unsigned char* scr, int32_t* out_ids, uint32_t* out_d) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = lane_id();
    uint64_t* fdoms = reinterpret_cast<uint64_t*>(scr);  // [16][2]
    uint64_t* fdomby = fdoms + 32;                        // [16][2]
    uint8_t* rk = reinterpret_cast<uint8_t*>(fdomby + 32);  // [128]
    uint8_t* fpos = rk + 128;                             // [16]
    // rank by key (keys are distinct): position of each of this lane's candidates
    uint64_t kk[4];
    int rank[4] = {0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < 4; ++q) kk[q] = lane + 32 * q < n ? cand[lane + 32 * q] : UMAX;
    for (int j = 0; j < n; ++j) {
        const uint64_t kj = cand[j];
#pragma unroll
        for (int q = 0; q < 4; ++q) rank[q] += kj < kk[q];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (lane + 32 * q < n) rk[rank[q]] = (uint8_t)(lane + 32 * q);
    __syncwarp();
    // this lane's ranked positions lane + 32 q: candidate index, key distance, row id, norm
    int ic[4];
    float dt[4], nc[4];
    uint32_t fm[4];
    int nf = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int c = lane + 32 * q;
        ic[q] = c < n ? rk[c] : 0;
        const uint64_t kc = cand[ic[q]];
        dt[q] = __uint_as_float((uint32_t)(kc >> 32));
        nc[q] = __ldg(m.norms + (uint32_t)(kc & 0xFFFFFFFFull));
        fm[q] = __ballot_sync(FULL, c < n && ic[q] >= hd);
        if (c < n && ic[q] >= hd) fpos[nf + __popc(fm[q] & lanemask_lt())] = (uint8_t)c;
        nf += __popc(fm[q]);
    }
    __syncwarp();
    const int D = m.D;
    for (int f = 0; f < nf; ++f) {
        const int pf = fpos[f];
        const uint64_t kf = cand[rk[pf]];
        const uint32_t idf = (uint32_t)(kf & 0xFFFFFFFFull);
        const float dtf = __uint_as_float((uint32_t)(kf >> 32));
        __syncwarp();
        m.load_pivot(pv, idf);  // f's row + norm
        const float* fv = reinterpret_cast<const float*>(pv);
        const float nf_ = fv[(D + 3) & ~3];
        uint64_t dlo = 0, dhi = 0, blo = 0, bhi = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = lane + 32 * q;
            bool d = false, b = false;
            if (c < n && c != pf) {
                const uint32_t idc = (uint32_t)(cand[ic[q]] & 0xFFFFFFFFull);
                const float dot = a1_dot<false>(m.data + (size_t)idc * D, fv, D);
                if (c > pf) {  // does f (as the star) prune c?
                    const float dfc = exact_from_dot(nc[q], dot, nf_);
                    d = !(__dmul_rn(alpha2, (double)dfc) > (double)dt[q]);
                } else {       // does c (as the star) prune f?
                    const float dcf = exact_from_dot(nf_, dot, nc[q]);
                    b = !(__dmul_rn(alpha2, (double)dcf) > (double)dtf);
                }
            }
            const uint32_t dm = __ballot_sync(FULL, d), bm = __ballot_sync(FULL, b);
            if (q < 2) { dlo |= (uint64_t)dm << (32 * q); blo |= (uint64_t)bm << (32 * q); }
            else { dhi |= (uint64_t)dm << (32 * (q - 2)); bhi |= (uint64_t)bm << (32 * (q - 2)); }
        }
        if (lane == 0) {
            fdoms[2 * f] = dlo; fdoms[2 * f + 1] = dhi;
            fdomby[2 * f] = blo; fdomby[2 * f + 1] = bhi;
        }
    }
    __syncwarp();
    // scan in rank order: c kept iff no kept candidate before it prunes it
    const uint64_t flo = (uint64_t)fm[0] | ((uint64_t)fm[1] << 32), fhi = (uint64_t)fm[2] | ((uint64_t)fm[3] << 32);
    uint64_t klo = 0, khi = 0, kdlo = 0, kdhi = 0;
    int kept = 0, f = 0;
    for (int c = 0; c < n && kept < R; ++c) {
        const bool hi = c >= 64;
        const uint64_t bit = 1ull << (c & 63);
        const bool isf = ((hi ? fhi : flo) & bit) != 0;
        bool dominated;
        if (isf) dominated = ((fdomby[2 * f] & klo) | (fdomby[2 * f + 1] & khi)) != 0;
        else dominated = ((hi ? kdhi : kdlo) & bit) != 0;
        if (!dominated) {
            if (hi) khi |= bit; else klo |= bit;
            if (isf) { kdlo |= fdoms[2 * f]; kdhi |= fdoms[2 * f + 1]; }
            if (lane == 0) {
                const uint64_t kc = cand[rk[c]];
                out_ids[kept] = (int32_t)(kc & 0xFFFFFFFFull);
                out_d[kept] = (uint32_t)(kc >> 32);
            }
            ++kept;
        }
        if (isf) ++f;
    }
    __syncwarp();
    return kept;
}

// MODE 0: every target (append, or prune with staged rows); MODE 1 (light, no row
// staging, high occupancy): append where the fresh sources fit, defer the rest to
// defer[] (targets needing a prune or the global pool) — except closed f32 rows
// whose candidates fit `crows` (MODE 1's crows = the closed pass's staging size),
// which go to defer[dstride + ...]; MODE 2: the deferred list (staged rows, Gram
// screen); MODE 3: the closed list (almost every prune of a bulk build), the same
// staged path on a persistent grid of 1-warp blocks (1M x 128 build 0.472 -> 0.454 s,
// identical graphs).
template <class M, int MODE>
__device__ __forceinline__ void owner_one(const M& m, double alpha2, int R, int always_prune, const uint32_t* __restrict__ tgt,
                   const uint64_t* __restrict__ key, int64_t total, const int32_t* __restrict__ seg_start, int64_t s,
                   uint64_t* __restrict__ pool, unsigned long long* __restrict__ pool_top,
                   int pool_cap, int32_t* __restrict__ adj, int32_t* __restrict__ deg, int* __restrict__ err, int crows,
                   unsigned char* base, int32_t* __restrict__ defer, int* __restrict__ ndefer, uint32_t& sph,
                   int64_t dstride) {
    const int lane = threadIdx.x & 31;
    constexpr int SC = OWNER_SC;
    uint64_t* scand = reinterpret_cast<uint64_t*>(base);
    // F32: Gram block (16 B aligned) and rank list of warp_prune_gram
    constexpr int GB = (std::is_same<M, F32Metric>::value && MODE != 1) ? GP_BYTES : 0;
    float* gb = reinterpret_cast<float*>(base + SC * 8);
    uint8_t* rk = reinterpret_cast<uint8_t*>(base + SC * 8 + 16 * GP_MAX * 4 + GP_MAX * 4);
    uint32_t* pv = reinterpret_cast<uint32_t*>(base + SC * 8 + GB);
    uint32_t* rows = pv + m.pivot_words();
    uint32_t* cn = rows + (size_t)crows * m.stage_stride_words();
    int32_t* have = MODE == 1 ? reinterpret_cast<int32_t*>(base + SC * 8)
                              : reinterpret_cast<int32_t*>(pv + vertex_warp_words(m, crows));
    int32_t* kid = have + R;
    uint32_t* kd = reinterpret_cast<uint32_t*>(kid + R);
    // Dependent global round trips kept to three: the segment start; its first 32
    // targets and keys together; the target's degree and whole row together.
    const int64_t g0 = seg_start[s];
    const uint32_t tl = (g0 + lane < total) ? tgt[g0 + lane] : NO_TARGET;
    const uint64_t kl = (g0 + lane < total) ? key[g0 + lane] : 0;
    const uint32_t t = __shfl_sync(0xFFFFFFFFu, tl, 0);
    int64_t g1 = g0 + __popc(__ballot_sync(0xFFFFFFFFu, tl == t));
    if (g1 - g0 == 32) {
        for (;;) {  // group end: first index whose target differs
            const int64_t i = g1 + lane;
            const bool same = i < total && tgt[i] == t;
            const uint32_t msk = __ballot_sync(0xFFFFFFFFu, same);
            g1 += __popc(msk);
            if (msk != 0xFFFFFFFFu) break;
        }
    }
    const int g = (int)(g1 - g0);
    int hd;
    {
        const int32_t* row = adj + (size_t)t * R;
        int32_t r0 = lane < R ? row[lane] : -1;
        hd = deg[t];
        if (lane < hd) have[lane] = r0;
        for (int j = lane + 32; j < hd; j += 32) have[j] = row[j];
    }
    __syncwarp();
    // candidate storage: smem when it fits, else a bump-allocated global slice
    uint64_t* cand = scand;
    if (MODE == 1 && hd + g > SC) {  // needs the global pool: the deferred pass
        if (lane == 0) defer[atomicAdd(ndefer, 1)] = (int32_t)s;
        return;
    }
    if (hd + g > SC) {
        unsigned long long off = 0;
        if (lane == 0) off = atomicAdd(pool_top, (unsigned long long)(hd + g));
        off = __shfl_sync(0xFFFFFFFFu, off, 0);
        if (off + hd + g > (unsigned long long)pool_cap) {
            if (lane == 0) atomicExch(err, 1);
            return;
        }
        cand = pool + off;
    }
    // fresh = group sources not already neighbours, in (dist, source) order
    int nf = 0;
    for (int b = 0; b < g; b += 32) {
        const int j = b + lane;
        bool fresh = false;
        uint64_t k = 0;
        if (j < g) {
            k = b == 0 ? kl : key[g0 + j];
            const int32_t src = (int32_t)(k & 0xFFFFFFFFull);
            fresh = true;
            for (int e = 0; e < hd; ++e) fresh &= (have[e] != src);
        }
        const uint32_t msk = __ballot_sync(0xFFFFFFFFu, fresh);
        if (fresh) cand[hd + nf + __popc(msk & lanemask_lt())] = k;
        nf += __popc(msk);
    }
    __syncwarp();
    if (nf == 0) return;
    if (!always_prune && hd + nf <= R) {  // append in (dist, source) order
        for (int j = lane; j < nf; j += 32) adj[(size_t)t * R + hd + j] = (int32_t)(cand[hd + j] & 0xFFFFFFFFull);
        if (lane == 0) {
            deg[t] = hd + nf;
            m.open_row(t);  // appended, not pruned: no closure
        }
        return;
    }
    if (MODE == 1) {  // a prune: the deferred pass (staged rows, Gram screen) or the closed pass
        bool closed = false;
        if constexpr (std::is_same<M, F32Metric>::value)
            closed = dstride > 0 && hd + nf <= crows && m.row_closed(t, alpha2);
        if (lane == 0) {
            if (closed) defer[dstride + atomicAdd(ndefer + 1, 1)] = (int32_t)s;
            else defer[atomicAdd(ndefer, 1)] = (int32_t)s;
        }
        return;
    }
    // existing neighbours get recomputed distances d(t, e) (target is the pivot);
    // fresh entries already hold (stored triple dist << 32 | source) keys
    m.load_pivot_async(pv, t);  // overlaps the staging copies below
    const int n = hd + nf;
    int k;
#ifdef JB_OWNER_STATS
    if (lane == 0) {
        atomicAdd(&g_owner_stats[0], 1ull);                      // pruned targets
        atomicAdd(&g_owner_stats[1], (unsigned long long)n);     // candidates
        if (n > crows) {
            atomicAdd(&g_owner_stats[2], 1ull);                  // unstaged targets
            atomicAdd(&g_owner_stats[3], (unsigned long long)n); // their candidates
        }
        atomicAdd(&g_owner_stats[4 + min(n / 16, 11)], 1ull);    // histogram of n in 16s
    }
#endif
    if (n <= crows) {
        for (int j = lane; j < hd; j += 32) cand[j] = (uint64_t)(uint32_t)have[j];  // id only, for staging
        __syncwarp();
        m.stage(rows, cn, cand, n, stage_bar(cn, crows), &sph);
        for (int j = lane; j < hd; j += 32) cand[j] = key_of(m.dist_pivot_staged(pv, rows, cn, j), (uint32_t)have[j]);
        __syncwarp();
        bool done = false;
        if constexpr (std::is_same<M, F32Metric>::value) {
            if (m.gram_ok(n, GP_MAX)) {
                k = warp_prune_gram(cand, n, alpha2, R, m, rows, cn, rk, gb, kid, kd,
                                    m.row_closed(t, alpha2) ? hd : -1);
                done = true;
            }
        }
        if (!done) k = warp_prune_staged(cand, n, alpha2, R, m, rows, cn, stage_list(cn, crows), kid, kd);
    } else if (MODE != 1) {
        cp_async_wait_all();
        __syncwarp();
        for (int j = lane; j < hd; j += 32) {
            const uint32_t e = (uint32_t)have[j];
            cand[j] = key_of(m.dist(pv, e), e);
        }
        __syncwarp();
        bool done = false;
        if constexpr (std::is_same<M, F32Metric>::value) {
            if (n - hd >= 1 && n - hd <= 16 && n <= 128 && m.row_closed(t, alpha2)) {
                k = prune_closed_global(cand, n, hd, alpha2, R, m, pv, reinterpret_cast<unsigned char*>(gb), kid, kd);
                done = true;
            }
        }
        if (!done) k = warp_prune(cand, n, alpha2, R, m, pv, kid, kd);
    }
    write_row(m, alpha2, adj, deg, R, t, kid, k);
}

template <class M, int MODE>
__global__ void __launch_bounds__(BW * 32)
owner_merge_kernel(const M m, double alpha2, int R, int always_prune, const uint32_t* __restrict__ tgt,
                   const uint64_t* __restrict__ key, int64_t total, const int32_t* __restrict__ seg_start,
                   const int* __restrict__ n_seg, uint64_t* __restrict__ pool, unsigned long long* __restrict__ pool_top,
                   int pool_cap, int32_t* __restrict__ adj, int32_t* __restrict__ deg, int* __restrict__ err, int crows,
                   int32_t* __restrict__ defer, int* __restrict__ ndefer, int64_t dstride) {
    extern __shared__ __align__(16) unsigned char shb[];
    const int warp = threadIdx.x >> 5;
    const int per_warp = MODE == 1 ? owner_light_per_warp(R) : owner_per_warp(m, R, crows);
    unsigned char* base = shb + (size_t)warp * per_warp;
    uint32_t sph = 0;  // the warp's staging-barrier phase (MODE 0 / 2 stage rows)
    if (MODE != 1) {
        constexpr int GB = std::is_same<M, F32Metric>::value ? GP_BYTES : 0;
        uint32_t* cn = reinterpret_cast<uint32_t*>(base + OWNER_SC * 8 + GB) + m.pivot_words() +
                       (size_t)crows * m.stage_stride_words();
        init_stage_bar(cn, crows);
    }
    if (MODE >= 2) {  // persistent over the deferred (2) or closed (3) targets
        const int nd = ndefer[MODE - 2];
        const int32_t* list = defer + (MODE == 3 ? dstride : 0);
        const int wpb = (int)(blockDim.x >> 5);
        for (int64_t i = (int64_t)blockIdx.x * wpb + warp; i < nd; i += (int64_t)gridDim.x * wpb)
            owner_one<M, MODE>(m, alpha2, R, always_prune, tgt, key, total, seg_start, list[i], pool, pool_top,
                               pool_cap, adj, deg, err, crows, base, defer, ndefer, sph, dstride);
    } else {
        const int64_t s = (int64_t)blockIdx.x * BW + warp;
        if (s >= *n_seg) return;
        owner_one<M, MODE>(m, alpha2, R, always_prune, tgt, key, total, seg_start, s, pool, pool_top, pool_cap, adj,
                           deg, err, crows, base, defer, ndefer, sph, dstride);
    }
}

// ---- phase 3 for rows too large to stage per warp (f32, e.g. 960-d) ----------
// One block per target. Warp 0 does the owner's group / fresh / append logic;
// when the prune has n <= MX - 1 candidates the block computes the full A1 dot
// matrix of the candidates and the target (MX x MX tile, 4 x 4 pairs per
// thread, the donor scan's k-step order: 16-element blocks as vectors 3,2,1,0,
// then the tail forward) so every row is read once instead of once per round.
// dot(a, b) == dot(b, a) bit for bit (same products, same order), so each
// operand-role distance follows from the matrix and the two norms:
// d(p -> c) = max((xn[c] - 2 dot) + xn[p], 0). Warp 0 then runs the rounds from
// smem. Larger groups fall back to the global-row prune on warp 0.
constexpr int MX = 64;
#ifdef JB_NO_MATRIX
constexpr bool kNoMatrix = true;  // dev A/B: warp kernels only
#else
constexpr bool kNoMatrix = false;
#endif
__global__ void __launch_bounds__(256, 2)
owner_matrix_kernel(const F32Metric m, double alpha2, int R, int always_prune, const uint32_t* __restrict__ tgt,
                    const uint64_t* __restrict__ key, int64_t total, const int32_t* __restrict__ seg_start,
                    uint64_t* __restrict__ pool, unsigned long long* __restrict__ pool_top, int pool_cap,
                    int32_t* __restrict__ adj, int32_t* __restrict__ deg, int* __restrict__ err) {
    extern __shared__ __align__(16) unsigned char shm[];
    float* dotm = reinterpret_cast<float*>(shm);                  // [MX][MX + 1]
    float* S = dotm + MX * (MX + 1);                              // [MX][17] k-step slice
    float* nrm = S + MX * 17;                                     // [MX]
    int32_t* ids = reinterpret_cast<int32_t*>(nrm + MX);          // [MX]
    uint64_t* scand = reinterpret_cast<uint64_t*>(ids + MX);      // [OWNER_SC] (8 B aligned: MX even)
    int32_t* have = reinterpret_cast<int32_t*>(scand + OWNER_SC); // [R]
    int32_t* kid = have + R;
    uint32_t* kd = reinterpret_cast<uint32_t*>(kid + R);
    uint32_t* pv = kd + R;                                        // pivot row (fallback path), 16 B aligned below
    __shared__ int mode_s, n_s, hdc_s;
    __shared__ uint64_t* cand_s;
    pv = reinterpret_cast<uint32_t*>((reinterpret_cast<uintptr_t>(pv) + 15) & ~uintptr_t(15));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t s = blockIdx.x;
    const int64_t g0 = seg_start[s];
    const uint32_t t = tgt[g0];
    const int D = m.D;
    if (warp == 0) {
        int64_t g1 = g0;
        for (;;) {
            const int64_t i = g1 + lane;
            const bool same = i < total && tgt[i] == t;
            const uint32_t msk = __ballot_sync(0xFFFFFFFFu, same);
            g1 += __popc(msk);
            if (msk != 0xFFFFFFFFu) break;
        }
        const int g = (int)(g1 - g0);
        const int hd = deg[t];
        for (int j = lane; j < hd; j += 32) have[j] = adj[(size_t)t * R + j];
        __syncwarp();
        uint64_t* cand = scand;
        int mode = 0;  // 0 done, 1 matrix, 2 fallback
        if (hd + g > OWNER_SC) {
            unsigned long long off = 0;
            if (lane == 0) off = atomicAdd(pool_top, (unsigned long long)(hd + g));
            off = __shfl_sync(0xFFFFFFFFu, off, 0);
            if (off + hd + g > (unsigned long long)pool_cap) {
                if (lane == 0) atomicExch(err, 1);
                cand = nullptr;
            } else {
                cand = pool + off;
            }
        }
        int nf = 0;
        if (cand != nullptr) {
            for (int b = 0; b < g; b += 32) {
                const int j = b + lane;
                bool fresh = false;
                uint64_t k = 0;
                if (j < g) {
                    k = key[g0 + j];
                    const int32_t src = (int32_t)(k & 0xFFFFFFFFull);
                    fresh = true;
                    for (int e = 0; e < hd; ++e) fresh &= (have[e] != src);
                }
                const uint32_t msk = __ballot_sync(0xFFFFFFFFu, fresh);
                if (fresh) cand[hd + nf + __popc(msk & lanemask_lt())] = k;
                nf += __popc(msk);
            }
            __syncwarp();
            if (nf > 0) {
                if (!always_prune && hd + nf <= R) {
                    for (int j = lane; j < nf; j += 32)
                        adj[(size_t)t * R + hd + j] = (int32_t)(cand[hd + j] & 0xFFFFFFFFull);
                    if (lane == 0) {
                        deg[t] = hd + nf;
                        m.open_row(t);  // appended, not pruned: no closure
                    }
                } else {
                    mode = (hd + nf <= MX - 1) ? 1 : 2;
                }
            }
        }
        if (mode == 1) {
            const int n = hd + nf;
            for (int j = lane; j < MX; j += 32) {
                const int32_t id = j < hd ? have[j] : j < n ? (int32_t)(cand[j] & 0xFFFFFFFFull) : j == n ? (int32_t)t : -1;
                ids[j] = id;
                nrm[j] = id >= 0 ? __ldg(m.norms + id) : 0.0f;
            }
        }
        if (lane == 0) {
            mode_s = mode; n_s = hd + nf; cand_s = cand;
            // closed row with few fresh sources: only the fresh and target rows of the matrix
            hdc_s = (mode == 1 && nf <= 16 && m.row_closed(t, alpha2)) ? hd : -1;
        }
    }
    __syncthreads();
    const int mode = mode_s;
    if (mode == 0) return;
    const int n = n_s;
    const int hdc = hdc_s;
    uint64_t* cand = cand_s;
    if (mode == 2) {  // hub target: the global-row prune on warp 0
        if (warp != 0) return;
        const int hd = deg[t];
        m.load_pivot(pv, t);
        for (int j = lane; j < hd; j += 32) {
            const uint32_t e = (uint32_t)have[j];
            cand[j] = key_of(m.dist(pv, e), e);
        }
        __syncwarp();
        const int k = warp_prune(cand, n, alpha2, R, m, pv, kid, kd);
        write_row(m, alpha2, adj, deg, R, t, kid, k);
        return;
    }
    // ---- dot matrix of the n candidates and the target (row n) ----
    const int tx = tid & 15, ty = tid >> 4;
    const int N = n + 1;
    Acc4 acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b].zero();
    constexpr int KB = 16;
    // sub-tiles wholly past the N live rows / columns skip the math (warp-uniform in ty);
    // for a closed row only the row groups holding the fresh rows and the target
    // (rows hdc .. n) are needed
    const bool live = ty * 4 < N && tx * 4 < N && (hdc < 0 || ty * 4 + 3 >= hdc);
    // each thread's 4 slice elements: rows tid/16 + 16h, column tid%16; the next
    // k-step's are loaded into registers while the current one is consumed
    const int srow = tid / KB, scol = tid % KB;
    const float* rp[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const int row = srow + 16 * h;
        rp[h] = row < N ? m.data + (size_t)ids[row] * D : nullptr;
    }
    float pf[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) pf[h] = (rp[h] && scol < D) ? __ldg(rp[h] + scol) : 0.0f;
    for (int k0 = 0; k0 < D; k0 += KB) {
        const int kl = min(KB, D - k0);
#pragma unroll
        for (int h = 0; h < 4; ++h) S[(srow + 16 * h) * 17 + scol] = pf[h];
        __syncthreads();
        if (k0 + KB < D) {
            const int e = k0 + KB + scol;
#pragma unroll
            for (int h = 0; h < 4; ++h) pf[h] = (rp[h] && e < D) ? __ldg(rp[h] + e) : 0.0f;
        }
        if (!live) {
        } else if (kl == KB) {
#pragma unroll
            for (int v = 3; v >= 0; --v) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float av[4], bv[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) av[a] = S[(ty * 4 + a) * 17 + 4 * v + j];
#pragma unroll
                    for (int b = 0; b < 4; ++b) bv[b] = S[(tx * 4 + b) * 17 + 4 * v + j];
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            const float p = __fmul_rn(bv[b], av[a]);
                            if (j == 0) acc[a][b].l0 = __fadd_rn(p, acc[a][b].l0);
                            else if (j == 1) acc[a][b].l1 = __fadd_rn(p, acc[a][b].l1);
                            else if (j == 2) acc[a][b].l2 = __fadd_rn(p, acc[a][b].l2);
                            else acc[a][b].l3 = __fadd_rn(p, acc[a][b].l3);
                        }
                }
            }
        } else {
            for (int e = 0; e < kl; ++e) {  // tail: forward
                float av[4], bv[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) av[a] = S[(ty * 4 + a) * 17 + e];
#pragma unroll
                for (int b = 0; b < 4; ++b) bv[b] = S[(tx * 4 + b) * 17 + e];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) acc[a][b].madd1((k0 + e) & 3, bv[b], av[a]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dotm[(ty * 4 + a) * (MX + 1) + tx * 4 + b] = acc[a][b].reduce();
    __syncthreads();
    if (warp != 0) return;
    // existing neighbours: d(t -> e) with the target as the pivot; fresh keys stay
    // (row n of the matrix: dot(a, b) == dot(b, a) bit for bit)
    const int hd = deg[t];
    for (int j = lane; j < hd; j += 32)
        cand[j] = key_of(__float_as_uint(exact_from_dot(nrm[j], dotm[n * (MX + 1) + j], nrm[n])), (uint32_t)ids[j]);
    __syncwarp();
    if (hdc >= 0) {
        // closed row: only pairs with a fresh source (candidate index >= hd) can prune
        // (warp_prune_gram's closed path, with exact dots from the matrix rows hd .. n-1)
        uint8_t* rk = reinterpret_cast<uint8_t*>(S);                 // [MX] ranked -> candidate
        uint64_t* fdoms = reinterpret_cast<uint64_t*>(S + MX);       // [16]
        uint64_t* fdomby = fdoms + 16;                               // [16]
        uint8_t* fpos = reinterpret_cast<uint8_t*>(fdomby + 16);     // [16]
        const unsigned FULL = 0xFFFFFFFFu;
        const uint64_t k0 = lane < n ? cand[lane] : UMAX, k1 = lane + 32 < n ? cand[lane + 32] : UMAX;
        int c0 = 0, c1 = 0;
        for (int j = 0; j < n; ++j) {
            const uint64_t kj = cand[j];
            c0 += kj < k0;
            c1 += kj < k1;
        }
        if (lane < n) rk[c0] = (uint8_t)lane;
        if (lane + 32 < n) rk[c1] = (uint8_t)(lane + 32);
        __syncwarp();
        const int i0 = lane < n ? rk[lane] : 0, i1 = lane + 32 < n ? rk[lane + 32] : 0;
        const bool fr0 = lane < n && i0 >= hd, fr1 = lane + 32 < n && i1 >= hd;
        const uint32_t fm0 = __ballot_sync(FULL, fr0), fm1 = __ballot_sync(FULL, fr1);
        const int nfr = __popc(fm0) + __popc(fm1);
        if (fr0) fpos[__popc(fm0 & lanemask_lt())] = (uint8_t)lane;
        if (fr1) fpos[__popc(fm0) + __popc(fm1 & lanemask_lt())] = (uint8_t)(lane + 32);
        __syncwarp();
        const float dt0 = __uint_as_float((uint32_t)(cand[i0] >> 32)), dt1 = __uint_as_float((uint32_t)(cand[i1] >> 32));
        // does candidate `is` (as the star) prune candidate `ic`? d(is -> ic) from the fresh row f
        auto prunes = [&](int f, int is, int ic, float dtc) -> bool {
            const float d = exact_from_dot(nrm[ic], dotm[f * (MX + 1) + (f == is ? ic : is)], nrm[is]);
            return !(__dmul_rn(alpha2, (double)d) > (double)dtc);
        };
        for (int q = 0; q < nfr; ++q) {
            const int pf = fpos[q];
            const int ifr = rk[pf];
            const float dtf = __uint_as_float((uint32_t)(cand[ifr] >> 32));
            bool d0 = false, b0 = false, d1 = false, b1 = false;
            if (lane < n && lane != pf) {
                if (lane > pf) d0 = prunes(ifr, ifr, i0, dt0);
                else b0 = prunes(ifr, i0, ifr, dtf);
            }
            if (lane + 32 < n && lane + 32 != pf) {
                if (lane + 32 > pf) d1 = prunes(ifr, ifr, i1, dt1);
                else b1 = prunes(ifr, i1, ifr, dtf);
            }
            const uint64_t dm = (uint64_t)__ballot_sync(FULL, d0) | ((uint64_t)__ballot_sync(FULL, d1) << 32);
            const uint64_t bm = (uint64_t)__ballot_sync(FULL, b0) | ((uint64_t)__ballot_sync(FULL, b1) << 32);
            if (lane == 0) { fdoms[q] = dm; fdomby[q] = bm; }
        }
        __syncwarp();
        const uint64_t fmask = (uint64_t)fm0 | ((uint64_t)fm1 << 32);
        uint64_t kept_mask = 0, kdoms = 0;
        int kept = 0, q = 0;
        for (int c = 0; c < n && kept < R; ++c) {
            const bool isf = (fmask >> c) & 1ull;
            const bool dominated = isf ? (fdomby[q] & kept_mask) != 0 : ((kdoms >> c) & 1ull) != 0;
            if (!dominated) {
                kept_mask |= 1ull << c;
                if (isf) kdoms |= fdoms[q];
                if (lane == 0) {
                    const uint64_t kc = cand[rk[c]];
                    kid[kept] = (int32_t)(kc & 0xFFFFFFFFull);
                    kd[kept] = (uint32_t)(kc >> 32);
                }
                ++kept;
            }
            if (isf) ++q;
        }
        __syncwarp();
        write_row(m, alpha2, adj, deg, R, t, kid, kept);
        return;
    }
    // robust prune from the matrix (same extraction sequence as warp_prune)
    int kept = 0;
    while (kept < R) {
        uint64_t mk = UMAX;
        int mi = -1;
        for (int i = lane; i < n; i += 32) {
            const uint64_t c = cand[i];
            if (c < mk) { mk = c; mi = i; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t om = shfl_xor_u64(mk, o);
            const int oi = __shfl_xor_sync(0xFFFFFFFFu, mi, o);
            if (om < mk) { mk = om; mi = oi; }
        }
        if (mk == UMAX) break;
        __syncwarp();  // every lane's argmin reads of cand precede lane 0's write (WAR)
        if (lane == 0) {
            kid[kept] = (int32_t)(mk & 0xFFFFFFFFull);
            kd[kept] = (uint32_t)(mk >> 32);
            cand[mi] = UMAX;
        }
        ++kept;
        __syncwarp();
        if (kept >= R) break;
        for (int i = lane; i < n; i += 32) {
            const uint64_t c = cand[i];
            if (c == UMAX) continue;
            const float dsp = exact_from_dot(nrm[i], dotm[i * (MX + 1) + mi], nrm[mi]);
            if (!(__dmul_rn(alpha2, (double)dsp) > (double)__uint_as_float((uint32_t)(c >> 32)))) cand[i] = UMAX;
        }
        __syncwarp();
    }
    __syncwarp();
    write_row(m, alpha2, adj, deg, R, t, kid, kept);
}

// ---- repair: BFS ------------------------------------------------------------
constexpr int BFS_BATCH = 8;           // BFS levels enqueued per host read
constexpr int BFS_MAX_LEVELS = 1 << 16;

__global__ void bfs_init_kernel(int32_t* __restrict__ seen, int64_t n, int64_t entry, int32_t* __restrict__ front,
                                int* __restrict__ fcount) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) seen[i] = (i == entry);
    if (i == 0) { front[0] = (int32_t)entry; *fcount = 1; }
}

// Append `v` to list[] for the lanes with `take`: one atomicAdd per warp (a single
// global counter taking one atomic per element serialises at 10M-vertex scale).
// Every lane of the warp must call. List order is irrelevant to the callers.
__device__ __forceinline__ void warp_append(bool take, int32_t v, int32_t* __restrict__ list, int* __restrict__ count) {
    const unsigned m = __ballot_sync(0xFFFFFFFFu, take);
    if (m == 0) return;
    const int lane = lane_id(), leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(count, __popc(m));
    base = __shfl_sync(0xFFFFFFFFu, base, leader);
    if (take) list[base + __popc(m & lanemask_lt())] = v;
}

// One warp per frontier vertex (grid-stride), lane j reads edge j of its row: a
// coalesced 4R-byte row read and no per-edge index division. Level l reads the
// frontier size cnt[l] and appends the next frontier with cnt[l + 1] (zeroed
// beforehand), so a run of levels is enqueued without reading anything back;
// levels past the last non-empty frontier exit at once. New vertices gather in a
// per-block smem list flushed with one global atomic per block step (a single
// frontier counter taking one atomic per warp serialised the big levels).
constexpr int BFS_T = 512;  // threads per block of bfs_expand_kernel
__global__ void __launch_bounds__(BFS_T)
bfs_expand_kernel(const int32_t* __restrict__ adj, int R, const int32_t* __restrict__ front,
                  const int* __restrict__ fcount, int32_t* __restrict__ seen, int32_t* __restrict__ next,
                  int* __restrict__ ncount) {
    __shared__ int32_t buf[BFS_T];  // one step: <= 32 new vertices per warp
    __shared__ int bn, gbase;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int WPB = BFS_T / 32;
    const int n = *fcount;
    if (threadIdx.x == 0) bn = 0;
    __syncthreads();
    for (int64_t f0 = (int64_t)blockIdx.x * WPB; f0 < n; f0 += (int64_t)gridDim.x * WPB) {
        const int64_t f = f0 + warp;
        for (int j0 = 0; j0 < R; j0 += 32) {  // block-uniform trip count
            bool found = false;
            int32_t v = -1;
            if (f < n) {
                const int j = j0 + lane;
                v = j < R ? adj[(size_t)front[f] * R + j] : -1;
                if (v >= 0 && !seen[v]) found = atomicExch(&seen[v], 1) == 0;
            }
            const unsigned m = __ballot_sync(0xFFFFFFFFu, found);
            int base = 0;
            if (lane == 0 && m) base = atomicAdd(&bn, __popc(m));
            base = __shfl_sync(0xFFFFFFFFu, base, 0);
            if (found) buf[base + __popc(m & lanemask_lt())] = v;
            __syncthreads();
            const int cnt = bn;
            if (cnt > 0) {
                if (threadIdx.x == 0) gbase = atomicAdd(ncount, cnt);
                __syncthreads();
                for (int i = threadIdx.x; i < cnt; i += BFS_T) next[gbase + i] = buf[i];
                __syncthreads();
                if (threadIdx.x == 0) bn = 0;
            }
            __syncthreads();
        }
    }
}

__global__ void split_kernel(const int32_t* __restrict__ seen, int64_t n, int32_t* __restrict__ lost,
                             int* __restrict__ nlost, int32_t* __restrict__ reach, int* __restrict__ nreach) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool in = i < n;
    const bool r = in && seen[i];
    warp_append(r, (int32_t)i, reach, nreach);
    warp_append(in && !r, (int32_t)i, lost, nlost);
}

// Sorted top-`fan` list held one key per lane (lanes >= fan hold UMAX): insert every
// lane's candidate key c (UMAX = none) in turn. Keys are distinct (unique ids), so
// the list after all insertions is the `fan` smallest of list u candidates.
__device__ __forceinline__ void topk_insert_all(uint64_t& t, uint64_t c, int fan) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = lane_id();
    for (uint32_t mm = __ballot_sync(FULL, c != UMAX); mm; mm &= mm - 1) {
        const uint64_t k = shfl_u64(c, __ffs(mm) - 1);
        const uint64_t worst = shfl_u64(t, fan - 1);
        if (k >= worst) continue;  // uniform
        const int pos = __popc(__ballot_sync(FULL, lane < fan && t < k));
        const uint64_t up = __shfl_up_sync(FULL, t, 1);
        if (lane < fan) {
            if (lane > pos) t = up;
            else if (lane == pos) t = k;
        }
    }
}

// ---- repair: nearest reachable donors (build.py:185-192) --------------------
// Block tile: 64 stranded x 64 reachable rows staged in smem; each thread owns a
// 4x4 pair sub-tile with four A1 accumulator lanes per pair. Distances use the
// stranded vertex as the pivot. Each block keeps a running top-16 per stranded
// row over its slice of the reachable list; slices are merged afterwards.
constexpr int DT = 64;      // tile edge
constexpr int FAN = 16;     // min(R, 16) donors, upper bound

// RES: the 64 stranded rows stay resident in smem for the whole slice (D <= 256);
// otherwise (high D) their k-step slices stream through smem beside the reachable ones.
template <bool RES>
__global__ void __launch_bounds__(256, 2)
donor_scan_kernel(const float* __restrict__ data, const float* __restrict__ norms, int D, const int32_t* __restrict__ lost,
                  int nlost, const int32_t* __restrict__ reach, int nreach, int slices, int fan,
                  uint64_t* __restrict__ part) {
    extern __shared__ __align__(16) unsigned char dsh[];
    const int KB = 16;  // elements per k-step (one A1 block)
    const int AS = RES ? D + 1 : KB + 1;                   // stranded tile row stride
    float* Ares = reinterpret_cast<float*>(dsh);           // [DT][AS]   stranded rows (whole, or the k-step)
    float* Bs = Ares + DT * AS;                            // [DT][KB+1] reachable k-step
    float* dist = Bs + DT * (KB + 1);                      // [DT][DT+1]
    uint64_t* top = reinterpret_cast<uint64_t*>(dist + DT * (DT + 1) + ((DT * AS + DT * (KB + 1) + DT * (DT + 1)) & 1));
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads, 4x4 pairs each
    const int s0 = blockIdx.x * DT;
    const int slice = blockIdx.y;
    const int64_t per = (nreach + slices - 1) / slices;
    const int64_t r_begin = slice * per, r_end = (nreach < r_begin + per) ? (int64_t)nreach : r_begin + per;
    for (int i = tid; i < DT * FAN; i += 256) top[i] = UMAX;
    // the 64 stranded rows stay in smem for the whole slice
    if (RES) {
        for (int i = tid; i < DT * D; i += 256) {
            const int row = i / D, e = i % D;
            Ares[row * AS + e] = (s0 + row < nlost) ? data[(size_t)lost[s0 + row] * D + e] : 0.f;
        }
    }
    __syncthreads();
    // reachable rows stream through a 64 x 16 smem tile; each thread prefetches its 4
    // elements of the next k-step into registers while the current one is consumed
    for (int64_t r0 = r_begin; r0 < r_end; r0 += DT) {
        Acc4 acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b].zero();
        // prefetch k-step 0
        float pf[4], pa[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const int i = tid + 256 * h, row = i / KB, e = i % KB;
            pf[h] = (e < min(KB, D) && r0 + row < r_end) ? __ldg(data + (size_t)reach[r0 + row] * D + e) : 0.f;
            if (!RES) pa[h] = (e < min(KB, D) && s0 + row < nlost) ? __ldg(data + (size_t)lost[s0 + row] * D + e) : 0.f;
        }
        for (int k0 = 0; k0 < D; k0 += KB) {
            const int kl = min(KB, D - k0);
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const int i = tid + 256 * h, row = i / KB, e = i % KB;
                Bs[row * (KB + 1) + e] = pf[h];
                if (!RES) Ares[row * AS + e] = pa[h];
            }
            __syncthreads();
            if (k0 + KB < D) {  // next k-step's loads in flight during this step's math
                const int kn = min(KB, D - k0 - KB);
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const int i = tid + 256 * h, row = i / KB, e = i % KB;
                    pf[h] = (e < kn && r0 + row < r_end) ? __ldg(data + (size_t)reach[r0 + row] * D + k0 + KB + e) : 0.f;
                    if (!RES)
                        pa[h] = (e < kn && s0 + row < nlost) ? __ldg(data + (size_t)lost[s0 + row] * D + k0 + KB + e) : 0.f;
                }
            }
            const float* Ak = RES ? Ares + k0 : Ares;
            if (kl == KB) {
                // A1 order inside a 16-block: vectors 3,2,1,0; lane j = element % 4
#pragma unroll
                for (int v = 3; v >= 0; --v) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        float av[4], bv[4];
#pragma unroll
                        for (int a = 0; a < 4; ++a) av[a] = Ak[(ty * 4 + a) * AS + 4 * v + j];
#pragma unroll
                        for (int b = 0; b < 4; ++b) bv[b] = Bs[(tx * 4 + b) * (KB + 1) + 4 * v + j];
#pragma unroll
                        for (int a = 0; a < 4; ++a)
#pragma unroll
                            for (int b = 0; b < 4; ++b) {
                                const float p = __fmul_rn(bv[b], av[a]);
                                if (j == 0) acc[a][b].l0 = __fadd_rn(p, acc[a][b].l0);
                                else if (j == 1) acc[a][b].l1 = __fadd_rn(p, acc[a][b].l1);
                                else if (j == 2) acc[a][b].l2 = __fadd_rn(p, acc[a][b].l2);
                                else acc[a][b].l3 = __fadd_rn(p, acc[a][b].l3);
                            }
                    }
                }
            } else {
                for (int e = 0; e < kl; ++e) {  // tail: forward
                    float av[4], bv[4];
#pragma unroll
                    for (int a = 0; a < 4; ++a) av[a] = Ak[(ty * 4 + a) * AS + e];
#pragma unroll
                    for (int b = 0; b < 4; ++b) bv[b] = Bs[(tx * 4 + b) * (KB + 1) + e];
#pragma unroll
                    for (int a = 0; a < 4; ++a)
#pragma unroll
                        for (int b = 0; b < 4; ++b) acc[a][b].madd1((k0 + e) & 3, bv[b], av[a]);
                }
            }
            __syncthreads();
        }
        // distances: row = reachable r (data role), pivot = stranded x (norm added last)
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const int si = s0 + ty * 4 + a;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int64_t ri = r0 + tx * 4 + b;
                float d = __int_as_float(0x7F800000);
                if (si < nlost && ri < r_end) {
                    const uint32_t r = (uint32_t)reach[ri];
                    d = exact_from_dot(__ldg(norms + r), acc[a][b].reduce(), __ldg(norms + lost[si]));
                }
                dist[(ty * 4 + a) * (DT + 1) + tx * 4 + b] = d;
            }
        }
        __syncthreads();
        // merge the 64 new candidates of each stranded row into its top-`fan`
        const int warp = tid >> 5, lane = tid & 31;
        for (int row = warp; row < DT; row += 8) {
            if (s0 + row >= nlost) continue;
            uint64_t* tp = top + row * FAN;
            const uint64_t worst = tp[fan - 1];
            uint64_t k0v = UMAX, k1v = UMAX;
            if (r0 + lane < r_end) k0v = pack_key(dist[row * (DT + 1) + lane], (uint32_t)reach[r0 + lane]);
            if (r0 + 32 + lane < r_end) k1v = pack_key(dist[row * (DT + 1) + 32 + lane], (uint32_t)reach[r0 + 32 + lane]);
            if (k0v >= worst) k0v = UMAX;
            if (k1v >= worst) k1v = UMAX;
            if (!__any_sync(0xFFFFFFFFu, k0v != UMAX || k1v != UMAX)) continue;
            // insert the survivors one at a time into the sorted top list (lanes < fan)
            uint64_t t = lane < fan ? tp[lane] : UMAX;
            topk_insert_all(t, k0v, fan);
            topk_insert_all(t, k1v, fan);
            if (lane < fan) tp[lane] = t;
            __syncwarp();
        }
        __syncthreads();
    }
    for (int i = tid; i < DT * FAN; i += 256) {
        const int row = i / FAN, j = i % FAN;
        if (s0 + row < nlost && j < fan) part[((size_t)slice * nlost + s0 + row) * fan + j] = top[row * FAN + j];
    }
}

// Generic nearest-donor scan (any metric): block = 8 warps = 8 stranded pivots
// staged in smem, each warp scans a slice of the reachable list one row per lane
// and keeps a running top-`fan` by (dist, id) key in registers (lane j = j-th best). Output layout as donor_scan_kernel.
template <class M>
__global__ void __launch_bounds__(256)
donor_scan_generic_kernel(const M m, const int32_t* __restrict__ lost, int nlost, const int32_t* __restrict__ reach,
                          int nreach, int slices, int fan, uint64_t* __restrict__ part) {
    extern __shared__ __align__(16) uint32_t gsh[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t* pv = gsh + warp * m.pivot_words();
    const int si = blockIdx.x * 8 + warp;
    if (si >= nlost) return;
    const int slice = blockIdx.y;
    const int64_t per = (nreach + slices - 1) / slices;
    const int64_t r_begin = slice * per, r_end = (nreach < r_begin + per) ? (int64_t)nreach : r_begin + per;
    m.load_pivot(pv, (uint32_t)lost[si]);
    __syncwarp();
    // lane j holds the j-th best key (j < fan); candidates enter by warp insertion
    uint64_t t = UMAX;
    for (int64_t r0 = r_begin; r0 < r_end; r0 += 32) {
        const int64_t ri = r0 + lane;
        uint64_t k = UMAX;
        if (ri < r_end) {
            const uint32_t r = (uint32_t)reach[ri];
            k = key_of(m.dist(pv, r), r);
        }
        topk_insert_all(t, k, fan);
    }
    if (lane < fan) part[((size_t)slice * nlost + si) * fan + lane] = t;
}

// merge slice top-lists: warp per stranded vertex; writes donors and the sort key
// (nearest-donor dist bits << 32 | stranded id) for the processing order.
__global__ void donor_merge_kernel(const uint64_t* __restrict__ part, int slices, int nlost, int fan,
                                   const int32_t* __restrict__ lost, int32_t* __restrict__ donors,
                                   uint64_t* __restrict__ order_key, int32_t* __restrict__ order_val) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= nlost) return;
    uint64_t best = UMAX;
    // repeated extraction of the minimum: slices*fan <= 64*16 candidates
    uint64_t taken_last = 0;
    bool first = true;
    for (int j = 0; j < fan; ++j) {
        uint64_t m = UMAX;
        for (int i = lane; i < slices * fan; i += 32) {
            const int sl = i / fan, q = i % fan;
            const uint64_t k = part[((size_t)sl * nlost + warp) * fan + q];
            if ((first || k > taken_last) && k < m) m = k;
        }
        m = warp_min_u64(m);
        if (lane == 0) donors[(size_t)warp * fan + j] = (m == UMAX) ? -1 : (int32_t)(m & 0xFFFFFFFFull);
        if (j == 0) best = m;
        taken_last = m;
        first = false;
        if (m == UMAX) {
            for (int jj = j + 1 + lane; jj < fan; jj += 32) donors[(size_t)warp * fan + jj] = -1;
            break;
        }
    }
    if (lane == 0) {
        order_key[warp] = (best & 0xFFFFFFFF00000000ull) | (uint32_t)lost[warp];
        order_val[warp] = warp;
    }
}

// ---- repair: ordered sequential attach (build.py:193-224), one warp ----------
template <class M>
__global__ void attach_kernel(const M m, int32_t* __restrict__ adj, int32_t* __restrict__ deg, int R, uint8_t* __restrict__ pinned,
                              int32_t* __restrict__ seen, const int32_t* __restrict__ lost,
                              const int32_t* __restrict__ order, int nlost, const int32_t* __restrict__ donors, int fan,
                              int32_t* __restrict__ queue, unsigned long long* __restrict__ bridges,
                              int* __restrict__ err, int32_t* __restrict__ err_vertex, int* __restrict__ evictions) {
    extern __shared__ __align__(16) uint32_t ash[];
    uint32_t* pv = ash;
    const int lane = threadIdx.x;
    unsigned long long added = 0;
    int evicted = 0;
    for (int oi = 0; oi < nlost; ++oi) {
        const int i = order[oi];
        const int32_t x = lost[i];
        if (*((volatile int32_t*)seen + x)) continue;
        bool placed = false;
        for (int j = 0; j < fan && !placed; ++j) {
            const int32_t u = donors[(size_t)i * fan + j];
            if (u < 0) break;
            int du = deg[u];
            int32_t* row = adj + (size_t)u * R;
            uint8_t* pin = pinned + (size_t)u * R;
            if (du >= R) {
                // farthest non-pinned neighbour by d(u, e) (u is the pivot), first index on
                // ties; distance words compare like the distances (non-negative)
                m.load_pivot(pv, (uint32_t)u);
                long long bestd = -1;
                int bests = R;
                for (int s = lane; s < du; s += 32) {
                    if (pin[s]) continue;
                    const long long d = (long long)m.dist(pv, (uint32_t)row[s]);
                    if (d > bestd || (d == bestd && s < bests)) { bestd = d; bests = s; }
                }
                for (int o = 16; o > 0; o >>= 1) {
                    const long long od = __shfl_xor_sync(0xFFFFFFFFu, bestd, o);
                    const int os = __shfl_xor_sync(0xFFFFFFFFu, bests, o);
                    if (od > bestd || (od == bestd && os < bests)) { bestd = od; bests = os; }
                }
                __syncwarp();
                if (bests >= R) continue;  // saturated with bridges: next donor
                ++evicted;
                // remove slot `bests`, keeping order (and pins): ascending 32-wide chunks
                for (int c = bests; c < du - 1; c += 32) {
                    const int sidx = c + lane;
                    int32_t rv = -1; uint8_t pv = 0;
                    if (sidx < du - 1) { rv = row[sidx + 1]; pv = pin[sidx + 1]; }
                    __syncwarp();
                    if (sidx < du - 1) { row[sidx] = rv; pin[sidx] = pv; }
                    __syncwarp();
                }
                du -= 1;
            }
            if (lane == 0) {
                row[du] = x;
                pin[du] = 1;
                deg[u] = du + 1;
                m.open_row((uint32_t)u);  // bridged (and maybe evicted): no closure
            }
            __syncwarp();
            placed = true;
            ++added;
        }
        if (!placed) {
            if (lane == 0) { *err = 1; *err_vertex = x; }
            return;
        }
        // BFS-extend reachability from x
        if (lane == 0) { seen[x] = 1; queue[0] = x; }
        __syncwarp();
        int head = 0, tail = 1;
        while (head < tail) {
            const int32_t v = queue[head++];
            const int dv = deg[v];
            for (int s = lane; s < dv; s += 32) {
                const int32_t w = adj[(size_t)v * R + s];
                bool nw = (w >= 0) && !seen[w];
                // lanes hold distinct neighbours of one row, so no duplicate pushes
                const uint32_t m = __ballot_sync(__activemask(), nw);
                if (nw) { seen[w] = 1; queue[tail + __popc(m & lanemask_lt())] = w; }
                tail += __popc(m);
            }
            tail = __shfl_sync(0xFFFFFFFFu, tail, 0);
            __syncwarp();
        }
    }
    if (lane == 0) {
        *bridges += added;
        *evictions = evicted;
    }
}

// ---- host orchestration -----------------------------------------------------
struct Bufs {
    std::vector<Scratch*> owned;
    ~Bufs() { for (auto* s : owned) delete s; }
    template <class T> T* get(size_t n, cudaStream_t st, cudaError_t& e) {
        auto* s = new Scratch();
        owned.push_back(s);
        e = s->alloc(n * sizeof(T), st);
        return s->as<T>();
    }
};

#define BALLOC(var, T, n)                       \
    T* var = bufs.get<T>((n), st, _ce);         \
    JB_CUDA(_ce);

// JB_PROFILE=1: per-batch phase timings on stderr (stream events; diagnostics only)
struct PhaseTimer {
    bool on = false;
    cudaStream_t st = nullptr;
    std::vector<std::pair<const char*, cudaEvent_t>> ev;
    explicit PhaseTimer(cudaStream_t s) : st(s) {
        const char* e = getenv("JB_PROFILE");
        on = e && e[0] == '1';
        mark("start");
    }
    void mark(const char* name) {
        if (!on) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, st);
        ev.emplace_back(name, e);
    }
    void report(int64_t start, int64_t stop, const char* what = "batch") {
        if (!on) return;
        mark("end");
        cudaEventSynchronize(ev.back().second);
        fprintf(stderr, "[jb] %s [%lld, %lld):", what, (long long)start, (long long)stop);
        for (size_t i = 1; i < ev.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i - 1].second, ev[i].second);
            fprintf(stderr, " %s %.2fms", ev[i].first, ms);
        }
        fprintf(stderr, "\n");
        for (auto& p : ev) cudaEventDestroy(p.second);
        ev.clear();
    }
};

// Per-warp candidate-row staging budget (~26 KB per warp beside the pivot).
template <class M>
static int staged_rows(const M& m, int want, int R, int budget_kb = JB_STAGE_KB) {
    if (!M::kStage) return 0;
    int crows = std::min(want, (budget_kb * 1024 - m.pivot_words() * 4) / (m.stage_stride_words() * 4 + 4));
    return crows < R + 1 ? 0 : crows;
}

// ---- repair, approximate donors (extension, jb_insert_args.repair_beam_width) ----
// dst[i] = src row ids[i] (row_bytes each; word copies when rows are 4-byte multiples)
__global__ void gather_rows_kernel(const uint8_t* __restrict__ src, int64_t row_bytes, const int32_t* __restrict__ ids,
                                   int n, uint8_t* __restrict__ dst) {
    const int64_t total = (int64_t)n * row_bytes;
    if ((row_bytes & 3) == 0) {
        const int64_t rw = row_bytes >> 2;
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total / 4; i += (int64_t)gridDim.x * blockDim.x) {
            const int64_t r = i / rw, w = i % rw;
            reinterpret_cast<uint32_t*>(dst)[i] = reinterpret_cast<const uint32_t*>(src)[(int64_t)ids[r] * rw + w];
        }
    } else {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
            const int64_t r = i / row_bytes, b = i % row_bytes;
            dst[i] = src[(int64_t)ids[r] * row_bytes + b];
        }
    }
}

// part[w, j] = frontier key j of stranded vertex w (j < fan; UMAX past the frontier)
__global__ void frontier_head_kernel(const uint64_t* __restrict__ fk, int nlost, int L, int fan,
                                     uint64_t* __restrict__ part) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)nlost * fan) return;
    const int64_t w = i / fan;
    const int j = (int)(i % fan);
    part[i] = j < L ? fk[w * L + j] : UMAX;
}

static unsigned gather_blocks(int64_t work) {
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 8 * sm_count_current()));
}

// Donor candidates of the stranded vertices from one batched beam search (width
// repair_beam_width) from the entry point with the stranded rows as queries: the
// search only walks edges out of the reachable set, so every frontier vertex is
// reachable, and its keys are d(x, r) with r in the data role and x's norm added
// last, as in the exact scan. The top `fan` frontier keys become slice 0 of `part`.
static int approx_donors(const jb_insert_args& a, const int32_t* lost, int nlost, int64_t n_active, int64_t entry,
                         int fan, Bufs& bufs, cudaStream_t st, uint64_t*& part) {
    cudaError_t _ce;
    const int D = a.dims, Ls = a.repair_beam_width;
    jb_search_args s{};
    s.adjacency = a.adjacency; s.degree_cap = a.degree_cap; s.active_count = n_active; s.dims = D;
    auto gather = [&](const void* src, int64_t row_bytes, void*& out) -> int {
        BALLOC(buf, uint8_t, (size_t)nlost * row_bytes);
        gather_rows_kernel<<<gather_blocks((int64_t)nlost * row_bytes / 4), 256, 0, st>>>(
            static_cast<const uint8_t*>(src), row_bytes, lost, nlost, buf);
        JB_LAUNCH_CHECK();
        out = buf;
        return JB_OK;
    };
    void *q = nullptr, *qa = nullptr, *qs = nullptr;
    int rc;
    if (a.quantized) {
        s.source = JB_SRC_RABITQ;
        s.records = a.records; s.record_bytes = a.record_bytes; s.bits = a.bits;
        if ((rc = gather(a.bound_rotated, (int64_t)D * 4, q)) || (rc = gather(a.bound_qadd, 4, qa)) ||
            (rc = gather(a.bound_qsumq, 4, qs)))
            return rc;
        s.queries = static_cast<const float*>(q); s.query_add = static_cast<const float*>(qa);
        s.query_sumq = static_cast<const float*>(qs);
    } else if (a.element_kind == JB_KIND_U8) {
        s.source = JB_SRC_EXACT_U8;
        s.data_u8 = a.data_u8; s.norms_u32 = a.norms_u32;
        if ((rc = gather(a.data_u8, D, q)) || (rc = gather(a.norms_u32, 4, qa))) return rc;
        s.queries_u8 = static_cast<const uint8_t*>(q); s.query_norms_u32 = static_cast<const uint32_t*>(qa);
    } else {
        s.source = JB_SRC_EXACT;
        s.data = a.data; s.data_norms = a.data_norms;
        if ((rc = gather(a.data, (int64_t)D * 4, q)) || (rc = gather(a.data_norms, 4, qa))) return rc;
        s.queries = static_cast<const float*>(q); s.query_add = static_cast<const float*>(qa);
    }
    BALLOC(fk, uint64_t, (size_t)nlost * Ls);
    s.nq = nlost; s.starts = nullptr; s.start_vertex = entry;
    s.beam_width = Ls; s.hash_slots = 0; s.trace_cap = 0; s.frontier_keys = fk;
    if ((rc = jb_beam_search(&s, st)) != JB_OK) return rc;
    part = bufs.get<uint64_t>((size_t)nlost * fan, st, _ce); JB_CUDA(_ce);
    frontier_head_kernel<<<(unsigned)(((int64_t)nlost * fan + 255) / 256), 256, 0, st>>>(fk, nlost, Ls, fan, part);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

template <class M>
static int repair(const M& m, const jb_insert_args& a, int64_t n_active, int64_t entry, cudaStream_t st,
                  int64_t* bridges_out) {
    *bridges_out = 0;
    if (n_active < 2) return JB_OK;
    const int R = a.degree_cap, D = a.dims;
    const int fan = std::min(R, 16);
    Bufs bufs;
    cudaError_t _ce;
    BALLOC(seen, int32_t, n_active);
    BALLOC(fa, int32_t, n_active);
    BALLOC(fb, int32_t, n_active);
    BALLOC(counts, int, 8);
    BALLOC(lvl, int, BFS_MAX_LEVELS + 1);  // frontier size per BFS level
    BALLOC(lost, int32_t, n_active);
    BALLOC(reach, int32_t, n_active);
    BALLOC(pinned, uint8_t, (size_t)n_active * R);
    BALLOC(bridges, unsigned long long, 1);
    BALLOC(err, int, 3);  // no-donor flag, its vertex, evictions of the round
    JB_CUDA(cudaMemsetAsync(pinned, 0, (size_t)n_active * R, st));
    JB_CUDA(cudaMemsetAsync(bridges, 0, sizeof(unsigned long long), st));
    JB_CUDA(cudaMemsetAsync(err, 0, 3 * sizeof(int), st));
    const int T = 256;
    const unsigned nblk = (unsigned)((n_active + T - 1) / T);
    for (int round = 0;; ++round) {
        PhaseTimer rt(st);
        // BFS from the entry
        // levels are enqueued JB_BFS_BATCH at a time (one host read per batch, not per level)
        bfs_init_kernel<<<nblk, T, 0, st>>>(seen, n_active, entry, fa, lvl);
        int levels = 0;
        const unsigned eb = (unsigned)std::min<int64_t>(((int64_t)n_active * 32 + BFS_T - 1) / BFS_T, 4 * sm_count_current());
        for (int fcount = 1; fcount > 0;) {
            if (levels + BFS_BATCH >= BFS_MAX_LEVELS) { set_error("connectivity repair: BFS depth"); return JB_ECUDA; }
            JB_CUDA(cudaMemsetAsync(lvl + levels + 1, 0, BFS_BATCH * sizeof(int), st));
            for (int l = levels; l < levels + BFS_BATCH; ++l) {
                const bool odd = (l & 1) != 0;
                bfs_expand_kernel<<<eb, BFS_T, 0, st>>>(a.adjacency, R, odd ? fb : fa, lvl + l, seen, odd ? fa : fb,
                                                    lvl + l + 1);
                JB_LAUNCH_CHECK();
            }
            levels += BFS_BATCH;
            JB_CUDA(cudaMemcpyAsync(&fcount, lvl + levels, sizeof(int), cudaMemcpyDeviceToHost, st));
            JB_CUDA(cudaStreamSynchronize(st));
        }
        JB_CUDA(cudaMemsetAsync(counts + 2, 0, 2 * sizeof(int), st));
        split_kernel<<<nblk, T, 0, st>>>(seen, n_active, lost, counts + 2, reach, counts + 3);
        int h[2];
        JB_CUDA(cudaMemcpyAsync(h, counts + 2, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
        JB_CUDA(cudaStreamSynchronize(st));
        const int nlost = h[0], nreach = h[1];
        rt.mark("bfs");
        if (getenv("JB_PROFILE") && getenv("JB_PROFILE")[0] == '1')
            fprintf(stderr, "[jb]   repair round %d: stranded %d reachable %d (BFS levels %d)\n", round, nlost, nreach,
                    levels);
        if (nlost == 0) {
            rt.report(round, round, "  repair timings round");
            break;
        }
        // donors: top-`fan` reachable by (d(x, r), r) for every stranded x (build.py:185-192)
        BALLOC(donors, int32_t, (size_t)nlost * fan);
        BALLOC(okey, uint64_t, nlost);
        BALLOC(oval, int32_t, nlost);
        BALLOC(okey2, uint64_t, nlost);
        BALLOC(oval2, int32_t, nlost);
        int slices;
        uint64_t* part;
        if (a.repair_beam_width > 0) {  // approximate donors (extension)
            slices = 1;
            const int rc = approx_donors(a, lost, nlost, n_active, entry, fan, bufs, st, part);
            if (rc != JB_OK) return rc;
        } else if (std::is_same<M, F32Metric>::value) {
            // tiled A1 scan on the f32 rows of `ls` (n stranded) -> sl slices of partial top lists
            auto exact_scan = [&](const int32_t* ls, int n, uint64_t*& pt, int& sl) -> int {
                const bool res = D <= 256;
                const int sblocks = (n + DT - 1) / DT;
                sl = std::max(1, std::min(128, 4 * sm_count_current() / sblocks));  // whole waves at 2 blocks/SM
                sl = (int)std::min<int64_t>(sl, std::max<int64_t>(1, (nreach + DT - 1) / DT));
                pt = bufs.get<uint64_t>((size_t)sl * n * fan, st, _ce); JB_CUDA(_ce);
                const size_t dsm = (size_t)(DT * (res ? D + 1 : 17) + DT * 17 + DT * (DT + 1) + 1) * 4 + DT * FAN * 8;
                if (res) {
                    JB_CUDA_RC(grow_smem(donor_scan_kernel<true>, (int)dsm));
                    donor_scan_kernel<true><<<dim3(sblocks, sl), 256, dsm, st>>>(a.data, a.data_norms, D, ls, n, reach,
                                                                                nreach, sl, fan, pt);
                } else {
                    JB_CUDA_RC(grow_smem(donor_scan_kernel<false>, (int)dsm));
                    donor_scan_kernel<false><<<dim3(sblocks, sl), 256, dsm, st>>>(a.data, a.data_norms, D, ls, n, reach,
                                                                                 nreach, sl, fan, pt);
                }
                JB_LAUNCH_CHECK();
                return JB_OK;
            };
            if (donor_tc_supported(D, n_active)) {
                // tensor-core screen + exact re-rank (donor_tc.cu); uncertified rows rescanned exactly
                slices = 1;
                part = bufs.get<uint64_t>((size_t)nlost * fan, st, _ce); JB_CUDA(_ce);
                BALLOC(redo, int32_t, nlost);
                BALLOC(nredo, int, 1);
                JB_CUDA_RC(donor_scan_tc(a.data, a.data_norms, D, a.adjacency, R, seen, n_active, lost, nlost, fan, part,
                                         redo, nredo, st));
                int hredo = 0;
                JB_CUDA(cudaMemcpyAsync(&hredo, nredo, sizeof(int), cudaMemcpyDeviceToHost, st));
                JB_CUDA(cudaStreamSynchronize(st));
                if (getenv("JB_PROFILE") && getenv("JB_PROFILE")[0] == '1')
                    fprintf(stderr, "[jb]   tensor-core donor screen: %d of %d stranded rows rescanned exactly\n", hredo,
                            nlost);
                if (a.stats_out_host) {
                    a.stats_out_host[6] += nlost;
                    a.stats_out_host[7] += hredo;
                }
                if (hredo > 0) {
                    BALLOC(lost2, int32_t, hredo);
                    JB_CUDA_RC(donor_redo_ids(lost, redo, hredo, lost2, st));
                    uint64_t* part2;
                    int sl2;
                    JB_CUDA_RC(exact_scan(lost2, hredo, part2, sl2));
                    JB_CUDA_RC(donor_redo_merge(part2, sl2, hredo, fan, redo, part, st));
                }
            } else {
                JB_CUDA_RC(exact_scan(lost, nlost, part, slices));
            }
        } else {
            const int sblocks = (nlost + 7) / 8;
            slices = std::max(1, std::min(64, 8 * sm_count_current() / sblocks));
            slices = (int)std::min<int64_t>(slices, std::max<int64_t>(1, (nreach + 31) / 32));
            part = bufs.get<uint64_t>((size_t)slices * nlost * fan, st, _ce); JB_CUDA(_ce);
            const size_t gsm = (size_t)8 * m.pivot_words() * 4;
            JB_CUDA_RC(grow_smem(donor_scan_generic_kernel<M>, (int)gsm));
            donor_scan_generic_kernel<M><<<dim3(sblocks, slices), 256, gsm, st>>>(m, lost, nlost, reach, nreach, slices,
                                                                                 fan, part);
        }
        JB_LAUNCH_CHECK();
        rt.mark("scan");
        donor_merge_kernel<<<(unsigned)((nlost * 32 + 255) / 256), 256, 0, st>>>(part, slices, nlost, fan, lost, donors,
                                                                               okey, oval);
        JB_LAUNCH_CHECK();
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, okey, okey2, oval, oval2, nlost, 0, 64, st);
        BALLOC(tmp, unsigned char, tb);
        JB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, okey, okey2, oval, oval2, nlost, 0, 64, st));
        const int asm_bytes = m.pivot_words() * 4;
        JB_CUDA_RC(grow_smem(attach_kernel<M>, asm_bytes));
        rt.mark("order");
        attach_kernel<M><<<1, 32, asm_bytes, st>>>(m, a.adjacency, a.degrees, R, pinned, seen, lost, oval2, nlost,
                                                    donors, fan, fa, bridges, err, err + 1, err + 2);
        JB_LAUNCH_CHECK();
        rt.mark("attach");
        rt.report(round, round, "  repair timings round");
        int herr[3];
        JB_CUDA(cudaMemcpyAsync(herr, err, 3 * sizeof(int), cudaMemcpyDeviceToHost, st));
        JB_CUDA(cudaStreamSynchronize(st));
        if (herr[0]) {
            set_error("connectivity repair: no donor for vertex %d", herr[1]);
            return JB_ENODONOR;
        }
        // Without evictions the round only added edges: every vertex reachable before
        // still is, and the attach kernel's BFS-extend marked each bridged vertex and
        // what it reaches, so the next round's BFS would find nothing stranded.
        if (herr[2] == 0) {
            if (getenv("JB_PROFILE") && getenv("JB_PROFILE")[0] == '1')
                fprintf(stderr, "[jb]   repair round %d: no evictions, reachability complete\n", round);
            break;
        }
        if (round > 10000) { set_error("connectivity repair did not converge"); return JB_ECUDA; }
    }
    unsigned long long hb = 0;
    JB_CUDA(cudaMemcpyAsync(&hb, bridges, sizeof(hb), cudaMemcpyDeviceToHost, st));
    JB_CUDA(cudaStreamSynchronize(st));
    *bridges_out = (int64_t)hb;
    return JB_OK;
}

// Phase-1 search with visited-trace capture: queries are rows [q0, q0 + nq) of the
// dataset, the graph shows `active` vertices. The trace capacity is generous
// (8 B per slot); a longer trace re-runs the batch with an exact-size buffer.
// Trace distances are the keys' 32-bit words (f32 bits, or u32 integer distances).
static int trace_search(const jb_insert_args& a, int64_t q0, int64_t nq, int64_t active, int64_t entry, Bufs& bufs,
                        cudaStream_t st, int& cap, int32_t*& hops, int32_t*& evals, int32_t*& tids, uint32_t*& tdst) {
    cudaError_t _ce;
    const int R = a.degree_cap, D = a.dims, L = a.build_beam_width;
    cap = std::max(4 * L, L + 512);
    BALLOC(fk, uint64_t, (size_t)nq * L);
    BALLOC(h, int32_t, nq);
    BALLOC(ev, int32_t, nq);
    BALLOC(flags, int32_t, nq);
    hops = h;
    evals = ev;
    for (int attempt = 0; attempt < 2; ++attempt) {
        tids = bufs.get<int32_t>((size_t)nq * cap, st, _ce); JB_CUDA(_ce);
        tdst = bufs.get<uint32_t>((size_t)nq * cap, st, _ce); JB_CUDA(_ce);
        jb_search_args s{};
        s.adjacency = a.adjacency; s.degree_cap = R; s.active_count = active; s.dims = D;
        if (a.quantized) {  // run_beam_searches(graph, quantizer, rows) (build.py:322-325)
            s.source = JB_SRC_RABITQ;
            s.records = a.records; s.record_bytes = a.record_bytes; s.bits = a.bits;
            s.queries = a.bound_rotated + (size_t)q0 * D; s.query_add = a.bound_qadd + q0;
            s.query_sumq = a.bound_qsumq + q0;
        } else if (a.element_kind == JB_KIND_U8) {
            s.source = JB_SRC_EXACT_U8;
            s.data_u8 = a.data_u8; s.norms_u32 = a.norms_u32;
            s.queries_u8 = a.data_u8 + (size_t)q0 * D; s.query_norms_u32 = a.norms_u32 + q0;
        } else {
            s.source = JB_SRC_EXACT;
            s.data = a.data; s.data_norms = a.data_norms;
            s.queries = a.data + (size_t)q0 * D; s.query_add = a.data_norms + q0;
            s.screen = a.screen; s.screen_center = a.screen_center;
        }
        s.nq = nq; s.starts = nullptr; s.start_vertex = entry;
        s.beam_width = L; s.hash_slots = 0; s.trace_cap = cap;
        s.frontier_keys = fk; s.hops = h; s.evals = ev; s.trace_ids = tids;
        s.trace_dists = reinterpret_cast<float*>(tdst); s.flags = flags;
        int rc = jb_beam_search(&s, st);
        if (rc) return rc;
        size_t tb = 0;
        BALLOC(mx, int32_t, 1);
        cub::DeviceReduce::Max(nullptr, tb, h, mx, (int)nq, st);
        BALLOC(tmp, unsigned char, tb);
        JB_CUDA(cub::DeviceReduce::Max(tmp, tb, h, mx, (int)nq, st));
        int hmax = 0;
        JB_CUDA(cudaMemcpyAsync(&hmax, mx, sizeof(int), cudaMemcpyDeviceToHost, st));
        JB_CUDA(cudaStreamSynchronize(st));
        if (hmax <= cap) break;
        cap = hmax;  // re-run with an exact-size trace buffer (rare)
    }
    return JB_OK;
}

// Global-pool slots the owner of segment s takes: deg[t] + g when that exceeds the
// OWNER_SC smem candidate slots (else 0). Summed to size the pool exactly (with
// R = 64 nearly every target spills, so no fixed multiple of the triple count fits).
__global__ void owner_pool_need_kernel(const uint32_t* __restrict__ tgt, int64_t total,
                                       const int32_t* __restrict__ seg_start, int nseg,
                                       const int32_t* __restrict__ deg, unsigned long long* __restrict__ need) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nseg) return;
    const int64_t g0 = seg_start[s];
    const uint32_t t = tgt[g0];
    int64_t g1 = s + 1 < nseg ? (int64_t)seg_start[s + 1] : g0 + 1;
    if (s + 1 >= nseg)
        while (g1 < total && tgt[g1] == t) ++g1;  // last segment: ends at the NO_TARGET tail
    const int64_t c = (int64_t)deg[t] + (g1 - g0);
    need[s] = c > OWNER_SC ? (unsigned long long)c : 0ull;
}

// JB_P2_SCREEN=0: phase 2 stages f32 rows even when screen records are given (A/B)
static bool p2_screen_on() {
    const char* e = getenv("JB_P2_SCREEN");
    return !(e && e[0] == '0');
}

// JB_CLOSED_PASS=0: closed rows stay on the staged deferred pass (A/B)
static bool closed_pass_on() {
    const char* e = getenv("JB_CLOSED_PASS");  // read per batch (A/B within one process)
    return !(e && e[0] == '0');
}

// staging rows beyond R of the closed pass (JB_CLOSED_EXTRA; default the deferred
// pass's R + JB_OWNER_EXTRA: fewer rows measured no faster, 1M x 128 build 0.454 s at
// +16 vs 0.457-0.460 s at +6..+12, `tools/exp_build_ab.py`)
static int closed_extra() {
    const char* e = getenv("JB_CLOSED_EXTRA");
    return e ? std::max(1, atoi(e)) : JB_OWNER_EXTRA;
}

// Phase 3 (build.py:269-293): (target, dist, source) order via two stable radix
// sorts of the reverse triples, segment heads, one owner warp per target.
template <class M>
static int merge_phase(const M& m, const jb_insert_args& a, double alpha2, uint32_t* tt, uint64_t* tk, int64_t ntri,
                       Bufs& bufs, cudaStream_t st, int& hseg) {
    cudaError_t _ce;
    const int R = a.degree_cap;
    BALLOC(tt2, uint32_t, ntri);
    BALLOC(tk2, uint64_t, ntri);
    {
        size_t tb1 = 0, tb2 = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb1, tk, tk2, tt, tt2, (int)ntri, 0, 64, st);
        cub::DeviceRadixSort::SortPairs(nullptr, tb2, tt2, tt, tk2, tk, (int)ntri, 0, 32, st);
        BALLOC(tmp, unsigned char, std::max(tb1, tb2));
        size_t tb = std::max(tb1, tb2);
        JB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, tk, tk2, tt, tt2, (int)ntri, 0, 64, st));  // by (dist, source)
        tb = std::max(tb1, tb2);
        JB_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, tt2, tt, tk2, tk, (int)ntri, 0, 32, st));  // stable by target
    }
    BALLOC(flag, uint8_t, ntri);
    BALLOC(seg, int32_t, ntri);
    BALLOC(nseg, int, 1);
    seg_head_kernel<<<(unsigned)((ntri + 255) / 256), 256, 0, st>>>(tt, ntri, flag);
    {
        size_t tb = 0;
        cub::DeviceSelect::Flagged(nullptr, tb, cub::CountingInputIterator<int32_t>(0), flag, seg, nseg, (int)ntri, st);
        BALLOC(tmp, unsigned char, tb);
        JB_CUDA(cub::DeviceSelect::Flagged(tmp, tb, cub::CountingInputIterator<int32_t>(0), flag, seg, nseg, (int)ntri,
                                           st));
    }
    hseg = 0;
    JB_CUDA(cudaMemcpyAsync(&hseg, nseg, sizeof(int), cudaMemcpyDeviceToHost, st));
    JB_CUDA(cudaStreamSynchronize(st));
    if (hseg > 0) {
        int pool_cap = 1024;
        {
            BALLOC(need, unsigned long long, hseg);
            BALLOC(need_sum, unsigned long long, 1);
            owner_pool_need_kernel<<<(unsigned)((hseg + 255) / 256), 256, 0, st>>>(tt, ntri, seg, hseg, a.degrees, need);
            JB_LAUNCH_CHECK();
            size_t tb = 0;
            cub::DeviceReduce::Sum(nullptr, tb, need, need_sum, hseg, st);
            BALLOC(tmp, unsigned char, tb);
            JB_CUDA(cub::DeviceReduce::Sum(tmp, tb, need, need_sum, hseg, st));
            unsigned long long hneed = 0;
            JB_CUDA(cudaMemcpyAsync(&hneed, need_sum, sizeof(hneed), cudaMemcpyDeviceToHost, st));
            JB_CUDA(cudaStreamSynchronize(st));
            if (hneed + 1024 > (unsigned long long)INT32_MAX) { set_error("phase 3: candidate pool too large"); return JB_EOVERFLOW; }
            pool_cap = (int)(hneed + 1024);
        }
        BALLOC(pool, uint64_t, pool_cap);
        BALLOC(ptop, unsigned long long, 1);
        BALLOC(err, int, 1);
        JB_CUDA(cudaMemsetAsync(ptop, 0, sizeof(unsigned long long), st));
        JB_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
        // owners stage up to R + 16 candidate rows in smem when they fit; R + 8 instead
        // when that lifts the kernel from 2 to 3 resident blocks per SM (short rows)
        int crows = staged_rows(m, R + JB_OWNER_EXTRA, R);
        const int crows_lo = staged_rows(m, R + JB_OWNER_EXTRA / 2, R);
        const int smem_sm = 227 * 1024;
        if (crows_lo > 0 && smem_sm / (owner_per_warp(m, R, crows) * BW) < 3 &&
            smem_sm / (owner_per_warp(m, R, crows_lo) * BW) >= 3)
            crows = crows_lo;
        bool launched = false;
        if constexpr (std::is_same<M, F32Metric>::value) {
            // rows too large to stage per warp: block per target, dot matrix — when the
            // candidate sets (R + a few fresh) fit the 64-row tile; else the warp kernel
            if (crows == 0 && R + 16 <= MX - 1 && !kNoMatrix) {
                const size_t msm = (size_t)(MX * (MX + 1) + MX * 17 + MX) * 4 + MX * 4 + OWNER_SC * 8 + 3 * R * 4 +
                                   (((size_t)a.dims + 3) / 4 * 4 + 4) * 4 + 16;
                JB_CUDA_RC(grow_smem(owner_matrix_kernel, (int)msm));
                owner_matrix_kernel<<<(unsigned)hseg, 256, msm, st>>>(m, alpha2, R, a.always_prune, tt, tk, ntri, seg,
                                                                       pool, ptop, pool_cap, a.adjacency, a.degrees, err);
                launched = true;
            }
        }
        const int osm = owner_per_warp(m, R, crows) * BW;
#ifdef JB_OWNER_SPLIT
        const M mo = split_prune(m);  // dev A/B
#else
        const M& mo = m;
#endif
        const char* oe = getenv("JB_OWNER_DEFER");
        if (launched) {
        } else if (oe && oe[0] == '0') {  // A/B: one pass, every target at the staging kernel's occupancy
            JB_CUDA_RC(grow_smem(owner_merge_kernel<M, 0>, osm));
            owner_merge_kernel<M, 0><<<(unsigned)((hseg + BW - 1) / BW), BW * 32, osm, st>>>(
                mo, alpha2, R, a.always_prune, tt, tk, ntri, seg, nseg, pool, ptop, pool_cap, a.adjacency, a.degrees, err,
                crows, nullptr, nullptr, 0);
        } else {
            // light pass (appends, no staged rows: high occupancy), then the targets
            // that need a prune on a persistent grid of the staging kernel
            // closed f32 rows (prune closure on) get their own list and pass (MODE 3)
            bool closed_pass = false;
            if constexpr (std::is_same<M, F32Metric>::value) closed_pass = m.closure != nullptr && closed_pass_on();
            const int64_t dstride = closed_pass ? hseg : 0;
            BALLOC(defer, int32_t, closed_pass ? 2 * (int64_t)hseg : hseg);
            BALLOC(ndefer, int, 2);
            JB_CUDA(cudaMemsetAsync(ndefer, 0, 2 * sizeof(int), st));
            const int lsm = owner_light_per_warp(R) * BW;
            JB_CUDA_RC(grow_smem(owner_merge_kernel<M, 1>, lsm));
            const int crows3 = closed_pass ? staged_rows(m, R + closed_extra(), R) : 0;
            owner_merge_kernel<M, 1><<<(unsigned)((hseg + BW - 1) / BW), BW * 32, lsm, st>>>(
                mo, alpha2, R, a.always_prune, tt, tk, ntri, seg, nseg, pool, ptop, pool_cap, a.adjacency, a.degrees, err,
                crows3, defer, ndefer, crows3 > 0 ? dstride : 0);
            JB_LAUNCH_CHECK();
            if (closed_pass && crows3 > 0) {
                // 1-warp blocks: the ~20 KB per-warp staging packs the SM best in single warps
                const int osm3 = owner_per_warp(m, R, crows3);
                JB_CUDA_RC(grow_smem(owner_merge_kernel<M, 3>, osm3));
                int per_sm3 = 0;
                JB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm3, owner_merge_kernel<M, 3>, 32, osm3));
                const unsigned g3 = (unsigned)std::max<int64_t>(
                    1, std::min<int64_t>(hseg, (int64_t)std::max(1, per_sm3) * sm_count_current()));
                owner_merge_kernel<M, 3><<<g3, 32, osm3, st>>>(mo, alpha2, R, a.always_prune, tt, tk, ntri, seg,
                                                              nseg, pool, ptop, pool_cap, a.adjacency, a.degrees,
                                                              err, crows3, defer, ndefer, dstride);
                JB_LAUNCH_CHECK();
            }
            const int osm2 = owner_per_warp(m, R, crows) * OWNER_BW;
            JB_CUDA_RC(grow_smem(owner_merge_kernel<M, 2>, osm2));
            int per_sm = 0;
            JB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, owner_merge_kernel<M, 2>, OWNER_BW * 32, osm2));
            const int64_t want = (hseg + OWNER_BW - 1) / OWNER_BW;
            const unsigned g2 = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)std::max(1, per_sm) *
                                                                                       sm_count_current()));
            owner_merge_kernel<M, 2><<<g2, OWNER_BW * 32, osm2, st>>>(mo, alpha2, R, a.always_prune, tt, tk, ntri, seg, nseg,
                                                               pool, ptop, pool_cap, a.adjacency, a.degrees, err, crows,
                                                               defer, ndefer, dstride);
        }
        JB_LAUNCH_CHECK();
        int herr = 0;
        JB_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
        JB_CUDA(cudaStreamSynchronize(st));
        if (herr) { set_error("phase 3: candidate pool overflow"); return JB_EOVERFLOW; }
    }
    return JB_OK;
}

// out[0] += sum(v[0..n)), out[1] += sum(w[0..n)) (work counters; int64 totals)
__global__ void sum2_kernel(const int32_t* __restrict__ v, const int32_t* __restrict__ w, int64_t n,
                            unsigned long long* __restrict__ out) {
    unsigned long long a = 0, b = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        a += (unsigned)v[i];
        b += (unsigned)w[i];
    }
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xFFFFFFFFu, a, o);
        b += __shfl_xor_sync(0xFFFFFFFFu, b, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out, a);
        atomicAdd(out + 1, b);
    }
}

static int sum2(const int32_t* v, const int32_t* w, int64_t n, Bufs& bufs, cudaStream_t st, unsigned long long out[2]) {
    cudaError_t _ce;
    BALLOC(work, unsigned long long, 2);
    JB_CUDA(cudaMemsetAsync(work, 0, 2 * sizeof(unsigned long long), st));
    sum2_kernel<<<std::max(1, std::min<int>((int)((n + 255) / 256), 4 * sm_count_current())), 256, 0, st>>>(v, w, n,
                                                                                                         work);
    JB_LAUNCH_CHECK();
    JB_CUDA(cudaMemcpyAsync(out, work, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    return JB_OK;
}


static int validate_insert(const jb_insert_args& a) {
    JB_CHECK_ARG(a.adjacency && a.degrees, "batch insert: missing graph arrays");
    if (a.quantized) {
        JB_CHECK_ARG(a.element_kind == JB_KIND_F32, "quantized construction requires f32 data");
        JB_CHECK_ARG(a.bits == 1 || a.bits == 2 || a.bits == 4 || a.bits == 8, "bits must be one of (1, 2, 4, 8)");
        JB_CHECK_ARG(a.records && a.bound_rotated && a.bound_qadd && a.bound_qsumq,
                     "quantized construction: missing records / bound rows");
        JB_CHECK_ARG(a.record_bytes == jb_rabitq_record_bytes(a.dims, a.bits), "quantized construction: record_bytes");
    }
    JB_CHECK_ARG(a.element_kind == JB_KIND_F32 || a.element_kind == JB_KIND_U8, "unknown element kind %d",
                 a.element_kind);
    if (a.element_kind == JB_KIND_U8) {
        JB_CHECK_ARG(a.data_u8 && a.norms_u32, "batch insert: missing u8 rows / norms");
        JB_CHECK_ARG((int64_t)a.dims * 255 * 255 < (1ll << 32), "u8 dims too large for 32-bit packed distances");
    } else {
        JB_CHECK_ARG(a.data && a.data_norms, "batch insert: missing arrays");
    }
    JB_CHECK_ARG(a.degree_cap >= 1 && a.dims >= 1, "batch insert: bad shape");
    JB_CHECK_ARG(a.alpha >= 1.0, "alpha must be >= 1");
    JB_CHECK_ARG(a.start >= 0 && a.start <= a.stop, "batch insert: bad range");
    JB_CHECK_ARG(a.stop <= a.count, "id range exceeds dataset count");
    JB_CHECK_ARG(a.stop <= a.capacity, "id range exceeds graph capacity");
    JB_CHECK_ARG(a.stop < (1ll << 31), "ids exceed int32");
    return JB_OK;
}

template <class M>
static int batch_insert_impl(const M& m, const jb_insert_args& a, cudaStream_t st) {
    int rc = 0;
    const int R = a.degree_cap, D = a.dims;
    const double alpha2 = a.alpha * a.alpha;
    int64_t entry = a.entry_point;
    int64_t bridges = 0;
    if (a.entry_point_out_host) *a.entry_point_out_host = entry;
    if (a.bridges_out_host) *a.bridges_out_host = 0;
    if (a.start == a.stop) return JB_OK;
    const int64_t nb = a.stop - a.start;
    Bufs bufs;
    cudaError_t _ce;
    PhaseTimer pt(st);

    if (a.start == 0) {  // seed batch: medoid entry + mutual pruning (build.py:246-266)
        rc = a.element_kind == JB_KIND_U8 ? jb_medoid_u8(a.data_u8, a.stop, D, &entry, st)
                                          : jb_medoid(a.data, a.stop, D, &entry, st);
        if (rc) return rc;
        if (nb > 1) {
            // pivots in tiles: scratch is tile x (nb - 1) keys (<= 1 GiB), not nb^2. The
            // reference's seed batch is all-pairs too (build.py:254-266); a tile's rows are
            // written as it finishes and no pivot reads adjacency, so tiling is exact.
            const int64_t tile = std::max<int64_t>(BW, std::min<int64_t>(nb, ((int64_t)1 << 27) / (nb - 1)));
            BALLOC(cand, uint64_t, (size_t)tile * (nb - 1));
            BALLOC(kid, int32_t, (size_t)tile * R);
            BALLOC(kd, uint32_t, (size_t)tile * R);
            const int smem = BW * m.pivot_words() * 4;
            JB_CUDA_RC(grow_smem(seed_prune_kernel<M>, smem));
            for (int64_t t0 = 0; t0 < nb; t0 += tile) {
                const int64_t t1 = std::min(nb, t0 + tile);
                seed_prune_kernel<M><<<(unsigned)((t1 - t0 + BW - 1) / BW), BW * 32, smem, st>>>(
                    m, a.start, a.stop, t0, t1, alpha2, R, cand, kid, kd, a.adjacency, a.degrees);
                JB_LAUNCH_CHECK();
            }
        }
        rc = repair(m, a, a.stop, entry, st, &bridges);
        if (a.entry_point_out_host) *a.entry_point_out_host = entry;
        if (a.bridges_out_host) *a.bridges_out_host = bridges;
        if (a.stats_out_host) {
            a.stats_out_host[2] += nb * (nb - 1);  // seed: every vertex prunes over all others
            a.stats_out_host[5] += bridges;
        }
        return rc;
    }

    // ---- phase 1: batched search of the new rows on the read-only graph ----
    int cap = 0;
    int32_t *hops = nullptr, *evals = nullptr, *tids = nullptr;
    uint32_t* tdst = nullptr;
    rc = trace_search(a, a.start, nb, a.start, entry, bufs, st, cap, hops, evals, tids, tdst);
    if (rc) return rc;
    unsigned long long hwork[2] = {0, 0};
    if (a.stats_out_host && (rc = sum2(hops, evals, nb, bufs, st, hwork))) return rc;
    pt.mark("search");

    // ---- phase 2: activate, prune each new vertex, emit reverse triples ----
    const int W = a.reverse_all_visited ? cap : R;
    const int64_t ntri = nb * (int64_t)W;
    JB_CHECK_ARG(ntri < INT32_MAX, "batch of %lld rows x %d reverse slots exceeds the 2^31 sort limit; "
                 "use a smaller max_batch", (long long)nb, W);
    BALLOC(cand, uint64_t, (size_t)nb * cap);
    BALLOC(kid, int32_t, (size_t)nb * R);
    BALLOC(kd, uint32_t, (size_t)nb * R);
    BALLOC(tt, uint32_t, ntri);
    BALLOC(tk, uint64_t, ntri);
    // smem-staged candidate rows when a trace fits in ~26 KB per warp; longer traces
    // prune from L1/L2 (staging them would cost more occupancy than it saves)
    // stage traces of up to P2_ROWS candidates (1-warp blocks: smem per warp sets the
    // occupancy exactly); longer traces prune from global rows
    const int crows2 = staged_rows(m, std::min(cap, a.build_beam_width + JB_P2_ROWS_OVER_L), R, JB_P2_KB);
    bool p2_done = false;
    if constexpr (std::is_same<M, F32Metric>::value) {
        // rows too large to stage per warp: block per vertex, dot matrix — when the
        // traces (about 1.1 x L_build) fit 128 rows; else the warp kernel
        if (crows2 == 0 && a.build_beam_width <= 96 && !kNoMatrix) {
            const size_t psm = (size_t)(MX2 * (MX2 + 1) + 2 * 64 * 17 + MX2) * 4 + MX2 * 4 +
                               (((size_t)a.dims + 3) / 4 * 4 + 4) * 4;
            JB_CUDA_RC(grow_smem(phase2_matrix_kernel, (int)psm));
            phase2_matrix_kernel<<<(unsigned)nb, 256, psm, st>>>(m, a.start, nb, alpha2, R, hops, tids, tdst, cap,
                                                                 a.reverse_all_visited, cand, kid, kd, a.adjacency,
                                                                 a.degrees, tt, tk, W);
            p2_done = true;
        }
    }
    if constexpr (std::is_same<M, F32Metric>::value) {
        // screen records available (f32 rows): the int8-screened staged prune
        if (!p2_done && a.screen != nullptr && p2_screen_on()) {
            const int rb = jb_screen_record_bytes(a.dims);
            const int srows = std::min(cap, a.build_beam_width + JB_P2_ROWS_OVER_L);
            const int sm = p2s_warp_bytes(srows, rb, a.dims);
            JB_CUDA_RC(grow_smem(phase2_screen_kernel, sm));
            phase2_screen_kernel<<<(unsigned)nb, 32, sm, st>>>(m, a.screen, rb, srows, a.start, nb, alpha2, R, hops, tids,
                                                                tdst, cap, a.reverse_all_visited, cand, kid, kd,
                                                                a.adjacency, a.degrees, tt, tk, W);
            p2_done = true;
        }
    }
    const int p2_smem = P2_BW * 4 * vertex_warp_words(m, crows2);
    JB_CUDA_RC(grow_smem(phase2_kernel<M>, p2_smem));
    if (!p2_done)
    phase2_kernel<M><<<(unsigned)((nb + P2_BW - 1) / P2_BW), P2_BW * 32, p2_smem, st>>>(
        split_prune(m), a.start, nb, alpha2, R, hops, tids, tdst, cap, a.reverse_all_visited, cand, kid, kd, a.adjacency, a.degrees,
        tt, tk, W, crows2);
    JB_LAUNCH_CHECK();
    pt.mark("prune");

    // ---- phase 3: grouped reverse-edge merge ----
    int hseg = 0;
    rc = merge_phase(m, a, alpha2, tt, tk, ntri, bufs, st, hseg);
    if (rc) return rc;
    pt.mark("merge");

    // ---- connectivity repair over the activated graph ----
    rc = repair(m, a, a.stop, entry, st, &bridges);
    pt.mark("repair");
    pt.report(a.start, a.stop);
    if (pt.on) fprintf(stderr, "[jb]   bridges %lld\n", (long long)bridges);
    if (a.entry_point_out_host) *a.entry_point_out_host = entry;
    if (a.bridges_out_host) *a.bridges_out_host = bridges;
    if (a.stats_out_host) {
        int64_t* w = a.stats_out_host;
        w[0] += (int64_t)hwork[0];
        w[1] += (int64_t)hwork[1];
        w[2] += (int64_t)hwork[0];  // each new vertex prunes over its visited trace
        w[3] += hseg;
        w[4] += ntri;
        w[5] += bridges;
    }
    return rc;
}

template <class M>
static int refine_batch_impl(const M& m, const jb_insert_args& a, int64_t active, cudaStream_t st) {
    const int R = a.degree_cap;
    const double alpha2 = a.alpha * a.alpha;
    const int64_t nb = a.stop - a.start;
    Bufs bufs;
    cudaError_t _ce;
    PhaseTimer pt(st);
    int cap = 0;
    int32_t *hops = nullptr, *evals = nullptr, *tids = nullptr;
    uint32_t* tdst = nullptr;
    int rc = trace_search(a, a.start, nb, active, a.entry_point, bufs, st, cap, hops, evals, tids, tdst);
    if (rc) return rc;
    pt.mark("search");
    const int64_t ntri = nb * (int64_t)R;
    BALLOC(cand, uint64_t, (size_t)nb * (cap + R));
    BALLOC(kid, int32_t, (size_t)nb * R);
    BALLOC(kd, uint32_t, (size_t)nb * R);
    BALLOC(tt, uint32_t, ntri);
    BALLOC(tk, uint64_t, ntri);
    BALLOC(ncand, int32_t, nb);
    const int crows = staged_rows(m, cap + R, R);
    const int smem = BW * 4 * vertex_warp_words(m, crows);
    JB_CUDA_RC(grow_smem(refine_prune_kernel<M>, smem));
    refine_prune_kernel<M><<<(unsigned)((nb + BW - 1) / BW), BW * 32, smem, st>>>(
        split_prune(m), a.start, nb, alpha2, R, hops, tids, tdst, cap, cand, kid, kd, a.adjacency, a.degrees, tt, tk, crows, ncand);
    JB_LAUNCH_CHECK();
    pt.mark("prune");
    int hseg = 0;
    rc = merge_phase(m, a, alpha2, tt, tk, ntri, bufs, st, hseg);
    if (rc) return rc;
    pt.mark("merge");
    pt.report(a.start, a.stop);
    if (a.stats_out_host) {
        unsigned long long hw[2] = {0, 0}, pc[2] = {0, 0};
        if ((rc = sum2(hops, evals, nb, bufs, st, hw))) return rc;
        if ((rc = sum2(ncand, ncand, nb, bufs, st, pc))) return rc;
        JB_CUDA(cudaStreamSynchronize(st));
        int64_t* w = a.stats_out_host;
        w[0] += (int64_t)hw[0];
        w[1] += (int64_t)hw[1];
        w[2] += (int64_t)pc[0];
        w[3] += hseg;
        w[4] += ntri;
    }
    JB_CUDA(cudaStreamSynchronize(st));
    return JB_OK;
}

// Run f with the construction metric of the call: RaBitQ estimates, u8 or f32 rows.
template <class F>
static int with_metric(const jb_insert_args& a, F&& f) {
    if (a.quantized) {
        switch (a.bits) {
            case 1: return f(RabitqMetric<1>{a.records, a.record_bytes, a.bound_rotated, a.bound_qadd, a.bound_qsumq, a.dims});
            case 2: return f(RabitqMetric<2>{a.records, a.record_bytes, a.bound_rotated, a.bound_qadd, a.bound_qsumq, a.dims});
            case 4: return f(RabitqMetric<4>{a.records, a.record_bytes, a.bound_rotated, a.bound_qadd, a.bound_qsumq, a.dims});
            default: return f(RabitqMetric<8>{a.records, a.record_bytes, a.bound_rotated, a.bound_qadd, a.bound_qsumq, a.dims});
        }
    }
    if (a.element_kind == JB_KIND_U8) return f(U8Metric{a.data_u8, a.norms_u32, a.dims});
    F32Metric m{a.data, a.data_norms, a.dims};
    const char* e = getenv("JB_GRAM");
    m.gram = !(e && e[0] == '0');
    const char* c = getenv("JB_CLOSURE");
    m.closure = (c && c[0] == '0') ? nullptr : a.closure;  // JB_CLOSURE=0: full prunes (A/B)
    return f(m);
}

}  // namespace jb

using namespace jb;

extern "C" {

int jb_repair_connectivity(const jb_insert_args* args, void* stream) {
    JB_CHECK_ARG(args, "null args");
    const jb_insert_args& a = *args;
    int rc = validate_insert(a);
    if (rc) return rc;
    int64_t b = 0;
    cudaStream_t st = as_stream(stream);
    rc = with_metric(a, [&](auto m) { return repair(m, a, a.stop, a.entry_point, st, &b); });
    if (a.bridges_out_host) *a.bridges_out_host = b;
    if (a.entry_point_out_host) *a.entry_point_out_host = a.entry_point;
    return rc;
}

int jb_batch_insert(const jb_insert_args* args, void* stream) {
    JB_CHECK_ARG(args, "null args");
    const jb_insert_args& a = *args;
    int rc = validate_insert(a);
    if (rc) return rc;
    cudaStream_t st = as_stream(stream);
    return with_metric(a, [&](auto m) { return batch_insert_impl(m, a, st); });
}

int jb_refine_batch(const jb_insert_args* args, void* stream) {
    JB_CHECK_ARG(args, "null args");
    const jb_insert_args& a = *args;
    int rc = validate_insert(a);
    if (rc) return rc;
    const int64_t active = a.active_count > 0 ? a.active_count : a.stop;
    JB_CHECK_ARG(a.stop <= active && active <= a.capacity && active <= a.count, "refine: range beyond the active graph");
    JB_CHECK_ARG(a.entry_point >= 0 && a.entry_point < active, "refine: entry point out of range");
    if (a.entry_point_out_host) *a.entry_point_out_host = a.entry_point;  // refinement never moves the entry
    if (a.bridges_out_host) *a.bridges_out_host = 0;
    if (a.start == a.stop) return JB_OK;
    cudaStream_t st = as_stream(stream);
    return with_metric(a, [&](auto m) { return refine_batch_impl(m, a, active, st); });
}

int jb_robust_prune(const float* data, const float* data_norms, int32_t dims, const int64_t* pivots, int64_t count,
                    const int64_t* offsets, const int32_t* cand_ids, const float* cand_dists, double alpha,
                    int32_t degree_cap, int32_t* out_ids, float* out_dists, int32_t* out_counts, void* stream) {
    JB_CHECK_ARG(alpha >= 1.0, "alpha must be >= 1");
    JB_CHECK_ARG(degree_cap >= 1, "degree_cap must be >= 1");
    JB_CHECK_ARG(dims >= 1, "dims must be >= 1");
    if (count == 0) return JB_OK;
    cudaStream_t st = as_stream(stream);
    int64_t total = 0;
    JB_CUDA(cudaMemcpyAsync(&total, offsets + count, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    JB_CUDA(cudaStreamSynchronize(st));
    Scratch cand;
    JB_CUDA(cand.alloc((size_t)std::max<int64_t>(total, 1) * 8, st));
    const F32Metric m{data, data_norms, dims};
    const int smem = BW * m.pivot_words() * 4;
    JB_CUDA_RC(grow_smem(prune_batch_kernel, smem));
    prune_batch_kernel<<<(unsigned)((count + BW - 1) / BW), BW * 32, smem, st>>>(
        m, pivots, count, offsets, cand_ids, cand_dists, alpha * alpha, degree_cap, cand.as<uint64_t>(), out_ids,
        out_dists, out_counts);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

}  // extern "C"
