// donor_tc.cu — tensor-core screened nearest-donor scan for connectivity repair.
//
// Replaces the CUDA-core exact scan (donor_scan_kernel, build.cu) for f32 rows
// with D % 4 == 0 and D <= 128. The reference (build.py:185-192) picks, for every
// stranded vertex x, the `fan` reachable vertices r with the smallest keys
// (d(x, r), r), d in the reference's f32 einsum order (A1) with r in the data
// role and x's norm added last. Results here are identical; the work is split as
//
//   1. seed  (donor_seed_kernel, warp per x): exact keys of the reachable vertices
//      within two hops of x in the graph; the fan-th smallest distinct one is an
//      upper bound tau_x on x's fan-th donor distance (+inf if fewer than fan);
//   2. screen (donor_screen_tc_kernel): every (data row r, stranded x) dot product
//      on the 5th-gen tensor cores — tcgen05.mma kind::tf32, f32 rows fed by TMA
//      (128 B swizzle) straight from the dataset, accumulators in TMEM — and the
//      epilogue keeps r as a candidate of x iff r is reachable and
//        d~(x, r) - err(x, r) <= tau_x,
//      d~ = |r|^2 + |x|^2 - 2 <r, x>_tf32 and err a rigorous bound on
//      |d~ - d_A1| (below), so every true donor is kept;
//   3. exact (donor_exact_kernel, warp per x): A1-order keys of the candidates,
//      top `fan` by (dist, id) -> the slice layout donor_merge_kernel consumes.
// A stranded row whose candidate list overflows gets a second screen pass with
// tau refined from its first candidates; one with no finite tau, or a second
// overflow, is rescanned by the exact CUDA-core kernel (build.cu), so the output
// never depends on the screen's selectivity.
//
// Error bound (per pair; tf32 keeps 10 mantissa bits, |rel err| < 2^-10 per
// operand; f32 accumulation over K <= 128 terms adds < 2^-17 relative):
//   |<r,x>_tf32 - <r,x>| < (2^-9 + 2^-17 + 2^-20) sum_e |r_e x_e| <= 2^-8.99 |r| |x|
//   |<r,x>_A1  - <r,x>|  < 2^-19 |r| |x|       (4 chains of <= 32 adds + 2)
//   rounding of the two distance evaluations < 2^-21 (|r|^2 + |x|^2)
// so err = 2^-7 |r| |x| + 2^-18 (|r|^2 + |x|^2) holds with a 2x (8x) margin on each term.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include "common.cuh"
#include "runtime.cuh"
#include "donor_tc.cuh"

namespace jb {

constexpr int TC_M = 128;        // data rows per tile (TMEM lanes)
constexpr int TC_N = 256;        // stranded rows per CTA (TMEM columns per accumulator)
constexpr int TC_KC = 32;        // f32 elements per K chunk (one 128 B swizzle row)
constexpr int TC_MAX_STAGES = 8; // A-chunk pipeline depth: as many 16 KB stages as fit beside B
constexpr int TC_MAXK = 4;       // D <= 128
constexpr int TC_EPI_WARPS = 8;  // two epilogue warps per TMEM lane quarter (128 columns each)
constexpr int TC_THREADS = 64 + 32 * TC_EPI_WARPS;  // warp 0 TMA, warp 1 MMA + TMEM owner, warps 2.. epilogue
constexpr int TC_CAP = 1024;     // candidate slots per stranded row
constexpr float TC_E1 = 0x1p-7f;   // error bound: E1 |r| |x| + E2 (|r|^2 + |x|^2) (see top)
constexpr float TC_E2 = 0x1p-18f;
constexpr float TC_E = 0.5f * TC_E1 + TC_E2;  // <= E (|r|^2 + |x|^2) form of the same bound
constexpr uint32_t TC_A_BYTES = TC_M * 128;   // 16 KB per stage
constexpr uint32_t TC_B_BYTES = TC_N * 128;   // 32 KB per K chunk

__host__ __device__ constexpr size_t tc_smem_bytes(int nk, int stages) {
    return 1024 /* align slack */ + (size_t)nk * TC_B_BYTES + (size_t)stages * TC_A_BYTES + TC_N * 4 + 512;
}
__host__ __device__ constexpr int tc_stages(int nk) {
    int st = TC_MAX_STAGES;
    while (st > 2 && tc_smem_bytes(nk, st) > 227 * 1024) --st;
    return st;
}

// ---- PTX wrappers ------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    return ok != 0;
}
// spin with a short back-off: the waiting warps share SM sub-partitions with the
// epilogue warps, whose issue slots a hot spin loop would take
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    const uint32_t a = smem_u32(b);
    while (!mbar_try(a, parity)) __nanosleep(32);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major operand, 128 B swizzle: 8-row core groups 1024 B apart (SBO), LBO 16 B
// (unused by the swizzled K-major layout), descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
    return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::tf32, f32 accumulate, A and B K-major, M = 128, N = 256
constexpr uint32_t TC_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_N >> 3) << 17) |
                              ((uint32_t)(TC_M >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
        "l"(adesc), "l"(bdesc), "r"(TC_IDESC), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// 32 consecutive f32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// ---- 2. screen ---------------------------------------------------------------
// grid (persistent over data tiles, stranded chunks of TC_N); one CTA per SM.
__global__ void __launch_bounds__(TC_THREADS, 1)
donor_screen_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b, int nk,
                       int64_t n_rows, int64_t tiles, const int32_t* __restrict__ seen, const float* __restrict__ norms,
                       const float4* __restrict__ sinfo, int nlost, int* __restrict__ cnt, int32_t* __restrict__ list,
                       int cap) {
    extern __shared__ __align__(1024) unsigned char tsm_raw[];
    // 1024 B alignment for the 128 B swizzle atoms (pointer arithmetic keeps the shared window)
    unsigned char* tsm = tsm_raw + ((1024u - (smem_u32(tsm_raw) & 1023u)) & 1023u);
    unsigned char* sB = tsm;                                       // nk x [256 rows x 128 B]
    unsigned char* sA = sB + (size_t)nk * TC_B_BYTES;              // STAGES x [128 rows x 128 B]
    const int STAGES = tc_stages(nk);
    float* sC = reinterpret_cast<float*>(sA + (size_t)STAGES * TC_A_BYTES);  // [256] c_x per column
    uint64_t* bars = reinterpret_cast<uint64_t*>(sC + TC_N);
    uint64_t* full = bars;                    // [STAGES]
    uint64_t* empty = bars + STAGES;          // [STAGES]
    uint64_t* bfull = bars + 2 * STAGES;      // [1]
    uint64_t* tfull = bfull + 1;              // [2]
    uint64_t* tempty = tfull + 2;             // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int s_base = blockIdx.y * TC_N;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < STAGES; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
        mbar_init(bfull, 1);
        for (int i = 0; i < 2; ++i) { mbar_init(tfull + i, 1); mbar_init(tempty + i, TC_EPI_WARPS); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    }
    if (warp == 1) {  // the whole warp allocates all 512 TMEM columns (2 accumulators of 256)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // per stranded column: c_x = (tau_x - |x|^2 (1 - E)) / 2; -inf: no column (a row
    // without a finite tau is rescanned exactly anyway)
    for (int i = threadIdx.x; i < TC_N; i += TC_THREADS) {
        const int s = s_base + i;
        float c = -__int_as_float(0x7F800000);
        if (s < nlost) {
            const float4 si = sinfo[s];
            if (si.z < __int_as_float(0x7F800000)) c = 0.5f * (si.z - si.x * (1.0f - TC_E));
        }
        sC[i] = c;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // TMA producer
            mbar_expect_tx(bfull, (uint32_t)nk * TC_B_BYTES);
            for (int kc = 0; kc < nk; ++kc) tma_load_2d(sB + (size_t)kc * TC_B_BYTES, &map_b, kc * TC_KC, s_base, bfull);
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
                for (int kc = 0; kc < nk; ++kc) {
                    mbar_wait(empty + stage, phase ^ 1);
                    mbar_expect_tx(full + stage, TC_A_BYTES);
                    tma_load_2d(sA + (size_t)stage * TC_A_BYTES, &map_a, kc * TC_KC, (int)(t * TC_M), full + stage);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // MMA issuer
            mbar_wait(bfull, 0);
            int stage = 0, acc = 0;
            uint32_t phase = 0, aphase = 0;
            const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
            for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
                mbar_wait(tempty + acc, aphase ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * TC_N);
                for (int kc = 0; kc < nk; ++kc) {
                    mbar_wait(full + stage, phase);
                    tc_fence_after();
#pragma unroll
                    for (int k = 0; k < TC_KC / 8; ++k) {  // UMMA_K = 8 tf32 = 32 B along the swizzled row
                        const uint64_t ad = sw128_desc(a0 + stage * TC_A_BYTES + 32 * k);
                        const uint64_t bd = sw128_desc(b0 + kc * TC_B_BYTES + 32 * k);
                        mma_tf32(d, ad, bd, (kc | k) != 0);
                    }
                    mma_commit(empty + stage);  // frees the A stage once these MMAs have read it
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                mma_commit(tfull + acc);  // accumulator ready for the epilogue
                acc ^= 1;
                if (acc == 0) aphase ^= 1;
            }
        }
        __syncwarp();
    } else {
        // epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 = data rows of the tile, and
        // one half of the 256 stranded columns. With err <= E (|r|^2 + |x|^2),
        // E = E1 / 2 + E2 (E1 |r||x| <= E1 (|r|^2 + |x|^2) / 2), keep (r, x) iff
        //   <r, x>  >=  h_r - c_x,   h_r = |r|^2 (1 - E) / 2,   c_x = (tau_x - |x|^2 (1 - E)) / 2
        // (the rearrangement's roundings are inside E2 = 2^-18, 4x the bound's own term).
        const int q = warp & 3;
        const int half = (warp - 2) >> 2;
        const int col0 = half * (TC_N / 2);
        const int ncol = min(TC_N / 2, max(0, nlost - s_base - col0));  // valid stranded columns of this half
        int acc = 0;
        uint32_t aphase = 0;
        for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
            const int64_t r = t * TC_M + 32 * q + lane;
            float h = __int_as_float(0x7F800000);  // unreachable / past the end: never a candidate
            if (r < n_rows && seen[r] != 0) h = __ldg(norms + r) * (0.5f - 0.5f * TC_E);
            const bool any_row = __any_sync(0xFFFFFFFFu, h < __int_as_float(0x7F800000));
            mbar_wait(tfull + acc, aphase);
            tc_fence_after();
            const uint32_t base = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(acc * TC_N + col0);
            if (any_row) {
#pragma unroll 1
                for (int c0 = 0; c0 < ncol; c0 += 32) {
                    float v[32];
                    tmem_ld32(base + c0, v);
                    const float4* cv = reinterpret_cast<const float4*>(sC + col0 + c0);
                    bool hit = false;
#pragma unroll
                    for (int j4 = 0; j4 < 8; ++j4) {
                        const float4 c = cv[j4];
                        hit |= v[4 * j4] >= h - c.x;
                        hit |= v[4 * j4 + 1] >= h - c.y;
                        hit |= v[4 * j4 + 2] >= h - c.z;
                        hit |= v[4 * j4 + 3] >= h - c.w;
                    }
                    if (hit) {  // rare: append this group's candidates
                        for (int j = 0; j < 32; ++j) {
                            if (v[j] >= h - sC[col0 + c0 + j]) {
                                const int s = s_base + col0 + c0 + j;
                                const int slot = atomicAdd(cnt + s, 1);
                                if (slot < cap) list[(size_t)s * cap + slot] = (int32_t)r;
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty + acc);
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---- 1. seed: tau_x from the two-hop neighbourhood -------------------------------
// Sorted top-`fan` keys one per lane; insert the lanes' candidates, skipping keys
// already present (a vertex reached along two paths).
__device__ __forceinline__ void topk_insert_distinct(uint64_t& t, uint64_t c, int fan) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = lane_id();
    for (uint32_t mm = __ballot_sync(FULL, c != UMAX); mm; mm &= mm - 1) {
        const uint64_t k = shfl_u64(c, __ffs(mm) - 1);
        const uint64_t worst = shfl_u64(t, fan - 1);
        if (k >= worst) continue;
        if (__ballot_sync(FULL, lane < fan && t == k)) continue;
        const int pos = __popc(__ballot_sync(FULL, lane < fan && t < k));
        const uint64_t up = __shfl_up_sync(FULL, t, 1);
        if (lane < fan) {
            if (lane > pos) t = up;
            else if (lane == pos) t = k;
        }
    }
}

// the reference's key of reachable r for stranded x: (d(x, r), r), r in the data role
__device__ __forceinline__ uint64_t donor_key(const float* __restrict__ data, const float* __restrict__ norms, int D,
                                              uint32_t r, uint32_t x) {
    const float dot = a1_dot<false>(data + (size_t)r * D, data + (size_t)x * D, D);
    return pack_key(exact_from_dot(__ldg(norms + r), dot, __ldg(norms + x)), r);
}

__global__ void donor_seed_kernel(const float* __restrict__ data, const float* __restrict__ norms, int D,
                                  const int32_t* __restrict__ adj, int R, const int32_t* __restrict__ seen,
                                  int64_t n_rows, const int32_t* __restrict__ lost, int nlost, int fan,
                                  float4* __restrict__ sinfo) {
    const int w = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (w >= nlost) return;
    const uint32_t x = (uint32_t)lost[w];
    uint64_t t = UMAX;
    const int32_t* row = adj + (size_t)x * R;
    for (int j = 0; j < R; ++j) {
        const int32_t u = __ldg(row + j);
        if (u < 0) continue;
        // u itself (slot R) and u's out-neighbours
        for (int c0 = 0; c0 <= R; c0 += 32) {
            const int c = c0 + lane;
            int32_t v = -1;
            if (c < R) v = __ldg(adj + (size_t)u * R + c);
            else if (c == R) v = u;
            uint64_t k = UMAX;
            if (v >= 0 && v < n_rows && (uint32_t)v != x && seen[v]) k = donor_key(data, norms, D, (uint32_t)v, x);
            topk_insert_distinct(t, k, fan);
        }
    }
    const uint64_t last = shfl_u64(t, fan - 1);
    if (lane == 0) {
        const float xn = __ldg(norms + x);
        const float tau = last == UMAX ? __int_as_float(0x7F800000) : key_dist(last);
        sinfo[w] = make_float4(xn, sqrtf(xn) * (1.0f + 0x1p-10f), tau, 0.0f);
    }
}

// ---- 3. exact keys of the candidates, top `fan` -----------------------------------
// part[w * fan + j] (one slice); rows whose list overflowed or had no finite tau
// are flagged in redo[] for the exact CUDA-core scan.
// Row w (of this pass's list; part row remap[w], or w): rows whose list overflowed
// or that had no finite tau go to redo[] (as part rows). An overflowed row's first
// `cap` candidates are distinct reachable vertices, so the fan-th smallest of their
// exact distances is a valid (and usually much tighter) tau for a second screen
// pass: written to tau2[w] (+inf when unusable).
__global__ void donor_exact_kernel(const float* __restrict__ data, const float* __restrict__ norms, int D,
                                   const int32_t* __restrict__ lost, int nlost, const float4* __restrict__ sinfo,
                                   const int* __restrict__ cnt, const int32_t* __restrict__ list, int cap, int fan,
                                   const int32_t* __restrict__ remap, uint64_t* __restrict__ part,
                                   int32_t* __restrict__ redo, int* __restrict__ nredo, float* __restrict__ tau2) {
    const int w = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (w >= nlost) return;
    const int pr = remap ? remap[w] : w;
    const int n = cnt[w];
    const bool finite = sinfo[w].z < __int_as_float(0x7F800000);
    const uint32_t x = (uint32_t)lost[w];
    uint64_t t = UMAX;
    if (finite) {
        for (int i0 = 0; i0 < min(n, cap); i0 += 32) {
            const int i = i0 + lane;
            uint64_t k = UMAX;
            if (i < min(n, cap)) k = donor_key(data, norms, D, (uint32_t)list[(size_t)w * cap + i], x);
            topk_insert_distinct(t, k, fan);
        }
    }
    if (!finite || n > cap) {
        const uint64_t last = shfl_u64(t, fan - 1);
        if (lane == 0) {
            redo[atomicAdd(nredo, 1)] = pr;
            if (tau2) tau2[w] = (finite && last != UMAX) ? key_dist(last) : __int_as_float(0x7F800000);
        }
        return;
    }
    if (lane < fan) part[(size_t)pr * fan + lane] = t;
}

// second pass inputs for the redo rows: ids, and sinfo with the refined tau
__global__ void donor_pass2_kernel(const int32_t* __restrict__ lost, const float4* __restrict__ sinfo,
                                   const int32_t* __restrict__ redo, int n2, const float* __restrict__ tau2,
                                   int32_t* __restrict__ lost2, float4* __restrict__ sinfo2) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n2) return;
    const int w = redo[i];  // part row == pass-1 row
    lost2[i] = lost[w];
    float4 si = sinfo[w];
    si.z = tau2[w];
    sinfo2[i] = si;
}

// Rows rescanned by the exact kernel: top `fan` over its `slices` partial lists
// -> part row redo[i] (keys are distinct: every r lives in one slice).
__global__ void donor_redo_merge_kernel(const uint64_t* __restrict__ part2, int slices, int n2, int fan,
                                        const int32_t* __restrict__ redo, uint64_t* __restrict__ part) {
    const int i = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= n2) return;
    uint64_t t = UMAX;
    for (int j0 = 0; j0 < slices * fan; j0 += 32) {
        const int j = j0 + lane;
        const uint64_t k = j < slices * fan ? part2[((size_t)(j / fan) * n2 + i) * fan + j % fan] : UMAX;
        topk_insert_distinct(t, k, fan);
    }
    if (lane < fan) part[(size_t)redo[i] * fan + lane] = t;
}

__global__ void donor_redo_ids_kernel(const int32_t* __restrict__ lost, const int32_t* __restrict__ redo, int n2,
                                      int32_t* __restrict__ lost2) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n2) lost2[i] = lost[redo[i]];
}

int donor_redo_ids(const int32_t* lost, const int32_t* redo, int n2, int32_t* lost2, cudaStream_t st) {
    donor_redo_ids_kernel<<<(n2 + 255) / 256, 256, 0, st>>>(lost, redo, n2, lost2);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

int donor_redo_merge(const uint64_t* part2, int slices, int n2, int fan, const int32_t* redo, uint64_t* part,
                     cudaStream_t st) {
    donor_redo_merge_kernel<<<(unsigned)(((int64_t)n2 * 32 + 255) / 256), 256, 0, st>>>(part2, slices, n2, fan, redo,
                                                                                      part);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

// ---- host ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// [rows, D] f32 row-major, box {32, box_rows}, 128 B swizzle, OOB zero fill
static bool make_map(CUtensorMap* m, const float* base, int D, int64_t rows, int box_rows) {
    auto enc = encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)D * 4};
    cuuint32_t box[2] = {(cuuint32_t)TC_KC, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool donor_tc_supported(int D, int64_t n_rows) {
    const char* e = std::getenv("JB_DONOR_TC");
    if (e && e[0] == '0') return false;
    return D % 4 == 0 && D <= TC_KC * TC_MAXK && n_rows < (1ll << 31) && encode_fn() != nullptr;
}

// dst[i] = row lost[i] of data (f32, D elements)
__global__ void gather_f32_rows_kernel(const float* __restrict__ data, int D, const int32_t* __restrict__ ids, int n,
                                       float* __restrict__ dst) {
    const int64_t total = (int64_t)n * D;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = data[(int64_t)ids[i / D] * D + i % D];
}

// One screen pass over `n` stranded rows (ids ls, seeds si) -> exact top lists in
// part rows (remap), uncertified rows appended to redo (+ refined tau in tau2).
static int screen_pass(const float* data, const float* norms, int D, const int32_t* seen, int64_t n_rows,
                       const int32_t* ls, const float4* si, int n, int fan, const int32_t* remap, uint64_t* part,
                       int32_t* redo, int* nredo, float* tau2, cudaStream_t st) {
    const int cap = TC_CAP;
    const int sp = (n + TC_N - 1) / TC_N * TC_N;
    Scratch s_rows, s_cnt, s_list;
    JB_CUDA(s_rows.alloc((size_t)sp * D * 4, st));
    JB_CUDA(s_cnt.alloc((size_t)n * sizeof(int), st));
    JB_CUDA(s_list.alloc((size_t)n * cap * sizeof(int32_t), st));
    float* srows = s_rows.as<float>();
    int* cnt = s_cnt.as<int>();
    int32_t* list = s_list.as<int32_t>();
    JB_CUDA(cudaMemsetAsync(cnt, 0, (size_t)n * sizeof(int), st));
    JB_CUDA(cudaMemsetAsync(srows, 0, (size_t)sp * D * 4, st));
    gather_f32_rows_kernel<<<(unsigned)std::min<int64_t>(((int64_t)n * D + 255) / 256, 4096), 256, 0, st>>>(
        data, D, ls, n, srows);
    JB_LAUNCH_CHECK();
    CUtensorMap ma, mb;
    JB_CHECK_ARG(make_map(&ma, data, D, n_rows, TC_M) && make_map(&mb, srows, D, sp, TC_N),
                 "donor scan: cuTensorMapEncodeTiled failed");
    const int nk = (D + TC_KC - 1) / TC_KC;
    const size_t smem = tc_smem_bytes(nk, tc_stages(nk));
    JB_CUDA_RC(grow_smem(donor_screen_tc_kernel, (int)smem));
    const int64_t tiles = (n_rows + TC_M - 1) / TC_M;
    const int chunks = sp / TC_N;
    const int gx = (int)std::min<int64_t>(tiles, std::max(1, sm_count_current() / chunks));
    donor_screen_tc_kernel<<<dim3(gx, chunks), TC_THREADS, smem, st>>>(ma, mb, nk, n_rows, tiles, seen, norms, si, n,
                                                                       cnt, list, cap);
    JB_LAUNCH_CHECK();
    donor_exact_kernel<<<(unsigned)(((int64_t)n * 32 + 255) / 256), 256, 0, st>>>(
        data, norms, D, ls, n, si, cnt, list, cap, fan, remap, part, redo, nredo, tau2);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

int donor_scan_tc(const float* data, const float* norms, int D, const int32_t* adj, int R, const int32_t* seen,
                  int64_t n_rows, const int32_t* lost, int nlost, int fan, uint64_t* part, int32_t* redo, int* nredo,
                  cudaStream_t st) {
    Scratch s_info, s_tau2, s_redo1, s_n1;
    JB_CUDA(s_info.alloc((size_t)nlost * sizeof(float4), st));
    JB_CUDA(s_tau2.alloc((size_t)nlost * sizeof(float), st));
    JB_CUDA(s_redo1.alloc((size_t)nlost * sizeof(int32_t), st));
    JB_CUDA(s_n1.alloc(sizeof(int), st));
    float4* sinfo = s_info.as<float4>();
    int32_t* redo1 = s_redo1.as<int32_t>();
    int* n1 = s_n1.as<int>();
    JB_CUDA(cudaMemsetAsync(n1, 0, sizeof(int), st));
    JB_CUDA(cudaMemsetAsync(nredo, 0, sizeof(int), st));
    donor_seed_kernel<<<(unsigned)(((int64_t)nlost * 32 + 255) / 256), 256, 0, st>>>(data, norms, D, adj, R, seen, n_rows,
                                                                                   lost, nlost, fan, sinfo);
    JB_LAUNCH_CHECK();
    // pass 1: two-hop seeds
    JB_CUDA_RC(screen_pass(data, norms, D, seen, n_rows, lost, sinfo, nlost, fan, nullptr, part, redo1, n1,
                           s_tau2.as<float>(), st));
    int h1 = 0;
    JB_CUDA(cudaMemcpyAsync(&h1, n1, sizeof(int), cudaMemcpyDeviceToHost, st));
    JB_CUDA(cudaStreamSynchronize(st));
    if (h1 == 0) return JB_OK;
    // pass 2: the uncertified rows again with tau refined from their pass-1 candidates;
    // what still fails (no finite tau, or a second overflow) is left to the exact scan
    Scratch s_l2, s_i2;
    JB_CUDA(s_l2.alloc((size_t)h1 * sizeof(int32_t), st));
    JB_CUDA(s_i2.alloc((size_t)h1 * sizeof(float4), st));
    donor_pass2_kernel<<<(h1 + 255) / 256, 256, 0, st>>>(lost, sinfo, redo1, h1, s_tau2.as<float>(), s_l2.as<int32_t>(),
                                                         s_i2.as<float4>());
    JB_LAUNCH_CHECK();
    return screen_pass(data, norms, D, seen, n_rows, s_l2.as<int32_t>(), s_i2.as<float4>(), h1, fan, redo1, part, redo,
                       nredo, nullptr, st);
}

}  // namespace jb
