// search.cu — batched greedy beam search (Vamana GreedySearch) on sm_100a.
//
// Replaces the reference's lockstep numpy engine, `_run_lockstep`
// (search.py:171-269) driven by `run_beam_searches` (search.py:272-304), and
// the rerank/top-k tail of `search_knn_batch` (search.py:351-383).
//
// Design (one warp per query, persistent grid, everything per query in smem):
//  * beam: L u64 keys kept sorted ascending; key = (f32 dist bits << 32) | id,
//    exactly the reference's key (search.py:139-145). Bit 31 of the id word is
//    the device-only "expanded" flag, so a key carries its visited state when
//    the beam is shifted by a merge.
//  * visited ("seen") set: a 4-way set-associative id table in smem (one 16 B
//    probe). It never yields a false positive. When a bucket is full an id is
//    evicted and may later be re-evaluated; its key is then either already in
//    the beam (dropped by the equal-key dedupe, the incumbent keeps its flag) or
//    worse than the full beam's last key (dropped by the filter), because the
//    beam is always the top-L of every key evaluated so far. Frontier and trace
//    are therefore identical to the reference's exact `seen` matrix; only
//    `evals` can count re-evaluations, and flags[q] bit0 reports evictions.
//  * expansion: the first unexpanded key in ascending order (search.py:202-210).
//    Neighbours are checked 32 per step (one per lane); each new neighbour's
//    distance is computed by its lane in the reference's exact f32 rounding
//    order (A1) and merged into the beam by rank (one binary search per
//    surviving key, a ballot loop for ranks among survivors), shifting beam
//    entries right in 32-wide chunks from the top. Candidates worse than a full
//    beam's last key are dropped before any of that.
//  * exact rows are staged into smem with coalesced cp.async (one 512 B row per
//    warp instruction at D=128) and then read per lane (16 B skew per row keeps
//    the per-lane float4 reads bank-conflict free). RaBitQ records are read
//    directly, one 32 B record per lane (two 128-bit loads).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include "common.cuh"
#include "metric.cuh"
#include "runtime.cuh"

namespace jb {

#ifndef JB_WPB
#define JB_WPB 4
#endif
constexpr int WPB = JB_WPB;     // warps per block
#ifndef JB_RR_WARPS
#define JB_RR_WARPS 4
#endif
#ifndef JB_RR_ROWS
#define JB_RR_ROWS 8
#endif
constexpr int RR_WARPS = JB_RR_WARPS;  // warps per block of the rerank kernel
constexpr int RR_ROWS = JB_RR_ROWS;    // frontier rows staged per step (4 lanes each, RR_ROWS <= 8)
constexpr int MAX_CHUNKS = 4;   // neighbour slots per hop: R <= 32 * MAX_CHUNKS
#ifndef JB_EXACT_CHUNK
#define JB_EXACT_CHUNK 128      // exact source: row elements staged per pass (multiple of 32)
#endif
#ifndef JB_LDG256_R1
#define JB_LDG256_R1 1  // 32 B records of the float estimator (m = 1) in one 256-bit load
#endif
#ifndef JB_LDG256_R64
#define JB_LDG256_R64 1  // 64 B multi-bit records in two 256-bit loads, estimated from registers
#endif
#ifndef JB_COOP_MAX
#define JB_COOP_MAX 2
#endif
constexpr int COOP_MAX = JB_COOP_MAX;  // merge: warp-cooperative placement up to this many candidates

struct SearchLayout {
    int q_off, beam_off, hash_off, newk_off, cid_off, bar_off, stage_off, plane_off, rec_off, bytes;
    int rec_stride;  // SREC: staged record stride (bytes, = 16 mod 128: conflict-free 16 B lane reads)
    int chunk;      // staged elements per row chunk (multiple of 32, <= 128)
    int sstride;    // staged row stride in floats (chunk + 4)
    int hbits;      // log2(number of 4-way buckets)
    int scr_off;    // EXACT: int8 code of the centred query (screen), 16 B aligned
    int srows;      // EXACT: rows staged per pass (32; 16 with the screen: fewer survivors, more warps)
    int srb;        // screen record bytes
    int spf;        // 1: prefetch the speculative next hop's screen records into L2
    int snext;      // 1: stage the speculative next hop's screen records into smem (nrec_off)
    int nrec_off;   // snext: 32 records + their mbarrier (16 B)
};

static int pow2_ceil(int v) { int p = 1; while (p < v) p <<= 1; return p; }
__host__ __device__ constexpr int log2i(int v) { int l = 0; while ((1 << l) < v) ++l; return l; }

// Per-warp smem layout. The fixed-size pieces come first and the beam (L keys)
// last, so for a compile-time D and visited-table size every offset is a
// constant (the specialised kernels then address smem as base + immediate).
__host__ __device__ constexpr SearchLayout make_layout(int src, int D, int L, int hash_slots, int qb,
                                                      bool direct = false, int rec_bytes = 0, int srows = 32) {
    SearchLayout s{};
    int off = 0;
    s.q_off = off; off += ((D * 4) + 15) & ~15;
    s.scr_off = off;
    if (src == JB_SRC_EXACT) off += (D + 15) & ~15;
    s.hbits = log2i(hash_slots / 4 > 1 ? hash_slots / 4 : 1);   // 4-way buckets
    s.hash_off = off; off += (4 << s.hbits) * 4;
    s.newk_off = off; off += 32 * 4;
    s.cid_off = off; off += 32 * 4;
    s.bar_off = off; off += 16;   // per-warp mbarrier of the bulk row staging
    s.chunk = ((D + 31) / 32) * 32 < JB_EXACT_CHUNK ? ((D + 31) / 32) * 32 : JB_EXACT_CHUNK;
    s.sstride = s.chunk + 4;
    s.stage_off = off;
    s.srows = srows;
    s.srb = ((D + 15) & ~15) + 16;
    s.spf = 0;
    if (src == JB_SRC_EXACT && !direct) off += srows * s.sstride * 4;
    s.plane_off = off;
    if (src == JB_SRC_RABITQ_FAST) off += qb * ((((D + 31) / 32) + 3) & ~3) * 4;
    off = (off + 15) & ~15;
    s.rec_off = off;
    s.rec_stride = 0;
    if (rec_bytes > 0) {  // staged records, one slot per lane
        s.rec_stride = ((rec_bytes - 16 + 127) / 128) * 128 + 16;
        off += 32 * s.rec_stride;
    }
    s.snext = 0;
    s.nrec_off = off;  // (sized by with_snext)
    s.beam_off = off; off += ((L * 8) + 15) & ~15;
    s.bytes = (off + 15) & ~15;
    return s;
}


// Visited table: 4-way set-associative buckets of ids in smem, one 16 B load per
// probe. A miss inserts into the first empty way, else evicts a pseudo-random way.
// No atomics: the lanes of one warp probe and insert concurrently, so two lanes
// whose ids hash to one bucket may read it while the other writes (RAW) and may
// both claim the same empty way (WAW). These races are intended and harmless:
//  * the bucket load and the slot store are volatile (PTX relaxed, morally
//    strong) 32-bit accesses, so a racing read returns the old or the new word
//    and a racing write leaves exactly one of the written ids — never a torn or
//    invented value;
//  * every id written in a hop is an id evaluated in that hop (a lane writes only
//    after deciding its own id is new), so whichever write survives, the table
//    never reports an unevaluated id as seen (no false positive);
//  * an id whose write lost (or was evicted later) is only forgotten: if it comes
//    back it is re-evaluated to the same key, which the merge drops (equal-key
//    dedupe, or the full beam's worst-key filter), so frontier and trace stay
//    exact; the loser notices (re-read after __syncwarp) and flags `lossy`;
//  * a racing reader's own id differs from the writers' ids (an adjacency row
//    holds distinct ids), so what it reads only affects which way it picks.
// compute-sanitizer racecheck reports exactly these two accesses.
__device__ __forceinline__ bool visit(uint32_t* tab, int hbits, uint32_t id, int& lossy, uint32_t*& slot) {
    const uint32_t h = id * 0x9E3779B1u;
    const uint32_t b = h >> (32 - hbits);
    uint4* bucket = reinterpret_cast<uint4*>(tab) + b;
    uint4 v;
    asm volatile("ld.volatile.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"((uint32_t)__cvta_generic_to_shared(bucket)));
    slot = nullptr;
    if (v.x == id || v.y == id || v.z == id || v.w == id) return false;
    int way;
    if (v.x == EMPTY_SLOT) way = 0;
    else if (v.y == EMPTY_SLOT) way = 1;
    else if (v.z == EMPTY_SLOT) way = 2;
    else if (v.w == EMPTY_SLOT) way = 3;
    else { way = (h >> 3) & 3; lossy = 1; }
    slot = reinterpret_cast<uint32_t*>(bucket) + way;
    asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(slot)), "r"(id)
                 : "memory");
    return true;
}

// Popcount estimator (fast mode, m = 1): the rotated query is quantized per query
// to QB-bit integers qq = round((q - lo) / delta) and stored as QB bit-planes
// (built with warp ballots, element e <-> bit e % 32 of word e / 32, the same
// layout as the packed 1-bit codes), so
//   <u, q> ~= lo * popc(u) + delta * sum_b 2^b popc(u & plane_b)
// replaces the 128 ordered float adds with 4 * (QB + 1) popcounts at D = 128.
#ifndef JB_FAST_QB
#define JB_FAST_QB 6
#endif
#ifndef JB_FAST_MINB
#define JB_FAST_MINB 10  // blocks/SM of the popcount kernel: 12 is 3% faster alone but slows the
                        // two-lane step (the other lane's bind / rerank lose their SM share)
#endif
#ifndef JB_RQ_MINB
#define JB_RQ_MINB 8  // blocks/SM of the bit-exact RaBitQ kernel
#endif
#ifndef JB_OTHER_MINB
#define JB_OTHER_MINB 8  // blocks/SM of the exact-row kernels (smem-bound: staged rows)
#endif
constexpr int FAST_QB = JB_FAST_QB;   // query bit-planes of the popcount estimator

// planes: FAST_QB planes of `pw` words each (pw = nwords rounded up to 4, zero padded)
// PW > 0: plane stride known at compile time (PW = 4 covers D <= 128 in one piece).
// m-bit codes (MB > 1) are read as MB code bit-planes of `pw` words (plane records,
// jb_rabitq_pack_planes): u = sum_b' 2^b' c_b', so
//   <u, q> ~= lo * sum_b' 2^b' popc(c_b') + delta * sum_b' sum_b 2^(b'+b) popc(c_b' & plane_b).
// For MB = 1 the plane record is the packed record itself.
template <int QB, int PW = 0, int MB = 1, bool GL = true>
__device__ __forceinline__ float rabitq_dd_fast(const uint8_t* __restrict__ rec, uint4 first,
                                               const uint32_t* __restrict__ planes, int pw_rt, float lo, float delta) {
    const int pw = PW > 0 ? PW : pw_rt;
    int pc = 0;
    int acc[QB];
#pragma unroll
    for (int b = 0; b < QB; ++b) acc[b] = 0;
    int s = 0;
    // runtime stride (long records, e.g. 4 planes x 128 B at D = 960): the next word
    // group's MB plane loads are issued before this group's popcounts
    uint4 cur[MB];
#pragma unroll
    for (int bp = 0; bp < MB; ++bp)
        cur[bp] = bp == 0 ? first : ld16<GL>(rec + 4 * (bp * pw));
#pragma unroll
    for (int w0 = 0; w0 < pw; w0 += 4) {
        uint4 nxt[MB];
#pragma unroll
        for (int bp = 0; bp < MB; ++bp)
            nxt[bp] = (w0 + 4 < pw) ? ld16<GL>(rec + 4 * (bp * pw + w0 + 4)) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int bp = 0; bp < MB; ++bp) {
            const uint4 c = cur[bp];
            pc += (__popc(c.x) + __popc(c.y) + __popc(c.z) + __popc(c.w)) << bp;
#pragma unroll
            for (int b = 0; b < QB; ++b) {
                const uint4 p = *reinterpret_cast<const uint4*>(planes + b * pw + w0);
                const int t = __popc(c.x & p.x) + __popc(c.y & p.y) + __popc(c.z & p.z) + __popc(c.w & p.w);
                if (MB == 1) acc[b] += t;
                else s += t << (b + bp);
            }
        }
#pragma unroll
        for (int bp = 0; bp < MB; ++bp) cur[bp] = nxt[bp];
    }
    if (MB == 1) {
#pragma unroll
        for (int b = 0; b < QB; ++b) s += acc[b] << b;
    }
    return fmaf(delta, (float)s, lo * (float)pc);
}

template <int QB, int MB = 1>
__device__ __forceinline__ float rabitq_estimate_fast(const uint8_t* __restrict__ rec, const uint32_t* __restrict__ planes,
                                                      int nwords, int meta_off, float lo, float delta, float qadd,
                                                      float qsumq) {
    const uint4 first = __ldg(reinterpret_cast<const uint4*>(rec));
    const float dd = rabitq_dd_fast<QB, 0, MB>(rec, first, planes, nwords, lo, delta);
    const float2 m = __ldg(reinterpret_cast<const float2*>(rec + meta_off));
    const float est = (qadd + m.x) + m.y * (dd - qsumq);
    return est > 0.0f ? est : 0.0f;
}

// Build the query bit-planes in smem (one warp): lo/delta from a warp min/max.
template <int QB>
__device__ __forceinline__ void build_planes(const float* qv, int D, uint32_t* planes, float& lo, float& delta) {
    const int lane = lane_id();
    float mn = 3.4e38f, mx = -3.4e38f;
    for (int e = lane; e < D; e += 32) { mn = fminf(mn, qv[e]); mx = fmaxf(mx, qv[e]); }
    for (int o = 16; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xFFFFFFFFu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    }
    lo = mn;
    const float levels = (float)((1 << QB) - 1);
    delta = (mx > mn) ? (mx - mn) / levels : 1.0f;
    const int pw = (((D + 31) / 32) + 3) & ~3;
    for (int w = 0; w < pw; ++w) {
        const int e = w * 32 + lane;
        uint32_t qq = 0;
        if (e < D) qq = (uint32_t)min((int)levels, max(0, __float2int_rn((qv[e] - lo) / delta)));
#pragma unroll
        for (int b = 0; b < QB; ++b) {
            const uint32_t bits = __ballot_sync(0xFFFFFFFFu, (qq >> b) & 1u);
            if (lane == 0) planes[b * pw + w] = bits;
        }
    }
    __syncwarp();
}

// First index >= s (< n) whose key is not expanded; n if none.
__device__ __forceinline__ int first_unexpanded(const uint64_t* beam, int s, int n) {
    const int lane = lane_id();
    for (int b = s; b < n; b += 32) {
        int i = b + lane;
        bool un = (i < n) && !(beam[i] & EXPANDED);
        uint32_t m = __ballot_sync(0xFFFFFFFFu, un);
        if (m) return b + __ffs(m) - 1;
    }
    return n;
}

// Merge up to 32 candidate keys (one per lane, UMAX = none) into the sorted beam
// (search.py:232-237: stable sort of beam + candidates, first L kept). Keys are
// distinct except a re-evaluated id equal to a beam key (dropped: the incumbent
// keeps its expanded flag). No sort: each surviving key's final position is
//   fs = lower_bound(beam, key) + #survivors below it,
// distinct across survivors, recorded as bits of a per-warp position mask. Beam
// entries are then gathered top-down, one 32-entry chunk per step: output j
// (not a survivor slot) takes old entry j - #survivor slots below j, a popcount
// of the mask. Returns the smallest insertion position (bcount if none).
#ifdef JB_MERGE_STATS
// dev builds only (-DJB_MERGE_STATS): [0..32] histogram of candidates per merge
// after the beam-worst filter, [33..65] of evaluated candidates per merge.
__device__ unsigned long long g_merge_stats[66];
#endif

__device__ __forceinline__ int merge_into_beam(uint64_t* beam, int& bcount, int L, uint64_t key,
                                               uint32_t* fmask) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = lane_id();
#ifdef JB_MERGE_STATS
    const int nin = __popc(__ballot_sync(FULL, key != UMAX));
#endif
    if (key != UMAX && bcount == L && key >= key_mask(beam[L - 1])) key = UMAX;
    const uint32_t cm = __ballot_sync(FULL, key != UMAX);
#ifdef JB_MERGE_STATS
    if (lane == 0) {
        atomicAdd(&g_merge_stats[__popc(cm)], 1ull);
        atomicAdd(&g_merge_stats[33 + nin], 1ull);
    }
#endif
    if (cm == 0) return bcount;  // most hops: nothing beats the full beam
    int p = 0, rank = 0;
    uint32_t sm;
    if (__popc(cm) <= COOP_MAX) {
        // Few candidates (the common case): the whole warp locates each one in
        // turn. Lane g holds the last key of beam group g (G = ceil(bcount/32)
        // entries per group): popc(ballot(split < k)) counts the groups wholly
        // below k, then lanes j < G compare k with that group's entries. Ranks
        // among survivors and the equal-key dedupe come out of the same loop.
        const int G = (bcount + 31) >> 5;
        const int si = G * lane + G - 1;
        const uint64_t split = si < bcount ? key_mask(beam[si]) : UMAX;
        bool dup_mine = false;
        for (uint32_t mm = cm; mm; mm &= mm - 1) {
            const int t = __ffs(mm) - 1;
            const uint64_t kt = shfl_u64(key, t);
            const int g0 = G * __popc(__ballot_sync(FULL, split < kt));
            const int e = g0 + lane;
            const uint64_t ev = (lane < G && e < bcount) ? key_mask(beam[e]) : UMAX;
            const int pt = g0 + __popc(__ballot_sync(FULL, ev < kt));
            const bool dup = __ballot_sync(FULL, ev == kt) != 0;
            if (!dup && kt < key) ++rank;
            if (lane == t) { p = pt; dup_mine = dup; }
        }
        if (dup_mine) key = UMAX;
        sm = __ballot_sync(FULL, key != UMAX);
        if (sm == 0) return bcount;
        if (key == UMAX) rank = 0;
    } else {
        if (key != UMAX) {
            p = lower_bound_masked(beam, bcount, key);
            if (p < bcount && key_mask(beam[p]) == key) key = UMAX;
        }
        sm = __ballot_sync(FULL, key != UMAX);
        if (sm == 0) return bcount;
        for (uint32_t mm = sm; mm; mm &= mm - 1) {
            const int t = __ffs(mm) - 1;
            rank += (shfl_u64(key, t) < key) ? 1 : 0;
        }
    }
    const int m2 = __popc(sm);
    const int fs = p + rank;
    const bool live = key != UMAX && fs < L;
    if (live) atomicOr(&fmask[fs >> 5], 1u << (fs & 31));
    const uint32_t lm = __ballot_sync(FULL, live);
    const int mlive = __popc(lm);
    // the rank-0 survivor lands exactly at its lower bound, the smallest position
    const int p0 = __shfl_sync(FULL, fs, __ffs(__ballot_sync(FULL, key != UMAX && rank == 0)) - 1);
    const int nb = min(L, bcount + m2);
    __syncwarp();
    int above = 0;  // live survivor slots in chunks above the current one
    const uint32_t lt = lanemask_lt();
    for (int ob = ((nb - 1) >> 5) << 5; ob >= (p0 & ~31); ob -= 32) {
        const uint32_t w = fmask[ob >> 5];
        const int j = ob + lane;
        const int pw = __popc(w);
        const bool mv = j >= p0 && j < nb && !((w >> lane) & 1u);
        uint64_t v = 0;
        if (mv) v = beam[j - (mlive - above - pw + __popc(w & lt))];
        __syncwarp();
        if (mv) beam[j] = v;
        above += pw;
    }
    __syncwarp();
    if (live) beam[fs] = key;
    if (lane >= (p0 >> 5) && lane <= ((nb - 1) >> 5)) fmask[lane] = 0;
    __syncwarp();
    bcount = nb;
    return p0;
}

// Per-query state shared by the two search kernels (pointers into the warp's smem).
struct QueryCtx {
    const float* qv;          // query (EXACT) or rotated query (RaBitQ), D f32
    const uint32_t* planes;   // popcount query bit-planes
    int32_t* cid;             // EXACT: compacted new ids, 32
    float* stage;             // EXACT: staged rows, 32 x sstride
    float qadd, qsumq, qlo, qdelta;
    int nwords, meta_off;
    uint32_t qn;              // EXACT_U8: integer query norm (query bytes at qv)
    uint64_t* bar;            // EXACT / SREC: bulk-staging mbarrier
    unsigned char* recs;      // SREC: staged records (rec_stride apart, slot = lane)
    const uint32_t* sa;       // screen: int8 code words of the centred query (nullptr: off)
    float sq, sa2, seps, smq; // screen: query scale, sq^2 |a|^2, eps_q, (D + 32) 2^-24
};

// Screen (jb_search_args.screen, screen.cu): true when the new neighbour `nb` is
// provably worse than the full beam's worst key. s0 >= sqrt(worst distance).
// |q~ - x~|^2 from exact integer <a, b> (dp4a) with f32 roundings absorbed by a
// 2^-19 (A + B) slack (~10 ulps needed); g <= |q~ - x~|, h >= eps + eps_q + s0 +
// sqrt(M) with M = (D + 32) 2^-24 (|x|^2 + |q|^2) >= |d_f32 - |q - x|^2| (the A1
// dot and norms: chains of D/4 products, two combining adds, three final ops).
// g > h => |q - x|^2 > worst + M => the exact f32 key is above the worst key.
__device__ __forceinline__ bool screen_drop(const jb_search_args& a, const QueryCtx& c, int D, uint32_t nb, float s0,
                                            const uint8_t* srec = nullptr) {
    const int dp = (D + 15) & ~15;
    const bool sm = srec != nullptr;  // staged one hop ahead in smem (snext)
    const uint8_t* rec = sm ? srec : a.screen + (size_t)nb * (dp + 16);
    const uint4* r = reinterpret_cast<const uint4*>(rec);
    const float4 m = sm ? *reinterpret_cast<const float4*>(rec + dp) : __ldg(reinterpret_cast<const float4*>(rec + dp));
    int dot = 0;
    for (int w = 0; w < (dp >> 4); ++w) {
        const uint4 b = sm ? r[w] : __ldg(r + w);
        const uint4 q = *reinterpret_cast<const uint4*>(c.sa + 4 * w);
        dot = __dp4a((int)b.x, (int)q.x, dot);
        dot = __dp4a((int)b.y, (int)q.y, dot);
        dot = __dp4a((int)b.z, (int)q.z, dot);
        dot = __dp4a((int)b.w, (int)q.w, dot);
    }
    const float A = c.sa2, B = m.x * m.x * m.y;
    const float dd = fmaf(-2.0f * c.sq * m.x, (float)dot, A + B) - 0x1p-19f * (A + B);
    if (!(dd > 0.0f)) return false;
    const float g = sqrtf(dd) * (1.0f - 0x1p-20f);
    const float h = (m.z + c.seps + s0 + sqrtf(c.smq * (m.w + c.qadd)) * (1.0f + 0x1p-20f)) * (1.0f + 0x1p-20f);
    return g > h;
}

// Screen setup for one query (warp): a = rint((q - c) / sq) in [-127, 127] (int8,
// zero padded to 16 B), sq = max|q - c| / 127, eps_q >= |sq a - (q - c)|_2 (f64, up).
__device__ __forceinline__ void screen_query(const float* qv, const float* __restrict__ center, int D, uint32_t* sa,
                                             float& sq, float& sa2, float& seps) {
    const int lane = lane_id();
    const int dp = (D + 15) & ~15;
    double mx = 0.0;
    for (int e = lane; e < D; e += 32) mx = fmax(mx, fabs((double)qv[e] - (double)center[e]));
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    const float s = mx > 0.0 ? (float)(mx / 127.0) : 1.0f;
    double err = 0.0, nrm = 0.0;
    int aa = 0;
    int8_t* a8 = reinterpret_cast<int8_t*>(sa);
    for (int e = lane; e < dp; e += 32) {
        int b = 0;
        if (e < D) {
            const double qc = (double)qv[e] - (double)center[e];
            b = (int)rint(qc / (double)s);
            b = b > 127 ? 127 : (b < -127 ? -127 : b);
            const double t = (double)s * (double)b - qc;
            err += t * t;
            nrm += fabs((double)qv[e]) + fabs((double)center[e]);
        }
        aa += b * b;
        a8[e] = (int8_t)b;
    }
    for (int o = 16; o > 0; o >>= 1) {
        err += __shfl_xor_sync(0xFFFFFFFFu, err, o);
        nrm += __shfl_xor_sync(0xFFFFFFFFu, nrm, o);
        aa += __shfl_xor_sync(0xFFFFFFFFu, aa, o);
    }
    sq = s;
    sa2 = s * s * (float)aa;
    seps = __double2float_ru(sqrt(err) * (1.0 + 0x1p-30) + 0x1p-30 * nrm);
    __syncwarp();
}

// One neighbour per lane (nb = -1: none): visited check, then the distance of
// every new neighbour, returned as the lane's candidate key (UMAX = none; EXACT
// compacts the new ids to lanes 0..nnew-1). Adds the new count to `evals`.
// DIRECT (exact source, 16 B aligned rows): the lane that owns a new neighbour reads
// its row straight from global memory instead of the warp staging rows in smem —
// faster when the rows are L2-resident, slower from HBM (uncoalesced sectors).
#ifndef JB_BULK
#define JB_BULK 1  // exact rows staged by cp.async.bulk (one instruction per row); 0: warp-wide 16 B cp.async
#endif
template <int SRC, int BITS, bool ALIGNED, int KD = 0, bool DIRECT = false, bool SREC = false>
__device__ __forceinline__ uint64_t eval_chunk(const jb_search_args& a, const SearchLayout& lay, const QueryCtx& c,
                                               uint32_t* tab, int nb, int& evals, int& lossy, uint32_t& bphase,
                                               float s0 = __builtin_huge_valf(), const uint8_t* srec = nullptr) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = lane_id();
    const int D = KD > 0 ? KD : a.dims;
    // compile-time record size for the specialised popcount kernels (KD > 0: m = 1 plane
    // records of KD bits + 8 B metadata, rounded to 16 B)
    const int RB = (SRC == JB_SRC_RABITQ_FAST && KD > 0 && BITS == 1) ? ((((KD + 31) / 32 + 3) & ~3) * 4 + 8 + 15) / 16 * 16
                                                                      : a.record_bytes;
    // RaBitQ: issue the candidate's record loads before the visited check
    // (32 and 64 B records: whole record in 256-bit loads, one L1 request per 32 B;
    // R64: 64 B records estimated from registers, multi-bit codes only)
    constexpr bool R64 = BITS >= 2 && JB_LDG256_R64;
    uint4 rc0 = make_uint4(0, 0, 0, 0), rc1 = make_uint4(0, 0, 0, 0), rc2 = make_uint4(0, 0, 0, 0),
          rc3 = make_uint4(0, 0, 0, 0);
    if (SRC != JB_SRC_EXACT && !SREC && nb >= 0) {
        const uint8_t* rec = a.records + (size_t)nb * RB;
        if (RB == 32 && (SRC == JB_SRC_RABITQ_FAST || JB_LDG256_R1)) ldg32(rec, rc0, rc1);
        else if (RB == 64 && R64) { ldg32(rec, rc0, rc1); ldg32(rec + 32, rc2, rc3); }
        else {
            rc0 = __ldg(reinterpret_cast<const uint4*>(rec));
            if (RB == 32) rc1 = __ldg(reinterpret_cast<const uint4*>(rec + 16));
        }
    }
    bool isnew = false;
    uint32_t* slot = nullptr;
    if (nb >= 0) isnew = visit(tab, lay.hbits, (uint32_t)nb, lossy, slot);
    __syncwarp();
    // two lanes may have claimed the same empty way: the loser's id is
    // forgotten (safe, but it may be re-evaluated later -> flag it)
    if (slot != nullptr && *reinterpret_cast<volatile uint32_t*>(slot) != (uint32_t)nb) lossy = 1;
    const uint32_t nm = __ballot_sync(FULL, isnew);
    int nnew = __popc(nm);
    if (nnew == 0) return UMAX;
    evals += nnew;

    if (SRC == JB_SRC_EXACT_U8) {  // integer distance, evaluated by the lane that owns the neighbour
        if (!isnew) return UMAX;
        const uint32_t dot = u8_dot(a.data_u8 + (size_t)nb * D, reinterpret_cast<const uint8_t*>(c.qv), D);
        return ((uint64_t)u8_dist(__ldg(a.norms_u32 + nb), dot, c.qn) << 32) | (uint32_t)nb;
    }
    float d = 0.0f;
    int myid = 0;
    if (SRC == JB_SRC_EXACT && ALIGNED && DIRECT) {
        // the lane that owns the neighbour reads its row straight from global (A1 order)
        myid = nb;
        if (isnew) {
            Acc4 acc; acc.zero();
            a1_range<true, false>(acc, a.data + (size_t)nb * D, c.qv, 0, D);
            d = exact_from_dot(__ldg(a.data_norms + nb), acc.reduce(), c.qadd);
        }
    } else if (SRC == JB_SRC_EXACT) {
        // screen (beam full): only neighbours not provably worse than its worst key
        // get the exact A1 distance; the others return no key, as the merge would
        const bool ex = isnew && !(c.sa != nullptr && s0 < __builtin_huge_valf() &&
                                   screen_drop(a, c, D, (uint32_t)nb, s0, srec));
        const uint32_t em = __ballot_sync(FULL, ex);
        nnew = __popc(em);
        if (nnew == 0) return UMAX;
        if (ex) c.cid[__popc(em & lanemask_lt())] = nb;
        __syncwarp();
        myid = (lane < nnew) ? c.cid[lane] : 0;
        // few rows (<= 16, e.g. the screen's survivors): 4 lanes per row, lane j of a
        // group runs A1 chain j (elements j mod 4 of each 16-block, vectors 3..0, then
        // the tail forward) — the same sums as one lane running all four, in a
        // quarter (one pass) or half (two passes) of the dependent steps. Rows are
        // staged lay.srows at a time (16 with the screen: a smaller stage, more warps).
        const int srows = lay.srows;
        const bool split = nnew <= 16 || srows < 32;
        const int grp = lane >> 2, cj = lane & 3;
        uint64_t skey = UMAX;
        Acc4 acc; acc.zero();
        for (int b0 = 0; b0 < nnew; b0 += srows) {
            const int nr = min(srows, nnew - b0);
            float sacc0 = 0.0f, sacc1 = 0.0f;
            const int rid = lane < nr ? c.cid[b0 + lane] : 0;
            for (int e0 = 0; e0 < D; e0 += lay.chunk) {
                const int clen = min(lay.chunk, D - e0);
                if (ALIGNED && JB_BULK) {  // lane j copies row b0 + j's chunk (clen * 4 B, a 16 B multiple)
                    const uint32_t bytes = (uint32_t)clen * 4;
                    wbar_expect(c.bar, bytes * (uint32_t)nr);
                    if (lane < nr) bulk_row(c.stage + lane * lay.sstride, a.data + (size_t)rid * D + e0, bytes, c.bar);
                    wbar_wait(c.bar, bphase);
                } else if (ALIGNED) {
                    const int nv = clen >> 2;
                    for (int j = 0; j < nr; ++j) {
                        const float* src = a.data + (size_t)c.cid[b0 + j] * D + e0;
                        float* dst = c.stage + j * lay.sstride;
                        for (int f = lane; f < nv; f += 32) cp_async16(dst + 4 * f, src + 4 * f);
                    }
                } else {
                    for (int j = 0; j < nr; ++j) {
                        const float* src = a.data + (size_t)c.cid[b0 + j] * D + e0;
                        float* dst = c.stage + j * lay.sstride;
                        for (int f = lane; f < clen; f += 32) cp_async4(dst + f, src + f);
                    }
                }
                if (!(ALIGNED && JB_BULK)) cp_async_wait_all();
                __syncwarp();
                if (split) {
#pragma unroll
                    for (int pp = 0; pp < 2; ++pp) {
                        const int r = pp * 8 + grp;
                        if (r < nr) {
                            const float* row = c.stage + r * lay.sstride;
                            const float* qq = c.qv + e0;
                            float l = pp == 0 ? sacc0 : sacc1;
                            int t = 0;
                            for (; t + 16 <= clen; t += 16) {
#pragma unroll
                                for (int i = 3; i >= 0; --i)
                                    l = __fadd_rn(__fmul_rn(row[t + 4 * i + cj], qq[t + 4 * i + cj]), l);
                            }
                            for (int u = t + cj; u < clen; u += 4) l = __fadd_rn(__fmul_rn(row[u], qq[u]), l);
                            if (pp == 0) sacc0 = l; else sacc1 = l;
                        }
                    }
                } else if (lane < nr) {
                    a1_range<ALIGNED, false>(acc, c.stage + lane * lay.sstride - e0, c.qv, e0, e0 + clen);
                }
                __syncwarp();
            }
            if (split) {
                // (l0 + l1) + (l2 + l3) over the group; row b0 + 8 pp + grp's key ends in
                // lane 4 grp + b0 / 8 + pp (at most one key per lane for nnew <= 32)
#pragma unroll
                for (int pp = 0; pp < 2; ++pp) {
                    const float l = pp == 0 ? sacc0 : sacc1;
                    float t = __fadd_rn(l, __shfl_xor_sync(FULL, l, 1));
                    t = __fadd_rn(t, __shfl_xor_sync(FULL, t, 2));
                    const int r = pp * 8 + grp;
                    uint64_t kp = UMAX;
                    if (cj == 0 && r < nr) {
                        const int id = c.cid[b0 + r];
                        kp = pack_key(exact_from_dot(__ldg(a.data_norms + id), t, c.qadd), (uint32_t)id);
                    }
                    const uint64_t mv = shfl_u64(kp, lane & ~3);
                    if (cj == (b0 >> 3) + pp) skey = mv;
                }
            }
        }
        if (split) return skey;
        if (lane < nnew) d = exact_from_dot(__ldg(a.data_norms + myid), acc.reduce(), c.qadd);
    } else if (SREC) {
        // long records (high D): each new lane's record is staged into its smem slot
        // by one cp.async.bulk (issued together), then read conflict-free from smem
        myid = nb;
        unsigned char* srec = c.recs + lane * lay.rec_stride;
        wbar_expect(c.bar, (uint32_t)RB * (uint32_t)nnew);
        if (isnew) bulk_row(srec, a.records + (size_t)myid * RB, (uint32_t)RB, c.bar);
        wbar_wait(c.bar, bphase);
        if (isnew) {
            const uint4 f = ld16<false>(srec);
            const float2 m = *reinterpret_cast<const float2*>(srec + c.meta_off);
            if (SRC == JB_SRC_RABITQ_FAST) {
                const float dd = rabitq_dd_fast<FAST_QB, 0, BITS, false>(srec, f, c.planes, c.nwords, c.qlo, c.qdelta);
                const float est = (c.qadd + m.x) + m.y * (dd - c.qsumq);
                d = est > 0.0f ? est : 0.0f;
            } else {
                d = rabitq_finish(rabitq_dd<BITS, false>(srec, f, c.qv, D), m, c.qadd, c.qsumq);
            }
        }
    } else {
        // the lane that owns the neighbour evaluates it from its registers
        myid = nb;
        if (isnew) {
            const uint8_t* rec = a.records + (size_t)myid * RB;
            // metadata: in the loaded registers for 32 / 64 B records (16 B aligned offset)
            const uint4 mp = (RB == 32) ? rc1 : (c.meta_off == 16 ? rc1 : (c.meta_off == 32 ? rc2 : rc3));
            const float2 m = (RB == 32 || (RB == 64 && R64)) ? make_float2(__uint_as_float(mp.x), __uint_as_float(mp.y))
                                                             : __ldg(reinterpret_cast<const float2*>(rec + c.meta_off));
            if (SRC == JB_SRC_RABITQ_FAST) {
                const float dd = (BITS == 1 && c.nwords == 4)
                                     ? rabitq_dd_fast<FAST_QB, 4, 1>(rec, rc0, c.planes, 4, c.qlo, c.qdelta)
                                     : rabitq_dd_fast<FAST_QB, 0, BITS>(rec, rc0, c.planes, c.nwords, c.qlo, c.qdelta);
                const float est = (c.qadd + m.x) + m.y * (dd - c.qsumq);
                d = est > 0.0f ? est : 0.0f;
            } else if (R64 && RB == 64) {
                d = rabitq_finish(rabitq_dd_regs<BITS>(rc0, rc1, rc2, c.qv, D), m, c.qadd, c.qsumq);
            } else {
                d = rabitq_finish(rabitq_dd<BITS>(rec, rc0, c.qv, D), m, c.qadd, c.qsumq);
            }
        }
    }
    const bool have = (SRC == JB_SRC_EXACT && !(ALIGNED && DIRECT)) ? (lane < nnew) : isnew;
    return have ? pack_key(d, (uint32_t)myid) : UMAX;
}

// KD > 0 and KHB > 0: compile-time dims and visited-table buckets (log2), so the
// per-warp smem offsets are constants; the beam length (L) stays a runtime value.
// warps per block: 2 for exact f32 rows (smem-bound by the staged rows: finer
// blocks fit more warps per SM — the insert-path search 18.3 -> 15.7 ms per 100K at
// 3M, 0.57 -> 0.66 of HBM), WPB otherwise (the popcount kernel: 4 measured best)
template <int SRC>
constexpr int warps_per_block() { return SRC == JB_SRC_EXACT ? 2 : WPB; }

template <int SRC, int BITS, bool ALIGNED, int CH, int MINB, int KD = 0, int KHB = 0, bool DIRECT = false,
          bool SREC = false>
__global__ void __launch_bounds__(warps_per_block<SRC>() * 32, MINB)
beam_search_kernel(const jb_search_args a, const SearchLayout lay_arg, int* __restrict__ counter) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    SearchLayout lay = lay_arg;
    if (KD > 0 && KHB > 0) {
        constexpr SearchLayout c = make_layout(SRC, KD > 0 ? KD : 1, 0, 4 << (KHB > 0 ? KHB : 1), FAST_QB);
        lay = c;
        lay.bytes = lay_arg.bytes;
    }
    unsigned char* base = smem + (size_t)warp * lay.bytes;
    float* qv = reinterpret_cast<float*>(base + lay.q_off);
    uint64_t* beam = reinterpret_cast<uint64_t*>(base + lay.beam_off);
    uint32_t* tab = reinterpret_cast<uint32_t*>(base + lay.hash_off);
    uint32_t* fmask = reinterpret_cast<uint32_t*>(base + lay.newk_off);  // survivor-slot mask, L/32 words
    int32_t* cid = reinterpret_cast<int32_t*>(base + lay.cid_off);
    float* stage = reinterpret_cast<float*>(base + lay.stage_off);
    uint64_t* wbar = reinterpret_cast<uint64_t*>(base + lay.bar_off);
    uint32_t bphase = 0;
    unsigned char* srecs = base + lay.rec_off;
    if ((SRC == JB_SRC_EXACT && ALIGNED && !DIRECT && JB_BULK) || SREC) {
        if (lane == 0) wbar_init(wbar);
        __syncwarp();
    }
    // snext: the speculative next hop's screen records, staged into smem one hop ahead
    unsigned char* nrec = base + lay.nrec_off;
    uint64_t* nbar = reinterpret_cast<uint64_t*>(nrec + 32 * lay.srb);
    uint32_t nphase = 0;
    if (SRC == JB_SRC_EXACT && lay.snext) {
        if (lane == 0) wbar_init(nbar);
        __syncwarp();
    }
    uint32_t* planes = reinterpret_cast<uint32_t*>(base + lay.plane_off);
    const int D = KD > 0 ? KD : a.dims;
    const int nwords = (((D + 31) / 32) + 3) & ~3;  // plane stride (16 B aligned)

    const int L = a.beam_width;
    const int R = a.degree_cap;
    const int H = 4 << lay.hbits;
    const int RB = a.record_bytes;
    // packed record: code zero-padded to 16 B; popcount plane record: BITS planes of nwords words
    const int meta_off = SRC == JB_SRC_RABITQ_FAST ? BITS * nwords * 4 : ((((D * BITS) + 7) / 8 + 15) / 16) * 16;
    const unsigned FULL = 0xFFFFFFFFu;

    for (;;) {
        int64_t qi = 0;
        if (lane == 0) qi = atomicAdd(counter, 1);
        qi = __shfl_sync(FULL, (long long)qi, 0);
        if (qi >= a.nq) break;

        if (SRC == JB_SRC_EXACT_U8) {
            const uint8_t* q8 = a.queries_u8 + qi * D;
            for (int e = lane; e < D; e += 32) reinterpret_cast<uint8_t*>(qv)[e] = q8[e];
        } else {
            const float* q = a.queries + qi * D;
            for (int e = lane; e < D; e += 32) qv[e] = q[e];
        }
        for (int i = lane; i < L; i += 32) beam[i] = UMAX;
        fmask[lane] = 0;
        for (int i = lane; i < H / 4; i += 32) reinterpret_cast<uint4*>(tab)[i] = make_uint4(EMPTY_SLOT, EMPTY_SLOT, EMPTY_SLOT, EMPTY_SLOT);
        const float qadd = (SRC == JB_SRC_EXACT_U8) ? 0.0f : a.query_add[qi];
        const uint32_t qn = (SRC == JB_SRC_EXACT_U8) ? a.query_norms_u32[qi] : 0u;
        const float qsumq = (SRC != JB_SRC_EXACT) ? a.query_sumq[qi] : 0.0f;
        const uint32_t start = a.starts ? (uint32_t)a.starts[qi] : (uint32_t)a.start_vertex;
        __syncwarp();
        float qlo = 0.0f, qdelta = 0.0f;
        if (SRC == JB_SRC_RABITQ_FAST) build_planes<FAST_QB>(qv, D, planes, qlo, qdelta);
        uint32_t* sa = nullptr;
        float ssq = 0.0f, ssa2 = 0.0f, sseps = 0.0f;
        if (SRC == JB_SRC_EXACT && a.screen != nullptr) {
            sa = reinterpret_cast<uint32_t*>(base + lay.scr_off);
            screen_query(qv, a.screen_center, D, sa, ssq, ssa2, sseps);
        }
        const QueryCtx qc{qv, planes, cid, stage, qadd, qsumq, qlo, qdelta, nwords, meta_off, qn, wbar, srecs,
                          sa, ssq, ssa2, sseps, (float)(D + 32) * 0x1p-24f};

        int lossy = 0;
        if (lane == 0) {
            float d0 = 0.0f;
            if (SRC == JB_SRC_EXACT_U8) {
                const uint32_t dot = u8_dot(a.data_u8 + (size_t)start * D, reinterpret_cast<const uint8_t*>(qv), D);
                beam[0] = ((uint64_t)u8_dist(a.norms_u32[start], dot, qn) << 32) | start;
            } else if (SRC == JB_SRC_EXACT) {
                const float dot = a1_dot<false>(a.data + (size_t)start * D, qv, D);
                d0 = exact_from_dot(a.data_norms[start], dot, qadd);
            } else if (SRC == JB_SRC_RABITQ_FAST) {
                d0 = rabitq_estimate_fast<FAST_QB, BITS>(a.records + (size_t)start * RB, planes, nwords, meta_off, qlo, qdelta, qadd,
                                          qsumq);
            } else {
                d0 = rabitq_estimate<BITS>(a.records + (size_t)start * RB, qv, D, meta_off, qadd, qsumq);
            }
            if (SRC != JB_SRC_EXACT_U8) beam[0] = pack_key(d0, start);
            uint32_t* sl;
            visit(tab, lay.hbits, start, lossy, sl);
        }
        __syncwarp();

        int bcount = 1, cursor = 0, hops = 0, evals = 1;
        const int tcap = a.trace_cap;
        int32_t* tids = a.trace_ids ? a.trace_ids + qi * (int64_t)tcap : nullptr;
        float* tdst = a.trace_dists ? a.trace_dists + qi * (int64_t)tcap : nullptr;

        // Speculative adjacency prefetch: the next expansion is guessed as the first
        // unexpanded key after the cursor in the pre-merge beam (right whenever this
        // hop inserts nothing in front of it). Its row is loaded while this hop runs.
        int spec = -1;
        int nxt_for = -1;     // snext: the vertex whose neighbours' records are staged
        bool nxt_pend = false;
        int spec_nb[CH];
#pragma unroll
        for (int c = 0; c < CH; ++c) spec_nb[c] = -1;

        while (cursor < bcount) {
            const uint64_t ukey = beam[cursor];
            const uint32_t u = key_id(ukey);
            bool nxt_hit = false;
            if (SRC == JB_SRC_EXACT && CH == 1 && lay.snext && nxt_pend) {
                wbar_wait(nbar, nphase);
                nxt_pend = false;
                nxt_hit = nxt_for == (int)u;
            }
            const int sidx = first_unexpanded(beam, cursor + 1, bcount);
            const int nspec = sidx < bcount ? (int)key_id(beam[sidx]) : -1;
            __syncwarp();
            if (lane == 0) {
                beam[cursor] = ukey | EXPANDED;
                if (hops < tcap) {  // the key's distance word (f32 bits, or the u32 integer distance)
                    tids[hops] = (int32_t)u;
                    reinterpret_cast<uint32_t*>(tdst)[hops] = (uint32_t)(ukey >> 32);
                }
            }
            ++hops;
            int s_min = cursor + 1;
            int p_ins = bcount;  // CH == 1: smallest insertion position of this hop's merge
            int nbv[CH];
            const int32_t* adj_u = a.adjacency + (size_t)u * R;
            const int32_t* adj_s = a.adjacency + (size_t)(nspec < 0 ? 0 : nspec) * R;
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int r = c * 32 + lane;
                nbv[c] = (spec == (int)u) ? spec_nb[c] : ((r < R) ? __ldg(adj_u + r) : -1);
                spec_nb[c] = (nspec >= 0 && r < R) ? __ldg(adj_s + r) : -1;
            }
            spec = nspec;

#pragma unroll
            for (int c = 0; c < CH; ++c) {
                if (c * 32 >= R) break;
                float s0 = __builtin_huge_valf();  // sqrt(worst distance), rounded up; inf: no screen
                if (SRC == JB_SRC_EXACT && sa != nullptr && bcount == L)
                    s0 = sqrtf(__uint_as_float((uint32_t)(beam[L - 1] >> 32))) * (1.0f + 0x1p-20f);
                const uint8_t* srec = (SRC == JB_SRC_EXACT && nxt_hit) ? nrec + lane * lay.srb : nullptr;
                const uint64_t key = eval_chunk<SRC, BITS, ALIGNED, KD, DIRECT, SREC>(a, lay, qc, tab, nbv[c], evals,
                                                                                     lossy, bphase, s0, srec);
                if (SRC == JB_SRC_EXACT && CH == 1 && lay.snext && sa != nullptr && bcount == L) {
                    // stage the speculative next hop's records (its adjacency row has arrived)
                    const int have = spec_nb[0] >= 0;
                    const uint32_t cnt = (uint32_t)__popc(__ballot_sync(0xFFFFFFFFu, have));
                    if (cnt > 0) {
                        wbar_expect(nbar, cnt * (uint32_t)lay.srb);
                        if (have)
                            bulk_row(nrec + lane * lay.srb, a.screen + (size_t)spec_nb[0] * lay.srb, (uint32_t)lay.srb,
                                     nbar);
                        nxt_for = spec;
                        nxt_pend = true;
                    }
                } else if (SRC == JB_SRC_EXACT && sa != nullptr && lay.spf && spec_nb[c] >= 0) {
                    // the speculative next hop's screen records into L2 (its adjacency row
                    // has arrived by now): the next hop's screen then reads L2, not HBM
                    const char* pr = reinterpret_cast<const char*>(a.screen) + (size_t)spec_nb[c] * lay.srb;
                    if (lay.spf == 2) {  // the copy engine's L2 prefetch of the whole record
                        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pr), "r"(lay.srb) : "memory");
                    } else {
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(pr));
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(pr + lay.srb - 16));
                    }
                }
                const int p0 = merge_into_beam(beam, bcount, L, key, fmask);
                s_min = min(s_min, p0);
                p_ins = p0;
            }
            if (CH == 1) {
                // One merge per hop: the keys it inserted are unexpanded and the smallest
                // landed at p_ins (the pre-merge bcount when nothing was inserted);
                // entries before it are unchanged. So the first unexpanded key is at
                // p_ins if that is at or before the pre-merge candidate sidx, else sidx
                // did not move (nothing was inserted in front of it).
                cursor = min(p_ins, sidx);
            } else {
                cursor = first_unexpanded(beam, s_min, bcount);
            }
        }

        if (SRC == JB_SRC_EXACT && CH == 1 && lay.snext && nxt_pend) {  // drain before the buffer is reused
            wbar_wait(nbar, nphase);
            nxt_pend = false;
        }
        // ---- outputs ----
        uint64_t* fk = a.frontier_keys + qi * (int64_t)L;
        for (int i = lane; i < L; i += 32) {
            const uint64_t k = beam[i];
            fk[i] = (k == UMAX) ? UMAX : key_mask(k);
        }
        lossy = __reduce_or_sync(FULL, lossy);
        if (lane == 0) {
            if (a.hops) a.hops[qi] = hops;
            if (a.evals) a.evals[qi] = evals;
            if (a.flags) a.flags[qi] = lossy ? 1 : 0;
        }
        __syncwarp();
    }
}


// ---- exact rerank of the frontier (search.py:318-320, 375-382) -----------
// One warp per query, 8 frontier rows at a time: the rows are staged into smem
// with coalesced cp.async (512 B per warp instruction at D = 128), then 4 lanes
// per row each run one A1 accumulator chain j of einsum(x - q, x - q) (elements
// e = j mod 4, 16-element blocks with vectors 3,2,1,0, then the tail forward;
// conflict-free scalar smem reads) and the chains combine as (l0 + l1) + (l2 + l3)
// over two shuffles. ~6 KB of smem per warp keeps ~32 warps per SM loading.
// Keys (dist, id) are then sorted (bitonic, smem) and the first k written.
__global__ void __launch_bounds__(RR_WARPS * 32)
rerank_kernel(const float* __restrict__ data, int D, const float* __restrict__ queries, int64_t nq,
              const uint64_t* __restrict__ fkeys, int L, int k, int lpad, int rstride, int per_warp,
              int32_t* __restrict__ out_ids, double* __restrict__ out_dists) {
    const int wpb = blockDim.x >> 5;
    extern __shared__ __align__(16) unsigned char smem[];
    const unsigned FULL = 0xFFFFFFFFu;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* base = smem + (size_t)warp * per_warp;
    float* qv = reinterpret_cast<float*>(base);
    uint64_t* keys = reinterpret_cast<uint64_t*>(base + ((D * 4 + 15) / 16) * 16);
    float* stage = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(keys) + (size_t)lpad * 8);
    const int64_t qi = (int64_t)blockIdx.x * wpb + warp;
    if (qi >= nq) return;
    const float* q = queries + qi * D;
    for (int e = lane; e < D; e += 32) qv[e] = q[e];
    const uint64_t* fk = fkeys + qi * (int64_t)L;
    // valid keys (the frontier is sorted; UMAX padding at the end)
    int n = 0;
    for (int b = 0; b < L; b += 32) {
        const int i = b + lane;
        n += __popc(__ballot_sync(FULL, i < L && fk[i] != UMAX));
    }
    for (int i = lane; i < lpad; i += 32) keys[i] = UMAX;
    __syncwarp();
    const int r = lane >> 2, j = lane & 3;
    const int D16 = D & ~15;
    const bool vec = (D & 3) == 0;
    const int nv = D >> 2;  // 16 B chunks per row
    const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
    for (int c = 0; c < n; c += RR_ROWS) {
        const int cnt = min(RR_ROWS, n - c);
        const uint32_t myid = lane < cnt ? (uint32_t)(fk[c + lane] & 0xFFFFFFFFull) : 0u;
        if (vec && nv <= 32) {  // one 16 B chunk per lane per row (D <= 128)
#pragma unroll
            for (int t = 0; t < RR_ROWS; ++t) {
                const uint32_t id = __shfl_sync(FULL, myid, t);
                if (t < cnt && lane < nv) {
                    const float* src = data + (size_t)id * D + 4 * lane;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(stage_s + (t * rstride + 4 * lane) * 4),
                                 "l"(src));
                }
            }
        } else {
            for (int t = 0; t < cnt; ++t) {
                const uint32_t id = __shfl_sync(FULL, myid, t);
                const float* src = data + (size_t)id * D;
                float* dst = stage + t * rstride;
                if (vec) { for (int f = lane; f < nv; f += 32) cp_async16(dst + 4 * f, src + 4 * f); }
                else { for (int f = lane; f < D; f += 32) cp_async4(dst + f, src + f); }
            }
        }
        cp_async_wait_all();
        __syncwarp();
        const bool on = r < cnt;
        const float* row = stage + r * rstride;
        float acc = 0.0f;
        if (on) {
            for (int b = 0; b < D16; b += 16) {
#pragma unroll
                for (int i = 3; i >= 0; --i) {
                    const int e = b + 4 * i + j;
                    const float d = __fsub_rn(row[e], qv[e]);
                    acc = __fadd_rn(__fmul_rn(d, d), acc);
                }
            }
            for (int e = D16 + j; e < D; e += 4) {  // tail: forward, element e -> chain e % 4
                const float d = __fsub_rn(row[e], qv[e]);
                acc = __fadd_rn(__fmul_rn(d, d), acc);
            }
        }
        // (l0 + l1) + (l2 + l3)
        const float pair = __fadd_rn(acc, __shfl_down_sync(FULL, acc, 1));
        const float tot = __fadd_rn(pair, __shfl_down_sync(FULL, pair, 2));
        const uint32_t rid = __shfl_sync(FULL, myid, r);
        if (on && j == 0) keys[c + r] = pack_key(tot, rid);
        __syncwarp();
    }
    __syncwarp();
    if (k <= 32) {  // the k smallest (dist, id) keys in order: repeated warp minimum
        uint64_t mine = UMAX;  // this lane's answer slot (rank == lane)
        for (int jj = 0; jj < k; ++jj) {
            uint64_t m = UMAX;
            int mi = -1;
            for (int i = lane; i < n; i += 32) {
                const uint64_t c = keys[i];
                if (c < m) { m = c; mi = i; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const uint64_t om = shfl_xor_u64(m, o);
                const int oi = __shfl_xor_sync(FULL, mi, o);
                if (om < m) { m = om; mi = oi; }
            }
            if (lane == jj) mine = m;
            if (lane == 0 && mi >= 0) keys[mi] = UMAX;
            __syncwarp();
        }
        if (lane < k) {
            const int64_t o = qi * k + lane;
            if (mine != UMAX) {
                out_ids[o] = (int32_t)(mine & 0xFFFFFFFFull);
                out_dists[o] = (double)__uint_as_float((uint32_t)(mine >> 32));
            } else {
                out_ids[o] = -1;
                out_dists[o] = __longlong_as_double(0x7FF0000000000000ll);
            }
        }
        return;
    }
    warp_bitonic_sort_smem(keys, lpad);
    for (int jj = lane; jj < k; jj += 32) {
        const uint64_t key = keys[jj];
        const int64_t o = qi * k + jj;
        if (jj < n) {
            out_ids[o] = (int32_t)(key & 0xFFFFFFFFull);
            out_dists[o] = (double)__uint_as_float((uint32_t)(key >> 32));
        } else {
            out_ids[o] = -1;
            out_dists[o] = __longlong_as_double(0x7FF0000000000000ll);
        }
    }
}


// ---- reference-defined eval counts (search.py:211-226) ----------------------
// evals = |{start} U N(u) for every expanded u|: the reference evaluates every
// valid neighbour of an expanded vertex exactly once (its `seen` matrix). The
// search kernel counts its own evaluations, which include re-evaluations after
// visited-table evictions (flags bit 0); this recount is exact. Warp per query
// (persistent), an open-addressing id set in a per-warp global scratch slice of
// `slots` (pow2 >= 2 x the largest possible set).
__global__ void __launch_bounds__(256)
count_evals_kernel(const int32_t* __restrict__ adj, int R, const int32_t* __restrict__ tids, int cap,
                   const int32_t* __restrict__ hops, const int32_t* __restrict__ starts, int64_t start_vertex,
                   const int32_t* __restrict__ flags, int64_t nq, uint32_t* __restrict__ scratch, int slots,
                   int32_t* __restrict__ evals) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    uint32_t* tab = scratch + w0 * (int64_t)slots;
    const int hb = log2i(slots);
    for (int64_t q = w0; q < nq; q += nw) {
        if (flags && !(flags[q] & 1)) continue;  // no eviction: the kernel's own count is exact
        for (int i = lane; i < slots; i += 32) tab[i] = EMPTY_SLOT;
        __syncwarp();
        const int h = min(hops[q], cap);
        int cnt = 0;
        auto insert = [&](uint32_t v) {
            uint32_t b = (v * 0x9E3779B1u) >> (32 - hb);
            for (;;) {
                const uint32_t old = atomicCAS(tab + b, EMPTY_SLOT, v);
                if (old == EMPTY_SLOT) { ++cnt; return; }
                if (old == v) return;
                b = (b + 1) & (uint32_t)(slots - 1);
            }
        };
        if (lane == 0) insert(starts ? (uint32_t)starts[q] : (uint32_t)start_vertex);
        for (int i = 0; i < h; ++i) {
            const int32_t u = tids[q * (int64_t)cap + i];
            for (int j = lane; j < R; j += 32) {
                const int32_t v = adj[(size_t)u * R + j];
                if (v >= 0) insert((uint32_t)v);
            }
        }
        for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
        if (lane == 0) evals[q] = cnt;
        __syncwarp();
    }
}

using SearchKernel = void (*)(const jb_search_args, const SearchLayout, int*);

// Exact rows small enough to stay in L2 (<= half of it) are read lane-by-lane from
// global memory (measured: +22-33% QPS on 100K x 128); larger sets are staged with
// coalesced cp.async (direct reads halved QPS on 10M x 96 rows in HBM).
// JB_EXACT_DIRECT=0/1 forces either (A/B).
static bool rows_l2_resident(const jb_search_args& a) {
    const char* e = std::getenv("JB_EXACT_DIRECT");
    if (e && (e[0] == '0' || e[0] == '1')) return e[0] == '1';
    static thread_local int dev = -1, l2 = 0;
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) return false;
    if (d != dev) {
        if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, d) != cudaSuccess) l2 = 0;
        dev = d;
    }
    return (double)a.active_count * a.dims * 4.0 <= 0.5 * (double)l2;
}

// The screen adds one dependent record fetch per hop in front of the survivors'
// row fetch. Where the records stay largely L2-resident (or the rows are long) the
// next hop's records are prefetched into L2; beyond that (HBM-resident short rows)
// they are staged into smem one hop ahead instead (snext: +32 records per warp,
// fewer warps, but the fetch is off the hop's critical path). Measured, phase-1
// search per 100K (8-row stage, 14-block kernel): 1M x 128 (144 MB of records)
// 19.8 -> 13.5 ms with L2 prefetch (16.2 with snext); 96-d with L2 prefetch: 3M
// (336 MB) 16.0 -> 13.8, 4.5M 16.4 -> 18.3, 6M 16.7 -> 21.1, 12.5M 17.3 -> 24.4 ms;
// with snext: 6M 16.9 -> 16.2, 12.5M 17.5 -> 16.7 ms. So snext when the records
// exceed 3 x L2 (378 MB on B200) and D < 256. JB_SCREEN_FORCE=0 turns the screen
// off; JB_SCREEN_NEXT=0 / 1 forces the staging mode (A/B).
static bool screen_big(const jb_search_args& a) {
    static thread_local int dev = -1, l2 = 0;
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) return false;
    if (d != dev) {
        if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, d) != cudaSuccess) l2 = 0;
        dev = d;
    }
    const double rec = (double)a.active_count * (((a.dims + 15) & ~15) + 16);
    return rec > 3.0 * (double)l2 && a.dims < 256;
}
static bool screen_off() {
    const char* e = std::getenv("JB_SCREEN_FORCE");
    return e && e[0] == '0';
}

#ifndef JB_SREC_MIN
#define JB_SREC_MIN 256  // records of at least this many bytes are staged into smem (SREC kernels)
#endif
// JB_SREC=0 keeps high-D records on per-lane global loads (A/B)
static bool srec_on() {
    static const bool on = [] {
        const char* e = std::getenv("JB_SREC");
        return !(e && e[0] == '0');
    }();
    return on;
}

// JB_SEARCH_SPEC=0 disables the compile-time-shape kernels (A/B and debugging)
static bool specialize_off() {
    static const bool off = [] {
        const char* e = std::getenv("JB_SEARCH_SPEC");
        return e && e[0] == '0';
    }();
    return off;
}

// Occupancy per (kernel, smem size) is cached: the attribute/occupancy queries
// cost more than the launch itself for small batches.
static int launch_search_kernel(SearchKernel kern, const SearchLayout& lay, const jb_search_args& a, cudaStream_t st,
                                int nw = WPB) {
    const int smem = lay.bytes * nw;
    JB_CHECK_ARG(smem <= 227 * 1024, "beam search: per-block shared memory %d B exceeds 227 KB", smem);
    // The smem attribute only grows, process-wide (grow_smem), so no host thread can
    // lower it below another thread's cached launch configuration. Occupancy per
    // (kernel, smem, device) is cached per thread (the query costs more than a launch).
    struct Entry { SearchKernel k; int smem, dev, per_sm; };
    static thread_local Entry cache[16] = {};
    static thread_local int next = 0;
    int dev = 0;
    JB_CUDA(cudaGetDevice(&dev));
    int per_sm = 0;
    for (const Entry& e : cache)
        if (e.k == kern && e.smem == smem && e.dev == dev) per_sm = e.per_sm;
    if (per_sm == 0) {
        JB_CUDA_RC(grow_smem(kern, smem));
        JB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem));
        JB_CHECK_ARG(per_sm >= 1, "beam search: kernel does not fit on an SM");
        cache[next] = Entry{kern, smem, dev, per_sm};
        next = (next + 1) % 16;
    }
    int64_t need = (a.nq + nw - 1) / nw;
    int grid = (int)std::min<int64_t>(need, (int64_t)per_sm * sm_count_current());
    Scratch ctr;
    JB_CUDA(ctr.alloc(sizeof(int), st));
    JB_CUDA(cudaMemsetAsync(ctr.p, 0, sizeof(int), st));
    kern<<<grid, nw * 32, smem, st>>>(a, lay, ctr.as<int>());
    JB_LAUNCH_CHECK();
    return JB_OK;
}

// rows staged per pass with the screen (JB_SCREEN_SROWS, 8..32; default 8 with the
// 14-block kernel: 13.5 ms per 100K at 1M vs 14.0 for 16 rows at 8 blocks)
static int screen_srows() {
    const char* e = std::getenv("JB_SCREEN_SROWS");
    const int v = e ? std::atoi(e) : 8;
    return v >= 32 ? 32 : (v <= 8 ? 8 : 16);
}

// stage the speculative next hop's screen records into smem (see screen_big)
static bool screen_next(const jb_search_args& a) {
    const char* e = std::getenv("JB_SCREEN_NEXT");
    if (e && (e[0] == '0' || e[0] == '1')) return e[0] == '1';
    return screen_big(a);
}

// resident blocks the screened exact kernel is compiled for (JB_SCREEN_MINB: 8 or 14,
// default 14: 72 registers with a few spills, 28 warps/SM with the 8-row stage)
static int screen_minb() {
    const char* e = std::getenv("JB_SCREEN_MINB");
    return (e && std::atoi(e) == 8) ? 8 : 14;
}

// JB_SCREEN_PF: 0 = no prefetch of the next hop's screen records, 1 = prefetch.global.L2
// (default), 2 = cp.async.bulk.prefetch.L2 (better at 6M x 96, worse at 1M x 128)
static int screen_prefetch() {
    const char* e = std::getenv("JB_SCREEN_PF");
    return e ? std::atoi(e) : 1;
}

// R <= 32: one neighbour chunk per hop (single merge, no rescan of the beam);
// MAX_CHUNKS for wider rows. Blocks/SM: the popcount kernel is issue-bound and
// gains from 10 resident blocks; the float estimators keep 8.
template <int SRC, int BITS, bool ALIGNED>
static int launch_search(const jb_search_args& a, int hash_slots, cudaStream_t st) {
    // multi-bit popcount records keep MB code planes live: 8 blocks/SM (64 registers) instead of spilling
    constexpr int MINB = SRC == JB_SRC_RABITQ_FAST ? (BITS == 1 ? JB_FAST_MINB : 8)
                         : SRC == JB_SRC_RABITQ    ? JB_RQ_MINB
                                                   : JB_OTHER_MINB;
    constexpr int NW = warps_per_block<SRC>();
    const int L = a.beam_width;
    SearchLayout lay = make_layout(SRC, a.dims, L, hash_slots, FAST_QB, false, 0,
                                   (SRC == JB_SRC_EXACT && a.screen != nullptr) ? screen_srows() : 32);
    lay.spf = (SRC == JB_SRC_EXACT && a.screen != nullptr) ? screen_prefetch() : 0;
    if (SRC == JB_SRC_EXACT && a.screen != nullptr && a.degree_cap <= 32 && screen_next(a)) {
        // 32 staged records + mbarrier in front of the beam (the beam moves up)
        const int extra = 32 * lay.srb + 16;
        lay.snext = 1;
        lay.nrec_off = lay.beam_off;
        lay.beam_off += extra;
        lay.bytes += extra;
    }
    if (a.degree_cap <= 32 && SRC == JB_SRC_RABITQ_FAST && BITS == 1) {
        // specialised shapes: D in {96, 128} with a 512- or 1024-slot visited table (popcount
        // estimator only: measured -2% at L=128; the float estimators got slower, +4%)
        const int hb = lay.hbits;
#define JB_SPEC(KD_, KHB_)                                                                                   \
    if (a.dims == KD_ && hb == KHB_)                                                                         \
        return launch_search_kernel(beam_search_kernel<SRC, BITS, ALIGNED, 1, MINB, KD_, KHB_>, lay, a, st, NW);
        if (ALIGNED && !specialize_off()) {
            JB_SPEC(128, 7) JB_SPEC(128, 8) JB_SPEC(96, 7) JB_SPEC(96, 8)
        }
#undef JB_SPEC
    }
    if constexpr (SRC == JB_SRC_RABITQ || SRC == JB_SRC_RABITQ_FAST) {
        if (a.degree_cap <= 32 && a.record_bytes >= JB_SREC_MIN && srec_on()) {
            // high-D records (e.g. 496 B at D = 960, m = 4): staged per lane by the copy engine
            const SearchLayout lr = make_layout(SRC, a.dims, L, hash_slots, FAST_QB, false, a.record_bytes);
            return launch_search_kernel(beam_search_kernel<SRC, BITS, ALIGNED, 1, 8, 0, 0, false, true>, lr, a, st, NW);
        }
    }
    if (SRC == JB_SRC_EXACT && ALIGNED && a.degree_cap <= 32 && rows_l2_resident(a)) {
        const SearchLayout ld = make_layout(SRC, a.dims, L, hash_slots, FAST_QB, true);
        return launch_search_kernel(beam_search_kernel<SRC, BITS, ALIGNED, 1, MINB, 0, 0, true>, ld, a, st, NW);
    }
    if constexpr (SRC == JB_SRC_EXACT) {
        // screened exact rows (16- or 8-row stage): registers, not smem, cap the warps
        // per SM at 8 blocks; the 14-block build trades a few spills for occupancy
        if (a.degree_cap <= 32 && a.screen != nullptr && screen_minb() == 14)
            return launch_search_kernel(beam_search_kernel<SRC, BITS, ALIGNED, 1, 14>, lay, a, st, NW);
    }
    if (a.degree_cap <= 32) return launch_search_kernel(beam_search_kernel<SRC, BITS, ALIGNED, 1, MINB>, lay, a, st, NW);
    return launch_search_kernel(beam_search_kernel<SRC, BITS, ALIGNED, MAX_CHUNKS, 8>, lay, a, st, NW);
}

}  // namespace jb

using namespace jb;

extern "C" {

#ifdef JB_MERGE_STATS
int jb_debug_merge_stats(unsigned long long* out) {
    JB_CUDA(cudaMemcpyFromSymbol(out, g_merge_stats, sizeof(unsigned long long) * 66));
    static const unsigned long long zero[66] = {};
    JB_CUDA(cudaMemcpyToSymbol(g_merge_stats, zero, sizeof(zero)));
    return JB_OK;
}
#endif

int jb_beam_search(const jb_search_args* args, void* stream) {
    JB_CHECK_ARG(args != nullptr, "jb_beam_search: null args");
    const jb_search_args& a = *args;
    JB_CHECK_ARG(a.active_count > 0, "search on an empty graph");
    JB_CHECK_ARG(a.beam_width >= 1 && a.beam_width <= 1024, "beam_width must be in [1, 1024]");
    JB_CHECK_ARG(a.degree_cap >= 1 && a.degree_cap <= 32 * MAX_CHUNKS, "degree_cap must be in [1, %d]",
                 32 * MAX_CHUNKS);
    JB_CHECK_ARG(a.dims >= 1, "dims must be >= 1");
    JB_CHECK_ARG(a.active_count < (1ll << 31), "active_count exceeds int32 ids");
    JB_CHECK_ARG(a.trace_cap == 0 || (a.trace_ids && a.trace_dists), "trace buffers required when trace_cap > 0");
    JB_CHECK_ARG(a.starts != nullptr || (a.start_vertex >= 0 && a.start_vertex < a.active_count),
                 "start vertex out of range");
    if (a.nq == 0) return JB_OK;
    int hs = a.hash_slots;
    // Small tables win: evictions only cost re-evaluations (results stay exact),
    // while smem per warp sets occupancy (measured at L=128: 1024 slots 19% faster
    // than 2048; 512 slots 1% faster than 1024 with 10 blocks/SM).
    if (hs <= 0) hs = std::min(2048, std::max(512, pow2_ceil(4 * a.beam_width)));
    hs = std::max(32, pow2_ceil(hs));
    cudaStream_t st = as_stream(stream);
    if (a.source == JB_SRC_EXACT_U8) {
        JB_CHECK_ARG(a.data_u8 && a.norms_u32 && a.queries_u8 && a.query_norms_u32, "u8 search: missing arrays");
        JB_CHECK_ARG((int64_t)a.dims * 255 * 255 < (1ll << 32), "u8 dims too large for 32-bit packed distances");
        return launch_search<JB_SRC_EXACT_U8, 1, true>(a, hs, st);
    }
    if (a.source == JB_SRC_EXACT) {
        JB_CHECK_ARG(a.data && a.data_norms && a.queries && a.query_add, "exact search: missing arrays");
        JB_CHECK_ARG(a.screen == nullptr || (a.screen_center != nullptr && a.dims <= 1040),
                     "exact search: screen records need their centre (dims <= 1040)");
        if (a.screen != nullptr && screen_off()) {  // A/B: unscreened
            jb_search_args b = a;
            b.screen = nullptr;
            if ((b.dims & 3) == 0) return launch_search<JB_SRC_EXACT, 1, true>(b, hs, st);
            return launch_search<JB_SRC_EXACT, 1, false>(b, hs, st);
        }
        if ((a.dims & 3) == 0) return launch_search<JB_SRC_EXACT, 1, true>(a, hs, st);
        return launch_search<JB_SRC_EXACT, 1, false>(a, hs, st);
    }
    JB_CHECK_ARG(a.source == JB_SRC_RABITQ || a.source == JB_SRC_RABITQ_FAST, "unknown distance source %d", a.source);
    JB_CHECK_ARG(a.records && a.queries && a.query_add && a.query_sumq, "rabitq search: missing arrays");
    if (a.source == JB_SRC_RABITQ_FAST) {  // bit-plane records (jb_rabitq_pack_planes; = packed for m = 1)
        JB_CHECK_ARG(a.record_bytes == jb_rabitq_plane_record_bytes(a.dims, a.bits),
                     "popcount search: record_bytes mismatch (plane records expected)");
        switch (a.bits) {
            case 1: return launch_search<JB_SRC_RABITQ_FAST, 1, true>(a, hs, st);
            case 2: return launch_search<JB_SRC_RABITQ_FAST, 2, true>(a, hs, st);
            case 4: return launch_search<JB_SRC_RABITQ_FAST, 4, true>(a, hs, st);
            case 8: return launch_search<JB_SRC_RABITQ_FAST, 8, true>(a, hs, st);
            default: JB_CHECK_ARG(false, "bits must be one of (1, 2, 4, 8)");
        }
    }
    JB_CHECK_ARG(a.record_bytes == jb_rabitq_record_bytes(a.dims, a.bits), "rabitq search: record_bytes mismatch");
    switch (a.bits) {
        case 1: return launch_search<JB_SRC_RABITQ, 1, true>(a, hs, st);
        case 2: return launch_search<JB_SRC_RABITQ, 2, true>(a, hs, st);
        case 4: return launch_search<JB_SRC_RABITQ, 4, true>(a, hs, st);
        case 8: return launch_search<JB_SRC_RABITQ, 8, true>(a, hs, st);
        default: JB_CHECK_ARG(false, "bits must be one of (1, 2, 4, 8)");
    }
}

int jb_count_evals(const int32_t* adjacency, int32_t degree_cap, const int32_t* trace_ids, int32_t trace_cap,
                   const int32_t* hops, const int32_t* starts, int64_t start_vertex, const int32_t* flags, int64_t nq,
                   int32_t* evals, void* stream) {
    JB_CHECK_ARG(adjacency && trace_ids && hops && evals, "jb_count_evals: missing arrays");
    JB_CHECK_ARG(degree_cap >= 1 && trace_cap >= 1, "jb_count_evals: bad degree_cap / trace_cap");
    if (nq == 0) return JB_OK;
    const int64_t most = (int64_t)trace_cap * degree_cap + 1;
    JB_CHECK_ARG(most < (1ll << 28), "jb_count_evals: trace too long");
    const int slots = pow2_ceil((int)(2 * most));
    cudaStream_t st = as_stream(stream);
    const int64_t warps = std::min<int64_t>(nq, (int64_t)sm_count_current() * 32);
    Scratch tab;
    JB_CUDA(tab.alloc((size_t)warps * slots * sizeof(uint32_t), st));
    count_evals_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(
        adjacency, degree_cap, trace_ids, trace_cap, hops, starts, start_vertex, flags, nq, tab.as<uint32_t>(), slots,
        evals);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

int jb_rerank_topk(const float* data, int32_t dims, const float* queries, int64_t nq,
                   const uint64_t* frontier_keys, int32_t beam_width, int32_t k,
                   int32_t* out_ids, double* out_dists, void* stream) {
    JB_CHECK_ARG(k >= 1 && k <= beam_width, "k must satisfy 1 <= k <= beam_width");
    JB_CHECK_ARG(dims >= 1, "dims must be >= 1");
    if (nq == 0) return JB_OK;
    const int lpad = std::max(32, pow2_ceil(beam_width));
    // staged row stride: 16 B aligned, and 4 (mod 32) words so the 8 rows x 4 chains
    // of a scalar smem read hit 32 distinct banks
    const int rstride = ((dims + 3) & ~3) + ((4 - (((dims + 3) & ~3) % 32) + 32) % 32);
    const int per_warp = ((dims * 4 + 15) / 16) * 16 + lpad * 8 + RR_ROWS * rstride * 4;
    const int wpb = std::max(1, std::min(RR_WARPS, (200 * 1024) / per_warp));  // high-D rows: fewer warps per block
    const int smem = per_warp * wpb;
    JB_CHECK_ARG(smem <= 227 * 1024, "rerank: shared memory %d B exceeds 227 KB", smem);
    cudaStream_t st = as_stream(stream);
    const unsigned grid = (unsigned)((nq + wpb - 1) / wpb);
    JB_CUDA_RC(grow_smem(rerank_kernel, smem));
    rerank_kernel<<<grid, wpb * 32, smem, st>>>(data, dims, queries, nq, frontier_keys, beam_width, k, lpad, rstride,
                                                per_warp, out_ids, out_dists);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

}  // extern "C"
