/*
 * jasper_b200.h — C ABI of the B200-native hot paths of the `beamann` reference
 * (arxiv 2601.07048, "Jasper"): Vamana greedy beam search, RaBitQ estimation +
 * fp32 rerank, batch-parallel lock-free insertion, sharded top-k merge.
 *
 * Conventions
 *  - Every entry point returns an int status (JB_OK == 0). On failure
 *    jb_last_error() returns a thread-local, NUL-terminated message.
 *  - All array arguments are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *    unless the name ends in `_host`. The caller owns every buffer passed in;
 *    the library only allocates stream-ordered scratch (cudaMallocAsync) that
 *    it frees before returning.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    Calls are asynchronous w.r.t. the host unless documented otherwise; calls
 *    that must read a device value back (loop trip counts) synchronize `stream`.
 *  - Arithmetic follows the reference's numpy rounding order bit-exactly
 *    ("A1": 4-lane SSE einsum order, separate multiply and add, no FMA), so
 *    device results are identical to the reference on the same inputs.
 *  - Search keys are the reference's u64 keys: (f32 bits of max(d,0)) << 32 | id
 *    (search.py:139-156). Bit 31 of the low word is used on device only as the
 *    "expanded" flag and is always cleared in outputs.
 *
 * Each function names the reference function it replaces (file:line relative
 * to pkg/src/beamann/ of the reference).
 */
#ifndef JASPER_B200_H
#define JASPER_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define JB_OK 0
#define JB_EINVAL 1        /* bad argument (mirrors the reference's ValueError) */
#define JB_ECUDA 2         /* CUDA runtime / launch failure                     */
#define JB_ENODONOR 3      /* connectivity repair found no donor (RuntimeError) */
#define JB_EOVERFLOW 4     /* a bounded device buffer overflowed                */

/* ---- library ---------------------------------------------------------- */
const char* jb_last_error(void);
int jb_abi_version(void);
/* Number of SMs of `device` (grids are sized in multiples of it). */
int jb_sm_count(int device, int32_t* out);

/* ---- data model -------------------------------------------------------- */

/* Row squared norms in A1 order: out[i] = einsum("nd,nd->n", x, x)[i].
 * Replaces ExactDistances.__init__ xnorm (search.py:101),
 * ExactDistances.bind qnorm (search.py:113) and _PairwiseDistances norms
 * (build.py:120). */
int jb_row_sq_norms(const float* x, int64_t n, int32_t dims, float* out, void* stream);

/* Extension (no reference counterpart): int8 screen records for the exact search
 * (jb_search_args.screen). Record of row i (jb_screen_record_bytes(dims) bytes):
 * int8 codes b of x_i - center (per-row scale s = max|x_i - center| / 127, codes
 * zero-padded to a 16 B multiple), then f32 {s, |b|^2, eps, norms[i]} with
 * eps >= |s b - (x_i - center)|_2 (f64, rounded up). */
int32_t jb_screen_record_bytes(int32_t dims);
int jb_screen_records(const float* x, const float* norms, int64_t n, int32_t dims, const float* center,
                      uint8_t* out, void* stream);

/* Medoid: argmin_i ||x_i - mean||^2 in f64 (mean = sequential f64 row sum / n,
 * distance = 2-lane einsum order), lowest id on ties. Writes the index to
 * *out_host (synchronizes). Replaces graph.medoid (graph.py:159-171). */
int jb_medoid(const float* x, int64_t n, int32_t dims, int64_t* out_host, void* stream);

/* u8 element kind (ElementKind.U8, core.py:32-37): integer-exact row norms
 * sum(x*x) (core.py:162-166, search.py:94-96) and the medoid of u8 rows (the
 * reference's f64 path on x.astype(f64): identical to jb_medoid on exact f32
 * copies of the rows, which this entry point makes on the device). */
int jb_row_sq_norms_u8(const uint8_t* x, int64_t n, int32_t dims, uint32_t* out, void* stream);
int jb_medoid_u8(const uint8_t* x, int64_t n, int32_t dims, int64_t* out_host, void* stream);
/* u8 rows -> exact f32 copy (for the f64 ground truth / medoid paths). */
int jb_u8_to_f32(const uint8_t* x, int64_t count, float* out, void* stream);

/* Element kinds of jb_insert_args.element_kind. */
#define JB_KIND_F32 0
#define JB_KIND_U8 1

/* ---- search (north-star 1) -------------------------------------------- */

/* Distance source of a search. */
#define JB_SRC_EXACT 0     /* ExactDistances over raw f32 rows (search.py:82-130) */
#define JB_SRC_RABITQ 1    /* RaBitQ estimator (rabitq.py:225-244), bit-exact      */
#define JB_SRC_RABITQ_FAST 2 /* RaBitQ: query quantized to 6-bit planes, <u,q> by
                              * AND + popcount over the code bit-planes (m = 1, 2, 4, 8;
                              * records from jb_rabitq_pack_planes) (north-star 2).
                              * Numerics differ from the reference estimator;
                              * validated by recall.                              */
#define JB_SRC_EXACT_U8 3  /* ExactDistances over u8 rows: integer distances
                              * ||x||^2 - 2<x,q> + ||q||^2 (search.py:92-99,
                              * 126-130), key word = the u32 distance            */

typedef struct jb_search_args {
    /* graph (GraphIndex, graph.py:36-99): fixed-stride int32 slab padded -1 */
    const int32_t* adjacency;      /* [capacity, degree_cap]                   */
    int32_t degree_cap;            /* R                                        */
    int64_t active_count;          /* vertices visible to the search           */
    /* distance source */
    int32_t source;                /* JB_SRC_*                                 */
    int32_t dims;                  /* D                                        */
    const float* data;             /* EXACT: [N, D] f32 rows                   */
    const float* data_norms;       /* EXACT: [N] A1 row norms                  */
    const uint8_t* records;        /* RABITQ: [N, record_bytes] packed records */
    int32_t record_bytes;          /* RABITQ: see jb_rabitq_pack_records        */
    int32_t bits;                  /* RABITQ: 1, 2, 4 or 8                      */
    /* queries */
    const float* queries;          /* EXACT: [nq, D] f32; RABITQ: rotated [nq, D] */
    const float* query_add;        /* EXACT: [nq] qnorm; RABITQ: [nq] query_add  */
    const float* query_sumq;       /* RABITQ: [nq] query_sumq; EXACT: unused     */
    int64_t nq;
    const int32_t* starts;         /* [nq] start vertices, or NULL => start_vertex */
    int64_t start_vertex;
    /* search parameters */
    int32_t beam_width;            /* L, 1..1024                               */
    int32_t hash_slots;            /* visited-table slots per query (pow2) or 0 = auto */
    int32_t trace_cap;             /* visited-trace capacity per query; 0 = no trace */
    /* outputs */
    uint64_t* frontier_keys;       /* [nq, L] ascending keys, UMAX padded      */
    int32_t* hops;                 /* [nq] SearchStats.hops                    */
    int32_t* evals;                /* [nq] device distance evaluations          */
    int32_t* trace_ids;            /* [nq, trace_cap] visited ids in hop order  */
    float* trace_dists;            /* [nq, trace_cap] their f32 distances       */
    int32_t* flags;                /* [nq] bit0: visited table overflowed (lossy) */
    /* EXACT_U8 source (the f32 data/queries fields are unused) */
    const uint8_t* data_u8;        /* [N, D] u8 rows                            */
    const uint32_t* norms_u32;     /* [N] integer row norms                     */
    const uint8_t* queries_u8;     /* [nq, D] u8 queries                        */
    const uint32_t* query_norms_u32; /* [nq] integer query norms                */
    /* Extension (EXACT source, not in the reference; NULL = off): int8 screen
     * records of the rows (jb_screen_records) and their centre. While the beam is
     * full, a new neighbour whose rigorous lower bound on the exact distance
     * (triangle inequality on int8-quantised centred rows, both quantisation
     * errors and the f32 rounding of the exact formula accounted for) exceeds the
     * beam's worst key is dropped without reading its f32 row: the merge would
     * drop its exact key too, so frontier, trace and evals are unchanged. */
    const uint8_t* screen;
    const float* screen_center;    /* [D] f32 centre the records were built with */
} jb_search_args;

/* Batched greedy beam search, one warp per query (persistent grid).
 * Replaces run_beam_searches/_run_lockstep (search.py:171-304). Frontier and
 * visited trace are identical to the reference's (same keys, same order). */
int jb_beam_search(const jb_search_args* args, void* stream);

/* Reference-defined distance-evaluation counts (SearchStats.distance_evals,
 * search.py:211-226): |{start} U N(u) for every expanded u| per query, from the
 * visited traces (trace_ids [nq, trace_cap], hops[q] <= trace_cap). Queries whose
 * flags bit 0 is clear (no visited-table eviction) keep evals[q] as given; with
 * flags NULL every query is recounted. Replaces the host recount of lossy queries. */
int jb_count_evals(const int32_t* adjacency, int32_t degree_cap, const int32_t* trace_ids, int32_t trace_cap,
                   const int32_t* hops, const int32_t* starts, int64_t start_vertex, const int32_t* flags, int64_t nq,
                   int32_t* evals, void* stream);

/* Top-k extraction from frontier keys: ids (int32, -1 padded) and dists (f64,
 * +inf padded). Replaces the exact-source branch of search_knn_batch
 * (search.py:366-383). */
int jb_frontier_topk(const uint64_t* frontier_keys, int64_t nq, int32_t beam_width, int32_t k,
                     int32_t* out_ids, double* out_dists, void* stream);
/* Same for integer (u8-source) keys: the key word is the u32 distance. */
int jb_frontier_topk_u8(const uint64_t* frontier_keys, int64_t nq, int32_t beam_width, int32_t k,
                        int32_t* out_ids, double* out_dists, void* stream);

/* Exact fp32 rerank of the full frontier: dist = einsum(x-q, x-q) (A1),
 * ordered by (dist, id), first k. Replaces _exact_rescore + lexsort
 * (search.py:318-320, 375-382). */
int jb_rerank_topk(const float* data, int32_t dims, const float* queries, int64_t nq,
                   const uint64_t* frontier_keys, int32_t beam_width, int32_t k,
                   int32_t* out_ids, double* out_dists, void* stream);

/* Host-buffer search: the whole search_knn_batch call (search.py:351-383) in
 * native code. `search` carries the graph and distance source (device pointers;
 * its query/output/trace fields are ignored). Queries are read from host memory,
 * (ids int32, dists f64) [nq, k] written to host memory (-1 / +inf padded), in
 * pipelined chunks over two streams (pinned staging, H2D, bind, search, rerank,
 * D2H). Returns after the results are in the caller's arrays. */
typedef struct jb_knn_plan {
    jb_search_args search;         /* graph + source + beam_width + hash_slots   */
    const float* centroid;         /* RABITQ: f32 [D] (device)                   */
    const double* rotation;        /* RABITQ: f64 [D, D] (device)                */
    const float* rerank_data;      /* f32 [N, D] rows for the exact rerank, or NULL
                                    * for the frontier's own top-k               */
    int32_t k;
    int32_t chunk;                 /* queries per pipeline chunk, 0 = auto       */
} jb_knn_plan;

int jb_search_knn_host(const jb_knn_plan* plan, const float* queries, int64_t nq,
                       int32_t* out_ids, double* out_dists, void* stream);

/* Same with HBM-resident queries [nq, D] and outputs [nq, k] (device pointers):
 * enqueues the chunks on the two lanes and makes `stream` wait for them. */
int jb_search_knn_device(const jb_knn_plan* plan, const float* queries, int64_t nq,
                         int32_t* out_ids, double* out_dists, void* stream);

/* ---- RaBitQ (north-star 2) --------------------------------------------- */

/* Packed device record of one vector: code bytes, zero padding to 16, then
 * (data_add, data_rescale) f32, total rounded up to 16 bytes (32 B at D=128, m=1). */
int32_t jb_rabitq_record_bytes(int32_t dims, int32_t bits);

/* Bit-plane records for the popcount estimator (JB_SRC_RABITQ_FAST, any m):
 * per vector m planes of ceil(D/32) words (rounded up to 4), plane b' bit e =
 * bit b' of the code of dimension e, then (data_add, data_rescale). For m = 1
 * the layout equals jb_rabitq_pack_records'. */
int32_t jb_rabitq_plane_record_bytes(int32_t dims, int32_t bits);
int jb_rabitq_pack_planes(const uint8_t* codes, const float* meta, int64_t n, int32_t dims, int32_t bits,
                          uint8_t* records, void* stream);

/* Build records from reference-layout codes [n, ceil(D*m/8)] and meta [n, 2].
 * (RaBitQIndex layout, rabitq.py:113-168). */
int jb_rabitq_pack_records(const uint8_t* codes, const float* meta, int64_t n, int32_t dims,
                           int32_t bits, uint8_t* records, void* stream);

/* Quantize rows: codes [n, ceil(D*m/8)] and meta [n, 2], bit-exact with
 * rabitq.fit's per-block math (rabitq.py:282-299) given the same centroid (f32)
 * and rotation (f64 [D, D], from the seed on the host). */
int jb_rabitq_encode(const float* x, int64_t n, int32_t dims, int32_t bits,
                     const float* centroid, const double* rotation,
                     uint8_t* codes, float* meta, void* stream);

/* Centroid: f32(sequential f64 column mean) (rabitq.py:273). */
int jb_column_mean_f32(const float* x, int64_t n, int32_t dims, float* out, void* stream);

/* Per-query prep (RaBitQIndex.bind, rabitq.py:170-181): rotated = f32(f64(q-c) @ rot^T),
 * query_add = A1 dot(q-c, q-c), query_sumq = f32(pairwise_sum_f32(rotated) * mid). */
int jb_rabitq_bind(const float* queries, int64_t nq, int32_t dims, int32_t bits,
                   const float* centroid, const double* rotation,
                   float* rotated, float* query_add, float* query_sumq, void* stream);

/* ---- construction / insertion (north-star 3) --------------------------- */

typedef struct jb_insert_args {
    /* graph, mutated in place on device */
    int32_t* adjacency;            /* [capacity, R] */
    int32_t* degrees;              /* [capacity]    */
    int32_t degree_cap;            /* R             */
    int64_t capacity;
    /* dataset (exact construction only) */
    const float* data;             /* [count, D]    */
    const float* data_norms;       /* [count]       */
    int32_t dims;
    int64_t count;
    /* BuildParams (build.py:35-62) */
    int32_t build_beam_width;
    double alpha;
    int32_t always_prune;
    int32_t reverse_all_visited;
    /* batch */
    int64_t start, stop;           /* new ids [start, stop); start == active_count */
    int64_t entry_point;           /* in: current entry point                */
    /* outputs (host) */
    int64_t* entry_point_out_host; /* entry point after the batch            */
    int64_t* bridges_out_host;     /* bridges added by connectivity repair   */
    int64_t* stats_out_host;       /* [8] work counters of the batch, added to
                                    * (may be NULL): [0] phase-1 hops, [1] phase-1
                                    * distance evals, [2] phase-2 prune candidates,
                                    * [3] phase-3 touched targets, [4] reverse
                                    * triples, [5] repair bridges, [6] stranded
                                    * rows through the tensor-core donor screen,
                                    * [7] of those rescanned exactly              */
    int64_t active_count;          /* jb_refine_batch: vertices visible to the
                                    * search (0 => stop); ignored elsewhere     */
    int32_t element_kind;          /* JB_KIND_F32 (data, data_norms) or
                                    * JB_KIND_U8 (data_u8, norms_u32)           */
    const uint8_t* data_u8;        /* [count, D] u8 rows                        */
    const uint32_t* norms_u32;     /* [count] integer row norms                 */
    /* quantized construction (build.py:105-111, 124-129; f32 rows only): every
     * construction distance is the RaBitQ estimate of a row's record against
     * the pivot's own row bound as a query (jb_rabitq_bind over the dataset) */
    int32_t quantized;             /* 0: exact distances; 1: RaBitQ estimates  */
    const uint8_t* records;        /* [count, record_bytes] packed records      */
    int32_t record_bytes;
    int32_t bits;                  /* 1, 2, 4 or 8                              */
    const float* bound_rotated;    /* [count, D] rows bound as queries          */
    const float* bound_qadd;       /* [count]                                   */
    const float* bound_qsumq;      /* [count]                                   */
    /* Extension (not in the reference; default 0 = the reference's exact repair):
     * > 0 makes connectivity repair take each stranded vertex's donors from the
     * frontier of a beam search of this width from the entry point (which only
     * reaches reachable vertices) instead of the exact scan over all reachable
     * rows (build.py:185-192), for 10M-row streaming. */
    int32_t repair_beam_width;
    /* Extension: per-vertex prune closure, [capacity] f64 on device (or NULL = off;
     * f32 builds only). closure[v] = alpha^2 of the robust prune that last wrote
     * v's row, 0 after an append or a bridge; the owner merge of a row closed at
     * alpha_a^2 <= alpha^2 only tests the pairs that involve its fresh sources
     * (same result). Must be zeroed whenever the adjacency is written outside
     * these calls (the Python GraphIndex does so on every host upload). */
    double* closure;
    /* Extension: int8 screen records of data (jb_screen_records) + centre for the
     * phase-1 exact search (jb_search_args.screen); NULL = off. */
    const uint8_t* screen;
    const float* screen_center;
} jb_insert_args;

/* One three-phase batch: search -> prune + reverse triples -> grouped merge,
 * then connectivity repair. On an empty graph (start == 0) the batch seeds it
 * by mutual pruning. Replaces batch_insert (build.py:296-348) with
 * _seed_batch (246-266), _merge_reverse_edges (269-293) and
 * _repair_connectivity (154-224). Synchronizes `stream`. */
int jb_batch_insert(const jb_insert_args* args, void* stream);

/* One batch of the two_pass refinement (_refine_pass, build.py:351-386): search
 * rows [start, stop) on the active graph (active_count vertices), prune each
 * vertex over its visited trace (itself excluded) plus the current neighbours
 * missing from the trace at the final alpha, rewrite its row, then the grouped
 * reverse-edge merge. The caller runs jb_repair_connectivity after the last
 * batch, as the reference does. Synchronizes `stream`. */
int jb_refine_batch(const jb_insert_args* args, void* stream);

/* Connectivity repair only (after the entry point moves, build.py:415-418). */
int jb_repair_connectivity(const jb_insert_args* args, void* stream);

/* Batched robust prune (graph.robust_prune, graph.py:174-228) of `count`
 * independent pivots: pivots[i] with candidates cand_ids/cand_dists[offsets[i]:offsets[i+1]]
 * (f32 distances to the pivot; any order). Kept ids/dists written to
 * out_ids/out_dists[i*degree_cap ...], out_counts[i] = number kept. */
int jb_robust_prune(const float* data, const float* data_norms, int32_t dims,
                    const int64_t* pivots, int64_t count, const int64_t* offsets,
                    const int32_t* cand_ids, const float* cand_dists,
                    double alpha, int32_t degree_cap,
                    int32_t* out_ids, float* out_dists, int32_t* out_counts, void* stream);

/* ---- distance-source protocol (search.py:82-168, rabitq.py:225-244) ------ */

/* `bind_distance_source(source, queries).distances(qrows, ids)` on the device:
 * out[i] = d(query qrows[i], vector ids[i]) for i < n, in the search kernel's
 * rounding. args: the source + bound-query fields of jb_search_args (source,
 * dims, data/data_norms | records/record_bytes/bits | data_u8/norms_u32,
 * queries/query_add/query_sumq | queries_u8/query_norms_u32); graph fields are
 * ignored. query_stride: elements between bound query rows (0 = dims); RABITQ
 * rows need a multiple of 4 floats and U8 rows a multiple of 16 bytes (16 B
 * aligned). out: f32 [n] (EXACT, RABITQ reference estimator) or u32 [n] (U8). */
int jb_bound_distances(const jb_search_args* args, int64_t query_stride, const int64_t* qrows,
                       const int64_t* ids, int64_t n, void* out, void* stream);

/* robust_prune (graph.py:174-228) of one candidate set given its pairwise
 * matrix dmat[i * n + j] = dist_fn(ids[i], [ids[j]]) (f64), candidate dists
 * to the pivot `dists` (f64) and ids (for the (dist, id) order): writes the
 * kept candidate POSITIONS in extraction order to out_pos[<= degree_cap] and
 * their number to *out_count (device). */
int jb_robust_prune_matrix(const double* dmat, const int64_t* ids, const double* dists, int32_t n,
                           double alpha, int32_t degree_cap, int32_t* out_pos, int32_t* out_count,
                           void* stream);

/* ---- measurement -------------------------------------------------------- */

/* Exact top-k in f64 (oracle.exact_knn, oracle.py:20-62): (dist, id) ascending. */
int jb_exact_knn(const float* data, int64_t n, int32_t dims, const float* queries, int64_t nq,
                 int32_t k, int32_t* out_ids, float* out_dists, void* stream);

/* exact_knn with a distance kind (oracle.py:20-62): inner_product = 0 ranks by
 * the squared Euclidean score above, 1 by -(q . x) (DistanceKind.INNER_PRODUCT,
 * oracle.py:53-54); ties by id. */
int jb_exact_knn_kind(const float* data, int64_t n, int32_t dims, const float* queries, int64_t nq, int32_t k,
                      int32_t inner_product, int32_t* out_ids, float* out_dists, void* stream);

/* ---- MIPS reduction (core.py:169-206) ----------------------------------- */

/* mips_augment on the device: aug_data [n, dims+1] = [x, f32(sqrt(M^2 - ||x||^2))]
 * with M^2 the largest f64 row norm (numpy einsum order), aug_queries
 * [nq, dims+1] = [q, 0]; M^2 written to *max_sq_out_host. Synchronizes. */
int jb_mips_augment(const float* data, int64_t n, int32_t dims, const float* queries, int64_t nq,
                    float* aug_data, float* aug_queries, double* max_sq_out_host, void* stream);

/* ---- sharding (north-star 4) ------------------------------------------- */

/* Merge per-shard top-k lists gathered from `shards` ranks into a global top-k
 * by (dist, global id). in_ids/in_dists: [shards, nq, k] with shard-local ids;
 * id_offsets[s] converts to global ids. -1 ids are padding. */
int jb_merge_shard_topk(const int32_t* in_ids, const double* in_dists, int32_t shards, int64_t nq,
                        int32_t k, const int64_t* id_offsets_host, int64_t* out_ids,
                        double* out_dists, void* stream);

/* Exchange format of the sharded path: a shard's top-k (local int32 ids, f64
 * dists, [nq, k]) packed into 16-byte records {f64 dist, i64 global id}
 * (id + id_offset; -1 padding kept) so one all-gather moves ids and dists. */
int jb_pack_shard_topk(const int32_t* ids, const double* dists, int64_t nq, int32_t k, int64_t id_offset,
                       void* out_records, void* stream);

/* Global top-k by (dist, global id) from all-gathered records [shards, nq, k].
 * Stream-ordered: no allocation, no synchronization. */
int jb_merge_shard_records(const void* records, int32_t shards, int64_t nq, int32_t k, int64_t* out_ids,
                           double* out_dists, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* JASPER_B200_H */
