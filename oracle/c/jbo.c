/* ORACLE — TEST INFRASTRUCTURE ONLY. Not part of the product.
 *
 * A plain-C, multi-threaded (OpenMP) restatement of the reference package
 * beamann's hot path (/root/reference/pkg/src/beamann), the same algorithm as
 * the numpy oracle (oracle/search.py, vamana.py), so that the CPU side of bench.py can build
 * and search a 1M-vector index on the host cores in minutes instead of days.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs load it; the
 * product (paper_2601_07048_b200) never does.
 *
 * Rounding is the reference's (numpy 2.x on x86-64), restated operation by
 * operation; compile with -ffp-contract=off (no FMA contraction):
 *   A1  f32 einsum('md,md->m'): 4 accumulator lanes (element e -> lane e % 4),
 *       multiply then add, each 16-element block visited as 4-wide vectors
 *       3,2,1,0, the tail forward, reduce (l0 + l1) + (l2 + l3).
 *   A1d f64 einsum: 2 lanes, 8-element blocks, vectors 3,2,1,0, reduce l0 + l1.
 *   A3  mean(axis=0) of f64 rows: sequential row sum, then / n.
 *
 * Functions and the reference lines they follow (pkg/src/beamann/...):
 *   jbo_row_norms        search.py:101,113 / build.py:120   einsum('nd,nd->n')
 *   exact distance       search.py:126-130                  max((xn - 2 dot) + qn, 0) in f32
 *   pair distance        build.py:120-134                   rows in the data role, pivot norm last
 *   rabitq estimate      rabitq.py:235-244                  qadd + add + rescale * (<u, q> - sumq), >= 0
 *   jbo_search           search.py:171-304                  lockstep beam search, keys search.py:139-156
 *   jbo_rerank_topk      search.py:318-320, 366-383         einsum(x - q, x - q), lexsort((ids, d))
 *   robust_prune         graph.py:174-228                   (dist, id) order, alpha^2 * d(s, c) > d(p, c)
 *   jbo_batch_insert     build.py:246-348                   seed batch, 3 phases, EdgeBuffer order build.py:65-102
 *   jbo_repair           build.py:137-224                   BFS, nearest-16 donors, ordered attach with pins
 *   jbo_medoid           graph.py:159-171                   f64 mean, f64 einsum, lowest id
 *   jbo_topk_rows        oracle.py:20-62                    stable argsort of a score row, first k
 *
 * Parity: tests/test_oracle_c.py pins every function to the live-reference
 * fixtures in tests/golden (the same ones the numpy oracle is pinned to) and
 * to the numpy oracle on random cases.
 */
#include <math.h>
#include <omp.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define UMAX 0xFFFFFFFFFFFFFFFFull

/* ------------------------------------------------------------------ */
/* arithmetic                                                          */

static inline float a1_dot(const float *a, const float *b, int D) {
    float l0 = 0.f, l1 = 0.f, l2 = 0.f, l3 = 0.f;
    int e = 0;
    for (; e + 16 <= D; e += 16) {
        for (int i = 3; i >= 0; --i) {
            const float *pa = a + e + 4 * i, *pb = b + e + 4 * i;
            l0 = pa[0] * pb[0] + l0;
            l1 = pa[1] * pb[1] + l1;
            l2 = pa[2] * pb[2] + l2;
            l3 = pa[3] * pb[3] + l3;
        }
    }
    for (; e < D; ++e) {
        float p = a[e] * b[e];
        switch (e & 3) {
            case 0: l0 = p + l0; break;
            case 1: l1 = p + l1; break;
            case 2: l2 = p + l2; break;
            default: l3 = p + l3; break;
        }
    }
    return (l0 + l1) + (l2 + l3);
}

/* four A1 dots against one shared row, interleaved for instruction-level parallelism;
 * each result has exactly a1_dot's operation order */
static inline void a1_dot4(const float *a0, const float *a1, const float *a2, const float *a3, const float *b, int D,
                           float out[4]) {
    float acc[4][4] = {{0.f}};
    const float *rows[4] = {a0, a1, a2, a3};
    int e = 0;
    for (; e + 16 <= D; e += 16) {
        for (int i = 3; i >= 0; --i) {
            const float *pb = b + e + 4 * i;
            for (int r = 0; r < 4; ++r) {
                const float *pa = rows[r] + e + 4 * i;
                for (int j = 0; j < 4; ++j) acc[r][j] = pa[j] * pb[j] + acc[r][j];
            }
        }
    }
    for (; e < D; ++e)
        for (int r = 0; r < 4; ++r) acc[r][e & 3] = rows[r][e] * b[e] + acc[r][e & 3];
    for (int r = 0; r < 4; ++r) out[r] = (acc[r][0] + acc[r][1]) + (acc[r][2] + acc[r][3]);
}

/* einsum over the direct difference (search.py:318-320) */
static inline float a1_dsq(const float *a, const float *b, int D) {
    float l0 = 0.f, l1 = 0.f, l2 = 0.f, l3 = 0.f;
    int e = 0;
    for (; e + 16 <= D; e += 16) {
        for (int i = 3; i >= 0; --i) {
            const float *pa = a + e + 4 * i, *pb = b + e + 4 * i;
            float d0 = pa[0] - pb[0], d1 = pa[1] - pb[1], d2 = pa[2] - pb[2], d3 = pa[3] - pb[3];
            l0 = d0 * d0 + l0;
            l1 = d1 * d1 + l1;
            l2 = d2 * d2 + l2;
            l3 = d3 * d3 + l3;
        }
    }
    for (; e < D; ++e) {
        float d = a[e] - b[e];
        float p = d * d;
        switch (e & 3) {
            case 0: l0 = p + l0; break;
            case 1: l1 = p + l1; break;
            case 2: l2 = p + l2; break;
            default: l3 = p + l3; break;
        }
    }
    return (l0 + l1) + (l2 + l3);
}

static inline double a1d_sq(const double *a, int D) {
    double l0 = 0.0, l1 = 0.0;
    int e = 0;
    for (; e + 8 <= D; e += 8) {
        for (int i = 3; i >= 0; --i) {
            const double *p = a + e + 2 * i;
            l0 = p[0] * p[0] + l0;
            l1 = p[1] * p[1] + l1;
        }
    }
    for (; e < D; ++e) {
        double p = a[e] * a[e];
        if (e & 1) l1 = p + l1; else l0 = p + l0;
    }
    return l0 + l1;
}

static inline float clamp0(float d) { return d > 0.f ? d : 0.f; }

/* search.py:126-130 / build.py:130-134: rows in the data role, query/pivot norm added last */
static inline float exact_from_dot(float xn, float dot, float qn) { return clamp0((xn - 2.0f * dot) + qn); }

static inline uint64_t pack_key(float d, uint32_t id) {
    union { float f; uint32_t u; } c;
    c.f = clamp0(d);
    return ((uint64_t)c.u << 32) | (uint64_t)id;
}

static inline double key_dist(uint64_t k) {
    union { float f; uint32_t u; } c;
    c.u = (uint32_t)(k >> 32);
    return (double)c.f;
}

/* ------------------------------------------------------------------ */
/* distance sources                                                    */

typedef struct {
    int kind; /* 0 exact f32, 1 rabitq */
    int D;
    const float *x, *xn;            /* exact: rows + A1 norms */
    const uint8_t *codes;           /* rabitq: packed codes [n, cb] */
    const float *meta;              /* rabitq: (add, rescale) [n, 2] */
    int bits, cb;
} Source;

typedef struct {
    const float *q; /* exact: the query row; rabitq: the rotated query */
    float qn;       /* exact: query norm; rabitq: qadd */
    float sumq;     /* rabitq */
} Bound;

/* byte -> its `8 / m` code values as f32 (rabitq.py:90-101, LSB-first), m = 1, 2, 4, 8 */
static float UNPACK_LUT[9][256][8];

__attribute__((constructor)) static void init_unpack_lut(void) {
    for (int m = 1; m <= 8; m <<= 1)
        for (int b = 0; b < 256; ++b)
            for (int t = 0; t < 8 / m; ++t) UNPACK_LUT[m][b][t] = (float)((b >> (m * t)) & ((1 << m) - 1));
}

/* the unpacked f32 code row u[0, D) (zero-padded to a whole byte) */
static inline void rabitq_unpack(const Source *s, int64_t id, float *u) {
    const uint8_t *c = s->codes + id * (int64_t)s->cb;
    const int m = s->bits, per = 8 / m;
    for (int bi = 0; bi < s->cb; ++bi) memcpy(u + bi * per, UNPACK_LUT[m][c[bi]], sizeof(float) * (size_t)per);
}

static inline float rabitq_dot(const Source *s, int64_t id, const float *rq) {
    /* unpack to f32 and einsum with the rotated query (A1) */
    float u[4096 + 8];
    rabitq_unpack(s, id, u);
    return a1_dot(u, rq, s->D);
}

static inline float src_dist(const Source *s, const Bound *b, int64_t id) {
    if (s->kind == 0) return exact_from_dot(s->xn[id], a1_dot(s->x + id * (int64_t)s->D, b->q, s->D), b->qn);
    float dot = rabitq_dot(s, id, b->q);
    float est = (b->qn + s->meta[2 * id]) + s->meta[2 * id + 1] * (dot - b->sumq);
    return clamp0(est);
}

/* build.py:120-134: dist(pivot, id) with the row in the data role */
static inline float pair_dist(const float *x, const float *xn, int D, int64_t pivot, int64_t id) {
    return exact_from_dot(xn[id], a1_dot(x + id * (int64_t)D, x + pivot * (int64_t)D, D), xn[pivot]);
}

/* out[j] = dist(pivot, ids[j]) for j < n, four at a time */
static inline void pair_dists(const float *x, const float *xn, int D, int64_t pivot, const int64_t *ids, int64_t n,
                              int64_t stride, float *out) {
    const float *pv = x + pivot * (int64_t)D;
    int64_t j = 0;
    for (; j + 4 <= n; j += 4) {
        float d4[4];
        int64_t i0 = ids[j * stride], i1 = ids[(j + 1) * stride], i2 = ids[(j + 2) * stride],
                i3 = ids[(j + 3) * stride];
        a1_dot4(x + i0 * D, x + i1 * D, x + i2 * D, x + i3 * D, pv, D, d4);
        out[j] = exact_from_dot(xn[i0], d4[0], xn[pivot]);
        out[j + 1] = exact_from_dot(xn[i1], d4[1], xn[pivot]);
        out[j + 2] = exact_from_dot(xn[i2], d4[2], xn[pivot]);
        out[j + 3] = exact_from_dot(xn[i3], d4[3], xn[pivot]);
    }
    for (; j < n; ++j) out[j] = pair_dist(x, xn, D, pivot, ids[j * stride]);
}

/* ------------------------------------------------------------------ */
/* lockstep beam search for one query (search.py:171-269)               */

typedef struct {
    uint32_t *stamp; /* visited epochs, one per vertex */
    uint32_t epoch;
    int64_t cap;
    uint64_t *beam, *cand;
    uint8_t *done;
    uint64_t *trace;
    int64_t trace_n, trace_cap;
} Scratch;

static void scratch_init(Scratch *w, int64_t n, int L, int R) {
    w->stamp = (uint32_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(uint32_t));
    w->epoch = 0;
    w->cap = n;
    w->beam = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(L + R + 1));
    w->cand = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)(R + 1));
    w->done = (uint8_t *)malloc((size_t)(L + R + 1));
    w->trace_cap = 256;
    w->trace = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)w->trace_cap);
    w->trace_n = 0;
}

static void scratch_free(Scratch *w) {
    free(w->stamp); free(w->beam); free(w->cand); free(w->done); free(w->trace);
}

static inline void next_epoch(Scratch *w) {
    if (++w->epoch == 0) {
        memset(w->stamp, 0, sizeof(uint32_t) * (size_t)w->cap);
        w->epoch = 1;
    }
}

static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : x > y;
}

/* Returns the number of valid beam keys; beam holds them sorted, trace the
 * expanded keys in order when want_trace. */
static int search_one(const int32_t *adj, int R, int64_t active, const Source *s, const Bound *b, int64_t start,
                      int L, Scratch *w, int want_trace, int64_t *hops_out, int64_t *evals_out) {
    next_epoch(w);
    uint64_t *beam = w->beam, *cand = w->cand;
    uint8_t *done = w->done;
    int n = 1;
    beam[0] = pack_key(src_dist(s, b, start), (uint32_t)start);
    done[0] = 0;
    w->stamp[start] = w->epoch;
    int64_t hops = 0, evals = 1;
    w->trace_n = 0;
    int cursor = 0; /* every slot before cursor is expanded */
    for (;;) {
        while (cursor < n && done[cursor]) ++cursor;
        if (cursor >= n) break;
        uint64_t k = beam[cursor];
        done[cursor] = 1;
        ++hops;
        if (want_trace) {
            if (w->trace_n == w->trace_cap) {
                w->trace_cap *= 2;
                w->trace = (uint64_t *)realloc(w->trace, sizeof(uint64_t) * (size_t)w->trace_cap);
            }
            w->trace[w->trace_n++] = k;
        }
        const int32_t *row = adj + (int64_t)(uint32_t)(k & 0xFFFFFFFFu) * R;
        int nc = 0;
        /* claim the fresh neighbours first and prefetch their rows (memory-level
         * parallelism; the evaluation order below is unchanged) */
        for (int r = 0; r < R; ++r) {
            int32_t v = row[r];
            if (v < 0 || w->stamp[v] == w->epoch) continue;
            w->stamp[v] = w->epoch;
            cand[nc++] = (uint64_t)(uint32_t)v;
            const char *p = s->kind == 0 ? (const char *)(s->x + (int64_t)v * s->D)
                                         : (const char *)(s->codes + (int64_t)v * s->cb);
            const int nbytes = s->kind == 0 ? 4 * s->D : s->cb;
            for (int o = 0; o < nbytes; o += 64) __builtin_prefetch(p + o);
            if (s->kind == 1) __builtin_prefetch(s->meta + 2 * (int64_t)v);
        }
        int c = 0;
        if (s->kind == 1 && s->D <= 1024) {
            float u[4][1024 + 8], d4[4];
            for (; c + 4 <= nc; c += 4) {
                for (int r = 0; r < 4; ++r) rabitq_unpack(s, (uint32_t)cand[c + r], u[r]);
                a1_dot4(u[0], u[1], u[2], u[3], b->q, s->D, d4);
                for (int r = 0; r < 4; ++r) {
                    const uint32_t v = (uint32_t)cand[c + r];
                    const float est = (b->qn + s->meta[2 * (int64_t)v]) + s->meta[2 * (int64_t)v + 1] * (d4[r] - b->sumq);
                    cand[c + r] = pack_key(est, v);
                }
            }
        }
        if (s->kind == 0) {
            for (; c + 4 <= nc; c += 4) {
                float d4[4];
                const int64_t D = s->D;
                uint32_t v0 = (uint32_t)cand[c], v1 = (uint32_t)cand[c + 1], v2 = (uint32_t)cand[c + 2],
                         v3 = (uint32_t)cand[c + 3];
                a1_dot4(s->x + v0 * D, s->x + v1 * D, s->x + v2 * D, s->x + v3 * D, b->q, (int)D, d4);
                cand[c] = pack_key(exact_from_dot(s->xn[v0], d4[0], b->qn), v0);
                cand[c + 1] = pack_key(exact_from_dot(s->xn[v1], d4[1], b->qn), v1);
                cand[c + 2] = pack_key(exact_from_dot(s->xn[v2], d4[2], b->qn), v2);
                cand[c + 3] = pack_key(exact_from_dot(s->xn[v3], d4[3], b->qn), v3);
            }
        }
        for (; c < nc; ++c) {
            uint32_t v = (uint32_t)cand[c];
            cand[c] = pack_key(src_dist(s, b, v), v);
        }
        evals += nc;
        if (!nc) continue;
        /* insertion sort of the (<= R) new keys, then a stable merge truncated to L;
         * keys are unique (one per id), so stable == sorted */
        for (int i = 1; i < nc; ++i) {
            uint64_t t = cand[i];
            int j = i - 1;
            while (j >= 0 && cand[j] > t) { cand[j + 1] = cand[j]; --j; }
            cand[j + 1] = t;
        }
        int i = n - 1, j = nc - 1, o = n + nc - 1;
        int first_new = n + nc;
        while (j >= 0) {
            if (i >= 0 && beam[i] > cand[j]) { beam[o] = beam[i]; done[o] = done[i]; --i; }
            else { beam[o] = cand[j]; done[o] = 0; first_new = o; --j; }
            --o;
        }
        n += nc;
        if (n > L) n = L;
        if (first_new < cursor) cursor = first_new;
    }
    *hops_out = hops;
    *evals_out = evals;
    return n;
}

/* run_beam_searches over a bound source (search.py:272-304). out_keys [nq, L]
 * (UMAX padded), hops / evals per query. kind 0: q = queries, qv = query norms;
 * kind 1: q = rotated queries, qv = qadd, sumq. */
int jbo_search(const int32_t *adj, int R, int64_t active, int kind, const float *x, const float *xn,
               const uint8_t *codes, const float *meta, int bits, int D, const float *q, const float *qv,
               const float *sumq, int64_t nq, const int64_t *starts, int L, int threads, uint64_t *out_keys,
               int64_t *out_hops, int64_t *out_evals) {
    if (active <= 0) return -1;
    if (L < 1 || L > 1024) return -2;
    if (D > 4096) return -3;
    Source s = {kind, D, x, xn, codes, meta, bits, (D * bits + 7) / 8};
    int rc = 0;
#pragma omp parallel num_threads(threads > 0 ? threads : omp_get_max_threads())
    {
        Scratch w;
        scratch_init(&w, active, L, R);
#pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < nq; ++i) {
            if (starts[i] < 0 || starts[i] >= active) { rc = -4; continue; }
            Bound b = {q + i * (int64_t)D, qv[i], kind == 1 ? sumq[i] : 0.f};
            int64_t h, e;
            int n = search_one(adj, R, active, &s, &b, starts[i], L, &w, 0, &h, &e);
            uint64_t *o = out_keys + i * (int64_t)L;
            memcpy(o, w.beam, sizeof(uint64_t) * (size_t)n);
            for (int j = n; j < L; ++j) o[j] = UMAX;
            out_hops[i] = h;
            out_evals[i] = e;
        }
        scratch_free(&w);
    }
    return rc;
}

/* ------------------------------------------------------------------ */
/* exact rerank + top-k (search.py:318-320, 366-383)                   */

typedef struct { double d; int64_t id; } DI;

static int cmp_di(const void *a, const void *b) {
    const DI *x = (const DI *)a, *y = (const DI *)b;
    if (x->d < y->d) return -1;
    if (x->d > y->d) return 1;
    return (x->id > y->id) - (x->id < y->id);
}

int jbo_rerank_topk(const float *x, int D, const float *q, int64_t nq, const int32_t *fids, int L, int k,
                    int threads, int32_t *out_ids, double *out_d) {
#pragma omp parallel num_threads(threads > 0 ? threads : omp_get_max_threads())
    {
        DI *c = (DI *)malloc(sizeof(DI) * (size_t)L);
#pragma omp for schedule(dynamic, 16)
        for (int64_t i = 0; i < nq; ++i) {
            int n = 0;
            for (int j = 0; j < L; ++j) {
                int32_t id = fids[i * (int64_t)L + j];
                if (id < 0) continue;
                c[n].d = (double)a1_dsq(x + (int64_t)id * D, q + i * (int64_t)D, D);
                c[n].id = id;
                ++n;
            }
            qsort(c, (size_t)n, sizeof(DI), cmp_di);
            for (int j = 0; j < k; ++j) {
                out_ids[i * (int64_t)k + j] = j < n ? (int32_t)c[j].id : -1;
                out_d[i * (int64_t)k + j] = j < n ? c[j].d : INFINITY;
            }
        }
        free(c);
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* norms, medoid, ground-truth selection                                */

void jbo_row_norms(const float *x, int64_t n, int D, float *out, int threads) {
#pragma omp parallel for num_threads(threads > 0 ? threads : omp_get_max_threads()) schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = a1_dot(x + i * (int64_t)D, x + i * (int64_t)D, D);
}

/* graph.py:159-171: argmin of the f64 squared distance to the f64 mean (A3), lowest id */
int64_t jbo_medoid(const float *x, int64_t n, int D) {
    if (n <= 0 || D > 4096) return -1;
    double mean[4096], diff[4096];
    for (int d = 0; d < D; ++d) mean[d] = 0.0;
    for (int64_t i = 0; i < n; ++i)
        for (int d = 0; d < D; ++d) mean[d] += (double)x[i * (int64_t)D + d];
    for (int d = 0; d < D; ++d) mean[d] /= (double)n;
    int64_t best = 0;
    double bd = INFINITY;
    for (int64_t i = 0; i < n; ++i) {
        for (int d = 0; d < D; ++d) diff[d] = (double)x[i * (int64_t)D + d] - mean[d];
        double v = a1d_sq(diff, D);
        if (v < bd) { bd = v; best = i; }
    }
    return best;
}

/* oracle.py:20-62 tail: per row of a score matrix, the k smallest by (score, column)
 * (a stable argsort's first k). */
int jbo_topk_rows(const double *s, int64_t rows, int64_t cols, int k, int threads, int32_t *out_i, double *out_d) {
#pragma omp parallel num_threads(threads > 0 ? threads : omp_get_max_threads())
    {
        DI *h = (DI *)malloc(sizeof(DI) * (size_t)(k + 1));
#pragma omp for schedule(dynamic, 4)
        for (int64_t r = 0; r < rows; ++r) {
            const double *row = s + r * cols;
            int n = 0;
            for (int64_t c = 0; c < cols; ++c) {
                double v = row[c];
                if (n == k && !(v < h[k - 1].d)) continue; /* ties keep the earlier column */
                int j = n < k ? n++ : k - 1;
                while (j > 0 && h[j - 1].d > v) { h[j] = h[j - 1]; --j; }
                h[j].d = v;
                h[j].id = c;
            }
            for (int j = 0; j < k; ++j) {
                out_i[r * k + j] = j < n ? (int32_t)h[j].id : -1;
                out_d[r * k + j] = j < n ? h[j].d : INFINITY;
            }
        }
        free(h);
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* robust prune (graph.py:174-228)                                     */

typedef struct {
    const float *x, *xn;
    int D;
} Rows;

/* cands sorted in place by (d, id); writes the kept ids/dists, returns the count */
static int robust_prune(const Rows *rw, int64_t p, DI *c, int n, double a2, int R, int32_t *out_i, double *out_d) {
    (void)p;
    qsort(c, (size_t)n, sizeof(DI), cmp_di);
    int kept = 0, head = 0;
    while (head < n && kept < R) {
        int64_t s = c[head].id;
        out_i[kept] = (int32_t)s;
        if (out_d) out_d[kept] = c[head].d;
        ++kept;
        ++head;
        int m = head;
        float dd[4];
        int j = head;
        for (; j < n; j += 4) {
            int cntj = n - j < 4 ? n - j : 4;
            pair_dists(rw->x, rw->xn, rw->D, s, &c[j].id, cntj, 2, dd);
            for (int t = 0; t < cntj; ++t)
                if (a2 * (double)dd[t] > c[j + t].d) c[m++] = c[j + t];
        }
        n = m;
    }
    return kept;
}

/* ------------------------------------------------------------------ */
/* connectivity repair (build.py:137-224)                              */

typedef struct { int64_t u, x; } Pin;

typedef struct {
    int32_t *adj, *deg;
    int R;
    int64_t active, entry;
} G;

static void bfs_from(const G *g, uint8_t *seen, int64_t src, int64_t *queue) {
    int64_t qh = 0, qt = 0;
    queue[qt++] = src;
    seen[src] = 1;
    while (qh < qt) {
        int64_t u = queue[qh++];
        const int32_t *row = g->adj + u * g->R;
        for (int r = 0; r < g->R; ++r) {
            int32_t v = row[r];
            if (v >= 0 && !seen[v]) { seen[v] = 1; queue[qt++] = v; }
        }
    }
}

typedef struct { double best; int64_t x; int64_t donors[16]; int nd; } Stranded;

static int cmp_stranded(const void *a, const void *b) {
    const Stranded *p = (const Stranded *)a, *q = (const Stranded *)b;
    if (p->best < q->best) return -1;
    if (p->best > q->best) return 1;
    return (p->x > q->x) - (p->x < q->x);
}

static int64_t repair(G *g, const Rows *rw, int threads, Pin **pins, int64_t *npins, int64_t *pcap) {
    const int64_t n = g->active;
    if (n < 2) return 0;
    const int R = g->R, fan = R < 16 ? R : 16;
    int64_t added = 0;
    uint8_t *seen = (uint8_t *)malloc((size_t)n);
    int64_t *queue = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    int64_t *ok = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    for (;;) {
        memset(seen, 0, (size_t)n);
        bfs_from(g, seen, g->entry, queue);
        int64_t nl = 0, nok = 0;
        for (int64_t i = 0; i < n; ++i) {
            if (seen[i]) ok[nok++] = i; else ++nl;
        }
        if (!nl) break;
        Stranded *st = (Stranded *)malloc(sizeof(Stranded) * (size_t)nl);
        int64_t j = 0;
        for (int64_t i = 0; i < n; ++i)
            if (!seen[i]) st[j++].x = i;
        /* nearest reachable donors: the fan smallest (d(x, r), r) (argpartition + lexsort) */
#pragma omp parallel for num_threads(threads > 0 ? threads : omp_get_max_threads()) schedule(dynamic, 1)
        for (int64_t i = 0; i < nl; ++i) {
            int64_t x = st[i].x;
            DI top[17];
            int nt = 0;
            float d4[4];
            for (int64_t t0 = 0; t0 < nok; t0 += 4) {
                const int cnt = nok - t0 < 4 ? (int)(nok - t0) : 4;
                pair_dists(rw->x, rw->xn, rw->D, x, ok + t0, cnt, 1, d4);
                for (int u = 0; u < cnt; ++u) {
                    const double d = (double)d4[u];
                    const int64_t t = t0 + u;
                    if (nt == fan && !(d < top[fan - 1].d)) continue;
                    int q = nt < fan ? nt++ : fan - 1;
                    while (q > 0 && top[q - 1].d > d) { top[q] = top[q - 1]; --q; }
                    top[q].d = d;
                    top[q].id = ok[t];
                }
            }
            st[i].nd = nt;
            for (int q = 0; q < nt; ++q) st[i].donors[q] = top[q].id;
            st[i].best = top[0].d;
        }
        qsort(st, (size_t)nl, sizeof(Stranded), cmp_stranded);
        for (int64_t i = 0; i < nl; ++i) {
            int64_t x = st[i].x;
            if (seen[x]) continue;
            int placed = 0;
            for (int q = 0; q < st[i].nd && !placed; ++q) {
                int64_t u = st[i].donors[q];
                int32_t *row = g->adj + u * R;
                int d = g->deg[u];
                if (d >= R) {
                    /* evict the farthest non-pinned neighbour (first max of dist(u, ev)) */
                    int drop = -1;
                    double dmax = -1.0;
                    for (int r = 0; r < d; ++r) {
                        int pinned = 0;
                        for (int64_t pp = 0; pp < *npins; ++pp)
                            if ((*pins)[pp].u == u && (*pins)[pp].x == row[r]) { pinned = 1; break; }
                        if (pinned) continue;
                        double dd = (double)pair_dist(rw->x, rw->xn, rw->D, u, row[r]);
                        if (drop < 0 || dd > dmax) { dmax = dd; drop = r; }
                    }
                    if (drop < 0) continue; /* donor saturated with bridges */
                    for (int r = drop; r + 1 < d; ++r) row[r] = row[r + 1];
                    --d;
                }
                row[d++] = (int32_t)x;
                for (int r = d; r < R; ++r) row[r] = -1;
                g->deg[u] = d;
                if (*npins == *pcap) {
                    *pcap = *pcap ? 2 * *pcap : 64;
                    *pins = (Pin *)realloc(*pins, sizeof(Pin) * (size_t)*pcap);
                }
                (*pins)[(*npins)++] = (Pin){u, x};
                ++added;
                placed = 1;
            }
            if (!placed) {
                free(st); free(seen); free(queue); free(ok);
                return -(x + 1) - 1000000000000LL; /* "no donor for vertex x" */
            }
            bfs_from(g, seen, x, queue);
        }
        free(st);
    }
    free(seen); free(queue); free(ok);
    return added;
}

int64_t jbo_repair(int32_t *adj, int32_t *deg, int R, int64_t active, int64_t entry, const float *x,
                   const float *xn, int D, int threads) {
    G g = {adj, deg, R, active, entry};
    Rows rw = {x, xn, D};
    Pin *pins = NULL;
    int64_t np = 0, pc = 0;
    int64_t r = repair(&g, &rw, threads, &pins, &np, &pc);
    free(pins);
    return r;
}

/* ------------------------------------------------------------------ */
/* batch insert (build.py:246-348)                                     */

typedef struct { int64_t t; double d; int64_t s; } Triple;

static int cmp_triple(const void *a, const void *b) {
    const Triple *x = (const Triple *)a, *y = (const Triple *)b;
    if (x->t != y->t) return x->t < y->t ? -1 : 1;
    if (x->d < y->d) return -1;
    if (x->d > y->d) return 1;
    return (x->s > y->s) - (x->s < y->s);
}

static void put_row(G *g, int64_t u, const int32_t *ids, int n) {
    int32_t *row = g->adj + u * g->R;
    memcpy(row, ids, sizeof(int32_t) * (size_t)n);
    for (int r = n; r < g->R; ++r) row[r] = -1;
    g->deg[u] = n;
}

/* *active / *entry are in-out. seed_entry: the medoid of x[:stop] (used when the graph is
 * empty). Returns the repair bridge count, or < 0 on error. */
int64_t jbo_batch_insert(int32_t *adj, int32_t *deg, int R, int64_t *active, int64_t *entry, const float *x,
                         const float *xn, int D, int64_t start, int64_t stop, int L, double alpha,
                         int64_t seed_entry, int always_prune, int reverse_all, int threads) {
    if (start == stop) return 0;
    if (D > 4096) return -3;
    G g = {adj, deg, R, *active, *entry};
    Rows rw = {x, xn, D};
    const double a2 = alpha * alpha;
    const int nth = threads > 0 ? threads : omp_get_max_threads();
    const int64_t nb = stop - start;
    const int prof = getenv("JBO_PROFILE") != NULL;
    double t0 = omp_get_wtime(), t1 = t0, t2 = t0;
    if (g.active == 0) {
        /* seed batch (build.py:254-266): every vertex pruned over all the others */
        g.active = stop;
        g.entry = seed_entry;
        if (nb > 1) {
#pragma omp parallel num_threads(nth)
            {
                DI *c = (DI *)malloc(sizeof(DI) * (size_t)nb);
                int32_t *ki = (int32_t *)malloc(sizeof(int32_t) * (size_t)R);
#pragma omp for schedule(dynamic, 1)
                for (int64_t v = start; v < stop; ++v) {
                    int n = 0;
                    for (int64_t u = start; u < stop; ++u) {
                        if (u == v) continue;
                        c[n].id = u;
                        c[n].d = (double)pair_dist(x, xn, D, v, u);
                        ++n;
                    }
                    int k = robust_prune(&rw, v, c, n, a2, R, ki, NULL);
                    put_row(&g, v, ki, k);
                }
                free(c); free(ki);
            }
        }
    } else {
        /* phase 1 (build.py:310-326): search every new row on the current graph, with the
         * expansion trace; phase 2 (327-335): prune each over its trace, write its row and its
         * reverse-edge triples */
        const int64_t base_active = g.active;
        int64_t *tri_off = (int64_t *)calloc((size_t)nb + 1, sizeof(int64_t));
        Triple **tri = (Triple **)calloc((size_t)nb, sizeof(Triple *));
        int32_t *kept_rows = (int32_t *)malloc(sizeof(int32_t) * (size_t)nb * R);
        int *kept_n = (int *)malloc(sizeof(int) * (size_t)nb);
        Source s = {0, D, x, xn, NULL, NULL, 0, 0};
#pragma omp parallel num_threads(nth)
        {
            Scratch w;
            scratch_init(&w, base_active, L, R);
            DI *c = NULL;
            int64_t ccap = 0;
            double *kd = (double *)malloc(sizeof(double) * (size_t)R);
#pragma omp for schedule(dynamic, 4)
            for (int64_t i = 0; i < nb; ++i) {
                int64_t v = start + i;
                Bound b = {x + v * (int64_t)D, xn[v], 0.f};
                int64_t h, e;
                search_one(adj, R, base_active, &s, &b, g.entry, L, &w, 1, &h, &e);
                if (w.trace_n > ccap) {
                    ccap = w.trace_n;
                    c = (DI *)realloc(c, sizeof(DI) * (size_t)ccap);
                }
                for (int64_t t = 0; t < w.trace_n; ++t) {
                    c[t].id = (int64_t)(w.trace[t] & 0xFFFFFFFFu);
                    c[t].d = key_dist(w.trace[t]);
                }
                int n = (int)w.trace_n;
                int64_t ne = 0;
                Triple *tp = NULL;
                if (reverse_all) {
                    ne = n;
                    tp = (Triple *)malloc(sizeof(Triple) * (size_t)(ne ? ne : 1));
                    for (int t = 0; t < n; ++t) tp[t] = (Triple){c[t].id, c[t].d, v};
                }
                int k = robust_prune(&rw, v, c, n, a2, R, kept_rows + i * R, kd);
                kept_n[i] = k;
                if (!reverse_all) {
                    ne = k;
                    tp = (Triple *)malloc(sizeof(Triple) * (size_t)(ne ? ne : 1));
                    for (int t = 0; t < k; ++t) tp[t] = (Triple){kept_rows[i * R + t], kd[t], v};
                }
                tri[i] = tp;
                tri_off[i + 1] = ne;
            }
            free(c); free(kd);
            scratch_free(&w);
        }
        t1 = omp_get_wtime();
        g.active = stop;
        for (int64_t i = 0; i < nb; ++i) put_row(&g, start + i, kept_rows + i * R, kept_n[i]);
        for (int64_t i = 0; i < nb; ++i) tri_off[i + 1] += tri_off[i];
        const int64_t nt = tri_off[nb];
        Triple *all = (Triple *)malloc(sizeof(Triple) * (size_t)(nt ? nt : 1));
        for (int64_t i = 0; i < nb; ++i) {
            memcpy(all + tri_off[i], tri[i], sizeof(Triple) * (size_t)(tri_off[i + 1] - tri_off[i]));
            free(tri[i]);
        }
        free(tri); free(tri_off); free(kept_rows); free(kept_n);
        /* phase 3 (build.py:269-293, 336-347): EdgeBuffer order (target, dist, source),
         * one merge per target; a target's merge touches only its own row */
        /* bucket by target (counting sort), then each group sorted by (dist, source)
         * inside the parallel loop: the same order as one sort by (target, dist, source) */
        int64_t *cnt = (int64_t *)calloc((size_t)stop + 1, sizeof(int64_t));
        for (int64_t i = 0; i < nt; ++i) ++cnt[all[i].t + 1];
        for (int64_t t = 0; t < stop; ++t) cnt[t + 1] += cnt[t];
        Triple *sorted = (Triple *)malloc(sizeof(Triple) * (size_t)(nt ? nt : 1));
        {
            int64_t *pos = (int64_t *)malloc(sizeof(int64_t) * (size_t)(stop + 1));
            memcpy(pos, cnt, sizeof(int64_t) * (size_t)(stop + 1));
            for (int64_t i = 0; i < nt; ++i) sorted[pos[all[i].t]++] = all[i];
            free(pos);
        }
        free(all);
        all = sorted;
        int64_t ngroups = 0;
        int64_t *heads = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nt + 1));
        for (int64_t t = 0; t < stop; ++t)
            if (cnt[t + 1] > cnt[t]) heads[ngroups++] = cnt[t];
        heads[ngroups] = nt;
        free(cnt);
#pragma omp parallel num_threads(nth)
        {
            int64_t ccap = 0;
            DI *c = NULL;
            int32_t *ki = (int32_t *)malloc(sizeof(int32_t) * (size_t)R);
#pragma omp for schedule(dynamic, 16)
            for (int64_t gi = 0; gi < ngroups; ++gi) {
                const int64_t a = heads[gi], b = heads[gi + 1], t = all[a].t;
                qsort(all + a, (size_t)(b - a), sizeof(Triple), cmp_triple);
                int32_t *row = adj + t * R;
                const int have = deg[t];
                if (have + (b - a) > ccap) {
                    ccap = have + (b - a);
                    c = (DI *)realloc(c, sizeof(DI) * (size_t)ccap);
                }
                int nf = 0;
                for (int64_t j = a; j < b; ++j) {
                    int dup = 0;
                    for (int r = 0; r < have; ++r)
                        if (row[r] == all[j].s) { dup = 1; break; }
                    if (!dup) { c[have + nf].id = all[j].s; c[have + nf].d = all[j].d; ++nf; }
                }
                if (!nf) continue;
                if (!always_prune && have + nf <= R) {
                    for (int f = 0; f < nf; ++f) row[have + f] = (int32_t)c[have + f].id;
                    deg[t] = have + nf;
                    continue;
                }
                for (int r = 0; r < have; ++r) {
                    c[r].id = row[r];
                    c[r].d = (double)pair_dist(x, xn, D, t, row[r]);
                }
                int k = robust_prune(&rw, t, c, have + nf, a2, R, ki, NULL);
                put_row(&g, t, ki, k);
            }
            free(c); free(ki);
        }
        free(heads); free(all);
    }
    t2 = omp_get_wtime();
    Pin *pins = NULL;
    int64_t np = 0, pc = 0;
    int64_t r = repair(&g, &rw, nth, &pins, &np, &pc);
    free(pins);
    if (prof)
        fprintf(stderr, "[jbo] batch [%ld, %ld) search+prune %.3f s merge %.3f s repair %.3f s (%ld bridges)\n",
                (long)start, (long)stop, t1 - t0, t2 - t1, omp_get_wtime() - t2, (long)r);
    *active = g.active;
    *entry = g.entry;
    return r;
}

int jbo_num_threads(void) { return omp_get_max_threads(); }
