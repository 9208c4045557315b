// shard.cu — per-shard top-k exchange and merge (north-star 4).
//
// Each rank searches its own shard and produces a (dist, local id) top-k list
// per query, ascending by (dist, id). For the exchange the rank packs its list
// into 16-byte records {f64 dist, i64 global id} (global id = local id + the
// shard's offset, -1 padding kept), so ONE all-gather moves the whole exchange
// and the merge needs no offsets. After the all-gather every rank holds
// [shards, nq, k] records; the global top-k is the first k of their union by
// (dist, global id). One thread per query walks the S sorted lists. Nothing
// here synchronizes the stream or allocates.
#include "common.cuh"
#include "runtime.cuh"

namespace jb {

constexpr int MAX_SHARDS = 64;

struct ShardOffsets {
    int64_t v[MAX_SHARDS];
};

struct __align__(16) TopkRecord {
    double d;
    int64_t id;  // global id, -1 = padding
};

__global__ void pack_shard_topk_kernel(const int32_t* __restrict__ ids, const double* __restrict__ dists, int64_t n,
                                       int64_t offset, TopkRecord* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t id = ids[i];
    TopkRecord r;
    r.d = dists[i];
    r.id = id < 0 ? -1 : (int64_t)id + offset;
    out[i] = r;
}

// rec(s, q, j) -> (dist, global id); returns false for padding
template <bool PACKED>
struct ShardLists {
    const int32_t* ids;
    const double* dists;
    const TopkRecord* recs;
    ShardOffsets offs;
    __device__ __forceinline__ bool get(int64_t o, int s, double& d, int64_t& gid) const {
        if (PACKED) {
            const TopkRecord r = recs[o];
            d = r.d;
            gid = r.id;
            return r.id >= 0;
        }
        const int32_t id = ids[o];
        if (id < 0) return false;
        d = dists[o];
        gid = (int64_t)id + offs.v[s];
        return true;
    }
};

template <bool PACKED>
__global__ void merge_shard_topk_kernel(ShardLists<PACKED> lists, int S, int64_t nq, int k,
                                        int64_t* __restrict__ out_ids, double* __restrict__ out_d) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    int pos[MAX_SHARDS];
    for (int s = 0; s < S; ++s) pos[s] = 0;
    for (int j = 0; j < k; ++j) {
        int best = -1;
        double bd = 0.0;
        int64_t bid = 0;
        for (int s = 0; s < S; ++s) {
            if (pos[s] >= k) continue;
            double d;
            int64_t gid;
            if (!lists.get(((int64_t)s * nq + q) * k + pos[s], s, d, gid)) continue;
            if (best < 0 || d < bd || (d == bd && gid < bid)) { best = s; bd = d; bid = gid; }
        }
        const int64_t w = q * k + j;
        if (best < 0) {
            out_ids[w] = -1;
            out_d[w] = __longlong_as_double(0x7FF0000000000000ll);
        } else {
            out_ids[w] = bid;
            out_d[w] = bd;
            ++pos[best];
        }
    }
}

}  // namespace jb

using namespace jb;

extern "C" int jb_merge_shard_topk(const int32_t* in_ids, const double* in_dists, int32_t shards, int64_t nq, int32_t k,
                                   const int64_t* id_offsets_host, int64_t* out_ids, double* out_dists, void* stream) {
    JB_CHECK_ARG(shards >= 1 && shards <= MAX_SHARDS, "shards must be in [1, %d]", MAX_SHARDS);
    JB_CHECK_ARG(k >= 1, "k must be >= 1");
    if (nq == 0) return JB_OK;
    ShardLists<false> lists{in_ids, in_dists, nullptr, {}};
    for (int s = 0; s < shards; ++s) lists.offs.v[s] = id_offsets_host[s];  // kernel parameter: no copy, no sync
    merge_shard_topk_kernel<false><<<(unsigned)((nq + 127) / 128), 128, 0, as_stream(stream)>>>(
        lists, shards, nq, k, out_ids, out_dists);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

extern "C" int jb_pack_shard_topk(const int32_t* ids, const double* dists, int64_t nq, int32_t k, int64_t id_offset,
                                  void* out_records, void* stream) {
    JB_CHECK_ARG(k >= 1, "k must be >= 1");
    const int64_t n = nq * k;
    if (n == 0) return JB_OK;
    pack_shard_topk_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
        ids, dists, n, id_offset, reinterpret_cast<TopkRecord*>(out_records));
    JB_LAUNCH_CHECK();
    return JB_OK;
}

extern "C" int jb_merge_shard_records(const void* records, int32_t shards, int64_t nq, int32_t k, int64_t* out_ids,
                                      double* out_dists, void* stream) {
    JB_CHECK_ARG(shards >= 1 && shards <= MAX_SHARDS, "shards must be in [1, %d]", MAX_SHARDS);
    JB_CHECK_ARG(k >= 1, "k must be >= 1");
    if (nq == 0) return JB_OK;
    ShardLists<true> lists{nullptr, nullptr, reinterpret_cast<const TopkRecord*>(records), {}};
    merge_shard_topk_kernel<true><<<(unsigned)((nq + 127) / 128), 128, 0, as_stream(stream)>>>(
        lists, shards, nq, k, out_ids, out_dists);
    JB_LAUNCH_CHECK();
    return JB_OK;
}
