// shard.cu — merge of per-shard top-k lists (north-star 4).
//
// After the NCCL all-gather every rank holds [shards, nq, k] (local id, dist)
// lists, each ascending by (dist, id). The global top-k is the first k of their
// union by (dist, global id); one thread per query walks the S sorted lists.
#include "common.cuh"
#include "runtime.cuh"

namespace jb {

constexpr int MAX_SHARDS = 64;

__global__ void merge_shard_topk_kernel(const int32_t* __restrict__ ids, const double* __restrict__ dists, int S,
                                        int64_t nq, int k, const int64_t* __restrict__ offs, int64_t* __restrict__ out_ids,
                                        double* __restrict__ out_d) {
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
            const int64_t o = ((int64_t)s * nq + q) * k + pos[s];
            const int32_t id = ids[o];
            if (id < 0) continue;
            const double d = dists[o];
            const int64_t gid = id + offs[s];
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
    cudaStream_t st = as_stream(stream);
    Scratch offs;
    JB_CUDA(offs.alloc(sizeof(int64_t) * shards, st));
    JB_CUDA(cudaMemcpyAsync(offs.p, id_offsets_host, sizeof(int64_t) * shards, cudaMemcpyHostToDevice, st));
    merge_shard_topk_kernel<<<(unsigned)((nq + 127) / 128), 128, 0, st>>>(in_ids, in_dists, shards, nq, k,
                                                                          offs.as<int64_t>(), out_ids, out_dists);
    JB_LAUNCH_CHECK();
    // offs is freed stream-ordered after the kernel; the host array must stay valid until then
    JB_CUDA(cudaStreamSynchronize(st));
    return JB_OK;
}
