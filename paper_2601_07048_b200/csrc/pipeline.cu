// pipeline.cu — host-buffer search entry point (the C-ABI call a host binding makes).
//
// Replaces the reference's per-call path of `search_knn_batch`
// (search.py:351-383: bind the distance source, run the lockstep search, top-k
// or exact rerank) for callers that hold the queries and want the results in
// host memory. Everything between the two host arrays runs in native code:
//
//   chunk c (lane c % 2, one CUDA stream per lane):
//     host memcpy queries -> pinned staging      (CPU; overlaps chunk c-1 on the GPU;
//                                                 skipped when the caller's buffer is pinned)
//     H2D, bind (rotate GEMM + finish) or A1 query norms, beam search, rerank/top-k,
//     D2H ids + dists -> pinned, event
//   lane reuse / drain: event sync, pinned -> caller's arrays
//
// Two lanes let the search kernel of chunk c+1 fill the SMs freed by the tail of
// chunk c (each persistent grid is sized to its own chunk), and hide the host
// copies behind device work. Per-thread context (streams, events, pinned and
// device buffers) is cached and grown on demand, so concurrent host threads
// (the reference's run_queries thread pool, bench.py:69-91) never share state.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>
#include "runtime.cuh"

namespace jb {
namespace {

// Host memcpy split over a few persistent worker threads: one core copies ~17 GB/s,
// which alone would cost ~0.3 ms per 10K x 128 f32 query batch.
class CopyPool {
  public:
    explicit CopyPool(int workers) {
        for (int i = 0; i < workers; ++i) threads_.emplace_back([this, i] { run(i + 1); });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
    }
    void copy(void* dst, const void* src, size_t bytes) {
        const int parts = (int)threads_.size() + 1;
        if (bytes < ((size_t)256 << 10) || parts == 1) {
            std::memcpy(dst, src, bytes);
            return;
        }
        {
            std::lock_guard<std::mutex> g(mu_);
            dst_ = static_cast<char*>(dst);
            src_ = static_cast<const char*>(src);
            bytes_ = bytes;
            pending_ = parts - 1;
            ++gen_;
        }
        cv_.notify_all();
        part(0, parts);
        std::unique_lock<std::mutex> lk(mu_);
        done_.wait(lk, [this] { return pending_ == 0; });
    }

  private:
    void part(int i, int parts) {
        const size_t per = ((bytes_ + parts - 1) / parts + 63) & ~(size_t)63;
        const size_t lo = std::min(bytes_, per * i), hi = std::min(bytes_, lo + per);
        if (hi > lo) std::memcpy(dst_ + lo, src_ + lo, hi - lo);
    }
    void run(int i) {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
            }
            part(i, (int)threads_.size() + 1);
            {
                std::lock_guard<std::mutex> g(mu_);
                if (--pending_ == 0) done_.notify_one();
            }
        }
    }
    std::vector<std::thread> threads_;
    std::mutex mu_;
    std::condition_variable cv_, done_;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
    int pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// JB_PIPE_PROFILE=1: per-call host phase timings on stderr (tuning aid)
struct PhaseTimer {
    bool on = getenv("JB_PIPE_PROFILE") != nullptr;
    double t[5] = {0, 0, 0, 0, 0};  // copy-in, enqueue, wait, copy-out, total
    std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now(), t0 = last;
    void tick(int i) {
        if (!on) return;
        auto now = std::chrono::steady_clock::now();
        t[i] += std::chrono::duration<double, std::micro>(now - last).count();
        last = now;
    }
    void report() {
        if (!on) return;
        t[4] = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        fprintf(stderr, "[jb pipeline] copy-in %.0f us, enqueue %.0f us, wait %.0f us, copy-out %.0f us, total %.0f us\n",
                t[0], t[1], t[2], t[3], t[4]);
    }
};

int copy_workers() {
    const char* e = getenv("JB_COPY_THREADS");
    if (e) return std::max(0, atoi(e));
    const unsigned hc = std::thread::hardware_concurrency();
    return (int)std::min(3u, hc > 1 ? hc - 1 : 0u);
}

struct Lane {
    cudaStream_t s = nullptr;
    cudaEvent_t done = nullptr;
    float* h_q = nullptr;        // pinned [C, D]
    int32_t* h_ids = nullptr;    // pinned [C, k]
    double* h_d = nullptr;       // pinned [C, k]
    float* d_q = nullptr;        // [C, D]
    float* d_rot = nullptr;      // [C, D]
    float* d_qadd = nullptr;     // [C]
    float* d_sumq = nullptr;     // [C]
    uint64_t* d_fk = nullptr;    // [C, L]
    int32_t* d_ids = nullptr;    // [C, k]
    double* d_d = nullptr;       // [C, k]
    int64_t pend_q0 = -1, pend_m = 0;
    bool pend_direct = false;    // results went straight into the caller's pinned arrays
};

struct Ctx {
    int dev = -1;
    int64_t cap_q = 0, cap_qd = 0, cap_fk = 0, cap_k = 0;  // element capacities per lane
    Lane lane[2];
    cudaEvent_t start = nullptr;
    CopyPool* pool = nullptr;
    // thread exit: stop the copy workers (CUDA buffers are left to process teardown)
    ~Ctx() { delete pool; }

    void release_buffers() {
        for (Lane& l : lane) {
            cudaFreeHost(l.h_q); cudaFreeHost(l.h_ids); cudaFreeHost(l.h_d);
            cudaFree(l.d_q); cudaFree(l.d_rot); cudaFree(l.d_qadd); cudaFree(l.d_sumq);
            cudaFree(l.d_fk); cudaFree(l.d_ids); cudaFree(l.d_d);
            l.h_q = nullptr; l.h_ids = nullptr; l.h_d = nullptr;
            l.d_q = l.d_rot = l.d_qadd = l.d_sumq = nullptr;
            l.d_fk = nullptr; l.d_ids = nullptr; l.d_d = nullptr;
        }
        cap_q = cap_qd = cap_fk = cap_k = 0;
    }
};

thread_local Ctx g_ctx;

int ensure(Ctx& c, int64_t C, int D, int L, int k) {
    int dev = 0;
    JB_CUDA(cudaGetDevice(&dev));
    if (c.dev != dev) {
        if (c.dev >= 0) c.release_buffers();  // another device: drop the old context's buffers
        for (Lane& l : c.lane) {
            JB_CUDA(cudaStreamCreateWithFlags(&l.s, cudaStreamNonBlocking));
            JB_CUDA(cudaEventCreateWithFlags(&l.done, cudaEventDisableTiming));
        }
        JB_CUDA(cudaEventCreateWithFlags(&c.start, cudaEventDisableTiming));
        if (!c.pool) c.pool = new CopyPool(copy_workers());  // lives as long as the thread's context
        c.dev = dev;
    }
    const int64_t need_qd = C * D, need_fk = C * L, need_k = C * k;
    if (C <= c.cap_q && need_qd <= c.cap_qd && need_fk <= c.cap_fk && need_k <= c.cap_k) return JB_OK;
    for (Lane& l : c.lane) JB_CUDA(cudaStreamSynchronize(l.s));
    c.release_buffers();
    const int64_t cq = C, cqd = need_qd, cfk = need_fk, ck = need_k;
    for (Lane& l : c.lane) {
        JB_CUDA(cudaMallocHost(&l.h_q, sizeof(float) * cqd));
        JB_CUDA(cudaMallocHost(&l.h_ids, sizeof(int32_t) * ck));
        JB_CUDA(cudaMallocHost(&l.h_d, sizeof(double) * ck));
        JB_CUDA(cudaMalloc(&l.d_q, sizeof(float) * cqd));
        JB_CUDA(cudaMalloc(&l.d_rot, sizeof(float) * cqd));
        JB_CUDA(cudaMalloc(&l.d_qadd, sizeof(float) * cq));
        JB_CUDA(cudaMalloc(&l.d_sumq, sizeof(float) * cq));
        JB_CUDA(cudaMalloc(&l.d_fk, sizeof(uint64_t) * cfk));
        JB_CUDA(cudaMalloc(&l.d_ids, sizeof(int32_t) * ck));
        JB_CUDA(cudaMalloc(&l.d_d, sizeof(double) * ck));
    }
    c.cap_q = cq; c.cap_qd = cqd; c.cap_fk = cfk; c.cap_k = ck;
    return JB_OK;
}

// Wait for the lane's in-flight chunk and copy its results to the caller.
int drain(Ctx& c, Lane& l, int k, int32_t* out_ids, double* out_d, PhaseTimer& pt) {
    if (l.pend_q0 < 0) return JB_OK;
    pt.tick(1);
    JB_CUDA(cudaEventSynchronize(l.done));
    pt.tick(2);
    if (!l.pend_direct) {
        c.pool->copy(out_ids + l.pend_q0 * k, l.h_ids, sizeof(int32_t) * l.pend_m * k);
        c.pool->copy(out_d + l.pend_q0 * k, l.h_d, sizeof(double) * l.pend_m * k);
    }
    pt.tick(3);
    l.pend_q0 = -1;
    return JB_OK;
}

}  // namespace
}  // namespace jb

using namespace jb;

// Device work of one chunk on its lane: bind (or query norms), beam search,
// rerank / top-k into (ids, dists) — device pointers, `q` already in HBM.
static int run_chunk(const jb_knn_plan* plan, Lane& l, const float* q, int64_t m, int32_t* ids, double* dists) {
    const jb_search_args& base = plan->search;
    const int D = base.dims, L = base.beam_width, k = plan->k;
    jb_search_args a = base;
    int st;
    if (base.source != JB_SRC_EXACT) {
        st = jb_rabitq_bind(q, m, D, base.bits, plan->centroid, plan->rotation, l.d_rot, l.d_qadd, l.d_sumq, l.s);
        a.queries = l.d_rot;
        a.query_sumq = l.d_sumq;
    } else {
        st = jb_row_sq_norms(q, m, D, l.d_qadd, l.s);
        a.queries = q;
        a.query_sumq = nullptr;
    }
    if (st != JB_OK) return st;
    a.query_add = l.d_qadd;
    a.nq = m;
    a.starts = nullptr;
    a.trace_cap = 0;
    a.trace_ids = nullptr;
    a.trace_dists = nullptr;
    a.frontier_keys = l.d_fk;
    a.hops = a.evals = a.flags = nullptr;
    if ((st = jb_beam_search(&a, l.s)) != JB_OK) return st;
    if (plan->rerank_data) return jb_rerank_topk(plan->rerank_data, D, q, m, l.d_fk, L, k, ids, dists, l.s);
    return jb_frontier_topk(l.d_fk, m, L, k, ids, dists, l.s);
}

static int check_plan(const jb_knn_plan* plan) {
    JB_CHECK_ARG(plan != nullptr, "knn search: null plan");
    const jb_search_args& base = plan->search;
    JB_CHECK_ARG(base.dims >= 1, "dims must be >= 1");
    JB_CHECK_ARG(base.beam_width >= 1 && base.beam_width <= 1024, "beam_width must be in [1, 1024]");
    JB_CHECK_ARG(plan->k >= 1 && plan->k <= base.beam_width, "k must satisfy 1 <= k <= beam_width");
    JB_CHECK_ARG(base.source == JB_SRC_EXACT || (plan->centroid && plan->rotation),
                 "quantized source: centroid and rotation required");
    return JB_OK;
}

// Lanes start after everything already queued on the caller's stream (uploads, builds).
static int fork_lanes(Ctx& c, cudaStream_t caller) {
    JB_CUDA(cudaEventRecord(c.start, caller));
    for (Lane& l : c.lane) JB_CUDA(cudaStreamWaitEvent(l.s, c.start, 0));
    return JB_OK;
}

static int search_knn_host(const jb_knn_plan* plan, const float* queries, int64_t nq, int32_t* out_ids,
                           double* out_dists, void* stream) {
    int st = check_plan(plan);
    if (st != JB_OK || nq == 0) return st;
    JB_CHECK_ARG(queries && out_ids && out_dists, "jb_search_knn_host: null host buffer");
    const int D = plan->search.dims, L = plan->search.beam_width, k = plan->k;
    // chunks: two lanes, ~nq/2 each by default (concurrent kernels fill each other's tails)
    int64_t C = plan->chunk > 0 ? plan->chunk : std::max<int64_t>(1024, ((nq + 1) / 2 + 255) / 256 * 256);
    C = std::min<int64_t>(C, nq);
    Ctx& c = g_ctx;
    if ((st = ensure(c, C, D, L, k)) != JB_OK) return st;
    if ((st = fork_lanes(c, as_stream(stream))) != JB_OK) return st;

    // Queries already in page-locked memory (cudaHostAlloc / registered) are copied
    // to HBM straight from the caller's buffer; pageable ones go through staging.
    // Likewise results: page-locked output arrays receive the D2H copies directly.
    auto pinned = [](const void* p) {
        cudaPointerAttributes pa{};
        const bool r = cudaPointerGetAttributes(&pa, p) == cudaSuccess && pa.type == cudaMemoryTypeHost;
        cudaGetLastError();  // a pageable pointer may leave an error behind on older drivers
        return r;
    };
    const bool pinned_in = pinned(queries);
    const bool pinned_out = pinned(out_ids) && pinned(out_dists);

    PhaseTimer pt;
    int64_t chunk_i = 0;
    for (int64_t q0 = 0; q0 < nq; q0 += C, ++chunk_i) {
        Lane& l = c.lane[chunk_i & 1];
        const int64_t m = std::min<int64_t>(C, nq - q0);
        if ((st = drain(c, l, k, out_ids, out_dists, pt)) != JB_OK) return st;
        pt.tick(1);
        const float* src = queries + q0 * D;
        if (!pinned_in) {
            c.pool->copy(l.h_q, src, sizeof(float) * m * D);
            src = l.h_q;
        }
        pt.tick(0);
        JB_CUDA(cudaMemcpyAsync(l.d_q, src, sizeof(float) * m * D, cudaMemcpyHostToDevice, l.s));
        if ((st = run_chunk(plan, l, l.d_q, m, l.d_ids, l.d_d)) != JB_OK) return st;
        int32_t* hi = pinned_out ? out_ids + q0 * k : l.h_ids;
        double* hd = pinned_out ? out_dists + q0 * k : l.h_d;
        JB_CUDA(cudaMemcpyAsync(hi, l.d_ids, sizeof(int32_t) * m * k, cudaMemcpyDeviceToHost, l.s));
        JB_CUDA(cudaMemcpyAsync(hd, l.d_d, sizeof(double) * m * k, cudaMemcpyDeviceToHost, l.s));
        JB_CUDA(cudaEventRecord(l.done, l.s));
        l.pend_q0 = q0;
        l.pend_m = m;
        l.pend_direct = pinned_out;
    }
    for (int i = 0; i < 2; ++i) {
        // drain in submission order
        Lane& l = c.lane[(chunk_i + i) & 1];
        if ((st = drain(c, l, k, out_ids, out_dists, pt)) != JB_OK) return st;
    }
    pt.report();
    return JB_OK;
}

extern "C" int jb_search_knn_host(const jb_knn_plan* plan, const float* queries, int64_t nq, int32_t* out_ids,
                                  double* out_dists, void* stream) {
    const int st = search_knn_host(plan, queries, nq, out_ids, out_dists, stream);
    if (st != JB_OK) {
        // a failed call leaves no chunk pending for the next one
        for (Lane& l : g_ctx.lane) {
            if (l.s) cudaStreamSynchronize(l.s);
            l.pend_q0 = -1;
        }
    }
    return st;
}

// HBM-resident variant: queries and outputs are device arrays; the call only
// enqueues (two lanes, joined back into the caller's stream).
extern "C" int jb_search_knn_device(const jb_knn_plan* plan, const float* queries, int64_t nq, int32_t* out_ids,
                                    double* out_dists, void* stream) {
    int st = check_plan(plan);
    if (st != JB_OK || nq == 0) return st;
    const int D = plan->search.dims, L = plan->search.beam_width, k = plan->k;
    int64_t C = plan->chunk > 0 ? plan->chunk : (nq >= 2048 ? (nq + 1) / 2 : nq);
    C = std::min<int64_t>(C, nq);
    Ctx& c = g_ctx;
    if ((st = ensure(c, C, D, L, k)) != JB_OK) return st;
    cudaStream_t caller = as_stream(stream);
    if ((st = fork_lanes(c, caller)) != JB_OK) return st;
    int64_t chunk_i = 0;
    for (int64_t q0 = 0; q0 < nq; q0 += C, ++chunk_i) {
        Lane& l = c.lane[chunk_i & 1];
        const int64_t m = std::min<int64_t>(C, nq - q0);
        if ((st = run_chunk(plan, l, queries + q0 * D, m, out_ids + q0 * k, out_dists + q0 * k)) != JB_OK) return st;
        JB_CUDA(cudaEventRecord(l.done, l.s));
    }
    for (int i = 0; i < 2 && i < chunk_i; ++i) JB_CUDA(cudaStreamWaitEvent(caller, c.lane[i].done, 0));
    return JB_OK;
}
