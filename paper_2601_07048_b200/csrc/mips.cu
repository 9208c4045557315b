// mips.cu — maximum-inner-product reduction to Euclidean search, on the device.
//
// Replaces `mips_augment` (core.py:169-206): data row x -> [x, sqrt(M^2 - ||x||^2)]
// with M^2 the largest f64 row norm, query row q -> [q, 0], so argmax <q, x> is
// argmin ||q' - x'||^2. Norms follow numpy's f64 einsum('nd,nd->n') order (2
// lanes, 8-element blocks visited as pairs 3,2,1,0, the tail forward), the max is
// exact, and the extra coordinate is f32(sqrt_rn(max(M^2 - n, 0))), as in the
// reference. The augmented rows are written straight into HBM ([n, D+1] f32).
#include <algorithm>
#include <cstring>
#include "common.cuh"
#include "runtime.cuh"

namespace jb {

__device__ __forceinline__ double f64_row_norm(const float* __restrict__ r, int D) {
    Acc2d acc; acc.zero();
    int e = 0;
    for (; e + 8 <= D; e += 8) {
#pragma unroll
        for (int i = 3; i >= 0; --i) {
            const double a0 = (double)r[e + 2 * i], a1 = (double)r[e + 2 * i + 1];
            acc.l0 = __dadd_rn(__dmul_rn(a0, a0), acc.l0);
            acc.l1 = __dadd_rn(__dmul_rn(a1, a1), acc.l1);
        }
    }
    for (; e < D; ++e) {
        const double a = (double)r[e];
        if (e & 1) acc.l1 = __dadd_rn(__dmul_rn(a, a), acc.l1);
        else acc.l0 = __dadd_rn(__dmul_rn(a, a), acc.l0);
    }
    return acc.reduce();
}

// norms[i] and the running max (non-negative doubles order like their bit patterns)
__global__ void mips_norms_kernel(const float* __restrict__ x, int64_t n, int D, double* __restrict__ norms,
                                  unsigned long long* __restrict__ max_bits) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long b = 0;
    if (i < n) {
        const double s = f64_row_norm(x + i * D, D);
        norms[i] = s;
        b = (unsigned long long)__double_as_longlong(s);
    }
    for (int o = 16; o > 0; o >>= 1) b = max(b, __shfl_xor_sync(0xFFFFFFFFu, b, o));
    if ((threadIdx.x & 31) == 0) atomicMax(max_bits, b);
}

// one thread per output element of the augmented rows [n, D+1]
__global__ void mips_rows_kernel(const float* __restrict__ x, int64_t n, int D, const double* __restrict__ norms,
                                 const unsigned long long* __restrict__ max_bits, float* __restrict__ out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * (D + 1)) return;
    const int64_t i = t / (D + 1);
    const int e = (int)(t - i * (D + 1));
    if (e < D) {
        out[t] = x[i * D + e];
    } else if (norms != nullptr) {
        const double m2 = __longlong_as_double((long long)*max_bits);
        const double r = __dsub_rn(m2, norms[i]);
        out[t] = __double2float_rn(__dsqrt_rn(r > 0.0 ? r : 0.0));
    } else {
        out[t] = 0.0f;  // query rows: [q, 0]
    }
}

}  // namespace jb

using namespace jb;

extern "C" int jb_mips_augment(const float* data, int64_t n, int32_t dims, const float* queries, int64_t nq,
                               float* aug_data, float* aug_queries, double* max_sq_out_host, void* stream) {
    JB_CHECK_ARG(n >= 1, "mips_augment requires non-empty data");
    JB_CHECK_ARG(dims >= 1 && nq >= 0, "mips_augment: bad shape");
    cudaStream_t st = as_stream(stream);
    Scratch norms, mx;
    JB_CUDA(norms.alloc(sizeof(double) * n, st));
    JB_CUDA(mx.alloc(sizeof(unsigned long long), st));
    JB_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(unsigned long long), st));
    mips_norms_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(data, n, dims, norms.as<double>(),
                                                                   mx.as<unsigned long long>());
    JB_LAUNCH_CHECK();
    const int64_t td = n * (dims + 1), tq = nq * (dims + 1);
    mips_rows_kernel<<<(unsigned)((td + 255) / 256), 256, 0, st>>>(data, n, dims, norms.as<double>(),
                                                                   mx.as<unsigned long long>(), aug_data);
    JB_LAUNCH_CHECK();
    if (nq > 0) {
        mips_rows_kernel<<<(unsigned)((tq + 255) / 256), 256, 0, st>>>(queries, nq, dims, nullptr, nullptr,
                                                                       aug_queries);
        JB_LAUNCH_CHECK();
    }
    unsigned long long hb = 0;
    JB_CUDA(cudaMemcpyAsync(&hb, mx.p, sizeof(hb), cudaMemcpyDeviceToHost, st));
    JB_CUDA(cudaStreamSynchronize(st));
    if (max_sq_out_host) std::memcpy(max_sq_out_host, &hb, sizeof(double));
    return JB_OK;
}
