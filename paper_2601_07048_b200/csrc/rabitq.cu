// rabitq.cu — RaBitQ quantization on sm_100a.
//
//  * jb_rabitq_encode   replaces the per-block body of rabitq.fit (rabitq.py:282-299)
//  * jb_rabitq_bind     replaces RaBitQIndex.bind (rabitq.py:170-181)
//  * jb_rabitq_pack_records builds the packed device record used by the search
//    estimator (rabitq.py:235-244): code bytes | zero pad to 16 | data_add, data_rescale
//    | pad to 16, so one vector is one aligned request (32 B at D=128, m=1).
//
// Bit-exactness: every f64 step follows the reference formula in the same
// operation order; the only order difference is the f64 rotation GEMM
// (OpenBLAS dgemm vs. a per-output warp reduction here). f64 rounding
// differences there sit ~29 bits below the f32 / code decision boundaries, so
// codes and metadata match bit-for-bit in practice; the tests assert it.
#include <algorithm>
#include "common.cuh"
#include "runtime.cuh"

namespace jb {

__host__ __device__ inline int code_bytes_of(int D, int bits) { return (D * bits + 7) / 8; }
__host__ __device__ inline int meta_off_of(int D, int bits) { return ((code_bytes_of(D, bits) + 15) / 16) * 16; }
__host__ __device__ inline int record_bytes_of(int D, int bits) { return ((meta_off_of(D, bits) + 8 + 15) / 16) * 16; }

__host__ __device__ inline int plane_words_of(int D) { return (((D + 31) / 32) + 3) & ~3; }
__host__ __device__ inline int plane_record_bytes_of(int D, int bits) {
    return ((bits * plane_words_of(D) * 4 + 8 + 15) / 16) * 16;
}

// Bit-plane records for the popcount estimator: plane b' word w bit i = bit b' of the
// code of dimension 32w + i; (data_add, data_rescale) after the planes. One thread per
// (vector, word).
__global__ void pack_planes_kernel(const uint8_t* __restrict__ codes, const float* __restrict__ meta, int64_t n, int D,
                                   int bits, int cb, int pw, int rb, uint8_t* __restrict__ rec) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * pw) return;
    const int64_t v = t / pw;
    const int w = (int)(t % pw);
    const uint8_t* c = codes + v * cb;
    uint32_t* out = reinterpret_cast<uint32_t*>(rec + v * rb);
    const uint32_t mask = (1u << bits) - 1u;
    for (int bp = 0; bp < bits; ++bp) {
        uint32_t word = 0;
        for (int i = 0; i < 32; ++i) {
            const int e = 32 * w + i;
            if (e >= D) break;
            const int off = e * bits;
            const uint32_t u = (c[off >> 3] >> (off & 7)) & mask;  // codes never straddle a byte
            word |= ((u >> bp) & 1u) << i;
        }
        out[bp * pw + w] = word;
    }
    if (w == 0) {
        *reinterpret_cast<float2*>(rec + v * rb + bits * pw * 4) = make_float2(meta[2 * v], meta[2 * v + 1]);
        for (int i = bits * pw * 4 + 8; i < rb; ++i) rec[v * rb + i] = 0;
    }
}

__global__ void pack_records_kernel(const uint8_t* __restrict__ codes, const float* __restrict__ meta, int64_t n,
                                    int cb, int moff, int rb, uint8_t* __restrict__ rec) {
    int64_t v = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (v >= n) return;
    const int lane = threadIdx.x & 31;
    uint8_t* r = rec + v * rb;
    for (int i = lane; i < rb; i += 32) {
        uint8_t b = 0;
        if (i < cb) b = codes[v * cb + i];
        r[i] = b;
    }
    __syncwarp();
    if (lane == 0) {
        float2 m = make_float2(meta[2 * v], meta[2 * v + 1]);
        *reinterpret_cast<float2*>(r + moff) = m;
    }
}

// ---- encode --------------------------------------------------------------
// Block = 4 warps handling TV vectors:
//   1. nres[v][d] = f64(f32(x - c)) / norm   (norm = sqrt(A1-f64 of resid))
//   2. o[v][i]    = sum_d nres[v][d] * rot[i][d]    (warp per output i, coalesced rot row)
//   3. per vector (warp): delta, codes, obar, <o, obar> (2-lane order), meta.
constexpr int ENC_WARPS = 4;

__device__ __forceinline__ double a1f64_self(const double* r, int D) {
    Acc2d acc; acc.zero();
    int e = 0;
    for (; e + 8 <= D; e += 8) {
#pragma unroll
        for (int i = 3; i >= 0; --i) {
            acc.l0 = __dadd_rn(__dmul_rn(r[e + 2 * i], r[e + 2 * i]), acc.l0);
            acc.l1 = __dadd_rn(__dmul_rn(r[e + 2 * i + 1], r[e + 2 * i + 1]), acc.l1);
        }
    }
    for (; e < D; ++e) {
        if (e & 1) acc.l1 = __dadd_rn(__dmul_rn(r[e], r[e]), acc.l1);
        else acc.l0 = __dadd_rn(__dmul_rn(r[e], r[e]), acc.l0);
    }
    return acc.reduce();
}

__global__ void __launch_bounds__(ENC_WARPS * 32)
encode_kernel(const float* __restrict__ x, int64_t n, int D, int bits, const float* __restrict__ centroid,
              const double* __restrict__ rot, int TV, uint8_t* __restrict__ codes, float* __restrict__ meta) {
    extern __shared__ __align__(16) double esh[];
    double* nres = esh;                      // [TV][D]
    double* o = esh + (size_t)TV * D;        // [TV][D]
    double* norms = o + (size_t)TV * D;      // [TV]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t v0 = (int64_t)blockIdx.x * TV;
    const int nv = (int)std::min<int64_t>(TV, n - v0);
    const int levels = (1 << bits) - 1;
    const double mid = levels / 2.0;

    // resid (f32 subtract, widened)
    for (int idx = threadIdx.x; idx < nv * D; idx += blockDim.x) {
        int v = idx / D, d = idx - v * D;
        nres[idx] = (double)__fsub_rn(x[(v0 + v) * D + d], centroid[d]);
    }
    __syncthreads();
    for (int v = warp; v < nv; v += ENC_WARPS) {
        if (lane == 0) norms[v] = __dsqrt_rn(a1f64_self(nres + (size_t)v * D, D));
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < nv * D; idx += blockDim.x) {
        int v = idx / D;
        double nr = norms[v];
        double safe = nr > 0.0 ? nr : 1.0;
        nres[idx] = __ddiv_rn(nres[idx], safe);
    }
    __syncthreads();
    // rotation: o[v][i] = sum_d nres[v][d] * rot[i][d]
    for (int i = warp; i < D; i += ENC_WARPS) {
        const double* rr = rot + (size_t)i * D;
        for (int vb = 0; vb < nv; vb += 8) {
            double s[8];
#pragma unroll
            for (int t = 0; t < 8; ++t) s[t] = 0.0;
            for (int d = lane; d < D; d += 32) {
                const double rv = __ldg(rr + d);
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    if (vb + t < nv) s[t] = fma(nres[(size_t)(vb + t) * D + d], rv, s[t]);
            }
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                double vsum = s[t];
                for (int off = 16; off > 0; off >>= 1) vsum += __shfl_xor_sync(0xFFFFFFFFu, vsum, off);
                if (lane == 0 && vb + t < nv) o[(size_t)(vb + t) * D + i] = vsum;
            }
        }
    }
    __syncthreads();
    // quantize per vector
    const int cb = (D * bits + 7) / 8;
    const int per = 8 / bits;
    for (int v = warp; v < nv; v += ENC_WARPS) {
        const double* ov = o + (size_t)v * D;
        double mx = 0.0;
        for (int d = lane; d < D; d += 32) mx = fmax(mx, fabs(ov[d]));
        for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, off));
        const double norm = norms[v];
        const bool nonzero = norm > 0.0;
        const double delta = __ddiv_rn(__dmul_rn(2.0, mx), (double)levels);
        const double sdelta = delta > 0.0 ? delta : 1.0;
        // codes -> reuse nres row as obar storage
        double* obar = nres + (size_t)v * D;
        uint8_t* crow = codes + (v0 + v) * cb;
        for (int byte = lane; byte < cb; byte += 32) {
            uint32_t packed = 0;
            for (int j = 0; j < per; ++j) {
                const int d = byte * per + j;
                uint32_t u = 0;
                if (d < D) {
                    if (nonzero) {
                        double t = rint(__dadd_rn(__ddiv_rn(ov[d], sdelta), mid));
                        t = t < 0.0 ? 0.0 : (t > (double)levels ? (double)levels : t);
                        u = (uint32_t)t;
                    } else {
                        u = 1u << (bits - 1);
                    }
                    obar[d] = __dmul_rn(sdelta, __dsub_rn((double)u, mid));
                }
                packed |= u << (bits * j);
            }
            crow[byte] = (uint8_t)packed;
        }
        __syncwarp();
        if (lane == 0) {
            Acc2d acc; acc.zero();
            int e = 0;
            for (; e + 8 <= D; e += 8) {
#pragma unroll
                for (int i = 3; i >= 0; --i) {
                    acc.l0 = __dadd_rn(__dmul_rn(ov[e + 2 * i], obar[e + 2 * i]), acc.l0);
                    acc.l1 = __dadd_rn(__dmul_rn(ov[e + 2 * i + 1], obar[e + 2 * i + 1]), acc.l1);
                }
            }
            for (; e < D; ++e) {
                if (e & 1) acc.l1 = __dadd_rn(__dmul_rn(ov[e], obar[e]), acc.l1);
                else acc.l0 = __dadd_rn(__dmul_rn(ov[e], obar[e]), acc.l0);
            }
            const double ip = acc.reduce();
            const bool ok = nonzero && (ip > 1e-12);
            const double rescale = ok ? __ddiv_rn(__dmul_rn(__dmul_rn(-2.0, norm), delta), ip) : 0.0;
            meta[2 * (v0 + v)] = __double2float_rn(nonzero ? __dmul_rn(norm, norm) : 0.0);
            meta[2 * (v0 + v) + 1] = __double2float_rn(rescale);
        }
    }
}

// ---- bind ----------------------------------------------------------------
// numpy pairwise summation for f32 (A2), n = row length, unit stride.
__device__ float pairwise_sum_f32(const float* a, int n) {
    if (n < 8) {
        float r = 0.0f;
        for (int i = 0; i < n; ++i) r = __fadd_rn(r, a[i]);
        return r;
    }
    if (n <= 128) {
        float r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] = __fadd_rn(r[j], a[i + j]);
        float res = __fadd_rn(__fadd_rn(__fadd_rn(r[0], r[1]), __fadd_rn(r[2], r[3])),
                              __fadd_rn(__fadd_rn(r[4], r[5]), __fadd_rn(r[6], r[7])));
        for (; i < n; ++i) res = __fadd_rn(res, a[i]);
        return res;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __fadd_rn(pairwise_sum_f32(a, n2), pairwise_sum_f32(a + n2, n - n2));
}

// rotated = f32(f64(q - c) @ rot^T) as a tiled f64 GEMM: 256 threads with TM x TM
// outputs each on a (16 TM) x (16 TM) tile, 16-wide k-steps through k-major smem
// tiles. TM = 2 for small D (many small blocks: a 5K-query lane still puts ~40
// warps on every SM), TM = 4 for large D (twice the FMAs per smem read). Every
// output is one sequential FMA chain over d = 0..D-1 (the order the tests pin
// against the reference's dgemm results).
constexpr int RK = 16;

template <int TM>
__global__ void __launch_bounds__(256)
rotate_gemm_kernel(const float* __restrict__ queries, int64_t nq, int D, const float* __restrict__ centroid,
                   const double* __restrict__ rot, float* __restrict__ rotated) {
    constexpr int RT = 16 * TM;
    __shared__ __align__(16) double As[RK][RT + 2];
    __shared__ __align__(16) double Bs[RK][RT + 2];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int64_t q0 = (int64_t)blockIdx.x * RT;
    const int o0 = blockIdx.y * RT;
    double acc[TM][TM];
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TM; ++b) acc[a][b] = 0.0;
    // each thread's slice elements of the next k-step are loaded into registers while
    // the current k-step is consumed (RT * RK / 256 = TM * TM elements of each operand)
    constexpr int PER = RT * RK / 256;
    double pa[PER], pb[PER];
    auto fetch = [&](int k0) {
#pragma unroll
        for (int h = 0; h < PER; ++h) {
            const int i = tid + 256 * h;
            const int r = i / RK, e = i % RK, d = k0 + e;
            double va = 0.0, vb = 0.0;
            if (d < D) {
                if (q0 + r < nq) va = (double)__fsub_rn(__ldg(queries + (q0 + r) * D + d), __ldg(centroid + d));
                if (o0 + r < D) vb = __ldg(rot + (size_t)(o0 + r) * D + d);
            }
            pa[h] = va;
            pb[h] = vb;
        }
    };
    fetch(0);
    for (int k0 = 0; k0 < D; k0 += RK) {
#pragma unroll
        for (int h = 0; h < PER; ++h) {
            const int i = tid + 256 * h;
            As[i % RK][i / RK] = pa[h];
            Bs[i % RK][i / RK] = pb[h];
        }
        __syncthreads();
        if (k0 + RK < D) fetch(k0 + RK);
#pragma unroll
        for (int e = 0; e < RK; ++e) {
            double av[TM], bv[TM];
#pragma unroll
            for (int h = 0; h < TM; h += 2) {
                const double2 a2 = *reinterpret_cast<const double2*>(&As[e][ty * TM + h]);
                const double2 b2 = *reinterpret_cast<const double2*>(&Bs[e][tx * TM + h]);
                av[h] = a2.x; av[h + 1] = a2.y;
                bv[h] = b2.x; bv[h + 1] = b2.y;
            }
#pragma unroll
            for (int a = 0; a < TM; ++a)
#pragma unroll
                for (int b = 0; b < TM; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < TM; ++a) {
        const int64_t q = q0 + ty * TM + a;
        if (q >= nq) continue;
#pragma unroll
        for (int b = 0; b < TM; ++b) {
            const int o = o0 + tx * TM + b;
            if (o < D) rotated[q * D + o] = __double2float_rn(acc[a][b]);
        }
    }
}

// Per query (one warp): query_add = A1 dot(q - c, q - c), query_sumq =
// f32(pairwise_sum_f32(rotated) * mid) — both sequential orders, done by lane 0.
__global__ void bind_finish_kernel(const float* __restrict__ queries, int64_t nq, int D, int bits,
                                   const float* __restrict__ centroid, const float* __restrict__ rotated,
                                   float* __restrict__ qadd, float* __restrict__ qsumq) {
    extern __shared__ __align__(16) float fsh[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t qi = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    if (qi >= nq) return;
    float* qc = fsh + (size_t)warp * ((D + 3) & ~3);
    for (int d = lane; d < D; d += 32) qc[d] = __fsub_rn(queries[qi * D + d], centroid[d]);
    __syncwarp();
    if (lane == 0) {
        qadd[qi] = a1_dot<false>(qc, qc, D);
        const float mid = (float)(((1 << bits) - 1) / 2.0);
        qsumq[qi] = __fmul_rn(pairwise_sum_f32(rotated + qi * D, D), mid);
    }
}

}  // namespace jb

using namespace jb;

extern "C" {

int32_t jb_rabitq_record_bytes(int32_t dims, int32_t bits) { return record_bytes_of(dims, bits); }
int32_t jb_rabitq_plane_record_bytes(int32_t dims, int32_t bits) { return plane_record_bytes_of(dims, bits); }

int jb_rabitq_pack_planes(const uint8_t* codes, const float* meta, int64_t n, int32_t dims, int32_t bits,
                          uint8_t* records, void* stream) {
    JB_CHECK_ARG(bits == 1 || bits == 2 || bits == 4 || bits == 8, "bits must be one of (1, 2, 4, 8)");
    JB_CHECK_ARG(dims >= 1, "dims must be >= 1");
    if (n == 0) return JB_OK;
    const int pw = plane_words_of(dims);
    const int64_t threads = n * pw;
    pack_planes_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, as_stream(stream)>>>(
        codes, meta, n, dims, bits, code_bytes_of(dims, bits), pw, plane_record_bytes_of(dims, bits), records);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

int jb_rabitq_pack_records(const uint8_t* codes, const float* meta, int64_t n, int32_t dims, int32_t bits,
                           uint8_t* records, void* stream) {
    JB_CHECK_ARG(bits == 1 || bits == 2 || bits == 4 || bits == 8, "bits must be one of (1, 2, 4, 8)");
    JB_CHECK_ARG(dims >= 1, "dims must be >= 1");
    if (n == 0) return JB_OK;
    const int wpb = 8;
    pack_records_kernel<<<(unsigned)((n + wpb - 1) / wpb), wpb * 32, 0, as_stream(stream)>>>(
        codes, meta, n, code_bytes_of(dims, bits), meta_off_of(dims, bits), record_bytes_of(dims, bits), records);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

int jb_rabitq_encode(const float* x, int64_t n, int32_t dims, int32_t bits, const float* centroid,
                     const double* rotation, uint8_t* codes, float* meta, void* stream) {
    JB_CHECK_ARG(bits == 1 || bits == 2 || bits == 4 || bits == 8, "bits must be one of (1, 2, 4, 8)");
    JB_CHECK_ARG(dims >= 1, "dims must be >= 1");
    if (n == 0) return JB_OK;
    const size_t budget = 200 * 1024;
    int TV = (int)std::min<size_t>(64, (budget - 64 * 8) / (size_t)(16 * dims));
    JB_CHECK_ARG(TV >= 1, "rabitq encode: dims %d too large for shared memory", dims);
    const size_t smem = (size_t)TV * dims * 16 + (size_t)TV * 8;
    cudaStream_t st = as_stream(stream);
    JB_CUDA_RC(grow_smem(encode_kernel, (int)smem));
    encode_kernel<<<(unsigned)((n + TV - 1) / TV), ENC_WARPS * 32, smem, st>>>(x, n, dims, bits, centroid, rotation,
                                                                               TV, codes, meta);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

int jb_rabitq_bind(const float* queries, int64_t nq, int32_t dims, int32_t bits, const float* centroid,
                   const double* rotation, float* rotated, float* query_add, float* query_sumq, void* stream) {
    JB_CHECK_ARG(bits == 1 || bits == 2 || bits == 4 || bits == 8, "bits must be one of (1, 2, 4, 8)");
    if (nq == 0) return JB_OK;
    cudaStream_t st = as_stream(stream);
    if (dims >= 256) {
        dim3 grid((unsigned)((nq + 63) / 64), (unsigned)((dims + 63) / 64));
        rotate_gemm_kernel<4><<<grid, 256, 0, st>>>(queries, nq, dims, centroid, rotation, rotated);
    } else {
        dim3 grid((unsigned)((nq + 31) / 32), (unsigned)((dims + 31) / 32));
        rotate_gemm_kernel<2><<<grid, 256, 0, st>>>(queries, nq, dims, centroid, rotation, rotated);
    }
    JB_LAUNCH_CHECK();
    const int wpb = 8;
    const size_t smem = (size_t)wpb * ((dims + 3) & ~3) * 4;
    JB_CUDA_RC(grow_smem(bind_finish_kernel, (int)smem));
    bind_finish_kernel<<<(unsigned)((nq + wpb - 1) / wpb), wpb * 32, smem, st>>>(queries, nq, dims, bits, centroid,
                                                                               rotated, query_add, query_sumq);
    JB_LAUNCH_CHECK();
    return JB_OK;
}

}  // extern "C"
