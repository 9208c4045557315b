// screen.cu — int8 screen records for the exact-row beam search (extension).
//
// The exact search (search.cu, jb_search_args.screen) evaluates every new
// neighbour's f32 row in the reference's A1 order (search.py:101-113), but once
// the beam is full most of them (~80% in the build's phase-1 searches) are worse
// than its worst key and the merge drops them. A record of int8 codes of the
// centred row lets the kernel prove that first from 144 B instead of 512 B
// (D = 128): with x~ = s b, q~ = s_q a and eps >= |x~ - (x - c)|, eps_q >= |q~ - (q - c)|,
//   |q - x| >= |q~ - x~| - eps - eps_q,   |q~ - x~|^2 = s_q^2 |a|^2 + s^2 |b|^2 - 2 s_q s <a, b>
// (<a, b> exact in integers, dp4a). Dropped neighbours never touch the frontier,
// the trace or the stats, so the search stays identical to the reference's.
#include <algorithm>
#include <cmath>
#include "common.cuh"
#include "runtime.cuh"

namespace jb {

// one warp per row: centred row in f64, per-row scale, codes, |b|^2, eps (f64, up)
__global__ void screen_records_kernel(const float* __restrict__ x, const float* __restrict__ norms, int64_t n, int D,
                                      const float* __restrict__ center, uint8_t* __restrict__ out, int rb) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int dp = rb - 16;
    for (int64_t i = w; i < n; i += nw) {
        const float* r = x + i * D;
        double mx = 0.0;
        for (int e = lane; e < D; e += 32) mx = fmax(mx, fabs((double)r[e] - (double)center[e]));
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
        const float s = mx > 0.0 ? (float)(mx / 127.0) : 1.0f;
        uint8_t* rec = out + i * (int64_t)rb;
        double err = 0.0, nrm = 0.0;
        int bb = 0;
        for (int e = lane; e < dp; e += 32) {
            int b = 0;
            if (e < D) {
                const double xc = (double)r[e] - (double)center[e];
                b = (int)rint(xc / (double)s);
                b = b > 127 ? 127 : (b < -127 ? -127 : b);
                const double t = (double)s * (double)b - xc;
                err += t * t;
                nrm += fabs((double)r[e]) + fabs((double)center[e]);
            }
            bb += b * b;
            rec[e] = (uint8_t)(int8_t)b;
        }
        for (int o = 16; o > 0; o >>= 1) {
            err += __shfl_xor_sync(0xFFFFFFFFu, err, o);
            nrm += __shfl_xor_sync(0xFFFFFFFFu, nrm, o);
            bb += __shfl_xor_sync(0xFFFFFFFFu, bb, o);
        }
        if (lane == 0) {
            // f64 roundings of the residuals are ~2^-52 of the operands: a 2^-30
            // relative and a 2^-30 x sum|operand| absolute slack cover them
            const double eps = sqrt(err) * (1.0 + 0x1p-30) + 0x1p-30 * nrm;
            float* meta = reinterpret_cast<float*>(rec + dp);
            meta[0] = s;
            meta[1] = (float)bb;  // exact: |b|^2 <= D * 127^2 < 2^24 for D <= 1040
            meta[2] = __double2float_ru(eps);
            meta[3] = norms[i];
        }
    }
}

}  // namespace jb

using namespace jb;

extern "C" int32_t jb_screen_record_bytes(int32_t dims) { return ((dims + 15) & ~15) + 16; }

extern "C" int jb_screen_records(const float* x, const float* norms, int64_t n, int32_t dims, const float* center,
                                 uint8_t* out, void* stream) {
    JB_CHECK_ARG(dims >= 1 && dims <= 1040 && n >= 0, "jb_screen_records: bad shape (dims in [1, 1040])");
    JB_CHECK_ARG(n == 0 || (x && norms && center && out), "jb_screen_records: null buffer");
    if (n == 0) return JB_OK;
    const int64_t blocks = std::min<int64_t>((n + 7) / 8, 148 * 16);
    screen_records_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(x, norms, n, dims, center, out,
                                                                           jb_screen_record_bytes(dims));
    JB_LAUNCH_CHECK();
    return JB_OK;
}
