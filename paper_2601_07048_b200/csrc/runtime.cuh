// runtime.cuh — host-side error plumbing shared by every translation unit.
#pragma once
#include <cstdio>
#include <string>
#include <cuda_runtime.h>
#include "../../include/jasper_b200.h"

namespace jb {

void set_error(const char* fmt, ...);

#define JB_CHECK_ARG(cond, ...)                 \
    do {                                        \
        if (!(cond)) {                          \
            ::jb::set_error(__VA_ARGS__);       \
            return JB_EINVAL;                   \
        }                                       \
    } while (0)

#define JB_CUDA(expr)                                                                  \
    do {                                                                               \
        cudaError_t _e = (expr);                                                       \
        if (_e != cudaSuccess) {                                                       \
            ::jb::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,                 \
                            cudaGetErrorString(_e));                                   \
            return JB_ECUDA;                                                           \
        }                                                                              \
    } while (0)

#define JB_LAUNCH_CHECK() JB_CUDA(cudaGetLastError())

// propagate a JB_* status from a helper
#define JB_CUDA_RC(expr)            \
    do {                            \
        const int _rc = (expr);     \
        if (_rc != JB_OK) return _rc; \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count_current();

// Raise a kernel's dynamic smem limit to at least `bytes` on the current device.
// The limit is process-wide state of the kernel, so it only ever grows (under a
// lock): concurrent host threads launching the same kernel with different smem
// sizes cannot lower it under each other.
int grow_smem_attr(const void* func, int bytes);
template <class F>
inline int grow_smem(F* func, size_t bytes) { return grow_smem_attr(reinterpret_cast<const void*>(func), (int)bytes); }

// Once per device: keep freed stream-ordered memory in the default pool instead
// of returning it to the driver at every synchronization (the default release
// threshold 0 turned each launch's small scratch allocation into a ~0.5 ms remap).
void retain_pool_memory();

// Stream-ordered scratch that frees itself (cudaFreeAsync) on scope exit.
struct Scratch {
    void* p = nullptr;
    cudaStream_t s = nullptr;
    Scratch() = default;
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    cudaError_t alloc(size_t bytes, cudaStream_t st) {
        retain_pool_memory();
        s = st;
        if (bytes == 0) bytes = 16;
        return cudaMallocAsync(&p, bytes, st);
    }
    template <class T> T* as() const { return reinterpret_cast<T*>(p); }
    ~Scratch() { if (p) cudaFreeAsync(p, s); }
};

}  // namespace jb
