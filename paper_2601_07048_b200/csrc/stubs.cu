// stubs.cu — entry points whose kernels land in later commits (return JB_EINVAL).
#include "runtime.cuh"
using namespace jb;
extern "C" {
int jb_exact_knn(const float*, int64_t, int32_t, const float*, int64_t, int32_t, int32_t*, float*, void*) {
    set_error("jb_exact_knn: not built yet"); return JB_EINVAL; }
}
