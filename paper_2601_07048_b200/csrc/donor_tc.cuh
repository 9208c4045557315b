// donor_tc.cuh — tensor-core screened donor scan (donor_tc.cu), called by the
// connectivity repair in build.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace jb {

// D % 4 == 0, D <= 128, the driver's tensor-map encoder available, JB_DONOR_TC != 0
bool donor_tc_supported(int D, int64_t n_rows);

// For every stranded x = lost[w]: the `fan` reachable (seen[r] != 0) vertices with
// the smallest reference keys (d(x, r), r) -> part[w * fan + j] (one slice, UMAX
// padded). Rows the screen could not certify are listed in redo[0 .. *nredo)
// (device) and their part rows are left unwritten: rescan them exactly.
int donor_scan_tc(const float* data, const float* norms, int D, const int32_t* adj, int R, const int32_t* seen,
                  int64_t n_rows, const int32_t* lost, int nlost, int fan, uint64_t* part, int32_t* redo, int* nredo,
                  cudaStream_t st);

// lost2[i] = lost[redo[i]]; then, after the exact scan of lost2 into `slices`
// partial lists part2, merge them into part rows redo[i].
int donor_redo_ids(const int32_t* lost, const int32_t* redo, int n2, int32_t* lost2, cudaStream_t st);
int donor_redo_merge(const uint64_t* part2, int slices, int n2, int fan, const int32_t* redo, uint64_t* part,
                     cudaStream_t st);

}  // namespace jb
