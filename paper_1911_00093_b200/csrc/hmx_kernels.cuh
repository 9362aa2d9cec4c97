#pragma once
#include <type_traits>

#include "hmx_internal.cuh"

namespace hmx {

// stage-1 segments [seg_begin, seg_begin + seg_count) (count < 0: to the end)
cudaError_t launch_stage1(const DevPlan& P, const double* x, cudaStream_t st,
                          const int* skip = nullptr, int seg_begin = 0, int seg_count = -1);
cudaError_t launch_stage2(const DevPlan& P, const double* x, const S2Out& out, cudaStream_t st,
                          bool pdl);
// once per plan: kernel attributes (shared-memory opt-in of the FP32 stage 2)
cudaError_t configure_kernels();
cudaError_t launch_gather_perm(const double* x, const int32_t* perm, double* xp, int n,
                               cudaStream_t st);
cudaError_t launch_probe(const DevPlan& P, const double* x, unsigned long long* first_bad,
                         cudaStream_t st);

}  // namespace hmx
