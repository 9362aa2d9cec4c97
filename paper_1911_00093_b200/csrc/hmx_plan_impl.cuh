// Host-side plan object shared by hmx_plan.cu (flattener, matvec C ABI) and
// hmx_solver.cu (BiCG-STAB).
#pragma once

#include <cuda_runtime.h>

#include <mutex>
#include <string>
#include <vector>

#include "hmx_gpu.h"
#include "hmx_kernels.cuh"

namespace hmx {

void set_error(const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define HMX_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, #call);  \
  } while (0)

// Restores the caller's current device on scope exit.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// BiCG-STAB device workspace (allocated on a plan's first solve).
struct Workspace {
  int64_t n = 0;
  double *b = nullptr, *x = nullptr, *r = nullptr, *rhat = nullptr, *p = nullptr, *v = nullptr,
         *s = nullptr, *t = nullptr, *y = nullptr, *orig = nullptr;
  double* sc = nullptr;    // device scalars
  double* h_sc = nullptr;  // pinned mirror (+ flags)
  int* flags = nullptr;    // non-finite flags of the solver's matvecs
  double* partials = nullptr;
  uint32_t* done = nullptr;
  int* stop = nullptr;      // solver decision word [stop, reason, iteration, spare]
  double* hist = nullptr;   // device residual history
  int hist_cap = 0;
  int grid = 0;
};

}  // namespace hmx

struct hmx_plan {
  std::mutex mu;
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t n = 0;
  int scheme = 0;
  hmx::DevPlan dp{};
  int s1_grid = 0;
  std::vector<void*> allocs;
  std::vector<void*> pinned;
  hmx::Workspace* ws = nullptr;
  hmx_plan_info info{};

  // per-matvec device buffers
  double* d_xin = nullptr;     // original-order input staging (n)
  double* d_xp = nullptr;      // permuted input (n)
  double* d_y = nullptr;       // output (n)
  int* d_nonfinite = nullptr;
  double* d_seg_dots = nullptr;  // 2 per stage-2 segment
  uint32_t* d_done = nullptr;
  double* d_dots = nullptr;      // 2 reduced dots
  unsigned long long* d_first_bad = nullptr;
  // pinned host staging
  int* h_flag = nullptr;
  // input of the most recent matvec (for the non-finite probe)
  const double* last_xp = nullptr;
  cudaEvent_t ev[8] = {};

  template <typename T>
  T* alloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    if (cudaMalloc(&p, count * sizeof(T)) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
};

namespace hmx {

// Enqueues y = A xp (both device, permuted order unless permute_out) on the
// plan's stream with the stage-2 epilogue options `out` (y/nonfinite filled
// in by the caller).
int enqueue_matvec(hmx_plan* p, const double* xp, const S2Out& out);

}  // namespace hmx
