// Host-side plan object shared by hmx_plan.cu (flattener, matvec C ABI) and
// hmx_solver.cu (BiCG-STAB).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
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

// NVTX range for the host-side phases (plan build, matvec call, solve,
// compression): free when no profiler is attached (nvtx3 is header-only and
// resolves its tool at run time), visible on nsys / ncu timelines otherwise.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

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
  int* ictl = nullptr;      // iteration control [i, max_iter, -, -]
  // graph-resident iteration loop (CUDA graph with a WHILE conditional node),
  // built on first use; rebuilt when the history buffer moves
  cudaGraph_t loop_graph = nullptr;
  cudaGraphExec_t loop_exec = nullptr;
  const double* loop_hist = nullptr;
  bool loop_failed = false;
  // (copied by value into solver contexts: the owner, hmx_plan_destroy,
  // releases the graph)
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
  // input of the most recent matvec (for the non-finite probe; the caller of
  // hmx_apply_local keeps it alive until hmx_nonfinite_block returns)
  const double* last_xp = nullptr;
  cudaEvent_t ev[8] = {};
  // end of the plan's most recent asynchronous work (any stream); see plan_enter
  cudaEvent_t ev_tail = nullptr;

  template <typename T>
  T* alloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    if (cudaMalloc(&p, count * sizeof(T)) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
};

// FP64 masters resident on a device (hmx_master_create / hmx_master_build).
// A plan's device work may be queued on several streams (its own, a caller's
// in hmx_apply_local / hmx_dist_matvec) and it shares per-plan scratch (z,
// chunk partials, arrival counters, flags).  Every entry point makes its
// stream wait for the plan's previous asynchronous work first (plan_enter);
// the asynchronous ones record their end (plan_leave).  The plan mutex orders
// the enqueues, these events order the device work.
inline cudaError_t plan_enter(hmx_plan* p, cudaStream_t st) {
  return p->ev_tail ? cudaStreamWaitEvent(st, p->ev_tail, 0) : cudaSuccess;
}
inline cudaError_t plan_leave(hmx_plan* p, cudaStream_t st) {
  return p->ev_tail ? cudaEventRecord(p->ev_tail, st) : cudaSuccess;
}

struct hmx_master {
  int device = 0;
  int64_t n = 0, nb = 0, n_data = 0, rank_sum = 0, max_rank = 0;
  cudaStream_t stream = nullptr;
  // host copies for the flattener
  std::vector<int64_t> perm, table, offset, rank, roff;
  std::vector<int32_t> kind;
  // device
  double* data = nullptr;
  int64_t* d_table = nullptr;
  int64_t* d_offset = nullptr;
  int64_t* d_rank = nullptr;
  int64_t* d_roff = nullptr;
  int32_t* d_kind = nullptr;
  std::vector<void*> allocs;

  template <typename T>
  T* alloc(size_t count) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
};

namespace hmx {

// Device-side payload source of hmx_plan_create_prepared: the resident FP64
// masters plus the per-rank scaling/classification computed on the device.
struct DevSource {
  const double* data = nullptr;     // masters (hmx_master_desc layout)
  const int64_t* table = nullptr;   // n_blocks x 5
  const int64_t* offset = nullptr;  // per block
  const int64_t* rank = nullptr;    // per block (full rank)
  const int64_t* roff = nullptr;    // per block: first rank slot (prefix of ranks)
  const int64_t* khi = nullptr;     // per block: FP64-class ranks
  const int32_t* cls_idx = nullptr; // per rank slot: original rank index, class order (hi, then lo)
  const double* colmag = nullptr;   // per rank slot (original order), nullptr = unscaled
  const double* rowmag = nullptr;
  unsigned long long* lost = nullptr;  // FP32 underflow counter
  long long* overflow = nullptr;       // first overflowing block (min)
};

// Pack program for the device: one unit per stage-1 segment / stage-2 part.
struct PackS1 {
  int64_t dst;      // element offset in blob64 / blob32
  int64_t rows;     // offset into the (block, class position) row list
  int32_t R, rp, w, c0;
  int32_t is32, cls;  // cls 1 = FP64 class / plain factors, 2 = FP32 class
  int32_t chunk, pad; // chunk 1: SGEMV chunk layout (chunk_off), m1-single
};
struct PackS2 {
  int64_t dst;
  int32_t R, rp, row0, item0, nitems, is32;
};
struct PackItem {
  int32_t block, cls, width, pad;  // cls 0 dense, 1 hi, 2 lo; pad 1: SGEMV chunk layout (chunk_off)
};
struct PackRow {
  int32_t block, q;
};
int device_pack(const DevSource& src, const std::vector<PackS1>& s1, const std::vector<PackRow>& rows,
                const std::vector<PackS2>& s2, const std::vector<PackItem>& items, double* b64, float* b32,
                cudaStream_t st);

int plan_create_impl(const hmx_matrix_desc* d, int device, const hmx_plan_options* opt, hmx_plan* p,
                     const DevSource* dsrc);

// Enqueues y = A xp (both device, permuted order unless permute_out) on the
// plan's stream with the stage-2 epilogue options `out` (y/nonfinite filled
// in by the caller).
int enqueue_matvec(hmx_plan* p, const double* xp, const S2Out& out);

}  // namespace hmx
