// H-matrix compression on the GPU ("GPU ACA +
// kernel-entry assembly"): the FP64 masters of one H-matrix are built straight
// into device memory -- dense near-field blocks by kernel-entry assembly,
// admissible blocks by adaptive cross approximation -- ready for
// hmx_plan_create_prepared, with no payload crossing the host link.
//
// Arithmetic restates reference pkg/src/hmx/compress.py:79-207 (ACA with
// partial pivoting) and :256-282 (kernel entries) exactly as the host
// builder does (csrc/aca_core.h): every floating-point operation is an
// explicit IEEE intrinsic in the host's order (no FMA contraction; the
// norm/cross dot products are the host's FMA chains, each run sequentially
// by one lane), pivots are first-index argmax like the host loops, so the
// device masters are BIT-IDENTICAL to the host builder's
// (tests/test_gpu_build.py).
//
// One warp per admissible block (grid-stride over blocks sorted by size):
// lanes evaluate residual rows/columns entry-parallel, warp shuffles find
// the max and the pivots, lanes run the 2 + 2 rank dot-product chains in
// parallel.  Two passes: pass 1 finds every rank (factors in bounded,
// batched scratch of kAcaCap columns), pass 2 recomputes and writes the
// factors straight into the packed master layout.  Blocks that need more
// than kAcaCap ranks, or that take the reference's "ran out of pivot rows"
// path (exact remainder, possible dense fallback), are completed on the host
// with the host builder's aca_block -- the same arithmetic.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <numeric>
#include <thread>
#include <vector>

#include "aca_core.h"
#include "hmx_plan_impl.cuh"

namespace hmx {
namespace {

constexpr int kCap1 = 24;   // ranks per block in pass-1 scratch (config 4: max rank 19)
constexpr int kCap1Small = 16;  // ... when 24 would not fit in one batch (config 5: max rank 14)
constexpr int kCap2 = 96;   // retry round for the blocks that exhaust kCap1
constexpr int kAcaWarps = 8;             // warps per CTA
constexpr double kPiD = 3.141592653589793;
constexpr double kFourPiD = 4.0 * kPiD;  // compress.py:38
constexpr double kEpsD = 2.220446049250313e-16;

struct AcaTask {
  int64_t r0, c0;
  int64_t u_off;     // U element (i, k) at base[u_off + k * m + i] (column-major: the chains stream)
  int64_t vt_off;    // Vt element (k, j) at base[vt_off + k * n + j]
  int64_t flag_off;  // byte flags: rows [0, m), columns [m, m + n)
  int32_t m, n, budget, cap;
};

enum : int32_t { ACA_OK = 0, ACA_HOST = 1, ACA_CAP = 2 };

__device__ __forceinline__ double kentry_dev(const double* __restrict__ pc, const double* __restrict__ pa,
                                             int64_t gi, int64_t gj) {
  if (gi == gj) return __dmul_rn(0.5, __dsqrt_rn(__ddiv_rn(pa[gi], kPiD)));
  const double* a = pc + 3 * gi;
  const double* b = pc + 3 * gj;
  const double dx = __dsub_rn(a[0], b[0]), dy = __dsub_rn(a[1], b[1]), dz = __dsub_rn(a[2], b[2]);
  const double d = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
  return __ddiv_rn(pa[gj], __dmul_rn(kFourPiD, d));
}

// (value, index) argmax over the warp: larger value, then smaller index
__device__ __forceinline__ void warp_argmax(double& v, int& idx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    if (v2 > v || (v2 == v && i2 < idx)) {
      v = v2;
      idx = i2;
    }
  }
}

// One warp per task.  out_rank/out_status per task.
__global__ void __launch_bounds__(32 * kAcaWarps) aca_kernel(const AcaTask* __restrict__ tasks,
                                                             const int32_t* __restrict__ which, int ntask,
                                                             const double* __restrict__ pc,
                                                             const double* __restrict__ pa, double tol,
                                                             double* base, uint8_t* flags, int32_t* out_rank,
                                                             int32_t* out_status) {
  __shared__ double sab[kAcaWarps][2 * kCap2 + 2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* ab = sab[wid];
  for (int tt = blockIdx.x * kAcaWarps + wid; tt < ntask; tt += gridDim.x * kAcaWarps) {
    const int t = which[tt];
    const AcaTask T = tasks[t];
    const int m = T.m, n = T.n, cap = T.cap;
    double* U = base + T.u_off;
    double* Vt = base + T.vt_off;
    uint8_t* rowu = flags + T.flag_off;
    uint8_t* colu = rowu + m;
    for (int i = lane; i < m + n; i += 32) rowu[i] = 0;
    __syncwarp();
    double frob_sq = 0.0, max_seen = 0.0;
    int rank = 0, i_star = 0, status = ACA_OK;
    bool converged = false;
    while (rank < T.budget && i_star >= 0) {
      if (rank == cap) {  // scratch columns exhausted: retried with more
        status = ACA_CAP;
        break;
      }
      // residual row i_star, written into the next Vt row
      double* row = Vt + (int64_t)rank * n;
      const double* urow = U + i_star;  // U(i_star, k) at urow[k * m]
      double rmax = 0.0, best = -1.0;
      int jbest = 0;
      for (int j = lane; j < n; j += 32) {
        double v = kentry_dev(pc, pa, T.r0 + i_star, T.c0 + j);
        if (rank) {
          double s = 0.0;
          for (int k = 0; k < rank; ++k) s = __dadd_rn(s, __dmul_rn(urow[(int64_t)k * m], Vt[(int64_t)k * n + j]));
          v = __dsub_rn(v, s);
        }
        row[j] = v;
        const double a = fabs(v);
        rmax = (rmax < a) ? a : rmax;
        const double mv = colu[j] ? 0.0 : a;
        if (mv > best) {
          best = mv;
          jbest = j;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double r2 = __shfl_xor_sync(0xffffffffu, rmax, o);
        rmax = (rmax < r2) ? r2 : rmax;
      }
      warp_argmax(best, jbest);
      __syncwarp();
      if (lane == 0) rowu[i_star] = 1;
      max_seen = (max_seen < rmax) ? rmax : max_seen;
      const double pivot = colu[jbest] ? 0.0 : row[jbest];
      __syncwarp();
      if (fabs(pivot) <= __dmul_rn(kEpsD, max_seen)) {
        // vanished pivot: next unused row (compress.py:155-158)
        int first = m;
        for (int i = lane; i < m; i += 32)
          if (!rowu[i]) {
            first = i;
            break;
          }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
        i_star = first < m ? first : -1;
        __syncwarp();
        continue;
      }
      for (int j = lane; j < n; j += 32) row[j] = __ddiv_rn(row[j], pivot);
      // residual column j_star, written into U column `rank`
      for (int i = lane; i < m; i += 32) {
        double v = kentry_dev(pc, pa, T.r0 + i, T.c0 + jbest);
        if (rank) {
          const double* ui = U + i;
          double s = 0.0;
          for (int k = 0; k < rank; ++k) s = __dadd_rn(s, __dmul_rn(ui[(int64_t)k * m], Vt[(int64_t)k * n + jbest]));
          v = __dsub_rn(v, s);
        }
        U[(int64_t)rank * m + i] = v;
      }
      __syncwarp();
      if (lane == 0) colu[jbest] = 1;
      // the host's FMA chains, one per lane: |u|, |v|, a_k = U_k . u, b_k = Vt_k . v
      const int nch = 2 + 2 * rank;
      for (int c = lane; c < nch; c += 32) {
        // one loop for every chain (lanes stay converged), loads batched
        // ahead of the sequential FMA chain
        const double *pa_, *pb_;
        int len;
        if (c == 0) {
          pa_ = pb_ = U + (int64_t)rank * m;
          len = m;
        } else if (c == 1) {
          pa_ = pb_ = row;
          len = n;
        } else if (c < 2 + rank) {
          pa_ = U + (int64_t)(c - 2) * m;
          pb_ = U + (int64_t)rank * m;
          len = m;
        } else {
          pa_ = Vt + (int64_t)(c - 2 - rank) * n;
          pb_ = row;
          len = n;
        }
        double s = 0.0;
        int i = 0;
        for (; i + 16 <= len; i += 16) {
          double a[16], b[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            a[u] = pa_[i + u];
            b[u] = pb_[i + u];
          }
#pragma unroll
          for (int u = 0; u < 16; ++u) s = fma(a[u], b[u], s);
        }
        for (; i < len; ++i) s = fma(pa_[i], pb_[i], s);
        ab[c] = s;
      }
      __syncwarp();
      const double u_norm = __dsqrt_rn(ab[0]), v_norm = __dsqrt_rn(ab[1]);
      double cross = 0.0;
      if (rank) {
        double s = 0.0;
        for (int k = 0; k < rank; ++k) s = fma(ab[2 + k], ab[2 + rank + k], s);
        cross = __dmul_rn(2.0, s);
      }
      __syncwarp();
      const double uv = __dmul_rn(u_norm, v_norm);
      const double f = __dadd_rn(__dadd_rn(frob_sq, __dmul_rn(uv, uv)), cross);
      frob_sq = (f < 0.0) ? 0.0 : f;
      ++rank;
      if (uv <= __dmul_rn(tol, __dsqrt_rn(frob_sq))) {
        converged = true;
        break;
      }
      // next pivot row: largest |u_new| among unused rows (first index)
      double cb = -1.0;
      int ib = 0;
      for (int i = lane; i < m; i += 32) {
        const double cv = rowu[i] ? -1.0 : fabs(U[(int64_t)(rank - 1) * m + i]);
        if (cv > cb) {
          cb = cv;
          ib = i;
        }
      }
      warp_argmax(cb, ib);
      i_star = cb < 0.0 ? -1 : ib;
      __syncwarp();
    }
    // "ran out of pivot rows" (compress.py:191-205): the host measures the
    // remainder and decides between these factors and the dense fallback
    if (status == ACA_OK && !converged && rank < T.budget) status = ACA_HOST;
    if (lane == 0) {
      out_rank[t] = rank;
      out_status[t] = status;
    }
    __syncwarp();
  }
}

// ---- one CTA per large block (m + n >= kBigMN, cap <= kCtaCap): the same
// arithmetic as aca_kernel (bitwise), with 256 threads on the residual row /
// column and the dot-product chains fed through shared memory in chunks
// loaded by the whole CTA (one lane streaming a 10^5-10^6-long chain from
// global memory is bound by its own few loads in flight).
constexpr int kCtaThreads = 256;
constexpr int kCtaCap = 32;
constexpr int kCtaArrays = 2 * kCtaCap;
constexpr int kCtaChunk = 128;
constexpr int64_t kBigMN = 8192;
constexpr size_t kCtaSmem = (size_t)kCtaArrays * kCtaChunk * sizeof(double);

__device__ __forceinline__ void cta_argmax(double& v, int& idx, double* sv, int* si) {
  warp_argmax(v, idx);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) {
    sv[w] = v;
    si[w] = idx;
  }
  __syncthreads();
  v = sv[0];
  idx = si[0];
  for (int q = 1; q < kCtaThreads / 32; ++q)
    if (sv[q] > v || (sv[q] == v && si[q] < idx)) {
      v = sv[q];
      idx = si[q];
    }
}

__device__ __forceinline__ double cta_max(double v, double* sv) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double r2 = __shfl_xor_sync(0xffffffffu, v, o);
    v = (v < r2) ? r2 : v;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sv[threadIdx.x >> 5] = v;
  __syncthreads();
  v = sv[0];
  for (int q = 1; q < kCtaThreads / 32; ++q) v = (v < sv[q]) ? sv[q] : v;
  return v;
}

__device__ __forceinline__ int cta_min(int v, int* si) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) si[threadIdx.x >> 5] = v;
  __syncthreads();
  v = si[0];
  for (int q = 1; q < kCtaThreads / 32; ++q) v = min(v, si[q]);
  return v;
}

__global__ void __launch_bounds__(kCtaThreads) aca_cta_kernel(const AcaTask* __restrict__ tasks,
                                                              const int32_t* __restrict__ which,
                                                              const double* __restrict__ pc,
                                                              const double* __restrict__ pa, double tol,
                                                              double* base, uint8_t* flags, int32_t* out_rank,
                                                              int32_t* out_status) {
  extern __shared__ double chunk[];  // [kCtaArrays][kCtaChunk]
  __shared__ double sv[kCtaThreads / 32];
  __shared__ int si[kCtaThreads / 32];
  __shared__ double ab[kCtaArrays + 2];
  const int tid = threadIdx.x;
  const int t = which[blockIdx.x];
  const AcaTask T = tasks[t];
  const int m = T.m, n = T.n, cap = T.cap;
  double* U = base + T.u_off;
  double* Vt = base + T.vt_off;
  uint8_t* rowu = flags + T.flag_off;
  uint8_t* colu = rowu + m;
  for (int i = tid; i < m + n; i += kCtaThreads) rowu[i] = 0;
  __syncthreads();
  double frob_sq = 0.0, max_seen = 0.0;
  int rank = 0, i_star = 0, status = ACA_OK;
  bool converged = false;
  while (rank < T.budget && i_star >= 0) {
    if (rank == cap) {
      status = ACA_CAP;
      break;
    }
    double* row = Vt + (int64_t)rank * n;
    const double* urow = U + i_star;
    double rmax = 0.0, best = -1.0;
    int jbest = 0;
    for (int j = tid; j < n; j += kCtaThreads) {
      double v = kentry_dev(pc, pa, T.r0 + i_star, T.c0 + j);
      if (rank) {
        double s = 0.0;
        for (int k = 0; k < rank; ++k) s = __dadd_rn(s, __dmul_rn(urow[(int64_t)k * m], Vt[(int64_t)k * n + j]));
        v = __dsub_rn(v, s);
      }
      row[j] = v;
      const double a = fabs(v);
      rmax = (rmax < a) ? a : rmax;
      const double mv = colu[j] ? 0.0 : a;
      if (mv > best) {
        best = mv;
        jbest = j;
      }
    }
    rmax = cta_max(rmax, sv);
    cta_argmax(best, jbest, sv, si);
    max_seen = (max_seen < rmax) ? rmax : max_seen;
    const double pivot = colu[jbest] ? 0.0 : row[jbest];
    __syncthreads();
    if (tid == 0) rowu[i_star] = 1;
    __syncthreads();
    if (fabs(pivot) <= __dmul_rn(kEpsD, max_seen)) {
      int first = m;
      for (int i = tid; i < m; i += kCtaThreads)
        if (!rowu[i]) {
          first = i;
          break;
        }
      first = cta_min(first, si);
      i_star = first < m ? first : -1;
      __syncthreads();
      continue;
    }
    for (int j = tid; j < n; j += kCtaThreads) row[j] = __ddiv_rn(row[j], pivot);
    for (int i = tid; i < m; i += kCtaThreads) {
      double v = kentry_dev(pc, pa, T.r0 + i, T.c0 + jbest);
      if (rank) {
        const double* ui = U + i;
        double s = 0.0;
        for (int k = 0; k < rank; ++k) s = __dadd_rn(s, __dmul_rn(ui[(int64_t)k * m], Vt[(int64_t)k * n + jbest]));
        v = __dsub_rn(v, s);
      }
      U[(int64_t)rank * m + i] = v;
    }
    __syncthreads();
    if (tid == 0) colu[jbest] = 1;
    // chains (the host's FMA chains, one thread each, same order as
    // aca_kernel): array c is chain c's first operand -- 0: U col rank,
    // 1: v (row), 2+k: U col k, 2+rank+k: Vt row k; the second operand is
    // array 0 (chains 0 and 2+k) or array 1 (chains 1 and 2+rank+k)
    const int nch = 2 + 2 * rank;
    double s = 0.0;
    const int maxlen = max(m, n);
    for (int i0 = 0; i0 < maxlen; i0 += kCtaChunk) {
      for (int idx = tid; idx < nch * kCtaChunk; idx += kCtaThreads) {
        const int a = idx / kCtaChunk, e = idx - a * kCtaChunk, i = i0 + e;
        const double* p;
        int len;
        if (a == 0) {
          p = U + (int64_t)rank * m;
          len = m;
        } else if (a == 1) {
          p = row;
          len = n;
        } else if (a < 2 + rank) {
          p = U + (int64_t)(a - 2) * m;
          len = m;
        } else {
          p = Vt + (int64_t)(a - 2 - rank) * n;
          len = n;
        }
        chunk[idx] = i < len ? p[i] : 0.0;
      }
      __syncthreads();
      if (tid < nch) {
        const int len = (tid == 0 || (tid >= 2 && tid < 2 + rank)) ? m : n;
        const double* A = chunk + tid * kCtaChunk;
        const double* B = chunk + ((tid == 0 || (tid >= 2 && tid < 2 + rank)) ? 0 : kCtaChunk);
        const int e1 = min(kCtaChunk, len - i0);
        for (int e = 0; e < e1; ++e) s = fma(A[e], B[e], s);
      }
      __syncthreads();
    }
    if (tid < nch) ab[tid] = s;
    __syncthreads();
    const double u_norm = __dsqrt_rn(ab[0]), v_norm = __dsqrt_rn(ab[1]);
    double cross = 0.0;
    if (rank) {
      double c2 = 0.0;
      for (int k = 0; k < rank; ++k) c2 = fma(ab[2 + k], ab[2 + rank + k], c2);
      cross = __dmul_rn(2.0, c2);
    }
    const double uv = __dmul_rn(u_norm, v_norm);
    const double f = __dadd_rn(__dadd_rn(frob_sq, __dmul_rn(uv, uv)), cross);
    frob_sq = (f < 0.0) ? 0.0 : f;
    ++rank;
    if (uv <= __dmul_rn(tol, __dsqrt_rn(frob_sq))) {
      converged = true;
      break;
    }
    double cb = -1.0;
    int ib = 0;
    for (int i = tid; i < m; i += kCtaThreads) {
      const double cv = rowu[i] ? -1.0 : fabs(U[(int64_t)(rank - 1) * m + i]);
      if (cv > cb) {
        cb = cv;
        ib = i;
      }
    }
    cta_argmax(cb, ib, sv, si);
    i_star = cb < 0.0 ? -1 : ib;
    __syncthreads();
  }
  if (status == ACA_OK && !converged && rank < T.budget) status = ACA_HOST;
  if (tid == 0) {
    out_rank[t] = rank;
    out_status[t] = status;
  }
}

// Dense near-field blocks (and ACA dense fallbacks): compress.py:272-282.
struct DenseTask {
  int64_t r0, c0, off;
  int32_t m, n;
};

__global__ void dense_fill_kernel(const DenseTask* __restrict__ tasks, const double* __restrict__ pc,
                                  const double* __restrict__ pa, double* base) {
  const DenseTask T = tasks[blockIdx.x];
  const int64_t total = (int64_t)T.m * T.n;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    const int64_t i = e / T.n, j = e - i * T.n;
    base[T.off + e] = kentry_dev(pc, pa, T.r0 + i, T.c0 + j);
  }
}

// Scratch factors (U m x cap column-major, Vt cap x n) into the packed layout
// (U m x r, then Vt r x n).
struct CopyTask {
  int64_t src_u, src_vt, dst;
  int32_t m, n, cap, r;
};

__global__ void compact_kernel(const CopyTask* __restrict__ tasks, const double* __restrict__ src,
                               double* dst) {
  const CopyTask T = tasks[blockIdx.x];
  const int64_t nu = (int64_t)T.m * T.r, nv = (int64_t)T.r * T.n;
  for (int64_t e = threadIdx.x; e < nu; e += blockDim.x) {
    const int64_t i = e / T.r, k = e - i * T.r;
    dst[T.dst + e] = src[T.src_u + k * T.m + i];
  }
  for (int64_t e = threadIdx.x; e < nv; e += blockDim.x) dst[T.dst + nu + e] = src[T.src_vt + e];
}

template <typename T, typename F>
int launch_tasks(const std::vector<T>& v, cudaStream_t st, F&& launch) {
  for (size_t b0 = 0; b0 < v.size(); b0 += (size_t)1 << 20) {
    const size_t cnt = std::min<size_t>(v.size() - b0, (size_t)1 << 20);
    T* d = nullptr;
    HMX_CUDA(cudaMalloc(&d, cnt * sizeof(T)));
    cudaError_t e = cudaMemcpyAsync(d, v.data() + b0, cnt * sizeof(T), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) {
      launch(d, (unsigned)cnt);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d);
    if (e != cudaSuccess) return cuda_fail(e, "build kernel");
  }
  return HMX_OK;
}

int run_aca(const std::vector<AcaTask>& tasks, const double* d_pc, const double* d_pa, double tol,
            double* base, uint8_t* d_flags, int32_t* d_rank, int32_t* d_status, cudaStream_t st, int sms) {
  if (tasks.empty()) return HMX_OK;
  // large blocks: a CTA each, on a side stream, concurrently with the
  // warp-per-block kernel over the rest
  std::vector<int32_t> big, small;
  for (size_t i = 0; i < tasks.size(); ++i) {
    const AcaTask& T = tasks[i];
    ((int64_t)T.m + T.n >= kBigMN && T.cap <= kCtaCap ? big : small).push_back((int32_t)i);
  }
  AcaTask* d_tasks = nullptr;
  int32_t* d_which = nullptr;
  cudaStream_t side = nullptr;
  cudaEvent_t ev = nullptr;
  cudaError_t e = cudaMalloc(&d_tasks, tasks.size() * sizeof(AcaTask));
  if (e == cudaSuccess) e = cudaMalloc(&d_which, tasks.size() * sizeof(int32_t));
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_tasks, tasks.data(), tasks.size() * sizeof(AcaTask), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && !small.empty())
    e = cudaMemcpyAsync(d_which, small.data(), small.size() * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && !big.empty())
    e = cudaMemcpyAsync(d_which + small.size(), big.data(), big.size() * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && !big.empty()) {
    e = cudaFuncSetAttribute(aca_cta_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kCtaSmem);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ev, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(side, ev, 0);
    if (e == cudaSuccess) {
      aca_cta_kernel<<<(unsigned)big.size(), kCtaThreads, kCtaSmem, side>>>(
          d_tasks, d_which + small.size(), d_pc, d_pa, tol, base, d_flags, d_rank, d_status);
      e = cudaGetLastError();
    }
  }
  if (e == cudaSuccess && !small.empty()) {
    const int64_t want = ((int64_t)small.size() + kAcaWarps - 1) / kAcaWarps;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * 8));
    aca_kernel<<<grid, 32 * kAcaWarps, 0, st>>>(d_tasks, d_which, (int)small.size(), d_pc, d_pa, tol, base,
                                                d_flags, d_rank, d_status);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess && side) e = cudaStreamSynchronize(side);
  if (ev) cudaEventDestroy(ev);
  if (side) cudaStreamDestroy(side);
  cudaFree(d_which);
  cudaFree(d_tasks);
  if (e != cudaSuccess) return cuda_fail(e, "aca kernels");
  return HMX_OK;
}

}  // namespace
}  // namespace hmx

using namespace hmx;

extern "C" {

int hmx_master_build(const hmx_build_desc* d, int device, hmx_master** out, int32_t* kinds, int64_t* ranks,
                     int64_t* offsets, int64_t* n_data, int64_t* fallbacks) {
  NvtxRange nvtx("hmx_master_build");
  if (!d || !out || !kinds || !ranks || !offsets || !n_data || !d->pcent || !d->parea || !d->perm ||
      !d->table) {
    set_error("null argument");
    return HMX_ERR_ARG;
  }
  *out = nullptr;
  const int64_t N = d->n, nb = d->n_blocks;
  if (N < 1 || nb < 1 || !(d->tol > 0.0) || d->max_rank < 0) {
    set_error("invalid build descriptor (n, n_blocks >= 1, tol > 0, max_rank >= 0)");
    return HMX_ERR_ARG;
  }
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    set_error("no CUDA device is available");
    return HMX_ERR_CUDA;
  }
  if (device < 0 || device >= count) {
    set_error("device index out of range");
    return HMX_ERR_ARG;
  }
  DeviceGuard guard(device);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const bool timing = std::getenv("HMX_BUILD_TIMING") != nullptr;
  auto t_start = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!timing) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[hmx_master_build] %-28s %8.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t_start).count());
    t_start = now;
  };
  const int64_t row_lo = d->row_lo, row_hi = d->row_hi > 0 ? d->row_hi : N;

  auto* M = new hmx_master();
  auto fail = [&](int rc) {
    hmx_master_destroy(M);
    return rc;
  };
  M->device = device;
  M->n = N;
  M->nb = nb;
  M->perm.assign(d->perm, d->perm + N);
  M->table.assign(d->table, d->table + 5 * nb);
  cudaError_t e = cudaStreamCreateWithFlags(&M->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return fail(cuda_fail(e, "cudaStreamCreate"));
  cudaStream_t st = M->stream;

  // geometry on the device
  double* d_pc = M->alloc<double>((size_t)(3 * N));
  double* d_pa = M->alloc<double>((size_t)N);
  if (!d_pc || !d_pa) {
    set_error("cudaMalloc failed for the mesh geometry");
    return fail(HMX_ERR_CUDA);
  }
  if ((e = cudaMemcpyAsync(d_pc, d->pcent, (size_t)(3 * N) * 8, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
      (e = cudaMemcpyAsync(d_pa, d->parea, (size_t)N * 8, cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return fail(cuda_fail(e, "geometry upload"));

  // block classes: 0 dense, 1 ACA, 2 not built (outside the row range)
  std::vector<int32_t> kind((size_t)nb), rank((size_t)nb, 0);
  std::vector<int64_t> aca_blocks;
  for (int64_t k = 0; k < nb; ++k) {
    const int64_t* t = d->table + 5 * k;
    if (t[1] <= t[0] || t[3] <= t[2] || t[0] < 0 || t[1] > N || t[2] < 0 || t[3] > N) {
      set_error("block " + std::to_string(k) + " is outside the matrix");
      return fail(HMX_ERR_ARG);
    }
    if (t[1] <= row_lo || t[0] >= row_hi) kind[(size_t)k] = 2;
    else if (t[4]) {
      kind[(size_t)k] = 1;
      aca_blocks.push_back(k);
    } else {
      kind[(size_t)k] = 0;
    }
  }
  // largest blocks first (their sequential chains are the longest)
  std::stable_sort(aca_blocks.begin(), aca_blocks.end(), [&](int64_t a, int64_t b) {
    const int64_t* ta = d->table + 5 * a;
    const int64_t* tb = d->table + 5 * b;
    return (ta[1] - ta[0]) + (ta[3] - ta[2]) > (tb[1] - tb[0]) + (tb[3] - tb[2]);
  });
  auto budget_of = [&](int64_t k) {
    const int64_t* t = d->table + 5 * k;
    int64_t b = std::min(t[1] - t[0], t[3] - t[2]);
    if (d->max_rank > 0) b = std::min(b, d->max_rank);
    return b;
  };
  const size_t na = aca_blocks.size();
  int32_t *d_rank = nullptr, *d_status = nullptr;
  d_rank = M->alloc<int32_t>(std::max<size_t>(na, 1));
  d_status = M->alloc<int32_t>(std::max<size_t>(na, 1));
  if (!d_rank || !d_status) {
    set_error("cudaMalloc failed for the ACA results");
    return fail(HMX_ERR_CUDA);
  }

  // ---- ACA rounds.  A round runs the ACA of a set of blocks in batches of
  // bounded scratch (U m x cap column-major, then Vt cap x n per block) and
  // hands every finished batch to `done`.  Pass 1: ranks with kCap1 columns;
  // when one batch holds every block (config 4: 14 GB) its scratch is kept
  // and compacted into the masters.  Retry: the blocks that exhausted kCap1,
  // with kCap2.  Pass 2: the blocks whose factors were not kept, recomputed
  // with their final rank as cap and compacted batch by batch.
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const int64_t scratch_budget = std::max<int64_t>((int64_t)1 << 27, (int64_t)(free_b / 8) * 60 / 100);
  // pass-1 columns per block: 24, or 16 when that keeps pass 1 in one batch
  // (its scratch is then compacted instead of recomputed; blocks that need
  // more are retried)
  int64_t cap1 = kCap1;
  {
    int64_t need24 = 0, need16 = 0;
    for (int64_t k : aca_blocks) {
      const int64_t* t = d->table + 5 * k;
      const int64_t mn = (t[1] - t[0]) + (t[3] - t[2]);
      need24 += std::min<int64_t>(budget_of(k), kCap1) * mn;
      need16 += std::min<int64_t>(budget_of(k), kCap1Small) * mn;
    }
    if (need24 > scratch_budget && need16 <= scratch_budget) cap1 = kCap1Small;
  }
  std::vector<int32_t> h_rank(na, 0), h_status(na, 0);
  auto aca_round = [&](const std::vector<size_t>& idx_in, const std::function<int64_t(size_t)>& cap_of,
                       const std::function<int(const std::vector<AcaTask>&, const std::vector<int32_t>&,
                                               const std::vector<int32_t>&, const std::vector<size_t>&,
                                               double*, bool)>& done)
      -> int {
    // more than one batch: deal the (size-sorted) blocks round-robin so
    // every batch mixes large and small blocks (a batch of only the largest
    // leaves most warps idle behind their long sequential chains)
    std::vector<size_t> idx = idx_in;
    {
      int64_t total = 0;
      for (size_t q : idx_in) {
        const int64_t* t = d->table + 5 * aca_blocks[q];
        total += cap_of(q) * ((t[1] - t[0]) + (t[3] - t[2]));
      }
      const int64_t nbat = (total + scratch_budget - 1) / scratch_budget;
      if (nbat > 1) {
        idx.clear();
        for (int64_t b = 0; b < nbat; ++b)
          for (size_t i = (size_t)b; i < idx_in.size(); i += (size_t)nbat) idx.push_back(idx_in[i]);
      }
    }
    uint8_t* fl = nullptr;
    double* sc = nullptr;
    int64_t sc_cap = 0, fl_cap = 0;
    size_t b0 = 0;
    int rc = HMX_OK;
    bool kept = false;
    while (b0 < idx.size() && rc == HMX_OK) {
      std::vector<AcaTask> batch;
      int64_t used = 0, fused = 0;
      size_t b1 = b0;
      for (; b1 < idx.size(); ++b1) {
        const int64_t k = aca_blocks[idx[b1]];
        const int64_t* t = d->table + 5 * k;
        const int64_t m = t[1] - t[0], n = t[3] - t[2];
        const int64_t cap = cap_of(idx[b1]);
        const int64_t need = cap * (m + n);
        if (!batch.empty() && used + need > scratch_budget) break;
        AcaTask T{};
        T.r0 = t[0];
        T.c0 = t[2];
        T.m = (int32_t)m;
        T.n = (int32_t)n;
        T.budget = (int32_t)budget_of(k);
        T.cap = (int32_t)cap;
        T.u_off = used;
        T.vt_off = used + m * cap;
        T.flag_off = fused;
        used += need;
        fused += m + n;
        batch.push_back(T);
      }
      const bool only = b0 == 0 && b1 == idx.size();
      if (used > sc_cap) {
        cudaFree(sc);
        sc = nullptr;
        if (cudaMalloc(&sc, (size_t)std::max<int64_t>(used, 1) * 8) != cudaSuccess) {
          set_error("cudaMalloc failed for the ACA scratch");
          rc = HMX_ERR_CUDA;
          break;
        }
        sc_cap = used;
      }
      if (fused > fl_cap) {
        cudaFree(fl);
        fl = nullptr;
        if (cudaMalloc(&fl, (size_t)fused) != cudaSuccess) {
          set_error("cudaMalloc failed for the ACA flags");
          rc = HMX_ERR_CUDA;
          break;
        }
        fl_cap = fused;
      }
      rc = run_aca(batch, d_pc, d_pa, d->tol, sc, fl, d_rank, d_status, st, sms);
      if (rc) break;
      std::vector<int32_t> r(batch.size()), q(batch.size());
      if ((e = cudaMemcpy(r.data(), d_rank, batch.size() * 4, cudaMemcpyDeviceToHost)) != cudaSuccess ||
          (e = cudaMemcpy(q.data(), d_status, batch.size() * 4, cudaMemcpyDeviceToHost)) != cudaSuccess) {
        rc = cuda_fail(e, "ACA ranks");
        break;
      }
      rc = done(batch, r, q, std::vector<size_t>(idx.begin() + (ptrdiff_t)b0, idx.begin() + (ptrdiff_t)b1), sc,
                only);
      if (rc == -1) {  // the callback keeps the scratch
        kept = true;
        rc = HMX_OK;
      }
      b0 = b1;
    }
    cudaFree(fl);
    if (!kept) cudaFree(sc);
    return rc;
  };
  // pass 1
  double* kept_scratch = nullptr;
  std::vector<AcaTask> kept_tasks;
  {
    std::vector<size_t> all(na);
    std::iota(all.begin(), all.end(), (size_t)0);
    const int rc = aca_round(
        all, [&](size_t q) { return std::min<int64_t>(budget_of(aca_blocks[q]), cap1); },
        [&](const std::vector<AcaTask>& b, const std::vector<int32_t>& r, const std::vector<int32_t>& q,
            const std::vector<size_t>& qs, double* sc, bool only) -> int {
          for (size_t i = 0; i < b.size(); ++i) {
            h_rank[qs[i]] = r[i];
            h_status[qs[i]] = q[i];
          }
          if (!only) return HMX_OK;
          kept_scratch = sc;
          kept_tasks = b;
          return -1;
        });
    if (rc) return fail(rc);
  }
  struct FreeOnExit {
    double** p;
    ~FreeOnExit() { cudaFree(*p); }
  } scratch_guard{&kept_scratch};
  lap("pass 1 (ranks)");
  // retry round for the blocks that exhausted kCap1
  {
    std::vector<size_t> retry;
    for (size_t q = 0; q < na; ++q)
      if (h_status[q] == ACA_CAP) retry.push_back(q);
    if (timing && na) {
      const int64_t* t = d->table + 5 * aca_blocks[0];
      std::fprintf(stderr, "[hmx_master_build] %zu ACA blocks, largest %lld x %lld (rank %d), %zu retried with %d columns, "
                   "pass-1 scratch %s\n", na, (long long)(t[1] - t[0]), (long long)(t[3] - t[2]), h_rank[0],
                   retry.size(), kCap2, kept_scratch ? "kept" : "batched");
    }
    if (!retry.empty()) {
      const int rc = aca_round(
          retry, [&](size_t q) { return std::min<int64_t>(budget_of(aca_blocks[q]), kCap2); },
          [&](const std::vector<AcaTask>& b, const std::vector<int32_t>& r, const std::vector<int32_t>& q,
              const std::vector<size_t>& qs, double*, bool) -> int {
            for (size_t i = 0; i < b.size(); ++i) {
              h_rank[qs[i]] = r[i];
              h_status[qs[i]] = q[i];
            }
            return HMX_OK;
          });
      if (rc) return fail(rc);
    }
  }
  // pass-1 blocks whose factors are in the kept scratch
  std::vector<char> in_kept(na, 0);
  if (kept_scratch)
    for (size_t q = 0; q < na; ++q) in_kept[q] = h_status[q] == ACA_OK && h_rank[q] <= kept_tasks[q].cap;
  // ---- host completion of the rare blocks (same arithmetic: aca_core.h)
  std::vector<size_t> host_idx;
  for (size_t q = 0; q < na; ++q)
    if (h_status[q] != ACA_OK) host_idx.push_back(q);  // remainder path, or beyond kCap2 ranks
  std::vector<hmx_aca::BlockResult> host_res(host_idx.size());
  int64_t nfall = 0;
  {
    hmx_aca::Geom G{d->pcent, d->parea};
    std::vector<char> fb(host_idx.size(), 0);
    std::atomic<size_t> next{0};
    const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(),
                                                        (unsigned)std::max<size_t>(host_idx.size(), 1)));
    std::vector<std::thread> pool;
    for (unsigned w = 0; w < nt; ++w)
      pool.emplace_back([&]() {
        for (;;) {
          const size_t h = next.fetch_add(1);
          if (h >= host_idx.size()) break;
          const int64_t k = aca_blocks[host_idx[h]];
          const int64_t* t = d->table + 5 * k;
          bool f = false;
          hmx_aca::aca_block(G, t[0], t[1] - t[0], t[2], t[3] - t[2], d->tol, d->max_rank, host_res[h], f);
          fb[h] = f ? 1 : 0;
        }
      });
    for (auto& th : pool) th.join();
    for (size_t h = 0; h < host_idx.size(); ++h) {
      const size_t q = host_idx[h];
      const int64_t k = aca_blocks[q];
      if (fb[h]) {
        kind[(size_t)k] = 0;  // dense fallback (the host builder stores it dense too)
        ++nfall;
      } else {
        h_rank[q] = (int32_t)host_res[h].rank;
      }
    }
  }
  for (size_t q = 0; q < na; ++q)
    if (kind[(size_t)aca_blocks[q]] == 1) rank[(size_t)aca_blocks[q]] = h_rank[q];
  if (timing) std::fprintf(stderr, "[hmx_master_build] %zu of %zu ACA blocks completed on the host\n",
                           host_idx.size(), na);
  lap("host completion");

  // ---- layout (hb_build_layout's): dense m*n, low rank r*(m+n), skipped 0
  int64_t off = 0;
  M->kind.resize((size_t)nb);
  M->offset.resize((size_t)nb);
  M->rank.resize((size_t)nb);
  M->roff.resize((size_t)nb);
  for (int64_t k = 0; k < nb; ++k) {
    const int64_t* t = d->table + 5 * k;
    const int64_t m = t[1] - t[0], n = t[3] - t[2];
    const int32_t kd = kind[(size_t)k];
    const int64_t r = kd == 1 ? rank[(size_t)k] : 0;
    kinds[k] = kd;
    ranks[k] = r;
    offsets[k] = off;
    M->kind[(size_t)k] = kd;
    M->rank[(size_t)k] = r;
    M->offset[(size_t)k] = off;
    M->roff[(size_t)k] = M->rank_sum;
    M->rank_sum += r;
    M->max_rank = std::max(M->max_rank, r);
    off += kd == 0 ? m * n : kd == 1 ? r * (m + n) : 0;
  }
  *n_data = off;
  M->n_data = off;
  if (fallbacks) *fallbacks = nfall;
  M->data = M->alloc<double>((size_t)std::max<int64_t>(off, 1));
  if (!M->data && kept_scratch) {
    // no room next to the kept pass-1 scratch: drop it, recompute in pass 2
    cudaFree(kept_scratch);
    kept_scratch = nullptr;
    std::fill(in_kept.begin(), in_kept.end(), 0);
    cudaGetLastError();
    M->data = M->alloc<double>((size_t)std::max<int64_t>(off, 1));
  }
  if (!M->data) {
    set_error("cudaMalloc failed for the masters (out of device memory?)");
    return fail(HMX_ERR_CUDA);
  }

  // ---- dense blocks: kernel-entry assembly
  {
    std::vector<DenseTask> dt;
    for (int64_t k = 0; k < nb; ++k)
      if (kind[(size_t)k] == 0) {
        const int64_t* t = d->table + 5 * k;
        dt.push_back({t[0], t[2], offsets[k], (int32_t)(t[1] - t[0]), (int32_t)(t[3] - t[2])});
      }
    const int rc = launch_tasks(dt, st, [&](const DenseTask* t, unsigned cnt) {
      dense_fill_kernel<<<cnt, 256, 0, st>>>(t, d_pc, d_pa, M->data);
    });
    if (rc) return fail(rc);
  }
  // ---- factors into the packed layout (U m x r row-major, then Vt r x n)
  auto compact = [&](const std::vector<AcaTask>& b, const std::vector<size_t>& qs, const double* sc) -> int {
    std::vector<CopyTask> ct;
    for (size_t i = 0; i < b.size(); ++i) {
      const size_t q = qs[i];
      const int64_t k = aca_blocks[q];
      if (kind[(size_t)k] != 1 || h_status[q] != ACA_OK) continue;
      ct.push_back({b[i].u_off, b[i].vt_off, offsets[k], b[i].m, b[i].n, b[i].cap, (int32_t)rank[(size_t)k]});
    }
    return launch_tasks(ct, st, [&](const CopyTask* dt, unsigned cnt) {
      compact_kernel<<<cnt, 256, 0, st>>>(dt, sc, M->data);
    });
  };
  if (kept_scratch) {
    std::vector<size_t> qs(na);
    std::iota(qs.begin(), qs.end(), (size_t)0);
    std::vector<AcaTask> b;
    std::vector<size_t> bq;
    for (size_t q = 0; q < na; ++q)
      if (in_kept[q]) {
        b.push_back(kept_tasks[q]);
        bq.push_back(q);
      }
    const int rc = compact(b, bq, kept_scratch);
    if (rc) return fail(rc);
    cudaFree(kept_scratch);
    kept_scratch = nullptr;
  }
  lap("layout + dense + compaction");
  // pass 2: the GPU-finished blocks whose factors were not kept, recomputed
  // with their rank as cap (same arithmetic: the ranks must reproduce)
  {
    std::vector<size_t> redo;
    for (size_t q = 0; q < na; ++q)
      if (h_status[q] == ACA_OK && !in_kept[q] && kind[(size_t)aca_blocks[q]] == 1) redo.push_back(q);
    if (!redo.empty()) {
      const int rc = aca_round(
          redo, [&](size_t q) { return std::max<int64_t>(h_rank[q], 1); },
          [&](const std::vector<AcaTask>& b, const std::vector<int32_t>& r, const std::vector<int32_t>& q,
              const std::vector<size_t>& qs, double* sc, bool) -> int {
            for (size_t i = 0; i < b.size(); ++i) {
              if (r[i] != h_rank[qs[i]] || q[i] != ACA_OK) {
                set_error("ACA pass 2 diverged from pass 1");
                return HMX_ERR_CUDA;
              }
            }
            return compact(b, qs, sc);
          });
      if (rc) return fail(rc);
    }
  }
  lap("pass 2 (factors)");
  // host-completed low-rank blocks
  for (size_t h = 0; h < host_idx.size(); ++h) {
    const int64_t k = aca_blocks[host_idx[h]];
    if (kind[(size_t)k] != 1) continue;
    const hmx_aca::BlockResult& R = host_res[h];
    const int64_t* t = d->table + 5 * k;
    const int64_t m = t[1] - t[0];
    if (R.rank > 0) {
      if ((e = cudaMemcpy(M->data + offsets[k], R.u.data(), R.u.size() * 8, cudaMemcpyHostToDevice)) != cudaSuccess ||
          (e = cudaMemcpy(M->data + offsets[k] + m * R.rank, R.vt.data(), R.vt.size() * 8,
                          cudaMemcpyHostToDevice)) != cudaSuccess)
        return fail(cuda_fail(e, "host ACA upload"));
    }
  }

  // ---- device tables (as hmx_master_create)
  auto up = [&](auto** dst, const auto* src, size_t cnt) -> int {
    using T = typename std::remove_pointer<typename std::remove_reference<decltype(*dst)>::type>::type;
    *dst = M->alloc<T>(cnt);
    if (!*dst) {
      set_error("cudaMalloc failed for the master tables");
      return HMX_ERR_CUDA;
    }
    if (cnt) HMX_CUDA(cudaMemcpy(*dst, src, cnt * sizeof(T), cudaMemcpyHostToDevice));
    return HMX_OK;
  };
  int rc = up(&M->d_table, M->table.data(), (size_t)(5 * nb));
  if (!rc) rc = up(&M->d_kind, M->kind.data(), (size_t)nb);
  if (!rc) rc = up(&M->d_offset, M->offset.data(), (size_t)nb);
  if (!rc) rc = up(&M->d_rank, M->rank.data(), (size_t)nb);
  if (!rc) rc = up(&M->d_roff, M->roff.data(), (size_t)nb);
  if (rc) return fail(rc);
  *out = M;
  return HMX_OK;
}

int hmx_master_download(hmx_master* m, double* data) {
  if (!m || (!data && m->n_data > 0)) {
    set_error("null argument");
    return HMX_ERR_ARG;
  }
  DeviceGuard guard(m->device);
  if (m->n_data > 0) HMX_CUDA(cudaMemcpy(data, m->data, (size_t)m->n_data * 8, cudaMemcpyDeviceToHost));
  return HMX_OK;
}

}  // extern "C"
