// Internal data layout and device helpers of the sm_100a H-matvec library.
//
// One H-matvec y = A x runs as two streaming kernels over two device blobs
// built by the flattener (hmx_plan.cu):
//
//  stage 1  z = Vt x for every low-rank block (and FP64/FP32 class of a
//           Method-3 block).  Vt rows are stored row-major (ld = n padded to a
//           16-byte multiple).  Work unit = one warp task: <= 16 rank rows x a
//           column chunk; lanes stride over columns with 16-byte loads, keep x
//           in registers across the rank rows, and reduce with a transpose
//           butterfly.  Blocks wider than one chunk are summed by the last
//           arriving task (fixed chunk order => deterministic, atomic-free
//           arithmetic).
//  stage 2  y = sum over the items of every leaf row segment: dense blocks
//           (A x) and U slabs (U z).  Each segment's items are stored
//           column-major (column stride = rows padded to 16 bytes) so a row
//           segment is one contiguous stream; one CTA per segment, thread
//           groups own contiguous column ranges, and the per-row partials are
//           reduced across groups in a fixed order.  No atomics touch y.
//
// Precision pipelines reproduce reference pkg/src/hmx/matvec.py:55-110.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hmx {

// ---- stage 1 -----------------------------------------------------------------
struct S1Task {          // 32 bytes; one warp
  int64_t vt_off;        // element offset of (rank row 0, first column) in vt64/vt32
  int32_t ld;            // row stride in elements
  int32_t ncols;         // columns in this chunk
  int32_t xoff;          // x index of the first column
  int32_t seg;           // stage-1 segment
  int16_t chunk;         // chunk index within the segment
  int8_t R;              // rank rows (1..16)
  int8_t is32;           // float32 storage
  int32_t pad;
};
static_assert(sizeof(S1Task) == 32, "S1Task layout");

struct S1Seg {           // 16 bytes
  int32_t zoff;          // first z entry
  int32_t R;             // rank rows
  int32_t nchunks;       // tasks contributing
  int32_t part_off;      // partial slots (nchunks * R doubles) or -1
};

// ---- stage 2 -----------------------------------------------------------------
struct S2Seg {           // 48 bytes
  int64_t off64;         // element offset of the FP64 column-major part in blob64
  int64_t off32;         // element offset of the FP32 part in blob32
  int32_t row0;          // first (permuted) row
  int32_t R;             // rows (<= 64)
  int32_t W64, W32;      // columns in each part
  int32_t run0;          // first run; FP64 runs then FP32 runs
  int32_t nrun64, nrun32;
  int32_t pad;
};
static_assert(sizeof(S2Seg) == 48, "S2Seg layout");

enum : int32_t { RUN_Z = 1, RUN_ROUND = 2, RUN_ACC32 = 4 };

struct Run {             // one item (block slab) of a segment part
  int32_t src;           // first source index (x, or z if RUN_Z)
  int32_t width;         // columns
  int32_t col0;          // first column within the part
  int32_t flags;
};

// Precision pipelines (hmx_scheme order).
enum Pipe : int { P_M1D = 0, P_M1S = 1, P_M1M = 2, P_M2D = 3, P_M2S = 4, P_M2M = 5, P_M3 = 6 };

// FP32-part accumulation modes for stage 2
enum F32Mode : int { F32_ALL64 = 0, F32_ALL32 = 1, F32_MIXED = 2 };

constexpr int kS2Rows = 64;       // max rows per stage-2 segment
constexpr int kS2Threads = 256;   // stage-2 CTA size
constexpr int kS2WMax = 2048;     // columns of g staged in shared memory per tile
constexpr int kS1Threads = 256;   // stage-1 CTA size (8 warps)
constexpr int kS1RMax = 16;       // rank rows per stage-1 task

// Device-visible plan (passed by value to kernels).
struct DevPlan {
  int32_t n;
  int32_t row_begin, row_end;     // rows computed by this plan
  int32_t pipe;
  // stage 1
  const S1Task* tasks;
  const int32_t* warp_ptr;        // tasks of global warp w: [warp_ptr[w], warp_ptr[w+1])
  const S1Seg* s1segs;
  const double* vt64;
  const float* vt32;
  const double* zscale;           // d per z entry (methods 2, 3)
  double* z;
  double* part;
  uint32_t* seg_count;
  int32_t n_warps;
  // stage 2
  const S2Seg* s2segs;
  const Run* runs;
  const double* blob64;
  const float* blob32;
  int32_t n_s2;
  int32_t f32mode;
  const int32_t* perm;            // permuted -> original (int32)
  const int32_t* run_block;       // run -> block index (non-finite probe)
};

// Per-matvec stage-2 epilogue options.
struct S2Out {
  double* y;            // output
  int permute_out;      // write y[perm[i]] instead of y[i]
  const double* w1;     // if non-null: dot partial sum(y * w1) per segment
  int yy;               // if non-zero: dot partial sum(y * y)
  double* seg_dots;     // 2 doubles per segment
  uint32_t* done;       // last-CTA counter
  double* dots_out;     // final [sum y*w1, sum y*y] (fixed-order reduction)
  int* nonfinite;       // set to 1 when any y entry is not finite
};

// ---- device helpers ------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Streaming 16-byte loads of read-once payload: no L1 allocation, L2
// evict-first so x, z and the tables stay L2-resident.
__device__ __forceinline__ double2 ld_stream(const double* p, uint64_t pol) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ float4 ld_stream(const float* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}

}  // namespace hmx
