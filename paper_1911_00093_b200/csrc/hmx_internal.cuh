// Internal data layout and device helpers of the sm_100a H-matvec library.
//
// One H-matvec y = A x runs as two launches of ONE segmented column-major
// GEMV kernel over device blobs built by the flattener (hmx_plan.cu):
//
//  stage 1  z = Vt x.  Low-rank blocks are grouped by column cluster: every
//           block with the same column range reads the same x segment, so
//           their rank rows stack into one tall (sum r) x n matrix.  It is cut
//           into segments of <= 64 rank rows (and column chunks of ~256 KB),
//           stored column-major, one CTA each.  z is laid out in the same
//           order, so a segment writes a contiguous z range.
//  stage 2  y = sum of the items covering every leaf row segment: dense
//           blocks (A x) and U slabs (U z), column-major, one CTA each.
//
// In both, a CTA stages its source vector g (x segments / z vectors) in
// shared memory, thread groups stream contiguous column ranges with 16-byte
// loads (2 FP64 or 4 FP32 rows per thread), and per-row partials are reduced
// across groups in a fixed order.  Column-chunked stage-1 segments are summed
// by the last arriving CTA in chunk order.  No atomics touch y or z values:
// results are bit-reproducible.
//
// Precision pipelines reproduce reference pkg/src/hmx/matvec.py:55-110.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace hmx {

// ---- segments (both stages) ----------------------------------------------------
struct Seg {             // 64 bytes; one CTA
  int64_t off64;         // element offset of the FP64 column-major part in blob64
  int64_t off32;         // element offset of the FP32 part in blob32
  int32_t row0;          // first output row: y row (stage 2) or z index (stage 1)
  int32_t R;             // rows (<= 64)
  int32_t W64, W32;      // columns in each part
  int32_t run0;          // first run; FP64 runs then FP32 runs
  int32_t nrun64, nrun32;
  int32_t red;           // stage 1: reduction group of a column-chunked segment, or -1
  int32_t chunk, nchunks;  // stage 1: column chunk / count; stage 2: chunk = wb, the first
                           // thread of the FP32-accumulated groups of a mixed FP32 part (0: none)
  int32_t part_off;      // partial slots (nchunks * R doubles)
  int32_t gtab;          // FP32 part: group cuts gtab[gtab..gtab+G], the first FP32-accumulated
                         // column, then per cut the index of the first run at or after it;
                         // <= -2: that column alone at gtab[-2-gtab]; -1: none
};
static_assert(sizeof(Seg) == 64, "Seg layout");

// RUN_CHUNK: a stage-1 FP32-accumulated segment (m1-single) in SGEMV chunk layout (below)
enum : int32_t { RUN_Z = 1, RUN_ROUND = 2, RUN_ACC32 = 4, RUN_CHUNK = 8 };
// RUN_CHUNK items: bits 4..31 of Run.flags locate, within the segment, the
// row classes OpenBLAS SGEMV-T computes the item's block in (it takes the
// rows of an m-row block 16, then 8, then 4 at a time, then a 2-row and a
// 1-row remainder kernel, whose summation orders differ): four 7-bit
// segment-relative row bounds e16 | e8 << 7 | e4 << 14 | e2 << 21
// (chain_row_kind: p < e16 -> 16, < e8 -> 8, < e4 -> 4, < e2 -> 2, else 1)
constexpr int kRunKindShift = 4;
__host__ __device__ __forceinline__ int chain_row_kind(uint32_t bits, int p) {
  const int e16 = bits & 127, e8 = (bits >> 7) & 127, e4 = (bits >> 14) & 127, e2 = (bits >> 21) & 127;
  return p < e16 ? 16 : p < e8 ? 8 : p < e4 ? 4 : p < e2 ? 2 : 1;
}
// the same classes for row i of an m-row block
__host__ __device__ __forceinline__ int sgemv_row_kind(int64_t i, int64_t m) {
  const int64_t a16 = m & ~int64_t(15), b8 = a16 + (m & 8), c4 = b8 + (m & 4);
  return i < a16 ? 16 : i < b8 ? 8 : i < c4 ? 4 : ((m & 3) >= 2 && i < c4 + 2) ? 2 : 1;
}

// ---- FP32-accumulated stage-2 items: the reference's summation order ---------
// The reference's FP32 products (`A32 @ x32`, `U32 @ z32`; matvec.py:57, :73)
// run through OpenBLAS SGEMV-T.  Its summation tree for one n-wide row,
// recovered by probing (tools/sgemv_order_probe.py; CPU model and bitwise
// check against numpy in tools/fp32_accum_emulation.py), with nch = n / 4
// chunks of 4 columns and T = n % 4 tail columns:
//   * two 4-wide FMA accumulators A and B over the chunks (nch even: A takes
//     the even chunks, B the odd ones; nch odd: A = {0, 1, 3, 5, ..},
//     B = {2, 4, ..}); l = A + B lane-wise; main = (l0 + l1) + (l2 + l3);
//   * tail: T = 1: fma(a_m, g_m, main); T = 2: main + fma(a_m, g_m, a_{m+1}
//     g_{m+1}); T = 3: main + fma(a_{m+2}, g_{m+2}, that)   (m = 4 nch);
//   * n = 8: l_j = a_{2j} g_{2j} + a_{2j+1} g_{2j+1}, then main as above;
//   * n <= 3 and 5 <= n <= 7: one forward FMA chain.
// The stage-2 kernel evaluates exactly this per row, one row per thread.  Such
// an item (R rows padded to rp, n columns) is stored as its nch chunks, each
// rp rows x 4 floats (16 bytes per row: one vector load), then the T tail
// columns rp floats each; chain-shaped widths store every column that way.
// Same element count (rp * n) as the column-major items.
__host__ __device__ __forceinline__ bool chain_shaped(int n) { return n <= 3 || (n >= 5 && n <= 7); }
__host__ __device__ __forceinline__ int64_t chunk_off(int n, int rp, int row, int k) {
  const int nch = chain_shaped(n) ? 0 : n >> 2;
  if (k < 4 * nch) return ((int64_t)(k >> 2) * rp + row) * 4 + (k & 3);
  return (int64_t)4 * nch * rp + (int64_t)(k - 4 * nch) * rp + row;
}

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

// Stage-1 epilogue per pipe (z = op(sum)).
enum ZEpi : int { Z_NONE = 0, Z_ROUND32 = 1, Z_SCALE = 2 };

constexpr int kSegRows = 64;      // max rows per stage-2 segment (leaf rows)
constexpr int kS1Rows = 256;      // max rank rows per stage-1 segment
constexpr int kSegThreads = 256;  // stage-2 CTA size (thread-group layout of gtab)
constexpr int kS1Threads = 128;   // stage-1 CTA size
constexpr int kS1Threads32 = 64;  // stage-1 CTA size for widened-FP32-only stage 1 (<= 256 rows)
constexpr int kSegWMax = 2048;    // columns of g staged in shared memory per tile (stage 2)
constexpr int kS1WMax = 1024;     // max columns per stage-1 segment chunk
#ifndef HMX_S1X_ROWS
#define HMX_S1X_ROWS 128
#endif
constexpr int kS1ExactRows = HMX_S1X_ROWS;  // m1-single stage 1: rank rows per CTA (one thread each)
#ifndef HMX_CHAIN_WARPS_MIXED
#define HMX_CHAIN_WARPS_MIXED 6
#endif
constexpr int kChainWarpsMixed = HMX_CHAIN_WARPS_MIXED;
constexpr int kChainRunsMax = 1024;  // most runs of a stage-2 FP32 part with SGEMV-order chain lanes (meta in shared memory)  // SGEMV-order stage 2: most chain warps beside widened warps in one CTA
constexpr int kSgemvBlock = 1024; // OpenBLAS SGEMV-T column blocking: 4096 columns = 1024 chunks

// Device-visible plan (passed by value to kernels).
struct DevPlan {
  int32_t n;
  int32_t row_begin, row_end;     // rows computed by this plan
  int32_t pipe;
  const Seg* seg1;                // stage-1 segments (CTA order)
  const Seg* seg2;                // stage-2 segments (row order)
  int32_t n_seg1, n_seg2;
  const Run* runs;
  const double* blob64;
  const float* blob32;
  int32_t f32mode1, f32mode2;
  int32_t zepi;
  int32_t s1_narrow;              // every stage-1 segment is widened FP32: 64-thread CTAs
  int32_t s2_deep;                // FP64-accumulating stage 2 with an FP64 part: deep pipeline
  int32_t s1_exact;               // m1-single: stage 1 in SGEMV order (1: s1_exact_kernel, 2: s1_exact4_kernel)
  int32_t chain_exact;            // stage-2 FP32-accumulated items in SGEMV order (chain_stream)
  int32_t chain_warps;            // most chain warps (groups) of any stage-2 segment
  int32_t n_seg1_local;           // leading stage-1 segments reading only x[row_begin, row_end)
  const int32_t* gtab;            // item-aligned FP32 group boundaries (stage 2)
  const double* zscale;           // d per z entry (methods 2, 3)
  const uint8_t* zkind;           // m1-single: SGEMV row kernel (4, 2, 1) per z entry
  double* z;
  double* part;                   // stage-1 chunk partials
  uint32_t* red_count;            // stage-1 arrival counters
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
  const int* skip;      // if non-null and *skip != 0 the launch is a no-op (solver guards)
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
