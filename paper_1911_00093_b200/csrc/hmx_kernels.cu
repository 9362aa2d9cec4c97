// sm_100a kernels of the H-matrix vector product.  See hmx_internal.cuh for
// the data layout; precision pipelines follow reference
// pkg/src/hmx/matvec.py:55-110 (table in SURVEY.md s0.1):
//
//   pipe  stage 1: z = Vt x                    stage 2: per item partial
//   m1d   f64                                  f64
//   m1s   f32 data . f32(x), f32 acc, z f32    dense A32.x32 f32-acc; U32.z32 f32-acc
//   m1m   f32 widened . x, f64 acc, z -> f32   dense widened f64; U32.z32 f32-acc
//   m2d   f64, z *= d                          f64
//   m2s   f32 widened . widen(f32(x)), z *= d  dense A32.x32 f32-acc; U widened f64
//   m2m   f32 widened . x, z *= d              dense widened f64; U widened f64
//   m3    hi f64 / lo f32 widened, z *= d      dense f64; U_hi f64; U_lo widened f64
//
// Every f32-accumulated partial is widened once and added in f64.
#include <algorithm>
#include <type_traits>

#include "hmx_kernels.cuh"

#ifndef HMX_MIXED_MINB
#define HMX_MIXED_MINB 4
#endif
#ifndef HMX_FIFO_BATCHES_MIXED
#define HMX_FIFO_BATCHES_MIXED 3  // chain lanes' FIFO depth (batches) in parts with widened warps (A/B at config 4: 2: +3 %, 4: +5 % on m1-mixed stage 2)
#endif
#ifndef HMX_FIFO_BATCHES_ALL32
#define HMX_FIFO_BATCHES_ALL32 3  // ... in all-chain parts (m1-single: eight chain warps, three CTAs per SM)
#endif
#ifndef HMX_S1X_WIN
#define HMX_S1X_WIN 8  // s1_exact_kernel: chunk loads per batch and thread
#endif
#ifndef HMX_CHAIN_PAIR
#define HMX_CHAIN_PAIR 0  // chain lanes: reduce the A and B chunk of a pair after one wait
#endif
#ifndef HMX_EXACT_MINB_ALL32
#define HMX_EXACT_MINB_ALL32 3
#endif
#ifndef HMX_EXACT_MINB
#define HMX_EXACT_MINB 3  // CTAs per SM of the SGEMV-order stage-2 kernels with <= 5 chain warps (registers; FIFOs)
#endif

namespace hmx {

enum Out : int { OUT_Y = 0, OUT_Z = 1 };

// a / b for the small non-negative integers of the thread-group arithmetic
// (0 <= a <= 2048 * 257, 1 <= b <= 256): (a + 0.5) / b is at least 0.5 / b away
// from an integer, far more than the rounding of the reciprocal and the
// product (checked exhaustively over that range).  A runtime integer
// division costs ~45 instructions per thread at every CTA start; this ~5.
__device__ __forceinline__ int fast_div(int a, int b) {
  return (int)(((float)a + 0.5f) * __frcp_rn((float)b));
}

// Shared-memory slot of an FP32-accumulated column: the FP32 source value in
// the low word, 1 in the high word on the first column of an item.
__device__ __forceinline__ double acc32_slot(float g, bool start) {
  return __hiloint2double(start ? 1 : 0, __float_as_int(g));
}

// 8-byte asynchronous global -> shared copies (the x / z segments of a tile)
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// Stage a tile [tc0, tc0+tw) of one part's source vector g (x segments and z
// vectors, in item order) into shared memory with cp.async; FP32-accumulated
// columns are then rewritten as acc32_slot and FP32-shadow columns rounded
// (fl: scratch flags, bit 0 item start, bit 1 FP32 item).  A single run
// (every stage-1 segment) is a contiguous copy.  Otherwise the runs are first
// expanded into a per-column source index in shared memory, so every
// column's copy is independent (no dependent run lookups).
constexpr int32_t kTagZ = 1 << 30, kTagRound = 1 << 29, kIdxMask = kTagRound - 1;
template <bool FLAGS, int NT, int WMAX>
__device__ __forceinline__ void gather_g(const DevPlan& P, const Run* __restrict__ runs, int nrun,
                                         int tc0, int tw, const double* __restrict__ x,
                                         double* gs, uint8_t* fl, int32_t* sidx) {
  constexpr int PER = WMAX / NT;  // columns per thread
  if (nrun == 1) {
    const Run r = runs[0];
    const double* src = ((r.flags & RUN_Z) ? P.z : x) + r.src + (tc0 - r.col0);
    const bool rnd = (r.flags & RUN_ROUND) != 0;
    const bool f32 = FLAGS && (r.flags & RUN_ACC32);
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int c = threadIdx.x + u * NT;
      if (c < tw) cp_async8(gs + c, src + c);
    }
    cp_async_wait_all();
    if (rnd || f32) {
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int c = threadIdx.x + u * NT;
        if (c < tw) {
          const double g = gs[c];
          gs[c] = f32 ? acc32_slot((float)g, tc0 + c == r.col0) : (double)(float)g;
        }
      }
    }
    return;
  }
  // runs whose columns meet the tile: scatter their source indices
  for (int j = threadIdx.x; j < nrun; j += NT) {
    const Run r = runs[j];
    const int lo = max(r.col0, tc0), hi = min(r.col0 + r.width, tc0 + tw);
    const int32_t tag = ((r.flags & RUN_Z) ? kTagZ : 0) | ((r.flags & RUN_ROUND) ? kTagRound : 0);
    const uint8_t f32 = (r.flags & RUN_ACC32) ? 2 : 0;
    for (int col = lo; col < hi; ++col) {
      sidx[col - tc0] = (r.src + (col - r.col0)) | tag;
      if constexpr (FLAGS) fl[col - tc0] = (uint8_t)((col == r.col0 ? 1 : 0) | f32);
    }
  }
  __syncthreads();
  const double* __restrict__ z = P.z;
  int32_t id[PER];
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int c = threadIdx.x + u * NT;
    id[u] = c < tw ? sidx[c] : 0;
    if (c < tw) cp_async8(gs + c, ((id[u] & kTagZ) ? z : x) + (id[u] & kIdxMask));
  }
  cp_async_wait_all();
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int c = threadIdx.x + u * NT;
    if (c < tw) {
      const uint8_t f = FLAGS ? fl[c] : 0;
      if (FLAGS && (f & 2)) gs[c] = acc32_slot((float)gs[c], f & 1);
      else if (id[u] & kTagRound) gs[c] = (double)(float)gs[c];
    }
  }
}

__device__ __forceinline__ double z_epilogue(const DevPlan& P, double s, int zi) {
  if (P.zepi == Z_ROUND32) return (double)(float)s;   // FP32 intermediate (matvec.py:68-72)
  if (P.zepi == Z_SCALE) return s * P.zscale[zi];      // z *= diag (matvec.py:81, :88, :92)
  return s;
}

// FP32-accumulated items: each row's value in OpenBLAS SGEMV-T's order,
// widened once and added in FP64 (reference matvec.py:57, :73, then :106).
// Explicit _rn intrinsics: nothing is contracted or reassociated.
//
// Stage 2 gives these items to the lanes of the chain warps (chain_lane
// below): slots of rp / 4 lanes, four rows per lane, each slot one thread
// group of the segment (hmx_plan.cu deals the items to the groups and lays
// every group's items out contiguously, widest first).  A lane streams its
// slot's columns through a private cp.async FIFO in shared memory
// (ChainFifo) and reads back only its own copies: no barrier is shared
// between lanes or warps.
__device__ __forceinline__ float4 fma4(float4 a, float4 g, float4 c) {
  return make_float4(__fmaf_rn(a.x, g.x, c.x), __fmaf_rn(a.y, g.y, c.y), __fmaf_rn(a.z, g.z, c.z),
                     __fmaf_rn(a.w, g.w, c.w));
}
__device__ __forceinline__ float4 mad4(float4 a, float4 g, float4 c) {  // multiply, then add
  return make_float4(__fadd_rn(c.x, __fmul_rn(a.x, g.x)), __fadd_rn(c.y, __fmul_rn(a.y, g.y)),
                     __fadd_rn(c.z, __fmul_rn(a.z, g.z)), __fadd_rn(c.w, __fmul_rn(a.w, g.w)));
}
__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}
__device__ __forceinline__ float hsum4(float4 l) { return __fadd_rn(__fadd_rn(l.x, l.y), __fadd_rn(l.z, l.w)); }
__device__ __forceinline__ float4 ld_chunk(const float* p) {
  float4 r;  // L1-allocating: a thread's A and B chunks share 32-byte sectors
  asm volatile("ld.global.nc.L1::evict_first.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ float ld_one(const float* p) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ void chain_bar(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int kMetaW = 12;  // run meta in shared memory: col0 << 12 | width

// One row of an n-wide item in OpenBLAS SGEMV-T's order.  X4(c): the row's
// columns 4c .. 4c+3; E(k): its column k; G(k): the FP32 source value of the
// item's column k.
// `kind`: which OpenBLAS SGEMV-T row kernel computes this row of its block
// (sgemv_row_kind): 16, 8, 4 = the 16-, 8- and 4-row kernels (A/B FMA
// chains; rows shorter than 8 differ between them), 2 = the two-row
// remainder kernel (one 4-lane accumulator, multiply then add), 1 = the
// one-row remainder kernel (A/B, multiply then add).  All end with
// (l0 + l1) + (l2 + l3) and the same tail rule (tools/fp32_accum_emulation.py
// sgemv_kind: bitwise numpy's own for every row count 2..64, widths 1..48).
template <typename XF, typename EF, typename GF>
__device__ __forceinline__ float chain_item(XF X4, EF E, GF G, int n, int kind) {
  auto G4 = [&](int c) { return make_float4(G(c), G(c + 1), G(c + 2), G(c + 3)); };
  auto Pr = [&](int k) { return __fmul_rn(E(k), G(k)); };  // rounded product
  auto F = [&](int k, float acc) { return __fmaf_rn(E(k), G(k), acc); };
  if (n == 1) return Pr(0);
  if (kind >= 4 && n <= 7 && n != 4) {  // short rows of the 16-, 8- and 4-row kernels
    if (n == 2 && kind != 16) return __fadd_rn(Pr(0), Pr(1));
    if (kind == 4 && n == 3) return F(2, F(0, Pr(1)));
    if (kind == 4 && n == 6) return __fadd_rn(__fadd_rn(Pr(0), F(1, Pr(2))), __fadd_rn(Pr(3), F(4, Pr(5))));
    if (kind == 4 && n == 7)
      return __fadd_rn(__fadd_rn(F(0, Pr(1)), F(4, Pr(5))), __fadd_rn(F(2, Pr(3)), Pr(6)));
    float v = 0.f;  // one forward FMA chain
    for (int k = 0; k < n; ++k) v = F(k, v);
    return v;
  }
  if (kind < 4) {  // the 2- and 1-row remainder kernels, short rows
    if (kind == 1 && n == 3) return F(2, F(0, Pr(1)));
    if (kind == 2 && n == 8)
      return __fadd_rn(__fadd_rn(__fadd_rn(Pr(0), Pr(1)), __fadd_rn(Pr(4), Pr(5))),
                       __fadd_rn(__fadd_rn(Pr(2), Pr(3)), __fadd_rn(Pr(6), Pr(7))));
    if (n <= 7 && n != 4) {  // a sequential multiply-then-add chain
      float v = Pr(0);
      for (int k = 1; k < n; ++k) v = __fadd_rn(v, Pr(k));
      return v;
    }
  }
  const int nch = n >> 2, T = n & 3, m = 4 * nch;
  float4 l;
  bool seq = false;  // sequential horizontal sum (one-row kernel, n <= 8)
  if (n == 8 && kind >= 4) {  // l_j = a_2j g_2j + a_2j+1 g_2j+1
    const float4 x0 = X4(0), x1 = X4(1);
    const float4 g0 = G4(0), g1 = G4(4);
    l = make_float4(__fadd_rn(__fmul_rn(x0.x, g0.x), __fmul_rn(x0.y, g0.y)),
                    __fadd_rn(__fmul_rn(x0.z, g0.z), __fmul_rn(x0.w, g0.w)),
                    __fadd_rn(__fmul_rn(x1.x, g1.x), __fmul_rn(x1.y, g1.y)),
                    __fadd_rn(__fmul_rn(x1.z, g1.z), __fmul_rn(x1.w, g1.w)));
  } else {
    // chunks into A (and B): four-row and one-row kernels: nch even: A = even
    // chunks, B = odd; nch odd: A = {0, 1, 3, 5, ..}, B = {2, 4, ..}; two-row
    // kernel: every chunk into A
    float4 A = make_float4(0.f, 0.f, 0.f, 0.f), B = A;
    int c = 0;
    if (kind >= 4) {
      if (nch & 1) {
        A = fma4(X4(0), G4(0), A);
        c = 1;
      }
      for (; c < nch; c += 2) {
        const float4 xa = X4(c), xb = X4(c + 1);
        A = fma4(xa, G4(4 * c), A);
        B = fma4(xb, G4(4 * c + 4), B);
      }
    } else if (kind == 2) {
      for (; c < nch; ++c) A = mad4(X4(c), G4(4 * c), A);
    } else {
      if (nch & 1) {
        A = mad4(X4(0), G4(0), A);
        c = 1;
      }
      for (; c < nch; c += 2) {
        const float4 xa = X4(c), xb = X4(c + 1);
        A = mad4(xa, G4(4 * c), A);
        B = mad4(xb, G4(4 * c + 4), B);
      }
    }
    l = add4(A, B);
    seq = kind == 1 && n <= 8;
  }
  float v = seq ? __fadd_rn(__fadd_rn(__fadd_rn(l.x, l.y), l.z), l.w) : hsum4(l);
  if (T == 1) {
    v = __fmaf_rn(E(m), G(m), v);
  } else if (T >= 2) {
    float tv = __fmul_rn(E(m + 1), G(m + 1));
    tv = __fmaf_rn(E(m), G(m), tv);
    if (T == 3) tv = __fmaf_rn(E(m + 2), G(m + 2), tv);
    v = __fadd_rn(v, tv);
  }
  return v;
}
// the same row of an item stored in chunk layout (chunk_off) at element
// offsets L4(o) (16-byte vector) / L1(o)
template <typename LD4, typename LD1, typename GF>
__device__ __forceinline__ float chain_item_chunked(LD4 L4, LD1 L1, GF G, int n, int rp, int p, int kind) {
  auto X4 = [&](int c) { return L4(4 * (c * rp + p)); };
  auto E = [&](int k) {
    if (chain_shaped(n)) return L1(k * rp + p);
    const int m = n & ~3;
    return k < m ? L1(4 * ((k >> 2) * rp + p) + (k & 3)) : L1(m * rp + (k - m) * rp + p);
  };
  return chain_item(X4, E, G, n, kind);
}

// Four rows of a column-major item at once, every row in the 16-row kernel
// (n < 8) or in the 16/8/4-row kernels (n >= 8): chain_item's order per row,
// the source values shared.  C(k): column k of the four rows.
__device__ __forceinline__ float4 fmas4(float4 a, float g, float4 c) {
  return make_float4(__fmaf_rn(a.x, g, c.x), __fmaf_rn(a.y, g, c.y), __fmaf_rn(a.z, g, c.z), __fmaf_rn(a.w, g, c.w));
}
__device__ __forceinline__ float4 muls4(float4 a, float g) {
  return make_float4(__fmul_rn(a.x, g), __fmul_rn(a.y, g), __fmul_rn(a.z, g), __fmul_rn(a.w, g));
}
template <typename CF, typename GF>
__device__ __forceinline__ float4 chain_quad(CF C, GF G, int n) {
  const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
  if (n == 1) return muls4(C(0), G(0));
  if (n <= 7 && n != 4) {  // one forward FMA chain per row
    float4 v = zero;
    for (int k = 0; k < n; ++k) v = fmas4(C(k), G(k), v);
    return v;
  }
  if (n == 8) {  // l_j = a_2j g_2j + a_2j+1 g_2j+1, then (l0 + l1) + (l2 + l3)
    float4 l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) l[j] = add4(muls4(C(2 * j), G(2 * j)), muls4(C(2 * j + 1), G(2 * j + 1)));
    return add4(add4(l[0], l[1]), add4(l[2], l[3]));
  }
  const int nch = n >> 2, T = n & 3, m = 4 * nch;
  // A[j], B[j]: lane j of the row accumulators (column 4c + j), the four rows side by side
  float4 A[4] = {zero, zero, zero, zero}, B[4] = {zero, zero, zero, zero};
  int c = 0;
  if (nch & 1) {
#pragma unroll
    for (int j = 0; j < 4; ++j) A[j] = fmas4(C(j), G(j), A[j]);
    c = 1;
  }
  for (; c < nch; c += 2) {
#pragma unroll
    for (int j = 0; j < 4; ++j) A[j] = fmas4(C(4 * c + j), G(4 * c + j), A[j]);
#pragma unroll
    for (int j = 0; j < 4; ++j) B[j] = fmas4(C(4 * c + 4 + j), G(4 * c + 4 + j), B[j]);
  }
  float4 v = add4(add4(add4(A[0], B[0]), add4(A[1], B[1])), add4(add4(A[2], B[2]), add4(A[3], B[3])));
  if (T == 1) {
    v = fmas4(C(m), G(m), v);
  } else if (T >= 2) {
    float4 tv = muls4(C(m + 1), G(m + 1));
    tv = fmas4(C(m), G(m), tv);
    if (T == 3) tv = fmas4(C(m + 2), G(m + 2), tv);
    v = add4(v, tv);
  }
  return v;
}

// The generic-kind version of chain_quad for items wider than 8 columns: row
// i of the four in SGEMV row kernel kind[i] (any of 16, 8, 4, 2, 1), chunk by
// chunk.  C(k) / G(k) as in chain_quad; before(c) is called before chunk c
// (and before the tail, c = nch) so the caller can stage the columns.
template <typename CF, typename GF, typename BF>
__device__ __forceinline__ float4 chain_quad_kinds(CF C, GF G, BF before, int n, const int* kind) {
  const int nch = n >> 2, T = n & 3, m = 4 * nch;
  const bool odd = nch & 1;
  float A[4][4], B[4][4];  // [row][accumulator lane]
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) A[i][j] = B[i][j] = 0.f;
  for (int c = 0; c < nch; ++c) {
    before(c);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float4 x4 = C(4 * c + j);
      const float g = G(4 * c + j);
      const float x[4] = {x4.x, x4.y, x4.z, x4.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const bool inA = kind[i] == 2 || (odd ? (c == 0 || (c & 1)) : !(c & 1));
        const float X = inA ? A[i][j] : B[i][j];
        const float Y = kind[i] >= 4 ? __fmaf_rn(x[i], g, X) : __fadd_rn(X, __fmul_rn(x[i], g));
        if (inA) A[i][j] = Y;
        else B[i][j] = Y;
      }
    }
  }
  float v[4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    v[i] = __fadd_rn(__fadd_rn(__fadd_rn(A[i][0], B[i][0]), __fadd_rn(A[i][1], B[i][1])),
                     __fadd_rn(__fadd_rn(A[i][2], B[i][2]), __fadd_rn(A[i][3], B[i][3])));
  if (T > 0) {
    before(nch);
    const float4 c0 = C(m), c1 = T >= 2 ? C(m + 1) : c0, c2 = T == 3 ? C(m + 2) : c0;
    const float x0[4] = {c0.x, c0.y, c0.z, c0.w}, x1[4] = {c1.x, c1.y, c1.z, c1.w}, x2[4] = {c2.x, c2.y, c2.z, c2.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (T == 1) {
        v[i] = __fmaf_rn(x0[i], G(m), v[i]);
      } else {
        float tv = __fmul_rn(x1[i], G(m + 1));
        tv = __fmaf_rn(x0[i], G(m), tv);
        if (T == 3) tv = __fmaf_rn(x2[i], G(m + 2), tv);
        v[i] = __fadd_rn(v[i], tv);
      }
    }
  }
  return make_float4(v[0], v[1], v[2], v[3]);
}

// A chain lane's private FIFO in shared memory.  The lanes of one slot
// (rp / 4 lanes, four rows each) stream the columns of their group --
// contiguous in the blob -- with 16-byte cp.async copies in BATCHES: the
// 4-column chunks of each item and its 1..3 tail columns, one commit group
// per batch, NB batch slots per lane.  A batch is consumed whole (one chunk
// of SGEMV's A/B accumulators, or the tail), so while one is reduced the
// other NB - 1 are in flight.  Every lane reads back only what it
// copied itself: nothing is synchronised between lanes.
constexpr int kMetaWide = 1 << 30;  // run meta: an FP64-accumulated (widened) item on a chain lane
__device__ __forceinline__ int meta_col0(int32_t m) { return (m >> kMetaW) & 0x3ffff; }
__device__ __forceinline__ int meta_width(int32_t m) { return m & ((1 << kMetaW) - 1); }
template <int NB>  // batch slots per lane
struct ChainFifo {
  static constexpr int kBytes = NB * 4 * 512;  // per chain warp: 16 bytes x 32 lanes per column
  const float* srcp;     // this lane's four rows of the next column to copy
  const float* fifo;     // this lane's 16 bytes of batch slot 0, column 0 (column u: + 128 u, slot b: + 512 b floats)
  uint32_t fifo_s;       // ... its shared-space address
  const int32_t* meta;   // run meta in shared memory
  int rp;
  int ij, je;            // next item to copy from / end of the lane's items
  int irem;              // columns of item ij not yet copied
  int ib = 0;            // batches copied or in flight
  int cb = 0;            // batches consumed
  int islot = 0;         // ib mod NB
  int cslot = 0;         // cb mod NB

  // copy the next batch (a chunk or the tail of item ij); ij < je
  __device__ __forceinline__ void issue() {
    const int cols = min(4, irem);
    const uint32_t dst = fifo_s + (uint32_t)islot * 2048u;
    if (cols == 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 512u * u), "l"(srcp + (int64_t)u * rp) : "memory");
    } else {
#pragma unroll
      for (int u = 0; u < 3; ++u)
        if (u < cols)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst + 512u * u), "l"(srcp + (int64_t)u * rp) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    ++ib;
    islot = islot == NB - 1 ? 0 : islot + 1;
    srcp += (int64_t)cols * rp;
    irem -= cols;
    if (irem == 0 && ++ij < je) irem = meta_width(meta[ij]);
  }
  __device__ __forceinline__ void start(const int32_t* m, int jb, int je_) {
    meta = m;
    ij = jb;
    je = je_;
    irem = jb < je_ ? meta_width(m[jb]) : 0;
    while (ib < NB && ij < je) issue();
  }
  // batch bt (cb <= bt < ib) has landed
  __device__ __forceinline__ void need(int bt) {
    const int pend = ib - bt;  // 1 + the batches copied after it
    if (NB >= 4 && pend >= 4) asm volatile("cp.async.wait_group 3;\n" ::: "memory");
    else if (pend >= 3) asm volatile("cp.async.wait_group 2;\n" ::: "memory");
    else if (pend == 2) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  }
  // batches < bt are consumed (bt - cb <= NB): refill their slots
  __device__ __forceinline__ void done(int bt) {
    cslot += bt - cb;
    if (cslot >= NB) cslot -= NB;
    cb = bt;
    while (ib - cb < NB && ij < je) issue();
  }
  // one more batch is consumed
  __device__ __forceinline__ void done1() {
    ++cb;
    cslot = cslot == NB - 1 ? 0 : cslot + 1;
    if (ij < je) issue();  // (ib - cb was NB - 1 or the stream is exhausted)
  }
  // column u of batch bt (cb <= bt < cb + NB), this lane's four rows
  __device__ __forceinline__ float4 col(int bt, int u) const {
    int sl = cslot + (bt - cb);
    if (sl >= NB) sl -= NB;
    return *reinterpret_cast<const float4*>(fifo + sl * 512 + u * 128);
  }
  // this lane's 16 bytes of column 0 of the batch being consumed
  __device__ __forceinline__ const float* cur() const { return fifo + cslot * 512; }
  // ... of the batch after it
  __device__ __forceinline__ const float* nxt() const { return fifo + (cslot == NB - 1 ? 0 : cslot + 1) * 512; }
};

// One chain lane: items jb .. je-1 of the part (meta / kbits in shared memory)
// are its slot's group; rows 4t .. 4t+3.  Adds the widened item values into
// b[0..3] (FP64, item order).  Every row's value is in OpenBLAS SGEMV-T's
// order (chain_quad: all rows in the 16-row kernel / 16-8-4-row kernels;
// otherwise chain_item / chain_quad_kinds per row kind).
template <int NB>
__device__ __forceinline__ void chain_lane(ChainFifo<NB>& F, const int32_t* meta, const uint32_t* kbits, int jb, int je,
                                           const double* gs, int rp, int t, double* b) {
  F.start(meta, jb, je);
  int j = jb;
  // (uniform trip count over the warp, so the slots stay converged item by item)
  while (__any_sync(0xffffffffu, j < je)) {
    if (j < je) {
      const int32_t mj = meta[j];
      const int c0 = meta_col0(mj), n = meta_width(mj);
      const double* gj = gs + c0;
      if (mj & kMetaWide) {
        // an FP64-accumulated item (FP32 data widened; reference matvec.py:59, :86):
        // batch by batch straight into the row sums
        auto L = [](const float* p, int u) { return *reinterpret_cast<const float4*>(p + u * 128); };
        for (int k0 = 0; k0 < n; k0 += 4) {
          F.need(F.cb);
          const float* p = F.cur();
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (k0 + u < n) {
              const float4 x = L(p, u);
              const double g = gj[k0 + u];
              b[0] = fma((double)x.x, g, b[0]);
              b[1] = fma((double)x.y, g, b[1]);
              b[2] = fma((double)x.z, g, b[2]);
              b[3] = fma((double)x.w, g, b[3]);
            }
          F.done1();
        }
        ++j;
        continue;
      }
      const uint32_t kb = kbits[j];
      auto G = [&](int q) { return __int_as_float(__double2loint(gj[q])); };
      const int b0 = F.cb;  // the item's first batch; column q sits in batch b0 + q / 4
      auto C = [&](int q) { return F.col(b0 + (q >> 2), q & 3); };
      const bool fast = (int)((kb >> (n < 8 ? 0 : 14)) & 127) >= rp;
      const int nch = n >> 2, T = n & 3, m = 4 * nch;
      const int nb = chain_shaped(n) ? 1 + (n > 4) : nch + (T > 0);  // batches of the item (== ceil(n / 4))
      float4 v;
      if (n <= 8) {
        F.need(b0 + nb - 1);
        if (fast) {
          v = chain_quad(C, G, n);
        } else {
          float r[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            auto E = [&](int q) {
              const float4 x = C(q);
              return i == 0 ? x.x : i == 1 ? x.y : i == 2 ? x.z : x.w;
            };
            auto X4 = [&](int c) { return make_float4(E(4 * c), E(4 * c + 1), E(4 * c + 2), E(4 * c + 3)); };
            r[i] = chain_item(X4, E, G, n, chain_row_kind(kb, 4 * t + i));
          }
          v = make_float4(r[0], r[1], r[2], r[3]);
        }
        F.done(b0 + nb);
      } else if (fast) {
        const float4 zero = make_float4(0.f, 0.f, 0.f, 0.f);
        float4 A[4] = {zero, zero, zero, zero}, B[4] = {zero, zero, zero, zero};
        auto L = [](const float* p, int u) { return *reinterpret_cast<const float4*>(p + u * 128); };
        int c = 0;
        if (nch & 1) {
          F.need(F.cb);
          const float* p = F.cur();
#pragma unroll
          for (int q = 0; q < 4; ++q) A[q] = fmas4(L(p, q), G(q), A[q]);
          F.done1();
          c = 1;
        }
        for (; c < nch; c += 2) {
#if HMX_CHAIN_PAIR
          // the A and the B chunk of a pair together (one wait, eight loads in flight)
          F.need(F.cb + 1);
          const float* pa = F.cur();
          const float* pb = F.nxt();
#pragma unroll
          for (int q = 0; q < 4; ++q) A[q] = fmas4(L(pa, q), G(4 * c + q), A[q]);
#pragma unroll
          for (int q = 0; q < 4; ++q) B[q] = fmas4(L(pb, q), G(4 * c + 4 + q), B[q]);
          F.done1();
          F.done1();
#else
          F.need(F.cb);
          const float* pa = F.cur();
#pragma unroll
          for (int q = 0; q < 4; ++q) A[q] = fmas4(L(pa, q), G(4 * c + q), A[q]);
          F.done1();
          F.need(F.cb);
          const float* pb = F.cur();
#pragma unroll
          for (int q = 0; q < 4; ++q) B[q] = fmas4(L(pb, q), G(4 * c + 4 + q), B[q]);
          F.done1();
#endif
        }
        v = add4(add4(add4(A[0], B[0]), add4(A[1], B[1])), add4(add4(A[2], B[2]), add4(A[3], B[3])));
        if (T > 0) {
          F.need(F.cb);
          const float* p = F.cur();
          if (T == 1) {
            v = fmas4(L(p, 0), G(m), v);
          } else {
            float4 tv = muls4(L(p, 1), G(m + 1));
            tv = fmas4(L(p, 0), G(m), tv);
            if (T == 3) tv = fmas4(L(p, 2), G(m + 2), tv);
            v = add4(v, tv);
          }
          F.done1();
        }
      } else {
        int kind[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) kind[i] = chain_row_kind(kb, 4 * t + i);
        auto before = [&](int c) {
          F.done(b0 + c);
          F.need(b0 + c);
        };
        v = chain_quad_kinds(C, G, before, n, kind);
        F.done(b0 + nb);
      }
      b[0] += (double)v.x;
      b[1] += (double)v.y;
      b[2] += (double)v.z;
      b[3] += (double)v.w;
      ++j;
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// Stage 1 of m1-single: z = Vt32 . x32 accumulated in FP32 (reference
// matvec.py:70, numpy -> OpenBLAS SGEMV-T), in SGEMV's own order: one thread
// per rank row over the cluster's whole width, 4096-column blocks each
// reduced by the A/B lane tree of hmx_internal.cuh (the tail rule in the last
// block), the block values added in order (one CTA per block; the last one
// to arrive adds them).  Rows stored in chunk layout (chunk_off), so a warp's
// 16-byte loads cover 32 consecutive rows.
__global__ void __launch_bounds__(kS1ExactRows) s1_exact_kernel(DevPlan P, const Seg* __restrict__ segs,
                                                                const double* __restrict__ x, const int* skip) {
  if (skip != nullptr && *skip != 0) return;
  asm volatile("griddepcontrol.launch_dependents;");
  __shared__ unsigned ticket;
  const Seg sg = segs[blockIdx.x];
  const int t = threadIdx.x;
  const Run run = P.runs[sg.run0];
  const int n = sg.W32, rp = (sg.R + 3) & ~3;
  const float* __restrict__ it = P.blob32 + sg.off32;
  const double* __restrict__ xs = x + run.src;
  // the FP32 source shadow (matvec.py:119): x rounded once, staged in shared
  // memory for the whole CTA (a block is at most 4096 columns wide)
  __shared__ __align__(16) float xs32[4 * kSgemvBlock];
  for (int c = t; c < n; c += kS1ExactRows) xs32[c] = (float)__ldg(xs + c);
  __syncthreads();
  auto G = [&](int c) { return xs32[c]; };
  auto G4 = [&](int c) { return *reinterpret_cast<const float4*>(xs32 + c); };
  float y = 0.f;
  const int kind = t < sg.R ? P.zkind[sg.row0 + t] : 16;
  if (t >= sg.R) {
    // (idle row: no loads; joins the barrier below)
  } else if (n <= 8) {  // short rows (chain-shaped, n = 4, n = 8): the per-kernel rules
    y = chain_item_chunked([&](int o) { return ld_chunk(it + o); }, [&](int o) { return ld_one(it + o); }, G, n, rp, t, kind);
  } else {
    // this CTA's 4096-column block: the A/B lane tree (kinds 16/8/4: FMA
    // chains; 1: multiply then add; 2: one accumulator, multiply then add),
    // chunks loaded kS1Win at a time (all loads of a batch in flight before
    // the first is consumed -- measured faster than a rolling refill)
    const int nch = n >> 2, T = n & 3;
    const bool fm = kind >= 4, one = kind == 2, odd = nch & 1;
    const float* ch = it + 4 * t;  // chunk c at ch[4 c rp]
    float4 A = make_float4(0.f, 0.f, 0.f, 0.f), B = A;
    auto step = [&](const float4& x, int cc) {
      const bool inA = one || (odd ? (cc == 0 || (cc & 1)) : !(cc & 1));
      const float4 g = G4(4 * cc);
      const float4 X = inA ? A : B;
      const float4 Y = fm ? fma4(x, g, X)
                          : make_float4(__fadd_rn(X.x, __fmul_rn(x.x, g.x)), __fadd_rn(X.y, __fmul_rn(x.y, g.y)),
                                        __fadd_rn(X.z, __fmul_rn(x.z, g.z)), __fadd_rn(X.w, __fmul_rn(x.w, g.w)));
      if (inA) A = Y;
      else B = Y;
    };
    constexpr int kS1Win = HMX_S1X_WIN;
    for (int c = 0; c < nch; c += kS1Win) {
      float4 w[kS1Win];
#pragma unroll
      for (int u = 0; u < kS1Win; ++u)
        if (c + u < nch) w[u] = ld_chunk(ch + (int64_t)4 * (c + u) * rp);
#pragma unroll
      for (int u = 0; u < kS1Win; ++u)
        if (c + u < nch) step(w[u], c + u);
    }
    const float4 l = make_float4(__fadd_rn(A.x, B.x), __fadd_rn(A.y, B.y), __fadd_rn(A.z, B.z),
                                 __fadd_rn(A.w, B.w));
    y = __fadd_rn(__fadd_rn(l.x, l.y), __fadd_rn(l.z, l.w));
    if (T > 0) {
      const int m = 4 * nch;
      const float* tl = it + (int64_t)m * rp + t;
      if (T == 1) {
        y = __fmaf_rn(ld_one(tl), G(m), y);
      } else {
        float tv = __fmul_rn(ld_one(tl + rp), G(m + 1));
        tv = __fmaf_rn(ld_one(tl), G(m), tv);
        if (T == 3) tv = __fmaf_rn(ld_one(tl + 2 * rp), G(m + 2), tv);
        y = __fadd_rn(y, tv);
      }
    }
  }
  if (sg.nchunks == 1) {
    if (t < sg.R) P.z[sg.row0 + t] = (double)y;
    return;
  }
  // one 4096-column block per CTA: the last-arriving CTA adds the block
  // values in block order (y = (b0 + b1) + ..., as SGEMV)
  if (t < sg.R) P.part[sg.part_off + sg.chunk * sg.R + t] = (double)y;
  __threadfence();
  __syncthreads();
  if (t == 0) ticket = atomicAdd(P.red_count + sg.red, 1u);
  __syncthreads();
  if (ticket != (unsigned)(sg.nchunks - 1)) return;
  __threadfence();
  if (t < sg.R) {
    float f = (float)__ldcg(P.part + sg.part_off + t);
    for (int ch = 1; ch < sg.nchunks; ++ch) f = __fadd_rn(f, (float)__ldcg(P.part + sg.part_off + ch * sg.R + t));
    P.z[sg.row0 + t] = (double)f;
  }
  if (t == 0) P.red_count[sg.red] = 0u;  // ready for the next matvec
}

// The same stage 1 for SMALL plans (P.s1_exact == 2: under ~1 GB of stage-1
// payload, where the long rows of the wide column clusters bound the launch;
// config 3: 204 -> 164 us, config 2: 68 -> 52 us; at config 4 the one-thread
// kernel above is faster, 0.33 against 0.72 ms).  Per rank
// row, 4096-column blocks each reduced by the A/B lane tree of
// hmx_internal.cuh (the tail rule in the last block), the block values added
// in order (one CTA per block; the last one to arrive adds them).  FOUR
// threads per row: thread (row t, lane j) owns lane j of the row's A and B
// accumulators, i.e. column 4c + j of every chunk c -- a quarter of the row's
// serial chain each, and the 32 threads of a warp read 8 rows x 16 bytes of
// a chunk (chunk layout, chunk_off) as one 128-byte line.  The lanes meet in
// (l0 + l1) + (l2 + l3) through shuffles; lane 0 adds the tail and writes.
constexpr int kS1ExactThreads = 4 * kS1ExactRows;
__global__ void __launch_bounds__(kS1ExactThreads) s1_exact4_kernel(DevPlan P, const Seg* __restrict__ segs,
                                                                   const double* __restrict__ x, const int* skip) {
  if (skip != nullptr && *skip != 0) return;
  asm volatile("griddepcontrol.launch_dependents;");
  __shared__ unsigned ticket;
  const Seg sg = segs[blockIdx.x];
  const int tid = threadIdx.x;
  const int t = tid >> 2, j = tid & 3;
  const Run run = P.runs[sg.run0];
  const int n = sg.W32, rp = (sg.R + 3) & ~3;
  const float* __restrict__ it = P.blob32 + sg.off32;
  const double* __restrict__ xs = x + run.src;
  // the FP32 source shadow (matvec.py:119): x rounded once, staged in shared
  // memory for the whole CTA (a block is at most 4096 columns wide)
  __shared__ __align__(16) float xs32[4 * kSgemvBlock];
  for (int c = tid; c < n; c += kS1ExactThreads) xs32[c] = (float)__ldg(xs + c);
  __syncthreads();
  auto G = [&](int c) { return xs32[c]; };
  const bool row = t < sg.R;
  const int kind = row ? P.zkind[sg.row0 + t] : 16;
  float y = 0.f;
  if (n <= 8) {  // short rows (chain-shaped, n = 4, n = 8): the per-kernel rules, lane 0
    if (row && j == 0)
      y = chain_item_chunked([&](int o) { return ld_chunk(it + o); }, [&](int o) { return ld_one(it + o); }, G, n, rp, t,
                             kind);
  } else {
    // this CTA's 4096-column block: lane j of the A/B tree (kinds 16/8/4: FMA
    // chains; 1: multiply then add; 2: one accumulator, multiply then add),
    // chunks loaded kS1Win at a time (all loads of a batch in flight before
    // the first is consumed)
    const int nch = n >> 2, T = n & 3;
    const bool fm = kind >= 4, one = kind == 2, odd = nch & 1;
    const float* ch = it + 4 * t + j;  // this thread's element of chunk c at ch[4 c rp]
    float a = 0.f, b = 0.f;
    constexpr int kS1Win = HMX_S1X_WIN;
    for (int c = 0; c < nch; c += kS1Win) {
      float w[kS1Win];
#pragma unroll
      for (int u = 0; u < kS1Win; ++u)
        if (row && c + u < nch) w[u] = ld_one(ch + (int64_t)4 * (c + u) * rp);
#pragma unroll
      for (int u = 0; u < kS1Win; ++u)
        if (row && c + u < nch) {
          const int cc = c + u;
          const bool inA = one || (odd ? (cc == 0 || (cc & 1)) : !(cc & 1));
          const float g = G(4 * cc + j);
          const float X = inA ? a : b;
          const float Y = fm ? __fmaf_rn(w[u], g, X) : __fadd_rn(X, __fmul_rn(w[u], g));
          if (inA) a = Y;
          else b = Y;
        }
    }
    // l_j = A_j + B_j; (l0 + l1) + (l2 + l3) across the row's four lanes
    // (IEEE addition commutes, so every lane holds the same sums)
    const float l = __fadd_rn(a, b);
    const float s2 = __fadd_rn(l, __shfl_xor_sync(0xffffffffu, l, 1));
    y = __fadd_rn(s2, __shfl_xor_sync(0xffffffffu, s2, 2));
    if (T > 0 && row && j == 0) {
      const int m = 4 * nch;
      const float* tl = it + (int64_t)m * rp + t;
      if (T == 1) {
        y = __fmaf_rn(ld_one(tl), G(m), y);
      } else {
        float tv = __fmul_rn(ld_one(tl + rp), G(m + 1));
        tv = __fmaf_rn(ld_one(tl), G(m), tv);
        if (T == 3) tv = __fmaf_rn(ld_one(tl + 2 * rp), G(m + 2), tv);
        y = __fadd_rn(y, tv);
      }
    }
  }
  const bool writer = row && j == 0;
  if (sg.nchunks == 1) {
    if (writer) P.z[sg.row0 + t] = (double)y;
    return;
  }
  // one 4096-column block per CTA: the last-arriving CTA adds the block
  // values in block order (y = (b0 + b1) + ..., as SGEMV)
  if (writer) P.part[sg.part_off + sg.chunk * sg.R + t] = (double)y;
  __threadfence();
  __syncthreads();
  if (tid == 0) ticket = atomicAdd(P.red_count + sg.red, 1u);
  __syncthreads();
  if (ticket != (unsigned)(sg.nchunks - 1)) return;
  __threadfence();
  if (writer) {
    float f = (float)__ldcg(P.part + sg.part_off + t);
    for (int ch2 = 1; ch2 < sg.nchunks; ++ch2) f = __fadd_rn(f, (float)__ldcg(P.part + sg.part_off + ch2 * sg.R + t));
    P.z[sg.row0 + t] = (double)f;
  }
  if (tid == 0) P.red_count[sg.red] = 0u;  // ready for the next matvec
}

// One CTA = one segment: rows [row0, row0+R) of a column-major item stream.
// DEEP: stage 2 with an FP64 part, 12 FP64 columns in flight per thread at 3
// CTAs per SM (80 registers) instead of 8 at 4 (A/B on config 4: m1-double
// stage 2 -1.1 %, m2-double -2.4 %; FP32-only stage 2 prefers 8 at 4)
// EXACT (stage 2 with FP32-accumulated items): those items in SGEMV's order
// (chain_lane); otherwise one FP32 chain per (row, item) (HMX_PLAN_FP32_CHAIN).
// Separate instantiations keep each one's register allocation its own.
// XMINB: CTAs per SM of an EXACT instantiation: 3 (80 registers; the chain
// warps' FIFOs -- 6 KB each -- fit beside the static shared memory).
template <int F32MODE, int OUT, int NT, bool DEEP = false, bool EXACT = false, int XMINB = HMX_EXACT_MINB>
__global__ void __launch_bounds__(NT, DEEP ? 3 : (OUT == OUT_Y && F32MODE != F32_ALL64) ? (EXACT ? XMINB : HMX_MIXED_MINB) : 1024 / NT) seg_kernel(DevPlan P, const Seg* __restrict__ segs,
                                                          const double* __restrict__ x, S2Out out) {
  // stage 1 segments have a single run (no index expansion) and <= 1024 columns
  constexpr int WMAX = OUT == OUT_Z ? kS1WMax : kSegWMax;
  constexpr int D64 = DEEP ? 12 : 8;
  __shared__ double gs[WMAX];
  // XS: a stage-2 kernel with SGEMV-order chain lanes.  Its plans hold no FP64
  // part (pipes m1-single, m1-mixed, m2-single: FP32 storage throughout), and
  // its gather flags share red32 (flags: gather phases; red32: after them), so
  // three CTAs and their chain FIFOs fit an SM.
  constexpr bool XS = EXACT && OUT == OUT_Y && F32MODE != F32_ALL64;
  // the chain lanes' column FIFOs (stage-2 FP32 kernels; dynamic: ChainFifo<NB>::kBytes x P.chain_warps)
  extern __shared__ __align__(128) float chain_buf[];
  __shared__ uint8_t fl_own[XS ? 1 : WMAX];
  __shared__ int32_t sidx_own[(OUT == OUT_Z || (EXACT && F32MODE != F32_ALL64)) ? 1 : kSegWMax];
  __shared__ double red64[XS ? 1 : 2 * NT];
  __shared__ double red32[4 * NT];
  uint8_t* fl = XS ? reinterpret_cast<uint8_t*>(red32) : fl_own;
  // XS: the gather's source-index scratch shares the chain FIFOs' memory (the
  // FIFOs start after the gather); the chain items' meta / row-kernel bounds
  // then live in red32 (plans keep <= kChainRunsMax runs in such a part)
  int32_t* sidx = XS ? reinterpret_cast<int32_t*>(chain_buf) : sidx_own;
  __shared__ double wred[2][NT / 32];
  __shared__ unsigned ticket;

  if (out.skip != nullptr && *out.skip != 0) return;  // guarded launch (solver)
  // stage 1: let the dependent stage-2 grid launch as soon as every stage-1
  // CTA has started (its CTAs then fill the SMs stage 1's tail frees and
  // prefetch; griddepcontrol.wait in stage 2 still waits for all of stage 1).
  // The 64-thread FP32 stage 1 triggers at CTA end instead (measured).
  if (OUT == OUT_Z && NT >= 128) asm volatile("griddepcontrol.launch_dependents;");
  const Seg sg = segs[blockIdx.x];
  const int R = sg.R;
  const int tid = threadIdx.x;
  const uint64_t pol = policy_evict_first();

  // ---------------- FP64 part: 2 rows x 16 bytes per thread
  const int rp64 = (R + 1) & ~1;
  const int tpg64 = rp64 >> 1;
  const int g64 = fast_div(NT, tpg64);
  const int q64 = fast_div(tid, tpg64), p64 = tid - q64 * tpg64;
  double a0 = 0.0, a1 = 0.0;
  if constexpr (!XS) {
  for (int tc0 = 0; tc0 < sg.W64; tc0 += WMAX) {
    const int tw = min(WMAX, sg.W64 - tc0);
    const bool act = q64 < g64;
    const int cb = act ? fast_div(tw * q64, g64) : 0;
    const int ce = act ? fast_div(tw * (q64 + 1), g64) : 0;
    const double* __restrict__ col = P.blob64 + sg.off64 + (int64_t)tc0 * rp64 + 2 * p64;
    // D64 columns in flight per thread (stage 2, FP64-only kernels: deeper,
    // at fewer resident CTAs), predicated at the end of the range (a short
    // range -- small segments -- is still one batch, never a serial chain).
    // The first batch is independent of g: it is issued before the gather
    // (and, in stage 2, before waiting on stage 1) to hide one latency.
    double2 m[D64];
    int c = cb;
#pragma unroll
    for (int u = 0; u < D64; ++u)
      if (c + u < ce) m[u] = ld_stream(col + (int64_t)(c + u) * rp64, pol);
    if (OUT == OUT_Y && tc0 == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    gather_g<false, NT, WMAX>(P, P.runs + sg.run0, sg.nrun64, tc0, tw, x, gs, fl, sidx);
    __syncthreads();
    // rolling: each register is refilled with the column D64 ahead right
    // after it is consumed (D64 loads stay in flight); the tail is predicated
    for (;;) {
      if (c + 2 * D64 <= ce) {
#pragma unroll
        for (int u = 0; u < D64; ++u) {
          const double g = gs[c + u];
          a0 = fma(m[u].x, g, a0);
          a1 = fma(m[u].y, g, a1);
          m[u] = ld_stream(col + (int64_t)(c + D64 + u) * rp64, pol);
        }
      } else {
#pragma unroll
        for (int u = 0; u < D64; ++u) {
          if (c + u < ce) {
            const double g = gs[c + u];
            a0 = fma(m[u].x, g, a0);
            a1 = fma(m[u].y, g, a1);
          }
          if (c + D64 + u < ce) m[u] = ld_stream(col + (int64_t)(c + D64 + u) * rp64, pol);
        }
      }
      c += D64;
      if (c >= ce) break;
    }
  }

  // FP64-part partials go to shared memory now (frees their registers for
  // the FP32 part; red64 is read only in the epilogue)
  if (sg.W64 > 0 && q64 < g64) {
    red64[q64 * rp64 + 2 * p64] = a0;
    red64[q64 * rp64 + 2 * p64 + 1] = a1;
  }
  }

  // ---------------- FP32 part: 4 rows x 16 bytes per thread
  const int rp32 = (R + 3) & ~3;
  const int tpg32 = rp32 >> 2;
  int g32 = fast_div(NT, tpg32);
  int q32 = fast_div(tid, tpg32), p32 = tid - q32 * tpg32;
  // Stage-2 parts with a group table (every part of <= kSegWMax columns):
  // FP64-accumulated (widened) items on threads [0, wbc), 4 rows per thread
  // as above; the FP32-accumulated items on the warps of threads [wbc, NT),
  // each item evaluated in SGEMV's own order (chain_lane), 4 rows per lane.
  // wbc (plan: sg.chunk) is warp-aligned, so no warp runs both loops.
  bool chain_thr = false, chain_warp = false;
  int cg0 = 0, cg1 = 0;
  constexpr int NB = F32MODE == F32_ALL32 ? HMX_FIFO_BATCHES_ALL32 : HMX_FIFO_BATCHES_MIXED;
  ChainFifo<NB> cfifo;
  if constexpr (F32MODE == F32_MIXED && OUT == OUT_Y) {
    // (HMX_PLAN_FP32_CHAIN plans: one FP32 FMA chain per (row, item), 4 rows
    // per thread on both sides of the warp-aligned split at wb = sg.chunk)
    const int wb = sg.chunk;
    if (!EXACT && wb > 0 && sg.gtab >= 0) {
      const int ga = fast_div(wb, tpg32), gb = fast_div(NT - wb, tpg32);
      g32 = ga + gb;
      if (tid < wb) {
        if (q32 >= ga) q32 = g32;  // idle
      } else {
        const int u = tid - wb;
        const int qb = fast_div(u, tpg32);
        p32 = u - qb * tpg32;
        q32 = qb < gb ? ga + qb : g32;
      }
    }
  }
  if constexpr (EXACT && F32MODE != F32_ALL64 && OUT == OUT_Y) {
    if (sg.gtab >= 0) {
      const int wbc = sg.chunk;  // (0: every warp is a chain warp)
      // chain lanes: slots of tpg32 lanes inside each warp, one group per slot
      const int nslot = min(fast_div(32, tpg32), 8);
      const int ga = fast_div(wbc, tpg32), gb = ((NT - wbc) >> 5) * nslot;
      g32 = ga + gb;
      if (tid < wbc) {
        if (q32 >= ga) q32 = g32;  // idle
      } else {
        chain_warp = true;
        const int cw = (tid - wbc) >> 5, lane = tid & 31;
        const int slot = fast_div(lane, tpg32);
        p32 = lane - slot * tpg32;
        q32 = slot < nslot ? ga + cw * nslot + slot : g32;
        chain_thr = q32 < g32;
        if (chain_thr) {
          cg0 = P.gtab[sg.gtab + q32];
          cg1 = P.gtab[sg.gtab + q32 + 1];
          cfifo.rp = rp32;
          cfifo.srcp = P.blob32 + sg.off32 + (int64_t)cg0 * rp32 + 4 * p32;
          cfifo.fifo = chain_buf + (size_t)cw * (ChainFifo<NB>::kBytes / 4) + 4 * lane;
          cfifo.fifo_s = smem_addr(cfifo.fifo);
        }
      }
    }
  }
  double b[4] = {0.0, 0.0, 0.0, 0.0};
  float b32[4] = {0.f, 0.f, 0.f, 0.f};
  // the part holds FP64-accumulated items first, then FP32-accumulated ones
  // from column c32 on (plan: gtab after the group cuts, or alone at -2-gtab)
  int c32 = sg.W32;
  if constexpr (F32MODE == F32_ALL32) c32 = 0;
  if constexpr (F32MODE == F32_MIXED) {
    if (sg.gtab >= 0) c32 = P.gtab[sg.gtab + g32 + 1];
    else if (sg.gtab <= -2) c32 = P.gtab[-2 - sg.gtab];
  }
  // widened FP32 data, FP64 accumulation
  auto consume64 = [&](const float4& v, int cc) {
    const double g = gs[cc];
    b[0] = fma((double)v.x, g, b[0]);
    b[1] = fma((double)v.y, g, b[1]);
    b[2] = fma((double)v.z, g, b[2]);
    b[3] = fma((double)v.w, g, b[3]);
  };
  // FP32 chain per (row, item): the gathered slot holds the FP32 source in
  // its low word and "first column of an item" in its high word
  auto consume32 = [&](const float4& v, int cc) {
    const double e = gs[cc];
    // item start: close the previous FP32 partial (a real branch: the
    // compiler would otherwise predicate the flush onto every column)
    if (OUT == OUT_Y && __double2hiint(e) != 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        b[i] += (double)b32[i];
        b32[i] = 0.f;
      }
      __syncwarp(__activemask());
    }
    const float gf = __int_as_float(__double2loint(e));
    b32[0] = fmaf(v.x, gf, b32[0]);
    b32[1] = fmaf(v.y, gf, b32[1]);
    b32[2] = fmaf(v.z, gf, b32[2]);
    b32[3] = fmaf(v.w, gf, b32[3]);
  };
  for (int tc0 = 0; tc0 < sg.W32; tc0 += WMAX) {
    const int tw = min(WMAX, sg.W32 - tc0);
    const bool act = q32 < g32;
    int cb = act ? fast_div(tw * q32, g32) : 0;
    int ce = act ? fast_div(tw * (q32 + 1), g32) : 0;
    if (F32MODE != F32_ALL64 && OUT == OUT_Y && sg.gtab >= 0 && act) {
      // FP32-accumulated items are never split between groups: every item
      // row is one FP32 chain (reference: FP32 GEMV per block, matvec.py:57, :73)
      cb = P.gtab[sg.gtab + q32];
      ce = P.gtab[sg.gtab + q32 + 1];
      if (chain_thr) ce = cb;  // (their items: chain_lane after the tile loop)
    }
    // [cb, cm): FP64-accumulated columns, [cm, ce): FP32-accumulated ones
    const int cm = min(ce, max(cb, c32 - tc0));
    const float* __restrict__ col = P.blob32 + sg.off32 + (int64_t)tc0 * rp32 + 4 * p32;
    float4 m[8];
    {
      const int e0 = cb < cm ? cm : ce;
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (cb + u < e0) m[u] = ld_stream(col + (int64_t)(cb + u) * rp32, pol);
    }
    if (OUT == OUT_Y && tc0 == 0 && sg.W64 == 0) asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    gather_g<F32MODE != F32_ALL64, NT, WMAX>(P, P.runs + sg.run0 + sg.nrun64, sg.nrun32, tc0, tw, x, gs,
                                             fl, sidx);
    __syncthreads();
    // batches of 8 columns: unpredicated when full, predicated at the end
    // ROLL: refill each register 8 columns ahead right after consuming it (8
    // loads always in flight; measured faster for the widened FP64-accumulated
    // columns), else batch by batch (much faster around the FP32-chain
    // flushes: m1-single stage 2 0.38 vs 0.52 ms)
    auto drain = [&](int c, int e, auto&& consume, auto roll) {
      constexpr bool ROLL = decltype(roll)::value;
      if constexpr (!ROLL) {
        for (;;) {
          // two half-batches: refill the first four registers while the last
          // four columns are consumed (>= 4 loads stay in flight; A/B on
          // config 4: m1-mixed -0.4 %, m2-single -0.6 %, m1-single neutral)
          if (c + 16 <= e) {
#pragma unroll
            for (int u = 0; u < 4; ++u) consume(m[u], c + u);
#pragma unroll
            for (int u = 0; u < 4; ++u) m[u] = ld_stream(col + (int64_t)(c + 8 + u) * rp32, pol);
#pragma unroll
            for (int u = 4; u < 8; ++u) consume(m[u], c + u);
#pragma unroll
            for (int u = 4; u < 8; ++u) m[u] = ld_stream(col + (int64_t)(c + 8 + u) * rp32, pol);
            c += 8;
            continue;
          }
          if (c + 8 <= e) {
#pragma unroll
            for (int u = 0; u < 8; ++u) consume(m[u], c + u);
          } else {
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (c + u < e) consume(m[u], c + u);
          }
          c += 8;
          if (c >= e) break;
          if (c + 8 <= e) {
#pragma unroll
            for (int u = 0; u < 8; ++u) m[u] = ld_stream(col + (int64_t)(c + u) * rp32, pol);
          } else {
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (c + u < e) m[u] = ld_stream(col + (int64_t)(c + u) * rp32, pol);
          }
        }
        return;
      }
      for (;;) {
        if (c + 16 <= e) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            consume(m[u], c + u);
            m[u] = ld_stream(col + (int64_t)(c + 8 + u) * rp32, pol);
          }
        } else {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (c + u < e) consume(m[u], c + u);
            if (c + 8 + u < e) m[u] = ld_stream(col + (int64_t)(c + 8 + u) * rp32, pol);
          }
        }
        c += 8;
        if (c >= e) break;
      }
    };
    if constexpr (F32MODE != F32_ALL32) {
      if (cb < cm) {
        drain(cb, cm, consume64, std::true_type{});
        if (cm < ce) {
#pragma unroll
          for (int u = 0; u < 8; ++u)
            if (cm + u < ce) m[u] = ld_stream(col + (int64_t)(cm + u) * rp32, pol);
        }
      }
    }
    if constexpr (F32MODE != F32_ALL64) {
      if (cm < ce) drain(cm, ce, consume32, std::false_type{});
    }
  }
  if constexpr (F32MODE != F32_ALL64) {
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] += (double)b32[i];
  }

  if constexpr (F32MODE != F32_ALL64 && OUT == OUT_Y) {
    if (chain_warp) {
      // the part's run meta and per-item SGEMV row-kernel bounds into shared
      // memory (red32, unused until the epilogue), then a barrier among the
      // chain warps only: the widened warps stream on meanwhile
      int32_t* meta = reinterpret_cast<int32_t*>(red32);
      uint32_t* kbits = reinterpret_cast<uint32_t*>(red32) + kChainRunsMax;
      const int wbc = sg.chunk;  // (0: every warp is a chain warp)
      const Run* runs = P.runs + sg.run0 + sg.nrun64;
      for (int j = tid - wbc; j < sg.nrun32; j += NT - wbc) {
        const Run r = runs[j];
        meta[j] = ((r.flags & RUN_ACC32) ? 0 : kMetaWide) | (r.col0 << kMetaW) | r.width;
        kbits[j] = (uint32_t)r.flags >> kRunKindShift;
      }
      chain_bar(NT - wbc);
      // this lane's items (none on an idle lane): the run index ranges follow the
      // group cuts and the first FP32-accumulated column in the group table
      int jb = 0, je = 0;
      if (chain_thr) {
        jb = P.gtab[sg.gtab + g32 + 2 + q32];
        je = P.gtab[sg.gtab + g32 + 2 + q32 + 1];
      }
      chain_lane(cfifo, meta, kbits, jb, je, gs, rp32, p32, b);
    }
  }

  // ---------------- fixed-order reduction over thread groups
  __syncthreads();
  if (sg.W32 > 0 && q32 < g32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) red32[q32 * rp32 + 4 * p32 + i] = b[i];
  }
  __syncthreads();
  // row sums over groups (fixed order); a thread owns rows tid, tid + NT, ...
  auto row_sum = [&](int t) -> double {
    double s = 0.0;
    if constexpr (!XS) {
      if (sg.W64 > 0)
        for (int q = 0; q < g64; ++q) s += red64[q * rp64 + t];
    }
    if (sg.W32 > 0) {
      if (OUT == OUT_Z && F32MODE == F32_ALL32) {
        // stage 1, m1-single: z = Vt32 . x32 accumulated in FP32 throughout
        float f = 0.f;
        for (int q = 0; q < g32; ++q) f += (float)red32[q * rp32 + t];
        s = (double)f;
      } else {
        for (int q = 0; q < g32; ++q) s += red32[q * rp32 + t];
      }
    }
    return s;
  };

  if constexpr (OUT == OUT_Z) {
    // ---------------- stage-1 epilogue: z (or a chunk partial)
    if (sg.nchunks == 1) {
      for (int t = tid; t < R; t += NT) P.z[sg.row0 + t] = z_epilogue(P, row_sum(t), sg.row0 + t);
    } else {
      for (int t = tid; t < R; t += NT) P.part[sg.part_off + sg.chunk * R + t] = row_sum(t);
      __threadfence();
      __syncthreads();
      if (tid == 0) ticket = atomicAdd(P.red_count + sg.red, 1u);
      __syncthreads();
      if (ticket == (unsigned)(sg.nchunks - 1)) {
        __threadfence();
        for (int t = tid; t < R; t += NT) {
          double v = 0.0;
          if (F32MODE == F32_ALL32) {
            float f = 0.f;
            for (int ch = 0; ch < sg.nchunks; ++ch) f += (float)__ldcg(P.part + sg.part_off + ch * R + t);
            v = (double)f;
          } else {
            for (int ch = 0; ch < sg.nchunks; ++ch) v += __ldcg(P.part + sg.part_off + ch * R + t);
          }
          P.z[sg.row0 + t] = z_epilogue(P, v, sg.row0 + t);
        }
        if (tid == 0) P.red_count[sg.red] = 0u;  // ready for the next matvec
      }
    }
    if (NT < 128) asm volatile("griddepcontrol.launch_dependents;");

  } else {
    // ---------------- stage-2 epilogue: y, finite flag, fused dots
    double d0 = 0.0, d1 = 0.0;
    for (int t = tid; t < R; t += NT) {
      const double s = row_sum(t);
      const int row = sg.row0 + t;
      const int li = row - P.row_begin;
      if (!isfinite(s)) *out.nonfinite = 1;
      if (out.permute_out) out.y[P.perm[row]] = s;
      else out.y[li] = s;
      if (out.w1) d0 += s * out.w1[li];
      if (out.yy) d1 += s * s;
    }
    if (out.seg_dots == nullptr) return;
    // per-segment dot partials, then the last CTA reduces all segment
    // partials in segment order (deterministic)
    const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      d0 += __shfl_xor_sync(0xffffffffu, d0, o);
      d1 += __shfl_xor_sync(0xffffffffu, d1, o);
    }
    if (lane == 0) {
      wred[0][wid] = d0;
      wred[1][wid] = d1;
    }
    __syncthreads();
    if (tid == 0) {
      double e0 = 0.0, e1 = 0.0;
      for (int w = 0; w < NT / 32; ++w) {
        e0 += wred[0][w];
        e1 += wred[1][w];
      }
      out.seg_dots[2 * blockIdx.x] = e0;
      out.seg_dots[2 * blockIdx.x + 1] = e1;
      __threadfence();
      ticket = atomicAdd(out.done, 1u);
    }
    __syncthreads();
    if (ticket != gridDim.x - 1) return;
    __threadfence();
    double e0 = 0.0, e1 = 0.0;
    for (int i = tid; i < (int)gridDim.x; i += NT) {
      e0 += __ldcg(out.seg_dots + 2 * i);
      e1 += __ldcg(out.seg_dots + 2 * i + 1);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      e0 += __shfl_xor_sync(0xffffffffu, e0, o);
      e1 += __shfl_xor_sync(0xffffffffu, e1, o);
    }
    __syncthreads();
    if (lane == 0) {
      wred[0][wid] = e0;
      wred[1][wid] = e1;
    }
    __syncthreads();
    if (tid == 0) {
      double f0 = 0.0, f1 = 0.0;
      for (int w = 0; w < NT / 32; ++w) {
        f0 += wred[0][w];
        f1 += wred[1][w];
      }
      out.dots_out[0] = f0;
      out.dots_out[1] = f1;
      *out.done = 0u;
    }
  }
}

// ------------------------------------------------------------------------------
// boundary kernels

__global__ void gather_perm_kernel(const double* __restrict__ x, const int32_t* __restrict__ perm,
                                   double* __restrict__ xp, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) xp[i] = x[perm[i]];
}

// Non-finite probe (reference _check_finite, matvec.py:123-135): evaluates
// every stage-2 item (block slab) on its own, in the scheme's precision, and
// records the smallest block index whose contribution is not finite.
__global__ void probe_kernel(DevPlan P, const double* __restrict__ x, unsigned long long* first_bad) {
  const Seg sg = P.seg2[blockIdx.x];
  const int R = sg.R;
  const int nrun = sg.nrun64 + sg.nrun32;
  for (int j = 0; j < nrun; ++j) {
    const Run r = P.runs[sg.run0 + j];
    const bool f32part = j >= sg.nrun64;
    const int rp = f32part ? ((R + 3) & ~3) : ((R + 1) & ~1);
    const double* src = (r.flags & RUN_Z) ? P.z : x;
    for (int row = threadIdx.x; row < R; row += blockDim.x) {
      double s = 0.0;
      float s32 = 0.f;
      for (int c = 0; c < r.width; ++c) {
        double g = src[r.src + c];
        if (r.flags & RUN_ROUND) g = (double)(float)g;
        const int64_t e = (r.flags & RUN_CHUNK) ? (int64_t)r.col0 * rp + chunk_off(r.width, rp, row, c)
                                                : (int64_t)(r.col0 + c) * rp + row;
        if (f32part) {
          const float m = P.blob32[sg.off32 + e];
          if (r.flags & RUN_ACC32) s32 = fmaf(m, (float)g, s32);
          else s = fma((double)m, g, s);
        } else {
          s = fma(P.blob64[sg.off64 + e], g, s);
        }
      }
      if (f32part && (r.flags & RUN_ACC32)) s = (double)s32;
      if (!isfinite(s)) atomicMin(first_bad, (unsigned long long)P.run_block[sg.run0 + j]);
    }
  }
}

// ------------------------------------------------------------------------------
// launchers

// dynamic shared memory of a seg_kernel instantiation: the chain-item staging
// buffers of the stage-2 FP32 kernels
template <int M, int O, bool EXACT>
static size_t chain_smem(const DevPlan& P) {
  // (at least the gather's index scratch, which shares the memory)
  constexpr size_t fifo = ChainFifo<M == F32_ALL32 ? HMX_FIFO_BATCHES_ALL32 : HMX_FIFO_BATCHES_MIXED>::kBytes;
  return (EXACT && O == OUT_Y && M != F32_ALL64) ? std::max((size_t)P.chain_warps * fifo, (size_t)kSegWMax * 4) : 0;
}
constexpr int kChainSmemMax = (kSegThreads / 32) * 4 * 4 * 512;

template <int M, int O, int NT = kSegThreads, bool DEEP = false, bool EXACT = false, int XMINB = HMX_EXACT_MINB>
static cudaError_t launch_seg(const DevPlan& P, const Seg* segs, int nseg, const double* x,
                              const S2Out& out, cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nseg);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = chain_smem<M, O, EXACT>(P);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, seg_kernel<M, O, NT, DEEP, EXACT, XMINB>, P, segs, x, out);
}

cudaError_t launch_stage1(const DevPlan& P, const double* x, cudaStream_t st, const int* skip,
                          int seg_begin, int seg_count) {
  const int nseg = seg_count < 0 ? P.n_seg1 - seg_begin : std::min(seg_count, P.n_seg1 - seg_begin);
  if (nseg <= 0) return cudaSuccess;
  const Seg* segs = P.seg1 + seg_begin;
  S2Out none{};
  none.skip = skip;
  // every stage-1 segment FP32 data widened into FP64 sums (m1-mixed, m2-single,
  // m2-mixed, m3 with an all-FP32 class): 64-thread CTAs, 16 per SM (measured
  // -3..-4 % on stage 1 against 128 threads; the FP32-accumulating m1-single
  // stage 1 is faster on 128)
  if (P.s1_exact) {
    if (P.s1_exact == 2) s1_exact4_kernel<<<nseg, kS1ExactThreads, 0, st>>>(P, segs, x, skip);
    else s1_exact_kernel<<<nseg, kS1ExactRows, 0, st>>>(P, segs, x, skip);
    return cudaGetLastError();
  }
  switch (P.f32mode1) {
    case F32_ALL32: return launch_seg<F32_ALL32, OUT_Z, kS1Threads>(P, segs, nseg, x, none, st, false);
    default:
      return P.s1_narrow ? launch_seg<F32_ALL64, OUT_Z, kS1Threads32>(P, segs, nseg, x, none, st, false)
                         : launch_seg<F32_ALL64, OUT_Z, kS1Threads>(P, segs, nseg, x, none, st, false);
  }
}

cudaError_t launch_stage2(const DevPlan& P, const double* x, const S2Out& out, cudaStream_t st,
                          bool pdl) {
  if (P.n_seg2 == 0) return cudaSuccess;
  switch (P.f32mode2) {
    case F32_ALL32:
      return P.chain_exact ? launch_seg<F32_ALL32, OUT_Y, kSegThreads, false, true, HMX_EXACT_MINB_ALL32>(P, P.seg2, P.n_seg2, x, out, st, pdl)
                           : launch_seg<F32_ALL32, OUT_Y>(P, P.seg2, P.n_seg2, x, out, st, pdl);
    case F32_MIXED:
      if (!P.chain_exact) return launch_seg<F32_MIXED, OUT_Y>(P, P.seg2, P.n_seg2, x, out, st, pdl);
      return launch_seg<F32_MIXED, OUT_Y, kSegThreads, false, true>(P, P.seg2, P.n_seg2, x, out, st, pdl);
    default:
      return P.s2_deep ? launch_seg<F32_ALL64, OUT_Y, kSegThreads, true>(P, P.seg2, P.n_seg2, x, out, st, pdl)
                       : launch_seg<F32_ALL64, OUT_Y>(P, P.seg2, P.n_seg2, x, out, st, pdl);
  }
}

// The stage-2 FP32 kernels opt in to > 48 KB of shared memory (static + the
// chain staging buffers); called at plan creation, outside any capture.
cudaError_t configure_kernels() {
  cudaError_t e = cudaFuncSetAttribute(seg_kernel<F32_ALL32, OUT_Y, kSegThreads, false, true, HMX_EXACT_MINB_ALL32>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kChainSmemMax);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(seg_kernel<F32_MIXED, OUT_Y, kSegThreads, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, kChainSmemMax);
  return e;
}

cudaError_t launch_gather_perm(const double* x, const int32_t* perm, double* xp, int n,
                               cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  gather_perm_kernel<<<(n + 255) / 256, 256, 0, st>>>(x, perm, xp, n);
  return cudaGetLastError();
}

cudaError_t launch_probe(const DevPlan& P, const double* x, unsigned long long* first_bad,
                         cudaStream_t st) {
  if (P.n_seg2 == 0) return cudaSuccess;
  probe_kernel<<<P.n_seg2, 64, 0, st>>>(P, x, first_bad);
  return cudaGetLastError();
}

}  // namespace hmx
