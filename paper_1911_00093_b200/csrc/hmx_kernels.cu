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
#ifndef HMX_EXACT_MINB
#define HMX_EXACT_MINB 4  // CTAs per SM of the SGEMV-order stage-2 kernels (register budget)
#endif

namespace hmx {

enum Out : int { OUT_Y = 0, OUT_Z = 1 };

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

// FP32-accumulated items (RUN_CHUNK, layout chunk_off in hmx_internal.cuh):
// each row's value in OpenBLAS SGEMV-T's order, widened once and added in
// FP64 (reference matvec.py:57, :73, then :106).  Explicit _rn intrinsics:
// nothing is contracted or reassociated.
//
// The chain warps stage the segment's chain items through shared memory:
// windows of whole consecutive items (<= kChainWin bytes, contiguous in the
// blob), copied with cp.async by all chain threads into two buffers, the next
// window in flight while one is reduced; inside a window item i goes to slot i mod K (K = chain
// threads / rp), one row per thread.  Items larger than a window are read
// from global memory by slot 0.
__device__ __forceinline__ float4 fma4(float4 a, float4 g, float4 c) {
  return make_float4(__fmaf_rn(a.x, g.x, c.x), __fmaf_rn(a.y, g.y, c.y), __fmaf_rn(a.z, g.z, c.z),
                     __fmaf_rn(a.w, g.w, c.w));
}
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
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void chain_bar(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}
// mbarrier + 1-D bulk copy (TMA engine): one thread moves a whole window
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(b)) : "memory");
}
// arrive on `b` expecting `bytes` and start the copy (bytes = 0: plain arrive)
__device__ __forceinline__ void bulk_to_smem(float* dst, const float* src, uint32_t bytes, uint64_t* b) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
  if (bytes)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(b))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @P1 bra DONE;\n bra WAIT;\n "
      "DONE:\n }" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}

constexpr int kMetaW = 12;  // run meta in shared memory: col0 << 12 | width
#ifndef HMX_CHAIN_ROWS
#define HMX_CHAIN_ROWS 1  // rows per chain thread (1 or 2); the flattener's group count follows kChainRows
#endif
#ifndef HMX_CHAIN_WB
#define HMX_CHAIN_WB 8192
#endif
constexpr int kChainWin = HMX_CHAIN_WB;  // bytes per staging buffer (two buffers)

// row p of one n-wide item at `it` (global or shared memory, chunk layout).
// `kind`: which OpenBLAS SGEMV-T row kernel computes this row of its block
// (sgemv_row_kind): 16, 8, 4 = the 16-, 8- and 4-row kernels (A/B FMA
// chains; rows shorter than 8 differ between them), 2 = the two-row
// remainder kernel (one 4-lane accumulator, multiply then add), 1 = the
// one-row remainder kernel (A/B, multiply then add).  All end with
// (l0 + l1) + (l2 + l3) and the same tail rule (tools/fp32_accum_emulation.py
// sgemv_kind: bitwise numpy's own for every row count 2..64, widths 1..48).
// G(k): the FP32 source value of the item's column k.
template <bool GLOBAL, typename GF>
__device__ __forceinline__ float chain_item(const float* it, GF G, int n, int rp, int p, int kind) {
  constexpr int c0 = 0;
  auto G4 = [&](int c) { return make_float4(G(c), G(c + 1), G(c + 2), G(c + 3)); };
  auto L4 = [&](const float* q) {
    if constexpr (GLOBAL) return ld_chunk(q);
    else return *reinterpret_cast<const float4*>(q);
  };
  auto L1 = [&](const float* q) {
    if constexpr (GLOBAL) return ld_one(q);
    else return *q;
  };
  // element k of this row (chunk layout)
  auto E = [&](int k) {
    if (chain_shaped(n)) return L1(it + (int64_t)k * rp + p);
    const int m = n & ~3;
    return k < m ? L1(it + 4 * ((int64_t)(k >> 2) * rp + p) + (k & 3)) : L1(it + (int64_t)m * rp + (int64_t)(k - m) * rp + p);
  };
  auto Pr = [&](int k) { return __fmul_rn(E(k), G(c0 + k)); };  // rounded product
  auto F = [&](int k, float acc) { return __fmaf_rn(E(k), G(c0 + k), acc); };
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
  const float* ch = it + 4 * p;  // chunk c of row p at ch[4 c rp]
  float4 l;
  bool seq = false;  // sequential horizontal sum (one-row kernel, n <= 8)
  if (n == 8 && kind >= 4) {  // l_j = a_2j g_2j + a_2j+1 g_2j+1
    const float4 x0 = L4(ch), x1 = L4(ch + 4 * rp);
    const float4 g0 = G4(c0), g1 = G4(c0 + 4);
    l = make_float4(__fadd_rn(__fmul_rn(x0.x, g0.x), __fmul_rn(x0.y, g0.y)),
                    __fadd_rn(__fmul_rn(x0.z, g0.z), __fmul_rn(x0.w, g0.w)),
                    __fadd_rn(__fmul_rn(x1.x, g1.x), __fmul_rn(x1.y, g1.y)),
                    __fadd_rn(__fmul_rn(x1.z, g1.z), __fmul_rn(x1.w, g1.w)));
  } else {
    // chunks into A (and B): four-row and one-row kernels: nch even: A = even
    // chunks, B = odd; nch odd: A = {0, 1, 3, 5, ..}, B = {2, 4, ..}; two-row
    // kernel: every chunk into A
    float4 A = make_float4(0.f, 0.f, 0.f, 0.f), B = A;
    auto acc = [&](float4& X, const float4& x, const float4& g) {
      if (kind >= 4) X = fma4(x, g, X);
      else X = make_float4(__fadd_rn(X.x, __fmul_rn(x.x, g.x)), __fadd_rn(X.y, __fmul_rn(x.y, g.y)),
                           __fadd_rn(X.z, __fmul_rn(x.z, g.z)), __fadd_rn(X.w, __fmul_rn(x.w, g.w)));
    };
    int c = 0;
    if (kind == 2) {
      for (; c < nch; ++c) acc(A, L4(ch + (int64_t)4 * c * rp), G4(c0 + 4 * c));
    } else {
      if (nch & 1) {
        acc(A, L4(ch), G4(c0));
        c = 1;
      }
      for (; c < nch; c += 2) {
        const float4 xa = L4(ch + (int64_t)4 * c * rp), xb = L4(ch + (int64_t)4 * (c + 1) * rp);
        acc(A, xa, G4(c0 + 4 * c));
        acc(B, xb, G4(c0 + 4 * c + 4));
      }
    }
    l = make_float4(__fadd_rn(A.x, B.x), __fadd_rn(A.y, B.y), __fadd_rn(A.z, B.z), __fadd_rn(A.w, B.w));
    seq = kind == 1 && n <= 8;
  }
  float v = seq ? __fadd_rn(__fadd_rn(__fadd_rn(l.x, l.y), l.z), l.w)
                : __fadd_rn(__fadd_rn(l.x, l.y), __fadd_rn(l.z, l.w));
  const float* tl = it + (int64_t)m * rp + p;
  if (T == 1) {
    v = __fmaf_rn(L1(tl), G(c0 + m), v);
  } else if (T >= 2) {
    float tv = __fmul_rn(L1(tl + rp), G(c0 + m + 1));
    tv = __fmaf_rn(L1(tl), G(c0 + m), tv);
    if (T == 3) tv = __fmaf_rn(L1(tl + 2 * rp), G(c0 + m + 2), tv);
    v = __fadd_rn(v, tv);
  }
  return v;
}

// Rows r0 = h and r1 = h + half of one n-wide item in shared memory (chunk
// layout), both in the four-row kernel's order (kind 4): chain_item for two
// rows at once, sharing the source loads.
template <typename GF>
__device__ __forceinline__ float2 chain_item2(const float* it, GF G, int n, int rp, int r0, int r1) {
  auto G4 = [&](int c) { return make_float4(G(c), G(c + 1), G(c + 2), G(c + 3)); };
  if (chain_shaped(n)) {
    float v0 = 0.f, v1 = 0.f;
    for (int k = 0; k < n; ++k) {
      const float g = G(k);
      v0 = __fmaf_rn(it[(int64_t)k * rp + r0], g, v0);
      v1 = __fmaf_rn(it[(int64_t)k * rp + r1], g, v1);
    }
    return make_float2(v0, v1);
  }
  const int nch = n >> 2, T = n & 3, m = 4 * nch;
  const float4* c0p = reinterpret_cast<const float4*>(it) + r0;  // chunk c of row r at [c rp + r]
  const float4* c1p = reinterpret_cast<const float4*>(it) + r1;
  float4 l0, l1;
  if (n == 8) {  // l_j = a_2j g_2j + a_2j+1 g_2j+1
    const float4 g0 = G4(0), g1 = G4(4);
    auto pairs = [&](const float4& x, const float4& y) {
      return make_float4(__fadd_rn(__fmul_rn(x.x, g0.x), __fmul_rn(x.y, g0.y)),
                         __fadd_rn(__fmul_rn(x.z, g0.z), __fmul_rn(x.w, g0.w)),
                         __fadd_rn(__fmul_rn(y.x, g1.x), __fmul_rn(y.y, g1.y)),
                         __fadd_rn(__fmul_rn(y.z, g1.z), __fmul_rn(y.w, g1.w)));
    };
    l0 = pairs(c0p[0], c0p[rp]);
    l1 = pairs(c1p[0], c1p[rp]);
  } else {
    float4 A0 = make_float4(0.f, 0.f, 0.f, 0.f), B0 = A0, A1 = A0, B1 = A0;
    int c = 0;
    if (nch & 1) {
      const float4 g = G4(0);
      A0 = fma4(c0p[0], g, A0);
      A1 = fma4(c1p[0], g, A1);
      c = 1;
    }
    for (; c < nch; c += 2) {
      const float4 ga = G4(4 * c), gb = G4(4 * c + 4);
      A0 = fma4(c0p[c * rp], ga, A0);
      A1 = fma4(c1p[c * rp], ga, A1);
      B0 = fma4(c0p[(c + 1) * rp], gb, B0);
      B1 = fma4(c1p[(c + 1) * rp], gb, B1);
    }
    l0 = make_float4(__fadd_rn(A0.x, B0.x), __fadd_rn(A0.y, B0.y), __fadd_rn(A0.z, B0.z), __fadd_rn(A0.w, B0.w));
    l1 = make_float4(__fadd_rn(A1.x, B1.x), __fadd_rn(A1.y, B1.y), __fadd_rn(A1.z, B1.z), __fadd_rn(A1.w, B1.w));
  }
  float v0 = __fadd_rn(__fadd_rn(l0.x, l0.y), __fadd_rn(l0.z, l0.w));
  float v1 = __fadd_rn(__fadd_rn(l1.x, l1.y), __fadd_rn(l1.z, l1.w));
  const float* tl = it + (int64_t)m * rp;
  if (T == 1) {
    const float g = G(m);
    v0 = __fmaf_rn(tl[r0], g, v0);
    v1 = __fmaf_rn(tl[r1], g, v1);
  } else if (T >= 2) {
    const float ga = G(m + 1), gb = G(m);
    float t0 = __fmaf_rn(tl[r0], gb, __fmul_rn(tl[rp + r0], ga));
    float t1 = __fmaf_rn(tl[r1], gb, __fmul_rn(tl[rp + r1], ga));
    if (T == 3) {
      const float gc = G(m + 2);
      t0 = __fmaf_rn(tl[2 * rp + r0], gc, t0);
      t1 = __fmaf_rn(tl[2 * rp + r1], gc, t1);
    }
    v0 = __fadd_rn(v0, t0);
    v1 = __fadd_rn(v1, t1);
  }
  return make_float2(v0, v1);
}

// chain threads u = 0 .. nthr-1 (slot u / rp, row u % rp); items j0 .. nrun-1
// of the part (meta in shared memory, the part's blob at `part`); buf: two
// kChainWin-byte staging buffers, filled by bulk copies (thread 0 issues one
// per window; mb: their two mbarriers); wq: 6 ints of shared memory for the
// window bounds thread 0 keeps one window ahead.  Returns this thread's row sum.
__device__ __forceinline__ double chain_windows(const int32_t* meta, const uint32_t* kbits, int j0, int nrun,
                                                const float* part, const double* gs, int rp, int u, int nthr,
                                                float* buf, int* wq, uint64_t* mb, double& acc1) {
#if HMX_CHAIN_ROWS == 2
  const int half = rp >> 1;  // two rows per thread: p and p + half
  const int K = nthr / half;
  const int slot = u / half, p = u - slot * half, p1 = p + half;
#else
  const int K = nthr / rp;
  const int slot = u / rp, p = u - slot * rp;
#endif
  const bool act = slot < K;
  const int wmax = kChainWin / (4 * rp);  // columns per window
  auto col0 = [&](int j) { return meta[j] >> kMetaW; };
  auto width = [&](int j) { return meta[j] & ((1 << kMetaW) - 1); };
  // window starting at item j: [j, end) of <= wmax columns, or one oversize item
  auto wend = [&](int j) {
    if (j >= nrun) return j;
    const int cs = col0(j);
    int e = j + 1;
    if (width(j) > wmax) return e;
    while (e < nrun && col0(e) + width(e) - cs <= wmax) ++e;
    return e;
  };
  // (thread 0) copy window [j, e) into buffer b; an oversize item (read from
  // global memory) completes the buffer's phase with no bytes
  auto stage = [&](int j, int e, int b) {
    if (j >= nrun) return;
    uint32_t bytes = 0;
    const float* src = part;
    if (width(j) <= wmax) {
      const int cs = col0(j), ce = col0(e - 1) + width(e - 1);
      bytes = (uint32_t)((ce - cs) * rp * 4);
      src = part + (int64_t)cs * rp;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the buffer's last generic reads
    bulk_to_smem(buf + b * (kChainWin / 4), src, bytes, mb + b);
  };
  // window bounds: a ring of three (start, end) pairs in wq
  if (u == 0) {
    mbar_init(mb);
    mbar_init(mb + 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const int e0 = wend(j0), e1 = wend(e0);
    wq[0] = j0, wq[1] = e0, wq[2] = e0, wq[3] = e1;
    stage(j0, e0, 0);
  }
  chain_bar(nthr);
  double acc = 0.0;
  for (int w = 0;; ++w) {
    const int r = w % 3;
    const int j = wq[2 * r], e = wq[2 * r + 1];
    if (j >= nrun) break;
    if (u == 0) {  // the next window in flight while this one is reduced; bounds of the one after
      const int r1 = (w + 1) % 3, r2 = (w + 2) % 3;
      const int jn = wq[2 * r1], en = wq[2 * r1 + 1];
      stage(jn, en, (w + 1) & 1);
      wq[2 * r2] = en;
      wq[2 * r2 + 1] = wend(en);
    }
    mbar_wait(mb + (w & 1), (uint32_t)(w >> 1) & 1u);  // window [j, e) has landed
    if (act) {
      if (width(j) > wmax) {  // oversize item: straight from global memory
        if (slot == 0) {
          const int c0 = col0(j);
          auto G = [&](int k) { return __int_as_float(__double2loint(gs[c0 + k])); };
          acc += (double)chain_item<true>(part + (int64_t)c0 * rp, G, width(j), rp, p, chain_row_kind(kbits[j], p));
#if HMX_CHAIN_ROWS == 2
          acc1 += (double)chain_item<true>(part + (int64_t)c0 * rp, G, width(j), rp, p1, chain_row_kind(kbits[j], p1));
#endif
        }
      } else {
        const float* base = buf + (w & 1) * (kChainWin / 4);
        const int cs = col0(j);
        for (int i = j + slot; i < e; i += K) {
          const int c0 = col0(i);
          auto G = [&](int k) { return __int_as_float(__double2loint(gs[c0 + k])); };
          const float* it = base + (c0 - cs) * rp;
          // the common case first: every row of the segment in SGEMV's
          // 16-row kernel (n < 8), or in the 16/8/4-row kernels (n >= 8)
          const uint32_t kb = kbits[i];
          const int wi = width(i);
#if HMX_CHAIN_ROWS == 2
          if ((int)((kb >> (wi < 8 ? 0 : 14)) & 127) >= rp) {
            const float2 v = chain_item2(it, G, wi, rp, p, p1);
            acc += (double)v.x;
            acc1 += (double)v.y;
          } else {
            acc += (double)chain_item<false>(it, G, wi, rp, p, chain_row_kind(kb, p));
            acc1 += (double)chain_item<false>(it, G, wi, rp, p1, chain_row_kind(kb, p1));
          }
#else
          if ((int)((kb >> (wi < 8 ? 0 : 14)) & 127) >= rp) acc += (double)chain_item<false>(it, G, wi, rp, p, 16);
          else acc += (double)chain_item<false>(it, G, wi, rp, p, chain_row_kind(kb, p));
#endif
        }
      }
    }
    chain_bar(nthr);  // buffer w & 1 is free again; wq holds the next bounds
  }
  return acc;
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
  // the FP32 source shadow (matvec.py:119): x rounded once
  auto G = [&](int c) { return (float)__ldg(xs + c); };
  auto G4 = [&](int c) { return make_float4(G(c), G(c + 1), G(c + 2), G(c + 3)); };
  float y = 0.f;
  const int kind = t < sg.R ? P.zkind[sg.row0 + t] : 16;
  if (t >= sg.R) {
    // (idle row: no loads; joins the barrier below)
  } else if (n <= 8) {  // short rows (chain-shaped, n = 4, n = 8): the per-kernel rules
    y = chain_item<true>(it, G, n, rp, t, kind);
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
    constexpr int kS1Win = 8;
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

// One CTA = one segment: rows [row0, row0+R) of a column-major item stream.
// DEEP: stage 2 with an FP64 part, 12 FP64 columns in flight per thread at 3
// CTAs per SM (80 registers) instead of 8 at 4 (A/B on config 4: m1-double
// stage 2 -1.1 %, m2-double -2.4 %; FP32-only stage 2 prefers 8 at 4)
// EXACT (stage 2 with FP32-accumulated items): those items in SGEMV's order
// (chain_windows); otherwise one FP32 chain per (row, item) (HMX_PLAN_FP32_CHAIN).
// Separate instantiations keep each one's register allocation its own.
// XMINB: CTAs per SM of an EXACT instantiation (its register budget; m2-single
// measured faster at 3 = 80 registers, m1-mixed at 4).
template <int F32MODE, int OUT, int NT, bool DEEP = false, bool EXACT = false, int XMINB = HMX_EXACT_MINB>
__global__ void __launch_bounds__(NT, DEEP ? 3 : (OUT == OUT_Y && F32MODE != F32_ALL64) ? (EXACT ? XMINB : HMX_MIXED_MINB) : 1024 / NT) seg_kernel(DevPlan P, const Seg* __restrict__ segs,
                                                          const double* __restrict__ x, S2Out out) {
  // stage 1 segments have a single run (no index expansion) and <= 1024 columns
  constexpr int WMAX = OUT == OUT_Z ? kS1WMax : kSegWMax;
  constexpr int D64 = DEEP ? 12 : 8;
  __shared__ double gs[WMAX];
  __shared__ uint8_t fl[WMAX];
  __shared__ int32_t sidx[OUT == OUT_Z ? 1 : kSegWMax];
  __shared__ double red64[2 * NT];
  __shared__ double red32[4 * NT];
  __shared__ double wred[2][NT / 32];
  // chain-item staging buffers (stage-2 FP32 kernels: 2 x kChainWin bytes of dynamic shared memory)
  extern __shared__ __align__(16) float chain_buf[];
  __shared__ int chain_wq[6];  // chain-window bounds (chain_windows)
  __shared__ uint64_t chain_mb[2];  // their bulk copies' mbarriers
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
  const int g64 = NT / tpg64;
  const int q64 = tid / tpg64, p64 = tid - q64 * tpg64;
  double a0 = 0.0, a1 = 0.0;
  for (int tc0 = 0; tc0 < sg.W64; tc0 += WMAX) {
    const int tw = min(WMAX, sg.W64 - tc0);
    const bool act = q64 < g64;
    const int cb = act ? (int)((int64_t)tw * q64 / g64) : 0;
    const int ce = act ? (int)((int64_t)tw * (q64 + 1) / g64) : 0;
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

  // ---------------- FP32 part: 4 rows x 16 bytes per thread
  const int rp32 = (R + 3) & ~3;
  const int tpg32 = rp32 >> 2;
  int g32 = NT / tpg32;
  int q32 = tid / tpg32, p32 = tid - q32 * tpg32;
  // Stage-2 parts with a group table (every part of <= kSegWMax columns):
  // FP64-accumulated (widened) items on threads [0, wbc), 4 rows per thread
  // as above; the FP32-accumulated items (RUN_CHUNK) on threads [wbc, NT),
  // ONE row per thread, each item evaluated in SGEMV's own order (chain_items).
  // wbc (plan: sg.chunk) is warp-aligned, so no warp runs both loops.
  bool chain_thr = false;
  int pc = 0;
  if constexpr (F32MODE == F32_MIXED && OUT == OUT_Y) {
    // (HMX_PLAN_FP32_CHAIN plans: one FP32 FMA chain per (row, item), 4 rows
    // per thread on both sides of the warp-aligned split at wb = sg.chunk)
    const int wb = sg.chunk;
    if (!EXACT && wb > 0 && sg.gtab >= 0) {
      const int ga = wb / tpg32, gb = (NT - wb) / tpg32;
      g32 = ga + gb;
      if (tid < wb) {
        if (q32 >= ga) q32 = g32;  // idle
      } else {
        const int u = tid - wb;
        const int qb = u / tpg32;
        p32 = u - qb * tpg32;
        q32 = qb < gb ? ga + qb : g32;
      }
    }
  }
  if constexpr (EXACT && F32MODE != F32_ALL64 && OUT == OUT_Y) {
    if (sg.gtab >= 0) {
      const int wbc = F32MODE == F32_ALL32 ? 0 : sg.chunk;
      const int ga = wbc / tpg32, gb = (NT - wbc) / (rp32 / HMX_CHAIN_ROWS);
      g32 = ga + gb;
      if (tid < wbc) {
        if (q32 >= ga) q32 = g32;  // idle
      } else {
        const int u = tid - wbc;
        const int qb = u / (rp32 / HMX_CHAIN_ROWS);
        pc = u - qb * (rp32 / HMX_CHAIN_ROWS);
        q32 = qb < gb ? ga + qb : g32;
        chain_thr = true;
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
  double bc = 0.0, bc1 = 0.0;  // chain threads: their rows' FP64 sums of the widened item values
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
    int cb = act ? (int)((int64_t)tw * q32 / g32) : 0;
    int ce = act ? (int)((int64_t)tw * (q32 + 1) / g32) : 0;
    if (F32MODE != F32_ALL64 && OUT == OUT_Y && sg.gtab >= 0 && act) {
      // FP32-accumulated items are never split between groups: every item
      // row is one FP32 chain (reference: FP32 GEMV per block, matvec.py:57, :73)
      cb = P.gtab[sg.gtab + q32];
      ce = P.gtab[sg.gtab + q32 + 1];
      if (chain_thr) ce = cb;  // (their items: chain_items after the tile loop)
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
    if (chain_thr) {
      // (the per-item SGEMV row-kernel bounds live in red32, unused until the epilogue)
      uint32_t* kbits = reinterpret_cast<uint32_t*>(red32);
      // the part's run meta into shared memory (sidx is free after the
      // gather), then a barrier among the chain warps only: the widened
      // warps stream on meanwhile
      const int wbc = F32MODE == F32_ALL32 ? 0 : sg.chunk;
      const Run* runs = P.runs + sg.run0 + sg.nrun64;
      for (int j = tid - wbc; j < sg.nrun32; j += NT - wbc) {
        const Run r = runs[j];
        sidx[j] = (r.col0 << kMetaW) | r.width;
        kbits[j] = (uint32_t)r.flags >> kRunKindShift;
      }
      chain_bar(NT - wbc);
      int j0 = 0;  // the first chain item (they follow the widened ones)
      const int c32c = P.gtab[sg.gtab + g32 + 1];
      while (j0 < sg.nrun32 && (sidx[j0] >> kMetaW) < c32c) ++j0;
      bc = chain_windows(sidx, kbits, j0, sg.nrun32, P.blob32 + sg.off32, gs, rp32, tid - wbc, NT - wbc, chain_buf,
                         chain_wq, chain_mb, bc1);
    }
  }

  // ---------------- fixed-order reduction over thread groups
  __syncthreads();
  if (sg.W32 > 0 && q32 < g32) {
    if (chain_thr) {
      red32[q32 * rp32 + pc] = bc;
      if (HMX_CHAIN_ROWS == 2) red32[q32 * rp32 + pc + (rp32 >> 1)] = bc1;
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) red32[q32 * rp32 + 4 * p32 + i] = b[i];
    }
  }
  __syncthreads();
  // row sums over groups (fixed order); a thread owns rows tid, tid + NT, ...
  auto row_sum = [&](int t) -> double {
    double s = 0.0;
    if (sg.W64 > 0)
      for (int q = 0; q < g64; ++q) s += red64[q * rp64 + t];
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
constexpr size_t chain_smem() {
  return (EXACT && O == OUT_Y && M != F32_ALL64) ? 2 * (size_t)kChainWin : 0;
}

template <int M, int O, int NT = kSegThreads, bool DEEP = false, bool EXACT = false, int XMINB = HMX_EXACT_MINB>
static cudaError_t launch_seg(const DevPlan& P, const Seg* segs, int nseg, const double* x,
                              const S2Out& out, cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nseg);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = chain_smem<M, O, EXACT>();
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
    s1_exact_kernel<<<nseg, kS1ExactRows, 0, st>>>(P, segs, x, skip);
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
      return P.chain_exact ? launch_seg<F32_ALL32, OUT_Y, kSegThreads, false, true>(P, P.seg2, P.n_seg2, x, out, st, pdl)
                           : launch_seg<F32_ALL32, OUT_Y>(P, P.seg2, P.n_seg2, x, out, st, pdl);
    case F32_MIXED:
      if (!P.chain_exact) return launch_seg<F32_MIXED, OUT_Y>(P, P.seg2, P.n_seg2, x, out, st, pdl);
      return P.pipe == P_M2S ? launch_seg<F32_MIXED, OUT_Y, kSegThreads, false, true, 3>(P, P.seg2, P.n_seg2, x, out, st, pdl)
                             : launch_seg<F32_MIXED, OUT_Y, kSegThreads, false, true>(P, P.seg2, P.n_seg2, x, out, st, pdl);
    default:
      return P.s2_deep ? launch_seg<F32_ALL64, OUT_Y, kSegThreads, true>(P, P.seg2, P.n_seg2, x, out, st, pdl)
                       : launch_seg<F32_ALL64, OUT_Y>(P, P.seg2, P.n_seg2, x, out, st, pdl);
  }
}

// The stage-2 FP32 kernels opt in to > 48 KB of shared memory (static + the
// chain staging buffers); called at plan creation, outside any capture.
cudaError_t configure_kernels() {
  cudaError_t e = cudaFuncSetAttribute(seg_kernel<F32_ALL32, OUT_Y, kSegThreads, false, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)chain_smem<F32_ALL32, OUT_Y, true>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(seg_kernel<F32_MIXED, OUT_Y, kSegThreads, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chain_smem<F32_MIXED, OUT_Y, true>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(seg_kernel<F32_MIXED, OUT_Y, kSegThreads, false, true, 3>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)chain_smem<F32_MIXED, OUT_Y, true>());
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
