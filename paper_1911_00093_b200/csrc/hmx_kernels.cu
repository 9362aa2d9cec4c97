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

namespace hmx {

enum Out : int { OUT_Y = 0, OUT_Z = 1 };

// Shared-memory slot of an FP32-accumulated column: the FP32 source value in
// the low word, the column's tree code (OB_*, hmx_internal.cuh) in the high
// word (stage 1: OB_ITEM_CHAIN on a segment's first column, else 0).
__device__ __forceinline__ double acc32_slot(float g, int code) {
  return __hiloint2double(code, __float_as_int(g));
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
// (fl: scratch flags, the column's OB_* code and kFlAcc32).  RUN_OBL items
// are stored in SGEMV lane order, so column k reads source obl_col(k).  A single run
// (every stage-1 segment) is a contiguous copy.  Otherwise the runs are first
// expanded into a per-column source index in shared memory, so every
// column's copy is independent (no dependent run lookups).
constexpr int32_t kTagZ = 1 << 30, kTagRound = 1 << 29, kIdxMask = kTagRound - 1;
constexpr uint8_t kFlAcc32 = 16;  // fl: low 4 bits the OB_* code, bit 4 an FP32-accumulated column
template <bool FLAGS, int NT, int WMAX>
__device__ __forceinline__ void gather_g(const DevPlan& P, const Run* __restrict__ runs, int nrun,
                                         int tc0, int tw, const double* __restrict__ x,
                                         double* gs, uint8_t* fl, int32_t* sidx) {
  constexpr int PER = WMAX / NT;  // columns per thread
  if (nrun == 1) {
    const Run r = runs[0];
    const double* src = ((r.flags & RUN_Z) ? P.z : x) + r.src;
    const bool rnd = (r.flags & RUN_ROUND) != 0;
    const bool f32 = FLAGS && (r.flags & RUN_ACC32);
    const bool obl = FLAGS && (r.flags & RUN_OBL);
    int code[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int c = threadIdx.x + u * NT;
      const int k = tc0 + c - r.col0;
      code[u] = k == 0 ? OB_ITEM_CHAIN : OB_NONE;
      const int sc = obl ? obl_col(r.width, k, &code[u]) : k;
      if (c < tw) cp_async8(gs + c, src + sc);
    }
    cp_async_wait_all();
    if (rnd || f32) {
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int c = threadIdx.x + u * NT;
        if (c < tw) {
          const double g = gs[c];
          gs[c] = f32 ? acc32_slot((float)g, code[u]) : (double)(float)g;
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
    const uint8_t f32 = (r.flags & RUN_ACC32) ? kFlAcc32 : 0;
    const bool obl = FLAGS && (r.flags & RUN_OBL);
    for (int col = lo; col < hi; ++col) {
      int code = col == r.col0 ? OB_ITEM_CHAIN : OB_NONE;
      const int sc = obl ? obl_col(r.width, col - r.col0, &code) : col - r.col0;
      sidx[col - tc0] = (r.src + sc) | tag;
      if constexpr (FLAGS) fl[col - tc0] = (uint8_t)(code | f32);
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
      if (FLAGS && (f & kFlAcc32)) gs[c] = acc32_slot((float)gs[c], f & 15);
      else if (id[u] & kTagRound) gs[c] = (double)(float)gs[c];
    }
  }
}

__device__ __forceinline__ double z_epilogue(const DevPlan& P, double s, int zi) {
  if (P.zepi == Z_ROUND32) return (double)(float)s;   // FP32 intermediate (matvec.py:68-72)
  if (P.zepi == Z_SCALE) return s * P.zscale[zi];      // z *= diag (matvec.py:81, :88, :92)
  return s;
}

// One CTA = one segment: rows [row0, row0+R) of a column-major item stream.
// DEEP: stage 2 with an FP64 part, 12 FP64 columns in flight per thread at 3
// CTAs per SM (80 registers) instead of 8 at 4 (A/B on config 4: m1-double
// stage 2 -1.1 %, m2-double -2.4 %; FP32-only stage 2 prefers 8 at 4)
template <int F32MODE, int OUT, int NT, bool DEEP = false>
__global__ void __launch_bounds__(NT, DEEP ? 3 : (OUT == OUT_Y && F32MODE != F32_ALL64) ? HMX_MIXED_MINB : 1024 / NT) seg_kernel(DevPlan P, const Seg* __restrict__ segs,
                                                          const double* __restrict__ x, S2Out out) {
  // stage 1 segments have a single run (no index expansion) and <= 1024 columns
  constexpr int WMAX = OUT == OUT_Z ? kS1WMax : kSegWMax;
  constexpr int D64 = DEEP ? 12 : 8;
  __shared__ double gs[WMAX];
  __shared__ uint8_t fl[WMAX];
  __shared__ int32_t sidx[OUT == OUT_Z ? 1 : kSegWMax];
  __shared__ double red64[2 * NT];
  __shared__ double red32[4 * NT];
  // pending FP32 lane-tree values of stage 2's FP32-accumulated items
  // (consume32): dynamic shared memory, 3 x NT float4 (kTreeSmem)
  extern __shared__ float4 tstate[];
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
  if constexpr (F32MODE == F32_MIXED && OUT == OUT_Y) {
    // warp-aligned split (plan: sg.chunk = wb): groups of the FP64-accumulated
    // columns on threads [0, wb), of the FP32-accumulated ones from wb on, so
    // no warp runs both loops
    const int wb = sg.chunk;
    if (wb > 0 && sg.gtab >= 0) {
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
  // FP32-accumulated items (stage 2): per row, the SGEMV lane tree of
  // hmx_internal.cuh evaluated in storage order.  b32 is the running FMA
  // chain; the tree's pending values live in shared memory (touched only at
  // sub-chain starts, so they cost no registers in the streaming loop):
  // TS_P a finished A_j waiting for B_j, TS_01 = l0 (+ l1), TS_2 = l2.  They
  // are zero whenever tmode == 0 (0: plain chain, 1: lane tree open, 2: tail
  // chain after the tree).
  enum { TS_P = 0, TS_01 = 1, TS_2 = 2 };
  int tmode = 0;
  auto tload = [&](int k) { return tstate[k * NT + tid]; };
  auto tstore = [&](int k, float a, float b_, float c, float d) { tstate[k * NT + tid] = make_float4(a, b_, c, d); };
  // close the open tree: widen its value once and add it in FP64
  auto flush32 = [&]() {
    float v[4] = {b32[0], b32[1], b32[2], b32[3]};
    if (OUT == OUT_Y && tmode != 0) {
      const float4 s01 = tload(TS_01);
      if (tmode == 1) {
        const float4 pp = tload(TS_P), s2 = tload(TS_2);
        v[0] = s01.x + (s2.x + (pp.x + b32[0]));
        v[1] = s01.y + (s2.y + (pp.y + b32[1]));
        v[2] = s01.z + (s2.z + (pp.z + b32[2]));
        v[3] = s01.w + (s2.w + (pp.w + b32[3]));
        tstore(TS_P, 0.f, 0.f, 0.f, 0.f);
        tstore(TS_2, 0.f, 0.f, 0.f, 0.f);
      } else {
        v[0] = s01.x + b32[0];
        v[1] = s01.y + b32[1];
        v[2] = s01.z + b32[2];
        v[3] = s01.w + b32[3];
      }
      tstore(TS_01, 0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      b[i] += (double)v[i];
      b32[i] = 0.f;
    }
    tmode = 0;
  };
  // the gathered slot holds the FP32 source in its low word and the column's
  // OB_* code in its high word
  auto consume32 = [&](const float4& v, int cc) {
    const double e = gs[cc];
    // sub-chain start: fold the tree (a real branch: the compiler would
    // otherwise predicate the folds onto every column)
    if (OUT == OUT_Y && __double2hiint(e) != OB_NONE) {
      const int code = __double2hiint(e);
      if (code <= OB_ITEM_MAIN) {
        flush32();
        tmode = code == OB_ITEM_MAIN ? 1 : 0;
      } else if (code == OB_B) {
        tstore(TS_P, b32[0], b32[1], b32[2], b32[3]);
        tmode = 1;
      } else if (code < OB_TAIL1) {
        const float4 pp = tload(TS_P);
        const float l0 = pp.x + b32[0], l1 = pp.y + b32[1], l2 = pp.z + b32[2], l3 = pp.w + b32[3];
        if (code == OB_A1) {
          tstore(TS_01, l0, l1, l2, l3);
        } else if (code == OB_A1 + 1) {
          const float4 s01 = tload(TS_01);
          tstore(TS_01, s01.x + l0, s01.y + l1, s01.z + l2, s01.w + l3);
        } else {
          tstore(TS_2, l0, l1, l2, l3);
        }
        tstore(TS_P, 0.f, 0.f, 0.f, 0.f);
        tmode = 1;
      } else {
        const float4 pp = tload(TS_P), s01 = tload(TS_01), s2 = tload(TS_2);
        // main = (l0 + l1) + (l2 + l3)
        const float m0 = s01.x + (s2.x + (pp.x + b32[0])), m1 = s01.y + (s2.y + (pp.y + b32[1]));
        const float m2 = s01.z + (s2.z + (pp.z + b32[2])), m3 = s01.w + (s2.w + (pp.w + b32[3]));
        tstore(TS_P, 0.f, 0.f, 0.f, 0.f);
        tstore(TS_2, 0.f, 0.f, 0.f, 0.f);
        if (code == OB_TAIL1) {  // the one tail column is fused onto main
          tstore(TS_01, 0.f, 0.f, 0.f, 0.f);
          b32[0] = m0, b32[1] = m1, b32[2] = m2, b32[3] = m3;
          tmode = 0;
          goto fma32;
        }
        tstore(TS_01, m0, m1, m2, m3);
        tmode = 2;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) b32[i] = 0.f;
    fma32:
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
      flush32();  // (a tiled part may cut an item between tiles: each piece is closed)
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
        int code;
        double g = src[r.src + ((r.flags & RUN_OBL) ? obl_col(r.width, c, &code) : c)];
        if (r.flags & RUN_ROUND) g = (double)(float)g;
        const int64_t e = (int64_t)(r.col0 + c) * rp + row;
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

// dynamic shared memory of a seg_kernel instantiation: the FP32 lane-tree
// state of stage 2's FP32-accumulated items
template <int M, int O, int NT>
constexpr size_t tree_smem() {
  return (O == OUT_Y && M != F32_ALL64) ? 3 * NT * sizeof(float4) : 0;
}

template <int M, int O, int NT = kSegThreads, bool DEEP = false>
static cudaError_t launch_seg(const DevPlan& P, const Seg* segs, int nseg, const double* x,
                              const S2Out& out, cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)nseg);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = tree_smem<M, O, NT>();
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, seg_kernel<M, O, NT, DEEP>, P, segs, x, out);
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
    case F32_ALL32: return launch_seg<F32_ALL32, OUT_Y>(P, P.seg2, P.n_seg2, x, out, st, pdl);
    case F32_MIXED: return launch_seg<F32_MIXED, OUT_Y>(P, P.seg2, P.n_seg2, x, out, st, pdl);
    default:
      return P.s2_deep ? launch_seg<F32_ALL64, OUT_Y, kSegThreads, true>(P, P.seg2, P.n_seg2, x, out, st, pdl)
                       : launch_seg<F32_ALL64, OUT_Y>(P, P.seg2, P.n_seg2, x, out, st, pdl);
  }
}

// Opt the stage-2 FP32 kernels into > 48 KB of shared memory (static +
// the lane-tree state); called once per plan creation, outside any capture.
cudaError_t configure_kernels() {
  cudaError_t e = cudaFuncSetAttribute(seg_kernel<F32_ALL32, OUT_Y, kSegThreads, false>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)tree_smem<F32_ALL32, OUT_Y, kSegThreads>());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(seg_kernel<F32_MIXED, OUT_Y, kSegThreads, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tree_smem<F32_MIXED, OUT_Y, kSegThreads>());
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
