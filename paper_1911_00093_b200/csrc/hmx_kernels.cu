// sm_100a kernels of the H-matrix vector product.  See hmx_internal.cuh for
// the data layout; precision pipelines follow reference
// pkg/src/hmx/matvec.py:55-110 (table in SURVEY.md s0.1):
//
//   pipe  stage-1 z = Vt x                    stage-2 per item partial
//   m1d   f64                                 f64
//   m1s   f32 data, f32(x), f32 accumulate     dense A32.x32 f32-acc; U32.z32 f32-acc
//   m1m   f32 data widened, f64 acc, z->f32    dense widened f64; U32.z32 f32-acc
//   m2d   f64, z *= d                          f64
//   m2s   f32 widened . widen(f32(x)), z *= d  dense A32.x32 f32-acc; U widened f64
//   m2m   f32 widened . x, z *= d              dense widened f64; U widened f64
//   m3    hi f64 / lo f32 widened, z *= d      dense f64; U_hi f64; U_lo widened f64
//
// Every f32-accumulated item partial is widened once and added in f64.
#include "hmx_kernels.cuh"

namespace hmx {

// ------------------------------------------------------------------------------
// stage 1

template <int PIPE>
struct S1Pipe {
  // float32 tasks accumulate in float32 only for m1-single (matvec.py:68-69)
  static constexpr bool acc32 = PIPE == P_M1S;
  // the FP32 source shadow: m1-single (float) and m2-single (widened) (matvec.py:77-78, :119)
  static constexpr bool round_src = PIPE == P_M1S || PIPE == P_M2S;
  static constexpr bool has64 = PIPE == P_M1D || PIPE == P_M2D || PIPE == P_M3;
  static constexpr bool has32 = PIPE != P_M1D && PIPE != P_M2D;
};

// Transpose-butterfly warp reduction of N per-lane values (N = 2^b <= 16):
// each step halves the live values per lane; afterwards the lane holds the
// full sum of rank index k(lane) (see s1_rank_of_lane).  Fixed order.
template <int N, int S, typename A>
struct Butterfly {
  static __device__ __forceinline__ void run(A* acc, int lane) {
    if constexpr (S > 0) {
      if constexpr (N > 1) {
        constexpr int H = N / 2;
        const bool up = (lane & S) != 0;
#pragma unroll
        for (int j = 0; j < H; ++j) {
          const A send = up ? acc[j] : acc[j + H];
          const A keep = up ? acc[j + H] : acc[j];
          acc[j] = keep + __shfl_xor_sync(0xffffffffu, send, S);
        }
        Butterfly<H, S / 2, A>::run(acc, lane);
      } else {
        acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], S);
        Butterfly<1, S / 2, A>::run(acc, lane);
      }
    }
  }
};

template <int N>
__device__ __forceinline__ int s1_rank_of_lane(int lane, bool& writer) {
  constexpr int b = N == 16 ? 4 : N == 8 ? 3 : N == 4 ? 2 : N == 2 ? 1 : 0;
  int k = 0;
#pragma unroll
  for (int i = 0; i < b; ++i) k |= ((lane >> (4 - i)) & 1) << (b - 1 - i);
  writer = (lane & ((1 << (5 - b)) - 1)) == 0;
  return k;
}

template <typename T>
struct Vec16;
template <>
struct Vec16<double> {
  using type = double2;
  static constexpr int V = 2;
  static __device__ __forceinline__ double get(const double2& v, int i) { return i == 0 ? v.x : v.y; }
};
template <>
struct Vec16<float> {
  using type = float4;
  static constexpr int V = 4;
  static __device__ __forceinline__ float get(const float4& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
  }
};

template <int PIPE, typename T>
__device__ __forceinline__ double s1_epilogue(double v, const double* zscale, int zi) {
  if constexpr (PIPE == P_M1D) {
    return v;
  } else if constexpr (PIPE == P_M1S || PIPE == P_M1M) {
    // m1-single: float accumulator widened; m1-mixed: f64 product rounded
    // once into the FP32 intermediate (matvec.py:70-72)
    return (double)(float)v;
  } else {
    return v * zscale[zi];  // z *= diag (matvec.py:81, :88, :92)
  }
}

template <int PIPE, typename T, int RB>
__device__ __forceinline__ void s1_task(const DevPlan& P, const S1Task& t, const double* __restrict__ x,
                                        int lane, uint64_t pol) {
  using VT = typename Vec16<T>::type;
  constexpr int V = Vec16<T>::V;
  constexpr bool ACC32 = S1Pipe<PIPE>::acc32 && sizeof(T) == 4;
  constexpr bool ROUND = S1Pipe<PIPE>::round_src && sizeof(T) == 4;
  using A = typename std::conditional<ACC32, float, double>::type;

  const T* __restrict__ base = (sizeof(T) == 8 ? (const T*)P.vt64 : (const T*)P.vt32) + t.vt_off;
  const double* __restrict__ xs = x + t.xoff;
  const int R = t.R, ld = t.ld, ncols = t.ncols;
  A acc[RB];
#pragma unroll
  for (int k = 0; k < RB; ++k) acc[k] = A(0);

  for (int c = lane * V; c < ncols; c += 32 * V) {
    A xv[V];
#pragma unroll
    for (int i = 0; i < V; ++i) {
      double xi = (c + i < ncols) ? __ldg(xs + c + i) : 0.0;
      if constexpr (ROUND) xi = (double)(float)xi;
      xv[i] = (A)xi;
    }
    // rank rows in groups of <= 8 loads in flight per lane (register budget)
    constexpr int KG = RB < 8 ? RB : 8;
#pragma unroll
    for (int kb = 0; kb < RB; kb += KG) {
      VT m[KG];
#pragma unroll
      for (int k = 0; k < KG; ++k)
        if (kb + k < R) m[k] = ld_stream(base + (int64_t)(kb + k) * ld + c, pol);
#pragma unroll
      for (int k = 0; k < KG; ++k) {
        if (kb + k < R) {
#pragma unroll
          for (int i = 0; i < V; ++i) acc[kb + k] = fma((A)Vec16<T>::get(m[k], i), xv[i], acc[kb + k]);
        }
      }
    }
  }

  Butterfly<RB, 16, A>::run(acc, lane);
  bool writer;
  const int k = s1_rank_of_lane<RB>(lane, writer);
  const S1Seg sg = P.s1segs[t.seg];
  const bool mine = writer && k < R;
  if (sg.nchunks == 1) {
    if (mine) P.z[sg.zoff + k] = s1_epilogue<PIPE, T>((double)acc[0], P.zscale, sg.zoff + k);
    return;
  }
  // multi-chunk segment: publish the partial; the last arriving task sums
  // every chunk in chunk order (deterministic) and applies the epilogue.
  if (mine) P.part[sg.part_off + t.chunk * R + k] = (double)acc[0];
  __threadfence();
  __syncwarp();
  unsigned ticket = 0;
  if (lane == 0) ticket = atomicAdd(P.seg_count + t.seg, 1u);
  ticket = __shfl_sync(0xffffffffu, ticket, 0);
  if (ticket != (unsigned)(sg.nchunks - 1)) return;
  __threadfence();
  if (lane < R) {
    A s = A(0);
    for (int ch = 0; ch < sg.nchunks; ++ch) s += (A)__ldcg(P.part + sg.part_off + ch * R + lane);
    P.z[sg.zoff + lane] = s1_epilogue<PIPE, T>((double)s, P.zscale, sg.zoff + lane);
  }
  if (lane == 0) P.seg_count[t.seg] = 0u;  // ready for the next matvec
}

template <int PIPE>
__global__ void __launch_bounds__(kS1Threads, 2) s1_kernel(DevPlan P, const double* __restrict__ x) {
  const int warp = (int)((blockIdx.x * kS1Threads + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (warp >= P.n_warps) return;
  const uint64_t pol = policy_evict_first();
  const int t0 = P.warp_ptr[warp], t1 = P.warp_ptr[warp + 1];
  for (int ti = t0; ti < t1; ++ti) {
    const S1Task t = P.tasks[ti];
    if (t.is32) {
      if constexpr (S1Pipe<PIPE>::has32) {
        if (t.R <= 4) s1_task<PIPE, float, 4>(P, t, x, lane, pol);
        else if (t.R <= 8) s1_task<PIPE, float, 8>(P, t, x, lane, pol);
        else s1_task<PIPE, float, 16>(P, t, x, lane, pol);
      }
    } else {
      if constexpr (S1Pipe<PIPE>::has64) {
        if (t.R <= 4) s1_task<PIPE, double, 4>(P, t, x, lane, pol);
        else if (t.R <= 8) s1_task<PIPE, double, 8>(P, t, x, lane, pol);
        else s1_task<PIPE, double, 16>(P, t, x, lane, pol);
      }
    }
  }
  // let the dependent stage-2 grid start its z-independent prologue
  asm volatile("griddepcontrol.launch_dependents;");
}

// ------------------------------------------------------------------------------
// stage 2

// Stage a tile [tc0, tc0+tw) of one part's source vector g (x segments and z
// vectors, in item order) into shared memory, plus FP32-part item flags.
template <bool FLAGS>
__device__ __forceinline__ void s2_gather(const DevPlan& P, const Run* __restrict__ runs, int nrun,
                                          int tc0, int tw, const double* __restrict__ x,
                                          double* gs, uint8_t* fl) {
  for (int c = threadIdx.x; c < tw; c += blockDim.x) {
    const int col = tc0 + c;
    int lo = 0, hi = nrun - 1;  // last run with col0 <= col
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldg(&runs[mid].col0) <= col) lo = mid;
      else hi = mid - 1;
    }
    const Run r = runs[lo];
    const int off = col - r.col0;
    const double* src = (r.flags & RUN_Z) ? P.z : x;
    double g = src[r.src + off];
    if (r.flags & RUN_ROUND) g = (double)(float)g;
    gs[c] = g;
    if constexpr (FLAGS) fl[c] = (uint8_t)((off == 0 ? 1 : 0) | ((r.flags & RUN_ACC32) ? 2 : 0));
  }
}

template <int F32MODE>
__global__ void __launch_bounds__(kS2Threads) s2_kernel(DevPlan P, const double* __restrict__ x,
                                                         S2Out out) {
  __shared__ double gs[kS2WMax];
  __shared__ uint8_t fl[kS2WMax];
  __shared__ double red64[2 * kS2Threads];
  __shared__ double red32[4 * kS2Threads];
  __shared__ double wred[2][8];

  const S2Seg sg = P.s2segs[blockIdx.x];
  const int R = sg.R;
  const int tid = threadIdx.x;
  const uint64_t pol = policy_evict_first();

  // the z-independent prologue overlaps stage 1's tail (PDL); z is read only
  // after the dependency resolves
  asm volatile("griddepcontrol.wait;" ::: "memory");

  // ---------------- FP64 part: 2 rows x 16 bytes per thread
  const int rp64 = (R + 1) & ~1;
  const int tpg64 = rp64 >> 1;
  const int g64 = kS2Threads / tpg64;
  const int q64 = tid / tpg64, p64 = tid - q64 * tpg64;
  double a0 = 0.0, a1 = 0.0;
  for (int tc0 = 0; tc0 < sg.W64; tc0 += kS2WMax) {
    const int tw = min(kS2WMax, sg.W64 - tc0);
    __syncthreads();
    s2_gather<false>(P, P.runs + sg.run0, sg.nrun64, tc0, tw, x, gs, fl);
    __syncthreads();
    if (q64 < g64) {
      const int cb = (int)((int64_t)tw * q64 / g64), ce = (int)((int64_t)tw * (q64 + 1) / g64);
      const double* __restrict__ col = P.blob64 + sg.off64 + (int64_t)tc0 * rp64 + 2 * p64;
      int c = cb;
      for (; c + 8 <= ce; c += 8) {
        double2 m[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) m[u] = ld_stream(col + (int64_t)(c + u) * rp64, pol);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double g = gs[c + u];
          a0 = fma(m[u].x, g, a0);
          a1 = fma(m[u].y, g, a1);
        }
      }
      for (; c < ce; ++c) {
        const double2 m = ld_stream(col + (int64_t)c * rp64, pol);
        const double g = gs[c];
        a0 = fma(m.x, g, a0);
        a1 = fma(m.y, g, a1);
      }
    }
  }

  // ---------------- FP32 part: 4 rows x 16 bytes per thread
  const int rp32 = (R + 3) & ~3;
  const int tpg32 = rp32 >> 2;
  const int g32 = kS2Threads / tpg32;
  const int q32 = tid / tpg32, p32 = tid - q32 * tpg32;
  double b[4] = {0.0, 0.0, 0.0, 0.0};
  float b32[4] = {0.f, 0.f, 0.f, 0.f};
  for (int tc0 = 0; tc0 < sg.W32; tc0 += kS2WMax) {
    const int tw = min(kS2WMax, sg.W32 - tc0);
    __syncthreads();
    s2_gather<F32MODE != F32_ALL64>(P, P.runs + sg.run0 + sg.nrun64, sg.nrun32, tc0, tw, x, gs, fl);
    __syncthreads();
    if (q32 < g32) {
      const int cb = (int)((int64_t)tw * q32 / g32), ce = (int)((int64_t)tw * (q32 + 1) / g32);
      const float* __restrict__ col = P.blob32 + sg.off32 + (int64_t)tc0 * rp32 + 4 * p32;
      int c = cb;
      auto consume = [&](const float4& m, int cc) {
        const double g = gs[cc];
        const float mv[4] = {m.x, m.y, m.z, m.w};
        if constexpr (F32MODE == F32_ALL64) {
#pragma unroll
          for (int i = 0; i < 4; ++i) b[i] = fma((double)mv[i], g, b[i]);
        } else {
          const uint8_t f = fl[cc];
          if (f & 1) {  // first column of an item: close the previous f32 partial
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              b[i] += (double)b32[i];
              b32[i] = 0.f;
            }
          }
          if (F32MODE == F32_ALL32 || (f & 2)) {
            const float gf = (float)g;
#pragma unroll
            for (int i = 0; i < 4; ++i) b32[i] = fmaf(mv[i], gf, b32[i]);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) b[i] = fma((double)mv[i], g, b[i]);
          }
        }
      };
      for (; c + 8 <= ce; c += 8) {
        float4 m[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) m[u] = ld_stream(col + (int64_t)(c + u) * rp32, pol);
#pragma unroll
        for (int u = 0; u < 8; ++u) consume(m[u], c + u);
      }
      for (; c < ce; ++c) consume(ld_stream(col + (int64_t)c * rp32, pol), c);
    }
  }
  if constexpr (F32MODE != F32_ALL64) {
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] += (double)b32[i];
  }

  // ---------------- fixed-order reduction over thread groups
  __syncthreads();
  if (sg.W64 > 0 && q64 < g64) {
    red64[q64 * rp64 + 2 * p64] = a0;
    red64[q64 * rp64 + 2 * p64 + 1] = a1;
  }
  if (sg.W32 > 0 && q32 < g32) {
#pragma unroll
    for (int i = 0; i < 4; ++i) red32[q32 * rp32 + 4 * p32 + i] = b[i];
  }
  __syncthreads();

  double d0 = 0.0, d1 = 0.0;
  if (tid < R) {
    double s = 0.0;
    if (sg.W64 > 0)
      for (int q = 0; q < g64; ++q) s += red64[q * rp64 + tid];
    if (sg.W32 > 0)
      for (int q = 0; q < g32; ++q) s += red32[q * rp32 + tid];
    const int row = sg.row0 + tid;
    const int li = row - P.row_begin;
    if (!isfinite(s)) *out.nonfinite = 1;
    if (out.permute_out) out.y[P.perm[row]] = s;
    else out.y[li] = s;
    if (out.w1) d0 = s * out.w1[li];
    if (out.yy) d1 = s * s;
  }
  if (out.seg_dots == nullptr) return;

  // per-segment dot partials (rows < 64: warps 0 and 1), then the last CTA
  // reduces all segment partials in segment order
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    d0 += __shfl_xor_sync(0xffffffffu, d0, s);
    d1 += __shfl_xor_sync(0xffffffffu, d1, s);
  }
  if (lane == 0) {
    wred[0][wid] = d0;
    wred[1][wid] = d1;
  }
  __syncthreads();
  __shared__ unsigned ticket;
  if (tid == 0) {
    double e0 = 0.0, e1 = 0.0;
    for (int w = 0; w < kS2Threads / 32; ++w) {
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
  for (int i = tid; i < (int)gridDim.x; i += kS2Threads) {
    e0 += __ldcg(out.seg_dots + 2 * i);
    e1 += __ldcg(out.seg_dots + 2 * i + 1);
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    e0 += __shfl_xor_sync(0xffffffffu, e0, s);
    e1 += __shfl_xor_sync(0xffffffffu, e1, s);
  }
  __syncthreads();
  if (lane == 0) {
    wred[0][wid] = e0;
    wred[1][wid] = e1;
  }
  __syncthreads();
  if (tid == 0) {
    double f0 = 0.0, f1 = 0.0;
    for (int w = 0; w < kS2Threads / 32; ++w) {
      f0 += wred[0][w];
      f1 += wred[1][w];
    }
    out.dots_out[0] = f0;
    out.dots_out[1] = f1;
    *out.done = 0u;
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
// every item (block slab) on its own, in the scheme's precision, and records
// the smallest block index whose contribution is not finite.
__global__ void probe_kernel(DevPlan P, const double* __restrict__ x, unsigned long long* first_bad) {
  const S2Seg sg = P.s2segs[blockIdx.x];
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

cudaError_t launch_stage1(const DevPlan& P, const double* x, int grid, cudaStream_t st) {
  if (P.n_warps == 0) return cudaSuccess;
  switch (P.pipe) {
    case P_M1D: s1_kernel<P_M1D><<<grid, kS1Threads, 0, st>>>(P, x); break;
    case P_M1S: s1_kernel<P_M1S><<<grid, kS1Threads, 0, st>>>(P, x); break;
    case P_M1M: s1_kernel<P_M1M><<<grid, kS1Threads, 0, st>>>(P, x); break;
    case P_M2D: s1_kernel<P_M2D><<<grid, kS1Threads, 0, st>>>(P, x); break;
    case P_M2S: s1_kernel<P_M2S><<<grid, kS1Threads, 0, st>>>(P, x); break;
    case P_M2M: s1_kernel<P_M2M><<<grid, kS1Threads, 0, st>>>(P, x); break;
    default: s1_kernel<P_M3><<<grid, kS1Threads, 0, st>>>(P, x); break;
  }
  return cudaGetLastError();
}

template <int M>
static cudaError_t launch_s2_mode(const DevPlan& P, const double* x, const S2Out& out,
                                  cudaStream_t st, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)P.n_s2);
  cfg.blockDim = dim3(kS2Threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, s2_kernel<M>, P, x, out);
}

cudaError_t launch_stage2(const DevPlan& P, const double* x, const S2Out& out, cudaStream_t st,
                          bool pdl) {
  if (P.n_s2 == 0) return cudaSuccess;
  switch (P.f32mode) {
    case F32_ALL32: return launch_s2_mode<F32_ALL32>(P, x, out, st, pdl);
    case F32_MIXED: return launch_s2_mode<F32_MIXED>(P, x, out, st, pdl);
    default: return launch_s2_mode<F32_ALL64>(P, x, out, st, pdl);
  }
}

cudaError_t launch_gather_perm(const double* x, const int32_t* perm, double* xp, int n,
                               cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  gather_perm_kernel<<<(n + 255) / 256, 256, 0, st>>>(x, perm, xp, n);
  return cudaGetLastError();
}

cudaError_t launch_probe(const DevPlan& P, const double* x, unsigned long long* first_bad,
                         cudaStream_t st) {
  if (P.n_s2 == 0) return cudaSuccess;
  probe_kernel<<<P.n_s2, 64, 0, st>>>(P, x, first_bad);
  return cudaGetLastError();
}

int stage1_occupancy(int pipe) {
  int blocks = 0;
  switch (pipe) {
    case P_M1D: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, s1_kernel<P_M1D>, kS1Threads, 0); break;
    case P_M1S: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, s1_kernel<P_M1S>, kS1Threads, 0); break;
    case P_M1M: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, s1_kernel<P_M1M>, kS1Threads, 0); break;
    case P_M2D: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, s1_kernel<P_M2D>, kS1Threads, 0); break;
    case P_M2S: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, s1_kernel<P_M2S>, kS1Threads, 0); break;
    case P_M2M: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, s1_kernel<P_M2M>, kS1Threads, 0); break;
    default: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, s1_kernel<P_M3>, kS1Threads, 0); break;
  }
  return blocks > 0 ? blocks : 1;
}

}  // namespace hmx
