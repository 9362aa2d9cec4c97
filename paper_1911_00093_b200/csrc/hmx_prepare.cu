// prepare_scheme on the device (reference precision.py:121-162, :241-329).
//
// hmx_master_create uploads the FP64 masters of one H-matrix once.
// hmx_plan_create_prepared then builds a scheme's plan without moving any
// payload over the host link:
//   1. scale_kernel: per low-rank block, the per-column max-abs of U and the
//      per-row max-abs of Vt (scale_decompose, precision.py:121-141), their
//      product d, and for Method 3 the class of every rank,
//      d_i < max(d) * 10**(-c) (split_indices, precision.py:144-162);
//   2. the host flattener (hmx_plan.cu) lays the blobs out from the class
//      counts alone;
//   3. pack_s1_kernel / pack_s2_kernel write every blob element from the
//      masters: divided by the extracted magnitude (IEEE division, as numpy),
//      rounded to FP32 where the scheme stores FP32 (RNE, as astype), with the
//      reference's overflow check and underflow count (_cast_fp32).
// The result is bit-identical to the plan of the host-prepared payloads.
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstring>
#include <thread>
#include <type_traits>

#include "hmx_plan_impl.cuh"

namespace hmx {

// max of non-negative doubles through their bit patterns (order independent)
__device__ __forceinline__ void smem_max(unsigned long long* slot, double v) {
  atomicMax(slot, (unsigned long long)__double_as_longlong(v));
}

// One CTA per low-rank block: colmag/rowmag/d per rank slot, and for
// Method 3 (split) the class (1 = FP64, 2 = FP32) of every rank.
__global__ void scale_kernel(const double* __restrict__ data, const int64_t* __restrict__ table,
                             const int32_t* __restrict__ kind, const int64_t* __restrict__ offset,
                             const int64_t* __restrict__ rank, const int64_t* __restrict__ roff,
                             double* colmag, double* rowmag, double* diag, int8_t* cls, int32_t* nlo,
                             int split, double factor) {
  extern __shared__ unsigned long long mag[];  // 2 x r
  const int k = blockIdx.x;
  if (kind[k] != 1) return;
  const int64_t r = rank[k];
  if (r == 0) {
    if (threadIdx.x == 0) nlo[k] = 0;
    return;
  }
  const int64_t m = table[5 * k + 1] - table[5 * k], n = table[5 * k + 3] - table[5 * k + 2];
  const double* u = data + offset[k];
  const double* vt = u + m * r;
  for (int64_t q = threadIdx.x; q < 2 * r; q += blockDim.x) mag[q] = 0ull;
  __syncthreads();
  for (int64_t e = threadIdx.x; e < m * r; e += blockDim.x) smem_max(mag + e % r, fabs(u[e]));
  for (int64_t e = threadIdx.x; e < r * n; e += blockDim.x) smem_max(mag + r + e / n, fabs(vt[e]));
  __syncthreads();
  const int64_t base = roff[k];
  __shared__ unsigned long long dmax;
  if (threadIdx.x == 0) dmax = 0ull;
  __syncthreads();
  for (int64_t q = threadIdx.x; q < r; q += blockDim.x) {
    const double cm = __longlong_as_double((long long)mag[q]);
    const double rm = __longlong_as_double((long long)mag[r + q]);
    const double d = __dmul_rn(cm, rm);
    colmag[base + q] = cm;
    rowmag[base + q] = rm;
    diag[base + q] = d;
    smem_max(&dmax, d);
  }
  __syncthreads();
  // threshold = max(d) * 10**(-c): the factor is computed by the caller as
  // the reference computes it (precision.py:158)
  const double thr = __dmul_rn(__longlong_as_double((long long)dmax), factor);
  __shared__ int count;
  if (threadIdx.x == 0) count = 0;
  __syncthreads();
  for (int64_t q = threadIdx.x; q < r; q += blockDim.x) {
    const bool lo = split && diag[base + q] < thr;
    cls[base + q] = lo ? 2 : 1;
    if (lo) atomicAdd(&count, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) nlo[k] = count;
}

// returns 1 when the FP32 cast of a nonzero value lands below FLT_MIN
__device__ __forceinline__ unsigned put(double* b64, float* b32, int64_t i, bool is32, double v, int k,
                                        const DevSource& S) {
  if (!is32) {
    b64[i] = v;
    return 0u;
  }
  const float f = __double2float_rn(v);
  b32[i] = f;
  // _cast_fp32 (precision.py:241-253): overflow is an error, underflow counted
  if (isinf(f) && isfinite(v)) atomicMin(S.overflow, (long long)k);
  return (v != 0.0 && fabsf(f) < FLT_MIN) ? 1u : 0u;
}

__device__ __forceinline__ void add_lost(const DevSource& S, unsigned lost) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lost += __shfl_xor_sync(0xffffffffu, lost, o);
  if ((threadIdx.x & 31) == 0 && lost) atomicAdd(S.lost, (unsigned long long)lost);
}

__device__ __forceinline__ double unit(double v, const double* mag, int64_t slot) {
  if (!mag) return v;
  const double g = mag[slot];
  return __ddiv_rn(v, g == 0.0 ? 1.0 : g);  // a zero column/row divides by 1 (precision.py:133-135)
}

// Stage-1 unit: rows (block, class position) x chunk columns, column-major.
__global__ void pack_s1_kernel(DevSource S, const PackS1* __restrict__ units, const PackRow* __restrict__ rows,
                               double* b64, float* b32) {
  const PackS1 u = units[blockIdx.x];
  const int64_t total = (int64_t)u.R * u.w;
  unsigned lost = 0;
  for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
    const int t = (int)(e % u.R), j = (int)(e / u.R);
    const PackRow pr = rows[u.rows + t];
    const int k = pr.block;
    const int64_t* tb = S.table + 5 * k;
    const int64_t m = tb[1] - tb[0], n = tb[3] - tb[2], r = S.rank[k];
    const int64_t slot0 = S.roff[k];
    const int q = S.cls_idx[slot0 + (u.cls == 2 ? S.khi[k] : 0) + pr.q];
    const double v = S.data[S.offset[k] + m * r + (int64_t)q * n + u.c0 + j];
    const int64_t dst = u.dst + (u.chunk ? chunk_off(u.w, u.rp, t, j) : (int64_t)j * u.rp + t);
    lost += put(b64, b32, dst, u.is32, unit(v, S.rowmag, slot0 + q), k, S);
  }
  add_lost(S, lost);
}

// Stage-2 unit: segment rows x items (dense values or U slabs), column-major.
__global__ void pack_s2_kernel(DevSource S, const PackS2* __restrict__ units, const PackItem* __restrict__ items,
                               double* b64, float* b32) {
  const PackS2 u = units[blockIdx.x];
  int64_t col = 0;
  unsigned lost = 0;
  for (int it = 0; it < u.nitems; ++it) {
    const PackItem p = items[u.item0 + it];
    const int k = p.block;
    const int64_t* tb = S.table + 5 * k;
    const int64_t n = tb[3] - tb[2], r = S.rank[k];
    const int64_t r0 = u.row0 - tb[0];
    const int64_t total = (int64_t)u.R * p.width;
    for (int64_t e = threadIdx.x; e < total; e += blockDim.x) {
      const int i = (int)(e % u.R), c = (int)(e / u.R);
      // chain items of group-table parts: SGEMV chunk layout (hmx_internal.cuh)
      const int64_t dst = u.dst + col * u.rp + (p.pad ? chunk_off(p.width, u.rp, i, c) : (int64_t)c * u.rp + i);
      if (p.cls == 0) {
        lost += put(b64, b32, dst, u.is32, S.data[S.offset[k] + (r0 + i) * n + c], k, S);
      } else {
        const int64_t slot0 = S.roff[k];
        const int q = S.cls_idx[slot0 + (p.cls == 2 ? S.khi[k] : 0) + c];
        const double v = S.data[S.offset[k] + (r0 + i) * r + q];
        lost += put(b64, b32, dst, u.is32, unit(v, S.colmag, slot0 + q), k, S);
      }
    }
    col += p.width;
  }
  add_lost(S, lost);
}

// Host -> device copy of a large pageable buffer through pinned windows
// (parallel host copies overlapped with the transfers).
static int staged_upload(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  constexpr size_t kWin = size_t(64) << 20;
  constexpr int kBufs = 3;
  if (bytes < 2 * kWin) {
    HMX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    return cudaStreamSynchronize(st) == cudaSuccess ? HMX_OK : cuda_fail(cudaGetLastError(), "upload");
  }
  void* buf[kBufs] = {};
  cudaEvent_t ev[kBufs] = {};
  int rc = HMX_OK;
  for (int b = 0; b < kBufs && rc == HMX_OK; ++b)
    if (cudaMallocHost(&buf[b], kWin) != cudaSuccess || cudaEventCreateWithFlags(&ev[b], cudaEventDisableTiming) != cudaSuccess)
      rc = cuda_fail(cudaGetLastError(), "pinned staging");
  const int nt = (int)std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  for (size_t off = 0, w = 0; off < bytes && rc == HMX_OK; off += kWin, ++w) {
    const size_t len = std::min(kWin, bytes - off);
    const int b = (int)(w % kBufs);
    if (cudaEventSynchronize(ev[b]) != cudaSuccess) {
      rc = cuda_fail(cudaGetLastError(), "upload");
      break;
    }
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        const size_t a = len * t / nt, e = len * (t + 1) / nt;
        std::memcpy(static_cast<char*>(buf[b]) + a, static_cast<const char*>(src) + off + a, e - a);
      });
    for (auto& x : th) x.join();
    cudaError_t ce = cudaMemcpyAsync(static_cast<char*>(dst) + off, buf[b], len, cudaMemcpyHostToDevice, st);
    if (ce == cudaSuccess) ce = cudaEventRecord(ev[b], st);
    if (ce != cudaSuccess) rc = cuda_fail(ce, "upload");
  }
  cudaError_t ce = cudaStreamSynchronize(st);
  if (rc == HMX_OK && ce != cudaSuccess) rc = cuda_fail(ce, "upload");
  for (int b = 0; b < kBufs; ++b) {
    if (ev[b]) cudaEventDestroy(ev[b]);
    if (buf[b]) cudaFreeHost(buf[b]);
  }
  return rc;
}

template <typename T>
static int upload(std::vector<void*>& keep, T** dst, const std::vector<T>& v, cudaStream_t st) {
  void* p = nullptr;
  HMX_CUDA(cudaMalloc(&p, std::max<size_t>(v.size(), 1) * sizeof(T)));
  keep.push_back(p);
  if (!v.empty()) HMX_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  *dst = static_cast<T*>(p);
  return HMX_OK;
}

int device_pack(const DevSource& src, const std::vector<PackS1>& s1, const std::vector<PackRow>& rows,
                const std::vector<PackS2>& s2, const std::vector<PackItem>& items, double* b64, float* b32,
                cudaStream_t st) {
  std::vector<void*> tmp;
  PackS1* d_s1 = nullptr;
  PackRow* d_rows = nullptr;
  PackS2* d_s2 = nullptr;
  PackItem* d_items = nullptr;
  int rc = HMX_OK;
  if ((rc = upload(tmp, &d_s1, s1, st)) || (rc = upload(tmp, &d_rows, rows, st)) ||
      (rc = upload(tmp, &d_s2, s2, st)) || (rc = upload(tmp, &d_items, items, st))) {
    for (void* p : tmp) cudaFree(p);
    return rc;
  }
  if (!s1.empty()) pack_s1_kernel<<<(unsigned)s1.size(), 256, 0, st>>>(src, d_s1, d_rows, b64, b32);
  if (!s2.empty()) pack_s2_kernel<<<(unsigned)s2.size(), 256, 0, st>>>(src, d_s2, d_items, b64, b32);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  for (void* p : tmp) cudaFree(p);
  if (e != cudaSuccess) return cuda_fail(e, "device_pack");
  return HMX_OK;
}

}  // namespace hmx

using namespace hmx;

extern "C" {

void hmx_master_destroy(hmx_master* m) {
  if (!m) return;
  {
    DeviceGuard g(m->device);
    if (m->stream) cudaStreamSynchronize(m->stream);
    for (void* a : m->allocs) cudaFree(a);
    if (m->stream) cudaStreamDestroy(m->stream);
  }
  delete m;
}

int hmx_master_create(const hmx_master_desc* d, int device, hmx_master** out) {
  if (!d || !out || !d->perm || !d->table || !d->kind || !d->offset || !d->rank || !d->data) {
    set_error("null argument");
    return HMX_ERR_ARG;
  }
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    set_error("no CUDA device is available");
    return HMX_ERR_CUDA;
  }
  if (device < 0 || device >= count) {
    set_error("device index out of range");
    return HMX_ERR_ARG;
  }
  const int64_t n = d->n, nb = d->n_blocks;
  if (n < 1 || nb < 1 || d->n_data < 0) {
    set_error("invalid master descriptor");
    return HMX_ERR_ARG;
  }
  DeviceGuard guard(device);
  auto* m = new hmx_master();
  m->device = device;
  m->n = n;
  m->nb = nb;
  m->n_data = d->n_data;
  m->perm.assign(d->perm, d->perm + n);
  m->table.assign(d->table, d->table + 5 * nb);
  m->kind.assign(d->kind, d->kind + nb);
  m->offset.assign(d->offset, d->offset + nb);
  m->rank.assign(d->rank, d->rank + nb);
  m->roff.assign((size_t)nb, 0);
  for (int64_t k = 0; k < nb; ++k) {
    const int64_t* t = d->table + 5 * k;
    const int64_t rows = t[1] - t[0], cols = t[3] - t[2];
    const int64_t r = d->kind[k] == 1 ? d->rank[k] : 0;
    const int64_t need = d->kind[k] == 0 ? rows * cols : d->kind[k] == 1 ? r * (rows + cols) : 0;
    if (rows < 1 || cols < 1 || r < 0 || (need && (d->offset[k] < 0 || d->offset[k] + need > d->n_data))) {
      hmx_master_destroy(m);
      set_error("block " + std::to_string(k) + " exceeds the master buffer");
      return HMX_ERR_ARG;
    }
    m->roff[(size_t)k] = m->rank_sum;
    m->rank_sum += r;
    m->max_rank = std::max(m->max_rank, r);
  }
  cudaError_t e = cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    hmx_master_destroy(m);
    return cuda_fail(e, "cudaStreamCreate");
  }
  int rc = HMX_OK;
  auto up = [&](auto** dst, const auto* src, size_t count) {
    using T = typename std::remove_pointer<typename std::remove_reference<decltype(*dst)>::type>::type;
    *dst = m->alloc<T>(count);
    if (!*dst) {
      set_error("cudaMalloc failed while uploading the masters (out of device memory?)");
      rc = HMX_ERR_CUDA;
      return;
    }
    if (count) {
      cudaError_t ce = cudaMemcpyAsync(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice, m->stream);
      if (ce != cudaSuccess) rc = cuda_fail(ce, "master upload");
    }
  };
  m->data = m->alloc<double>((size_t)d->n_data);
  if (!m->data) {
    set_error("cudaMalloc failed while uploading the masters (out of device memory?)");
    rc = HMX_ERR_CUDA;
  } else if (d->n_data) {
    rc = staged_upload(m->data, d->data, (size_t)d->n_data * sizeof(double), m->stream);
  }
  if (!rc) up(&m->d_table, d->table, (size_t)(5 * nb));
  if (!rc) up(&m->d_kind, d->kind, (size_t)nb);
  if (!rc) up(&m->d_offset, d->offset, (size_t)nb);
  if (!rc) up(&m->d_rank, d->rank, (size_t)nb);
  if (!rc) up(&m->d_roff, m->roff.data(), (size_t)nb);
  if (!rc) {
    e = cudaStreamSynchronize(m->stream);
    if (e != cudaSuccess) rc = cuda_fail(e, "master upload");
  }
  if (rc) {
    hmx_master_destroy(m);
    return rc;
  }
  *out = m;
  return HMX_OK;
}

int hmx_plan_create_prepared(hmx_master* m, int scheme, double split_factor, const hmx_plan_options* opt,
                             hmx_plan** out, hmx_prepare_info* info) {
  NvtxRange nvtx("hmx_plan_create_prepared");
  if (!m || !out) {
    set_error("null argument");
    return HMX_ERR_ARG;
  }
  *out = nullptr;
  if (scheme < HMX_M1_DOUBLE || scheme > HMX_M3) {
    set_error("invalid scheme");
    return HMX_ERR_ARG;
  }
  if (info) *info = hmx_prepare_info{0, 0, -1, 0};
  DeviceGuard guard(m->device);
  const int64_t nb = m->nb, R = m->rank_sum;
  const bool scaled = scheme >= HMX_M2_DOUBLE, split = scheme == HMX_M3;
  // storage flags per scheme (precision.py:79-87, :271-320)
  const bool a32 = scheme == HMX_M1_SINGLE || scheme == HMX_M1_MIXED || scheme == HMX_M2_SINGLE ||
                   scheme == HMX_M2_MIXED;
  const bool hi32 = a32;

  std::vector<void*> tmp;
  auto cleanup = [&]() {
    for (void* p : tmp) cudaFree(p);
    tmp.clear();
  };
  auto dalloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(bytes, 8)) != cudaSuccess) return nullptr;
    tmp.push_back(p);
    return p;
  };
  double* colmag = (double*)dalloc(R * 8);
  double* rowmag = (double*)dalloc(R * 8);
  double* diag = (double*)dalloc(R * 8);
  int8_t* cls = (int8_t*)dalloc(R);
  int32_t* nlo = (int32_t*)dalloc(nb * 4);
  unsigned long long* lost = (unsigned long long*)dalloc(8);
  long long* ovf = (long long*)dalloc(8);
  if (!colmag || !rowmag || !diag || !cls || !nlo || !lost || !ovf) {
    cleanup();
    set_error("cudaMalloc failed while preparing the scheme (out of device memory?)");
    return HMX_ERR_CUDA;
  }
  cudaStream_t st = m->stream;
  const long long none = LLONG_MAX;
  HMX_CUDA(cudaMemsetAsync(lost, 0, 8, st));
  HMX_CUDA(cudaMemcpyAsync(ovf, &none, 8, cudaMemcpyHostToDevice, st));
  HMX_CUDA(cudaMemsetAsync(nlo, 0, nb * 4, st));

  std::vector<int8_t> h_cls((size_t)R, 1);
  std::vector<double> h_diag((size_t)R, 0.0);
  std::vector<int32_t> h_nlo((size_t)nb, 0);
  if (scaled && R > 0) {
    const size_t smem = (size_t)(2 * std::max<int64_t>(m->max_rank, 1)) * 8;
    if (smem > 200 * 1024) {
      cleanup();
      set_error("rank too large for the device scaling kernel");
      return HMX_ERR_ARG;
    }
    if (smem > 48 * 1024)
      HMX_CUDA(cudaFuncSetAttribute(scale_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    scale_kernel<<<(unsigned)nb, 256, smem, st>>>(m->data, m->d_table, m->d_kind, m->d_offset, m->d_rank,
                                                m->d_roff, colmag, rowmag, diag, cls, nlo, split ? 1 : 0,
                                                split_factor);
    HMX_CUDA(cudaGetLastError());
    HMX_CUDA(cudaMemcpyAsync(h_cls.data(), cls, (size_t)R, cudaMemcpyDeviceToHost, st));
    HMX_CUDA(cudaMemcpyAsync(h_diag.data(), diag, (size_t)R * 8, cudaMemcpyDeviceToHost, st));
    HMX_CUDA(cudaMemcpyAsync(h_nlo.data(), nlo, (size_t)nb * 4, cudaMemcpyDeviceToHost, st));
    HMX_CUDA(cudaStreamSynchronize(st));
  }

  // class order per block: FP64-class ranks ascending, then FP32-class ones
  // (split_indices returns ascending index lists, precision.py:160-162)
  std::vector<int64_t> khi((size_t)nb, 0), klo((size_t)nb, 0), dhi_off((size_t)nb, -1),
      dlo_off((size_t)nb, -1), zero((size_t)nb, 0);
  std::vector<int32_t> cls_idx((size_t)std::max<int64_t>(R, 1), 0);
  std::vector<double> diag_cls((size_t)std::max<int64_t>(R, 1), 0.0);
  for (int64_t k = 0; k < nb; ++k) {
    if (m->kind[(size_t)k] != 1) continue;
    const int64_t r = m->rank[(size_t)k], b = m->roff[(size_t)k];
    int64_t pos = b;
    for (int pass = 1; pass <= 2; ++pass)
      for (int64_t q = 0; q < r; ++q)
        if (h_cls[(size_t)(b + q)] == pass) {
          cls_idx[(size_t)pos] = (int32_t)q;
          diag_cls[(size_t)pos] = h_diag[(size_t)(b + q)];
          ++pos;
        }
    klo[(size_t)k] = split ? h_nlo[(size_t)k] : 0;
    khi[(size_t)k] = r - klo[(size_t)k];
    if (scaled) {
      dhi_off[(size_t)k] = b;
      dlo_off[(size_t)k] = b + khi[(size_t)k];
    }
  }
  int32_t* d_cls_idx = nullptr;
  int64_t* d_khi = nullptr;
  {
    int rc = upload(tmp, &d_cls_idx, cls_idx, st);
    if (!rc) rc = upload(tmp, &d_khi, khi, st);
    if (rc) {
      cleanup();
      return rc;
    }
  }

  // virtual descriptor: the flattener needs the layout (class counts, the
  // diagonal for z scaling); payload values come from DevSource
  const int64_t huge = INT64_MAX / 4;
  hmx_matrix_desc vd{};
  vd.n = m->n;
  vd.n_blocks = nb;
  vd.scheme = scheme;
  vd.a32 = a32;
  vd.hi32 = hi32;
  vd.perm = m->perm.data();
  vd.table = m->table.data();
  vd.kind = m->kind.data();
  vd.a_off = zero.data();
  vd.hi_off = zero.data();
  vd.khi = khi.data();
  vd.dhi_off = dhi_off.data();
  vd.lo_off = zero.data();
  vd.klo = klo.data();
  vd.dlo_off = dlo_off.data();
  vd.buf64 = diag_cls.data();
  vd.n64 = huge;
  vd.buf32 = nullptr;
  vd.n32 = huge;

  DevSource src;
  src.data = m->data;
  src.table = m->d_table;
  src.offset = m->d_offset;
  src.rank = m->d_rank;
  src.roff = m->d_roff;
  src.khi = d_khi;
  src.cls_idx = d_cls_idx;
  src.colmag = scaled ? colmag : nullptr;
  src.rowmag = scaled ? rowmag : nullptr;
  src.lost = lost;
  src.overflow = ovf;

  auto* p = new hmx_plan();
  p->device = m->device;
  p->n = m->n;
  p->scheme = scheme;
  cudaError_t e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete p;
    cleanup();
    return cuda_fail(e, "cudaStreamCreate");
  }
  // the pack kernels run on the plan's stream after the uploads above
  cudaStreamSynchronize(st);
  int rc = plan_create_impl(&vd, m->device, opt, p, &src);
  long long h_ovf = none;
  unsigned long long h_lost = 0;
  if (rc == HMX_OK) {
    cudaMemcpy(&h_ovf, ovf, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&h_lost, lost, 8, cudaMemcpyDeviceToHost);
  }
  cleanup();
  if (rc != HMX_OK) {
    hmx_plan_destroy(p);
    return rc;
  }
  int64_t lo_ranks = 0;
  for (int64_t k = 0; k < nb; ++k) lo_ranks += klo[(size_t)k];
  if (info) {
    info->payload_bytes = p->info.payload_bytes;
    info->underflow_count = (int64_t)h_lost;
    info->overflow_block = h_ovf == none ? -1 : (int64_t)h_ovf;
    info->fp32_ranks = lo_ranks;
  }
  if (h_ovf != none) {
    hmx_plan_destroy(p);
    set_error("FP32 overflow while casting block " + std::to_string(h_ovf));
    return HMX_ERR_OVERFLOW;
  }
  *out = p;
  return HMX_OK;
}

}  // extern "C"
