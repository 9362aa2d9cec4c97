// Host-side H-matrix builder: icosphere meshes, cluster tree, admissible
// block partition, ACA compression, dense near-field fill, and the per-scheme
// payload preparation (Method-2 scaling, Method-3 splitting).
//
// This is NOT the hot path (the reference builds and prepares untimed, see
// reference pkg/src/hmx/bench.py:174).  It exists because the GPU box has no
// copy of the reference, and because the reference's pure-Python build takes
// 442 s at N = 327,680.  Every routine restates the
// reference's algorithm with the same floating-point operation order where
// numpy's order is known:
//   * 1-D np.linalg.norm of a 3-vector is OpenBLAS ddot = an FMA chain
//     (measured in this container);
//   * numpy reductions over a length-3 axis are left-to-right, no FMA.
// BLAS-backed ACA updates (dgemv/ddot of arbitrary length) cannot be matched
// bit-for-bit; they agree to a few ulps (tests/test_builder_vs_reference.py).
//
// Build: g++ -O3 -std=c++17 -ffp-contract=off -fPIC -shared -pthread
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <unordered_map>
#include <numeric>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "aca_core.h"

namespace {

using namespace hmx_aca;

int run_parallel(int64_t count, int nthreads, const std::function<void(int64_t)>& fn) {
  if (nthreads <= 0) nthreads = (int)std::max(1u, std::thread::hardware_concurrency());
  if (count <= 0) return 0;
  if (nthreads == 1 || count == 1) {
    for (int64_t i = 0; i < count; ++i) fn(i);
    return 0;
  }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> pool;
  const int nt = (int)std::min<int64_t>(nthreads, count);
  for (int t = 0; t < nt; ++t) {
    pool.emplace_back([&]() {
      for (;;) {
        const int64_t i = next.fetch_add(1);
        if (i >= count) break;
        fn(i);
      }
    });
  }
  for (auto& th : pool) th.join();
  return 0;
}

void set_err(char* err, int errlen, const std::string& msg) {
  if (err && errlen > 0) {
    std::snprintf(err, (size_t)errlen, "%s", msg.c_str());
  }
}
}  // namespace

extern "C" {

// ---------------------------------------------------------------------------
// Icosphere (restates reference problem.py:99-143).

int64_t hb_icosphere_nverts(int level) { return 10 * (int64_t(1) << (2 * level)) + 2; }
int64_t hb_icosphere_nfaces(int level) { return 20 * (int64_t(1) << (2 * level)); }

// verts: (nverts x 3) float64, faces: (nfaces x 3) int64.  Vertex creation
// order and face order follow the reference's subdivision exactly so meshes
// are identical element-for-element.
int hb_icosphere(int level, double* verts, int64_t* faces) {
  if (level < 0) return -1;
  const double phi = (1.0 + std::sqrt(5.0)) / 2.0;
  const double base[12][3] = {
      {-1.0, phi, 0.0}, {1.0, phi, 0.0}, {-1.0, -phi, 0.0}, {1.0, -phi, 0.0},
      {0.0, -1.0, phi}, {0.0, 1.0, phi}, {0.0, -1.0, -phi}, {0.0, 1.0, -phi},
      {phi, 0.0, -1.0}, {phi, 0.0, 1.0}, {-phi, 0.0, -1.0}, {-phi, 0.0, 1.0}};
  const int64_t tris[20][3] = {
      {0, 11, 5}, {0, 5, 1}, {0, 1, 7}, {0, 7, 10}, {0, 10, 11},
      {1, 5, 9}, {5, 11, 4}, {11, 10, 2}, {10, 7, 6}, {7, 1, 8},
      {3, 9, 4}, {3, 4, 2}, {3, 2, 6}, {3, 6, 8}, {3, 8, 9},
      {4, 9, 5}, {2, 4, 11}, {6, 2, 10}, {8, 6, 7}, {9, 8, 1}};
  int64_t nv = 0;
  for (int i = 0; i < 12; ++i) {
    const double nrm = norm_fma(base[i], 3);
    for (int d = 0; d < 3; ++d) verts[3 * nv + d] = base[i][d] / nrm;
    ++nv;
  }
  std::vector<int64_t> cur(60), nxt;
  for (int i = 0; i < 20; ++i)
    for (int d = 0; d < 3; ++d) cur[3 * i + d] = tris[i][d];
  for (int round = 0; round < level; ++round) {
    // edge -> midpoint vertex; creation order = first visit order
    std::unordered_map<uint64_t, int64_t> cache;
    cache.reserve(cur.size());
    auto mid = [&](int64_t a, int64_t b) -> int64_t {
      const uint64_t key = a < b ? (uint64_t(a) << 32) | uint64_t(b) : (uint64_t(b) << 32) | uint64_t(a);
      auto it = cache.find(key);
      if (it != cache.end()) return it->second;
      double m[3];
      for (int d = 0; d < 3; ++d) m[d] = verts[3 * a + d] + verts[3 * b + d];
      const double nrm = norm_fma(m, 3);
      for (int d = 0; d < 3; ++d) verts[3 * nv + d] = m[d] / nrm;
      cache.emplace(key, nv);
      return nv++;
    };
    const size_t nf = cur.size() / 3;
    nxt.assign(nf * 12, 0);
    for (size_t f = 0; f < nf; ++f) {
      const int64_t a = cur[3 * f], b = cur[3 * f + 1], c = cur[3 * f + 2];
      const int64_t ab = mid(a, b), bc = mid(b, c), ca = mid(c, a);
      const int64_t quad[4][3] = {{a, ab, ca}, {b, bc, ab}, {c, ca, bc}, {ab, bc, ca}};
      for (int q = 0; q < 4; ++q)
        for (int d = 0; d < 3; ++d) nxt[12 * f + 3 * q + d] = quad[q][d];
    }
    cur.swap(nxt);
  }
  std::memcpy(faces, cur.data(), cur.size() * sizeof(int64_t));
  return 0;
}

// Row-wise v /= |v| (left-to-right sum of squares, no FMA).  Used by the
// BASELINE jittered-sphere recipe.
void hb_normalize_rows3(double* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    double* p = v + 3 * i;
    const double nrm = std::sqrt((p[0] * p[0] + p[1] * p[1]) + p[2] * p[2]);
    p[0] /= nrm;
    p[1] /= nrm;
    p[2] /= nrm;
  }
}

// ---------------------------------------------------------------------------
// Cluster tree (restates reference partition.py:74-105): median bisection
// along the longest bbox axis; ties broken by original index.

typedef struct {
  int64_t start, end;
  double bmin[3], bmax[3];
  int64_t left, right;  // node indices, -1 for leaves
} hb_node;

int hb_cluster_tree(const double* pts, int64_t n, int64_t leaf_size, int64_t* perm,
                    hb_node* nodes, int64_t node_cap, int64_t* n_nodes) {
  if (n < 1 || leaf_size < 1) return -1;
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  int64_t count = 0;
  std::vector<std::pair<double, int64_t>> keys;
  std::function<int64_t(int64_t, int64_t)> build = [&](int64_t s, int64_t e) -> int64_t {
    if (count >= node_cap) return -2;
    const int64_t id = count++;
    hb_node& nd = nodes[id];
    nd.start = s;
    nd.end = e;
    nd.left = nd.right = -1;
    for (int d = 0; d < 3; ++d) {
      double lo = pts[3 * perm[s] + d], hi = lo;
      for (int64_t i = s + 1; i < e; ++i) {
        const double v = pts[3 * perm[i] + d];
        lo = v < lo ? v : lo;
        hi = v > hi ? v : hi;
      }
      nd.bmin[d] = lo;
      nd.bmax[d] = hi;
    }
    if (e - s > leaf_size) {
      int axis = 0;
      double best = nd.bmax[0] - nd.bmin[0];
      for (int d = 1; d < 3; ++d) {
        const double ext = nd.bmax[d] - nd.bmin[d];
        if (ext > best) {  // np.argmax: first maximum wins
          best = ext;
          axis = d;
        }
      }
      keys.resize((size_t)(e - s));
      for (int64_t i = s; i < e; ++i) keys[(size_t)(i - s)] = {pts[3 * perm[i] + axis], perm[i]};
      std::sort(keys.begin(), keys.end());  // (coordinate, original index)
      for (int64_t i = s; i < e; ++i) perm[i] = keys[(size_t)(i - s)].second;
      const int64_t mid = s + (e - s) / 2;
      const int64_t l = build(s, mid);
      if (l < 0) return l;
      const int64_t r = build(mid, e);
      if (r < 0) return r;
      nodes[id].left = l;
      nodes[id].right = r;
    }
    return id;
  };
  const int64_t root = build(0, n);
  if (root < 0) return (int)root;
  *n_nodes = count;
  return 0;
}

// ---------------------------------------------------------------------------
// Block partition (restates reference partition.py:142-169): dual traversal
// from (root, root); emission order is the reference's recursion order.

static inline double node_diam(const hb_node& a) {
  double d[3];
  for (int k = 0; k < 3; ++k) d[k] = a.bmax[k] - a.bmin[k];
  return norm_fma(d, 3);
}

static inline double node_dist(const hb_node& a, const hb_node& b) {
  double g[3];
  for (int k = 0; k < 3; ++k) {
    const double x = a.bmin[k] - b.bmax[k], y = b.bmin[k] - a.bmax[k];
    const double m = x > y ? x : y;  // np.maximum (no NaNs here)
    g[k] = m > 0.0 ? m : 0.0;
  }
  return norm_fma(g, 3);
}

int hb_is_admissible(const hb_node* s, const hb_node* t, double eta) {
  const double dist = node_dist(*s, *t);
  const double ds = node_diam(*s), dt = node_diam(*t);
  return dist > 0.0 && (ds < dt ? ds : dt) <= eta * dist;
}

// blocks_out: rows of (row_start, row_end, col_start, col_end, admissible).
// Returns the number of blocks; writes at most `cap` rows (call with cap=0
// to size the output).
int64_t hb_partition(const hb_node* nodes, int64_t n_nodes, double eta, int64_t* blocks_out,
                     int64_t cap) {
  if (n_nodes < 1) return -1;
  std::vector<double> diam((size_t)n_nodes);
  for (int64_t i = 0; i < n_nodes; ++i) diam[(size_t)i] = node_diam(nodes[i]);
  int64_t count = 0;
  auto emit = [&](const hb_node& s, const hb_node& t, int adm) {
    if (count < cap) {
      int64_t* o = blocks_out + 5 * count;
      o[0] = s.start;
      o[1] = s.end;
      o[2] = t.start;
      o[3] = t.end;
      o[4] = adm;
    }
    ++count;
  };
  std::function<void(int64_t, int64_t)> visit = [&](int64_t si, int64_t ti) {
    const hb_node& s = nodes[si];
    const hb_node& t = nodes[ti];
    const double dist = node_dist(s, t);
    const double dm = diam[(size_t)si] < diam[(size_t)ti] ? diam[(size_t)si] : diam[(size_t)ti];
    if (dist > 0.0 && dm <= eta * dist) {
      emit(s, t, 1);
      return;
    }
    const bool sl = s.left < 0, tl = t.left < 0;
    if (sl && tl) {
      emit(s, t, 0);
      return;
    }
    const int64_t sc[2] = {sl ? si : s.left, s.right};
    const int64_t tc[2] = {tl ? ti : t.left, t.right};
    const int ns = sl ? 1 : 2, nt = tl ? 1 : 2;
    for (int a = 0; a < ns; ++a)
      for (int b = 0; b < nt; ++b) visit(sc[a], tc[b]);
  };
  visit(0, 0);
  return count;
}

// ---------------------------------------------------------------------------
// H-matrix compression (restates reference compress.py:79-342).

struct Builder : Geom {
  int64_t n = 0;
  std::vector<int64_t> blocks;  // nb x 5
  std::vector<BlockResult> res;
  int64_t fallbacks = 0;
};

// Builds every block.  pcent/parea must stay alive until hb_build_export.
// Blocks whose rows miss [row_lo, row_hi) are skipped (kind 2, no storage):
// a multi-GPU rank builds only the blocks its row slice needs.
void* hb_build(const double* pcent, const double* parea, int64_t n, const int64_t* blocks,
               int64_t nb, double tol, int64_t max_rank, int nthreads, int64_t row_lo,
               int64_t row_hi, char* err, int errlen) {
  if (tol <= 0.0) {
    set_err(err, errlen, "tol must be positive");
    return nullptr;
  }
  auto* B = new Builder();
  B->pc = pcent;
  B->pa = parea;
  B->n = n;
  B->blocks.assign(blocks, blocks + 5 * nb);
  B->res.resize((size_t)nb);
  std::atomic<int64_t> fb{0};
  run_parallel(nb, nthreads, [&](int64_t k) {
    const int64_t* b = B->blocks.data() + 5 * k;
    BlockResult& r = B->res[(size_t)k];
    if (b[1] <= row_lo || b[0] >= row_hi) {
      r.kind = 2;
    } else if (b[4]) {
      bool fallback = false;
      aca_block(*B, b[0], b[1] - b[0], b[2], b[3] - b[2], tol, max_rank, r, fallback);
      if (fallback) fb.fetch_add(1);
    } else {
      r.kind = 0;
    }
  });
  B->fallbacks = fb.load();
  return B;
}

int64_t hb_build_fallbacks(void* h) { return static_cast<Builder*>(h)->fallbacks; }

// kinds[nb] (0 dense / 1 low rank), ranks[nb] (0 for dense), offsets[nb]
// (float64 element offset of the block's storage: dense m*n values, or U
// m*r followed by Vt r*n).  Returns the total element count.
int64_t hb_build_layout(void* h, int32_t* kinds, int64_t* ranks, int64_t* offsets) {
  auto* B = static_cast<Builder*>(h);
  int64_t off = 0;
  const int64_t nb = (int64_t)B->res.size();
  for (int64_t k = 0; k < nb; ++k) {
    const int64_t* b = B->blocks.data() + 5 * k;
    const int64_t m = b[1] - b[0], n = b[3] - b[2];
    const BlockResult& r = B->res[(size_t)k];
    kinds[k] = r.kind;
    ranks[k] = r.rank;
    offsets[k] = off;
    off += r.kind == 0 ? m * n : r.kind == 1 ? r.rank * (m + n) : 0;
  }
  return off;
}

// Fills `data` (sized by hb_build_layout) and releases per-block scratch.
int hb_build_export(void* h, double* data, const int64_t* offsets, int nthreads) {
  auto* B = static_cast<Builder*>(h);
  const int64_t nb = (int64_t)B->res.size();
  run_parallel(nb, nthreads, [&](int64_t k) {
    const int64_t* b = B->blocks.data() + 5 * k;
    const int64_t r0 = b[0], m = b[1] - b[0], c0 = b[2], n = b[3] - b[2];
    BlockResult& r = B->res[(size_t)k];
    double* dst = data + offsets[k];
    if (r.kind == 2) return;
    if (r.kind == 0) {
      // _fill_dense_block (compress.py:272-282); ACA fallbacks evaluate the
      // same entries (u@vt with an identity factor is exact)
      for (int64_t i = 0; i < m; ++i)
        for (int64_t j = 0; j < n; ++j) dst[i * n + j] = kentry(*B, r0 + i, c0 + j);
    } else {
      std::memcpy(dst, r.u.data(), r.u.size() * sizeof(double));
      std::memcpy(dst + m * r.rank, r.vt.data(), r.vt.size() * sizeof(double));
    }
    std::vector<double>().swap(r.u);
    std::vector<double>().swap(r.vt);
  });
  return 0;
}

void hb_build_free(void* h) { delete static_cast<Builder*>(h); }

// ---------------------------------------------------------------------------
// Scheme preparation on the packed master (restates precision.py:121-162,
// :256-329).  Low-rank block k has U at master[off[k]] (m x r) and Vt right
// after it (r x n).

// Per-rank diagonal d = colmag(U) * rowmag(Vt) and, when split_scale > 0,
// the Method-3 class of each rank (1 = FP32 class): d_i < max(d) * split_scale.
// diag_out / lo_out are indexed by the packed rank offset roff[k].
int hb_scale_diag(const double* master, int64_t nb, const int32_t* kinds, const int64_t* ranks,
                  const int64_t* ms, const int64_t* ns, const int64_t* offs, const int64_t* roffs,
                  double split_scale, int do_split, double* diag_out, int8_t* lo_out,
                  int64_t* nlo_out, int nthreads) {
  run_parallel(nb, nthreads, [&](int64_t k) {
    nlo_out[k] = 0;
    if (kinds[k] != 1) return;
    const int64_t m = ms[k], n = ns[k], r = ranks[k];
    const double* u = master + offs[k];
    const double* vt = u + m * r;
    double* d = diag_out + roffs[k];
    for (int64_t q = 0; q < r; ++q) {
      double cm = 0.0, rm = 0.0;
      for (int64_t i = 0; i < m; ++i) cm = std::max(cm, std::fabs(u[i * r + q]));
      for (int64_t j = 0; j < n; ++j) rm = std::max(rm, std::fabs(vt[q * n + j]));
      d[q] = cm * rm;
    }
    if (do_split && r > 0) {
      double dmax = d[0];
      for (int64_t q = 1; q < r; ++q) dmax = std::max(dmax, d[q]);
      const double thr = dmax * split_scale;
      int64_t nlo = 0;
      for (int64_t q = 0; q < r; ++q) {
        const int8_t lo = d[q] < thr ? 1 : 0;
        lo_out[roffs[k] + q] = lo;
        nlo += lo;
      }
      nlo_out[k] = nlo;
    } else if (r > 0) {
      for (int64_t q = 0; q < r; ++q) lo_out[roffs[k] + q] = 0;
    }
  });
  return 0;
}

// Writes unit-scaled factors.  For every low-rank block, the FP64-class
// columns go to out64 (U_hi at hi_off[k], Vt_hi right after) and the
// FP32-class columns to out32 (U_lo at lo_off[k], Vt_lo right after), both
// stable in the original column order.  Division by the magnitude uses 1 for
// zero columns/rows (precision.py:135-137).  Method 2 passes an all-zero
// class array and out64 only (then cast by the caller for FP32 variants).
// diag_in (original rank order, from hb_scale_diag) is rewritten into
// diag_out at roffs[k] as [d_hi..., d_lo...].  lost_out[k] counts FP32-class
// values that lost all magnitude in the cast (precision.py:241-253).
int hb_scale_fill(const double* master, int64_t nb, const int32_t* kinds, const int64_t* ranks,
                  const int64_t* ms, const int64_t* ns, const int64_t* offs, const int64_t* roffs,
                  const int8_t* lo_cls, const int64_t* hi_off, const int64_t* lo_off,
                  double* out64, float* out32, const double* diag_in, double* diag_out,
                  int64_t* lost_out, int nthreads) {
  const float f32_tiny = 1.17549435e-38f;
  run_parallel(nb, nthreads, [&](int64_t k) {
    lost_out[k] = 0;
    if (kinds[k] != 1) return;
    const int64_t m = ms[k], n = ns[k], r = ranks[k];
    const double* u = master + offs[k];
    const double* vt = u + m * r;
    const int8_t* cls = lo_cls + roffs[k];
    int64_t khi = 0, klo = 0;
    for (int64_t q = 0; q < r; ++q) (cls[q] ? klo : khi)++;
    std::vector<double> cm((size_t)r), rm((size_t)r);
    for (int64_t q = 0; q < r; ++q) {
      double a = 0.0, b = 0.0;
      for (int64_t i = 0; i < m; ++i) a = std::max(a, std::fabs(u[i * r + q]));
      for (int64_t j = 0; j < n; ++j) b = std::max(b, std::fabs(vt[q * n + j]));
      cm[(size_t)q] = a == 0.0 ? 1.0 : a;
      rm[(size_t)q] = b == 0.0 ? 1.0 : b;
    }
    double* uh = out64 ? out64 + hi_off[k] : nullptr;
    double* vh = uh ? uh + m * khi : nullptr;
    float* ul = (out32 && klo) ? out32 + lo_off[k] : nullptr;
    float* vl = ul ? ul + m * klo : nullptr;
    int64_t ih = 0, il = 0, lost = 0;
    auto cast = [&](double v) -> float {
      const float f = (float)v;
      if (v != 0.0 && std::fabs(f) < f32_tiny) ++lost;
      return f;
    };
    std::vector<double> dlo;
    for (int64_t q = 0; q < r; ++q) {
      if (!cls[q]) {
        for (int64_t i = 0; i < m; ++i) uh[i * khi + ih] = u[i * r + q] / cm[(size_t)q];
        for (int64_t j = 0; j < n; ++j) vh[ih * n + j] = vt[q * n + j] / rm[(size_t)q];
        if (diag_out) diag_out[roffs[k] + ih] = diag_in[roffs[k] + q];
        ++ih;
      } else {
        for (int64_t i = 0; i < m; ++i) ul[i * klo + il] = cast(u[i * r + q] / cm[(size_t)q]);
        for (int64_t j = 0; j < n; ++j) vl[il * n + j] = cast(vt[q * n + j] / rm[(size_t)q]);
        dlo.push_back(diag_in[roffs[k] + q]);
        ++il;
      }
    }
    if (diag_out)
      for (int64_t q = 0; q < klo; ++q) diag_out[roffs[k] + khi + q] = dlo[(size_t)q];
    lost_out[k] = lost;
  });
  return 0;
}

}  // extern "C"

extern "C" {

// Round-to-nearest FP32 copy of `src` (precision.py:241-253): returns the
// index of the first element that overflows (finite -> inf), or -1, and the
// number of nonzero values that lost all magnitude (|f32| < FLT_MIN).
int64_t hb_cast_f32(const double* src, int64_t n, float* dst, int64_t* lost_out, int nthreads) {
  const float f32_tiny = 1.17549435e-38f;
  const int64_t chunk = 1 << 20;
  const int64_t nchunks = (n + chunk - 1) / chunk;
  std::vector<int64_t> first((size_t)std::max<int64_t>(nchunks, 1), -1), lost((size_t)std::max<int64_t>(nchunks, 1), 0);
  run_parallel(nchunks, nthreads, [&](int64_t c) {
    const int64_t a = c * chunk, b = std::min(n, a + chunk);
    int64_t f = -1, l = 0;
    for (int64_t i = a; i < b; ++i) {
      const double v = src[i];
      const float o = (float)v;
      dst[i] = o;
      if (f < 0 && std::isinf(o) && std::isfinite(v)) f = i;
      if (v != 0.0 && std::fabs(o) < f32_tiny) ++l;
    }
    first[(size_t)c] = f;
    lost[(size_t)c] = l;
  });
  int64_t f = -1, l = 0;
  for (int64_t c = 0; c < nchunks; ++c) {
    if (f < 0 && first[(size_t)c] >= 0) f = first[(size_t)c];
    l += lost[(size_t)c];
  }
  *lost_out = l;
  return f;
}

}  // extern "C"

extern "C" {

// dst[0:n] = src[0:n], in parallel chunks (host staging of large payloads).
void hb_copy_f64(const double* src, double* dst, int64_t n, int nthreads) {
  const int64_t chunk = 1 << 22;
  run_parallel((n + chunk - 1) / chunk, nthreads, [&](int64_t c) {
    const int64_t a = c * chunk, b = std::min(n, a + chunk);
    std::memcpy(dst + a, src + a, (size_t)(b - a) * sizeof(double));
  });
}

}  // extern "C"
