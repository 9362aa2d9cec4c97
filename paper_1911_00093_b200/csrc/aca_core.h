// ACA compression core shared by the host builder (hbuild.cpp) and the GPU
// builder's host-side completion of rare blocks (hmx_build.cu): kernel
// entries and adaptive cross approximation with partial pivoting, restating
// reference pkg/src/hmx/compress.py:79-207 and :256-282 with numpy's
// operation order where it is known (see hbuild.cpp).  Compile with
// -ffp-contract=off.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

namespace hmx_aca {

constexpr double kPi = 3.141592653589793;
constexpr double kFourPi = 4.0 * kPi;          // compress.py:38 (exact power-of-two product)
constexpr double kEps64 = 2.220446049250313e-16;  // compress.py:39

// np.linalg.norm(v) for a 1-D float64 vector == sqrt(ddot(v, v)); OpenBLAS'
// short ddot is a sequential FMA chain.
inline double norm_fma(const double* v, int64_t n, int64_t stride = 1) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s = std::fma(v[i * stride], v[i * stride], s);
  return std::sqrt(s);
}

// np.sqrt(np.sum(d*d, axis=-1)) with a length-3 last axis: left to right.
inline double dist3(const double* a, const double* b) {
  const double dx = a[0] - b[0], dy = a[1] - b[1], dz = a[2] - b[2];
  return std::sqrt((dx * dx + dy * dy) + dz * dz);
}

// Kernel geometry: permuted centroids (n x 3) and areas.
struct Geom {
  const double* pc = nullptr;
  const double* pa = nullptr;
};

struct BlockResult {
  int kind = 0;  // 0 dense (incl. ACA fallback), 1 low rank
  int64_t rank = 0;
  std::vector<double> u;   // m x rank row-major
  std::vector<double> vt;  // rank x n row-major
};

// compress.py:256-282 / problem.py:220-238: entry (gi, gj) in permuted indices.
inline double kentry(const Geom& B, int64_t gi, int64_t gj) {
  if (gi == gj) return 0.5 * std::sqrt(B.pa[gi] / kPi);
  const double d = dist3(B.pc + 3 * gi, B.pc + 3 * gj);
  return B.pa[gj] / (kFourPi * d);
}

// Adaptive cross approximation with partial pivoting (compress.py:79-207).
// Returns kind 1 with factors, or kind 0 when the reference would take the
// dense fallback (fallback counted by the caller).
inline void aca_block(const Geom& B, int64_t r0, int64_t m, int64_t c0, int64_t n, double tol,
                      int64_t max_rank, BlockResult& out, bool& fallback) {
  int64_t budget = std::min(m, n);
  if (max_rank > 0) budget = std::min(budget, max_rank);
  std::vector<double> U;   // column-major m x rank (column k at k*m)
  std::vector<double> Vt;  // row-major rank x n
  std::vector<char> row_used((size_t)m, 0), col_used((size_t)n, 0);
  std::vector<double> row((size_t)n), col((size_t)m), a, b;
  double frob_sq = 0.0, max_seen = 0.0;
  bool converged = false;
  int64_t rank = 0;
  int64_t i_star = 0;
  fallback = false;
  while (rank < budget && i_star >= 0) {
    // residual row i_star
    for (int64_t j = 0; j < n; ++j) {
      double v = kentry(B, r0 + i_star, c0 + j);
      if (rank) {
        double s = 0.0;
        for (int64_t k = 0; k < rank; ++k) s += U[(size_t)(k * m + i_star)] * Vt[(size_t)(k * n + j)];
        v = v - s;
      }
      row[(size_t)j] = v;
    }
    row_used[(size_t)i_star] = 1;
    double rmax = 0.0;
    for (int64_t j = 0; j < n; ++j) rmax = std::max(rmax, std::fabs(row[(size_t)j]));
    max_seen = std::max(max_seen, rmax);
    int64_t j_star = 0;
    double best = -1.0;
    for (int64_t j = 0; j < n; ++j) {
      const double mv = col_used[(size_t)j] ? 0.0 : std::fabs(row[(size_t)j]);
      if (mv > best) {
        best = mv;
        j_star = j;
      }
    }
    const double pivot = col_used[(size_t)j_star] ? 0.0 : row[(size_t)j_star];
    if (std::fabs(pivot) <= kEps64 * max_seen) {
      i_star = -1;
      for (int64_t i = 0; i < m; ++i)
        if (!row_used[(size_t)i]) {
          i_star = i;
          break;
        }
      continue;
    }
    // v_new = row / pivot ; u_new = residual column j_star
    const size_t vbase = Vt.size();
    Vt.resize(vbase + (size_t)n);
    for (int64_t j = 0; j < n; ++j) Vt[vbase + (size_t)j] = row[(size_t)j] / pivot;
    for (int64_t i = 0; i < m; ++i) {
      double v = kentry(B, r0 + i, c0 + j_star);
      if (rank) {
        double s = 0.0;
        for (int64_t k = 0; k < rank; ++k) s += U[(size_t)(k * m + i)] * Vt[(size_t)(k * n + j_star)];
        v = v - s;
      }
      col[(size_t)i] = v;
    }
    col_used[(size_t)j_star] = 1;
    const size_t ubase = U.size();
    U.insert(U.end(), col.begin(), col.end());
    const double* u_new = U.data() + ubase;
    const double* v_new = Vt.data() + vbase;
    const double u_norm = norm_fma(u_new, m);
    const double v_norm = norm_fma(v_new, n);
    double cross = 0.0;
    if (rank) {
      a.assign((size_t)rank, 0.0);
      b.assign((size_t)rank, 0.0);
      for (int64_t k = 0; k < rank; ++k) {
        double sa = 0.0, sb = 0.0;
        const double* uk = U.data() + (size_t)(k * m);
        const double* vk = Vt.data() + (size_t)(k * n);
        for (int64_t i = 0; i < m; ++i) sa = std::fma(uk[i], u_new[i], sa);
        for (int64_t j = 0; j < n; ++j) sb = std::fma(vk[j], v_new[j], sb);
        a[(size_t)k] = sa;
        b[(size_t)k] = sb;
      }
      double s = 0.0;
      for (int64_t k = 0; k < rank; ++k) s = std::fma(a[(size_t)k], b[(size_t)k], s);
      cross = 2.0 * s;
    }
    const double uv = u_norm * v_norm;
    frob_sq = std::max(frob_sq + uv * uv + cross, 0.0);
    ++rank;
    if (uv <= tol * std::sqrt(frob_sq)) {
      converged = true;
      break;
    }
    i_star = -1;
    double cbest = -1.0;
    for (int64_t i = 0; i < m; ++i) {
      const double cv = row_used[(size_t)i] ? -1.0 : std::fabs(u_new[i]);
      if (cv > cbest) {
        cbest = cv;
        i_star = i;
      }
    }
    if (cbest < 0.0) i_star = -1;
  }
  if (!converged && rank < budget) {
    // ran out of pivot rows: measure the exact remainder (compress.py:191-205)
    double rem_sq = 0.0;
    for (int64_t i = 0; i < m; ++i) {
      double rr = 0.0;
      for (int64_t j = 0; j < n; ++j) {
        double v = kentry(B, r0 + i, c0 + j);
        if (rank) {
          double s = 0.0;
          for (int64_t k = 0; k < rank; ++k) s += U[(size_t)(k * m + i)] * Vt[(size_t)(k * n + j)];
          v = v - s;
        }
        rr = std::fma(v, v, rr);
      }
      rem_sq += rr;
    }
    if (std::sqrt(rem_sq) > tol * std::sqrt(frob_sq)) {
      fallback = true;
      out.kind = 0;
      out.rank = 0;
      return;
    }
  }
  out.kind = 1;
  out.rank = rank;
  out.u.resize((size_t)(m * rank));
  for (int64_t i = 0; i < m; ++i)
    for (int64_t k = 0; k < rank; ++k) out.u[(size_t)(i * rank + k)] = U[(size_t)(k * m + i)];
  out.vt.assign(Vt.begin(), Vt.begin() + (size_t)(rank * n));
}


}  // namespace hmx_aca
