// BiCG-STAB on the device (reference pkg/src/hmx/solver.py:68-168).
//
// Control flow and scalar arithmetic are the reference's: alpha, omega and
// beta are formed on the device with the same IEEE operations, vector
// updates keep the reference's operation order (no FMA contraction in the
// axpy's: x = (x + alpha p) + omega s etc.), dots and norms are deterministic
// two-level reductions (fixed grid, fixed order).
//
// Speculative batched launch: every kernel of an iteration first reads a
// device `stop` word and becomes a no-op once it is set.  The device itself
// records each decision the reference takes, at the same point and with the
// same values (rho breakdown, shadow-projection breakdown, early exit on |s|,
// stabilisation breakdown, convergence of |r|, omega breakdown, non-finite
// matvec), so the host can enqueue several iterations per synchronisation and
// act on the recorded outcome afterwards (FP64 true-residual confirmation,
// breakdown report).  Per iteration: p-update, v = A p (fused r^.v),
// s-update (fused |s|^2), t = A s (fused t.s, t.t), x/r-update (fused |r|^2,
// r^.r).
#include <dlfcn.h>
#include <nccl.h>

#include <type_traits>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "hmx_plan_impl.cuh"

namespace hmx {

constexpr int kVecThreads = 512;
constexpr double kBreakdownEps = 1e-300;  // solver.py:27

// scalar slots
enum : int {
  SC_BB = 0,      // |b|^2
  SC_RHO0 = 1,    // rho ring buffer slot 0
  SC_RHO1 = 2,    // rho ring buffer slot 1
  SC_ALPHA = 3,
  SC_OMEGA = 4,
  SC_SS = 5,      // |s|^2
  SC_RR = 6,      // |r|^2
  SC_RES = 7,     // |b - A x|^2
  SC_DV = 8,      // [r^.v, unused]
  SC_DT = 10,     // [t.s, t.t]
  SC_TMP = 12,    // [2 scratch]
  SC_NB = 14,     // |b|
  SC_BVAL = 15,   // value reported with a breakdown
  SC_TOL = 16,    // tol of the running solve
  SC_N = 18
};

// iteration control (int[4]): [current iteration i, max_iter, spare, spare]
__device__ __forceinline__ int rho_slot_of(int it) { return (it & 1) ? SC_RHO1 : SC_RHO0; }

// stop word layout (int[4]): [stop, reason, iteration, spare]
enum : int {
  R_NONE = 0, R_RHO = 1, R_DENOM = 2, R_TT = 3, R_OMEGA = 4, R_SEXIT = 5, R_CONV = 6,
  R_NONFINITE = 7
};

__device__ __forceinline__ void set_stop(int* stop, int reason, int it, double* sc, double val) {
  stop[1] = reason;
  stop[2] = it;
  sc[SC_BVAL] = val;
  __threadfence();
  stop[0] = 1;
}

struct VecRed {
  double* partials;  // 2 per CTA
  uint32_t* done;
  double* out;       // 2 results
};

// Deterministic two-level sum of (u, w) over the grid: per-CTA fixed-order
// block reduction, then the last CTA to finish sums the CTA partials in order.
__device__ __forceinline__ bool grid_reduce2(double u, double w, const VecRed& R) {
  __shared__ double su[kVecThreads / 32], sw[kVecThreads / 32];
  __shared__ unsigned ticket;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    u += __shfl_xor_sync(0xffffffffu, u, s);
    w += __shfl_xor_sync(0xffffffffu, w, s);
  }
  if (lane == 0) {
    su[wid] = u;
    sw[wid] = w;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < kVecThreads / 32; ++i) {
      a += su[i];
      b += sw[i];
    }
    R.partials[2 * blockIdx.x] = a;
    R.partials[2 * blockIdx.x + 1] = b;
    __threadfence();
    ticket = atomicAdd(R.done, 1u);
  }
  __syncthreads();
  if (ticket != gridDim.x - 1) return false;
  __threadfence();
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += kVecThreads) {
    a += __ldcg(R.partials + 2 * i);
    b += __ldcg(R.partials + 2 * i + 1);
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, s);
    b += __shfl_xor_sync(0xffffffffu, b, s);
  }
  __syncthreads();
  if (lane == 0) {
    su[wid] = a;
    sw[wid] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double fa = 0.0, fb = 0.0;
    for (int i = 0; i < kVecThreads / 32; ++i) {
      fa += su[i];
      fb += sw[i];
    }
    R.out[0] = fa;
    R.out[1] = fb;
    *R.done = 0u;
    return true;
  }
  return false;
}

// (|u|^2, u.w) style reductions: out = [sum a*b, sum c*d]
__global__ void __launch_bounds__(kVecThreads) dot2_kernel(const double* a, const double* b,
                                                            const double* c, const double* dd,
                                                            int n, VecRed R) {
  double u = 0.0, w = 0.0;
  for (int i = blockIdx.x * kVecThreads + threadIdx.x; i < n; i += gridDim.x * kVecThreads) {
    u += a[i] * b[i];
    if (c) w += c[i] * dd[i];
  }
  grid_reduce2(u, w, R);
}

// r = b - t ; r_hat = r ; x = 0 ; out = [|r|^2, unused]   (solver.py:99-102)
__global__ void __launch_bounds__(kVecThreads) init_kernel(const double* b, const double* t,
                                                            double* r, double* rhat, double* x,
                                                            int n, VecRed R) {
  double u = 0.0;
  for (int i = blockIdx.x * kVecThreads + threadIdx.x; i < n; i += gridDim.x * kVecThreads) {
    const double ri = __dsub_rn(b[i], t[i]);
    r[i] = ri;
    rhat[i] = ri;
    x[i] = 0.0;
    u += ri * ri;
  }
  grid_reduce2(u, 0.0, R);
}

// p = r (first iteration) or p = r + beta (p - omega v),
// beta = (rho / rho_prev) (alpha / omega)   (solver.py:112-120); first checks
// the rho breakdown of iteration `it` (solver.py:113-115)
__global__ void __launch_bounds__(kVecThreads) p_update_kernel(const double* r, const double* v,
                                                                double* p, int n, const int* ictl,
                                                                double* sc, int* stop) {
  if (*(volatile int*)stop) return;
  const int it = ictl[0];
  const int rho_slot = rho_slot_of(it), prev_slot = rho_slot_of(it - 1);
  const double rho = sc[rho_slot];
  if (fabs(rho) < kBreakdownEps) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_stop(stop, R_RHO, it, sc, rho);
    return;
  }
  double beta = 0.0, omega = 0.0;
  if (it > 1) {
    const double rho_prev = sc[prev_slot];
    const double alpha = sc[SC_ALPHA];
    omega = sc[SC_OMEGA];
    beta = __dmul_rn(__ddiv_rn(rho, rho_prev), __ddiv_rn(alpha, omega));
  }
  for (int i = blockIdx.x * kVecThreads + threadIdx.x; i < n; i += gridDim.x * kVecThreads) {
    if (it == 1) p[i] = r[i];
    else p[i] = __dadd_rn(r[i], __dmul_rn(beta, __dsub_rn(p[i], __dmul_rn(omega, v[i]))));
  }
}

// alpha = rho / (r^.v) ; s = r - alpha v ; |s|^2 ; early exit on |s|/|b| < tol
// (solver.py:122-136)
__global__ void __launch_bounds__(kVecThreads) s_update_kernel(const double* r, const double* v,
                                                                double* s, int n, double* sc,
                                                                VecRed R, const int* ictl,
                                                                double* hist, int* stop,
                                                                const int* nonfin, int dist = 0) {
  if (*(volatile int*)stop) return;
  const int it = ictl[0];
  const int rho_slot = rho_slot_of(it);
  const double tol = sc[SC_TOL];
  if (*nonfin) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_stop(stop, R_NONFINITE, it, sc, 0.0);
    return;
  }
  const double denom = sc[SC_DV];
  if (fabs(denom) < kBreakdownEps) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_stop(stop, R_DENOM, it, sc, denom);
    return;
  }
  const double alpha = __ddiv_rn(sc[rho_slot], denom);
  if (blockIdx.x == 0 && threadIdx.x == 0) sc[SC_ALPHA] = alpha;
  double u = 0.0;
  for (int i = blockIdx.x * kVecThreads + threadIdx.x; i < n; i += gridDim.x * kVecThreads) {
    const double si = __dsub_rn(r[i], __dmul_rn(alpha, v[i]));
    s[i] = si;
    u += si * si;
  }
  // last CTA, thread 0: the reduced |s|^2 (multi-GPU: a local partial,
  // decided on by decide_s_kernel after the allreduce)
  if (grid_reduce2(u, 0.0, R) && !dist) {
    const double s_rel = __ddiv_rn(sqrt(R.out[0]), sc[SC_NB]);
    if (s_rel < tol) {
      hist[it] = s_rel;
      set_stop(stop, R_SEXIT, it, sc, s_rel);
    }
  }
}

// x = x + alpha p (early exit on |s|, solver.py:131)
__global__ void __launch_bounds__(kVecThreads) x_alpha_p_kernel(double* x, const double* p, int n,
                                                                 const double* sc) {
  const double alpha = sc[SC_ALPHA];
  for (int i = blockIdx.x * kVecThreads + threadIdx.x; i < n; i += gridDim.x * kVecThreads)
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
}

// omega = (t.s)/(t.t); x = x + alpha p + omega s; r = s - omega t;
// |r|^2, r^.r (solver.py:139-158): records the history entry, the next rho,
// convergence of |r| and the omega breakdown.
__global__ void __launch_bounds__(kVecThreads) xr_update_kernel(double* x, double* r,
                                                                 const double* p, const double* s,
                                                                 const double* t,
                                                                 const double* rhat, int n,
                                                                 double* sc, VecRed R,
                                                                 const int* ictl, double* hist,
                                                                 int* stop, const int* nonfin,
                                                                 int dist = 0) {
  if (*(volatile int*)stop) return;
  const int it = ictl[0];
  const int next_slot = rho_slot_of(it + 1);
  const double tol = sc[SC_TOL];
  if (*nonfin) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_stop(stop, R_NONFINITE, it, sc, 0.0);
    return;
  }
  const double tt = sc[SC_DT + 1];
  if (tt == 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) set_stop(stop, R_TT, it, sc, 0.0);
    return;
  }
  const double omega = __ddiv_rn(sc[SC_DT], tt);
  const double alpha = sc[SC_ALPHA];
  if (blockIdx.x == 0 && threadIdx.x == 0) sc[SC_OMEGA] = omega;
  double u = 0.0, w = 0.0;
  for (int i = blockIdx.x * kVecThreads + threadIdx.x; i < n; i += gridDim.x * kVecThreads) {
    const double xi = __dadd_rn(__dadd_rn(x[i], __dmul_rn(alpha, p[i])), __dmul_rn(omega, s[i]));
    const double ri = __dsub_rn(s[i], __dmul_rn(omega, t[i]));
    x[i] = xi;
    r[i] = ri;
    u += ri * ri;
    w += rhat[i] * ri;
  }
  if (grid_reduce2(u, w, R) && !dist) {
    const double rel = __ddiv_rn(sqrt(R.out[0]), sc[SC_NB]);
    hist[it] = rel;
    sc[next_slot] = R.out[1];  // rho of the next iteration
    if (rel < tol) set_stop(stop, R_CONV, it, sc, rel);
    else if (fabs(omega) < kBreakdownEps) set_stop(stop, R_OMEGA, it, sc, omega);
  }
}

// Multi-GPU: the decisions s_update / xr_update take in their last CTA,
// taken instead on the allreduced sums (identical on every rank, so every
// rank records the same decision at the same point).
__global__ void decide_s_kernel(double* sc, const int* ictl, double* hist, int* stop) {
  if (*(volatile int*)stop) return;
  const int it = ictl[0];
  const double s_rel = __ddiv_rn(sqrt(sc[SC_SS]), sc[SC_NB]);
  if (s_rel < sc[SC_TOL]) {
    hist[it] = s_rel;
    set_stop(stop, R_SEXIT, it, sc, s_rel);
  }
}

__global__ void decide_r_kernel(double* sc, const int* ictl, double* hist, int* stop) {
  if (*(volatile int*)stop) return;
  const int it = ictl[0];
  const double rel = __ddiv_rn(sqrt(sc[SC_TMP]), sc[SC_NB]);
  hist[it] = rel;
  sc[rho_slot_of(it + 1)] = sc[SC_TMP + 1];
  if (rel < sc[SC_TOL]) set_stop(stop, R_CONV, it, sc, rel);
  else if (fabs(sc[SC_OMEGA]) < kBreakdownEps) set_stop(stop, R_OMEGA, it, sc, sc[SC_OMEGA]);
}

// out = [|b - y|^2, |b|^2]   (solver.py:60-62)
__global__ void __launch_bounds__(kVecThreads) resid_kernel(const double* b, const double* y, int n,
                                                             VecRed R) {
  double u = 0.0, w = 0.0;
  for (int i = blockIdx.x * kVecThreads + threadIdx.x; i < n; i += gridDim.x * kVecThreads) {
    const double e = __dsub_rn(b[i], y[i]);
    u += e * e;
    w += b[i] * b[i];
  }
  grid_reduce2(u, w, R);
}

// end of an iteration: next i; in the graph-resident loop also the loop
// condition (continue while no decision is recorded and i <= max_iter)
__global__ void advance_kernel(int* ictl, const int* stop, cudaGraphConditionalHandle loop, int in_graph) {
  const bool go = !*(volatile const int*)stop;
  if (go) ictl[0] += 1;
  if (in_graph) cudaGraphSetConditional(loop, (go && ictl[0] <= ictl[1]) ? 1u : 0u);
}

__global__ void permute_kernel(const double* src, const int32_t* perm, double* dst, int n,
                               int inverse) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (inverse) dst[perm[i]] = src[i];  // permuted -> original
  else dst[i] = src[perm[i]];          // original -> permuted
}

}  // namespace hmx

using namespace hmx;

namespace {

struct SolveCtx {
  hmx_plan* A;
  hmx_plan* A64;
  Workspace w;
  cudaStream_t st;
  int grid;
  VecRed red(int slot) const { return VecRed{w.partials, w.done, w.sc + slot}; }
};

int alloc_ws(hmx_plan* p, Workspace& w, int64_t n, int grid) {
  w.n = n;
  w.grid = grid;
  double** vecs[] = {&w.b, &w.x, &w.r, &w.rhat, &w.p, &w.v, &w.s, &w.t, &w.y, &w.orig};
  for (double** v : vecs) {
    *v = p->alloc<double>((size_t)n);
    if (!*v) {
      set_error("cudaMalloc failed for the solver workspace");
      return HMX_ERR_CUDA;
    }
  }
  w.sc = p->alloc<double>(SC_N);
  w.flags = p->alloc<int>(4);
  w.stop = p->alloc<int>(4);
  w.ictl = p->alloc<int>(4);
  w.partials = p->alloc<double>((size_t)2 * grid);
  w.done = p->alloc<uint32_t>(1);
  if (!w.sc || !w.flags || !w.stop || !w.ictl || !w.partials || !w.done) {
    set_error("cudaMalloc failed for the solver workspace");
    return HMX_ERR_CUDA;
  }
  HMX_CUDA(cudaMemset(w.done, 0, sizeof(uint32_t)));
  HMX_CUDA(cudaMemset(w.sc, 0, SC_N * sizeof(double)));
  HMX_CUDA(cudaMallocHost(&w.h_sc, (SC_N + 8) * sizeof(double)));
  p->pinned.push_back(w.h_sc);
  return HMX_OK;
}

// Stage-2 epilogue options: y (the plan's rows), dots y.w1 / y.y fused into
// sc[slot..slot+1], the non-finite flag, the stop word as launch guard.
S2Out solver_out(hmx_plan* A, double* sc, double* y, const double* w1, int yy, int slot, int* flag,
                 const int* skip) {
  S2Out out{};
  out.skip = skip;
  out.y = y;
  out.permute_out = 0;
  out.w1 = w1;
  out.yy = yy;
  if (w1 || yy) {
    out.seg_dots = A->d_seg_dots;
    out.done = A->d_done;
    out.dots_out = sc + slot;
  }
  out.nonfinite = flag;
  return out;
}

// y = A xp on stream st, fused dots into sc[slot..slot+1]
int apply_sc(hmx_plan* A, double* sc, cudaStream_t st, const double* xp, double* y,
             const double* w1, int yy, int slot, int* flag, const int* skip = nullptr) {
  if ((w1 || yy) && A->dp.n_seg2 == 0)  // no local rows: the dots are zero
    HMX_CUDA(cudaMemsetAsync(sc + slot, 0, 2 * sizeof(double), st));
  HMX_CUDA(launch_stage1(A->dp, xp, st, skip));
  HMX_CUDA(launch_stage2(A->dp, xp, solver_out(A, sc, y, w1, yy, slot, flag, skip), st, /*pdl=*/true));
  A->last_xp = xp;
  return HMX_OK;
}

int apply(hmx_plan* A, const Workspace& w, cudaStream_t st, const double* xp, double* y,
          const double* w1, int yy, int slot, int* flag, const int* skip = nullptr) {
  return apply_sc(A, w.sc, st, xp, y, w1, yy, slot, flag, skip);
}

// scalars, non-finite flags and the stop word in one pinned mirror
int sync_scalars(const SolveCtx& c) {
  HMX_CUDA(cudaMemcpyAsync(c.w.h_sc, c.w.sc, SC_N * sizeof(double), cudaMemcpyDeviceToHost, c.st));
  HMX_CUDA(cudaMemcpyAsync(c.w.h_sc + SC_N, c.w.flags, 4 * sizeof(int), cudaMemcpyDeviceToHost, c.st));
  HMX_CUDA(cudaMemcpyAsync(c.w.h_sc + SC_N + 2, c.w.stop, 4 * sizeof(int), cudaMemcpyDeviceToHost, c.st));
  HMX_CUDA(cudaStreamSynchronize(c.st));
  return HMX_OK;
}

const int* host_stop(const SolveCtx& c) { return reinterpret_cast<const int*>(c.w.h_sc + SC_N + 2); }

int flags_nonfinite(const SolveCtx& c) {
  const int* f = reinterpret_cast<const int*>(c.w.h_sc + SC_N);
  return f[0] | f[1] | f[2];
}

// One BiCG-STAB iteration (solver.py:112-158), every kernel guarded by the
// stop word; the iteration number and tol live on the device (ictl, SC_TOL)
// so the same launches serve every iteration and can be captured once.
int enqueue_iteration(const SolveCtx& c, int n32, cudaGraphConditionalHandle loop, int in_graph) {
  const Workspace& w = c.w;
  cudaStream_t st = c.st;
  int rc;
  p_update_kernel<<<c.grid, kVecThreads, 0, st>>>(w.r, w.v, w.p, n32, w.ictl, w.sc, w.stop);
  if ((rc = apply(c.A, w, st, w.p, w.v, w.rhat, 0, SC_DV, w.flags, w.stop))) return rc;
  s_update_kernel<<<c.grid, kVecThreads, 0, st>>>(w.r, w.v, w.s, n32, w.sc, c.red(SC_SS), w.ictl, w.hist,
                                                    w.stop, w.flags);
  if ((rc = apply(c.A, w, st, w.s, w.t, w.s, 1, SC_DT, w.flags + 1, w.stop))) return rc;
  xr_update_kernel<<<c.grid, kVecThreads, 0, st>>>(w.x, w.r, w.p, w.s, w.t, w.rhat, n32, w.sc,
                                                     VecRed{w.partials, w.done, w.sc + SC_TMP}, w.ictl,
                                                     w.hist, w.stop, w.flags + 1);
  advance_kernel<<<1, 1, 0, st>>>(w.ictl, w.stop, loop, in_graph);
  HMX_CUDA(cudaGetLastError());
  return HMX_OK;
}

// The whole iteration loop as one CUDA graph: a WHILE conditional node whose
// body is one captured iteration; advance_kernel clears the condition when a
// decision is recorded or max_iter is reached.  One launch and one host
// synchronisation per solve, no speculative iterations.
int build_loop_graph(const SolveCtx& c, Workspace& ws, int n32) {
  if (ws.loop_exec) cudaGraphExecDestroy(ws.loop_exec);
  if (ws.loop_graph) cudaGraphDestroy(ws.loop_graph);
  ws.loop_exec = nullptr;
  ws.loop_graph = nullptr;
  cudaGraph_t g = nullptr;
  HMX_CUDA(cudaGraphCreate(&g, 0));
  ws.loop_graph = g;
  cudaGraphConditionalHandle h;
  HMX_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np{};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  HMX_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  HMX_CUDA(cudaStreamBeginCaptureToGraph(c.st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  const int rc = enqueue_iteration(c, n32, h, 1);
  cudaGraph_t captured = nullptr;
  const cudaError_t e = cudaStreamEndCapture(c.st, &captured);
  if (rc) return rc;
  HMX_CUDA(e);
  HMX_CUDA(cudaGraphInstantiate(&ws.loop_exec, g, 0));
  ws.loop_hist = c.w.hist;
  return HMX_OK;
}

// |b - A64 x| / |b| with x, b device, permuted; result on the host
int true_residual_dev(SolveCtx& c, double* out) {
  int rc = apply(c.A64, c.w, c.st, c.w.x, c.w.y, nullptr, 0, 0, c.w.flags + 2);
  if (rc) return rc;
  resid_kernel<<<c.grid, kVecThreads, 0, c.st>>>(c.w.b, c.w.y, (int)c.w.n, c.red(SC_RES));
  HMX_CUDA(cudaGetLastError());
  if ((rc = sync_scalars(c))) return rc;
  if (flags_nonfinite(c)) {
    set_error("non-finite matvec result");
    return HMX_ERR_NONFINITE;
  }
  const double nr = std::sqrt(c.w.h_sc[SC_RES]), nb = std::sqrt(c.w.h_sc[SC_RES + 1]);
  if (nb == 0.0) *out = nr == 0.0 ? 0.0 : INFINITY;
  else *out = nr / nb;
  return HMX_OK;
}

// Iterations completed and operator applications run for a recorded
// decision (or none: max_iter reached); returns the completed count.
int account_iterations(int reason, int stop_it, int max_iter, hmx_solve_report* rep) {
  int completed;
  if (reason == R_NONE) completed = max_iter;
  else if (reason == R_RHO || reason == R_DENOM || reason == R_TT || reason == R_NONFINITE)
    completed = stop_it - 1;
  else completed = stop_it;  // R_SEXIT, R_CONV, R_OMEGA complete their iteration
  rep->iterations = completed;
  rep->matvecs += 2 * completed;
  if (reason == R_DENOM) rep->matvecs += 1;
  if (reason == R_SEXIT) rep->matvecs -= 1;  // t = A s skipped on the early exit
  if (reason == R_TT) rep->matvecs += 2;
  return completed;
}

void report_breakdown(int reason, int stop_it, double bval, hmx_solve_report* rep) {
  if (reason == R_TT) {  // solver.py:139-142
    rep->breakdown = 3;
    rep->breakdown_iteration = stop_it;
    return;
  }
  // rho (solver.py:113-115), shadow projection (:123-125), omega (:155-157)
  rep->breakdown = reason == R_RHO ? 1 : reason == R_DENOM ? 2 : 4;
  rep->breakdown_value = bval;
  rep->breakdown_iteration = stop_it;
}

int workspace_for(hmx_plan* p, Workspace& out, int grid) {
  if (!p->ws) {
    auto* w = new Workspace();
    int rc = alloc_ws(p, *w, p->n, grid);
    if (rc) {
      delete w;
      return rc;
    }
    p->ws = w;
  }
  out = *p->ws;
  return HMX_OK;
}

}  // namespace

extern "C" {

int hmx_true_residual(hmx_plan* p64, const double* x, const double* b, double* out) {
  NvtxRange nvtx("hmx_true_residual");
  if (!p64 || !x || !b || !out) {
    set_error("null argument");
    return HMX_ERR_ARG;
  }
  std::lock_guard<std::mutex> lock(p64->mu);
  DeviceGuard guard(p64->device);
  int sms = 0;  // (cudaGetDeviceProperties costs milliseconds; the attribute does not)
  HMX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p64->device));
  SolveCtx c{};
  c.A = c.A64 = p64;
  c.st = p64->stream;
  HMX_CUDA(plan_enter(p64, c.st));
  c.grid = 2 * sms;
  int rc = workspace_for(p64, c.w, c.grid);
  if (rc) return rc;
  const int64_t n = p64->n;
  const int nb = (int)((n + 255) / 256);
  HMX_CUDA(cudaMemcpyAsync(c.w.orig, x, n * sizeof(double), cudaMemcpyHostToDevice, c.st));
  permute_kernel<<<nb, 256, 0, c.st>>>(c.w.orig, p64->dp.perm, c.w.x, (int)n, 0);
  HMX_CUDA(cudaMemcpyAsync(c.w.orig, b, n * sizeof(double), cudaMemcpyHostToDevice, c.st));
  permute_kernel<<<nb, 256, 0, c.st>>>(c.w.orig, p64->dp.perm, c.w.b, (int)n, 0);
  HMX_CUDA(cudaMemsetAsync(c.w.flags, 0, 4 * sizeof(int), c.st));
  return true_residual_dev(c, out);
}

int hmx_bicgstab(hmx_plan* A, hmx_plan* A64, const double* b, double tol, int max_iter, double* x,
                 double* history, hmx_solve_report* rep) {
  NvtxRange nvtx("hmx_bicgstab");
  if (!A || !b || !x || !history || !rep) {
    set_error("null argument");
    return HMX_ERR_ARG;
  }
  if (!A64) A64 = A;
  if (A64->n != A->n || A64->device != A->device) {
    set_error("plan and FP64 plan differ in size or device");
    return HMX_ERR_ARG;
  }
  if (!(tol > 0.0) || max_iter < 1) {
    set_error("tol must be positive and max_iter >= 1");
    return HMX_ERR_ARG;
  }
  std::unique_lock<std::mutex> l1(A->mu, std::defer_lock), l2(A64->mu, std::defer_lock);
  if (A == A64) l1.lock();
  else std::lock(l1, l2);
  DeviceGuard guard(A->device);
  *rep = hmx_solve_report{};
  int sms = 0;
  HMX_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, A->device));
  SolveCtx c{};
  c.A = A;
  c.A64 = A64;
  c.st = A->stream;
  HMX_CUDA(plan_enter(A, c.st));
  if (A64 != A) HMX_CUDA(plan_enter(A64, c.st));
  c.grid = 2 * sms;
  int rc = workspace_for(A, c.w, c.grid);
  if (rc) return rc;
  const int64_t n = A->n;
  const int n32 = (int)n;
  const int pgrid = (int)((n + 255) / 256);
  Workspace& w = c.w;
  cudaStream_t st = c.st;

  HMX_CUDA(cudaEventRecord(A->ev[6], st));
  HMX_CUDA(cudaMemcpyAsync(w.orig, b, n * sizeof(double), cudaMemcpyHostToDevice, st));
  permute_kernel<<<pgrid, 256, 0, st>>>(w.orig, A->dp.perm, w.b, n32, 0);
  HMX_CUDA(cudaMemsetAsync(w.flags, 0, 4 * sizeof(int), st));
  // |b| (solver.py:91)
  dot2_kernel<<<c.grid, kVecThreads, 0, st>>>(w.b, w.b, nullptr, nullptr, n32, c.red(SC_BB));
  HMX_CUDA(cudaGetLastError());
  if ((rc = sync_scalars(c))) return rc;
  const double nb = std::sqrt(w.h_sc[SC_BB]);
  int hlen = 0;
  auto finish = [&](int status) -> int {
    rep->history_len = hlen;
    if (status == HMX_OK) {
      permute_kernel<<<pgrid, 256, 0, st>>>(w.x, A->dp.perm, w.orig, n32, 1);
      HMX_CUDA(cudaMemcpyAsync(x, w.orig, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    HMX_CUDA(cudaEventRecord(A->ev[7], st));
    HMX_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, A->ev[6], A->ev[7]);
    rep->device_ms = ms;
    return status;
  };
  if (nb == 0.0) {  // zero data: x = 0 is exact (solver.py:92-97)
    HMX_CUDA(cudaMemsetAsync(w.x, 0, n * sizeof(double), st));
    history[hlen++] = 0.0;
    rep->converged = 1;
    rep->has_true_residual = 1;
    rep->true_residual = 0.0;
    return finish(HMX_OK);
  }

  // x = 0 ; r = b - A x ; r_hat = r   (solver.py:99-102)
  if (w.hist_cap < max_iter + 2) {
    double* hd = A->alloc<double>((size_t)max_iter + 2);
    if (!hd) {
      set_error("cudaMalloc failed for the residual history");
      return HMX_ERR_CUDA;
    }
    A->ws->hist = w.hist = hd;
    A->ws->hist_cap = w.hist_cap = max_iter + 2;
  }
  HMX_CUDA(cudaMemsetAsync(w.p, 0, n * sizeof(double), st));
  HMX_CUDA(cudaMemsetAsync(w.stop, 0, 4 * sizeof(int), st));
  if ((rc = apply(A, w, st, w.p, w.t, nullptr, 0, 0, w.flags))) return rc;
  rep->matvecs++;
  init_kernel<<<c.grid, kVecThreads, 0, st>>>(w.b, w.t, w.r, w.rhat, w.x, n32, c.red(SC_RHO1));
  HMX_CUDA(cudaGetLastError());
  // |b| for the device-side relative residuals
  HMX_CUDA(cudaMemcpyAsync(w.sc + SC_NB, &nb, sizeof(double), cudaMemcpyHostToDevice, st));
  if ((rc = sync_scalars(c))) return rc;
  if (flags_nonfinite(c)) {
    set_error("non-finite matvec result");
    return finish(HMX_ERR_NONFINITE);
  }
  // rho_1 = r^.r = |r|^2 lives in ring slot (1 & 1) = SC_RHO1
  history[hlen++] = std::sqrt(w.h_sc[SC_RHO1]) / nb;

  // iteration control on the device: i = 1, max_iter, tol
  {
    const int ctl[4] = {1, max_iter, 0, 0};
    HMX_CUDA(cudaMemcpyAsync(w.ictl, ctl, sizeof(ctl), cudaMemcpyHostToDevice, st));
    HMX_CUDA(cudaMemcpyAsync(w.sc + SC_TOL, &tol, sizeof(double), cudaMemcpyHostToDevice, st));
  }
  int reason = R_NONE, stop_it = 0;
  bool looped = false;
  Workspace& ws = *A->ws;
  if (!ws.loop_failed && !std::getenv("HMX_SOLVER_NO_GRAPH")) {
    if (!ws.loop_exec || ws.loop_hist != w.hist) {
      if (build_loop_graph(c, ws, n32) != HMX_OK) {
        // e.g. a driver without conditional graph nodes: keep the batched path
        cudaStreamCaptureStatus cs;
        if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
          cudaGraph_t junk = nullptr;
          cudaStreamEndCapture(st, &junk);
          if (junk) cudaGraphDestroy(junk);
        }
        cudaGetLastError();
        ws.loop_failed = true;
      }
    }
    if (!ws.loop_failed) {
      HMX_CUDA(cudaGraphLaunch(ws.loop_exec, st));
      if ((rc = sync_scalars(c))) return rc;
      looped = true;
    }
  }
  if (!looped) {
    // speculative batches: kernels after a recorded decision are no-ops, so
    // over-enqueueing only costs launches
    int done_through = 0;
    int batch = 2;
    while (done_through < max_iter) {
      const int last = std::min(max_iter, done_through + batch);
      for (int i = done_through + 1; i <= last; ++i)
        if ((rc = enqueue_iteration(c, n32, 0, 0))) return rc;
      done_through = last;
      if ((rc = sync_scalars(c))) return rc;
      if (host_stop(c)[0]) break;
      batch = std::min(batch * 2, 16);
    }
  }
  {
    const int* sw = host_stop(c);
    if (sw[0]) {
      reason = sw[1];
      stop_it = sw[2];
    }
  }
  const int completed = account_iterations(reason, stop_it, max_iter, rep);
  if (completed > 0) {
    HMX_CUDA(cudaMemcpyAsync(history + 1, w.hist + 1, (size_t)completed * sizeof(double),
                             cudaMemcpyDeviceToHost, st));
    HMX_CUDA(cudaStreamSynchronize(st));
    hlen += completed;
  }
  const double bval = w.h_sc[SC_BVAL];
  switch (reason) {
    case R_NONFINITE: {
      const int* f = reinterpret_cast<const int*>(w.h_sc + SC_N);
      A->last_xp = f[0] ? w.p : w.s;  // the failing product's input, for the probe
      set_error("non-finite matvec result");
      return finish(HMX_ERR_NONFINITE);
    }
    case R_RHO:
    case R_DENOM:
    case R_OMEGA:
    case R_TT:
      report_breakdown(reason, stop_it, bval, rep);
      break;
    case R_SEXIT:  // solver.py:130-136: x = x + alpha p, then confirm
      x_alpha_p_kernel<<<c.grid, kVecThreads, 0, st>>>(w.x, w.p, n32, w.sc);
      HMX_CUDA(cudaGetLastError());
      /* fallthrough */
    case R_CONV: {  // solver.py:151-154
      double tr = 0.0;
      if ((rc = true_residual_dev(c, &tr))) return finish(rc);
      rep->matvecs++;
      rep->has_true_residual = 1;
      rep->true_residual = tr;
      rep->converged = tr < tol;
      break;
    }
    default:
      break;
  }
  return finish(HMX_OK);
}

}  // extern "C"

// ==============================================================================
// Multi-GPU mode: row slices, one NCCL allgather of the iterate
// per operator application, small NCCL allreduces for the dot products.  The
// iteration is the single-GPU one (same kernels, same IEEE scalar
// arithmetic, same stop word); the kernels' grid reductions produce local
// partials and the decisions move to decide_s/decide_r after the allreduce.
// Iterations are enqueued in speculative batches guarded by the stop word
// (one host synchronisation per batch); collectives are always enqueued, so
// every rank issues the same sequence.

struct hmx_comm {
  std::mutex mu;
  ncclComm_t nc = nullptr;
  int world = 1, rank = 0, device = 0;
  std::vector<int64_t> cuts;
  int64_t n = 0, r0 = 0, r1 = 0;
  std::vector<void*> allocs;
  // full permuted vectors (allgather targets)
  double *x_full = nullptr, *p_full = nullptr, *s_full = nullptr;
  // local rows
  double *b = nullptr, *x = nullptr, *r = nullptr, *rhat = nullptr, *v = nullptr, *t = nullptr,
         *y = nullptr;
  double* sc = nullptr;
  double* h_sc = nullptr;  // pinned mirror: scalars, flags, stop word
  int* flags = nullptr;
  int* stop = nullptr;
  int* ictl = nullptr;
  double* partials = nullptr;
  uint32_t* done = nullptr;
  double* hist = nullptr;
  int hist_cap = 0;
  int grid = 0;
  cudaEvent_t ev[2] = {};
  // overlap of the allgather with the stage-1 work on the local x slice
  cudaStream_t side = nullptr;
  cudaEvent_t ev_x = nullptr, ev_local = nullptr;
  bool overlap = false;

  template <typename T>
  T* alloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    if (cudaMalloc(&p, count * sizeof(T)) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
};

// NCCL is resolved at run time (first hmx_comm_* call) rather than linked:
// dlopen("libnccl.so.2") returns the NCCL the process already holds -- the
// one torch loaded -- so a single NCCL serves torch.distributed and this
// library (linking it would put the system libnccl in the process first,
// and torch's libtorch_cuda needs symbols of its own, newer copy).
// HMX_NCCL_LIB names a specific library instead.
struct NcclApi {
  bool ok = false;
  std::string error;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
};

static NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    const char* env = std::getenv("HMX_NCCL_LIB");
    void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h && !env) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      a.error = std::string("cannot load NCCL: ") + dlerror();
      return a;
    }
    bool all = true;
    auto get = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) {
        all = false;
        a.error += std::string(" missing ") + name;
      }
    };
    get(a.GetUniqueId, "ncclGetUniqueId");
    get(a.CommInitRank, "ncclCommInitRank");
    get(a.CommDestroy, "ncclCommDestroy");
    get(a.GetErrorString, "ncclGetErrorString");
    get(a.GroupStart, "ncclGroupStart");
    get(a.GroupEnd, "ncclGroupEnd");
    get(a.Send, "ncclSend");
    get(a.Recv, "ncclRecv");
    get(a.AllReduce, "ncclAllReduce");
    a.ok = all;
    return a;
  }();
  return api;
}

#define HMX_NCCL(call)                                                                    \
  do {                                                                                    \
    ncclResult_t _r = (call);                                                             \
    if (_r != ncclSuccess) {                                                              \
      hmx::set_error(std::string("NCCL error in " #call ": ") + nccl_api().GetErrorString(_r));    \
      return HMX_ERR_COMM;                                                                \
    }                                                                                     \
  } while (0)

namespace {

// The one exchange per operator application: every rank's slice of `full`
// (its rows [cuts[q], cuts[q+1])) to every other rank, grouped NCCL
// send/recv straight into place (uneven slices, no padding, no copies).
int allgather_rows(hmx_comm* c, double* full, cudaStream_t st) {
  if (c->world == 1) return HMX_OK;
  const int64_t m = c->r1 - c->r0;
  HMX_NCCL(nccl_api().GroupStart());
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) continue;
    const int64_t mq = c->cuts[(size_t)q + 1] - c->cuts[(size_t)q];
    if (m > 0) HMX_NCCL(nccl_api().Send(full + c->r0, (size_t)m, ncclFloat64, q, c->nc, st));
    if (mq > 0) HMX_NCCL(nccl_api().Recv(full + c->cuts[(size_t)q], (size_t)mq, ncclFloat64, q, c->nc, st));
  }
  HMX_NCCL(nccl_api().GroupEnd());
  return HMX_OK;
}

int allreduce_sum(hmx_comm* c, double* v, int count, cudaStream_t st) {
  HMX_NCCL(nccl_api().AllReduce(v, v, (size_t)count, ncclFloat64, ncclSum, c->nc, st));
  return HMX_OK;
}

// dot partials (sum) and a non-finite flag (max) in one NCCL group
int allreduce_dots_flag(hmx_comm* c, double* dots, int count, int* flag, cudaStream_t st) {
  HMX_NCCL(nccl_api().GroupStart());
  if (count > 0) HMX_NCCL(nccl_api().AllReduce(dots, dots, (size_t)count, ncclFloat64, ncclSum, c->nc, st));
  HMX_NCCL(nccl_api().AllReduce(flag, flag, 1, ncclInt32, ncclMax, c->nc, st));
  HMX_NCCL(nccl_api().GroupEnd());
  return HMX_OK;
}

// y_local = rows of A full, with the one exchange: `full` holds this rank's
// slice (written on st); the allgather of the other slices runs on st while
// the plan's leading stage-1 segments that read only the local slice
// (HMX_PLAN_LOCAL_FIRST) run on the side stream; then the rest of stage 1
// and stage 2 (dots fused as in apply_sc).  Without local-first segments
// this is allgather + apply_sc.
int dist_apply(hmx_comm* c, hmx_plan* A, double* sc, cudaStream_t st, double* full, double* y,
               const double* w1, int yy, int slot, int* flag, const int* skip = nullptr) {
  // (one rank has nothing to gather: a single stream is cheaper, except
  // under the test hook that exercises the two-stream path)
  const int nloc = c->overlap ? A->dp.n_seg1_local : 0;
  if (nloc > 0) {
    HMX_CUDA(cudaEventRecord(c->ev_x, st));
    HMX_CUDA(cudaStreamWaitEvent(c->side, c->ev_x, 0));
    HMX_CUDA(launch_stage1(A->dp, full, c->side, skip, 0, nloc));
    HMX_CUDA(cudaEventRecord(c->ev_local, c->side));
  }
  int rc = allgather_rows(c, full, st);
  if (rc) return rc;
  if ((w1 || yy) && A->dp.n_seg2 == 0) HMX_CUDA(cudaMemsetAsync(sc + slot, 0, 2 * sizeof(double), st));
  const S2Out out = solver_out(A, sc, y, w1, yy, slot, flag, skip);
  HMX_CUDA(launch_stage1(A->dp, full, st, skip, nloc, -1));
  if (nloc > 0) HMX_CUDA(cudaStreamWaitEvent(st, c->ev_local, 0));
  HMX_CUDA(launch_stage2(A->dp, full, out, st, /*pdl=*/true));
  A->last_xp = full;
  return HMX_OK;
}

struct DistCtx {
  hmx_plan* A;
  hmx_plan* A64;
  hmx_comm* c;
  cudaStream_t st;
  int grid;
  int nl;
  VecRed red(int slot) const { return VecRed{c->partials, c->done, c->sc + slot}; }
};

int dist_sync(const DistCtx& d) {
  hmx_comm* c = d.c;
  HMX_CUDA(cudaMemcpyAsync(c->h_sc, c->sc, SC_N * sizeof(double), cudaMemcpyDeviceToHost, d.st));
  HMX_CUDA(cudaMemcpyAsync(c->h_sc + SC_N, c->flags, 4 * sizeof(int), cudaMemcpyDeviceToHost, d.st));
  HMX_CUDA(cudaMemcpyAsync(c->h_sc + SC_N + 2, c->stop, 4 * sizeof(int), cudaMemcpyDeviceToHost, d.st));
  HMX_CUDA(cudaStreamSynchronize(d.st));
  return HMX_OK;
}

const int* dist_host_stop(const DistCtx& d) { return reinterpret_cast<const int*>(d.c->h_sc + SC_N + 2); }
const int* dist_host_flags(const DistCtx& d) { return reinterpret_cast<const int*>(d.c->h_sc + SC_N); }

// one iteration on the local rows (the single-GPU enqueue_iteration with the
// collectives between its kernels)
int enqueue_iteration_dist(const DistCtx& d) {
  hmx_comm* c = d.c;
  cudaStream_t st = d.st;
  double* pl = c->p_full + c->r0;
  double* sl = c->s_full + c->r0;
  int rc;
  p_update_kernel<<<d.grid, kVecThreads, 0, st>>>(c->r, c->v, pl, d.nl, c->ictl, c->sc, c->stop);
  if ((rc = dist_apply(c, d.A, c->sc, st, c->p_full, c->v, c->rhat, 0, SC_DV, c->flags, c->stop))) return rc;
  if ((rc = allreduce_dots_flag(c, c->sc + SC_DV, 1, c->flags, st))) return rc;
  s_update_kernel<<<d.grid, kVecThreads, 0, st>>>(c->r, c->v, sl, d.nl, c->sc, d.red(SC_SS), c->ictl,
                                                    c->hist, c->stop, c->flags, 1);
  if ((rc = allreduce_sum(c, c->sc + SC_SS, 1, st))) return rc;
  decide_s_kernel<<<1, 1, 0, st>>>(c->sc, c->ictl, c->hist, c->stop);
  if ((rc = dist_apply(c, d.A, c->sc, st, c->s_full, c->t, sl, 1, SC_DT, c->flags + 1, c->stop))) return rc;
  if ((rc = allreduce_dots_flag(c, c->sc + SC_DT, 2, c->flags + 1, st))) return rc;
  xr_update_kernel<<<d.grid, kVecThreads, 0, st>>>(c->x, c->r, pl, sl, c->t, c->rhat, d.nl, c->sc,
                                                     d.red(SC_TMP), c->ictl, c->hist, c->stop,
                                                     c->flags + 1, 1);
  if ((rc = allreduce_sum(c, c->sc + SC_TMP, 2, st))) return rc;
  decide_r_kernel<<<1, 1, 0, st>>>(c->sc, c->ictl, c->hist, c->stop);
  advance_kernel<<<1, 1, 0, st>>>(c->ictl, c->stop, 0, 0);
  HMX_CUDA(cudaGetLastError());
  return HMX_OK;
}

// |b - A64 x| / |b| over all ranks (solver.py:56-65)
int true_residual_dist(const DistCtx& d, double* out) {
  hmx_comm* c = d.c;
  cudaStream_t st = d.st;
  int rc;
  if (d.nl > 0)
    HMX_CUDA(cudaMemcpyAsync(c->x_full + c->r0, c->x, (size_t)d.nl * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if ((rc = dist_apply(c, d.A64, c->sc, st, c->x_full, c->y, nullptr, 0, 0, c->flags + 2))) return rc;
  resid_kernel<<<d.grid, kVecThreads, 0, st>>>(c->b, c->y, d.nl, d.red(SC_RES));
  HMX_CUDA(cudaGetLastError());
  if ((rc = allreduce_dots_flag(c, c->sc + SC_RES, 2, c->flags + 2, st))) return rc;
  if ((rc = dist_sync(d))) return rc;
  if (dist_host_flags(d)[2]) {
    set_error("non-finite matvec result");
    return HMX_ERR_NONFINITE;
  }
  const double nr = std::sqrt(c->h_sc[SC_RES]), nb = std::sqrt(c->h_sc[SC_RES + 1]);
  if (nb == 0.0) *out = nr == 0.0 ? 0.0 : INFINITY;
  else *out = nr / nb;
  return HMX_OK;
}

bool plan_matches(const hmx_plan* p, const hmx_comm* c) {
  return p->n == c->n && p->dp.row_begin == c->r0 && p->dp.row_end == c->r1 && p->device == c->device;
}

}  // namespace

extern "C" {

int hmx_comm_unique_id(uint8_t id[128]) {
  if (!id) return HMX_ERR_ARG;
  if (!nccl_api().ok) {
    set_error(nccl_api().error);
    return HMX_ERR_COMM;
  }
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
  ncclUniqueId u;
  HMX_NCCL(nccl_api().GetUniqueId(&u));
  std::memcpy(id, &u, sizeof(u));
  return HMX_OK;
}

void hmx_comm_destroy(hmx_comm* c) {
  if (!c) return;
  {
    DeviceGuard g(c->device);
    cudaDeviceSynchronize();
    if (c->nc) nccl_api().CommDestroy(c->nc);
    for (void* a : c->allocs) cudaFree(a);
    if (c->h_sc) cudaFreeHost(c->h_sc);
    for (auto& e : c->ev)
      if (e) cudaEventDestroy(e);
    if (c->ev_x) cudaEventDestroy(c->ev_x);
    if (c->ev_local) cudaEventDestroy(c->ev_local);
    if (c->side) cudaStreamDestroy(c->side);
  }
  delete c;
}

int hmx_comm_create(const uint8_t id[128], int world, int rank, int device, const int64_t* cuts,
                    hmx_comm** out) {
  if (!id || !cuts || !out || world < 1 || rank < 0 || rank >= world) {
    set_error("hmx_comm_create: bad arguments");
    return HMX_ERR_ARG;
  }
  *out = nullptr;
  if (!nccl_api().ok) {
    set_error(nccl_api().error);
    return HMX_ERR_COMM;
  }
  if (cuts[0] != 0) {
    set_error("hmx_comm_create: cuts[0] must be 0");
    return HMX_ERR_ARG;
  }
  for (int q = 0; q < world; ++q)
    if (cuts[q + 1] < cuts[q]) {
      set_error("hmx_comm_create: cuts must be non-decreasing");
      return HMX_ERR_ARG;
    }
  if (cuts[world] > INT32_MAX || cuts[world] < 1) {
    set_error("hmx_comm_create: n out of range");
    return HMX_ERR_ARG;
  }
  DeviceGuard guard(device);
  HMX_CUDA(cudaSetDevice(device));
  auto* c = new hmx_comm();
  c->world = world;
  c->rank = rank;
  c->device = device;
  c->cuts.assign(cuts, cuts + world + 1);
  c->n = cuts[world];
  c->r0 = cuts[rank];
  c->r1 = cuts[rank + 1];
  c->overlap = world > 1 || std::getenv("HMX_TEST_SPLIT_STAGE1") != nullptr;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  const ncclResult_t r = nccl_api().CommInitRank(&c->nc, world, u, rank);
  if (r != ncclSuccess) {
    set_error(std::string("ncclCommInitRank: ") + nccl_api().GetErrorString(r));
    c->nc = nullptr;
    hmx_comm_destroy(c);
    return HMX_ERR_COMM;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  c->grid = 2 * sms;
  const size_t n = (size_t)c->n, nl = (size_t)(c->r1 - c->r0);
  c->x_full = c->alloc<double>(n);
  c->p_full = c->alloc<double>(n);
  c->s_full = c->alloc<double>(n);
  double** loc[] = {&c->b, &c->x, &c->r, &c->rhat, &c->v, &c->t, &c->y};
  bool ok = c->x_full && c->p_full && c->s_full;
  for (double** v : loc) ok = ok && (*v = c->alloc<double>(nl)) != nullptr;
  c->sc = c->alloc<double>(SC_N);
  c->flags = c->alloc<int>(4);
  c->stop = c->alloc<int>(4);
  c->ictl = c->alloc<int>(4);
  c->partials = c->alloc<double>((size_t)2 * c->grid);
  c->done = c->alloc<uint32_t>(1);
  ok = ok && c->sc && c->flags && c->stop && c->ictl && c->partials && c->done;
  if (!ok || cudaMallocHost(&c->h_sc, (SC_N + 8) * sizeof(double)) != cudaSuccess ||
      cudaMemset(c->done, 0, sizeof(uint32_t)) != cudaSuccess ||
      cudaMemset(c->sc, 0, SC_N * sizeof(double)) != cudaSuccess ||
      cudaMemset(c->x_full, 0, n * sizeof(double)) != cudaSuccess ||
      cudaEventCreate(&c->ev[0]) != cudaSuccess || cudaEventCreate(&c->ev[1]) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_x, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_local, cudaEventDisableTiming) != cudaSuccess) {
    set_error("hmx_comm_create: device allocation failed");
    hmx_comm_destroy(c);
    return HMX_ERR_CUDA;
  }
  *out = c;
  return HMX_OK;
}

int hmx_dist_matvec(hmx_plan* p, hmx_comm* c, const double* x_local, double* y_local, int* nonfinite,
                    uint64_t stream) {
  NvtxRange nvtx("hmx_dist_matvec");
  if (!p || !c || (!x_local && c->r1 > c->r0) || (!y_local && c->r1 > c->r0)) {
    set_error("null argument");
    return HMX_ERR_ARG;
  }
  if (!plan_matches(p, c)) {
    set_error("plan rows / device do not match this rank's slice");
    return HMX_ERR_ARG;
  }
  std::scoped_lock lock(c->mu, p->mu);
  DeviceGuard guard(p->device);
  cudaStream_t st = stream == UINT64_MAX ? p->stream : reinterpret_cast<cudaStream_t>(stream);
  const int64_t nl = c->r1 - c->r0;
  HMX_CUDA(plan_enter(p, st));
  if (nl > 0 && x_local != c->x_full + c->r0)
    HMX_CUDA(cudaMemcpyAsync(c->x_full + c->r0, x_local, (size_t)nl * sizeof(double), cudaMemcpyDeviceToDevice, st));
  const int rc = dist_apply(c, p, c->sc, st, c->x_full, y_local, nullptr, 0, 0,
                            nonfinite ? nonfinite : p->d_nonfinite);
  if (rc) return rc;
  HMX_CUDA(plan_leave(p, st));
  return HMX_OK;
}

int hmx_bicgstab_dist(hmx_plan* A, hmx_plan* A64, hmx_comm* c, const double* b_local, double tol,
                      int max_iter, double* x_local, double* history, hmx_solve_report* rep) {
  NvtxRange nvtx("hmx_bicgstab_dist");
  if (!A || !c || !history || !rep || ((!b_local || !x_local) && c->r1 > c->r0)) {
    set_error("null argument");
    return HMX_ERR_ARG;
  }
  if (!A64) A64 = A;
  if (!plan_matches(A, c) || !plan_matches(A64, c)) {
    set_error("plan rows / device do not match this rank's slice");
    return HMX_ERR_ARG;
  }
  if (!(tol > 0.0) || max_iter < 1) {
    set_error("tol must be positive and max_iter >= 1");
    return HMX_ERR_ARG;
  }
  std::unique_lock<std::mutex> l0(c->mu, std::defer_lock), l1(A->mu, std::defer_lock),
      l2(A64->mu, std::defer_lock);
  if (A == A64) std::lock(l0, l1);
  else std::lock(l0, l1, l2);
  DeviceGuard guard(A->device);
  *rep = hmx_solve_report{};
  DistCtx d{A, A64, c, A->stream, c->grid, (int)(c->r1 - c->r0)};
  cudaStream_t st = d.st;
  HMX_CUDA(plan_enter(A, st));
  if (A64 != A) HMX_CUDA(plan_enter(A64, st));
  const size_t nlb = (size_t)d.nl * sizeof(double);
  int rc;

  HMX_CUDA(cudaEventRecord(c->ev[0], st));
  if (d.nl > 0) HMX_CUDA(cudaMemcpyAsync(c->b, b_local, nlb, cudaMemcpyHostToDevice, st));
  HMX_CUDA(cudaMemsetAsync(c->flags, 0, 4 * sizeof(int), st));
  HMX_CUDA(cudaMemsetAsync(c->stop, 0, 4 * sizeof(int), st));
  // |b| (solver.py:91)
  dot2_kernel<<<d.grid, kVecThreads, 0, st>>>(c->b, c->b, nullptr, nullptr, d.nl, d.red(SC_BB));
  HMX_CUDA(cudaGetLastError());
  if ((rc = allreduce_sum(c, c->sc + SC_BB, 1, st))) return rc;
  if ((rc = dist_sync(d))) return rc;
  const double nb = std::sqrt(c->h_sc[SC_BB]);
  int hlen = 0;
  auto finish = [&](int status) -> int {
    rep->history_len = hlen;
    if (status == HMX_OK && d.nl > 0) HMX_CUDA(cudaMemcpyAsync(x_local, c->x, nlb, cudaMemcpyDeviceToHost, st));
    HMX_CUDA(cudaEventRecord(c->ev[1], st));
    HMX_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev[0], c->ev[1]);
    rep->device_ms = ms;
    return status;
  };
  if (nb == 0.0) {  // zero data: x = 0 is exact (solver.py:92-97)
    if (d.nl > 0) HMX_CUDA(cudaMemsetAsync(c->x, 0, nlb, st));
    history[hlen++] = 0.0;
    rep->converged = 1;
    rep->has_true_residual = 1;
    rep->true_residual = 0.0;
    return finish(HMX_OK);
  }
  if (c->hist_cap < max_iter + 2) {
    double* hd = c->alloc<double>((size_t)max_iter + 2);
    if (!hd) {
      set_error("cudaMalloc failed for the residual history");
      return HMX_ERR_CUDA;
    }
    c->hist = hd;
    c->hist_cap = max_iter + 2;
  }
  // x = 0 ; r = b - A x ; r_hat = r   (solver.py:99-102)
  HMX_CUDA(cudaMemsetAsync(c->p_full, 0, (size_t)c->n * sizeof(double), st));
  if ((rc = apply_sc(A, c->sc, st, c->p_full, c->t, nullptr, 0, 0, c->flags))) return rc;
  rep->matvecs++;
  if ((rc = allreduce_dots_flag(c, nullptr, 0, c->flags, st))) return rc;
  init_kernel<<<d.grid, kVecThreads, 0, st>>>(c->b, c->t, c->r, c->rhat, c->x, d.nl, d.red(SC_RHO1));
  HMX_CUDA(cudaGetLastError());
  if ((rc = allreduce_sum(c, c->sc + SC_RHO1, 1, st))) return rc;
  HMX_CUDA(cudaMemcpyAsync(c->sc + SC_NB, &nb, sizeof(double), cudaMemcpyHostToDevice, st));
  if ((rc = dist_sync(d))) return rc;
  if (dist_host_flags(d)[0]) {
    set_error("non-finite matvec result");
    return finish(HMX_ERR_NONFINITE);
  }
  history[hlen++] = std::sqrt(c->h_sc[SC_RHO1]) / nb;
  {
    const int ctl[4] = {1, max_iter, 0, 0};
    HMX_CUDA(cudaMemcpyAsync(c->ictl, ctl, sizeof(ctl), cudaMemcpyHostToDevice, st));
    HMX_CUDA(cudaMemcpyAsync(c->sc + SC_TOL, &tol, sizeof(double), cudaMemcpyHostToDevice, st));
  }
  // speculative batches (identical on every rank: the stop word is)
  int done_through = 0, batch = 2;
  while (done_through < max_iter) {
    const int last = std::min(max_iter, done_through + batch);
    for (int i = done_through + 1; i <= last; ++i)
      if ((rc = enqueue_iteration_dist(d))) return rc;
    done_through = last;
    if ((rc = dist_sync(d))) return rc;
    if (dist_host_stop(d)[0]) break;
    batch = std::min(batch * 2, 16);
  }
  int reason = R_NONE, stop_it = 0;
  if (dist_host_stop(d)[0]) {
    reason = dist_host_stop(d)[1];
    stop_it = dist_host_stop(d)[2];
  }
  const int completed = account_iterations(reason, stop_it, max_iter, rep);
  if (completed > 0) {
    HMX_CUDA(cudaMemcpyAsync(history + 1, c->hist + 1, (size_t)completed * sizeof(double),
                             cudaMemcpyDeviceToHost, st));
    HMX_CUDA(cudaStreamSynchronize(st));
    hlen += completed;
  }
  const double bval = c->h_sc[SC_BVAL];
  switch (reason) {
    case R_NONFINITE:
      A->last_xp = dist_host_flags(d)[0] ? c->p_full : c->s_full;
      set_error("non-finite matvec result");
      return finish(HMX_ERR_NONFINITE);
    case R_RHO:
    case R_DENOM:
    case R_OMEGA:
    case R_TT:
      report_breakdown(reason, stop_it, bval, rep);
      break;
    case R_SEXIT:  // solver.py:130-136
      x_alpha_p_kernel<<<d.grid, kVecThreads, 0, st>>>(c->x, c->p_full + c->r0, d.nl, c->sc);
      HMX_CUDA(cudaGetLastError());
      /* fallthrough */
    case R_CONV: {  // solver.py:151-154
      double tr = 0.0;
      if ((rc = true_residual_dist(d, &tr))) return finish(rc);
      rep->matvecs++;
      rep->has_true_residual = 1;
      rep->true_residual = tr;
      rep->converged = tr < tol;
      break;
    }
    default:
      break;
  }
  return finish(HMX_OK);
}

}  // extern "C"
