// Flattener + plan lifetime + matvec C ABI.
//
// hmx_plan_create turns the packed payloads of one prepared scheme
// (python PackedScheme; reference SchemeHMatrix, precision.py:209-234) into
// the two streaming blobs of hmx_internal.cuh and uploads them:
//   * stage-1 blob: the Vt rank rows of every low-rank block (class), stacked
//     per column cluster, cut into segments of rank rows and column chunks,
//     column-major (m1-single in SGEMV order: chunk layout, chunk_off);
//   * stage-2 blob: for every leaf row segment (<= 64 rows), the rows of every
//     block covering it (dense values or U slab), column-major, FP64 items
//     and FP32 items in two parts; the FP32 part ordered by thread group
//     (widened items, streamed FP32-accumulated items, the chain lanes' items
//     slot by slot; plan_fp32_groups).
// Every stored payload byte appears exactly once on the device.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <tuple>
#include <numeric>
#include <queue>
#include <chrono>
#include <cstdlib>
#include <thread>

#include "hmx_plan_impl.cuh"

namespace hmx {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
  return HMX_ERR_CUDA;
}

static void parallel_for(int64_t count, const std::function<void(int64_t)>& fn) {
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(count, std::thread::hardware_concurrency()));
  if (nt <= 1) {
    for (int64_t i = 0; i < count; ++i) fn(i);
    return;
  }
  std::atomic<int64_t> next{0};
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&]() {
      for (int64_t i; (i = next.fetch_add(1)) < count;) fn(i);
    });
  for (auto& th : pool) th.join();
}

static inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

struct ItemRef {
  int32_t block;
  int8_t cls;  // 0 dense, 1 hi, 2 lo
};

int enqueue_matvec(hmx_plan* p, const double* xp, const S2Out& out) {
  HMX_CUDA(launch_stage1(p->dp, xp, p->stream));
  HMX_CUDA(launch_stage2(p->dp, xp, out, p->stream, /*pdl=*/true));
  return HMX_OK;
}

}  // namespace hmx

using namespace hmx;

extern "C" {

const char* hmx_last_error(void) { return g_last_error.c_str(); }

int hmx_device_count(int* count) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) {
    *count = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  *count = c;
  return HMX_OK;
}

void hmx_plan_destroy(hmx_plan* p) {
  if (!p) return;
  {
    DeviceGuard g(p->device);
    if (p->stream) cudaStreamSynchronize(p->stream);
    for (void* a : p->allocs) cudaFree(a);
    if (p->h_flag) cudaFreeHost(p->h_flag);
    for (void* h : p->pinned) cudaFreeHost(h);
    if (p->ws) {
      if (p->ws->loop_exec) cudaGraphExecDestroy(p->ws->loop_exec);
      if (p->ws->loop_graph) cudaGraphDestroy(p->ws->loop_graph);
    }
    delete p->ws;
    if (p->ev_tail) cudaEventSynchronize(p->ev_tail);
    for (auto& e : p->ev)
      if (e) cudaEventDestroy(e);
    if (p->ev_tail) cudaEventDestroy(p->ev_tail);
    if (p->stream) cudaStreamDestroy(p->stream);
  }
  delete p;
}

int hmx_plan_get_info(const hmx_plan* p, hmx_plan_info* info) {
  if (!p || !info) return HMX_ERR_ARG;
  *info = p->info;
  return HMX_OK;
}

int hmx_host_alloc(int64_t bytes, void** out) {
  if (!out || bytes <= 0) {
    set_error("hmx_host_alloc: bad size or null output");
    return HMX_ERR_ARG;
  }
  *out = nullptr;
  // portable: the buffer serves copies on any device's stream
  HMX_CUDA(cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable));
  return HMX_OK;
}

void hmx_host_free(void* ptr) {
  if (ptr) cudaFreeHost(ptr);
}

}  // extern "C"

int hmx::plan_create_impl(const hmx_matrix_desc* d, int device, const hmx_plan_options* opt,
                          hmx_plan* p, const DevSource* dsrc) {
  NvtxRange nvtx("hmx plan: flatten + upload");
  const int64_t n = d->n, nb = d->n_blocks;
  if (n < 1 || n > INT32_MAX / 2 || nb < 1 || d->scheme < 0 || d->scheme > HMX_M3) {
    set_error("invalid matrix descriptor (n, n_blocks or scheme)");
    return HMX_ERR_ARG;
  }
  const int pipe = d->scheme;
  const bool has_lo = pipe == P_M3;
  // FP32-accumulated products: SGEMV's order (default) or one FMA chain per (row, block)
  const bool chain_order = opt && (opt->flags & HMX_PLAN_FP32_CHAIN);
  HMX_CUDA(configure_kernels());
  const int64_t rb = opt && opt->row_end > 0 ? opt->row_begin : 0;
  const int64_t re = opt && opt->row_end > 0 ? opt->row_end : n;
  if (rb < 0 || re > n || rb >= re) {
    set_error("invalid row range");
    return HMX_ERR_ARG;
  }
  const auto t_start = std::chrono::steady_clock::now();
  auto secs = [&]() { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count(); };
  int64_t s1_target = opt && opt->s1_chunk_bytes > 0 ? opt->s1_chunk_bytes : 256 * 1024;
  const size_t a_es = d->a32 ? 4 : 8, hi_es = d->hi32 ? 4 : 8;

  // ---- validate blocks and collect the ones touching rows [rb, re)
  std::vector<int32_t> blocks;
  blocks.reserve((size_t)nb);
  int64_t payload = 0;
  for (int64_t k = 0; k < nb; ++k) {
    const int64_t* t = d->table + 5 * k;
    const int64_t m = t[1] - t[0], nc = t[3] - t[2];
    if (t[0] < 0 || t[1] > n || t[2] < 0 || t[3] > n || m < 1 || nc < 1) {
      set_error("block " + std::to_string(k) + " has an invalid range");
      return HMX_ERR_ARG;
    }
    if (d->kind[k] == 2) {  // not built (row-restricted host build)
      if (t[1] > rb && t[0] < re) {
        set_error("block " + std::to_string(k) + " meets the plan's rows but was not built");
        return HMX_ERR_ARG;
      }
      continue;
    }
    if (d->kind[k] == 0) {
      if (d->a_off[k] < 0 || d->a_off[k] + m * nc > (d->a32 ? d->n32 : d->n64)) {
        set_error("dense block " + std::to_string(k) + " exceeds its payload buffer");
        return HMX_ERR_ARG;
      }
      payload += m * nc * (int64_t)a_es;
    } else {
      const int64_t kh = d->khi[k], kl = has_lo ? d->klo[k] : 0;
      if (kh < 0 || kl < 0 || d->hi_off[k] + kh * (m + nc) > (d->hi32 ? d->n32 : d->n64) ||
          (kl && d->lo_off[k] + kl * (m + nc) > d->n32)) {
        set_error("low-rank block " + std::to_string(k) + " exceeds its payload buffer");
        return HMX_ERR_ARG;
      }
      if (pipe >= P_M2D && ((kh && (d->dhi_off[k] < 0 || d->dhi_off[k] + kh > d->n64)) ||
                            (kl && (d->dlo_off[k] < 0 || d->dlo_off[k] + kl > d->n64)))) {
        set_error("low-rank block " + std::to_string(k) + " lacks its scale diagonal");
        return HMX_ERR_ARG;
      }
      payload += kh * (m + nc) * (int64_t)hi_es + kl * (m + nc) * 4;
      if (pipe >= P_M2D) payload += (kh + kl) * 8;
    }
    if (t[1] > rb && t[0] < re) blocks.push_back((int32_t)k);
  }

  // ---- stage-2 row segments: every block row boundary, chunks of <= 64 rows
  std::vector<int64_t> bounds = {rb, re};
  for (int32_t k : blocks) {
    const int64_t* t = d->table + 5 * k;
    if (t[0] > rb) bounds.push_back(t[0]);
    if (t[1] < re) bounds.push_back(t[1]);
  }
  std::sort(bounds.begin(), bounds.end());
  bounds.erase(std::unique(bounds.begin(), bounds.end()), bounds.end());
  std::vector<int64_t> seg_start;
  for (size_t i = 0; i + 1 < bounds.size(); ++i) {
    const int64_t a = bounds[i], b = bounds[i + 1];
    const int64_t pieces = (b - a + kSegRows - 1) / kSegRows;
    for (int64_t q = 0; q < pieces; ++q) seg_start.push_back(a + (b - a) * q / pieces);
  }
  const int64_t nseg2 = (int64_t)seg_start.size();
  seg_start.push_back(re);

  // ---- stage-1 groups: rank rows of the blocks sharing a column cluster
  // (and a storage class); z is laid out group by group so every stage-1
  // segment writes a contiguous z range.
  std::map<std::tuple<int, int64_t, int64_t>, std::vector<int32_t>> groups;
  for (int32_t k : blocks) {
    if (d->kind[k] != 1) continue;
    const int64_t* t = d->table + 5 * k;
    if (d->khi[k] > 0) groups[std::make_tuple(1, t[2], t[3])].push_back(k);
    if (has_lo && d->klo[k] > 0) groups[std::make_tuple(2, t[2], t[3])].push_back(k);
  }
  std::vector<int64_t> zoff_hi((size_t)nb, -1), zoff_lo((size_t)nb, -1);
  int64_t Z = 0;
  for (auto& g : groups) {
    const int cls = std::get<0>(g.first);
    for (int32_t k : g.second) {
      (cls == 1 ? zoff_hi : zoff_lo)[(size_t)k] = Z;
      Z += cls == 1 ? d->khi[k] : d->klo[k];
    }
  }
  if (Z > INT32_MAX) {
    set_error("rank sum exceeds the 32-bit index range");
    return HMX_ERR_ARG;
  }

  // Stage-1 CTA shape.  A chunk of C bytes streams for about C / (NT x 8 x
  // 16 B) memory latencies on one CTA, so small problems want small chunks
  // (about one per resident CTA slot, 64-256 KB: config 2 is best at 64 KB,
  // configs 3-4 at 256 KB).  When every stage-1 row is widened FP32 and the
  // stage holds several waves of 256 KB chunks (config 4 and up), 64-thread
  // CTAs, 16 per SM, are faster (measured -3..-4 %); below that they lose.
  int64_t s1_total = 0;
  bool fp32_only = pipe != P_M1S && !groups.empty();
  for (auto& g : groups) {
    const int cls = std::get<0>(g.first);
    const int64_t ncol = std::get<2>(g.first) - std::get<1>(g.first);
    const bool is32 = cls == 2 || d->hi32;
    if (!is32) fp32_only = false;
    for (int32_t k : g.second) s1_total += (cls == 1 ? d->khi[k] : d->klo[k]) * ncol * (is32 ? 4 : 8);
  }
  int sms = 148;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) sms = 148;
  // (Method 3 with FP64-class rows too: 64-thread CTAs with <= 128-row
  // segments, measured -5 % on m3:c=3's stage 1; neutral-to-worse for the
  // all-FP64 schemes, which keep 128 threads)
  const bool s1_big = s1_total >= (int64_t)sms * (1024 / kS1Threads32) * (256 << 10);
  const bool s1_narrow = s1_big && (fp32_only || pipe == P_M3);
  const int64_t s1_rows = (s1_narrow && !fp32_only) ? 2 * kS1Threads32 : kS1Rows;
  if (!(opt && opt->s1_chunk_bytes > 0) && !s1_narrow) {
    const int64_t slots = (int64_t)std::max(sms, 1) * (1024 / kS1Threads);
    s1_target = std::min<int64_t>(s1_target, std::max<int64_t>(64 * 1024, s1_total / slots));
  }
  std::vector<Seg> seg1, seg2((size_t)nseg2);
  std::vector<int32_t> gtab;
  std::vector<Run> runs;
  std::vector<int32_t> run_block;
  int64_t off64 = 0, off32 = 0;

  // ---- stage-1 segments
  const bool src_round = pipe == P_M1S || pipe == P_M2S;  // FP32 source shadow (matvec.py:119)
  struct S1Fill {
    int32_t seg;       // index into seg1 (pre-sort)
    int32_t cls;
    int64_t cs, ncol;  // cluster columns
    int64_t c0;        // first column of this chunk within the cluster
    std::vector<std::pair<int32_t, int32_t>>* rows;  // (block, rank) per output row
    int32_t r0;
  };
  std::vector<std::vector<std::pair<int32_t, int32_t>>> group_rows;
  group_rows.reserve(groups.size());
  std::vector<S1Fill> fills;
  std::vector<double> zscale(pipe >= P_M2D ? (size_t)std::max<int64_t>(Z, 1) : 1, 1.0);
  // m1-single stage 1: the SGEMV row kernel of every z entry (its rank index
  // q within its block's rank r: sgemv_row_kind(q, r))
  std::vector<uint8_t> zkind(pipe == P_M1S ? (size_t)std::max<int64_t>(Z, 1) : 1, 16);
  int64_t part_len = 0;
  int32_t n_red = 0;
  int64_t s1_bytes = 0, s2_bytes = 0;
  for (auto& g : groups) {
    const int cls = std::get<0>(g.first);
    const int64_t cs = std::get<1>(g.first), ncol = std::get<2>(g.first) - cs;
    group_rows.emplace_back();
    auto& rows = group_rows.back();
    for (int32_t k : g.second) {
      const int64_t kk = cls == 1 ? d->khi[k] : d->klo[k];
      for (int64_t q = 0; q < kk; ++q) rows.push_back({k, (int32_t)q});
      if (pipe == P_M1S) {
        const int64_t z0 = cls == 1 ? zoff_hi[(size_t)k] : zoff_lo[(size_t)k];
        for (int64_t q = 0; q < kk; ++q) zkind[(size_t)(z0 + q)] = (uint8_t)sgemv_row_kind(q, kk);
      }
      if (pipe >= P_M2D) {
        const double* dsrc = d->buf64 + (cls == 1 ? d->dhi_off[k] : d->dlo_off[k]);
        const int64_t z0 = cls == 1 ? zoff_hi[(size_t)k] : zoff_lo[(size_t)k];
        for (int64_t q = 0; q < kk; ++q) zscale[(size_t)(z0 + q)] = dsrc[q];
      }
    }
    const bool is32 = cls == 2 || d->hi32;
    const int64_t es = is32 ? 4 : 8;
    const int64_t rg = (int64_t)rows.size();
    // m1-single: z = Vt32 . x32 accumulated in FP32 in SGEMV's order over the
    // whole cluster width (s1_exact_kernel: one thread per rank row, no
    // column chunks), stored in chunk layout
    const bool exact1 = is32 && pipe == P_M1S && !chain_order;
    const int64_t rows_cap = exact1 ? kS1ExactRows : s1_rows;
    const int64_t pieces = (rg + rows_cap - 1) / rows_cap;
    for (int64_t pc = 0; pc < pieces; ++pc) {
      const int64_t r0 = rg * pc / pieces, r1 = rg * (pc + 1) / pieces, R = r1 - r0;
      const int64_t rp = round_up(R, is32 ? 4 : 2);
      // (exact: OpenBLAS's own 4096-column blocks, one CTA each, added in order)
      int64_t C = exact1 ? 4 * (int64_t)kSgemvBlock : std::max<int64_t>(1, s1_target / (rp * es));
      const int64_t nch = (ncol + C - 1) / C;
      if (!exact1) C = (ncol + nch - 1) / nch;
      const int32_t red = nch > 1 ? n_red++ : -1;
      const int32_t poff = nch > 1 ? (int32_t)part_len : -1;
      if (nch > 1) part_len += nch * R;
      const auto& first = rows[(size_t)r0];
      const int64_t zrow0 = (cls == 1 ? zoff_hi : zoff_lo)[(size_t)first.first] + first.second;
      for (int64_t ch = 0; ch < nch; ++ch) {
        const int64_t c0 = ch * C, w = std::min(C, ncol - c0);
        Seg s{};
        s.row0 = (int32_t)zrow0;
        s.R = (int32_t)R;
        s.run0 = (int32_t)runs.size();
        s.red = red;
        s.chunk = (int32_t)ch;
        s.nchunks = (int32_t)nch;
        s.part_off = poff;
        s.gtab = -1;
        Run r{};
        r.src = (int32_t)(cs + c0);
        r.width = (int32_t)w;
        r.col0 = 0;
        r.flags = (src_round ? RUN_ROUND : 0) | ((is32 && pipe == P_M1S) ? (RUN_ACC32 | (exact1 ? RUN_CHUNK : 0)) : 0);
        runs.push_back(r);
        run_block.push_back(-1);
        if (is32) {
          s.off32 = off32;
          s.W32 = (int32_t)w;
          s.nrun32 = 1;
          off32 += w * rp;
        } else {
          s.off64 = off64;
          s.W64 = (int32_t)w;
          s.nrun64 = 1;
          off64 += w * rp;
        }
        s1_bytes += R * w * es;
        fills.push_back({(int32_t)seg1.size(), cls, cs, ncol, c0, &rows, (int32_t)r0});
        seg1.push_back(s);
      }
    }
  }
  if (part_len > INT32_MAX) {
    set_error("too many stage-1 partials");
    return HMX_ERR_ARG;
  }

  // ---- stage-2 items per row segment, in partition order
  std::vector<std::vector<ItemRef>> items64((size_t)nseg2), items32((size_t)nseg2);
  for (int32_t k : blocks) {
    const int64_t* t = d->table + 5 * k;
    const int64_t lo = std::max(t[0], rb), hi = std::min(t[1], re);
    int64_t s = std::upper_bound(seg_start.begin(), seg_start.begin() + nseg2, lo) - seg_start.begin() - 1;
    for (; s < nseg2 && seg_start[(size_t)s] < hi; ++s) {
      if (d->kind[k] == 0) {
        (d->a32 ? items32 : items64)[(size_t)s].push_back({k, 0});
      } else {
        if (d->khi[k] > 0) (d->hi32 ? items32 : items64)[(size_t)s].push_back({k, 1});
        if (has_lo && d->klo[k] > 0) items32[(size_t)s].push_back({k, 2});
      }
    }
  }
  auto item_width = [&](const ItemRef& it) -> int64_t {
    const int64_t* t = d->table + 5 * it.block;
    return it.cls == 0 ? t[3] - t[2] : it.cls == 1 ? d->khi[it.block] : d->klo[it.block];
  };
  // cost of an FP64-accumulated (widened) column relative to an FP32-chain
  // column in a mixed FP32 part (A/B on config 4 with the warp-aligned split:
  // m1-mixed best at 0.8-1.0, m2-single at 1/1.0-1/1.2)
  const char* aw_env = std::getenv("HMX_ACC64_WEIGHT");
  // (SGEMV-order plans: 2.0 and 4 columns per chain item -- config 4 is flat between
  // 1.0-2.5 / 4-12, config 5's m1-mixed stage 2 takes 3.98 ms at 1.4 / 8, 3.84 at 2.0 / 4
  // and 3.66 at 3.0 / 2, where config 4's m2-single loses 8 %)
  const double acc64_weight = aw_env ? std::atof(aw_env) : (chain_order ? 0.85 : 2.0);
  const char* al_env = std::getenv("HMX_ALL_LANES");
  const bool all_lanes = al_env ? std::atoi(al_env) != 0 : false;
  const char* ss_env = std::getenv("HMX_STREAM_SMALL");
  const bool stream_small = ss_env ? std::atoi(ss_env) != 0 : true;
  const char* sw_env = std::getenv("HMX_STREAM_WEIGHT");
  // (a streamed chain column against a lane-tree column; measured at config 5,
  // where most items are streamed: 1.0: 4.33 ms, 2.5: 3.98, 3.5: 3.94, 5: 4.08; flat at config 4)
  const double stream_weight = sw_env ? std::atof(sw_env) : 3.0;
  const char* s4_env = std::getenv("HMX_S1_EXACT4_BELOW");
  const int64_t s1_exact4_below = s4_env ? std::atoll(s4_env) : int64_t(800) << 20;
  const char* ic_env = std::getenv("HMX_CHAIN_ITEM_COST");
  const int64_t chain_item_cost = ic_env ? std::atoll(ic_env) : 4;
  const bool dense_single = pipe == P_M1S || pipe == P_M2S;  // A32 . x32 in FP32
  const bool u_acc32 = pipe == P_M1S || pipe == P_M1M;       // U32 . z32 in FP32
  bool any_acc32 = false, any_acc64_in32 = false;
  // FP32 part: FP64-accumulated items first, then FP32-accumulated ones, so
  // the kernel switches accumulation mode once per part instead of testing
  // every column (the switch column is stored after the group table)
  auto item_acc32 = [&](const ItemRef& it) {
    return it.cls == 0 ? dense_single : (it.cls == 1 && u_acc32);
  };
  for (auto& lst : items32)
    std::stable_sort(lst.begin(), lst.end(), [&](const ItemRef& a, const ItemRef& b) {
      return (int)item_acc32(a) < (int)item_acc32(b);
    });

  // Thread groups of a stage-2 FP32 part that holds FP32-accumulated
  // (chain) items, i.e. the schemes whose reference GEMV accumulates in FP32
  // (matvec.py:57, :73).  Each (row, chain item) stays ONE FP32 chain, so a
  // chain item is never split between groups: chain items are dealt to
  // groups by LPT (widest first, to the least-loaded group) and laid out
  // group by group (partition order inside a group), which balances far
  // better than cutting the partition-order stream at item boundaries (a
  // 40-column dense item against ~66-column group shares).  FP64-accumulated
  // (widened) items come first and are cut anywhere.  When the part has
  // both kinds, the two run different loops, so each kind gets its own
  // warps: threads [0, wb) for the widened columns, [wb, 256) for the
  // chains, wb (a multiple of 32) minimising the larger estimated group
  // cost, a widened column costing acc64_weight of a chain column.
  struct FP32Groups {
    std::vector<int64_t> cuts;  // G + 1 column boundaries; empty: no group table
    int64_t c32 = 0;            // first chain column
    int64_t wb = 0;
    int64_t cw = 0;             // chain warps (SGEMV-order plans)
  };
  auto lpt = [](const std::vector<int64_t>& w, int64_t G, std::vector<int32_t>* owner) {
    std::vector<int32_t> order(w.size());
    for (size_t i = 0; i < w.size(); ++i) order[i] = (int32_t)i;
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return w[(size_t)a] > w[(size_t)b]; });
    std::vector<int64_t> load((size_t)G, 0);
    if (owner) owner->assign(w.size(), 0);
    for (int32_t i : order) {
      const size_t g = (size_t)(std::min_element(load.begin(), load.end()) - load.begin());
      load[g] += w[(size_t)i];
      if (owner) (*owner)[(size_t)i] = (int32_t)g;
    }
    return *std::max_element(load.begin(), load.end());
  };
  // row-kernel bounds of block k's rows seen from a segment starting at row0
  // (7-bit segment-relative bounds e16 | e8 << 7 | e4 << 14 | e2 << 21, hmx_internal.cuh)
  auto kind_bits = [&](int64_t k, int64_t row0) {
    const int64_t* t = d->table + 5 * k;
    const int64_t mb = t[1] - t[0], d0 = row0 - t[0];  // block row of segment row 0
    const int64_t a16 = mb & ~int64_t(15), b8 = a16 + (mb & 8), c4 = b8 + (mb & 4);
    const int64_t c2 = c4 + ((mb & 3) >= 2 ? 2 : 0);
    auto rel = [&](int64_t bound) { return (uint32_t)std::min<int64_t>(std::max<int64_t>(bound - d0, 0), 127); };
    return rel(a16) | rel(b8) << 7 | rel(c4) << 14 | rel(c2) << 21;
  };
  // An FP32-accumulated item whose SGEMV order is ONE forward FMA chain per
  // row: widths 1, 3, 5, 6, 7 when every row of the segment is in the 16- or
  // 8-row kernel, width 2 in the 16-row kernel (hmx_kernels.cu chain_item).
  // That is exactly what the streaming threads' FP32 chain computes (one chain
  // per (row, item), started at the item's first column), so SGEMV-order
  // plans leave such items to the streaming warps, at no per-item cost.
  auto stream_exact = [&](const ItemRef& it, int64_t row0, int64_t R) {
    const int64_t n = item_width(it);
    if (!(n <= 3 || (n >= 5 && n <= 7))) return false;
    const uint32_t bits = kind_bits(it.block, row0);
    const int64_t e16 = bits & 127, e8 = (bits >> 7) & 127;
    return n == 2 ? e16 >= R : e8 >= R;
  };
  auto plan_fp32_groups = [&](std::vector<ItemRef>& lst, int64_t R, int64_t row0) {
    FP32Groups fg;
    if (!(dense_single || u_acc32) || lst.empty()) return fg;
    int64_t W = 0;
    for (const ItemRef& it : lst) W += item_width(it);
    if (W > kSegWMax) return fg;  // tiled part: no group table
    if (!chain_order && (int64_t)lst.size() > kChainRunsMax) return fg;  // (the chain lanes' meta table)
    // widened groups: 4 rows per thread (tpg threads per group)
    const int64_t rp = round_up(R, 4), tpg = rp / 4, G = kSegThreads / tpg;
    // chain groups: HMX_PLAN_FP32_CHAIN plans: tpg threads each, anywhere; SGEMV-order
    // plans: slots of tpg lanes inside a warp, 32 / tpg (<= 8) slots per warp
    const int64_t nslot = std::min<int64_t>(32 / tpg, 8);
    auto chain_groups = [&](int64_t threads) { return chain_order ? threads / tpg : threads / 32 * nslot; };
    const int64_t Gc = chain_groups(kSegThreads);
    size_t nA = 0;
    while (nA < lst.size() && !item_acc32(lst[nA])) ++nA;
    int64_t colsA = 0;
    for (size_t i = 0; i < nA; ++i) colsA += item_width(lst[i]);
    // wB: chain item widths; cB: their estimated costs in columns (SGEMV-order
    // plans: a fixed per-item overhead -- accumulator set-up, the lane tree,
    // FIFO bookkeeping -- measured at about kChainItemCost columns)
    std::vector<int64_t> wB, cB;
    for (size_t i = nA; i < lst.size(); ++i) {
      wB.push_back(item_width(lst[i]));
      cB.push_back(wB.back() + (chain_order ? 0 : chain_item_cost));
    }
    fg.c32 = colsA;
    int64_t gA = 0, gB = Gc;
    if (all_lanes && !chain_order && nA > 0 && !wB.empty()) {
      // SGEMV-order plans, all-lanes mode: no widened warps.  Every item of the
      // part -- widened ones too (FP64 accumulation on the same lanes) -- is
      // dealt to the lane slots of all eight warps by LPT on its estimated
      // cost, so no warp waits for the other kind.  A slot's widened items come
      // first, then its chain items widest first.
      std::vector<int64_t> cost(lst.size());
      for (size_t i = 0; i < lst.size(); ++i)
        cost[i] = i < nA ? (int64_t)std::ceil(acc64_weight * (double)item_width(lst[i])) + 2
                         : item_width(lst[i]) + chain_item_cost;
      std::vector<int32_t> owner;
      lpt(cost, Gc, &owner);
      const std::vector<ItemRef> all(lst.begin(), lst.end());
      fg.cuts.push_back(0);
      size_t k = 0;
      for (int64_t g = 0; g < Gc; ++g) {
        std::vector<size_t> mine;
        for (size_t i = 0; i < all.size(); ++i)
          if (owner[i] == g) mine.push_back(i);
        std::stable_sort(mine.begin(), mine.end(), [&](size_t a, size_t b) {
          if ((a < nA) != (b < nA)) return a < nA;
          return a >= nA && item_width(all[a]) > item_width(all[b]);
        });
        int64_t load = 0;
        for (size_t i : mine) {
          lst[k++] = all[i];
          load += item_width(all[i]);
        }
        fg.cuts.push_back(fg.cuts.back() + load);
      }
      fg.c32 = 0;
      fg.wb = 0;
      fg.cw = kSegThreads / 32;
      return fg;
    }
    if (!chain_order && stream_small && !wB.empty()) {
      // SGEMV-order plans: [widened | streamed chain items | lane-tree chain items].
      // Threads [0, wb): gW widened groups (even column cuts) then gS groups of
      // streamed chain items (whole items, LPT); the chain warps' slots take
      // the rest.  wb, gW and gS minimise the largest estimated group cost.
      std::vector<size_t> iS, iT;
      for (size_t i = nA; i < lst.size(); ++i) (stream_exact(lst[i], row0, R) ? iS : iT).push_back(i);
      if (!iS.empty()) {
        std::vector<int64_t> wS, cT;
        int64_t colsS = 0;
        for (size_t i : iS) {
          wS.push_back(item_width(lst[i]));
          colsS += wS.back();
        }
        for (size_t i : iT) cT.push_back(item_width(lst[i]) + chain_item_cost);
        const double ws = stream_weight;  // a streamed chain column against a lane-tree column
        double best = 1e300;
        int64_t bwb = 0, bgW = 0, bgS = 0;
        std::vector<double> tS_of((size_t)G + 1, -1.0);  // LPT makespan of the streamed items over gS groups
        for (int64_t wb = 32; wb <= kSegThreads; wb += 32) {
          const int64_t ga = wb / tpg, cw = (kSegThreads - wb) / 32;
          if (cT.empty() != (cw == 0)) continue;
          if (nA > 0 && cw > kChainWarpsMixed) continue;
          if (ga < (nA > 0 ? 2 : 1)) continue;
          const double tT = cT.empty() ? 0.0 : (double)lpt(cT, cw * nslot, nullptr);
          for (int64_t gS = 1; gS <= ga - (nA > 0 ? 1 : 0); ++gS) {
            const int64_t gW = ga - gS;
            if ((nA > 0) != (gW > 0)) continue;
            if (tS_of[(size_t)gS] < 0.0) tS_of[(size_t)gS] = (double)lpt(wS, gS, nullptr);
            const double tS = ws * tS_of[(size_t)gS];
            const double tW = nA > 0 ? acc64_weight * (double)colsA / (double)gW : 0.0;
            const double t = std::max(tT, std::max(tS, tW));
            if (t < best) {
              best = t;
              bwb = wb;
              bgW = gW;
              bgS = gS;
            }
          }
        }
        if (bwb > 0) {
          const std::vector<ItemRef> all(lst.begin(), lst.end());
          size_t k = nA;
          fg.cuts.push_back(0);
          for (int64_t q = 1; q <= bgW; ++q) fg.cuts.push_back(colsA * q / bgW);
          std::vector<int32_t> owner;
          lpt(wS, bgS, &owner);
          for (int64_t g = 0; g < bgS; ++g) {
            int64_t load = 0;
            for (size_t i = 0; i < iS.size(); ++i)
              if (owner[i] == g) {
                lst[k++] = all[iS[i]];
                load += wS[i];
              }
            fg.cuts.push_back(fg.cuts.back() + load);
          }
          const int64_t cw = (kSegThreads - bwb) / 32, gT = cw * nslot;
          if (gT > 0) {
            lpt(cT, gT, &owner);
            for (int64_t g = 0; g < gT; ++g) {
              std::vector<size_t> mine;
              for (size_t i = 0; i < iT.size(); ++i)
                if (owner[i] == g) mine.push_back(i);
              std::stable_sort(mine.begin(), mine.end(), [&](size_t a, size_t b) { return cT[a] > cT[b]; });
              int64_t load = 0;
              for (size_t i : mine) {
                lst[k++] = all[iT[i]];
                load += item_width(all[iT[i]]);
              }
              fg.cuts.push_back(fg.cuts.back() + load);
            }
          }
          fg.wb = bwb;
          fg.cw = cw;
          return fg;
        }
      }
    }
    if (nA > 0 && !wB.empty()) {
      double best = 1e300;
      for (int64_t wb = 32; wb < kSegThreads; wb += 32) {
        const int64_t ga = wb / tpg, gb = chain_groups(kSegThreads - wb);
        if (ga < 1 || gb < 1) continue;
        // (SGEMV-order plans: at most kChainWarpsMixed chain warps, so that three
        // CTAs with their column FIFOs fit an SM)
        if (!chain_order && (kSegThreads - wb) / 32 > kChainWarpsMixed) continue;
        const double t = std::max(acc64_weight * (double)colsA / (double)ga, (double)lpt(cB, gb, nullptr));
        if (t < best) {
          best = t;
          fg.wb = wb;
          gA = ga;
          gB = gb;
        }
      }
    } else if (nA > 0) {
      gA = G;
      gB = 0;
      fg.wb = kSegThreads;  // no chain threads
    }
    // widened range [0, colsA): even cuts over gA groups (or all G groups
    // when there are no chains)
    fg.cuts.push_back(0);
    for (int64_t q = 1; q <= gA; ++q) fg.cuts.push_back(colsA * q / gA);
    fg.cw = (wB.empty() || chain_order) ? 0 : (kSegThreads - fg.wb) / 32;
    if (gB > 0) {
      std::vector<int32_t> owner;
      lpt(cB, gB, &owner);
      std::vector<ItemRef> chains(lst.begin() + (ptrdiff_t)nA, lst.end());
      std::vector<int64_t> load((size_t)gB, 0);
      size_t k = nA;
      for (int64_t g = 0; g < gB; ++g) {
        // a group's items widest first (SGEMV-order plans: neighbouring items
        // of equal width share a pass of the chain warp without diverging)
        std::vector<size_t> mine;
        for (size_t i = 0; i < chains.size(); ++i)
          if (owner[i] == g) mine.push_back(i);
        if (!chain_order)
          std::stable_sort(mine.begin(), mine.end(), [&](size_t a, size_t b) { return wB[a] > wB[b]; });
        for (size_t i : mine) {
          lst[k++] = chains[i];
          load[(size_t)g] += wB[i];
        }
        fg.cuts.push_back(fg.cuts.back() + load[(size_t)g]);
      }
    }
    return fg;
  };
  int64_t chain_warps_max = 0, n_chain_fallback = 0;
  for (int64_t s = 0; s < nseg2; ++s) {
    Seg& sg = seg2[(size_t)s];
    sg.row0 = (int32_t)seg_start[(size_t)s];
    sg.R = (int32_t)(seg_start[(size_t)s + 1] - seg_start[(size_t)s]);
    sg.run0 = (int32_t)runs.size();
    sg.red = -1;
    sg.nchunks = 1;
    sg.part_off = -1;
    const FP32Groups fg = plan_fp32_groups(items32[(size_t)s], sg.R, sg.row0);  // may reorder chain items
    chain_warps_max = std::max<int64_t>(chain_warps_max, fg.cw);
    for (int part = 0; part < 2; ++part) {
      const auto& lst = part == 0 ? items64[(size_t)s] : items32[(size_t)s];
      int64_t col = 0;
      for (const ItemRef& it : lst) {
        const int64_t* t = d->table + 5 * it.block;
        Run r{};
        r.width = (int32_t)item_width(it);
        r.col0 = (int32_t)col;
        if (it.cls == 0) {
          r.src = (int32_t)t[2];
          r.flags = (part == 1 && dense_single) ? (RUN_ROUND | RUN_ACC32) : 0;
        } else {
          r.src = (int32_t)(it.cls == 1 ? zoff_hi[(size_t)it.block] : zoff_lo[(size_t)it.block]);
          r.flags = RUN_Z | ((part == 1 && it.cls == 1 && u_acc32) ? RUN_ACC32 : 0);
        }
        if (part == 1) {
          if (r.flags & RUN_ACC32) any_acc32 = true;
          else any_acc64_in32 = true;
          // parts with a group table: chain items carry the segment rows of
          // each SGEMV row kernel (sgemv_row_kind of the block's rows, as 7-bit
          // segment-relative bounds)
          if ((r.flags & RUN_ACC32) && !fg.cuts.empty() && !chain_order) {
            const uint32_t bits = kind_bits(it.block, sg.row0);
            r.flags |= (int32_t)(bits << kRunKindShift);
          }
        }
        runs.push_back(r);
        run_block.push_back(it.block);
        col += r.width;
      }
      if (part == 0) {
        sg.W64 = (int32_t)col;
        sg.nrun64 = (int32_t)lst.size();
      } else {
        sg.W32 = (int32_t)col;
        sg.nrun32 = (int32_t)lst.size();
      }
    }
    // group boundaries of the FP32 part (plan_fp32_groups): gtab[0..G] then
    // the first FP32-accumulated column; sg.chunk = wb of a warp-split part
    sg.gtab = -1;
    sg.chunk = 0;
    if (!fg.cuts.empty()) {
      sg.gtab = (int32_t)gtab.size();
      for (int64_t c : fg.cuts) gtab.push_back((int32_t)c);
      gtab.push_back((int32_t)fg.c32);
      // ... then, per cut, the index of the first run of the part starting at
      // or after it (the chain lanes' item ranges, hmx_kernels.cu)
      {
        int32_t j = 0;
        for (int64_t c : fg.cuts) {
          while (j < sg.nrun32 && runs[(size_t)(sg.run0 + sg.nrun64 + j)].col0 < c) ++j;
          gtab.push_back(j);
        }
      }
      sg.chunk = (int32_t)fg.wb;
    } else if (sg.W32 > 0 && (dense_single || u_acc32)) {
      // (a part wider than the staging tile, or with too many runs: its FP32-
      // accumulated items fall back to one FP32 chain per (row, item))
      ++n_chain_fallback;
      // wide part (tiled, no group cuts): only the first FP32-accumulated column
      int32_t first = sg.W32;
      for (int32_t j = 0; j < sg.nrun32; ++j) {
        const Run& r = runs[(size_t)(sg.run0 + sg.nrun64 + j)];
        if (r.flags & RUN_ACC32) {
          first = r.col0;
          break;
        }
      }
      sg.gtab = -2 - (int32_t)gtab.size();
      gtab.push_back(first);
    }
    sg.off64 = off64;
    sg.off32 = off32;
    off64 += (int64_t)sg.W64 * round_up(sg.R, 2);
    off32 += (int64_t)sg.W32 * round_up(sg.R, 4);
    s2_bytes += (int64_t)sg.R * (sg.W64 * 8 + sg.W32 * 4);
  }
  if ((int64_t)runs.size() > INT32_MAX || off64 < 0) {
    set_error("plan too large");
    return HMX_ERR_ARG;
  }
  const int f32mode2 = !any_acc32 ? F32_ALL64 : (any_acc64_in32 ? F32_MIXED : F32_ALL32);
  if (!chain_order && f32mode2 != F32_ALL64 && off64 != 0) {
    set_error("internal: FP64 part in a plan with FP32-accumulated items");  // (the SGEMV-order kernels skip it)
    return HMX_ERR_ARG;
  }

  // ---- packing of one blob unit (a stage-1 segment, or one part of a
  // stage-2 segment) into a staging window whose first element is blob
  // element w0; padding rows stay zero
  const std::vector<Seg> seg1_fill = seg1;  // fill order (seg1 is re-sorted below)
  auto pack_s1 = [&](int64_t i, double* b64, float* b32, int64_t w0) {
    const S1Fill& f = fills[(size_t)i];
    const Seg& s = seg1_fill[(size_t)f.seg];
    const bool is32 = s.W32 > 0;
    const int64_t rp = round_up(s.R, is32 ? 4 : 2);
    const int64_t w = is32 ? s.W32 : s.W64;
    const int64_t o = (is32 ? s.off32 : s.off64) - w0;
    for (int64_t t = 0; t < s.R; ++t) {
      const auto& row = (*f.rows)[(size_t)(f.r0 + t)];
      const int32_t k = row.first;
      const int64_t* tb = d->table + 5 * k;
      const int64_t m = tb[1] - tb[0];
      const int64_t kk = f.cls == 1 ? d->khi[k] : d->klo[k];
      const int64_t base = (f.cls == 1 ? d->hi_off[k] : d->lo_off[k]) + m * kk + (int64_t)row.second * f.ncol + f.c0;
      const bool src32 = f.cls == 2 || d->hi32;
      const bool chunk = (runs[(size_t)s.run0].flags & RUN_CHUNK) != 0;
      for (int64_t j = 0; j < w; ++j) {
        const int64_t e = chunk ? chunk_off((int)w, (int)rp, (int)t, (int)j) : j * rp + t;
        if (is32) b32[(size_t)(o + e)] = src32 ? d->buf32[base + j] : (float)d->buf64[base + j];
        else b64[(size_t)(o + e)] = src32 ? d->buf32[base + j] : d->buf64[base + j];
      }
    }
  };
  auto pack_s2 = [&](int64_t s, int part, double* b64, float* b32, int64_t w0) {
    const Seg& sg = seg2[(size_t)s];
    const auto& lst = part == 0 ? items64[(size_t)s] : items32[(size_t)s];
    const int64_t rp = part == 0 ? round_up(sg.R, 2) : round_up(sg.R, 4);
    const int64_t o = (part == 0 ? sg.off64 : sg.off32) - w0;
    int64_t col = 0;
    for (const ItemRef& it : lst) {
      const int64_t* t = d->table + 5 * it.block;
      const int64_t r0 = sg.row0 - t[0];
      const int64_t w = item_width(it);
      int64_t src_off;
      bool src32;
      if (it.cls == 0) {
        src_off = d->a_off[it.block];
        src32 = d->a32;
      } else if (it.cls == 1) {
        src_off = d->hi_off[it.block];
        src32 = d->hi32;
      } else {
        src_off = d->lo_off[it.block];
        src32 = true;
      }
      for (int64_t i = 0; i < sg.R; ++i) {
        const int64_t e0 = src_off + (r0 + i) * w;
        for (int64_t c = 0; c < w; ++c) {
          const int64_t dst = o + (col + c) * rp + i;  // every stage-2 item is column-major
          if (part == 0) b64[(size_t)dst] = src32 ? d->buf32[e0 + c] : d->buf64[e0 + c];
          else b32[(size_t)dst] = src32 ? d->buf32[e0 + c] : (float)d->buf64[e0 + c];
        }
      }
      col += w;
    }
  };
  // units per blob, in offset order (offsets were handed out sequentially)
  struct Unit {
    int64_t off, len;  // elements
    int32_t idx;
    int8_t stage, part;
  };
  std::vector<Unit> units[2];
  for (int64_t i = 0; i < (int64_t)fills.size(); ++i) {
    const Seg& s = seg1[(size_t)fills[(size_t)i].seg];
    const bool is32 = s.W32 > 0;
    if (is32) units[1].push_back({s.off32, (int64_t)s.W32 * round_up(s.R, 4), (int32_t)i, 1, 1});
    else units[0].push_back({s.off64, (int64_t)s.W64 * round_up(s.R, 2), (int32_t)i, 1, 0});
  }
  for (int64_t s = 0; s < nseg2; ++s) {
    const Seg& sg = seg2[(size_t)s];
    if (sg.W64) units[0].push_back({sg.off64, (int64_t)sg.W64 * round_up(sg.R, 2), (int32_t)s, 2, 0});
    if (sg.W32) units[1].push_back({sg.off32, (int64_t)sg.W32 * round_up(sg.R, 4), (int32_t)s, 2, 1});
  }
  for (auto& u : units)
    std::sort(u.begin(), u.end(), [](const Unit& a, const Unit& b) { return a.off < b.off; });
  std::vector<int32_t> perm32((size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    if (d->perm[i] < 0 || d->perm[i] >= n) {
      set_error("permutation entry out of range");
      return HMX_ERR_ARG;
    }
    perm32[(size_t)i] = (int32_t)d->perm[i];
  }
  // stage-1 CTAs in decreasing size: chunked (long) segments start first and
  // the many small ones fill the tail
  // (HMX_PLAN_LOCAL_FIRST: the segments that read only this plan's own x
  // slice first, so the multi-GPU mode can run them during the allgather)
  const bool local_first = opt && (opt->flags & HMX_PLAN_LOCAL_FIRST);
  auto s1_local = [&](const Seg& sg) {
    const Run& r = runs[(size_t)sg.run0];
    return local_first && r.src >= rb && (int64_t)r.src + r.width <= re;
  };
  std::stable_sort(seg1.begin(), seg1.end(), [&](const Seg& a, const Seg& b) {
    const bool la = s1_local(a), lb = s1_local(b);
    if (la != lb) return la;
    return (int64_t)a.R * (a.W64 * 2 + a.W32) > (int64_t)b.R * (b.W64 * 2 + b.W32);
  });
  int32_t n_seg1_local = 0;
  for (const Seg& sg : seg1) n_seg1_local += s1_local(sg) ? 1 : 0;
  // test hook: split the stage-1 launch in two at world 1 too (where every
  // segment is local), to exercise the two-stream path
  if (local_first && std::getenv("HMX_TEST_SPLIT_STAGE1")) n_seg1_local = (int32_t)seg1.size() / 2;

  DevPlan& dp = p->dp;
  dp.n = (int32_t)n;
  dp.row_begin = (int32_t)rb;
  dp.row_end = (int32_t)re;
  dp.pipe = pipe;
  auto up = [&](auto* dst, const auto& vec) -> int {
    using T = typename std::decay<decltype(vec[0])>::type;
    if (!dst) {
      set_error("cudaMalloc failed while uploading the plan (out of device memory?)");
      return HMX_ERR_CUDA;
    }
    if (!vec.empty()) HMX_CUDA(cudaMemcpy(dst, vec.data(), vec.size() * sizeof(T), cudaMemcpyHostToDevice));
    return HMX_OK;
  };
  int rc;
  Seg* d_seg1 = p->alloc<Seg>(std::max<size_t>(seg1.size(), 1));
  if ((rc = up(d_seg1, seg1))) return rc;
  Seg* d_seg2 = p->alloc<Seg>(seg2.size());
  if ((rc = up(d_seg2, seg2))) return rc;
  Run* d_runs = p->alloc<Run>(runs.size());
  if ((rc = up(d_runs, runs))) return rc;
  int32_t* d_rb = p->alloc<int32_t>(run_block.size());
  if ((rc = up(d_rb, run_block))) return rc;
  const double t_meta = secs();
  // ---- blobs: packed window by window into pinned staging buffers and
  // uploaded asynchronously, so packing overlaps the copies and the host
  // never holds a second full copy of the payload
  double* d_b64 = p->alloc<double>((size_t)std::max<int64_t>(off64, 2));
  float* d_b32 = p->alloc<float>((size_t)std::max<int64_t>(off32, 4));
  if (!d_b64 || !d_b32) {
    set_error("cudaMalloc failed while uploading the plan (out of device memory?)");
    return HMX_ERR_CUDA;
  }
  HMX_CUDA(cudaMemsetAsync(d_b64, 0, (size_t)std::max<int64_t>(off64, 2) * 8, p->stream));
  HMX_CUDA(cudaMemsetAsync(d_b32, 0, (size_t)std::max<int64_t>(off32, 4) * 4, p->stream));
  if (dsrc) {
    // payload values come from the device-resident masters (hmx_prepare.cu)
    std::vector<PackRow> prow;
    std::vector<size_t> gbase(group_rows.size());
    for (size_t g = 0; g < group_rows.size(); ++g) {
      gbase[g] = prow.size();
      for (const auto& r : group_rows[g]) prow.push_back({r.first, r.second});
    }
    std::vector<PackS1> ps1;
    ps1.reserve(fills.size());
    for (const S1Fill& f : fills) {
      const Seg& sg = seg1_fill[(size_t)f.seg];
      const bool is32 = sg.W32 > 0;
      PackS1 u{};
      u.dst = is32 ? sg.off32 : sg.off64;
      u.rows = (int64_t)gbase[(size_t)(f.rows - group_rows.data())] + f.r0;
      u.R = sg.R;
      u.rp = (int32_t)round_up(sg.R, is32 ? 4 : 2);
      u.w = is32 ? sg.W32 : sg.W64;
      u.c0 = (int32_t)f.c0;
      u.is32 = is32;
      u.cls = f.cls;
      u.chunk = (runs[(size_t)sg.run0].flags & RUN_CHUNK) ? 1 : 0;
      ps1.push_back(u);
    }
    std::vector<PackS2> ps2;
    std::vector<PackItem> pit;
    for (int64_t q = 0; q < nseg2; ++q) {
      const Seg& sg = seg2[(size_t)q];
      for (int part = 0; part < 2; ++part) {
        const auto& lst = part == 0 ? items64[(size_t)q] : items32[(size_t)q];
        if (lst.empty()) continue;
        PackS2 u{};
        u.dst = part == 0 ? sg.off64 : sg.off32;
        u.R = sg.R;
        u.rp = (int32_t)round_up(sg.R, part == 0 ? 2 : 4);
        u.row0 = sg.row0;
        u.item0 = (int32_t)pit.size();
        u.nitems = (int32_t)lst.size();
        u.is32 = part;
        for (const ItemRef& it : lst)
          pit.push_back({it.block, it.cls, (int32_t)item_width(it),
                         0});
        ps2.push_back(u);
      }
    }
    const int prc = device_pack(*dsrc, ps1, prow, ps2, pit, d_b64, d_b32, p->stream);
    if (prc != HMX_OK) return prc;
  } else {
    const int64_t kWinBytes = int64_t(64) << 20;
    int64_t max_unit = 0;
    for (int b = 0; b < 2; ++b)
      for (const Unit& u : units[b]) max_unit = std::max(max_unit, u.len * (b ? 4 : 8));
    const size_t stage_bytes = (size_t)std::max(kWinBytes, max_unit);
    constexpr int kBufs = 3;
    struct Stage {
      void* h = nullptr;
      cudaEvent_t ev = nullptr;
    } st[kBufs];
    int rc2 = HMX_OK;
    for (auto& b : st) {
      if (cudaMallocHost(&b.h, stage_bytes) != cudaSuccess || cudaEventCreateWithFlags(&b.ev, cudaEventDisableTiming) != cudaSuccess) {
        rc2 = cuda_fail(cudaGetLastError(), "pinned staging for the plan upload");
        break;
      }
    }
    int64_t win_no = 0;
    for (int b = 0; b < 2 && rc2 == HMX_OK; ++b) {
      const auto& us = units[b];
      const int64_t es = b ? 4 : 8;
      for (size_t i = 0; i < us.size() && rc2 == HMX_OK;) {
        size_t j = i + 1;
        const int64_t w0 = us[i].off;
        int64_t w1 = us[i].off + us[i].len;
        while (j < us.size() && (us[j].off + us[j].len - w0) * es <= kWinBytes) w1 = us[j].off + us[j++].len;
        Stage& sb = st[win_no++ % kBufs];
        if (cudaEventSynchronize(sb.ev) != cudaSuccess) {
          rc2 = cuda_fail(cudaGetLastError(), "plan upload");
          break;
        }
        std::memset(sb.h, 0, (size_t)((w1 - w0) * es));
        double* h64 = static_cast<double*>(sb.h);
        float* h32 = static_cast<float*>(sb.h);
        parallel_for((int64_t)(j - i), [&](int64_t q) {
          const Unit& u = us[i + (size_t)q];
          if (u.stage == 1) pack_s1(u.idx, h64, h32, w0);
          else pack_s2(u.idx, u.part, h64, h32, w0);
        });
        void* dst = b ? (void*)(d_b32 + w0) : (void*)(d_b64 + w0);
        cudaError_t e1 = cudaMemcpyAsync(dst, sb.h, (size_t)((w1 - w0) * es), cudaMemcpyHostToDevice, p->stream);
        if (e1 == cudaSuccess) e1 = cudaEventRecord(sb.ev, p->stream);
        if (e1 != cudaSuccess) rc2 = cuda_fail(e1, "plan upload");
        i = j;
      }
    }
    cudaError_t es_ = cudaStreamSynchronize(p->stream);
    if (rc2 == HMX_OK && es_ != cudaSuccess) rc2 = cuda_fail(es_, "plan upload");
    for (auto& b : st) {
      if (b.ev) cudaEventDestroy(b.ev);
      if (b.h) cudaFreeHost(b.h);
    }
    if (rc2 != HMX_OK) return rc2;
  }
  if (std::getenv("HMX_PLAN_TIMING"))
    std::fprintf(stderr,
                 "hmx_plan_create: layout %.3f s, pack+upload %.3f s (%.2f GB); stage-2 segments %lld, "
                 "chain warps <= %lld, parts without a group table (FP32 items as plain chains) %lld\n",
                 t_meta, secs() - t_meta, (off64 * 8.0 + off32 * 4.0) / 1e9, (long long)nseg2,
                 (long long)chain_warps_max, (long long)n_chain_fallback);
  double* d_zs = p->alloc<double>(zscale.size());
  if ((rc = up(d_zs, zscale))) return rc;
  uint8_t* d_zk = p->alloc<uint8_t>(zkind.size());
  if ((rc = up(d_zk, zkind))) return rc;
  int32_t* d_perm = p->alloc<int32_t>(perm32.size());
  if ((rc = up(d_perm, perm32))) return rc;
  int32_t* d_gtab = p->alloc<int32_t>(std::max<size_t>(gtab.size(), 1));
  if ((rc = up(d_gtab, gtab))) return rc;
  double* d_z = p->alloc<double>((size_t)std::max<int64_t>(Z, 1));
  double* d_part = p->alloc<double>((size_t)std::max<int64_t>(part_len, 1));
  uint32_t* d_cnt = p->alloc<uint32_t>((size_t)std::max<int32_t>(n_red, 1));
  if (!d_z || !d_part || !d_cnt) {
    set_error("cudaMalloc failed (out of device memory?)");
    return HMX_ERR_CUDA;
  }
  HMX_CUDA(cudaMemset(d_cnt, 0, (size_t)std::max<int32_t>(n_red, 1) * sizeof(uint32_t)));

  dp.seg1 = d_seg1;
  dp.seg2 = d_seg2;
  dp.n_seg1 = (int32_t)seg1.size();
  dp.n_seg1_local = n_seg1_local;
  dp.n_seg2 = (int32_t)nseg2;
  dp.runs = d_runs;
  dp.blob64 = d_b64;
  dp.blob32 = d_b32;
  dp.f32mode1 = pipe == P_M1S ? F32_ALL32 : F32_ALL64;
  dp.s1_narrow = s1_narrow ? 1 : 0;
  // m1-single stage 1 in SGEMV's order: one thread per rank row, or four (small plans)
  dp.s1_exact = (pipe == P_M1S && !chain_order) ? (s1_bytes < s1_exact4_below ? 2 : 1) : 0;
  dp.chain_exact = chain_order ? 0 : 1;
  dp.chain_warps = (int32_t)chain_warps_max;  // dynamic shared memory: one ring per chain warp
  {
    // deep FP64 pipeline when the FP64 part carries most of stage 2's bytes
    int64_t b64 = 0, b32 = 0;
    for (const Seg& a : seg2) {
      b64 += (int64_t)a.W64 * a.R * 8;
      b32 += (int64_t)a.W32 * a.R * 4;
    }
    // ... and only with several waves of row segments (4 per SM): small
    // plans prefer more resident CTAs (A/B: config 2 m3:c=3 65.0 -> 59.9 us,
    // m1-double 51.8 -> 51.0 us; config 3 neutral; config 4 keeps the deep
    // pipeline, -1.1 % / -2.4 % for m1-/m2-double)
    const bool many = nseg2 >= (int64_t)4 * 4 * sms;
    dp.s2_deep = (f32mode2 == F32_ALL64 && b64 > 0 && b64 >= b32 && many && !std::getenv("HMX_S2_NO_DEEP")) ? 1 : 0;
  }
  dp.f32mode2 = f32mode2;
  dp.zepi = pipe == P_M1D ? Z_NONE : (pipe == P_M1S || pipe == P_M1M) ? Z_ROUND32 : Z_SCALE;
  dp.zscale = d_zs;
  dp.zkind = d_zk;
  dp.z = d_z;
  dp.part = d_part;
  dp.red_count = d_cnt;
  dp.perm = d_perm;
  dp.gtab = d_gtab;
  dp.run_block = d_rb;

  // per-matvec buffers
  p->d_xin = p->alloc<double>((size_t)n);
  p->d_xp = p->alloc<double>((size_t)n);
  p->d_y = p->alloc<double>((size_t)n);
  p->d_nonfinite = p->alloc<int>(1);
  p->d_seg_dots = p->alloc<double>((size_t)(2 * nseg2));
  p->d_done = p->alloc<uint32_t>(1);
  p->d_dots = p->alloc<double>(2);
  p->d_first_bad = p->alloc<unsigned long long>(1);
  if (!p->d_xin || !p->d_xp || !p->d_y || !p->d_nonfinite || !p->d_seg_dots || !p->d_done ||
      !p->d_dots || !p->d_first_bad) {
    set_error("cudaMalloc failed (out of device memory?)");
    return HMX_ERR_CUDA;
  }
  HMX_CUDA(cudaMemset(p->d_done, 0, sizeof(uint32_t)));
  HMX_CUDA(cudaMallocHost(&p->h_flag, 4 * sizeof(int)));
  for (auto& e : p->ev) HMX_CUDA(cudaEventCreate(&e));
  HMX_CUDA(cudaEventCreateWithFlags(&p->ev_tail, cudaEventDisableTiming));

  hmx_plan_info& info = p->info;
  info.n = n;
  info.payload_bytes = payload;
  info.device_bytes = off64 * 8 + off32 * 4 +
                      (int64_t)((seg1.size() + seg2.size()) * sizeof(Seg) + runs.size() * (sizeof(Run) + 4)) +
                      (Z * 2 + part_len + 3 * n) * 8 + n * 4;
  info.s1_segments = (int64_t)seg1.size();
  info.s1_tasks = n_red;
  info.s2_segments = nseg2;
  info.s2_runs = (int64_t)runs.size();
  info.z_len = Z;
  info.stage1_bytes = s1_bytes;
  info.stage2_bytes = s2_bytes;
  info.s1_grid = (int32_t)seg1.size();
  info.s1_block = dp.s1_narrow ? kS1Threads32 : kS1Threads;
  info.s2_grid = (int32_t)nseg2;
  info.s2_block = kSegThreads;
  return HMX_OK;
}

extern "C" {

int hmx_plan_create(const hmx_matrix_desc* d, int device, const hmx_plan_options* opt,
                    hmx_plan** out) {
  if (!d || !out) {
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
  DeviceGuard guard(device);
  auto* p = new hmx_plan();
  p->device = device;
  p->n = d->n;
  p->scheme = d->scheme;
  cudaError_t e = cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete p;
    return cuda_fail(e, "cudaStreamCreate");
  }
  const int rc = plan_create_impl(d, device, opt, p, nullptr);
  if (rc != HMX_OK) {
    hmx_plan_destroy(p);
    return rc;
  }
  *out = p;
  return HMX_OK;
}

int hmx_matvec(hmx_plan* p, const double* x, double* y, int flags) {
  NvtxRange nvtx("hmx_matvec");
  if (!p || !x || !y) {
    set_error("null argument");
    return HMX_ERR_ARG;
  }
  if (p->dp.row_begin != 0 || p->dp.row_end != p->dp.n) {
    set_error("hmx_matvec needs a full-matrix plan");
    return HMX_ERR_ARG;
  }
  std::lock_guard<std::mutex> lock(p->mu);
  DeviceGuard guard(p->device);
  const int64_t n = p->n;
  const bool dev = flags & HMX_DEVICE_PTRS, permuted = flags & HMX_PERMUTED;
  cudaStream_t st = p->stream;
  HMX_CUDA(plan_enter(p, st));
  const double* src;
  if (dev) {
    src = x;
  } else {
    // pageable source: the driver's own staged copy beats memcpy into our
    // pinned buffer followed by a pinned transfer (measured on the B200 host)
    HMX_CUDA(cudaMemcpyAsync(p->d_xin, x, (size_t)n * sizeof(double), cudaMemcpyHostToDevice, st));
    src = p->d_xin;
  }
  const double* xp = src;
  if (!permuted) {
    HMX_CUDA(launch_gather_perm(src, p->dp.perm, p->d_xp, (int)n, st));
    xp = p->d_xp;
  } else if (!dev) {
    xp = p->d_xin;
  }
  HMX_CUDA(cudaMemsetAsync(p->d_nonfinite, 0, sizeof(int), st));
  S2Out out{};
  out.y = dev ? y : p->d_y;
  out.permute_out = permuted ? 0 : 1;
  out.nonfinite = p->d_nonfinite;
  int rc = enqueue_matvec(p, xp, out);
  if (rc) return rc;
  p->last_xp = xp;
  HMX_CUDA(cudaMemcpyAsync(p->h_flag, p->d_nonfinite, sizeof(int), cudaMemcpyDeviceToHost, st));
  if (!dev) HMX_CUDA(cudaMemcpyAsync(y, p->d_y, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost, st));
  HMX_CUDA(cudaStreamSynchronize(st));
  if (*p->h_flag) {
    set_error("non-finite matvec result");
    return HMX_ERR_NONFINITE;
  }
  return HMX_OK;
}

int hmx_nonfinite_block(hmx_plan* p, int64_t* block) {
  if (!p || !block) return HMX_ERR_ARG;
  std::lock_guard<std::mutex> lock(p->mu);
  DeviceGuard guard(p->device);
  if (!p->last_xp) {
    *block = -1;
    return HMX_OK;
  }
  cudaStream_t st = p->stream;
  HMX_CUDA(plan_enter(p, st));
  HMX_CUDA(cudaMemsetAsync(p->d_first_bad, 0xff, sizeof(unsigned long long), st));
  HMX_CUDA(launch_probe(p->dp, p->last_xp, p->d_first_bad, st));
  unsigned long long v = 0;
  HMX_CUDA(cudaMemcpyAsync(&v, p->d_first_bad, sizeof(v), cudaMemcpyDeviceToHost, st));
  HMX_CUDA(cudaStreamSynchronize(st));
  *block = v == ~0ull ? -1 : (int64_t)v;
  return HMX_OK;
}

int hmx_apply_local(hmx_plan* p, const double* xp, double* y, const double* w1, int yy,
                    double* dots, int* nonfinite, uint64_t stream) {
  if (!p || !xp || !y) {
    set_error("null argument");
    return HMX_ERR_ARG;
  }
  std::lock_guard<std::mutex> lock(p->mu);
  DeviceGuard guard(p->device);
  // UINT64_MAX selects the plan's own stream; any other value (including 0,
  // the legacy default stream) is used as given
  cudaStream_t st = stream == UINT64_MAX ? p->stream : reinterpret_cast<cudaStream_t>(stream);
  S2Out out{};
  out.y = y;
  out.permute_out = 0;
  out.w1 = w1;
  out.yy = yy;
  if (dots) {
    out.seg_dots = p->d_seg_dots;
    out.done = p->d_done;
    out.dots_out = dots;
  }
  out.nonfinite = nonfinite ? nonfinite : p->d_nonfinite;
  HMX_CUDA(plan_enter(p, st));
  HMX_CUDA(launch_stage1(p->dp, xp, st));
  HMX_CUDA(launch_stage2(p->dp, xp, out, st, /*pdl=*/true));
  HMX_CUDA(plan_leave(p, st));
  p->last_xp = xp;
  return HMX_OK;
}

int hmx_bench_matvec(hmx_plan* p, int warmup, int iters, int64_t flush_l2, double* out_ms) {
  if (!p || iters < 1 || !out_ms) return HMX_ERR_ARG;
  std::lock_guard<std::mutex> lock(p->mu);
  DeviceGuard guard(p->device);
  cudaStream_t st = p->stream;
  HMX_CUDA(plan_enter(p, st));
  void* flush = nullptr;
  if (flush_l2 > 0) HMX_CUDA(cudaMalloc(&flush, (size_t)flush_l2));
  S2Out out{};
  out.y = p->d_y;
  out.nonfinite = p->d_nonfinite;
  const double* xp = p->d_xp;
  for (int i = 0; i < warmup; ++i) {
    int rc = enqueue_matvec(p, xp, out);
    if (rc) return rc;
  }
  HMX_CUDA(cudaStreamSynchronize(st));
  // (1) the timed steps: `iters` matvecs back to back (stage 2 launched with
  // programmatic dependent launch, as in the solver), one event pair
  float total = 0.f;
  if (!flush) {
    HMX_CUDA(cudaEventRecord(p->ev[0], st));
    for (int i = 0; i < iters; ++i) {
      int rc = enqueue_matvec(p, xp, out);
      if (rc) return rc;
    }
    HMX_CUDA(cudaEventRecord(p->ev[1], st));
    HMX_CUDA(cudaEventSynchronize(p->ev[1]));
    cudaEventElapsedTime(&total, p->ev[0], p->ev[1]);
  }
  // (2) per-stage breakdown: events around each launch (no PDL), optional
  // L2 flush between matvecs outside the events
  double t1 = 0, t2 = 0, best = 1e30;
  const int reps = flush ? iters : std::max(3, std::min(iters, 50));
  for (int i = 0; i < reps; ++i) {
    if (flush) HMX_CUDA(cudaMemsetAsync(flush, i & 0xff, (size_t)flush_l2, st));
    HMX_CUDA(cudaEventRecord(p->ev[2], st));
    HMX_CUDA(launch_stage1(p->dp, xp, st));
    HMX_CUDA(cudaEventRecord(p->ev[3], st));
    HMX_CUDA(launch_stage2(p->dp, xp, out, st, /*pdl=*/false));
    HMX_CUDA(cudaEventRecord(p->ev[4], st));
    HMX_CUDA(cudaEventSynchronize(p->ev[4]));
    float a = 0, b = 0;
    cudaEventElapsedTime(&a, p->ev[2], p->ev[3]);
    cudaEventElapsedTime(&b, p->ev[3], p->ev[4]);
    t1 += a;
    t2 += b;
    best = std::min(best, (double)(a + b));
  }
  if (flush) cudaFree(flush);
  out_ms[0] = flush ? (t1 + t2) / reps : (double)total / iters;
  out_ms[1] = t1 / reps;
  out_ms[2] = t2 / reps;
  out_ms[3] = best;
  return HMX_OK;
}

}  // extern "C"
