/*
 * hmx_gpu.h - C ABI of the B200 (sm_100a) H-matrix matvec / BiCG-STAB library.
 *
 * This is the drop-in boundary for the reference package `hmx`
 * (/root/reference/pkg/src/hmx).  The reference is pure Python, so its
 * "operator API" is a set of Python signatures; each entry point below
 * replaces one of them, and paper_1911_00093_b200/_gpu.py binds them with
 * ctypes (INTEGRATION.md shows the binding):
 *
 *   hmx_plan_create     <- the payload layout fixed by prepare_scheme /
 *                          SchemeHMatrix (precision.py:169-234, :256-329);
 *                          the plan is the device-resident, flattened form
 *   hmx_matvec          <- matvec(sh, x)                  (matvec.py:138-147)
 *                          and matvec_threaded(sh, x, t)  (matvec.py:161-197)
 *   hmx_nonfinite_block <- _check_finite's block rescan   (matvec.py:123-135)
 *   hmx_true_residual   <- true_residual(h64, x, b)       (solver.py:56-65)
 *   hmx_bicgstab        <- bicgstab(sh, h64, b, cfg)      (solver.py:68-168)
 *   hmx_master_create + hmx_plan_create_prepared
 *                       <- prepare_scheme(h, scheme) run on the device from
 *                          FP64 masters uploaded once: scale_decompose,
 *                          split_indices, _cast_fp32 (precision.py:121-162,
 *                          :241-329), then the plan, with no payload upload
 *
 * All vectors are float64.  Pointers are host pointers unless a flag says
 * device.  Every call returns an hmx_status; hmx_last_error() describes the
 * last failure on the calling thread.  Calls on one plan are serialised by
 * the plan's mutex (host side) and by an event chained through every call's
 * stream (device side: work a call enqueues on a caller's stream finishes
 * before the plan's next call starts on any stream); distinct plans may be
 * used concurrently.
 */
#ifndef HMX_GPU_H
#define HMX_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HMX_OK = 0,
  HMX_ERR_ARG = 1,        /* invalid argument or inconsistent descriptor */
  HMX_ERR_CUDA = 2,       /* CUDA runtime failure (no device, OOM, ...) */
  HMX_ERR_NONFINITE = 3,  /* matvec result not finite: FloatingPointError */
  HMX_ERR_SHAPE = 4,      /* vector length does not match the matrix: ValueError */
  HMX_ERR_OVERFLOW = 5,   /* FP32 cast overflow while preparing a scheme: OverflowError */
  HMX_ERR_COMM = 6        /* NCCL failure in the multi-GPU entry points */
} hmx_status;

/* Precision schemes of the reference (precision.py:46-104). */
typedef enum {
  HMX_M1_DOUBLE = 0,
  HMX_M1_SINGLE = 1,
  HMX_M1_MIXED = 2,
  HMX_M2_DOUBLE = 3,
  HMX_M2_SINGLE = 4,
  HMX_M2_MIXED = 5,
  HMX_M3 = 6 /* m3:c=<int>; the split is already applied in the payloads */
} hmx_scheme;

/*
 * Host-side packed payloads of one prepared scheme (python: PackedScheme).
 * Block k covers rows [table[5k], table[5k+1]) and columns
 * [table[5k+2], table[5k+3]) of the permuted index space.
 *   kind[k] == 0  dense: m x n row-major at a_off[k] in buf32 (a32) or buf64
 *   kind[k] == 1  low rank:
 *       FP64 class ("hi"): U m x khi then Vt khi x n, row-major, at hi_off[k]
 *                          in buf32 (hi32) or buf64; diagonal d_hi (buf64) at
 *                          dhi_off[k], or -1 for Method 1 (no diagonal)
 *       FP32 class ("lo", Method 3 only): U m x klo then Vt klo x n at
 *                          lo_off[k] in buf32; d_lo at dlo_off[k] in buf64
 * perm[i] is the original index of permuted index i (partition.py:66).
 */
typedef struct {
  int64_t n;
  int64_t n_blocks;
  int32_t scheme; /* hmx_scheme */
  int32_t a32;
  int32_t hi32;
  int32_t reserved;
  const int64_t* perm;
  const int64_t* table;
  const int32_t* kind;
  const int64_t* a_off;
  const int64_t* hi_off;
  const int64_t* khi;
  const int64_t* dhi_off;
  const int64_t* lo_off;
  const int64_t* klo;
  const int64_t* dlo_off;
  const double* buf64;
  int64_t n64;
  const float* buf32;
  int64_t n32;
} hmx_matrix_desc;

/* Optional row restriction (multi-GPU row partition): the plan computes only
 * rows [row_begin, row_end) of y.  Pass NULL options for the full matrix. */
typedef struct {
  int64_t row_begin;
  int64_t row_end;
  int32_t s1_chunk_bytes; /* stage-1 column-chunk target; 0 = adaptive (64-256 KB) */
  int32_t flags;          /* HMX_PLAN_* bits, 0 = none */
} hmx_plan_options;

/* hmx_plan_options.flags: order the stage-1 work so the part that reads
 * only x[row_begin, row_end) -- this rank's own slice of the iterate in the
 * multi-GPU mode -- can run while the allgather brings the other slices
 * (hmx_dist_matvec, hmx_bicgstab_dist). */
#define HMX_PLAN_LOCAL_FIRST 1

/* hmx_plan_options.flags: the FP32-accumulated products (m1-single,
 * m1-mixed U slabs, m2-single dense blocks) as ONE sequential FP32 FMA chain
 * per (row, block) -- the faster round-1 order -- instead of the default,
 * OpenBLAS SGEMV-T's own summation order (bitwise the reference's FP32
 * products). */
#define HMX_PLAN_FP32_CHAIN 2

typedef struct hmx_plan hmx_plan;

typedef struct {
  int64_t n;
  int64_t payload_bytes;   /* algorithmic matrix bytes (precision.py:332-334) */
  int64_t device_bytes;    /* device memory held by the plan */
  int64_t s1_segments;  /* stage-1 segments (one CTA each) */
  int64_t s1_tasks;     /* column-chunked stage-1 row groups (last-arriver reductions) */
  int64_t s2_segments, s2_runs, z_len;
  int64_t stage1_bytes, stage2_bytes; /* stored payload bytes read per stage */
  int32_t s1_grid, s1_block, s2_grid, s2_block;
} hmx_plan_info;

/*
 * FP64 masters of one H-matrix (python PackedMaster; reference HMatrixF64,
 * compress.py:236-253), uploaded once by hmx_master_create:
 *   kind[k] == 0  dense m x n row-major at offset[k]
 *   kind[k] == 1  low rank: U m x rank[k] then Vt rank[k] x n at offset[k]
 *   kind[k] == 2  not built (row-restricted build)
 */
typedef struct {
  int64_t n;
  int64_t n_blocks;
  const int64_t* perm;
  const int64_t* table;
  const int32_t* kind;
  const int64_t* offset;
  const int64_t* rank;
  const double* data;
  int64_t n_data;
} hmx_master_desc;

typedef struct hmx_master hmx_master;

/* What prepare_scheme reports besides the payloads (SchemeHMatrix fields). */
typedef struct {
  int64_t payload_bytes;   /* precision.py:332-334 */
  int64_t underflow_count; /* nonzero values whose FP32 cast is below FLT_MIN (precision.py:241-253) */
  int64_t overflow_block;  /* first block (partition order) whose FP32 cast overflows, else -1 */
  int64_t fp32_ranks;      /* Method 3: ranks in the FP32 class */
} hmx_prepare_info;

/* matvec flags */
#define HMX_DEVICE_PTRS 1 /* x and y are device pointers */
#define HMX_PERMUTED 2    /* x and y are in permuted (cluster-tree) order */

typedef struct {
  int32_t converged;
  int32_t iterations;
  int32_t has_true_residual;
  int32_t breakdown;        /* 0 none, 1 rho, 2 shadow projection, 3 stabilisation, 4 omega */
  double true_residual;
  double breakdown_value;
  int32_t breakdown_iteration;
  int32_t history_len;      /* entries written to `history` */
  int32_t matvecs;          /* operator applications incl. the true-residual check */
  int32_t reserved;
  double device_ms;         /* GPU time of the solve (CUDA events) */
} hmx_solve_report;

const char* hmx_last_error(void);
int hmx_device_count(int* count);

int hmx_plan_create(const hmx_matrix_desc* desc, int device, const hmx_plan_options* opt,
                    hmx_plan** out);
void hmx_plan_destroy(hmx_plan* plan);
int hmx_plan_get_info(const hmx_plan* plan, hmx_plan_info* info);

/* y = A x (matvec.py:138).  Blocks until y is written.  Returns
 * HMX_ERR_NONFINITE when any y entry is not finite (y is still written). */
int hmx_matvec(hmx_plan* plan, const double* x, double* y, int flags);

/* After HMX_ERR_NONFINITE: index of the first block (partition order) whose
 * own contribution is not finite for the last x, or -1 if every block is
 * finite on its own (overflow in the summation). */
int hmx_nonfinite_block(hmx_plan* plan, int64_t* block);

/* ||b - A64 x|| / ||b|| with A64 an m1-double plan (solver.py:56-65). */
int hmx_true_residual(hmx_plan* plan64, const double* x, const double* b, double* out);

/* BiCG-STAB from x0 = 0 (solver.py:68-168).  `plan` applies the scheme's
 * operator, `plan64` (an m1-double plan of the same H-matrix, may equal
 * `plan`) confirms convergence.  history needs max_iter + 1 entries. */
int hmx_bicgstab(hmx_plan* plan, hmx_plan* plan64, const double* b, double tol, int max_iter,
                 double* x, double* history, hmx_solve_report* report);

/* Row-restricted product for the multi-GPU mode: rows [row_begin, row_end)
 * of y = A xp for a plan created with hmx_plan_options.  xp is the FULL
 * iterate in permuted order (device), y the local slice (device).  When
 * `dots` (device, 2 doubles) is non-NULL it receives [y . w1, y . y] over the
 * local rows (w1: local slice, device, may be NULL; yy: compute y . y).
 * `nonfinite` (device int, may be NULL) is set to 1 when a y entry is not
 * finite.  Enqueued on `stream` (a cudaStream_t, 0 being the legacy default
 * stream; UINT64_MAX = the plan's own stream); returns without
 * synchronising.  xp must stay valid until the product completes, and, if a
 * non-finite result is reported, until hmx_nonfinite_block has named the
 * block (the probe re-reads the most recent input). */
int hmx_apply_local(hmx_plan* plan, const double* xp, double* y, const double* w1, int yy,
                    double* dots, int* nonfinite, uint64_t stream);

/*
 * Build the FP64 masters of one H-matrix on the device (reference
 * compress.py:285-342: ACA of the admissible blocks, compress.py:79-207,
 * kernel-entry assembly of the near field, :256-282), bit-identical to the
 * host builder; the result serves hmx_plan_create_prepared like an uploaded
 * master.  Fills kinds / ranks / offsets (n_blocks each, the host builder's
 * packed layout: 0 dense m*n, 1 low rank U m x r then Vt r x n, 2 not built),
 * n_data (float64 elements) and fallbacks (ACA blocks stored dense).
 */
typedef struct {
  int64_t n;
  int64_t n_blocks;
  const double* pcent;   /* n x 3 panel centroids, permuted order */
  const double* parea;   /* n panel areas, permuted order */
  const int64_t* perm;   /* permuted -> original */
  const int64_t* table;  /* n_blocks x 5: rs, re, cs, ce, admissible */
  double tol;            /* ACA tolerance */
  int64_t max_rank;      /* 0: min(m, n) */
  int64_t row_lo;        /* build only blocks meeting rows [row_lo, row_hi) */
  int64_t row_hi;        /* 0: n */
} hmx_build_desc;

int hmx_master_build(const hmx_build_desc* desc, int device, hmx_master** out, int32_t* kinds,
                     int64_t* ranks, int64_t* offsets, int64_t* n_data, int64_t* fallbacks);
/* Copies the packed master data (n_data float64) to the host. */
int hmx_master_download(hmx_master* master, double* data);

/* Upload the FP64 masters of one H-matrix once (device-resident). */
int hmx_master_create(const hmx_master_desc* desc, int device, hmx_master** out);
void hmx_master_destroy(hmx_master* master);

/* prepare_scheme(h, scheme) on the device followed by hmx_plan_create: the
 * scaling (scale_decompose), the Method-3 split (split_indices, with the
 * threshold factor 10**(-c) passed as split_factor, computed by the caller
 * exactly as the reference does) and the FP32 casts run on the GPU, reading
 * the resident masters; no payload crosses the host link.  The plan is
 * identical to hmx_plan_create on the host-prepared payloads of the same
 * scheme.  Returns HMX_ERR_OVERFLOW (info->overflow_block set) when an FP32
 * cast overflows.  underflow_count covers the whole matrix for a full plan
 * (opt NULL). */
int hmx_plan_create_prepared(hmx_master* master, int scheme, double split_factor,
                             const hmx_plan_options* opt, hmx_plan** out, hmx_prepare_info* info);

/* Benchmark helper: `iters` device matvecs in permuted order on device
 * buffers, timed with CUDA events on the plan's stream after `warmup`
 * untimed ones.  flush_l2 > 0 writes a buffer of that many bytes between
 * timed matvecs (excluded from the timing via per-matvec events).
 * out_ms[0] = mean matvec ms, out_ms[1] = mean stage-1 ms, out_ms[2] = mean
 * stage-2 ms, out_ms[3] = min matvec ms. */
int hmx_bench_matvec(hmx_plan* plan, int warmup, int iters, int64_t flush_l2, double* out_ms);

/*
 * Multi-GPU mode: rows of the permuted index space are cut into
 * contiguous slices [cuts[k], cuts[k+1]), one per rank (one process per GPU);
 * each rank holds a row-restricted plan of its slice (hmx_plan_options).
 * Per operator application there is exactly one exchange, the allgather of
 * the iterate's slices over NCCL (grouped send/recv straight into the full
 * permuted vector, no padding); solver dot products are local partials fused
 * into the kernels plus one small NCCL allreduce per reduction point.  The
 * reference has no multi-process mode; its single-process semantics
 * (solver.py:68-168) are kept on every rank.
 */
typedef struct hmx_comm hmx_comm;

/* NCCL unique id (128 bytes) for hmx_comm_create; made on rank 0 and passed
 * to every rank by the caller (e.g. torch.distributed.broadcast_object_list). */
int hmx_comm_unique_id(uint8_t id[128]);
/* Joins the NCCL communicator (blocks until every rank has joined).  cuts has
 * world + 1 entries, cuts[0] = 0, cuts[world] = n. */
int hmx_comm_create(const uint8_t id[128], int world, int rank, int device, const int64_t* cuts,
                    hmx_comm** out);
void hmx_comm_destroy(hmx_comm* comm);

/* y_local = rows [cuts[rank], cuts[rank+1]) of A x (permuted order, device
 * pointers): x_local, this rank's slice of x, is allgathered into the full
 * iterate, then the local two-stage product runs.  Enqueued on `stream`
 * (UINT64_MAX = the plan's stream) without synchronising.  `nonfinite`
 * (device int, may be NULL) is set when a local y entry is not finite. */
int hmx_dist_matvec(hmx_plan* plan, hmx_comm* comm, const double* x_local, double* y_local,
                    int* nonfinite, uint64_t stream);

/* BiCG-STAB over row slices (solver.py:68-168, from x0 = 0), every rank
 * calling with its own slice: b_local / x_local are this rank's rows of b / x
 * in permuted order (host).  Same report on every rank; decisions are taken
 * on the device from allreduced scalars, so all ranks stop together. */
int hmx_bicgstab_dist(hmx_plan* plan, hmx_plan* plan64, hmx_comm* comm, const double* b_local,
                      double tol, int max_iter, double* x_local, double* history,
                      hmx_solve_report* report);

/* Page-locked host memory for matvec results (no reference counterpart: the
 * reference returns a fresh numpy array, matvec.py:145-147, and the Python
 * layer hands out fresh arrays backed by a pool of these buffers so the
 * device->host copy of y is one DMA instead of a driver-staged pageable
 * copy).  hmx_host_free accepts NULL. */
int hmx_host_alloc(int64_t bytes, void** out);
void hmx_host_free(void* ptr);

#ifdef __cplusplus
}
#endif

#endif /* HMX_GPU_H */
