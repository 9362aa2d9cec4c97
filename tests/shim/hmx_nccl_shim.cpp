// TEST INFRASTRUCTURE: a host-shared-memory stand-in for the nine NCCL calls
// libhmx_gpu's multi-GPU mode resolves at run time (hmx_solver.cu,
// nccl_api(); selected with HMX_NCCL_LIB).  It lets the production C++ path
// -- hmx_dist_matvec / hmx_bicgstab_dist with their grouped send/recv
// allgather, the side-stream local-first stage 1 and the allreduce sequence
// -- run with world > 1 as separate processes on ONE GPU, for correctness
// (tests/test_gpu_dist_shim.py).  It is not a transport and never timed.
//
// Semantics: every operation is blocking on the host.  It first synchronises
// the caller's stream (so the device data it reads or overwrites is settled),
// then moves bytes through a shared file mapping (/tmp, sparse) named by the
// unique id: one single-slot mailbox per ordered rank pair for send/recv, one slot
// per rank for allreduce (reduced in rank order on the host).  Grouped calls
// are queued and run at ncclGroupEnd: sends, then receives, then allreduces.
// No kernel ever waits on another process's kernel.
#ifdef HMX_SHIM_HOST_ONLY
// CPU build for the protocol test (tests/test_abi.py): buffers are host memory
#include <cstring>
typedef void* cudaStream_t;
typedef int cudaError_t;
enum { cudaSuccess = 0, cudaMemcpyDeviceToHost = 2, cudaMemcpyHostToDevice = 1 };
static inline cudaError_t cudaStreamSynchronize(cudaStream_t) { return cudaSuccess; }
static inline cudaError_t cudaMemcpy(void* d, const void* s, size_t n, int) {
  std::memcpy(d, s, n);
  return cudaSuccess;
}
static inline cudaError_t cudaMemcpyAsync(void* d, const void* s, size_t n, int k, cudaStream_t) {
  return cudaMemcpy(d, s, n, k);
}
#else
#include <cuda_runtime.h>
#endif
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <random>
#include <string>
#include <vector>

extern "C" {
typedef int ncclResult_t;            // ncclSuccess = 0
typedef struct ShimComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclDataType_t;          // nccl.h: ncclInt32 = 2, ncclFloat64 = 8
typedef int ncclRedOp_t;             // nccl.h: ncclSum = 0, ncclMax = 2
}

namespace {

constexpr int kInternalError = 3, kInvalidArgument = 4, kSystemError = 2;
constexpr int kMaxWorld = 8;
constexpr size_t kChanBytes = size_t(8) << 20;  // one message: <= 8 MB (N <= 1M doubles)
constexpr size_t kArBytes = 4096;                // allreduce payload: <= 512 doubles

struct Chan {
  std::atomic<uint64_t> written, read;
  uint64_t bytes;
  alignas(64) unsigned char data[kChanBytes];
};
struct ArSlot {
  std::atomic<uint64_t> seq, done;
  uint64_t bytes;
  alignas(64) unsigned char data[kArBytes];
};
struct Shm {
  std::atomic<int> attached;
  int world;
  ArSlot ar[kMaxWorld];
  Chan chan[kMaxWorld * kMaxWorld];  // [src * world + dst]
};

struct Op {
  int kind;  // 0 send, 1 recv, 2 allreduce
  const void* sbuf;
  void* rbuf;
  size_t count;
  int type, op, peer;
  cudaStream_t st;
};

size_t type_size(int t) { return t == 8 ? 8 : t == 2 ? 4 : 0; }

// HMX_SHIM_TRACE=1: one stderr line per operation; a wait longer than
// HMX_SHIM_WAIT_S (default 120 s) prints what it waited for and aborts
bool trace() {
  static const bool t = std::getenv("HMX_SHIM_TRACE") != nullptr;
  return t;
}
double wait_limit() {
  static const double w = std::getenv("HMX_SHIM_WAIT_S") ? std::atof(std::getenv("HMX_SHIM_WAIT_S")) : 120.0;
  return w;
}
thread_local const char* g_waiting = "";
thread_local timespec g_t0;
void spin(int& n) {
  if (n == 0) clock_gettime(CLOCK_MONOTONIC, &g_t0);
  if (++n > 64) {
    usleep(20);
    if ((n & 1023) == 0) {
      timespec t;
      clock_gettime(CLOCK_MONOTONIC, &t);
      if ((double)(t.tv_sec - g_t0.tv_sec) + 1e-9 * (double)(t.tv_nsec - g_t0.tv_nsec) > wait_limit()) {
        std::fprintf(stderr, "hmx_nccl_shim: pid %d stuck waiting for %s\n", (int)getpid(), g_waiting);
        std::fflush(stderr);
        std::abort();
      }
    }
  } else {
    sched_yield();
  }
}

thread_local int g_group = 0;
thread_local std::vector<Op> g_ops;

}  // namespace

struct ShimComm {
  Shm* shm = nullptr;
  size_t len = 0;
  int world = 0, rank = 0;
  std::string name;
  uint64_t sent[kMaxWorld] = {}, recvd[kMaxWorld] = {}, rounds = 0;
};

namespace {

Chan& chan(ShimComm* c, int src, int dst) { return c->shm->chan[src * c->world + dst]; }

// Host -> device on the operation's stream, complete when this returns (a
// plain cudaMemcpy from pageable memory can return before its DMA lands, and
// the library's kernels run on non-blocking streams that do not order after
// the legacy stream).
cudaError_t h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
  return e == cudaSuccess ? cudaStreamSynchronize(st) : e;
}

ncclResult_t do_send(ShimComm* c, const Op& o) {
  const size_t bytes = o.count * type_size(o.type);
  if (bytes > kChanBytes || o.peer < 0 || o.peer >= c->world) return kInvalidArgument;
  if (cudaStreamSynchronize(o.st) != cudaSuccess) return kInternalError;
  Chan& ch = chan(c, c->rank, o.peer);
  int n = 0;
  g_waiting = "a send slot to be consumed";
  if (trace()) std::fprintf(stderr, "shim r%d send #%llu to %d: %zu B\n", c->rank, (unsigned long long)c->sent[o.peer] + 1, o.peer, bytes);
  while (ch.read.load(std::memory_order_acquire) != ch.written.load(std::memory_order_acquire)) spin(n);
  if (cudaMemcpy(ch.data, o.sbuf, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return kInternalError;
  ch.bytes = bytes;
  ch.written.store(++c->sent[o.peer], std::memory_order_release);
  return 0;
}

ncclResult_t do_recv(ShimComm* c, const Op& o) {
  const size_t bytes = o.count * type_size(o.type);
  if (o.peer < 0 || o.peer >= c->world) return kInvalidArgument;
  if (cudaStreamSynchronize(o.st) != cudaSuccess) return kInternalError;
  Chan& ch = chan(c, o.peer, c->rank);
  const uint64_t want = ++c->recvd[o.peer];
  int n = 0;
  g_waiting = "a message";
  if (trace()) std::fprintf(stderr, "shim r%d recv #%llu from %d: %zu B\n", c->rank, (unsigned long long)want, o.peer, bytes);
  while (ch.written.load(std::memory_order_acquire) < want) spin(n);
  if (ch.bytes != bytes) return kInvalidArgument;
  if (h2d(o.rbuf, ch.data, bytes, o.st) != cudaSuccess) return kInternalError;
  ch.read.store(want, std::memory_order_release);
  return 0;
}

ncclResult_t do_allreduce(ShimComm* c, const Op& o) {
  const size_t es = type_size(o.type), bytes = o.count * es;
  if (!es || bytes > kArBytes || (o.op != 0 && o.op != 2)) return kInvalidArgument;
  if (cudaStreamSynchronize(o.st) != cudaSuccess) return kInternalError;
  const uint64_t r = ++c->rounds;
  Shm* s = c->shm;
  int n = 0;
  g_waiting = "an allreduce round";
  if (trace()) std::fprintf(stderr, "shim r%d allreduce #%llu: %zu x type %d op %d\n", c->rank, (unsigned long long)r, o.count, o.type, o.op);
  for (int q = 0; q < c->world; ++q)  // everyone has read the previous round's slots
    while (s->ar[q].done.load(std::memory_order_acquire) + 1 < r) spin(n);
  ArSlot& mine = s->ar[c->rank];
  if (cudaMemcpy(mine.data, o.sbuf, bytes, cudaMemcpyDeviceToHost) != cudaSuccess) return kInternalError;
  mine.bytes = bytes;
  mine.seq.store(r, std::memory_order_release);
  for (int q = 0; q < c->world; ++q)
    while (s->ar[q].seq.load(std::memory_order_acquire) < r) spin(n);
  std::vector<unsigned char> acc(bytes);
  std::memcpy(acc.data(), s->ar[0].data, bytes);
  for (int q = 1; q < c->world; ++q) {  // rank order: deterministic
    for (size_t i = 0; i < o.count; ++i) {
      if (o.type == 8) {
        double a, b;
        std::memcpy(&a, acc.data() + 8 * i, 8);
        std::memcpy(&b, s->ar[q].data + 8 * i, 8);
        a = o.op == 0 ? a + b : (b > a ? b : a);
        std::memcpy(acc.data() + 8 * i, &a, 8);
      } else {
        int32_t a, b;
        std::memcpy(&a, acc.data() + 4 * i, 4);
        std::memcpy(&b, s->ar[q].data + 4 * i, 4);
        a = o.op == 0 ? a + b : (b > a ? b : a);
        std::memcpy(acc.data() + 4 * i, &a, 4);
      }
    }
  }
  mine.done.store(r, std::memory_order_release);
  if (trace()) {
    for (size_t i = 0; i < o.count && i < 2; ++i) {
      if (o.type == 8) {
        double a, m;
        std::memcpy(&a, acc.data() + 8 * i, 8);
        std::memcpy(&m, mine.data + 8 * i, 8);
        std::fprintf(stderr, "shim r%d   = %.17g (mine %.17g)\n", c->rank, a, m);
      } else {
        int32_t a;
        std::memcpy(&a, acc.data() + 4 * i, 4);
        std::fprintf(stderr, "shim r%d   = %d\n", c->rank, a);
      }
    }
  }
  if (h2d(o.rbuf, acc.data(), bytes, o.st) != cudaSuccess) return kInternalError;
  return 0;
}

ncclResult_t run(ShimComm* c, const Op& o) {
  return o.kind == 0 ? do_send(c, o) : o.kind == 1 ? do_recv(c, o) : do_allreduce(c, o);
}

thread_local ShimComm* g_group_comm = nullptr;

ncclResult_t submit(ShimComm* c, const Op& o) {
  if (!c) return kInvalidArgument;
  if (g_group > 0) {  // (one communicator per process in the tests)
    g_group_comm = c;
    g_ops.push_back(o);
    return 0;
  }
  return run(c, o);
}

}  // namespace

extern "C" {

const char* ncclGetErrorString(ncclResult_t r) {
  switch (r) {
    case 0: return "no error (shim)";
    case kSystemError: return "shim: shared mapping setup failed";
    case kInternalError: return "shim: CUDA call failed";
    case kInvalidArgument: return "shim: invalid argument or message too large";
    default: return "shim: unknown error";
  }
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  std::memset(id->internal, 0, sizeof(id->internal));
  std::random_device rd;
  std::snprintf(id->internal, sizeof(id->internal), "/hmxshim_%d_%08x%08x", (int)getpid(), rd(), rd());
  return 0;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
  if (nranks < 1 || nranks > kMaxWorld || rank < 0 || rank >= nranks) return kInvalidArgument;
  auto* c = new ShimComm();
  c->world = nranks;
  c->rank = rank;
  c->name.assign(id.internal, strnlen(id.internal, sizeof(id.internal)));
  c->len = sizeof(Shm);
  c->name = "/tmp" + c->name;
  const int fd = open(c->name.c_str(), O_CREAT | O_RDWR, 0600);
  if (fd < 0 || ftruncate(fd, (off_t)c->len) != 0) {
    delete c;
    return kSystemError;
  }
  void* p = mmap(nullptr, c->len, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) {
    delete c;
    return kSystemError;
  }
  c->shm = static_cast<Shm*>(p);  // a fresh segment is zero-filled
  c->shm->attached.fetch_add(1);
  int n = 0;
  while (c->shm->attached.load() < nranks) spin(n);
  *comm = c;
  return 0;
}

ncclResult_t ncclCommDestroy(ncclComm_t c) {
  if (!c) return 0;
  const int left = c->shm->attached.fetch_sub(1) - 1;
  munmap(c->shm, c->len);
  if (left == 0) unlink(c->name.c_str());
  delete c;
  return 0;
}

ncclResult_t ncclGroupStart() {
  ++g_group;
  return 0;
}

ncclResult_t ncclGroupEnd() {
  if (g_group <= 0) return kInvalidArgument;
  if (--g_group > 0) return 0;
  std::vector<Op> ops;
  ops.swap(g_ops);
  ShimComm* c = g_group_comm;
  g_group_comm = nullptr;
  for (int kind = 0; kind < 3; ++kind)
    for (const Op& o : ops)
      if (o.kind == kind) {
        const ncclResult_t r = run(c, o);
        if (r) return r;
      }
  return 0;
}

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t type, int peer, ncclComm_t c,
                      cudaStream_t st) {
  return submit(c, Op{0, buf, nullptr, count, type, 0, peer, st});
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t type, int peer, ncclComm_t c,
                      cudaStream_t st) {
  return submit(c, Op{1, nullptr, buf, count, type, 0, peer, st});
}

ncclResult_t ncclAllReduce(const void* sbuf, void* rbuf, size_t count, ncclDataType_t type,
                           ncclRedOp_t op, ncclComm_t c, cudaStream_t st) {
  return submit(c, Op{2, sbuf, rbuf, count, type, op, -1, st});
}

}  // extern "C"
