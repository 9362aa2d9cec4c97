// Streaming-read ceiling of this GPU: every byte of a large buffer read once
// with 16-byte non-allocating loads (the access pattern of the H-matvec
// streams), a trivial reduction, one write per thread.  Reports GB/s for a
// few grid shapes.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 ld_nc(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

template <int UNROLL>
__global__ void __launch_bounds__(256) read_kernel(const double2* __restrict__ a, size_t n2, double* out) {
  double s0 = 0, s1 = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (UNROLL - 1) * stride < n2; i += UNROLL * stride) {
    double2 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) v[u] = ld_nc(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      s0 += v[u].x;
      s1 += v[u].y;
    }
  }
  for (; i < n2; i += stride) {
    double2 v = ld_nc(a + i);
    s0 += v.x;
    s1 += v.y;
  }
  if (s0 + s1 == 12345.678) out[0] = s0;  // keep the loads
}

int main() {
  const size_t bytes = (size_t)8 << 30;
  const size_t n2 = bytes / 16;
  double2* a;
  double* out;
  cudaMalloc(&a, bytes);
  cudaMalloc(&out, 8);
  cudaMemset(a, 0, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int per_sm : {4, 8}) {
    const int grid = sms * per_sm;
    for (int rep = 0; rep < 2; ++rep) {
      read_kernel<8><<<grid, 256>>>(a, n2, out);
      cudaEventRecord(e0);
      const int iters = 20;
      for (int k = 0; k < iters; ++k) read_kernel<8><<<grid, 256>>>(a, n2, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("read-only stream: %d CTAs x 256 threads, 8 x 16 B in flight per thread: %.1f GB/s\n",
                      grid, bytes * (double)iters / (ms * 1e6));
    }
  }
  return 0;
}
