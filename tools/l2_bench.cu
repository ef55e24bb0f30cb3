// L2-resident read bandwidth: repeatedly stream a buffer that fits in L2
// (bulk TMA copies into smem, and plain 16-B loads), report GB/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1802_09113_b200/csrc/snx_pipe.cuh"
using namespace snx;

__global__ void bulk_read(const char* src, size_t bytes, int seg, int reps, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bar[4];
  if (threadIdx.x == 0) { for (int s = 0; s < 4; ++s) mbar_init(&bar[s], 1); mbar_fence_init(); }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t nseg = bytes / seg;
  int it = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t q = blockIdx.x; q < nseg; q += gridDim.x, ++it) {
      const int s = it & 3;
      if (it >= 4) mbar_wait(&bar[s], ((it >> 2) - 1) & 1);
      mbar_arrive_expect_tx(&bar[s], seg);
      bulk_g2s(smem + (size_t)s * seg, src + q * seg, seg, &bar[s]);
    }
  for (int k = (it > 4 ? it - 4 : 0); k < it; ++k) mbar_wait(&bar[k & 3], (k >> 2) & 1);
  sink[blockIdx.x] = smem[3];
}

__global__ void ldg_read(const uint4* src, size_t n, int reps, unsigned long long* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int r = 0; r < reps; ++r)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      uint4 v = __ldcg(src + i);
      acc.x ^= v.x; acc.y ^= v.y;
    }
  if (acc.x == 12345) sink[0] = acc.y;
}

int main() {
  unsigned long long* sink; cudaMalloc(&sink, 4096 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  size_t sizes[] = {32ull << 20, 60ull << 20, 96ull << 20, 1ull << 30};
  for (size_t bytes : sizes) {
    char* src; cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes);
    int reps = bytes > (256ull << 20) ? 2 : 20;
    int seg = 32768;
    cudaFuncSetAttribute(bulk_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * seg);
    bulk_read<<<148, 32, 4 * seg>>>(src, bytes, seg, 2, sink);
    cudaEventRecord(e0);
    bulk_read<<<148, 32, 4 * seg>>>(src, bytes, seg, reps, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("bulk32K %6zu MB x%2d: %8.1f GB/s\n", bytes >> 20, reps, (double)bytes * reps / ms / 1e6);
    ldg_read<<<148 * 8, 256>>>((const uint4*)src, bytes / 16, 2, sink);
    cudaEventRecord(e0);
    ldg_read<<<148 * 8, 256>>>((const uint4*)src, bytes / 16, reps, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ldg.cg  %6zu MB x%2d: %8.1f GB/s\n", bytes >> 20, reps, (double)bytes * reps / ms / 1e6);
    cudaFree(src);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
