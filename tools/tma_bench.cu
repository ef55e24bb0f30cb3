// Microbenchmark: TMA bulk copy (cp.async.bulk) vs LDGSTS (cp.async 16B) throughput
// for row-segment sizes typical of the row-pass kernels.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_1802_09113_b200/csrc/snx_pipe.cuh"
using namespace snx;

__global__ void bulk_kernel(const char* src, size_t total, int seg, int per_stage, int iters, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  __syncthreads();
  const int lane = threadIdx.x;
  size_t off = ((size_t)blockIdx.x * 7919 * seg) % (total - (size_t)seg * per_stage);
  for (int it = 0; it < iters; ++it) {
    if (lane == 0) mbar_arrive_expect_tx(&bar, (unsigned)seg * per_stage);
    __syncwarp();
    for (int i = lane; i < per_stage; i += 32)
      bulk_g2s(smem + (size_t)i * seg, src + off + (size_t)i * seg * 3, seg, &bar);
    mbar_wait(&bar, it & 1);
    off = (off + (size_t)seg * per_stage * 3 * 148) % (total - (size_t)seg * per_stage * 3);
  }
  if (lane == 0) sink[blockIdx.x] = smem[5];
}

__global__ void ldgsts_kernel(const char* src, size_t total, int seg, int per_stage, int iters, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  size_t off = ((size_t)blockIdx.x * 7919 * seg) % (total - (size_t)seg * per_stage);
  const int vec_per_seg = seg / 16;
  for (int it = 0; it < iters; ++it) {
    for (int t = threadIdx.x; t < per_stage * vec_per_seg; t += blockDim.x) {
      int r = t / vec_per_seg, q = t - r * vec_per_seg;
      unsigned s = smem_u32(smem + (size_t)r * seg + q * 16);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(s), "l"(src + off + (size_t)r * seg * 3 + q * 16));
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    off = (off + (size_t)seg * per_stage * 3 * 148) % (total - (size_t)seg * per_stage * 3);
  }
  if (threadIdx.x == 0) sink[blockIdx.x] = smem[5];
}

int main() {
  size_t total = 1ull << 31;  // 2 GB source
  char* src; cudaMalloc(&src, total); cudaMemset(src, 1, total);
  unsigned long long* sink; cudaMalloc(&sink, 148 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int segs[] = {256, 512, 768, 1536, 3072, 12288};
  for (int si = 0; si < 6; ++si) {
    int seg = segs[si];
    int per_stage = (96 * 1024) / seg; if (per_stage < 1) per_stage = 1;
    int iters = 200;
    size_t smem = (size_t)seg * per_stage;
    cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(ldgsts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int w = 0; w < 2; ++w) bulk_kernel<<<148, 32, smem>>>(src, total, seg, per_stage, 20, sink);
    cudaEventRecord(e0);
    bulk_kernel<<<148, 32, smem>>>(src, total, seg, per_stage, iters, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = 148.0 * iters * per_stage * seg;
    printf("bulk   seg %6d B x %4d per stage: %8.1f GB/s  (%.1f ns per copy per SM)\n", seg, per_stage, bytes / ms / 1e6, ms * 1e6 / (iters * per_stage));
    for (int w = 0; w < 2; ++w) ldgsts_kernel<<<148, 256, smem>>>(src, total, seg, per_stage, 20, sink);
    cudaEventRecord(e0);
    ldgsts_kernel<<<148, 256, smem>>>(src, total, seg, per_stage, iters, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ldgsts seg %6d B x %4d per stage: %8.1f GB/s\n", seg, per_stage, bytes / ms / 1e6);
  }
  cudaError_t e = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(e));
  return 0;
}
