// Unit test of the tcgen05 kind::f16 (bf16) path of snx_umma.cuh: K-major and
// MN-major (128-B swizzle) A operands, M=128 N=32 / N=16 MMAs, and the
// bf16x2 split X = X1 + X2, q = Q1 + Q2 (X1.Q1 + X1.Q2 + X2.Q1).
#include <cuda_bf16.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "snx_umma.cuh"

using namespace snx;
constexpr int M = 128, KD = 64;  // one 128-B bf16 row = 64 elements

__device__ __forceinline__ uint32_t sw128(uint32_t off) { return off ^ (((off >> 7) & 7) << 4); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(umma::smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, int phase) {
  asm volatile(
      "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}\n" ::"r"(
          umma::smem_u32(b)),
      "r"(phase));
}

// mode 0: A K-major; mode 1: A MN-major (two 64-wide MN blocks, LBO 8 KB)
__global__ void __launch_bounds__(128) t_kernel(const float* A, const float* B, float* D, int mode) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA1 = sm, *sA2 = sm + 16384, *sB = sm + 32768;  // B: 32 rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) umma::tmem_alloc(&tbase, 32);
  if (tid == 0) mbar_init(&bar, 1);
  for (int e = tid; e < M * KD; e += 128) {
    int m = e / KD, k = e % KD;
    float x = A[m * KD + k];
    __nv_bfloat16 x1 = __float2bfloat16_rn(x);
    __nv_bfloat16 x2 = __float2bfloat16_rn(x - __bfloat162float(x1));
    uint32_t off = mode == 1 ? (m / 64) * 8192 + sw128(k * 128 + (m % 64) * 2) : sw128(m * 128 + k * 2);
    *reinterpret_cast<__nv_bfloat16*>(sA1 + off) = x1;
    *reinterpret_cast<__nv_bfloat16*>(sA2 + off) = x2;
  }
  for (int e = tid; e < 16 * KD; e += 128) {
    int n = e / KD, k = e % KD;
    float q = B[n * KD + k];
    __nv_bfloat16 q1 = __float2bfloat16_rn(q);
    __nv_bfloat16 q2 = __float2bfloat16_rn(q - __bfloat162float(q1));
    *reinterpret_cast<__nv_bfloat16*>(sB + sw128(n * 128 + k * 2)) = q1;
    *reinterpret_cast<__nv_bfloat16*>(sB + sw128((16 + n) * 128 + k * 2)) = q2;
  }
  umma::fence_proxy_async_smem();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  uint32_t tm = tbase;
  if (tid == 0) {
    uint32_t id32 = umma::idesc_bf16(M, 32, mode == 1, false);
    uint32_t id16 = umma::idesc_bf16(M, 16, mode == 1, false);
    uint32_t a1 = umma::smem_u32(sA1), a2 = umma::smem_u32(sA2), b0 = umma::smem_u32(sB);
    for (int k = 0; k < KD / 16; ++k) {
      uint64_t d1, d2;
      if (mode == 1) {
        d1 = umma::desc_sw128(a1 + k * 2048, 8192, 1024);
        d2 = umma::desc_sw128(a2 + k * 2048, 8192, 1024);
      } else {
        d1 = umma::desc_k_sw128(a1 + k * 32);
        d2 = umma::desc_k_sw128(a2 + k * 32);
      }
      uint64_t bd = umma::desc_k_sw128(b0 + k * 32);
      umma::mma_bf16(tm, d1, bd, id32, k > 0);
      umma::mma_bf16(tm, d2, bd, id16, 1);
    }
    umma::commit(&bar);
  }
  mbar_wait(&bar, 0);
  umma::fence_after();
  float v0[16], v1[16];
  umma::tmem_ld16(tm + (static_cast<uint32_t>(warp * 32) << 16), v0);
  umma::tmem_ld16(tm + (static_cast<uint32_t>(warp * 32) << 16) + 16, v1);
  int row = warp * 32 + lane;
  for (int j = 0; j < 16; ++j) D[row * 16 + j] = v0[j] + v1[j];
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tm, 32);
}

int main() {
  std::vector<float> A(M * KD), B(16 * KD), D(M * 16);
  srand(3);
  for (auto& x : A) x = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
  for (auto& x : B) x = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(t_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  int fails = 0;
  for (int mode = 0; mode < 2; ++mode) {
    t_kernel<<<1, 128, 48 * 1024>>>(dA, dB, dD, mode);
    if (cudaDeviceSynchronize() != cudaSuccess) {
      printf("mode %d: CUDA error\n", mode);
      return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0, nrm = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < 16; ++n) {
        double s = 0;
        for (int k = 0; k < KD; ++k) s += (double)A[m * KD + k] * B[n * KD + k];
        err = fmax(err, fabs(D[m * 16 + n] - s));
        nrm = fmax(nrm, fabs(s));
      }
    printf("mode %d (%s): max abs err %.3e (max |D| %.2f)\n", mode, mode ? "MN-major" : "K-major", err, nrm);
    if (!(err < 1e-4 * nrm)) ++fails;
  }
  printf(fails ? "BF16 UMMA TEST FAILED\n" : "BF16 UMMA TEST PASSED\n");
  return fails;
}
