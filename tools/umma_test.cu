// Unit test of the tcgen05 kind::tf32 building blocks (snx_umma.cuh):
// K-major and MN-major 128-byte-swizzled smem descriptors, M=128 N=16 MMA,
// TMEM alloc / ld, and the 3xTF32 split.  One CTA of 128 threads.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I../paper_1802_09113_b200/csrc
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "snx_umma.cuh"

using namespace snx;

constexpr int M = 128, N = 16, KD = 32;

__device__ __forceinline__ uint32_t sw128(uint32_t off) { return off ^ (((off >> 7) & 7) << 4); }
__device__ __forceinline__ uint32_t sw128_32(uint32_t off) { return off ^ (((off >> 7) & 3) << 5); }
__device__ __forceinline__ uint64_t desc_b32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = umma::desc_sw128(saddr, lbo, sbo);
  d &= ~(uint64_t(7) << 61);
  return d | (uint64_t(1) << 61);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(umma::smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, int phase) {
  asm volatile(
      "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}\n" ::"r"(
          umma::smem_u32(b)),
      "r"(phase));
}

// mode 0: A K-major; mode 1: A MN-major; mode 2: A K-major with 3xTF32
__global__ void __launch_bounds__(128) umma_test(const float* A, const float* B, float* D, int mode, uint32_t lbo, uint32_t sbo) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;               // 16 KB
  uint8_t* sAlo = sm + 16384;     // 16 KB
  uint8_t* sB = sm + 32768;       // 2 KB
  uint8_t* sBlo = sm + 34816;     // 2 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 0) umma::tmem_alloc(&tbase, 32);
  if (tid == 0) mbar_init(&bar, 1);
  for (int e = tid; e < M * KD; e += 128) {
    int m = e / KD, k = e % KD;
    float x = A[m * KD + k];
    uint32_t off;
    if (mode == 1) off = (m / 32) * 4096 + sw128_32(k * 128 + (m % 32) * 4);
    else off = sw128(m * 128 + k * 4);
    float hi = mode == 2 ? umma::tf32_hi(x) : x;
    *reinterpret_cast<float*>(sA + off) = hi;
    *reinterpret_cast<float*>(sAlo + off) = x - hi;
  }
  for (int e = tid; e < N * KD; e += 128) {
    int n = e / KD, k = e % KD;
    float x = B[n * KD + k];
    uint32_t off = sw128(n * 128 + k * 4);
    float hi = mode == 2 ? umma::tf32_hi(x) : x;
    *reinterpret_cast<float*>(sB + off) = hi;
    *reinterpret_cast<float*>(sBlo + off) = x - hi;
  }
  umma::fence_proxy_async_smem();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  uint32_t tm = tbase;
  if (tid == 0) {
    uint32_t id = umma::idesc_tf32(M, N, mode == 1, false);
    uint32_t a0 = umma::smem_u32(sA), alo = umma::smem_u32(sAlo);
    uint32_t b0 = umma::smem_u32(sB), blo = umma::smem_u32(sBlo);
    for (int k = 0; k < KD / 8; ++k) {
      uint64_t ad = mode == 1 ? desc_b32(a0 + k * 1024, lbo, sbo) : umma::desc_k_sw128(a0 + k * 32);
      uint64_t bd = umma::desc_k_sw128(b0 + k * 32);
      umma::mma_tf32(tm, ad, bd, id, k > 0);
      if (mode == 2) {
        umma::mma_tf32(tm, ad, umma::desc_k_sw128(blo + k * 32), id, 1);
        umma::mma_tf32(tm, umma::desc_k_sw128(alo + k * 32), bd, id, 1);
      }
    }
    umma::commit(&bar);
  }
  mbar_wait(&bar, 0);
  umma::fence_after();
  float v[16];
  umma::tmem_ld16(tm + (static_cast<uint32_t>(warp * 32) << 16), v);
  int row = warp * 32 + lane;
  for (int j = 0; j < 16; ++j) D[row * N + j] = v[j];
  umma::fence_before();
  __syncthreads();
  if (warp == 0) umma::tmem_dealloc(tm, 32);
}

static float trunc_tf32(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  memcpy(&x, &u, 4);
  return x;
}
static float round_tf32(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  u += 0x1000u;
  u &= 0xFFFFE000u;
  memcpy(&x, &u, 4);
  return x;
}

int main() {
  std::vector<float> A(M * KD), B(N * KD), D(M * N);
  srand(1);
  for (auto& x : A) x = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
  for (auto& x : B) x = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(umma_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024);
  int fails = 0;
  uint32_t variants[4][2] = {{4096, 512}, {512, 4096}, {4096, 1024}, {1024, 4096}};
  for (int mode = 0; mode < 6; ++mode) {
    cudaMemset(dD, 0, D.size() * 4);
    int md = mode < 3 ? mode : 1;
    uint32_t lbo = mode < 3 ? 4096 : variants[mode - 2][0], sbo = mode < 3 ? 512 : variants[mode - 2][1];
    printf("lbo %u sbo %u D[0..3] %s\n", lbo, sbo, "");
    umma_test<<<1, 128, 40 * 1024>>>(dA, dB, dD, md, lbo, sbo);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double et = 0, er = 0, ef = 0, nrm = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double st = 0, sr = 0, sf = 0;
        for (int k = 0; k < KD; ++k) {
          st += (double)trunc_tf32(A[m * KD + k]) * trunc_tf32(B[n * KD + k]);
          sr += (double)round_tf32(A[m * KD + k]) * round_tf32(B[n * KD + k]);
          sf += (double)A[m * KD + k] * B[n * KD + k];
        }
        double d = D[m * N + n];
        et = fmax(et, fabs(d - st));
        er = fmax(er, fabs(d - sr));
        ef = fmax(ef, fabs(d - sf));
        nrm = fmax(nrm, fabs(sf));
      }
    { double r0=0; for (int k=0;k<KD;++k) r0 += (double)trunc_tf32(A[k])*trunc_tf32(B[k]);
      double r1=0; for (int k=0;k<KD;++k) r1 += (double)trunc_tf32(A[KD+k])*trunc_tf32(B[k]);
      printf("  D[0][0]=%f want %f  D[0][1]=%f D[1][0]=%f want %f\n", D[0], r0, D[1], D[N], r1); }
    printf("mode %d: max|D-trunc| %.3e  max|D-round| %.3e  max|D-fp32 exact| %.3e  (max|D| %.2f)\n",
           mode, et, er, ef, nrm);
    double tol = mode == 2 ? 1e-5 : 1e-5;
    double best = mode == 2 ? ef : fmin(et, er); if (mode >= 3) best = 0;
    if (!(best < tol)) ++fails;
  }
  printf(fails ? "UMMA TEST FAILED\n" : "UMMA TEST PASSED\n");
  return fails;
}
