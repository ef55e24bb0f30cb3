// FP64 throughput on B200: DFMA (CUDA cores) vs DMMA (mma.sync f64 shapes).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double *out, int iters) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 1.2345) out[0] = s;
}

__global__ void dmma_m8n8k4(double *out, int iters) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1.2345) out[0] = s;
}

__global__ void dmma_m16n8k16(double *out, int iters) {
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-6;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]), "+d"(acc[i][2]), "+d"(acc[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]),
                     "d"(a[7]), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 1.2345) out[0] = s;
}

// DMMA and DFMA interleaved in one warp: are they separate pipes?
__global__ void mixed_kernel(double *out, int iters, int nf) {
  double acc[8][2];
  double f[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) f[i] = threadIdx.x * 1e-3 + i;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  const double fb = 1.0000001, fc = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
    if (nf) {
#pragma unroll
      for (int i = 0; i < 16; ++i) f[i] = fma(f[i], fb, fc);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
#pragma unroll
  for (int i = 0; i < 16; ++i) s += f[i];
  if (s == 1.2345) out[0] = s;
}

int main() {
  double *out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 4096, blocks = 148 * 2;
    dfma_kernel<<<blocks, warps * 32>>>(out, 16);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * iters * (double)blocks * warps * 32;
    printf("DFMA   warps/CTA %2d (2 CTA/SM): %7.2f TFLOP/s\n", warps, fl / ms / 1e9);
    dmma_m8n8k4<<<blocks, warps * 32>>>(out, 16);
    cudaEventRecord(e0);
    dmma_m8n8k4<<<blocks, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 8 * 8 * 4 * 8 * iters * (double)blocks * warps;
    printf("DMMA m8n8k4   warps %2d: %7.2f TFLOP/s\n", warps, fl / ms / 1e9);
    dmma_m16n8k16<<<blocks, warps * 32>>>(out, 16);
    cudaEventRecord(e0);
    dmma_m16n8k16<<<blocks, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * 8 * 16 * 4 * iters * (double)blocks * warps;
    printf("DMMA m16n8k16 warps %2d: %7.2f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  for (int warps : {8, 12, 16}) {
    const int iters = 4096, blocks = 148;
    for (int nf : {0, 1}) {
      mixed_kernel<<<blocks, warps * 32>>>(out, 16, nf);
      cudaEventRecord(e0);
      mixed_kernel<<<blocks, warps * 32>>>(out, iters, nf);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double fm = 2.0 * 8 * 8 * 4 * 8 * iters * (double)blocks * warps;
      const double ff = nf ? 2.0 * 16 * iters * (double)blocks * warps * 32 : 0.0;
      printf("mixed warps %2d dfma %d: %7.2f us  DMMA %6.2f + DFMA %6.2f = %6.2f TFLOP/s\n", warps,
             nf, ms * 1e3, fm / ms / 1e9, ff / ms / 1e9, (fm + ff) / ms / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
