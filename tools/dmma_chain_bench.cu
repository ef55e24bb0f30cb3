// DMMA m8n8k4.f64 latency and the V phase's accumulator-chain count: one warp
// running a dependent chain gives the latency; 8 warps per SM running the V
// phase of one 8-row block (NCH 16-column chunks, weights in registers) with
// 1, 2, 4 or 8 independent accumulator chains give its per-block time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dcb tools/dmma_chain_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

__global__ void latency(double *out, int n, long long *cyc) {
  double c[2] = {0, 0};
  const double a = 1e-3 * threadIdx.x, b = 2e-3;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) dmma(c, a, b);
  const long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  out[threadIdx.x] = c[0] + c[1];
}

constexpr int WS = 770;

template <int NCH, int CH>
__global__ void __launch_bounds__(256, 1) vphase(double *out, int reps) {
  extern __shared__ double sm[];
  double *tile = sm;
  for (int i = threadIdx.x; i < 8 * WS; i += blockDim.x) sm[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
  double qf[NCH][4];
  for (int i = 0; i < NCH; ++i)
    for (int s = 0; s < 4; ++s) qf[i][s] = 1e-3 * (i + s + lane);
  double tot = 0.0;
  const double *xrow = tile + g * WS + 4 * t;
  for (int r = 0; r < reps; ++r) {
    double c[CH][2];
#pragma unroll
    for (int k = 0; k < CH; ++k) c[k][0] = c[k][1] = 0.0;
#pragma unroll
    for (int i = 0; i < NCH; ++i) {
      const int ch = warp + 8 * i;
      const double2 xa = *reinterpret_cast<const double2 *>(xrow + 16 * ch);
      const double2 xb = *reinterpret_cast<const double2 *>(xrow + 16 * ch + 2);
      dmma(c[(4 * i + 0) % CH], xa.x, qf[i][0]);
      dmma(c[(4 * i + 1) % CH], xb.x, qf[i][2]);
      dmma(c[(4 * i + 2) % CH], xa.y, qf[i][1]);
      dmma(c[(4 * i + 3) % CH], xb.y, qf[i][3]);
    }
#pragma unroll
    for (int k = 0; k < CH; ++k) tot += c[k][0] + c[k][1];
    __syncwarp();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = tot;
}

template <int NCH, int CH>
static void run_v(double *out, int sms) {
  const int reps = 2000;
  cudaFuncSetAttribute(vphase<NCH, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * WS * 8);
  vphase<NCH, CH><<<sms, 256, 8 * WS * 8>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  vphase<NCH, CH><<<sms, 256, 8 * WS * 8>>>(out, reps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("V phase NCH=%d chains=%d: %.3f us per 8-row block (%d DMMA per warp)\n", NCH, CH,
         ms * 1e3 / reps, 4 * NCH);
}

int main() {
  double *out;
  long long *cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 8);
  latency<<<1, 32>>>(out, 100, cyc);
  latency<<<1, 32>>>(out, 4096, cyc);
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("dependent DMMA m8n8k4: %.1f cycles each\n", (double)h / 4096);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run_v<6, 1>(out, sms);
  run_v<6, 2>(out, sms);
  run_v<6, 4>(out, sms);
  run_v<6, 8>(out, sms);
  run_v<4, 2>(out, sms);
  run_v<4, 4>(out, sms);
  run_v<4, 8>(out, sms);
  return 0;
}
