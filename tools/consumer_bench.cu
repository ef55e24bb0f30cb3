// Standalone replica of the fp64 GEMM1 consumer inner loop (lanes own 3 rows of
// a 96-row x 16-column swizzled box, W broadcasts, 9 classes) on shared-memory
// data, no TMA: how close does this instruction mix get to the FP64 peak?
#include <cstdio>
#include <cuda_runtime.h>

template <int K, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 1) consumer(double *out, int stages) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int BOX = 96 * 128, NB = 4, CHUNK = 64;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < (NB * BOX + K * CHUNK * 8) / 8; i += blockDim.x)
    reinterpret_cast<double *>(smem)[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int box = (warp >> 1) % NB, c0 = (warp & 1) * 4, sw = lane & 7;
  const unsigned char *xa = smem + box * BOX + lane * 128;
  const double *wp = reinterpret_cast<const double *>(smem + NB * BOX) + (warp % 8) * 8;
  double acc0[K], acc1[K], acc2[K];
#pragma unroll
  for (int c = 0; c < K; ++c) acc0[c] = acc1[c] = acc2[c] = 0.0;
  for (int s = 0; s < stages; ++s) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int off = ((c0 + q) ^ sw) * 16;
      const double2 x0 = *reinterpret_cast<const double2 *>(xa + off);
      const double2 x1 = *reinterpret_cast<const double2 *>(xa + 32 * 128 + off);
      const double2 x2 = *reinterpret_cast<const double2 *>(xa + 64 * 128 + off);
      double2 w[K];
#pragma unroll
      for (int c = 0; c < K; ++c) w[c] = *reinterpret_cast<const double2 *>(wp + c * CHUNK + q * 2);
#pragma unroll
      for (int c = 0; c < K; ++c) {
        acc0[c] = fma(x0.x, w[c].x, acc0[c]);
        acc1[c] = fma(x1.x, w[c].x, acc1[c]);
        acc2[c] = fma(x2.x, w[c].x, acc2[c]);
      }
#pragma unroll
      for (int c = 0; c < K; ++c) {
        acc0[c] = fma(x0.y, w[c].y, acc0[c]);
        acc1[c] = fma(x1.y, w[c].y, acc1[c]);
        acc2[c] = fma(x2.y, w[c].y, acc2[c]);
      }
    }
    __syncwarp();
  }
  double t = 0;
#pragma unroll
  for (int c = 0; c < K; ++c) t += acc0[c] + acc1[c] + acc2[c];
  if (t == 1.2345) out[0] = t;
}

template <int WARPS>
void run(double *out) {
  const int stages = 2000;
  const size_t sm = 4 * 96 * 128 + 9 * 64 * 8;
  cudaFuncSetAttribute(consumer<9, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  consumer<9, WARPS><<<148, WARPS * 32, sm>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  consumer<9, WARPS><<<148, WARPS * 32, sm>>>(out, stages);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * 148 * WARPS * 32 * 216.0 * stages;
  printf("warps %2d: %.2f TFLOP/s fp64, %.3f us per stage (8-warp-equivalent)\n", WARPS,
         fl / ms / 1e9, ms * 1e3 / stages * 8 / WARPS);
}

// R rows per lane (R x 32 rows per box)
template <int K, int R>
__global__ void __launch_bounds__(256, 1) consumerR(double *out, int stages) {
  extern __shared__ __align__(1024) unsigned char smem[];
  constexpr int BOX = R * 32 * 128, NB = 4, CHUNK = 64;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < (NB * BOX + K * CHUNK * 8) / 8; i += blockDim.x)
    reinterpret_cast<double *>(smem)[i] = 1e-3 * (i % 97);
  __syncthreads();
  const int box = warp >> 1, c0 = (warp & 1) * 4, sw = lane & 7;
  const unsigned char *xa = smem + box * BOX + lane * 128;
  const double *wp = reinterpret_cast<const double *>(smem + NB * BOX) + warp * 8;
  double acc[R][K];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < K; ++c) acc[r][c] = 0.0;
  for (int s = 0; s < stages; ++s) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int off = ((c0 + q) ^ sw) * 16;
      double2 x[R];
#pragma unroll
      for (int r = 0; r < R; ++r) x[r] = *reinterpret_cast<const double2 *>(xa + r * 32 * 128 + off);
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const double2 w = *reinterpret_cast<const double2 *>(wp + c * CHUNK + q * 2);
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r][c] = fma(h ? x[r].y : x[r].x, h ? w.y : w.x, acc[r][c]);
        }
    }
    __syncwarp();
  }
  double t = 0;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < K; ++c) t += acc[r][c];
  if (t == 1.2345) out[0] = t;
}

template <int R>
void runR(double *out) {
  const int stages = 2000;
  const size_t sm = 4 * R * 32 * 128 + 9 * 64 * 8;
  cudaFuncSetAttribute(consumerR<9, R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  consumerR<9, R><<<148, 256, sm>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  consumerR<9, R><<<148, 256, sm>>>(out, stages);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * 148 * 256 * (R * 72.0) * stages;
  printf("R %d rows/lane: %.2f TFLOP/s fp64\n", R, fl / ms / 1e9);
}

int main() {
  {
    double *o;
    cudaMalloc(&o, 8);
    runR<3>(o);
    runR<4>(o);
    runR<6>(o);
  }
  double *out;
  cudaMalloc(&out, 8);
  run<8>(out);
  run<12>(out);
  run<16>(out);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
