// Fixed per-kernel cost on this GPU: empty persistent kernels back to back,
// with small and large dynamic shared memory, with and without PDL.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty_kernel(int* p) { extern __shared__ int s[]; if (threadIdx.x == 0 && p[0] == 12345) s[0] = 1; }
__global__ void empty_pdl(int* p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  extern __shared__ int s[]; if (threadIdx.x == 0 && p[0] == 12345) s[0] = 1; }
int main() {
  int* p; cudaMalloc(&p, 4); cudaMemset(p, 0, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaStream_t st; cudaStreamCreate(&st);
  size_t smems[] = {0, 64 << 10, 190 << 10};
  for (size_t smem : smems) {
    cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(empty_pdl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int mode = 0; mode < 3; ++mode) {
      // mode 0: plain stream launches; 1: PDL launches; 2: CUDA graph of plain launches
      auto run = [&](int n) {
        for (int i = 0; i < n; ++i) {
          if (mode == 1) {
            cudaLaunchConfig_t cfg = {}; cfg.gridDim = 148; cfg.blockDim = 288; cfg.dynamicSmemBytes = smem; cfg.stream = st;
            cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at; cfg.numAttrs = 1; cudaLaunchKernelEx(&cfg, empty_pdl, p);
          } else empty_kernel<<<148, 288, smem, st>>>(p);
        }
      };
      float ms;
      if (mode == 2) {
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal); run(100); cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0); cudaGraphLaunch(ge, st); cudaStreamSynchronize(st);
        cudaEventRecord(e0, st); cudaGraphLaunch(ge, st); cudaEventRecord(e1, st); cudaEventSynchronize(e1);
      } else {
        run(20); cudaStreamSynchronize(st);
        cudaEventRecord(e0, st); run(100); cudaEventRecord(e1, st); cudaEventSynchronize(e1);
      }
      cudaEventElapsedTime(&ms, e0, e1);
      printf("smem %6zu mode %d (%s): %.2f us per kernel\n", smem, mode, mode == 0 ? "stream" : mode == 1 ? "pdl" : "graph", ms * 10);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
