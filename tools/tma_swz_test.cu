// Which shared-memory layout does a 2-D TMA box land in for a given swizzle
// mode?  Loads a 32-col x 32-row f32 box (value = row*1000 + col) and checks
// candidate address formulas.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>

__global__ void load_box(const __grid_constant__ CUtensorMap map, float* out) {
  __shared__ __align__(1024) float sm[32 * 32];
  __shared__ uint64_t bar;
  uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(4096));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(sm)),
        "l"(&map), "r"(0), "r"(0), "r"(b)
        : "memory");
    asm volatile(
        "{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n" ::"r"(b));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = sm[i];
}

int main() {
  const int R = 64, Cn = 64;
  std::vector<float> h(R * Cn);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < Cn; ++c) h[r * Cn + c] = r * 1000 + c;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4);
  cudaMalloc(&o, 4096);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMapSwizzle modes[3] = {CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                                 CU_TENSOR_MAP_SWIZZLE_128B_ATOM_64B};
  const char* names[3] = {"128B", "128B_ATOM_32B", "128B_ATOM_64B"};
  for (int mi = 0; mi < 3; ++mi) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)Cn, (cuuint64_t)R};
    cuuint64_t strides[1] = {(cuuint64_t)Cn * 4};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, modes[mi], CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("%s: encode failed %d\n", names[mi], (int)r);
      continue;
    }
    load_box<<<1, 128>>>(map, o);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("%s: %s\n", names[mi], cudaGetErrorString(e));
      return 1;
    }
    std::vector<float> s(1024);
    cudaMemcpy(s.data(), o, 4096, cudaMemcpyDeviceToHost);
    // candidate formulas: byte offset of element (row, col)
    auto f16 = [](unsigned off) { return off ^ (((off >> 7) & 7) << 4); };
    auto f32a = [](unsigned off) { return off ^ (((off >> 7) & 3) << 5); };
    auto f32b = [](unsigned off) { return off ^ (((off >> 8) & 3) << 5); };
    auto f64a = [](unsigned off) { return off ^ (((off >> 7) & 1) << 6); };
    unsigned (*cands[4])(unsigned) = {+f16, +f32a, +f32b, +f64a};
    const char* cn[4] = {"x^(((x>>7)&7)<<4)", "x^(((x>>7)&3)<<5)", "x^(((x>>8)&3)<<5)",
                         "x^(((x>>7)&1)<<6)"};
    printf("%s: first row in smem:", names[mi]);
    for (int i = 0; i < 12; ++i) printf(" %g", s[i]);
    printf("\n  second 128B:");
    for (int i = 32; i < 44; ++i) printf(" %g", s[i]);
    printf("\n");
    for (int ci = 0; ci < 4; ++ci) {
      int bad = 0;
      for (int rr = 0; rr < 32; ++rr)
        for (int c = 0; c < 32; ++c) {
          unsigned off = cands[ci](rr * 128 + c * 4);
          if (s[off / 4] != rr * 1000 + c) ++bad;
        }
      printf("  candidate %-22s mismatches %d\n", cn[ci], bad);
    }
  }
  return 0;
}
