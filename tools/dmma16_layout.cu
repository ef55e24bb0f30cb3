// Fragment layout check for mma.sync.m16n8k8.row.col.f64 (A 16x8, B 8x8, C 16x8):
// A[m][k] = 100 m + k, B[k][n] = (k == n) -> C = A[:, :8] restricted to n < 8.
// The assumed layout (lane = 4 g + t):
//   a0 (g, t), a1 (g + 8, t), a2 (g, t + 4), a3 (g + 8, t + 4)
//   b0 (k = t, n = g), b1 (k = t + 4, n = g)
//   c0 (g, 2t), c1 (g, 2t + 1), c2 (g + 8, 2t), c3 (g + 8, 2t + 1)
#include <cstdio>
__global__ void k(double *out) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a0 = 100 * g + t, a1 = 100 * (g + 8) + t, a2 = 100 * g + t + 4, a3 = 100 * (g + 8) + t + 4;
  double b0 = (t == g) ? 1.0 : 0.0, b1 = (t + 4 == g) ? 1.0 : 0.0;
  double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
               "{%8,%9}, {%0,%1,%2,%3};"
               : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
               : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  out[lane * 4 + 0] = c0;
  out[lane * 4 + 1] = c1;
  out[lane * 4 + 2] = c2;
  out[lane * 4 + 3] = c3;
}
int main() {
  double *d, h[128];
  cudaMalloc(&d, 128 * 8);
  k<<<1, 32>>>(d);
  cudaMemcpy(h, d, 128 * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int lane = 0; lane < 32; ++lane) {
    const int g = lane >> 2, t = lane & 3;
    const double want[4] = {100.0 * g + 2 * t, 100.0 * g + 2 * t + 1, 100.0 * (g + 8) + 2 * t,
                            100.0 * (g + 8) + 2 * t + 1};
    for (int i = 0; i < 4; ++i)
      if (h[lane * 4 + i] != want[i]) {
        if (bad < 8) printf("lane %d c%d = %g want %g\n", lane, i, h[lane * 4 + i], want[i]);
        ++bad;
      }
  }
  printf(bad ? "LAYOUT MISMATCH (%d)\n" : "layout ok\n", bad);
  return bad != 0;
}
