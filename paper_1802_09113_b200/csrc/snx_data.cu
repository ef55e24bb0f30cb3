// Dataset preparation on the device: column normalisation (the reference's
// normalize_columns, dataset.py:314-324 over DesignMatrix.column_norms /
// scale_columns, dataset.py:103-118).  X is row-major [n][ld]; a block owns a
// 256-column strip of a fixed row segment, threads walk down the rows of
// their column (coalesced 2 KB rows per step), and the per-segment partial
// sums of squares are reduced in segment order -- a fixed summation order, so
// the norms are bit-identical run to run.
#include "snx_common.cuh"
#include "snx_internal.h"

namespace snx {

constexpr int kColThreads = 256;
constexpr int kColSegments = 64;  // row segments (partials per column)

template <typename T>
__global__ void __launch_bounds__(kColThreads)
    colsq_part_kernel(const T *__restrict__ X, int64_t ldx, int64_t n, int p,
                      double *__restrict__ part) {
  const int j = blockIdx.x * kColThreads + threadIdx.x;
  const int seg = blockIdx.y;
  const int64_t per = (n + kColSegments - 1) / kColSegments;
  const int64_t r0 = seg * per, r1 = min(n, r0 + per);
  if (j >= p) return;
  double acc = 0.0;
#pragma unroll 8
  for (int64_t r = r0; r < r1; ++r) {
    const double x = (double)__ldg(X + r * ldx + j);
    acc += x * x;
  }
  part[(int64_t)seg * p + j] = acc;
}

// norms[j] = sqrt(sum_seg part[seg][j]); scale[j] = 1 / norms[j] where the
// norm is nonzero, else 1 (zero columns are left untouched, dataset.py:321-323).
__global__ void colsq_final_kernel(const double *__restrict__ part, int p,
                                   double *__restrict__ norms, double *__restrict__ scale) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= p) return;
  double s = 0.0;
  for (int seg = 0; seg < kColSegments; ++seg) s += part[(int64_t)seg * p + j];
  const double nj = sqrt(s);
  if (norms) norms[j] = nj;
  scale[j] = nj > 0.0 ? __ddiv_rn(1.0, nj) : 1.0;
}

// Y[r][j] = X[r][j] * scale[j] (numpy `A * scale`, one rounding; f32 data is
// scaled in fp64 and rounded once to f32).  Pad columns j >= p stay zero.
template <typename T>
__global__ void scale_cols_kernel(const T *__restrict__ X, int64_t ldx, int64_t n, int p,
                                  int64_t ld, const double *__restrict__ scale,
                                  T *__restrict__ Y, int64_t ldy) {
  const int64_t total = n * ld;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ld;
    const int j = (int)(i - r * ld);
    Y[r * ldy + j] = j < p ? (T)__dmul_rn((double)X[r * ldx + j], scale[j]) : T(0);
  }
}

}  // namespace snx

using namespace snx;

extern "C" {

size_t snx_colnorm_workspace_bytes(int32_t p) {
  return (size_t)kColSegments * (size_t)(p > 0 ? p : 1) * sizeof(double);
}

int snx_column_norms(int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p,
                     double *norms, double *scale, void *ws, size_t ws_bytes, void *stream) {
  if (p <= 0) return 0;
  if (ws_bytes < snx_colnorm_workspace_bytes(p)) {
    set_error("snx_column_norms: workspace of %zu bytes < %zu", ws_bytes,
              snx_colnorm_workspace_bytes(p));
    return 1;
  }
  if (ldx < p || nrows < 0) {
    set_error("snx_column_norms: bad shape (ldx %lld < p %d or nrows < 0)", (long long)ldx, p);
    return 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  double *part = static_cast<double *>(ws);
  const dim3 grid((p + kColThreads - 1) / kColThreads, kColSegments);
  if (dtype == SNX_F64)
    colsq_part_kernel<double><<<grid, kColThreads, 0, st>>>(static_cast<const double *>(X), ldx,
                                                           nrows, p, part);
  else
    colsq_part_kernel<float><<<grid, kColThreads, 0, st>>>(static_cast<const float *>(X), ldx,
                                                          nrows, p, part);
  if (check_launch("colsq_part")) return 1;
  colsq_final_kernel<<<(p + 255) / 256, 256, 0, st>>>(part, p, norms, scale);
  return check_launch("colsq_final");
}

int snx_scale_columns(int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p,
                      int64_t ld, const double *scale, void *Y, int64_t ldy, void *stream) {
  if (nrows == 0 || ld == 0) return 0;
  if (ld < p || ldx < ld || ldy < ld) {
    set_error("snx_scale_columns: need p <= ld <= ldx, ldy");
    return 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int blocks = 148 * 8;
  if (dtype == SNX_F64)
    scale_cols_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double *>(X), ldx, nrows,
                                                     p, ld, scale, static_cast<double *>(Y), ldy);
  else
    scale_cols_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float *>(X), ldx, nrows, p,
                                                    ld, scale, static_cast<float *>(Y), ldy);
  return check_launch("scale_columns");
}

}  // extern "C"
