// Host-side internals shared by the libsnx translation units.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/snx.h"

namespace snx {

// thread-local last-error message (snx_last_error)
void set_error(const char *fmt, ...);
int check_launch(const char *what);

inline size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline size_t dtype_bytes(int dtype) { return dtype == SNX_F64 ? 8 : 4; }

// Row-pass launch geometry (shared by workspace sizing and the launchers).
struct Geometry {
  int rows_per_warp;
  int warps;
  int64_t rowpass_blocks;  // blocks of the GEMM1+epilogue kernel
  int xtu_tiles;           // column tiles of the GEMM2 kernel
  int64_t splits;          // row splits of the GEMM2 kernel
  int64_t rows_per_split;
};
Geometry geometry(int dtype, int64_t nrows, int32_t P);

// Workspace carve-up (byte offsets), all 256-B aligned.
struct Workspace {
  size_t weights;     // K*P of T: weights converted to the X dtype
  size_t rowbuf;      // nrows*K of T: R / W / U per row
  size_t partial;     // splits*K*P of T: GEMM2 partials
  size_t loss_part;   // rowpass_blocks doubles
  size_t corr_part;   // rowpass_blocks uint64
  size_t dot_part;    // 4*kDotBlocks doubles (w.w, v.Hv, v.v)
  size_t counters;    // 16 uint32 (zero at rest; kernels restore zero)
  size_t total;
};
Workspace workspace_layout(int dtype, int64_t nrows, int32_t p, int32_t K);
inline int32_t padded(int32_t p) { return (p + 3) / 4 * 4; }

// vector kernels (snx_vec.cu)
int launch_prep_weights(int dtype, const double *w, const double *dir, double alpha, int K,
                        int p, int P, void *Wt, double *wsq_partials, unsigned *counter,
                        double *wsq_out, cudaStream_t st);

}  // namespace snx
