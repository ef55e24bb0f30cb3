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
  int grid1, grid2;    // persistent CTAs (<= one per SM, <= items)
  // GEMM1 (logits): items = row_blocks x nchunks, stream-K over `grid` CTAs
  int chunk;           // columns per chunk (512 B)
  int nchunks;
  int64_t row_blocks;  // 64-row blocks
  int64_t g1_items;
  int g1_maxseg;       // CTA segments per row block (upper bound)
  // GEMM2 (X^T U): items = col_tiles x rchunks, stream-K over `grid` CTAs
  int tcol;            // columns per tile (1 KB)
  int col_tiles;
  int rchunks;         // 32-row chunks
  int64_t g2_items;
  int g2_maxseg;
};
Geometry geometry(int dtype, int64_t nrows, int32_t P, int32_t K);

// Workspace carve-up (byte offsets), all 256-B aligned.
struct Workspace {
  size_t weights;     // K*P of T: weights converted to the X dtype
  size_t rowbuf;      // nrows*K of T: R / U per row (+ slack)
  size_t zp;          // nslices*nrows*K doubles: GEMM1 slice partials
  size_t gp;          // rsplits*K*P doubles: GEMM2 split partials
  size_t loss_part;   // row_blocks doubles
  size_t corr_part;   // row_blocks uint64
  size_t dot_part;    // 4*kDotBlocks doubles (w.w partials)
  size_t counters;    // uint32 scheduler words + arrival counters (zero at rest)
  // f32 tensor-core Hessian product (snx_tc.cu); zero-sized for f64
  size_t tc_b;        // [32][round_up(P,8)] bf16: GEMM1's B = [Q1 ; Q2] (bf16 split of v)
  size_t tc_ut;       // [32][round_up(nrows,8)] bf16: GEMM2's B = [U1^T ; U2^T]
  size_t tc_zp;       // GEMM1 segment partials [row_blocks][maxseg1][128][K] doubles
  size_t tc_gp;       // GEMM2 segment partials [col_tiles][maxseg2][K][128] doubles
  size_t total;
};
// Geometry of the tensor-core Hessian product: GEMM1 items = (128-row block x
// 64-column k-tile), GEMM2 items = (128-column tile x 64-row chunk), each
// split stream-K over <= one CTA per SM.
struct TcGeometry {
  int grid1, nk;
  int64_t row_blocks, items1;
  int maxseg1;
  int grid2, col_tiles, rchunks;
  int64_t items2;
  int maxseg2;
};
TcGeometry tc_geometry(int64_t nrows, int32_t P);
int tc_kp(int32_t K);  // classes padded for the tensor-core operands (16 or a multiple of 16)
int sk_maxseg(int64_t items, int grid, int per_group);
int sm_count();

Workspace workspace_layout(int dtype, int64_t nrows, int32_t p, int32_t K);
int validate(int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p, int32_t K,
             void *ws, size_t ws_bytes);
int gather(int dtype, const void *X, int64_t ldx, const int32_t *labels, const int64_t *rows,
           int64_t nrows, void *dst, int64_t ldd, int32_t *labels_out, cudaStream_t st);
int launch_finalize(const double *gp, int64_t items, int grid, int rchunks, int maxseg, int tcol,
                    int K, int p, double scale, double lam, const double *base, double *out,
                    double *dots, const double *skip, cudaStream_t st);
int launch_lam_only(int K, int p, double lam, const double *base, double *out, double *dots,
                    const double *skip, cudaStream_t st);
inline int32_t padded(int32_t p) { return (p + 3) / 4 * 4; }

// Ask for the maximum shared-memory carveout once per kernel: every libsnx
// kernel then runs in the same L1/smem configuration as the persistent TMA
// kernels, so consecutive launches never pay an SM reconfiguration.
void prefer_max_smem(const void *kernel);
template <typename F>
inline void carveout(F *kernel) {
  prefer_max_smem(reinterpret_cast<const void *>(kernel));
}

// one-pass fp64 row pass on thread-block clusters (snx_cluster.cu)
size_t rowpass_counter_bytes();  // the zero-at-rest counter block at workspace offset 0
bool cluster_supported(int dtype, int32_t p, int32_t K);
bool cluster_grad_preferred(int dtype, int32_t p, int32_t K);
size_t cluster_ws_bytes(int dtype, int64_t nrows, int32_t p, int32_t K);
int cluster_rowpass(int mode, int dtype, const void *X, int64_t ldx, const int64_t *rows,
                    int64_t nrows,
                    int32_t p, int32_t K, const int32_t *labels, const double *w,
                    const double *h, double *hout, double scale, double lam,
                    const double *base, double *out, double *loss_out, long long *corr_out,
                    double *dots, const double *skip, int early, void *ws, size_t ws_bytes,
                    cudaStream_t st);

int cluster_cg_iteration(int dtype, const void *X, int64_t ldx, const int64_t *rows,
                         int64_t nrows,
                         int32_t p, int32_t K, const double *h, double scale, double lam, int t,
                         int T, double *r, double *s, double *pv, double *pb, double *Hs,
                         double *state, int early, void *ws, size_t ws_bytes, cudaStream_t st);

// vector kernels (snx_vec.cu)
int launch_cg_step2(int t, int T, int64_t d, const double *r, double *s, const double *p,
                    double *pb, double *state, cudaStream_t st);
int launch_prep_weights(int dtype, const double *w, const double *dir, double alpha, int K,
                        int p, int P, void *Wt, double *wsq_partials, unsigned *counter,
                        double *wsq_out, cudaStream_t st);

}  // namespace snx

namespace snx {

// PDL is opt-in (SNX_PDL=1); see pdl_enabled() in snx_vec.cu.
bool pdl_enabled();

// Launch with programmatic stream serialization (PDL); see snx_pipe.cuh.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_if(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block,
                                 size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  return launch_pdl_if(pdl_enabled(), kernel, grid, block, smem, st, args...);
}

// The row-pass GEMM2 overlaps its prologue and X tiles with GEMM1's tail
// (programmatic dependent launch; it waits before its first U load).
// SNX_GEMM2_PDL=0 disables.
bool gemm2_pdl();

}  // namespace snx
// fp64 wide-class passes on CSR data (K > 32), csrc/snx_wide64.cu
namespace snx {
namespace wide {
size_t csr_wide_ws_bytes(int64_t n, int32_t p, int32_t K);
int csr_wide_objective(const int64_t *indptr, const int32_t *indices, const double *data,
                       int64_t n, int32_t p, int32_t K, const int32_t *labels, const double *w,
                       const double *dir, double alpha, double *out, int64_t *correct_out,
                       void *ws, size_t ws_bytes, cudaStream_t st);
int csr_wide_objective_grad(const int64_t *indptr, const int32_t *indices, const double *data,
                            const int64_t *colptr, const int32_t *rowidx, const double *cdata,
                            int64_t n, int32_t p, int32_t K, const int32_t *labels,
                            const double *w, double scale, double lam, double *out, double *G,
                            void *ws, size_t ws_bytes, cudaStream_t st);
int csr_wide_probs(const int64_t *indptr, const int32_t *indices, const double *data, int64_t n,
                   int32_t p, int32_t K, const int32_t *labels, const double *w, double *P,
                   int32_t *Y, double *S, void *ws, size_t ws_bytes, cudaStream_t st);
int csr_wide_hess_prepare(const int64_t *indptr, const int32_t *indices, const double *data,
                          int64_t n, int32_t p, int32_t K, const double *w, double *H,
                          void *ws, size_t ws_bytes, cudaStream_t st);
int csr_wide_hess_apply(const int64_t *indptr, const int32_t *indices, const double *data,
                        const int64_t *colptr, const int32_t *rowidx, const double *cdata,
                        int64_t n, int32_t p, int32_t K, const double *H, const double *v,
                        double scale, double lam, double *out, double *dots, const double *skip,
                        void *ws, size_t ws_bytes, cudaStream_t st);
}  // namespace wide
}  // namespace snx


