// fp64 data with many classes (K = C-1 >= 17; the reference is fp64 for
// any C, softmax.py:85-212): the feature products are library DGEMMs
// (cuBLAS, column-major views of the row-major arrays) and the per-row softmax
// algebra is one warp per row here.  Rows are processed in chunks of `zrows`
// so the logits buffer stays bounded (Z: zrows x K doubles in the caller's
// scratch).  Every reduction has a fixed order (reruns are bit-identical).
//
// Column-major views: X row-major [n][ld] is X^c (ld x n); the class-major
// weights w[c*p + j] are W^c (p x K, ld p); Z row-major [m][K] is Z^c (K x m).
//   Z^c  = W^c^T X^c        (cublasDgemm T, N: K x m, inner p)
//   G^c += X^c  Z^c^T       (cublasDgemm N, T: p x K, inner m)
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "snx.h"
#include "snx_common.cuh"
#include "snx_internal.h"

namespace snx {
namespace wide {

constexpr int kKMax = 128;        // K <= 128 (C <= 129), 4 classes per lane
constexpr int kCPL = kKMax / 32;  // classes per lane
constexpr int kKAny = 1 << 16;    // K > 128: row_kernel_any (logits re-read from L1 / L2)
constexpr int kRowWarps = 8;      // rows per 256-thread block
constexpr int kRedThreads = 1024;

enum Mode { kObj = 0, kGrad = 1, kPrep = 2, kApply = 3, kProbs = 4 };

static cublasHandle_t handle() {
  static cublasHandle_t h = nullptr;
  static void *wsp = nullptr;
  if (h == nullptr) {
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
    // a fixed workspace, so the calls can be captured in a CUDA graph
    const size_t bytes = (size_t)32 << 20;
    if (cudaMalloc(&wsp, bytes) == cudaSuccess) cublasSetWorkspace(h, wsp, bytes);
  }
  return h;
}

// first NaN wins, else the larger value, ties to the lower index (numpy argmax)
__device__ __forceinline__ void amax_merge(double &v, int &i, double v2, int i2) {
  const bool n1 = isnan(v), n2 = isnan(v2);
  bool take;
  if (n1 || n2)
    take = n2 && (!n1 || i2 < i);
  else
    take = v2 > v || (v2 == v && i2 < i);
  if (take) {
    v = v2;
    i = i2;
  }
}

struct RowArgs {
  int mode;
  int64_t m, row0;    // rows of this chunk, first row's global index
  int K;
  double *Z;          // [m][K]: logits (V for apply); R / U written in place
  const int32_t *y;   // labels of the chunk (obj / grad / probs stats)
  const double *h;    // apply: h rows of the chunk [m][K]
  double *hout;       // prep: h rows out [m][K]
  double *rl;         // obj / grad: per-row loss (global row index)
  int32_t *rc;        // obj / grad: per-row correct flag (nullable)
  double *P;          // probs: [m][K+1] (nullable)
  int32_t *Y;         // probs: prediction (nullable)
  double *S;          // probs: [m][3] row stats (nullable)
  const double *skip;
};

// softmax.py:91-98 per row: M = max(0, max_c z) (NaN propagates),
// E = exp(z - M), alpha = e^-M + sum E; then the mode's lines.
__global__ void __launch_bounds__(32 * kRowWarps) row_kernel(const RowArgs a) {
  if (a.skip != nullptr && *a.skip != 0.0) return;
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (r >= a.m) return;
  const int K = a.K;
  double *zr = a.Z + r * K;
  double z[kCPL];
#pragma unroll
  for (int j = 0; j < kCPL; ++j) {
    const int c = lane + 32 * j;
    z[j] = c < K ? zr[c] : 0.0;
  }
  if (a.mode == kApply) {  // softmax.py:206-208: VW = V*W; U = VW - W*rowsum(VW)
    const double *hr = a.h + r * K;
    double hv[kCPL], vw[kCPL], s = 0.0;
#pragma unroll
    for (int j = 0; j < kCPL; ++j) {
      const int c = lane + 32 * j;
      hv[j] = c < K ? hr[c] : 0.0;
      vw[j] = z[j] * hv[j];
      s += vw[j];
    }
    s = warp_allsum(s);
#pragma unroll
    for (int j = 0; j < kCPL; ++j) {
      const int c = lane + 32 * j;
      if (c < K) zr[c] = vw[j] - hv[j] * s;
    }
    return;
  }
  double M = 0.0;  // max(0, max_c z) with NaN propagation
#pragma unroll
  for (int j = 0; j < kCPL; ++j)
    if (lane + 32 * j < K && (z[j] > M || isnan(z[j]))) M = z[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double q = __shfl_xor_sync(0xffffffffu, M, o);
    if (isnan(q) || q > M) M = q;
  }
  double E[kCPL], se = 0.0;
#pragma unroll
  for (int j = 0; j < kCPL; ++j) {
    E[j] = lane + 32 * j < K ? exp(z[j] - M) : 0.0;
    se += E[j];
  }
  se = warp_allsum(se);
  const double eM = exp(-M), alpha = eM + se;
  if (a.mode == kPrep) {
    double *ho = a.hout + r * K;
#pragma unroll
    for (int j = 0; j < kCPL; ++j)
      if (lane + 32 * j < K) ho[lane + 32 * j] = E[j] / alpha;
    return;
  }
  const int y = a.y != nullptr ? a.y[r] : -1;
  double lin = 0.0;  // z_{r,y} (0 for the reference class)
#pragma unroll
  for (int j = 0; j < kCPL; ++j)
    if (lane + 32 * j == y) lin = z[j];
  lin = warp_allsum(lin);
  // argmax over [E/alpha, e^-M/alpha] (softmax.py:224-240)
  double bv = (double)NAN;
  int bi = 1 << 30;
  bool have = false;
#pragma unroll
  for (int j = 0; j < kCPL; ++j) {
    const int c = lane + 32 * j;
    if (c < K) {
      const double pc = E[j] / alpha;
      if (!have) {
        bv = pc;
        bi = c;
        have = true;
      } else {
        amax_merge(bv, bi, pc, c);
      }
    }
  }
  if (lane == 0) {
    if (!have) {
      bv = eM / alpha;
      bi = K;
      have = true;
    } else {
      amax_merge(bv, bi, eM / alpha, K);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    const bool h2 = __shfl_xor_sync(0xffffffffu, (int)have, o) != 0;
    if (h2) {
      if (!have) {
        bv = v2;
        bi = i2;
        have = true;
      } else {
        amax_merge(bv, bi, v2, i2);
      }
    }
  }
  if (a.mode == kProbs) {
    if (a.P != nullptr) {
      double *pr = a.P + r * (K + 1);
#pragma unroll
      for (int j = 0; j < kCPL; ++j)
        if (lane + 32 * j < K) pr[lane + 32 * j] = E[j] / alpha;
      if (lane == 0) pr[K] = eM / alpha;
    }
    if (lane == 0) {
      if (a.Y != nullptr) a.Y[r] = bi;
      if (a.S != nullptr) {
        a.S[r * 3 + 0] = M;
        a.S[r * 3 + 1] = se;
        a.S[r * 3 + 2] = lin;
      }
    }
    return;
  }
  if (lane == 0) {
    a.rl[a.row0 + r] = (M + log(alpha)) - lin;  // softmax.py:134
    if (a.rc != nullptr) a.rc[a.row0 + r] = bi == y ? 1 : 0;
  }
  if (a.mode == kGrad) {  // softmax.py:157-161: R = E/alpha - onehot
#pragma unroll
    for (int j = 0; j < kCPL; ++j) {
      const int c = lane + 32 * j;
      if (c < K) zr[c] = E[j] / alpha - (c == y ? 1.0 : 0.0);
    }
  }
}

// The same row algebra for K > 128 (any C): each lane walks its classes
// c = lane, lane + 32, ... through the chunk's logits in global memory (L1 /
// L2-resident), recomputing E where needed -- same values and the same
// summation order as row_kernel.
__global__ void __launch_bounds__(32 * kRowWarps) row_kernel_any(const RowArgs a) {
  if (a.skip != nullptr && *a.skip != 0.0) return;
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5);
  if (r >= a.m) return;
  const int K = a.K;
  double *zr = a.Z + r * K;
  if (a.mode == kApply) {
    const double *hr = a.h + r * K;
    double s = 0.0;
    for (int c = lane; c < K; c += 32) s += zr[c] * hr[c];
    s = warp_allsum(s);
    __syncwarp();
    for (int c = lane; c < K; c += 32) {
      const double vw = zr[c] * hr[c];
      zr[c] = vw - hr[c] * s;
    }
    return;
  }
  double M = 0.0;
  for (int c = lane; c < K; c += 32) {
    const double z = zr[c];
    if (z > M || isnan(z)) M = z;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double q = __shfl_xor_sync(0xffffffffu, M, o);
    if (isnan(q) || q > M) M = q;
  }
  double se = 0.0;
  for (int c = lane; c < K; c += 32) se += exp(zr[c] - M);
  se = warp_allsum(se);
  const double eM = exp(-M), alpha = eM + se;
  if (a.mode == kPrep) {
    double *ho = a.hout + r * K;
    for (int c = lane; c < K; c += 32) ho[c] = exp(zr[c] - M) / alpha;
    return;
  }
  const int y = a.y != nullptr ? a.y[r] : -1;
  double lin = 0.0;
  if (y >= 0 && y < K && (y & 31) == lane) lin = zr[y];
  lin = warp_allsum(lin);
  double bv = (double)NAN;
  int bi = 1 << 30;
  bool have = false;
  for (int c = lane; c < K; c += 32) {
    const double pc = exp(zr[c] - M) / alpha;
    if (!have) {
      bv = pc;
      bi = c;
      have = true;
    } else {
      amax_merge(bv, bi, pc, c);
    }
  }
  if (lane == 0) {
    if (!have) {
      bv = eM / alpha;
      bi = K;
      have = true;
    } else {
      amax_merge(bv, bi, eM / alpha, K);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    const bool h2 = __shfl_xor_sync(0xffffffffu, (int)have, o) != 0;
    if (h2) {
      if (!have) {
        bv = v2;
        bi = i2;
        have = true;
      } else {
        amax_merge(bv, bi, v2, i2);
      }
    }
  }
  if (a.mode == kProbs) {
    if (a.P != nullptr) {
      double *pr = a.P + r * (K + 1);
      for (int c = lane; c < K; c += 32) pr[c] = exp(zr[c] - M) / alpha;
      if (lane == 0) pr[K] = eM / alpha;
    }
    if (lane == 0) {
      if (a.Y != nullptr) a.Y[r] = bi;
      if (a.S != nullptr) {
        a.S[r * 3 + 0] = M;
        a.S[r * 3 + 1] = se;
        a.S[r * 3 + 2] = lin;
      }
    }
    return;
  }
  if (lane == 0) {
    a.rl[a.row0 + r] = (M + log(alpha)) - lin;
    if (a.rc != nullptr) a.rc[a.row0 + r] = bi == y ? 1 : 0;
  }
  if (a.mode == kGrad)
    for (int c = lane; c < K; c += 32) zr[c] = exp(zr[c] - M) / alpha - (c == y ? 1.0 : 0.0);
}

// f32 rows widened to fp64 (exact), row-major [mc][ldo]
__global__ void widen_kernel(const float *X, int64_t ldx, int64_t mc, int32_t p, double *out,
                             int64_t ldo) {
  const int64_t total = mc * (int64_t)p;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / p, j = e - r * p;
    out[r * ldo + j] = (double)X[r * ldx + j];
  }
}

// w_eff = w + alpha * dir (numpy rounding, newton.py:92)
__global__ void weff_kernel(const double *w, const double *dir, double alpha, int64_t d,
                            double *out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = dir != nullptr ? __dadd_rn(w[i], __dmul_rn(alpha, dir[i])) : w[i];
}

// out[0] = sum rl (fixed order), out[1] = ||w||^2, *corr = sum rc
__global__ void __launch_bounds__(kRedThreads)
    reduce_kernel(const double *rl, const int32_t *rc, int64_t n, const double *w, int64_t d,
                  double *out, long long *corr) {
  __shared__ double sh[kRedThreads / 32];
  double s = 0.0, q = 0.0;
  long long c = 0;
  for (int64_t i = threadIdx.x; i < n; i += kRedThreads) {
    s += rl[i];
    if (rc != nullptr) c += rc[i];
  }
  for (int64_t i = threadIdx.x; i < d; i += kRedThreads) q += w[i] * w[i];
  const double ts = block_sum<kRedThreads>(s, sh);
  const double tq = block_sum<kRedThreads>(q, sh);
  __shared__ long long shc[kRedThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) shc[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int k = 0; k < kRedThreads / 32; ++k) t += shc[k];
    out[0] = ts;
    out[1] = tq;
    if (corr != nullptr) *corr = t;
  }
}

// out = scale * acc + lam * base (numpy rounding), + CG dot partials
// (dots[b] = base.out, dots[B + b] = base.base, the snx_hess_apply layout)
__global__ void __launch_bounds__(kDotThreads)
    finish_kernel(const double *acc, double scale, double lam, const double *base, int64_t d,
                  double *out, double *dots, const double *skip) {
  if (skip != nullptr && *skip != 0.0) return;
  __shared__ double sh[kDotThreads / 32];
  double bo = 0.0, bb = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
       i += (int64_t)kDotBlocks * kDotThreads) {
    const double b = base[i];
    const double o = __dadd_rn(__dmul_rn(scale, acc[i]), __dmul_rn(lam, b));
    out[i] = o;
    bo += b * o;
    bb += b * b;
  }
  if (dots == nullptr) return;
  const double so = block_sum<kDotThreads>(bo, sh);
  const double sb = block_sum<kDotThreads>(bb, sh);
  if (threadIdx.x == 0) {
    dots[blockIdx.x] = so;
    dots[kDotBlocks + blockIdx.x] = sb;
  }
}

static int check_args(const char *who, const void *X, int64_t ldx, int64_t n, int32_t p,
                      int32_t K, const double *scratch, int64_t zrows) {
  if (K < 1 || K > kKAny) {
    set_error("%s: K = C-1 = %d outside [1, %d]", who, K, kKAny);
    return 1;
  }
  if (p < 1 || ldx < p || n < 0 || (n > 0 && X == nullptr)) {
    set_error("%s: bad shape (n=%lld p=%d ldx=%lld) or NULL X", who, (long long)n, p,
              (long long)ldx);
    return 1;
  }
  if (scratch == nullptr || zrows < 1) {
    set_error("%s: NULL scratch or zrows < 1", who);
    return 1;
  }
  if (handle() == nullptr) {
    set_error("%s: cublasCreate failed", who);
    return 1;
  }
  return 0;
}

static int gemm_check(cublasStatus_t s, const char *who) {
  if (s != CUBLAS_STATUS_SUCCESS) {
    set_error("%s: cublasDgemm failed (status %d)", who, (int)s);
    return 1;
  }
  return check_launch(who);
}

// Z^c (K x mc) = W^c^T (K x p) X^c (p x mc)
static int logits(const double *X, int64_t ldx, int64_t mc, int32_t p, int32_t K,
                  const double *W, double *Z, cudaStream_t st) {
  cublasHandle_t h = handle();
  cublasSetStream(h, st);
  const double one = 1.0, zero = 0.0;
  return gemm_check(cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, K, (int)mc, p, &one, W, p, X,
                                (int)ldx, &zero, Z, K),
                    "wide logits");
}

// G^c (p x K) (+)= X^c (p x mc) Z^c^T (mc x K)
static int xtz(const double *X, int64_t ldx, int64_t mc, int32_t p, int32_t K, const double *Z,
               double *G, bool accumulate, cudaStream_t st) {
  cublasHandle_t h = handle();
  cublasSetStream(h, st);
  const double one = 1.0, beta = accumulate ? 1.0 : 0.0;
  return gemm_check(cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_T, p, K, (int)mc, &one, X, (int)ldx,
                                Z, K, &beta, G, p),
                    "wide X^T Z");
}

static int rows_launch(const RowArgs &a, cudaStream_t st) {
  if (a.m <= 0) return 0;
  const unsigned blocks = (unsigned)((a.m + kRowWarps - 1) / kRowWarps);
  if (a.K <= kKMax)
    row_kernel<<<blocks, 32 * kRowWarps, 0, st>>>(a);
  else
    row_kernel_any<<<blocks, 32 * kRowWarps, 0, st>>>(a);
  return check_launch("wide row pass");
}

// scratch layout (doubles): Z [zrows*K] | row loss [n] | row correct [n ints] |
// w_eff / product accumulator [d] | 2 spare
struct Scratch {
  double *Z, *rl, *acc;
  int32_t *rc;
};
static Scratch carve(double *s, int64_t zrows, int32_t K, int64_t n) {
  Scratch c;
  c.Z = s;
  c.rl = s + zrows * K;
  c.rc = reinterpret_cast<int32_t *>(c.rl + n);
  c.acc = c.rl + n + (n + 1) / 2;
  return c;
}

// ---------------------------------------------------------------- CSR data
// Sparse rows with many classes (K > 32; the CSR kernels of snx_csr.cu keep a
// row's logits in registers): logits by a warp per row over the row's entries
// in stored order (lanes over classes, weights transposed to [p][K] so the
// loads coalesce), X^T R by a warp per CSC column -- both fixed-order -- and
// the row algebra of row_kernel.  One chunk (Z: nrows x K doubles).

// wt[j*K + c] = (w + alpha*dir)[c*p + j]; block partials not needed here
__global__ void transpose_w_kernel(const double *w, const double *dir, double alpha, int32_t p,
                                   int32_t K, double *wt) {
  const int64_t d = (int64_t)K * p;
  for (int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; f < d;
       f += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = f / p, j = f - c * p;
    wt[j * K + c] = dir != nullptr ? __dadd_rn(w[f], __dmul_rn(alpha, dir[f])) : w[f];
  }
}

__global__ void __launch_bounds__(256)
    csr_logits_kernel(const int64_t *indptr, const int32_t *indices, const double *data,
                      int64_t nrows, const double *wt, int32_t K, double *Z,
                      const double *skip) {
  if (skip != nullptr && *skip != 0.0) return;
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (r >= nrows) return;
  const int64_t e0 = indptr[r], e1 = indptr[r + 1];
  for (int c0 = 0; c0 < K; c0 += 32) {
    const int c = c0 + lane;
    double acc = 0.0;
    if (c < K)
      for (int64_t t = e0; t < e1; ++t) acc = fma(data[t], __ldg(wt + (int64_t)indices[t] * K + c), acc);
    if (c < K) Z[r * K + c] = acc;
  }
}

// acc[c*p + j] = sum over column j's entries (stored order) of cdata * R[row][c]
__global__ void __launch_bounds__(256)
    csc_xtr_kernel(const int64_t *colptr, const int32_t *rowidx, const double *cdata, int32_t p,
                   const double *R, int32_t K, double *acc, const double *skip) {
  if (skip != nullptr && *skip != 0.0) return;
  const int lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (j >= p) return;
  const int64_t e0 = colptr[j], e1 = colptr[j + 1];
  for (int c0 = 0; c0 < K; c0 += 32) {
    const int c = c0 + lane;
    double s = 0.0;
    if (c < K)
      for (int64_t t = e0; t < e1; ++t) s = fma(cdata[t], R[(int64_t)rowidx[t] * K + c], s);
    if (c < K) acc[(int64_t)c * p + j] = s;
  }
}

// workspace (bytes) of the sparse wide passes: wt [d] | Z [n*K] | rl [n] |
// rc [n ints] | acc [d] | 2
size_t csr_wide_ws_bytes(int64_t n, int32_t p, int32_t K) {
  const int64_t d = (int64_t)K * p;
  return (size_t)(d + (int64_t)n * K + n + (n + 1) / 2 + d + 2) * sizeof(double);
}

struct CsrWs {
  double *wt, *Z, *rl, *acc;
  int32_t *rc;
};
static int csr_carve(const char *who, void *ws, size_t ws_bytes, int64_t n, int32_t p, int32_t K,
                     CsrWs &c) {
  if (ws == nullptr || ws_bytes < csr_wide_ws_bytes(n, p, K)) {
    set_error("%s: workspace of %zu bytes < %zu", who, ws_bytes, csr_wide_ws_bytes(n, p, K));
    return 1;
  }
  const int64_t d = (int64_t)K * p;
  double *s = static_cast<double *>(ws);
  c.wt = s;
  c.Z = s + d;
  c.rl = c.Z + n * K;
  c.rc = reinterpret_cast<int32_t *>(c.rl + n);
  c.acc = c.rl + n + (n + 1) / 2;
  return 0;
}

static int csr_logits(const int64_t *indptr, const int32_t *indices, const double *data,
                      int64_t n, int32_t p, int32_t K, const double *w, const double *dir,
                      double alpha, const CsrWs &c, const double *skip, cudaStream_t st) {
  transpose_w_kernel<<<296, 256, 0, st>>>(w, dir, alpha, p, K, c.wt);
  if (check_launch("csr wide transpose")) return 1;
  if (n > 0) {
    csr_logits_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(indptr, indices, data, n, c.wt, K,
                                                            c.Z, skip);
    if (check_launch("csr wide logits")) return 1;
  }
  return 0;
}

int csr_wide_objective(const int64_t *indptr, const int32_t *indices, const double *data,
                       int64_t n, int32_t p, int32_t K, const int32_t *labels, const double *w,
                       const double *dir, double alpha, double *out, int64_t *correct_out,
                       void *ws, size_t ws_bytes, cudaStream_t st) {
  CsrWs c;
  if (csr_carve("snx_csr_objective", ws, ws_bytes, n, p, K, c)) return 1;
  if (csr_logits(indptr, indices, data, n, p, K, w, dir, alpha, c, nullptr, st)) return 1;
  RowArgs a{};
  a.mode = kObj;
  a.m = n;
  a.K = K;
  a.Z = c.Z;
  a.y = labels;
  a.rl = c.rl;
  a.rc = correct_out != nullptr ? c.rc : nullptr;
  if (rows_launch(a, st)) return 1;
  // ||w_eff||^2 from the transposed copy (same values, a different order)
  reduce_kernel<<<1, kRedThreads, 0, st>>>(c.rl, a.rc, n, c.wt, (int64_t)K * p, out,
                                           reinterpret_cast<long long *>(correct_out));
  return check_launch("csr wide reduce");
}

int csr_wide_objective_grad(const int64_t *indptr, const int32_t *indices, const double *data,
                            const int64_t *colptr, const int32_t *rowidx, const double *cdata,
                            int64_t n, int32_t p, int32_t K, const int32_t *labels,
                            const double *w, double scale, double lam, double *out, double *G,
                            void *ws, size_t ws_bytes, cudaStream_t st) {
  CsrWs c;
  if (csr_carve("snx_csr_objective_grad", ws, ws_bytes, n, p, K, c)) return 1;
  if (csr_logits(indptr, indices, data, n, p, K, w, nullptr, 0.0, c, nullptr, st)) return 1;
  RowArgs a{};
  a.mode = kGrad;
  a.m = n;
  a.K = K;
  a.Z = c.Z;
  a.y = labels;
  a.rl = c.rl;
  if (rows_launch(a, st)) return 1;
  csc_xtr_kernel<<<(unsigned)((p + 7) / 8), 256, 0, st>>>(colptr, rowidx, cdata, p, c.Z, K, c.acc,
                                                        nullptr);
  if (check_launch("csr wide X^T R")) return 1;
  reduce_kernel<<<1, kRedThreads, 0, st>>>(c.rl, nullptr, n, w, (int64_t)K * p, out, nullptr);
  if (check_launch("csr wide reduce")) return 1;
  finish_kernel<<<kDotBlocks, kDotThreads, 0, st>>>(c.acc, scale, lam, w, (int64_t)K * p, G,
                                                   nullptr, nullptr);
  return check_launch("csr wide gradient finish");
}

int csr_wide_probs(const int64_t *indptr, const int32_t *indices, const double *data, int64_t n,
                   int32_t p, int32_t K, const int32_t *labels, const double *w, double *P,
                   int32_t *Y, double *S, void *ws, size_t ws_bytes, cudaStream_t st) {
  CsrWs c;
  if (csr_carve("snx_csr_class_probabilities", ws, ws_bytes, n, p, K, c)) return 1;
  if (csr_logits(indptr, indices, data, n, p, K, w, nullptr, 0.0, c, nullptr, st)) return 1;
  RowArgs a{};
  a.mode = kProbs;
  a.m = n;
  a.K = K;
  a.Z = c.Z;
  a.y = labels;
  a.P = P;
  a.Y = Y;
  a.S = S;
  return rows_launch(a, st);
}

int csr_wide_hess_prepare(const int64_t *indptr, const int32_t *indices, const double *data,
                          int64_t n, int32_t p, int32_t K, const double *w, double *H,
                          void *ws, size_t ws_bytes, cudaStream_t st) {
  CsrWs c;
  if (csr_carve("snx_csr_hess_prepare", ws, ws_bytes, n, p, K, c)) return 1;
  if (csr_logits(indptr, indices, data, n, p, K, w, nullptr, 0.0, c, nullptr, st)) return 1;
  RowArgs a{};
  a.mode = kPrep;
  a.m = n;
  a.K = K;
  a.Z = c.Z;
  a.hout = H;
  return rows_launch(a, st);
}

int csr_wide_hess_apply(const int64_t *indptr, const int32_t *indices, const double *data,
                        const int64_t *colptr, const int32_t *rowidx, const double *cdata,
                        int64_t n, int32_t p, int32_t K, const double *H, const double *v,
                        double scale, double lam, double *out, double *dots, const double *skip,
                        void *ws, size_t ws_bytes, cudaStream_t st) {
  CsrWs c;
  if (csr_carve("snx_csr_hess_apply", ws, ws_bytes, n, p, K, c)) return 1;
  if (csr_logits(indptr, indices, data, n, p, K, v, nullptr, 0.0, c, skip, st)) return 1;
  RowArgs a{};
  a.mode = kApply;
  a.m = n;
  a.K = K;
  a.Z = c.Z;
  a.h = H;
  a.skip = skip;
  if (rows_launch(a, st)) return 1;
  csc_xtr_kernel<<<(unsigned)((p + 7) / 8), 256, 0, st>>>(colptr, rowidx, cdata, p, c.Z, K, c.acc,
                                                        skip);
  if (check_launch("csr wide X^T U")) return 1;
  finish_kernel<<<kDotBlocks, kDotThreads, 0, st>>>(c.acc, scale, lam, v, (int64_t)K * p, out,
                                                   dots, skip);
  return check_launch("csr wide product finish");
}

}  // namespace wide
}  // namespace snx

using namespace snx;
using namespace snx::wide;

extern "C" {

int64_t snx_wide_scratch_doubles(int64_t n, int32_t p, int32_t K, int64_t zrows) {
  return zrows * K + n + (n + 1) / 2 + (int64_t)K * p + 2;
}

int snx_wide_objective(const double *X, int64_t ldx, int64_t n, int32_t p, int32_t K,
                       const int32_t *labels, const double *w, const double *dir, double alpha,
                       double *out, long long *correct_out, double *scratch, int64_t zrows,
                       void *stream) {
  if (check_args("snx_wide_objective", X, ldx, n, p, K, scratch, zrows)) return 1;
  if (w == nullptr || out == nullptr || (n > 0 && labels == nullptr)) {
    set_error("snx_wide_objective: NULL w, out or labels");
    return 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  Scratch sc = carve(scratch, zrows, K, n);
  const int64_t d = (int64_t)K * p;
  weff_kernel<<<148, 256, 0, st>>>(w, dir, alpha, d, sc.acc);
  if (check_launch("wide w_eff")) return 1;
  for (int64_t r0 = 0; r0 < n; r0 += zrows) {
    const int64_t mc = n - r0 < zrows ? n - r0 : zrows;
    if (logits(X + r0 * ldx, ldx, mc, p, K, sc.acc, sc.Z, st)) return 1;
    RowArgs a{};
    a.mode = kObj;
    a.m = mc;
    a.row0 = r0;
    a.K = K;
    a.Z = sc.Z;
    a.y = labels + r0;
    a.rl = sc.rl;
    a.rc = correct_out != nullptr ? sc.rc : nullptr;
    if (rows_launch(a, st)) return 1;
  }
  reduce_kernel<<<1, kRedThreads, 0, st>>>(sc.rl, correct_out != nullptr ? sc.rc : nullptr, n,
                                           sc.acc, d, out, correct_out);
  return check_launch("wide reduce");
}

int snx_wide_objective_grad(const double *X, int64_t ldx, int64_t n, int32_t p, int32_t K,
                            const int32_t *labels, const double *w, double scale, double lam,
                            double *out, double *G, double *scratch, int64_t zrows,
                            void *stream) {
  if (check_args("snx_wide_objective_grad", X, ldx, n, p, K, scratch, zrows)) return 1;
  if (w == nullptr || out == nullptr || G == nullptr || (n > 0 && labels == nullptr)) {
    set_error("snx_wide_objective_grad: NULL w, out, G or labels");
    return 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  Scratch sc = carve(scratch, zrows, K, n);
  const int64_t d = (int64_t)K * p;
  if (n == 0) cudaMemsetAsync(sc.acc, 0, d * sizeof(double), st);
  for (int64_t r0 = 0; r0 < n; r0 += zrows) {
    const int64_t mc = n - r0 < zrows ? n - r0 : zrows;
    if (logits(X + r0 * ldx, ldx, mc, p, K, w, sc.Z, st)) return 1;
    RowArgs a{};
    a.mode = kGrad;
    a.m = mc;
    a.row0 = r0;
    a.K = K;
    a.Z = sc.Z;
    a.y = labels + r0;
    a.rl = sc.rl;
    if (rows_launch(a, st)) return 1;
    if (xtz(X + r0 * ldx, ldx, mc, p, K, sc.Z, sc.acc, r0 > 0, st)) return 1;
  }
  reduce_kernel<<<1, kRedThreads, 0, st>>>(sc.rl, nullptr, n, w, d, out, nullptr);
  if (check_launch("wide reduce")) return 1;
  finish_kernel<<<kDotBlocks, kDotThreads, 0, st>>>(sc.acc, scale, lam, w, d, G, nullptr,
                                                   nullptr);
  return check_launch("wide gradient finish");
}

int snx_wide_hess_prepare(const double *X, int64_t ldx, const int64_t *rows, int64_t nrows,
                          int32_t p, int32_t K, const double *w, double *Xs_out, int64_t ld_out,
                          double *H_out, double *scratch, int64_t zrows, void *stream) {
  if (check_args("snx_wide_hess_prepare", X, ldx, nrows, p, K, scratch, zrows)) return 1;
  if (w == nullptr || H_out == nullptr || (rows != nullptr && Xs_out == nullptr)) {
    set_error("snx_wide_hess_prepare: NULL w or H_out (or Xs_out with rows)");
    return 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const double *Xs = X;
  int64_t lds = ldx;
  if (rows != nullptr) {
    if (snx_gather_rows(SNX_F64, X, ldx, nullptr, rows, nrows, Xs_out, ld_out, nullptr, st))
      return 1;
    Xs = Xs_out;
    lds = ld_out;
  }
  Scratch sc = carve(scratch, zrows, K, nrows);
  for (int64_t r0 = 0; r0 < nrows; r0 += zrows) {
    const int64_t mc = nrows - r0 < zrows ? nrows - r0 : zrows;
    if (logits(Xs + r0 * lds, lds, mc, p, K, w, sc.Z, st)) return 1;
    RowArgs a{};
    a.mode = kPrep;
    a.m = mc;
    a.K = K;
    a.Z = sc.Z;
    a.hout = H_out + r0 * K;
    if (rows_launch(a, st)) return 1;
  }
  return 0;
}

int snx_wide_hess_apply(const double *Xs, int64_t lds, int64_t m, int32_t p, int32_t K,
                        const double *H, const double *v, double scale, double lam, double *out,
                        double *dots, const double *skip, double *scratch, int64_t zrows,
                        void *stream) {
  if (check_args("snx_wide_hess_apply", Xs, lds, m, p, K, scratch, zrows)) return 1;
  if (H == nullptr || v == nullptr || out == nullptr) {
    set_error("snx_wide_hess_apply: NULL H, v or out");
    return 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  Scratch sc = carve(scratch, zrows, K, m);
  const int64_t d = (int64_t)K * p;
  if (m == 0) cudaMemsetAsync(sc.acc, 0, d * sizeof(double), st);
  for (int64_t r0 = 0; r0 < m; r0 += zrows) {
    const int64_t mc = m - r0 < zrows ? m - r0 : zrows;
    if (logits(Xs + r0 * lds, lds, mc, p, K, v, sc.Z, st)) return 1;  // V = X_S v^T
    RowArgs a{};
    a.mode = kApply;
    a.m = mc;
    a.K = K;
    a.Z = sc.Z;
    a.h = H + r0 * K;
    a.skip = skip;
    if (rows_launch(a, st)) return 1;
    if (xtz(Xs + r0 * lds, lds, mc, p, K, sc.Z, sc.acc, r0 > 0, st)) return 1;
  }
  finish_kernel<<<kDotBlocks, kDotThreads, 0, st>>>(sc.acc, scale, lam, v, d, out, dots, skip);
  return check_launch("wide product finish");
}

int snx_wide_class_probabilities(const double *X, int64_t ldx, int64_t n, int32_t p, int32_t K,
                                 const int32_t *labels, const double *w, double *probs_out,
                                 int32_t *pred_out, double *stats_out, double *scratch,
                                 int64_t zrows, void *stream) {
  if (check_args("snx_wide_class_probabilities", X, ldx, n, p, K, scratch, zrows)) return 1;
  if (w == nullptr || (n > 0 && stats_out != nullptr && labels == nullptr)) {
    set_error("snx_wide_class_probabilities: NULL w (or labels with stats_out)");
    return 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  Scratch sc = carve(scratch, zrows, K, n);
  for (int64_t r0 = 0; r0 < n; r0 += zrows) {
    const int64_t mc = n - r0 < zrows ? n - r0 : zrows;
    if (logits(X + r0 * ldx, ldx, mc, p, K, w, sc.Z, st)) return 1;
    RowArgs a{};
    a.mode = kProbs;
    a.m = mc;
    a.K = K;
    a.Z = sc.Z;
    a.y = labels != nullptr ? labels + r0 : nullptr;
    a.P = probs_out != nullptr ? probs_out + r0 * (K + 1) : nullptr;
    a.Y = pred_out != nullptr ? pred_out + r0 : nullptr;
    a.S = stats_out != nullptr ? stats_out + r0 * 3 : nullptr;
    if (rows_launch(a, st)) return 1;
  }
  return 0;
}

int64_t snx_wide_f32_scratch_doubles(int64_t n, int32_t p, int32_t K, int64_t zrows) {
  (void)n;
  return zrows * K + zrows * (int64_t)p + 2;
}

int snx_wide_class_probabilities_f32(const float *X, int64_t ldx, int64_t n, int32_t p,
                                     int32_t K, const int32_t *labels, const double *w,
                                     double *probs_out, int32_t *pred_out, double *stats_out,
                                     double *scratch, int64_t zrows, void *stream) {
  if (check_args("snx_wide_class_probabilities_f32", X, ldx, n, p, K, scratch, zrows))
    return 1;
  if (w == nullptr || (n > 0 && stats_out != nullptr && labels == nullptr)) {
    set_error("snx_wide_class_probabilities_f32: NULL w (or labels with stats_out)");
    return 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  double *Z = scratch, *Xd = scratch + zrows * K;
  for (int64_t r0 = 0; r0 < n; r0 += zrows) {
    const int64_t mc = n - r0 < zrows ? n - r0 : zrows;
    widen_kernel<<<296, 256, 0, st>>>(X + r0 * ldx, ldx, mc, p, Xd, p);
    if (check_launch("wide widen")) return 1;
    if (logits(Xd, p, mc, p, K, w, Z, st)) return 1;
    RowArgs a{};
    a.mode = kProbs;
    a.m = mc;
    a.K = K;
    a.Z = Z;
    a.y = labels != nullptr ? labels + r0 : nullptr;
    a.P = probs_out != nullptr ? probs_out + r0 * (K + 1) : nullptr;
    a.Y = pred_out != nullptr ? pred_out + r0 : nullptr;
    a.S = stats_out != nullptr ? stats_out + r0 * 3 : nullptr;
    if (rows_launch(a, st)) return 1;
  }
  return 0;
}

}  // extern "C"
