// Sparse (CSR) feature storage: the reference's sparse DesignMatrix
// (dataset.py:21-147; scipy CSR products in matmat / rmatmat :80-88) and the
// paper's cuSPARSE path, fp64, K = C - 1 <= 32 (Newsgroups20: 19).
//
// Data: CSR  indptr[n+1] (int64), indices[nnz] (int32 columns), data[nnz]
//       CSC  colptr[p+1] (int64), rowidx[nnz] (int32 rows),    cdata[nnz]
// (the CSC copy is the transpose, so X^T R contracts per column with no
// atomics: every reduction has a fixed order and reruns are bit-identical).
//
// Passes (all HBM / L2 gather-bound: SpMM with K <= 16 dense columns):
//   rows pass   one warp per row: z = a_i . W over the row's nonzeros (lanes
//               stride the nonzeros, butterfly per class), then the row
//               algebra of softmax.py:85-99 (loss, argmax, residual E/alpha -
//               onehot, probabilities h, or ComputeU of softmax.py:206-208);
//   cols pass   a lane per short column, a warp (lanes stride the entries) per
//               long one: out[c][j] = scale * sum_i a_ij R_ic + lam*base
//               (softmax.py:154-169 / :209-210) + CG dot partials;
//   gather      the sample S of sampling.py:79-80 as its own CSR (row copy)
//               and CSC (the full CSC filtered by a row -> sample-position map,
//               order kept), so each Hessian product touches only the sample.
#include <type_traits>

#include "snx_common.cuh"
#include "snx_internal.h"

namespace snx {
namespace {

constexpr int kCsrThreads = 256;
constexpr int kCsrWarps = kCsrThreads / 32;
constexpr int kRowBlocks = 148 * 4;  // fixed grid of the rows pass (loss partials)

enum CsrMode { kObj = 0, kGrad = 1, kPrep = 2, kApply = 3, kProbs = 4 };

__host__ __device__ constexpr size_t al256(size_t x) { return (x + 255) / 256 * 256; }

// workspace layout (bytes)
struct CsrWs {
  double *wt;            // [p][K] weights (or v) transposed: row j holds its K classes
  double *rowbuf;        // [rows][K] residual R / probabilities / U
  double *loss_part;     // [kRowBlocks]
  unsigned long long *corr_part;  // [kRowBlocks]
  double *wsq_part;      // [kDotBlocks]
  int32_t *pos;          // [n] row -> first sample position (or -1)
  int32_t *mult;         // [n] multiplicity of the row in the sample
  int64_t *scan;         // [max(n, p) + 1] scan input
};

__host__ __device__ inline size_t csr_ws_layout(int64_t n, int p, int K, char *base, CsrWs *w) {
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char *q = base ? base + off : nullptr;
    off += al256(bytes);
    return q;
  };
  const int64_t nn = n > 0 ? n : 1;
  const int64_t pp = p > 0 ? p : 1;
  const int64_t big = (nn > pp ? nn : pp) + 1;
  char *a = take((size_t)pp * K * 8);
  char *b = take((size_t)nn * K * 8);
  char *c = take((size_t)kRowBlocks * 8);
  char *d = take((size_t)kRowBlocks * 8);
  char *e = take((size_t)kDotBlocks * 8);
  char *f = take((size_t)nn * 4);
  char *g = take((size_t)nn * 4);
  char *h = take((size_t)big * 8);
  if (w) {
    w->wt = reinterpret_cast<double *>(a);
    w->rowbuf = reinterpret_cast<double *>(b);
    w->loss_part = reinterpret_cast<double *>(c);
    w->corr_part = reinterpret_cast<unsigned long long *>(d);
    w->wsq_part = reinterpret_cast<double *>(e);
    w->pos = reinterpret_cast<int32_t *>(f);
    w->mult = reinterpret_cast<int32_t *>(g);
    w->scan = reinterpret_cast<int64_t *>(h);
  }
  return off;
}

// Wt[j*K + c] = (w + alpha*dir)[c*p + j] with numpy rounding, as a tiled
// transpose (each warp: 32 columns x K classes through shared memory, loads
// and stores coalesced); block partials of ||w + alpha*dir||^2 (the lam/2
// ||x||^2 term of softmax.py:141).  Exactly kDotBlocks blocks.
template <int K>
__global__ void __launch_bounds__(kCsrThreads)
    csr_prep_w_kernel(const double *__restrict__ w, const double *__restrict__ dir, double alpha,
                      int p, double *__restrict__ wt, double *__restrict__ wsq_part,
                      const double *skip) {
  if (skip != nullptr && *skip != 0.0) return;
  constexpr int TW = K <= 23 ? 32 : 16;  // columns per warp tile (static smem <= 48 KB)
  __shared__ double tile[kCsrWarps][TW * K + 1];
  __shared__ double sh[kCsrThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0.0;
  double *tw = tile[warp];
  for (int64_t j0 = ((int64_t)blockIdx.x * kCsrWarps + warp) * TW; j0 < p;
       j0 += (int64_t)gridDim.x * kCsrWarps * TW) {
    const int64_t j = j0 + lane;
    const int nj = (int)min((int64_t)TW, (int64_t)p - j0);
#pragma unroll
    for (int c = 0; c < K; ++c) {
      if (lane < nj) {
        const int64_t f = (int64_t)c * p + j;
        const double v = dir ? np_axpy(w[f], alpha, dir[f]) : w[f];
        tw[lane * K + c] = v;
        acc += v * v;
      }
    }
    __syncwarp();
    for (int t = lane; t < nj * K; t += 32) wt[j0 * K + t] = tw[t];
    __syncwarp();
  }
  if (wsq_part == nullptr) return;
  const double b = block_sum<kCsrThreads>(acc, sh);
  if (threadIdx.x == 0) wsq_part[blockIdx.x] = b;
}

// One warp per row: logits of the row (or V = a_i Q for kApply) and the row algebra.
template <int K>
__global__ void __launch_bounds__(kCsrThreads)
    csr_rows_kernel(int mode, const int64_t *__restrict__ indptr,
                    const int32_t *__restrict__ indices, const double *__restrict__ data,
                    int64_t nrows, const double *__restrict__ wt, const int32_t *__restrict__ labels,
                    const double *__restrict__ H, double *__restrict__ rowout,
                    double *__restrict__ loss_part, unsigned long long *__restrict__ corr_part,
                    const double *skip, int32_t *__restrict__ pred_out = nullptr,
                    double *__restrict__ stats_out = nullptr) {
  if (skip != nullptr && *skip != 0.0) return;
  __shared__ double shl[kCsrWarps];
  __shared__ unsigned long long shc[kCsrWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * kCsrWarps + warp;
  const int64_t stride = (int64_t)gridDim.x * kCsrWarps;
  double lacc = 0.0;
  unsigned long long cacc = 0;
  for (int64_t r = gw; r < nrows; r += stride) {
    const int64_t e0 = indptr[r], e1 = indptr[r + 1];
    double z[K];
#pragma unroll
    for (int c = 0; c < K; ++c) z[c] = 0.0;
    for (int64_t t = e0 + lane; t < e1; t += 32) {
      const double a = data[t];
      const double *wr = wt + (int64_t)indices[t] * K;
#pragma unroll
      for (int c = 0; c < K; ++c) z[c] = fma(a, __ldg(wr + c), z[c]);
    }
#pragma unroll
    for (int c = 0; c < K; ++c) z[c] = warp_allsum(z[c]);  // every lane holds the row
    if (mode == kApply) {
      // softmax.py:206-208: VW = V*W; U = VW - W*rowsum(VW)
      double hw[K], vw[K], s = 0.0;
#pragma unroll
      for (int c = 0; c < K; ++c) {
        hw[c] = H[r * K + c];
        vw[c] = z[c] * hw[c];
        s += vw[c];
      }
#pragma unroll
      for (int c = 0; c < K; ++c)
        if (lane == c) rowout[r * K + c] = vw[c] - hw[c] * s;
      continue;
    }
    // softmax.py:91-98
    double M = 0.0;
#pragma unroll
    for (int c = 0; c < K; ++c) M = (z[c] > M || isnan(z[c])) ? z[c] : M;
    double E[K], se = 0.0;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      E[c] = exp(z[c] - M);
      se += E[c];
    }
    const double alpha = exp(-M) + se;
    if (mode == kPrep) {
#pragma unroll
      for (int c = 0; c < K; ++c)
        if (lane == c) rowout[r * K + c] = E[c] / alpha;
      continue;
    }
    if (mode == kProbs) {  // softmax.py:224-240 and row_stats :107-122
      if (rowout != nullptr) {
#pragma unroll
        for (int c = 0; c < K; ++c)
          if (lane == c) rowout[r * (K + 1) + c] = E[c] / alpha;
        if (lane == 31) rowout[r * (K + 1) + K] = exp(-M) / alpha;
      }
      if (lane == 0 && stats_out != nullptr) {
        const int yy = labels[r];
        double lin = 0.0;
#pragma unroll
        for (int c = 0; c < K; ++c)
          if (c == yy) lin = z[c];
        stats_out[r * 3 + 0] = M;
        stats_out[r * 3 + 1] = se;
        stats_out[r * 3 + 2] = lin;
      }
      if (lane == 0 && pred_out != nullptr) {
        int best = 0;
        double bv = E[0] / alpha;
        bool nan_hit = isnan(bv);
#pragma unroll
        for (int c = 1; c <= K; ++c) {
          const double pc = (c < K ? E[c] : exp(-M)) / alpha;
          if (!nan_hit && (isnan(pc) || pc > bv)) {
            best = c;
            bv = pc;
            nan_hit = isnan(pc);
          }
        }
        pred_out[r] = best;
      }
      continue;
    }
    const int y = labels[r];
    double lin = 0.0;
#pragma unroll
    for (int c = 0; c < K; ++c)
      if (c == y) lin = z[c];
    lacc += (M + log(alpha)) - lin;  // softmax.py:134, rows in a fixed order per warp
    if (mode == kGrad) {
#pragma unroll
      for (int c = 0; c < K; ++c)
        if (lane == c) rowout[r * K + c] = E[c] / alpha - (c == y ? 1.0 : 0.0);
    } else if (corr_part != nullptr) {
      // softmax.py:224-240: argmax over [E/alpha, e^-M/alpha], first max wins
      int best = 0;
      double bv = E[0] / alpha;
      bool nan_hit = isnan(bv);
#pragma unroll
      for (int c = 1; c <= K; ++c) {
        const double pc = (c < K ? E[c] : exp(-M)) / alpha;
        if (!nan_hit && (isnan(pc) || pc > bv)) {
          best = c;
          bv = pc;
          nan_hit = isnan(pc);
        }
      }
      cacc += (best == y) ? 1ull : 0ull;
    }
  }
  if (mode == kPrep || mode == kApply || mode == kProbs || loss_part == nullptr) return;
  if (lane == 0) {
    shl[warp] = lacc;
    shc[warp] = cacc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    unsigned long long u = 0;
#pragma unroll
    for (int i = 0; i < kCsrWarps; ++i) {
      t += shl[i];
      u += shc[i];
    }
    loss_part[blockIdx.x] = t;
    if (corr_part) corr_part[blockIdx.x] = u;
  }
}

// out[0] = sum of the row-block loss partials, out[1] = ||w_eff||^2, correct count.
__global__ void csr_final_kernel(const double *loss_part, const unsigned long long *corr_part,
                                 const double *wsq_part, double *out, long long *corr_out) {
  const int lane = threadIdx.x;
  double l = 0.0;
  unsigned long long u = 0;
  for (int i = lane; i < kRowBlocks; i += 32) {
    l += loss_part[i];
    if (corr_out) u += corr_part[i];
  }
  l = warp_allsum(l);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
  const double q = warp_sum_partials(wsq_part);
  if (lane == 0) {
    out[0] = l;
    out[1] = q;
    if (corr_out) *corr_out = (long long)u;
  }
}

// Columns pass: out[c*p + j] = scale * sum_i a_ij R[i][c] + lam * base[c*p + j]
// (numpy rounding of `scale * acc + lam * v`), and the CG dot partials
// (base . out | base . base) of this block.  A warp owns 32 consecutive
// columns, one per lane (short columns: the lane walks its entries, class
// writes coalesced across lanes); columns longer than kLongCol are summed by
// the whole warp (lane-strided + butterfly).  Exactly kDotBlocks blocks.
constexpr int kLongCol = 48;

template <int K>
__global__ void __launch_bounds__(kCsrThreads)
    csc_cols_kernel(const int64_t *__restrict__ colptr, const int32_t *__restrict__ rowidx,
                    const double *__restrict__ cdata, int p, const double *__restrict__ R,
                    double scale, double lam, const double *__restrict__ base,
                    double *__restrict__ out, double *__restrict__ dots, const double *skip) {
  if (skip != nullptr && *skip != 0.0) return;
  __shared__ double sh[kCsrThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double bo = 0.0, bb = 0.0;
  for (int64_t j0 = ((int64_t)blockIdx.x * kCsrWarps + warp) * 32; j0 < p;
       j0 += (int64_t)gridDim.x * kCsrWarps * 32) {
    const int64_t j = j0 + lane;
    int64_t e0 = 0, e1 = 0;
    if (j < p) {
      e0 = colptr[j];
      e1 = colptr[j + 1];
    }
    const bool lng = e1 - e0 > kLongCol;
    double acc[K];
#pragma unroll
    for (int c = 0; c < K; ++c) acc[c] = 0.0;
    if (!lng) {
      for (int64_t t = e0; t < e1; ++t) {
        const double a = cdata[t];
        const double *rr = R + (int64_t)rowidx[t] * K;
#pragma unroll
        for (int c = 0; c < K; ++c) acc[c] = fma(a, __ldg(rr + c), acc[c]);
      }
    }
    for (unsigned lm = __ballot_sync(0xffffffffu, lng); lm != 0u; lm &= lm - 1u) {
      const int src = __ffs(lm) - 1;
      const int64_t l0 = __shfl_sync(0xffffffffu, e0, src), l1 = __shfl_sync(0xffffffffu, e1, src);
      double t2[K];
#pragma unroll
      for (int c = 0; c < K; ++c) t2[c] = 0.0;
      for (int64_t t = l0 + lane; t < l1; t += 32) {
        const double a = cdata[t];
        const double *rr = R + (int64_t)rowidx[t] * K;
#pragma unroll
        for (int c = 0; c < K; ++c) t2[c] = fma(a, __ldg(rr + c), t2[c]);
      }
#pragma unroll
      for (int c = 0; c < K; ++c) {
        t2[c] = warp_allsum(t2[c]);
        if (lane == src) acc[c] = t2[c];
      }
    }
    if (j < p) {
#pragma unroll
      for (int c = 0; c < K; ++c) {
        const int64_t f = (int64_t)c * p + j;
        const double b = base ? base[f] : 0.0;
        const double o = __dadd_rn(__dmul_rn(scale, acc[c]), __dmul_rn(lam, b));
        out[f] = o;
        bo += b * o;
        bb += b * b;
      }
    }
  }
  if (dots == nullptr) return;
  const double so = block_sum<kCsrThreads>(bo, sh);
  const double sb = block_sum<kCsrThreads>(bb, sh);
  if (threadIdx.x == 0) {
    dots[blockIdx.x] = so;
    dots[kDotBlocks + blockIdx.x] = sb;
  }
}

// ---------------------------------------------------------------- sample gather
__global__ void fill_i32_kernel(int32_t *a, int64_t n, int32_t v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

__global__ void sample_rowlen_kernel(const int64_t *__restrict__ indptr,
                                     const int64_t *__restrict__ rows, int64_t m,
                                     int64_t *__restrict__ len) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = rows[r];
    len[r] = indptr[i + 1] - indptr[i];
  }
}

// Exclusive scan of in[0..n) into out[0..n] (out[n] = total); one block.
__global__ void __launch_bounds__(1024) scan_kernel(const int64_t *__restrict__ in, int64_t n,
                                                    int64_t *__restrict__ out) {
  __shared__ int64_t sh[1024];
  const int t = threadIdx.x;
  const int64_t per = (n + 1023) / 1024;
  const int64_t b0 = t * per, b1 = min(n, b0 + per);
  int64_t s = 0;
#pragma unroll 8
  for (int64_t i = b0; i < b1; ++i) s += __ldg(in + i);
  sh[t] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {  // Hillis-Steele inclusive scan of the chunk sums
    const int64_t v = t >= o ? sh[t - o] : 0;
    __syncthreads();
    sh[t] += v;
    __syncthreads();
  }
  int64_t run = sh[t] - s;
#pragma unroll 8
  for (int64_t i = b0; i < b1; ++i) {
    const int64_t v = __ldg(in + i);
    out[i] = run;
    run += v;
  }
  if (t == 1023) out[n] = sh[1023];
}

// Sample CSR: warp per sample row copies the row's entries (dataset.py:90-97).
__global__ void __launch_bounds__(kCsrThreads)
    sample_copy_kernel(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                       const double *__restrict__ data, const int64_t *__restrict__ rows,
                       int64_t m, const int64_t *__restrict__ sptr, int32_t *__restrict__ sind,
                       double *__restrict__ sdat) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t r = (int64_t)blockIdx.x * kCsrWarps + warp; r < m;
       r += (int64_t)gridDim.x * kCsrWarps) {
    const int64_t i = rows[r], e0 = indptr[i], e1 = indptr[i + 1], o = sptr[r];
    for (int64_t t = e0 + lane; t < e1; t += 32) {
      sind[o + (t - e0)] = indices[t];
      sdat[o + (t - e0)] = data[t];
    }
  }
}

// pos[i] = first position of row i in the sorted sample, mult[i] = its count
// (duplicates only with replacement, sampling.py:41-42).
__global__ void sample_mark_kernel(const int64_t *__restrict__ rows, int64_t m,
                                   int32_t *__restrict__ pos, int32_t *__restrict__ mult) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = rows[r];
    if (r > 0 && rows[r - 1] == i) continue;
    int64_t e = r + 1;
    while (e < m && rows[e] == i) ++e;
    pos[i] = (int32_t)r;
    mult[i] = (int32_t)(e - r);
  }
}

__global__ void __launch_bounds__(kCsrThreads)
    sample_colcount_kernel(const int64_t *__restrict__ colptr, const int32_t *__restrict__ rowidx,
                           int p, const int32_t *__restrict__ pos, int64_t *__restrict__ cnt) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = blockIdx.x * kCsrWarps + warp; j < p; j += gridDim.x * kCsrWarps) {
    int64_t c = 0;
    for (int64_t t = colptr[j] + lane; t < colptr[j + 1]; t += 32) c += pos[rowidx[t]] >= 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[j] = c;
  }
}

// Sample CSC: the full column filtered to sampled rows (order kept: ballot
// compaction), rows renumbered to sample positions, duplicated rows weighted
// by their multiplicity (their U rows are identical).
__global__ void __launch_bounds__(kCsrThreads)
    sample_colfill_kernel(const int64_t *__restrict__ colptr, const int32_t *__restrict__ rowidx,
                          const double *__restrict__ cdata, int p, const int32_t *__restrict__ pos,
                          const int32_t *__restrict__ mult, const int64_t *__restrict__ scol,
                          int32_t *__restrict__ srow, double *__restrict__ sdat) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = blockIdx.x * kCsrWarps + warp; j < p; j += gridDim.x * kCsrWarps) {
    int64_t o = scol[j];
    const int64_t e1 = colptr[j + 1];
    for (int64_t t0 = colptr[j]; t0 < e1; t0 += 32) {
      const int64_t t = t0 + lane;
      int32_t q = -1, i = 0;
      if (t < e1) {
        i = rowidx[t];
        q = pos[i];
      }
      const unsigned keep = __ballot_sync(0xffffffffu, q >= 0);
      if (q >= 0) {
        const int64_t at = o + __popc(keep & ((1u << lane) - 1u));
        srow[at] = q;
        const int32_t k = mult[i];
        sdat[at] = k == 1 ? cdata[t] : __dmul_rn((double)k, cdata[t]);
      }
      o += __popc(keep);
    }
  }
}

// ---------------------------------------------------------------- column scaling
// normalize_columns on CSR storage (dataset.py:103-107 column_norms: sum of the
// squared stored values per column; :109-118 scale_columns: data *= scale[col]).
// Norms come from the CSC copy (one warp per column, lane-strided + butterfly:
// fixed order); both copies are scaled.
__global__ void __launch_bounds__(kCsrThreads)
    csc_colnorm_kernel(const int64_t *__restrict__ colptr, const double *__restrict__ cdata,
                       int p, double *__restrict__ norms, double *__restrict__ scale) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = blockIdx.x * kCsrWarps + warp; j < p; j += gridDim.x * kCsrWarps) {
    double acc = 0.0;
    for (int64_t t = colptr[j] + lane; t < colptr[j + 1]; t += 32) {
      const double v = cdata[t];
      acc += v * v;
    }
    acc = warp_allsum(acc);
    if (lane == 0) {
      const double nj = sqrt(acc);
      if (norms) norms[j] = nj;
      scale[j] = nj > 0.0 ? __ddiv_rn(1.0, nj) : 1.0;
    }
  }
}

__global__ void scale_entries_kernel(const int32_t *__restrict__ col_of, const double *__restrict__ in,
                                     int64_t nnz, const double *__restrict__ scale,
                                     double *__restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nnz;
       t += (int64_t)gridDim.x * blockDim.x)
    out[t] = __dmul_rn(in[t], scale[col_of[t]]);
}

__global__ void csc_col_index_kernel(const int64_t *__restrict__ colptr, int p,
                                     int32_t *__restrict__ col_of) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = blockIdx.x * kCsrWarps + warp; j < p; j += gridDim.x * kCsrWarps)
    for (int64_t t = colptr[j] + lane; t < colptr[j + 1]; t += 32) col_of[t] = j;
}

template <typename Fn>
int dispatch_k(int K, Fn &&fn) {
  switch (K) {
#define SNX_K(k) \
  case k:        \
    return fn(std::integral_constant<int, k>());
    SNX_K(1) SNX_K(2) SNX_K(3) SNX_K(4) SNX_K(5) SNX_K(6) SNX_K(7) SNX_K(8)
    SNX_K(9) SNX_K(10) SNX_K(11) SNX_K(12) SNX_K(13) SNX_K(14) SNX_K(15) SNX_K(16)
    SNX_K(17) SNX_K(18) SNX_K(19) SNX_K(20) SNX_K(21) SNX_K(22) SNX_K(23) SNX_K(24)
    SNX_K(25) SNX_K(26) SNX_K(27) SNX_K(28) SNX_K(29) SNX_K(30) SNX_K(31) SNX_K(32)
#undef SNX_K
    default:
      set_error("snx_csr: K = %d weighted classes not supported (1..32)", K);
      return 1;
  }
}

int check_ws(const char *who, int64_t n, int p, int K, size_t ws_bytes) {
  const size_t need = csr_ws_layout(n, p, K, nullptr, nullptr);
  if (ws_bytes < need) {
    set_error("%s: workspace of %zu bytes < %zu", who, ws_bytes, need);
    return 1;
  }
  if (K < 1 || K > 32 || p < 0 || n < 0) {
    set_error("%s: bad shape (n=%lld, p=%d, K=%d)", who, (long long)n, p, K);
    return 1;
  }
  return 0;
}

}  // namespace
}  // namespace snx

using namespace snx;

extern "C" {

size_t snx_csr_workspace_bytes(int64_t nrows, int32_t p, int32_t K) {
  if (K > 32) {  // the wide-class passes (and the row gather's K = 1 layout)
    const size_t a = csr_ws_layout(nrows, p, 1, nullptr, nullptr);
    const size_t b = snx::wide::csr_wide_ws_bytes(nrows, p, K);
    return a > b ? a : b;
  }
  return csr_ws_layout(nrows, p, K, nullptr, nullptr);
}

int snx_csr_column_norms(const int64_t *colptr, const double *cdata, int32_t p, double *norms,
                         double *scale, void *stream) {
  if (p <= 0) return 0;
  csc_colnorm_kernel<<<148 * 4, kCsrThreads, 0, (cudaStream_t)stream>>>(colptr, cdata, p, norms,
                                                                       scale);
  return check_launch("csc_colnorm");
}

int snx_csr_scale_columns(const int32_t *indices, const double *data, const int64_t *colptr,
                          const double *cdata, int64_t nnz, int32_t p, const double *scale,
                          double *data_out, double *cdata_out, int32_t *col_scratch,
                          void *stream) {
  if (nnz == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  scale_entries_kernel<<<148 * 8, 256, 0, st>>>(indices, data, nnz, scale, data_out);
  if (check_launch("scale_entries(csr)")) return 1;
  csc_col_index_kernel<<<148 * 4, kCsrThreads, 0, st>>>(colptr, p, col_scratch);
  if (check_launch("csc_col_index")) return 1;
  scale_entries_kernel<<<148 * 8, 256, 0, st>>>(col_scratch, cdata, nnz, scale, cdata_out);
  return check_launch("scale_entries(csc)");
}

int snx_csr_objective(const int64_t *indptr, const int32_t *indices, const double *data,
                      int64_t nrows, int32_t p, int32_t K, const int32_t *labels, const double *w,
                      const double *dir, double alpha, double *out, int64_t *correct_out,
                      void *ws, size_t ws_bytes, void *stream) {
  if (K > 32)
    return wide::csr_wide_objective(indptr, indices, data, nrows, p, K, labels, w, dir, alpha,
                                    out, correct_out, ws, ws_bytes, (cudaStream_t)stream);
  if (check_ws("snx_csr_objective", nrows, p, K, ws_bytes)) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  CsrWs W;
  csr_ws_layout(nrows, p, K, static_cast<char *>(ws), &W);
  int rc = dispatch_k(K, [&](auto kk) {
    constexpr int KK = decltype(kk)::value;
    csr_prep_w_kernel<KK><<<kDotBlocks, kCsrThreads, 0, st>>>(w, dir, alpha, p, W.wt, W.wsq_part,
                                                             nullptr);
    if (check_launch("csr_prep_w")) return 1;
    csr_rows_kernel<KK><<<kRowBlocks, kCsrThreads, 0, st>>>(
        kObj, indptr, indices, data, nrows, W.wt, labels, nullptr, nullptr, W.loss_part,
        correct_out ? W.corr_part : nullptr, nullptr);
    return check_launch("csr_rows(objective)");
  });
  if (rc) return rc;
  csr_final_kernel<<<1, 32, 0, st>>>(W.loss_part, W.corr_part, W.wsq_part, out,
                                     reinterpret_cast<long long *>(correct_out));
  return check_launch("csr_final");
}

int snx_csr_class_probabilities(const int64_t *indptr, const int32_t *indices,
                                const double *data, int64_t nrows, int32_t p, int32_t K,
                                const int32_t *labels, const double *w, double *probs_out,
                                int32_t *pred_out, double *stats_out, void *ws, size_t ws_bytes,
                                void *stream) {
  if (K > 32)
    return wide::csr_wide_probs(indptr, indices, data, nrows, p, K, labels, w, probs_out,
                                pred_out, stats_out, ws, ws_bytes, (cudaStream_t)stream);
  if (check_ws("snx_csr_class_probabilities", nrows, p, K, ws_bytes)) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  CsrWs W;
  csr_ws_layout(nrows, p, K, static_cast<char *>(ws), &W);
  return dispatch_k(K, [&](auto kk) {
    constexpr int KK = decltype(kk)::value;
    csr_prep_w_kernel<KK><<<kDotBlocks, kCsrThreads, 0, st>>>(w, nullptr, 0.0, p, W.wt, nullptr,
                                                             nullptr);
    if (check_launch("csr_prep_w")) return 1;
    csr_rows_kernel<KK><<<kRowBlocks, kCsrThreads, 0, st>>>(
        kProbs, indptr, indices, data, nrows, W.wt, labels, nullptr, probs_out, nullptr, nullptr,
        nullptr, pred_out, stats_out);
    return check_launch("csr_rows(probabilities)");
  });
}

int snx_csr_objective_grad(const int64_t *indptr, const int32_t *indices, const double *data,
                           const int64_t *colptr, const int32_t *rowidx, const double *cdata,
                           int64_t nrows, int32_t p, int32_t K, const int32_t *labels,
                           const double *w, double scale, double lam, double *out, double *G_out,
                           void *ws, size_t ws_bytes, void *stream) {
  if (K > 32)
    return wide::csr_wide_objective_grad(indptr, indices, data, colptr, rowidx, cdata, nrows, p,
                                         K, labels, w, scale, lam, out, G_out, ws, ws_bytes,
                                         (cudaStream_t)stream);
  if (check_ws("snx_csr_objective_grad", nrows, p, K, ws_bytes)) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  CsrWs W;
  csr_ws_layout(nrows, p, K, static_cast<char *>(ws), &W);
  return dispatch_k(K, [&](auto kk) {
    constexpr int KK = decltype(kk)::value;
    csr_prep_w_kernel<KK><<<kDotBlocks, kCsrThreads, 0, st>>>(w, nullptr, 0.0, p, W.wt,
                                                             W.wsq_part, nullptr);
    if (check_launch("csr_prep_w")) return 1;
    csr_rows_kernel<KK><<<kRowBlocks, kCsrThreads, 0, st>>>(kGrad, indptr, indices, data, nrows,
                                                           W.wt, labels, nullptr, W.rowbuf,
                                                           W.loss_part, nullptr, nullptr);
    if (check_launch("csr_rows(gradient)")) return 1;
    csr_final_kernel<<<1, 32, 0, st>>>(W.loss_part, W.corr_part, W.wsq_part, out, nullptr);
    if (check_launch("csr_final")) return 1;
    csc_cols_kernel<KK><<<kDotBlocks, kCsrThreads, 0, st>>>(colptr, rowidx, cdata, p, W.rowbuf,
                                                           scale, lam, w, G_out, nullptr, nullptr);
    return check_launch("csc_cols(gradient)");
  });
}

int snx_csr_gather(const int64_t *indptr, const int32_t *indices, const double *data,
                   const int64_t *colptr, const int32_t *rowidx, const double *cdata,
                   int64_t nrows, int32_t p, const int64_t *rows, int64_t m, int64_t *s_indptr,
                   int32_t *s_indices, double *s_data, int64_t *s_colptr, int32_t *s_rowidx,
                   double *s_cdata, void *ws, size_t ws_bytes, void *stream) {
  if (check_ws("snx_csr_gather", nrows, p, 1, ws_bytes)) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  CsrWs W;
  csr_ws_layout(nrows, p, 1, static_cast<char *>(ws), &W);
  const int grid = 148 * 4;
  sample_rowlen_kernel<<<grid, 256, 0, st>>>(indptr, rows, m, W.scan);
  scan_kernel<<<1, 1024, 0, st>>>(W.scan, m, s_indptr);
  sample_copy_kernel<<<grid, kCsrThreads, 0, st>>>(indptr, indices, data, rows, m, s_indptr,
                                                    s_indices, s_data);
  if (check_launch("csr_gather(rows)")) return 1;
  fill_i32_kernel<<<grid, 256, 0, st>>>(W.pos, nrows, -1);
  sample_mark_kernel<<<grid, 256, 0, st>>>(rows, m, W.pos, W.mult);
  sample_colcount_kernel<<<grid, kCsrThreads, 0, st>>>(colptr, rowidx, p, W.pos, W.scan);
  scan_kernel<<<1, 1024, 0, st>>>(W.scan, p, s_colptr);
  sample_colfill_kernel<<<grid, kCsrThreads, 0, st>>>(colptr, rowidx, cdata, p, W.pos, W.mult,
                                                       s_colptr, s_rowidx, s_cdata);
  return check_launch("csr_gather(columns)");
}

int snx_csr_hess_prepare(const int64_t *indptr, const int32_t *indices, const double *data,
                         int64_t nrows, int32_t p, int32_t K, const double *w, double *H_out,
                         void *ws, size_t ws_bytes, void *stream) {
  if (K > 32)
    return wide::csr_wide_hess_prepare(indptr, indices, data, nrows, p, K, w, H_out, ws, ws_bytes,
                                       (cudaStream_t)stream);
  if (check_ws("snx_csr_hess_prepare", nrows, p, K, ws_bytes)) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  CsrWs W;
  csr_ws_layout(nrows, p, K, static_cast<char *>(ws), &W);
  return dispatch_k(K, [&](auto kk) {
    constexpr int KK = decltype(kk)::value;
    csr_prep_w_kernel<KK><<<kDotBlocks, kCsrThreads, 0, st>>>(w, nullptr, 0.0, p, W.wt, nullptr,
                                                             nullptr);
    if (check_launch("csr_prep_w")) return 1;
    csr_rows_kernel<KK><<<kRowBlocks, kCsrThreads, 0, st>>>(kPrep, indptr, indices, data, nrows,
                                                           W.wt, nullptr, nullptr, H_out, nullptr,
                                                           nullptr, nullptr);
    return check_launch("csr_rows(prepare)");
  });
}

int snx_csr_hess_apply(const int64_t *indptr, const int32_t *indices, const double *data,
                       const int64_t *colptr, const int32_t *rowidx, const double *cdata,
                       int64_t nrows, int32_t p, int32_t K, const double *H, const double *v,
                       double scale, double lam, double *Hv_out, double *dots, const double *skip,
                       void *ws, size_t ws_bytes, void *stream) {
  if (K > 32)
    return wide::csr_wide_hess_apply(indptr, indices, data, colptr, rowidx, cdata, nrows, p, K, H,
                                     v, scale, lam, Hv_out, dots, skip, ws, ws_bytes,
                                     (cudaStream_t)stream);
  if (check_ws("snx_csr_hess_apply", nrows, p, K, ws_bytes)) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  CsrWs W;
  csr_ws_layout(nrows, p, K, static_cast<char *>(ws), &W);
  return dispatch_k(K, [&](auto kk) {
    constexpr int KK = decltype(kk)::value;
    csr_prep_w_kernel<KK><<<kDotBlocks, kCsrThreads, 0, st>>>(v, nullptr, 0.0, p, W.wt, nullptr,
                                                             skip);
    if (check_launch("csr_prep_w")) return 1;
    csr_rows_kernel<KK><<<kRowBlocks, kCsrThreads, 0, st>>>(kApply, indptr, indices, data, nrows,
                                                           W.wt, nullptr, H, W.rowbuf, nullptr,
                                                           nullptr, skip);
    if (check_launch("csr_rows(apply)")) return 1;
    csc_cols_kernel<KK><<<kDotBlocks, kCsrThreads, 0, st>>>(colptr, rowidx, cdata, p, W.rowbuf,
                                                           scale, lam, v, Hv_out, dots, skip);
    return check_launch("csc_cols(apply)");
  });
}

}  // extern "C"
