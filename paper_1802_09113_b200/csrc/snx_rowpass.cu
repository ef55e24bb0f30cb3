// Row-pass kernels: the two feature products of every softmax quantity.
//
//   GEMM1 + row epilogue  (rowpass_kernel): z_r = X[row_r] . W  (K logits per
//       row, softmax.py:91 / :206) followed by the per-row softmax algebra of
//       softmax.py:85-99 (objective, accuracy), :157-161 (gradient residual),
//       :189-195 (Hessian probabilities) or :206-208 (ComputeU).
//   GEMM2 (xtu_kernel + finalize_kernel): out = scale * X_rows^T U + lam * base
//       (softmax.py:162 / :209-210) with a split over rows and a fixed-order
//       reduction of the split partials (no float atomics => reruns are
//       bit-identical).
//
// v1 layout: X row-major (ldx), rows optionally gathered through an index
// array (the sample S_H / S_g, no materialised X_S copy).  GEMM1 maps lanes to
// features with 16-byte vector loads (coalesced row streams) and one warp to
// RW rows; GEMM2 maps threads to feature columns and streams rows.
#include <stdarg.h>
#include <stdio.h>

#include "snx_common.cuh"
#include "snx_internal.h"

namespace snx {

enum Mode { kObjective = 0, kGradient = 1, kHessPrep = 2, kHessApply = 3 };

struct RowArgs {
  const void *X;
  int64_t ldx;
  const int64_t *rows;
  int64_t nrows;
  int P;
  const int32_t *labels;
  const void *W;      // K*P weights (X dtype), class-major
  const void *H;      // kHessApply: nrows*K probabilities (X dtype)
  void *rowout;       // nrows*K: R (gradient), h (prep), U (apply)
  double *loss_part;  // per-block partial losses
  unsigned long long *corr_part;
  unsigned *counter;
  double *loss_out;
  long long *corr_out;
  const double *skip;
};

constexpr int kWarps = 8;

template <typename T, int K, int MODE, int RW>
__global__ void __launch_bounds__(kWarps * 32) rowpass_kernel(RowArgs a) {
  if (a.skip != nullptr && *a.skip != 0.0) return;
  constexpr int V = Vec<T>::N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r0 = ((int64_t)blockIdx.x * kWarps + warp) * RW;
  const T *__restrict__ X = static_cast<const T *>(a.X);
  const T *__restrict__ W = static_cast<const T *>(a.W);

  const T *xr[RW];
#pragma unroll
  for (int q = 0; q < RW; ++q) {
    int64_t r = r0 + q;
    if (r >= a.nrows) r = a.nrows - 1;  // clamp; results of padding rows are dropped
    const int64_t g = a.rows ? a.rows[r] : r;
    xr[q] = X + g * a.ldx;
  }

  T acc[RW][K];
#pragma unroll
  for (int q = 0; q < RW; ++q)
#pragma unroll
    for (int c = 0; c < K; ++c) acc[q][c] = T(0);

  for (int j = lane * V; j < a.P; j += 32 * V) {
    T w[K][V];
#pragma unroll
    for (int c = 0; c < K; ++c) ldv(W + (size_t)c * a.P + j, w[c]);
#pragma unroll
    for (int q = 0; q < RW; ++q) {
      T x[V];
      ldv(xr[q] + j, x);
#pragma unroll
      for (int c = 0; c < K; ++c)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[q][c] = fma(x[v], w[c][v], acc[q][c]);
    }
  }
#pragma unroll
  for (int q = 0; q < RW; ++q)
#pragma unroll
    for (int c = 0; c < K; ++c) acc[q][c] = warp_allsum(acc[q][c]);

  // lane q < RW runs the epilogue of row r0+q in fp64
  double z[K];
#pragma unroll
  for (int c = 0; c < K; ++c) z[c] = (double)acc[0][c];
#pragma unroll
  for (int q = 1; q < RW; ++q)
    if (lane == q) {
#pragma unroll
      for (int c = 0; c < K; ++c) z[c] = (double)acc[q][c];
    }
  const int64_t r = r0 + lane;
  const bool mine = lane < RW && r < a.nrows;
  double loss = 0.0;
  unsigned long long corr = 0;
  if (mine) {
    const int64_t g = a.rows ? a.rows[r] : r;
    if (MODE == kHessApply) {
      // softmax.py:206-208: VW = V*W; U = VW - W*rowsum(VW)
      const T *h = static_cast<const T *>(a.H) + r * K;
      double hw[K], vw[K], s = 0.0;
#pragma unroll
      for (int c = 0; c < K; ++c) {
        hw[c] = (double)h[c];
        vw[c] = z[c] * hw[c];
        s += vw[c];
      }
      T *u = static_cast<T *>(a.rowout) + r * K;
#pragma unroll
      for (int c = 0; c < K; ++c) u[c] = (T)(vw[c] - hw[c] * s);
    } else {
      // softmax.py:91-98: M = max(0, max_c z); E = exp(z - M); alpha = e^-M + sum E
      double M = 0.0;
#pragma unroll
      for (int c = 0; c < K; ++c) M = (z[c] > M || isnan(z[c])) ? z[c] : M;  // NaN propagates
      double E[K], alpha = exp(-M);
      double se = 0.0;
#pragma unroll
      for (int c = 0; c < K; ++c) {
        E[c] = exp(z[c] - M);
        se += E[c];
      }
      alpha += se;
      if (MODE == kHessPrep) {
        T *h = static_cast<T *>(a.rowout) + r * K;
#pragma unroll
        for (int c = 0; c < K; ++c) h[c] = (T)(E[c] / alpha);
      } else {
        const int y = a.labels[g];
        double lin = 0.0;
#pragma unroll
        for (int c = 0; c < K; ++c)
          if (c == y) lin = z[c];
        loss = (M + log(alpha)) - lin;  // softmax.py:134
        if (MODE == kGradient) {
          T *R = static_cast<T *>(a.rowout) + r * K;
#pragma unroll
          for (int c = 0; c < K; ++c) R[c] = (T)(E[c] / alpha - (c == y ? 1.0 : 0.0));
        } else if (a.corr_out != nullptr) {
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
          corr = (best == y) ? 1ull : 0ull;
        }
      }
    }
  }
  if (MODE == kObjective || MODE == kGradient) {
    // fixed-order per-block sums, then the last block reduces the partials
    __shared__ double sl[kWarps];
    __shared__ unsigned long long sc[kWarps];
    __shared__ bool last;
    double wl = 0.0;
    unsigned long long wc = 0;
#pragma unroll
    for (int q = 0; q < RW; ++q) {
      wl += __shfl_sync(0xffffffffu, loss, q);
      wc += __shfl_sync(0xffffffffu, corr, q);
    }
    if (lane == 0) {
      sl[warp] = wl;
      sc[warp] = wc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double bl = 0.0;
      unsigned long long bc = 0;
#pragma unroll
      for (int i = 0; i < kWarps; ++i) {
        bl += sl[i];
        bc += sc[i];
      }
      a.loss_part[blockIdx.x] = bl;
      a.corr_part[blockIdx.x] = bc;
      __threadfence();
      last = atomicAdd(a.counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      __shared__ double sh[kWarps];
      double t = 0.0;
      unsigned long long tc = 0;
      for (int i = threadIdx.x; i < (int)gridDim.x; i += kWarps * 32) {
        t += ((volatile double *)a.loss_part)[i];
        tc += ((volatile unsigned long long *)a.corr_part)[i];
      }
      const double tot = block_sum<kWarps * 32>(t, sh);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tc += __shfl_xor_sync(0xffffffffu, tc, o);
      __shared__ unsigned long long shc[kWarps];
      if (lane == 0) shc[warp] = tc;
      __syncthreads();
      if (threadIdx.x == 0) {
        unsigned long long ct = 0;
        for (int i = 0; i < kWarps; ++i) ct += shc[i];
        a.loss_out[0] = tot;
        if (a.corr_out) a.corr_out[0] = (long long)ct;
        *a.counter = 0u;  // leave the counter at rest
      }
    }
  }
}

// GEMM2 partials: partial[s][c][j] = sum_{r in split s} X[row_r][j] * U[r][c]
template <typename T, int K>
__global__ void __launch_bounds__(128) xtu_kernel(const T *__restrict__ X, int64_t ldx,
                                                  const int64_t *__restrict__ rows,
                                                  int64_t nrows, int P,
                                                  const T *__restrict__ U, int64_t rps,
                                                  T *__restrict__ partial,
                                                  const double *skip) {
  if (skip != nullptr && *skip != 0.0) return;
  constexpr int V = Vec<T>::N, CH = 64;
  __shared__ T su[CH * K];
  __shared__ int64_t sr[CH];
  const int j = (blockIdx.x * 128 + threadIdx.x) * V;
  const bool active = j < P;
  const int64_t rb = (int64_t)blockIdx.y * rps;
  const int64_t re = min(rb + rps, nrows);
  T acc[V][K];
#pragma unroll
  for (int v = 0; v < V; ++v)
#pragma unroll
    for (int c = 0; c < K; ++c) acc[v][c] = T(0);
  for (int64_t c0 = rb; c0 < re; c0 += CH) {
    const int nch = (int)min((int64_t)CH, re - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < nch * K; t += 128) su[t] = U[c0 * K + t];
    for (int t = threadIdx.x; t < nch; t += 128) sr[t] = rows ? rows[c0 + t] : c0 + t;
    __syncthreads();
    if (active) {
#pragma unroll 4
      for (int r = 0; r < nch; ++r) {
        T x[V];
        ldv(X + sr[r] * ldx + j, x);
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const T u = su[r * K + c];
#pragma unroll
          for (int v = 0; v < V; ++v) acc[v][c] = fma(x[v], u, acc[v][c]);
        }
      }
    }
  }
  if (active) {
#pragma unroll
    for (int c = 0; c < K; ++c)
#pragma unroll
      for (int v = 0; v < V; ++v)
        partial[((int64_t)blockIdx.y * K + c) * P + j + v] = acc[v][c];
  }
}

// out[c*p + j] = scale * sum_s partial[s][c*P + j] + lam * base[c*p + j]
// (numpy rounding: two products, one add), optional per-block partials of
// base.out and base.base (the CG curvature test).
template <typename T>
__global__ void __launch_bounds__(kDotThreads)
    finalize_kernel(const T *__restrict__ partial, int64_t splits, int K, int p, int P,
                    double scale, double lam, const double *__restrict__ base,
                    double *__restrict__ out, double *dots, const double *skip) {
  if (skip != nullptr && *skip != 0.0) return;
  __shared__ double sh[kDotThreads / 32];
  double bo = 0.0, bb = 0.0;
  const int64_t d = (int64_t)K * p, stride = (int64_t)K * P;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
       i += (int64_t)kDotBlocks * kDotThreads) {
    const int64_t c = i / p;
    const int64_t pi = c * P + (i - c * p);
    double s = 0.0;
    for (int64_t k = 0; k < splits; ++k) s += (double)partial[k * stride + pi];
    const double b = base[i];
    const double o = __dadd_rn(__dmul_rn(scale, s), __dmul_rn(lam, b));
    out[i] = o;
    bo += b * o;
    bb += b * b;
  }
  if (dots != nullptr) {
    const double so = block_sum<kDotThreads>(bo, sh);
    const double sb = block_sum<kDotThreads>(bb, sh);
    if (threadIdx.x == 0) {
      dots[blockIdx.x] = so;
      dots[kDotBlocks + blockIdx.x] = sb;
    }
  }
}

// ---------------------------------------------------------------- host side
Geometry geometry(int dtype, int64_t nrows, int32_t P) {
  Geometry g{};
  g.rows_per_warp = 4;
  g.warps = kWarps;
  const int64_t per_block = (int64_t)g.rows_per_warp * g.warps;
  g.rowpass_blocks = nrows > 0 ? (nrows + per_block - 1) / per_block : 0;
  const int V = dtype == SNX_F64 ? 2 : 4;
  g.xtu_tiles = (P + 128 * V - 1) / (128 * V);
  if (g.xtu_tiles < 1) g.xtu_tiles = 1;
  int64_t s = (4 * 148 + g.xtu_tiles - 1) / g.xtu_tiles;
  const int64_t by_rows = (nrows + 31) / 32;
  if (s > by_rows) s = by_rows;
  if (s > 128) s = 128;
  if (s < 1) s = 1;
  g.rows_per_split = nrows > 0 ? (nrows + s - 1) / s : 1;
  g.splits = nrows > 0 ? (nrows + g.rows_per_split - 1) / g.rows_per_split : 1;
  return g;
}

Workspace workspace_layout(int dtype, int64_t nrows, int32_t p, int32_t K) {
  const int32_t P = padded(p);
  const Geometry g = geometry(dtype, nrows, P);
  const size_t tb = dtype_bytes(dtype);
  Workspace w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = round_up(off + bytes, 256);
    return o;
  };
  w.weights = take((size_t)K * P * tb);
  w.rowbuf = take((size_t)(nrows > 0 ? nrows : 1) * K * tb);
  w.partial = take((size_t)g.splits * K * P * tb);
  w.loss_part = take((size_t)(g.rowpass_blocks + 1) * 8);
  w.corr_part = take((size_t)(g.rowpass_blocks + 1) * 8);
  w.dot_part = take((size_t)4 * kDotBlocks * 8);
  w.counters = take(16 * 4);
  w.total = off;
  return w;
}

template <typename T, int K>
static void launch_rowpass(int mode, const RowArgs &a, int64_t blocks, cudaStream_t st) {
  const dim3 grid((unsigned)blocks), block(kWarps * 32);
  switch (mode) {
    case kObjective: rowpass_kernel<T, K, kObjective, 4><<<grid, block, 0, st>>>(a); break;
    case kGradient: rowpass_kernel<T, K, kGradient, 4><<<grid, block, 0, st>>>(a); break;
    case kHessPrep: rowpass_kernel<T, K, kHessPrep, 4><<<grid, block, 0, st>>>(a); break;
    default: rowpass_kernel<T, K, kHessApply, 4><<<grid, block, 0, st>>>(a); break;
  }
}

template <typename T, int K>
static void launch_xtu(const RowArgs &a, const Geometry &g, const void *U, void *partial,
                       const double *skip, cudaStream_t st) {
  const dim3 grid((unsigned)g.xtu_tiles, (unsigned)g.splits), block(128);
  xtu_kernel<T, K><<<grid, block, 0, st>>>(static_cast<const T *>(a.X), a.ldx, a.rows,
                                           a.nrows, a.P, static_cast<const T *>(U),
                                           g.rows_per_split, static_cast<T *>(partial), skip);
}

#define SNX_K_SWITCH(K, CALL)                         \
  switch (K) {                                        \
    case 1: { constexpr int KK = 1; CALL; } break;    \
    case 2: { constexpr int KK = 2; CALL; } break;    \
    case 3: { constexpr int KK = 3; CALL; } break;    \
    case 4: { constexpr int KK = 4; CALL; } break;    \
    case 5: { constexpr int KK = 5; CALL; } break;    \
    case 6: { constexpr int KK = 6; CALL; } break;    \
    case 7: { constexpr int KK = 7; CALL; } break;    \
    case 8: { constexpr int KK = 8; CALL; } break;    \
    case 9: { constexpr int KK = 9; CALL; } break;    \
    case 10: { constexpr int KK = 10; CALL; } break;  \
    case 11: { constexpr int KK = 11; CALL; } break;  \
    case 12: { constexpr int KK = 12; CALL; } break;  \
    case 13: { constexpr int KK = 13; CALL; } break;  \
    case 14: { constexpr int KK = 14; CALL; } break;  \
    case 15: { constexpr int KK = 15; CALL; } break;  \
    case 16: { constexpr int KK = 16; CALL; } break;  \
    default: break;                                   \
  }

static int validate(int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p,
                    int32_t K, void *ws, size_t ws_bytes) {
  if (dtype != SNX_F64 && dtype != SNX_F32) {
    set_error("snx: unknown dtype %d", dtype);
    return 1;
  }
  if (K < 1 || K > 16) {
    set_error("snx: K = C-1 = %d outside the supported range [1, 16]", K);
    return 1;
  }
  if (p < 1 || ldx < padded(p) || ldx % 4 != 0) {
    set_error("snx: p=%d needs ldx >= round_up(p,4) and ldx %% 4 == 0 (ldx=%lld)", p,
              (long long)ldx);
    return 1;
  }
  if (nrows < 0) {
    set_error("snx: negative row count");
    return 1;
  }
  if (nrows > 0 && X == nullptr) {
    set_error("snx: X is NULL");
    return 1;
  }
  const Workspace w = workspace_layout(dtype, nrows, p, K);
  if (ws == nullptr || ws_bytes < w.total) {
    set_error("snx: workspace too small (%zu < %zu bytes)", ws_bytes, w.total);
    return 1;
  }
  return 0;
}

// Common driver of the four row-pass entry points.
static int rowpass(int mode, int dtype, const void *X, int64_t ldx, const int64_t *rows,
                   int64_t nrows, int32_t p, int32_t K, const int32_t *labels,
                   const double *w, const double *dir, double alpha, const void *H,
                   void *rowout, double scale, double lam, const double *base, double *out,
                   long long *corr_out, double *vec_out, double *dots, const double *skip,
                   void *ws, size_t ws_bytes, cudaStream_t st) {
  if (validate(dtype, X, ldx, nrows, p, K, ws, ws_bytes)) return 1;
  const int32_t P = padded(p);
  const Geometry g = geometry(dtype, nrows, P);
  const Workspace lay = workspace_layout(dtype, nrows, p, K);
  char *wsb = static_cast<char *>(ws);
  unsigned *counters = reinterpret_cast<unsigned *>(wsb + lay.counters);
  double *dotp = reinterpret_cast<double *>(wsb + lay.dot_part);

  // Weights in the X dtype, padded to P columns (and ||w_eff||^2 for the
  // objective's regulariser).
  const void *Wt = w;
  const bool need_wsq = (mode == kObjective || mode == kGradient) && out != nullptr;
  const bool convert = dtype == SNX_F32 || dir != nullptr || P != p;
  if (convert || need_wsq) {
    void *dst = convert ? (void *)(wsb + lay.weights) : nullptr;
    if (launch_prep_weights(dtype, w, dir, alpha, K, p, P, dst, dotp, counters + 1,
                            need_wsq ? out + 1 : nullptr, st))
      return 1;
    if (dst) Wt = dst;
  }
  if (nrows == 0) {
    // empty dataset: data terms vanish (tests/test_softmax.py:121-125,146-151)
    if (mode == kObjective || mode == kGradient) {
      if (cudaMemsetAsync(out, 0, sizeof(double), st) != cudaSuccess)
        return check_launch("memset");
      if (corr_out && cudaMemsetAsync(corr_out, 0, sizeof(long long), st) != cudaSuccess)
        return check_launch("memset");
    }
    if (mode == kHessPrep) return 0;
    if (mode == kGradient || mode == kHessApply) {
      // out = lam * base (scale * 0 + lam * base)
      cudaMemsetAsync(wsb + lay.partial, 0, (size_t)K * P * dtype_bytes(dtype), st);
      if (dtype == SNX_F64)
        finalize_kernel<double><<<kDotBlocks, kDotThreads, 0, st>>>(
            reinterpret_cast<const double *>(wsb + lay.partial), 1, K, p, P, scale, lam,
            base, vec_out, dots, skip);
      else
        finalize_kernel<float><<<kDotBlocks, kDotThreads, 0, st>>>(
            reinterpret_cast<const float *>(wsb + lay.partial), 1, K, p, P, scale, lam,
            base, vec_out, dots, skip);
      return check_launch("finalize");
    }
    return check_launch("objective(empty)");
  }

  RowArgs a{};
  a.X = X;
  a.ldx = ldx;
  a.rows = rows;
  a.nrows = nrows;
  a.P = P;
  a.labels = labels;
  a.W = Wt;
  a.H = H;
  a.rowout = rowout ? rowout : (void *)(wsb + lay.rowbuf);
  a.loss_part = reinterpret_cast<double *>(wsb + lay.loss_part);
  a.corr_part = reinterpret_cast<unsigned long long *>(wsb + lay.corr_part);
  a.counter = counters;
  a.loss_out = out;
  a.corr_out = corr_out;
  a.skip = skip;
  if (dtype == SNX_F64) {
    SNX_K_SWITCH(K, (launch_rowpass<double, KK>(mode, a, g.rowpass_blocks, st)));
  } else {
    SNX_K_SWITCH(K, (launch_rowpass<float, KK>(mode, a, g.rowpass_blocks, st)));
  }
  if (check_launch("rowpass")) return 1;
  if (mode == kGradient || mode == kHessApply) {
    void *partial = wsb + lay.partial;
    if (dtype == SNX_F64) {
      SNX_K_SWITCH(K, (launch_xtu<double, KK>(a, g, a.rowout, partial, skip, st)));
      if (check_launch("xtu")) return 1;
      finalize_kernel<double><<<kDotBlocks, kDotThreads, 0, st>>>(
          static_cast<const double *>(partial), g.splits, K, p, P, scale, lam, base, vec_out,
          dots, skip);
    } else {
      SNX_K_SWITCH(K, (launch_xtu<float, KK>(a, g, a.rowout, partial, skip, st)));
      if (check_launch("xtu")) return 1;
      finalize_kernel<float><<<kDotBlocks, kDotThreads, 0, st>>>(
          static_cast<const float *>(partial), g.splits, K, p, P, scale, lam, base, vec_out,
          dots, skip);
    }
    if (check_launch("finalize")) return 1;
  }
  return 0;
}

}  // namespace snx

using namespace snx;

extern "C" {

size_t snx_workspace_bytes(int dtype, int64_t nrows, int32_t p, int32_t K) {
  return workspace_layout(dtype, nrows, p, K).total;
}

int snx_objective(int dtype, const void *X, int64_t ldx, const int64_t *rows, int64_t nrows,
                  int32_t p, int32_t K, const int32_t *labels, const double *w,
                  const double *dir, double alpha, double *out, int64_t *correct_out,
                  void *ws, size_t ws_bytes, void *stream) {
  if (out == nullptr || w == nullptr || (nrows > 0 && labels == nullptr)) {
    set_error("snx_objective: NULL out/w/labels");
    return 1;
  }
  return rowpass(kObjective, dtype, X, ldx, rows, nrows, p, K, labels, w, dir, alpha, nullptr,
                 nullptr, 1.0, 0.0, nullptr, out, reinterpret_cast<long long *>(correct_out),
                 nullptr, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

int snx_objective_grad(int dtype, const void *X, int64_t ldx, const int64_t *rows,
                       int64_t nrows, int32_t p, int32_t K, const int32_t *labels,
                       const double *w, double scale, double lam, double *out, double *G_out,
                       void *ws, size_t ws_bytes, void *stream) {
  if (out == nullptr || w == nullptr || G_out == nullptr || (nrows > 0 && labels == nullptr)) {
    set_error("snx_objective_grad: NULL out/w/G_out/labels");
    return 1;
  }
  return rowpass(kGradient, dtype, X, ldx, rows, nrows, p, K, labels, w, nullptr, 0.0, nullptr,
                 nullptr, scale, lam, w, out, nullptr, G_out, nullptr, nullptr, ws, ws_bytes,
                 (cudaStream_t)stream);
}

int snx_hess_prepare(int dtype, const void *X, int64_t ldx, const int64_t *rows,
                     int64_t nrows, int32_t p, int32_t K, const int32_t *labels,
                     const double *w, void *H_out, void *ws, size_t ws_bytes, void *stream) {
  (void)labels;  // h does not depend on the labels (softmax.py:189-195)
  if (w == nullptr || (nrows > 0 && H_out == nullptr)) {
    set_error("snx_hess_prepare: NULL w/H_out");
    return 1;
  }
  return rowpass(kHessPrep, dtype, X, ldx, rows, nrows, p, K, nullptr, w, nullptr, 0.0,
                 nullptr, H_out, 1.0, 0.0, nullptr, nullptr, nullptr, nullptr, nullptr,
                 nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

int snx_hess_apply(int dtype, const void *X, int64_t ldx, const int64_t *rows, int64_t nrows,
                   int32_t p, int32_t K, const void *H, const double *v, double scale,
                   double lam, double *Hv_out, double *dots, const double *skip, void *ws,
                   size_t ws_bytes, void *stream) {
  if (v == nullptr || Hv_out == nullptr || (nrows > 0 && H == nullptr)) {
    set_error("snx_hess_apply: NULL v/Hv_out/H");
    return 1;
  }
  return rowpass(kHessApply, dtype, X, ldx, rows, nrows, p, K, nullptr, v, nullptr, 0.0, H,
                 nullptr, scale, lam, v, nullptr, nullptr, Hv_out, dots, skip, ws, ws_bytes,
                 (cudaStream_t)stream);
}

}  // extern "C"
