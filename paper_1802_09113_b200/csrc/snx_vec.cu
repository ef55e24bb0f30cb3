// d-vector kernels: weight preparation, dot products, numpy-rounded axpy and
// the device-resident CG iteration of cg.py:51-98.  All of them run on a fixed
// grid of SNX_DOT_BLOCKS blocks so every reduction has one summation order.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>

#include "snx_common.cuh"
#include "snx_internal.h"
#include "snx_pipe.cuh"

namespace snx {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

bool pdl_enabled() {
  // Off by default: measured on B200, dependent CTAs made resident early slow
  // the short epilogue/finalize kernels 2-4x; SNX_PDL=1 re-enables it.
  static int on = -1;
  if (on < 0) {
    const char *e = getenv("SNX_PDL");
    on = (e != nullptr && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

bool gemm2_pdl() {
  static int on = -1;
  if (on < 0) {
    const char *e = getenv("SNX_GEMM2_PDL");
    on = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

void prefer_max_smem(const void *kernel) {
  static const void *seen[256];
  static int nseen = 0;
  for (int i = 0; i < nseen; ++i)
    if (seen[i] == kernel) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  cudaGetLastError();  // the preference is advisory
  if (nseen < 256) seen[nseen++] = kernel;
}

int check_launch(const char *what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("snx: %s failed: %s", what, cudaGetErrorString(e));
    return 1;
  }
  return 0;
}

// Wt[c*P + j] = T(w + alpha*dir)[c*p + j] (zero in the pad columns j >= p);
// block partials of ||w + alpha*dir||^2; the last block writes the total to
// wsq_out (if given).
template <typename T>
__global__ void __launch_bounds__(kDotThreads)
    prep_weights_kernel(const double *__restrict__ w, const double *__restrict__ dir,
                        double alpha, int K, int p, int P, T *__restrict__ Wt, double *part,
                        unsigned *counter, double *wsq_out) {
  pdl_wait();  // successor launches when this grid exits (implicit trigger)
  __shared__ double sh[kDotThreads / 32];
  __shared__ bool last;
  double acc = 0.0;
  const int64_t total = (int64_t)K * P;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < total;
       i += (int64_t)kDotBlocks * kDotThreads) {
    const int64_t c = i / P;
    const int j = (int)(i - c * P);
    double v = 0.0;
    if (j < p) {
      const int64_t f = c * p + j;
      v = dir ? np_axpy(w[f], alpha, dir[f]) : w[f];
      acc += v * v;
    }
    if (Wt) Wt[i] = (T)v;
  }
  if (wsq_out == nullptr) return;
  const double b = block_sum<kDotThreads>(acc, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = b;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    if (threadIdx.x < 32) {
      double t = 0.0;
      const volatile double *vp = part;
#pragma unroll
      for (int i = 0; i < kDotBlocks / 32; ++i) t += vp[threadIdx.x + 32 * i];
      t = warp_allsum(t);
      if (threadIdx.x == 0) {
        *wsq_out = t;
        *counter = 0u;
      }
    }
  }
}

int launch_prep_weights(int dtype, const double *w, const double *dir, double alpha, int K,
                        int p, int P, void *Wt, double *part, unsigned *counter,
                        double *wsq_out, cudaStream_t st) {
  if (dtype == SNX_F64) {
    launch_pdl(prep_weights_kernel<double>, dim3(kDotBlocks), dim3(kDotThreads), 0, st, 
        w, dir, alpha, K, p, P, static_cast<double *>(Wt), part, counter, wsq_out);
  } else {
    launch_pdl(prep_weights_kernel<float>, dim3(kDotBlocks), dim3(kDotThreads), 0, st, 
        w, dir, alpha, K, p, P, static_cast<float *>(Wt), part, counter, wsq_out);
  }
  return check_launch("prep_weights");
}

__global__ void __launch_bounds__(kDotThreads)
    dot_part_kernel(const double *__restrict__ x, const double *__restrict__ y, int64_t d,
                    double *part) {
  pdl_wait();  // successor launches when this grid exits (implicit trigger)
  __shared__ double sh[kDotThreads / 32];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
       i += (int64_t)kDotBlocks * kDotThreads)
    acc += x[i] * y[i];
  const double b = block_sum<kDotThreads>(acc, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = b;
}

__global__ void dot_final_kernel(const double *part, double *out) {
  pdl_wait();  // successor launches when this grid exits (implicit trigger)
  const double t = warp_sum_partials(part);
  if (threadIdx.x == 0) *out = t;
}

__global__ void __launch_bounds__(kDotThreads)
    axpy_kernel(const double *__restrict__ x, const double *__restrict__ p, double alpha,
                int64_t d, double *__restrict__ out) {
  pdl_wait();  // successor launches when this grid exits (implicit trigger)
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
       i += (int64_t)kDotBlocks * kDotThreads)
    out[i] = np_axpy(x[i], alpha, p[i]);
}

__global__ void __launch_bounds__(kDotThreads)
    axpby_kernel(double a, const double *__restrict__ x, double b, const double *__restrict__ y,
                 int64_t d, double *__restrict__ out) {
  pdl_wait();  // successor launches when this grid exits (implicit trigger)
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
       i += (int64_t)kDotBlocks * kDotThreads)
    out[i] = __dadd_rn(__dmul_rn(a, x[i]), __dmul_rn(b, y[i]));
}

__global__ void __launch_bounds__(kDotThreads)
    finish_hv_kernel(const double *__restrict__ v, double lam, int64_t d, double *out,
                     double *dots, const double *skip) {
  pdl_wait();
  if (skip != nullptr && *skip != 0.0) return;
  __shared__ double sh[kDotThreads / 32];
  double bo = 0.0, bb = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
       i += (int64_t)kDotBlocks * kDotThreads) {
    const double b = v[i];
    const double o = np_axpy(out[i], lam, b);
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

#ifdef SNX_TIMELINE
__device__ unsigned long long g_vec_timeline[2][256][2];
#define SNX_VTL(slot, ev)                                              \
  do {                                                                 \
    unsigned long long t_;                                             \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));             \
    g_vec_timeline[slot][blockIdx.x][ev] = t_;                         \
  } while (0)
#else
#define SNX_VTL(slot, ev) \
  do {                    \
  } while (0)
#endif

// ------------------------------------------------------------------ CG (cg.py)

__global__ void __launch_bounds__(kDotThreads)
    cg_init_kernel(const double *__restrict__ g, int64_t d, int max_iters, double *r,
                   double *s, double *p, double *pb, double *state) {
  pdl_wait();  // successor launches when this grid exits (implicit trigger)
  __shared__ double sh[kDotThreads / 32];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
       i += (int64_t)kDotBlocks * kDotThreads) {
    const double gi = g[i];
    r[i] = -gi;  // cg.py:65-69: r = -g, s = r, p = 0, p_best = s
    s[i] = -gi;
    p[i] = 0.0;
    pb[i] = -gi;
    acc += gi * gi;
  }
  const double b = block_sum<kDotThreads>(acc, sh);
  if (threadIdx.x == 0) {
    scratch(state, max_iters)[blockIdx.x] = b;
    scratch(state, max_iters)[kDotBlocks + blockIdx.x] = b;  // s.s of s = -g (fused CG update)
  }
  // zero every slot's flags (block 0)
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < (max_iters + 2) * SNX_CG_SLOT; i += kDotThreads)
      state[i] = 0.0;
}

__global__ void cg_init_final_kernel(double theta, int max_iters, double *state) {
  pdl_wait();  // successor launches when this grid exits (implicit trigger)
  const double gg = warp_sum_partials(scratch(state, max_iters));
  if (threadIdx.x == 0) {
    double *s0 = slot(state, 0);
    const double gn = sqrt(gg);  // np.linalg.norm = sqrt(dot)
    s0[kRs] = gg;                // (-g).(-g) == g.g bitwise
    s0[kBest] = gn;
    s0[kThr] = theta * gn;
    s0[kIters] = 0.0;
    s0[kConv] = gn == 0.0 ? 1.0 : 0.0;
    s0[kDone] = gn == 0.0 ? 1.0 : 0.0;  // cg.py:61-62
  }
}

// Iteration t, part 1 (cg.py:77-86): curvature test, alpha, p += a s, r -= a Hs.
__global__ void __launch_bounds__(kDotThreads)
    cg_step1_kernel(int t, int max_iters, int64_t d, const double *__restrict__ Hs,
                    const double *__restrict__ dots, double *r, const double *s, double *p,
                    double *state) {
  pdl_wait();  // successor launches when this grid exits (implicit trigger)
  if (threadIdx.x == 0) SNX_VTL(0, 0);
  const double *st = slot(state, t);
  if (st[kDone] != 0.0) return;
  __shared__ double sh[kDotThreads / 32];
  __shared__ double s_alpha;
  __shared__ bool s_bad;
  if (threadIdx.x < 32) {
    const double curv = warp_sum_partials(dots);            // s.Hs
    const double ss = warp_sum_partials(dots + kDotBlocks);  // s.s
    if (threadIdx.x == 0) {
      s_bad = curv <= 1e-32 * ss;  // cg.py:16, :79
      s_alpha = st[kRs] / curv;
      if (s_bad && blockIdx.x == 0) {
        slot(state, t + 1)[kErr] = 1.0;
        slot(state, t + 1)[kCurv] = curv;
      }
    }
  }
  __syncthreads();
  if (s_bad) return;
  const double alpha = s_alpha;
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
       i += (int64_t)kDotBlocks * kDotThreads) {
    p[i] = np_axpy(p[i], alpha, s[i]);
    const double ri = np_axmy(r[i], alpha, Hs[i]);
    r[i] = ri;
    acc += ri * ri;
  }
  const double b = block_sum<kDotThreads>(acc, sh);
  if (threadIdx.x == 0) scratch(state, max_iters)[blockIdx.x] = b;
  if (threadIdx.x == 0) SNX_VTL(0, 1);
}

// Iteration t, part 2 (cg.py:87-96): best-iterate copy, stop test, new direction.
__global__ void __launch_bounds__(kDotThreads)
    cg_step2_kernel(int t, int max_iters, int64_t d, const double *__restrict__ r, double *s,
                    const double *__restrict__ p, double *pb, double *state) {
  // the next product's GEMM1 (a programmatic dependent) may stage its X tiles
  // while this runs; it waits for this grid before reading s or the done flag
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) SNX_VTL(1, 0);
  const double *st = slot(state, t);
  double *nx = slot(state, t + 1);
  // the first element's operands load alongside the flags and the r.r
  // partials (no dependent round trip before the update)
  const int64_t i0 = (int64_t)blockIdx.x * kDotThreads + threadIdx.x;
  const double r0 = i0 < d ? r[i0] : 0.0, s0 = i0 < d ? s[i0] : 0.0, p0 = i0 < d ? p[i0] : 0.0;
  const double done = st[kDone], err = nx[kErr];
  __shared__ double s_rr;
  if (threadIdx.x < 32) {
    const double rr = warp_sum_partials(scratch(state, max_iters));
    if (threadIdx.x == 0) s_rr = rr;
  }
  if (done != 0.0) {
    if (blockIdx.x == 0 && threadIdx.x < SNX_CG_SLOT) nx[threadIdx.x] = st[threadIdx.x];
    return;
  }
  if (err != 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      nx[kRs] = st[kRs];
      nx[kBest] = st[kBest];
      nx[kThr] = st[kThr];
      nx[kConv] = 0.0;
      nx[kIters] = t + 1;
      nx[kDone] = 1.0;
    }
    return;
  }
  __syncthreads();
  const double rr = s_rr;
  const double rn = sqrt(rr);
  const bool best = rn <= st[kBest];
  const bool conv = rn <= st[kThr];
  const double beta = rr / st[kRs];
  double ss = 0.0;
  for (int64_t i = i0; i < d; i += (int64_t)kDotBlocks * kDotThreads) {
    const bool first = i == i0;
    if (best) pb[i] = first ? p0 : p[i];
    if (!conv) {
      const double si = np_axpy(first ? r0 : r[i], beta, first ? s0 : s[i]);
      s[i] = si;
      ss += si * si;
    }
  }
  // s.s partials of the new direction (the fused CG update's curvature, second
  // scratch row; every block reaches this point: no early return above here)
  __shared__ double sh2[kDotThreads / 32];
  const double bs = block_sum<kDotThreads>(ss, sh2);
  if (threadIdx.x == 0) scratch(state, max_iters)[kDotBlocks + blockIdx.x] = bs;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    nx[kRs] = conv ? st[kRs] : rr;
    nx[kBest] = best ? rn : st[kBest];
    nx[kThr] = st[kThr];
    nx[kConv] = conv ? 1.0 : 0.0;
    nx[kIters] = t + 1;
    nx[kDone] = (conv || t + 1 >= max_iters) ? 1.0 : 0.0;
  }
  if (threadIdx.x == 0) SNX_VTL(1, 1);
}

// ------------------------------------------------- power iteration (bench.py:116-138)
// state: [rayleigh, ||w||, zero_flag, pad] + kDotBlocks (v.w) + kDotBlocks (w.w) partials.
// Step part 1: block partials of v.w and w.w (skipped once a zero w was seen, so
// the partials of that iteration stay in place).
__global__ void __launch_bounds__(kDotThreads)
    power_part_kernel(const double *__restrict__ v, const double *__restrict__ w, int64_t d,
                      double *state) {
  if (state[2] != 0.0) return;
  __shared__ double sh[kDotThreads / 32];
  double vw = 0.0, ww = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
       i += (int64_t)kDotBlocks * kDotThreads) {
    const double wi = w[i];
    vw += v[i] * wi;
    ww += wi * wi;
  }
  const double a = block_sum<kDotThreads>(vw, sh);
  const double b = block_sum<kDotThreads>(ww, sh);
  if (threadIdx.x == 0) {
    state[4 + blockIdx.x] = a;
    state[4 + kDotBlocks + blockIdx.x] = b;
  }
}

// Step part 2: every block reduces the partials in the same fixed order;
// rayleigh = v.w, ||w|| = sqrt(w.w) (np.linalg.norm); ||w|| == 0 -> the
// estimate is 0 and the iteration stops (bench.py:133-135); else v = w / ||w||.
__global__ void __launch_bounds__(kDotThreads)
    power_scale_kernel(double *__restrict__ v, const double *__restrict__ w, int64_t d,
                       double *state) {
  __shared__ double s_vw, s_nw;
  if (threadIdx.x < 32) {
    const double vw = warp_sum_partials(state + 4);
    const double ww = warp_sum_partials(state + 4 + kDotBlocks);
    if (threadIdx.x == 0) {
      s_vw = vw;
      s_nw = sqrt(ww);
    }
  }
  __syncthreads();
  const double nw = s_nw;
  if (nw == 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      state[0] = 0.0;
      state[1] = 0.0;
      state[2] = 1.0;
    }
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    state[0] = s_vw;
    state[1] = nw;
  }
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
       i += (int64_t)kDotBlocks * kDotThreads)
    v[i] = __ddiv_rn(w[i], nw);
}

// ------------------------------------------------ Steihaug-CG (trust region)
// N&W Alg. 7.2 as in oracle/trust_region.py steihaug_cg, device resident.  state:
// (T + 2) slots of SNX_CG_SLOT doubles, slot j = the scalars entering iteration
// j: [rr, done, boundary, iters, m, tol, -, -], then 4 x kDotBlocks partials
// (z.d | z.z | znew.znew | r.r).  Every kernel of iteration j reads slot j and
// writes slot j + 1 only (no block reads a field another block of the same
// launch writes); every block reduces the partials in the same fixed order.
enum { kTrRs = 0, kTrDone = 1, kTrBnd = 2, kTrIters = 3, kTrM = 4, kTrTol = 5 };

__device__ __forceinline__ double *tr_scratch(double *state, int T) {
  return state + (T + 2) * SNX_CG_SLOT;
}

__global__ void __launch_bounds__(kDotThreads)
    tr_init_kernel(const double *__restrict__ g, int64_t d, int T, double *z, double *r,
                   double *dv, double *state) {
  __shared__ double sh[kDotThreads / 32];
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
       i += (int64_t)kDotBlocks * kDotThreads) {
    const double gi = g[i];
    z[i] = 0.0;
    r[i] = gi;   // r0 = g
    dv[i] = -gi; // d0 = -r0
    acc += gi * gi;
  }
  const double b = block_sum<kDotThreads>(acc, sh);
  if (threadIdx.x == 0) tr_scratch(state, T)[3 * kDotBlocks + blockIdx.x] = b;
  if (blockIdx.x == 0)
    for (int i = threadIdx.x; i < (T + 2) * SNX_CG_SLOT; i += kDotThreads) state[i] = 0.0;
}

__global__ void tr_init_final_kernel(double theta, int T, double *state) {
  const double gg = warp_sum_partials(tr_scratch(state, T) + 3 * kDotBlocks);
  if (threadIdx.x == 0) {
    double *s0 = slot(state, 0);
    const double gn = sqrt(gg);  // np.linalg.norm(g)
    s0[kTrRs] = gg;
    s0[kTrTol] = theta * gn;
    s0[kTrDone] = gn == 0.0 ? 1.0 : 0.0;  // zero step, 0 iterations
  }
}

// Iteration j, part 1: alpha = rr / dHd; znew = z + alpha d; partials of z.d,
// z.z, znew.znew (the boundary root and the |z_{j+1}| >= radius test).
__global__ void __launch_bounds__(kDotThreads)
    tr_step1_kernel(int j, int T, int64_t d, const double *__restrict__ dots,
                    const double *__restrict__ z, const double *__restrict__ dv,
                    double *__restrict__ znew, double *state) {
  const double *st = slot(state, j);
  if (st[kTrDone] != 0.0) return;
  __shared__ double sh[kDotThreads / 32];
  __shared__ double s_a;
  if (threadIdx.x < 32) {
    const double dhd = warp_sum_partials(dots);
    if (threadIdx.x == 0) s_a = st[kTrRs] / dhd;
  }
  __syncthreads();
  const double a = s_a;
  double zd = 0.0, zz = 0.0, nn = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
       i += (int64_t)kDotBlocks * kDotThreads) {
    const double zi = z[i], di = dv[i];
    const double zn = np_axpy(zi, a, di);  // z + a * d
    znew[i] = zn;
    zd += zi * di;
    zz += zi * zi;
    nn += zn * zn;
  }
  double *sc = tr_scratch(state, T);
  const double b0 = block_sum<kDotThreads>(zd, sh);
  const double b1 = block_sum<kDotThreads>(zz, sh);
  const double b2 = block_sum<kDotThreads>(nn, sh);
  if (threadIdx.x == 0) {
    sc[blockIdx.x] = b0;
    sc[kDotBlocks + blockIdx.x] = b1;
    sc[2 * kDotBlocks + blockIdx.x] = b2;
  }
}

// Iteration j, part 2: negative curvature or |znew| >= radius -> the boundary
// step z + tau d (done); else z = znew, r += alpha Hd, partials of r.r.
__global__ void __launch_bounds__(kDotThreads)
    tr_step2_kernel(int j, int T, int64_t d, const double *__restrict__ radius,
                    const double *__restrict__ Hd, const double *__restrict__ dots,
                    double *z, double *r, const double *__restrict__ dv,
                    const double *__restrict__ znew, double *state) {
  const double *st = slot(state, j);
  if (st[kTrDone] != 0.0) return;
  __shared__ double sh[kDotThreads / 32];
  __shared__ double s_v[6];
  if (threadIdx.x < 32) {
    const double *sc = tr_scratch(state, T);
    const double dhd = warp_sum_partials(dots);
    const double dd = warp_sum_partials(dots + kDotBlocks);
    const double zd = warp_sum_partials(sc);
    const double zz = warp_sum_partials(sc + kDotBlocks);
    const double nn = warp_sum_partials(sc + 2 * kDotBlocks);
    if (threadIdx.x == 0) {
      const double rr = st[kTrRs], rad = *radius;
      const bool bnd = dhd <= 0.0 || sqrt(nn) >= rad;
      double step;
      if (bnd) {  // _to_boundary(z, d, radius)
        const double disc = zd * zd + dd * (rad * rad - zz);
        step = (-zd + sqrt(fmax(disc, 0.0))) / dd;
      } else {
        step = rr / dhd;
      }
      s_v[0] = bnd ? 1.0 : 0.0;
      s_v[1] = step;
      s_v[2] = st[kTrM] + (-step * rr + 0.5 * step * step * dhd);
    }
  }
  __syncthreads();
  const bool bnd = s_v[0] != 0.0;
  const double step = s_v[1];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double *nx = slot(state, j + 1);
    nx[kTrRs] = st[kTrRs];
    nx[kTrTol] = st[kTrTol];
    nx[kTrM] = s_v[2];
    nx[kTrBnd] = bnd ? 1.0 : 0.0;
    nx[kTrIters] = j + 1;
    nx[kTrDone] = bnd ? 1.0 : 0.0;
  }
  double acc = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
       i += (int64_t)kDotBlocks * kDotThreads) {
    if (bnd) {
      z[i] = np_axpy(z[i], step, dv[i]);
    } else {
      z[i] = znew[i];
      const double ri = np_axpy(r[i], step, Hd[i]);  // r + a * Hd
      r[i] = ri;
      acc += ri * ri;
    }
  }
  if (bnd) return;
  const double b = block_sum<kDotThreads>(acc, sh);
  if (threadIdx.x == 0) tr_scratch(state, T)[3 * kDotBlocks + blockIdx.x] = b;
}

// Iteration j, part 3: |r| <= tol -> done; else d = -r + (rr_next / rr) d.
__global__ void __launch_bounds__(kDotThreads)
    tr_step3_kernel(int j, int T, int64_t d, const double *__restrict__ r, double *dv,
                    double *state) {
  // the next product's GEMM1 (a programmatic dependent) may stage its X tiles
  // now; it waits for this grid before reading d or the done flag
  pdl_trigger();
  const double *st = slot(state, j);
  double *nx = slot(state, j + 1);
  if (st[kTrDone] != 0.0) {  // finished earlier: carry the scalars forward
    if (blockIdx.x == 0 && threadIdx.x < SNX_CG_SLOT) nx[threadIdx.x] = st[threadIdx.x];
    return;
  }
  if (nx[kTrBnd] != 0.0) return;  // boundary step taken in part 2
  __shared__ double s_rr;
  if (threadIdx.x < 32) {
    const double rr = warp_sum_partials(tr_scratch(state, T) + 3 * kDotBlocks);
    if (threadIdx.x == 0) s_rr = rr;
  }
  __syncthreads();
  const double rrn = s_rr;
  const bool conv = sqrt(rrn) <= st[kTrTol];
  if (!conv) {
    const double beta = rrn / st[kTrRs];
    for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
         i += (int64_t)kDotBlocks * kDotThreads)
      dv[i] = __dadd_rn(-r[i], __dmul_rn(beta, dv[i]));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    nx[kTrRs] = conv ? st[kTrRs] : rrn;
    nx[kTrDone] = (conv || j + 1 >= T) ? 1.0 : 0.0;
  }
}

template <typename T>
__global__ void pack_rows_kernel(const double *__restrict__ src, int64_t nrows, int p,
                                 T *__restrict__ dst, int64_t ldd) {
  const int64_t total = nrows * ldd;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ldd;
    const int64_t j = i - r * ldd;
    dst[i] = j < p ? (T)src[r * p + j] : T(0);
  }
}

}  // namespace snx

using namespace snx;

extern "C" {

#ifdef SNX_TIMELINE
int snx_debug_vec_timeline(unsigned long long *host_out) {
  return cudaMemcpyFromSymbol(host_out, g_vec_timeline, sizeof(g_vec_timeline)) == cudaSuccess
             ? 0
             : 1;
}
#endif

int snx_abi_version(void) { return SNX_ABI_VERSION; }

const char *snx_last_error(void) { return g_err; }

int snx_dot(const double *x, const double *y, int64_t d, double *out, void *stream) {
  // out holds 1 + SNX_DOT_BLOCKS doubles: the partials go to out[1..]
  cudaStream_t st = (cudaStream_t)stream;
  launch_pdl(dot_part_kernel, dim3(kDotBlocks), dim3(kDotThreads), 0, st, x, y, d, out + 1);
  if (check_launch("dot")) return 1;
  launch_pdl(dot_final_kernel, dim3(1), dim3(32), 0, st, out + 1, out);
  return check_launch("dot_final");
}

int snx_dot_partials(const double *x, const double *y, int64_t d, double *part, void *stream) {
  launch_pdl(dot_part_kernel, dim3(kDotBlocks), dim3(kDotThreads), 0, (cudaStream_t)stream, x, y, d, part);
  return check_launch("dot_partials");
}

int snx_axpy(const double *x, const double *p, double alpha, int64_t d, double *x_out,
             void *stream) {
  launch_pdl(axpy_kernel, dim3(kDotBlocks), dim3(kDotThreads), 0, (cudaStream_t)stream, x, p, alpha, d, x_out);
  return check_launch("axpy");
}

int snx_axpby(double a, const double *x, double b, const double *y, int64_t d, double *out,
              void *stream) {
  launch_pdl(axpby_kernel, dim3(kDotBlocks), dim3(kDotThreads), 0, (cudaStream_t)stream, a, x, b, y, d, out);
  return check_launch("axpby");
}

int snx_finish_hv(const double *v, double lam, int64_t d, double *out, double *dots,
                  const double *skip, void *stream) {
  launch_pdl(finish_hv_kernel, dim3(kDotBlocks), dim3(kDotThreads), 0, (cudaStream_t)stream, v,
             lam, d, out, dots, skip);
  return check_launch("finish_hv");
}

int snx_cg_init(const double *g, int64_t d, double theta, int32_t max_iters, double *r,
                double *s, double *p, double *p_best, double *state, void *stream) {
  if (max_iters < 1) {
    set_error("snx_cg_init: max_iters must be >= 1");
    return 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  launch_pdl(cg_init_kernel, dim3(kDotBlocks), dim3(kDotThreads), 0, st, g, d, max_iters, r, s, p, p_best, state);
  if (check_launch("cg_init")) return 1;
  launch_pdl(cg_init_final_kernel, dim3(1), dim3(32), 0, st, theta, max_iters, state);
  return check_launch("cg_init_final");
}

int snx_cg_update(int32_t t, int32_t max_iters, int64_t d, const double *Hs,
                  const double *dots, double *r, double *s, double *p, double *p_best,
                  double *state, void *stream) {
  if (t < 0 || t >= max_iters) {
    set_error("snx_cg_update: iteration %d outside [0, %d)", t, max_iters);
    return 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  launch_pdl(cg_step1_kernel, dim3(kDotBlocks), dim3(kDotThreads), 0, st, t, max_iters, d, Hs, dots, r, s, p,
                                                      state);
  if (check_launch("cg_step1")) return 1;
  launch_pdl(cg_step2_kernel, dim3(kDotBlocks), dim3(kDotThreads), 0, st, t, max_iters, d, r, s, p, p_best, state);
  return check_launch("cg_step2");
}

}  // extern "C"

namespace snx {
int launch_cg_step2(int t, int T, int64_t d, const double *r, double *s, const double *p,
                    double *pb, double *state, cudaStream_t st) {
  launch_pdl(cg_step2_kernel, dim3(kDotBlocks), dim3(kDotThreads), 0, st, t, T, d, r, s, p, pb,
             state);
  return check_launch("cg_step2");
}
}  // namespace snx

extern "C" {

const double *snx_cg_done_flag(const double *state, int32_t t) {
  return state + (size_t)t * SNX_CG_SLOT + kDone;
}

int snx_power_step(double *v, const double *w, int64_t d, double *state, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  power_part_kernel<<<kDotBlocks, kDotThreads, 0, st>>>(v, w, d, state);
  if (check_launch("power_part")) return 1;
  power_scale_kernel<<<kDotBlocks, kDotThreads, 0, st>>>(v, w, d, state);
  return check_launch("power_scale");
}

int snx_tr_init(const double *g, int64_t d, double theta, int32_t max_iters, double *z,
                double *r, double *dvec, double *state, void *stream) {
  if (max_iters < 1) {
    set_error("snx_tr_init: max_iters must be >= 1");
    return 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  tr_init_kernel<<<kDotBlocks, kDotThreads, 0, st>>>(g, d, max_iters, z, r, dvec, state);
  if (check_launch("tr_init")) return 1;
  tr_init_final_kernel<<<1, 32, 0, st>>>(theta, max_iters, state);
  return check_launch("tr_init_final");
}

int snx_tr_update(int32_t j, int32_t max_iters, int64_t d, const double *radius,
                  const double *Hd, const double *dots, double *z, double *r, double *dvec,
                  double *znew, double *state, void *stream) {
  if (j < 0 || j >= max_iters) {
    set_error("snx_tr_update: iteration %d outside [0, %d)", j, max_iters);
    return 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  tr_step1_kernel<<<kDotBlocks, kDotThreads, 0, st>>>(j, max_iters, d, dots, z, dvec, znew,
                                                      state);
  if (check_launch("tr_step1")) return 1;
  tr_step2_kernel<<<kDotBlocks, kDotThreads, 0, st>>>(j, max_iters, d, radius, Hd, dots, z, r,
                                                      dvec, znew, state);
  if (check_launch("tr_step2")) return 1;
  tr_step3_kernel<<<kDotBlocks, kDotThreads, 0, st>>>(j, max_iters, d, r, dvec, state);
  return check_launch("tr_step3");
}

int snx_pack_rows(int dtype, const double *src, int64_t nrows, int32_t p, void *dst,
                  int64_t ldd, void *stream) {
  if (ldd < p) {
    set_error("snx_pack_rows: ldd < p");
    return 1;
  }
  if (nrows == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int blocks = 148 * 8;
  if (dtype == SNX_F64) {
    pack_rows_kernel<double><<<blocks, 256, 0, st>>>(src, nrows, p, static_cast<double *>(dst),
                                                     ldd);
  } else {
    pack_rows_kernel<float><<<blocks, 256, 0, st>>>(src, nrows, p, static_cast<float *>(dst),
                                                    ldd);
  }
  return check_launch("pack_rows");
}

}  // extern "C"
