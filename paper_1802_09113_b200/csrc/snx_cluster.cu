// One-pass fp64 row pass on thread-block clusters (sm_100a).
//
// The sampled Hessian product of softmax.py:197-210
//     V = X_S Q(v),  U = V.h - h.rowsum(V.h),  Hv = scale * X_S^T U + lam * v
// and the full-data objective + gradient of softmax.py:125-169
//     Z = X W,  R = E/alpha - onehot,  G = scale * X^T R + lam * w
// have the same shape: a K-wide contraction of every row over all p features,
// a row-local epilogue, and the transposed product with the SAME rows.  The
// two-GEMM path (snx_rowpass.cu) streams X twice with a grid-wide dependency
// between the GEMMs; this kernel streams every row ONCE:
//
//   * a cluster of CS CTAs owns a contiguous range of rows; CTA q of the
//     cluster owns the column slice [q*wc, (q+1)*wc) of every row.  A row
//     block of R rows arrives in shared memory by TMA bulk copies (one per
//     row slice, gathered through the sample's row indices -- the gather is
//     fused, no X_S copy is materialised);
//   * consumers compute the slice's partial logits V_q = X[:, slice] Q[slice]
//     (register tiles, fixed-order in-warp butterflies, fixed-order sum over
//     warps) and push them into every peer's shared memory with st.async
//     (distributed shared memory, completion counted on the peer's mbarrier);
//   * every CTA sums the CS slice partials in rank order -- identical bits on
//     all peers -- and runs the row algebra (U, or the residual + loss);
//   * the same shared-memory tile then feeds the transposed product: each
//     thread owns a few columns x K classes of X^T U in registers for the
//     whole kernel.  The block after next is already streaming in (3-4 stage
//     ring), and the peers' partial logits of the NEXT block are computed
//     before this block's X^T U, so the exchange latency hides behind it;
//   * at the end each cluster writes its K x p partial; a small finalize
//     kernel sums the cluster partials in a fixed order, applies scale, lam
//     and emits the CG dot partials (the SNX_DOT_BLOCKS layout of
//     snx_hess_apply).
//
// Every reduction has a fixed order and there are no float atomics: results
// are bit-identical run to run.  fp64 only, K <= 9 (the BASELINE shapes:
// covertype K = 6, MNIST / CIFAR-10 K = 9); other shapes use snx_rowpass.cu.
#include <stdio.h>

#include "snx_common.cuh"
#include "snx_internal.h"
#include "snx_pipe.cuh"

namespace snx {
namespace clp {

enum Mode { kPrep = 0, kApply = 1, kGrad = 2 };

constexpr int kNW = 8;               // consumer warps
constexpr int kNC = kNW * 32;        // consumer threads
constexpr int kNT = kNC + 32;        // + one producer warp
constexpr int kMaxK = 9;

// Thread-work shapes.
//  V phase (partial logits): lane = (row group rg < RGL, k-slice ksl < KSL);
//    a thread owns RT rows (rt*RGL + rg) x K classes over the column pairs
//    2*(i*KS + kslice), i < npi; the KSL lanes of a row group read one 16-B
//    pair each (a contiguous 16*KSL-byte run: no bank conflicts) and share the
//    weight pairs (smem broadcasts).
//  X^T U phase: thread t owns CPT consecutive columns of NCI chunks strided by
//    NCOLT*CPT, x K classes, over the rows r = rsub (mod RS); U rows are smem
//    broadcasts.
template <int RGL_, int RT_, int NCOLT_, int CPT_, int NCI_, bool DM_ = false, int NMT_ = 1>
struct Cfg {
  static constexpr int RGL = RGL_, RT = RT_, NCOLT = NCOLT_, CPT = CPT_, NCI = NCI_;
  static constexpr bool DM = DM_;   // fp64 tensor-core MMAs (m8n8k4) for classes 0..7
  static constexpr int NMT = NMT_;  // DM: X^T U column tiles (8 wide) per warp
  static constexpr int R = RGL * RT;      // rows per block
  static constexpr int KSL = 32 / RGL;    // k-slices per warp
  static constexpr int KS = kNW * KSL;    // k-slices per CTA
  static constexpr int RS = kNC / NCOLT;  // row subsets of X^T U
  static constexpr int LV = KSL == 1 ? 0 : KSL == 2 ? 1 : KSL == 4 ? 2 : KSL == 8 ? 3 : 4;
  static constexpr int LR = RT == 1 ? 0 : RT == 2 ? 1 : RT == 4 ? 2 : 3;
  static constexpr int LS = LV < LR ? LV : LR;  // reduce-scatter levels
};
// CfgA (DM): 8-row blocks, 16-column chunks; V = X Q on mma.m8n8k4.f64 (rows x
//   classes 0..7 per warp, k split over the warps), class 8 by DFMA from the
//   same fragments; X^T U on m8n8k4 with 8-column tiles owned by warps.
using CfgA = Cfg<4, 2, 256, 1, 3, true, 12>;  // column slices of 65..768
using CfgB = Cfg<16, 4, 16, 4, 1>;   // column slices of <= 64 (64-row blocks)

struct Args {
  const double *X;
  int64_t ldx;
  const int64_t *rows;    // nullable: sample position -> source row
  int64_t nrows;
  int p, K, cs, ncl, wc, npi, S, WS, WQ;
  int mode;
  const double *w;        // [K][p] class-major weights (v for the Hessian product)
  const double *h;        // apply: [nrows][K] probabilities
  const int32_t *labels;  // grad: labels of the (source) rows
  double *hout;           // prep: [nrows][K]
  double *gp;             // [ncl][K*p] cluster partials of X^T U
  double *lossp;          // grad: [ncl]
  unsigned long long *corrp;  // grad: [ncl]
  const double *skip;
  int early;              // programmatic dependent: stage rows before waiting
  int qbulk;              // weight slices are 16-B aligned: TMA bulk copies
  // shared-memory carve-up (byte offsets)
  int o_tiles, o_q, o_side, o_u, o_vr, o_red, o_bar;
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_id() {
  unsigned r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned mapa(unsigned addr, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// remote (or local) 8-B store into a cluster peer's shared memory, counted as
// 8 transaction bytes on the peer's mbarrier
__device__ __forceinline__ void st_async(unsigned raddr, double v, unsigned rbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(raddr),
      "d"(v), "r"(rbar)
      : "memory");
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
// arrive on `bar` once this thread's cp.async copies have landed (counts as one
// of the barrier's expected arrivals)
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t *bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// D = A B + C on the fp64 tensor cores: A 8x4 (row), B 4x8 (col), C/D 8x8.
// Lane l = 4g + t holds a = A[g][t], b = B[t][g], c = (C[g][2t], C[g][2t+1]).
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// half-warp (16-lane) butterflies: fixed order, identical bits on every lane
__device__ __forceinline__ double hsum(double v) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double hmax_nan(double v) {  // NaN wins (np.max propagates it)
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    v = isnan(v) ? v : (isnan(u) ? u : (u > v ? u : v));
  }
  return v;
}
// argmax with numpy's rules: the first NaN, else the largest, ties -> lowest index
__device__ __forceinline__ int hargmax(double v, int idx) {
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    const int j = __shfl_xor_sync(0xffffffffu, idx, o);
    const bool vn = isnan(v), un = isnan(u);
    bool take;
    if (vn || un)
      take = un && (!vn || j < idx);
    else
      take = u > v || (u == v && j < idx);
    if (take) {
      v = u;
      idx = j;
    }
  }
  return idx;
}

// Optional per-CTA timeline (-DSNX_CL_TIMELINE; tools/cl_timeline.py): warp
// 0 lane 0 and the producer stamp %globaltimer at fixed events per block.
#ifdef SNX_CL_TIMELINE
constexpr int kTlBlocks = 24;
__device__ unsigned long long g_cl_tl[160][kTlBlocks + 2][10];
__device__ __forceinline__ void cl_stamp(int b, int ev) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (blockIdx.x < 160 && b + 1 < kTlBlocks + 2) g_cl_tl[blockIdx.x][b + 1][ev] = t;
}
#define CL_TL(b, ev)                          \
  do {                                        \
    if (threadIdx.x == 0) cl_stamp((b), (ev)); \
  } while (0)
#define CL_TLP(b, ev)                          \
  do {                                         \
    if (threadIdx.x == kNC) cl_stamp((b), (ev)); \
  } while (0)
#else
#define CL_TL(b, ev) \
  do {               \
  } while (0)
#define CL_TLP(b, ev) \
  do {                \
  } while (0)
#endif

// ---------------------------------------------------------------- kernel
template <int K, typename C>
__global__ void __launch_bounds__(kNT, 1) cluster_rowpass_kernel(const __grid_constant__ Args a) {
  constexpr int R = C::R, RT = C::RT, RGL = C::RGL, KSL = C::KSL, KS = C::KS;
  // U row stride: 16-B multiple; DM: classes 0..8 + pad (10 doubles) so the
  // X^T U B fragments (U[2t+s][g]) hit each bank at most twice
  constexpr int KP = C::DM ? 10 : K + (K & 1);
  constexpr int KQ = C::DM ? (K > 8 ? K : 8) : K;  // weight rows (DM: classes >= K zero)
  pdl_trigger();  // the finalize kernel may launch now (it waits for this grid)
  extern __shared__ __align__(1024) unsigned char smem[];
  double *tiles = reinterpret_cast<double *>(smem + a.o_tiles);  // [S][R][WS]
  double *Qs = reinterpret_cast<double *>(smem + a.o_q);         // [K][WQ]
  double *side = reinterpret_cast<double *>(smem + a.o_side);    // [S][R][K] h | [S][R] int
  double *Us = reinterpret_cast<double *>(smem + a.o_u);         // [2][R][KP]
  double *Vr = reinterpret_cast<double *>(smem + a.o_vr);        // [2][cs][R][K]
  double *red = reinterpret_cast<double *>(smem + a.o_red);      // [2][NW][R][K]
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + a.o_bar);
  uint64_t *empty = full + a.S;
  uint64_t *vfull = empty + a.S;  // [2]
  uint64_t *qbar = vfull + 2;
  __shared__ double sh_loss[kNW];
  __shared__ unsigned long long sh_corr[kNW];
  __shared__ int sh_skip;

  // the warp index through a shuffle: provably warp-uniform for the compiler,
  // so shuffles under warp-indexed loops need no divergent-collective lowering
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int S = a.S, WS = a.WS, WQ = a.WQ, cs = a.cs;
  CL_TL(-1, 0);
  const unsigned q = cluster_rank();
  const int cl = (int)cluster_id();
  const int64_t row_lo = a.nrows * cl / a.ncl, row_hi = a.nrows * (cl + 1) / a.ncl;
  const int nb = (int)((row_hi - row_lo + R - 1) / R);
  const int c0 = (int)q * a.wc;                                 // first column of the slice
  const int wq = max(0, min(a.wc, ((a.p + 3) & ~3) - c0));      // slice width (even)
  const bool apply = a.mode == kApply, grad = a.mode == kGrad;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 32);
      mbar_init(&empty[s], kNW);
    }
    mbar_init(&vfull[0], 1);
    mbar_init(&vfull[1], 1);
    mbar_init(qbar, 1);
    mbar_fence_init();
  }
  // zero the tile columns no bulk copy writes (the V phase streams zero pairs there)
  for (int i = tid; i < S * R * (WS - wq); i += kNT) {
    const int r = i / (WS - wq), j = i - r * (WS - wq);
    tiles[(size_t)r * WS + wq + j] = 0.0;
  }
  __syncthreads();
  if (tid == 0 && nb > 0) {
    const int nr0 = (int)min((int64_t)R, row_hi - row_lo);
    mbar_arrive_expect_tx(&vfull[0], (unsigned)(cs * nr0 * K * 8));
  }
  cluster_sync_all();  // peers' barriers initialised before any st.async

  // ------------------------------------------------------------ producer warp
  if (warp == kNW) {
    constexpr int IPL = (R + 31) / 32;  // row indices per lane and block
    // source rows of block b (the next block's are loaded one block ahead, so
    // their latency hides behind the current block's issue)
    auto load_idx = [&](int b, int64_t(&dst)[IPL]) {
      const int64_t r0 = row_lo + (int64_t)b * R;
      const int nr = (int)min((int64_t)R, row_hi - r0);
#pragma unroll
      for (int j = 0; j < IPL; ++j) {
        const int e = lane + 32 * j;
        dst[j] = e < nr ? (a.rows ? a.rows[r0 + e] : r0 + e) : 0;
      }
    };
    // X slices of block b: TMA bulk copies, tx bytes announced without arriving
    auto issue_x = [&](int b, const int64_t(&idx)[IPL]) {
      const int s = b % S;
      if (b >= S) mbar_wait(&empty[s], ((b / S) - 1) & 1);
      const int64_t r0 = row_lo + (int64_t)b * R;
      const int nr = (int)min((int64_t)R, row_hi - r0);
      double *tile = tiles + (size_t)s * R * WS;
      const unsigned bytes = (unsigned)wq * 8u;
      if (lane == 0) mbar_expect_tx(&full[s], bytes * (unsigned)nr);
      if (bytes > 0) {
#pragma unroll
        for (int j = 0; j < IPL; ++j) {
          const int e = lane + 32 * j;
          if (e < nr) bulk_g2s(tile + (size_t)e * WS, a.X + idx[j] * a.ldx + c0, bytes, &full[s]);
        }
      }
    };
    // side data of block b (h rows / labels: possibly the predecessor's
    // outputs) by cp.async; each lane's arrival fires when its copies land
    auto issue_side = [&](int b, const int64_t(&idx)[IPL]) {
      const int s = b % S;
      const int64_t r0 = row_lo + (int64_t)b * R;
      const int nr = (int)min((int64_t)R, row_hi - r0);
      if (apply) {
        double *hs = side + (size_t)s * R * K;
        for (int e = lane; e < nr * K; e += 32) cp_async8(hs + e, a.h + r0 * K + e);
      } else if (grad) {
        int *ls = reinterpret_cast<int *>(side) + s * R;
#pragma unroll
        for (int j = 0; j < IPL; ++j) {
          const int e = lane + 32 * j;
          if (e < nr) cp_async4(ls + e, a.labels + idx[j]);
        }
      }
      cp_async_mbar_arrive(&full[s]);
    };
    int64_t idx[2][IPL];
    int b = 0;
    if (nb > 0) load_idx(0, idx[0]);
    if (a.early) {  // X and the row indices are older than the predecessor
      for (; b < nb && b < S; ++b) {
        if (b + 1 < nb) load_idx(b + 1, idx[(b + 1) & 1]);
        issue_x(b, idx[b & 1]);
      }
    }
    pdl_wait();
    if (lane == 0) sh_skip = (a.skip != nullptr && *a.skip != 0.0) ? 1 : 0;
    __syncwarp();
    if (sh_skip) {  // complete the staged phases (so no copy is in flight), then leave
      for (int bb = 0; bb < b; ++bb) {
        mbar_arrive(&full[bb % S]);
        mbar_wait(&full[bb % S], (bb / S) & 1);
      }
    } else {
      // the weight slice (consumers wait on qbar): one bulk copy per class
      if (a.qbulk && lane < K) {
        const int qc = min(wq, a.p - c0);
        if (lane == 0) mbar_arrive_expect_tx(qbar, (unsigned)(K * max(qc, 0) * 8));
        if (qc > 0)
          bulk_g2s(Qs + lane * WQ, a.w + (int64_t)lane * a.p + c0, (unsigned)qc * 8u, qbar);
      }
      // early-staged blocks only need their side data now (h never needs idx)
      for (int bb = 0; bb < b; ++bb) issue_side(bb, idx[bb & 1]);
      for (; b < nb; ++b) {
        if (b + 1 < nb) load_idx(b + 1, idx[(b + 1) & 1]);
        issue_x(b, idx[b & 1]);
        issue_side(b, idx[b & 1]);
      }
    }
    cluster_sync_all();
    return;
  }

  // ------------------------------------------------------------ consumers
  pdl_wait();  // the weights and the skip flag are the predecessor's outputs
  if (a.skip != nullptr && *a.skip != 0.0) {
    cluster_sync_all();
    return;
  }
  // weight slice Qs[c][j] = w[c*p + c0 + j], zero past the slice / p: the
  // producer's bulk copies (qbulk) or direct loads (batched: one round trip)
  {
    const int qc = a.qbulk ? max(0, min(wq, a.p - c0)) : 0;  // columns the copies bring
    for (int i0 = tid; i0 < KQ * WQ; i0 += 8 * kNC) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {  // loads first: one round trip per 8
        const int i = i0 + u * kNC;
        const int c = i / WQ, j = i - c * WQ, gc = c0 + j;
        v[u] = (!a.qbulk && c < K && j < wq && gc < a.p) ? a.w[(int64_t)c * a.p + gc] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * kNC;
        const int c = i / WQ;
        if (i < KQ * WQ && (c >= K || i - c * WQ >= qc)) Qs[i] = v[u];
      }
    }
    if (a.qbulk) mbar_wait(qbar, 0);
  }
  consumer_sync(kNC);

  const int rg = lane / KSL, ksl = lane % KSL;
  const int kslice = warp * KSL + ksl;
  // X^T U ownership
  const int cg = tid % C::NCOLT, rsub = tid / C::NCOLT;
  constexpr int AI = C::DM ? 1 : C::NCI, AE = C::DM ? 1 : C::CPT;
  double acc[AI][AE][K];
#pragma unroll
  for (int i = 0; i < AI; ++i)
#pragma unroll
    for (int e = 0; e < AE; ++e)
#pragma unroll
      for (int c = 0; c < K; ++c) acc[i][e][c] = 0.0;
  // DM: X^T U tiles (classes 2t, 2t+1 of column 8*tile + g) and class-8 partials
  constexpr int MT = C::DM ? C::NMT : 1;
  double dacc[MT][2], dacc8[MT];
#pragma unroll
  for (int m = 0; m < MT; ++m) dacc[m][0] = dacc[m][1] = dacc8[m] = 0.0;
  const int g8 = lane >> 2, t4 = lane & 3;
  double loss_acc = 0.0;
  unsigned long long corr_acc = 0;

  // V phase of block b: partial logits of this slice, reduced over the CTA and
  // pushed to every peer's Vr[b & 1][q]
  auto vphase = [&](int b) {
    const int s = b % S;
    const int64_t r0 = row_lo + (int64_t)b * R;
    const int nr = (int)min((int64_t)R, row_hi - r0);
    const int rtv = (nr + RGL - 1) / RGL;  // valid row slots (warp-uniform)
    mbar_wait(&full[s], (b / S) & 1);
    const double *tile = tiles + (size_t)s * R * WS;
    if constexpr (C::DM) {
      // 16-column chunks ch = warp, warp + 8, ...; physical column of (step s,
      // lane t) = 16 ch + 4 t + s, so a lane's 4 A (and B) values are contiguous
      double c2[2] = {0.0, 0.0}, v8 = 0.0;
      const double *xrow = tile + (size_t)g8 * WS + 4 * t4;
      const double *qrow = Qs + (size_t)g8 * WQ + 4 * t4;
      const double *q8row = Qs + (size_t)8 * WQ + 4 * t4;
      const int nch = (wq + 15) >> 4;
#pragma unroll 2
      for (int ch = warp; ch < nch; ch += kNW) {
        const double2 xa = *reinterpret_cast<const double2 *>(xrow + 16 * ch);
        const double2 xb = *reinterpret_cast<const double2 *>(xrow + 16 * ch + 2);
        const double2 qa = *reinterpret_cast<const double2 *>(qrow + 16 * ch);
        const double2 qb = *reinterpret_cast<const double2 *>(qrow + 16 * ch + 2);
        dmma(c2, xa.x, qa.x);
        dmma(c2, xa.y, qa.y);
        dmma(c2, xb.x, qb.x);
        dmma(c2, xb.y, qb.y);
        if constexpr (K == 9) {
          const double2 ra = *reinterpret_cast<const double2 *>(q8row + 16 * ch);
          const double2 rb2 = *reinterpret_cast<const double2 *>(q8row + 16 * ch + 2);
          v8 = fma(xa.x, ra.x, v8);
          v8 = fma(xa.y, ra.y, v8);
          v8 = fma(xb.x, rb2.x, v8);
          v8 = fma(xb.y, rb2.y, v8);
        }
      }
      double *rbw = red + (size_t)(b & 1) * kNW * R * K + (size_t)warp * R * K + g8 * K;
      if (2 * t4 < K) rbw[2 * t4] = c2[0];
      if (2 * t4 + 1 < K) rbw[2 * t4 + 1] = c2[1];
      if constexpr (K == 9) {
        v8 += __shfl_xor_sync(0xffffffffu, v8, 1);
        v8 += __shfl_xor_sync(0xffffffffu, v8, 2);
        if (t4 == 0) rbw[8] = v8;
      }
      return;
    }
    double v[RT][K];
#pragma unroll
    for (int rt = 0; rt < RT; ++rt)
#pragma unroll
      for (int c = 0; c < K; ++c) v[rt][c] = 0.0;
#pragma unroll 2
    for (int i = 0; i < a.npi; ++i) {
      const int col = 2 * (i * KS + kslice);
      double2 qv[K];
#pragma unroll
      for (int c = 0; c < K; ++c) qv[c] = *reinterpret_cast<const double2 *>(Qs + c * WQ + col);
#pragma unroll
      for (int rt = 0; rt < RT; ++rt) {
        if (rt < rtv) {
          const double2 x =
              *reinterpret_cast<const double2 *>(tile + (size_t)(rt * RGL + rg) * WS + col);
#pragma unroll
          for (int c = 0; c < K; ++c) {
            v[rt][c] = fma(x.x, qv[c].x, v[rt][c]);
            v[rt][c] = fma(x.y, qv[c].y, v[rt][c]);
          }
        }
      }
    }
    // in-warp reduction over the KSL lanes of a row group: reduce-scatter over
    // the row slots, then full butterflies (fixed order)
    int slot0 = 0;
#pragma unroll
    for (int L = 0; L < C::LV; ++L) {
      const int o = 1 << L;
      if (L < C::LS) {
        const int half = RT >> (L + 1);
        const int bit = (ksl >> L) & 1;
#pragma unroll
        for (int j = 0; j < (RT >> 1); ++j) {
          if (j < half) {
#pragma unroll
            for (int c = 0; c < K; ++c) {
              const double send = bit ? v[j][c] : v[j + half][c];
              const double keep = bit ? v[j + half][c] : v[j][c];
              v[j][c] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
          }
        }
        slot0 += bit * half;
      } else {
#pragma unroll
        for (int j = 0; j < (RT >> C::LS); ++j)
#pragma unroll
          for (int c = 0; c < K; ++c) v[j][c] += __shfl_xor_sync(0xffffffffu, v[j][c], o);
      }
    }
    // writers: lanes whose full-butterfly bits are zero
    double *rb = red + (size_t)(b & 1) * kNW * R * K + (size_t)warp * R * K;
    if ((ksl >> C::LS) == 0) {
#pragma unroll
      for (int j = 0; j < (RT >> C::LS); ++j) {
        const int row = (slot0 + j) * RGL + rg;
#pragma unroll
        for (int c = 0; c < K; ++c) rb[row * K + c] = v[j][c];
      }
    }
  };

  // sum of the warp partials (fixed order) -> every peer's receive buffer
  auto vsend = [&](int b) {
    const int64_t r0 = row_lo + (int64_t)b * R;
    const int nr = (int)min((int64_t)R, row_hi - r0);
    const double *rb = red + (size_t)(b & 1) * kNW * R * K;
    const unsigned vr_local = smem_u32(Vr + ((size_t)(b & 1) * cs + q) * R * K);
    const unsigned bar_local = smem_u32(&vfull[b & 1]);
    for (int e = tid; e < nr * K; e += kNC) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < kNW; ++w) s += rb[w * R * K + e];
      for (int pq = 0; pq < cs; ++pq)
        st_async(mapa(vr_local + e * 8, pq), s, mapa(bar_local, pq));
    }
  };

  // row algebra of block b (half-warp per row, lanes over classes): U rows
  // into Us[b & 1]; h (prep), loss / correct (grad)
  auto rowalg = [&](int b) {
    const int s = b % S;
    const int64_t r0 = row_lo + (int64_t)b * R;
    const int nr = (int)min((int64_t)R, row_hi - r0);
    mbar_wait_cluster(&vfull[b & 1], (b >> 1) & 1);
    CL_TL(b, 6);
    if (tid == 0 && b + 1 < nb) {  // the next use of this buffer pair's other barrier
      const int nr1 = (int)min((int64_t)R, row_hi - (r0 + R));
      mbar_arrive_expect_tx(&vfull[(b + 1) & 1], (unsigned)(cs * nr1 * K * 8));
    }
    CL_TL(b, 8);
    const double *vr = Vr + (size_t)(b & 1) * cs * R * K;
    double *u = Us + (size_t)(b & 1) * R * KP;
    const int hw = lane >> 4, c = lane & 15;
    for (int rp = warp; rp < R / 2; rp += kNW) {  // warp-uniform trip count
      const int row = 2 * rp + hw;
      const bool rv = row < nr;
      double z = 0.0;
      if (rv && c < K)
        for (int pq = 0; pq < cs; ++pq) z += vr[(pq * R + row) * K + c];
      CL_TL(b, 7);
      if (apply) {
        const double hv = (rv && c < K) ? side[((size_t)s * R + row) * K + c] : 0.0;
        const double vw = z * hv;
        const double sm = hsum(vw);  // softmax.py:207 rowsum(VW)
        if (c < KP) u[row * KP + c] = (rv && c < K) ? vw - hv * sm : 0.0;
        continue;
      }
      // softmax.py:91-98: M = max(0, max_c z); E = exp(z - M); alpha = e^-M + sum E
      const double zc = (c < K) ? z : 0.0;
      const double M = hmax_nan(zc);  // lanes >= K contribute 0 = the reference class logit
      const double E = (c < K) ? exp(z - M) : 0.0;
      const double alpha = exp(-M) + hsum(E);
      if (a.mode == kPrep) {
        if (rv && c < K && q == 0) a.hout[(r0 + row) * K + c] = E / alpha;
        continue;
      }
      // grad: residual (softmax.py:157-161), loss (:134), accuracy (:224-247)
      const int y = rv ? reinterpret_cast<const int *>(side)[s * R + row] : 0;
      const double pr = (c < K) ? E / alpha : (c == K ? exp(-M) / alpha : -INFINITY);
      if (c < KP) u[row * KP + c] = (rv && c < K) ? pr - (c == y ? 1.0 : 0.0) : 0.0;
      const double lin = hsum((c < K && c == y) ? z : 0.0);
      if (rv && c == 0 && q == 0) loss_acc += (M + log(alpha)) - lin;
      const int best = hargmax(pr, c);
      if (rv && c == 0 && q == 0 && best == y) corr_acc += 1ull;
    }
    CL_TL(b, 9);
  };

  auto xtu = [&](int b) {
    const int s = b % S;
    const int64_t r0 = row_lo + (int64_t)b * R;
    const int nr = (int)min((int64_t)R, row_hi - r0);
    const double *tile = tiles + (size_t)s * R * WS;
    const double *u = Us + (size_t)(b & 1) * R * KP;
    if constexpr (C::DM) {
      // rows of step s, lane t: 2t + s (each bank hit by two of the four rows)
      const double ua0 = u[(2 * t4) * KP + g8], ua1 = u[(2 * t4 + 1) * KP + g8];
      const double u80 = K == 9 ? u[(2 * t4) * KP + 8] : 0.0;
      const double u81 = K == 9 ? u[(2 * t4 + 1) * KP + 8] : 0.0;
      const bool ok0 = 2 * t4 < nr, ok1 = 2 * t4 + 1 < nr;
      const double *x0 = tile + (size_t)(2 * t4) * WS + g8;
      const double *x1 = x0 + WS;
      const int nmt = (wq + 7) >> 3;
#pragma unroll
      for (int m = 0; m < C::NMT; ++m) {
        const int mt = warp + kNW * m;
        if (mt < nmt) {
          const double a0 = ok0 ? x0[8 * mt] : 0.0;
          const double a1 = ok1 ? x1[8 * mt] : 0.0;
          dmma(dacc[m], a0, ua0);
          dmma(dacc[m], a1, ua1);
          if constexpr (K == 9) {
            dacc8[m] = fma(a0, u80, dacc8[m]);
            dacc8[m] = fma(a1, u81, dacc8[m]);
          }
        }
      }
      return;
    }
    int nci = 0;  // active column chunks of this warp (warp-uniform)
#pragma unroll
    for (int i = 0; i < C::NCI; ++i)
      if ((i * C::NCOLT + ((warp * 32) % C::NCOLT)) * C::CPT < wq) nci = i + 1;
    for (int r = rsub; r < nr; r += C::RS) {
      double ur[KP];
#pragma unroll
      for (int c = 0; c < KP; c += 2) {
        const double2 t2 = *reinterpret_cast<const double2 *>(u + r * KP + c);
        ur[c] = t2.x;
        ur[c + 1] = t2.y;
      }
      const double *xr = tile + (size_t)r * WS;
#pragma unroll
      for (int i = 0; i < C::NCI; ++i) {
        if (i < nci) {
          double x[C::CPT];
          const int col = (i * C::NCOLT + cg) * C::CPT;
          if constexpr (C::CPT == 1) {
            x[0] = xr[col];
          } else {
#pragma unroll
            for (int e = 0; e < C::CPT; e += 2) {
              const double2 t2 = *reinterpret_cast<const double2 *>(xr + col + e);
              x[e] = t2.x;
              x[e + 1] = t2.y;
            }
          }
#pragma unroll
          for (int e = 0; e < C::CPT; ++e)
#pragma unroll
            for (int c = 0; c < K; ++c) acc[i][e][c] = fma(x[e], ur[c], acc[i][e][c]);
        }
      }
    }
  };

  CL_TL(-1, 1);
  if (nb > 0) {
    vphase(0);
    consumer_sync(kNC);
    vsend(0);
  }
  CL_TL(-1, 2);
  for (int b = 0; b < nb; ++b) {
    CL_TL(b, 0);
    rowalg(b);
    CL_TL(b, 1);
    if (b + 1 < nb) vphase(b + 1);
    CL_TL(b, 2);
    consumer_sync(kNC);  // U(b) and the warp partials of b + 1 visible
    CL_TL(b, 3);
    if (b + 1 < nb) vsend(b + 1);
    CL_TL(b, 4);
    if (a.mode != kPrep) xtu(b);
    CL_TL(b, 5);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[b % S]);
  }
  CL_TL(-1, 3);

  // ------------------------------------------------------------ epilogue
  if (grad) {
    double l = warp_allsum(loss_acc);
    unsigned long long cc = corr_acc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cc += __shfl_xor_sync(0xffffffffu, cc, o);
    if (lane == 0) {
      sh_loss[warp] = l;
      sh_corr[warp] = cc;
    }
  }
  if (a.mode != kPrep) {
    const int64_t d = (int64_t)K * a.p;
    double *g = a.gp + (int64_t)cl * d;
    if constexpr (C::DM) {
      const int nmt = (wq + 7) >> 3;
#pragma unroll
      for (int m = 0; m < C::NMT; ++m) {
        const int mt = warp + kNW * m;
        double s8 = dacc8[m];
        if constexpr (K == 9) {
          s8 += __shfl_xor_sync(0xffffffffu, s8, 1);
          s8 += __shfl_xor_sync(0xffffffffu, s8, 2);
        }
        const int col = 8 * mt + g8, gc = c0 + col;
        if (mt < nmt && col < wq && gc < a.p) {
          if (2 * t4 < K) g[(int64_t)(2 * t4) * a.p + gc] = dacc[m][0];
          if (2 * t4 + 1 < K) g[(int64_t)(2 * t4 + 1) * a.p + gc] = dacc[m][1];
          if (K == 9 && t4 == 0) g[(int64_t)8 * a.p + gc] = s8;
        }
      }
    } else if constexpr (C::RS == 1) {
#pragma unroll
      for (int i = 0; i < C::NCI; ++i)
#pragma unroll
        for (int e = 0; e < C::CPT; ++e) {
          const int col = (i * C::NCOLT + cg) * C::CPT + e;
          const int gc = c0 + col;
          if (col < wq && gc < a.p) {
#pragma unroll
            for (int c = 0; c < K; ++c) g[(int64_t)c * a.p + gc] = acc[i][e][c];
          }
        }
    } else {
      // combine the RS row subsets in order through shared memory (the tiles are free)
      consumer_sync(kNC);
      constexpr int NCOL = C::NCOLT * C::CPT * C::NCI;
      double *comb = tiles;  // [RS][NCOL][K]
#pragma unroll
      for (int i = 0; i < C::NCI; ++i)
#pragma unroll
        for (int e = 0; e < C::CPT; ++e)
#pragma unroll
          for (int c = 0; c < K; ++c)
            comb[((size_t)rsub * NCOL + (i * C::NCOLT + cg) * C::CPT + e) * K + c] =
                acc[i][e][c];
      consumer_sync(kNC);
      for (int t = tid; t < NCOL * K; t += kNC) {
        const int c = t / NCOL, col = t - c * NCOL;
        double s = 0.0;
        for (int r = 0; r < C::RS; ++r) s += comb[((size_t)r * NCOL + col) * K + c];
        const int gc = c0 + col;
        if (col < wq && gc < a.p) g[(int64_t)c * a.p + gc] = s;
      }
    }
  }
  if (grad) {
    consumer_sync(kNC);
    if (tid == 0 && q == 0) {
      double l = 0.0;
      unsigned long long cc = 0;
      for (int w = 0; w < kNW; ++w) {
        l += sh_loss[w];
        cc += sh_corr[w];
      }
      a.lossp[cl] = l;
      a.corrp[cl] = cc;
    }
  }
  CL_TL(-1, 4);
  cluster_sync_all();  // no CTA leaves while a peer may still address its smem
  CL_TL(-1, 5);
}

// out[i] = scale * sum_cl gp[cl][i] + lam * base[i] (fixed order: F lanes per
// element sum the partials cl = f (mod F) in order, then an xor butterfly),
// block b owns elements [b*EPB, (b+1)*EPB) -> dots[b] = base.out, dots[B+b] =
// base.base; block 0 also sums the loss / correct partials.
constexpr int kFinThreads = 512;

__global__ void __launch_bounds__(kFinThreads)
    finalize_kernel(const double *__restrict__ gp, int ncl, int64_t d, int64_t epb, int F,
                    double scale, double lam, const double *__restrict__ base,
                    double *__restrict__ out, double *dots, const double *skip,
                    const double *lossp, const unsigned long long *corrp, double *loss_out,
                    long long *corr_out) {
  pdl_wait();
  if (skip != nullptr && *skip != 0.0) return;
  __shared__ double sh[kFinThreads / 32];
  const int t = threadIdx.x;
  const int64_t i = (int64_t)blockIdx.x * epb + t / F;
  const int f = t % F;
  const bool own = (t / F) < epb && i < d;
  double s = 0.0;
  if (own) {
    int c = f;
    for (; c + 7 * F < ncl; c += 8 * F) {
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = __ldcg(gp + (int64_t)(c + k * F) * d + i);
#pragma unroll
      for (int k = 0; k < 8; ++k) s += v[k];
    }
    for (; c < ncl; c += F) s += __ldcg(gp + (int64_t)c * d + i);
  }
  for (int o = 1; o < F; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  double bo = 0.0, bb = 0.0;
  if (own && f == 0) {
    const double b = base[i];
    const double o = __dadd_rn(__dmul_rn(scale, s), __dmul_rn(lam, b));
    out[i] = o;
    bo = b * o;
    bb = b * b;
  }
  if (dots != nullptr) {
    const double so = block_sum<kFinThreads>(bo, sh);
    const double sb = block_sum<kFinThreads>(bb, sh);
    if (t == 0) {
      dots[blockIdx.x] = so;
      dots[kDotBlocks + blockIdx.x] = sb;
    }
  }
  if (blockIdx.x == 0 && loss_out != nullptr && t < 32) {
    double l = 0.0;
    unsigned long long cc = 0;
    for (int c = t; c < ncl; c += 32) {
      l += __ldcg(lossp + c);
      cc += __ldcg(corrp + c);
    }
    l = warp_allsum(l);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cc += __shfl_xor_sync(0xffffffffu, cc, o);
    if (t == 0) {
      *loss_out = l;
      if (corr_out != nullptr) *corr_out = (long long)cc;
    }
  }
}

// ---------------------------------------------------------------- host side
struct Plan {
  int ok;
  int cfg;  // 0: CfgA, 1: CfgB
  int cs, ncl, wc, npi, S, WS, WQ, R;
  size_t smem;
  int o_tiles, o_q, o_side, o_u, o_vr, o_red, o_bar;
};

template <int K, typename C>
static void layout(Plan &pl, int S) {
  constexpr int KP = C::DM ? 10 : K + (K & 1);
  constexpr int KQ = C::DM ? (K > 8 ? K : 8) : K;
  size_t off = 0;
  auto take = [&](size_t bytes, size_t align) {
    off = (off + align - 1) / align * align;
    const size_t o = off;
    off += bytes;
    return (int)o;
  };
  pl.o_tiles = take((size_t)S * C::R * pl.WS * 8, 1024);
  pl.o_q = take((size_t)KQ * pl.WQ * 8, 16);
  pl.o_side = take((size_t)S * C::R * K * 8, 16);
  pl.o_u = take((size_t)2 * C::R * KP * 8, 16);
  pl.o_vr = take((size_t)2 * pl.cs * C::R * K * 8, 16);
  pl.o_red = take((size_t)2 * kNW * C::R * K * 8, 16);
  pl.o_bar = take((size_t)(2 * S + 3) * 8, 8);
  pl.smem = off;
  pl.S = S;
}

// the dynamic shared-memory ceiling is raised once to the maximum: plans of
// different sizes share one instantiation
// (opt-in per-block maximum minus the kernel's static shared memory)
template <int K, typename C>
static size_t smem_cap() {
  static size_t cap = 0;
  if (cap == 0) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) !=
            cudaSuccess ||
        optin <= 0)
      optin = 227 * 1024;
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, cluster_rowpass_kernel<K, C>);
    cudaGetLastError();
    cap = (size_t)optin - fa.sharedSizeBytes;
  }
  return cap;
}

template <int K, typename C>
static bool set_max_smem() {
  static bool done = false;
  if (!done) {
    if (cudaFuncSetAttribute(cluster_rowpass_kernel<K, C>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem_cap<K, C>()) != cudaSuccess)
      return false;
    done = true;
  }
  return true;
}

template <int K, typename C>
static int max_clusters(int cs, size_t smem) {
  static int cache[9][2048];
  static bool init = false;
  if (!init) {
    for (auto &row : cache)
      for (int &v : row) v = -1;
    init = true;
  }
  const int key = (int)(smem / 1024);
  const int ci = cs == 1 ? 0 : cs == 2 ? 1 : cs == 4 ? 2 : 3;
  int &slot = cache[ci * 2 + (C::R == 8 ? 0 : 1)][key < 2048 ? key : 2047];
  if (slot >= 0) return slot;
  auto kern = cluster_rowpass_kernel<K, C>;
  set_max_smem<K, C>();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs * 64);
  cfg.blockDim = dim3(kNT);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = sm_count() / cs;
  }
  slot = n;
  return n;
}

template <int K, typename C>
static Plan plan_cfg(int P, int64_t nrows, int cs, int cfg_id) {
  Plan pl{};
  pl.cfg = cfg_id;
  pl.cs = cs;
  pl.R = C::R;
  pl.wc = ((P + cs - 1) / cs + 1) & ~1;
  if constexpr (C::DM) {
    // 16-column chunks; row strides = 2 (mod 16) doubles: the fragment loads of
    // neighbouring rows interleave across the banks
    pl.npi = (pl.wc + 15) / 16;
    pl.WQ = pl.npi * 16 + 2;
    pl.WS = pl.npi * 16 + 2;
    if ((pl.wc + 7) / 8 > kNW * C::NMT) return pl;  // slice too wide for the tiles
  } else {
    pl.npi = (pl.wc / 2 + C::KS - 1) / C::KS;
    pl.WQ = 2 * C::KS * pl.npi;
    const int xcols = (pl.wc + 32 * C::CPT - 1) / (32 * C::CPT) * (32 * C::CPT);
    const int need = pl.WQ > xcols ? pl.WQ : xcols;
    pl.WS = (need + 15) / 16 * 16 + 4;  // row stride: 4 doubles of bank skew
  }
  int S = 4;
  const size_t cap = smem_cap<K, C>();
  for (; S >= 3; --S) {
    layout<K, C>(pl, S);
    if (pl.smem <= cap) break;
  }
  if (pl.smem > cap) return pl;  // ok = 0
  const int maxcl = max_clusters<K, C>(cs, pl.smem);
  const int64_t want = nrows > 0 ? (nrows + C::R - 1) / C::R : 1;
  pl.ncl = (int)(want < maxcl ? want : maxcl);
  if (pl.ncl < 1) pl.ncl = 1;
  pl.ok = 1;
  return pl;
}

template <int K>
static Plan make_plan(int P, int64_t nrows) {
  Plan none{};
  for (int cs : {1, 2, 4, 8}) {
    const int wc = ((P + cs - 1) / cs + 1) & ~1;
    if (cs == 1 && wc <= 64) return plan_cfg<K, CfgB>(P, nrows, cs, 1);
    if (wc <= 768) {
      Plan pl = plan_cfg<K, CfgA>(P, nrows, cs, 0);
      if (pl.ok) return pl;
    }
  }
  return none;
}

static Plan plan_for(int dtype, int p, int K, int64_t nrows) {
  Plan none{};
  // A/B switch (work in progress: opt in with SNX_CLUSTER=1)
  static const bool off = getenv("SNX_TWO_PASS") != nullptr || getenv("SNX_CLUSTER") == nullptr;
  if (dtype != SNX_F64 || K < 1 || K > kMaxK || off) return none;
  const int P = padded(p);
  switch (K) {
#define SNX_CL_K(KK) \
  case KK:           \
    return make_plan<KK>(P, nrows);
    SNX_CL_K(1) SNX_CL_K(2) SNX_CL_K(3) SNX_CL_K(4) SNX_CL_K(5) SNX_CL_K(6) SNX_CL_K(7)
    SNX_CL_K(8) SNX_CL_K(9)
#undef SNX_CL_K
    default:
      return none;
  }
}

template <int K, typename C>
static int launch_main(const Plan &pl, Args &a, cudaStream_t st) {
  auto kern = cluster_rowpass_kernel<K, C>;
  if (!set_max_smem<K, C>()) return check_launch("cluster_rowpass attributes");
  carveout(kern);
  a.cs = pl.cs;
  a.ncl = pl.ncl;
  a.wc = pl.wc;
  a.npi = pl.npi;
  a.S = pl.S;
  a.WS = pl.WS;
  a.WQ = pl.WQ;
  a.o_tiles = pl.o_tiles;
  a.o_q = pl.o_q;
  a.o_side = pl.o_side;
  a.o_u = pl.o_u;
  a.o_vr = pl.o_vr;
  a.o_red = pl.o_red;
  a.o_bar = pl.o_bar;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.ncl * pl.cs);
  cfg.blockDim = dim3(kNT);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = pl.cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = a.early ? 2 : 1;
  cudaLaunchKernelEx(&cfg, kern, a);
  return check_launch("cluster_rowpass");
}

static int launch_any(const Plan &pl, int K, Args &a, cudaStream_t st) {
  int rc = 1;
  switch (K) {
#define SNX_CL_K(KK)                                                                  \
  case KK:                                                                            \
    rc = pl.cfg == 0 ? launch_main<KK, CfgA>(pl, a, st) : launch_main<KK, CfgB>(pl, a, st); \
    break;
    SNX_CL_K(1) SNX_CL_K(2) SNX_CL_K(3) SNX_CL_K(4) SNX_CL_K(5) SNX_CL_K(6) SNX_CL_K(7)
    SNX_CL_K(8) SNX_CL_K(9)
#undef SNX_CL_K
    default:
      set_error("snx: cluster row pass: K = %d unsupported", K);
  }
  return rc;
}

// Workspace: [counters (shared with the two-pass layout) | gp[ncl][K*p] | lossp | corrp]
struct ClWs {
  double *gp, *lossp;
  unsigned long long *corrp;
  size_t total;
};

static ClWs ws_layout(void *ws, const Plan &pl, int p, int K) {
  ClWs w{};
  char *b = static_cast<char *>(ws);
  size_t off = round_up(rowpass_counter_bytes(), 256);
  const size_t gbytes = (size_t)pl.ncl * K * p * 8;
  w.gp = reinterpret_cast<double *>(b + off);
  off = round_up(off + gbytes, 256);
  w.lossp = reinterpret_cast<double *>(b + off);
  off = round_up(off + (size_t)pl.ncl * 8, 256);
  w.corrp = reinterpret_cast<unsigned long long *>(b + off);
  off = round_up(off + (size_t)pl.ncl * 8, 256);
  w.total = off;
  return w;
}

}  // namespace clp

// ---- entry points used by snx_rowpass.cu's dispatcher --------------------------------
bool cluster_supported(int dtype, int32_t p, int32_t K) {
  return clp::plan_for(dtype, p, K, 1).ok != 0;
}

size_t cluster_ws_bytes(int dtype, int64_t nrows, int32_t p, int32_t K) {
  const clp::Plan pl = clp::plan_for(dtype, p, K, nrows);
  if (!pl.ok) return 0;
  char dummy;
  return clp::ws_layout(&dummy, pl, p, K).total;
}

// mode: 0 prep (hout), 1 apply (h, skip, dots -> out), 2 grad (labels, loss/corr -> out)
int cluster_rowpass(int mode, const double *X, int64_t ldx, const int64_t *rows, int64_t nrows,
                    int32_t p, int32_t K, const int32_t *labels, const double *w,
                    const double *h, double *hout, double scale, double lam,
                    const double *base, double *out, double *loss_out, long long *corr_out,
                    double *dots, const double *skip, int early, void *ws, size_t ws_bytes,
                    cudaStream_t st) {
  using namespace clp;
  const Plan pl = plan_for(SNX_F64, p, K, nrows);
  if (!pl.ok) {
    set_error("snx: no cluster row-pass plan for p=%d K=%d", p, K);
    return 1;
  }
  const ClWs cw = ws_layout(ws, pl, p, K);
  if (ws == nullptr || ws_bytes < cw.total) {
    set_error("snx: workspace too small for the cluster row pass (%zu < %zu)", ws_bytes,
              cw.total);
    return 1;
  }
  Args a{};
  a.X = X;
  a.ldx = ldx;
  a.rows = rows;
  a.nrows = nrows;
  a.p = p;
  a.K = K;
  a.mode = mode;
  a.w = w;
  a.h = h;
  a.labels = labels;
  a.hout = hout;
  a.gp = cw.gp;
  a.lossp = cw.lossp;
  a.corrp = cw.corrp;
  a.skip = skip;
  a.early = early;
  // weight slices by TMA: every class row slice 16-B aligned, whole 16-B units
  a.qbulk = (reinterpret_cast<uintptr_t>(w) % 16 == 0 && p % 2 == 0 && pl.wc % 2 == 0) ? 1 : 0;
  if (launch_any(pl, K, a, st)) return 1;
  if (mode == kPrep) return 0;
  const int64_t d = (int64_t)K * p;
  const int64_t epb = (d + kDotBlocks - 1) / kDotBlocks;
  int F = 1;
  while (F < 32 && (int64_t)(2 * F) * epb <= kFinThreads) F *= 2;
  launch_pdl_if(true, finalize_kernel, dim3(kDotBlocks), dim3(kFinThreads), 0, st, cw.gp,
                pl.ncl, d, epb, F, scale, lam, base, out, dots, skip,
                mode == kGrad ? (const double *)cw.lossp : nullptr,
                mode == kGrad ? (const unsigned long long *)cw.corrp : nullptr,
                mode == kGrad ? loss_out : nullptr, corr_out);
  return check_launch("cluster finalize");
}

}  // namespace snx

#ifdef SNX_CL_TIMELINE
extern "C" int snx_debug_cl_timeline(unsigned long long *host_out) {
  return cudaMemcpyFromSymbol(host_out, snx::clp::g_cl_tl, sizeof(snx::clp::g_cl_tl)) ==
                 cudaSuccess
             ? 0
             : 1;
}
#endif
