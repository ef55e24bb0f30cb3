// One-pass fp64 row pass (sm_100a): every row of X streamed ONCE per product.
//
// The sampled Hessian product of softmax.py:197-210
//     V = X_S Q(v),  U = V.h - h.rowsum(V.h),  Hv = scale * X_S^T U + lam * v
// and the full-data objective + gradient of softmax.py:125-169
//     Z = X W,  R = E/alpha - onehot,  G = scale * X^T R + lam * w
// have the same shape: a K-wide contraction of every row over all p features,
// a row-local epilogue, and the transposed product with the SAME rows.  The
// two-GEMM path (snx_rowpass.cu) streams X twice with a grid-wide dependency
// between the GEMMs; the kernels here keep a block of rows in shared memory
// for both products.  The contractions run on the fp64 tensor cores
// (mma.sync.m8n8k4.f64, classes 0..7; class 8 of C = 10 by DFMA from the same
// fragments); the row gather of a sample is fused into the TMA bulk copies
// (one per row slice, through the sample's row indices: no X_S copy).
//
// Two shapes of work decomposition:
//   * column split (cluster_rowpass_kernel, p > 64): a cluster of CS CTAs
//     owns a contiguous range of rows, CTA q of the cluster the column slice
//     [q*wc, (q+1)*wc).  Per 8-row block, the 8 compute warps form the slice's
//     partial logits (k split over the warps); an EXCHANGE warp sums the warp
//     partials, pushes them into every peer's shared memory with st.async
//     (distributed shared memory, completion counted on the peer's mbarrier),
//     waits for the peers' partials, sums them in rank order (identical bits
//     on every peer) and runs the row algebra -- all off the compute warps'
//     critical path: they meanwhile compute the NEXT block's logits.  The
//     transposed product then reuses the block's tile; each compute warp owns
//     8-column tiles of X^T U in registers for the whole kernel;
//   * row split (rowsplit_kernel, p <= 64, covertype): each warp owns 8 rows
//     of a 64-row block completely, the row algebra runs in its registers, no
//     block-level synchronisation at all.
// Each cluster / CTA writes a K x p partial; a finalize kernel sums them in a
// fixed order, applies scale and lam and emits the CG dot partials (the
// SNX_DOT_BLOCKS layout of snx_hess_apply).  Every reduction has a fixed order
// and there are no float atomics: results are bit-identical run to run.
// fp64, K <= 9 (the BASELINE shapes: covertype K = 6, MNIST / CIFAR-10 K = 9);
// other shapes use snx_rowpass.cu.
#include <stdio.h>

#include "snx_common.cuh"
#include "snx_internal.h"
#include "snx_pipe.cuh"

namespace snx {
namespace clp {

enum Mode { kPrep = 0, kApply = 1, kGrad = 2 };

constexpr int kNW = 8;             // compute warps (2 per SM sub-partition)
constexpr int kNC = kNW * 32;      // compute threads
constexpr int kNTR = kNC + 32;     // row split: + producer warp
constexpr int kMaxK = 9;
constexpr int kRA = 8;             // rows per block, column split
constexpr int kRR = 8 * kNW;       // rows per block, row split (8 per warp)
constexpr int kNMT = 12;           // column split: X^T U tiles (8 columns) per warp -> wc <= 768
constexpr int kUP = 10;            // U row stride: classes 0..8 + pad (bank spread)
constexpr int kNCH = 6;            // V phase: 16-column chunks per warp (wc <= 768, p <= 64)
constexpr int kNWA = 8;            // column split: compute warps (16 measured slower: the
                                   // larger partial ring forces 8-CTA clusters at p = 3072)
constexpr int kNCA = kNWA * 32;
constexpr int kNMTA = 96 / kNWA;   // column split: X^T U tiles per warp (wc <= 768)
constexpr int kNCHA = 48 / kNWA;   // column split: V chunks per warp
// column split block: compute warps + producer + send warp + NRW row-algebra
// warps (1 for the Hessian passes; 2 for the gradient pass, whose exp / log row
// algebra would otherwise bound the block rate -- they take alternate blocks)
template <int NRW>
constexpr int nta() { return kNCA + 32 * (2 + NRW); }
constexpr int kNTA = nta<2>();     // the larger block (occupancy queries)
#ifndef SNX_KLA
#define SNX_KLA 2
#endif
constexpr int kLA = SNX_KLA;       // column split: logits computed kLA blocks ahead of X^T U
constexpr int kNB3 = kLA + 1;      // red / U rings (blocks in flight between V and X^T U)
constexpr int kSA = kLA + 2;       // column split: ring stages (V(b + kLA), the tiles waiting
                                   // for X^T U, one loading)

struct Args {
  const void *X;          // [n][ldx] fp64 or f32 (the kernels' element type T)
  int64_t ldx;
  const int64_t *rows;    // nullable: sample position -> source row
  int64_t nrows;
  int p, K, cs, ncl, wc, S, WS, WQ;
  int mode;
  const double *w;        // [K][p] class-major weights (v for the Hessian product)
  const double *h;        // apply: [nrows][K] probabilities
  const int32_t *labels;  // grad: labels of the (source) rows
  double *hout;           // prep: [nrows][K]
  double *gp;             // [ncl][K*p] partials of X^T U
  double *lossp;          // grad: [ncl]
  unsigned long long *corrp;  // grad: [ncl]
  const double *skip;
  int early;              // programmatic dependent: stage rows before waiting
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
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
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
// split-phase cluster barrier: arrive now, wait only where a peer's shared
// memory is first addressed (every thread pairs each arrive with one wait)
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// exit barrier of warps that issued no remote shared-memory operation: the
// arrive need not order their (global) stores, so no GPU-scope fence
__device__ __forceinline__ void cluster_sync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// arrive on an mbarrier in a cluster peer's shared memory (release at cluster scope)
__device__ __forceinline__ void mbar_remote_arrive(unsigned raddr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(raddr)
               : "memory");
}
// Relaxed remote arrive (no GPU-scope fence): for a credit that releases only
// shared-memory reads whose values the caller has already consumed.
__device__ __forceinline__ void mbar_remote_arrive_relaxed(unsigned raddr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(raddr)
               : "memory");
}
// spin on a phase (test_wait polls: a thread parked in try_wait is not woken
// promptly by remote complete-tx).  The phase completes only once the peers'
// st.async bytes have landed in this CTA's shared memory.
__device__ __forceinline__ void mbar_poll(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITP_%=:\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITP_%=;\n"
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

// xor butterflies over lane groups of width W (fixed order: identical bits on
// every lane of a group)
template <int W>
__device__ __forceinline__ double gsum(double v) {
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double max_nan(double v, double u) {  // NaN wins (np.max)
  return isnan(v) ? v : (isnan(u) ? u : (u > v ? u : v));
}
template <int W>
__device__ __forceinline__ double gmax_nan(double v) {
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) v = max_nan(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// argmax with numpy's rules: the first NaN, else the largest, ties -> lowest index
__device__ __forceinline__ void amax_take(double &v, int &idx, double u, int j) {
  const bool vn = isnan(v), un = isnan(u);
  const bool take = (vn || un) ? (un && (!vn || j < idx)) : (u > v || (u == v && j < idx));
  if (take) {
    v = u;
    idx = j;
  }
}
template <int W>
__device__ __forceinline__ void gargmax(double &v, int &idx) {
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) {
    const double u = __shfl_xor_sync(0xffffffffu, v, o);
    const int j = __shfl_xor_sync(0xffffffffu, idx, o);
    amax_take(v, idx, u, j);
  }
}

// pairwise (fixed-order) tree over v[B..E): short dependent chains
template <int B, int E, int N>
__device__ __forceinline__ double tree_sum(const double (&v)[N]) {
  if constexpr (E - B == 1) {
    return v[B];
  } else {
    constexpr int M = B + (E - B) / 2;
    return tree_sum<B, M>(v) + tree_sum<M, E>(v);
  }
}

// Optional per-CTA timeline (-DSNX_CL_TIMELINE; tools/cl_timeline.py): compute
// thread 0 and exchange-warp lane 0 stamp %globaltimer at fixed events.
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
#define CL_TLX(b, ev)                                                  \
  do {                                                                 \
    if (threadIdx.x == kNCA + 32 || threadIdx.x == kNCA + 64) cl_stamp((b), (ev)); \
  } while (0)
#define CL_TLP(b, ev)                               \
  do {                                              \
    if (R == kRR && threadIdx.x == kNC) cl_stamp((b), (ev)); \
  } while (0)
#else
#define CL_TLP(b, ev) \
  do {                \
  } while (0)
#define CL_TL(b, ev) \
  do {               \
  } while (0)
#define CL_TLX(b, ev) \
  do {                \
  } while (0)
#endif

// ---------------------------------------------------------------- shared pieces
struct Ring {
  void *tiles;  // [S][R][WS] elements of the data type
  double *Qs, *side;
  uint64_t *full, *empty;
};

// X elements of either data type, widened to fp64 for the fp64 MMAs (f32 data:
// exact conversion, the arithmetic stays fp64)
__device__ __forceinline__ double2 ld2d(const double *p) {
  return *reinterpret_cast<const double2 *>(p);
}
__device__ __forceinline__ double2 ld2d(const float *p) {
  const float2 v = *reinterpret_cast<const float2 *>(p);
  return make_double2((double)v.x, (double)v.y);
}

// Producer warp: the row indices of the first S blocks are loaded at once and
// later ones one block ahead (registers: the ping-pong below keeps every array
// index compile-time); X slices by TMA bulk copies (one per row), or by 16-B
// cp.async pieces in the row split's Hessian passes; side data (h rows /
// labels) by cp.async; each lane arrives on the stage's full barrier once its
// copies have landed.  Launched as a programmatic dependent (`early`), the
// first S stages' X copies go out before griddepcontrol.wait (X and the row
// indices are older than the predecessor grid); everything the predecessor may
// write (weights, h, labels, the skip flag) waits.
template <int R, int K, typename T>
__device__ __forceinline__ void produce(const Args &a, const Ring &rg, int64_t row_lo,
                                        int64_t row_hi, int nb, int c0, int wq, int lane,
                                        int *sh_skip) {
  const int S = R == kRA ? kSA : a.S;  // column split: compile-time ring depth
  const int WS = a.WS;
  const T *X = static_cast<const T *>(a.X);
  const bool apply = a.mode == kApply, grad = a.mode == kGrad;
  // row split, Hessian passes: X by cp.async pieces with the lane's own arrive
  // per block; the consumers read h themselves (no side data)
  const bool pieces_path = R == kRR && !grad;
  constexpr int IPL = (R + 31) / 32;
  constexpr int kSMax = 4;
  auto load_idx = [&](int b, int64_t(&dst)[IPL]) {
    const int64_t r0 = row_lo + (int64_t)b * R;
    const int nr = (int)min((int64_t)R, row_hi - r0);
#pragma unroll
    for (int j = 0; j < IPL; ++j) {
      const int e = lane + 32 * j;
      dst[j] = e < nr ? (a.rows ? a.rows[r0 + e] : r0 + e) : 0;
    }
  };
  auto issue_x = [&](int b, const int64_t(&idx)[IPL]) {
    const int s = b % S;
    if (b >= S) mbar_wait(&rg.empty[s], ((b / S) - 1) & 1);
    const int64_t r0 = row_lo + (int64_t)b * R;
    const int nr = (int)min((int64_t)R, row_hi - r0);
    T *tile = static_cast<T *>(rg.tiles) + (size_t)s * R * WS;
    const unsigned bytes = (unsigned)(wq * sizeof(T));
    if (pieces_path) {
      // rows of a few hundred bytes: one TMA request per row serialises on the
      // copy engine (covertype product 18.2 -> 15.9 us), so 16-B cp.async
      // pieces, each lane its own rows (a lane-contiguous mapping costs a
      // division and two shuffles per piece: 4x slower to issue); each lane's
      // noinc arrive covers this block and the earlier ones only.  The
      // streaming gradient pass keeps the bulk copies (5 % faster there).
      const int pieces = (int)(bytes / 16u);
#pragma unroll
      for (int j = 0; j < IPL; ++j) {
        const int e = lane + 32 * j;
        if (e < nr) {
          const char *src = reinterpret_cast<const char *>(X + idx[j] * a.ldx + c0);
          char *dst = reinterpret_cast<char *>(tile + (size_t)e * WS);
          for (int c = 0; c < pieces; ++c) cp_async16(dst + 16 * c, src + 16 * c);
        }
      }
      cp_async_mbar_arrive(&rg.full[s]);
    } else {
      if (lane == 0) mbar_expect_tx(&rg.full[s], bytes * (unsigned)nr);
      if (bytes > 0) {
#pragma unroll
        for (int j = 0; j < IPL; ++j) {
          const int e = lane + 32 * j;
          if (e < nr)
            bulk_g2s(tile + (size_t)e * WS, X + idx[j] * a.ldx + c0, bytes, &rg.full[s]);
        }
      }
    }
  };
  auto issue_side = [&](int b, const int64_t(&idx)[IPL]) {
    if (pieces_path) return;
    const int s = b % S;
    const int64_t r0 = row_lo + (int64_t)b * R;
    const int nr = (int)min((int64_t)R, row_hi - r0);
    if (apply) {
      double *hs = rg.side + (size_t)s * R * K;
      for (int e = lane; e < nr * K; e += 32) cp_async8(hs + e, a.h + r0 * K + e);
    } else if (grad) {
      int *ls = reinterpret_cast<int *>(rg.side) + s * R;
#pragma unroll
      for (int j = 0; j < IPL; ++j) {
        const int e = lane + 32 * j;
        if (e < nr) cp_async4(ls + e, a.labels + idx[j]);
      }
    }
    cp_async_mbar_arrive(&rg.full[s]);
  };
  // A programmatic dependent (apply) stages the first min(S, nb) blocks' X
  // before griddepcontrol.wait, all their indices in flight at once; the side
  // data (h) follows the wait.  Otherwise each block's side data goes right
  // behind its X.  (grad is never launched early: its labels need the indices.)
  const bool early = a.early && !grad;
  const int nb0 = early ? min(nb, S) : 0;
  if (early) {
    int64_t e_idx[kSMax][IPL];
#pragma unroll
    for (int k = 0; k < kSMax; ++k)
      if (k < nb0) load_idx(k, e_idx[k]);
#pragma unroll
    for (int k = 0; k < kSMax; ++k) {
      if (k < nb0) issue_x(k, e_idx[k]);
      CL_TLP(k, 2);
    }
  }
  pdl_wait();
  if (lane == 0) *sh_skip = (a.skip != nullptr && *a.skip != 0.0) ? 1 : 0;
  __syncwarp();
  if (*sh_skip) {  // complete the staged phases (no copy left in flight), then leave
    cp_async_wait_all();
    for (int bb = 0; bb < nb0; ++bb) {
      if (!pieces_path) mbar_arrive(&rg.full[bb % S]);  // the side arrivals
      mbar_wait(&rg.full[bb % S], (bb / S) & 1);
    }
    return;
  }
  CL_TLP(-1, 7);
  int64_t cur[IPL], nxt[IPL];
#pragma unroll
  for (int j = 0; j < IPL; ++j) cur[j] = nxt[j] = 0;
  for (int bb = 0; bb < nb0; ++bb) issue_side(bb, cur);  // apply: no use of the indices
  // the rest: indices one block ahead
  if (nb0 < nb) load_idx(nb0, cur);
  for (int b = nb0; b < nb; ++b) {
    if (b + 1 < nb) load_idx(b + 1, nxt);
    issue_x(b, cur);
    CL_TLP(b, 2);
    issue_side(b, cur);
#pragma unroll
    for (int j = 0; j < IPL; ++j) cur[j] = nxt[j];
  }
}

// The weights stay in registers for the whole kernel: a warp's V chunks are
// fixed (ch = ch0 + step i), so lane (g, t) keeps the B fragments
// w[g][16 ch + 4 t + s] (s = 0..3) of its NCH chunks (zero past the slice, past
// p, or for classes >= K).  Class 8 (K = 9) is a shared-memory row (smem
// broadcasts: the four lanes of a group read one 16-B pair).
template <int K, int NCH>
__device__ __forceinline__ void load_qfrag(const Args &a, int c0, int wq, int g, int t, int ch0,
                                           int step, int nch, double (&qf)[NCH][4]) {
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    const int ch = ch0 + step * i;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int j = 16 * ch + 4 * t + s, gc = c0 + j;
      qf[i][s] = (ch < nch && g < K && j < wq && gc < a.p) ? a.w[(int64_t)g * a.p + gc] : 0.0;
    }
  }
}
// class-8 row by cp.async (all copies in flight at once); the caller waits
// with cp_async_wait_all() before the consumers' barrier
template <int K>
__device__ __forceinline__ void load_q8(const Args &a, double *q8, int c0, int wq, int n,
                                        int tid, int nthreads) {
  if constexpr (K == 9)
    for (int j = tid; j < n; j += nthreads) {
      if (j < wq && c0 + j < a.p)
        cp_async8(q8 + j, a.w + (int64_t)8 * a.p + c0 + j);
      else
        q8[j] = 0.0;
    }
}


// V phase of one 8-row group: C = X[8 rows][chunks] Q^T on m8n8k4, the 16
// columns of chunk ch at physical column 16 ch + 4 t + s for step s (so a
// lane's A and B values are 2 contiguous 16-B loads each).  Returns the lane's
// C = (V[g][2t], V[g][2t+1]) and v8 = the row's class-8 logit partial (summed
// over the 4 lanes of the group, K == 9).
template <int K, int NCH, typename T>
__device__ __forceinline__ void vgroup(const T *xrow, const double *q8row,
                                       const double (&qf)[NCH][4], int ch0, int step, int nch,
                                       double (&c2)[2], double &v8) {
  // two independent accumulator chains (steps 0,1 and 2,3), added at the end
  double ca[2] = {0.0, 0.0}, cb[2] = {0.0, 0.0}, va = 0.0, vb = 0.0;
#pragma unroll
  for (int i = 0; i < NCH; ++i) {
    const int ch = ch0 + step * i;
    if (ch < nch) {
      const double2 xa = ld2d(xrow + 16 * ch);
      const double2 xb = ld2d(xrow + 16 * ch + 2);
      dmma(ca, xa.x, qf[i][0]);
      dmma(cb, xb.x, qf[i][2]);
      dmma(ca, xa.y, qf[i][1]);
      dmma(cb, xb.y, qf[i][3]);
      if constexpr (K == 9) {
        const double2 ra = *reinterpret_cast<const double2 *>(q8row + 16 * ch);
        const double2 rb = *reinterpret_cast<const double2 *>(q8row + 16 * ch + 2);
        va = fma(xa.x, ra.x, va);
        vb = fma(xb.x, rb.x, vb);
        va = fma(xa.y, ra.y, va);
        vb = fma(xb.y, rb.y, vb);
      }
    }
  }
  c2[0] = ca[0] + cb[0];
  c2[1] = ca[1] + cb[1];
  v8 = 0.0;
  if constexpr (K == 9) v8 = gsum<4>(va + vb);
}

// X^T U of one 8-row group into the warp's column tiles: tile m covers
// columns 8 (m0 + mstep m) .. +7; rows of step s, lane t: 2t + s (each bank
// hit by two of the four rows).  u points at the group's U rows (stride kUP).
template <int K, int NMT, typename T>
__device__ __forceinline__ void xgroup(const T *x0, int WS, const double *u, int nr, int g,
                                       int t, int m0, int mstep, int nmt, double (&acc)[NMT][2],
                                       double (&acc8)[NMT]) {
  const double ua0 = u[(2 * t) * kUP + g], ua1 = u[(2 * t + 1) * kUP + g];
  const double u80 = K == 9 ? u[(2 * t) * kUP + 8] : 0.0;
  const double u81 = K == 9 ? u[(2 * t + 1) * kUP + 8] : 0.0;
  const bool ok0 = 2 * t < nr, ok1 = 2 * t + 1 < nr;
  const T *xa = x0 + (size_t)(2 * t) * WS + g;
  const T *xb = xa + WS;
#pragma unroll
  for (int m = 0; m < NMT; ++m) {
    const int mt = m0 + mstep * m;
    if (mt < nmt) {
      const double a0 = ok0 ? xa[8 * mt] : 0.0;
      const double a1 = ok1 ? xb[8 * mt] : 0.0;
      dmma(acc[m], a0, ua0);
      dmma(acc[m], a1, ua1);
      if constexpr (K == 9) {
        acc8[m] = fma(a0, u80, acc8[m]);
        acc8[m] = fma(a1, u81, acc8[m]);
      }
    }
  }
}

// X^T U of one 8-row block on m16n8k8: tile m covers columns 16 mt .. +15
// (mt = m0 + mstep m); lane (g, t) holds A = X^T values of columns g, g + 8 at
// rows 2t, 2t + 1, B = U rows 2t, 2t + 1 at class g, C = (columns g, g + 8) x
// (classes 2t, 2t + 1); class 8 by DFMA (per lane: rows 2t, 2t + 1 of columns
// g, g + 8; the four lanes of a group cover the 8 rows).
template <int K, int NMT, typename T>
__device__ __forceinline__ void xgroup16(const T *x0, int WS, const double *u, int nr, int g,
                                         int t, int m0, int mstep, int nmt16,
                                         double (&acc)[NMT][4], double (&acc8)[NMT][2]) {
  // the MMA's k index runs over the block's rows permuted (k = t -> row 2t,
  // k = t + 4 -> row 2t + 1), the same for A and B: a warp's A loads then hit
  // every bank pair exactly twice (rows 4 x WS = 2 mod 16 apart)
  const double b0 = u[(2 * t) * kUP + g], b1 = u[(2 * t + 1) * kUP + g];
  const double u8a = K == 9 ? u[(2 * t) * kUP + 8] : 0.0;
  const double u8b = K == 9 ? u[(2 * t + 1) * kUP + 8] : 0.0;
  const bool okt = 2 * t < nr, okt4 = 2 * t + 1 < nr;
  const T *xa = x0 + (size_t)(2 * t) * WS + g;
  const T *xb = xa + WS;
#pragma unroll
  for (int m = 0; m < NMT; ++m) {
    const int mt = m0 + mstep * m;
    if (mt < nmt16) {
      const double a0 = okt ? xa[16 * mt] : 0.0, a1 = okt ? xa[16 * mt + 8] : 0.0;
      const double a2 = okt4 ? xb[16 * mt] : 0.0, a3 = okt4 ? xb[16 * mt + 8] : 0.0;
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+d"(acc[m][0]), "+d"(acc[m][1]), "+d"(acc[m][2]), "+d"(acc[m][3])
          : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
      if constexpr (K == 9) {
        acc8[m][0] = fma(a0, u8a, acc8[m][0]);
        acc8[m][1] = fma(a1, u8a, acc8[m][1]);
        acc8[m][0] = fma(a2, u8b, acc8[m][0]);
        acc8[m][1] = fma(a3, u8b, acc8[m][1]);
      }
    }
  }
}

// Send warp, one block: the CTA's partial logits (the compute warps' partials
// summed in a fixed tree) -> every peer's Vr[B & 1][q] by st.async, counted on
// the peer's vfull[B & 1].  B: the block's position in the CTA's ring sequence.
template <int K>
__device__ __forceinline__ void send_block(const double *red, double *Vr, uint64_t *vfull,
                                           unsigned q, int cs, int lane, int64_t B, int nr) {
  constexpr int R = kRA;
  const double *rb = red + (size_t)(B % kNB3) * kNWA * R * K;
  const unsigned vr_local = smem_u32(Vr + ((size_t)(B & 1) * cs + q) * R * K);
  const unsigned bar_local = smem_u32(&vfull[B & 1]);
  constexpr int EPL = (R * K + 31) / 32;
  double tot[EPL];
#pragma unroll
  for (int h = 0; h < kNWA / 8; ++h) {  // eight warps' partials at a time
    double v[EPL][8];
#pragma unroll
    for (int j = 0; j < EPL; ++j) {
      const int e = lane + 32 * j;
#pragma unroll
      for (int w = 0; w < 8; ++w) v[j][w] = e < nr * K ? rb[(8 * h + w) * R * K + e] : 0.0;
    }
#pragma unroll
    for (int j = 0; j < EPL; ++j) tot[j] = h == 0 ? tree_sum<0, 8>(v[j]) : tot[j] + tree_sum<0, 8>(v[j]);
  }
#pragma unroll
  for (int j = 0; j < EPL; ++j) {
    const int e = lane + 32 * j;
    const double sm = tot[j];
    if (e < nr * K)
      for (int pq = 0; pq < cs; ++pq)
        st_async(mapa(vr_local + e * 8, pq), sm, mapa(bar_local, pq));
  }
}

// Row-algebra warp, one block (lanes: 4 per row): z = the peers' partial
// logits summed in rank order, then the mode's row algebra (apply: U =
// diag(h) z - h (h.z), the V.U curvature sum; prep: h; grad: residual, loss,
// accuracy), U rows -> Us[B % 3], ufull[B % 3], and the credit for Vr[B & 1]
// to every peer.
template <int K>
__device__ __forceinline__ void rows_block(const Args &a, const Ring &rg, const double *Vr,
                                           double *Us, uint64_t *ufull, uint64_t *credit,
                                           unsigned q, int cs, int lane, int64_t B, int s,
                                           int64_t r0, int nr, double &loss_acc,
                                           unsigned long long &corr_acc) {
  constexpr int R = kRA;
  const bool apply = a.mode == kApply, prep = a.mode == kPrep;
  // all 8 rows at once: 4 lanes per row, lane `sub` owns classes sub,
  // sub + 4, sub + 8
  const double *vr = Vr + (size_t)(B & 1) * cs * R * K;
  double *u = Us + (size_t)(B % kNB3) * R * kUP;
  const int row = lane >> 2, sub = lane & 3;
  const bool rv = row < nr;
  double z[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int c = sub + 4 * j;
    double pz[4] = {0.0, 0.0, 0.0, 0.0};
    if (rv && c < K) {
#pragma unroll
      for (int pq = 0; pq < 4; ++pq)
        if (pq < cs) pz[pq] = vr[(pq * R + row) * K + c];
#pragma unroll
      for (int pq = 4; pq < 8; ++pq)
        if (pq < cs) pz[pq - 4] += vr[(pq * R + row) * K + c];
    }
    z[j] = (pz[0] + pz[1]) + (pz[2] + pz[3]);
  }
  double uo[3] = {0.0, 0.0, 0.0};
  if (apply) {
    double hv[3], vw[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int c = sub + 4 * j;
      hv[j] = (rv && c < K) ? rg.side[((size_t)s * R + row) * K + c] : 0.0;
      vw[j] = z[j] * hv[j];
    }
    const double sm = gsum<4>((vw[0] + vw[1]) + vw[2]);  // softmax.py:207 rowsum(VW)
#pragma unroll
    for (int j = 0; j < 3; ++j) uo[j] = vw[j] - hv[j] * sm;
    // curvature pieces: s.(X^T U) = sum over rows of V.U (the fused CG update)
    if (rv) loss_acc += (z[0] * uo[0] + z[1] * uo[1]) + z[2] * uo[2];
  } else {
    // softmax.py:91-98: M = max(0, max_c z); E = exp(z - M); alpha = e^-M + sum E
    double M = 0.0;
#pragma unroll
    for (int j = 0; j < 3; ++j)
      if (sub + 4 * j < K) M = max_nan(M, z[j]);
    M = gmax_nan<4>(M);
    double E[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) E[j] = (sub + 4 * j < K) ? exp(z[j] - M) : 0.0;
    const double eM = exp(-M);
    const double alpha = eM + gsum<4>((E[0] + E[1]) + E[2]);
    const double ia = 1.0 / alpha;  // one division per lane (alpha >= 1 for finite rows)
    if (prep) {
#pragma unroll
      for (int j = 0; j < 3; ++j)
        if (rv && sub + 4 * j < K && q == 0) a.hout[(r0 + row) * K + sub + 4 * j] = E[j] * ia;
    } else {
      // grad: residual (softmax.py:157-161), loss (:134), accuracy (:224-247)
      const int y = rv ? reinterpret_cast<const int *>(rg.side)[s * R + row] : -1;
      double pr[3], lin = 0.0;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int c = sub + 4 * j;
        pr[j] = E[j] * ia;
        uo[j] = pr[j] - (c == y ? 1.0 : 0.0);
        if (c < K && c == y) lin = z[j];
      }
      lin = gsum<4>(lin);
      if (rv && sub == 0 && q == 0) loss_acc += (M + log(alpha)) - lin;
      double bv = -INFINITY;
      int bi = K + 1;
#pragma unroll
      for (int j = 0; j < 3; ++j)
        if (sub + 4 * j < K) amax_take(bv, bi, pr[j], sub + 4 * j);
      gargmax<4>(bv, bi);
      amax_take(bv, bi, eM * ia, K);  // the reference class
      if (rv && sub == 0 && q == 0 && bi == y) corr_acc += 1ull;
    }
  }
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int c = sub + 4 * j;
    if (c < kUP) u[row * kUP + c] = (rv && c < K) ? uo[j] : 0.0;
  }
  CL_TLX((int)B, 9);
  mbar_arrive(&ufull[B % kNB3]);  // each lane releases its own U stores
  // this CTA's receive slot (B & 1) is read -- the U stores above consumed
  // every value read, so those loads have completed: hand the credit to
  // every sender with a relaxed arrive (no GPU-scope fence per block)
  __syncwarp();
  if (lane < cs) mbar_remote_arrive_relaxed(mapa(smem_u32(&credit[B & 1]), (unsigned)lane));
}

// ---------------------------------------------------------------- column split
template <int K, int NRW, typename T>
__global__ void __launch_bounds__(nta<NRW>(), 1)
    cluster_rowpass_kernel(const __grid_constant__ Args a) {
  constexpr int R = kRA;
  pdl_trigger();  // the finalize kernel may launch now (it waits for this grid)
  extern __shared__ __align__(1024) unsigned char smem[];
  Ring rg;
  rg.tiles = smem + a.o_tiles;                                       // [S][R][WS] T
  T *tiles = static_cast<T *>(rg.tiles);
  rg.side = reinterpret_cast<double *>(smem + a.o_side);            // [S][R][K] h | [S][R] int
  double *Q8 = reinterpret_cast<double *>(smem + a.o_q);            // [WQ] class-8 weights
  double *Us = reinterpret_cast<double *>(smem + a.o_u);            // [3][R][kUP]
  double *Vr = reinterpret_cast<double *>(smem + a.o_vr);           // [2][cs][R][K]
  double *red = reinterpret_cast<double *>(smem + a.o_red);         // [3][NW][R][K]
  rg.full = reinterpret_cast<uint64_t *>(smem + a.o_bar);
  rg.empty = rg.full + a.S;
  uint64_t *vfull = rg.empty + a.S;  // [2] peers' partial logits landed
  uint64_t *credit = vfull + 2;      // [2] every peer has consumed this CTA's slot (b & 1)
  uint64_t *redfull = credit + 2;    // [3] compute warps' partials written
  uint64_t *ufull = redfull + kNB3;  // [3] U rows ready
  uint64_t *redfree = ufull + kNB3;  // [3] prep: the send warp has read red[b % 3]
  __shared__ int sh_skip;

  // the warp index through a shuffle: provably warp-uniform for the compiler
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  constexpr int S = kSA;
  const int WS = a.WS, cs = a.cs;
  CL_TL(-1, 0);
  const unsigned q = cluster_rank();
  const int cl = (int)cluster_id();
  const int64_t row_lo = a.nrows * cl / a.ncl, row_hi = a.nrows * (cl + 1) / a.ncl;
  const int nb = (int)((row_hi - row_lo + R - 1) / R);
  const int c0 = (int)q * a.wc;                                 // first column of the slice
  const int wq = max(0, min(a.wc, ((a.p + 3) & ~3) - c0));      // slice width (even)
  const bool apply = a.mode == kApply, grad = a.mode == kGrad, prep = a.mode == kPrep;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&rg.full[s], 32);
      mbar_init(&rg.empty[s], kNWA);
    }
    for (int j = 0; j < 2; ++j) {
      mbar_init(&vfull[j], 1);
      mbar_init(&credit[j], a.cs);
    }
    for (int j = 0; j < kNB3; ++j) {
      mbar_init(&redfull[j], kNWA);
      mbar_init(&ufull[j], 32);
      mbar_init(&redfree[j], 1);
    }
    mbar_fence_init();
  }
  // zero the tile columns no bulk copy writes (the chunks / tiles read them)
  for (int i = tid; i < S * R * (WS - wq); i += nta<NRW>()) {
    const int r = i / (WS - wq), j = i - r * (WS - wq);
    tiles[(size_t)r * WS + wq + j] = T(0);
  }
  __syncthreads();
  CL_TL(-1, 6);
  if (tid == 0) {  // the first block of each row-algebra warp
    for (int b = 0; b < NRW && b < nb; ++b) {
      const int nr0 = (int)min((int64_t)R, row_hi - (row_lo + (int64_t)b * R));
      mbar_arrive_expect_tx(&vfull[b & 1], (unsigned)(cs * nr0 * K * 8));
    }
  }
  // peers' barriers must be initialised before any st.async / remote arrive:
  // arrive here, wait only in the two warps that address peers (the others
  // pair their wait before the exit barrier)
  cluster_arrive();
  CL_TL(-1, 7);

  if (warp == kNWA) {  // ---------------------------------------- producer
    produce<R, K, T>(a, rg, row_lo, row_hi, nb, c0, wq, lane, &sh_skip);
    cluster_wait();
    cluster_sync_relaxed();
    return;
  }
  pdl_wait();  // the weights, h and the skip flag may be the predecessor's outputs
  CL_TL(-1, 8);
  const int g8 = lane >> 2, t4 = lane & 3;
  const int nch = (wq + 15) >> 4, nmt = (wq + 7) >> 3;
  double qf[kNCHA][4];
  if (warp < kNWA) {  // weight loads in flight before the skip test
    load_qfrag<K, kNCHA>(a, c0, wq, g8, t4, warp, kNWA, nch, qf);
    load_q8<K>(a, Q8, c0, wq, a.WQ, tid, kNCA);
  }
  if (a.skip != nullptr && *a.skip != 0.0) {
    cp_async_wait_all();
    cluster_wait();
    cluster_sync_relaxed();
    return;
  }

  if (warp == kNWA + 1) {  // ---------------------------------------- send warp
    cluster_wait();
    // the CTA's partial logits of block b -> every peer's Vr[b & 1][q].  The
    // FP64 pipe is shared with the compute warps' MMA stream, so the dependent
    // FP64 chains here are kept short (independent elements per lane,
    // pairwise fixed-order trees).
    for (int b = 0; b < nb; ++b) {
      const int64_t r0 = row_lo + (int64_t)b * R;
      const int nr = (int)min((int64_t)R, row_hi - r0);
      mbar_wait(&redfull[b % kNB3], (b / kNB3) & 1);
      // credit: every peer has read its slot (b & 1) of block b - 2 (so its
      // receive buffer and vfull phase are free for block b)
      if (b >= 2) mbar_wait(&credit[b & 1], ((b >> 1) - 1) & 1);
      __syncwarp();  // lanes leave a polling loop one by one: reconverge
      CL_TLX(b, 6);
      send_block<K>(red, Vr, vfull, q, cs, lane, b, nr);
      // prep: the compute warps do not wait for U, so red[b % 3] is handed
      // back explicitly (the sums above consumed every value read)
      __syncwarp();
      if (prep && lane == 0) mbar_arrive(&redfree[b % kNB3]);
      CL_TLX(b, 7);
    }
    cluster_sync_all();
    return;
  }

  if (warp >= kNWA + 2) {  // --------------------------- row-algebra warps
    // warp j takes blocks j, j + NRW, ...; block b's receive slot is vfull[b & 1],
    // re-armed for block b + NRW once this block's phase is done
    static_assert(NRW == 1 || NRW == 2, "two receive slots");
    cluster_wait();
    const int j = warp - (kNWA + 2);
    double loss_acc = 0.0;
    unsigned long long corr_acc = 0;
    for (int b = j; b < nb; b += NRW) {
      const int s = b % S;
      const int64_t r0 = row_lo + (int64_t)b * R;
      const int nr = (int)min((int64_t)R, row_hi - r0);
      // the peers' partials of block b, summed in rank order -> row algebra
      mbar_poll(&vfull[b & 1], (b >> 1) & 1);
      __syncwarp();
      CL_TLX(b, 8);
      if (lane == 0 && b + NRW < nb) {  // arm slot (b + NRW) & 1 for block b + NRW
        const int nrn = (int)min((int64_t)R, row_hi - (r0 + NRW * R));
        mbar_arrive_expect_tx(&vfull[(b + NRW) & 1], (unsigned)(cs * nrn * K * 8));
      }
      rows_block<K>(a, rg, Vr, Us, ufull, credit, q, cs, lane, b, s, r0, nr, loss_acc, corr_acc);
    }
    if (grad || apply) {  // apply: lossp[cl] = the cluster's sum of V.U (curvature)
      double l = warp_allsum(loss_acc);
      unsigned long long cc = corr_acc;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cc += __shfl_xor_sync(0xffffffffu, cc, o);
      if constexpr (NRW == 2) {  // fixed order: warp 0's sum + warp 1's
        __shared__ double sh_rl;
        __shared__ unsigned long long sh_rc;
        if (j == 1 && lane == 0) {
          sh_rl = l;
          sh_rc = cc;
        }
        asm volatile("bar.sync 2, 64;\n" ::: "memory");  // the two row-algebra warps
        l += sh_rl;
        cc += sh_rc;
      }
      if (j == 0 && lane == 0 && q == 0) {
        a.lossp[cl] = l;
        a.corrp[cl] = cc;
      }
    }
    cluster_sync_all();
    return;
  }

  // ---------------------------------------------------------- compute warps
  CL_TL(-1, 9);
  cp_async_wait_all();
  consumer_sync(kNCA);
  CL_TL(-1, 1);
  constexpr int NM16 = kNMTA / 2;  // 16-column X^T U tiles per warp
  const int nmt16 = (wq + 15) >> 4;
  double acc[NM16][4], acc8[NM16][2];
#pragma unroll
  for (int m = 0; m < NM16; ++m) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = acc8[m][0] =
      acc8[m][1] = 0.0;

  // partial logits of block b (k split over the warps) -> red[b & 1][warp]
  auto vphase = [&](int b) {
    const int s = b % S;
    mbar_wait(&rg.full[s], (b / S) & 1);
    __syncwarp();  // reconverge before the warp-wide MMAs
    const T *tile = tiles + (size_t)s * R * WS;
    double c2[2], v8;
    vgroup<K, kNCHA, T>(tile + (size_t)g8 * WS + 4 * t4, Q8 + 4 * t4, qf, warp, kNWA, nch, c2, v8);
    double *rbw = red + (size_t)(b % kNB3) * kNWA * R * K + (size_t)warp * R * K + g8 * K;
    if (2 * t4 < K) rbw[2 * t4] = c2[0];
    if (2 * t4 + 1 < K) rbw[2 * t4 + 1] = c2[1];
    if (K == 9 && t4 == 0) rbw[8] = v8;
    __syncwarp();
    if (lane == 0) mbar_arrive(&redfull[b % kNB3]);
  };

  // logits run kLA blocks ahead of X^T U: the exchange (warp sums, DSMEM
  // push, peers' partials, row algebra) of a block has kLA blocks of compute
  // to hide behind.  (Compile-time full-slice variants of the two MMA streams,
  // without the per-chunk / per-tile bounds tests, measured 1 us slower.)
  if (prep) {
    // h only: no X^T U, so a stage is released right after its logits and the
    // logits stream at the rate the exchange and the row algebra drain them
    CL_TL(-1, 2);
    for (int b = 0; b < nb; ++b) {
      CL_TL(b, 0);
      if (b >= kNB3) mbar_wait(&redfree[b % kNB3], ((b / kNB3) - 1) & 1);
      __syncwarp();
      CL_TL(b, 2);
      vphase(b);
      CL_TL(b, 1);
      if (lane == 0) mbar_arrive(&rg.empty[b % S]);
    }
    CL_TL(-1, 3);
    CL_TL(-1, 4);
    cluster_wait();          // the prologue's arrive
    cluster_sync_relaxed();  // no CTA leaves while a peer may still address its smem
    CL_TL(-1, 5);
    return;
  }
  for (int b = 0; b < kLA && b < nb; ++b) vphase(b);
  CL_TL(-1, 2);
  for (int b = 0; b < nb; ++b) {
    CL_TL(b, 0);
    if (b + kLA < nb) vphase(b + kLA);
    CL_TL(b, 1);
    mbar_wait(&ufull[b % kNB3], (b / kNB3) & 1);
    __syncwarp();
    CL_TL(b, 2);
    if (!prep) {
      const int64_t r0 = row_lo + (int64_t)b * R;
      const int nr = (int)min((int64_t)R, row_hi - r0);
      xgroup16<K, NM16, T>(tiles + (size_t)(b % S) * R * WS, WS,
                        Us + (size_t)(b % kNB3) * R * kUP, nr, g8, t4, warp, kNWA, nmt16, acc,
                        acc8);
    }
    CL_TL(b, 3);
    __syncwarp();
    if (lane == 0) mbar_arrive(&rg.empty[b % S]);
  }
  CL_TL(-1, 3);
  if (!prep) {
    const int64_t d = (int64_t)K * a.p;
    double *gq = a.gp + (int64_t)cl * d;
#pragma unroll
    for (int m = 0; m < NM16; ++m) {
      const int mt = warp + kNWA * m;
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // columns g (c0, c1) and g + 8 (c2, c3)
        const double s8 = K == 9 ? gsum<4>(acc8[m][h]) : 0.0;
        const int col = 16 * mt + g8 + 8 * h, gc = c0 + col;
        if (mt < nmt16 && col < wq && gc < a.p) {
          if (2 * t4 < K) gq[(int64_t)(2 * t4) * a.p + gc] = acc[m][2 * h];
          if (2 * t4 + 1 < K) gq[(int64_t)(2 * t4 + 1) * a.p + gc] = acc[m][2 * h + 1];
          if (K == 9 && t4 == 0) gq[(int64_t)8 * a.p + gc] = s8;
        }
      }
    }
  }
  CL_TL(-1, 4);
  cluster_wait();          // the prologue's arrive
  cluster_sync_relaxed();  // no CTA leaves while a peer may still address its smem
  CL_TL(-1, 5);
}

// ---------------------------------------------------------------- row split
// p <= 64: warp w owns rows 8w..8w+7 of every 64-row block completely (V over
// all columns, the row algebra in registers, X^T U of its rows); the CTA's
// K x p partial is reduced over the warps once at the end.
template <int K, typename T>
__global__ void __launch_bounds__(kNTR, 1) rowsplit_kernel(const __grid_constant__ Args a) {
  constexpr int R = kRR;
  constexpr int NMT = 8;  // column tiles: p <= 64
  CL_TL(-1, 0);
  pdl_trigger();
  extern __shared__ __align__(1024) unsigned char smem[];
  Ring rg;
  rg.tiles = smem + a.o_tiles;  // [S][R][WS] T
  T *tiles = static_cast<T *>(rg.tiles);
  rg.side = reinterpret_cast<double *>(smem + a.o_side);    // [S][R][K] h | [S][R] int
  double *Q8 = reinterpret_cast<double *>(smem + a.o_q);    // [WQ] class-8 weights
  double *Uw = reinterpret_cast<double *>(smem + a.o_u);    // [NW][8][kUP] per warp
  rg.full = reinterpret_cast<uint64_t *>(smem + a.o_bar);
  rg.empty = rg.full + a.S;
  __shared__ int sh_skip;
  __shared__ double sh_loss[kNW];
  __shared__ unsigned long long sh_corr[kNW];

  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const int S = a.S, WS = a.WS;
  const int cl = blockIdx.x;
  const int64_t row_lo = a.nrows * cl / a.ncl, row_hi = a.nrows * (cl + 1) / a.ncl;
  const int nb = (int)((row_hi - row_lo + R - 1) / R);
  const int wq = (a.p + 3) & ~3;  // the whole (padded) row
  const bool apply = a.mode == kApply, grad = a.mode == kGrad, prep = a.mode == kPrep;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&rg.full[s], 32);
      mbar_init(&rg.empty[s], kNW);
    }
    mbar_fence_init();
  }
  for (int i = tid; i < S * R * (WS - wq); i += kNTR) {
    const int r = i / (WS - wq), j = i - r * (WS - wq);
    tiles[(size_t)r * WS + wq + j] = T(0);
  }
  __syncthreads();
  CL_TL(-1, 6);
  if (warp == kNW) {
    produce<R, K, T>(a, rg, row_lo, row_hi, nb, 0, wq, lane, &sh_skip);
    return;
  }
  pdl_wait();
  CL_TL(-1, 8);
  if (a.skip != nullptr && *a.skip != 0.0) return;
  const int g = lane >> 2, t = lane & 3;
  const int nch = (wq + 15) >> 4, nmt = (wq + 7) >> 3;
  double qf[kNCH][4];
  load_qfrag<K, kNCH>(a, 0, wq, g, t, 0, 1, nch, qf);
  CL_TL(-1, 9);
  load_q8<K>(a, Q8, 0, wq, a.WQ, tid, kNC);
  cp_async_wait_all();
  consumer_sync(kNC);
  CL_TL(-1, 1);
  double acc[NMT][2], acc8[NMT];
#pragma unroll
  for (int m = 0; m < NMT; ++m) acc[m][0] = acc[m][1] = acc8[m] = 0.0;
  double loss_acc = 0.0;
  unsigned long long corr_acc = 0;
  double *u = Uw + (size_t)warp * 8 * kUP;
  const bool c0v = 2 * t < K, c1v = 2 * t + 1 < K;

  int s = 0;         // ring stage of block b (S is a runtime 2..4: no division per block)
  unsigned ph = 0;   // its phase parity
  for (int b = 0; b < nb; ++b) {
    const int64_t r0 = row_lo + (int64_t)b * R;
    const int nr = (int)min((int64_t)R, row_hi - r0);
    const int gr0 = 8 * warp;          // the warp's first row in the block
    const int ng = min(8, nr - gr0);   // its valid rows (warp-uniform)
    mbar_wait(&rg.full[s], ph);
    CL_TL(b, 0);
    __syncwarp();  // reconverge before the warp-wide MMAs
    if (ng > 0) {
      const T *tile = tiles + (size_t)s * R * WS + (size_t)gr0 * WS;
      const int row = gr0 + g;
      const bool rv = g < ng;
      // apply: the lane's h values straight from global memory, in flight
      // during the logits MMAs
      double h0 = 0.0, h1 = 0.0, h8 = 0.0;
      if (apply && rv) {
        const double *hr = a.h + (r0 + row) * K;
        if (c0v) h0 = __ldcg(hr + 2 * t);
        if (c1v) h1 = __ldcg(hr + 2 * t + 1);
        if (K == 9) h8 = __ldcg(hr + (K == 9 ? 8 : 0));
      }
      double c2[2], v8;
      vgroup<K, kNCH, T>(tile + (size_t)g * WS + 4 * t, Q8 + 4 * t, qf, 0, 1, nch, c2, v8);
      // row algebra: lane (g, t) holds classes 2t, 2t+1 of row g (+ class 8)
      const double z0 = c0v ? c2[0] : 0.0, z1 = c1v ? c2[1] : 0.0, z8 = K == 9 ? v8 : 0.0;
      double u0 = 0.0, u1 = 0.0, u8 = 0.0;
      if (apply) {
        const double w0 = z0 * h0, w1 = z1 * h1, w8 = z8 * h8;
        const double sm = gsum<4>(w0 + w1) + w8;  // softmax.py:207 rowsum(VW)
        u0 = w0 - h0 * sm;
        u1 = w1 - h1 * sm;
        u8 = w8 - h8 * sm;
        if (rv) loss_acc += (z0 * u0 + z1 * u1) + (t == 0 ? z8 * u8 : 0.0);  // V.U
      } else {
        // softmax.py:91-98: M = max(0, max_c z); E = exp(z - M); alpha = e^-M + sum E
        double M = max_nan(c0v ? z0 : 0.0, c1v ? z1 : 0.0);
        M = gmax_nan<4>(M);
        if (K == 9) M = max_nan(M, z8);
        M = max_nan(M, 0.0);
        const double E0 = c0v ? exp(z0 - M) : 0.0, E1 = c1v ? exp(z1 - M) : 0.0;
        const double E8 = K == 9 ? exp(z8 - M) : 0.0;
        const double eM = exp(-M);
        const double alpha = eM + (gsum<4>(E0 + E1) + E8);
        const double ia = 1.0 / alpha;  // one division per lane
        if (prep) {
          if (rv) {
            double *ho = a.hout + (r0 + row) * K;
            if (c0v) ho[2 * t] = E0 * ia;
            if (c1v) ho[2 * t + 1] = E1 * ia;
            if (K == 9 && t == 0) ho[K == 9 ? 8 : 0] = E8 * ia;
          }
        } else {
          // grad: residual (softmax.py:157-161), loss (:134), accuracy (:224-247)
          const int y = rv ? reinterpret_cast<const int *>(rg.side)[s * R + row] : -1;
          const double p0 = E0 * ia, p1 = E1 * ia, p8 = E8 * ia;
          u0 = p0 - (2 * t == y ? 1.0 : 0.0);
          u1 = p1 - (2 * t + 1 == y ? 1.0 : 0.0);
          u8 = p8 - (y == 8 ? 1.0 : 0.0);
          const double lin = gsum<4>((c0v && 2 * t == y ? z0 : 0.0) +
                                     (c1v && 2 * t + 1 == y ? z1 : 0.0)) +
                             (K == 9 && y == 8 ? z8 : 0.0);
          if (rv && t == 0) loss_acc += (M + log(alpha)) - lin;
          // argmax over [p_0..p_{K-1}, e^-M/alpha]: first NaN / first max wins
          double bv = c0v ? p0 : -INFINITY;
          int bi = 2 * t;
          if (c1v) amax_take(bv, bi, p1, 2 * t + 1);
          gargmax<4>(bv, bi);
          if (K == 9) amax_take(bv, bi, p8, 8);
          amax_take(bv, bi, eM * ia, K);
          if (rv && t == 0 && bi == y) corr_acc += 1ull;
        }
      }
      if (!rv) u0 = u1 = u8 = 0.0;
      u[g * kUP + 2 * t] = u0;
      u[g * kUP + 2 * t + 1] = u1;
      if (t == 0) {
        u[g * kUP + 8] = u8;
        u[g * kUP + 9] = 0.0;
      }
      __syncwarp();
      if (!prep)
        xgroup<K, NMT, T>(tiles + (size_t)s * R * WS + (size_t)gr0 * WS, WS, u, ng, g, t, 0, 1,
                       nmt, acc, acc8);
      __syncwarp();
    }
    CL_TL(b, 3);
    if (lane == 0) mbar_arrive(&rg.empty[s]);
    if (++s == S) {
      s = 0;
      ph ^= 1u;
    }
  }
  // the CTA's partial: warps reduced in order through shared memory (the tiles)
  CL_TL(-1, 3);
  consumer_sync(kNC);
  if (!prep) {
    double *comb = static_cast<double *>(rg.tiles);  // [NW][64 columns][kUP] (over the tiles)
#pragma unroll
    for (int m = 0; m < NMT; ++m) {
      const double s8 = K == 9 ? gsum<4>(acc8[m]) : 0.0;
      double *cp = comb + ((size_t)warp * 64 + 8 * m + g) * kUP;
      cp[2 * t] = acc[m][0];
      cp[2 * t + 1] = acc[m][1];
      if (t == 0) cp[8] = s8;
    }
    consumer_sync(kNC);
    const int64_t d = (int64_t)K * a.p;
    for (int e = tid; e < K * 64; e += kNC) {
      const int c = e / 64, col = e - c * 64;
      double sm = 0.0;
#pragma unroll
      for (int w = 0; w < kNW; ++w) sm += comb[((size_t)w * 64 + col) * kUP + c];
      if (col < a.p) a.gp[(int64_t)cl * d + (int64_t)c * a.p + col] = sm;
    }
  }
  CL_TL(-1, 4);
  if (grad || apply) {  // apply: lossp[cl] = the CTA's sum of V.U (curvature)
    const double l = warp_allsum(loss_acc);
    unsigned long long cc = corr_acc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cc += __shfl_xor_sync(0xffffffffu, cc, o);
    if (lane == 0) {
      sh_loss[warp] = l;
      sh_corr[warp] = cc;
    }
    consumer_sync(kNC);
    if (tid == 0) {
      double lt = 0.0;
      unsigned long long ct = 0;
      for (int w = 0; w < kNW; ++w) {
        lt += sh_loss[w];
        ct += sh_corr[w];
      }
      a.lossp[cl] = lt;
      a.corrp[cl] = ct;
    }
  }
  CL_TL(-1, 5);
}

#ifdef SNX_CL_TIMELINE
__device__ unsigned long long g_cgr_tl[256][6];  // cg_step1_rows: entry, dependency met, exit, loads, alpha, stores
#define CGR_TL(ev)                                                   \
  do {                                                               \
    if (threadIdx.x == 0) {                                          \
      unsigned long long t_;                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));         \
      g_cgr_tl[blockIdx.x][(ev)] = t_;                               \
    }                                                                \
  } while (0)
#else
#define CGR_TL(ev) \
  do {             \
  } while (0)
#endif

// ---------------------------------------------------------------- finalize
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
  CGR_TL(0);
  pdl_trigger();  // the next row pass may start staging its X tiles (it waits for this grid)
  pdl_wait();
  CGR_TL(1);
  if (skip != nullptr && *skip != 0.0) return;
  __shared__ double sh[kFinThreads / 32];
  __shared__ double part[kFinThreads];
  const int t = threadIdx.x;
  // thread (f, e) as in cg_step1_rows_kernel: coalesced partial rows, the F sums
  // of an element added in f order by its lead thread
  const int e = t % (int)epb, f = t / (int)epb;
  const int64_t i = (int64_t)blockIdx.x * epb + e;
  const bool own = f < F && i < d;
  const int64_t il = (int64_t)blockIdx.x * epb + t;
  const bool lead = t < epb && il < d;
  const double b = lead ? base[il] : 0.0;
  {
    constexpr int kML = 16;
    double v[kML];
#pragma unroll
    for (int k = 0; k < kML; ++k) {
      const int c = f + k * F;
      v[k] = own && c < ncl ? __ldcg(gp + (int64_t)c * d + i) : 0.0;
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kML; ++k)
      if (f + k * F < ncl) s += v[k];
    if (own)
      for (int c = f + kML * F; c < ncl; c += F) s += __ldcg(gp + (int64_t)c * d + i);
    if (own) part[f * epb + e] = s;
  }
  __syncthreads();
  double bo = 0.0, bb = 0.0;
  if (lead) {
    double s = 0.0;
    for (int ff = 0; ff < F; ++ff) s += part[ff * epb + t];
    const double o = __dadd_rn(__dmul_rn(scale, s), __dmul_rn(lam, b));
    out[il] = o;
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
  CGR_TL(2);
}

// The CG iteration's first half (cg.py:77-86) fused with the product's
// finalize: the curvature s.Hs = scale * sum_rows V.U + lam * s.s comes from
// the kernel's per-cluster V.U sums (lossp) and the s.s partials cg_step2 /
// cg_init leave in the state's second scratch row, so alpha is known before
// any element of H s exists; then per element H s = scale * sum_cl gp + lam s
// (written, for the record), p += alpha s, r -= alpha H s and the r.r block
// partials cg_step2 reduces.  Same decisions as cg_step1_kernel (curvature test
// of cg.py:79); the curvature's rounding differs from the dot of s and H s.
__global__ void __launch_bounds__(kFinThreads)
    cg_step1_rows_kernel(int t, int T, const double *__restrict__ gp, int ncl, int64_t d,
                         int64_t epb, int F, double scale, double lam,
                         const double *__restrict__ vup, const double *__restrict__ s, double *r,
                         double *p, double *Hs, double *state) {
  CGR_TL(0);
  pdl_trigger();  // cg_step2, then the next row pass, may launch early (both wait)
  pdl_wait();
  CGR_TL(1);
  const double *st = slot(state, t);
  __shared__ double sh[kFinThreads / 32];
  __shared__ double s_alpha;
  __shared__ int s_bad;
  const int tid = threadIdx.x;
  // every load that does not need alpha goes out first: the partials of H s
  // and s, p, r overlap the curvature reduction below
  const double done = st[kDone];
  // thread (f, e): element e of the block, partials cl = f, f + F, ...; a warp
  // covers consecutive elements of one partial row (coalesced); the F sums of
  // an element meet in shared memory and its lead thread adds them in f order
  const int e = tid % (int)epb, f = tid / (int)epb;
  const int64_t i = (int64_t)blockIdx.x * epb + e;
  const bool own = f < F && i < d;
  const int64_t il = (int64_t)blockIdx.x * epb + tid;
  const bool lead = tid < epb && il < d;
  const double si = lead ? s[il] : 0.0, pi = lead ? p[il] : 0.0, ri0 = lead ? r[il] : 0.0;
  __shared__ double part[kFinThreads];
  constexpr int kML = 16;
  {
    double v[kML];
#pragma unroll
    for (int k = 0; k < kML; ++k) {
      const int c = f + k * F;
      v[k] = own && c < ncl ? __ldcg(gp + (int64_t)c * d + i) : 0.0;
    }
    double sum = 0.0;
#pragma unroll
    for (int k = 0; k < kML; ++k)
      if (f + k * F < ncl) sum += v[k];
    if (own)
      for (int c = f + kML * F; c < ncl; c += F) sum += __ldcg(gp + (int64_t)c * d + i);
    if (own) part[f * epb + e] = sum;
  }
  if (tid < 32) {
    double vv[8];  // the clusters' V.U sums: lane-strided, loads first
#pragma unroll
    for (int k = 0; k < 8; ++k) vv[k] = tid + 32 * k < ncl ? __ldcg(vup + tid + 32 * k) : 0.0;
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (tid + 32 * k < ncl) v += vv[k];
    for (int c = tid + 256; c < ncl; c += 32) v += __ldcg(vup + c);
    v = warp_allsum(v);
    const double ss = warp_sum_partials_cg(scratch(state, T) + kDotBlocks);
    if (tid == 0) {
      const double curv = __dadd_rn(__dmul_rn(scale, v), __dmul_rn(lam, ss));
      s_bad = curv <= 1e-32 * ss;  // cg.py:16, :79
      s_alpha = st[kRs] / curv;
      if (s_bad && blockIdx.x == 0 && done == 0.0) {
        slot(state, t + 1)[kErr] = 1.0;
        slot(state, t + 1)[kCurv] = curv;
      }
    }
  }
  CGR_TL(3);
  __syncthreads();
  CGR_TL(4);
  if (done != 0.0 || s_bad) return;
  const double alpha = s_alpha;
  double acc = 0.0;
  if (lead) {
    double sum = 0.0;
    for (int ff = 0; ff < F; ++ff) sum += part[ff * epb + tid];
    const double o = __dadd_rn(__dmul_rn(scale, sum), __dmul_rn(lam, si));
    Hs[il] = o;
    p[il] = np_axpy(pi, alpha, si);
    const double ri = np_axmy(ri0, alpha, o);
    r[il] = ri;
    acc = ri * ri;
  }
  CGR_TL(5);
  const double b = block_sum<kFinThreads>(acc, sh);
  if (tid == 0) scratch(state, T)[blockIdx.x] = b;
  CGR_TL(2);
}

// ---------------------------------------------------------------- host side
struct Plan {
  int ok;
  int split;  // 0: column split (clusters), 1: row split
  int cs, ncl, wc, S, WS, WQ, R;
  size_t smem;
  int o_tiles, o_q, o_side, o_u, o_vr, o_red, o_bar;
};

template <typename KernT>
static size_t smem_cap(KernT kern) {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) !=
          cudaSuccess ||
      optin <= 0)
    optin = 227 * 1024;
  cudaFuncAttributes fa{};
  cudaFuncGetAttributes(&fa, kern);
  cudaGetLastError();
  return (size_t)optin - fa.sharedSizeBytes;
}

template <int K, typename T>
static size_t cap_a() {
  static size_t c = 0;
  if (!c) c = smem_cap(cluster_rowpass_kernel<K, 2, T>);
  return c;
}
template <int K, typename T>
static size_t cap_r() {
  static size_t c = 0;
  if (!c) c = smem_cap(rowsplit_kernel<K, T>);
  return c;
}

template <int K, typename T>
static void layout(Plan &pl, int S) {
  size_t off = 0;
  auto take = [&](size_t bytes, size_t align) {
    off = (off + align - 1) / align * align;
    const size_t o = off;
    off += bytes;
    return (int)o;
  };
  pl.o_tiles = take((size_t)S * pl.R * pl.WS * sizeof(T), 1024);
  pl.o_q = take((size_t)pl.WQ * 8, 16);
  pl.o_side = take((size_t)S * pl.R * K * 8, 16);
  if (pl.split == 0) {
    pl.o_u = take((size_t)kNB3 * kRA * kUP * 8, 16);
    pl.o_vr = take((size_t)2 * pl.cs * kRA * K * 8, 16);
    pl.o_red = take((size_t)kNB3 * kNWA * kRA * K * 8, 16);
    pl.o_bar = take((size_t)(2 * S + 4 + 3 * kNB3) * 8, 8);
  } else {
    pl.o_u = take((size_t)kNW * 8 * kUP * 8, 16);
    pl.o_vr = pl.o_red = 0;
    pl.o_bar = take((size_t)(2 * S) * 8, 8);
    // the final warp reduction reuses the tiles: [NW][64][kUP] doubles
    if ((size_t)S * pl.R * pl.WS * sizeof(T) < (size_t)kNW * 64 * kUP * 8) off = (size_t)1 << 30;
  }
  pl.smem = off;
  pl.S = S;
}

template <int K, typename T>
static int max_clusters(int cs, size_t smem) {
  static int cache[4] = {-1, -1, -1, -1};
  static size_t cache_smem[4] = {0, 0, 0, 0};
  const int ci = cs == 1 ? 0 : cs == 2 ? 1 : cs == 4 ? 2 : 3;
  if (cache[ci] >= 0 && cache_smem[ci] == smem) return cache[ci];
  auto kern = cluster_rowpass_kernel<K, 2, T>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap_a<K, T>());
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs * 64);
  cfg.blockDim = dim3(kNTA);
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
  cache[ci] = n;
  cache_smem[ci] = smem;
  return n;
}

template <int K, typename T>
static Plan make_plan(int P, int64_t nrows) {
  Plan pl{};
  if (P <= 64) {  // row split: the whole row in one CTA
    pl.split = 1;
    pl.cs = 1;
    pl.R = kRR;
    pl.wc = P;
    // = 2 (mod 16) doubles: fragment loads spread over banks; f32 rows: = 4
    // (mod 16) floats (16-B aligned for the copies)
    pl.WS = pl.WQ = (P + 15) / 16 * 16 + (sizeof(T) == 8 ? 2 : 4);
    int S = 4;
    for (; S >= 2; --S) {
      layout<K, T>(pl, S);
      if (pl.smem <= cap_r<K, T>()) break;
    }
    if (pl.smem > cap_r<K, T>()) return Plan{};
    const int64_t want = nrows > 0 ? (nrows + kRR - 1) / kRR : 1;
    pl.ncl = (int)(want < sm_count() ? want : sm_count());
    pl.ok = 1;
    return pl;
  }
  for (int cs : {1, 2, 4, 8}) {
    // slice width: even (fp64: 16-B aligned slices), a multiple of 4 for f32
    const int wc = sizeof(T) == 8 ? ((P + cs - 1) / cs + 1) & ~1 : ((P + cs - 1) / cs + 3) & ~3;
    if ((wc + 7) / 8 > kNWA * kNMTA) continue;  // > 768 columns per CTA
    pl = Plan{};
    pl.split = 0;
    pl.cs = cs;
    pl.R = kRA;
    pl.wc = wc;
    pl.WS = pl.WQ = (wc + 15) / 16 * 16 + (sizeof(T) == 8 ? 2 : 4);
    layout<K, T>(pl, kSA);
    if (pl.smem > cap_a<K, T>()) continue;
    const int maxcl = max_clusters<K, T>(cs, pl.smem);
    const int64_t want = nrows > 0 ? (nrows + kRA - 1) / kRA : 1;
    pl.ncl = (int)(want < maxcl ? want : maxcl);
    if (pl.ncl < 1) pl.ncl = 1;
    pl.ok = 1;
    return pl;
  }
  return Plan{};
}

static bool disabled() {
  static const int off = getenv("SNX_TWO_PASS") != nullptr ? 1 : 0;  // A/B: snx_rowpass.cu
  return off != 0;
}

// fp64 data, or f32 data widened to fp64 in shared memory (the arithmetic is
// the fp64 path's either way)
static Plan plan_for(int dtype, int p, int K, int64_t nrows) {
  if ((dtype != SNX_F64 && dtype != SNX_F32) || K < 1 || K > kMaxK || disabled()) return Plan{};
  const int P = padded(p);
  const bool f32 = dtype == SNX_F32;
  switch (K) {
#define SNX_CL_K(KK) \
  case KK:           \
    return f32 ? make_plan<KK, float>(P, nrows) : make_plan<KK, double>(P, nrows);
    SNX_CL_K(1) SNX_CL_K(2) SNX_CL_K(3) SNX_CL_K(4) SNX_CL_K(5) SNX_CL_K(6) SNX_CL_K(7)
    SNX_CL_K(8) SNX_CL_K(9)
#undef SNX_CL_K
    default:
      return Plan{};
  }
}

static void fill(Args &a, const Plan &pl) {
  a.cs = pl.cs;
  a.ncl = pl.ncl;
  a.wc = pl.wc;
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
}

template <int K, typename T>
static int launch_k(const Plan &pl, Args &a, cudaStream_t st) {
  fill(a, pl);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pl.split == 0) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = pl.cs;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  if (a.early) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.gridDim = dim3(pl.ncl * pl.cs);
  cfg.dynamicSmemBytes = pl.smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = na;
  if (pl.split == 0) {
    static bool attr = false;
    auto k1 = cluster_rowpass_kernel<K, 1, T>;
    auto k2 = cluster_rowpass_kernel<K, 2, T>;
    if (!attr) {
      if (cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)cap_a<K, T>()) != cudaSuccess ||
          cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)cap_a<K, T>()) != cudaSuccess)
        return check_launch("cluster_rowpass attributes");
      attr = true;
    }
    const bool two = a.mode != kApply;  // exp / log row algebra: two row warps
    carveout(two ? k2 : k1);
    cfg.blockDim = dim3(two ? nta<2>() : nta<1>());
    cudaLaunchKernelEx(&cfg, two ? k2 : k1, a);
    return check_launch("cluster_rowpass");
  }
  static bool attr = false;
  auto kern = rowsplit_kernel<K, T>;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)cap_r<K, T>()) != cudaSuccess)
      return check_launch("rowsplit attributes");
    attr = true;
  }
  carveout(kern);
  cfg.blockDim = dim3(kNTR);
  cudaLaunchKernelEx(&cfg, kern, a);
  return check_launch("rowsplit_rowpass");
}

static int launch_any(const Plan &pl, int K, int dtype, Args &a, cudaStream_t st) {
  const bool f32 = dtype == SNX_F32;
  switch (K) {
#define SNX_CL_K(KK) \
  case KK:           \
    return f32 ? launch_k<KK, float>(pl, a, st) : launch_k<KK, double>(pl, a, st);
    SNX_CL_K(1) SNX_CL_K(2) SNX_CL_K(3) SNX_CL_K(4) SNX_CL_K(5) SNX_CL_K(6) SNX_CL_K(7)
    SNX_CL_K(8) SNX_CL_K(9)
#undef SNX_CL_K
    default:
      set_error("snx: one-pass row pass: K = %d unsupported", K);
      return 1;
  }
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

// The full-data objective + gradient pass runs on the one-pass kernel (X read
// once): the row split at p <= 64, the column split with two row-algebra warps
// otherwise (CIFAR 365 vs 415 us for the two GEMMs of snx_rowpass.cu, which read
// X twice; with one row-algebra warp the exp / log per row bounded it at 522 us).
// SNX_TWO_PASS_GRAD=1 selects the two GEMMs, for A/B runs.
bool cluster_grad_preferred(int dtype, int32_t p, int32_t K) {
  static const bool off = getenv("SNX_TWO_PASS_GRAD") != nullptr;  // A/B: snx_rowpass.cu
  const clp::Plan pl = clp::plan_for(dtype, p, K, 1);
  return pl.ok && !off;
}

size_t cluster_ws_bytes(int dtype, int64_t nrows, int32_t p, int32_t K) {
  const clp::Plan pl = clp::plan_for(dtype, p, K, nrows);
  if (!pl.ok) return 0;
  char dummy;
  return clp::ws_layout(&dummy, pl, p, K).total;
}

// mode: 0 prep (hout), 1 apply (h, skip, dots -> out), 2 grad (labels, loss/corr -> out)
int cluster_rowpass(int mode, int dtype, const void *X, int64_t ldx, const int64_t *rows,
                    int64_t nrows,
                    int32_t p, int32_t K, const int32_t *labels, const double *w,
                    const double *h, double *hout, double scale, double lam,
                    const double *base, double *out, double *loss_out, long long *corr_out,
                    double *dots, const double *skip, int early, void *ws, size_t ws_bytes,
                    cudaStream_t st) {
  using namespace clp;
  const Plan pl = plan_for(dtype, p, K, nrows);
  if (!pl.ok) {
    set_error("snx: no one-pass row-pass plan for p=%d K=%d", p, K);
    return 1;
  }
  const ClWs cw = ws_layout(ws, pl, p, K);
  if (ws == nullptr || ws_bytes < cw.total) {
    set_error("snx: workspace too small for the one-pass row pass (%zu < %zu)", ws_bytes,
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
  if (launch_any(pl, K, dtype, a, st)) return 1;
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
  return check_launch("one-pass finalize");
}

// One CG iteration t on the sampled Hessian (cg.py:77-96): the one-pass product
// of s (skipped once the solve is done) without a finalize pass, the fused
// cg_step1 above, then cg_step2.
int cluster_cg_iteration(int dtype, const void *X, int64_t ldx, const int64_t *rows,
                         int64_t nrows,
                         int32_t p, int32_t K, const double *h, double scale, double lam, int t,
                         int T, double *r, double *s, double *pv, double *pb, double *Hs,
                         double *state, int early, void *ws, size_t ws_bytes, cudaStream_t st) {
  using namespace clp;
  const Plan pl = plan_for(dtype, p, K, nrows);
  if (!pl.ok || nrows < 1) {
    set_error("snx: no one-pass plan for the fused CG iteration (p=%d K=%d rows=%lld)", p, K,
              (long long)nrows);
    return 1;
  }
  const ClWs cw = ws_layout(ws, pl, p, K);
  if (ws == nullptr || ws_bytes < cw.total) {
    set_error("snx: workspace too small for the one-pass row pass (%zu < %zu)", ws_bytes,
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
  a.mode = kApply;
  a.w = s;
  a.h = h;
  a.gp = cw.gp;
  a.lossp = cw.lossp;
  a.corrp = cw.corrp;
  a.skip = state + (size_t)t * SNX_CG_SLOT + kDone;
  a.early = early;
  if (launch_any(pl, K, dtype, a, st)) return 1;
  const int64_t d = (int64_t)K * p;
  const int64_t epb = (d + kDotBlocks - 1) / kDotBlocks;
  int F = 1;
  while (F < 32 && (int64_t)(2 * F) * epb <= kFinThreads) F *= 2;
  launch_pdl_if(true, cg_step1_rows_kernel, dim3(kDotBlocks), dim3(kFinThreads), 0, st, t, T,
                cw.gp, pl.ncl, d, epb, F, scale, lam, (const double *)cw.lossp,
                (const double *)s, r, pv, Hs, state);
  if (check_launch("cg_step1_rows")) return 1;
  return launch_cg_step2(t, T, d, r, s, pv, pb, state, st);
}


}  // namespace snx

#ifdef SNX_CL_TIMELINE
extern "C" int snx_debug_cgr_timeline(unsigned long long *host_out) {
  return cudaMemcpyFromSymbol(host_out, snx::clp::g_cgr_tl, sizeof(snx::clp::g_cgr_tl)) ==
                 cudaSuccess
             ? 0
             : 1;
}
extern "C" int snx_debug_cl_timeline(unsigned long long *host_out) {
  return cudaMemcpyFromSymbol(host_out, snx::clp::g_cl_tl, sizeof(snx::clp::g_cl_tl)) ==
                 cudaSuccess
             ? 0
             : 1;
}
#endif
