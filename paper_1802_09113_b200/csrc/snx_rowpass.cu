// Row-pass kernels: the two feature products of every softmax quantity.
//
//   GEMM1 + row epilogue (gemm1_kernel): z_r = X[r] . W (K logits per row,
//     softmax.py:91 / :206) followed by the per-row softmax algebra of
//     softmax.py:85-99 (objective, accuracy), :157-161 (gradient residual),
//     :189-195 (Hessian probabilities) or :206-208 (ComputeU).
//   GEMM2 (gemm2_kernel): out = scale * X^T U + lam * base
//     (softmax.py:162 / :209-210), plus the CG dot partials of out.
//
// Both kernels are persistent and warp-specialised (sm_100a):
//   * one producer warp streams tiles into a ring of shared-memory stages with
//     2-D tensor-map TMA (cp.async.bulk.tensor, 8-32 KB boxes; out-of-range
//     rows/columns arrive zero-filled) completing on mbarriers; eight consumer
//     warps do the fp64/fp32 FMAs from shared memory.  Rows are contiguous: a
//     sample S_H is materialised once per outer iteration (snx_gather_rows /
//     snx_hess_prepare), then every Hessian product streams it as tiles;
//   * work units are handed out dynamically (one atomic ticket per unit) so
//     all SMs stay busy to the end;
//   * GEMM1 unit = (64-row block, feature slice).  X boxes are 64 rows x 128 B
//     with the 128-B swizzle, so lanes can own rows (2 each) without bank
//     conflicts while the weights are smem broadcasts; warps own 64-B column
//     strips.  The 8 warp partials are reduced in smem, the slice partial goes
//     to L2, and the last slice to arrive for a row block (arrival counter)
//     sums the slices in fixed order and runs the epilogue;
//   * GEMM2 unit = (feature tile, row split).  Lanes own 2 x 16 B of
//     consecutive columns, U rows are smem broadcasts, warps split rows; the
//     last row split to arrive for a tile sums the split partials in fixed
//     order and writes scale*X^T U + lam*base and the tile's dot partials.
// Every reduction has a fixed order and there are no float atomics: results
// are bit-identical run to run.
#include <stdarg.h>
#include <stdio.h>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "snx_common.cuh"
#include "snx_internal.h"
#include "snx_pipe.cuh"

namespace snx {

enum Mode { kObjective = 0, kGradient = 1, kHessPrep = 2, kHessApply = 3, kProbs = 4 };

constexpr int kWarps = 8;                    // consumer warps
constexpr int kConsumers = kWarps * 32;      // consumer threads
constexpr int kThreads = kConsumers + 32;    // + one producer warp
constexpr int kRB = 96;                      // rows per GEMM1 item (3 per lane)
constexpr int kG2Rows = 32;                  // rows per GEMM2 item
constexpr int kMaxTiles = kDotBlocks;
constexpr size_t kSmemBudget = 220 * 1024;
constexpr int64_t kMaxRowBlocks = 1 << 17;   // 12.5M rows per call
constexpr int kCounterWords = 16 + kMaxTiles + kMaxRowBlocks;

__host__ __device__ constexpr size_t cround(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Optional per-CTA timeline (compile with -DSNX_TIMELINE; tools/timeline.py):
// globaltimer stamps at kernel entry, first data ready, last item done, exit.
#ifdef SNX_TIMELINE
__device__ unsigned long long g_timeline[3][160][8];
#define SNX_TL(slot, ev)                                                   \
  do {                                                                     \
    unsigned long long t_;                                                 \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
    if (blockIdx.x < 160) g_timeline[slot][blockIdx.x][ev] = t_;          \
  } while (0)
#else
#define SNX_TL(slot, ev) \
  do {                   \
  } while (0)
#endif

// GEMM1 shape: an item is (96-row block) x (512 B of columns).  X arrives as
// four 96-row x 128-B boxes with the 128-B swizzle; warp w owns the 64-B strip
// (w & 1) of box (w >> 1); lanes own rows lane, lane+32, lane+64 (they share
// the swizzle phase lane & 7), so the weights are smem broadcasts.
template <typename T, int K> struct G1Shape {
  static constexpr int V = 16 / (int)sizeof(T);
  static constexpr int BOXC = 128 / (int)sizeof(T);
  static constexpr int WC = 64 / (int)sizeof(T);
  static constexpr int CHUNK = kWarps * WC;
  static constexpr int NB = CHUNK / BOXC;
  static constexpr size_t BOX = (size_t)kRB * 128;
  static constexpr size_t WBYTES = (size_t)K * CHUNK * sizeof(T);
  static constexpr size_t STAGE = cround(NB * BOX + WBYTES, 1024);
  static constexpr size_t RED = (size_t)(kWarps / 2) * kRB * K * 8;
  static constexpr int S = (3 * STAGE + RED + 256 <= kSmemBudget) ? 3 : 2;
  static constexpr size_t SMEM = S * STAGE + RED + 2 * S * 8 + 64;
};

// GEMM2 shape: an item is (1-KB column tile) x (32 rows); lanes own 2 x 16 B (one per tile half) of
// consecutive columns; U rows are padded to a 16-B multiple (KP) so each row
// is a few 128-bit smem broadcasts.
template <typename T, int K> struct G2Shape {
  static constexpr int V = 16 / (int)sizeof(T);
  static constexpr int LC = 2 * V;
  static constexpr int TCOL = 32 * LC;
  static constexpr int KP = (int)(cround(K * sizeof(T), 16) / sizeof(T));
  static constexpr size_t XB = (size_t)kG2Rows * TCOL * sizeof(T);
  static constexpr size_t UB = (size_t)kG2Rows * KP * sizeof(T);
  static constexpr size_t STAGE = cround(XB + UB, 128);
  static constexpr size_t RED = (size_t)(kWarps / 2) * K * TCOL * 8;
  static constexpr int S = (4 * STAGE + RED + 256 <= kSmemBudget)   ? 4
                           : (3 * STAGE + RED + 256 <= kSmemBudget) ? 3
                                                                    : 2;
  static constexpr size_t SMEM = S * STAGE + RED + 2 * S * 8 + 64;
};

inline int u_stride(int dtype, int K) {  // padded U row stride (elements)
  const int tb = dtype == SNX_F64 ? 8 : 4;
  return (int)(cround((size_t)K * tb, 16) / tb);
}

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ void lds(const double *p, double (&o)[2]) {
  const double2 v = *reinterpret_cast<const double2 *>(p);
  o[0] = v.x;
  o[1] = v.y;
}
__device__ __forceinline__ void lds(const float *p, float (&o)[4]) {
  const float4 v = *reinterpret_cast<const float4 *>(p);
  o[0] = v.x;
  o[1] = v.y;
  o[2] = v.z;
  o[3] = v.w;
}

// fixed-order u64 sum over the block; valid in thread 0
template <int NT>
__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v,
                                                            unsigned long long *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  unsigned long long t = 0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) t += sh[i];
  }
  __syncthreads();
  return t;
}

// fixed-order sums over the 256 consumer threads (named barrier 1; the
// producer warp never joins); valid in consumer thread 0
__device__ __forceinline__ double consumer_sum(double v, double *sh) {
  v = warp_allsum(v);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  consumer_sync(kConsumers);
  double t = 0.0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < kWarps; ++i) t += sh[i];
  }
  consumer_sync(kConsumers);
  return t;
}

__device__ __forceinline__ unsigned long long consumer_sum_u64(unsigned long long v,
                                                               unsigned long long *sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  consumer_sync(kConsumers);
  unsigned long long t = 0;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < kWarps; ++i) t += sh[i];
  }
  consumer_sync(kConsumers);
  return t;
}


// ---------------------------------------------------------------- GEMM1
struct G1Args {
  CUtensorMap xmap;  // X: [nrows][P] boxes of 96 rows x 128 B, 128-B swizzle
  CUtensorMap wmap;  // W: [K][P] boxes of K rows x CHUNK columns
  int64_t nrows;
  int nchunks;     // CHUNK-column chunks per row (ceil(P / CHUNK))
  int maxseg;      // max CTA segments per row block
  int64_t items;   // row_blocks * nchunks, split evenly over the CTAs
  int64_t row_blocks;
  int mode;        // Mode: which row epilogue the last segment of a row block runs
  int ustride;     // row stride of rowout (K for h, padded KP for R / U)
  double *zp;      // [row_blocks][maxseg][kRB][K] segment partial logits
  unsigned *rb_count;  // [row_blocks] segment arrivals (zero at rest)
  unsigned *done_rb;   // finished row blocks (zero at rest)
  const int32_t *labels;
  const void *H;       // kHessApply: nrows*K probabilities
  void *rowout;        // R (gradient), h (prep), U (apply)
  double *loss_part;   // [row_blocks]
  unsigned long long *corr_part;
  double *loss_out;
  long long *corr_out;
  const double *skip;
  int32_t *pred_out;   // kProbs: most probable class per row (nullable)
  double *stats_out;   // kProbs: [M, sum E, linear] per row (nullable)
  int early_x;         // launched as a programmatic dependent: stage the first X
                       // tiles before waiting for the previous kernel (X_S is
                       // older than it; the weights and the skip flag are not)
};

// Per-row softmax algebra on the summed logits z (softmax.py:85-99 and the
// mode-specific lines); returns the row loss / correct flag.  hw: the row's
// probabilities (kHessApply), y: its label (objective / gradient), both
// loaded by the caller ahead of the segment sums.
template <typename T, int K>
__device__ __forceinline__ void row_epilogue(const G1Args &a, int64_t r, const double (&z)[K],
                                             const double (&hw)[K], int y, double &loss,
                                             unsigned long long &corr) {
  if (a.mode == kHessApply) {
    // softmax.py:206-208: VW = V*W; U = VW - W*rowsum(VW)
    double vw[K], s = 0.0;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      vw[c] = z[c] * hw[c];
      s += vw[c];
    }
    T *u = static_cast<T *>(a.rowout) + r * a.ustride;
#pragma unroll
    for (int c = 0; c < K; ++c) u[c] = (T)(vw[c] - hw[c] * s);
    return;
  }
  // softmax.py:91-98: M = max(0, max_c z); E = exp(z - M); alpha = e^-M + sum E
  double M = 0.0;
#pragma unroll
  for (int c = 0; c < K; ++c) M = (z[c] > M || isnan(z[c])) ? z[c] : M;  // NaN propagates
  double E[K], se = 0.0;
#pragma unroll
  for (int c = 0; c < K; ++c) {
    E[c] = exp(z[c] - M);
    se += E[c];
  }
  const double alpha = exp(-M) + se;
  if (a.mode == kHessPrep) {
    T *h = static_cast<T *>(a.rowout) + r * a.ustride;
#pragma unroll
    for (int c = 0; c < K; ++c) h[c] = (T)(E[c] / alpha);
    return;
  }
  if (a.mode == kProbs) {
    // softmax.py:224-235 class_probabilities (reference class last), :238-240
    // predict (first max wins), :107-122 row_stats (max, sum of E, linear part)
    if (a.rowout != nullptr) {
      double *pr = static_cast<double *>(a.rowout) + r * (K + 1);
#pragma unroll
      for (int c = 0; c < K; ++c) pr[c] = E[c] / alpha;
      pr[K] = exp(-M) / alpha;
    }
    if (a.stats_out != nullptr) {
      double lin = 0.0;
#pragma unroll
      for (int c = 0; c < K; ++c)
        if (c == y) lin = z[c];
      a.stats_out[r * 3 + 0] = M;
      a.stats_out[r * 3 + 1] = se;
      a.stats_out[r * 3 + 2] = lin;
    }
    if (a.pred_out != nullptr) {
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
      a.pred_out[r] = best;
    }
    return;
  }
  double lin = 0.0;
#pragma unroll
  for (int c = 0; c < K; ++c)
    if (c == y) lin = z[c];
  loss = (M + log(alpha)) - lin;  // softmax.py:134
  if (a.mode == kGradient) {
    T *R = static_cast<T *>(a.rowout) + r * a.ustride;
#pragma unroll
    for (int c = 0; c < K; ++c) R[c] = (T)(E[c] / alpha - (c == y ? 1.0 : 0.0));
  }
  if (a.corr_out != nullptr) {
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

// Fixed-order sum over segments of kPer strided elements per thread: loads of
// up to kBatch segments are issued together (one L2 round trip per batch),
// then added in segment order -- the same rounding as a sequential sum.
template <int kPer, int kBatch>
__device__ __forceinline__ void segment_sums(const double *base, int64_t seg_stride, int nseg,
                                             int tid, int stride, int nvalid,
                                             double (&acc)[kPer]) {
#pragma unroll
  for (int q = 0; q < kPer; ++q) acc[q] = 0.0;
  for (int s0 = 0; s0 < nseg; s0 += kBatch) {
    double v[kBatch][kPer];
#pragma unroll
    for (int b = 0; b < kBatch; ++b)
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int e = tid + q * stride;
        v[b][q] = (s0 + b < nseg && e < nvalid) ? __ldcg(base + (int64_t)(s0 + b) * seg_stride + e)
                                                : 0.0;
      }
#pragma unroll
    for (int b = 0; b < kBatch; ++b)
#pragma unroll
      for (int q = 0; q < kPer; ++q)
        if (s0 + b < nseg) acc[q] += v[b][q];
  }
}

// Epilogue of row block rb by the CTA that delivered its last segment: the
// consumer threads sum the CTA segments (fixed order), then one thread per
// row runs the row algebra; loss / correct counts reduce per row block and,
// by the CTA that finishes the last row block, over all row blocks (fixed order).
template <typename T, int K>
__device__ __forceinline__ void block_epilogue(const G1Args &a, int64_t rb, int G, double *zsum,
                                            double *shd, unsigned long long *shu, int *flag,
                                            unsigned epoch) {
  const int tid = threadIdx.x;
  const int nrows = (int)min((int64_t)kRB, a.nrows - rb * kRB);
  const int64_t r = rb * kRB + tid;
  // row inputs first: their latency overlaps the segment loads
  double hw[K];
  int y = -1;
  if (tid < nrows) {
    if (a.mode == kHessApply) {
      const T *h = static_cast<const T *>(a.H) + r * K;
#pragma unroll
      for (int c = 0; c < K; ++c) hw[c] = (double)h[c];
    } else if (a.mode != kHessPrep && a.labels != nullptr) {
      y = a.labels[r];
    }
  }
  // 1) segment sums: element e = row*K + c
  {
    const int c_lo = sk_owner(a.items, G, rb * a.nchunks);
    const int nseg = sk_owner(a.items, G, (rb + 1) * a.nchunks - 1) - c_lo + 1;
    const double *zb = a.zp + rb * a.maxseg * (int64_t)kRB * K;
    constexpr int kPer = (kRB * K + kConsumers - 1) / kConsumers;
    double acc[kPer];
    segment_sums<kPer, (kPer <= 4 ? 8 : 4)>(zb, (int64_t)kRB * K, nseg, tid, kConsumers,
                                            nrows * K, acc);
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int e = tid + q * kConsumers;
      if (e < kRB * K) zsum[e] = acc[q];
    }
  }
  consumer_sync(kConsumers);
  // 2) row algebra, one thread per row
  double loss = 0.0;
  unsigned long long corr = 0;
  if (tid < nrows) {
    double z[K];
#pragma unroll
    for (int c = 0; c < K; ++c) z[c] = zsum[tid * K + c];
    row_epilogue<T, K>(a, r, z, hw, y, loss, corr);
  }
  if (tid == 0) a.rb_count[rb] = 0u;  // rest state for the next launch
  if (a.mode != kObjective && a.mode != kGradient) return;
  const double bl = consumer_sum(loss, shd);
  const unsigned long long bc = consumer_sum_u64(corr, shu);
  if (tid == 0) {
    a.loss_part[rb] = bl;
    a.corr_part[rb] = bc;
    *flag = atomic_add_acq_rel(a.done_rb, 1u) == (unsigned)(a.row_blocks - 1);
  }
  consumer_sync(kConsumers);
  if (!*flag) return;
  double t = 0.0;
  unsigned long long tc = 0;
  for (int64_t i = tid; i < a.row_blocks; i += kConsumers) {
    t += __ldcg(a.loss_part + i);
    tc += __ldcg(a.corr_part + i);
  }
  const double tot = consumer_sum(t, shd);
  const unsigned long long ct = consumer_sum_u64(tc, shu);
  if (tid == 0) {
    a.loss_out[0] = tot;
    if (a.corr_out) a.corr_out[0] = (long long)ct;
    *a.done_rb = 0u;
  }
}

// GEMM1 work of one CTA (items of the stream-K split over G CTAs), shared by
// gemm1_kernel and the persistent CG kernel.  itp / itc: the producer's and
// the consumers' running stage counters of the (full, empty) ring, kept
// across calls by the persistent kernel.
template <typename T, int K, int S>
__device__ __forceinline__ void gemm1_body(const G1Args &a, unsigned char *smem, double *red,
                                           uint64_t *full, uint64_t *empty, int G, int64_t &itp,
                                           int64_t &itc, unsigned epoch) {
  using Sh = G1Shape<T, K>;
  constexpr int V = Sh::V;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x;
  if (cta >= G) return;
  const int64_t i0 = sk_begin(a.items, G, cta), i1 = sk_begin(a.items, G, cta + 1);
  if (i0 == i1) return;  // more CTAs than items (the host never launches that)
  const int64_t rb0 = i0 / a.nchunks;
  __shared__ double shd[2 * kWarps];
  __shared__ unsigned long long shu[kWarps];
  __shared__ int flag;
  __shared__ long long epi_rb;
  const int ch0 = (int)(i0 - rb0 * a.nchunks);

  if (warp == kWarps) {
    // ------------------------------------------------ producer warp (TMA)
    if (lane == 0) {
      tma_prefetch_desc(&a.xmap);
      tma_prefetch_desc(&a.wmap);
      constexpr unsigned kTx = (unsigned)(Sh::NB * Sh::BOX + Sh::WBYTES);
      // early_x: the X boxes of the first S items go out before the wait for
      // the previous kernel (fresh ring: the empty waits pass at once)
      const int64_t npre = a.early_x ? min((int64_t)S, i1 - i0) : 0;
      {
        int64_t rb = rb0;
        int ch = ch0;
        for (int64_t j = 0; j < npre; ++j) {
          const int s = (int)((itp + j) % S);
          mbar_arrive_expect_tx(&full[s], kTx);
          unsigned char *st = smem + s * Sh::STAGE;
          const int col = ch * Sh::CHUNK, row = (int)(rb * kRB);
#pragma unroll
          for (int b = 0; b < Sh::NB; ++b)
            tma_load_2d(st + b * Sh::BOX, &a.xmap, col + b * Sh::BOXC, row, &full[s]);
          if (++ch == a.nchunks) {
            ch = 0;
            ++rb;
          }
        }
      }
      bool skipped = false;
      if (a.early_x) {
        pdl_wait();
        skipped = a.skip != nullptr && *a.skip != 0.0;
      }
      int64_t rb = rb0;
      int ch = ch0;
      for (int64_t i = i0; i < i1; ++i, ++itp) {
        const int s = (int)(itp % S);
        const bool pre = i - i0 < npre;
        if (skipped && !pre) break;
        if (!pre) {
          mbar_wait(&empty[s], (unsigned)((itp / S) & 1) ^ 1u);
          mbar_arrive_expect_tx(&full[s], kTx);
        }
        unsigned char *st = smem + s * Sh::STAGE;
        const int col = ch * Sh::CHUNK, row = (int)(rb * kRB);
        if (!pre) {
#pragma unroll
          for (int b = 0; b < Sh::NB; ++b)
            tma_load_2d(st + b * Sh::BOX, &a.xmap, col + b * Sh::BOXC, row, &full[s]);
        }
        tma_load_2d(st + Sh::NB * Sh::BOX, &a.wmap, col, 0, &full[s]);
        if (++ch == a.nchunks) {
          ch = 0;
          ++rb;
        }
      }
      if (skipped)  // no consumer will read them: let the staged copies land before exit
        for (int64_t j = 0; j < npre; ++j) mbar_wait(&full[(int)(j % S)], 0u);
    }
    return;
  }

  // -------------------------------------------------- consumer warps
  if (a.early_x) {  // everything below may depend on the previous kernel
    pdl_wait();
    if (a.skip != nullptr && *a.skip != 0.0) return;
  }
  const int box = warp >> 1;
  const int c0 = (warp & 1) * 4;  // first 16-B chunk of this warp's strip
  const int sw = lane & 7;        // swizzle phase of rows lane, lane+32, lane+64
  T acc0[K], acc1[K], acc2[K];
#pragma unroll
  for (int c = 0; c < K; ++c) acc0[c] = acc1[c] = acc2[c] = T(0);
  // deferred last-arriver check (thread 0): the segment counter of the row
  // block flushed last time, read one flush later so its latency is hidden
  long long pend_rb = -1;
  unsigned pend_prev = 0;
  int64_t rb = rb0;
  int ch = ch0;
  for (int64_t i = i0; i <= i1; ++i) {
    if (i == i1 || (ch == 0 && i > i0)) {
      if (i == i1 && tid == 0) SNX_TL(0, 2);
      // flush the segment partial of the row block just finished: warp pairs
      // (w, w+4) in smem, then the 4 pair sums in order
      const int64_t frb = (i == i1 && ch != 0) ? rb : rb - 1;
      double *mine = red + (size_t)(warp & 3) * kRB * K;
      if (warp >= 4) {
#pragma unroll
        for (int c = 0; c < K; ++c) {
          mine[lane * K + c] = (double)acc0[c];
          mine[(lane + 32) * K + c] = (double)acc1[c];
          mine[(lane + 64) * K + c] = (double)acc2[c];
        }
      }
      consumer_sync(kConsumers);
      if (warp < 4) {
#pragma unroll
        for (int c = 0; c < K; ++c) {
          mine[lane * K + c] = (double)acc0[c] + mine[lane * K + c];
          mine[(lane + 32) * K + c] = (double)acc1[c] + mine[(lane + 32) * K + c];
          mine[(lane + 64) * K + c] = (double)acc2[c] + mine[(lane + 64) * K + c];
        }
      }
#pragma unroll
      for (int c = 0; c < K; ++c) acc0[c] = acc1[c] = acc2[c] = T(0);
      consumer_sync(kConsumers);
      const int c_lo = sk_owner(a.items, G, frb * a.nchunks);
      double *zb = a.zp + (frb * a.maxseg + (cta - c_lo)) * (int64_t)kRB * K;
      const int valid = (int)min((int64_t)kRB, a.nrows - frb * kRB) * K;
      for (int t = tid; t < valid; t += kConsumers) {
        const double z = ((red[t] + red[kRB * K + t]) + red[2 * kRB * K + t]) +
                         red[3 * kRB * K + t];
        zb[t] = z;
      }
      consumer_sync(kConsumers);  // segment written; red free again
      if (i == i1 && tid == 0) SNX_TL(0, 4);
      // resolve the previous arrival, publish this one (release), and on the
      // final flush also resolve this one
      if (tid == 0) {
        epi_rb = -1;
        if (pend_rb >= 0) {
          const int n_prev = sk_owner(a.items, G, (pend_rb + 1) * a.nchunks - 1) -
                             sk_owner(a.items, G, pend_rb * a.nchunks) + 1;
          if (pend_prev == (unsigned)(n_prev - 1)) epi_rb = pend_rb;
        }
        pend_rb = frb;
        pend_prev = atomic_add_acq_rel(&a.rb_count[frb], 1u);  // release our segment
      }
      consumer_sync(kConsumers);
      if (i == i1 && tid == 0) SNX_TL(0, 5);
      for (int pass = 0; pass < 2; ++pass) {
        if (epi_rb >= 0) {  // the acq_rel arrival already acquired the other segments
          block_epilogue<T, K>(a, epi_rb, G, red, shd, shu, &flag, epoch);
          consumer_sync(kConsumers);
          if (i == i1 && tid == 0) SNX_TL(0, 6 + pass);
        }
        if (i != i1 || pass == 1) break;
        // final flush: wait for this CTA's own arrival and resolve it too
        if (tid == 0) {
          const int n_cur = sk_owner(a.items, G, (frb + 1) * a.nchunks - 1) - c_lo + 1;
          epi_rb = (pend_prev == (unsigned)(n_cur - 1)) ? frb : -1;
        }
        consumer_sync(kConsumers);
      }
    }
    if (i == i1) {
      if (tid == 0) SNX_TL(0, 3);
      break;
    }
    const int s = (int)(itc % S);
    mbar_wait(&full[s], (unsigned)((itc / S) & 1));
    if (tid == 0 && i == i0) SNX_TL(0, 1);
    const unsigned char *st = smem + s * Sh::STAGE;
    const unsigned char *xa = st + box * Sh::BOX + lane * 128;
    const T *wp = reinterpret_cast<const T *>(st + Sh::NB * Sh::BOX) + warp * Sh::WC;
#ifndef SNX_DIAG_NOMATH  // diagnostic build: data movement only
    // software-pipelined over the 4 16-B column chunks of this warp's strip:
    // the operands of chunk q+1 load while chunk q's 6K FMAs issue (two warps
    // per SM sub-partition cannot hide the shared-memory latency otherwise)
    T xv[2][3][V], wv[2][K][V];
    auto load_q = [&](int q, T (&x)[3][V], T (&w)[K][V]) {
      const int off = ((c0 + q) ^ sw) * 16;
      lds(reinterpret_cast<const T *>(xa + off), x[0]);
      lds(reinterpret_cast<const T *>(xa + 32 * 128 + off), x[1]);
      lds(reinterpret_cast<const T *>(xa + 64 * 128 + off), x[2]);
#pragma unroll
      for (int c = 0; c < K; ++c) lds(wp + c * Sh::CHUNK + q * V, w[c]);  // broadcasts
    };
    load_q(0, xv[0], wv[0]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q < 3) load_q(q + 1, xv[(q + 1) & 1], wv[(q + 1) & 1]);
      const T(&v0)[V] = xv[q & 1][0];
      const T(&v1)[V] = xv[q & 1][1];
      const T(&v2)[V] = xv[q & 1][2];
      const T(&w)[K][V] = wv[q & 1];
      // column-outer order: consecutive FMAs hit different accumulators, the
      // same accumulator recurs only every 3K instructions
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int c = 0; c < K; ++c) {
          acc0[c] = fma(v0[v], w[c][v], acc0[c]);
          acc1[c] = fma(v1[v], w[c][v], acc1[c]);
          acc2[c] = fma(v2[v], w[c][v], acc2[c]);
        }
    }
#endif
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    ++itc;
    if (++ch == a.nchunks) {
      ch = 0;
      ++rb;
    }
  }
}

template <typename T, int K>
__global__ void __launch_bounds__(kThreads, 1) gemm1_kernel(const __grid_constant__ G1Args a) {
  pdl_trigger();  // all CTAs are resident (one per SM): safe to let the successor queue
  if (!a.early_x) {
    pdl_wait();
    if (a.skip != nullptr && *a.skip != 0.0) return;
  }
  using Sh = G1Shape<T, K>;
  constexpr int S = Sh::S;
  extern __shared__ __align__(1024) unsigned char smem[];
  double *red = reinterpret_cast<double *>(smem + S * Sh::STAGE);  // [4][kRB][K]
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + S * Sh::STAGE + Sh::RED);
  uint64_t *empty = full + S;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) SNX_TL(0, 0);
  int64_t itp = 0, itc = 0;
  gemm1_body<T, K, S>(a, smem, red, full, empty, gridDim.x, itp, itc, 0u);
}

// ---------------------------------------------------------------- GEMM2
struct G2Args {
  CUtensorMap xmap;  // X: [nrows][P] boxes of 32 rows x TCOL columns
  int64_t nrows;
  int rchunks;     // 32-row chunks (ceil(nrows / 32))
  int maxseg;      // max CTA segments per column tile
  int64_t items;   // col_tiles * rchunks, split evenly over the CTAs
  const void *U;   // nrows rows of KP (padded) elements, X dtype
  double *gp;      // [col_tiles][maxseg][K][TCOL] segment partials
  const double *skip;
  // fused finalize (by the last segment to arrive for a column tile)
  unsigned *tile_count;  // [col_tiles] arrivals (zero at rest)
  int col_tiles;
  int p;
  double scale, lam;
  const double *base;    // v (Hessian) / w (gradient)
  double *out;           // scale * X^T U + lam * base, flat class-major
  double *dots;          // nullable: [tile] partials of base.out, [kDotBlocks + tile] of base.base
};

// out[c*p + j] = scale * sum_seg gp[tile][seg][c][jj] + lam * base[c*p + j] for
// the columns j of one tile, the segments summed in CTA order (numpy rounding:
// two products, one add), plus the tile's partials of base.out and base.base
// (the CG curvature test; tile 0 zeroes the unused partial slots).
template <int K, int TCOL>
__device__ __forceinline__ void tile_finalize(const G2Args &a, int tile, int G, double *shd) {
  const int tid = threadIdx.x;
  const int c_lo = sk_owner(a.items, G, (int64_t)tile * a.rchunks);
  const int nseg = sk_owner(a.items, G, (int64_t)(tile + 1) * a.rchunks - 1) - c_lo + 1;
  constexpr int kPer = (K * TCOL + kConsumers - 1) / kConsumers;
  // the base values first: their loads overlap the segment loads (one L2
  // round trip for both when nseg <= kBatch)
  double bv[kPer];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int e = tid + q * kConsumers;
    const int c = e / TCOL, j = tile * TCOL + (e - c * TCOL);
    bv[q] = (e < K * TCOL && j < a.p) ? __ldcg(a.base + (int64_t)c * a.p + j)  // may be written
                                      : 0.0;                                  // by other CTAs
  }
  double acc[kPer];
  segment_sums<kPer, (kPer <= 8 ? 8 : 4)>(a.gp + (int64_t)tile * a.maxseg * K * TCOL,
                                          (int64_t)K * TCOL, nseg, tid, kConsumers, K * TCOL,
                                          acc);
  double bo = 0.0, bb = 0.0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int e = tid + q * kConsumers;
    const int c = e / TCOL, j = tile * TCOL + (e - c * TCOL);
    if (e < K * TCOL && j < a.p) {
      const double b = bv[q];
      const double o = __dadd_rn(__dmul_rn(a.scale, acc[q]), __dmul_rn(a.lam, b));
      a.out[(int64_t)c * a.p + j] = o;
      bo += b * o;
      bb += b * b;
    }
  }
  if (a.dots == nullptr) return;
  // both curvature partials in one fixed-order block reduction
  bo = warp_allsum(bo);
  bb = warp_allsum(bb);
  if ((tid & 31) == 0) {
    shd[tid >> 5] = bo;
    shd[kWarps + (tid >> 5)] = bb;
  }
  consumer_sync(kConsumers);
  if (tid == 0) {
    double so = 0.0, sb = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      so += shd[w];
      sb += shd[kWarps + w];
    }
    a.dots[tile] = so;
    a.dots[kDotBlocks + tile] = sb;
  }
  consumer_sync(kConsumers);
  if (tile == 0)
    for (int t = a.col_tiles + tid; t < kDotBlocks; t += kConsumers) {
      a.dots[t] = 0.0;
      a.dots[kDotBlocks + t] = 0.0;
    }
}

// GEMM2 work of one CTA (see gemm1_body).
template <typename T, int K, int S>
__device__ __forceinline__ void gemm2_body(const G2Args &a, unsigned char *smem, double *red,
                                           uint64_t *full, uint64_t *empty, int G, int64_t &itp,
                                           int64_t &itc, unsigned epoch) {
  using Sh = G2Shape<T, K>;
  constexpr int V = Sh::V, LC = Sh::LC, TCOL = Sh::TCOL, KP = Sh::KP;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x;
  if (cta >= G) return;
  const int64_t i0 = sk_begin(a.items, G, cta), i1 = sk_begin(a.items, G, cta + 1);
  if (i0 == i1) return;
  const int tile0 = (int)(i0 / a.rchunks);
  const int rc0 = (int)(i0 - (int64_t)tile0 * a.rchunks);
  __shared__ double shd[2 * kWarps];
  __shared__ int last_tile;

  if (warp == kWarps) {
    // ------------------------------------------------ producer warp (TMA)
    if (lane == 0) {
      tma_prefetch_desc(&a.xmap);
      const T *U = static_cast<const T *>(a.U);
      int tile = tile0, rc = rc0;
      for (int64_t i = i0; i < i1; ++i, ++itp) {
        const int64_t c0 = (int64_t)rc * kG2Rows;
        const int nr = (int)min((int64_t)kG2Rows, a.nrows - c0);
        const int s = (int)(itp % S);
        mbar_wait(&empty[s], (unsigned)((itp / S) & 1) ^ 1u);
        const unsigned ub = (unsigned)(nr * KP * sizeof(T));
        mbar_arrive_expect_tx(&full[s], (unsigned)Sh::XB + ub);
        unsigned char *st = smem + s * Sh::STAGE;
        tma_load_2d(st, &a.xmap, tile * TCOL, (int)c0, &full[s]);
        if (i == i0) pdl_wait();  // no-op unless launched as a programmatic dependent
        bulk_g2s(st + Sh::XB, U + c0 * KP, ub, &full[s]);
        // the done flag of a captured CG loop is read only after the wait: the
        // kernel that writes it (cg_step2 / the fused tail) may still be running
        // when this grid starts (GEMM1 lets its dependents launch early)
        if (i == i0 && a.skip != nullptr && *a.skip != 0.0) {
          mbar_wait(&full[s], (unsigned)((itp / S) & 1));  // the staged copy lands first
          break;
        }
        if (++rc == a.rchunks) {
          rc = 0;
          ++tile;
        }
      }
    }
    return;
  }

  // -------------------------------------------------- consumer warps
  pdl_wait();  // no-op unless launched as a programmatic dependent
  if (a.skip != nullptr && *a.skip != 0.0) return;
  T acc[LC][K];
#pragma unroll
  for (int v = 0; v < LC; ++v)
#pragma unroll
    for (int c = 0; c < K; ++c) acc[v][c] = T(0);
  int tile = tile0, rc = rc0;
  for (int64_t i = i0; i <= i1; ++i) {
    if (i == i1 || (rc == 0 && i > i0)) {
      if (i == i1 && tid == 0) SNX_TL(1, 2);
      // flush the segment partial of the tile just finished: warp pairs
      // (w, w+4), then the 4 pair sums in order
      const int ftile = (i == i1 && rc != 0) ? tile : tile - 1;
      // lane columns: acc[v] is column V*lane + v (v < V) of the tile's first
      // half and 32V + V*lane + v - V of its second half (conflict-free loads)
      double *mine = red + (size_t)(warp & 3) * K * TCOL;
      auto col_of = [&](int v) { return v < V ? V * lane + v : 32 * V + V * lane + (v - V); };
      if (warp >= 4) {
#pragma unroll
        for (int c = 0; c < K; ++c)
#pragma unroll
          for (int v = 0; v < LC; ++v) mine[c * TCOL + col_of(v)] = (double)acc[v][c];
      }
      consumer_sync(kConsumers);
      if (warp < 4) {
#pragma unroll
        for (int c = 0; c < K; ++c)
#pragma unroll
          for (int v = 0; v < LC; ++v)
            mine[c * TCOL + col_of(v)] = (double)acc[v][c] + mine[c * TCOL + col_of(v)];
      }
#pragma unroll
      for (int v = 0; v < LC; ++v)
#pragma unroll
        for (int c = 0; c < K; ++c) acc[v][c] = T(0);
      consumer_sync(kConsumers);
      const int c_lo = sk_owner(a.items, G, (int64_t)ftile * a.rchunks);
      double *gb = a.gp + ((int64_t)ftile * a.maxseg + (cta - c_lo)) * K * TCOL;
      for (int t = tid; t < K * TCOL; t += kConsumers)
        gb[t] = ((red[t] + red[K * TCOL + t]) + red[2 * K * TCOL + t]) + red[3 * K * TCOL + t];
      consumer_sync(kConsumers);  // segment written; red free again
      if (i == i1 && tid == 0) SNX_TL(1, 4);
      if (tid == 0) {
        const int nseg = sk_owner(a.items, G, (int64_t)(ftile + 1) * a.rchunks - 1) - c_lo + 1;
        const unsigned prev = atomic_add_acq_rel(&a.tile_count[ftile], 1u);  // publish / acquire
        last_tile = prev == (unsigned)(nseg - 1);
        if (last_tile) a.tile_count[ftile] = 0u;  // rest state for the next launch
      }
      consumer_sync(kConsumers);
      if (i == i1 && tid == 0) SNX_TL(1, 5);
      if (last_tile) {
        tile_finalize<K, TCOL>(a, ftile, G, shd);
        consumer_sync(kConsumers);
        if (i == i1 && tid == 0) SNX_TL(1, 6);
      }
    }
    if (i == i1) {
      if (tid == 0) SNX_TL(1, 3);
      break;
    }
    const int s = (int)(itc % S);
    mbar_wait(&full[s], (unsigned)((itc / S) & 1));
    if (tid == 0 && i == i0) SNX_TL(1, 1);
    const int nr = (int)min((int64_t)kG2Rows, a.nrows - (int64_t)rc * kG2Rows);
    const T *xs = reinterpret_cast<const T *>(smem + s * Sh::STAGE);
    const T *us = reinterpret_cast<const T *>(smem + s * Sh::STAGE + Sh::XB);
    if (nr == kG2Rows) {
      // full chunk: rows warp + 8j, j < 4, software-pipelined (row j+1's
      // operands load while row j's 2VK FMAs issue)
      T xb[2][2][V], ub[2][KP];
      auto load_r = [&](int r, T (&x)[2][V], T (&u)[KP]) {
        lds(xs + r * TCOL + lane * V, x[0]);
        lds(xs + r * TCOL + 32 * V + lane * V, x[1]);
#pragma unroll
        for (int k = 0; k < KP; k += V) {  // 128-bit broadcasts of the U row
          T t4[V];
          lds(us + r * KP + k, t4);
#pragma unroll
          for (int v = 0; v < V; ++v) u[k + v] = t4[v];
        }
      };
      load_r(warp, xb[0], ub[0]);
#pragma unroll
      for (int j = 0; j < kG2Rows / kWarps; ++j) {
        if (j + 1 < kG2Rows / kWarps) load_r(warp + kWarps * (j + 1), xb[(j + 1) & 1], ub[(j + 1) & 1]);
        const T(&x)[2][V] = xb[j & 1];
        const T(&u)[KP] = ub[j & 1];
#pragma unroll
        for (int c = 0; c < K; ++c) {
#pragma unroll
          for (int v = 0; v < V; ++v) {
            acc[v][c] = fma(x[0][v], u[c], acc[v][c]);
            acc[V + v][c] = fma(x[1][v], u[c], acc[V + v][c]);
          }
        }
      }
    } else
    for (int r = warp; r < nr; r += kWarps) {
      T x0[V], x1[V];
      lds(xs + r * TCOL + lane * V, x0);
      lds(xs + r * TCOL + 32 * V + lane * V, x1);
      T u[KP];
#pragma unroll
      for (int k = 0; k < KP; k += V) {  // 128-bit broadcasts of the U row
        T t4[V];
        lds(us + r * KP + k, t4);
#pragma unroll
        for (int v = 0; v < V; ++v) u[k + v] = t4[v];
      }
#pragma unroll
      for (int c = 0; c < K; ++c) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          acc[v][c] = fma(x0[v], u[c], acc[v][c]);
          acc[V + v][c] = fma(x1[v], u[c], acc[V + v][c]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    ++itc;
    if (++rc == a.rchunks) {
      rc = 0;
      ++tile;
    }
  }
}

template <typename T, int K>
__global__ void __launch_bounds__(kThreads, 1) gemm2_kernel(const __grid_constant__ G2Args a) {
  pdl_trigger();  // all CTAs are resident (one per SM): safe to let the successor queue
  // launched as a programmatic dependent of GEMM1: X_S is older than both, the
  // U rows, the done flag and the CG state are not -- the producer waits
  // (griddepcontrol.wait) right before its first U load, the consumers before
  // anything else (gemm2_body)
  using Sh = G2Shape<T, K>;
  constexpr int S = Sh::S;
  extern __shared__ __align__(1024) unsigned char smem[];
  double *red = reinterpret_cast<double *>(smem + S * Sh::STAGE);  // [4][K][TCOL]
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + S * Sh::STAGE + Sh::RED);
  uint64_t *empty = full + S;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) SNX_TL(1, 0);
  int64_t itp = 0, itc = 0;
  gemm2_body<T, K, S>(a, smem, red, full, empty, gridDim.x, itp, itc, 0u);
}

// out[c*p + j] = scale * sum_seg gp[tile][seg][c][j % TCOL] + lam * base[c*p + j]
// with the segments (CTAs that covered the tile) summed in CTA order (numpy
// rounding: two products, one add), plus kDotBlocks fixed-order partials of
// base.out and base.base (the CG curvature test).
__global__ void __launch_bounds__(kDotThreads)
    finalize_kernel(const double *__restrict__ gp, int64_t items, int grid, int rchunks,
                    int maxseg, int tcol, int K, int p, double scale, double lam,
                    const double *__restrict__ base, double *__restrict__ out, double *dots,
                    const double *skip) {
  pdl_wait();  // successor launches when this grid exits (implicit trigger)
  if (skip != nullptr && *skip != 0.0) return;
  if (threadIdx.x == 0) SNX_TL(2, 0);
  __shared__ double sh[kDotThreads / 32];
  double bo = 0.0, bb = 0.0;
  const int64_t d = (int64_t)K * p;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
       i += (int64_t)kDotBlocks * kDotThreads) {
    const int c = (int)(i / p);
    const int j = (int)(i - (int64_t)c * p);
    const int tile = j / tcol;
    const int c_lo = sk_owner(items, grid, (int64_t)tile * rchunks);
    const int nseg = sk_owner(items, grid, (int64_t)(tile + 1) * rchunks - 1) - c_lo + 1;
    const double *g = gp + ((int64_t)tile * maxseg * K + c) * tcol + (j - tile * tcol);
    const int64_t sstride = (int64_t)K * tcol;
    double s = 0.0;
    int sg = 0;
    for (; sg + 4 <= nseg; sg += 4) {  // independent loads first, fixed-order sum
      double v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] = __ldcg(g + (sg + k) * sstride);
#pragma unroll
      for (int k = 0; k < 4; ++k) s += v[k];
    }
    for (; sg < nseg; ++sg) s += __ldcg(g + sg * sstride);
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
  if (threadIdx.x == 0) SNX_TL(2, 3);
}

// out = lam * base (the empty dataset: every data term vanishes), with the
// dot partials the CG expects.
__global__ void __launch_bounds__(kDotThreads)
    lam_only_kernel(int K, int p, double lam, const double *__restrict__ base,
                    double *__restrict__ out, double *dots, const double *skip) {
  pdl_wait();  // successor launches when this grid exits (implicit trigger)
  if (skip != nullptr && *skip != 0.0) return;
  __shared__ double sh[kDotThreads / 32];
  double bo = 0.0, bb = 0.0;
  const int64_t d = (int64_t)K * p;
  for (int64_t i = (int64_t)blockIdx.x * kDotThreads + threadIdx.x; i < d;
       i += (int64_t)kDotBlocks * kDotThreads) {
    const double b = base[i];
    const double o = __dadd_rn(0.0, __dmul_rn(lam, b));
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

int launch_finalize(const double *gp, int64_t items, int grid, int rchunks, int maxseg, int tcol,
                    int K, int p, double scale, double lam, const double *base, double *out,
                    double *dots, const double *skip, cudaStream_t st) {
  launch_pdl(finalize_kernel, dim3(kDotBlocks), dim3(kDotThreads), 0, st, gp, items, grid,
             rchunks, maxseg, tcol, K, p, scale, lam, base, out, dots, skip);
  return check_launch("finalize");
}

int launch_lam_only(int K, int p, double lam, const double *base, double *out, double *dots,
                    const double *skip, cudaStream_t st) {
  launch_pdl(lam_only_kernel, dim3(kDotBlocks), dim3(kDotThreads), 0, st, K, p, lam, base, out,
             dots, skip);
  return check_launch("lam_only");
}

// Row gather (dataset.py:90-97 `take`): dst[r][0:ldd] = X[rows[r]][0:ldd],
// labels_out[r] = labels[rows[r]]; one warp per row, 16-B vectors.
template <typename T>
__global__ void __launch_bounds__(256)
    gather_rows_kernel(const T *__restrict__ X, int64_t ldx, const int32_t *__restrict__ labels,
                       const int64_t *__restrict__ rows, int64_t nrows, T *__restrict__ dst,
                       int64_t ldd, int32_t *__restrict__ labels_out) {
  constexpr int V = Vec<T>::N;
  const int lane = threadIdx.x & 31;
  const int64_t nvec = ldd / V;
  for (int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); r < nrows;
       r += (int64_t)gridDim.x * 8) {
    const int64_t g = rows[r];
    const uint4 *src = reinterpret_cast<const uint4 *>(X + g * ldx);
    uint4 *out = reinterpret_cast<uint4 *>(dst + r * ldd);
    for (int64_t q = lane; q < nvec; q += 32) out[q] = __ldg(src + q);
    if (lane == 0 && labels_out != nullptr) labels_out[r] = labels[g];
  }
}

// ---------------------------------------------------------------- host side
static int g_sms = 0;  // cached SM count

int sm_count() {
  if (g_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        g_sms <= 0)
      g_sms = 148;
  }
  return g_sms;
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static bool have_encode() {
  if (g_encode == nullptr) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        fn == nullptr) {
      set_error("snx: cuTensorMapEncodeTiled unavailable (driver too old?)");
      return false;
    }
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  return true;
}

int make_tmap(CUtensorMap *m, bool f64, const void *base, uint64_t cols, uint64_t rows,
              uint64_t ld, uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swz) {
  if (!have_encode()) return 1;
  const size_t tb = f64 ? 8 : 4;
  const cuuint64_t dims[2] = {cols, rows > 0 ? rows : 1};
  const cuuint64_t strides[1] = {ld * tb};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = g_encode(
      m, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
      const_cast<void *>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("snx: cuTensorMapEncodeTiled failed (%d) for %llux%llu ld=%llu box %ux%u", (int)r,
              (unsigned long long)rows, (unsigned long long)cols, (unsigned long long)ld,
              box_rows, box_cols);
    return 1;
  }
  return 0;
}

// bf16 [rows][ld] tensor, 128-B swizzled boxes (box_cols * 2 == 128)
int make_tmap_bf16(CUtensorMap *m, const void *base, uint64_t cols, uint64_t rows, uint64_t ld,
                   uint32_t box_cols, uint32_t box_rows) {
  if (!have_encode()) return 1;
  const cuuint64_t dims[2] = {cols, rows > 0 ? rows : 1};
  const cuuint64_t strides[1] = {ld * 2};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base),
                              dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("snx: cuTensorMapEncodeTiled(bf16) failed (%d) for %llux%llu ld=%llu box %ux%u",
              (int)r, (unsigned long long)rows, (unsigned long long)cols, (unsigned long long)ld,
              box_rows, box_cols);
    return 1;
  }
  return 0;
}

static int make_map(CUtensorMap *m, int dtype, const void *base, uint64_t cols, uint64_t rows,
                    uint64_t ld, uint32_t box_cols, uint32_t box_rows, bool swizzle) {
  return make_tmap(m, dtype == SNX_F64, base, cols, rows, ld, box_cols, box_rows,
                   swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE);
}

size_t rowpass_counter_bytes() { return (size_t)kCounterWords * 4; }

int sk_maxseg(int64_t items, int grid, int per_group) {
  const int64_t per = items / grid > 0 ? items / grid : 1;
  return (int)((per_group + per - 1) / per + 1);
}

Geometry geometry(int dtype, int64_t nrows, int32_t P, int32_t K) {
  (void)K;
  Geometry g{};
  const int sms = sm_count();
  const size_t tb = dtype_bytes(dtype);
  // GEMM1: (96-row block x 512-B column chunk) items, stream-K over the CTAs
  g.chunk = (int)(512 / tb);
  g.nchunks = (P + g.chunk - 1) / g.chunk;
  g.row_blocks = nrows > 0 ? (nrows + kRB - 1) / kRB : 0;
  g.g1_items = g.row_blocks * g.nchunks;
  // never more CTAs than items: every CTA between a group's first and last
  // owner then holds a segment of it
  g.grid1 = (int)(g.g1_items < sms ? (g.g1_items > 0 ? g.g1_items : 1) : sms);
  g.g1_maxseg = sk_maxseg(g.g1_items, g.grid1, g.nchunks);
  // GEMM2: (1-KB column tile x 32-row chunk) items, stream-K over the CTAs
  g.tcol = (int)(1024 / tb);
  g.col_tiles = (P + g.tcol - 1) / g.tcol;
  g.rchunks = nrows > 0 ? (int)((nrows + kG2Rows - 1) / kG2Rows) : 0;
  g.g2_items = (int64_t)g.col_tiles * g.rchunks;
  g.grid2 = (int)(g.g2_items < sms ? (g.g2_items > 0 ? g.g2_items : 1) : sms);
  g.g2_maxseg = sk_maxseg(g.g2_items, g.grid2, g.rchunks);
  return g;
}

Workspace workspace_layout(int dtype, int64_t nrows, int32_t p, int32_t K) {
  const int32_t P = padded(p);
  const Geometry g = geometry(dtype, nrows, P, K);
  const size_t tb = dtype_bytes(dtype);
  Workspace w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = round_up(off + bytes, 256);
    return o;
  };
  const int64_t nr = nrows > 0 ? nrows : 1;
  // The counters sit at offset 0 with a size independent of nrows, so one
  // zero-filled workspace serves calls of every row count (they stay zero at
  // rest).
  w.counters = take((size_t)kCounterWords * 4);
  w.weights = take((size_t)K * P * tb);
  w.rowbuf = take((size_t)nr * u_stride(dtype, K) * tb);  // R / U rows, 16-B padded
  w.zp = take((size_t)(g.row_blocks > 0 ? g.row_blocks : 1) * g.g1_maxseg * kRB * K * 8);
  w.gp = take((size_t)g.col_tiles * g.g2_maxseg * K * g.tcol * 8);
  w.loss_part = take((size_t)(g.row_blocks + 1) * 8);
  w.corr_part = take((size_t)(g.row_blocks + 1) * 8);
  w.dot_part = take((size_t)4 * kDotBlocks * 8);
  if (dtype == SNX_F32) {  // tensor-core Hessian product (snx_tc.cu)
    const TcGeometry t = tc_geometry(nrows, P);
    const size_t kp2 = 2 * (size_t)tc_kp(K);  // [B1 ; B2] rows
    w.tc_b = take(kp2 * round_up((size_t)P, 8) * 2);
    w.tc_ut = take(kp2 * round_up((size_t)nr, 8) * 2);
    w.tc_zp = take((size_t)(t.row_blocks > 0 ? t.row_blocks : 1) * t.maxseg1 * 128 * K * 8);
    w.tc_gp = take((size_t)t.col_tiles * t.maxseg2 * K * 128 * 8);
  }
  // the one-pass cluster row pass (snx_cluster.cu) shares the counter block and
  // carves its cluster partials out of the same buffer
  const size_t cl = cluster_ws_bytes(dtype, nrows, p, K);
  w.total = off > cl ? off : cl;
  return w;
}

template <typename KernelT, typename ArgT>
static int launch_persistent(KernelT kernel, int grid, size_t smem, size_t *configured,
                             cudaStream_t st, const ArgT &args, const char *what,
                             bool pdl = false) {
  if (smem > *configured) {
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
      return check_launch(what);
    *configured = smem;
  }
  carveout(kernel);
  launch_pdl_if(pdl || pdl_enabled(), kernel, dim3(grid), dim3(kThreads), smem, st,
                args);  // one CTA per SM
  return check_launch(what);
}

// SNX_G1_PDL=0: GEMM1 of the Hessian product waits for the previous kernel
// before staging anything (A/B switch for the early X prefetch)
static bool gemm1_early_x() {
  static int on = -1;
  if (on < 0) {
    const char *e = getenv("SNX_G1_PDL");
    on = (e != nullptr && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

template <typename T, int K>
static int launch_gemm1(const G1Args &a, int grid, cudaStream_t st) {
  static size_t configured = 0;
  return launch_persistent(gemm1_kernel<T, K>, grid, G1Shape<T, K>::SMEM, &configured, st, a,
                           "gemm1", a.early_x != 0);
}

template <typename T, int K>
static int launch_gemm2(const G2Args &a, int grid, cudaStream_t st) {
  static size_t configured = 0;
  return launch_persistent(gemm2_kernel<T, K>, grid, G2Shape<T, K>::SMEM, &configured, st, a,
                           "gemm2", gemm2_pdl());
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

int validate(int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p,
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
  if (nrows > 0 && (X == nullptr || (reinterpret_cast<uintptr_t>(X) & 15) != 0)) {
    set_error("snx: X must be a non-NULL 16-byte aligned device pointer");
    return 1;
  }
  const Geometry g = geometry(dtype, nrows, padded(p), K);
  if (g.row_blocks > kMaxRowBlocks || nrows > (int64_t)0x7fffffff) {
    set_error("snx: %lld rows exceed one call's limit (%lld); shard the rows", (long long)nrows,
              (long long)(kMaxRowBlocks * kRB));
    return 1;
  }
  if (g.col_tiles > kMaxTiles) {
    set_error("snx: p=%d too wide for this build (max %d column tiles)", p, kMaxTiles);
    return 1;
  }
  const Workspace w = workspace_layout(dtype, nrows, p, K);
  if (ws == nullptr || ws_bytes < w.total) {
    set_error("snx: workspace too small (%zu < %zu bytes)", ws_bytes, w.total);
    return 1;
  }
  return 0;
}

// Common driver of the row-pass entry points (rows contiguous).
struct ProbsOut {
  int32_t *pred;
  double *stats;
};

static int rowpass(int mode, int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p,
                   int32_t K, const int32_t *labels, const double *w, const double *dir,
                   double alpha, const void *H, void *rowout, double scale, double lam,
                   const double *base, double *out, long long *corr_out, double *vec_out,
                   double *dots, const double *skip, void *ws, size_t ws_bytes,
                   cudaStream_t st, const ProbsOut *po = nullptr) {
  if (validate(dtype, X, ldx, nrows, p, K, ws, ws_bytes)) return 1;
  const int32_t P = padded(p);
  const Geometry g = geometry(dtype, nrows, P, K);
  const Workspace lay = workspace_layout(dtype, nrows, p, K);
  char *wsb = static_cast<char *>(ws);
  unsigned *counters = reinterpret_cast<unsigned *>(wsb + lay.counters);
  double *dotp = reinterpret_cast<double *>(wsb + lay.dot_part);

  // fp64, K <= 9: the one-pass cluster kernel (X streamed once per product)
  // (f32 data: the gradient; its Hessian passes take the one-pass kernel only
  // through the row-index entry points, whose h is fp64)
  if (nrows > 0 &&
      ((mode == kHessApply && dtype == SNX_F64 && cluster_supported(dtype, p, K)) ||
       (mode == kGradient && cluster_grad_preferred(dtype, p, K)))) {
    if (mode == kGradient && out != nullptr &&
        launch_prep_weights(dtype, w, nullptr, 0.0, K, p, P, nullptr, dotp, counters + 15,
                            out + 1, st))
      return 1;
    return cluster_rowpass(mode == kHessApply ? 1 : 2, dtype, X, ldx,
                           nullptr, nrows, p, K, labels, w, static_cast<const double *>(H),
                           nullptr, scale, lam, base, vec_out, out, corr_out, dots, skip,
                           (mode == kHessApply && gemm1_early_x()) ? 1 : 0, ws, ws_bytes, st);
  }

  // Weights in the X dtype, padded to P columns (and ||w_eff||^2 for the
  // objective's regulariser).
  const void *Wt = w;
  const bool need_wsq = (mode == kObjective || mode == kGradient) && out != nullptr;
  const bool convert = dtype == SNX_F32 || dir != nullptr || P != p;
  if (convert || need_wsq) {
    void *dst = convert ? (void *)(wsb + lay.weights) : nullptr;
    if (launch_prep_weights(dtype, w, dir, alpha, K, p, P, dst, dotp, counters + 15,
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
    if (mode == kGradient || mode == kHessApply) {
      launch_pdl(lam_only_kernel, dim3(kDotBlocks), dim3(kDotThreads), 0, st, K, p, lam, base, vec_out, dots, skip);
      return check_launch("lam_only");
    }
    return 0;
  }

  const size_t tb = dtype_bytes(dtype);
  void *rowbuf = (rowout || mode == kProbs) ? rowout : (void *)(wsb + lay.rowbuf);
  double *zp = reinterpret_cast<double *>(wsb + lay.zp);
  G1Args a{};
  if (make_map(&a.xmap, dtype, X, P, nrows, ldx, (uint32_t)(128 / tb), kRB, true)) return 1;
  if (make_map(&a.wmap, dtype, Wt, P, K, P, (uint32_t)(512 / tb), K, false)) return 1;
  a.nrows = nrows;
  a.nchunks = g.nchunks;
  a.maxseg = g.g1_maxseg;
  a.items = g.g1_items;
  a.zp = zp;
  a.skip = skip;
  a.row_blocks = g.row_blocks;
  a.mode = mode;
  a.ustride = mode == kHessPrep ? K : u_stride(dtype, K);
  a.rb_count = counters + 16 + kMaxTiles;  // [row_blocks]
  a.done_rb = counters + 2;
  a.labels = labels;
  a.H = H;
  a.rowout = rowbuf;
  a.loss_part = reinterpret_cast<double *>(wsb + lay.loss_part);
  a.corr_part = reinterpret_cast<unsigned long long *>(wsb + lay.corr_part);
  a.loss_out = out;
  a.corr_out = corr_out;
  // the CG loop's product: X_S is older than the kernel before (cg_step2), the
  // weights s and the skip flag are its outputs -> stage X early (PDL)
  a.early_x = (mode == kHessApply && !convert && gemm1_early_x()) ? 1 : 0;
  a.pred_out = po ? po->pred : nullptr;
  a.stats_out = po ? po->stats : nullptr;
  int rc = 1;
  if (dtype == SNX_F64) {
    SNX_K_SWITCH(K, (rc = launch_gemm1<double, KK>(a, g.grid1, st)));
  } else {
    SNX_K_SWITCH(K, (rc = launch_gemm1<float, KK>(a, g.grid1, st)));
  }
  if (rc) return rc;
  if (mode != kGradient && mode != kHessApply) return 0;

  G2Args b{};
  if (make_map(&b.xmap, dtype, X, P, nrows, ldx, (uint32_t)g.tcol, kG2Rows, false)) return 1;
  b.nrows = nrows;
  b.rchunks = g.rchunks;
  b.maxseg = g.g2_maxseg;
  b.items = g.g2_items;
  b.U = rowbuf;
  b.gp = reinterpret_cast<double *>(wsb + lay.gp);
  b.skip = skip;
  b.tile_count = counters + 16;  // [col_tiles <= kMaxTiles]
  b.col_tiles = g.col_tiles;
  b.p = p;
  b.scale = scale;
  b.lam = lam;
  b.base = base;
  b.out = vec_out;
  b.dots = dots;
  if (dtype == SNX_F64) {
    SNX_K_SWITCH(K, (rc = launch_gemm2<double, KK>(b, g.grid2, st)));
  } else {
    SNX_K_SWITCH(K, (rc = launch_gemm2<float, KK>(b, g.grid2, st)));
  }
  return rc;
}

int gather(int dtype, const void *X, int64_t ldx, const int32_t *labels,
                  const int64_t *rows, int64_t nrows, void *dst, int64_t ldd,
                  int32_t *labels_out, cudaStream_t st) {
  if (nrows == 0) return 0;
  if (X == nullptr || rows == nullptr || dst == nullptr || ldd > ldx || ldd % 4 != 0 ||
      ldx % 4 != 0) {
    set_error("snx_gather_rows: bad arguments (NULL pointer or ld_out > ldx / not %% 4)");
    return 1;
  }
  if (labels_out != nullptr && labels == nullptr) {
    set_error("snx_gather_rows: labels_out without labels");
    return 1;
  }
  const int64_t blocks64 = (nrows + 7) / 8;
  const int blocks = (int)(blocks64 < 8 * sm_count() ? blocks64 : 8 * sm_count());
  if (dtype == SNX_F64) {
    gather_rows_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double *>(X), ldx,
                                                        labels, rows, nrows,
                                                        static_cast<double *>(dst), ldd,
                                                        labels_out);
  } else {
    gather_rows_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float *>(X), ldx,
                                                       labels, rows, nrows,
                                                       static_cast<float *>(dst), ldd,
                                                       labels_out);
  }
  return check_launch("gather_rows");
}

}  // namespace snx

using namespace snx;

extern "C" {

#ifdef SNX_TIMELINE
int snx_debug_timeline(unsigned long long *host_out) {
  return cudaMemcpyFromSymbol(host_out, g_timeline, sizeof(g_timeline)) == cudaSuccess ? 0 : 1;
}
#endif

size_t snx_workspace_bytes(int dtype, int64_t nrows, int32_t p, int32_t K) {
  return workspace_layout(dtype, nrows, p, K).total;
}

int snx_gather_rows(int dtype, const void *X, int64_t ldx, const int32_t *labels,
                    const int64_t *rows, int64_t nrows, void *X_out, int64_t ld_out,
                    int32_t *labels_out, void *stream) {
  if (dtype != SNX_F64 && dtype != SNX_F32) {
    set_error("snx_gather_rows: unknown dtype %d", dtype);
    return 1;
  }
  return gather(dtype, X, ldx, labels, rows, nrows, X_out, ld_out, labels_out,
                (cudaStream_t)stream);
}

int snx_objective(int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p, int32_t K,
                  const int32_t *labels, const double *w, const double *dir, double alpha,
                  double *out, int64_t *correct_out, void *ws, size_t ws_bytes, void *stream) {
  if (out == nullptr || w == nullptr || (nrows > 0 && labels == nullptr)) {
    set_error("snx_objective: NULL out/w/labels");
    return 1;
  }
  return rowpass(kObjective, dtype, X, ldx, nrows, p, K, labels, w, dir, alpha, nullptr,
                 nullptr, 1.0, 0.0, nullptr, out, reinterpret_cast<long long *>(correct_out),
                 nullptr, nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

int snx_objective_grad(int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p,
                       int32_t K, const int32_t *labels, const double *w, double scale,
                       double lam, double *out, double *G_out, void *ws, size_t ws_bytes,
                       void *stream) {
  if (out == nullptr || w == nullptr || G_out == nullptr || (nrows > 0 && labels == nullptr)) {
    set_error("snx_objective_grad: NULL out/w/G_out/labels");
    return 1;
  }
  return rowpass(kGradient, dtype, X, ldx, nrows, p, K, labels, w, nullptr, 0.0, nullptr,
                 nullptr, scale, lam, w, out, nullptr, G_out, nullptr, nullptr, ws, ws_bytes,
                 (cudaStream_t)stream);
}

int snx_class_probabilities(int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p,
                            int32_t K, const int32_t *labels, const double *w, double *probs_out,
                            int32_t *pred_out, double *stats_out, void *ws, size_t ws_bytes,
                            void *stream) {
  if (w == nullptr || (nrows > 0 && stats_out != nullptr && labels == nullptr)) {
    set_error("snx_class_probabilities: NULL w (or labels with stats_out)");
    return 1;
  }
  const ProbsOut po{pred_out, stats_out};
  return rowpass(kProbs, dtype, X, ldx, nrows, p, K, labels, w, nullptr, 0.0, nullptr,
                 probs_out, 1.0, 0.0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, ws,
                 ws_bytes, (cudaStream_t)stream, &po);
}

int snx_objective_grad_acc(int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p,
                           int32_t K, const int32_t *labels, const double *w, double scale,
                           double lam, double *out, int64_t *correct_out, double *G_out, void *ws,
                           size_t ws_bytes, void *stream) {
  if (out == nullptr || w == nullptr || G_out == nullptr || (nrows > 0 && labels == nullptr)) {
    set_error("snx_objective_grad_acc: NULL out/w/G_out/labels");
    return 1;
  }
  return rowpass(kGradient, dtype, X, ldx, nrows, p, K, labels, w, nullptr, 0.0, nullptr,
                 nullptr, scale, lam, w, out, reinterpret_cast<long long *>(correct_out), G_out,
                 nullptr, nullptr, ws, ws_bytes, (cudaStream_t)stream);
}

int snx_hess_prepare(int dtype, const void *X, int64_t ldx, const int64_t *rows, int64_t nrows,
                     int32_t p, int32_t K, const double *w, void *Xs_out, int64_t ld_out,
                     void *H_out, void *ws, size_t ws_bytes, void *stream) {
  if (w == nullptr || (nrows > 0 && H_out == nullptr)) {
    set_error("snx_hess_prepare: NULL w/H_out");
    return 1;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (nrows > 0 && cluster_supported(dtype, p, K) && (dtype == SNX_F64 || Xs_out == nullptr)) {
    // one pass over X[rows]: the row gather is fused into the TMA loads; X_S is
    // materialised only if the caller asks for it (Xs_out != NULL).  f32 data:
    // only without X_S (the fused path), and H_out is fp64
    if (validate(dtype, X, ldx, nrows, p, K, ws, ws_bytes)) return 1;
    if (rows != nullptr && Xs_out != nullptr &&
        gather(dtype, X, ldx, nullptr, rows, nrows, Xs_out, ld_out, nullptr, st))
      return 1;
    return cluster_rowpass(0, dtype, X, ldx, rows, nrows, p, K, nullptr, w,
                           nullptr, static_cast<double *>(H_out), 1.0, 0.0, nullptr, nullptr,
                           nullptr, nullptr, nullptr, nullptr, 0, ws, ws_bytes, st);
  }
  const void *Xs = X;
  int64_t lds = ldx;
  if (rows != nullptr) {  // materialise X_S = X[rows] (dataset.py:90-97)
    if (gather(dtype, X, ldx, nullptr, rows, nrows, Xs_out, ld_out, nullptr, st)) return 1;
    Xs = Xs_out;
    lds = ld_out;
  }
  return rowpass(kHessPrep, dtype, Xs, lds, nrows, p, K, nullptr, w, nullptr, 0.0, nullptr,
                 H_out, 1.0, 0.0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, ws,
                 ws_bytes, st);
}

int snx_hess_apply(int dtype, const void *Xs, int64_t ldx, int64_t nrows, int32_t p, int32_t K,
                   const void *H, const double *v, double scale, double lam, double *Hv_out,
                   double *dots, const double *skip, void *ws, size_t ws_bytes, void *stream) {
  if (v == nullptr || Hv_out == nullptr || (nrows > 0 && H == nullptr)) {
    set_error("snx_hess_apply: NULL v/Hv_out/H");
    return 1;
  }
  return rowpass(kHessApply, dtype, Xs, ldx, nrows, p, K, nullptr, v, nullptr, 0.0, H, nullptr,
                 scale, lam, v, nullptr, nullptr, Hv_out, dots, skip, ws, ws_bytes,
                 (cudaStream_t)stream);
}

int snx_hess_apply_cg_rows(int dtype, const void *X, int64_t ldx, const int64_t *rows,
                           int64_t nrows, int32_t p, int32_t K, const void *H, double scale,
                           double lam, int32_t t, int32_t max_iters, double *r, double *s,
                           double *p_vec, double *p_best, double *Hs, double *state, void *ws,
                           size_t ws_bytes, void *stream) {
  if (s == nullptr || Hs == nullptr || state == nullptr || r == nullptr || p_vec == nullptr ||
      p_best == nullptr || H == nullptr) {
    set_error("snx_hess_apply_cg_rows: NULL argument");
    return 1;
  }
  if (t < 0 || t >= max_iters) {
    set_error("snx_hess_apply_cg_rows: iteration %d outside [0, %d)", t, max_iters);
    return 1;
  }
  if (!cluster_supported(dtype, p, K) || nrows < 1) {
    set_error("snx_hess_apply_cg_rows: K <= 9 and nrows >= 1 only (snx_rowpass_fused)");
    return 1;
  }
  if (validate(dtype, X, ldx, nrows, p, K, ws, ws_bytes)) return 1;
  return cluster_cg_iteration(dtype, X, ldx, rows, nrows, p, K,
                              static_cast<const double *>(H), scale, lam, t, max_iters, r, s,
                              p_vec, p_best, Hs, state, gemm1_early_x() ? 1 : 0, ws, ws_bytes,
                              (cudaStream_t)stream);
}

int snx_rowpass_fused(int dtype, int32_t p, int32_t K) {
  return cluster_supported(dtype, p, K) ? 1 : 0;
}

int snx_hess_apply_rows(int dtype, const void *X, int64_t ldx, const int64_t *rows,
                        int64_t nrows, int32_t p, int32_t K, const void *H, const double *v,
                        double scale, double lam, double *Hv_out, double *dots,
                        const double *skip, void *ws, size_t ws_bytes, void *stream) {
  if (v == nullptr || Hv_out == nullptr || (nrows > 0 && H == nullptr)) {
    set_error("snx_hess_apply_rows: NULL v/Hv_out/H");
    return 1;
  }
  if (nrows == 0 || (rows == nullptr && dtype == SNX_F64))
    return snx_hess_apply(dtype, X, ldx, nrows, p, K, H, v, scale, lam, Hv_out, dots, skip, ws,
                          ws_bytes, stream);
  if (!cluster_supported(dtype, p, K)) {
    set_error("snx_hess_apply_rows: K <= 9 only (snx_rowpass_fused)");
    return 1;
  }
  if (validate(dtype, X, ldx, nrows, p, K, ws, ws_bytes)) return 1;
  return cluster_rowpass(1, dtype, X, ldx, rows, nrows, p, K, nullptr, v,
                         static_cast<const double *>(H), nullptr, scale, lam, v, Hv_out, nullptr,
                         nullptr, dots, skip, gemm1_early_x() ? 1 : 0, ws, ws_bytes,
                         (cudaStream_t)stream);
}

}  // extern "C"
