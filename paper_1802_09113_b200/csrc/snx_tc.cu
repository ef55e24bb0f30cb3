// Tensor-core Hessian-vector product for f32 data (the declared 1e-4 path):
// softmax.py:197-210 with both feature products on the 5th-generation tensor
// cores (tcgen05.mma kind::tf32, accumulators in TMEM, operands staged by TMA).
//
// tf32 keeps 10 mantissa bits, so each product is split 3xTF32-style:
//   A.B ~= A_hi.B_hi + A_hi.B_lo + A_lo.B_hi,   x_lo = x - tf32(x),
// where the hardware truncation of an f32 operand IS x_hi.  X_lo is
// materialised once per sample (snx_hess_prepare_tc), the small operand is
// stacked as [B ; B_lo] (N = 32), so one MMA with N = 32 gives A_hi.B_hi and
// A_hi.B_lo and a second with N = 16 adds A_lo.B_hi into the first 16 columns.
//
//   GEMM1 (tc_gemm1_kernel): V = X_S Q(v).  Items (128-row block x 32-column
//     k-tile), stream-K over one CTA per SM; A = X / X_lo tiles (K-major,
//     128-B swizzle), B = [Q ; Q_lo] (K-major).  The segment partial of a row
//     block leaves TMEM as doubles; the last segment to arrive (acq_rel
//     counter) sums the segments in fixed order and applies ComputeU
//     (softmax.py:206-208), writing U^T and U^T_lo as GEMM2's B operand.
//   GEMM2 (tc_gemm2_kernel): X_S^T U.  Items (128-column tile x 32-row chunk);
//     A = X tile read MN-major (128-B swizzle, 32-B atoms), B = [U^T ; U^T_lo].
//     Segment partials go to finalize_kernel (scale, + lam v, CG dots).
// Warp roles (192 threads, one CTA per SM): warp 0 TMA producer, warp 1 MMA
// issuer (one thread) and TMEM owner, warps 2-5 epilogue (TMEM lane quarters).
// All reductions are in a fixed order: reruns are bit-identical.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "snx_common.cuh"
#include "snx_internal.h"
#include "snx_pipe.cuh"
#include "snx_umma.cuh"

namespace snx {

int make_tmap(CUtensorMap *m, bool f64, const void *base, uint64_t cols, uint64_t rows,
              uint64_t ld, uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swz);

#ifdef SNX_TIMELINE
__device__ unsigned long long g_tc_timeline[2][160][4];
#define SNX_TC_TL(slot, ev)                                                \
  do {                                                                     \
    unsigned long long t_;                                                 \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
    if (blockIdx.x < 160) g_tc_timeline[slot][blockIdx.x][ev] = t_;       \
  } while (0)
#else
#define SNX_TC_TL(slot, ev) \
  do {                      \
  } while (0)
#endif

namespace {

constexpr int kThreads = 192;
constexpr int kS = 5;                          // pipeline stages
constexpr uint32_t kXB = 16384;                // X tile: 128 x 32 f32
constexpr uint32_t kBB = 4096;                 // B tile: 32 x 32 f32
constexpr uint32_t kStage = 2 * kXB + kBB;     // X, X_lo, B
constexpr size_t kSmem = kS * kStage + 1024;   // + alignment slack
constexpr uint32_t kTmemCols = 64;             // two 32-column accumulators

__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
  return reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// named barrier over the 128 epilogue threads (warps 2-5)
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 2, 128;\n" ::: "memory"); }

struct Tc1Args {
  CUtensorMap xmap;   // X    [nrows][P]: boxes 32 cols x 128 rows, 128-B swizzle
  CUtensorMap lmap;   // X_lo [nrows][P]: same
  CUtensorMap bmap;   // [Q ; Q_lo] [32][P]: boxes 32 x 32, 128-B swizzle
  int64_t nrows;
  int nk;             // 32-column k-tiles per row
  int64_t items;      // row_blocks * nk
  int maxseg;
  const float *H;     // [nrows][K] probabilities
  float *ut;          // [32][ldu]: U^T rows 0..K-1, U^T_lo rows 16..16+K-1
  int64_t ldu;
  double *zp;         // [row_blocks][maxseg][128][K] segment partials
  unsigned *rb_count; // [row_blocks] arrivals (zero at rest)
  const double *skip;
};

struct Tc2Args {
  CUtensorMap xmap;   // X    [nrows][P]: boxes 32 cols x 32 rows, 128-B swizzle 32-B atoms
  CUtensorMap lmap;   // X_lo [nrows][P]: same
  CUtensorMap umap;   // [U^T ; U^T_lo] [32][ldu]: boxes 32 x 32, 128-B swizzle
  int64_t nrows;
  int rchunks;        // 32-row chunks
  int64_t items;      // col_tiles * rchunks
  int maxseg;
  double *gp;         // [col_tiles][maxseg][K][128] segment partials
  const double *skip;
};

// Common skeleton: barriers, TMEM, warp roles.  LOAD(i, stage, bar) issues the
// TMA of item i; MMA(stage_addr, d_tmem, first) issues its MMAs; SEG_END(i) is
// true when item i closes a segment; EPI(seg_first_item, v0, v1) consumes the
// accumulator of one segment (epilogue threads).
struct Barriers {
  uint64_t full[kS], empty[kS], accf[2], acce[2];
  uint32_t tbase;
  int flag;
};

__device__ __forceinline__ void setup(Barriers &b, int warp) {
  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < kS; ++s) {
      mbar_init(&b.full[s], 1);
      mbar_init(&b.empty[s], 1);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      mbar_init(&b.accf[k], 1);
      mbar_init(&b.acce[k], 4);
    }
    mbar_fence_init();
  }
  if (warp == 1) umma::tmem_alloc(&b.tbase, kTmemCols);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
}

__device__ __forceinline__ void teardown(Barriers &b, int warp) {
  umma::fence_before();
  __syncthreads();
  if (warp == 1) {
    umma::fence_after();
    umma::tmem_dealloc(b.tbase, kTmemCols);
  }
}

// Epilogue threads: wait for the accumulator of segment `n` (buffer n & 1) and
// load this thread's TMEM lane (32 columns), then release the buffer.
__device__ __forceinline__ void acc_take(Barriers &b, int n, int warp, int lane, float (&v0)[16],
                                         float (&v1)[16]) {
  const int buf = n & 1;
  mbar_wait(&b.accf[buf], (unsigned)((n >> 1) & 1));
  umma::fence_after();
  const uint32_t t = b.tbase + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(buf * 32);
  umma::tmem_ld16(t, v0);
  umma::tmem_ld16(t + 16, v1);
  umma::fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive(&b.acce[buf]);
}

// MMA issuer loop (one thread).  a_mn selects the MN-major A layout (GEMM2).
template <bool kAmn, typename SegStart, typename SegEnd>
__device__ __forceinline__ void mma_loop(Barriers &b, uint8_t *sm, int64_t i0, int64_t i1,
                                         SegStart seg_start, SegEnd seg_end) {
  constexpr int slot = kAmn ? 1 : 0;
  (void)slot;
  constexpr uint32_t id32 = umma::idesc_tf32(128, 32, kAmn, false);
  constexpr uint32_t id16 = umma::idesc_tf32(128, 16, kAmn, false);
  int nseg = 0;
  for (int64_t i = i0, it = 0; i < i1; ++i, ++it) {
    const bool first = i == i0 || seg_start(i);
    const int buf = nseg & 1;
    if (first) {
      mbar_wait(&b.acce[buf], (unsigned)(((nseg >> 1) & 1) ^ 1));
      umma::fence_after();
    }
    const int s = (int)(it % kS);
    mbar_wait(&b.full[s], (unsigned)((it / kS) & 1));
    umma::fence_after();
    if (it == 0) SNX_TC_TL(slot, 1);
    const uint32_t st = umma::smem_u32(sm + s * kStage);
    const uint32_t d = b.tbase + (uint32_t)(buf * 32);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint64_t ax, al;
      if (kAmn) {  // 8 K-rows of 128 B per MMA; 32-column blocks 4 KB apart
        ax = umma::desc_mn_sw128_32b(st + k * 1024, 4096);
        al = umma::desc_mn_sw128_32b(st + kXB + k * 1024, 4096);
      } else {     // 8 K-columns (32 B) per MMA inside the 128-B rows
        ax = umma::desc_k_sw128(st + k * 32);
        al = umma::desc_k_sw128(st + kXB + k * 32);
      }
      const uint64_t bd = umma::desc_k_sw128(st + 2 * kXB + k * 32);
      umma::mma_tf32(d, ax, bd, id32, (first && k == 0) ? 0u : 1u);  // A_hi.[B_hi | B_lo]
      umma::mma_tf32(d, al, bd, id16, 1u);                            // + A_lo.B_hi
    }
    umma::commit(&b.empty[s]);  // stage free once these MMAs completed
    if (i + 1 == i1 || seg_end(i)) {
      umma::commit(&b.accf[buf]);
      ++nseg;
    }
  }
  SNX_TC_TL(slot, 2);
}

// ---------------------------------------------------------------- GEMM1
template <int K>
__global__ void __launch_bounds__(kThreads, 1) tc_gemm1_kernel(const __grid_constant__ Tc1Args a) {
  if (a.skip != nullptr && *a.skip != 0.0) return;
  extern __shared__ uint8_t smraw[];
  uint8_t *sm = align1024(smraw);
  __shared__ Barriers b;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  const int64_t i0 = sk_begin(a.items, G, cta), i1 = sk_begin(a.items, G, cta + 1);
  if (i0 == i1) return;
  if (tid == 0) SNX_TC_TL(0, 0);
  setup(b, warp);
  const int nk = a.nk;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&a.xmap);
      tma_prefetch_desc(&a.lmap);
      tma_prefetch_desc(&a.bmap);
      for (int64_t i = i0, it = 0; i < i1; ++i, ++it) {
        const int s = (int)(it % kS);
        mbar_wait(&b.empty[s], (unsigned)(((it / kS) & 1) ^ 1));
        mbar_arrive_expect_tx(&b.full[s], kStage);
        uint8_t *st = sm + s * kStage;
        const int rb = (int)(i / nk), kt = (int)(i - (int64_t)rb * nk);
        tma_load_2d(st, &a.xmap, kt * 32, rb * 128, &b.full[s]);
        tma_load_2d(st + kXB, &a.lmap, kt * 32, rb * 128, &b.full[s]);
        tma_load_2d(st + 2 * kXB, &a.bmap, kt * 32, 0, &b.full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0)
      mma_loop<false>(
          b, sm, i0, i1, [&](int64_t i) { return i % nk == 0; },
          [&](int64_t i) { return (i + 1) % nk == 0; });
    __syncwarp();
  } else {
    // ------------------------------------------------ epilogue warps 2-5
    const int row = (warp & 3) * 32 + lane;  // TMEM lane = row within the block
    const int et = tid - 64;
    int n = 0;
    for (int64_t rb = i0 / nk; rb <= (i1 - 1) / nk; ++rb, ++n) {
      float v0[16], v1[16];
      acc_take(b, n, warp, lane, v0, v1);
      const int c_lo = sk_owner(a.items, G, rb * nk);
      const int nseg = sk_owner(a.items, G, (rb + 1) * nk - 1) - c_lo + 1;
      const int64_t r = rb * 128 + row;
      double *zrow = a.zp + ((rb * a.maxseg + (cta - c_lo)) * 128 + row) * K;
      if (r < a.nrows) {
#pragma unroll
        for (int c = 0; c < K; ++c) zrow[c] = (double)v0[c] + (double)v1[c];
      }
      epi_sync();
      if (et == 0) {
        const unsigned prev = atomic_add_acq_rel(&a.rb_count[rb], 1u);  // publish / acquire
        b.flag = prev == (unsigned)(nseg - 1);
        if (b.flag) a.rb_count[rb] = 0u;  // rest state for the next launch
      }
      epi_sync();
      if (b.flag && r < a.nrows) {
        // last segment of this row block: fixed-order segment sum, ComputeU
        const double *z0 = a.zp + (rb * a.maxseg * 128 + row) * K;
        double V[K];
#pragma unroll
        for (int c = 0; c < K; ++c) V[c] = 0.0;
        for (int sg = 0; sg < nseg; ++sg) {
#pragma unroll
          for (int c = 0; c < K; ++c) V[c] += __ldcg(z0 + (int64_t)sg * 128 * K + c);
        }
        const float *h = a.H + r * K;
        double hw[K], vw[K], s = 0.0;
#pragma unroll
        for (int c = 0; c < K; ++c) {
          hw[c] = (double)h[c];
          vw[c] = V[c] * hw[c];
          s += vw[c];
        }
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const float u = (float)(vw[c] - hw[c] * s);
          a.ut[(int64_t)c * a.ldu + r] = u;
          a.ut[(int64_t)(16 + c) * a.ldu + r] = u - umma::tf32_hi(u);
        }
      }
      epi_sync();
    }
    if (et == 0) SNX_TC_TL(0, 3);
  }
  teardown(b, warp);
}

// ---------------------------------------------------------------- GEMM2
template <int K>
__global__ void __launch_bounds__(kThreads, 1) tc_gemm2_kernel(const __grid_constant__ Tc2Args a) {
  if (a.skip != nullptr && *a.skip != 0.0) return;
  extern __shared__ uint8_t smraw[];
  uint8_t *sm = align1024(smraw);
  __shared__ Barriers b;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x, cta = blockIdx.x;
  const int64_t i0 = sk_begin(a.items, G, cta), i1 = sk_begin(a.items, G, cta + 1);
  if (i0 == i1) return;
  if (tid == 0) SNX_TC_TL(1, 0);
  setup(b, warp);
  const int rch = a.rchunks;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&a.xmap);
      tma_prefetch_desc(&a.lmap);
      tma_prefetch_desc(&a.umap);
      for (int64_t i = i0, it = 0; i < i1; ++i, ++it) {
        const int s = (int)(it % kS);
        mbar_wait(&b.empty[s], (unsigned)(((it / kS) & 1) ^ 1));
        mbar_arrive_expect_tx(&b.full[s], kStage);
        uint8_t *st = sm + s * kStage;
        const int tile = (int)(i / rch), rc = (int)(i - (int64_t)tile * rch);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          tma_load_2d(st + q * 4096, &a.xmap, tile * 128 + q * 32, rc * 32, &b.full[s]);
          tma_load_2d(st + kXB + q * 4096, &a.lmap, tile * 128 + q * 32, rc * 32, &b.full[s]);
        }
        tma_load_2d(st + 2 * kXB, &a.umap, rc * 32, 0, &b.full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0)
      mma_loop<true>(
          b, sm, i0, i1, [&](int64_t i) { return i % rch == 0; },
          [&](int64_t i) { return (i + 1) % rch == 0; });
    __syncwarp();
  } else {
    const int col = (warp & 3) * 32 + lane;  // TMEM lane = column within the tile
    int n = 0;
    for (int64_t tile = i0 / rch; tile <= (i1 - 1) / rch; ++tile, ++n) {
      float v0[16], v1[16];
      acc_take(b, n, warp, lane, v0, v1);
      const int seg = cta - sk_owner(a.items, G, tile * rch);
      double *g = a.gp + ((tile * a.maxseg + seg) * K) * 128 + col;
#pragma unroll
      for (int c = 0; c < K; ++c) g[c * 128] = (double)v0[c] + (double)v1[c];
    }
    if (tid == 64) SNX_TC_TL(1, 3);
  }
  teardown(b, warp);
}

// [Q ; Q_lo] from v (class-major d = K*p, fp64): rows c < K: f32(v[c*p + j]),
// rows 16 + c: the tf32 remainder; other rows and columns >= p zero.
__global__ void tc_prep_b_kernel(const double *__restrict__ v, int K, int p, int P,
                                 float *__restrict__ B) {
  const int64_t n = (int64_t)32 * P;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / P), j = (int)(e - (int64_t)r * P);
    const int c = r & 15;
    const float f = (c < K && j < p) ? (float)v[(int64_t)c * p + j] : 0.0f;
    B[e] = r < 16 ? f : f - umma::tf32_hi(f);
  }
}

// X_lo = X - tf32(X) over nrows x ld (float4 vectors).
__global__ void tc_split_kernel(const float4 *__restrict__ X, float4 *__restrict__ L,
                                int64_t n4) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4;
       e += (int64_t)gridDim.x * blockDim.x) {
    const float4 x = X[e];
    L[e] = make_float4(x.x - umma::tf32_hi(x.x), x.y - umma::tf32_hi(x.y),
                       x.z - umma::tf32_hi(x.z), x.w - umma::tf32_hi(x.w));
  }
}

template <typename KernelT, typename ArgT>
int launch_tc(KernelT kernel, int grid, const ArgT &args, cudaStream_t st, size_t *configured,
              const char *what) {
  if (kSmem > *configured) {
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem) !=
        cudaSuccess)
      return check_launch(what);
    *configured = kSmem;
  }
  carveout(kernel);
  kernel<<<grid, kThreads, kSmem, st>>>(args);
  return check_launch(what);
}

template <int K>
int run_tc(const Tc1Args &a1, int g1, const Tc2Args &a2, int g2, cudaStream_t st) {
  static size_t c1 = 0, c2 = 0;
  if (launch_tc(tc_gemm1_kernel<K>, g1, a1, st, &c1, "tc_gemm1")) return 1;
  return launch_tc(tc_gemm2_kernel<K>, g2, a2, st, &c2, "tc_gemm2");
}

}  // namespace

TcGeometry tc_geometry(int64_t nrows, int32_t P) {
  TcGeometry t{};
  const int sms = sm_count();
  t.nk = (P + 31) / 32;
  t.row_blocks = nrows > 0 ? (nrows + 127) / 128 : 0;
  t.items1 = t.row_blocks * t.nk;
  t.grid1 = (int)(t.items1 < sms ? (t.items1 > 0 ? t.items1 : 1) : sms);
  t.maxseg1 = sk_maxseg(t.items1, t.grid1, t.nk);
  t.col_tiles = (P + 127) / 128;
  t.rchunks = nrows > 0 ? (int)((nrows + 31) / 32) : 0;
  t.items2 = (int64_t)t.col_tiles * t.rchunks;
  t.grid2 = (int)(t.items2 < sms ? (t.items2 > 0 ? t.items2 : 1) : sms);
  t.maxseg2 = sk_maxseg(t.items2, t.grid2, t.rchunks);
  return t;
}

static int tc_apply(const float *Xs, const float *Xlo, int64_t ldx, int64_t nrows, int32_t p,
                    int32_t K, const float *H, const double *v, double scale, double lam,
                    double *out, double *dots, const double *skip, void *ws, size_t ws_bytes,
                    cudaStream_t st) {
  if (validate(SNX_F32, Xs, ldx, nrows, p, K, ws, ws_bytes)) return 1;
  if (nrows > 0 && (Xlo == nullptr || (reinterpret_cast<uintptr_t>(Xlo) & 15) != 0)) {
    set_error("snx_hess_apply_tc: Xlo must be a 16-byte aligned device pointer");
    return 1;
  }
  if (nrows == 0) return launch_lam_only(K, p, lam, v, out, dots, skip, st);
  const int32_t P = padded(p);
  const TcGeometry t = tc_geometry(nrows, P);
  const Workspace lay = workspace_layout(SNX_F32, nrows, p, K);
  char *wsb = static_cast<char *>(ws);
  unsigned *counters = reinterpret_cast<unsigned *>(wsb + lay.counters);
  float *B = reinterpret_cast<float *>(wsb + lay.tc_b);
  float *UT = reinterpret_cast<float *>(wsb + lay.tc_ut);
  const int64_t ldu = (int64_t)round_up((size_t)nrows, 4);
  // (the workspace is sized for its dataset's row count >= nrows; UT's row
  //  stride follows this call's nrows, the rows past K stay zero)
  tc_prep_b_kernel<<<64, 256, 0, st>>>(v, K, p, P, B);
  if (check_launch("tc_prep_b")) return 1;

  Tc1Args a1{};
  if (make_tmap(&a1.xmap, false, Xs, P, nrows, ldx, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      make_tmap(&a1.lmap, false, Xlo, P, nrows, ldx, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      make_tmap(&a1.bmap, false, B, P, 32, P, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B))
    return 1;
  a1.nrows = nrows;
  a1.nk = t.nk;
  a1.items = t.items1;
  a1.maxseg = t.maxseg1;
  a1.H = H;
  a1.ut = UT;
  a1.ldu = ldu;
  a1.zp = reinterpret_cast<double *>(wsb + lay.tc_zp);
  a1.rb_count = counters + 16 + SNX_DOT_BLOCKS;
  a1.skip = skip;

  Tc2Args a2{};
  if (make_tmap(&a2.xmap, false, Xs, P, nrows, ldx, 32, 32,
                CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ||
      make_tmap(&a2.lmap, false, Xlo, P, nrows, ldx, 32, 32,
                CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ||
      make_tmap(&a2.umap, false, UT, nrows, 32, ldu, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B))
    return 1;
  a2.nrows = nrows;
  a2.rchunks = t.rchunks;
  a2.items = t.items2;
  a2.maxseg = t.maxseg2;
  a2.gp = reinterpret_cast<double *>(wsb + lay.tc_gp);
  a2.skip = skip;

  int rc = 1;
  switch (K) {
#define SNX_TC_CASE(KK) \
  case KK:              \
    rc = run_tc<KK>(a1, t.grid1, a2, t.grid2, st); \
    break;
    SNX_TC_CASE(1) SNX_TC_CASE(2) SNX_TC_CASE(3) SNX_TC_CASE(4) SNX_TC_CASE(5) SNX_TC_CASE(6)
    SNX_TC_CASE(7) SNX_TC_CASE(8) SNX_TC_CASE(9) SNX_TC_CASE(10) SNX_TC_CASE(11)
    SNX_TC_CASE(12) SNX_TC_CASE(13) SNX_TC_CASE(14) SNX_TC_CASE(15) SNX_TC_CASE(16)
#undef SNX_TC_CASE
    default:
      set_error("snx: K = %d outside [1, 16]", K);
      return 1;
  }
  if (rc) return rc;
  return launch_finalize(a2.gp, t.items2, t.grid2, t.rchunks, t.maxseg2, 128, K, p, scale, lam,
                         v, out, dots, skip, st);
}

}  // namespace snx

using namespace snx;

extern "C" {

#ifdef SNX_TIMELINE
int snx_debug_tc_timeline(unsigned long long *host_out) {
  return cudaMemcpyFromSymbol(host_out, g_tc_timeline, sizeof(g_tc_timeline)) == cudaSuccess ? 0
                                                                                             : 1;
}
#endif

int snx_hess_prepare_tc(const float *X, int64_t ldx, const int64_t *rows, int64_t nrows,
                        int32_t p, int32_t K, const double *w, float *Xs_out, float *Xlo_out,
                        int64_t ld_out, float *H_out, void *ws, size_t ws_bytes, void *stream) {
  if (nrows > 0 && (Xlo_out == nullptr || (reinterpret_cast<uintptr_t>(Xlo_out) & 15) != 0)) {
    set_error("snx_hess_prepare_tc: Xlo_out must be a 16-byte aligned device pointer");
    return 1;
  }
  if (snx_hess_prepare(SNX_F32, X, ldx, rows, nrows, p, K, w, Xs_out, ld_out, H_out, ws,
                       ws_bytes, stream))
    return 1;
  if (nrows == 0) return 0;
  const float *Xs = rows != nullptr ? Xs_out : X;
  const int64_t ld = rows != nullptr ? ld_out : ldx;
  const int64_t n4 = nrows * ld / 4;
  const int blocks = (int)((n4 + 255) / 256 < 4 * sm_count() ? (n4 + 255) / 256 : 4 * sm_count());
  tc_split_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const float4 *>(Xs), reinterpret_cast<float4 *>(Xlo_out), n4);
  return check_launch("tc_split");
}

int snx_hess_apply_tc(const float *Xs, const float *Xlo, int64_t ldx, int64_t nrows, int32_t p,
                      int32_t K, const float *H, const double *v, double scale, double lam,
                      double *Hv_out, double *dots, const double *skip, void *ws,
                      size_t ws_bytes, void *stream) {
  if (v == nullptr || Hv_out == nullptr || (nrows > 0 && H == nullptr)) {
    set_error("snx_hess_apply_tc: NULL v/Hv_out/H");
    return 1;
  }
  return tc_apply(Xs, Xlo, ldx, nrows, p, K, H, v, scale, lam, Hv_out, dots, skip, ws, ws_bytes,
                  (cudaStream_t)stream);
}

}  // extern "C"
