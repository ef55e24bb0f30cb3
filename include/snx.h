/*
 * snx.h -- C ABI of libsnx, the sm_100a kernels behind the sub-sampled
 * Newton-CG hot path (arXiv 1802.09113).
 *
 * The reference (/root/reference/pkg/src/subnewton) is pure Python on numpy;
 * it has no FFI.  Its plugin seam is Python callables:
 *   objective_fn(x), oracle.gradient(x), oracle.hessian_operator(x)(v),
 *   cg_solve(apply_H, g, cfg), line_search(f, f0, slope, cfg).
 * Each entry point below replaces the arithmetic of one of those callables;
 * the Python package paper_1802_09113_b200 binds them with ctypes and keeps
 * the reference's names, argument meaning and exceptions.
 *
 * Conventions
 *   - All pointers are DEVICE pointers unless stated; the library never
 *     allocates persistent memory (workspace is passed in, sized by
 *     snx_workspace_bytes).  `stream` is a cudaStream_t (NULL = legacy).
 *   - dtype: SNX_F64 (X stored fp64, fp64 math: 1e-10 parity path) or
 *     SNX_F32 (X stored fp32, fp32 products, fp64 reductions: 1e-4 path).
 *   - X is row-major with leading dimension ldx (elements).  p is the true
 *     feature count; kernels stream P = round_up(p, 4) columns, so ldx >= P,
 *     ldx % 4 == 0 and columns p..P-1 must be zero (snx_pack_rows does this).
 *   - Weight-shaped vectors (x, v, gradients, Hv, CG vectors) are fp64 and
 *     flat class-major, d = K*p, w[c*p + j] for weighted class c < K = C-1:
 *     exactly the reference layout x.reshape((p, C-1), order="F")
 *     (softmax.py:62-74).
 *   - rows: int64 row indices of a sorted sample S (sampling.py:38-45);
 *     labels are int32 in [0, C).  X pointers must be 16-byte aligned.
 *   - Return 0 on success; non-zero => snx_last_error() has the message.
 *   - Every reduction runs in a fixed order: results are bit-identical run
 *     to run (the reference's reruns are, tests/test_newton.py:102-114).
 */
#ifndef SNX_H
#define SNX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SNX_ABI_VERSION 1
#define SNX_F64 0
#define SNX_F32 1
#define SNX_DOT_BLOCKS 256 /* fixed partial count of every dot product */
#define SNX_CG_SLOT 8      /* doubles per CG state slot */

int snx_abi_version(void);
const char *snx_last_error(void);

/* Bytes of workspace the calls below need for nrows rows of p features, K
 * weighted classes (any of the row-pass calls).  The workspace must be
 * zero-filled once when allocated; calls leave its counters at zero. */
size_t snx_workspace_bytes(int dtype, int64_t nrows, int32_t p, int32_t K);

/* Row gather (the reference's dataset.take, dataset.py:90-97, 180-185):
 * X_out[r][0:ld_out] = X[rows[r]][0:ld_out]; labels_out[r] = labels[rows[r]]
 * (labels/labels_out nullable).  Materialises a sample S once so every later
 * pass streams contiguous rows through TMA tiles. */
int snx_gather_rows(int dtype, const void *X, int64_t ldx, const int32_t *labels,
                    const int64_t *rows, int64_t nrows, void *X_out, int64_t ld_out,
                    int32_t *labels_out, void *stream);

/* softmax.py:125-141 (data_objective/objective) + softmax.py:239-247
 * (predict/accuracy) over rows 0..nrows-1 of X, evaluated at
 * w_eff = w + alpha*dir (dir may be NULL; the line-search trial x + a*p of
 * newton.py:92 without materialising it).
 *   out[0] = sum_i (M_i + log alpha_i - lin_i)   (data loss)
 *   out[1] = ||w_eff||^2                          (for lam/2 ||x||^2)
 *   correct_out[0] (nullable) = #rows with argmax prob == label. */
int snx_objective(int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p, int32_t K,
                  const int32_t *labels, const double *w, const double *dir, double alpha,
                  double *out, int64_t *correct_out, void *ws, size_t ws_bytes, void *stream);

/* softmax.py:144-169 (data_gradient/gradient), sampling.py:84-87:
 *   G_out = scale * vec(X^T (E/alpha - onehot)) + lam * w
 * plus out[0..1] as snx_objective (the loss comes for free). */
int snx_objective_grad(int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p,
                       int32_t K, const int32_t *labels, const double *w, double scale,
                       double lam, double *out, double *G_out, void *ws, size_t ws_bytes,
                       void *stream);

/* snx_objective_grad plus the accuracy count of snx_objective (correct_out,
 * nullable) in the same pass: the Newton loop evaluates its first line-search
 * trial F(x + p) together with the gradient at x + p (newton.py:92-99). */
int snx_objective_grad_acc(int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p,
                           int32_t K, const int32_t *labels, const double *w, double scale,
                           double lam, double *out, int64_t *correct_out, double *G_out, void *ws,
                           size_t ws_bytes, void *stream);

/* softmax.py:224-240 class_probabilities / predict and :107-122 row_stats in
 * one row pass (each output nullable):
 *   probs_out[r*(K+1) + c] = E_rc / alpha_r (c < K), [K] = e^-M_r / alpha_r
 *   pred_out[r]  = argmax over the K+1 probabilities, first max wins
 *   stats_out[r*3 + 0..2] = (M_r, sum_c E_rc, linear part z_{r,y_r})  (labels needed) */
int snx_class_probabilities(int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p,
                            int32_t K, const int32_t *labels, const double *w, double *probs_out,
                            int32_t *pred_out, double *stats_out, void *ws, size_t ws_bytes,
                            void *stream);

/* softmax.py:181-195 (HessianOperator.__init__) on the sample rows S_H:
 * when rows != NULL the sample is X[rows] (gathered into Xs_out (ld_out) when
 * Xs_out != NULL; with Xs_out == NULL nothing is materialised and the product
 * is snx_hess_apply_rows -- fp64 data, K <= 9 only), else X itself is the
 * sample (the f = 1 identity, dataset.py:94-96).
 *   H_out[r*K + c] = h(a_r, x_c) = E_rc / alpha_r, stored in the X dtype. */
int snx_hess_prepare(int dtype, const void *X, int64_t ldx, const int64_t *rows, int64_t nrows,
                     int32_t p, int32_t K, const double *w, void *Xs_out, int64_t ld_out,
                     void *H_out, void *ws, size_t ws_bytes, void *stream);

/* softmax.py:197-210 (HessianOperator.apply), scale = n/|S_H| (sampling.py:82),
 * on the contiguous sample Xs prepared above:
 *   Hv_out = scale * vec(Xs^T (V.W - W.rowsum(V.W))) + lam * v,  V = Xs Q(v)
 * dots (nullable, 2*SNX_DOT_BLOCKS doubles): fixed-count partials of v.Hv and
 * v.v (the CG curvature test, cg.py:78).  skip (nullable): if *skip != 0 the
 * call is a no-op (device-side early exit of a captured CG loop). */
int snx_hess_apply(int dtype, const void *Xs, int64_t ldx, int64_t nrows, int32_t p, int32_t K,
                   const void *H, const double *v, double scale, double lam, double *Hv_out,
                   double *dots, const double *skip, void *ws, size_t ws_bytes, void *stream);

/* The gather-fused form of snx_hess_apply: the sample is rows[0..nrows) of X
 * (sorted int64 indices, duplicates allowed), read in place -- no X_S copy.
 * H comes from snx_hess_prepare(..., rows, ..., Xs_out = NULL, ...), which
 * fuses the same gather.  K <= 9 (snx_rowpass_fused != 0): the one-pass
 * cluster kernel (csrc/snx_cluster.cu) streams every sample row once per
 * product -- fp64 data, or f32 data widened to fp64 in shared memory (fp64
 * arithmetic); H is fp64 for both (rows may be NULL: all nrows rows). */
int snx_rowpass_fused(int dtype, int32_t p, int32_t K);
int snx_hess_apply_rows(int dtype, const void *X, int64_t ldx, const int64_t *rows,
                        int64_t nrows, int32_t p, int32_t K, const void *H, const double *v,
                        double scale, double lam, double *Hv_out, double *dots,
                        const double *skip, void *ws, size_t ws_bytes, void *stream);

/* Tensor-core variant of the two calls above for f32 data (the declared 1e-4
 * path; tcgen05 kind::f16 MMAs on a two-term bf16 split, see csrc/snx_tc.cu).
 * snx_hess_prepare_tc = snx_hess_prepare(SNX_F32, ...) plus the split of the
 * sample rows Xs (or X when rows == NULL):
 *   X1[r][j] = bf16(Xs[r][j]),  X2[r][j] = bf16(Xs[r][j] - X1[r][j])
 * as [nrows][ldb] bf16 arrays, ldb >= snx_tc_ld(p) (a multiple of 8); every
 * product of this sample reuses them. */
int64_t snx_tc_ld(int32_t p);
int snx_hess_prepare_tc(const float *X, int64_t ldx, const int64_t *rows, int64_t nrows,
                        int32_t p, int32_t K, const double *w, float *Xs_out, int64_t ld_out,
                        float *H_out, void *X1_out, void *X2_out, int64_t ldb, void *ws,
                        size_t ws_bytes, void *stream);

/* snx_hess_apply(SNX_F32, ...) on the tensor cores from the split sample. */
int snx_hess_apply_tc(const void *X1, const void *X2, int64_t ldb, int64_t nrows, int32_t p,
                      int32_t K, const float *H, const double *v, double scale, double lam,
                      double *Hv_out, double *dots, const double *skip, void *ws,
                      size_t ws_bytes, void *stream);

/* Wide classes (16 < K <= 128) on f32 data: the full-data passes of
 * snx_objective / snx_objective_grad on the tensor cores, reading the bf16
 * split of the rows (snx_tc_split: X1 = bf16(X), X2 = bf16(X - X1), [nrows][ldb]).
 * Same outputs and conventions as the SNX_F32 calls above. */
int snx_tc_split(const float *X, int64_t ldx, int64_t nrows, int32_t p, void *X1, void *X2,
                 int64_t ldb, void *stream);
int snx_objective_tc(const void *X1, const void *X2, int64_t ldb, int64_t nrows, int32_t p,
                     int32_t K, const int32_t *labels, const double *w, const double *dir,
                     double alpha, double *out, int64_t *correct_out, void *ws, size_t ws_bytes,
                     void *stream);
int snx_objective_grad_tc(const void *X1, const void *X2, int64_t ldb, int64_t nrows, int32_t p,
                          int32_t K, const int32_t *labels, const double *w, double scale,
                          double lam, double *out, double *G_out, void *ws, size_t ws_bytes,
                          void *stream);

/* Fixed-order dot product: out[0] = x . y (np.dot / np.linalg.norm**2).
 * out must hold 1 + SNX_DOT_BLOCKS doubles (out[1..] = block partials). */
int snx_dot(const double *x, const double *y, int64_t d, double *out, void *stream);

/* SNX_DOT_BLOCKS fixed-order block partials of x . y into part (the layout
 * snx_cg_update expects for its dots argument: [s.Hs partials | s.s partials]). */
int snx_dot_partials(const double *x, const double *y, int64_t d, double *part, void *stream);

/* x_out = x + alpha * p, rounded as numpy's `x + alpha * p` (no FMA):
 * newton.py:97 and the trial points of newton.py:92. */
int snx_axpy(const double *x, const double *p, double alpha, int64_t d, double *x_out,
             void *stream);

/* out = a*x + b*y with numpy rounding of `a * x + b * y` (two products, one
 * add, no FMA); the vector updates of Steihaug-CG (trust region). */
int snx_axpby(double a, const double *x, double b, const double *y, int64_t d, double *out,
              void *stream);

/* Finish a row-sharded product after the cross-rank sum:
 *   out = out + lam * v   (numpy rounding of `sum + lam * v`)
 * and, when dots != NULL, the SNX_DOT_BLOCKS-partials layout of snx_hess_apply
 * (v.out | v.v) for the CG update. */
int snx_finish_hv(const double *v, double lam, int64_t d, double *out, double *dots,
                  const double *skip, void *stream);

/* Device CG (cg.py:51-98).  state: (max_iters+2)*SNX_CG_SLOT + 2*SNX_DOT_BLOCKS
 * doubles (the tail is reduction scratch: r.r and s.s partials); slot t
 * holds the scalars entering iteration t: [rs, best_norm, done, iters,
 * converged, threshold, err, curvature].  Vectors r, s, p, p_best have d
 * entries.  snx_cg_init sets r = s = -g, p = 0, p_best = -g and slot 0; a
 * zero g finishes immediately (cg.py:61-62). */
int snx_cg_init(const double *g, int64_t d, double theta, int32_t max_iters,
                double *r, double *s, double *p, double *p_best, double *state,
                void *stream);

/* One CG iteration t after Hs = H s was written with its dot partials
 * (snx_hess_apply(..., dots, skip = &state slot t done flag)). */
int snx_cg_update(int32_t t, int32_t max_iters, int64_t d, const double *Hs,
                  const double *dots, double *r, double *s, double *p, double *p_best,
                  double *state, void *stream);

/* One CG iteration t with the one-pass product (K <= 9: snx_rowpass_fused):
 * equivalent to snx_hess_apply_rows(s -> Hs, skip = done flag of slot t) +
 * snx_cg_update(t, ...), with the product's finalize fused into the CG's first
 * kernel -- the curvature s.Hs = scale * sum_rows V.U + lam * s.s is formed from
 * per-cluster row sums of the product itself and the s.s partials snx_cg_init /
 * snx_cg_update leave in the state (so the iterates agree with the unfused
 * pair to rounding, not bitwise).  rows: NULL for the contiguous sample X. */
int snx_hess_apply_cg_rows(int dtype, const void *X, int64_t ldx, const int64_t *rows,
                           int64_t nrows, int32_t p, int32_t K, const void *H, double scale,
                           double lam, int32_t t, int32_t max_iters, double *r, double *s,
                           double *p_vec, double *p_best, double *Hs, double *state, void *ws,
                           size_t ws_bytes, void *stream);

/* Address of the "done" field of slot t (pass as snx_hess_apply's skip). */
const double *snx_cg_done_flag(const double *state, int32_t t);

/* Power iteration of the reference's estimate_lipschitz (bench.py:116-138),
 * one step after w = H v was written (snx_hess_apply(v -> w, skip = state+2)):
 *   rayleigh = v.w, ||w|| = sqrt(w.w); ||w|| == 0 -> estimate 0 and stop
 *   (sticky flag state[2]); else v = w / ||w||.
 * state: SNX_POWER_STATE doubles, zero-filled before the first step;
 * state[0] = current estimate (v.w of the last step), state[1] = ||w||. */
#define SNX_POWER_STATE (4 + 2 * SNX_DOT_BLOCKS)
int snx_power_step(double *v, const double *w, int64_t d, double *state, void *stream);

/* Column normalisation (normalize_columns, dataset.py:314-324):
 *   norms[j] = sqrt(sum_i X[i][j]^2)  (fixed-order; norms nullable)
 *   scale[j] = 1 / norms[j] if norms[j] > 0 else 1
 * ws: snx_colnorm_workspace_bytes(p) bytes of scratch. */
size_t snx_colnorm_workspace_bytes(int32_t p);
int snx_column_norms(int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p,
                     double *norms, double *scale, void *ws, size_t ws_bytes, void *stream);

/* Y[i][j] = X[i][j] * scale[j] for j < p, 0 for p <= j < ld (scale_columns,
 * dataset.py:109-118); Y may alias X. */
int snx_scale_columns(int dtype, const void *X, int64_t ldx, int64_t nrows, int32_t p,
                      int64_t ld, const double *scale, void *Y, int64_t ldy, void *stream);

/* ------------------------------------------------------------------ sparse
 * CSR feature storage (the reference's sparse DesignMatrix, dataset.py:21-147;
 * the paper's cuSPARSE path), fp64 only, K <= 32:
 *   CSR  indptr[n+1] (int64), indices[nnz] (int32 column ids), data[nnz]
 *   CSC  colptr[p+1] (int64), rowidx[nnz] (int32 row ids),    cdata[nnz]
 * (the CSC copy is the transpose; X^T R contracts column by column in a fixed
 * order, no atomics).  Same outputs and conventions as the dense calls;
 * ws: snx_csr_workspace_bytes(n, p, K) bytes (n = rows of the FULL dataset
 * for snx_csr_gather). */
size_t snx_csr_workspace_bytes(int64_t nrows, int32_t p, int32_t K);
int snx_csr_objective(const int64_t *indptr, const int32_t *indices, const double *data,
                      int64_t nrows, int32_t p, int32_t K, const int32_t *labels, const double *w,
                      const double *dir, double alpha, double *out, int64_t *correct_out,
                      void *ws, size_t ws_bytes, void *stream);
int snx_csr_objective_grad(const int64_t *indptr, const int32_t *indices, const double *data,
                           const int64_t *colptr, const int32_t *rowidx, const double *cdata,
                           int64_t nrows, int32_t p, int32_t K, const int32_t *labels,
                           const double *w, double scale, double lam, double *out, double *G_out,
                           void *ws, size_t ws_bytes, void *stream);
int snx_csr_class_probabilities(const int64_t *indptr, const int32_t *indices,
                                const double *data, int64_t nrows, int32_t p, int32_t K,
                                const int32_t *labels, const double *w, double *probs_out,
                                int32_t *pred_out, double *stats_out, void *ws, size_t ws_bytes,
                                void *stream);
/* normalize_columns on CSR storage (dataset.py:103-118, 314-324): norms[j] =
 * sqrt(sum of the column's squared stored values) from the CSC copy (norms
 * nullable), scale[j] = 1/norms[j] (1 for an empty column); then both copies
 * scaled: data_out = data * scale[indices], cdata_out = cdata * scale[column]
 * (col_scratch: nnz int32). */
int snx_csr_column_norms(const int64_t *colptr, const double *cdata, int32_t p, double *norms,
                         double *scale, void *stream);
int snx_csr_scale_columns(const int32_t *indices, const double *data, const int64_t *colptr,
                          const double *cdata, int64_t nnz, int32_t p, const double *scale,
                          double *data_out, double *cdata_out, int32_t *col_scratch,
                          void *stream);
/* The row sample S (sorted int64, duplicates allowed: sampling with
 * replacement) as its own CSR (s_indptr[m+1], entries in the order of the
 * source rows) and CSC (s_colptr[p+1], rows renumbered to sample positions,
 * a duplicated row weighted by its multiplicity); s_* capacities must hold
 * sum_r nnz(row S[r]) entries (dataset.py:90-97 take / sampling.py:79-80). */
int snx_csr_gather(const int64_t *indptr, const int32_t *indices, const double *data,
                   const int64_t *colptr, const int32_t *rowidx, const double *cdata,
                   int64_t nrows, int32_t p, const int64_t *rows, int64_t m, int64_t *s_indptr,
                   int32_t *s_indices, double *s_data, int64_t *s_colptr, int32_t *s_rowidx,
                   double *s_cdata, void *ws, size_t ws_bytes, void *stream);
/* softmax.py:181-195 on a (gathered) CSR sample: H_out[r*K + c] = h(a_r, x_c). */
int snx_csr_hess_prepare(const int64_t *indptr, const int32_t *indices, const double *data,
                         int64_t nrows, int32_t p, int32_t K, const double *w, double *H_out,
                         void *ws, size_t ws_bytes, void *stream);
/* softmax.py:197-210 on the CSR + CSC of the sample; dots / skip as snx_hess_apply. */
int snx_csr_hess_apply(const int64_t *indptr, const int32_t *indices, const double *data,
                       const int64_t *colptr, const int32_t *rowidx, const double *cdata,
                       int64_t nrows, int32_t p, int32_t K, const double *H, const double *v,
                       double scale, double lam, double *Hv_out, double *dots, const double *skip,
                       void *ws, size_t ws_bytes, void *stream);

/* ------------------------------------------------------------------ ingest
 * LIBSVM / svmlight text (dataset.py:242-293 load_libsvm), HOST memory:
 * snx_libsvm_scan parses `path` (whitespace tokens, blank lines skipped,
 * "<label> <idx>:<val> ..." with 1-based idx) and returns the sizes;
 * snx_libsvm_fetch copies the parse out (raw float labels[nrows], CSR
 * indptr[nrows+1], 0-based indices[nnz], data[nnz]).  Returns 2 on a parse
 * error ("line N: ..." in snx_last_error), 1 on an I/O error. */
int snx_libsvm_scan(const char *path, int64_t *nrows, int64_t *nnz, int64_t *max_index);
int snx_libsvm_fetch(const char *path, double *labels, int64_t *indptr, int32_t *indices,
                     double *data);

/* Steihaug-CG of the sub-sampled trust-region Newton variant (BASELINE config
 * #4; no reference counterpart -- oracle/trust_region.py steihaug_cg, N&W
 * Alg. 7.2), device resident.  state: (max_iters + 2) * SNX_CG_SLOT +
 * 4 * SNX_DOT_BLOCKS doubles; slot j = [rr, done, boundary, iters, model m,
 * tol]; snx_tr_init sets z = 0, r = g, d = -g and slot 0.  Iteration j:
 * snx_hess_apply(d -> Hd, dots = [d.Hd | d.d], skip = snx_cg_done_flag-style
 * &state[j * SNX_CG_SLOT + 1]) then snx_tr_update(j, ...) (radius: device
 * scalar).  The step is z; slot max_iters holds m(z), iterations, boundary. */
int snx_tr_init(const double *g, int64_t d, double theta, int32_t max_iters, double *z,
                double *r, double *dvec, double *state, void *stream);
int snx_tr_update(int32_t j, int32_t max_iters, int64_t d, const double *radius,
                  const double *Hd, const double *dots, double *z, double *r, double *dvec,
                  double *znew, double *state, void *stream);

/* Copy+convert host-layout helpers (device to device). */
int snx_pack_rows(int dtype, const double *src, int64_t nrows, int32_t p, void *dst,
                  int64_t ldd, void *stream);

/* ---- fp64 data with many classes (K = C-1 >= 17, any C: up to 4 classes
 * per lane in registers to K = 128, a loop variant beyond; the fast paths
 * above stop at K = 16).  The reference computes in fp64 for any C
 * (softmax.py:85-212); here the feature products are library DGEMMs (cuBLAS)
 * and the per-row softmax algebra is one warp per row (csrc/snx_wide64.cu).
 * X is row-major [n][ldx] fp64, weights class-major fp64 as everywhere.
 * Rows are processed in chunks of zrows; `scratch` holds
 * snx_wide_scratch_doubles(n, p, K, zrows) doubles (n = the rows of the call). */
int64_t snx_wide_scratch_doubles(int64_t n, int32_t p, int32_t K, int64_t zrows);
/* snx_objective on wide-class data: out = [data loss, ||w_eff||^2], w_eff =
 * w + alpha*dir (dir nullable); correct_out (nullable) = rows whose argmax
 * probability is their label (softmax.py:125-141, :224-247). */
int snx_wide_objective(const double *X, int64_t ldx, int64_t n, int32_t p, int32_t K,
                       const int32_t *labels, const double *w, const double *dir, double alpha,
                       double *out, long long *correct_out, double *scratch, int64_t zrows,
                       void *stream);
/* snx_objective_grad on wide-class data: G = scale * data_gradient + lam * w,
 * out = [data loss, ||w||^2] (softmax.py:144-169). */
int snx_wide_objective_grad(const double *X, int64_t ldx, int64_t n, int32_t p, int32_t K,
                            const int32_t *labels, const double *w, double scale, double lam,
                            double *out, double *G, double *scratch, int64_t zrows,
                            void *stream);
/* snx_hess_prepare on wide-class data (softmax.py:181-195): with rows != NULL
 * the sample X[rows] is gathered into Xs_out (ld_out); H_out[r*K + c] = h_rc. */
int snx_wide_hess_prepare(const double *X, int64_t ldx, const int64_t *rows, int64_t nrows,
                          int32_t p, int32_t K, const double *w, double *Xs_out, int64_t ld_out,
                          double *H_out, double *scratch, int64_t zrows, void *stream);
/* snx_hess_apply on wide-class data (softmax.py:197-212): out = scale *
 * X_S^T U + lam * v, U = h*V - h*rowsum(h*V), V = X_S v^T; dots / skip as in
 * snx_hess_apply (with *skip != 0 the result and dots are left untouched). */
int snx_wide_hess_apply(const double *Xs, int64_t lds, int64_t m, int32_t p, int32_t K,
                        const double *H, const double *v, double scale, double lam, double *out,
                        double *dots, const double *skip, double *scratch, int64_t zrows,
                        void *stream);
/* snx_class_probabilities on wide-class data (same outputs, each nullable). */
int snx_wide_class_probabilities(const double *X, int64_t ldx, int64_t n, int32_t p, int32_t K,
                                 const int32_t *labels, const double *w, double *probs_out,
                                 int32_t *pred_out, double *stats_out, double *scratch,
                                 int64_t zrows, void *stream);
/* snx_class_probabilities on f32 data with C = 18..129: each chunk of zrows
 * rows is widened to fp64 (exact) and goes through the fp64 path above, so the
 * results are the fp64 arithmetic on the f32-rounded data; scratch holds
 * snx_wide_f32_scratch_doubles(n, p, K, zrows) doubles. */
int64_t snx_wide_f32_scratch_doubles(int64_t n, int32_t p, int32_t K, int64_t zrows);
int snx_wide_class_probabilities_f32(const float *X, int64_t ldx, int64_t n, int32_t p,
                                     int32_t K, const int32_t *labels, const double *w,
                                     double *probs_out, int32_t *pred_out, double *stats_out,
                                     double *scratch, int64_t zrows, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SNX_H */
