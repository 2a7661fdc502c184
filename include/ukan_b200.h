/*
 * ukan_b200.h — C ABI of the B200 (sm_100a) matrix-form B-spline KAN / UKAN hot path.
 *
 * This is the drop-in boundary of the rebuild of arXiv 2408.11200's accelerated path
 * (reference: /root/reference/pkg/src/ukan, a float64 NumPy implementation).  Every entry
 * point below replaces one fused graph op (or a fused group of them) of the reference's
 * `ukan.layers` module; the reference-side binding (a ctypes stub) is in INTEGRATION.md and
 * the Python mirror of the reference API is `paper_2408_11200_b200.layers`.
 *
 * Conventions
 *  - all tensor pointers are DEVICE pointers, caller-owned (allocated by the caller, e.g. by
 *    torch's caching allocator), row-major and contiguous; no allocation happens inside;
 *  - `stream` is a cudaStream_t passed as void*; all work is enqueued on it; no host
 *    synchronisation happens inside any call except where documented (ukan_ukan_build_keys);
 *  - return value: 0 = ok, < 0 = argument error (UKAN_E_*), > 0 = a cudaError_t;
 *  - every call is re-entrant and stateless (workspace is passed in), and deterministic:
 *    identical inputs give bitwise identical outputs run to run (no float atomics);
 *  - storage is fp32; grid indices are computed in fp64 with the reference's exact
 *    expression order and are bit-exact against it; backward reductions are fp64.
 */
#ifndef UKAN_B200_H
#define UKAN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define UKAN_OK 0
#define UKAN_E_ARG (-1)        /* bad shape / size / pointer                         */
#define UKAN_E_DEGREE (-2)     /* spline degree outside [0, 10]  (bspline.py:21,72)   */
#define UKAN_E_GRID (-3)       /* g_min >= g_max or G < 1        (layers.py:152-153)  */
#define UKAN_E_WORKSPACE (-4)  /* workspace too small                                  */
#define UKAN_E_CAPACITY (-5)   /* data-dependent capacity exceeded (see ukan_ukan_*)   */

#define UKAN_MAX_DEGREE 10

/* Library version (major*10000 + minor*100 + patch). */
int ukan_version(void);

/* Number of kernels this library has launched in the process so far (monotonic; for
 * benchmarks and tests that check the native path actually ran). */
int64_t ukan_launch_count(void);

/* Exact K x K basis matrix (K = k+1) of the uniform degree-k B-spline in monomial form,
 * row i = coefficient of u^i, column j = window slot j; computed by the Cox-de Boor recursion
 * in exact rational arithmetic and rounded once to double.  Replaces
 * bspline.basis_matrix (bspline.py:24-80).  Host function; M_out has K*K doubles. */
int ukan_basis_matrix(int k, double* M_out);

/* ---------------------------------------------------------------------------------------
 * KAN layer (bounded grid).  Replaces kan_forward (layers.py:304-318) =
 *   _kan_locate (294-301) + span_gather (57-75) + basis_features (40-54) +
 *   edge_combine (78-105) [+ silu base branch (316-317)].
 * x [B, d_in], coeffs [d_in, G+k, d_out], scale [d_in, d_out], base_weight [d_in, d_out]
 * (nullable = no base branch), y [B, d_out].
 * ------------------------------------------------------------------------------------- */
int ukan_kan_forward(const float* x, const float* coeffs, const float* scale,
                     const float* base_weight, float* y,
                     int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k,
                     double g_min, double g_max, int32_t* err_flag, void* stream);

/* Same as ukan_kan_forward with a caller-provided device workspace (needed when the batch is
 * too small to fill the GPU and d_in is split across CTAs: fp32 partial outputs, reduced in
 * fixed order).  ukan_kan_forward itself takes it from a stream-ordered allocation. */
int64_t ukan_kan_forward_workspace_size(int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k);
int ukan_kan_forward_ws(const float* x, const float* coeffs, const float* scale,
                        const float* base_weight, float* y,
                        int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k,
                        double g_min, double g_max, int32_t* err_flag,
                        void* workspace, int64_t workspace_bytes, void* stream);

/* Backward of ukan_kan_forward given gy = dL/dy [B, d_out].  Replaces the bwd closures of
 * span_gather (layers.py:67-70), basis_features (44-46), edge_combine (84-88), clamp
 * (tensor.py:330-333) and the base branch.  dx [B, d_in] may be NULL (x not a recorded node,
 * tensor.py:455-456); dbase_weight must be NULL iff base_weight is NULL.  dcoeffs / dscale /
 * dbase_weight are OVERWRITTEN (not accumulated).  fp64 products and accumulators. */
int ukan_kan_backward(const float* x, const float* coeffs, const float* scale,
                      const float* base_weight, const float* gy,
                      float* dx, float* dcoeffs, float* dscale, float* dbase_weight,
                      int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k,
                      double g_min, double g_max, void* stream);

/* Same as ukan_kan_backward with an explicit caller workspace (stream-ordered, no allocation
 * inside; the size query covers every kernel choice). */
int64_t ukan_kan_backward_workspace_size(int64_t B, int64_t d_in, int64_t d_out, int64_t G,
                                         int k);
int ukan_kan_backward_ws(const float* x, const float* coeffs, const float* scale,
                         const float* base_weight, const float* gy, float* dx, float* dcoeffs,
                         float* dscale, float* dbase_weight, int64_t B, int64_t d_in,
                         int64_t d_out, int64_t G, int k, double g_min, double g_max,
                         void* workspace, int64_t workspace_bytes, void* stream);

/* Split form of the backward: ukan_kan_backward_prep depends on x only and fills the sorted
 * per-chunk records of the FP64 tensor-core path into the workspace, so a caller can run it
 * early on another stream (overlapping the layers above); *prepared (host) is set to 1 when it
 * launched the prep, 0 when that path does not apply (nothing done).  Pass flags = *prepared to
 * ukan_kan_backward_ws2 with the same workspace (after the prep's stream work) to reuse them;
 * flags = 0 is ukan_kan_backward_ws. */
int ukan_kan_backward_prep(const float* x, const float* base_weight, int64_t B, int64_t d_in,
                           int64_t d_out, int64_t G, int k, double g_min, double g_max,
                           void* workspace, int64_t workspace_bytes, int32_t* prepared,
                           void* stream);
int ukan_kan_backward_ws2(const float* x, const float* coeffs, const float* scale,
                          const float* base_weight, const float* gy, float* dx, float* dcoeffs,
                          float* dscale, float* dbase_weight, int64_t B, int64_t d_in,
                          int64_t d_out, int64_t G, int k, double g_min, double g_max,
                          void* workspace, int64_t workspace_bytes, int flags, void* stream);

/* Feature-sliced backward for data-parallel callers (k = 3, G <= 64, no base branch,
 * d_out >= 64 and a multiple of 4: ukan_kan_backward_part_supported returns 1).  After
 * ukan_kan_backward_prep has filled `workspace` for the WHOLE layer (prepared = 1), each call
 * computes, for features [i_lo, i_hi) only: what & 1 -> dcoeffs / dscale rows of those features
 * (written), what & 2 -> dx[:, i_lo:i_hi) (written; dx is the full [B, d_in] buffer).  The
 * slices of one layer are independent, so a caller can all-reduce a finished dcoeffs slice while
 * the next slice is computed (SURVEY 8e E1 bucketing).  Results equal ukan_kan_backward_ws2
 * bitwise. */
int ukan_kan_backward_part_supported(int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k);
int ukan_kan_backward_part(const float* coeffs, const float* scale, const float* gy, float* dx,
                           float* dcoeffs, float* dscale, int64_t B, int64_t d_in, int64_t d_out,
                           int64_t G, int k, double g_min, double g_max, void* workspace,
                           int64_t workspace_bytes, int64_t i_lo, int64_t i_hi, int what, void* stream);

/* Grid location only (for parity tests / tooling): cell [B, d_in] int32 and u [B, d_in]
 * double exactly as layers.py:296-300 compute them. */
int ukan_kan_locate(const float* x, int32_t* cell, double* u,
                    int64_t B, int64_t d_in, int64_t G, double g_min, double g_max,
                    void* stream);

/* Naive comparison arm (naive_kan_forward, layers.py:321-370): all G+k bases per input by the
 * Cox-de Boor recursion over the full knot vector, dotted with the whole coefficient table.
 * tmp [B, d_in, d_out] receives sum_s B_s C[i,s,o] (needed by the backward).  The backward
 * writes dcoeffs / dscale only (no dx, as the reference arm). */
int ukan_kan_naive_forward(const float* x, const float* coeffs, const float* scale, float* y,
                           float* tmp, int64_t B, int64_t d_in, int64_t d_out, int64_t G, int k,
                           double g_min, double g_max, void* stream);
int ukan_kan_naive_backward(const float* x, const float* scale, const float* tmp, const float* gy,
                            float* dcoeffs, float* dscale, int64_t B, int64_t d_in, int64_t d_out,
                            int64_t G, int k, double g_min, double g_max, void* stream);

/* Forward tangent (JVP) of the KAN layer and its backward (the tangent channel of
 * basis_features / edge_combine / clamp / silu, layers.py:49-53, 91-104, tensor.py:236-241,
 * 336-337, used by pinn_loss, tasks.py:153-166).  ty = (dy/dx) . tx per sample.  The backward
 * WRITES the gradients of sum(ty * gt): dx (tangent path only, nullable), dtx (nullable),
 * dcoeffs, dscale, dbase_weight (iff base_weight).  fp64 evaluation and sums, deterministic. */
int ukan_kan_jvp_forward(const float* x, const float* tx, const float* coeffs, const float* scale,
                         const float* base_weight, float* ty, int64_t B, int64_t d_in, int64_t d_out,
                         int64_t G, int k, double g_min, double g_max, void* stream);
int ukan_kan_jvp_backward(const float* x, const float* tx, const float* coeffs, const float* scale,
                          const float* base_weight, const float* gt, float* dx, float* dtx,
                          float* dcoeffs, float* dscale, float* dbase_weight, int64_t B, int64_t d_in,
                          int64_t d_out, int64_t G, int k, double g_min, double g_max, void* stream);

/* ---------------------------------------------------------------------------------------
 * UKAN layer (unbounded grid, coefficient generator).  Replaces ukan_forward
 * (layers.py:254-291), _cg_eval (232-243) and positional_encoding (112-123).
 *
 * Key order: the unique (feature, group) keys are stored FEATURE-MAJOR, sorted by
 * (f, group).  The reference sorts the int64 key group*d_in+f (np.unique, layers.py:275);
 * both orders hold the same set.  Feature-major order makes the window of cell g_id the
 * K consecutive rows  base = idx(f, g_id div K)*K + (g_id mod K)  of the flat
 * [n_u*K, d_out] coefficient table, because (f, g+1) always directly follows (f, g).
 * ------------------------------------------------------------------------------------- */

/* Bytes of device workspace ukan_ukan_build_keys needs for a key capacity of max_keys. */
int64_t ukan_ukan_keys_workspace_size(int64_t B, int64_t d_in, int64_t max_keys);

/* Locate every x[b, f] (g_id = floor(x * (1/delta_g)), layers.py:261-263), collect the unique
 * (f, group) and (f, group+1) keys (layers.py:266-278), sort them feature-major, and write
 *   key_f[n_u] int32 (feature), key_g[n_u] int64 (group), seg_start[d_in+1] int32 (row
 *   segment of each feature in key order), base_row[B, d_in] int32 (first of the K table rows
 *   of cell g_id: idx(f, g_id div K)*K + g_id mod K), and on the host *n_unique_host and
 *   *max_rows_host (largest per-feature key count).
 * Capacity: key_f / key_g must hold max_keys entries; UKAN_E_CAPACITY is returned when more
 * unique keys exist (retry with a larger max_keys).  *nonfinite_host = 1 when any input is
 * NaN/inf (the reference raises DomainError, layers.py:257-258) and = 2 when |g_id| >= 2^42
 * (outside the packed-key range).  This is the one call that synchronises the stream, because
 * n_u is data dependent. */
int ukan_ukan_build_keys(const float* x, int64_t B, int64_t d_in, int k, double delta_g,
                         int32_t* key_f, int64_t* key_g, int32_t* seg_start, int32_t* base_row,
                         int64_t max_keys, void* workspace, int64_t workspace_bytes,
                         int64_t* n_unique_host, int64_t* max_rows_host,
                         int32_t* nonfinite_host, void* stream);

/* Coefficient-generator input rows: inp[n_u, d_femb + d_pe] = [emb[f] || PE(group)] in fp64
 * (the PE evaluated and KEPT in fp64 as the reference does, layers.py:112-123, 238-240; the
 * embedding is widened exactly).  The whole CG chain stays fp64 between its GEMMs. */
int ukan_ukan_cg_input(const int32_t* key_f, const int64_t* key_g, const float* emb,
                       double* inp, int64_t n_u, int64_t d_femb, int64_t d_pe, void* stream);

/* Dense row-major GEMM family used by the CG MLP (layers.py:241-242, tensor.py:189-197):
 *   C[M,N] = act(A[M,K] @ B[K,N] + bias[N])         (ukan_gemm_bias_act, act 0=none 1=silu,
 *                                                     pre_out optional: pre-activation)
 *   C[M,N] = A[M,K] @ B[N,K]^T                       (ukan_gemm_nt)
 *   C[M,N] = A[K,M]^T @ B[K,N], bias_grad[N] = sum_K B (ukan_gemm_tn, fp64 split-K)
 * fp32 storage; ukan_gemm_nt / ukan_gemm_tn accumulate in fp64 (gradient GEMMs). */
int ukan_gemm_bias_act(const float* A, const float* Bm, const float* bias, float* C,
                       float* pre_out, int64_t M, int64_t N, int64_t K, int act, void* stream);
int ukan_gemm_nt(const float* A, const float* Bm, float* C, int64_t M, int64_t N, int64_t K,
                 void* stream);
int ukan_gemm_tn(const float* A, const float* Bm, float* C, float* colsum_B,
                 int64_t M, int64_t N, int64_t K, void* stream);

/* Diagnostic, not used by the product path: C[M,N] = A[K,M]^T @ B[K,N] on the tcgen05 tensor
 * cores in the 3xTF32 form SURVEY 8c C5 proposed for the CG gradient GEMMs (round-to-nearest
 * tf32 operand splits, fp64 promotion per 32-wide K chunk, split-K over 4096 rows summed in
 * fp64).  Kept so tests can measure why ukan_gemm_tn runs on FP64 DMMA instead (the fp32 tensor
 * core accumulator keeps ~22 bits).  M, N multiples of 4; A, B 16-byte aligned. */
int ukan_gemm_tn_tf32x3_probe(const float* A, const float* Bm, float* C, int64_t M, int64_t N,
                              int64_t K, void* stream);

/* d(silu): dpre = dH * (s + pre*s*(1-s)), s = sigmoid(pre)  (tensor.py:232-233), fp64. */
int ukan_silu_backward(const double* pre, const double* dH, double* dpre, int64_t n, void* stream);

/* GEMM on the FP64 tensor cores (mma.sync m8n8k4 f64, fp64 products and sums, split-K partials
 * reduced in fixed order) with fp32 or fp64 operands (dtype UKAN_F32 / UKAN_F64, widened exactly):
 *   op 0 (NN): A [M,K], B [K,N];  op 1 (NT): A [M,K], B [N,K];  op 2 (TN): A [K,M], B [K,N].
 * Epilogue in fp64: v = A.B + bias[n] (bias nullable); pre_out = v; v = silu(v) if act;
 * C64 = v; C32 = (float)v (each output nullable, at least one given).  colsum_B (op 2 only,
 * nullable) = column sums of B in fp64 (the bias gradient of a TN weight-gradient GEMM).
 * Used for the CG MLP (layers.py:241-242, tensor.py:189-197) in fp64. */
#define UKAN_F32 0
#define UKAN_F64 1
int ukan_gemm_f64(int op, const void* A, int a_dtype, const void* Bm, int b_dtype, const float* bias,
                  int act, double* pre_out, float* C32, double* C64, float* colsum_B, int64_t M,
                  int64_t N, int64_t K, void* stream);

/* Embedding gradient: d_emb[f, :] = sum over the rows of feature f (seg_start[f] ..
 * seg_start[f+1]) of dinp[r, :d_femb] (gather_rows bwd, tensor.py:265-268; dinp fp64), fp64 sum
 * in key order (deterministic). */
int ukan_ukan_emb_backward(const int32_t* seg_start, const double* dinp, float* d_emb,
                           int64_t d_in, int64_t d_femb, int64_t d_cg_in, void* stream);

/* UKAN spline forward over the generated table: table [n_u*K, d_out] (slot-major view of the
 * CG output [n_u, K*d_out]), base_row from ukan_ukan_build_keys. */
int ukan_ukan_forward(const float* x, const int32_t* base_row, const float* table,
                      const float* scale, float* y, int64_t B, int64_t d_in, int64_t d_out,
                      int k, double delta_g, void* stream);

/* UKAN spline backward: dtable [n_u*K, d_out] (overwritten), dscale [d_in, d_out]
 * (overwritten), dx [B, d_in] (nullable; layers.py:264: du/dx = 1/delta_g, no clamp).
 * seg_start gives each feature's key segment.  fp64 products / accumulators; the workspace
 * holds the fp64 accumulator (see ukan_ukan_backward_workspace_size). */
int64_t ukan_ukan_backward_workspace_size(int64_t B, int64_t d_in, int64_t d_out, int64_t n_u,
                                          int k);
int ukan_ukan_backward(const float* x, const int32_t* base_row, const int32_t* seg_start,
                       const float* table, const float* scale, const float* gy,
                       float* dx, float* dtable, float* dscale,
                       int64_t B, int64_t d_in, int64_t d_out, int64_t n_u, int k,
                       double delta_g, void* workspace, int64_t workspace_bytes,
                       void* stream);

/* ukan_ukan_backward with the key build's *max_rows_host: dense layers take
 * ukan_ukan_backward_dense, the others the sorted-merge path with max_rows bounding the per-feature
 * row histogram (which admits large batches to the per-feature sorted sweep). */
int64_t ukan_ukan_backward2_workspace_size(int64_t B, int64_t d_in, int64_t d_out, int64_t n_u,
                                           int64_t max_rows, int k);
int ukan_ukan_backward2(const float* x, const int32_t* base_row, const int32_t* seg_start,
                        const float* table, const float* scale, const float* gy,
                        float* dx, float* dtable, float* dscale,
                        int64_t B, int64_t d_in, int64_t d_out, int64_t n_u, int64_t max_rows, int k,
                        double delta_g, void* workspace, int64_t workspace_bytes, void* stream);

/* Dense UKAN forward (max_rows <= 67, k = 3, d_out >= 128): ukan_ukan_forward's result through the
 * TMEM-gather forward over the features' table segments.  Size 0 = the layer does not qualify. */
int64_t ukan_ukan_forward_dense_workspace_size(int64_t B, int64_t d_in, int64_t d_out, int64_t max_rows, int k);
int ukan_ukan_forward_dense(const float* x, const int32_t* base_row, const int32_t* seg_start,
                            const float* table, const float* scale, float* y, int64_t B, int64_t d_in,
                            int64_t d_out, int64_t max_rows, int k, double delta_g, void* workspace,
                            int64_t workspace_bytes, void* stream);

/* Dense UKAN layers (every feature's virtual table has max_rows <= 67 rows, k = 3, d_out >= 64,
 * d_out % 4 == 0): the same gradients as ukan_ukan_backward (layers.py:254-291 backward) on the
 * KAN FP64 tensor-core backward — cell-sorted records per (feature, 256-sample chunk), the banded
 * DMMA table-gradient sweep writing each feature's row segment of dtable (or, for segments of
 * fewer than 24 rows, the sorted-merge sweep of ukan_ukan_backward), and the DMMA dx.
 * max_rows is the *max_rows_host of ukan_ukan_build_keys.  The workspace size is 0 when the layer
 * does not qualify (call ukan_ukan_backward then).  Deterministic. */
int64_t ukan_ukan_backward_dense_workspace_size(int64_t B, int64_t d_in, int64_t d_out, int64_t n_u,
                                                int64_t max_rows, int k);
int ukan_ukan_backward_dense(const float* x, const int32_t* base_row, const int32_t* seg_start,
                             const float* table, const float* scale, const float* gy,
                             float* dx, float* dtable, float* dscale,
                             int64_t B, int64_t d_in, int64_t d_out, int64_t n_u, int64_t max_rows, int k,
                             double delta_g, void* workspace, int64_t workspace_bytes, void* stream);

/* Forward tangent of the UKAN spline over the generated table (u = x/dg - g_id carries tx/dg,
 * layers.py:264; the table has no tangent) and its backward: dx (tangent share, nullable), dtx
 * (nullable), dtable [n_u*K, d_out] (written), dscale (written).  Same key layout as above. */
int ukan_ukan_jvp_forward(const float* x, const float* tx, const int32_t* base_row, const float* table,
                          const float* scale, float* ty, int64_t B, int64_t d_in, int64_t d_out, int k,
                          double delta_g, void* stream);
int ukan_ukan_jvp_backward(const float* x, const float* tx, const int32_t* base_row,
                           const int32_t* seg_start, const float* table, const float* scale,
                           const float* gt, float* dx, float* dtx, float* dtable, float* dscale,
                           int64_t B, int64_t d_in, int64_t d_out, int64_t n_u, int k, double delta_g,
                           void* stream);

/* ---------------------------------------------------------------------------------------
 * Training-step kernels (train.py:142-150, optim.py:31-54, tensor.py:368-400).
 * ------------------------------------------------------------------------------------- */

/* Mean softmax cross-entropy over logits [n, c] and int64 labels [n] (tensor.py:377-400):
 * loss points at 1 + n device doubles; loss[0] = sum of this shard's row losses / n_global
 * (loss[1..n] is per-row scratch); dlogits = grad_scale * (softmax - onehot) / n_global.
 * A label outside [0, c) is never dereferenced: its row loss is NaN, its gradient row 0, and
 * bit 1 (value 2) is OR-ed into *err_flag (device int32, nullable) so the caller can raise the
 * reference's IndexError (tensor.py:388-392) at its next host read. */
int ukan_softmax_xent(const float* logits, const int64_t* labels, double* loss,
                      float* dlogits, int64_t n, int64_t c, int64_t n_global,
                      double grad_scale, int32_t* err_flag, void* stream);

/* Mean squared error over pred/target [n] elements (tensor.py:368-374): loss points at
 * 1 + n device doubles (loss[1..] is scratch: per-256-element partial sums), loss[0] = sum (pred-target)^2
 * / n_global; dpred = 2*(pred-target)/n_global. */
int ukan_mse(const float* pred, const float* target, double* loss, float* dpred,
             int64_t n, int64_t n_global, void* stream);

/* One Adam step with coupled L2 over a flat fp32 parameter buffer (optim.py:31-54):
 *   g += wd*p; m = b1*m + (1-b1)*g; v = b2*v + (1-b2)*g*g;
 *   p -= lr * (m/bc1) / (sqrt(v/bc2) + eps),  bc_i = 1 - b_i^t.
 * guard (nullable, device double): when *guard is not finite the update is skipped, so a
 * diverged loss leaves the parameters untouched without a host round trip (the reference
 * raises DivergedError before updating, train.py:143-144). */
int ukan_adam_step(float* p, const float* g, float* m, float* v, int64_t n, double lr,
                   double beta1, double beta2, double eps, double weight_decay, int64_t t,
                   const double* guard, void* stream);

/* SGD step p -= lr*g (optim.py:18-21), same guard semantics. */
/* Graph-replayable Adam (for a step captured as a CUDA graph): unless *guard is non-finite
 * (skipped step, counter unchanged, as the reference raises before state.t += 1) increments the
 * device step counter *t, computes the bias corrections 1 - beta^t into bc[2] (device), reads the learning
 * rate from *lr (device) and updates as ukan_adam_step.  All of t, bc, lr are device pointers. */
int ukan_adam_step_dev(float* p, const float* g, float* m, float* v, int64_t n, const double* lr,
                       double beta1, double beta2, double eps, double weight_decay, int64_t* t,
                       double* bc, const double* guard, void* stream);
int ukan_sgd_step(float* p, const float* g, int64_t n, double lr, const double* guard,
                  void* stream);

/* Fill helper: sets n fp32 values to `value` (used to zero flat gradient buffers). */
int ukan_fill_f32(float* p, int64_t n, float value, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* UKAN_B200_H */
