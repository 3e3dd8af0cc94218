/* brk.h — C-ABI of libbrk_sm100.so, the B200 (sm_100a) batch-reduce GEMM
 * engine and the DL primitives built on it.
 *
 * The reference (arxiv 1906.06440, package `brkernels`, pure Python/NumPy)
 * has no native boundary; these entry points are what its Python operator
 * API binds through ctypes.  Each function cites the
 * reference interface it replaces.
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless stated; the caller owns memory.
 *  - Every call is stream-ordered on `stream` (a cudaStream_t, may be NULL)
 *    and never synchronises the device.
 *  - Return 0 (BRK_OK) on success, BRK_ERR_CONTRACT (1) for a shape / layout
 *    contract violation (the Python shim maps it to BrgemmError/LayoutError),
 *    BRK_ERR_CUDA (2) for a CUDA error.  brk_last_error() returns the
 *    thread-local message of the last failure.
 *  - dtype codes: BRK_F32 / BRK_BF16 storage; compute codes BRK_COMPUTE_TF32
 *    (kind::tf32 tensor cores) / BRK_COMPUTE_BF16 (kind::f16, bf16 inputs);
 *    accumulation is always fp32 in TMEM.
 */
#ifndef BRK_H_
#define BRK_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define BRK_API __attribute__((visibility("default")))
#else
#define BRK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define BRK_OK 0
#define BRK_ERR_CONTRACT 1
#define BRK_ERR_CUDA 2

#define BRK_F32 0
#define BRK_BF16 1

#define BRK_COMPUTE_TF32 0
#define BRK_COMPUTE_BF16 1

/* Library / device information. */
BRK_API const char* brk_last_error(void);
BRK_API int brk_version(void);
/* Number of kernel launches issued by this library since load (host counter). */
BRK_API uint64_t brk_launch_count(void);

/* ---------------------------------------------------------------------------
 * BRGEMM, address variant.   Replaces brkernels.brgemm.brgemm
 * (reference pkg/src/brkernels/brgemm.py:260-293) and, with batch=1 per job,
 * brkernels.brgemm.batched_gemm (brgemm.py:340-353).
 *
 * For each job j in [0, n_jobs):
 *   C_j = beta*C_j + alpha * sum_{i<batch} B_ji @ A_ji     (reference view)
 * a_ptrs/b_ptrs: device arrays of n_jobs*batch block addresses (job-major);
 * c_ptrs: device array of n_jobs output block addresses.
 * Block shapes: A (k, m) row stride lda; B (n, k) row stride ldb; C (n, m)
 * row stride ldc (brgemm.py:5-15).  The accumulator for one C block stays in
 * TMEM for the whole batch; C is read (beta != 0) and written once.
 * ------------------------------------------------------------------------- */
BRK_API int brk_brgemm_addr(const void* const* a_ptrs, const void* const* b_ptrs, void* const* c_ptrs,
                    int n_jobs, int m, int n, int k, int batch, int64_t lda, int64_t ldb,
                    int64_t ldc, float alpha, float beta, int in_dtype, int out_dtype,
                    int compute, void* stream);
/* The address variant with registered views: a_view (a_view_elems elements) and b_view
 * (b_view_elems) are allocations that hold the A / B blocks.  The kernel turns each entry's
 * pointers into (row, column) coordinates of a 2-d view of its allocation and fetches blocks
 * that lie inside it with TMA (bf16); entries outside the views take the gather path, as in
 * brk_brgemm_addr.  Results are identical to brk_brgemm_addr. */
BRK_API int brk_brgemm_addr_views(const void* const* a_ptrs, const void* const* b_ptrs, void* const* c_ptrs,
                                  const void* a_view, int64_t a_view_elems, const void* b_view,
                                  int64_t b_view_elems, int n_jobs, int m, int n, int k, int batch, int64_t lda,
                                  int64_t ldb, int64_t ldc, float alpha, float beta, int in_dtype,
                                  int out_dtype, int compute, void* stream);

/* Grouped address-variant BRGEMM with general block strides and a fused
 * epilogue — the batch-list interface the FC/LSTM/conv drivers use for block
 * factors the TMA engine does not serve (reference drivers fc.py:139-160,
 * lstm.py:268-317, cnn.py:290-320 issue one brgemm per output block; here all
 * output blocks of a pass go in one launch).
 *   A_ji element (kk, col) at a_ptrs[j*batch+i][kk*a_sk + col*a_sm]
 *   B_ji element (row, kk) at b_ptrs[j*batch+i][row*b_sn + kk*b_sk]
 *   C_j  element (row, col) at c_ptrs[j][row*ldc + col]
 *   C_j = act(alpha*sum_i B_ji@A_ji + beta*C_j + bias[bias_offs[j]+col]) * (mask_j > 0)
 * act: 0 identity, 1 relu, 2 sigmoid.  bias / mask_ptrs may be NULL; mask_j
 * has the layout and dtype of C_j.  All tables are device arrays. */
typedef struct brk_grouped_desc {
  int n_jobs, m, n, k, batch;
  int64_t a_sk, a_sm, b_sn, b_sk, ldc;
  float alpha, beta;
  int in_dtype, out_dtype, compute;
  const void* const* a_ptrs;
  const void* const* b_ptrs;
  void* const* c_ptrs;
  const float* bias;
  const int64_t* bias_offs;
  int act;
  const void* const* mask_ptrs;
} brk_grouped_desc;

BRK_API int brk_brgemm_grouped(const brk_grouped_desc* desc, void* stream);

/* BRGEMM, offset variant (north star; no reference function — equivalent to
 * the address variant with A_ji = a_base + a_offs[j*batch+i] elements). */
BRK_API int brk_brgemm_offs(const void* a_base, const void* b_base, const int64_t* a_offs,
                    const int64_t* b_offs, void* const* c_ptrs, int n_jobs, int m, int n, int k,
                    int batch, int64_t lda, int64_t ldb, int64_t ldc, float alpha, float beta,
                    int in_dtype, int out_dtype, int compute, void* stream);

/* BRGEMM, stride variant.  Replaces brkernels.brgemm.brgemm_strided
 * (brgemm.py:296-337): A_ji = a_base + j*jstride_a + i*stride_a elements,
 * likewise B; C_j = c_base + j*jstride_c elements. */
BRK_API int brk_brgemm_stride(const void* a_base, const void* b_base, int64_t stride_a, int64_t stride_b,
                      void* c_base, int n_jobs, int64_t jstride_a, int64_t jstride_b,
                      int64_t jstride_c, int m, int n, int k, int batch, int64_t lda, int64_t ldb,
                      int64_t ldc, float alpha, float beta, int in_dtype, int out_dtype,
                      int compute, void* stream);

/* ---------------------------------------------------------------------------
 * Fully-connected layer passes on the reference's blocked layouts
 * (fc.py:99-163; tensor.py:143-158, 237-247):
 *   x, dx, mask : [N/b_n][C/b_c][b_n][b_c]      w : [K/b_k][C/b_c][b_c][b_k]
 *   y, dz       : [N/b_n][K/b_k][b_n][b_k]      dw: like w, fp32
 * Engine path: bf16 storage, b_n=b_c=b_k=64, N, C, K multiples of 128.
 * ------------------------------------------------------------------------- */
/* Replaces brkernels.fc.fc_forward (fc.py:99-163): y = act(W x + bias);
 * act: 0 identity, 1 relu, 2 sigmoid (fc.py:29-40); bias (fp32, K) may be NULL. */
BRK_API int brk_fc_fwd(const void* x, const void* w, const float* bias, void* y, int N, int C, int K,
                       int b_n, int b_c, int b_k, int act, int dtype, void* stream);
/* Backward-data (north star): dx = (W^T dz) * (mask > 0); mask may be NULL.
 * colsum_ws (may be NULL): fp32 [N/32][C] column-sum partials of the stored dx
 * (the next weight update reduces them into that layer's bias gradient). */
BRK_API int brk_fc_bwd_data(const void* dz, const void* w, const void* mask, void* dx, float* colsum_ws,
                            int N, int C, int K, int b_n, int b_c, int b_k, int dtype, void* stream);
/* Weight update (north star): dw = dz x^T (fp32); if w_sgd != NULL also
 * w_sgd -= lr * dw (bf16 weights, fused in the epilogue).  If db_partials !=
 * NULL (db_parts rows of K column sums, e.g. from brk_fc_bwd_data's colsum_ws)
 * also db_out[K] = their ordered sum and bias_sgd -= bias_lr * db_out.
 * workspace (may be NULL = no split-K): brk_fc_upd_workspace(N, C, K) bytes,
 * zeroed once before first use (its counters self-reset). */
BRK_API int brk_fc_upd(const void* x, const void* dz, float* dw, void* w_sgd, float lr,
                       const float* db_partials, int db_parts, float* db_out, float* bias_sgd, float bias_lr,
                       void* workspace, size_t ws_bytes, int N, int C, int K, int b_n, int b_c, int b_k,
                       int dtype, void* stream);
BRK_API size_t brk_fc_upd_workspace(int N, int C, int K);
/* The whole MLP training step as ONE persistent launch (BASELINE config 2):
 * L forward layers y[l+1] = relu(W_l y[l] + b_l), the top gradient
 * dz[L] = dy * (y[L] > 0) (fused in the last forward epilogue), and per layer l
 * from the top bwd-data dz[l-1] = (W_{l-1}^T dz[l]) * (y[l-1] > 0) and the
 * weight update dW = dz[l] y[l-1]^T with fused SGD of W and b (lr).  Arrays of
 * device pointers: y, dz, colsum have L+1 entries (colsum[l]: fp32 [N/32][C]
 * column-sum partials of dz[l]), w, bias, dw, db have L.  Blocked bf16 layouts
 * as brk_fc_*, N and C multiples of 256, L <= 4.  w_next (may be NULL = in-place SGD)
 * receives the updated weights W - lr dW, so the weight updates need not wait
 * for the bwd-data passes that read W (double-buffered weights).  lr == 0: gradients
 * only, no weight or bias update (data parallel: all-reduce, then brk_sgd_apply).  workspace:
 * >= brk_mlp_step_workspace_bytes(L, N, C) bytes of device scratch (the tile dependency counters):
 * zero it once before the first call; every call leaves it zeroed again (no per-step memset). */
BRK_API int brk_mlp_step(int L, int N, int C, const void* const* y, void* const* dz, const void* dy,
                         void* const* w, void* const* w_next, float* const* bias, float* const* dw, float* const* db,
                         float* const* colsum, float lr, void* workspace, size_t ws_bytes, void* stream);
/* The same step with an explicit storage type: BRK_BF16 (= brk_mlp_step) or BRK_F32 (fp32
 * activations, weights and gradients in the same blocked layouts, kind::tf32 tensor-core math:
 * the reference's own fp32 storage, north_star "bf16 and TF32 inputs").  Replaces the
 * reference FC runner's per-pass fc_forward calls (bench.py:355-360) for the whole step. */
BRK_API int brk_mlp_step_dt(int L, int N, int C, const void* const* y, void* const* dz, const void* dy,
                            void* const* w, void* const* w_next, float* const* bias, float* const* dw,
                            float* const* db, float* const* colsum, float lr, void* workspace, size_t ws_bytes,
                            int dtype, void* stream);
BRK_API size_t brk_mlp_step_workspace_bytes(int L, int N, int C);
/* Bias gradient (north star): dz_out = dy * (y > 0) if y != NULL; db[K] = sum over N of dz;
 * if bias_sgd != NULL also bias_sgd -= lr * db (fused SGD).  Deterministic.
 * workspace: brk_fc_bias_grad_workspace(K) bytes, zeroed once before first use. */
BRK_API int brk_fc_bias_grad(const void* dy, const void* y, void* dz_out, float* db, void* workspace,
                             int N, int K, int b_n, int b_k, float* bias_sgd, float lr, void* stream);
BRK_API size_t brk_fc_bias_grad_workspace(int K);
/* The same with the storage dtype of dy / y / dz_out: BRK_BF16 or BRK_F32 (TF32 MLP step). */
BRK_API int brk_fc_bias_grad_dt(const void* dy, const void* y, void* dz_out, float* db, void* workspace,
                                int N, int K, int b_n, int b_k, float* bias_sgd, float lr, int dtype, void* stream);
/* Bias gradient for any block factors / dtype (dy, y, dz_out in the
 * [N/b_n][K/b_k][b_n][b_k] layout): dz_out = dy*(y>0) if y != NULL; db = sum_n dz. */
BRK_API int brk_colsum_blocked(const void* dy, const void* y, void* dz_out, float* db, int N, int K,
                               int b_n, int b_k, int dtype, void* stream);
/* SGD apply (north-star training step after the dW allreduce): w -= lr * dw, n elements,
 * w in BRK_F32 or BRK_BF16 storage, dw fp32 in the same layout. */
BRK_API int brk_sgd_apply(void* w, const float* dw, float lr, int64_t n, int w_dtype, void* stream);

/* ---------------------------------------------------------------------------
 * Device layout transform.  Replaces the reference's blocked-layout copies
 * (pkg/src/brkernels/tensor.py:143-275: block_weight_2d, block_conv_input,
 * block_conv_weight, block_fc_activation, unblock_*, pad_spatial) on device
 * tensors.  dst (contiguous, ndims <= 8 extents `shape`) receives
 *   dst[i] = src[sum_d (i_d - pad_lo[d]) * src_strides[d]]  when every
 *            0 <= i_d - pad_lo[d] < src_extent[d], else 0,
 * with src_strides in elements (any permutation / split of a tensor);
 * pad_lo / src_extent may be NULL (no padding).  in_dtype / out_dtype
 * BRK_F32 or BRK_BF16 (conversion fused).  One HBM read + write per element.
 * ------------------------------------------------------------------------- */
BRK_API int brk_layout_transform(const void* src, void* dst, int ndims, const int64_t* shape,
                                 const int64_t* src_strides, const int64_t* pad_lo, const int64_t* src_extent,
                                 int in_dtype, int out_dtype, void* stream);

/* ---------------------------------------------------------------------------
 * Direct convolution on the reference's blocked layouts (cnn.py:201-334;
 * tensor.py:160-235), implicit GEMM with TMA im2col operand fetch:
 *   in, din : [N][C/64][H][W][64]     out, dout : [N][K/64][P][Q][64]
 *   w       : [K/64][C/64][R][S][64 c][64 k]   dw : like w, fp32
 * Engine path: bf16 storage (dtype BRK_BF16) or fp32 storage with TF32 math (BRK_F32: k-steps
 * of 32 channels, fp32 outputs; no fused SGD), b_c = b_k = 64, C and K multiples of 64; stride
 * 1 (pad <= 15, R, S <= 16) or 1x1 stride 2 without padding.
 * ------------------------------------------------------------------------- */
/* Replaces brkernels.cnn.conv2d_forward (cnn.py:201-334): out = act(conv(in, w) + bias);
 * bias (fp32, K) may be NULL; act as brk_fc_fwd. */
BRK_API int brk_conv_fwd(const void* in, const void* w, const float* bias, void* out, int N, int C, int K, int H,
                         int W, int R, int S, int stride, int pad_h, int pad_w, int b_c, int b_k, int act, int dtype,
                         void* stream);
/* Backward-data (north star, the paper's dual convolution): din = conv^T(dout, w).
 * Every element of din is written (1x1 stride 2: zeros at the odd positions). */
BRK_API int brk_conv_bwd_data(const void* dout, const void* w, void* din, int N, int C, int K, int H, int W, int R,
                              int S, int stride, int pad_h, int pad_w, int b_c, int b_k, int dtype, void* stream);
/* Weight update (north star): dw = sum over (n, p, q) of dout x in (fp32); if w_sgd != NULL also
 * w_sgd -= lr * dw (bf16 weights).  workspace: brk_conv_upd_workspace(...) bytes (may be 0 = NULL ok);
 * deterministic (split partials are summed in split order). */
BRK_API int brk_conv_upd(const void* in, const void* dout, float* dw, void* w_sgd, float lr, void* workspace,
                         size_t ws_bytes, int N, int C, int K, int H, int W, int R, int S, int stride, int pad_h,
                         int pad_w, int b_c, int b_k, int dtype, void* stream);
BRK_API size_t brk_conv_upd_workspace(int N, int C, int K, int H, int W, int R, int S, int stride, int pad_h,
                                      int pad_w);
/* Diagnostic: engine tile plan of a pass (0 fwd, 1 bwd-data, 2 upd) -> out3 = {pair, bn, splits}. */
/* Small-channel convolutions (C < 64, e.g. the 3-channel stem; reference cnn.py:201-334 with
 * b_c = C): explicit im2col + brk_gemm_dense.  col[(n,p,q)][(r*S+s)*C+c] (bf16, row stride ldcol,
 * a multiple of 8 >= R*S*C, zero outside the image; columns past R*S*C are left as they are) from the blocked input
 * [N][C_b][H][W][b_c]; col2im sums dcol back onto the input pixels (gather, fp32, deterministic). */
BRK_API int brk_conv_im2col(const void* in, void* col, int N, int C, int H, int W, int R, int S, int stride,
                            int pad_h, int pad_w, int b_c, int64_t ldcol, void* stream);
BRK_API int brk_conv_col2im(const void* dcol, void* dx, int N, int C, int H, int W, int R, int S, int stride,
                            int pad_h, int pad_w, int b_c, int64_t ldcol, void* stream);
BRK_API int brk_conv_plan(int pass, int N, int C, int K, int H, int W, int R, int S, int stride, int pad_h,
                          int pad_w, int* out3);
/* Stride-2 small-channel convolutions (C <= 4 in one channel block, e.g. the ResNet-50
 * stem 3->64, 7x7, stride 2, pad 3; reference cnn.py:201-334) as space-to-depth implicit GEMMs:
 * the input is unfolded into 64 channels per output pixel (xs[N][1][P+R'-1][Q][64], bf16:
 * (horizontal tap v, row/column parity a/b, channel c) -> v*16 + (2a+b)*C + c) and the conv
 * runs on the engine as an R' x 1 stride-1 conv (R' = ceil((R + pad_h%2)/2)).
 * x [N][1][H][W][C], w [K/64][1][R][S][C][64], out/dout [N][K/64][P][Q][64] (bf16),
 * dw like w in fp32, dx like x.  workspace: brk_conv_s2d_workspace(...) bytes (no init). */
BRK_API int brk_conv_s2d_shape(int N, int C, int K, int H, int W, int R, int S, int pad_h, int pad_w, int* out4);
BRK_API size_t brk_conv_s2d_workspace(int N, int C, int K, int H, int W, int R, int S, int pad_h, int pad_w);
BRK_API int brk_conv_s2d_unfold(const void* x, void* xs, int N, int C, int H, int W, int R, int S, int pad_h,
                                int pad_w, void* stream);
BRK_API int brk_conv_s2d_fwd(const void* x, const void* w, void* out, void* workspace, size_t ws_bytes, int N, int C,
                             int K, int H, int W, int R, int S, int pad_h, int pad_w, void* stream);
BRK_API int brk_conv_s2d_upd(const void* x, const void* dout, float* dw, void* workspace, size_t ws_bytes, int N,
                             int C, int K, int H, int W, int R, int S, int pad_h, int pad_w, void* stream);
BRK_API int brk_conv_s2d_bwd_data(const void* dout, const void* w, void* dx, void* workspace, size_t ws_bytes, int N,
                                  int C, int K, int H, int W, int R, int S, int pad_h, int pad_w, void* stream);

/* ---------------------------------------------------------------------------
 * Dense row-major GEMM on the same engine (batch list = the K/64 consecutive
 * 64-wide slices of the operands): C[M][N] = act(alpha*A.B^T + bias) + beta*C,
 * A M x K (a_kmajor: A[m][k] at m*lda+k, else k*lda+m), B N x K (b_kmajor: B[n][k]
 * at n*ldb+k, else k*ldb+n), bf16 operands, C fp32 (c_bf16=0) or bf16, row stride
 * ldc.  N, K multiples of 64.  workspace (may be NULL): brk_gemm_dense_workspace
 * bytes enable deterministic split-K for fp32 outputs without epilogue ops.
 * Used by the LSTM drivers (input projection, backward-data, weight gradients).
 * ------------------------------------------------------------------------- */
BRK_API int brk_gemm_dense(const void* a, int64_t lda, int a_kmajor, const void* b, int64_t ldb, int b_kmajor,
                           void* c, int64_t ldc, int c_bf16, int64_t M, int N, int K, float alpha, float beta,
                           const float* bias, int act, void* workspace, size_t ws_bytes, void* stream);
/* fp32 operands on the TF32 tensor cores (kind::tf32; the fp32 bit patterns are
 * consumed as TF32 — pre-round with brk_round_tf32 for round-to-nearest);
 * otherwise exactly brk_gemm_dense (same workspace query). */
BRK_API int brk_gemm_dense_f32(const float* a, int64_t lda, int a_kmajor, const float* b, int64_t ldb,
                               int b_kmajor, void* c, int64_t ldc, int c_bf16, int64_t M, int N, int K, float alpha,
                               float beta, const float* bias, int act, void* workspace, size_t ws_bytes,
                               void* stream);
/* dst = round-to-nearest (ties away, cvt.rna) of fp32 src to TF32 precision, stored as fp32
 * (dst may alias src).  The engine's TF32 paths feed on these. */
BRK_API int brk_round_tf32(const float* src, float* dst, int64_t n, void* stream);
BRK_API size_t brk_gemm_dense_workspace(int64_t M, int N, int K);

/* ---------------------------------------------------------------------------
 * LSTM over a whole sequence, one persistent launch per direction (reference
 * lstm.py:217-327; BPTT restated in oracle/brk_oracle.py:305-350).  bf16
 * tensor-core operands, fp32 state.  N <= 256, K % 64 == 0, K <= 1024.
 *   gx      [T][N][4][K] fp32   W_g x_t + b_g (gate order i, c, f, o)
 *   r_cat   [4K][K] bf16        rows g*K + k = R_g[k][:]
 *   rt_cat  [4K][K] bf16        rows g*K + j = R_g[:][j]  (transposed)
 *   h_bf    [T+1][N][K] bf16    slot 0 = h0 (caller), slot t+1 = h_t (kernel)
 *   flags   brk_lstm_seq_flags_bytes(K) bytes of device scratch
 * fwd writes h, s [T][N][K] and the activated gates [T][N][4][K] (fp32).
 * bwd reads dh [T][N][K] (dL/dh_t), gates, s, s0 (may be NULL) and writes
 * dpre [T][N][4][K] (bf16 pre-activation gradients) and ds0 [N][K].
 * ------------------------------------------------------------------------- */
BRK_API size_t brk_lstm_seq_flags_bytes(int K);
/* Diagnostic: per-step %globaltimer stamps of CTA 0 ([T][8] u64) for subsequent sequence launches; NULL disables. */
BRK_API void brk_diag_lstm_timestamps(unsigned long long* ts);
BRK_API int brk_lstm_seq_fwd(const float* gx, const void* r_cat, const float* s0, void* h_bf, float* h_out,
                             float* s_out, float* gates_out, unsigned* flags, int T, int N, int K, void* stream);
BRK_API int brk_lstm_seq_bwd(const float* dh, const float* gates, const float* s, const float* s0,
                             const void* rt_cat, void* dpre, float* ds0, unsigned* flags, int T, int N, int K,
                             void* stream);

/* ---------------------------------------------------------------------------
 * LSTM recurrent steps (reference lstm.py:217-327, Eqs. 1-6; gate order
 * i, c, f, o per lstm.py:28).  Storage fp32 (h, s, gates, gradients as in
 * the reference), tensor-core inputs TF32 or BF16 (compute code).
 *   R  : [4][K/b_k][K/b_k][b_k][b_k]  the four recurrent matrices, blocked as
 *        block_weight_2d(r_g, b_k, b_k) (tensor.py:143-158)
 *   gx : [N][4][K] = W_g x_t + b_g (precomputed for all t by one grouped BRGEMM)
 * ------------------------------------------------------------------------- */
/* Replaces the per-step work item of lstm_forward (lstm.py:268-317): one launch
 * computes h_t, s_t and the activated gates [N][4][K] of all items. s_prev may be NULL (zeros). */
BRK_API int brk_lstm_fwd_step(const float* h_prev, const float* s_prev, const float* gx, const float* R,
                              float* h_out, float* s_out, float* gates_out, int N, int K, int b_k, int compute,
                              void* stream);
/* BPTT step (north star): dpre_t [N][4][K] and ds_out = ds * f from dh_in (dL/dh_t
 * from the output), the recurrent gradient sum_g dpre_{t+1,g} R_g (dpre_next may be
 * NULL at t = T-1), the stored gates / s_t / s_{t-1} (NULL = 0) and ds_in (NULL = 0). */
BRK_API int brk_lstm_bwd_step(const float* dpre_next, const float* R, const float* dh_in, const float* gates,
                              const float* s_cur, const float* s_prev, const float* ds_in, float* dpre_out,
                              float* ds_out, int N, int K, int b_k, int compute, void* stream);
/* out[N][K] = sum_g dpre[N][g][:] R_g  (gradient w.r.t. h_init). */
BRK_API int brk_lstm_recurrent_grad(const float* dpre, const float* R, float* out, int N, int K, int b_k,
                                    int compute, void* stream);

/* Diagnostic (not on the product path): TMA global->shared streaming
 * throughput of `ctas` CTAs, each moving `iters` slots of loads_per_slot
 * boxes (64 bf16 x box_rows) of a rows x cols bf16 matrix through a ring of
 * `stages`; `spin` > 1 uses that many issuing warps.  Synchronous; returns
 * device microseconds and bytes moved. */
BRK_API int brk_diag_tma_bw(const void* buf, int rows, int cols, int box_rows, int loads_per_slot, int stages,
                            int ctas, int iters, int spin, float* us, double* bytes);
/* Diagnostic: subsequent engine launches record per-CTA %globaltimer phase
 * stamps into ts[8 * blockIdx.x + phase] (device buffer); NULL disables. */
BRK_API void brk_diag_set_timestamps(unsigned long long* ts);
/* Diagnostics: the host list schedule of the chain-first MLP step (brk_mlp_step) for L layers of
 * width C, batch N over `pairs` CTA pairs: units[offsets[c] .. offsets[c+1]) is pair c's list,
 * tiles[q] / dep[q] each problem's unit count and dependency; returns the unit count (0: none). */
BRK_API int brk_diag_mlp_schedule(int L, int N, int C, int pairs, int16_t* units, int16_t* offsets, int* tiles,
                                  int* dep);
/* Diagnostic: TMA throughput when the first `lanes` lanes of ONE warp per CTA each keep two boxes
 * (64 bf16 x box_rows) in flight; synchronous; device microseconds and bytes moved. */
BRK_API int brk_diag_tma_lanes(const void* buf, int rows, int cols, int box_rows, int lanes, int ctas, int iters,
                               float* us, double* bytes);
/* Diagnostic: per-warp clock64 cycles of iters x (tcgen05.ld.32x32b.x32 + wait); synchronous. */
BRK_API int brk_diag_tmem_ld(int ctas, int iters, long long* cycles_dev, float* sink_dev);
/* Diagnostic: clock64 cycles per CTA of iters x 4 back-to-back SS-mode MMAs (M = 128, N = n, K = 16
 * bf16; b_mn: MN-major B) from fixed shared-memory operands; synchronous. */
BRK_API int brk_diag_mma_rate(int n, int b_mn, int ctas, int iters, long long* cycles_dev);

#ifdef __cplusplus
}
#endif

#endif /* BRK_H_ */
