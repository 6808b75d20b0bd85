/*
 * sparsecross_b200.h -- C ABI of the B200 (sm_100a) sparse cross-encoder hot path.
 *
 * Drop-in boundary for the asymmetric windowed self-attention of
 * arXiv 2312.17649 and the backward-free encoder loop around it.  The
 * reference (`sparsecross` 0.1.0, pure Python/numpy) has no FFI; each entry
 * point below replaces the Python function cited beside it
 * (R/ = /root/reference/pkg/src/sparsecross/).
 *
 * Conventions
 *   - All data pointers are caller-owned DEVICE memory; nothing allocates.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream);
 *     every call is stream-ordered and asynchronous.
 *   - Return 0 (SC_OK) on success; on failure a non-zero SC_ERR_* code and a
 *     thread-local message readable through sc_last_error().  The Python
 *     facade maps SC_ERR_INVALID / SC_ERR_NO_VALID_ROW to the reference's
 *     ValueError subclasses (AttentionError, BandShapeError, EncoderError).
 *   - Reentrant: concurrent calls on shared read-only inputs are safe.
 *
 * Packed varlen layout (new; the reference batches one partition only,
 * R/encoder.py:461-468):
 *   cu_seqlens[nseq+1]  int32 prefix of sequence lengths (token rows)
 *   qgroup_len[nseq]    int32 query-group length m+1 of each sequence
 *                       (query tokens + its [SEP]); cls group is 1 row,
 *                       doc group = s - 1 - qgroup_len (R/encoder.py:58-94,
 *                       R/encoder.py:154-177 span convention)
 *
 * Attention pattern = `links[9]`, int32, row-major [src][tgt] over groups
 * (0 cls, 1 query, 2 doc): SC_LINK_NONE, SC_LINK_FULL or a window w >= 0
 * (R/attention.py:55-157; FULL = math.inf at R/attention.py:40).
 */
#ifndef SPARSECROSS_B200_H
#define SPARSECROSS_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SC_API __attribute__((visibility("default")))
#else
#define SC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SC_OK 0
#define SC_ERR_INVALID 1        /* bad shape/window/pattern argument            */
#define SC_ERR_CUDA 2           /* CUDA runtime/launch failure                  */
#define SC_ERR_UNSUPPORTED 3    /* valid request this build does not implement  */
#define SC_ERR_NO_VALID_ROW 4   /* a row has zero valid keys (R/attention.py:250-251) */

#define SC_LINK_NONE (-2)
#define SC_LINK_FULL (-1)

#define SC_DTYPE_F32 0
#define SC_DTYPE_BF16 1

#define SC_PAD_EXCLUDE 0        /* R/attention.py:8-12   */
#define SC_PAD_ZERO_LOGIT 1     /* R/attention.py:13-16  */

#define SC_ATTN_AUTO 0          /* pick the fastest kernel for the pattern      */
#define SC_ATTN_GENERIC 1       /* warp-per-row CUDA-core kernel (any pattern)  */
#define SC_ATTN_BAND_MMA 2      /* tiled band kernel (finite doc window)        */
#define SC_ATTN_TC 3            /* tcgen05/TMEM kernel (wide or dense doc band) */
#define SC_ATTN_HEAD_ROWS 4     /* only the cls + query-group rows of every sequence
                                   (other rows untouched): a last layer whose only
                                   consumer is the [CLS] score, R/encoder.py:506 */

SC_API const char* sc_last_error(void);
SC_API int sc_version(void);
/* Kernels launched by this library so far in this process (all streams). */
SC_API uint64_t sc_kernel_launches(void);

/* ---- K1: device index / mask construction ------------------------------ */

/* Per-token sequence id, group id (0/1/2), group-relative index and position
 * (token index within its sequence), plus per-sequence prefixes of doc-row
 * tiles of `tile_rows` rows (seq_tile_base[nseq+1], the band kernel's
 * scheduler) and of head rows = cls + query-group rows (seq_head_base[nseq+1]).  Replaces SubsequencePartition/_split_groups/_locate
 * (R/encoder.py:58-94, :299-303; R/reference.py:22-27).  qds_every > 0 also
 * fills tok_flags bit0 for QDS global doc tokens (R/encoder.py:180-193) and
 * their CSR lists glob_cu[nseq+1]/glob_pos (doc-relative); pass NULLs when 0.
 * glob_pos must hold at least total_tokens entries. */
SC_API int sc_index_build(const int32_t* cu_seqlens, const int32_t* qgroup_len, int32_t nseq,
                   int32_t total_tokens, int32_t tile_rows, int32_t qds_every,
                   int32_t* tok_seq, int32_t* tok_group, int32_t* tok_rel, int32_t* tok_pos,
                   int32_t* seq_tile_base, int32_t* seq_head_base, uint8_t* tok_flags,
                   int32_t* glob_cu, int32_t* glob_pos, void* stream);

/* Dense (s x s) attendability bitmap of sequence `seq` (uint8, 1 = may attend),
 * exactly the attention kernels' predicate.  Replaces pattern_mask
 * (R/reference.py:30-57); debug/parity export.  seq_len must equal the
 * sequence's length (the caller sizes mask_out = seq_len^2 bytes). */
SC_API int sc_mask_export(const int32_t* cu_seqlens, const int32_t* qgroup_len, int32_t nseq,
                   int32_t seq, int32_t seq_len, const int32_t* links, const uint8_t* tok_flags,
                   uint8_t* mask_out, void* stream);

/* Band validity (rows x (2w+1), uint8) -- R/band.py:48-52. */
SC_API int sc_band_validity(int32_t rows, int32_t window, int32_t target_len, uint8_t* out, void* stream);

/* ---- L1 band kernels ---------------------------------------------------- */

/* out[b, i, j] = q[b, i, :] . k[b, i+j-w, :], 0 where out of range.
 * q: [batch, s, d], k: [batch, t, d], out: [batch, s, 2w+1] (row-major,
 * contiguous), all of `dtype`.  Replaces band_scores / band_qk
 * (R/band.py:154-194, :290-303). */
SC_API int sc_band_scores(const void* q, const void* k, void* out, int64_t batch, int32_t s,
                   int32_t t, int32_t d, int32_t window, int32_t dtype, void* stream);

/* out[b, i, :] = sum_j p[b, i, j] v[b, i+j-w, :]; invalid slots never read.
 * Replaces band_apply / band_pv (R/band.py:197-236, :306-313). */
SC_API int sc_band_apply(const void* p, const void* v, void* out, int64_t batch, int32_t s,
                  int32_t t, int32_t d, int32_t window, int32_t dtype, void* stream);

/* Adjoint of sc_band_scores (R/band.py:239-253): grad_q[b,i,:] = sum_j
 * g[b,i,j] k[b,i+j-w,:], grad_k[b,r,:] = sum over slots addressing key r of
 * g * q; invalid slots of grad_band are never read.  grad_q [batch,s,d],
 * grad_k [batch,t,d], written (not accumulated). */
SC_API int sc_band_scores_backward(const void* grad_band, const void* q, const void* k, void* grad_q,
                   void* grad_k, int64_t batch, int32_t s, int32_t t, int32_t d, int32_t window,
                   int32_t dtype, void* stream);

/* Adjoint of sc_band_apply (R/band.py:256-274): grad_p[b,i,j] =
 * grad_out[b,i,:] . v[b,i+j-w,:] (0 at invalid slots), grad_v[b,r,:] = sum
 * over slots addressing r of p * grad_out.  Written, not accumulated. */
SC_API int sc_band_apply_backward(const void* grad_out, const void* p, const void* v, void* grad_p,
                   void* grad_v, int64_t batch, int32_t s, int32_t t, int32_t d, int32_t window,
                   int32_t dtype, void* stream);

/* ---- K2/K3: fused asymmetric windowed attention ------------------------- */

/* Workspace for sc_attn_fwd: split-softmax partials of the head rows that
 * attend the whole document (CLS; query rows too under longformer/full),
 * one (m, l, acc[d]) record per doc tile x head x full row.  max_qgroup_len
 * is the largest qgroup_len of the batch. */
SC_API size_t sc_attn_workspace_bytes(int32_t nseq, int32_t total_tokens, int32_t heads,
                               int32_t head_dim, int32_t tile_rows, int32_t max_qgroup_len,
                               const int32_t* links);

/* The same for a batch with QDS global doc tokens (R/attention.py:403-470):
 * adds room for n_global_tokens compact [q|k|v] rows (the dense global-key
 * segment and the global rows' full attention run from that copy).  The
 * workspace must be zero-filled before its first use (self-resetting
 * counters live in it); sc_attn_fwd leaves it reusable. */
SC_API size_t sc_attn_workspace_bytes_qds(int32_t nseq, int32_t total_tokens, int32_t heads,
                               int32_t head_dim, int32_t tile_rows, int32_t max_qgroup_len,
                               const int32_t* links, int32_t n_global_tokens);

/* Attention of every token row of a packed batch under one pattern:
 * all three groups (cls, query, doc) of every sequence in one call.
 * q/k/v: row r, head h at base + r*row_stride + h*head_dim (elements of
 * `dtype`); typical packed QKV [T][3][H][d]: k = q + H*d, v = q + 2*H*d,
 * row_stride = 3*H*d.  out: [T][H][d] with out_row_stride.  scale divides
 * the logits (sqrt(d) in the encoder, R/encoder.py:329).  tok_* /
 * seq_tile_base / seq_head_base come from sc_index_build with the same
 * tile_rows; max_qgroup_len is the host-known max of qgroup_len (kernel
 * selection only).  algo picks the kernel (SC_ATTN_*); AUTO runs, in bf16
 * with d = 64: the tiled band kernel for doc windows <= 56 without QDS
 * globals, else the tcgen05 kernel (wider or full windows, and QDS with its
 * globals) -- each plus the head-row combine -- and the generic kernel for
 * everything else (fp32, other head dims, windowed head-row links).
 * status (optional, device int32) gets bit0 set if a row had zero valid keys.
 * Replaces group_attention x3 (R/attention.py:416-473), apply_pattern
 * (:510-537), attend_segments (:290-345), masked_segment_softmax (:228-257)
 * and the band kernels underneath (R/band.py:154-236). */
SC_API int sc_attn_fwd(const void* q, const void* k, const void* v, int64_t row_stride,
                void* out, int64_t out_row_stride,
                const int32_t* cu_seqlens, const int32_t* qgroup_len, int32_t nseq,
                int32_t total_tokens, int32_t heads, int32_t head_dim,
                const int32_t* links, int32_t padding, float scale, int32_t dtype,
                const int32_t* tok_seq, const int32_t* seq_tile_base,
                const int32_t* seq_head_base, int32_t tile_rows, int32_t max_qgroup_len,
                const uint8_t* tok_flags, const int32_t* glob_cu, const int32_t* glob_pos,
                int32_t algo, void* workspace, size_t workspace_bytes, int32_t* status,
                void* stream);

/* Backward of sc_attn_fwd for fine-tuning (R/attention.py:260-269, :348-378,
 * :476-507; R/band.py:239-274): given q/k/v and the forward output `out`
 * (same layout, dtype and pattern arguments as sc_attn_fwd) and the output
 * gradient `dout` ([T][H][d], dout_row_stride, `dtype`), writes dq, dk and
 * dv in `grad_dtype` (fp32 accumulation either way; row r, head h at base +
 * r*grad_row_stride + h*d; e.g. the thirds of one [T][3][H][d] buffer).  Deterministic: two gather-form kernels, no
 * atomics.  Rows whose forward had no valid key get zero gradients.
 * tok_flags/glob_cu/glob_pos, seq_tile_base/tile_rows (from sc_index_build)
 * and max_qgroup_len as in sc_attn_fwd (QDS pointers NULL without QDS).
 * bf16, head_dim 64, no QDS, a finite doc window <= 24, tile_rows 64 and
 * max_qgroup_len <= 31 take the tiled tensor-core path for the doc band;
 * anything else the generic kernels.  n_tiles = seq_tile_base[nseq] when the
 * caller knows it (then the call never synchronises and is CUDA-graph
 * capturable), or -1 to read it from the device.
 * workspace: sc_attn_bwd_workspace_bytes(T, H, nseq, max_qgroup_len) bytes
 * (per-row softmax statistics + per-tile head-key partials of the tiled
 * path; T*H*8 bytes is the minimum).  head_dim <= 128. */
SC_API size_t sc_attn_bwd_workspace_bytes(int32_t total_tokens, int32_t heads, int32_t nseq,
                                          int32_t max_qgroup_len);
SC_API int sc_attn_bwd(const void* q, const void* k, const void* v, int64_t row_stride,
                const void* out, int64_t out_row_stride, const void* dout, int64_t dout_row_stride,
                void* dq, void* dk, void* dv, int64_t grad_row_stride, int32_t grad_dtype,
                const int32_t* cu_seqlens, const int32_t* qgroup_len, int32_t nseq,
                int32_t total_tokens, int32_t heads, int32_t head_dim,
                const int32_t* links, int32_t padding, float scale, int32_t dtype,
                const uint8_t* tok_flags, const int32_t* glob_cu, const int32_t* glob_pos,
                const int32_t* seq_tile_base, int32_t tile_rows, int32_t max_qgroup_len,
                int32_t n_tiles, void* workspace, size_t workspace_bytes, void* stream);

/* ---- Encoder-loop kernels (R/encoder.py:306-371, :475-509) -------------- */

/* x[t] = tok_emb[ids[t]] + pos_emb[tok_pos[t]] (R/encoder.py:483); fp32 x
 * and bf16 xh are each optional (not both NULL).  emb tables are fp32 [*, hidden]. */
SC_API int sc_embed(const int32_t* ids, const int32_t* tok_pos, const float* tok_emb,
             const float* pos_emb, float* x, void* xh, int32_t total_tokens, int32_t hidden,
             void* stream);

/* x_out = LN(resid + y (+ bias)) * gamma + beta, eps 1e-12, biased variance
 * (R/encoder.py:267-273 after the residuals at :346 and :353).  resid/x_out
 * fp32 (may alias); y of y_dtype; bias may be NULL; out_h (bf16) may be NULL. */
SC_API int sc_residual_layernorm(const float* resid, const void* y, int32_t y_dtype,
                          const float* bias, const float* gamma, const float* beta,
                          float* x_out, void* out_h, int32_t rows, int32_t hidden,
                          void* stream);

/* Generalised residual LayerNorm: resid of resid_dtype (fp32 or bf16; the
 * bf16 encoder keeps its residual stream in bf16), y of y_dtype, x_out (fp32)
 * and out_h (bf16) each optional (not both NULL); resid may alias either
 * output.  nonfinite_count (device int32, may be NULL) is incremented once per
 * warp whose output holds a NaN/Inf: the reference's per-layer finite check
 * (R/encoder.py:356-357) fused into the pass that writes the layer output. */
SC_API int sc_residual_layernorm_ex(const void* resid, int32_t resid_dtype, const void* y,
                             int32_t y_dtype, const float* bias, const float* gamma,
                             const float* beta, float* x_out, void* out_h,
                             int32_t* nonfinite_count, int32_t rows, int32_t hidden,
                             void* stream);

/* Fused FFN up-projection (bf16): out[M][N] = gelu_erf(a[M][K] w[N][K]^T + bias)
 * (R/encoder.py:350-351 with :258-259), one tcgen05 GEMM whose epilogue applies
 * bias and GELU before the single bf16 store.  a, w, out bf16 row-major with
 * row strides lda / ldw / ldo (elements); bias fp32 [N] or NULL.  Returns
 * SC_ERR_UNSUPPORTED unless N % 256 == 0, K % 64 == 0 and rows are 16-byte
 * aligned (callers then use cuBLAS + sc_bias_gelu). */
SC_API int sc_gemm_bias_gelu(const void* a, int64_t lda, const void* w, int64_t ldw, const float* bias,
                      void* out, int64_t ldo, int32_t M, int32_t N, int32_t K, void* stream);

/* Fused output projection + residual + LayerNorm (bf16): out[M][768] =
 * LN(resid + a[M][K] w[768][K]^T + bias) * gamma + beta, eps 1e-12 (R/encoder.py:345-347,
 * :352-354, :267-273): a cluster of three CTAs per 128-row block, each owning a
 * 256-column slice, exchanging per-row (mean, M2) through distributed shared
 * memory.  resid/out bf16 (may not alias), out_f32 (fp32 copy) and
 * nonfinite_count (R/encoder.py:356-357) optional.  SC_ERR_UNSUPPORTED unless
 * N == 768, K % 64 == 0 and rows are 16-byte aligned. */
SC_API int sc_gemm_residual_layernorm(const void* a, int64_t lda, const void* w, int64_t ldw, const float* bias,
                               const void* resid, int64_t ldr, const float* gamma, const float* beta,
                               void* out, int64_t ldo, float* out_f32, int64_t ldf,
                               int32_t* nonfinite_count, int32_t M, int32_t N, int32_t K, void* stream);

/* ---- Fine-tuning --------------------------------------- */

/* sc_gemm_bias_gelu that also stores the pre-activation pre = A W^T + b
 * (bf16, row stride ldp): the fine-tuning forward keeps it for the GELU
 * adjoint (R/encoder.py:262-264, :408).  Same envelope. */
SC_API int sc_gemm_bias_gelu_pre(const void* a, int64_t lda, const void* w, int64_t ldw, const float* bias,
                          void* out, int64_t ldo, void* pre, int64_t ldp, int32_t M, int32_t N, int32_t K,
                          void* stream);

/* One fused AdamW step over a flat fp32 buffer of n parameters (R/training.py:
 * 114-137): m = b1 m + (1-b1) g, v = b2 v + (1-b2) g^2,
 * w -= lr * ((m/bc1) / (sqrt(v/bc2) + eps) + weight_decay * w) with
 * bc = 1 - beta^step; fp64 arithmetic, fp32 storage; w_bf16 (optional)
 * receives a bf16 copy of the updated weights.  lr is the scheduled rate of
 * this step.  All buffers 16-byte aligned. */
SC_API int sc_adamw_step(float* w, const float* g, float* m, float* v, void* w_bf16, int64_t n, double lr,
                  double beta1, double beta2, double eps, double weight_decay, int64_t step, void* stream);

/* y = LN(a + b) (b may be NULL) with gamma/beta, eps, fp32 y (plus an
 * optional bf16 copy y_bf16 for the next GEMM) and per-row mean / rstd for
 * sc_layernorm_bwd (R/encoder.py:267-273).  a, b: [rows x
 * cols] contiguous, fp32 or bf16.  cols % 4 == 0, cols <= 1024, 8-byte
 * aligned rows (else SC_ERR_UNSUPPORTED). */
SC_API int sc_layernorm_fwd(const void* a, int32_t a_dtype, const void* b, int32_t b_dtype, const float* gamma,
                     const float* beta, float* y, void* y_bf16, float* mean, float* rstd, int32_t rows,
                     int32_t cols, float eps, void* stream);

/* Adjoint of sc_layernorm_fwd (R/encoder.py:276-285) for the upstream
 * gradient dy (+ dy_bf16, the gradient of the bf16 copy, optional): dx (fp32,
 * the gradient of both a and b) and dgamma / dbeta (fp32 [cols], written).  partials:
 * 2 * sc_ln_partials(rows) * cols floats of scratch.  Deterministic. */
SC_API int sc_layernorm_bwd(const float* dy, const void* dy_bf16, const void* a, int32_t a_dtype, const void* b,
                     int32_t b_dtype,
                     const float* gamma, const float* mean, const float* rstd, float* dx, void* dx_bf16, float* dgamma,
                     float* dbeta, float* partials, int32_t rows, int32_t cols, void* stream);

/* out[c] = sum_r x[r, c] (fp32 out; x fp32 or bf16 with row stride ld): the
 * bias gradients of layer_backward (R/encoder.py:403-441).  partials:
 * sc_ln_partials(rows) * cols floats of scratch.  Deterministic. */
SC_API int sc_colsum(const void* x, int32_t dtype, int64_t ld, int32_t rows, int32_t cols, float* out,
              float* partials, void* stream);

/* Exact-erf GELU (R/encoder.py:258-259), out of place; n % 8 == 0, 16-byte
 * aligned (else SC_ERR_UNSUPPORTED).  fp32: erff; bf16: one-MUFU erfc fit
 * (|error| <= 2e-6, below bf16 resolution), as in the forward epilogue. */
SC_API int sc_gelu_fwd(const void* x, void* y, int32_t dtype, int64_t n, void* stream);

/* dx = dy * gelu'(x) (R/encoder.py:262-264, :408) over [rows x cols]
 * contiguous, and (dbias != NULL) the column sums of dx in fp32 -- the bias
 * gradient of the GEMM that produced x -- with sc_ln_partials(rows) * cols
 * floats of partials.  cols % 8 == 0, 16-byte aligned.  Deterministic. */
SC_API int sc_gelu_bwd(const void* x, const void* dy, void* dx, int32_t dtype, int32_t rows, int32_t cols,
                float* dbias, float* partials, void* stream);

/* Number of per-CTA partial rows the two reductions above use for `rows`. */
SC_API int sc_ln_partials(int32_t rows);

/* In-place exact-erf GELU with optional bias (R/encoder.py:258-259). */
SC_API int sc_bias_gelu(void* x, const float* bias, int32_t dtype, int64_t rows, int32_t cols,
                 void* stream);

/* score[j] = x[cu_seqlens[j]] . head_w + head_b (R/encoder.py:506). */
SC_API int sc_cls_score(const float* x, const int32_t* cu_seqlens, int32_t nseq, int32_t hidden,
                 const float* head_w, float head_b, float* scores, void* stream);

/* Count of rows with a non-finite value in x[rows][cols] (fp32) accumulated
 * into *count (device int32); the encoder raises NonFiniteActivationError
 * when non-zero (R/encoder.py:356-357). */
SC_API int sc_count_nonfinite(const float* x, int64_t n, int32_t* count, void* stream);

/* fp32 GEMM operand -> three bf16 planes for the ranking-exact fp32 mode
 * (CrossEncoder(fp32_gemm="bf16x6"); replaces the fp32 operands of the
 * reference's projections R/encoder.py:322-324, :345, :350, :352).
 * v = x[r][c] (+ bias[c]) (then exact-erf GELU if gelu != 0, R/encoder.py:258-259);
 * y[r][c] = v if y != NULL (may alias x); planes row r = [p1 | p2 | p0 | p1 | p0]
 * (each `cols` wide, row stride ldp >= 5*cols) with p0 = bf16_rn(v),
 * p1 = bf16_rn(v - p0), p2 = bf16_rn(v - p0 - p1).  Strides in elements. */
SC_API int sc_split_bf16x3(const float* x, int64_t ldx, const float* bias, int32_t gelu, float* y, int64_t ldy,
                           void* planes, int64_t ldp, int64_t rows, int32_t cols, void* stream);

/* fp32 GEMM operand -> two fp16 planes for the fast fp32 mode (CrossEncoder(fp32_gemm="f16x3"),
 * the same projections): v as above, y as above; planes row r = [h0 | h1] (onehot == 0) or
 * [h0 | 1 0 0 0 0 0 0 0 | h1] (onehot != 0: a constant column that carries the projection's bias
 * through the GEMM), row stride ldp >= 2*cols (+8), with h0 = fp16_rn(v), h1 = fp16_rn(v - h0),
 * v = h0 + h1 + O(2^-22 |v|).  A value outside fp16 range (|v| >= 65504 or not finite) writes 1
 * to *status (device int, may be NULL).  Strides in elements. */
SC_API int sc_split_f16x2(const float* x, int64_t ldx, const float* bias, int32_t gelu, float* y, int64_t ldy,
                          void* planes, int64_t ldp, int64_t rows, int32_t cols, int32_t onehot, int32_t* status,
                          void* stream);

/* sc_residual_layernorm_ex for fp32 (resid, y, x_out fp32) that also writes the sc_split_f16x2
 * planes of x_out ([h0 | h1], or [h0 | 1 0 .. 0 | h1] with onehot) -- the split pass of the fast
 * fp32 mode fused into the LayerNorm that produces the next GEMM's operand (R/encoder.py:346-347,
 * :353-354 feeding :322-324 / :350).  range_status as sc_split_f16x2's status.  SC_ERR_UNSUPPORTED
 * unless hidden is one of 128, 256, 384, 512, 768, 1024 and pointers are 16-byte aligned. */
SC_API int sc_residual_layernorm_f16x2(const float* resid, const float* y, const float* bias, const float* gamma,
                                       const float* beta, float* x_out, void* planes, int64_t ldp, int32_t onehot,
                                       int32_t* range_status, int32_t* nonfinite_count, int32_t rows,
                                       int32_t hidden, void* stream);

/* Fused FFN up-projection of the fast fp32 mode (CrossEncoder(fp32_gemm="f16x3")): out_planes =
 * sc_split_f16x2 planes of gelu_erf(x1 W1^T + b1) (R/encoder.py:350-351, :258-259) with x1 W1^T as
 * three fp16 tensor-core products in one tcgen05 GEMM: a_planes [M, 2K] = [h0 | h1] of x1,
 * w_planes [N, 2K] = [g1 | g0] of W1 * 2^e (w_scale = 2^-e), accumulating h0 g1 + h1 g0 + h0 g0 in
 * fp32; the epilogue adds the bias, applies erff GELU and writes [M, 2N] = [hi | lo] fp16 planes
 * (the fp32 activation is never stored).  range_status as sc_split_f16x2's status.
 * SC_ERR_UNSUPPORTED unless N % 256 == 0, K % 64 == 0 and rows are 16-byte aligned. */
SC_API int sc_gemm_x3h_gelu_planes(const void* a_planes, int64_t lda, const void* w_planes, int64_t ldw,
                                   float w_scale, const float* bias, void* out_planes, int64_t ldo,
                                   int32_t* range_status, int32_t M, int32_t N, int32_t K, void* stream);

/* fp32 projection of the fast fp32 mode on the same tcgen05 GEMM: out[M][N] (fp32) =
 * w_scale * ([h0 | e | h1] . [g1 | b1 | g0] + [h0 | e] . [g0 | b0]) -- x W^T (+ the bias carried by
 * the constant column e when bias_cols == 8; bias_cols == 0: plain [h0 | h1] and [g1 | g0]) as the
 * three fp16 products of encoder.py _linear_x3h (R/encoder.py:322-324, :345), accumulated in one
 * fp32 TMEM accumulator.  a_planes as sc_split_f16x2 writes them, w_planes [N, 2K + 2*bias_cols].
 * SC_ERR_UNSUPPORTED unless N % 256 == 0, K % 64 == 0 and rows are 16-byte aligned. */
SC_API int sc_gemm_x3h(const void* a_planes, int64_t lda, const void* w_planes, int64_t ldw, float w_scale,
                       float* out, int64_t ldo, int32_t M, int32_t N, int32_t K, int32_t bias_cols, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARSECROSS_B200_H */
