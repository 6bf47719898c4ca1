/*
 * zq_b200.h — C ABI of the B200-native ZeroQuant hot path (libzq_b200.so).
 *
 * Every entry point takes caller-owned DEVICE buffers (plain pointers + sizes),
 * enqueues asynchronously on `stream` (a cudaStream_t passed as void*), and
 * returns a status code.  No torch types cross this boundary.
 *
 * Status codes map onto the reference's error taxonomy
 * (pkg/src/lowbit/errors.py:8-13):
 *   ZQ_OK            0
 *   ZQ_ERR_USAGE     1  -> lowbit.errors.UsageError
 *   ZQ_ERR_SHAPE     2  -> lowbit.errors.ShapeError
 *   ZQ_ERR_CUDA      3  -> RuntimeError (launch / driver failure)
 *   ZQ_ERR_UNSUPPORTED 4 -> UsageError (shape outside what the kernel handles)
 * Non-finite inputs are reported through `nonfinite_flag` (device int32,
 * caller-zeroed; set to 1 by the kernel), which the host raises as ValueError
 * (pkg/src/lowbit/quant.py:109-110, :247-248, :265-266).
 *
 * Layouts (row-major, C order):
 *   activations  f32 [rows, cols], row stride ld (elements)
 *   int8 payload [rows, ld_q] with ld_q % 16 == 0 and zero padding past cols
 *   weights      int8 [N, ld_w] output-major (igemm.py:66-80 reads w row j for
 *                output channel j); W4 packed: uint8 [N, ld_w/2], element 2k in
 *                the low nibble of byte k (two's complement)
 *   row scales   f32 [N]   (QuantizedMatrix.row_scales(), quant.py:165-170)
 *   token scales f32 [rows]
 */
#ifndef ZQ_B200_H_
#define ZQ_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ZQ_OK 0
#define ZQ_ERR_USAGE 1
#define ZQ_ERR_SHAPE 2
#define ZQ_ERR_CUDA 3
#define ZQ_ERR_UNSUPPORTED 4

/* output element types of the dequant epilogue */
#define ZQ_OUT_F32 0
#define ZQ_OUT_F16 1
#define ZQ_OUT_BF16 2

/* library version / build identification (for the loaded-.so audit) */
const char* zq_version(void);

/* Last error message of the calling thread (static storage). */
const char* zq_last_error(void);

/* Replaces quant.quantize_activation_tokenwise (pkg/src/lowbit/quant.py:258-269):
 * per-row scale s = f32(max|x| / qmax) (0 -> 1.0), q = clamp(RHAFZ(x/s)). */
int zq_quantize_tokenwise(const float* x, int64_t rows, int64_t cols, int64_t ld_x, int bits,
                          int8_t* q, int64_t ld_q, float* token_scales, int32_t* nonfinite_flag,
                          void* stream);

/* Replaces quant.quantize_activation_static (pkg/src/lowbit/quant.py:272-281) and
 * quant.quantize_array (quant.py:103-113): q = clamp(RHAFZ(f64(x) / scale)). */
int zq_quantize_static(const float* x, int64_t rows, int64_t cols, int64_t ld_x, double scale,
                       int bits, int8_t* q, int64_t ld_q, int32_t* nonfinite_flag, void* stream);

/* float64 inputs, as the reference reads them (no f32 round trip):
 * compute_scale's max |x| per row (quant.py:80-95) and quantize_array's
 * clamp(RHAFZ(x / scale)) with the f64 division (quant.py:98-113). */
int zq_row_absmax_f64(const double* x, int64_t rows, int64_t cols, int64_t ld_x, double* amax,
                      int32_t* nonfinite_flag, void* stream);
int zq_quantize_array_f64(const double* x, int64_t n, double scale, int bits, int8_t* q,
                          int32_t* nonfinite_flag, void* stream);

/* Replaces quant.quantize_weight_groupwise (pkg/src/lowbit/quant.py:236-255):
 * contiguous row groups (group_layout_for, quant.py:211-219), one f32 scale per
 * group, also writes the expanded per-row scale vector (QuantizedMatrix.row_scales).
 * `packed4` (nullable, bits==4 only) additionally receives the packed INT4 payload
 * [rows, ld_q/2]. */
int zq_quantize_weight_groupwise(const float* w, int64_t rows, int64_t cols, int64_t groups,
                                 int bits, int8_t* q, int64_t ld_q, float* group_scales,
                                 float* row_scales, uint8_t* packed4, int32_t* nonfinite_flag,
                                 void* stream);

/* Packs an int8 payload with values in [-7, 7] into two's-complement nibbles. */
int zq_pack_int4(const int8_t* q, int64_t rows, int64_t ld_q, uint8_t* packed, void* stream);

/* Replaces igemm.layer_norm_quantize (pkg/src/lowbit/igemm.py:150-157) over
 * tensor.layer_norm (pkg/src/lowbit/tensor.py:59-73), optionally fused with the
 * residual add that feeds it in block_forward (transformer.py:477, :486):
 * y = LN(x [+ residual]) with numpy's pairwise f32 reductions; writes the float
 * LN output (nullable) and its token-wise quantization. */
int zq_layer_norm_quantize(const float* x, const float* residual, const float* gamma,
                           const float* beta, int64_t rows, int64_t cols, float eps, int bits,
                           float* ln_out, int8_t* q, int64_t ld_q, float* token_scales,
                           int32_t* nonfinite_flag, void* stream);

/* Replaces igemm.gelu_quantize (pkg/src/lowbit/igemm.py:160-161) over tensor.gelu
 * (pkg/src/lowbit/tensor.py:76-83): exact-erf GeLU in f64 rounded once to f32,
 * then token-wise quantization.  gelu_out (nullable) receives the f32 GeLU. */
int zq_gelu_quantize(const float* x, int64_t rows, int64_t cols, int64_t ld_x, int bits,
                     float* gelu_out, int8_t* q, int64_t ld_q, float* token_scales,
                     int32_t* nonfinite_flag, void* stream);

/* Replaces igemm.igemm (pkg/src/lowbit/igemm.py:66-80): exact int32
 * acc[M,N] = xq[M,K] . wq[N,K]^T on tcgen05 kind::i8 tensor cores.
 * w_bits: 8 (int8 payload, ld_w bytes per row) or 4 (packed payload, ld_w/2 bytes per row). */
int zq_igemm_s32(const int8_t* xq, int64_t ld_x, const void* wq, int64_t ld_w, int w_bits,
                 int64_t M, int64_t N, int64_t K, int32_t* acc, int64_t ld_acc, void* stream);

/* Replaces igemm.quantized_linear for Dynamic/Static activations
 * (pkg/src/lowbit/igemm.py:115-139) after the activation quantizer: the fused
 * igemm + dequant_epilogue (igemm.py:83-112):
 *   out = ((f32(acc) * s_tok[i]) * s_w[j]) + bias[j]
 * token_scales == NULL selects the static path with `static_scale` (f32-rounded,
 * igemm.py:98-99).  bias nullable.  out_type: ZQ_OUT_F32/F16/BF16 (RN cast of
 * the exact f32 value). */
int zq_linear(const int8_t* xq, int64_t ld_x, const float* token_scales, float static_scale,
              const void* wq, int64_t ld_w, int w_bits, const float* w_row_scales,
              const float* bias, int64_t M, int64_t N, int64_t K, void* out, int64_t ld_out,
              int out_type, void* stream);

/* Fused row-parallel projection + residual + LayerNorm + token-wise quantize
 * (transformer.py:474-477 and :484-486 as one kernel): y = LN(residual + linear)
 * with the exact epilogue of zq_linear, numpy's pairwise LN of
 * zq_layer_norm_quantize, and its token-wise quantization; writes y (f32) and
 * q / q_scales, never the linear output.  Needs w_bits 8 and a row width whose
 * pairwise tree is balanced with 96- or 128-element leaves (768, 1024, 2048,
 * 3072, 4096, 6144, ...); returns ZQ_ERR_UNSUPPORTED otherwise (callers then
 * run zq_linear + zq_layer_norm_quantize).  `workspace`: device memory of at
 * least 4*ceil(M/256) + 16 + 12*M*(N/(2*leaf)) bytes, zero-initialised once and
 * then reused by every call with the same N on the same stream. */
int zq_linear_ln_quantize(const int8_t* xq, int64_t ld_x, const float* token_scales, const void* wq,
                          int64_t ld_w, int w_bits, const float* w_row_scales, const float* bias, int64_t M,
                          int64_t N, int64_t K, const float* residual, const float* gamma, const float* beta,
                          float eps, int bits, float* ln_out, int8_t* q, int64_t ld_q, float* q_scales,
                          void* workspace, int64_t workspace_bytes, int32_t* nonfinite_flag, void* stream);

/* zq_igemm_s32 with the stream-K workspace of zq_linear_ws for decode-sized calls
 * (the tensor-parallel row-parallel partial GEMM before the int32 SUM all-reduce). */
int zq_igemm_s32_ws(const int8_t* xq, int64_t ld_x, const void* wq, int64_t ld_w, int w_bits, int64_t M, int64_t N,
                    int64_t K, int32_t* acc, int64_t ld_acc, void* workspace, int64_t workspace_bytes, void* stream);

/* Standalone dequant epilogue over an int32 accumulator (igemm.py:83-112); used
 * after the tensor-parallel int32 all-reduce. */
int zq_dequant_epilogue(const int32_t* acc, int64_t ld_acc, const float* token_scales,
                        float static_scale, const float* w_row_scales, const float* bias,
                        int64_t M, int64_t N, void* out, int64_t ld_out, int out_type,
                        void* stream);

/* Replaces igemm.quantized_linear(FullAct) (pkg/src/lowbit/igemm.py:127-130):
 * weight-only path, out = matmul(x, dequant(w).T) + bias with the reference's
 * sequential f32 accumulation order (tensor.py:37-56). */
int zq_linear_full(const float* x, int64_t ld_x, const void* wq, int64_t ld_w, int w_bits,
                   const float* w_row_scales, const float* bias, int64_t M, int64_t N,
                   int64_t K, float* out, int64_t ld_out, void* stream);

/* Weight-only tensor-core path (tolerance mode of igemm.quantized_linear(FullAct),
 * pkg/src/lowbit/igemm.py:127-130; the paper's W8A16 / A8/16 deployment).
 * Step 1 splits each activation row, scaled by a power of two 2^e that puts its
 * max in [2^14, 2^15), into terms = 1 (fp16, "A16") or 2 (fp16 hi + lo, ~22
 * significant bits) 16-bit arrays [M, ld_h] and writes row_inv[i] = 2^-e. */
int zq_act_split16(const float* x, int64_t ld_x, int64_t M, int64_t K, int terms, void* hi, void* lo,
                   int64_t ld_h, float* row_inv, int32_t* nonfinite_flag, void* stream);

/* Step 2: out = ((acc * row_inv[i]) * s_w[j]) + bias[j], acc = sum_k (hi [+ lo])[i,k] * q[j,k]
 * on tcgen05 kind::f16 CTA pairs (f32 accumulators), the int8 / packed INT4 weight
 * rows converted to f16 in shared memory (exact).  a_lo = NULL for one term.
 * ld_a % 8 == 0, ld_w % 32 == 0 (weight rows as zq_linear).  out_type ZQ_OUT_*. */
int zq_linear_wo(const void* a_hi, const void* a_lo, int64_t ld_a, const float* row_inv, const void* wq,
                 int64_t ld_w, int w_bits, const float* w_row_scales, const float* bias, int64_t M, int64_t N,
                 int64_t K, void* out, int64_t ld_out, int out_type, void* stream);

/* Row absmax (f32 bit patterns, non-negative) for the tensor-parallel token-scale
 * all-reduce: amax[i] = max_j |x[i, j]|. */
int zq_row_absmax(const float* x, int64_t rows, int64_t cols, int64_t ld_x, float* amax,
                  int32_t* nonfinite_flag, void* stream);

/* Token-wise quantization with externally supplied per-row absmax (the
 * all-reduced global max in the row-parallel TP path). */
int zq_quantize_with_absmax(const float* x, int64_t rows, int64_t cols, int64_t ld_x,
                            const float* amax, int bits, int8_t* q, int64_t ld_q,
                            float* token_scales, void* stream);

/* Float attention of the block (transformer.py:413-440) for `batch` packed
 * sequences: qkv [batch*seq, ld_qkv] holds q | k | v (heads*head_dim columns
 * each), ctx [batch*seq, ld_ctx].  head_dim 64: tcgen05 (seq <= 128: kind::f16
 * with a two-term hi/lo split of power-of-two-scaled tiles; longer: kind::tf32
 * 3-term split with an online softmax), ~fp32 accuracy (tolerance parity).
 * Other head_dim (multiples of 16 up to 256): CUDA-core fp32 flash attention.
 * Returns ZQ_ERR_UNSUPPORTED otherwise. */
int zq_attention_f32(const float* qkv, int64_t ld_qkv, int batch, int seq, int heads,
                     int head_dim, int causal, float scale, float* ctx, int64_t ld_ctx,
                     void* stream);

/* Fused W8A8 QKV projection + attention for the encoder block (reference:
 * pkg/src/lowbit/transformer.py:395-440 — quantized_linear(attn_in) on the
 * concatenated QKV weight, then attention — which the reference runs as two
 * steps).  xq [batch*seq, ld_x] int8 with token_scales [batch*seq] (dynamic
 * token-wise), w_qkv [3*d, ld_w] int8 with w_row_scales [3*d] (expanded group
 * scales) and bias [3*d] or NULL, d = heads*head_dim.  ctx is bit-identical to
 * zq_linear(..., ZQ_OUT_F32) followed by zq_attention_f32; the f32 QKV
 * activation never reaches HBM.  ZQ_ERR_UNSUPPORTED unless head_dim == 64,
 * seq <= 128, d % 128 == 0 and ld_x, ld_w multiples of 16 (callers then run
 * the two kernels). */
int zq_qkv_attention(const int8_t* xq, int64_t ld_x, const float* token_scales, const int8_t* w_qkv,
                     int64_t ld_w, const float* w_row_scales, const float* bias, int batch, int seq,
                     int heads, int head_dim, int causal, float scale, float* ctx, int64_t ld_ctx,
                     void* stream);

/* GPT decode: scatter the k and v column blocks of the
 * fused QKV output qkv [batch*rows_per_seq, ld_qkv] (q | k | v, dmodel_local
 * columns each) into f32 caches [batch, max_ctx, dmodel_local] at rows
 * pos[b] .. pos[b]+rows_per_seq-1 (pos: device int32 [batch]).  The reference
 * recomputes the context each step (evaluate.py:96-98); cached rows are
 * bit-identical to the recomputed ones. */
int zq_kv_append(const float* qkv, int64_t ld_qkv, int batch, int rows_per_seq, int dmodel_local,
                 const int32_t* pos, float* kcache, float* vcache, int64_t max_ctx, void* stream);

/* zq_linear with a caller-owned int32 workspace for decode-sized calls (M <= 64,
 * int8 weights): the stream-K skinny kernel (k-block units split evenly over
 * two CTAs per SM, exact int32 partial sums added in the workspace, then a
 * light dequant-epilogue kernel that also re-zeroes it).  The workspace
 * (zq_linear_ws_bytes(M, N) bytes, 16-byte aligned) must be zeroed once before
 * first use; every launch leaves it zeroed.  Other shapes: exactly zq_linear. */
int64_t zq_linear_ws_bytes(int64_t M, int64_t N);
int zq_linear_ws(const int8_t* xq, int64_t ld_x, const float* token_scales, float static_scale, const void* wq,
                 int64_t ld_w, int w_bits, const float* w_row_scales, const float* bias, int64_t M, int64_t N,
                 int64_t K, void* out, int64_t ld_out, int out_type, void* workspace, int64_t workspace_bytes,
                 void* stream);

/* Decode QKV projection with the KV-cache append fused into the epilogue: as
 * zq_linear (f32 output, M <= 64 rows, one row per sequence) and additionally
 * kcache / vcache[m, pos[m], :] = columns [dl, 2 dl) / [2 dl, 3 dl) of row m
 * (N == 3 * dmodel_local).  ZQ_ERR_UNSUPPORTED for M > 64 (prefill): call
 * zq_linear then zq_kv_append. */
int zq_linear_kv(const int8_t* xq, int64_t ld_x, const float* token_scales, const void* wq, int64_t ld_w,
                 int w_bits, const float* w_row_scales, const float* bias, int64_t M, int64_t N, int64_t K,
                 float* out, int64_t ld_out, float* kcache, float* vcache, const int32_t* pos, int dmodel_local,
                 int64_t max_ctx, void* stream);
/* Prefill QKV projection (M > 64 token rows = whole sequences of rows_per_seq
 * tokens, the cache empty before it) with the KV-cache append done by the
 * CTA-pair GEMM's epilogue: row r's k / v columns also go to cache row
 * (r / rows_per_seq) * max_ctx + r % rows_per_seq.  ZQ_ERR_UNSUPPORTED where the
 * pair path does not apply (the caller runs zq_linear + zq_kv_append). */
int zq_linear_kv_prefill(const int8_t* xq, int64_t ld_x, const float* token_scales, const void* wq, int64_t ld_w,
                         int w_bits, const float* w_row_scales, const float* bias, int64_t M, int64_t N, int64_t K,
                         float* out, int64_t ld_out, float* kcache, float* vcache, int dmodel_local, int64_t max_ctx,
                         int rows_per_seq, void* stream);

/* The same with the stream-K workspace (see zq_linear_ws). */
int zq_linear_kv_ws(const int8_t* xq, int64_t ld_x, const float* token_scales, const void* wq, int64_t ld_w,
                    int w_bits, const float* w_row_scales, const float* bias, int64_t M, int64_t N, int64_t K,
                    float* out, int64_t ld_out, float* kcache, float* vcache, const int32_t* pos, int dmodel_local,
                    int64_t max_ctx, void* workspace, int64_t workspace_bytes, void* stream);

/* One-token-per-sequence attention against the caches (transformer.py:413-440
 * for the last query row): ctx[b, h] = softmax(q.K^T * scale) V over the first
 * lens[b] cached tokens (device int32).  head_dim % 32 == 0, <= 256.
 * `chunks` = context chunks per (sequence, head) merged by the flash-decoding
 * combine (1, 2, 4 or 8), or 0 for the occupancy rule.  The float result
 * depends on the chunking, so a tensor-parallel rank passes the count the
 * unsharded model would use (zq_decode_attention_chunks with the global head
 * count) to stay bit-identical to one GPU. */
int zq_decode_attention_f32(const float* q, int64_t ld_q, const float* kcache, const float* vcache,
                            int64_t max_ctx, int batch, int heads, int head_dim,
                            const int32_t* lens, float scale, float* ctx, int64_t ld_ctx,
                            int chunks, void* stream);

/* The occupancy rule behind chunks == 0: returns the chunk count for
 * batch x heads (sequence, head) pairs over a max_ctx cache. */
int zq_decode_attention_chunks(int batch, int heads, int64_t max_ctx);

/* L2 residency for an engine's hot activation pool: sets the persisting L2
 * set-aside (min(bytes, device max)) and an access-policy window on `stream`
 * (persisting hits inside [base, base + bytes), streaming misses).  Call outside
 * stream capture; kernels captured on the stream carry the window.  bytes == 0
 * clears the window.  *granted (nullable) receives the set-aside in bytes. */
int zq_l2_persist(void* stream, const void* base, int64_t bytes, int64_t* granted);

/* Tied LM head + greedy argmax of a decode step (logits = x @ emb^T, argmax per
 * row; float, tolerance parity): x [ntok <= 16, dim] f32 (row stride ld_x),
 * emb [vocab, dim] f32 row-major, emb_scale = a power of two with
 * max|emb| * emb_scale in [2^14, 2^15) (chosen once by the caller).  tcgen05
 * kind::f16 on a two-term f16 split of both operands (~fp32 accuracy); ties
 * resolve to the lowest index (numpy argmax).  Workspaces: xh_ws / xl_ws
 * 16*dim f16 each, xinv_ws 16 f32, keys_ws 16 u64.  ids: int64 [ntok]. */
int zq_lm_head_argmax(const float* x, int64_t ld_x, int ntok, const float* emb, int64_t vocab, int64_t dim,
                      float emb_scale, void* xh_ws, void* xl_ws, float* xinv_ws, unsigned long long* keys_ws,
                      int64_t* ids, void* stream);

/* The same head with the embedding pre-split once (zq_lm_embed_split: emb_hi /
 * emb_lo = f16 hi / lo terms of emb * emb_scale, [vocab, dim] each): the decode
 * step streams the two f16 terms by TMA with no per-step conversion. */
int zq_lm_embed_split(const float* emb, int64_t vocab, int64_t dim, float emb_scale, void* emb_hi, void* emb_lo,
                      void* stream);
int zq_lm_head_argmax_split(const float* x, int64_t ld_x, int ntok, const void* emb_hi, const void* emb_lo,
                            int64_t vocab, int64_t dim, float emb_scale, void* xh_ws, void* xl_ws, float* xinv_ws,
                            unsigned long long* keys_ws, int64_t* ids, void* stream);

/* Diagnostics / tests: the fp32 GeLU estimate the quantizer brackets with, and
 * its per-element relative error bound (x clamped to >= -5.5). */
int zq_gelu_estimate(const float* x, int64_t n, float* est, float* bound, void* stream);

/* Diagnostics: when buf != NULL, subsequent GEMM launches record per-CTA
 * %globaltimer stamps into buf[cta*64 + slot] (slot 0 entry, 1 setup done,
 * 2+4t / 3+4t MMA start / last operands landed for local tile t, 4+4t / 5+4t
 * epilogue start / end, 63 epilogue exit).  Not thread-safe; tooling only. */
int zq_gemm_set_trace(unsigned long long* buf);

/* Kept for ABI stability: mode 0 returns ZQ_OK, any other mode
 * ZQ_ERR_UNSUPPORTED (the phase timeline moved to zq_attention_set_trace). */
int zq_attention_debug(int mode);

/* Diagnostics: when buf != NULL (148 x 64 u64), the attention kernels launched
 * afterwards record %globaltimer stamps per CTA: attention_f16_kernel at
 * buf[cta*64 + head_iter*8 + phase] (phase 0 loop start, 1 operands landed,
 * 2 split done, 3 S done, 4 P in TMEM, 5 O done, 6 stored); the fused QKV +
 * attention kernel at buf[cta*64 + 8 + unit*8 + phase] (0 start, 1 S ready,
 * 2 P written, 3 next accumulator ready, 4 next split done, 5 P V done, 6 end,
 * 7 loop top), its prologue at [2], [3] and the GEMM warps at [52..63]
 * (tools/qa_trace.py reads them).  The pointer is a launch argument, so a
 * captured graph keeps the one set at capture. */
int zq_attention_set_trace(unsigned long long* buf);


/* ---- Order-exact float32 forward for static calibration (zq_calib.cu) ----
 * The reference calibrates on its FLOAT model (evaluate.py:168-196 over
 * transformer.py:405-440); these restate its numpy arithmetic so the
 * calibrated scales come out bit-identical. */

/* tensor.matmul(a, w.T) (+ bias) (tensor.py:37-56, transformer.py:405-410):
 * p-ascending f32 sum of separately rounded products from +0.0. */
int zq_matmul_f32_seq(const float* a, int64_t lda, const float* w, int64_t ldw, const float* bias, int64_t M,
                      int64_t N, int64_t K, float* out, int64_t ldo, void* stream);

/* transformer.attention (transformer.py:413-440) over one sequence of t tokens:
 * q, k, v = columns [0, d), [d, 2d), [2d, 3d) of qkv; numpy's f32 exp and
 * pairwise row sum inside tensor.softmax (tensor.py:94-99).  scratch: heads*t*t
 * floats. */
int zq_attention_exact_f32(const float* qkv, int64_t ld_qkv, int t, int heads, int head_dim, int causal,
                           float inv_scale, float* scratch, float* ctx, int64_t ld_ctx, void* stream);

/* out2 = [max, min] of x[0..n) (Calibrator.observe, quant.py:305-317). */
int zq_minmax_f32(const float* x, int64_t n, float* out2, int32_t* nonfinite_flag, void* stream);

/* y = numpy's float32 exp(x) (diagnostics / parity of the calibration forward). */
int zq_np_expf(const float* x, int64_t n, float* y, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ZQ_B200_H_ */
