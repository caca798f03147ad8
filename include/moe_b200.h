/*
 * moe_b200.h — C ABI of the B200-native W8A8 MoE hot path (arXiv 2508.07329,
 * reference package `moekit`).
 *
 * The reference exposes its operator API as module-level Python functions of
 * moekit.quant / moekit.trace / moekit.placement (re-exported in
 * moekit/__init__.py:15-17); it has no FFI. Each entry point below is the
 * device-side replacement of one of those functions (cited per function) or
 * of a forward-path step the reference leaves out (router, permutation,
 * grouped expert GEMM, combine — SURVEY.md §8a rows a'1..a'3). The Python
 * host layer `paper_2508_07329_b200` binds these with ctypes (see
 * INTEGRATION.md) and keeps the reference's names, argument meaning and
 * exception types.
 *
 * Conventions
 *  - All pointers are DEVICE pointers unless stated; callers own all memory;
 *    kernels never allocate (workspace sizes are queried).
 *  - Activations are tokens-major [rows, cols] (per_token == per row).
 *    Weights are [out rows, in cols] (quant.py:3-5). GEMM: Y = A * W^T.
 *  - Codes are unsigned 8-bit containers for 2..8-bit affine codes
 *    value = (code - zero_point) * scale (quant.py:15-16).
 *  - `stream` is a cudaStream_t (CUstream) passed as void*.
 *  - Every function returns a moe_status; on failure moe_last_error() holds
 *    a thread-local message. Status -> Python exception mapping:
 *    EINVAL -> ValueError, ENOTPD -> NotPositiveDefiniteError,
 *    EDEGENERATE -> DegenerateHessianError, EQUANTFAIL ->
 *    QuantizationFailedError (errors.py:11-35), ECUDA/EUNSUPPORTED ->
 *    RuntimeError.
 */
#ifndef MOE_B200_H
#define MOE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* moe_stream_t;

typedef enum {
  MOE_OK = 0,
  MOE_EINVAL = 1,
  MOE_ENOTPD = 2,
  MOE_EDEGENERATE = 3,
  MOE_EQUANTFAIL = 4,
  MOE_ECUDA = 5,
  MOE_EUNSUPPORTED = 6
} moe_status;

/* element types */
enum { MOE_DT_F32 = 0, MOE_DT_F64 = 1, MOE_DT_BF16 = 2, MOE_DT_F16 = 3, MOE_DT_U8 = 4, MOE_DT_I32 = 5 };
/* granularity tags == index in quant.GRANULARITIES (quant.py:40) */
enum { MOE_GRAN_PER_TENSOR = 0, MOE_GRAN_PER_TOKEN = 1, MOE_GRAN_PER_OUTPUT_ROW = 2 };
/* smoothing application (quant.py:314-324): activations divide, weights multiply */
enum { MOE_SMOOTH_NONE = 0, MOE_SMOOTH_DIVIDE = 1, MOE_SMOOTH_MULTIPLY = 2 };
/* GEMM epilogues */
enum { MOE_EPI_DEQUANT = 0, MOE_EPI_SWIGLU = 1, MOE_EPI_ACC_I32 = 2 };
/* OR-ed into `epilogue`: w_rowsum holds the pre-corrected weight term
 * rowsum_w - K * w_zp (precomputed once per weight matrix) instead of the
 * plain code row sums; saves one integer multiply per accumulator. */
enum { MOE_EPI_FLAG_WCORR = 0x100 };
/* OR-ed into moe_w8a8_gemm_combine's `epilogue`: the caller zeroed the
 * workspace already (earlier in the stream), so the call adds no memset
 * between the previous kernel and the GEMM (keeps the PDL overlap). */
enum { MOE_EPI_FLAG_WS_ZEROED = 0x200 };
/* OR-ed into moe_w8a8_gemm's `epilogue` with row_ext: the caller already set
 * every row's records to (min = ~0, max = 0) earlier in the stream, so the
 * call launches no initialisation kernel before the GEMM (keeps the PDL
 * chain from the previous kernel). */
enum { MOE_EPI_FLAG_EXT_READY = 0x400 };
/* channel ordering strategies (quant.py:42-45) */
enum { MOE_ORDER_MAX_ABS = 1, MOE_ORDER_SUM_SQUARES = 2 };

/* ---- library ------------------------------------------------------------ */
const char* moe_last_error(void);
/* Numeric detail of the last MOE_ENOTPD on this thread: the failing pivot
 * (0-based column, -1 if none) and its value (numkit.cholesky's
 * NotPositiveDefiniteError(pivot, value), numkit.py:89-90). */
moe_status moe_last_error_detail(int64_t* pivot, double* value);
int moe_abi_version(void);
/* Number of kernels this library has launched in the process (all entry
 * points count every launch they make) — the bench's gpu_launches. */
uint64_t moe_launch_count(void);
/* 0 if device `dev` is an sm_100 part the kernels were built for. */
moe_status moe_device_check(int dev);
/* Process-wide kernel-selection knobs (atomic; results never depend on them,
 * only which of the bit-identical kernels runs). Sets `key` to `value` and
 * returns the previous value in *old (optional); value < 0 only queries.
 *   MOE_TUNE_K1_SMALL_ROWS: per-token K1 calls with at most this many rows
 *   use the CTA-per-row kernel instead of the per-warp fast kernels
 *   (default 256; env MOE_B200_K1_SMALL sets the initial value).
 *   MOE_TUNE_ROUTER_CLUSTER_TILES: tensor-core router calls with at most
 *   this many 128-token tiles split K over a thread-block cluster; larger
 *   ones use the persistent multi-accumulator kernel (same logits;
 *   default 64 tiles).
 *   MOE_TUNE_FUSED_QUANT: 1 lets the MoE forward use moe_w8a8_gemm_quant_a
 *   for its second GEMM, 0 (default) the separate K1 + GEMM.
 *   MOE_TUNE_FUSED_COMBINE: 1 (default) lets the top-2 MoE forward use
 *   moe_w8a8_gemm_combine, 0 the separate GEMM + combine.
 *   MOE_TUNE_K1_TOKENS: x of the MoE forward quantized token-major
 *   (moe_act_quant_tokens, x read from HBM once per token): 2 (default) the
 *   row kernel walking tokens in order (a token's k rows on adjacent warps,
 *   32 warps per SM), 1 the register-resident one-warp-per-token kernel,
 *   0 the gathered moe_act_quant. (Same results every way.)
 *   MOE_TUNE_GPTQ_LANES: lanes per weight row of the moe_gptq_columns loop
 *   (0 = automatic: 16; 8, 16 or 32 forced).
 *   MOE_TUNE_BAND_MB: grouped-GEMM raster band — MB of activation rows kept
 *   L2-resident while the weight blocks stream past them (default 24; env
 *   MOE_B200_BAND_MB sets the initial value). */
enum {
  MOE_TUNE_K1_SMALL_ROWS = 1,
  MOE_TUNE_ROUTER_CLUSTER_TILES = 2,
  MOE_TUNE_FUSED_QUANT = 3,
  MOE_TUNE_FUSED_COMBINE = 4,
  MOE_TUNE_K1_TOKENS = 5,
  MOE_TUNE_GPTQ_LANES = 6,
  MOE_TUNE_BAND_MB = 7,
  MOE_TUNE_COUNT = 8
};
moe_status moe_tune(int key, int64_t value, int64_t* old);

/* ---- K1: smoothing + RTN affine quantization ----------------------------
 * Replaces quant.rtn_quantize (quant.py:214-231) applied to
 * apply_smoothing's operand (quant.py:314-324), i.e. the activation side of
 * quant_loss (quant.py:281-282) and of the W8A8 forward, and the weight side
 * of _quantize_weights (quant.py:262-264, MULTIPLY mode).
 *
 * Output row r reads input row gather_rows[r] (or r when NULL), smooths it
 * with table row row_group[r] (or 0) of `smooth` [G, cols] (with its
 * correctly-rounded reciprocal table `smooth_recip`, used for an exact
 * reciprocal-and-correct division; NULL -> plain IEEE division), then
 * quantizes with float64 semantics bit-identical to the reference. For bf16
 * input with per-row groups, `smooth_recip_f32` (RN32 of smooth_recip)
 * enables the float32-filtered kernel (exact float64 only where the float32
 * error interval could change the result; identical output):
 * scale = max((max-min)/qmax, 1e-12), zp = clip(rha(-min/scale)),
 * code = clip(rha(xs/scale)+zp), rha(v) = sign(v)*floor(|v|+0.5).
 * per_token / per_output_row: one group per output row. per_tensor: one
 * group (workspace >= moe_act_quant_workspace()). Outputs: codes [rows,
 * ldc], scale f64 [groups], scale_f32 (optional) [groups], zp [groups],
 * rowsum (optional) [rows] = sum of the row's codes (for the GEMM's
 * zero-point correction). row_ext (optional, per-row modes, bf16 input):
 * records [rows, 2] (min, max) of the float32 smoothed row (x * RN32(1/s)),
 * each (order-preserving key of the value << 32) | c with the extreme
 * element in columns [c, c + 32) (an exact column also qualifies), as produced by
 * moe_w8a8_gemm's SwiGLU epilogue — the kernel then speculates that the two
 * recorded elements are the exact extremes and streams the row once,
 * verifying the speculation while encoding (a failed check re-encodes the
 * row exactly); results are identical either way.
 */
int64_t moe_act_quant_workspace(int64_t rows, int64_t cols, int granularity);
moe_status moe_act_quant(const void* x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx,
                         const int32_t* gather_rows, const double* smooth, const double* smooth_recip,
                         const float* smooth_recip_f32, int smooth_mode, const int32_t* row_group,
                         int bits, int symmetric,
                         int granularity, uint8_t* codes, int64_t ldc, double* scale, float* scale_f32,
                         int32_t* zp, int32_t* rowsum, const unsigned long long* row_ext, void* workspace,
                         int64_t workspace_bytes, moe_stream_t stream);

/* Token-major K1 for the MoE dispatch (rtn_quantize per_token of
 * apply_smoothing's X / s, quant.py:214-231 / 314-324, as moe_act_quant):
 * output row r = token_pos[t * k + j] (t < T, j < k) holds token t of x
 * divided by smoothing row row_group[r]; every output row gets codes, scale,
 * scale_f32, zp and rowsum exactly as moe_act_quant(gather_rows = the
 * inverse of token_pos) would give. x is read from HBM once per token (a
 * token's k rows are encoded by adjacent warps at the same time, or from one
 * warp's registers: MOE_TUNE_K1_TOKENS). Requires bf16 x, cols % 8 == 0,
 * 16-byte aligned rows and the three smoothing tables; MOE_EINVAL otherwise.
 * The register variant is PDL-launched: x must not be written by the
 * immediately preceding kernel of the stream when that kernel triggers its
 * dependents early (none of this library's kernels that do write
 * activations). */
/* K1 with producer records (row_ext, as moe_act_quant(row_ext=...)) whose
 * row count lives on the device: rows r < *rows_dev of the capacity
 * rows_cap are quantized (the expert-parallel receiver, whose row count
 * comes from the device-side exchange plan). bf16 rows, cols % 8 == 0. */
moe_status moe_act_quant_given_dev(const void* x, int x_dtype, int64_t rows_cap, const int32_t* rows_dev,
                                   int64_t cols, int64_t ldx, const double* smooth, const double* smooth_recip,
                                   const float* smooth_recip_f32, const int32_t* row_group, int bits, int symmetric,
                                   uint8_t* codes, int64_t ldc, double* scale, float* scale_f32, int32_t* zp,
                                   int32_t* rowsum, const unsigned long long* row_ext, moe_stream_t stream);

moe_status moe_act_quant_tokens(const void* x, int x_dtype, int64_t T, int64_t cols, int64_t ldx, int k,
                                const int32_t* token_pos, const int32_t* row_group, const double* smooth,
                                const double* smooth_recip, const float* smooth_recip_f32, int bits, int symmetric,
                                uint8_t* codes, int64_t ldc, double* scale, float* scale_f32, int32_t* zp,
                                int32_t* rowsum, moe_stream_t stream);

/* out[i] = RN(1 / s[i]) (float64) and optionally out_f32[i] = RN32(out[i]);
 * feed smooth_recip / smooth_recip_f32. */
moe_status moe_reciprocal_f64(const double* s, int64_t n, double* out, float* out_f32, moe_stream_t stream);

/* dequantize (quant.py:234-240): out = (code - zp) * scale, float64. */
moe_status moe_dequantize(const uint8_t* codes, int64_t rows, int64_t cols, int64_t ldc,
                          const double* scale, const int32_t* zp, int granularity, double* out,
                          moe_stream_t stream);

/* apply_smoothing (quant.py:314-324): ws = w * f (cols), xs = x / f (rows of
 * the channels x tokens matrix). Either side may be NULL. */
moe_status moe_apply_smoothing(const double* w, int64_t R, int64_t n, const double* x, int64_t T,
                               const double* f, double* ws, double* xs, moe_stream_t stream);

/* channel statistics for channel_order (quant.py:346-363) and the smoothing
 * statistic of search_smoothing (quant.py:303): per row of x [n, T]:
 * MAX_ABS -> max |x|, SUM_SQUARES -> sum x^2 (row-order summation). */
moe_status moe_channel_stats(const double* x, int64_t n, int64_t T, int strategy, double* stat,
                             moe_stream_t stream);

/* ---- K2 / K5: W8A8 GEMM on tcgen05 kind::i8 -----------------------------
 * Replaces the fake-quant product of quant_loss (quant.py:281-283) and
 * quantize_layer (quant.py:475-478) with an exact integer product:
 *   acc[m,n] = sum_k (a[m,k] - a_zp[m]) * (w[n,k] - w_zp[n])   (int32, exact)
 * computed as u8*u8 UMMA plus zero-point correction with the code row sums.
 * Epilogues: DEQUANT  out = a_scale[m]*w_scale[n]*acc (+bias[n]) (*row_weight[m])
 *            SWIGLU   W rows interleaved in blocks of 128 (gate, up): out
 *                     [m, N/2] = silu(g) * u of the dequantized pair
 *            ACC_I32  acc_out[m, n] = acc (int32, exact)
 * Grouped (MoE, K5): A rows are grouped by expert; group g owns A rows
 * [group_offsets[g], group_offsets[g+1]) (device array) and W rows
 * [g*N, (g+1)*N) of the stacked weights. group_offsets == NULL -> one group
 * of M rows. K must be a multiple of 16; other shapes use a SIMT path with
 * identical integer results.
 * Fusion with the next K1 (SwiGLU epilogue, tensor-core path): when
 * row_ext [M, 2] is given, the epilogue also emits the (value, 32-column
 * chunk) records of the float32 min and max of each stored output row times the
 * next layer's RN32 reciprocal smoothing (table [G, next_ld]), so that
 * moe_act_quant(row_ext=...) reads h once. */
moe_status moe_w8a8_gemm(const uint8_t* a, int64_t M, int64_t K, int64_t lda, const float* a_scale,
                         const int32_t* a_zp, const int32_t* a_rowsum, const uint8_t* w, int64_t N,
                         int64_t ldw, const float* w_scale, const int32_t* w_zp, const int32_t* w_rowsum,
                         const float* bias, const float* row_weight, const int32_t* group_offsets,
                         int num_groups, int epilogue, void* out, int out_dtype, int64_t ldo,
                         int32_t* acc_out, int64_t ld_acc, const float* next_smooth_recip_f32,
                         int64_t next_ld, unsigned long long* row_ext, moe_stream_t stream);

/* Frobenius-loss reduction for quant_loss (quant.py:283) on the exact
 * accumulators: out = sum_{m,n} (a_scale[m]*w_scale[n]*acc[m,n] - ref[m,n])^2
 * with ref [M, N] float64. Scales are per row (per_tensor: stride 0 via
 * a_scale_stride = 0). Deterministic two-level reduction. */
moe_status moe_quant_sq_error(const int32_t* acc, int64_t M, int64_t N, const double* a_scale,
                              int a_scale_stride, const double* w_scale, const double* ref,
                              double* out, void* workspace, int64_t workspace_bytes, moe_stream_t stream);
int64_t moe_quant_sq_error_workspace(int64_t M, int64_t N);

/* ---- K3: router gating --------------------------------------------------
 * Not in the reference (its only trace of routing is the event format,
 * trace.py:40-44). logits[t, e] = x[t,:] . gate_w[e,:] (float32 accumulate);
 * top-k on logits, ties to the lower expert id, descending order; weights
 * = softmax over the selected logits. gate_bias [E] (optional) is added to the
 * logits. logits may be NULL (not stored). x rows are ldx (>= d) elements
 * apart. */
moe_status moe_router_gate(const void* x, int x_dtype, int64_t T, int64_t d, int64_t ldx, const float* gate_w,
                           const float* gate_bias, int E, int k, float* logits, int32_t* topk_idx,
                           float* topk_w, moe_stream_t stream);
/* top-k only, from given float32 logits [T, E]. */
/* Tensor-core K3: the same routing with logits from tcgen05.mma kind::f16
 * (x bf16 [T, d], d % 64 == 0, E <= 16). The float32 gate is first split
 * by moe_router_prepare into three bf16 pieces (hi + mid + lo = the exact
 * float32 value) in a caller buffer of moe_router_tc_workspace(d) bytes;
 * each product with a piece is exact and all accumulate in float32. */
int64_t moe_router_tc_workspace(int64_t d);
moe_status moe_router_prepare(const float* gate_w, int E, int64_t d, void* pieces, moe_stream_t stream);
moe_status moe_router_gate_tc(const void* x, int64_t T, int64_t d, int64_t ldx, const void* pieces,
                              const float* gate_bias, int E, int k, float* logits, int32_t* topk_idx,
                              float* topk_w, moe_stream_t stream);
moe_status moe_router_topk(const float* logits, int64_t T, int E, int k, int32_t* topk_idx, float* topk_w,
                           moe_stream_t stream);

/* ---- K4: token -> expert permutation (stable counting sort) -------------
 * expert_offsets [E+1]; for permuted row p: src_token[p], row_expert[p],
 * row_weight[p] (= topk_w of that pair, optional); token_pos[t*k+j] = p. */
int64_t moe_route_permute_workspace(int64_t T, int k, int E);
moe_status moe_route_permute(const int32_t* topk_idx, const float* topk_w, int64_t T, int k, int E,
                             int32_t* expert_offsets, int32_t* src_token, int32_t* row_expert,
                             float* row_weight, int32_t* token_pos, void* workspace,
                             int64_t workspace_bytes, moe_stream_t stream);

/* ---- K6: combine ----------------------------------------------------------
 * out[t, :] = sum_j y[token_pos[t*k+j], :] (row weights already applied by
 * the GEMM epilogue), summed in slot order j = 0..k-1 in float32. y rows are
 * contiguous [T*k, d]; out rows are ldo (>= d) elements apart. */
moe_status moe_combine(const void* y, int y_dtype, const int32_t* token_pos, int64_t T, int k, int64_t d,
                       void* out, int out_dtype, int64_t ldo, moe_stream_t stream);

/* ---- routing statistics (trace.expert_freq, trace.py:216-225) -----------
 * counts[layer*E + e] += number of (t, j) with topk_idx[t, j] == e. Path
 * keys for trace.path_stats (trace.py:207-213): path_codes[t] for this layer
 * = ascending pair of ids packed as lo*E + hi (k == 2) or a bitmask (k > 2). */
moe_status moe_expert_histogram(const int32_t* topk_idx, int64_t T, int k, int E, int layer,
                                int64_t* counts, int32_t* path_codes, moe_stream_t stream);

/* ---- K7: Hessian accumulation (build_hessian, quant.py:327-343) ----------
 * H[n, n] += 2 * xs^T xs over a tokens-major batch x [T, n] (xs = x / s when
 * smooth != NULL, exact division). Finalize symmetrises, adds
 * damping_fraction * mean(diag) on the diagonal and reports an all-zero
 * calibration (EDEGENERATE) via the nonzero counter. */
moe_status moe_hessian_accum(const void* x, int x_dtype, int64_t T, int64_t n, int64_t ldx,
                             const double* smooth, const double* smooth_recip, double* H,
                             unsigned long long* nonzero_count, moe_stream_t stream);
moe_status moe_hessian_finalize(double* H, int64_t n, double damping_fraction,
                                const unsigned long long* nonzero_count, moe_stream_t stream);

/* ---- K8: compensated column loop (hessian_quantize, quant.py:415-434) ----
 * W [R, n] float64 in the ORIGINAL column order (read-only); column i of
 * the loop is W[:, order[i]] (order NULL -> identity); U [n, n] is the upper
 * factor of the PERMUTED H^-1 (quant.py:366-385, 418-420). Per-row params
 * scale/zp are fixed for the loop (quant.py:415). Exactly the reference's
 * operation order per element: encode column i, err = (w_i - (c - zp)*scale)
 * / U_ii, then w_j = w_j - err*U_ij (separate multiply and subtract,
 * ascending i) -> bit-identical codes, written back to the original column
 * positions codes[r, order[i]] (quant.py:432-433). err_ws: workspace of
 * moe_gptq_workspace() bytes. */
int64_t moe_gptq_workspace(int64_t R, int64_t n);
moe_status moe_gptq_columns(const double* W, int64_t R, int64_t n, int64_t ldw, const int32_t* order,
                            const double* U, const double* scale, const int32_t* zp, int bits,
                            uint8_t* codes, int64_t ldc, void* err_ws, int64_t err_ws_bytes,
                            moe_stream_t stream);

/* ---- expert-parallel plumbing (no reference counterpart:
 * the reference has no forward, placement.py:1-256 only plans residency) --
 * route_keys: keys[i] = dest_rank[topk_idx[i]] * E + topk_idx[i], the sort
 *   key of moe_route_permute(E' = world * E) that makes each destination's
 *   rows contiguous and expert-sorted within it.
 * gather_rows: dst row r = src row index[r] (index NULL -> identity), rows
 *   of row_bytes bytes (16-byte vectors when aligned).
 * ep_pack_params: params[n, 4] int32 = (scale_f32 bits, zp, rowsum, weight
 *   bits; weight NULL -> 1.0f), the per-row sidecar of dispatched codes.
 * ep_unpack_params: SoA scale_f32/zp/rowsum/weight of params[index[r]] for
 *   r < n (r < min(n, *n_dev) with a device row count). */
moe_status moe_route_keys(const int32_t* topk_idx, int64_t n, const int32_t* dest_rank, int E, int32_t* keys,
                          moe_stream_t stream);
moe_status moe_gather_rows(const void* src, int64_t src_ld_bytes, const int32_t* index, int64_t n,
                           int64_t row_bytes, void* dst, int64_t dst_ld_bytes, moe_stream_t stream);
moe_status moe_ep_pack_params(const float* scale_f32, const int32_t* zp, const int32_t* rowsum,
                              const float* weight, int64_t n, int32_t* params, moe_stream_t stream);
moe_status moe_ep_unpack_params(const int32_t* params, const int32_t* index, int64_t n, const int32_t* n_dev,
                                float* scale_f32, int32_t* zp, int32_t* rowsum, float* weight, moe_stream_t stream);

/* Fused expert-parallel transport (peer memory over NVLink instead of an
 * NCCL all-to-all; buffers from torch symmetric memory):
 * act_quant_dispatch: K1 on gathered rows (as moe_act_quant per_token with
 *   gather_rows / row_group) writing each row's codes straight into
 *   codes_tab[dst_rank[r]] + dst_row[r] * ldc and its 16-byte sidecar
 *   (scale_f32, zp, rowsum, routing weight) into params_tab[...][dst_row[r]].
 * w8a8_gemm_scatter: moe_w8a8_gemm (DEQUANT) whose output row m is stored at
 *   out_tab[out_rank[m]] + out_row[m] * ldo (the combine's home buffers).
 *   With token_pos (output row of token t's j-th selection, rows = T * k)
 *   x is read once per token (token-major K1, as moe_act_quant_tokens);
 *   rows whose dst_rank is negative (refused plan) are skipped.
 * block_map: for rows in contiguous blocks [block_start[b], block_start[b+1]),
 *   out0[i] = val0[b], out1[i] = val1[b] + i - block_start[b], out2[i] =
 *   val2[b] (optional): the destination rank / row (and local expert) of
 *   every dispatched or returned row; i < n, or i < min(n, *n_dev) with a
 *   device row count; valid (optional, device): *valid == 0 makes every
 *   out0 -1.
 * ep_peer_plan: the exchange plan of one peer-memory EP forward computed on
 *   the device (no host round trip): from every rank's route_permute
 *   offsets over its W*E keys (offsets_all [W, W*E+1], key r*E + e = rows
 *   for expert e served by rank r, gathered by one all-gather), this
 *   rank's (me) send bases, receive blocks and grouped-GEMM offsets of its
 *   G local experts (local, ascending). plan (moe_ep_peer_plan_size ints):
 *   [valid, R, send_base[W*E], starts[G*W+1], ranks[G*W], homes[G*W],
 *   group[G*W], goff[G+1]]; valid = 0 (and R = 0) when some rank would
 *   receive more than cap rows, route more than cap_home rows, or this rank
 *   receives rows for an expert it does not hold. host_flag (optional,
 *   pinned host memory) receives valid too, stored by the kernel through
 *   the host mapping (no copy-engine transfer that could queue behind bulk
 *   D2H copies of other streams). */
moe_status moe_act_quant_dispatch(const void* x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx,
                                  const int32_t* gather_rows, const int32_t* token_pos, int k,
                                  const double* smooth, const double* smooth_recip,
                                  const float* smooth_recip_f32, const int32_t* row_group, int bits, int symmetric,
                                  void* const* codes_tab, void* const* params_tab, const int32_t* dst_rank,
                                  const int32_t* dst_row, const float* row_weight, int64_t ldc, moe_stream_t stream);
int64_t moe_ep_peer_plan_size(int W, int E, int G);
moe_status moe_ep_peer_plan(const int32_t* offsets_all, int W, int E, int me, const int32_t* local, int G,
                            int64_t cap, int64_t cap_home, int32_t* plan, int32_t* host_flag, moe_stream_t stream);
moe_status moe_block_map(int64_t n, const int32_t* n_dev, int nblocks, const int32_t* block_start,
                         const int32_t* val0, const int32_t* val1, const int32_t* val2, const int32_t* valid,
                         int32_t* out0, int32_t* out1, int32_t* out2, moe_stream_t stream);
moe_status moe_w8a8_gemm_scatter(const uint8_t* a, int64_t M, int64_t K, int64_t lda, const float* a_scale,
                                 const int32_t* a_zp, const int32_t* a_rowsum, const uint8_t* w, int64_t N,
                                 int64_t ldw, const float* w_scale, const int32_t* w_zp, const int32_t* w_rowsum,
                                 const float* bias, const float* row_weight, const int32_t* group_offsets,
                                 int num_groups, int epilogue, void* const* out_tab, const int32_t* out_rank,
                                 const int32_t* out_row, int out_dtype, int64_t ldo, moe_stream_t stream);
/* GEMM2 with its A operand's K1 fused in (MoE second grouped GEMM; replaces
 * moe_act_quant(row_ext=...) followed by moe_w8a8_gemm). x [M, K] bf16 (the
 * SwiGLU output h, ld ldx) is quantized per row exactly as moe_act_quant
 * with smoothing table rows row_group[m] and the producer records row_ext,
 * by the GEMM's epilogue warps while they wait for accumulators; the TMA
 * producer loads an A block once its rows are complete. Outputs: the codes
 * a [M, lda], a_scale64 / a_scale / a_zp / a_rowsum (as moe_act_quant) and
 * out (as moe_w8a8_gemm with the DEQUANT epilogue). Bit-identical to the
 * two separate calls. workspace: moe_w8a8_gemm_quant_a_workspace(M) bytes
 * (zeroed by the call). */
int64_t moe_w8a8_gemm_quant_a_workspace(int64_t M);
moe_status moe_w8a8_gemm_quant_a(const void* x, int64_t ldx, const double* smooth, const double* smooth_recip,
                                 const float* smooth_recip_f32, const int32_t* row_group,
                                 const unsigned long long* row_ext, uint8_t* a, int64_t lda, double* a_scale64,
                                 float* a_scale, int32_t* a_zp, int32_t* a_rowsum, int64_t M, int64_t K,
                                 const uint8_t* w, int64_t N, int64_t ldw, const float* w_scale, const int32_t* w_zp,
                                 const int32_t* w_rowsum, const float* bias, const float* row_weight,
                                 const int32_t* group_offsets, int num_groups, int epilogue, void* out,
                                 int out_dtype, int64_t ldo, void* workspace, int64_t workspace_bytes,
                                 moe_stream_t stream);
/* GEMM2 with the top-2 combine fused in (replaces moe_w8a8_gemm(DEQUANT,
 * bf16) followed by moe_combine for k == 2). A rows are the M = 2T
 * expert-sorted (token, slot) rows, src_token [M] their tokens, token_pos
 * [T, 2] each token's two rows. Per 32-column chunk, the first of a token's
 * two rows to finish stores its bf16 values in y [M, ldy] (scratch) and the
 * second adds them to its own ((0 + mine) + partner in float, which is the
 * combine kernel's sum: two-term addition commutes) and writes out [T, ldo]
 * bf16. Bit-identical to the two separate calls; y is only partly written.
 * workspace: moe_w8a8_gemm_combine_workspace(T, N) bytes (zeroed by the
 * call unless MOE_EPI_FLAG_WS_ZEROED). */
int64_t moe_w8a8_gemm_combine_workspace(int64_t T, int64_t N);
/* One kernel preparing a layer step's scratch ahead of its PDL-chained
 * kernels: zeroes `zero_bytes` (multiple of 16, 16-byte aligned) at `zero`
 * (the combine workspace; may be NULL) and sets `rows` extreme records of
 * row_ext (may be NULL) to (min = ~0, max = 0) for moe_w8a8_gemm with
 * MOE_EPI_FLAG_EXT_READY. */
moe_status moe_step_init(void* zero, int64_t zero_bytes, unsigned long long* row_ext, int64_t rows,
                         moe_stream_t stream);
moe_status moe_w8a8_gemm_combine(const uint8_t* a, int64_t M, int64_t K, int64_t lda, const float* a_scale,
                                 const int32_t* a_zp, const int32_t* a_rowsum, const uint8_t* w, int64_t N,
                                 int64_t ldw, const float* w_scale, const int32_t* w_zp, const int32_t* w_rowsum,
                                 const float* row_weight, const int32_t* group_offsets, int num_groups,
                                 int epilogue, void* y, int64_t ldy, const int32_t* src_token,
                                 const int32_t* token_pos, int64_t T, void* out, int64_t ldo, void* workspace,
                                 int64_t workspace_bytes, moe_stream_t stream);
/* MoE stack block glue (SURVEY.md C5 token path, pre-norm residual blocks):
 * s = bf16(x + y) (y == NULL: s = x), written to x_out when y is given, and
 * norm_out = bf16(s * rsqrt(mean(s^2) + eps)) (float32, fixed reduction
 * order per row; norm_out may be NULL). bf16 rows [T, d], d % 8 == 0,
 * d <= 8192, contiguous. */
moe_status moe_rmsnorm_residual(const void* x, const void* y, void* x_out, void* norm_out, int64_t T, int64_t d,
                                float eps, moe_stream_t stream);
/* Attention block glue (C5 token path): rotary position embedding in place
 * on `heads` heads of head_dim bf16 values at the start of each row of x
 * [T, ld] (rotate-half pairs (i, i + head_dim/2)); position of row t =
 * positions[t] (NULL: t); cos_tab / sin_tab float32 [max_pos, head_dim/2]
 * (cos / sin of position * theta^(-2i/head_dim), built in float64 by the
 * caller). head_dim % 16 == 0, 16-byte aligned rows. */
moe_status moe_rope_bf16(void* x, int64_t T, int heads, int head_dim, int64_t ld, const int32_t* positions,
                         const float* cos_tab, const float* sin_tab, moe_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* MOE_B200_H */
