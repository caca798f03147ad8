// K1 — smoothing + RTN affine quantization with moekit's exact float64
// semantics (quant.py:191-231, 314-324), plus the small elementwise pieces
// of the quantizer API: dequantize, apply_smoothing, channel statistics and
// reciprocal tables.
//
// Two kernels produce identical results:
//  * act_quant_fast.cu — the hot path (bf16 activations, per-token groups):
//    TMA-staged rows, float32 filter, float64 only where it can matter;
//  * act_quant_rows_kernel / per-tensor kernels here — the general exact
//    path for any input dtype (fp64 weights and calibration data, fp32,
//    fp16), any smoothing mode, and the per_tensor granularity.
#include <algorithm>

#include "k1_common.cuh"

namespace moe {

constexpr int kQuantThreads = 256;

// Pass 1 of the exact path: min/max of the smoothed row in float64.
__device__ __forceinline__ void row_minmax(const RowArgs& a, const RowView& v, double& mn, double& mx) {
  mn = DBL_MAX;
  mx = -DBL_MAX;
  for (int64_t j = threadIdx.x; j < a.cols; j += blockDim.x) {
    const double xs = smooth_value(load_as_f64(a.x, v.off + j, a.dt), a.sm, v.gbase, j);
    mn = fmin(mn, xs);
    mx = fmax(mx, xs);
  }
}

// Pass 2 of the exact path: encode with fixed params; returns the code sum.
__device__ __forceinline__ int64_t row_encode(const RowArgs& a, const RowView& v, const AffineParams& p, int qmax,
                                              uint8_t* out) {
  int64_t sum = 0;
  for (int64_t j = threadIdx.x; j < a.cols; j += blockDim.x) {
    const double xs = smooth_value(load_as_f64(a.x, v.off + j, a.dt), a.sm, v.gbase, j);
    const int code = encode_code(xs, p.scale, p.rscale, p.zp, qmax);
    sum += code;
    out[j] = (uint8_t)code;
  }
  return sum;
}

__device__ __forceinline__ void store_row_params(int64_t g, const AffineParams& p, double* scale, float* scale_f32,
                                                 int32_t* zp) {
  scale[g] = p.scale;
  if (scale_f32) scale_f32[g] = (float)p.scale;
  zp[g] = p.zp;
}

__global__ void __launch_bounds__(kQuantThreads) act_quant_rows_kernel(RowArgs a, int bits, int sym,
                                                                       uint8_t* codes, int64_t ldc,
                                                                       double* scale, float* scale_f32,
                                                                       int32_t* zp, int32_t* rowsum) {
  __shared__ double shd[kQuantThreads / 32];
  __shared__ int64_t shi[kQuantThreads / 32];
  const int64_t r = blockIdx.x;
  const RowView v = row_view(a, r);
  double mn, mx;
  row_minmax(a, v, mn, mx);
  mn = block_reduce(mn, shd, OpMin());
  mx = block_reduce(mx, shd, OpMax());
  const AffineParams p = affine_params(mn, mx, bits, sym);
  const int64_t s = row_encode(a, v, p, (1 << bits) - 1, codes + r * ldc);
  const int64_t t = rowsum ? block_reduce(s, shi, OpAdd()) : 0;
  if (threadIdx.x == 0) {
    if (rowsum) rowsum[r] = (int32_t)t;
    store_row_params(r, p, scale, scale_f32, zp);
  }
}

// per_tensor: global min/max by order-preserving atomics, then encode
__global__ void minmax_init_kernel(long long* ws) {
  ws[0] = 0x7FFFFFFFFFFFFFFFLL;
  ws[1] = (long long)0x8000000000000000ULL;
}

__global__ void __launch_bounds__(kQuantThreads) tensor_minmax_kernel(RowArgs a, long long* ws) {
  __shared__ double shd[kQuantThreads / 32];
  double mn, mx;
  row_minmax(a, row_view(a, blockIdx.x), mn, mx);
  mn = block_reduce(mn, shd, OpMin());
  mx = block_reduce(mx, shd, OpMax());
  if (threadIdx.x == 0) {
    atomicMin(&ws[0], dkey(mn));
    atomicMax(&ws[1], dkey(mx));
  }
}

__global__ void __launch_bounds__(kQuantThreads) tensor_encode_kernel(RowArgs a, const long long* ws, int bits,
                                                                      int sym, uint8_t* codes, int64_t ldc,
                                                                      double* scale, float* scale_f32,
                                                                      int32_t* zp, int32_t* rowsum) {
  __shared__ int64_t shi[kQuantThreads / 32];
  const int64_t r = blockIdx.x;
  const AffineParams p = affine_params(dunkey(ws[0]), dunkey(ws[1]), bits, sym);
  const int64_t s = row_encode(a, row_view(a, r), p, (1 << bits) - 1, codes + r * ldc);
  const int64_t t = rowsum ? block_reduce(s, shi, OpAdd()) : 0;
  if (threadIdx.x == 0) {
    if (rowsum) rowsum[r] = (int32_t)t;
    if (r == 0) store_row_params(0, p, scale, scale_f32, zp);
  }
}

__global__ void reciprocal_kernel(const double* s, int64_t n, double* out, float* out32) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double r = __drcp_rn(s[i]);
    out[i] = r;
    if (out32) out32[i] = __double2float_rn(r);
  }
}

__global__ void dequant_kernel(const uint8_t* codes, int64_t rows, int64_t cols, int64_t ldc, const double* scale,
                               const int32_t* zp, int per_row, double* out) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    const int64_t g = per_row ? r : 0;
    out[i] = __dmul_rn(__dsub_rn((double)codes[r * ldc + c], (double)zp[g]), scale[g]);
  }
}

__global__ void smooth_w_kernel(const double* w, int64_t R, int64_t n, const double* f, double* ws) {
  const int64_t total = R * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    ws[i] = __dmul_rn(w[i], f[i % n]);
}
__global__ void smooth_x_kernel(const double* x, int64_t n, int64_t T, const double* f, double* xs) {
  const int64_t total = n * T;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
    xs[i] = __ddiv_rn(x[i], f[i / T]);
}

// one CTA per channel row of x [n, T]; fixed tree order for the sums
__global__ void __launch_bounds__(256) channel_stats_kernel(const double* x, int64_t T, int strategy,
                                                            double* stat) {
  __shared__ double sh[256];
  const double* row = x + blockIdx.x * T;
  double acc = 0.0;
  if (strategy == MOE_ORDER_MAX_ABS) {
    for (int64_t j = threadIdx.x; j < T; j += blockDim.x) acc = fmax(acc, fabs(row[j]));
  } else {
    for (int64_t j = threadIdx.x; j < T; j += blockDim.x) acc = __dadd_rn(acc, __dmul_rn(row[j], row[j]));
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s)
      sh[threadIdx.x] = strategy == MOE_ORDER_MAX_ABS ? fmax(sh[threadIdx.x], sh[threadIdx.x + s])
                                                      : __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) stat[blockIdx.x] = sh[0];
}

static int grid_for(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 16;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace moe

using namespace moe;

extern "C" int64_t moe_act_quant_workspace(int64_t rows, int64_t cols, int granularity) {
  (void)rows;
  (void)cols;
  return granularity == MOE_GRAN_PER_TENSOR ? 2 * (int64_t)sizeof(long long) : 0;
}

extern "C" moe_status moe_act_quant(const void* x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx,
                                    const int32_t* gather_rows, const double* smooth, const double* smooth_recip,
                                    const float* smooth_recip_f32, int smooth_mode, const int32_t* row_group,
                                    int bits, int symmetric, int granularity, uint8_t* codes, int64_t ldc,
                                    double* scale, float* scale_f32, int32_t* zp, int32_t* rowsum,
                                    const unsigned long long* row_ext, void* workspace, int64_t workspace_bytes,
                                    moe_stream_t stream) {
  MOE_REQUIRE(x && codes && scale && zp, "act_quant: null pointer");
  MOE_REQUIRE(rows >= 1 && cols >= 1, "act_quant: matrix must be non-empty");
  MOE_REQUIRE(ldx >= cols && ldc >= cols, "act_quant: bad leading dimension");
  MOE_REQUIRE(bits >= 2 && bits <= 8, "bits must be in [2, 8]");
  MOE_REQUIRE(x_dtype == MOE_DT_F32 || x_dtype == MOE_DT_F64 || x_dtype == MOE_DT_BF16 || x_dtype == MOE_DT_F16,
              "act_quant: unsupported input dtype");
  MOE_REQUIRE(smooth_mode == MOE_SMOOTH_NONE || smooth, "act_quant: smoothing table missing");
  MOE_REQUIRE(granularity >= 0 && granularity <= 2, "act_quant: unknown granularity");
  const RowArgs a{x, x_dtype, rows, cols, ldx, gather_rows, row_group,
                  SmoothArgs{smooth, smooth_recip, smooth_mode, cols}};
  cudaStream_t s = as_stream(stream);
  if (granularity == MOE_GRAN_PER_TENSOR) {
    MOE_REQUIRE(workspace && workspace_bytes >= 16, "act_quant: per_tensor needs 16 B of workspace");
    long long* ws = static_cast<long long*>(workspace);
    minmax_init_kernel<<<1, 1, 0, s>>>(ws); ::moe::count_launch();
    tensor_minmax_kernel<<<(unsigned)rows, kQuantThreads, 0, s>>>(a, ws); ::moe::count_launch();
    tensor_encode_kernel<<<(unsigned)rows, kQuantThreads, 0, s>>>(a, ws, bits, symmetric, codes, ldc, scale,
                                                                   scale_f32, zp, rowsum); ::moe::count_launch();
  } else if (row_ext) {
    cudaError_t err = cudaSuccess;
    MOE_REQUIRE(launch_act_quant_given(a, smooth_recip_f32, row_ext, bits, symmetric, codes, ldc, scale,
                                       scale_f32, zp, rowsum, s, &err),
                "act_quant: row_ext needs bf16 rows (cols % 8 == 0) and float32 reciprocals");
    MOE_CUDA_TRY(err);
  } else {
    cudaError_t err = cudaSuccess;
    if (launch_act_quant_fast(a, smooth_recip_f32, bits, symmetric, codes, ldc, scale, scale_f32, zp, rowsum, s,
                              &err)) {
      MOE_CUDA_TRY(err);
    } else {
      act_quant_rows_kernel<<<(unsigned)rows, kQuantThreads, 0, s>>>(a, bits, symmetric, codes, ldc, scale,
                                                                      scale_f32, zp, rowsum); ::moe::count_launch();
    }
  }
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_act_quant_tokens(const void* x, int x_dtype, int64_t T, int64_t cols, int64_t ldx, int k,
                                           const int32_t* token_pos, const int32_t* row_group, const double* smooth,
                                           const double* smooth_recip, const float* smooth_recip_f32, int bits,
                                           int symmetric, uint8_t* codes, int64_t ldc, double* scale,
                                           float* scale_f32, int32_t* zp, int32_t* rowsum, moe_stream_t stream) {
  MOE_REQUIRE(x && token_pos && smooth && smooth_recip && smooth_recip_f32 && codes && scale && zp,
              "act_quant_tokens: null pointer");
  MOE_REQUIRE(T >= 1 && k >= 1 && cols >= 1 && ldx >= cols && ldc >= cols, "act_quant_tokens: bad shape");
  MOE_REQUIRE(bits >= 2 && bits <= 8, "bits must be in [2, 8]");
  const RowArgs a{x, x_dtype, T * k, cols, ldx, nullptr, row_group,
                  SmoothArgs{smooth, smooth_recip, MOE_SMOOTH_DIVIDE, cols}};
  cudaError_t err = cudaSuccess;
  MOE_REQUIRE(launch_act_quant_tokens(a, token_pos, k, T, smooth_recip_f32, bits, symmetric, codes, ldc, scale,
                                      scale_f32, zp, rowsum, as_stream(stream), &err),
              "act_quant_tokens: needs bf16 x with cols % 8 == 0 and 16-byte aligned rows");
  MOE_CUDA_TRY(err);
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_reciprocal_f64(const double* sv, int64_t n, double* out, float* out_f32,
                                         moe_stream_t stream) {
  MOE_REQUIRE(sv && out && n >= 1, "reciprocal: bad arguments");
  reciprocal_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(sv, n, out, out_f32); ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_dequantize(const uint8_t* codes, int64_t rows, int64_t cols, int64_t ldc,
                                     const double* scale, const int32_t* zp, int granularity, double* out,
                                     moe_stream_t stream) {
  MOE_REQUIRE(codes && scale && zp && out && rows >= 1 && cols >= 1 && ldc >= cols, "dequantize: bad arguments");
  dequant_kernel<<<grid_for(rows * cols, 256), 256, 0, as_stream(stream)>>>(
      codes, rows, cols, ldc, scale, zp, granularity != MOE_GRAN_PER_TENSOR, out); ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_apply_smoothing(const double* w, int64_t R, int64_t n, const double* x, int64_t T,
                                          const double* f, double* ws, double* xs, moe_stream_t stream) {
  MOE_REQUIRE(f && n >= 1, "apply_smoothing: bad arguments");
  cudaStream_t s = as_stream(stream);
  if (w) {
    MOE_REQUIRE(ws && R >= 1, "apply_smoothing: bad weight arguments");
    smooth_w_kernel<<<grid_for(R * n, 256), 256, 0, s>>>(w, R, n, f, ws); ::moe::count_launch();
  }
  if (x) {
    MOE_REQUIRE(xs && T >= 1, "apply_smoothing: bad activation arguments");
    smooth_x_kernel<<<grid_for(n * T, 256), 256, 0, s>>>(x, n, T, f, xs); ::moe::count_launch();
  }
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_channel_stats(const double* x, int64_t n, int64_t T, int strategy, double* stat,
                                        moe_stream_t stream) {
  MOE_REQUIRE(x && stat && n >= 1 && T >= 1, "channel_stats: bad arguments");
  MOE_REQUIRE(strategy == MOE_ORDER_MAX_ABS || strategy == MOE_ORDER_SUM_SQUARES, "channel_stats: bad strategy");
  channel_stats_kernel<<<(unsigned)n, 256, 0, as_stream(stream)>>>(x, T, strategy, stat); ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_act_quant_dispatch(const void* x, int x_dtype, int64_t rows, int64_t cols, int64_t ldx,
                                             const int32_t* gather_rows, const int32_t* token_pos, int k,
                                             const double* smooth, const double* smooth_recip,
                                             const float* smooth_recip_f32, const int32_t* row_group, int bits,
                                             int symmetric, void* const* codes_tab, void* const* params_tab,
                                             const int32_t* dst_rank, const int32_t* dst_row, const float* row_weight,
                                             int64_t ldc, moe_stream_t stream) {
  MOE_REQUIRE(x && (gather_rows || token_pos) && codes_tab && params_tab && dst_rank && dst_row,
              "act_quant_dispatch: null pointer");
  MOE_REQUIRE(rows >= 1 && cols >= 1 && ldx >= cols && ldc >= cols, "act_quant_dispatch: bad sizes");
  MOE_REQUIRE(x_dtype == MOE_DT_BF16 && smooth && smooth_recip && smooth_recip_f32,
              "act_quant_dispatch: bf16 rows with divide-smoothing tables (f64, RN(1/s) and its f32 copy)");
  MOE_REQUIRE(bits >= 2 && bits <= 8, "bits must be in [2, 8]");
  MOE_REQUIRE(!token_pos || (k >= 1 && rows % k == 0), "act_quant_dispatch: rows must be T * k");
  RowArgs a{x, x_dtype, rows, cols, ldx, token_pos ? nullptr : gather_rows, row_group,
            SmoothArgs{smooth, smooth_recip, MOE_SMOOTH_DIVIDE, cols}};
  a.ep = EpOut{reinterpret_cast<uint8_t* const*>(codes_tab), reinterpret_cast<int4* const*>(params_tab), dst_rank,
               dst_row, row_weight};
  cudaError_t err = cudaSuccess;
  // token-major (x read once per token) when token_pos is given and x fits
  // the register-resident kernel; else one warp per gathered row
  if (token_pos && launch_act_quant_tokens(a, token_pos, k, rows / k, smooth_recip_f32, bits, symmetric, nullptr,
                                           ldc, nullptr, nullptr, nullptr, nullptr, as_stream(stream), &err)) {
    MOE_CUDA_TRY(err);
    return MOE_OK;
  }
  MOE_REQUIRE(gather_rows, "act_quant_dispatch: token-major K1 not eligible and no gather_rows given");
  a.gather = gather_rows;
  MOE_REQUIRE(launch_act_quant_fast(a, smooth_recip_f32, bits, symmetric, nullptr, ldc, nullptr, nullptr, nullptr,
                                    nullptr, as_stream(stream), &err),
              "act_quant_dispatch: needs cols % 8 == 0 and 16-byte aligned rows");
  MOE_CUDA_TRY(err);
  return MOE_OK;
}

extern "C" moe_status moe_act_quant_given_dev(const void* x, int x_dtype, int64_t rows_cap, const int32_t* rows_dev,
                                              int64_t cols, int64_t ldx, const double* smooth,
                                              const double* smooth_recip, const float* smooth_recip_f32,
                                              const int32_t* row_group, int bits, int symmetric, uint8_t* codes,
                                              int64_t ldc, double* scale, float* scale_f32, int32_t* zp,
                                              int32_t* rowsum, const unsigned long long* row_ext,
                                              moe_stream_t stream) {
  MOE_REQUIRE(x && rows_dev && row_ext && codes && scale && zp && smooth && smooth_recip && smooth_recip_f32,
              "act_quant_given_dev: null pointer");
  MOE_REQUIRE(rows_cap >= 1 && cols >= 1 && ldx >= cols && ldc >= cols, "act_quant_given_dev: bad sizes");
  MOE_REQUIRE(bits >= 2 && bits <= 8, "bits must be in [2, 8]");
  RowArgs a{x, x_dtype, rows_cap, cols, ldx, nullptr, row_group,
            SmoothArgs{smooth, smooth_recip, MOE_SMOOTH_DIVIDE, cols}};
  a.rows_dev = rows_dev;
  cudaError_t err = cudaSuccess;
  MOE_REQUIRE(launch_act_quant_given(a, smooth_recip_f32, row_ext, bits, symmetric, codes, ldc, scale, scale_f32, zp,
                                     rowsum, as_stream(stream), &err),
              "act_quant_given_dev: needs bf16 rows (cols % 8 == 0, 16-byte aligned) and float32 reciprocals");
  MOE_CUDA_TRY(err);
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}
