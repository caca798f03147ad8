// K1 — smoothing + RTN affine quantization with moekit's exact float64
// semantics (quant.py:191-231, 314-324), plus the small elementwise pieces
// of the quantizer API: dequantize, apply_smoothing, channel statistics and
// reciprocal tables.
//
// Layout: one CTA per output row (rows are tokens for activations, output
// channels for weights). Pass 1 streams the row, applies the smoothing
// division (reciprocal-and-correct, exact) and reduces min/max in float64;
// pass 2 re-reads the row (L1/L2-resident) and encodes. HBM traffic is one
// read of x and one write of the codes.
#include <cfloat>

#include "common.cuh"

namespace moe {

constexpr int kQuantThreads = 256;

struct SmoothArgs {
  const double* s;
  const double* rs;
  int mode;
  int64_t cols;
};

__device__ __forceinline__ double smooth_value(double x, const SmoothArgs& sa, int64_t gbase, int64_t j) {
  if (sa.mode == MOE_SMOOTH_DIVIDE) {
    const double s = sa.s[gbase + j];
    return sa.rs ? div_rcp(x, s, sa.rs[gbase + j]) : __ddiv_rn(x, s);
  }
  if (sa.mode == MOE_SMOOTH_MULTIPLY) return __dmul_rn(x, sa.s[gbase + j]);
  return x;
}

template <typename T>
__device__ __forceinline__ double block_reduce_min(T v, T* sh) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = sh[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) v = fmin(v, sh[i]);
  return v;
}
template <typename T>
__device__ __forceinline__ double block_reduce_max(T v, T* sh) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = sh[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) v = fmax(v, sh[i]);
  return v;
}
__device__ __forceinline__ int64_t block_reduce_sum_i64(int64_t v, int64_t* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  int64_t t = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
  return t;
}

// order-preserving int64 key of a double (for atomic min/max)
__device__ __forceinline__ long long dkey(double d) {
  long long i = __double_as_longlong(d);
  return i >= 0 ? i : (i ^ 0x7FFFFFFFFFFFFFFFLL);
}
__device__ __forceinline__ double dunkey(long long k) {
  return __longlong_as_double(k >= 0 ? k : (k ^ 0x7FFFFFFFFFFFFFFFLL));
}

struct RowArgs {
  const void* x;
  int dt;
  int64_t rows, cols, ldx;
  const int32_t* gather;
  const int32_t* group;
  SmoothArgs sm;
};

// Generic element access: x value of output row r, column j (as float64).
struct RowView {
  const void* base;
  int dt;
  int64_t off;
  int64_t gbase;
};

__device__ __forceinline__ RowView row_view(const RowArgs& a, int64_t r) {
  const int64_t src = a.gather ? (int64_t)a.gather[r] : r;
  const int64_t g = a.group ? (int64_t)a.group[r] : 0;
  return RowView{a.x, a.dt, src * a.ldx, g * a.sm.cols};
}

// Pass 1: min/max of the smoothed row. Vectorised for bf16 (8 per 16 B).
__device__ __forceinline__ void row_minmax(const RowArgs& a, const RowView& v, double& mn, double& mx) {
  mn = DBL_MAX;
  mx = -DBL_MAX;
  const bool vec = a.dt == MOE_DT_BF16 && (a.cols % 8 == 0) && (a.ldx % 8 == 0) &&
                   ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
  if (vec) {
    const uint4* p = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.x) + v.off);
    for (int64_t c = threadIdx.x; c < a.cols / 8; c += blockDim.x) {
      const uint4 u = p[c];
      const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const double xs = smooth_value((double)__bfloat162float(h[e]), a.sm, v.gbase, c * 8 + e);
        mn = fmin(mn, xs);
        mx = fmax(mx, xs);
      }
    }
  } else {
    for (int64_t j = threadIdx.x; j < a.cols; j += blockDim.x) {
      const double xs = smooth_value(load_as_f64(a.x, v.off + j, a.dt), a.sm, v.gbase, j);
      mn = fmin(mn, xs);
      mx = fmax(mx, xs);
    }
  }
}

// Pass 2: encode the row with fixed params; returns this thread's code sum.
__device__ __forceinline__ int64_t row_encode(const RowArgs& a, const RowView& v, const AffineParams& p,
                                              int qmax, uint8_t* out) {
  int64_t sum = 0;
  const bool vec = a.dt == MOE_DT_BF16 && (a.cols % 8 == 0) && (a.ldx % 8 == 0) &&
                   ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(out) & 7) == 0);
  if (vec) {
    const uint4* src = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.x) + v.off);
    uint2* dst = reinterpret_cast<uint2*>(out);
    for (int64_t c = threadIdx.x; c < a.cols / 8; c += blockDim.x) {
      const uint4 u = src[c];
      const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u);
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const double xs = smooth_value((double)__bfloat162float(h[e]), a.sm, v.gbase, c * 8 + e);
        const uint32_t code = (uint32_t)encode_code(xs, p.scale, p.rscale, p.zp, qmax);
        sum += code;
        if (e < 4) lo |= code << (8 * e);
        else hi |= code << (8 * (e - 4));
      }
      dst[c] = make_uint2(lo, hi);
    }
  } else {
    for (int64_t j = threadIdx.x; j < a.cols; j += blockDim.x) {
      const double xs = smooth_value(load_as_f64(a.x, v.off + j, a.dt), a.sm, v.gbase, j);
      const int code = encode_code(xs, p.scale, p.rscale, p.zp, qmax);
      sum += code;
      out[j] = (uint8_t)code;
    }
  }
  return sum;
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
  mn = block_reduce_min(mn, shd);
  mx = block_reduce_max(mx, shd);
  const AffineParams p = affine_params(mn, mx, bits, sym);
  const int64_t s = row_encode(a, v, p, (1 << bits) - 1, codes + r * ldc);
  if (rowsum) {
    const int64_t t = block_reduce_sum_i64(s, shi);
    if (threadIdx.x == 0) rowsum[r] = (int32_t)t;
  }
  if (threadIdx.x == 0) {
    scale[r] = p.scale;
    if (scale_f32) scale_f32[r] = (float)p.scale;
    zp[r] = p.zp;
  }
}

__global__ void minmax_init_kernel(long long* ws) {
  ws[0] = 0x7FFFFFFFFFFFFFFFLL;
  ws[1] = (long long)0x8000000000000000ULL;
}

__global__ void __launch_bounds__(kQuantThreads) tensor_minmax_kernel(RowArgs a, long long* ws) {
  __shared__ double shd[kQuantThreads / 32];
  const RowView v = row_view(a, blockIdx.x);
  double mn, mx;
  row_minmax(a, v, mn, mx);
  mn = block_reduce_min(mn, shd);
  mx = block_reduce_max(mx, shd);
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
  if (rowsum) {
    const int64_t t = block_reduce_sum_i64(s, shi);
    if (threadIdx.x == 0) rowsum[r] = (int32_t)t;
  }
  if (r == 0 && threadIdx.x == 0) {
    scale[0] = p.scale;
    if (scale_f32) scale_f32[0] = (float)p.scale;
    zp[0] = p.zp;
  }
}

__global__ void reciprocal_kernel(const double* s, int64_t n, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __drcp_rn(s[i]);
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

// one CTA per channel row of x [n, T]; deterministic tree order for sums
__global__ void __launch_bounds__(256) channel_stats_kernel(const double* x, int64_t T, int strategy,
                                                            double* stat) {
  __shared__ double sh[256];
  const double* row = x + blockIdx.x * T;
  double acc = 0.0;
  if (strategy == MOE_ORDER_MAX_ABS) {
    acc = 0.0;
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
  int64_t b = (n + threads - 1) / threads;
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
                                    int smooth_mode, const int32_t* row_group, int bits, int symmetric,
                                    int granularity, uint8_t* codes, int64_t ldc, double* scale,
                                    float* scale_f32, int32_t* zp, int32_t* rowsum, void* workspace,
                                    int64_t workspace_bytes, moe_stream_t stream) {
  MOE_REQUIRE(x && codes && scale && zp, "act_quant: null pointer");
  MOE_REQUIRE(rows >= 1 && cols >= 1, "act_quant: matrix must be non-empty");
  MOE_REQUIRE(ldx >= cols && ldc >= cols, "act_quant: bad leading dimension");
  MOE_REQUIRE(bits >= 2 && bits <= 8, "bits must be in [2, 8]");
  MOE_REQUIRE(x_dtype == MOE_DT_F32 || x_dtype == MOE_DT_F64 || x_dtype == MOE_DT_BF16 || x_dtype == MOE_DT_F16,
              "act_quant: unsupported input dtype");
  MOE_REQUIRE(smooth_mode == MOE_SMOOTH_NONE || smooth, "act_quant: smoothing table missing");
  MOE_REQUIRE(granularity >= 0 && granularity <= 2, "act_quant: unknown granularity");
  RowArgs a{x, x_dtype, rows, cols, ldx, gather_rows, row_group, SmoothArgs{smooth, smooth_recip, smooth_mode, cols}};
  cudaStream_t s = as_stream(stream);
  if (granularity == MOE_GRAN_PER_TENSOR) {
    MOE_REQUIRE(workspace && workspace_bytes >= 16, "act_quant: per_tensor needs 16 B of workspace");
    long long* ws = static_cast<long long*>(workspace);
    minmax_init_kernel<<<1, 1, 0, s>>>(ws); ::moe::count_launch();
    tensor_minmax_kernel<<<(unsigned)rows, kQuantThreads, 0, s>>>(a, ws); ::moe::count_launch();
    tensor_encode_kernel<<<(unsigned)rows, kQuantThreads, 0, s>>>(a, ws, bits, symmetric, codes, ldc, scale,
                                                                   scale_f32, zp, rowsum); ::moe::count_launch();
  } else {
    act_quant_rows_kernel<<<(unsigned)rows, kQuantThreads, 0, s>>>(a, bits, symmetric, codes, ldc, scale,
                                                                    scale_f32, zp, rowsum); ::moe::count_launch();
  }
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_reciprocal_f64(const double* sv, int64_t n, double* out, moe_stream_t stream) {
  MOE_REQUIRE(sv && out && n >= 1, "reciprocal: bad arguments");
  reciprocal_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(sv, n, out); ::moe::count_launch();
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
