// Shared pieces of the K1 (smoothing + RTN) kernels: row addressing with
// gather / per-row smoothing groups and block-level reductions.
#pragma once

#include <cfloat>

#include "common.cuh"

namespace moe {

struct SmoothArgs {
  const double* s;    // [G, cols] smoothing factors
  const double* rs;   // [G, cols] RN(1/s) (optional)
  int mode;           // MOE_SMOOTH_*
  int64_t cols;
};

// Expert-parallel dispatch output: rows go straight into the receive
// buffers of their destination ranks (peer memory over NVLink), with the
// 16-byte sidecar (scale_f32, zp, rowsum, routing weight) beside them.
struct EpOut {
  uint8_t* const* codes_tab;   // [W] receive-buffer base per rank; NULL: ordinary local output
  int4* const* params_tab;     // [W] sidecar base per rank
  const int32_t* dst_rank;     // [rows]
  const int32_t* dst_row;      // [rows]
  const float* weight;         // [rows] routing weight (sidecar .w); NULL -> 1
};

struct RowArgs {
  const void* x;
  int dt;
  int64_t rows, cols, ldx;
  const int32_t* gather;  // output row -> input row (optional)
  const int32_t* group;   // output row -> smoothing table row (optional)
  SmoothArgs sm;
  EpOut ep;               // optional (zero: local output arrays)
  const int32_t* rows_dev = nullptr;  // optional: the row count lives on the device (<= rows, the capacity)
  // optional token-major walk (MoE dispatch): item i is output row order[i]
  // of source row i / order_k, so the k rows of a token go to adjacent warps
  // of one CTA at the same time and x is read from HBM once
  const int32_t* order = nullptr;
  int order_k = 1;
};

// Rows [lo, hi) of this CTA: `rows_per_cta` from the host, or, with a device
// row count, an even split of *rows_dev over the grid (launched for the
// capacity `rows`).
__device__ __forceinline__ void cta_row_range(const RowArgs& a, int64_t rows_per_cta, int64_t& lo, int64_t& hi) {
  int64_t rows = a.rows, rpc = rows_per_cta;
  if (a.rows_dev) {
    rows = min(rows, (int64_t)*a.rows_dev);
    rpc = (rows + gridDim.x - 1) / gridDim.x;
  }
  lo = (int64_t)blockIdx.x * rpc;
  hi = min(rows, lo + rpc);
}

// EP dispatch rows refused by the exchange plan (dst_rank < 0) are skipped.
__device__ __forceinline__ bool ep_row_dropped(const RowArgs& a, int64_t r) {
  return a.ep.codes_tab && a.ep.dst_rank[r] < 0;
}

__device__ __forceinline__ uint8_t* out_row_ptr(const RowArgs& a, uint8_t* codes, int64_t ldc, int64_t r) {
  return a.ep.codes_tab ? a.ep.codes_tab[a.ep.dst_rank[r]] + (int64_t)a.ep.dst_row[r] * ldc : codes + r * ldc;
}

struct RowView {
  int64_t off;    // element offset of the source row
  int64_t gbase;  // element offset of the smoothing table row
};

__device__ __forceinline__ RowView row_view(const RowArgs& a, int64_t r, int64_t src_item = -1) {
  const int64_t src = src_item >= 0 ? src_item / a.order_k : a.gather ? (int64_t)a.gather[r] : r;
  const int64_t g = a.group ? (int64_t)a.group[r] : 0;
  return RowView{src * a.ldx, g * a.sm.cols};
}

// x (already float64) smoothed exactly as apply_smoothing does (quant.py:324):
// RN(x / s) for activations, RN(w * s) for weights.
__device__ __forceinline__ double smooth_value(double x, const SmoothArgs& sa, int64_t gbase, int64_t j) {
  if (sa.mode == MOE_SMOOTH_DIVIDE) {
    const double s = sa.s[gbase + j];
    return sa.rs ? div_rcp(x, s, sa.rs[gbase + j]) : __ddiv_rn(x, s);
  }
  if (sa.mode == MOE_SMOOTH_MULTIPLY) return __dmul_rn(x, sa.s[gbase + j]);
  return x;
}

// Block reductions (any blockDim multiple of 32, <= 1024). All threads get
// the result. `sh` needs blockDim/32 slots.
template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, T* sh, Op op) {
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  T t = sh[0];
  for (int i = 1; i < (int)(blockDim.x >> 5); ++i) t = op(t, sh[i]);
  return t;
}

struct OpMin {
  __device__ double operator()(double a, double b) const { return fmin(a, b); }
  __device__ float operator()(float a, float b) const { return fminf(a, b); }
};
struct OpMax {
  __device__ double operator()(double a, double b) const { return fmax(a, b); }
  __device__ float operator()(float a, float b) const { return fmaxf(a, b); }
};
struct OpAdd {
  __device__ int64_t operator()(int64_t a, int64_t b) const { return a + b; }
};

// order-preserving int64 key of a double (atomic min/max of doubles)
__device__ __forceinline__ long long dkey(double d) {
  const long long i = __double_as_longlong(d);
  return i >= 0 ? i : (i ^ 0x7FFFFFFFFFFFFFFFLL);
}
__device__ __forceinline__ double dunkey(long long k) {
  return __longlong_as_double(k >= 0 ? k : (k ^ 0x7FFFFFFFFFFFFFFFLL));
}

// Host launcher of the TMA-staged bf16 fast path (act_quant_fast.cu).
// Returns false when the shape is outside its envelope.
bool launch_act_quant_fast(const RowArgs& a, const float* rs32, int bits, int sym, uint8_t* codes, int64_t ldc,
                           double* scale, float* scale_f32, int32_t* zp, int32_t* rowsum, cudaStream_t s,
                           cudaError_t* err);

// Token-major K1 for the MoE dispatch: output row token_pos[t * k + j] (j <
// k) = token t of x smoothed with group[row]; x read once per token. False
// if not eligible (bf16, cols % 8 == 0, cols <= 4096, divide smoothing).
bool launch_act_quant_tokens(const RowArgs& a, const int32_t* token_pos, int k, int64_t T, const float* rs32,
                             int bits, int sym, uint8_t* codes, int64_t ldc, double* scale, float* scale_f32,
                             int32_t* zp, int32_t* rowsum, cudaStream_t s, cudaError_t* err);

// K1 for rows whose float32 (min, max) records of the smoothed values were
// produced upstream (grouped GEMM SwiGLU epilogue) as (order key << 32 | col)
// `ext` [rows, 2]: a single speculative encode pass. False if not eligible.
bool launch_act_quant_given(const RowArgs& a, const float* rs32, const unsigned long long* ext, int bits, int sym,
                            uint8_t* codes, int64_t ldc, double* scale, float* scale_f32, int32_t* zp,
                            int32_t* rowsum, cudaStream_t s, cudaError_t* err);

}  // namespace moe
