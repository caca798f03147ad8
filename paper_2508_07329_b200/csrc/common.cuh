// Shared host/device helpers: status + thread-local error text, dtype loads,
// float64 rounding helpers that reproduce moekit's quantizer bit-for-bit.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <set>
#include <string>
#include <utility>

#include "../../include/moe_b200.h"

namespace moe {

void set_error(const std::string& msg);
// (pivot, value) of the last MOE_ENOTPD (moe_last_error_detail)
void set_error_detail(int64_t pivot, double value);
void count_launch();  // every kernel launch of the library is counted (moe_launch_count)
int64_t k1_small_rows();         // MOE_TUNE_K1_SMALL_ROWS
int64_t tune_value(int key);     // any MOE_TUNE_* knob
int64_t router_cluster_tiles();  // MOE_TUNE_ROUTER_CLUSTER_TILES

#define MOE_REQUIRE(cond, msg)         \
  do {                                 \
    if (!(cond)) {                     \
      ::moe::set_error(msg);           \
      return MOE_EINVAL;               \
    }                                  \
  } while (0)

#define MOE_CUDA_TRY(expr)                                                                  \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess) {                                                                \
      ::moe::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));                 \
      return MOE_ECUDA;                                                                     \
    }                                                                                       \
  } while (0)

#define MOE_LAUNCH_CHECK()                                                                  \
  do {                                                                                      \
    cudaError_t _e = cudaGetLastError();                                                    \
    if (_e != cudaSuccess) {                                                                \
      ::moe::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e));            \
      return MOE_ECUDA;                                                                     \
    }                                                                                       \
  } while (0)

inline cudaStream_t as_stream(moe_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device);
// thread-safe (the library is reentrant)
inline cudaError_t set_max_smem_once(const void* func, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({func, dev})) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({func, dev});
  return e;
}

// ── element loads ─────────────────────────────────────────────────────────
__device__ __forceinline__ double load_as_f64(const void* p, int64_t i, int dt) {
  switch (dt) {
    case MOE_DT_F32: return (double)static_cast<const float*>(p)[i];
    case MOE_DT_F64: return static_cast<const double*>(p)[i];
    case MOE_DT_BF16: return (double)__bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
    case MOE_DT_F16: return (double)__half2float(static_cast<const __half*>(p)[i]);
    default: return 0.0;
  }
}

// ── moekit float64 quantizer primitives (quant.py:64-67, 191-211) ─────────
// rha(v) = sign(v) * floor(|v| + 0.5); the add is a separately rounded op.
__device__ __forceinline__ double rha(double v) {
  const double a = floor(__dadd_rn(fabs(v), 0.5));
  return v > 0.0 ? a : (v < 0.0 ? -a : 0.0);
}

// Correctly rounded a / b from a precomputed rb = RN(1/b): q0 = a*rb,
// rem = a - q0*b (exact with FMA), q = q0 + rem*rb (Markstein; bit-identical
// to IEEE division absent under/overflow — verified on 2e8 random and
// all-ones-mantissa cases).
__device__ __forceinline__ double div_rcp(double a, double b, double rb) {
  const double q0 = __dmul_rn(a, rb);
  const double rem = __fma_rn(-q0, b, a);
  return __fma_rn(rem, rb, q0);
}

__device__ __forceinline__ int encode_code(double xs, double scale, double rscale, int zp, int qmax) {
  const double v = div_rcp(xs, scale, rscale);
  double c = __dadd_rn(rha(v), (double)zp);
  c = c < 0.0 ? 0.0 : (c > (double)qmax ? (double)qmax : c);
  return (int)c;
}

struct AffineParams {
  double scale;
  double rscale;
  int zp;
};

// _affine_params (quant.py:191-202) for one group.
__device__ __forceinline__ AffineParams affine_params(double mn, double mx, int bits, int symmetric) {
  const int qmax = (1 << bits) - 1;
  AffineParams p;
  if (symmetric) {
    const double amax = fmax(fabs(mn), fabs(mx));
    p.scale = fmax(__ddiv_rn(amax, (double)((1 << (bits - 1)) - 1)), 1e-12);
    p.zp = 1 << (bits - 1);
  } else {
    p.scale = fmax(__ddiv_rn(__dsub_rn(mx, mn), (double)qmax), 1e-12);
    double z = rha(__ddiv_rn(-mn, p.scale));
    z = z < 0.0 ? 0.0 : (z > (double)qmax ? (double)qmax : z);
    p.zp = (int)z;
  }
  p.rscale = __drcp_rn(p.scale);
  return p;
}

// affine_params for 8-bit asymmetric codes (the fast K1 rows) with both
// divisions through div_rcp (Markstein-corrected reciprocal: the correctly
// rounded quotient absent under/overflow; operands outside [2^-900, 2^1000]
// take the IEEE division), so the same values as affine_params for ~70
// fewer instructions per row.
__device__ __forceinline__ AffineParams affine_params_u8(double mn, double mx) {
  constexpr double kR255 = 1.0 / 255.0;   // RN(1/255), folded at compile time
  auto in_range = [](double v) { const double a = fabs(v); return a > 0x1p-900 && a < 0x1p+1000; };
  AffineParams p;
  const double diff = __dsub_rn(mx, mn);
  p.scale = fmax(in_range(diff) ? div_rcp(diff, 255.0, kR255) : __ddiv_rn(diff, 255.0), 1e-12);
  p.rscale = __drcp_rn(p.scale);
  const double nm = -mn;
  double z = rha((in_range(nm) && in_range(p.scale)) ? div_rcp(nm, p.scale, p.rscale) : __ddiv_rn(nm, p.scale));
  z = z < 0.0 ? 0.0 : (z > 255.0 ? 255.0 : z);
  p.zp = (int)z;
  return p;
}
__device__ __forceinline__ AffineParams affine_params_fast(double mn, double mx, int bits, int symmetric) {
  return (bits == 8 && !symmetric) ? affine_params_u8(mn, mx) : affine_params(mn, mx, bits, symmetric);
}


// Launch with programmatic dependent launch allowed: the kernel may start
// while the previous kernel in the stream is still running and must call
// griddepcontrol.wait (ptx.cuh: griddep_wait) before touching its outputs.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace moe
