// K1 hot path — bf16 rows, smoothing division, per-token RTN, bit-identical
// to the float64 reference semantics (quant.py:191-231, 314-324).
//
// Layout: one warp per row, 16 warps per CTA, rows gathered through the MoE
// permutation straight from x. A row is streamed up to three times — float32
// extremes (pass A, skipped when the producing GEMM epilogue already
// supplied them), exact float64 extremes over the few candidates (pass B),
// encode (pass C) — with 4 x 16-byte loads per lane in flight; the re-reads
// hit L1/L2 (a warp's row is 8-28 KB), so HBM sees one read of x and one
// write of the codes. No shared-memory staging and no block barriers: the
// reductions are warp shuffles. The float32 reciprocal table of the row's
// expert is read through L1 (a CTA's rows share an expert).
//
// Arithmetic: every element is first evaluated in float32 from correctly
// rounded reciprocals; the float32 value is within |v32| * 2^-21 of the
// float64 quotient (four float32 roundings of 2^-24). The row min/max are
// taken exactly (float64 reciprocal-and-correct division) over the few
// elements whose error interval can reach the extreme, and a code is taken
// from float32 when the interval cannot straddle a rounding boundary k+0.5
// (or lies far outside the clip range); the rest re-run the exact float64
// encode out of line. Codes, scales, zero points and row sums are identical
// to the exact kernel (tests/test_gpu_kernels.py).
#include <algorithm>

#include "k1_common.cuh"
#include "ptx.cuh"

namespace moe {

constexpr float kRelErr = 4.76837158203125e-07f;    // 2^-21
constexpr float kAbsErr = 7.174648137343064e-43f;   // 2^-140
constexpr int kWarpsPerCta = 16;
constexpr int kBatch = 4;                           // 16-byte vectors in flight per lane

__device__ __forceinline__ float err_bound(float v) { return fmaf(fabsf(v), kRelErr, kAbsErr); }

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

// xs = x * RN32(1/s) for 8 consecutive elements (table through L1)
__device__ __forceinline__ void smooth8(const uint4& u, const float* __restrict__ tab, int64_t c, float (&xs)[8]) {
  unpack8(u, xs);
  if (tab) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(tab) + 2 * c);
    const float4 b = __ldg(reinterpret_cast<const float4*>(tab) + 2 * c + 1);
    float2 p;
    p = __fmul2_rn(make_float2(xs[0], xs[1]), make_float2(a.x, a.y)); xs[0] = p.x; xs[1] = p.y;
    p = __fmul2_rn(make_float2(xs[2], xs[3]), make_float2(a.z, a.w)); xs[2] = p.x; xs[3] = p.y;
    p = __fmul2_rn(make_float2(xs[4], xs[5]), make_float2(b.x, b.y)); xs[4] = p.x; xs[5] = p.y;
    p = __fmul2_rn(make_float2(xs[6], xs[7]), make_float2(b.z, b.w)); xs[6] = p.x; xs[7] = p.y;
  }
}

// ── packed 8-bit encode (sm_100 FFMA2/FADD2 + I2IP saturating pack) ───────
// For |v| < 2^21: t = v + 1.5*2^23 rounds v to the nearest integer in its
// low mantissa bits (exact: rr = t - 1.5*2^23, d = v - rr). The element is
// "safe" when |d| + eb(v) < 0.5, i.e. the exact float64 quotient rounds to
// the same integer (round-half-away only differs from round-to-nearest-even
// at .5, which is never safe). code = clamp(R + zp, 0, 255) via I2IP.
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
constexpr int kMagicBits = 0x4B400000;

__device__ __forceinline__ uint32_t pack_sat_u8(int lo, int hi, uint32_t rest) {
  uint32_t d;
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(hi), "r"(lo), "r"(rest));
  return d;
}

__device__ __forceinline__ void enc2(float2 xs, float2 rsc2, int zpm, int& c0, int& c1, bool& unsafe) {
  const float2 v = __fmul2_rn(xs, rsc2);
  const float2 t = __fadd2_rn(v, make_float2(kMagic, kMagic));
  const float2 rr = __fadd2_rn(t, make_float2(-kMagic, -kMagic));
  const float2 d = __fadd2_rn(v, make_float2(-rr.x, -rr.y));
  const float2 s = __ffma2_rn(make_float2(fabsf(v.x), fabsf(v.y)), make_float2(kRelErr, kRelErr),
                              __fadd2_rn(make_float2(fabsf(d.x), fabsf(d.y)), make_float2(kAbsErr, kAbsErr)));
  unsafe |= (s.x >= 0.5f) | (s.y >= 0.5f);
  c0 = __float_as_int(t.x) + zpm;
  c1 = __float_as_int(t.y) + zpm;
}

// ── rare float64 paths, out of line ───────────────────────────────────────
__device__ __noinline__ double2 exact_extremes8(uint4 u, const double* srow, const double* rrow, int64_t c,
                                                 uint32_t cmax, uint32_t cmin) {
  float f[8];
  unpack8(u, f);
  double mn = DBL_MAX, mx = -DBL_MAX;
  for (int e = 0; e < 8; ++e) {
    if (!((cmax | cmin) >> e & 1u)) continue;
    const double xd = srow ? div_rcp((double)f[e], srow[c * 8 + e], rrow[c * 8 + e]) : (double)f[e];
    if (cmax >> e & 1u) mx = fmax(mx, xd);
    if (cmin >> e & 1u) mn = fmin(mn, xd);
  }
  return make_double2(mn, mx);
}

struct ExactParams {
  double scale, rscale;
  int zp, qmax;
};

__device__ __noinline__ uint2 exact_encode8(uint4 u, const double* srow, const double* rrow, int64_t c, uint32_t mask,
                                            uint2 packed, ExactParams p) {
  float f[8];
  unpack8(u, f);
  uint32_t w[2] = {packed.x, packed.y};
  for (int e = 0; e < 8; ++e) {
    if (!(mask >> e & 1u)) continue;
    const double xd = srow ? div_rcp((double)f[e], srow[c * 8 + e], rrow[c * 8 + e]) : (double)f[e];
    const uint32_t code = (uint32_t)encode_code(xd, p.scale, p.rscale, p.zp, p.qmax);
    const int sh = 8 * (e & 3);
    w[e >> 2] = (w[e >> 2] & ~(0xFFu << sh)) | (code << sh);
  }
  return make_uint2(w[0], w[1]);
}

__device__ __forceinline__ int bytesum(uint2 v) {
  return (int)__dp4a(v.y, 0x01010101u, __dp4a(v.x, 0x01010101u, 0u));
}

// Encoder of one row once its exact extremes (hence scale / zero point) are
// known: 8 elements per call, packed f32x2 path for 8-bit codes when the
// row's quotients stay below 2^21, general float32 path otherwise; either
// way elements whose float32 interval straddles a rounding boundary are
// re-encoded exactly (out of line).
struct RowEncoder {
  double scale, rscale;
  int zp, qmax;
  float rsc32, big;
  int zpm;
  bool packed, exact_all;

  __device__ __forceinline__ RowEncoder(const AffineParams& p, double mn, double mx, int bits, bool exact)
      : scale(p.scale), rscale(p.rscale), zp(p.zp), qmax((1 << bits) - 1) {
    rsc32 = __double2float_rn(p.rscale);
    big = (float)(qmax + zp + 2) * 1.001f;
    zpm = zp - kMagicBits;
    exact_all = exact;
    packed = bits == 8 && !exact && fmax(fabs(mn), fabs(mx)) * p.rscale < 2097152.0;
  }

  __device__ __forceinline__ uint2 encode8(const uint4& u, const float* tab, int64_t c, const double* srow,
                                           const double* rrow, int& sum) const {
    float xs[8];
    smooth8(u, tab, c, xs);
    uint2 out;
    uint32_t redo = 0;
    if (packed) {
      const float2 rsc2 = make_float2(rsc32, rsc32);
      int q[8];
      bool unsafe = false;
#pragma unroll
      for (int e = 0; e < 8; e += 2) enc2(make_float2(xs[e], xs[e + 1]), rsc2, zpm, q[e], q[e + 1], unsafe);
      out = make_uint2(pack_sat_u8(q[0], q[1], pack_sat_u8(q[2], q[3], 0u)),
                       pack_sat_u8(q[4], q[5], pack_sat_u8(q[6], q[7], 0u)));
      sum += bytesum(out);
      redo = unsafe ? 0xFFu : 0u;
    } else {
      uint32_t packedw[2] = {0u, 0u};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float v32 = xs[e] * rsc32;
        const float av = fabsf(v32);
        const float rr = rintf(av);
        const bool safe = 0.5f - fabsf(av - rr) > err_bound(av);
        const int R = (int)rr;
        int code = min(max((v32 < 0.f ? -R : R) + zp, 0), qmax);
        if (!safe) code = v32 < 0.f ? 0 : qmax;   // exact whenever av > big
        redo |= (uint32_t)(exact_all || (!safe && !(av > big))) << e;
        sum += code;
        packedw[e >> 2] |= (uint32_t)code << (8 * (e & 3));
      }
      out = make_uint2(packedw[0], packedw[1]);
    }
    if (redo) {
      const uint2 fixed = exact_encode8(u, srow, rrow, c, redo, out, ExactParams{scale, rscale, zp, qmax});
      sum += bytesum(fixed) - bytesum(out);
      out = fixed;
    }
    return out;
  }
};

// order-preserving int32 key of a float (atomic min/max of floats)
__device__ __forceinline__ float funkey(int k) { return __int_as_float(k >= 0 ? k : (k ^ 0x7FFFFFFF)); }

template <typename F>
__device__ __forceinline__ void for_row_batches(const uint4* src, int64_t nvec, int lane, F&& body) {
  for (int64_t c0 = lane; c0 < nvec; c0 += 32 * kBatch) {
    uint4 u[kBatch];
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const int64_t c = c0 + 32 * b;
      u[b] = c < nvec ? src[c] : make_uint4(0u, 0u, 0u, 0u);
    }
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const int64_t c = c0 + 32 * b;
      if (c < nvec) body(u[b], c);
    }
  }
}

template <bool GIVEN>
__global__ void __launch_bounds__(kWarpsPerCta * 32, 2)
    act_quant_warp_kernel(RowArgs a, const float* __restrict__ rs32_tab, const int* __restrict__ bounds, int bits,
                          int sym, uint8_t* codes, int64_t ldc, double* scale, float* scale_f32, int32_t* zp,
                          int32_t* rowsum, int64_t rows_per_cta) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t nvec = a.cols / 8;
  const bool smooth = a.sm.mode == MOE_SMOOTH_DIVIDE;
  // each CTA owns a contiguous range of rows (shared expert tables in L1)
  const int64_t r_lo = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r_hi = min(a.rows, r_lo + rows_per_cta);
  for (int64_t r = r_lo + warp; r < r_hi; r += kWarpsPerCta) {
    const RowView rv = row_view(a, r);
    const uint4* src = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.x) + rv.off);
    const float* tab = smooth ? rs32_tab + rv.gbase : nullptr;
    const double* srow = smooth ? a.sm.s + rv.gbase : nullptr;
    const double* rrow = smooth ? a.sm.rs + rv.gbase : nullptr;

    // pass A: float32 extremes (given by the producing epilogue, or computed)
    float M, m;
    if (GIVEN) {
      m = funkey(bounds[2 * r]);
      M = funkey(bounds[2 * r + 1]);
    } else {
      float tmax = -FLT_MAX, tmin = FLT_MAX;
      for_row_batches(src, nvec, lane, [&](const uint4& u, int64_t c) {
        float xs[8];
        smooth8(u, tab, c, xs);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          tmax = fmaxf(tmax, xs[e]);
          tmin = fminf(tmin, xs[e]);
        }
      });
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
        tmin = fminf(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
      }
      M = tmax;
      m = tmin;
    }
    const bool exact_all = !(isfinite(M) && isfinite(m));
    const float lb_max = exact_all ? -FLT_MAX : M - err_bound(M);   // the exact max is >= this
    const float ub_min = exact_all ? FLT_MAX : m + err_bound(m);    // the exact min is <= this

    // pass B: exact float64 extremes over the elements that can reach them
    double mn = DBL_MAX, mx = -DBL_MAX;
    for_row_batches(src, nvec, lane, [&](const uint4& u, int64_t c) {
      float xs[8];
      smooth8(u, tab, c, xs);
      uint32_t mmax = 0, mmin = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        mmax |= (uint32_t)(xs[e] + err_bound(xs[e]) >= lb_max) << e;
        mmin |= (uint32_t)(xs[e] - err_bound(xs[e]) <= ub_min) << e;
      }
      if (mmax | mmin) {
        const double2 ext = exact_extremes8(u, srow, rrow, c, mmax, mmin);
        mn = fmin(mn, ext.x);
        mx = fmax(mx, ext.y);
      }
    });
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    const AffineParams p = affine_params(mn, mx, bits, sym);
    const RowEncoder enc(p, mn, mx, bits, exact_all);

    // pass C: encode
    int sum = 0;
    uint2* dst = reinterpret_cast<uint2*>(codes + r * ldc);
    for_row_batches(src, nvec, lane,
                    [&](const uint4& u, int64_t c) { __stcs(dst + c, enc.encode8(u, tab, c, srow, rrow, sum)); });
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) {
      if (rowsum) rowsum[r] = sum;
      scale[r] = p.scale;
      if (scale_f32) scale_f32[r] = (float)p.scale;
      zp[r] = p.zp;
    }
  }
}

static bool eligible(const RowArgs& a, const float* rs32, uint8_t* codes, int64_t ldc) {
  const bool smooth = a.sm.mode == MOE_SMOOTH_DIVIDE;
  return a.dt == MOE_DT_BF16 && a.cols % 8 == 0 && a.ldx % 8 == 0 && ldc % 8 == 0 &&
         (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 && (reinterpret_cast<uintptr_t>(codes) & 7) == 0 &&
         (a.sm.mode == MOE_SMOOTH_NONE || (smooth && a.sm.rs && rs32));
}

template <bool GIVEN>
static cudaError_t launch_warp(const RowArgs& a, const float* rs32, const int* bounds, int bits, int sym,
                              uint8_t* codes, int64_t ldc, double* scale, float* scale_f32, int32_t* zp,
                              int32_t* rowsum, cudaStream_t s) {
  // contiguous row ranges, ~4 CTAs (64 warps) per SM
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>((a.rows + kWarpsPerCta - 1) / kWarpsPerCta,
                                                              4 * (int64_t)num_sms()));
  const int64_t rows_per_cta = (a.rows + ctas - 1) / ctas;
  const int64_t nblk = (a.rows + rows_per_cta - 1) / rows_per_cta;
  act_quant_warp_kernel<GIVEN><<<(unsigned)nblk, kWarpsPerCta * 32, 0, s>>>(
      a, rs32, bounds, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, rows_per_cta);
  count_launch();
  return cudaGetLastError();
}

bool launch_act_quant_given(const RowArgs& a, const float* rs32, const int* bounds, int bits, int sym,
                            uint8_t* codes, int64_t ldc, double* scale, float* scale_f32, int32_t* zp,
                            int32_t* rowsum, cudaStream_t s, cudaError_t* err) {
  if (!bounds || !eligible(a, rs32, codes, ldc)) return false;
  *err = launch_warp<true>(a, rs32, bounds, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, s);
  return true;
}

bool launch_act_quant_fast(const RowArgs& a, const float* rs32, int bits, int sym, uint8_t* codes, int64_t ldc,
                           double* scale, float* scale_f32, int32_t* zp, int32_t* rowsum, cudaStream_t s,
                           cudaError_t* err) {
  if (!eligible(a, rs32, codes, ldc)) return false;
  *err = launch_warp<false>(a, rs32, nullptr, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, s);
  return true;
}

}  // namespace moe
