// K1 device building blocks (bf16 rows, smoothing division, per-token RTN,
// bit-identical to the float64 reference semantics, quant.py:191-231,
// 314-324): the float32 filter, packed encode, speculative extremes and the
// exact fallbacks, and the per-row warp routine. Shared by the K1 kernels
// (act_quant_fast.cu) and the grouped GEMM that fuses K1 of its A operand
// (gemm_i8.cu). See act_quant_fast.cu for the algorithm notes.
#pragma once

#include <type_traits>

#include "k1_common.cuh"
#include "ptx.cuh"

namespace moe {

constexpr float kRelErr = 4.76837158203125e-07f;    // 2^-21
constexpr float kAbsErr = 7.174648137343064e-43f;   // 2^-140
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

// xs = x * RN32(1/s) for 8 consecutive elements (table through L1). The fast
// kernels always have a table (K1 without smoothing takes the exact kernel,
// or the host passes a table of ones), so the multiply is unconditional: a
// conditional one made the compiler merge both versions with moves.
__device__ __forceinline__ void smooth8(const uint4& u, const float* __restrict__ tab, int64_t c, float (&xs)[8]) {
  unpack8(u, xs);
  const float4 a = __ldg(reinterpret_cast<const float4*>(tab) + 2 * c);
  const float4 b = __ldg(reinterpret_cast<const float4*>(tab) + 2 * c + 1);
  float2 p;
  p = __fmul2_rn(make_float2(xs[0], xs[1]), make_float2(a.x, a.y)); xs[0] = p.x; xs[1] = p.y;
  p = __fmul2_rn(make_float2(xs[2], xs[3]), make_float2(a.z, a.w)); xs[2] = p.x; xs[3] = p.y;
  p = __fmul2_rn(make_float2(xs[4], xs[5]), make_float2(b.x, b.y)); xs[4] = p.x; xs[5] = p.y;
  p = __fmul2_rn(make_float2(xs[6], xs[7]), make_float2(b.z, b.w)); xs[6] = p.x; xs[7] = p.y;
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
static __device__ __noinline__ double2 exact_extremes8(uint4 u, const double* srow, const double* rrow, int64_t c,
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

static __device__ __noinline__ uint2 exact_encode8(uint4 u, const double* srow, const double* rrow, int64_t c, uint32_t mask,
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

  __device__ __forceinline__ uint2 encode8(const uint4& u, const float (&xs)[8], int64_t c, const double* srow,
                                           const double* rrow, int& sum) const {
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

// ── per-row extreme records ────────────────────────────────────────────────
// (float32 value, column) of the max and of the min of the smoothed row, as
// produced by the grouped GEMM's SwiGLU epilogue ((order key << 32) | col)
// or by pass A here.
struct RowExt {
  float M, m;
  int64_t cM, cm;
};

__device__ __forceinline__ float key_to_float(uint32_t k) {
  const int i = (int)(k ^ 0x80000000u);
  return __int_as_float(i >= 0 ? i : (i ^ 0x7FFFFFFF));
}

// Producer records (value key << 32 | c): the extreme element lies in columns
// [c, c + 32) (the GEMM epilogue records the 32-column chunk; an exact column
// also qualifies). The warp locates the first element of the chunk whose
// float32 smoothed value equals the recorded one; none -> column = cols
// (an inconsistent record, handled as such by the caller).
__device__ __forceinline__ int64_t locate32(const __nv_bfloat16* row, const float* tab, int64_t cols, int64_t base,
                                            float val, int lane) {
  const int64_t j = base + lane;
  bool hit = false;
  if (j < cols) {
    const float xf = __bfloat162float(row[j]);
    hit = (tab ? __fmul_rn(xf, tab[j]) : xf) == val;
  }
  const unsigned m = __ballot_sync(0xffffffffu, hit);
  return m ? base + __ffs(m) - 1 : cols;
}

__device__ __forceinline__ RowExt given_record(const __nv_bfloat16* row, const float* tab, int64_t cols,
                                               unsigned long long kmax, unsigned long long kmin, int lane) {
  RowExt rec{key_to_float((uint32_t)(kmax >> 32)), key_to_float((uint32_t)(kmin >> 32)), cols, cols};
  if (isfinite(rec.M) && isfinite(rec.m)) {
    rec.cM = locate32(row, tab, cols, (int64_t)(kmax & 0xFFFFFFFFu), rec.M, lane);
    rec.cm = locate32(row, tab, cols, (int64_t)(kmin & 0xFFFFFFFFu), rec.m, lane);
  }
  return rec;
}

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

// warp arg-reduce: larger value wins, ties to the lower column. Two REDUX
// instructions on order-preserving keys instead of five shuffle rounds
// (-0 is keyed as +0, so signed zeros tie like in a float compare; the
// returned value is then +0, which every caller treats like -0).
__device__ __forceinline__ uint32_t fkey32(float v) {
  const uint32_t b = __float_as_uint(v + 0.0f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float funkey32(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}
#ifndef MOE_K1_REDUX
#define MOE_K1_REDUX 1
#endif
#if MOE_K1_REDUX
__device__ __forceinline__ void warp_argmax(float& v, int64_t& col) {
  const uint32_t k = fkey32(v);
  const uint32_t km = __reduce_max_sync(0xffffffffu, k);
  col = (int64_t)__reduce_min_sync(0xffffffffu, k == km ? (uint32_t)col : 0xFFFFFFFFu);
  v = funkey32(km);
}
__device__ __forceinline__ void warp_argmin(float& v, int64_t& col) {
  const uint32_t k = fkey32(v);
  const uint32_t km = __reduce_min_sync(0xffffffffu, k);
  col = (int64_t)__reduce_min_sync(0xffffffffu, k == km ? (uint32_t)col : 0xFFFFFFFFu);
  v = funkey32(km);
}
// warp sums of the code sum and the candidate count (REDUX)
__device__ __forceinline__ void warp_sum2(int& sum, uint32_t& cnt) {
  sum = (int)__reduce_add_sync(0xffffffffu, (unsigned)sum);
  cnt = __reduce_add_sync(0xffffffffu, cnt);
}
#else   // shuffle trees (A/B reference)
__device__ __forceinline__ void warp_argmax(float& v, int64_t& col) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int64_t c2 = __shfl_xor_sync(0xffffffffu, col, o);
    if (v2 > v || (v2 == v && c2 < col)) { v = v2; col = c2; }
  }
}
__device__ __forceinline__ void warp_argmin(float& v, int64_t& col) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int64_t c2 = __shfl_xor_sync(0xffffffffu, col, o);
    if (v2 < v || (v2 == v && c2 < col)) { v = v2; col = c2; }
  }
}
__device__ __forceinline__ void warp_sum2(int& sum, uint32_t& cnt) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
}
#endif

// exact float64 value of element j of the row, and whether its float32
// evaluation matches the recorded extreme (record consistency check)
__device__ __forceinline__ double exact_at(const __nv_bfloat16* row, const float* tab, const double* srow,
                                           const double* rrow, int64_t j, float expect, bool& ok) {
  const float xf = __bfloat162float(row[j]);
  const float xs = tab ? __fmul_rn(xf, tab[j]) : xf;
  ok = ok && xs == expect;
  return srow ? div_rcp((double)xf, srow[j], rrow[j]) : (double)xf;
}


// ── 3-input min/max (FMNMX3) ───────────────────────────────────────────────
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float fmin3(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// NaN-propagating max of |a|, |b|, |c|
__device__ __forceinline__ float fmax3_abs_nan(float a, float b, float c) {
  float d;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(fabsf(a)), "f"(fabsf(b)), "f"(fabsf(c)));
  return d;
}
__device__ __forceinline__ float max8(const float (&v)[8]) {
  return fmax3(fmax3(v[0], v[1], v[2]), fmax3(v[3], v[4], v[5]), fmaxf(v[6], v[7]));
}
__device__ __forceinline__ float min8(const float (&v)[8]) {
  return fmin3(fmin3(v[0], v[1], v[2]), fmin3(v[3], v[4], v[5]), fminf(v[6], v[7]));
}

// ── fast 8-bit encode of one row (asymmetric, extremes at codes <= 0 / >= 255)
// t = RN(xs * rsc + (1.5*2^23 + zp)) holds round(p) + zp in its low mantissa
// bits (p = xs * rsc exact inside the FMA); d = RN(p - round(p)). A vector
// of 8 takes the fast path when every code is in [2, 253] and every |d| is
// below 0.5 - 2^-14 - 2^-24: those codes equal the float64 reference's
// (|p| <= 255 there and p = y (1 + e), |e| <= 3 2^-24 + 2^-50, so
// |p - y| <= 4.6e-5 < 2^-14; d itself carries one rounding of at most
// 2^-26, so y stays more than 1.5e-5 away from the rounding boundary).
// Everything else — clipping, rounding-boundary cases, non-finite values and
// the elements that could be row extremes (codes <= 1 / >= 254) — goes out
// of line. (The window was 0.5 - 2^-13 in round 1: twice as many boundary
// vectors on the slow path for the same proof.)
constexpr float kMagicF = 12582912.0f;
constexpr float kFastTlo = 12582914.0f;          // code 2
constexpr float kFastThi = 12583165.0f;          // code 253
constexpr float kFastThr = 0.49993890523910522f;  // 0.5 - 2^-14 - 2^-24

// Per-row constants of the fast encode. Two variants:
//  * two-sided rows (asymmetric, the extremes land on codes <= 0 / >= 255):
//    vectors are fast when every code is in [2, 253]; elements that could
//    be extremes necessarily fall outside and are counted out of line;
//  * general rows (one-sided, e.g. ReLU outputs with min 0, or symmetric):
//    codes in [0, 255] plus an explicit float32 candidate check
//    xlo <= xs <= xhi. An extreme that is exactly 0 needs no candidates:
//    zeros quantize exactly and only a strictly negative (positive) element
//    could beat a zero minimum (maximum).
struct FastRow {
  double scale, rscale;
  float rsc, magic;
  float tlo, thi;            // fast-vector t range (code window)
  float xlo, xhi;            // xs < xlo (> xhi) may be an exact min (max): counted
  uint32_t expect;           // candidate count that confirms the speculation (max | min << 16)
  int zp;
};
constexpr float kCodeT0 = 12582912.0f;          // t of code 0
constexpr float kCodeT255 = 12583167.0f;        // t of code 255

// 0: no fast path, 1: two-sided, 2: general
__device__ __forceinline__ int init_fast_row(FastRow& f, const AffineParams& p, float M, float m, double mn, double mx,
                                             int bits, int sym) {
  if (bits != 8) return 0;
  f.scale = p.scale;
  f.rscale = p.rscale;
  f.zp = p.zp;
  f.rsc = __double2float_rn(p.rscale);
  f.magic = kMagicF + (float)p.zp;
  const float cand_max = M - 3.f * fabsf(M) * kRelErr - 2.350988701644575e-38f;
  const float cand_min = m + 3.f * fabsf(m) * kRelErr + 2.350988701644575e-38f;
  f.xlo = nextafterf(cand_min, FLT_MAX);
  f.xhi = nextafterf(cand_max, -FLT_MAX);
  const double hc = __dadd_rn(rha(div_rcp(mx, p.scale, p.rscale)), (double)p.zp);
  const double lc = __dadd_rn(rha(div_rcp(mn, p.scale, p.rscale)), (double)p.zp);
  // two-sided window only when zero (hence the bulk of typical activations)
  // quantizes well inside [2, 253]; one-sided rows (zp at an edge, e.g. ReLU)
  // take the general window, where the edge codes stay on the fast path
  if (!sym && hc >= 255.0 && lc <= 0.0 && p.zp >= 16 && p.zp <= 239 && m != 0.f && M != 0.f) {
    f.tlo = kFastTlo;
    f.thi = kFastThi;
    f.expect = 0x10001u;
    return 1;
  }
  f.tlo = kCodeT0;
  f.thi = kCodeT255;
  uint32_t e = 0x10001u;
  if (m == 0.f) {           // zero minimum: only negatives are candidates
    f.xlo = 0.f;
    e -= 0x10000u;
  }
  if (M == 0.f) {
    f.xhi = 0.f;
    e -= 1u;
  }
  f.expect = e;
  return 2;
}

__device__ __forceinline__ uint32_t low_bytes4(float a, float b, float c, float d) {
  const uint32_t ab = __byte_perm(__float_as_uint(a), __float_as_uint(b), 0x0040);
  const uint32_t cd = __byte_perm(__float_as_uint(c), __float_as_uint(d), 0x0040);
  return __byte_perm(ab, cd, 0x5410);
}

// Fallback for a whole row: float64 extremes over every element that can
// reach them (pass B), then the generic encode (pass C). Used when the
// speculative extremes fail their check, for symmetric / non-8-bit codes
// and for rows outside the fast envelope.
static __device__ __noinline__ int fallback_row(const uint4* src, int64_t nvec, int lane, const float* tab,
                                         const double* srow, const double* rrow, float lb_max, float ub_min,
                                         bool exact_all, int bits, int sym, uint2* dst, AffineParams* out) {
  double mn = DBL_MAX, mx = -DBL_MAX;
  for_row_batches(src, nvec, lane, [&](const uint4& u, int64_t c) {
    float xs[8];
    smooth8(u, tab, c, xs);
    uint32_t mmax = 0, mmin = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      mmax |= (uint32_t)(!(xs[e] + err_bound(xs[e]) < lb_max)) << e;
      mmin |= (uint32_t)(!(xs[e] - err_bound(xs[e]) > ub_min)) << e;
    }
    if (mmax | mmin) {
      const double2 e2 = exact_extremes8(u, srow, rrow, c, mmax, mmin);
      mn = fmin(mn, e2.x);
      mx = fmax(mx, e2.y);
    }
  });
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const AffineParams p = affine_params(mn, mx, bits, sym);
  const RowEncoder enc(p, mn, mx, bits, exact_all);
  int sum = 0;
  for_row_batches(src, nvec, lane, [&](const uint4& u, int64_t c) {
    float xs[8];
    smooth8(u, tab, c, xs);
    __stcs(dst + c, enc.encode8(u, xs, c, srow, rrow, sum));
  });
  sum = (int)__reduce_add_sync(0xffffffffu, (unsigned)sum);
  *out = p;
  return sum;
}

template <bool GEN>
__device__ __forceinline__ bool fast_ok(const float (&xs)[8], const float (&t)[8], float dm, const FastRow& f) {
  // bitwise (not short-circuit): one predicate chain, no branches
  bool ok = (max8(t) <= f.thi) & (min8(t) >= f.tlo) & (dm < kFastThr);
  if (GEN) ok = ok & (max8(xs) <= f.xhi) & (min8(xs) >= f.xlo);
  return ok;
}

__device__ __forceinline__ float t_and_d(const float (&xs)[8], const FastRow& f, float (&t)[8]) {
  const float2 rsc2 = make_float2(f.rsc, f.rsc), mag2 = make_float2(f.magic, f.magic);
  float d[8];
#pragma unroll
  for (int e = 0; e < 8; e += 2) {
    const float2 x2 = make_float2(xs[e], xs[e + 1]);
    const float2 t2 = __ffma2_rn(x2, rsc2, mag2);
    const float2 nr = __fadd2_rn(mag2, make_float2(-t2.x, -t2.y));   // -round(p), exact
    const float2 d2 = __ffma2_rn(x2, rsc2, nr);
    t[e] = t2.x;
    t[e + 1] = t2.y;
    d[e] = d2.x;
    d[e + 1] = d2.y;
  }
  return fmax3_abs_nan(fmax3_abs_nan(d[0], d[1], d[2]), fmax3_abs_nan(d[3], d[4], d[5]),
                       fmax3_abs_nan(d[6], d[7], 0.f));
}

// Rare vectors (a code outside the fast window, a possible extreme, a
// rounding-boundary case): the count of possible-extreme elements plus the
// codes; clipping, boundary and non-finite elements re-run the float64
// reference encode. Returns (codes, cnt_max | cnt_min << 16). Two versions
// of the same result: slow_vec8 works element by element (the 64-register
// row kernels: K1-x 145 us, against 153 us with the packed one), and
// slow_vec8_packed handles the common rare vector — a row extreme, every code
// in [0, 255] and clear of rounding boundaries — with the packed float32
// encode, going element by element only for the rest (the bulk K1-h kernel:
// 309 -> 302 us).
static __device__ __noinline__ uint4 slow_vec8(uint4 u, const float* tab, int64_t c, const double* srow, const double* rrow,
                                        FastRow f) {
  float xv[8], xs[8];
  unpack8(u, xv);
  smooth8(u, tab, c, xs);
  uint32_t cnt = 0, w[2] = {0u, 0u};
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    cnt += (uint32_t)(xs[e] > f.xhi) + ((uint32_t)(xs[e] < f.xlo) << 16);
    const float t = fmaf(xs[e], f.rsc, f.magic);
    const float d = fmaf(xs[e], f.rsc, f.magic - t);   // magic - t = -round(p), exact
    uint32_t code;
    if (t >= kCodeT0 && t <= kCodeT255 && fabsf(d) < kFastThr) {   // in range: no clipping
      code = __float_as_uint(t) & 0xFFu;
    } else {   // clipping, rounding boundary, non-finite: the float64 reference encode
      const double xd = srow ? div_rcp((double)xv[e], srow[c * 8 + e], rrow[c * 8 + e]) : (double)xv[e];
      code = (uint32_t)encode_code(xd, f.scale, f.rscale, f.zp, 255);
    }
    w[e >> 2] |= code << (8 * (e & 3));
  }
  return make_uint4(w[0], w[1], cnt, 0u);
}

static __device__ __noinline__ uint4 slow_vec8_packed(uint4 u, const float* tab, int64_t c, const double* srow,
                                               const double* rrow, FastRow f) {
  float xs[8], t[8];
  smooth8(u, tab, c, xs);
  const float dm = t_and_d(xs, f, t);
  uint32_t cnt = 0;
  if (max8(xs) > f.xhi) {
#pragma unroll
    for (int e = 0; e < 8; ++e) cnt += (uint32_t)(xs[e] > f.xhi);
  }
  if (min8(xs) < f.xlo) {
#pragma unroll
    for (int e = 0; e < 8; ++e) cnt += (uint32_t)(xs[e] < f.xlo) << 16;
  }
  uint32_t w[2] = {low_bytes4(t[0], t[1], t[2], t[3]), low_bytes4(t[4], t[5], t[6], t[7])};
  if (!((max8(t) <= kCodeT255) & (min8(t) >= kCodeT0) & (dm < kFastThr))) {
    float xv[8];
    unpack8(u, xv);
#pragma unroll 1
    for (int e = 0; e < 8; ++e) {
      const float te = fmaf(xs[e], f.rsc, f.magic);
      const float de = fmaf(xs[e], f.rsc, f.magic - te);   // magic - t = -round(p), exact
      if (te >= kCodeT0 && te <= kCodeT255 && fabsf(de) < kFastThr) continue;   // in range, clear: byte stands
      // clipping, rounding boundary, non-finite: the float64 reference encode
      const double xd = srow ? div_rcp((double)xv[e], srow[c * 8 + e], rrow[c * 8 + e]) : (double)xv[e];
      const uint32_t code = (uint32_t)encode_code(xd, f.scale, f.rscale, f.zp, 255);
      const int sh = 8 * (e & 3);
      w[e >> 2] = (w[e >> 2] & ~(0xFFu << sh)) | (code << sh);
    }
  }
  return make_uint4(w[0], w[1], cnt, 0u);
}

template <bool GEN>
__device__ __forceinline__ uint2 fast_vec8(const uint4& u, int64_t c, const float* tab, const double* srow,
                                           const double* rrow, const FastRow& f, uint32_t& cnt) {
  float xs[8], t[8];
  smooth8(u, tab, c, xs);
  const float dm = t_and_d(xs, f, t);
  if (fast_ok<GEN>(xs, t, dm, f))
    return make_uint2(low_bytes4(t[0], t[1], t[2], t[3]), low_bytes4(t[4], t[5], t[6], t[7]));
  const uint4 sv = slow_vec8(u, tab, c, srow, rrow, f);
  cnt += sv.z;
  return make_uint2(sv.x, sv.y);
}

// xs = x * table for 8 elements, table slice preloaded (ta: elements 0-3, tb: 4-7)
__device__ __forceinline__ void smooth8_pre(const uint4& u, const float4& ta, const float4& tb, float (&xs)[8]) {
  unpack8(u, xs);
  float2 q;
  q = __fmul2_rn(make_float2(xs[0], xs[1]), make_float2(ta.x, ta.y)); xs[0] = q.x; xs[1] = q.y;
  q = __fmul2_rn(make_float2(xs[2], xs[3]), make_float2(ta.z, ta.w)); xs[2] = q.x; xs[3] = q.y;
  q = __fmul2_rn(make_float2(xs[4], xs[5]), make_float2(tb.x, tb.y)); xs[4] = q.x; xs[5] = q.y;
  q = __fmul2_rn(make_float2(xs[6], xs[7]), make_float2(tb.z, tb.w)); xs[6] = q.x; xs[7] = q.y;
}

// branch-free fast encode of 8 smoothed values; slow = the vector must take slow_vec8
template <bool GEN>
__device__ __forceinline__ uint2 fast_core(const float (&xs)[8], const FastRow& f, bool& slow) {
  float t[8];
  const float dm = t_and_d(xs, f, t);
  slow = !fast_ok<GEN>(xs, t, dm, f);
  return make_uint2(low_bytes4(t[0], t[1], t[2], t[3]), low_bytes4(t[4], t[5], t[6], t[7]));
}

// Load the lane's kBatch vectors of one batch (c = c0 + 32 b), zero past the row end.
template <int NB>
__device__ __forceinline__ void load_batch(const uint4* __restrict__ src, int c0, int nvec, uint4 (&u)[NB]) {
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    const int c = c0 + 32 * b;
    u[b] = c < nvec ? __ldg(src + c) : make_uint4(0u, 0u, 0u, 0u);
  }
}

// Pass A of one row (no producer records): float32 extremes and the first
// column holding each. Branch-free per vector (value and vector index), the
// element inside the winning vector is located once at the end.
__device__ __forceinline__ RowExt row_extremes_f32(const uint4* __restrict__ src, const float* __restrict__ tab,
                                                   int nvec, int lane) {
  float tmax = -FLT_MAX, tmin = FLT_MAX;
  int vM = 0, vm = 0;
  for (int c0 = lane; c0 < nvec; c0 += 32 * kBatch) {
    uint4 u[kBatch];
    load_batch<kBatch>(src, c0, nvec, u);
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const int c = c0 + 32 * b;
      if (c >= nvec) break;
      float xs[8];
      smooth8(u[b], tab, c, xs);
      const float vmax = max8(xs), vmin = min8(xs);
      const bool um = vmax > tmax, un = vmin < tmin;
      tmax = um ? vmax : tmax;
      vM = um ? c : vM;
      tmin = un ? vmin : tmin;
      vm = un ? c : vm;
    }
  }
  int64_t cM = vM, cm = vm;
  warp_argmax(tmax, cM);
  warp_argmin(tmin, cm);
  auto locate = [&](int64_t vc, float val) -> int64_t {
    float xs[8];
    smooth8(__ldg(src + vc), tab, vc, xs);
    int j = 0;
#pragma unroll
    for (int e = 7; e >= 0; --e) j = xs[e] == val ? e : j;
    return vc * 8 + j;
  };
  return RowExt{tmax, tmin, locate(cM, tmax), locate(cm, tmin)};
}

// Fast encode of one row with known exact parameters (FastRow): branch-free
// packed path per vector; vectors that need the slow path are remembered in
// a per-lane mask and redone after each segment of 64 vector steps, so the
// hot loop makes no calls. Returns the lane's code sum; *cnt accumulates the
// possible-extreme counts of the slow vectors.
struct NoPoll {
  __device__ __forceinline__ void operator()() const {}
};

template <bool GEN, int NB = kBatch, typename Poll = NoPoll>
__device__ __forceinline__ int encode_row_fast(const uint4* __restrict__ src, const float* __restrict__ tab,
                                               const double* srow, const double* rrow, int nvec, int lane,
                                               const FastRow& f, uint2* __restrict__ dst, uint32_t* cnt, Poll poll = Poll()) {
  int sum = 0;
  constexpr int kSeg = 32 * 64;   // vectors per segment (64 per lane)
  for (int s0 = 0; s0 < nvec; s0 += kSeg) {
    const int s1 = min(nvec, s0 + kSeg);
    uint64_t slow = 0;
    for (int base = s0; base < s1; base += 32 * NB) {   // same trip count on every lane (poll is warp-wide)
      const int c0 = base + lane;
      uint4 u[NB];
      load_batch<NB>(src, c0, s1, u);
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        const int c = c0 + 32 * b;
        if (c >= s1) break;
        float xs[8];
        smooth8(u[b], tab, c, xs);
        bool sl;
        const uint2 out = fast_core<GEN>(xs, f, sl);
        if (!sl) {
          sum += bytesum(out);
          __stcs(dst + c, out);
        }
        slow |= (uint64_t)sl << ((c - s0) >> 5);
      }
      poll();   // (fused K1: lets the caller service its other work between batches)
    }
    while (slow) {   // rare
      const int i = __ffsll((long long)slow) - 1;
      slow &= slow - 1;
      const int c = s0 + lane + 32 * i;
      const uint4 sv = slow_vec8(__ldg(src + c), tab, c, srow, rrow, f);
      *cnt += sv.z;
      const uint2 o2 = make_uint2(sv.x, sv.y);
      sum += bytesum(o2);
      __stcs(dst + c, o2);
    }
  }
  return sum;
}

// Row parameters (or the EP sidecar) of output row r.
__device__ __forceinline__ void store_row_params(const RowArgs& a, int64_t r, const AffineParams& p, int sum,
                                                 double* scale, float* scale_f32, int32_t* zp, int32_t* rowsum) {
  if (a.ep.codes_tab) {
    const float wgt = a.ep.weight ? a.ep.weight[r] : 1.0f;
    a.ep.params_tab[a.ep.dst_rank[r]][a.ep.dst_row[r]] =
        make_int4(__float_as_int((float)p.scale), p.zp, sum, __float_as_int(wgt));
  } else {
    if (rowsum) rowsum[r] = sum;
    scale[r] = p.scale;
    if (scale_f32) scale_f32[r] = (float)p.scale;
    zp[r] = p.zp;
  }
}

// One row of K1 by one warp (the per-row body of act_quant_warp_kernel;
// also run by the grouped GEMM's epilogue warps when K1 is fused into it).
template <bool GIVEN, int NB = kBatch, typename Poll = NoPoll>
__device__ __forceinline__ void k1_row_warp(const RowArgs& a, int64_t r, const float* __restrict__ rs32_tab,
                                            const unsigned long long* __restrict__ ext, int bits, int sym,
                                            uint8_t* codes, int64_t ldc, double* scale, float* scale_f32,
                                            int32_t* zp, int32_t* rowsum, int lane, Poll poll = Poll(),
                                            int64_t item = -1) {
  if (ep_row_dropped(a, r)) return;
  const int nvec = (int)(a.cols / 8);
  const bool smooth = a.sm.mode == MOE_SMOOTH_DIVIDE;
  const RowView rv = row_view(a, r, item);
  const __nv_bfloat16* row = static_cast<const __nv_bfloat16*>(a.x) + rv.off;
  const uint4* src = reinterpret_cast<const uint4*>(row);
  const float* tab = smooth ? rs32_tab + rv.gbase : nullptr;
  const double* srow = smooth ? a.sm.s + rv.gbase : nullptr;
  const double* rrow = smooth ? a.sm.rs + rv.gbase : nullptr;
  uint2* dst = reinterpret_cast<uint2*>(out_row_ptr(a, codes, ldc, r));

  // (value, column) records of the float32 extremes: producer's, or pass A
  const RowExt rec = GIVEN ? given_record(row, tab, a.cols, ext[2 * r + 1], ext[2 * r], lane)
                           : row_extremes_f32(src, tab, nvec, lane);
  const bool exact_all = !(isfinite(rec.M) && isfinite(rec.m)) || rec.cM >= a.cols || rec.cm >= a.cols;

  // speculative exact extremes: the recorded elements (verified below)
  bool spec = !exact_all;
  double mn = DBL_MAX, mx = -DBL_MAX;
  if (spec) {
    mx = exact_at(row, tab, srow, rrow, rec.cM, rec.M, spec);
    mn = exact_at(row, tab, srow, rrow, rec.cm, rec.m, spec);
  }
  // a record that names an element of the row bounds the exact extreme
  // (the max is >= lb_max, the min <= ub_min); an inconsistent one bounds nothing
  const float lb_max = spec ? rec.M - err_bound(rec.M) : -FLT_MAX;
  const float ub_min = spec ? rec.m + err_bound(rec.m) : FLT_MAX;

  AffineParams p{};
  int sum = 0;
  bool done = false;
  if (spec) {
    p = affine_params_fast(mn, mx, bits, sym);
    FastRow f;
    const int mode = init_fast_row(f, p, rec.M, rec.m, mn, mx, bits, sym);
    if (mode) {
      uint32_t cnt = 0;
      sum = mode == 1 ? encode_row_fast<false, NB>(src, tab, srow, rrow, nvec, lane, f, dst, &cnt, poll)
                      : encode_row_fast<true, NB>(src, tab, srow, rrow, nvec, lane, f, dst, &cnt, poll);
      warp_sum2(sum, cnt);
      // exactly the expected possible extremes (the recorded elements):
      // they are the exact extremes and the codes stand
      done = cnt == f.expect;
    }
  }
  if (!done) sum = fallback_row(src, nvec, lane, tab, srow, rrow, lb_max, ub_min, exact_all, bits, sym, dst, &p);
  if (lane == 0) store_row_params(a, r, p, sum, scale, scale_f32, zp, rowsum);
}

}  // namespace moe
