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

// warp arg-reduce: larger value wins, ties to the lower column
__device__ __forceinline__ void warp_argmax(float& v, int64_t& col) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int64_t c2 = __shfl_xor_sync(0xffffffffu, col, o);
    if (v2 > v || (v2 == v && c2 < col)) {
      v = v2;
      col = c2;
    }
  }
}
__device__ __forceinline__ void warp_argmin(float& v, int64_t& col) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int64_t c2 = __shfl_xor_sync(0xffffffffu, col, o);
    if (v2 < v || (v2 == v && c2 < col)) {
      v = v2;
      col = c2;
    }
  }
}

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
// below 0.5 - 2^-13: those codes equal the float64 reference's (|p| <= 254
// there and p = y (1 + e), |e| <= 3 2^-24 + 2^-50, so |p - y| < 2^-14; d
// itself carries one rounding of at most 2^-26). Everything else —
// clipping, rounding-boundary cases, non-finite values and the elements
// that could be row extremes (codes <= 1 / >= 254) — goes out of line.
constexpr float kMagicF = 12582912.0f;
constexpr float kFastTlo = 12582914.0f;          // code 2
constexpr float kFastThi = 12583165.0f;          // code 253
constexpr float kFastThr = 0.4998779296875f;     // 0.5 - 2^-13

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

// Rare vectors: generic float32 encode (clip, exact float64 redo) plus the
// count of possible-extreme elements. Returns (codes, cnt_max | cnt_min << 16).
__device__ __noinline__ uint4 slow_vec8(uint4 u, const float* tab, int64_t c, const double* srow, const double* rrow,
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

__device__ __forceinline__ uint32_t low_bytes4(float a, float b, float c, float d) {
  const uint32_t ab = __byte_perm(__float_as_uint(a), __float_as_uint(b), 0x0040);
  const uint32_t cd = __byte_perm(__float_as_uint(c), __float_as_uint(d), 0x0040);
  return __byte_perm(ab, cd, 0x5410);
}

// Fallback for a whole row: float64 extremes over every element that can
// reach them (pass B), then the generic encode (pass C). Used when the
// speculative extremes fail their check, for symmetric / non-8-bit codes
// and for rows outside the fast envelope.
__device__ __noinline__ int fallback_row(const uint4* src, int64_t nvec, int lane, const float* tab,
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
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  *out = p;
  return sum;
}

template <bool GEN>
__device__ __forceinline__ bool fast_ok(const float (&xs)[8], const float (&t)[8], float dm, const FastRow& f) {
  bool ok = max8(t) <= f.thi && min8(t) >= f.tlo && dm < kFastThr;
  if (GEN) ok = ok && max8(xs) <= f.xhi && min8(xs) >= f.xlo;
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
__device__ __forceinline__ void smooth8_pre(const uint4& u, bool has_tab, const float4& ta, const float4& tb,
                                            float (&xs)[8]) {
  unpack8(u, xs);
  if (has_tab) {
    float2 q;
    q = __fmul2_rn(make_float2(xs[0], xs[1]), make_float2(ta.x, ta.y)); xs[0] = q.x; xs[1] = q.y;
    q = __fmul2_rn(make_float2(xs[2], xs[3]), make_float2(ta.z, ta.w)); xs[2] = q.x; xs[3] = q.y;
    q = __fmul2_rn(make_float2(xs[4], xs[5]), make_float2(tb.x, tb.y)); xs[4] = q.x; xs[5] = q.y;
    q = __fmul2_rn(make_float2(xs[6], xs[7]), make_float2(tb.z, tb.w)); xs[6] = q.x; xs[7] = q.y;
  }
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
__device__ __forceinline__ void load_batch(const uint4* __restrict__ src, int c0, int nvec, uint4 (&u)[kBatch]) {
#pragma unroll
  for (int b = 0; b < kBatch; ++b) {
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
    load_batch(src, c0, nvec, u);
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
template <bool GEN>
__device__ __forceinline__ int encode_row_fast(const uint4* __restrict__ src, const float* __restrict__ tab,
                                               const double* srow, const double* rrow, int nvec, int lane,
                                               const FastRow& f, uint2* __restrict__ dst, uint32_t* cnt) {
  int sum = 0;
  constexpr int kSeg = 32 * 64;   // vectors per segment (64 per lane)
  for (int s0 = 0; s0 < nvec; s0 += kSeg) {
    const int s1 = min(nvec, s0 + kSeg);
    uint64_t slow = 0;
    for (int c0 = s0 + lane; c0 < s1; c0 += 32 * kBatch) {
      uint4 u[kBatch];
      load_batch(src, c0, s1, u);
#pragma unroll
      for (int b = 0; b < kBatch; ++b) {
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

template <bool GIVEN, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB)
    act_quant_warp_kernel(RowArgs a, const float* __restrict__ rs32_tab, const unsigned long long* __restrict__ ext,
                          int bits, int sym, uint8_t* codes, int64_t ldc, double* scale, float* scale_f32,
                          int32_t* zp, int32_t* rowsum, int64_t rows_per_cta) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nvec = (int)(a.cols / 8);
  const bool smooth = a.sm.mode == MOE_SMOOTH_DIVIDE;
  // each CTA owns a contiguous range of rows (shared expert tables in L1)
  const int64_t r_lo = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r_hi = min(a.rows, r_lo + rows_per_cta);
  for (int64_t r = r_lo + warp; r < r_hi; r += WARPS) {
    const RowView rv = row_view(a, r);
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
      p = affine_params(mn, mx, bits, sym);
      FastRow f;
      const int mode = init_fast_row(f, p, rec.M, rec.m, mn, mx, bits, sym);
      if (mode) {
        uint32_t cnt = 0;
        sum = mode == 1 ? encode_row_fast<false>(src, tab, srow, rrow, nvec, lane, f, dst, &cnt)
                        : encode_row_fast<true>(src, tab, srow, rrow, nvec, lane, f, dst, &cnt);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          sum += __shfl_xor_sync(0xffffffffu, sum, o);
          cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        }
        // exactly the expected possible extremes (the recorded elements):
        // they are the exact extremes and the codes stand
        done = cnt == f.expect;
      }
    }
    if (!done) sum = fallback_row(src, nvec, lane, tab, srow, rrow, lb_max, ub_min, exact_all, bits, sym, dst, &p);
    if (lane == 0) {
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
  }
  if (a.ep.codes_tab) __threadfence_system();   // peer writes visible before the rank barrier
}

// ── bulk-async (TMA) streaming variant ─────────────────────────────────────
// Same per-row algorithm as act_quant_warp_kernel, but rows are streamed
// through a per-warp ring of kRing x 2 KB shared-memory stages filled by
// cp.async.bulk (one elected lane issues, an mbarrier per stage completes
// on the byte count): 6 KB in flight per warp regardless of register
// pressure, ~100 KB per 16-warp CTA. Rows that fit the ring (d <= 3072) are
// held for the second pass; longer rows without records are streamed twice.
constexpr int kChunkBytes = 2048;
constexpr int kChunkVec = kChunkBytes / 16;   // 128 x 16 B: 4 vectors per lane
// 3 stages (6 KB per warp, 98 KB per CTA): the rest of the SM's 256 KB stays
// L1 and holds the expert's float32 reciprocal table (57 KB at ffn = 14336);
// 6 stages left ~30 KB of L1 and the table loads went to L2 (368 vs 346 us)
constexpr int kRing = 3;
constexpr int kBulkWarps = 16;       // (24 / 32 warps with smaller rings: register spills, 476 / 550 us)
constexpr int kVecStep = 2;     // vectors per lane processed together (register budget: 16 warps)
constexpr int kBulkSmem = kBulkWarps * kRing * (kChunkBytes + 8) + 128;

template <bool GIVEN>
__global__ void __launch_bounds__(kBulkWarps * 32, 1)
    act_quant_bulk_kernel(RowArgs a, const float* __restrict__ rs32_tab, const unsigned long long* __restrict__ ext,
                          int bits, int sym, uint8_t* codes, int64_t ldc, double* scale, float* scale_f32,
                          int32_t* zp, int32_t* rowsum, int64_t rows_per_cta) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint8_t* ring = smem_raw + warp * kRing * kChunkBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + kBulkWarps * kRing * kChunkBytes) + warp * kRing;
  if (lane == 0) {
    for (int i = 0; i < kRing; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncwarp();

  const int64_t nvec = a.cols / 8;
  const int64_t row_bytes = a.cols * 2;
  const int nchunks = (int)((nvec + kChunkVec - 1) / kChunkVec);
  const bool hold = !GIVEN && nchunks <= kRing;
  const int items_per_row = (GIVEN || hold) ? nchunks : 2 * nchunks;
  const bool smooth = a.sm.mode == MOE_SMOOTH_DIVIDE;
  const int64_t r_lo = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r_hi = min(a.rows, r_lo + rows_per_cta);
  const uint64_t pol = policy_evict_first();

  // producer: the warp's item stream (row, chunk) in consumption order
  int64_t prow = r_lo + warp;
  int pitem = 0;
  uint32_t pcount = 0;
  int64_t prow_off = prow < r_hi ? row_view(a, prow).off : 0;
  auto produce = [&]() {
    if (prow >= r_hi) return;
    if (lane == 0) {
      const int chunk = pitem % nchunks;
      const int64_t b0 = (int64_t)chunk * kChunkBytes;
      const uint32_t bytes = (uint32_t)min((int64_t)kChunkBytes, row_bytes - b0);
      const int st = (int)(pcount % kRing);
      fence_proxy_async_smem();
      mbar_expect_tx(&bars[st], bytes);
      bulk_load(ring + st * kChunkBytes, static_cast<const uint8_t*>(a.x) + prow_off * 2 + b0, bytes, &bars[st],
                pol);
    }
    ++pcount;
    if (++pitem == items_per_row) {
      pitem = 0;
      prow += kBulkWarps;
      if (prow < r_hi) prow_off = row_view(a, prow).off;
    }
  };
  for (int i = 0; i < kRing; ++i) produce();
  uint32_t ccount = 0;
  auto wait_item = [&](uint32_t it) { mbar_wait(&bars[it % kRing], (it / kRing) & 1u); };
  auto item_vec = [&](uint32_t it) { return reinterpret_cast<const uint4*>(ring + (it % kRing) * kChunkBytes); };
  for (int64_t r = r_lo + warp; r < r_hi; r += kBulkWarps) {
    const RowView rv = row_view(a, r);
    const __nv_bfloat16* row = static_cast<const __nv_bfloat16*>(a.x) + rv.off;
    const uint4* src = reinterpret_cast<const uint4*>(row);
    const float* tab = smooth ? rs32_tab + rv.gbase : nullptr;
    const double* srow = smooth ? a.sm.s + rv.gbase : nullptr;
    const double* rrow = smooth ? a.sm.rs + rv.gbase : nullptr;
    uint2* dst = reinterpret_cast<uint2*>(out_row_ptr(a, codes, ldc, r));
    const uint32_t base = ccount;
    ccount += items_per_row;

    RowExt rec;
    if (GIVEN) {
      const unsigned long long kmin = ext[2 * r], kmax = ext[2 * r + 1];
      rec = given_record(row, tab, a.cols, kmax, kmin, lane);
    } else {
      // per lane: running max / min and the vector holding them (first
      // occurrence), then the element inside that vector
      float tmax = -FLT_MAX, tmin = FLT_MAX;
      int64_t vmaxc = 0, vminc = 0;
      for (int k = 0; k < nchunks; ++k) {
        const uint32_t it = base + k;
        wait_item(it);
        const uint4* v = item_vec(it);
        const int64_t cb = (int64_t)k * kChunkVec + lane;
        const bool full = (int64_t)(k + 1) * kChunkVec <= nvec;
        uint4 u[4];
        float4 ta[4], tb[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const bool ok = full || cb + 32 * b < nvec;
          u[b] = ok ? v[lane + 32 * b] : make_uint4(0u, 0u, 0u, 0u);
          if (tab && ok) {
            ta[b] = __ldg(reinterpret_cast<const float4*>(tab) + 2 * (cb + 32 * b));
            tb[b] = __ldg(reinterpret_cast<const float4*>(tab) + 2 * (cb + 32 * b) + 1);
          }
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if (!(full || cb + 32 * b < nvec)) continue;
          float xs[8];
          smooth8_pre(u[b], tab != nullptr, ta[b], tb[b], xs);
          const float vmax = max8(xs), vmin = min8(xs);
          const bool um = vmax > tmax, un = vmin < tmin;
          tmax = um ? vmax : tmax;
          vmaxc = um ? cb + 32 * b : vmaxc;
          tmin = un ? vmin : tmin;
          vminc = un ? cb + 32 * b : vminc;
        }
        __syncwarp();
        if (!hold) produce();
      }
      warp_argmax(tmax, vmaxc);
      warp_argmin(tmin, vminc);
      // locate the element (first in the vector) from the resident chunk, or global
      auto locate = [&](int64_t vc, float val) -> int64_t {
        const uint4 u = hold ? item_vec(base + (uint32_t)(vc / kChunkVec))[vc % kChunkVec] : src[vc];
        float xs[8];
        smooth8(u, tab, vc, xs);
        int j = 0;
#pragma unroll
        for (int e = 7; e >= 0; --e) j = xs[e] == val ? e : j;
        return vc * 8 + j;
      };
      const int64_t imax = locate(vmaxc, tmax), imin = locate(vminc, tmin);
      rec = RowExt{tmax, tmin, imax, imin};
    }
    const uint32_t cfirst = (GIVEN || hold) ? base : base + nchunks;   // items of the encode pass
    const bool exact_all = !(isfinite(rec.M) && isfinite(rec.m)) || rec.cM >= a.cols || rec.cm >= a.cols;
    bool spec = !exact_all;
    double mn = DBL_MAX, mx = -DBL_MAX;
    if (spec) {
      mx = exact_at(row, tab, srow, rrow, rec.cM, rec.M, spec);
      mn = exact_at(row, tab, srow, rrow, rec.cm, rec.m, spec);
    }
    const float lb_max = spec ? rec.M - err_bound(rec.M) : -FLT_MAX;
    const float ub_min = spec ? rec.m + err_bound(rec.m) : FLT_MAX;

    AffineParams p{};
    int sum = 0;
    bool done = false;
    FastRow f;
    int mode = 0;
    if (spec) {
      p = affine_params(mn, mx, bits, sym);
      mode = init_fast_row(f, p, rec.M, rec.m, mn, mx, bits, sym);
    }
    if (mode) {
      uint32_t cnt = 0;
      auto run = [&](auto gen) {
      constexpr bool G = decltype(gen)::value;
      for (int k = 0; k < nchunks; ++k) {
        const uint32_t it = cfirst + k;
        wait_item(it);
        const uint4* v = item_vec(it);
        const int64_t cb = (int64_t)k * kChunkVec + lane;
        if ((int64_t)(k + 1) * kChunkVec <= nvec) {
          // full chunk, two vectors at a time: table loads up front, no
          // per-vector branches; the rare slow vectors are redone afterwards
          // from the staged copy (same lane, same addresses)
#pragma unroll
          for (int hf = 0; hf < 4; hf += kVecStep) {
            uint4 u[kVecStep];
            float4 ta[kVecStep], tb[kVecStep];
#pragma unroll
            for (int b = 0; b < kVecStep; ++b) {
              u[b] = v[lane + 32 * (hf + b)];
              if (tab) {
                ta[b] = __ldg(reinterpret_cast<const float4*>(tab) + 2 * (cb + 32 * (hf + b)));
                tb[b] = __ldg(reinterpret_cast<const float4*>(tab) + 2 * (cb + 32 * (hf + b)) + 1);
              }
            }
            uint2 out[kVecStep];
            uint32_t slowm = 0;
#pragma unroll
            for (int b = 0; b < kVecStep; ++b) {
              float xs[8];
              smooth8_pre(u[b], tab != nullptr, ta[b], tb[b], xs);
              bool sl;
              out[b] = fast_core<G>(xs, f, sl);
              slowm |= (uint32_t)sl << b;
            }
#pragma unroll
            for (int b = 0; b < kVecStep; ++b) {
              sum += bytesum(out[b]);
              __stcs(dst + cb + 32 * (hf + b), out[b]);
            }
            if (slowm) {
              for (int b = 0; b < kVecStep; ++b) {
                if (!(slowm >> b & 1u)) continue;
                const int64_t c = cb + 32 * (hf + b);
                const uint4 sv = slow_vec8(v[lane + 32 * (hf + b)], tab, c, srow, rrow, f);
                cnt += sv.z;
                const uint2 o2 = make_uint2(sv.x, sv.y);
                sum += bytesum(o2) - bytesum(out[b]);
                __stcs(dst + c, o2);
              }
            }
          }
        } else {
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int64_t c = cb + 32 * b;
            if (c < nvec) {
              const uint2 out = fast_vec8<G>(v[lane + 32 * b], c, tab, srow, rrow, f, cnt);
              sum += bytesum(out);
              __stcs(dst + c, out);
            }
          }
        }
        __syncwarp();
        produce();
      }
      };
      if (mode == 1) run(std::false_type{});
      else run(std::true_type{});
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        sum += __shfl_xor_sync(0xffffffffu, sum, o);
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
      }
      done = cnt == f.expect;
    } else {
      for (int k = 0; k < nchunks; ++k) {   // keep the ring in step
        wait_item(cfirst + k);
        __syncwarp();
        produce();
      }
    }
    if (!done) sum = fallback_row(src, nvec, lane, tab, srow, rrow, lb_max, ub_min, exact_all, bits, sym, dst, &p);
    if (lane == 0) {
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
  }
  if (a.ep.codes_tab) __threadfence_system();   // peer writes visible before the rank barrier
}

// ── CTA-per-row variant for small row counts ───────────────────────────────
// Decode-size batches have a few dozen rows: one warp per row leaves most
// SMs idle and runs each row as one long dependent chain (~25 us for 32
// rows). Here a 512-thread CTA owns one row, every thread holds up to four
// 16-byte vectors of it in registers (rows up to 16384 bf16), and the
// per-row reductions are block-wide; the per-vector arithmetic (float32
// filter, speculative extremes, candidate count, exact fallback) is the
// warp kernel's, so the results are identical.
constexpr int kCtaThreads = 512;
constexpr int kCtaNV = 4;

struct OpMaxU64 {
  __device__ unsigned long long operator()(unsigned long long a, unsigned long long b) const { return a > b ? a : b; }
};
struct OpMinU64 {
  __device__ unsigned long long operator()(unsigned long long a, unsigned long long b) const { return a < b ? a : b; }
};
// order-preserving 32-bit key of a float (no NaNs here)
__device__ __forceinline__ uint32_t fkey(float v) {
  const uint32_t b = __float_as_uint(v);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float funkey(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}

struct CtaRowState {
  RowExt rec;
  AffineParams p;
  FastRow f;
  float lb_max, ub_min;
  int mode;
  bool exact_all;
};

template <bool GIVEN>
__global__ void __launch_bounds__(kCtaThreads)
    act_quant_cta_kernel(RowArgs a, const float* __restrict__ rs32_tab, const unsigned long long* __restrict__ ext,
                         int bits, int sym, uint8_t* codes, int64_t ldc, double* scale, float* scale_f32,
                         int32_t* zp, int32_t* rowsum) {
  __shared__ unsigned long long sh64[kCtaThreads / 32];
  __shared__ double shd[kCtaThreads / 32];
  __shared__ int64_t shi[kCtaThreads / 32];
  __shared__ CtaRowState st;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r = blockIdx.x;
  const int64_t nvec = a.cols / 8;
  const bool smooth = a.sm.mode == MOE_SMOOTH_DIVIDE;
  const RowView rv = row_view(a, r);
  const __nv_bfloat16* row = static_cast<const __nv_bfloat16*>(a.x) + rv.off;
  const uint4* src = reinterpret_cast<const uint4*>(row);
  const float* tab = smooth ? rs32_tab + rv.gbase : nullptr;
  const double* srow = smooth ? a.sm.s + rv.gbase : nullptr;
  const double* rrow = smooth ? a.sm.rs + rv.gbase : nullptr;
  uint2* dst = reinterpret_cast<uint2*>(out_row_ptr(a, codes, ldc, r));

  uint4 u[kCtaNV];
#pragma unroll
  for (int i = 0; i < kCtaNV; ++i) {
    const int64_t c = tid + (int64_t)i * kCtaThreads;
    u[i] = c < nvec ? src[c] : make_uint4(0u, 0u, 0u, 0u);
  }
  if (GIVEN) {
    if (warp == 0) {
      const RowExt rec = given_record(row, tab, a.cols, ext[2 * r + 1], ext[2 * r], lane);
      if (lane == 0) st.rec = rec;
    }
  } else {
    // pass A: float32 extremes and a column holding each (larger / smaller
    // value wins, ties to the lower column)
    float tmax = -FLT_MAX, tmin = FLT_MAX;
    int64_t imax = 0, imin = 0;
#pragma unroll
    for (int i = 0; i < kCtaNV; ++i) {
      const int64_t c = tid + (int64_t)i * kCtaThreads;
      if (c >= nvec) continue;
      float xs[8];
      smooth8(u[i], tab, c, xs);
      const float vmax = max8(xs), vmin = min8(xs);
      if (vmax > tmax) {
        int j = 0;
#pragma unroll
        for (int e = 7; e >= 0; --e) j = xs[e] == vmax ? e : j;
        tmax = vmax;
        imax = c * 8 + j;
      }
      if (vmin < tmin) {
        int j = 0;
#pragma unroll
        for (int e = 7; e >= 0; --e) j = xs[e] == vmin ? e : j;
        tmin = vmin;
        imin = c * 8 + j;
      }
    }
    const unsigned long long kM = block_reduce(
        ((unsigned long long)fkey(tmax) << 32) | (0xFFFFFFFFu - (uint32_t)imax), sh64, OpMaxU64());
    const unsigned long long km = block_reduce(((unsigned long long)fkey(tmin) << 32) | (uint32_t)imin, sh64,
                                               OpMinU64());
    if (tid == 0)
      st.rec = RowExt{funkey((uint32_t)(kM >> 32)), funkey((uint32_t)(km >> 32)),
                      (int64_t)(0xFFFFFFFFu - (uint32_t)kM), (int64_t)(uint32_t)km};
  }
  __syncthreads();
  if (tid == 0) {
    const RowExt rec = st.rec;
    const bool exact_all = !(isfinite(rec.M) && isfinite(rec.m)) || rec.cM >= a.cols || rec.cm >= a.cols;
    bool spec = !exact_all;
    double mn = DBL_MAX, mx = -DBL_MAX;
    if (spec) {
      mx = exact_at(row, tab, srow, rrow, rec.cM, rec.M, spec);
      mn = exact_at(row, tab, srow, rrow, rec.cm, rec.m, spec);
    }
    st.lb_max = spec ? rec.M - err_bound(rec.M) : -FLT_MAX;
    st.ub_min = spec ? rec.m + err_bound(rec.m) : FLT_MAX;
    st.exact_all = exact_all;
    st.mode = 0;
    if (spec) {
      st.p = affine_params(mn, mx, bits, sym);
      st.mode = init_fast_row(st.f, st.p, rec.M, rec.m, mn, mx, bits, sym);
    }
  }
  __syncthreads();
  const int mode = st.mode;
  AffineParams p = st.p;
  int sum = 0;
  bool done = false;
  if (mode) {
    const FastRow f = st.f;
    uint32_t cnt = 0;
    auto run = [&](auto gen) {
      constexpr bool G = decltype(gen)::value;
#pragma unroll
      for (int i = 0; i < kCtaNV; ++i) {
        const int64_t c = tid + (int64_t)i * kCtaThreads;
        if (c >= nvec) continue;
        const uint2 out = fast_vec8<G>(u[i], c, tab, srow, rrow, f, cnt);
        sum += bytesum(out);
        __stcs(dst + c, out);
      }
    };
    if (mode == 1) run(std::false_type{});
    else run(std::true_type{});
    sum = (int)block_reduce((int64_t)sum, shi, OpAdd());
    done = (uint32_t)block_reduce((int64_t)cnt, shi, OpAdd()) == f.expect;
  }
  if (!done) {
    // exact extremes over every element that can reach them, then the
    // generic encode (as fallback_row, block-wide)
    const float lb_max = st.lb_max, ub_min = st.ub_min;
    double mn = DBL_MAX, mx = -DBL_MAX;
#pragma unroll
    for (int i = 0; i < kCtaNV; ++i) {
      const int64_t c = tid + (int64_t)i * kCtaThreads;
      if (c >= nvec) continue;
      float xs[8];
      smooth8(u[i], tab, c, xs);
      uint32_t mmax = 0, mmin = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        mmax |= (uint32_t)(!(xs[e] + err_bound(xs[e]) < lb_max)) << e;
        mmin |= (uint32_t)(!(xs[e] - err_bound(xs[e]) > ub_min)) << e;
      }
      if (mmax | mmin) {
        const double2 e2 = exact_extremes8(u[i], srow, rrow, c, mmax, mmin);
        mn = fmin(mn, e2.x);
        mx = fmax(mx, e2.y);
      }
    }
    mn = block_reduce(mn, shd, OpMin());
    mx = block_reduce(mx, shd, OpMax());
    p = affine_params(mn, mx, bits, sym);
    const RowEncoder enc(p, mn, mx, bits, st.exact_all);
    int s = 0;
#pragma unroll
    for (int i = 0; i < kCtaNV; ++i) {
      const int64_t c = tid + (int64_t)i * kCtaThreads;
      if (c >= nvec) continue;
      float xs[8];
      smooth8(u[i], tab, c, xs);
      __stcs(dst + c, enc.encode8(u[i], xs, c, srow, rrow, s));
    }
    sum = (int)block_reduce((int64_t)s, shi, OpAdd());
  }
  if (tid == 0) {
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
  if (a.ep.codes_tab) __threadfence_system();   // peer writes visible before the rank barrier
}

template <bool GIVEN>
static cudaError_t launch_bulk(const RowArgs& a, const float* rs32, const unsigned long long* ext, int bits, int sym,
                               uint8_t* codes, int64_t ldc, double* scale, float* scale_f32, int32_t* zp,
                               int32_t* rowsum, cudaStream_t s) {
  {
    const cudaError_t e = set_max_smem_once(reinterpret_cast<const void*>(act_quant_bulk_kernel<GIVEN>), kBulkSmem);
    if (e != cudaSuccess) return e;
  }
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>((a.rows + kBulkWarps - 1) / kBulkWarps, num_sms()));
  const int64_t rows_per_cta = (a.rows + ctas - 1) / ctas;
  const int64_t nblk = (a.rows + rows_per_cta - 1) / rows_per_cta;
  act_quant_bulk_kernel<GIVEN><<<(unsigned)nblk, kBulkWarps * 32, kBulkSmem, s>>>(
      a, rs32, ext, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, rows_per_cta);
  count_launch();
  return cudaGetLastError();
}

static bool eligible(const RowArgs& a, const float* rs32, uint8_t* codes, int64_t ldc) {
  const bool smooth = a.sm.mode == MOE_SMOOTH_DIVIDE;
  return a.dt == MOE_DT_BF16 && a.cols % 8 == 0 && a.ldx % 8 == 0 && ldc % 8 == 0 &&
         (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 && (reinterpret_cast<uintptr_t>(codes) & 7) == 0 &&
         (a.sm.mode == MOE_SMOOTH_NONE || (smooth && a.sm.rs && rs32));
}

template <bool GIVEN, int WARPS, int MINB>
static void launch_cfg(const RowArgs& a, const float* rs32, const unsigned long long* ext, int bits, int sym,
                       uint8_t* codes, int64_t ldc, double* scale, float* scale_f32, int32_t* zp, int32_t* rowsum,
                       cudaStream_t s) {
  // contiguous row ranges, MINB+ CTAs per SM
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>((a.rows + WARPS - 1) / WARPS,
                                                              (MINB + 2) * (int64_t)num_sms()));
  const int64_t rows_per_cta = (a.rows + ctas - 1) / ctas;
  const int64_t nblk = (a.rows + rows_per_cta - 1) / rows_per_cta;
  act_quant_warp_kernel<GIVEN, WARPS, MINB><<<(unsigned)nblk, WARPS * 32, 0, s>>>(
      a, rs32, ext, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, rows_per_cta);
}

// Kernel choice (measured on B200 at the Mixtral shape): rows with producer
// records (h) stream through the bulk-async ring (371 vs 387 us); rows that
// need their own extreme pass (x, gathered) use the register kernel, whose
// second pass and the router's just-read rows hit L1/L2 (in the step: 222 vs
// 258 us). MOE_B200_K1_CFG=0 / 7 forces one kernel for both (A/B runs).
// Calls with at most MOE_TUNE_K1_SMALL_ROWS rows (decode-size batches) use
// the CTA-per-row kernel (tools/k1_small.py).
template <bool GIVEN>
static cudaError_t launch_warp(const RowArgs& a, const float* rs32, const unsigned long long* ext, int bits, int sym,
                              uint8_t* codes, int64_t ldc, double* scale, float* scale_f32, int32_t* zp,
                              int32_t* rowsum, cudaStream_t s) {
  static const int forced = [] {
    const char* env = getenv("MOE_B200_K1_CFG");
    return env ? atoi(env) : -1;
  }();
  if (a.rows <= k1_small_rows() && a.cols <= (int64_t)kCtaNV * kCtaThreads * 8) {
    act_quant_cta_kernel<GIVEN><<<(unsigned)a.rows, kCtaThreads, 0, s>>>(a, rs32, ext, bits, sym, codes, ldc, scale,
                                                                          scale_f32, zp, rowsum);
    count_launch();
    return cudaGetLastError();
  }
  const bool bulk = forced == 7 || (forced < 0 && GIVEN);
  if (bulk) return launch_bulk<GIVEN>(a, rs32, ext, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, s);
  launch_cfg<GIVEN, 16, 2>(a, rs32, ext, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, s);
  count_launch();
  return cudaGetLastError();
}

bool launch_act_quant_given(const RowArgs& a, const float* rs32, const unsigned long long* ext, int bits, int sym,
                            uint8_t* codes, int64_t ldc, double* scale, float* scale_f32, int32_t* zp,
                            int32_t* rowsum, cudaStream_t s, cudaError_t* err) {
  if (!ext || !eligible(a, rs32, codes, ldc)) return false;
  *err = launch_warp<true>(a, rs32, ext, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, s);
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
