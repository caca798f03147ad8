// K1 hot path — bf16 rows, smoothing division, per-token RTN, bit-identical
// to the float64 reference semantics (quant.py:191-231, 314-324).
//
// Data movement (B200): a row is owned by a group of W warps (W = 1 for
// d = 4096, W = 4 for ffn = 14336). Each group streams its contiguous range
// of rows through a 2-stage shared-memory ring filled by 1-D bulk TMA copies
// (cp.async.bulk + mbarrier complete_tx): the next row is in flight while the
// current one is processed, without occupying registers. Rows are gathered
// through the MoE permutation straight from x. The float32 reciprocal table
// of the row's expert is read through L1 (a group's consecutive rows share
// an expert). HBM traffic = one read of x + one write of the codes.
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
constexpr int kStages = 2;
constexpr int64_t kSmemBudget = 220 * 1024;

__device__ __forceinline__ float err_bound(float v) { return fmaf(fabsf(v), kRelErr, kAbsErr); }

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

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

// 2 elements: returns codes (as ints, unclamped) and accumulates "unsafe".
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
                                            uint2 packed, ExactParams p, int* dsum) {
  float f[8];
  unpack8(u, f);
  uint32_t w[2] = {packed.x, packed.y};
  int delta = 0;
  for (int e = 0; e < 8; ++e) {
    if (!(mask >> e & 1u)) continue;
    const double xd = srow ? div_rcp((double)f[e], srow[c * 8 + e], rrow[c * 8 + e]) : (double)f[e];
    const uint32_t code = (uint32_t)encode_code(xd, p.scale, p.rscale, p.zp, p.qmax);
    const int sh = 8 * (e & 3);
    delta += (int)code - (int)((w[e >> 2] >> sh) & 0xFFu);
    w[e >> 2] = (w[e >> 2] & ~(0xFFu << sh)) | (code << sh);
  }
  *dsum += delta;
  return make_uint2(w[0], w[1]);
}

// Reduction across the W warps of a row group: warp shuffle, then smem +
// named barrier (id 1 + group) when W > 1.
template <int W, typename T, typename Op>
__device__ __forceinline__ T group_reduce(T v, T* slots, int gid, int wig, Op op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  if constexpr (W > 1) {
    if ((threadIdx.x & 31) == 0) slots[gid * W + wig] = v;
    named_bar_sync(1 + gid, W * 32);
    T t = slots[gid * W];
#pragma unroll
    for (int i = 1; i < W; ++i) t = op(t, slots[gid * W + i]);
    named_bar_sync(1 + gid, W * 32);
    return t;
  } else {
    return v;
  }
}

struct IntAdd {
  __device__ int operator()(int a, int b) const { return a + b; }
};

template <int W, int G>
__global__ void __launch_bounds__(W * G * 32, 1)
    act_quant_fast_kernel(RowArgs a, const float* __restrict__ rs32_tab, int bits, int sym, uint8_t* codes,
                          int64_t ldc, double* scale, float* scale_f32, int32_t* zp, int32_t* rowsum,
                          int64_t rows_per_group) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ float sf[G * W];
  __shared__ double sd[G * W];
  __shared__ int si[G * W];
  __shared__ __align__(8) uint64_t bars[G][kStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gid = warp / W, wig = warp % W;   // row group, warp in group
  const int glane = wig * 32 + lane;          // lane within the row group
  const int64_t cols = a.cols, nvec = cols / 8;
  const uint32_t row_bytes = (uint32_t)(cols * 2);
  const bool smooth = a.sm.mode == MOE_SMOOTH_DIVIDE;
  const int qmax = (1 << bits) - 1;
  uint4* ring = reinterpret_cast<uint4*>(sm) + (int64_t)gid * kStages * nvec;
  const int64_t r_lo = ((int64_t)blockIdx.x * G + gid) * rows_per_group;
  const int64_t r_hi = min(a.rows, r_lo + rows_per_group);
  const bool leader = glane == 0;

  auto issue = [&](int64_t r, int st) {
    const int64_t src = a.gather ? (int64_t)a.gather[r] : r;
    mbar_expect_tx(&bars[gid][st], row_bytes);
    bulk_g2s(ring + st * nvec, static_cast<const __nv_bfloat16*>(a.x) + src * a.ldx, row_bytes, &bars[gid][st]);
  };
  if (leader) {
    for (int st = 0; st < kStages; ++st) mbar_init(&bars[gid][st], 1);
    fence_mbar_init();
    for (int st = 0; st < kStages && r_lo + st < r_hi; ++st) issue(r_lo + st, st);
  }
  __syncthreads();
  if (r_lo >= r_hi) return;

  for (int64_t r = r_lo, it = 0; r < r_hi; ++r, ++it) {
    const int st = (int)(it & 1);
    const RowView rv = row_view(a, r);
    const float* tab = smooth ? rs32_tab + rv.gbase : nullptr;
    const double* srow = smooth ? a.sm.s + rv.gbase : nullptr;
    const double* rrow = smooth ? a.sm.rs + rv.gbase : nullptr;
    mbar_wait(&bars[gid][st], (uint32_t)((it >> 1) & 1));
    const uint4* xr = ring + st * nvec;

    // pass A: float32 extremes of the smoothed row
    float tmax = -FLT_MAX, tmin = FLT_MAX;
#pragma unroll 2
    for (int64_t c = glane; c < nvec; c += 32 * W) {
      float xs[8];
      smooth8(xr[c], tab, c, xs);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        tmax = fmaxf(tmax, xs[e]);
        tmin = fminf(tmin, xs[e]);
      }
    }
    const float M = group_reduce<W>(tmax, sf, gid, wig, OpMax());
    const float m = group_reduce<W>(tmin, sf, gid, wig, OpMin());
    const bool exact_all = !(isfinite(M) && isfinite(m));
    const float lb_max = M - err_bound(M);   // the exact max is >= this
    const float ub_min = m + err_bound(m);   // the exact min is <= this

    // pass B: exact float64 extremes over the elements that can reach them
    double mn = DBL_MAX, mx = -DBL_MAX;
    const bool scan_max = exact_all || tmax + err_bound(tmax) >= lb_max;
    const bool scan_min = exact_all || tmin - err_bound(tmin) <= ub_min;
    if (scan_max || scan_min) {
      for (int64_t c = glane; c < nvec; c += 32 * W) {
        float xs[8];
        smooth8(xr[c], tab, c, xs);
        uint32_t mmax = 0, mmin = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          mmax |= (uint32_t)(scan_max && (exact_all || xs[e] + err_bound(xs[e]) >= lb_max)) << e;
          mmin |= (uint32_t)(scan_min && (exact_all || xs[e] - err_bound(xs[e]) <= ub_min)) << e;
        }
        if (mmax | mmin) {
          const double2 ext = exact_extremes8(xr[c], srow, rrow, c, mmax, mmin);
          mn = fmin(mn, ext.x);
          mx = fmax(mx, ext.y);
        }
      }
    }
    mn = group_reduce<W>(mn, sd, gid, wig, OpMin());
    mx = group_reduce<W>(mx, sd, gid, wig, OpMax());
    const AffineParams p = affine_params(mn, mx, bits, sym);
    const float rsc32 = __double2float_rn(p.rscale);
    const float big = (float)(qmax + p.zp + 2) * 1.001f;

    // pass C: encode (float32 decision; float64 out of line near a boundary)
    int sum = 0;
    uint2* dst = reinterpret_cast<uint2*>(codes + r * ldc);
    const bool packed_ok = bits == 8 && !exact_all && fmax(fabs(mn), fabs(mx)) * p.rscale < 2097152.0;
    if (packed_ok) {
      const float2 rsc2 = make_float2(rsc32, rsc32);
      const int zpm = p.zp - kMagicBits;
#pragma unroll 2
      for (int64_t c = glane; c < nvec; c += 32 * W) {
        float xs[8];
        smooth8(xr[c], tab, c, xs);
        int q[8];
        bool unsafe = false;
#pragma unroll
        for (int e = 0; e < 8; e += 2) enc2(make_float2(xs[e], xs[e + 1]), rsc2, zpm, q[e], q[e + 1], unsafe);
        uint2 out = make_uint2(pack_sat_u8(q[0], q[1], pack_sat_u8(q[2], q[3], 0u)),
                               pack_sat_u8(q[4], q[5], pack_sat_u8(q[6], q[7], 0u)));
        sum = (int)__dp4a(out.x, 0x01010101u, (unsigned)sum);
        sum = (int)__dp4a(out.y, 0x01010101u, (unsigned)sum);
        if (unsafe) out = exact_encode8(xr[c], srow, rrow, c, 0xFFu, out, ExactParams{p.scale, p.rscale, p.zp, qmax}, &sum);
        __stcs(dst + c, out);
      }
    } else
#pragma unroll 2
    for (int64_t c = glane; c < nvec; c += 32 * W) {
      float xs[8];
      smooth8(xr[c], tab, c, xs);
      uint32_t packed[2] = {0u, 0u};
      uint32_t redo = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float v32 = xs[e] * rsc32;
        const float av = fabsf(v32);
        const float rr = rintf(av);
        const bool safe = 0.5f - fabsf(av - rr) > err_bound(av);
        const int R = (int)rr;
        int code = min(max((v32 < 0.f ? -R : R) + p.zp, 0), qmax);
        if (!safe) code = v32 < 0.f ? 0 : qmax;   // exact whenever av > big
        redo |= (uint32_t)(exact_all || (!safe && !(av > big))) << e;
        sum += code;
        packed[e >> 2] |= (uint32_t)code << (8 * (e & 3));
      }
      uint2 out = make_uint2(packed[0], packed[1]);
      if (redo) out = exact_encode8(xr[c], srow, rrow, c, redo, out, ExactParams{p.scale, p.rscale, p.zp, qmax}, &sum);
      __stcs(dst + c, out);
    }
    if (rowsum) sum = group_reduce<W>(sum, si, gid, wig, IntAdd());
    if (leader) {
      if (rowsum) rowsum[r] = sum;
      scale[r] = p.scale;
      if (scale_f32) scale_f32[r] = (float)p.scale;
      zp[r] = p.zp;
    }
    // refill this stage with row r + 2 once every lane of the group is done with it
    if constexpr (W > 1) named_bar_sync(1 + gid, W * 32);
    else __syncwarp();
    if (leader && r + kStages < r_hi) {
      fence_proxy_async_smem();
      issue(r + kStages, st);
    }
  }
}

template <int W, int G>
static cudaError_t launch_wg(const RowArgs& a, const float* rs32, int bits, int sym, uint8_t* codes, int64_t ldc,
                             double* scale, float* scale_f32, int32_t* zp, int32_t* rowsum, cudaStream_t s) {
  const int64_t smem = (int64_t)G * kStages * a.cols * 2;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(act_quant_fast_kernel<W, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSmemBudget);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  // persistent: one CTA per SM; every row group walks a contiguous row range
  const int64_t groups = std::min<int64_t>(a.rows, (int64_t)num_sms() * G);
  const int64_t rows_per_group = (a.rows + groups - 1) / groups;
  const int64_t used = (a.rows + rows_per_group - 1) / rows_per_group;
  const int64_t blocks = (used + G - 1) / G;
  act_quant_fast_kernel<W, G><<<(unsigned)blocks, W * G * 32, (size_t)smem, s>>>(
      a, rs32, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, rows_per_group);
  count_launch();
  return cudaGetLastError();
}

bool launch_act_quant_fast(const RowArgs& a, const float* rs32, int bits, int sym, uint8_t* codes, int64_t ldc,
                           double* scale, float* scale_f32, int32_t* zp, int32_t* rowsum, cudaStream_t s,
                           cudaError_t* err) {
  const bool smooth = a.sm.mode == MOE_SMOOTH_DIVIDE;
  const int64_t row_bytes = a.cols * 2;
  if (a.dt != MOE_DT_BF16 || a.cols % 8 || a.ldx % 8 || ldc % 8 ||
      (reinterpret_cast<uintptr_t>(a.x) & 15) || (reinterpret_cast<uintptr_t>(codes) & 7) ||
      !(a.sm.mode == MOE_SMOOTH_NONE || (smooth && a.sm.rs && rs32)))
    return false;
  // W warps per row (>= ~28 vectors per lane keeps the loop efficient),
  // G row groups per CTA so that G * 2 stages of rows fit in shared memory.
  auto fits = [&](int G) { return (int64_t)G * kStages * row_bytes <= kSmemBudget; };
  if (row_bytes <= 4096 && fits(16)) *err = launch_wg<1, 16>(a, rs32, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, s);
  else if (row_bytes <= 12 * 1024 && fits(8)) *err = launch_wg<1, 8>(a, rs32, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, s);
  else if (fits(4)) *err = launch_wg<4, 4>(a, rs32, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, s);
  else if (fits(2)) *err = launch_wg<8, 2>(a, rs32, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, s);
  else if (fits(1)) *err = launch_wg<16, 1>(a, rs32, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, s);
  else return false;
  return true;
}

}  // namespace moe
