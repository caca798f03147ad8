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

#include "k1_fast.cuh"

namespace moe {

template <bool GIVEN, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB)
    act_quant_warp_kernel(RowArgs a, const float* __restrict__ rs32_tab, const unsigned long long* __restrict__ ext,
                          int bits, int sym, uint8_t* codes, int64_t ldc, double* scale, float* scale_f32,
                          int32_t* zp, int32_t* rowsum, int64_t rows_per_cta) {
  griddep_launch_dependents();   // the next (PDL-launched) GEMM may start its weight prefetch
  griddep_wait();                // PDL-launched: the previous kernel's outputs are visible from here
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  // each CTA owns a contiguous range of rows (shared expert tables in L1)
  int64_t r_lo, r_hi;
  cta_row_range(a, rows_per_cta, r_lo, r_hi);
  for (int64_t i = r_lo + warp; i < r_hi; i += WARPS) {
    if (a.order)   // token-major walk: item i = (token i / k, its (i % k)-th row)
      k1_row_warp<GIVEN>(a, a.order[i], rs32_tab, ext, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, lane,
                         NoPoll(), i);
    else
      k1_row_warp<GIVEN>(a, i, rs32_tab, ext, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, lane);
  }
  if (a.ep.codes_tab) __threadfence_system();   // peer writes visible before the rank barrier
}

// ── bulk-async (TMA) streaming variant ─────────────────────────────────────
// Same per-row algorithm as act_quant_warp_kernel, but rows are streamed
// through a per-warp ring of kRing x kChunkBytes shared-memory stages filled
// by cp.async.bulk (one elected lane issues, an mbarrier per stage completes
// on the byte count): 8 KB in flight per warp regardless of register
// pressure, 128 KB per 16-warp CTA. Rows that fit the ring are held for the
// second pass; longer rows without records are streamed twice.
//
// Ring shape (K1 on h at the Mixtral shape, tools/k1x_ab.py, interleaved
// A/B): 2 x 4 KB 316 us, 3 x 2 KB 335 us, 3 x 4 KB 337 us (L1 left for the
// expert's 57 KB float32 reciprocal table shrinks), 6 x 2 KB 368 us. Larger
// chunks halve the per-chunk bookkeeping (ring wait, bulk issue), which
// ncu put at ~15 % of the kernel's instructions with 2 KB chunks.
// Deferring the rare slow vectors to one warp-wide pass per row measured
// slower (+1-2 %) and was dropped.
#ifndef MOE_K1_CHUNK
#define MOE_K1_CHUNK 4096
#endif
#ifndef MOE_K1_RING
#define MOE_K1_RING 2
#endif
constexpr int kChunkBytes = MOE_K1_CHUNK;
constexpr int kChunkVec = kChunkBytes / 16;   // 16-byte vectors per chunk
constexpr int kLaneVec = kChunkVec / 32;      // per lane (8 at 4 KB)
static_assert(kChunkBytes % 512 == 0, "chunk = whole 16-byte vectors for every lane");
constexpr int kRing = MOE_K1_RING;
constexpr int kBulkWarps = 16;       // (24 / 32 warps with smaller rings: register spills, 476 / 550 us)
constexpr int kVecStep = 4;     // vectors per lane processed together (119 registers, no spills; 2: 334 us, 4: 328 us)
constexpr int kBulkSmem = kBulkWarps * kRing * (kChunkBytes + 8) + 128;
static_assert(kLaneVec % kVecStep == 0, "a chunk's per-lane vectors come in kVecStep groups");

template <bool GIVEN>
__global__ void __launch_bounds__(kBulkWarps * 32, 1)
    act_quant_bulk_kernel(RowArgs a, const float* __restrict__ rs32_tab, const unsigned long long* __restrict__ ext,
                          int bits, int sym, uint8_t* codes, int64_t ldc, double* scale, float* scale_f32,
                          int32_t* zp, int32_t* rowsum, int64_t rows_per_cta) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  griddep_launch_dependents();   // the next (PDL-launched) GEMM may start its weight prefetch
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint8_t* ring = smem_raw + warp * kRing * kChunkBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw + kBulkWarps * kRing * kChunkBytes) + warp * kRing;
  if (lane == 0) {
    for (int i = 0; i < kRing; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  griddep_wait();   // PDL-launched: the producer's rows and records are visible from here

  const int64_t nvec = a.cols / 8;
  const int64_t row_bytes = a.cols * 2;
  const int nchunks = (int)((nvec + kChunkVec - 1) / kChunkVec);
  const bool hold = !GIVEN && nchunks <= kRing;
  const int items_per_row = (GIVEN || hold) ? nchunks : 2 * nchunks;
  const bool smooth = a.sm.mode == MOE_SMOOTH_DIVIDE;
  int64_t r_lo, r_hi;
  cta_row_range(a, rows_per_cta, r_lo, r_hi);
  const uint64_t pol = policy_evict_first();

  // producer: the warp's item stream (row, chunk) in consumption order
  int64_t prow = r_lo + warp;
  int pitem = 0;
  uint32_t pcount = 0;
  int64_t prow_off = prow < r_hi ? row_view(a, prow).off : 0;
  auto produce = [&]() {
    if (prow >= r_hi) return;
    if (lane == 0) {
      const int chunk = pitem >= nchunks ? pitem - nchunks : pitem;   // items_per_row <= 2 * nchunks
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
        uint4 u[kLaneVec];
        float4 ta[kLaneVec], tb[kLaneVec];
#pragma unroll
        for (int b = 0; b < kLaneVec; ++b) {
          const bool ok = full || cb + 32 * b < nvec;
          u[b] = ok ? v[lane + 32 * b] : make_uint4(0u, 0u, 0u, 0u);
          const int64_t ct = ok ? cb + 32 * b : 0;
          ta[b] = __ldg(reinterpret_cast<const float4*>(tab) + 2 * ct);
          tb[b] = __ldg(reinterpret_cast<const float4*>(tab) + 2 * ct + 1);
        }
#pragma unroll
        for (int b = 0; b < kLaneVec; ++b) {
          if (!(full || cb + 32 * b < nvec)) continue;
          float xs[8];
          smooth8_pre(u[b], ta[b], tb[b], xs);
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
      p = affine_params_fast(mn, mx, bits, sym);
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
          for (int hf = 0; hf < kLaneVec; hf += kVecStep) {
            uint4 u[kVecStep];
            float4 ta[kVecStep], tb[kVecStep];
#pragma unroll
            for (int b = 0; b < kVecStep; ++b) {
              u[b] = v[lane + 32 * (hf + b)];
              ta[b] = __ldg(reinterpret_cast<const float4*>(tab) + 2 * (cb + 32 * (hf + b)));
              tb[b] = __ldg(reinterpret_cast<const float4*>(tab) + 2 * (cb + 32 * (hf + b)) + 1);
            }
            uint2 out[kVecStep];
            uint32_t slowm = 0;
#pragma unroll
            for (int b = 0; b < kVecStep; ++b) {
              float xs[8];
              smooth8_pre(u[b], ta[b], tb[b], xs);
              bool sl;
              out[b] = fast_core<G>(xs, f, sl);
              slowm |= (uint32_t)sl << b;
            }
#pragma unroll
            for (int b = 0; b < kVecStep; ++b) {
              sum += (slowm >> b & 1u) ? 0 : bytesum(out[b]);
              __stcs(dst + cb + 32 * (hf + b), out[b]);
            }
            if (slowm) {
              for (int b = 0; b < kVecStep; ++b) {
                if (!(slowm >> b & 1u)) continue;
                const int64_t c = cb + 32 * (hf + b);
                const uint4 sv = slow_vec8_packed(v[lane + 32 * (hf + b)], tab, c, srow, rrow, f);
                cnt += sv.z;
                const uint2 o2 = make_uint2(sv.x, sv.y);
                sum += bytesum(o2);
                __stcs(dst + c, o2);
              }
            }
          }
        } else {
#pragma unroll
          for (int b = 0; b < kLaneVec; ++b) {
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
      warp_sum2(sum, cnt);
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

// ── token-major variant for the MoE dispatch (K1 on x) ─────────────────────
// The MoE layer quantizes each token once per selected expert (top-k rows,
// each with its expert's smoothing). Row-major K1 over the permuted rows
// reads a token's x row k times from unrelated warps (expert-sorted order),
// so the second read usually misses L2 (measured: 222 MB of DRAM reads for
// 134 MB of x). Here one warp owns a token: its x row is loaded once into
// registers (NV 16-byte vectors per lane, rows up to 256 * NV bf16), and
// for each of the token's k rows (output row token_pos[t, j], smoothing
// group group[row]) the float32 extremes, the speculative exact extremes
// and the packed encode run from those registers. Per-row arithmetic and
// fallbacks are k1_row_warp's, so the codes are identical.
// (NV = 16 holds 64 registers of x per lane: 12 warps per CTA leave it 168
// registers, no spills; 16 warps capped it at 128 and spilled)
template <int NV>
constexpr int tok_warps() { return NV > 8 ? 12 : 16; }

template <int NV, bool GEN>
__device__ __forceinline__ int encode_regs(const uint4 (&u)[NV], const uint4* __restrict__ src,
                                           const float* __restrict__ tab, const double* srow, const double* rrow,
                                           int nvec, int lane, const FastRow& f, uint2* __restrict__ dst,
                                           uint32_t* cnt) {
  int sum = 0;
  uint32_t slow = 0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    if (c < nvec) {
      float xs[8];
      smooth8(u[i], tab, c, xs);
      bool sl;
      const uint2 out = fast_core<GEN>(xs, f, sl);
      if (!sl) {
        sum += bytesum(out);
        __stcs(dst + c, out);
      }
      slow |= (uint32_t)sl << i;
    }
  }
  while (slow) {   // rare: the generic float32 encode / exact redo, from the (L1-resident) row
    const int i = __ffs(slow) - 1;
    slow &= slow - 1;
    const int c = lane + 32 * i;
    const uint4 sv = slow_vec8(__ldg(src + c), tab, c, srow, rrow, f);
    *cnt += sv.z;
    const uint2 o2 = make_uint2(sv.x, sv.y);
    sum += bytesum(o2);
    __stcs(dst + c, o2);
  }
  return sum;
}

template <int NV>
__global__ void __launch_bounds__(tok_warps<NV>() * 32, 1)
    act_quant_token_kernel(RowArgs a, const int32_t* __restrict__ token_pos, int k, int64_t T,
                           const float* __restrict__ rs32_tab, int bits, int sym, uint8_t* codes, int64_t ldc,
                           double* scale, float* scale_f32, int32_t* zp, int32_t* rowsum) {
  constexpr int kTokWarps = tok_warps<NV>();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nvec = (int)(a.cols / 8);
  const uint32_t row_bytes = (uint32_t)(a.cols * 2);
  const int64_t warps = (int64_t)gridDim.x * kTokWarps;
  // the warp's next token row is prefetched into L2 (bulk prefetch, no
  // shared memory: L1 keeps the experts' float32 reciprocal tables)
#ifndef MOE_K1_TOK_PREFETCH
#define MOE_K1_TOK_PREFETCH 1
#endif
  auto prefetch = [&](int64_t tt) {
    if (MOE_K1_TOK_PREFETCH && lane == 0 && tt < T) bulk_prefetch_l2(static_cast<const __nv_bfloat16*>(a.x) + tt * a.ldx, row_bytes);
  };
  int64_t t = (int64_t)blockIdx.x * kTokWarps + warp;
  uint4 u[NV];
  auto load_row = [&](int64_t tt) {
    const uint4* s0 = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.x) + tt * a.ldx);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int c = lane + 32 * i;
      u[i] = c < nvec ? __ldg(s0 + c) : make_uint4(0u, 0u, 0u, 0u);
    }
  };
  // PDL-launched behind the permutation: x is older than the router (whose
  // completion the permutation kernel waited for before letting this grid
  // launch), so the first row streams in while the permutation finishes;
  // token_pos / group are read only after griddep_wait
  if (t < T) load_row(t);
  prefetch(t + warps);
  griddep_wait();
  griddep_launch_dependents();   // the next (PDL-launched) GEMM may start its weight prefetch
  for (; t < T; t += warps) {
    const __nv_bfloat16* row = static_cast<const __nv_bfloat16*>(a.x) + t * a.ldx;
    const uint4* src = reinterpret_cast<const uint4*>(row);
    if (t != (int64_t)blockIdx.x * kTokWarps + warp) {
      load_row(t);
      prefetch(t + warps);
    }
    for (int j = 0; j < k; ++j) {
      const int64_t r = token_pos[t * k + j];
      if (ep_row_dropped(a, r)) continue;
      const int64_t gbase = a.group ? (int64_t)a.group[r] * a.sm.cols : 0;
      const float* tab = rs32_tab + gbase;
      const double* srow = a.sm.s + gbase;
      const double* rrow = a.sm.rs + gbase;
      uint2* dst = reinterpret_cast<uint2*>(out_row_ptr(a, codes, ldc, r));
      // pass A from registers: float32 extremes and the vector holding them
      float tmax = -FLT_MAX, tmin = FLT_MAX;
      int vM = 0, vm = 0;
#pragma unroll
      for (int i = 0; i < NV; ++i) {
        const int c = lane + 32 * i;
        if (c < nvec) {
          float xs[8];
          smooth8(u[i], tab, c, xs);
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
        int e0 = 0;
#pragma unroll
        for (int e = 7; e >= 0; --e) e0 = xs[e] == val ? e : e0;
        return vc * 8 + e0;
      };
      const RowExt rec{tmax, tmin, locate(cM, tmax), locate(cm, tmin)};
      const bool exact_all = !(isfinite(rec.M) && isfinite(rec.m));
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
      if (spec) {
        p = affine_params_fast(mn, mx, bits, sym);
        FastRow f;
        const int mode = init_fast_row(f, p, rec.M, rec.m, mn, mx, bits, sym);
        if (mode) {
          uint32_t cnt = 0;
          sum = mode == 1 ? encode_regs<NV, false>(u, src, tab, srow, rrow, nvec, lane, f, dst, &cnt)
                          : encode_regs<NV, true>(u, src, tab, srow, rrow, nvec, lane, f, dst, &cnt);
          warp_sum2(sum, cnt);
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
  griddep_wait();                // PDL-launched: the previous kernel's outputs are visible from here
  griddep_launch_dependents();   // the next (PDL-launched) GEMM may start its weight prefetch
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t r = blockIdx.x;
  if ((a.rows_dev && r >= *a.rows_dev) || ep_row_dropped(a, r)) return;
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
      st.p = affine_params_fast(mn, mx, bits, sym);
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
    p = affine_params_fast(mn, mx, bits, sym);
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
  const cudaError_t e = launch_pdl(act_quant_bulk_kernel<GIVEN>, dim3((unsigned)nblk), dim3(kBulkWarps * 32),
                                   (size_t)kBulkSmem, s, a, rs32, ext, bits, sym, codes, ldc, scale, scale_f32, zp,
                                   rowsum, rows_per_cta);
  if (e != cudaSuccess) return e;
  count_launch();
  return cudaGetLastError();
}

// The fast kernels need bf16 rows and the smoothing tables (float64 s and
// RN(1/s), float32 RN32(1/s)); unsmoothed rows take the exact kernel (the
// host layer passes a table of ones to keep them on the fast path).
static bool eligible(const RowArgs& a, const float* rs32, uint8_t* codes, int64_t ldc) {
  return a.dt == MOE_DT_BF16 && a.cols % 8 == 0 && a.ldx % 8 == 0 && ldc % 8 == 0 &&
         (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 && (reinterpret_cast<uintptr_t>(codes) & 7) == 0 &&
         a.sm.mode == MOE_SMOOTH_DIVIDE && a.sm.s && a.sm.rs && rs32;
}

template <bool GIVEN, int WARPS, int MINB>
static void launch_cfg(const RowArgs& a, const float* rs32, const unsigned long long* ext, int bits, int sym,
                       uint8_t* codes, int64_t ldc, double* scale, float* scale_f32, int32_t* zp, int32_t* rowsum,
                       cudaStream_t s, int extra_per_sm = 2) {
  // contiguous row ranges, MINB + extra_per_sm CTAs per SM (extra 0: exactly one resident wave)
  const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>((a.rows + WARPS - 1) / WARPS,
                                                              (MINB + extra_per_sm) * (int64_t)num_sms()));
  int64_t rows_per_cta = (a.rows + ctas - 1) / ctas;
  if (a.order) rows_per_cta = (rows_per_cta + a.order_k - 1) / a.order_k * a.order_k;   // a token's rows in one CTA
  const int64_t nblk = (a.rows + rows_per_cta - 1) / rows_per_cta;
  launch_pdl(act_quant_warp_kernel<GIVEN, WARPS, MINB>, dim3((unsigned)nblk), dim3(WARPS * 32), 0, s, a, rs32, ext,
             bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, rows_per_cta);
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
    const cudaError_t e = launch_pdl(act_quant_cta_kernel<GIVEN>, dim3((unsigned)a.rows), dim3(kCtaThreads), 0, s, a,
                                     rs32, ext, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum);
    if (e != cudaSuccess) return e;
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

bool launch_act_quant_tokens(const RowArgs& a, const int32_t* token_pos, int k, int64_t T, const float* rs32,
                             int bits, int sym, uint8_t* codes, int64_t ldc, double* scale, float* scale_f32,
                             int32_t* zp, int32_t* rowsum, cudaStream_t s, cudaError_t* err) {
  if (!eligible(a, rs32, codes, ldc) || a.gather || k < 1) return false;
  const int mode = tune_value(MOE_TUNE_K1_TOKENS);
  if (mode != 1 || a.cols > 256 * 16) {
    // token-major walk of the row kernel: the k rows of a token go to
    // adjacent warps of one CTA at the same time (x read from HBM once, the
    // second read an L1/L2 hit), 32 warps per SM of 64 registers
    RowArgs b = a;
    b.order = token_pos;
    b.order_k = k;
    b.rows = T * k;
    // (16 warps x 2 CTAs per SM: 148 us; 32 x 1: 162 us, 8 x 4: 168 us; and
    // exactly one resident wave of 2 x 148 CTAs: 134 us, against 145 us for
    // two waves, 158 us for 1.5 and 190 us for one CTA per SM)
    launch_cfg<false, 16, 2>(b, rs32, nullptr, bits, sym, codes, ldc, scale, scale_f32, zp, rowsum, s, 0);
    count_launch();
    *err = cudaGetLastError();
    return true;
  }
  const int nvec32 = (int)((a.cols / 8 + 31) / 32);
  // one warp per token; one CTA per SM (grid-stride over the tokens)
  auto go = [&](auto kern, int warps) {
    const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>((T + warps - 1) / warps, (int64_t)num_sms()));
    *err = launch_pdl(kern, dim3((unsigned)ctas), dim3(warps * 32), 0, s, a, token_pos, k, T, rs32, bits, sym,
                      codes, ldc, scale, scale_f32, zp, rowsum);
  };
  if (nvec32 <= 4) go(act_quant_token_kernel<4>, tok_warps<4>());
  else if (nvec32 <= 8) go(act_quant_token_kernel<8>, tok_warps<8>());
  else go(act_quant_token_kernel<16>, tok_warps<16>());
  count_launch();
  if (*err == cudaSuccess) *err = cudaGetLastError();
  return true;
}

}  // namespace moe
