// K3 router gating, K4 token->expert permutation, K6 combine and the routing
// statistics feeding placement. None of these exist in the reference; they
// implement the MoE forward around its quantizer (SURVEY.md §8a a'1, a'2)
// and emit statistics in the reference's trace semantics (trace.py:207-225).
#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"

namespace moe {

constexpr int kMaxE = 64;
constexpr int kMaxK = 8;

// Select top-k of E logits: descending, ties to the lower id; softmax over
// the selected logits. Returns via idx/w arrays.
__device__ __forceinline__ void topk_select(const float* l, int E, int k, int32_t* idx, float* w) {
  uint64_t taken = 0;
  float sel[kMaxK];
  for (int j = 0; j < k; ++j) {
    int best = -1;
    float bv = 0.f;
    for (int e = 0; e < E; ++e) {
      if (taken >> e & 1ull) continue;
      if (best < 0 || l[e] > bv) {
        best = e;
        bv = l[e];
      }
    }
    taken |= 1ull << best;
    idx[j] = best;
    sel[j] = bv;
  }
  float den = 0.f;
  float ex[kMaxK];
  for (int j = 0; j < k; ++j) {
    ex[j] = expf(sel[j] - sel[0]);
    den += ex[j];
  }
  for (int j = 0; j < k; ++j) w[j] = ex[j] / den;
}

// One warp per token: logits[t, e] = x[t] . gate_w[e] in float32, lane-strided
// then butterfly-reduced (fixed order -> deterministic), then top-k.
template <int E_T>
__global__ void __launch_bounds__(256) router_gate_kernel(const void* x, int dt, int64_t T, int64_t d, int64_t ldx,
                                                          const float* __restrict__ gw, const float* gb, int E,
                                                          int k, float* logits, int32_t* idx, float* w) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= T) return;
  float acc[E_T];
#pragma unroll
  for (int e = 0; e < E_T; ++e) acc[e] = 0.f;
  const int64_t row = (int64_t)warp * ldx;
  const bool vec = dt == MOE_DT_BF16 && d % 256 == 0 && ldx % 8 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  if (vec) {
    const uint4* xp = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(x) + row);
    for (int64_t c = lane; c < d / 8; c += 32) {
      const uint4 u = xp[c];
      const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u);
      float xv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) xv[i] = __bfloat162float(h[i]);
#pragma unroll
      for (int e = 0; e < E_T; ++e) {
        if (e >= E) break;
        const float4* g = reinterpret_cast<const float4*>(gw + (int64_t)e * d + c * 8);
        const float4 g0 = __ldg(g), g1 = __ldg(g + 1);
        acc[e] = fmaf(xv[0], g0.x, acc[e]);
        acc[e] = fmaf(xv[1], g0.y, acc[e]);
        acc[e] = fmaf(xv[2], g0.z, acc[e]);
        acc[e] = fmaf(xv[3], g0.w, acc[e]);
        acc[e] = fmaf(xv[4], g1.x, acc[e]);
        acc[e] = fmaf(xv[5], g1.y, acc[e]);
        acc[e] = fmaf(xv[6], g1.z, acc[e]);
        acc[e] = fmaf(xv[7], g1.w, acc[e]);
      }
    }
  } else {
    for (int64_t j = lane; j < d; j += 32) {
      const float xv = (float)load_as_f64(x, row + j, dt);
#pragma unroll
      for (int e = 0; e < E_T; ++e)
        if (e < E) acc[e] = fmaf(xv, gw[(int64_t)e * d + j], acc[e]);
    }
  }
#pragma unroll
  for (int e = 0; e < E_T; ++e)
    for (int o = 16; o > 0; o >>= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
  if (lane == 0) {
    float l[E_T];
#pragma unroll
    for (int e = 0; e < E_T; ++e) l[e] = (gb && e < E) ? acc[e] + gb[e] : acc[e];
    if (logits)
      for (int e = 0; e < E; ++e) logits[(int64_t)warp * E + e] = l[e];
    topk_select(l, E, k, idx + (int64_t)warp * k, w + (int64_t)warp * k);
  }
}

// Persistent variant: the gate matrix (E x d float32) is staged once per CTA
// in shared memory, each warp then streams tokens (x read exactly once from
// HBM, weights from smem instead of E*d*4 bytes of L2 per token). Same
// per-lane accumulation order as router_gate_kernel.
template <int E_T>
__global__ void __launch_bounds__(512) router_gate_smem_kernel(const __nv_bfloat16* __restrict__ x, int64_t T,
                                                               int64_t d, int64_t ldx, const float* __restrict__ gw,
                                                               const float* gb, int E, int k, float* logits,
                                                               int32_t* idx, float* w) {
  extern __shared__ __align__(16) float sgw[];
  for (int64_t i = threadIdx.x; i < (int64_t)E * d / 4; i += blockDim.x)
    reinterpret_cast<float4*>(sgw)[i] = reinterpret_cast<const float4*>(gw)[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int64_t t = (int64_t)blockIdx.x * nw + (threadIdx.x >> 5); t < T; t += (int64_t)gridDim.x * nw) {
    float acc[E_T];
#pragma unroll
    for (int e = 0; e < E_T; ++e) acc[e] = 0.f;
    // 4 elements (8 B of x, one conflict-free float4 of each gate row) per
    // lane and step; 4 steps in flight
    const uint2* xp = reinterpret_cast<const uint2*>(x + t * ldx);
    const int64_t n4 = d / 4;
#pragma unroll 4
    for (int64_t c = lane; c < n4; c += 32) {
      const uint2 u = __ldcs(xp + c);
      const float xv[4] = {__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xFFFF0000u),
                           __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xFFFF0000u)};
#pragma unroll
      for (int e = 0; e < E_T; ++e) {
        if (e >= E) break;
        const float4 g = reinterpret_cast<const float4*>(sgw + (int64_t)e * d)[c];
        acc[e] = fmaf(xv[0], g.x, acc[e]);
        acc[e] = fmaf(xv[1], g.y, acc[e]);
        acc[e] = fmaf(xv[2], g.z, acc[e]);
        acc[e] = fmaf(xv[3], g.w, acc[e]);
      }
    }
#pragma unroll
    for (int e = 0; e < E_T; ++e)
      for (int o = 16; o > 0; o >>= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
    if (lane == 0) {
      float l[E_T];
#pragma unroll
      for (int e = 0; e < E_T; ++e) l[e] = (gb && e < E) ? acc[e] + gb[e] : acc[e];
      if (logits)
        for (int e = 0; e < E; ++e) logits[t * E + e] = l[e];
      topk_select(l, E, k, idx + t * k, w + t * k);
    }
  }
}

// Register-resident gate: warp w of the CTA owns columns [256w, 256w + 256),
// lane l the 8 columns 256w + 8l .. +8 of all E <= 8 gate rows (64 floats in
// registers, loaded once per CTA). The CTA streams batches of 4 tokens:
// each lane loads 16 B of x per token, forms 4 x 8 partial dot products, a
// transpose-reduce across the warp leaves lane l with entry l of the 32
// (token, expert) sums, and warp 0 adds the per-warp partials (fixed order
// -> deterministic) and runs top-k. x is read once from HBM; no shared-memory
// traffic for the weights.
constexpr int kRouterTB = 4;

__global__ void __launch_bounds__(512, 1)
    router_gate_reg_kernel(const __nv_bfloat16* __restrict__ x, int64_t T, int64_t d, int64_t ldx,
                           const float* __restrict__ gw,
                           const float* gb, int E, int k, float* logits, int32_t* idx, float* w) {
  __shared__ float part[2][16][32];   // [buffer][warp][lane] -> entry lane = token * 8 + expert
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int64_t col0 = (int64_t)warp * 256 + lane * 8;
  float g[8][8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    if (e < E) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(gw + (int64_t)e * d + col0));
      const float4 b = __ldg(reinterpret_cast<const float4*>(gw + (int64_t)e * d + col0) + 1);
      g[e][0] = a.x; g[e][1] = a.y; g[e][2] = a.z; g[e][3] = a.w;
      g[e][4] = b.x; g[e][5] = b.y; g[e][6] = b.z; g[e][7] = b.w;
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) g[e][c] = 0.f;
    }
  }
  int buf = 0;
  for (int64_t t0 = (int64_t)blockIdx.x * kRouterTB; t0 < T; t0 += (int64_t)gridDim.x * kRouterTB, buf ^= 1) {
    uint4 u[kRouterTB];
#pragma unroll
    for (int t = 0; t < kRouterTB; ++t)
      u[t] = t0 + t < T ? __ldcs(reinterpret_cast<const uint4*>(x + (t0 + t) * ldx + col0)) : make_uint4(0, 0, 0, 0);
    float v[32];
#pragma unroll
    for (int t = 0; t < kRouterTB; ++t) {
      const uint32_t wd[4] = {u[t].x, u[t].y, u[t].z, u[t].w};
      float xv[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        xv[2 * i] = __uint_as_float(wd[i] << 16);
        xv[2 * i + 1] = __uint_as_float(wd[i] & 0xFFFF0000u);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float acc = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) acc = fmaf(xv[c], g[e][c], acc);
        v[t * 8 + e] = acc;
      }
    }
    // transpose-reduce: after the step with xor offset o the lane keeps the
    // upper half when (lane & o); finally lane l holds entry l
#pragma unroll
    for (int o = 16, half = 16; o >= 1; o >>= 1, half >>= 1) {
      const bool up = lane & o;
#pragma unroll
      for (int i = 0; i < half; ++i) {
        const float send = up ? v[i] : v[i + half];
        const float keep = up ? v[i + half] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    part[buf][warp][lane] = v[0];
    __syncthreads();
    // warp t finishes token t0 + t: lanes 0..7 = experts (fixed-order
    // sum over the warps' partials), top-k by shuffle arg-max rounds
    for (int t = warp; t < kRouterTB; t += nw) {   // d < 1024: fewer than 4 warps
      const int e = lane & 7;
      float sum = 0.f;
      for (int ww = 0; ww < nw; ++ww) sum += part[buf][ww][t * 8 + e];
      if (gb && e < E) sum += gb[e];
      const int64_t tok = t0 + t;
      if (logits && tok < T && e < E && lane < 8) logits[tok * E + e] = sum;
      if (tok < T) {
        // lanes >= 8 and experts >= E never win
        float l = (lane < 8 && e < E) ? sum : -INFINITY;
        float sel[kMaxK];
        int id[kMaxK];
#pragma unroll
        for (int j = 0; j < kMaxK; ++j) {
          if (j >= k) break;
          float bv = l;
          int bi = lane;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {   // larger value wins, ties -> lower id
            const float v2 = __shfl_xor_sync(0xffffffffu, bv, o);
            const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
            if (v2 > bv || (v2 == bv && i2 < bi)) {
              bv = v2;
              bi = i2;
            }
          }
          sel[j] = bv;
          id[j] = bi;
          if (lane == bi) l = -INFINITY;
        }
        if (lane == 0) {
          float den = 0.f, ex[kMaxK];
#pragma unroll
          for (int j = 0; j < kMaxK; ++j) {
            if (j >= k) break;
            ex[j] = expf(sel[j] - sel[0]);
            den += ex[j];
          }
#pragma unroll
          for (int j = 0; j < kMaxK; ++j) {
            if (j >= k) break;
            idx[tok * k + j] = id[j];
            w[tok * k + j] = ex[j] / den;
          }
        }
      }
    }
  }
}

__global__ void router_topk_kernel(const float* logits, int64_t T, int E, int k, int32_t* idx, float* w) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    float l[kMaxE];
    for (int e = 0; e < E; ++e) l[e] = logits[t * E + e];
    topk_select(l, E, k, idx + t * k, w + t * k);
  }
}

// ── stable counting sort ───────────────────────────────────────────────────
constexpr int kPermThreads = 256;
constexpr int kPermSingle = 1024;  // up to this many (token, slot) pairs: one single-block launch
constexpr int kPermChunk = 256;    // pairs per block of the multi-block path (one pass per block)
constexpr int kPermScanBlocks = 512;  // above this many blocks: separate scan launch

__global__ void permute_count_kernel(const int32_t* idx, int64_t n, int E, int32_t* block_counts) {
  __shared__ int cnt[kMaxE];
  griddep_wait();                 // PDL: the router's selections are visible from here
  griddep_launch_dependents();    // the scatter (PDL) may get ready meanwhile
  for (int e = threadIdx.x; e < E; e += blockDim.x) cnt[e] = 0;
  __syncthreads();
  const int64_t lo = (int64_t)blockIdx.x * kPermChunk;
  const int64_t hi = min(n, lo + kPermChunk);
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&cnt[idx[i]], 1);
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) block_counts[(int64_t)blockIdx.x * E + e] = cnt[e];
}


// stable scatter of pairs [lo, hi) given each expert's first free row (run[])
__device__ __forceinline__ void permute_scatter_range(const int32_t* idx, const float* topk_w, int64_t lo, int64_t hi,
                                                      int k, int E, int* run, int (*wcnt)[kMaxE],
                                                      int32_t* src_token, int32_t* row_expert, float* row_weight,
                                                      int32_t* token_pos) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t base = lo; base < hi; base += kPermThreads) {
    for (int i = threadIdx.x; i < (kPermThreads / 32) * E; i += blockDim.x) wcnt[i / E][i % E] = 0;
    __syncthreads();
    const int64_t i = base + threadIdx.x;
    const bool valid = i < hi;
    const int e = valid ? idx[i] : -1;
    const unsigned same = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(same & ((1u << lane) - 1u));
    if (valid && rank == 0) wcnt[warp][e] = __popc(same);
    __syncthreads();
    if (valid) {
      int pos = run[e] + rank;
      for (int w2 = 0; w2 < warp; ++w2) pos += wcnt[w2][e];
      src_token[pos] = (int32_t)(i / k);
      row_expert[pos] = e;
      if (row_weight) row_weight[pos] = topk_w[i];
      token_pos[i] = pos;
    }
    __syncthreads();
    for (int ee = threadIdx.x; ee < E; ee += blockDim.x) {
      int s = 0;
      for (int w2 = 0; w2 < kPermThreads / 32; ++w2) s += wcnt[w2][ee];
      run[ee] += s;
    }
    __syncthreads();
  }
}

// Large batches: one block per expert turns the per-block counts into
// exclusive per-block bases (bases[b * E + e]) and the expert total
// (bases[nblocks * E + e]), so the scatter blocks read O(E) values each
// instead of re-reading the whole nblocks x E table.
__global__ void __launch_bounds__(kPermThreads) permute_scan_kernel(const int32_t* block_counts, int nblocks, int E,
                                                                    int32_t* bases) {
  __shared__ int wsum[kPermThreads / 32];
  __shared__ int carry;
  const int e = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nblocks; b0 += kPermThreads) {
    const int b = b0 + threadIdx.x;
    const int c = b < nblocks ? block_counts[(int64_t)b * E + e] : 0;
    int v = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) wsum[warp] = v;
    __syncthreads();
    int before = carry;
    for (int w2 = 0; w2 < warp; ++w2) before += wsum[w2];
    if (b < nblocks) bases[(int64_t)b * E + e] = before + v - c;
    __syncthreads();
    if (threadIdx.x == kPermThreads - 1) carry = before + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) bases[(int64_t)nblocks * E + e] = carry;
}

// Every block derives its own bases: from the scanned table when `bases` is
// given, else from the per-block counts (nblocks x E ints, fine for small
// nblocks): expert offset = sum of earlier experts' totals, plus the counts
// of earlier blocks; block 0 also writes the offsets.
__global__ void __launch_bounds__(kPermThreads) permute_scatter_kernel(const int32_t* idx, const float* topk_w,
                                                                       int64_t n, int k, int E,
                                                                       const int32_t* block_counts, int nblocks,
                                                                       const int32_t* bases,
                                                                       int32_t* offsets, int32_t* src_token,
                                                                       int32_t* row_expert, float* row_weight,
                                                                       int32_t* token_pos) {
  __shared__ int run[kMaxE];
  __shared__ int tot[kMaxE];
  __shared__ int wcnt[kPermThreads / 32][kMaxE];
  griddep_wait();                 // PDL: the counts (and bases) are visible from here
  griddep_launch_dependents();    // K1 on x (PDL) may get ready meanwhile
  if (bases) {
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
      tot[e] = bases[(int64_t)nblocks * E + e];
      run[e] = bases[(int64_t)blockIdx.x * E + e];
    }
  } else {   // one warp per expert sums its column of the counts table
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int e = warp; e < E; e += kPermThreads / 32) {
      int t = 0, before = 0;
      for (int b = lane; b < nblocks; b += 32) {
        const int c = block_counts[(int64_t)b * E + e];
        t += c;
        if (b < (int)blockIdx.x) before += c;
      }
      t = (int)__reduce_add_sync(0xffffffffu, (unsigned)t);
      before = (int)__reduce_add_sync(0xffffffffu, (unsigned)before);
      if (lane == 0) {
        tot[e] = t;
        run[e] = before;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int e = 0; e < E; ++e) {
      run[e] += s;
      if (blockIdx.x == 0) offsets[e] = s;
      s += tot[e];
    }
    if (blockIdx.x == 0) offsets[E] = s;
  }
  __syncthreads();
  const int64_t lo = (int64_t)blockIdx.x * kPermChunk;
  permute_scatter_range(idx, topk_w, lo, min(n, lo + kPermChunk), k, E, run, wcnt, src_token, row_expert, row_weight,
                        token_pos);
}

// Batches of at most kPermChunk pairs (decode sizes): count, scan and
// scatter in one block — one launch instead of three, same permutation.
__global__ void __launch_bounds__(kPermThreads) permute_single_kernel(const int32_t* idx, const float* topk_w,
                                                                      int64_t n, int k, int E, int32_t* offsets,
                                                                      int32_t* src_token, int32_t* row_expert,
                                                                      float* row_weight, int32_t* token_pos) {
  __shared__ int run[kMaxE];
  __shared__ int wcnt[kPermThreads / 32][kMaxE];
  griddep_wait();                 // PDL: the router's selections are visible from here
  griddep_launch_dependents();
  for (int e = threadIdx.x; e < E; e += blockDim.x) run[e] = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&run[idx[i]], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int e = 0; e < E; ++e) {
      const int c = run[e];
      offsets[e] = s;
      run[e] = s;
      s += c;
    }
    offsets[E] = s;
  }
  __syncthreads();
  permute_scatter_range(idx, topk_w, 0, n, k, E, run, wcnt, src_token, row_expert, row_weight, token_pos);
}

// ── combine ────────────────────────────────────────────────────────────────
template <typename TIn, typename TOut>
__global__ void combine_kernel(const TIn* y, const int32_t* token_pos, int64_t T, int k, int64_t d, TOut* out,
                               int64_t ldo) {
  const int64_t t = blockIdx.x;
  for (int64_t c = threadIdx.x; c < d; c += blockDim.x) {
    float s = 0.f;
    for (int j = 0; j < k; ++j) {
      const int64_t r = token_pos[t * k + j];
      if constexpr (sizeof(TIn) == 2) s += __bfloat162float(y[r * d + c]);
      else s += y[r * d + c];
    }
    if constexpr (sizeof(TOut) == 2) out[t * ldo + c] = __float2bfloat16_rn(s);
    else out[t * ldo + c] = s;
  }
}

// vectorised bf16 -> bf16 / f32 -> f32 paths (8 / 4 elements per thread step)
__global__ void combine_bf16_vec_kernel(const __nv_bfloat16* y, const int32_t* token_pos, int k, int64_t d,
                                        __nv_bfloat16* out, int64_t ldo) {
  const int64_t t = blockIdx.x;
  int32_t rows[kMaxK];
  for (int j = 0; j < k; ++j) rows[j] = token_pos[t * k + j];
  for (int64_t c = threadIdx.x; c < d / 8; c += blockDim.x) {
    float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = 0; j < k; ++j) {
      const uint4 u = reinterpret_cast<const uint4*>(y + (int64_t)rows[j] * d)[c];
      const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
      for (int e = 0; e < 8; ++e) s[e] += __bfloat162float(h[e]);
    }
    uint4 o;
    __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int e = 0; e < 4; ++e) p[e] = __floats2bfloat162_rn(s[2 * e], s[2 * e + 1]);
    reinterpret_cast<uint4*>(out + t * ldo)[c] = o;
  }
}

// Residual + RMSNorm of the MoE stack (pre-norm blocks, SURVEY.md C5 token
// path): s = bf16(x + y) (y optional), norm = bf16(s * rsqrt(mean(s^2) + eps))
// in float32, one CTA per token row, each thread 8-element vectors. The sum of
// squares is reduced in a fixed order, so the norm of a row depends on that
// row alone.
__global__ void __launch_bounds__(256) rmsnorm_residual_kernel(const __nv_bfloat16* x, const __nv_bfloat16* y,
                                                               __nv_bfloat16* x_out, __nv_bfloat16* n_out,
                                                               int64_t d, float eps) {
  __shared__ float red[8];
  const int64_t t = blockIdx.x;
  const int nv = (int)(d / 8);
  constexpr int kMaxV = 4;   // d <= 256 * 8 * 4 = 8192
  float v[kMaxV][8];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxV; ++i) {
    const int c = threadIdx.x + i * 256;
    if (c >= nv) break;
    const uint4 ux = reinterpret_cast<const uint4*>(x + t * d)[c];
    const __nv_bfloat16* hx = reinterpret_cast<const __nv_bfloat16*>(&ux);
    uint4 uy = make_uint4(0u, 0u, 0u, 0u);
    if (y) uy = reinterpret_cast<const uint4*>(y + t * d)[c];
    const __nv_bfloat16* hy = reinterpret_cast<const __nv_bfloat16*>(&uy);
    uint4 os;
    __nv_bfloat16* ho = reinterpret_cast<__nv_bfloat16*>(&os);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float sv = y ? __bfloat162float(__float2bfloat16_rn(__bfloat162float(hx[e]) + __bfloat162float(hy[e])))
                         : __bfloat162float(hx[e]);
      ho[e] = __float2bfloat16_rn(sv);
      v[i][e] = sv;
      ss = fmaf(sv, sv, ss);
    }
    if (y && x_out) reinterpret_cast<uint4*>(x_out + t * d)[c] = os;
  }
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < 8; ++w) tot += red[w];
  const float r = rsqrtf(tot / (float)d + eps);
  if (!n_out) return;
#pragma unroll
  for (int i = 0; i < kMaxV; ++i) {
    const int c = threadIdx.x + i * 256;
    if (c >= nv) break;
    uint4 on;
    __nv_bfloat162* hn = reinterpret_cast<__nv_bfloat162*>(&on);
#pragma unroll
    for (int e = 0; e < 4; ++e) hn[e] = __floats2bfloat162_rn(v[i][2 * e] * r, v[i][2 * e + 1] * r);
    reinterpret_cast<uint4*>(n_out + t * d)[c] = on;
  }
}

__global__ void histogram_kernel(const int32_t* idx, int64_t T, int k, int E, int layer, int64_t* counts,
                                 int32_t* path_codes) {
  __shared__ unsigned long long cnt[kMaxE];
  for (int e = threadIdx.x; e < E; e += blockDim.x) cnt[e] = 0;
  __syncthreads();
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    uint32_t mask = 0;
    for (int j = 0; j < k; ++j) {
      const int e = idx[t * k + j];
      atomicAdd(&cnt[e], 1ull);
      mask |= 1u << e;
    }
    if (path_codes) path_codes[t] = (int32_t)mask;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(&counts[(int64_t)layer * E + e]), cnt[e]);
}

}  // namespace moe

using namespace moe;

extern "C" moe_status moe_router_gate(const void* x, int x_dtype, int64_t T, int64_t d, int64_t ldx, const float* gate_w,
                                      const float* gate_bias, int E, int k, float* logits, int32_t* topk_idx, float* topk_w, moe_stream_t stream) {
  MOE_REQUIRE(x && gate_w && topk_idx && topk_w, "router_gate: null pointer");
  MOE_REQUIRE(T >= 1 && d >= 1, "router_gate: empty input");
  MOE_REQUIRE(ldx >= d, "router_gate: row stride below d");
  MOE_REQUIRE(E >= 1 && E <= 32 && k >= 1 && k <= kMaxK && k <= E, "router_gate: need 1 <= k <= E <= 32");
  const int64_t threads = T * 32;
  const unsigned blocks = (unsigned)((threads + 255) / 256);
  cudaStream_t s = as_stream(stream);
  const int64_t gw_bytes = (int64_t)E * d * 4;
  if (x_dtype == MOE_DT_BF16 && d % 256 == 0 && d <= 4096 && E <= 8 && ldx % 8 == 0 &&
      (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(gate_w) & 15) == 0) {
    const int64_t grid = std::min<int64_t>((T + kRouterTB - 1) / kRouterTB, num_sms());
    router_gate_reg_kernel<<<(unsigned)grid, (unsigned)(d / 256 * 32), 0, s>>>(
        static_cast<const __nv_bfloat16*>(x), T, d, ldx, gate_w, gate_bias, E, k, logits, topk_idx, topk_w);
    ::moe::count_launch();
  } else if (x_dtype == MOE_DT_BF16 && d % 8 == 0 && ldx % 4 == 0 && E <= 8 && gw_bytes <= 200 * 1024 &&
      (reinterpret_cast<uintptr_t>(x) & 15) == 0 && (reinterpret_cast<uintptr_t>(gate_w) & 15) == 0) {
    MOE_CUDA_TRY(set_max_smem_once(reinterpret_cast<const void*>(router_gate_smem_kernel<8>), 200 * 1024));
    const int64_t grid = std::min<int64_t>((T + 15) / 16, num_sms());
    router_gate_smem_kernel<8><<<(unsigned)grid, 512, (size_t)gw_bytes, s>>>(
        static_cast<const __nv_bfloat16*>(x), T, d, ldx, gate_w, gate_bias, E, k, logits, topk_idx, topk_w);
    ::moe::count_launch();
  } else if (E <= 8) {
    router_gate_kernel<8><<<blocks, 256, 0, s>>>(x, x_dtype, T, d, ldx, gate_w, gate_bias, E, k, logits, topk_idx, topk_w); ::moe::count_launch();
  } else if (E <= 16) {
    router_gate_kernel<16><<<blocks, 256, 0, s>>>(x, x_dtype, T, d, ldx, gate_w, gate_bias, E, k, logits, topk_idx, topk_w); ::moe::count_launch();
  } else {
    router_gate_kernel<32><<<blocks, 256, 0, s>>>(x, x_dtype, T, d, ldx, gate_w, gate_bias, E, k, logits, topk_idx, topk_w); ::moe::count_launch();
  }
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_router_topk(const float* logits, int64_t T, int E, int k, int32_t* topk_idx,
                                      float* topk_w, moe_stream_t stream) {
  MOE_REQUIRE(logits && topk_idx && topk_w && T >= 1, "router_topk: bad arguments");
  MOE_REQUIRE(E >= 1 && E <= kMaxE && k >= 1 && k <= kMaxK && k <= E, "router_topk: need 1 <= k <= E <= 64");
  const unsigned blocks = (unsigned)((T + 255) / 256);
  router_topk_kernel<<<blocks, 256, 0, as_stream(stream)>>>(logits, T, E, k, topk_idx, topk_w); ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" int64_t moe_route_permute_workspace(int64_t T, int k, int E) {
  const int64_t nb = (T * k + kPermChunk - 1) / kPermChunk;
  return (2 * nb + 1) * E * (int64_t)sizeof(int32_t);
}

extern "C" moe_status moe_route_permute(const int32_t* topk_idx, const float* topk_w, int64_t T, int k, int E,
                                        int32_t* expert_offsets, int32_t* src_token, int32_t* row_expert,
                                        float* row_weight, int32_t* token_pos, void* workspace,
                                        int64_t workspace_bytes, moe_stream_t stream) {
  MOE_REQUIRE(topk_idx && expert_offsets && src_token && row_expert && token_pos, "route_permute: null pointer");
  MOE_REQUIRE(!row_weight || topk_w, "route_permute: row_weight needs topk_w");
  MOE_REQUIRE(T >= 1 && k >= 1 && E >= 1 && E <= kMaxE, "route_permute: bad sizes");
  MOE_REQUIRE(workspace && workspace_bytes >= moe_route_permute_workspace(T, k, E), "route_permute: workspace");
  const int64_t n = T * k;
  const int nb = (int)((n + kPermChunk - 1) / kPermChunk);
  int32_t* counts = static_cast<int32_t*>(workspace);
  cudaStream_t s = as_stream(stream);
  if (n <= kPermSingle) {
    MOE_CUDA_TRY(launch_pdl(permute_single_kernel, dim3(1), dim3(kPermThreads), 0, s, topk_idx, topk_w, n, k, E,
                            expert_offsets, src_token, row_expert, row_weight, token_pos));
    ::moe::count_launch();
    MOE_LAUNCH_CHECK();
    return MOE_OK;
  }
  MOE_CUDA_TRY(launch_pdl(permute_count_kernel, dim3(nb), dim3(kPermThreads), 0, s, topk_idx, n, E, counts));
  ::moe::count_launch();
  // beyond kPermScanBlocks blocks the per-block rescan (O(nb^2 E) reads) would
  // dominate: scan once in a separate launch
  int32_t* bases = nullptr;
  if (nb > kPermScanBlocks) {
    bases = counts + (int64_t)nb * E;
    permute_scan_kernel<<<E, kPermThreads, 0, s>>>(counts, nb, E, bases); ::moe::count_launch();
  }
  MOE_CUDA_TRY(launch_pdl(permute_scatter_kernel, dim3(nb), dim3(kPermThreads), 0, s, topk_idx, topk_w, n, k, E,
                          (const int32_t*)counts, nb, (const int32_t*)bases, expert_offsets, src_token, row_expert,
                          row_weight, token_pos));
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_combine(const void* y, int y_dtype, const int32_t* token_pos, int64_t T, int k, int64_t d,
                                  void* out, int out_dtype, int64_t ldo, moe_stream_t stream) {
  MOE_REQUIRE(y && token_pos && out && T >= 1 && d >= 1 && k >= 1 && k <= kMaxK, "combine: bad arguments");
  MOE_REQUIRE(ldo >= d, "combine: out row stride below d");
  MOE_REQUIRE((y_dtype == MOE_DT_F32 || y_dtype == MOE_DT_BF16) && (out_dtype == MOE_DT_F32 || out_dtype == MOE_DT_BF16),
              "combine: dtypes f32|bf16");
  cudaStream_t s = as_stream(stream);
  const unsigned threads = 256;
  if (y_dtype == MOE_DT_BF16 && out_dtype == MOE_DT_BF16 && d % 8 == 0 && ldo % 8 == 0 &&
      (reinterpret_cast<uintptr_t>(y) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    combine_bf16_vec_kernel<<<(unsigned)T, threads, 0, s>>>(static_cast<const __nv_bfloat16*>(y), token_pos, k, d,
                                                            static_cast<__nv_bfloat16*>(out), ldo);
  } else if (y_dtype == MOE_DT_F32 && out_dtype == MOE_DT_F32) {
    combine_kernel<float, float><<<(unsigned)T, threads, 0, s>>>(static_cast<const float*>(y), token_pos, T, k, d,
                                                                 static_cast<float*>(out), ldo);
  } else if (y_dtype == MOE_DT_F32) {
    combine_kernel<float, __nv_bfloat16><<<(unsigned)T, threads, 0, s>>>(
        static_cast<const float*>(y), token_pos, T, k, d, static_cast<__nv_bfloat16*>(out), ldo);
  } else if (out_dtype == MOE_DT_F32) {
    combine_kernel<__nv_bfloat16, float><<<(unsigned)T, threads, 0, s>>>(
        static_cast<const __nv_bfloat16*>(y), token_pos, T, k, d, static_cast<float*>(out), ldo);
  } else {
    combine_kernel<__nv_bfloat16, __nv_bfloat16><<<(unsigned)T, threads, 0, s>>>(
        static_cast<const __nv_bfloat16*>(y), token_pos, T, k, d, static_cast<__nv_bfloat16*>(out), ldo);
  }
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_expert_histogram(const int32_t* topk_idx, int64_t T, int k, int E, int layer,
                                           int64_t* counts, int32_t* path_codes, moe_stream_t stream) {
  MOE_REQUIRE(topk_idx && counts && T >= 1 && k >= 1 && E >= 1 && E <= 31 && layer >= 0,
              "expert_histogram: bad arguments");
  int64_t blocks = (T + 255) / 256;
  if (blocks > num_sms() * 4) blocks = num_sms() * 4;
  histogram_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(topk_idx, T, k, E, layer, counts, path_codes); ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_rmsnorm_residual(const void* x, const void* y, void* x_out, void* norm_out, int64_t T,
                                           int64_t d, float eps, moe_stream_t stream) {
  MOE_REQUIRE(x && T >= 1 && d >= 8 && d % 8 == 0 && d <= 8192, "rmsnorm_residual: bf16 rows, d % 8 == 0, d <= 8192");
  MOE_REQUIRE(norm_out || (y && x_out), "rmsnorm_residual: nothing to write");
  MOE_REQUIRE(((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(x_out) |
                reinterpret_cast<uintptr_t>(norm_out)) & 15) == 0,
              "rmsnorm_residual: 16-byte aligned rows");
  rmsnorm_residual_kernel<<<(unsigned)T, 256, 0, as_stream(stream)>>>(
      static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(y), static_cast<__nv_bfloat16*>(x_out),
      static_cast<__nv_bfloat16*>(norm_out), d, eps);
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}
