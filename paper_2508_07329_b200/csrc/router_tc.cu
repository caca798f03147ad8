// K3 router on the tensor cores: logits[T, E] = x[T, d] . Wg[E, d]^T with
// tcgen05.mma kind::f16 (bf16 x bf16 -> f32 in TMEM), top-k + softmax in the
// epilogue. The gate stays float32-accurate: it is split once into three
// bf16 pieces (hi + mid + lo hold all 24 significand bits), every product
// x * piece is exact in the f32 accumulator; the pieces sit side by side in
// one N = 48 MMA and are summed in the epilogue. x (bf16) is read once from
// HBM by TMA, so the kernel is HBM-bound instead of FMA/shared-memory bound
// (the gate is tiny: E <= 16 rows padded to N = 16).
//
// Split K over a thread-block cluster: a 128-token tile is computed by S
// CTAs (S <= 8, fixed by d alone), each accumulating a contiguous range of
// 64-column K blocks in its own TMEM. The partial sums meet in distributed
// shared memory and are added in rank order, each rank reducing and
// ranking its share of the tile's tokens. A decode-size batch (one tile)
// thus streams the gate and x over S SMs instead of one, and the result for
// a token does not depend on the batch it came in.
//
// CTA: warp 0 lane 0 = TMA producer, warp 1 lane 0 = MMA issuer, warps 0-3
// drain TMEM (one lane quarter each) into the shared-memory partial.
#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"

#include <cudaTypedefs.h>

namespace moe {

constexpr int kRtM = 128;                 // tokens per tile
constexpr int kRtN = 16;                  // experts padded to the UMMA N
constexpr int kRtPieces = 3;              // bf16 pieces of the float32 gate
constexpr int kRtCols = kRtPieces * kRtN;  // 48 accumulator columns
constexpr int kRtBK = 64;                 // bf16 elements per stage = one 128-byte swizzle atom row
constexpr int kRtStages = 4;
constexpr int kRtMaxSplit = 8;            // portable cluster size
constexpr int kRtA = kRtM * kRtBK * 2;                      // 16 KB
constexpr int kRtB = kRtCols * kRtBK * 2;                   // 6 KB
constexpr int kRtStage = kRtA + kRtB;
constexpr int kRtBarOff = kRtStages * kRtStage;
constexpr int kRtSmem = kRtBarOff + (2 * kRtStages + 1) * 8 + 16 + 1024;
// after the MMAs: partial [48][128] f32 and the reduced share [48][128] reuse the stage buffers
constexpr int kRtPartOff = 0;
constexpr int kRtRedOff = kRtCols * kRtM * 4;
static_assert(kRtRedOff + kRtCols * kRtM * 4 <= kRtBarOff, "router partials must fit the stage buffers");

// kind::f16 instruction descriptor: f32 D, bf16 A and B, both K-major
__host__ __device__ constexpr uint32_t idesc_bf16(uint32_t M, uint32_t N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((M >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// gate [E, d] f32 -> pieces [3 * 16, d] bf16 (rows >= E zero): hi, mid, lo
__global__ void router_split_gate_kernel(const float* gw, int E, int64_t d, __nv_bfloat16* pieces) {
  const int64_t n = (int64_t)kRtN * d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int e = (int)(i / d);
    const int64_t c = i - (int64_t)e * d;
    const float g = e < E ? gw[(int64_t)e * d + c] : 0.f;
    const __nv_bfloat16 hi = __float2bfloat16_rn(g);
    const float r1 = g - __bfloat162float(hi);                 // exact
    const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
    const float r2 = r1 - __bfloat162float(mid);               // exact
    pieces[i] = hi;
    pieces[n + i] = mid;
    pieces[2 * n + i] = __float2bfloat16_rn(r2);
  }
}

// K split of a d-wide row: S ranks of kpc K blocks each (no empty rank)
struct RtSplit {
  int S, kpc;
};
static inline RtSplit rt_split(int64_t d) {
  const int kblocks = (int)(d / kRtBK);
  const int s0 = std::min(kRtMaxSplit, kblocks);
  const int kpc = (kblocks + s0 - 1) / s0;
  return RtSplit{(kblocks + kpc - 1) / kpc, kpc};
}

// logits of one token -> top-k ids (descending, ties to the lower id) and
// softmax weights over the selected
__device__ __forceinline__ void rt_finish(const float (&l)[kRtN], int64_t tok, int E, int k, float* logits,
                                          int32_t* idx, float* w) {
  if (logits) {
#pragma unroll
    for (int e = 0; e < kRtN; ++e)
      if (e < E) logits[tok * E + e] = l[e];
  }
  uint32_t taken = 0;
  float sel[8], ex[8], den = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j >= k) break;
    int best = -1;
    float bv = 0.f;
#pragma unroll
    for (int e = 0; e < kRtN; ++e) {
      if (e >= E || (taken >> e & 1u)) continue;
      if (best < 0 || l[e] > bv) {
        best = e;
        bv = l[e];
      }
    }
    taken |= 1u << best;
    idx[tok * k + j] = best;
    sel[j] = bv;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j >= k) break;
    ex[j] = expf(sel[j] - sel[0]);
    den += ex[j];
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j >= k) break;
    w[tok * k + j] = ex[j] / den;
  }
}

__global__ void __launch_bounds__(128, 1)
    router_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmG, int64_t T,
                     int64_t d, int kpc, const float* __restrict__ gb, int E, int k, float* logits, int32_t* idx,
                     float* w) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRtBarOff);
  uint64_t* empty = full + kRtStages;
  uint64_t* done = empty + kRtStages;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  griddep_launch_dependents();   // the permutation kernel (PDL) may get ready meanwhile
  const uint32_t rank = cluster_ctarank(), nrank = cluster_nctarank();
  const int64_t row0 = (int64_t)(blockIdx.x / nrank) * kRtM;
  const int kblocks = (int)(d / kRtBK);
  const int kb0 = (int)rank * kpc, kb1 = min(kblocks, kb0 + kpc);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kRtStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmG);
  }
  if (warp == 0) {
    tmem_alloc(tmem_ptr, 64);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;
  if (warp == 0 && lane == 0) {
    // producer: x tile 128 x 64 and the three gate pieces 48 x 64 per stage
    const uint64_t pol_x = policy_evict_first(), pol_g = policy_evict_last();
    for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
      const int s = i % kRtStages;
      mbar_wait(&empty[s], ((i / kRtStages) & 1) ^ 1);
      uint8_t* sa = smem + s * kRtStage;
      mbar_expect_tx(&full[s], kRtStage);
      tma_load_2d(sa, &tmX, &full[s], kb * kRtBK, (int32_t)row0, pol_x);
      tma_load_2d(sa + kRtA, &tmG, &full[s], kb * kRtBK, 0, pol_g);
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer: 4 K-steps of 16 per stage, the three gate pieces side by side (N = 48)
    constexpr uint32_t idesc = idesc_bf16(kRtM, kRtCols);
    for (int kb = kb0, i = 0; kb < kb1; ++kb, ++i) {
      const int s = i % kRtStages;
      mbar_wait(&full[s], (i / kRtStages) & 1);
      tc_fence_after();
      const uint32_t a_addr = smem_u32(smem + s * kRtStage);
      const uint64_t adesc = sdesc_sw128(a_addr), bdesc = sdesc_sw128(a_addr + kRtA);
      // one N = 48 MMA per K step: TMEM columns [16p, 16p + 16) accumulate piece p
#pragma unroll
      for (int kk = 0; kk < kRtBK / 16; ++kk)
        umma_f16(tmem, adesc + (uint64_t)(kk * 2), bdesc + (uint64_t)(kk * 2), idesc, (i | kk) != 0);
      umma_commit(&empty[s]);
    }
    umma_commit(done);
  }
  __syncwarp();
  // this rank's partial sums: thread = token row, 48 f32 from TMEM -> smem [48][128]
  mbar_wait(done, 0);
  tc_fence_after();
  uint32_t v[kRtPieces][16];
#pragma unroll
  for (int p = 0; p < kRtPieces; ++p) tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + p * kRtN, v[p]);
  tmem_ld_wait();
  float* part = reinterpret_cast<float*>(smem + kRtPartOff);
#pragma unroll
  for (int p = 0; p < kRtPieces; ++p)
#pragma unroll
    for (int e = 0; e < 16; ++e) part[(p * kRtN + e) * kRtM + threadIdx.x] = __uint_as_float(v[p][e]);
  cluster_sync_all();   // every rank's partial written (release / acquire at cluster scope)

  // this rank reduces tokens [r0, r0 + nrows) of the tile over the ranks, in rank order
  const int rpr = (kRtM + (int)nrank - 1) / (int)nrank;
  const int r0 = (int)rank * rpr, nrows = max(0, min(kRtM, r0 + rpr) - r0);
  float* red = reinterpret_cast<float*>(smem + kRtRedOff);
  const uint32_t part_addr = smem_u32(part);
  for (int e = threadIdx.x; e < nrows * kRtCols; e += 128) {
    const int c = e / nrows, rr = e - c * nrows;
    const uint32_t off = (uint32_t)((c * kRtM + r0 + rr) * 4);
    float acc = ld_dsmem_f32(mapa_shared(part_addr + off, 0));
    for (uint32_t s = 1; s < nrank; ++s) acc += ld_dsmem_f32(mapa_shared(part_addr + off, s));
    red[c * kRtM + rr] = acc;
  }
  __syncthreads();
  const int64_t tok = row0 + r0 + threadIdx.x;
  if ((int)threadIdx.x < nrows && tok < T) {
    float l[kRtN];
#pragma unroll
    for (int e = 0; e < kRtN; ++e)
      l[e] = (red[e * kRtM + threadIdx.x] + red[(kRtN + e) * kRtM + threadIdx.x]) +
             red[(2 * kRtN + e) * kRtM + threadIdx.x] + ((gb && e < E) ? gb[e] : 0.f);
    rt_finish(l, tok, E, k, logits, idx, w);
  }
  tc_fence_before();
  cluster_sync_all();   // the peers are done reading this CTA's partial
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
  }
}

// Large batches: one persistent CTA per SM walks whole tiles; the S K ranges
// of a tile accumulate into S separate TMEM accumulators (S * 48 <= 384
// columns) that the epilogue adds in rank order — the same MMA sequence and
// the same additions as the cluster split, hence the same logits.
constexpr int kRtMultiStages = 6;
constexpr int kRtMultiBarOff = kRtMultiStages * kRtStage;
constexpr int kRtMultiSmem = kRtMultiBarOff + (2 * kRtMultiStages + 1) * 8 + 16 + 1024;

__global__ void __launch_bounds__(128, 1)
    router_tc_multi_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmG,
                           int64_t T, int64_t d, int S, int kpc, const float* __restrict__ gb, int E, int k,
                           float* logits, int32_t* idx, float* w) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRtMultiBarOff);
  uint64_t* empty = full + kRtMultiStages;
  uint64_t* done = empty + kRtMultiStages;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kblocks = (int)(d / kRtBK);
  const int64_t tiles = (T + kRtM - 1) / kRtM;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kRtMultiStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmG);
  }
  if (warp == 0) {
    tmem_alloc(tmem_ptr, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_ptr;
  uint32_t pit = 0, cit = 0, tile_no = 0;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++tile_no) {
    const int32_t row0 = (int32_t)(tile * kRtM);
    if (warp == 0 && lane == 0) {
      const uint64_t pol_x = policy_evict_first(), pol_g = policy_evict_last();
      for (int kb = 0; kb < kblocks; ++kb, ++pit) {
        const int s = pit % kRtMultiStages;
        mbar_wait(&empty[s], ((pit / kRtMultiStages) & 1) ^ 1);
        uint8_t* sa = smem + s * kRtStage;
        mbar_expect_tx(&full[s], kRtStage);
        tma_load_2d(sa, &tmX, &full[s], kb * kRtBK, row0, pol_x);
        tma_load_2d(sa + kRtA, &tmG, &full[s], kb * kRtBK, 0, pol_g);
      }
    } else if (warp == 1 && lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(kRtM, kRtCols);
      for (int kb = 0; kb < kblocks; ++kb, ++cit) {
        const int s = cit % kRtMultiStages;
        mbar_wait(&full[s], (cit / kRtMultiStages) & 1);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(smem + s * kRtStage);
        const uint64_t adesc = sdesc_sw128(a_addr), bdesc = sdesc_sw128(a_addr + kRtA);
        const uint32_t dt = tmem + (uint32_t)((kb / kpc) * kRtCols);   // accumulator of this K range
        const bool first = kb % kpc == 0;
#pragma unroll
        for (int kk = 0; kk < kRtBK / 16; ++kk)
          umma_f16(dt, adesc + (uint64_t)(kk * 2), bdesc + (uint64_t)(kk * 2), idesc, !(first && kk == 0));
        umma_commit(&empty[s]);
      }
      umma_commit(done);
    }
    __syncwarp();
    mbar_wait(done, tile_no & 1);
    tc_fence_after();
    float acc[kRtCols];
    for (int r = 0; r < S; ++r) {   // rank order, as the cluster reduction
      uint32_t v[kRtPieces][16];
#pragma unroll
      for (int p = 0; p < kRtPieces; ++p)
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(r * kRtCols + p * kRtN), v[p]);
      tmem_ld_wait();
#pragma unroll
      for (int p = 0; p < kRtPieces; ++p)
#pragma unroll
        for (int e = 0; e < 16; ++e)
          acc[p * kRtN + e] = r == 0 ? __uint_as_float(v[p][e]) : acc[p * kRtN + e] + __uint_as_float(v[p][e]);
    }
    tc_fence_before();
    __syncthreads();   // TMEM may be overwritten by the next tile's MMAs only after every warp read it
    const int64_t tok = (int64_t)row0 + threadIdx.x;
    if (tok < T) {
      float l[kRtN];
#pragma unroll
      for (int e = 0; e < kRtN; ++e)
        l[e] = (acc[e] + acc[kRtN + e]) + acc[2 * kRtN + e] + ((gb && e < E) ? gb[e] : 0.f);
      rt_finish(l, tok, E, k, logits, idx, w);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 rt_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

static bool rt_map(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld_bytes,
                   uint32_t box_rows) {
  auto enc = rt_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld_bytes};
  cuuint32_t box[2] = {(cuuint32_t)kRtBK, box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace moe

using namespace moe;

extern "C" int64_t moe_router_tc_workspace(int64_t d) { return (int64_t)kRtPieces * kRtN * d * 2; }

extern "C" moe_status moe_router_prepare(const float* gate_w, int E, int64_t d, void* pieces, moe_stream_t stream) {
  MOE_REQUIRE(gate_w && pieces && E >= 1 && E <= kRtN && d >= 1, "router_prepare: need 1 <= E <= 16");
  const int64_t n = (int64_t)kRtN * d;
  const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 4 * (int64_t)num_sms());
  router_split_gate_kernel<<<blocks, 256, 0, as_stream(stream)>>>(gate_w, E, d,
                                                                  static_cast<__nv_bfloat16*>(pieces));
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_router_gate_tc(const void* x, int64_t T, int64_t d, int64_t ldx, const void* pieces,
                                         const float* gate_bias, int E, int k, float* logits, int32_t* topk_idx,
                                         float* topk_w, moe_stream_t stream) {
  MOE_REQUIRE(x && pieces && topk_idx && topk_w && T >= 1, "router_gate_tc: null pointer / empty input");
  MOE_REQUIRE(E >= 1 && E <= kRtN && k >= 1 && k <= 8 && k <= E, "router_gate_tc: need 1 <= k <= E <= 16, k <= 8");
  MOE_REQUIRE(d % kRtBK == 0 && ldx >= d && (ldx * 2) % 16 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0,
              "router_gate_tc: d % 64 == 0 and 16-byte aligned rows");
  CUtensorMap tx, tg;
  if (!rt_map(&tx, x, (uint64_t)T, (uint64_t)d, (uint64_t)ldx * 2, kRtM) ||
      !rt_map(&tg, pieces, (uint64_t)kRtPieces * kRtN, (uint64_t)d, (uint64_t)d * 2, kRtPieces * kRtN)) {
    set_error("router_gate_tc: cuTensorMapEncodeTiled failed");
    return MOE_ECUDA;
  }
  const RtSplit sp = rt_split(d);
  const int64_t tiles = (T + kRtM - 1) / kRtM;
  if (tiles > router_cluster_tiles()) {
    MOE_CUDA_TRY(set_max_smem_once(reinterpret_cast<const void*>(router_tc_multi_kernel), kRtMultiSmem));
    const unsigned grid = (unsigned)std::min<int64_t>(tiles, num_sms());
    router_tc_multi_kernel<<<grid, 128, kRtMultiSmem, as_stream(stream)>>>(tx, tg, T, d, sp.S, sp.kpc, gate_bias,
                                                                           E, k, logits, topk_idx, topk_w);
  } else {
    MOE_CUDA_TRY(set_max_smem_once(reinterpret_cast<const void*>(router_tc_kernel), kRtSmem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)(tiles * sp.S));
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = kRtSmem;
    cfg.stream = as_stream(stream);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)sp.S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    MOE_CUDA_TRY(cudaLaunchKernelEx(&cfg, router_tc_kernel, tx, tg, T, d, sp.kpc, gate_bias, E, k, logits,
                                    topk_idx, topk_w));
  }
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}
