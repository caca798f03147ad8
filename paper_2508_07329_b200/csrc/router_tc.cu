// K3 router on the tensor cores: logits[T, E] = x[T, d] . Wg[E, d]^T with
// tcgen05.mma kind::f16 (bf16 x bf16 -> f32 in TMEM), top-k + softmax in the
// epilogue. The gate stays float32-accurate: it is split once into three
// bf16 pieces (hi + mid + lo hold all 24 significand bits), every product
// x * piece is exact in the f32 accumulator; the pieces sit side by side in
// one N = 48 MMA and are summed in the epilogue. x (bf16) is read once from HBM by TMA, so the
// kernel is HBM-bound instead of FMA/shared-memory bound (the gate is tiny:
// E <= 16 rows padded to N = 16).
//
// CTA = 128 tokens (UMMA M = 128), warp 0 lane 0 = TMA producer, warp 1
// lane 0 = MMA issuer, warps 0-3 = epilogue (one TMEM lane quarter each).
#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"

#include <cudaTypedefs.h>

namespace moe {

constexpr int kRtM = 128;                 // tokens per tile
constexpr int kRtN = 16;                  // experts padded to the UMMA N
constexpr int kRtPieces = 3;              // bf16 pieces of the float32 gate
constexpr int kRtBK = 64;                 // bf16 elements per stage = one 128-byte swizzle atom row
constexpr int kRtStages = 6;
constexpr int kRtA = kRtM * kRtBK * 2;                      // 16 KB
constexpr int kRtB = kRtPieces * kRtN * kRtBK * 2;          // 6 KB
constexpr int kRtStage = kRtA + kRtB;
constexpr int kRtBarOff = kRtStages * kRtStage;
constexpr int kRtSmem = kRtBarOff + (2 * kRtStages + 1) * 8 + 16 + 1024;

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

__global__ void __launch_bounds__(128, 1)
    router_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmG, int64_t T,
                     int64_t d, const float* __restrict__ gb, int E, int k, float* logits, int32_t* idx, float* w) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kRtBarOff);
  uint64_t* empty = full + kRtStages;
  uint64_t* done = empty + kRtStages;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kblocks = (int)((d + kRtBK - 1) / kRtBK);
  const int64_t tiles = (T + kRtM - 1) / kRtM;

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
  uint32_t pit = 0, cit = 0, tile_no = 0;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++tile_no) {
    const int32_t row0 = (int32_t)(tile * kRtM);
    if (warp == 0 && lane == 0) {
      // producer: x tile 128 x 64 and the three gate pieces 48 x 64 per stage
      const uint64_t pol_x = policy_evict_first(), pol_g = policy_evict_last();
      for (int kb = 0; kb < kblocks; ++kb, ++pit) {
        const int s = pit % kRtStages;
        mbar_wait(&empty[s], ((pit / kRtStages) & 1) ^ 1);
        uint8_t* sa = smem + s * kRtStage;
        mbar_expect_tx(&full[s], kRtStage);
        tma_load_2d(sa, &tmX, &full[s], kb * kRtBK, row0, pol_x);
        tma_load_2d(sa + kRtA, &tmG, &full[s], kb * kRtBK, 0, pol_g);
      }
    } else if (warp == 1 && lane == 0) {
      // MMA issuer: 4 K-steps of 16 per stage, the three gate pieces side by side (N = 48)
      constexpr uint32_t idesc = idesc_bf16(kRtM, kRtPieces * kRtN);
      for (int kb = 0; kb < kblocks; ++kb, ++cit) {
        const int s = cit % kRtStages;
        mbar_wait(&full[s], (cit / kRtStages) & 1);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(smem + s * kRtStage);
        const uint64_t adesc = sdesc_sw128(a_addr), bdesc = sdesc_sw128(a_addr + kRtA);
        // one N = 48 MMA per K step: TMEM columns [16p, 16p + 16) accumulate piece p
#pragma unroll
        for (int kk = 0; kk < kRtBK / 16; ++kk)
          umma_f16(tmem, adesc + (uint64_t)(kk * 2), bdesc + (uint64_t)(kk * 2), idesc, (kb | kk) != 0);
        umma_commit(&empty[s]);
      }
      umma_commit(done);
    }
    __syncwarp();
    // epilogue: thread = token row, 16 f32 logits from TMEM
    mbar_wait(done, tile_no & 1);
    tc_fence_after();
    uint32_t v[kRtPieces][16];
#pragma unroll
    for (int p = 0; p < kRtPieces; ++p) tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + p * kRtN, v[p]);
    tmem_ld_wait();
    tc_fence_before();
    __syncthreads();   // TMEM may be overwritten by the next tile's MMAs only after every warp read it
    const int64_t tok = (int64_t)row0 + threadIdx.x;
    if (tok < T) {
      float l[kRtN];
#pragma unroll
      for (int e = 0; e < kRtN; ++e)
        l[e] = (__uint_as_float(v[0][e]) + __uint_as_float(v[1][e])) + __uint_as_float(v[2][e]) +
               ((gb && e < E) ? gb[e] : 0.f);
      if (logits) {
#pragma unroll
        for (int e = 0; e < kRtN; ++e)
          if (e < E) logits[tok * E + e] = l[e];
      }
      // top-k: descending, ties to the lower id; softmax over the selected
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
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 64);
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
  MOE_CUDA_TRY(set_max_smem_once(reinterpret_cast<const void*>(router_tc_kernel), kRtSmem));
  const int64_t tiles = (T + kRtM - 1) / kRtM;
  const unsigned grid = (unsigned)std::min<int64_t>(tiles, num_sms());
  router_tc_kernel<<<grid, 128, kRtSmem, as_stream(stream)>>>(tx, tg, T, d, gate_bias, E, k, logits, topk_idx,
                                                              topk_w);
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}
