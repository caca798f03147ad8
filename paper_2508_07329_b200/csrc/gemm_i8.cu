// K2 / K5 — W8A8 GEMM on the 5th-generation tensor cores (tcgen05 kind::i8).
//
// Y[m, n] = epilogue( sum_k (a[m,k]-za[m]) * (w[n,k]-zw[n]) ), A [M, K] u8
// activation codes (tokens-major), W [G*N, K] u8 weight codes (per expert
// stacked), both K-major. Replaces the float64 fake-quant product of
// quant_loss / quantize_layer (quant.py:281-283, 475-478) with the exact
// integer product; the zero points are applied in the epilogue:
//   acc = sum a*w  - zw*rowsum_a - za*(rowsum_w - K*zw)    (wrapping int32,
//   exact because the true value satisfies |acc| <= K*255^2 < 2^31).
//
// Structure (persistent, warp-specialised, 384 threads per CTA):
//   warp 0 lane 0 : TMA producer — A tile 128 x 128 B, W tile (256/CG) x 128 B
//                   per stage, 128-byte swizzle, mbarrier complete_tx
//   warp 1 lane 0 : UMMA issuer — tcgen05.mma.kind::i8, N=256 K=32, int32
//                   accumulators in TMEM (2 x 256 columns, double-buffered)
//   warp 2        : TMEM allocator
//   warps 4..11   : epilogue — tcgen05.ld 32x32b, zero-point correction,
//                   dequant / SwiGLU / raw int32, global stores
// CG = 2 (the MoE hot path): a CTA pair on one TPC computes a 256 x 256 tile
// with tcgen05.mma.cta_group::2 issued by the leader; each CTA stages its own
// 128 A rows and half of the W tile, so per-SM shared-memory traffic per MMA
// drops from 12 KB to 8 KB and the W tile crosses L2 once per pair.
// Grouped mode (MoE): the tile scheduler walks experts from the device-side
// offsets, so routing never syncs with the host.
#include <algorithm>

#include "k1_fast.cuh"
#include "ptx.cuh"

#include <cudaTypedefs.h>

namespace moe {

constexpr int kBM = 128;           // rows per CTA (UMMA M per CTA)
constexpr int kBK = 128;           // bytes of K per stage = one SW128 atom row
constexpr int kUmmaK = 32;         // K per tcgen05.mma for 8-bit inputs
constexpr int kMaxGroups = 64;
#ifndef MOE_GEMM_EPI_WARPS
#define MOE_GEMM_EPI_WARPS 8
#endif
constexpr int kEpiWarps = MOE_GEMM_EPI_WARPS;         // epilogue warps: kEpiWarps / 4 per TMEM lane quarter
constexpr int kParts = kEpiWarps / 4;                  // column parts of a tile per lane quarter
constexpr int kGemmThreads = 128 + 32 * kEpiWarps;     // 4 control warps + the epilogue warps

struct GemmArgs {
  int M, N, K, G;
  int Kc;  // K of the zero-point correction term (0 when w_rowsum is pre-corrected)
  const int32_t* offsets;
  const float* a_scale;
  const int32_t* a_zp;
  const int32_t* a_rowsum;
  const float* w_scale;
  const int32_t* w_zp;
  const int32_t* w_rowsum;
  const float* bias;
  const float* row_weight;
  void* out;
  int64_t ldo;
  int32_t* acc_out;
  int64_t ld_acc;
  int vec_ok;      // output pointer / ldo allow 16-byte vector stores
  int acc_vec_ok;  // acc_out / ld_acc and the W zp / rowsum tables allow 16-byte vectors
  int param_vec_ok;  // W zp / rowsum / scale tables allow 16-byte vector loads
  int tma_out;              // bf16 output stored through smem + TMA (tensor map tmO)
  int band;                 // m-tiles per raster band (map_tile)
  int pf_kb;                // k blocks of the first weight tile to prefetch into L2 before griddep_wait
  int serp;                 // alternate the k direction tile by tile (exact int32 sums: order-free)
  int l2pol;                // L2 eviction priority of the A (bits 0-1) and W (bits 2-3) tile loads:
                            // 0 evict_last, 1 evict_normal, 2 evict_first
  void* const* out_tab;     // DEQUANT: row m goes to out_tab[out_rank[m]] + out_row[m] * ldo (EP combine)
  const int32_t* out_rank;
  const int32_t* out_row;
  // optional (SwiGLU): float32 per-row bounds of stored output * RN32(1/s_next)
  const float* ns_rs32;
  int64_t ns_ld;
  unsigned long long* row_ext;  // [M, 2] (min, max) records
  // fused K1 of the A operand (DEQUANT): the epilogue warps quantize A's
  // rows (K1 with producer records) while they wait for accumulators; the
  // TMA producer loads an A block once its 32-row blocks are complete
  int fq;
  RowArgs qa;                   // bf16 source rows of A, row -> smoothing group
  const float* q_rs32;
  const unsigned long long* q_ext;
  uint8_t* q_codes;             // = A
  int64_t q_ldc;
  double* q_scale;
  int* q_next;                  // next row to quantize
  int* q_blk;                   // completed rows per 32-row block
  // fused top-2 combine (DEQUANT, bf16): the second of a token's two rows
  // to finish a 32-column chunk adds the first's stored values and writes
  // the token's output row
  const int32_t* comb_src;      // row -> token
  const int32_t* comb_pos;      // [T, 2] token -> its two rows
  int* comb_cnt;                // [T, N / 32] chunk arrival counters (zeroed)
  int comb_chunks;
  __nv_bfloat16* comb_out;      // [T, comb_ldo]
  int64_t comb_ldo;
};

template <int BN, int STAGES, int CG, bool EPIBUF = true>
struct Smem {
  static constexpr int kA = kBM * kBK;
  static constexpr int kB = (BN / CG) * kBK;
  static constexpr int kStage = kA + kB;
  static constexpr int kBarOff = STAGES * kStage;
  static constexpr int kNumBars = 2 * STAGES + 4;
  static constexpr int kTmemPtrOff = kBarOff + kNumBars * 8;
  static constexpr int kTableOff = kTmemPtrOff + 16;                  // tile_start[G+1], off[G+1]
  static constexpr int kOutOff = (kTableOff + 2 * (kMaxGroups + 1) * 4 + 127) / 128 * 128;
  static constexpr int kOutBytes = EPIBUF ? kEpiWarps * 2 * 1024 : 0;  // per epilogue warp 2 x (32 rows x 32 B)
  // SwiGLU: per-tile W column parameters (zw, t = rowsum - Kc*zw, ws) and the
  // next layer's f32 reciprocal smoothing, staged by the epilogue warps while
  // they wait for the tile's accumulators (double-buffered)
  static constexpr int kParamBuf = EPIBUF ? BN * 12 + (BN / 2) * 4 : 0;   // (SwiGLU only)
  static constexpr int kParamOff = kOutOff + kOutBytes;
  static constexpr int kBytes = kParamOff + 2 * kParamBuf + 1024;     // + alignment slack
};

struct TileInfo {
  int g, m0, m_end, n0;
};

// tile t -> (group, first row, group end, first column). Within a group the
// m-tiles are walked in bands of `band` tiles: for each band every N block,
// m fastest inside the band. A band's activations (band * TM * K bytes) stay
// L2-resident while the weight blocks stream past them; the host sizes the
// band so that this fits (whole group when K is small, e.g. W13 at K=4096;
// 8 tiles for W2 at K=14336, where the full 59 MB group slice thrashed L2).
__device__ __forceinline__ TileInfo map_tile(int t, int G, const int* tile_start, const int* off, int TM, int BN,
                                             int n_tiles, int band) {
  int g = 0;
  while (g + 1 < G && t >= tile_start[g + 1]) ++g;
  const int local = t - tile_start[g];
  const int mt = (off[g + 1] - off[g] + TM - 1) / TM;
  const int bs = band < mt ? band : mt;
  const int full = mt / bs;                       // complete bands
  int m_tile, n_tile;
  if (local < full * bs * n_tiles) {
    const int b = local / (bs * n_tiles), w = local - b * bs * n_tiles;
    n_tile = w / bs;
    m_tile = b * bs + (w - n_tile * bs);
  } else {                                        // trailing partial band
    const int rm = mt - full * bs, w = local - full * bs * n_tiles;
    n_tile = w / rm;
    m_tile = full * bs + (w - n_tile * rm);
  }
  return TileInfo{g, off[g] + m_tile * TM, off[g + 1], n_tile * BN};
}

// Debug variant (-DMOE_GEMM_PROFILE=1, tools/gemm_waits.py): the MMA
// issuer and the producer accumulate the cycles they spend waiting on each
// barrier into a __device__ table (per CTA: [mma_tempty, mma_full,
// prod_empty, total]); off by default.
#ifndef MOE_GEMM_PROFILE
#define MOE_GEMM_PROFILE 0
#endif
#if MOE_GEMM_PROFILE
__device__ unsigned long long g_gemm_waits[1024][6];
#define MOE_PROF_T0() const long long _t0 = clock64()
#define MOE_PROF_ADD(slot) atomicAdd(&g_gemm_waits[blockIdx.x][slot], (unsigned long long)(clock64() - _t0))
#else
#define MOE_PROF_T0()
#define MOE_PROF_ADD(slot)
#endif

__device__ __forceinline__ uint64_t l2_policy(int which) {
  uint64_t pol;
  if (which == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  else if (which == 1) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  else asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ float silu_f(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

template <bool BF16>
__device__ __forceinline__ void store32(void* out, int64_t idx, const float (&v)[32], int nvalid, bool vec) {
  if (BF16) {
    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(out) + idx;
    if (vec && nvalid == 32) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u;
        __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) p[e] = __floats2bfloat162_rn(v[q * 8 + 2 * e], v[q * 8 + 2 * e + 1]);
        reinterpret_cast<uint4*>(o)[q] = u;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) o[j] = __float2bfloat16_rn(v[j]);
    }
  } else {
    float* o = static_cast<float*>(out) + idx;
    if (vec && nvalid == 32) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        reinterpret_cast<float4*>(o)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) o[j] = v[j];
    }
  }
}

// ── per-row float32 extreme records of stored output * RN32(1/s_next) ─────
// Feeds the next K1 (act_quant row_ext): the same float32 products K1 forms,
// reduced per thread to (value, 32-column chunk) of the max and of the min
// and merged per row with one 64-bit atomic each per tile: (order-preserving
// key << 32) | first column of the chunk. K1 locates the element in the
// chunk, divides the two extremes exactly and verifies during its single
// encode pass that no other element could be an extreme.
struct ExtRec {
  float M, m;
  int cM, cm;
};

__device__ __forceinline__ float fmax3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float fmin3f(float a, float b, float c) {
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// max / min of the 32 products of one chunk; the record keeps the chunk's
// first column (K1 locates the element inside the chunk with one warp ballot)
__device__ __forceinline__ void chunk_ext(const float (&hv)[32], const float* __restrict__ t32, int col0,
                                          ExtRec& r) {
  const float4* t = reinterpret_cast<const float4*>(t32);
  float xs[32];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const float4 tt = __ldg(t + q);
    const float2 a = __fmul2_rn(make_float2(hv[4 * q], hv[4 * q + 1]), make_float2(tt.x, tt.y));
    const float2 b = __fmul2_rn(make_float2(hv[4 * q + 2], hv[4 * q + 3]), make_float2(tt.z, tt.w));
    xs[4 * q] = a.x;
    xs[4 * q + 1] = a.y;
    xs[4 * q + 2] = b.x;
    xs[4 * q + 3] = b.y;
  }
  float M = xs[0], m = xs[0];
#pragma unroll
  for (int j = 1; j < 31; j += 2) {
    M = fmax3f(M, xs[j], xs[j + 1]);
    m = fmin3f(m, xs[j], xs[j + 1]);
  }
  M = fmaxf(M, xs[31]);
  m = fminf(m, xs[31]);
  if (M > r.M) {
    r.M = M;
    r.cM = col0;
  }
  if (m < r.m) {
    r.m = m;
    r.cm = col0;
  }
}

__device__ __forceinline__ unsigned long long ext_key(float v, int col) {
  const int i = __float_as_int(v);
  const uint32_t k = (uint32_t)(i >= 0 ? i : (i ^ 0x7FFFFFFF)) ^ 0x80000000u;  // unsigned float order
  return ((unsigned long long)k << 32) | (uint32_t)col;
}

__global__ void rowext_init_kernel(unsigned long long* re, int64_t M) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
    re[2 * i] = ~0ull;     // min record
    re[2 * i + 1] = 0ull;  // max record
  }
}

// zero-point corrected exact accumulator (wrapping int32 arithmetic)
__device__ __forceinline__ int32_t zp_correct(uint32_t acc, int32_t zw, int32_t rsw, int32_t za, int32_t rsa,
                                              int32_t K) {
  const uint32_t t = (uint32_t)rsw - (uint32_t)K * (uint32_t)zw;
  return (int32_t)(acc - (uint32_t)zw * (uint32_t)rsa - (uint32_t)za * t);
}

// Per-column W parameters of 32 consecutive columns starting at n (16-byte
// loads; all lanes of a warp read the same addresses -> L1 broadcast).
struct ColParams32 {
  int32_t zw[32], rsw[32];   // rsw: rowsum, or t = rowsum - K*zp when loaded by load_cols32_t
  float ws[32];
};
__device__ __forceinline__ void load_cols32(const GemmArgs& p, int n, ColParams32& c) {
  const int4* z = reinterpret_cast<const int4*>(p.w_zp + n);
  const int4* r = reinterpret_cast<const int4*>(p.w_rowsum + n);
  const float4* w = reinterpret_cast<const float4*>(p.w_scale + n);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int4 zz = __ldg(z + q), rr = __ldg(r + q);
    const float4 ww = __ldg(w + q);
    c.zw[4 * q] = zz.x; c.zw[4 * q + 1] = zz.y; c.zw[4 * q + 2] = zz.z; c.zw[4 * q + 3] = zz.w;
    c.rsw[4 * q] = rr.x; c.rsw[4 * q + 1] = rr.y; c.rsw[4 * q + 2] = rr.z; c.rsw[4 * q + 3] = rr.w;
    c.ws[4 * q] = ww.x; c.ws[4 * q + 1] = ww.y; c.ws[4 * q + 2] = ww.z; c.ws[4 * q + 3] = ww.w;
  }
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// SwiGLU epilogue hot path (vectorisable W tables, no bias): this thread's
// row, `half` of the tile's h columns, in 16-column sub-chunks with the next
// sub-chunk's TMEM loads in flight while the current one is computed.
// Zero-point correction in 2 IMADs per accumulator (row terms pre-negated,
// column term t = rowsum - Kc*zp), packed f32x2 math, silu through
// ex2/rcp.approx (what __expf / __fdividef compile to in range).
template <int BN, bool BF16>
__device__ __forceinline__ void swiglu_fast(const GemmArgs& p, const TileInfo& ti, int row, uint32_t tbase, int half,
                                            ExtRec& ext, bool rvalid, float sa, float rw, int32_t za, int32_t rsa,
                                            const CUtensorMap* tmO, uint8_t* obuf, uint32_t& ob,
                                            const uint8_t* pbuf) {
  constexpr int kSub = 16;
  constexpr int kNSubAll = BN / 2 / kSub;          // sub-chunks of a tile row (BN/2 h columns)
  constexpr int kIters = (kNSubAll + kParts - 1) / kParts;
  const int wbase = ti.g * p.N;
  const uint32_t nrsa = 0u - (uint32_t)rsa, nza = 0u - (uint32_t)za;
  const float2 sa2 = make_float2(sa, sa), srw2 = make_float2(sa * rw, sa * rw);
  const float2 nl2 = make_float2(-1.4426950408889634f, -1.4426950408889634f), one2 = make_float2(1.f, 1.f);
  // this tile's staged column parameters (shared memory)
  const int32_t* zw_s = reinterpret_cast<const int32_t*>(pbuf);
  const int32_t* t_s = zw_s + BN;
  const float* ws_s = reinterpret_cast<const float*>(t_s + BN);
  const float* ns_s = ws_s + BN;
  // whole-warp TMA store of the 32 x 16 h block when all 32 rows are in the group
  const bool tma = BF16 && p.tma_out && __all_sync(0xffffffffu, rvalid);
  const int lane = threadIdx.x & 31;
  uint32_t ag[2][kSub], au[2][kSub];
  tmem_ld16(tbase + half * kSub, ag[0]);
  tmem_ld16(tbase + BN / 2 + half * kSub, au[0]);
  tmem_ld_wait();
#pragma unroll
  for (int it = 0; it < kIters; ++it) {
    const int sc = half + it * kParts;             // this thread's sub-chunks: part, part + kParts, ...
    if (sc >= kNSubAll) break;
    const int cur = it & 1;
    const int hc = sc * kSub;                      // tile-relative h column of this sub-chunk
    if (sc + kParts < kNSubAll) {
      tmem_ld16(tbase + hc + kParts * kSub, ag[cur ^ 1]);
      tmem_ld16(tbase + BN / 2 + hc + kParts * kSub, au[cur ^ 1]);
    }
    const int4* gz = reinterpret_cast<const int4*>(zw_s + hc);
    const int4* gr = reinterpret_cast<const int4*>(t_s + hc);
    const float4* gs = reinterpret_cast<const float4*>(ws_s + hc);
    const int4* uz = reinterpret_cast<const int4*>(zw_s + BN / 2 + hc);
    const int4* ur = reinterpret_cast<const int4*>(t_s + BN / 2 + hc);
    const float4* us = reinterpret_cast<const float4*>(ws_s + BN / 2 + hc);
    uint32_t hb[kSub / 2];                         // packed bf16 pairs (BF16) 
    float h[kSub];
#pragma unroll
    for (int q = 0; q < kSub / 4; ++q) {
      const int4 z4g = gz[q], r4g = gr[q], z4u = uz[q], r4u = ur[q];
      const float4 s4g = gs[q], s4u = us[q];
      const int32_t zg[4] = {z4g.x, z4g.y, z4g.z, z4g.w}, rg[4] = {r4g.x, r4g.y, r4g.z, r4g.w};
      const int32_t zu[4] = {z4u.x, z4u.y, z4u.z, z4u.w}, ru[4] = {r4u.x, r4u.y, r4u.z, r4u.w};
      const float sg4[4] = {s4g.x, s4g.y, s4g.z, s4g.w}, su4[4] = {s4u.x, s4u.y, s4u.z, s4u.w};
#pragma unroll
      for (int e2 = 0; e2 < 4; e2 += 2) {
        const int j = 4 * q + e2;
        int32_t ai[4];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          ai[e] = (int32_t)(ag[cur][j + e] + (uint32_t)zg[e2 + e] * nrsa + (uint32_t)rg[e2 + e] * nza);
          ai[2 + e] = (int32_t)(au[cur][j + e] + (uint32_t)zu[e2 + e] * nrsa + (uint32_t)ru[e2 + e] * nza);
        }
        const float2 g = __fmul2_rn(make_float2((float)ai[0], (float)ai[1]),
                                    __fmul2_rn(sa2, make_float2(sg4[e2], sg4[e2 + 1])));
        const float2 u = __fmul2_rn(make_float2((float)ai[2], (float)ai[3]),
                                    __fmul2_rn(srw2, make_float2(su4[e2], su4[e2 + 1])));
        const float2 t = __fmul2_rn(g, nl2);
        const float2 den = __fadd2_rn(make_float2(ex2_approx(t.x), ex2_approx(t.y)), one2);
        const float2 sgv = __fmul2_rn(g, make_float2(rcp_approx(den.x), rcp_approx(den.y)));
        const float2 hv = __fmul2_rn(sgv, u);
        if (BF16) {   // the stored value, which K1 will read
          const __nv_bfloat162 b = __floats2bfloat162_rn(hv.x, hv.y);
          hb[j / 2] = *reinterpret_cast<const uint32_t*>(&b);
          h[j] = __low2float(b);
          h[j + 1] = __high2float(b);
        } else {
          h[j] = hv.x;
          h[j + 1] = hv.y;
        }
      }
    }
    if (tma) {
      uint8_t* buf = obuf + (ob & 1u) * 1024;
      if (lane == 0) bulk_wait_group_read<1>();   // the store that used this buffer has read it
      __syncwarp();
      uint4* d = reinterpret_cast<uint4*>(buf + lane * 32);
      d[0] = make_uint4(hb[0], hb[1], hb[2], hb[3]);
      d[1] = make_uint4(hb[4], hb[5], hb[6], hb[7]);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(tmO, buf, ti.n0 / 2 + hc, row);   // lane 0 holds the warp's first row
        bulk_commit_group();
      }
      ++ob;
    }
    if (!tma && rvalid) {
      const int64_t o = (int64_t)row * p.ldo + ti.n0 / 2 + hc;
      if (BF16 && p.vec_ok) {
        uint4* d = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(p.out) + o);
        d[0] = make_uint4(hb[0], hb[1], hb[2], hb[3]);
        d[1] = make_uint4(hb[4], hb[5], hb[6], hb[7]);
      } else if (BF16) {
        __nv_bfloat16* d = static_cast<__nv_bfloat16*>(p.out) + o;
#pragma unroll
        for (int j = 0; j < kSub; ++j) d[j] = __float2bfloat16_rn(h[j]);
      } else {
        float* d = static_cast<float*>(p.out) + o;
#pragma unroll
        for (int j = 0; j < kSub; ++j) d[j] = h[j];
      }
    }
    if (rvalid) {
      if (p.row_ext) {
        const float4* t4 = reinterpret_cast<const float4*>(ns_s + hc);
        float xs[kSub];
#pragma unroll
        for (int q = 0; q < kSub / 4; ++q) {
          const float4 tt = t4[q];
          const float2 a = __fmul2_rn(make_float2(h[4 * q], h[4 * q + 1]), make_float2(tt.x, tt.y));
          const float2 b = __fmul2_rn(make_float2(h[4 * q + 2], h[4 * q + 3]), make_float2(tt.z, tt.w));
          xs[4 * q] = a.x;
          xs[4 * q + 1] = a.y;
          xs[4 * q + 2] = b.x;
          xs[4 * q + 3] = b.y;
        }
        float M = xs[0], m = xs[0];
#pragma unroll
        for (int j = 1; j < kSub - 1; j += 2) {
          M = fmax3f(M, xs[j], xs[j + 1]);
          m = fmin3f(m, xs[j], xs[j + 1]);
        }
        M = fmaxf(M, xs[kSub - 1]);
        m = fminf(m, xs[kSub - 1]);
        // records carry a 32-column window start: [col, col + 32) holds the element
        const int col = ti.n0 / 2 + hc;
        if (M > ext.M) { ext.M = M; ext.cM = col; }
        if (m < ext.m) { ext.m = m; ext.cm = col; }
      }
    }
    if (sc + kParts < kNSubAll) tmem_ld_wait();
  }
}

// ── fused K1 of the A operand ──────────────────────────────────────────────
#ifndef MOE_FQ_BATCH
#define MOE_FQ_BATCH 16     // 16-byte vectors in flight per lane (8 KB per warp)
#endif
// Relaxed poll / release increment: no L1 invalidation (an acquire at GPU
// scope invalidates the SM's L1, which holds the K1 warps' reciprocal
// tables). The polled rows are read only through L2 (TMA, ld.cg).
__device__ __forceinline__ int ld_relaxed_s32(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ int ld_acquire_s32(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int atom_add_acquire_s32(int* p, int v) {
  int old;
  asm volatile("atom.acquire.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// TMA producer: wait until A rows [r0, r1) are quantized (whole 32-row blocks)
__device__ __forceinline__ void fq_wait_rows(const GemmArgs& p, int r0, int r1) {
  r1 = min(r1, p.M);
  for (int b = r0 >> 5; b * 32 < r1; ++b) {
    const int need = min(32, p.M - b * 32);
    while (ld_relaxed_s32(p.q_blk + b) < need) __nanosleep(64);
  }
  fence_acq_rel_gpu();           // acquire: order the polled flags before the TMA reads
  fence_proxy_async_global();
}

// Fused combine of one 32-column chunk of row `row` (y already dequantized
// and weighted, float): rounded to bf16 as the combine kernel would read it;
// the first of the token's two rows to get here stores it (y scratch) and
// publishes (+2); the second waits for that, adds ((0 + mine) + partner, the
// combine kernel's float order up to commutation of two terms) and stores
// the token's bf16 output.
__device__ __forceinline__ void comb_store(const GemmArgs& p, int row, int n_lo, float (&y)[32]) {
#pragma unroll
  for (int j = 0; j < 32; ++j) y[j] = __bfloat162float(__float2bfloat16_rn(y[j]));
  const int t = p.comb_src[row];
  int* ctr = p.comb_cnt + (int64_t)t * p.comb_chunks + (n_lo >> 5);
  // acquire on the arrival (and on the rare poll): when the partner has
  // already released (+2), its row is visible to the reads below
  const int old = atom_add_acquire_s32(ctr, 1);
  if (old == 0) {
    store32<true>(p.out, (int64_t)row * p.ldo + n_lo, y, 32, true);
    red_release_add(ctr, 2);
  } else {
    if (old < 3)
      while (ld_acquire_s32(ctr) < 4) __nanosleep(32);
    const int r0 = p.comb_pos[2 * t], r1 = p.comb_pos[2 * t + 1];
    const uint4* src = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.out) +
                                                      (int64_t)(r0 == row ? r1 : r0) * p.ldo + n_lo);
    float o[32];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint4 u = __ldcg(src + q);
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        o[q * 8 + 2 * e] = (0.f + y[q * 8 + 2 * e]) + __uint_as_float(w[e] << 16);
        o[q * 8 + 2 * e + 1] = (0.f + y[q * 8 + 2 * e + 1]) + __uint_as_float(w[e] & 0xFFFF0000u);
      }
    }
    store32<true>(p.comb_out, (int64_t)t * p.comb_ldo + n_lo, o, 32, true);
  }
}

// Epilogue of one tile for one thread: TMEM lane quarter q, column half
// `half` (8 epilogue warps split the 256 columns), output row `row`.
template <int BN, int EPI, bool BF16, bool CB = false>
__device__ __forceinline__ void epilogue_tile(const GemmArgs& p, const TileInfo& ti, int row, uint32_t tbase,
                                              int half, ExtRec& ext, const CUtensorMap* tmO, uint8_t* obuf,
                                              uint32_t& ob, const uint8_t* pbuf) {
  const bool rvalid = row < ti.m_end;
  float sa = 0.f, rw = 1.f;
  int32_t za = 0, rsa = 0;
  if (rvalid) {
    // through L2 (ld.cg): with K1 fused, these rows were written by other SMs during this kernel
    za = __ldcg(p.a_zp + row);
    rsa = __ldcg(p.a_rowsum + row);
    if (EPI != MOE_EPI_ACC_I32) {
      sa = __ldcg(p.a_scale + row);
      if (p.row_weight) rw = p.row_weight[row];
    }
  }
  const int wbase = ti.g * p.N;
  if (EPI == MOE_EPI_SWIGLU && p.param_vec_ok && !p.bias && (BN / 4) % 16 == 0) {
    swiglu_fast<BN, BF16>(p, ti, row, tbase, half, ext, rvalid, sa, rw, za, rsa, tmO, obuf, ob, pbuf);
  } else if (EPI == MOE_EPI_SWIGLU) {
    // tile columns [0, BN/2) are gate rows, [BN/2, BN) the matching up rows
#pragma unroll 1
    for (int c = half; c < BN / 64; c += kParts) {
      uint32_t vg[32], vu[32];
      tmem_ld32(tbase + c * 32, vg);
      tmem_ld32(tbase + BN / 2 + c * 32, vu);
      tmem_ld_wait();
      float h[32];
      const int ng0 = wbase + ti.n0 + c * 32;
      if (p.param_vec_ok) {
        ColParams32 cg, cu;
        load_cols32(p, ng0, cg);
        load_cols32(p, ng0 + BN / 2, cu);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int32_t ag = zp_correct(vg[j], cg.zw[j], cg.rsw[j], za, rsa, p.Kc);
          const int32_t au = zp_correct(vu[j], cu.zw[j], cu.rsw[j], za, rsa, p.Kc);
          float g = (float)ag * (sa * cg.ws[j]);
          float u = (float)au * (sa * cu.ws[j]);
          if (p.bias) {
            g += p.bias[ng0 + j];
            u += p.bias[ng0 + BN / 2 + j];
          }
          h[j] = silu_f(g) * u * rw;
          if (BF16) h[j] = __bfloat162float(__float2bfloat16_rn(h[j]));   // the value K1 will read
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int ng = ng0 + j;
          const int nu = ng + BN / 2;
          const int32_t ag = zp_correct(vg[j], p.w_zp[ng], p.w_rowsum[ng], za, rsa, p.Kc);
          const int32_t au = zp_correct(vu[j], p.w_zp[nu], p.w_rowsum[nu], za, rsa, p.Kc);
          float g = (float)ag * (sa * p.w_scale[ng]);
          float u = (float)au * (sa * p.w_scale[nu]);
          if (p.bias) {
            g += p.bias[ng];
            u += p.bias[nu];
          }
          h[j] = silu_f(g) * u * rw;
          if (BF16) h[j] = __bfloat162float(__float2bfloat16_rn(h[j]));   // the value K1 will read
        }
      }
      if (rvalid) {
        store32<BF16>(p.out, (int64_t)row * p.ldo + ti.n0 / 2 + c * 32, h, 32, p.vec_ok);
        if (p.row_ext) chunk_ext(h, p.ns_rs32 + ti.g * p.ns_ld + ti.n0 / 2 + c * 32, ti.n0 / 2 + c * 32, ext);
      }
    }
  } else {
#pragma unroll 1
    for (int c = half; c < BN / 32; c += kParts) {
      uint32_t v[32];
      tmem_ld32(tbase + c * 32, v);
      tmem_ld_wait();
      const int n_lo = ti.n0 + c * 32;
      int nvalid = p.N - n_lo;
      nvalid = nvalid > 32 ? 32 : nvalid;
      if (!rvalid || nvalid <= 0) continue;
      if (EPI == MOE_EPI_ACC_I32) {
        int32_t* o = p.acc_out + (int64_t)row * p.ld_acc + n_lo;
        if (nvalid == 32 && p.acc_vec_ok) {
          const int4* wz = reinterpret_cast<const int4*>(p.w_zp + wbase + n_lo);
          const int4* wr = reinterpret_cast<const int4*>(p.w_rowsum + wbase + n_lo);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int4 z = __ldg(wz + q), rs = __ldg(wr + q);
            reinterpret_cast<int4*>(o)[q] =
                make_int4(zp_correct(v[4 * q], z.x, rs.x, za, rsa, p.Kc), zp_correct(v[4 * q + 1], z.y, rs.y, za, rsa, p.Kc),
                          zp_correct(v[4 * q + 2], z.z, rs.z, za, rsa, p.Kc),
                          zp_correct(v[4 * q + 3], z.w, rs.w, za, rsa, p.Kc));
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (j < nvalid) {
              const int n = wbase + n_lo + j;
              o[j] = zp_correct(v[j], p.w_zp[n], p.w_rowsum[n], za, rsa, p.Kc);
            }
          }
        }
      } else {
        float y[32];
        if (nvalid == 32 && p.param_vec_ok) {
          ColParams32 cp;
          load_cols32(p, wbase + n_lo, cp);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int32_t a = zp_correct(v[j], cp.zw[j], cp.rsw[j], za, rsa, p.Kc);
            float val = (float)a * (sa * cp.ws[j]);
            if (p.bias) val += p.bias[wbase + n_lo + j];
            y[j] = val * rw;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int n = wbase + (j < nvalid ? n_lo + j : n_lo);
            const int32_t a = zp_correct(v[j], p.w_zp[n], p.w_rowsum[n], za, rsa, p.Kc);
            float val = (float)a * (sa * p.w_scale[n]);
            if (p.bias) val += p.bias[n];
            y[j] = val * rw;
          }
        }
        if constexpr (CB) {
          comb_store(p, row, n_lo, y);
        } else {
          void* obase = p.out_tab ? p.out_tab[p.out_rank[row]] : p.out;
          const int64_t orow = p.out_tab ? (int64_t)p.out_row[row] : (int64_t)row;
          store32<BF16>(obase, orow * p.ldo + n_lo, y, nvalid, p.vec_ok);
        }
      }
    }
  }
}

// Fused K1: drain one accumulator tile (its tfull phase already observed);
// out of line so the K1 loop that calls it keeps its registers.
template <int BN, bool BF16, int CG>
static __device__ __noinline__ void fq_drain(const GemmArgs& p, const TileInfo& ti, uint32_t as, uint32_t tmem_base,
                                             uint32_t rank, int q, int half, uint64_t* tempty,
                                             const CUtensorMap* tmO, uint8_t* obuf, uint32_t& ob,
                                             const uint8_t* pbuf) {
  const int lane = threadIdx.x & 31;
  tc_fence_after();
  const int row = ti.m0 + (int)rank * kBM + q * 32 + lane;
  const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + as * BN;
  ExtRec ext{-FLT_MAX, FLT_MAX, 0, 0};
  epilogue_tile<BN, MOE_EPI_DEQUANT, BF16>(p, ti, row, tbase, half, ext, tmO, obuf, ob, pbuf);
  tc_fence_before();
  if (CG == 2) mbar_arrive_leader(&tempty[as]);
  else mbar_arrive(&tempty[as]);
}

template <int BN, int STAGES, int EPI, bool BF16, int CG, bool FQ = false, bool CB = false>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_i8_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      const __grid_constant__ CUtensorMap tmO, GemmArgs p) {
  using L = Smem<BN, STAGES, CG, EPI == MOE_EPI_SWIGLU>;
  constexpr int TM = kBM * CG;  // tile rows (a CTA pair shares one 256-row tile)
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment for the 128B-swizzled TMA / UMMA tiles (same offset in both CTAs of a pair)
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(smem + L::kTmemPtrOff);
  int* tile_start = reinterpret_cast<int*>(smem + L::kTableOff);
  int* off = tile_start + (kMaxGroups + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_tiles = (p.N + BN - 1) / BN;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int unit = (int)blockIdx.x / CG;         // scheduling unit: a CTA or a CTA pair
  const int n_units = (int)gridDim.x / CG;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    // Launched with programmatic dependent launch: until griddep_wait() only
    // work independent of the previous kernel's outputs. At decode sizes the
    // grouped GEMM streams the weights; start pulling this unit's likely
    // first weight tile (group unit / n_tiles, n block unit % n_tiles — the
    // group offsets are not known yet) into L2 while the previous kernel runs.
    if (p.pf_kb > 0) {
      const int g = unit / n_tiles, nb = unit % n_tiles;
      if (g < p.G)
        for (int kb = 0; kb < p.pf_kb; ++kb)
          tma_prefetch_2d(&tmB, kb * kBK, g * p.N + nb * BN + (int)rank * (BN / CG));
    }
  }
  griddep_wait();
  if (threadIdx.x == 0) {
    if (p.offsets) {
      for (int g = 0; g <= p.G; ++g) off[g] = p.offsets[g];
    } else {
      off[0] = 0;
      off[1] = p.M;
    }
    int acc = 0;
    for (int g = 0; g < p.G; ++g) {
      tile_start[g] = acc;
      acc += ((off[g + 1] - off[g] + TM - 1) / TM) * n_tiles;
    }
    tile_start[p.G] = acc;
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], CG);        // leader: its own expect_tx arrive + the peer's arrive
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 32 * kEpiWarps * CG);  // all epilogue threads of the pair (leader's copy)
    }
    fence_mbar_init();
  }
  if (warp == 2) {
    if (CG == 2) {
      tmem_alloc_pair(tmem_ptr, 2 * BN);
      tmem_relinquish_pair();
    } else {
      tmem_alloc(tmem_ptr, 2 * BN);
      tmem_relinquish();
    }
  }
  tc_fence_before();
  if (CG == 2) cluster_sync_all();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_ptr;
  const int total_tiles = tile_start[p.G];

  if (warp == 0 && lane == 0) {
    // ===== TMA producer (both CTAs of a pair load their own halves) =====
    const uint64_t pol_a = l2_policy(p.l2pol & 3);
    const uint64_t pol_b = l2_policy((p.l2pol >> 2) & 3);
    const int kblocks = (p.K + kBK - 1) / kBK;
    uint32_t it = 0;
    uint32_t ptile = 0;
    for (int t = unit; t < total_tiles; t += n_units, ++ptile) {
      const TileInfo ti = map_tile(t, p.G, tile_start, off, TM, BN, n_tiles, p.band);
      const int arow = ti.m0 + (int)rank * kBM;
      const int wrow = ti.g * p.N + ti.n0 + (int)rank * (BN / CG);
      if constexpr (FQ) fq_wait_rows(p, arow, min(arow + kBM, ti.m_end));
      const bool down = p.serp && (ptile & 1);
      for (int kb = 0; kb < kblocks; ++kb, ++it) {
        const int kc = down ? kblocks - 1 - kb : kb;   // k block loaded into this stage
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        {
          MOE_PROF_T0();
          mbar_wait(&empty[s], ph ^ 1);
          MOE_PROF_ADD(2);
        }
        uint8_t* sa = smem + s * L::kStage;
        uint8_t* sb = sa + L::kA;
        if (CG == 2) {
          if (leader) mbar_expect_tx(&full[s], 2 * L::kStage);
          tma_load_2d_pair(sa, &tmA, &full[s], kc * kBK, arow, pol_a);
          tma_load_2d_pair(sb, &tmB, &full[s], kc * kBK, wrow, pol_b);
          if (!leader) mbar_arrive_leader(&full[s]);
        } else {
          mbar_expect_tx(&full[s], L::kStage);
          tma_load_2d(sa, &tmA, &full[s], kc * kBK, arow, pol_a);
          tma_load_2d(sb, &tmB, &full[s], kc * kBK, wrow, pol_b);
        }
      }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ===== UMMA issuer (the leader issues for the whole pair) =====
    constexpr uint32_t idesc = idesc_i8(TM, BN);
    const int kblocks = (p.K + kBK - 1) / kBK;
    uint32_t it = 0, tile_it = 0;
#if MOE_GEMM_PROFILE
    const long long _tall = clock64();
#endif
    for (int t = unit; t < total_tiles; t += n_units, ++tile_it) {
      const uint32_t as = tile_it & 1, aph = (tile_it >> 1) & 1;
      {
        MOE_PROF_T0();
        mbar_wait(&tempty[as], aph ^ 1);
        MOE_PROF_ADD(0);
      }
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + as * BN;
      for (int kb = 0; kb < kblocks; ++kb, ++it) {
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        {
          MOE_PROF_T0();
          mbar_wait(&full[s], ph);
          MOE_PROF_ADD(kb < STAGES ? 4 : 1);   // tile start vs steady state
        }
        tc_fence_after();
        const uint32_t a_addr = smem_u32(smem + s * L::kStage);
        const uint32_t b_addr = a_addr + L::kA;
        const uint64_t adesc = sdesc_sw128(a_addr);
        const uint64_t bdesc = sdesc_sw128(b_addr);
#pragma unroll
        for (int k = 0; k < kBK / kUmmaK; ++k) {
          // advance the start address by k*32 bytes inside the swizzle atom
          const uint64_t da = adesc + (uint64_t)(k * kUmmaK / 16), db = bdesc + (uint64_t)(k * kUmmaK / 16);
          if (CG == 2) umma_i8_pair(d_tmem, da, db, idesc, (kb | k) != 0);
          else umma_i8(d_tmem, da, db, idesc, (kb | k) != 0);
        }
        if (CG == 2) umma_commit_pair(&empty[s]);
        else umma_commit(&empty[s]);
      }
      if (CG == 2) umma_commit_pair(&tfull[as]);
      else umma_commit(&tfull[as]);
    }
#if MOE_GEMM_PROFILE
    atomicAdd(&g_gemm_waits[blockIdx.x][3], (unsigned long long)(clock64() - _tall));
#endif
  } else if (warp >= 4) {
    // ===== epilogue (each CTA drains its own 128 TMEM lanes) =====
    const int q = warp & 3;            // TMEM lane quarter this warp may access
    const int half = (warp - 4) >> 2;  // which column part of the tile (0 .. kParts-1)
    uint8_t* obuf = smem + L::kOutOff + (warp - 4) * 2048;   // this warp's TMA-store staging (2 x 1 KB)
    uint32_t ob = 0;
    uint32_t tile_it = 0;
    constexpr bool fused = FQ && EPI == MOE_EPI_DEQUANT;
    if constexpr (fused) {
      // K1 of A fused in: quantize rows (claimed in order from a global
      // counter), servicing ready accumulator tiles between 8 KB batches
      int t = unit;
      bool left = true;
      auto tile_ready = [&]() {
        int ok = 0;
        if (lane == 0) ok = t < total_tiles && mbar_try_wait(smem_u32(&tfull[tile_it & 1]), (tile_it >> 1) & 1);
        return __shfl_sync(0xffffffffu, ok, 0) != 0;
      };
      auto drain = [&]() {
        const uint32_t as = tile_it & 1;
        mbar_wait(&tfull[as], (tile_it >> 1) & 1);
        const TileInfo ti = map_tile(t, p.G, tile_start, off, TM, BN, n_tiles, p.band);
        fq_drain<BN, BF16, CG>(p, ti, as, tmem_base, rank, q, half, tempty, &tmO, obuf, ob,
                               smem + L::kParamOff + as * L::kParamBuf);
        t += n_units;
        ++tile_it;
      };
      auto poll = [&]() {
        while (tile_ready()) drain();
      };
      while (t < total_tiles || left) {
        poll();
        if (left) {
          int r = 0;
          if (lane == 0) r = atomicAdd(p.q_next, 1);
          r = __shfl_sync(0xffffffffu, r, 0);
          if (r >= p.M) {
            left = false;
            continue;
          }
          k1_row_warp<true, MOE_FQ_BATCH>(p.qa, r, p.q_rs32, p.q_ext, 8, 0, p.q_codes, p.q_ldc, p.q_scale,
                                          const_cast<float*>(p.a_scale), const_cast<int32_t*>(p.a_zp),
                                          const_cast<int32_t*>(p.a_rowsum), lane, poll);
          __syncwarp();
          if (lane == 0) {
            fence_proxy_async_global();   // the codes are read by TMA (async proxy)
            red_release_add(p.q_blk + (r >> 5), 1);
          }
        } else if (t < total_tiles) {
          drain();
        }
      }
    }
    for (int t = fused ? total_tiles : unit; t < total_tiles; t += n_units, ++tile_it) {
      const TileInfo ti = map_tile(t, p.G, tile_start, off, TM, BN, n_tiles, p.band);
      const uint32_t as = tile_it & 1, aph = (tile_it >> 1) & 1;
      uint8_t* pbuf = smem + L::kParamOff + (tile_it & 1) * L::kParamBuf;
      if constexpr (EPI == MOE_EPI_SWIGLU) {
        if (p.param_vec_ok && !p.bias) {
          // stage this tile's column parameters while the MMAs run (the loads'
          // latency overlaps the accumulator wait)
          int32_t* zw_s = reinterpret_cast<int32_t*>(pbuf);
          int32_t* t_s = zw_s + BN;
          float* ws_s = reinterpret_cast<float*>(t_s + BN);
          float* ns_s = ws_s + BN;
          for (int e = threadIdx.x - 128; e < BN; e += 32 * kEpiWarps) {
            const int n = ti.g * p.N + ti.n0 + e;
            const int32_t z = p.w_zp[n];
            zw_s[e] = z;
            t_s[e] = (int32_t)((uint32_t)p.w_rowsum[n] - (uint32_t)p.Kc * (uint32_t)z);
            ws_s[e] = p.w_scale[n];
            if (p.row_ext && e < BN / 2) ns_s[e] = p.ns_rs32[ti.g * p.ns_ld + ti.n0 / 2 + e];
          }
          named_bar_sync(1, 32 * kEpiWarps);
        }
      }
      mbar_wait(&tfull[as], aph);
      tc_fence_after();
      const int row = ti.m0 + (int)rank * kBM + q * 32 + lane;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + as * BN;
      ExtRec ext{-FLT_MAX, FLT_MAX, 0, 0};
      epilogue_tile<BN, EPI, BF16, CB>(p, ti, row, tbase, half, ext, &tmO, obuf, ob, pbuf);
      tc_fence_before();
      if (CG == 2) mbar_arrive_leader(&tempty[as]);
      else mbar_arrive(&tempty[as]);
      if (EPI == MOE_EPI_SWIGLU && p.row_ext && row < ti.m_end) {
        atomicMin(&p.row_ext[2 * (int64_t)row], ext_key(ext.m, ext.cm));
        atomicMax(&p.row_ext[2 * (int64_t)row + 1], ext_key(ext.M, ext.cM));
      }
    }
    if (lane == 0 && ob) bulk_wait_group<0>();   // TMA stores complete before the CTA retires
    if (p.out_tab) __threadfence_system();        // peer (home-rank) rows visible before the rank barrier
  }
  // (no early griddep_launch_dependents here: at decode sizes the next
  // kernels' CTAs, and behind them GEMM2's weight prefetch, then start during
  // this GEMM's weight-streaming tail: 269 -> 273 us at 16 tokens)
  tc_fence_before();
  if (CG == 2) cluster_sync_all();
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if (CG == 2) tmem_dealloc_pair(tmem_base, 2 * BN);
    else tmem_dealloc(tmem_base, 2 * BN);
  }
}

// ── SIMT path: small or unaligned shapes (same exact integer results) ─────
template <bool BF16>
__global__ void gemm_i8_simt_kernel(const uint8_t* a, int64_t lda, const uint8_t* w, int64_t ldw, GemmArgs p,
                                    int epi) {
  const int64_t total = (int64_t)p.M * (epi == MOE_EPI_SWIGLU ? p.N / 2 : p.N);
  const int ncols = epi == MOE_EPI_SWIGLU ? p.N / 2 : p.N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / ncols), c = (int)(i % ncols);
    int g = 0;
    if (p.offsets) {
      while (g + 1 < p.G && m >= p.offsets[g + 1]) ++g;
    }
    const int za = p.a_zp[m];
    auto dot = [&](int wr) {
      int32_t acc = 0;
      const int zw = p.w_zp[wr];
      for (int k = 0; k < p.K; ++k) acc += ((int)a[m * lda + k] - za) * ((int)w[(int64_t)wr * ldw + k] - zw);
      return acc;
    };
    float rw = p.row_weight ? p.row_weight[m] : 1.f;
    if (epi == MOE_EPI_SWIGLU) {
      const int blk = c / 128, j = c % 128;
      const int ng = g * p.N + blk * 256 + j, nu = ng + 128;
      float gg = (float)dot(ng) * (p.a_scale[m] * p.w_scale[ng]);
      float uu = (float)dot(nu) * (p.a_scale[m] * p.w_scale[nu]);
      if (p.bias) {
        gg += p.bias[ng];
        uu += p.bias[nu];
      }
      const float h = silu_f(gg) * uu * rw;
      if (BF16) static_cast<__nv_bfloat16*>(p.out)[m * p.ldo + c] = __float2bfloat16_rn(h);
      else static_cast<float*>(p.out)[m * p.ldo + c] = h;
    } else {
      const int n = g * p.N + c;
      const int32_t acc = dot(n);
      if (epi == MOE_EPI_ACC_I32) {
        p.acc_out[m * p.ld_acc + c] = acc;
      } else {
        float val = (float)acc * (p.a_scale[m] * p.w_scale[n]);
        if (p.bias) val += p.bias[n];
        val *= rw;
        if (BF16) static_cast<__nv_bfloat16*>(p.out)[m * p.ldo + c] = __float2bfloat16_rn(val);
        else static_cast<float*>(p.out)[m * p.ldo + c] = val;
      }
    }
  }
}

// ── host side ──────────────────────────────────────────────────────────────
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
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

static bool make_map_u8(CUtensorMap* m, const void* ptr, uint64_t rows, uint64_t cols, uint64_t ld,
                        uint32_t box_rows) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld};
  cuuint32_t box[2] = {(cuuint32_t)kBK, box_rows};
  cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(ptr), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN, int STAGES, int EPI, bool BF16, int CG, bool FQ = false, bool CB = false>
static moe_status launch_tc(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& to, const GemmArgs& p,
                            int grid, cudaStream_t s) {
  auto kern = gemm_i8_tc_kernel<BN, STAGES, EPI, BF16, CG, FQ, CB>;
  constexpr int bytes = Smem<BN, STAGES, CG, EPI == MOE_EPI_SWIGLU>::kBytes;
  static_assert(bytes <= 232448, "shared memory per CTA");
  MOE_CUDA_TRY(set_max_smem_once(reinterpret_cast<const void*>(kern), bytes));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  static const bool no_pdl = getenv("MOE_B200_NO_PDL") != nullptr;   // (A/B switch)
  if (!no_pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL (see griddep_wait)
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  if (CG == 2) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na++].val.clusterDim.z = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  MOE_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, ta, tb, to, p));
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

template <int CG>
static moe_status dispatch_tc(const uint8_t* a, int64_t M, int64_t K, int64_t lda, const uint8_t* w, int64_t N,
                              int64_t ldw, int num_groups, int epilogue, bool bf16, GemmArgs p,
                              cudaStream_t s) {
  constexpr int BN = 256;
  constexpr int ST = CG == 2 ? 6 : 4;
  CUtensorMap ta, tb;
  if (!make_map_u8(&ta, a, (uint64_t)M, (uint64_t)K, (uint64_t)lda, kBM) ||
      !make_map_u8(&tb, w, (uint64_t)N * num_groups, (uint64_t)K, (uint64_t)ldw, BN / CG)) {
    set_error("w8a8_gemm: cuTensorMapEncodeTiled failed");
    return MOE_ECUDA;
  }
  // SwiGLU bf16 output: stored through shared memory by TMA (32 x 16 boxes)
  CUtensorMap to = ta;
  p.tma_out = 0;
  if (epilogue == MOE_EPI_SWIGLU && bf16 && p.vec_ok && getenv("MOE_B200_NO_TMA_STORE") == nullptr) {
    auto enc = tensor_map_encoder();
    cuuint64_t dims[2] = {(cuuint64_t)(N / 2), (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)p.ldo * 2};
    cuuint32_t box[2] = {16, 32};
    cuuint32_t es[2] = {1, 1};
    if (enc && enc(&to, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, p.out, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      p.tma_out = 1;
  }
  const int64_t TM = kBM * CG;
  const int64_t n_tiles = (N + BN - 1) / BN;
  // raster band: keep ~24 MB of activations L2-resident per band
  {
    const int64_t budget = std::max<int64_t>(1, tune_value(MOE_TUNE_BAND_MB)) << 20;
    p.band = (int)std::max<int64_t>(1, std::min<int64_t>(1 << 20, budget / (TM * std::max<int64_t>(K, 1))));
  }
  // decode sizes (weight-stream bound): L2-prefetch the first 640 KB of each
  // unit's first weight tile during the previous kernel (PDL)
  {
    static const int env_pol = getenv("MOE_B200_GEMM_L2POL") ? atoi(getenv("MOE_B200_GEMM_L2POL")) : -1;
    p.l2pol = env_pol >= 0 ? env_pol : 0;
  }
  {
    static const int env_serp = getenv("MOE_B200_GEMM_SERP") ? atoi(getenv("MOE_B200_GEMM_SERP")) : 1;
    p.serp = env_serp;
  }
  p.pf_kb = (M <= 1024) ? (int)std::min<int64_t>((K + kBK - 1) / kBK, (640 << 10) / ((BN / CG) * kBK)) : 0;
  const int64_t units_bound = ((M + TM - 1) / TM + num_groups) * n_tiles;
  const int64_t max_units = num_sms() / CG;
  const int grid = (int)(std::min<int64_t>(units_bound, max_units) * CG);
  switch (epilogue) {
    case MOE_EPI_DEQUANT:
      // (a 7th stage fits the dequant kernels, which need no epilogue staging:
      // GEMM2 +2-3 %, tools/st2_ab.sh at the time — not kept)
      if (p.comb_cnt)   // fused top-2 combine (bf16 only, checked by the entry point)
        return launch_tc<BN, ST, MOE_EPI_DEQUANT, true, CG, false, true>(ta, tb, to, p, grid, s);
      if (p.fq)   // K1 of A fused in (separate instantiation: the plain kernel keeps its registers)
        return bf16 ? launch_tc<BN, ST, MOE_EPI_DEQUANT, true, CG, true>(ta, tb, to, p, grid, s)
                    : launch_tc<BN, ST, MOE_EPI_DEQUANT, false, CG, true>(ta, tb, to, p, grid, s);
      return bf16 ? launch_tc<BN, ST, MOE_EPI_DEQUANT, true, CG>(ta, tb, to, p, grid, s)
                  : launch_tc<BN, ST, MOE_EPI_DEQUANT, false, CG>(ta, tb, to, p, grid, s);
    case MOE_EPI_SWIGLU:
      return bf16 ? launch_tc<BN, ST, MOE_EPI_SWIGLU, true, CG>(ta, tb, to, p, grid, s)
                  : launch_tc<BN, ST, MOE_EPI_SWIGLU, false, CG>(ta, tb, to, p, grid, s);
    default:
      return launch_tc<BN, ST, MOE_EPI_ACC_I32, false, CG>(ta, tb, to, p, grid, s);
  }
}

}  // namespace moe

using namespace moe;

static moe_status gemm_entry(const uint8_t* a, int64_t M, int64_t K, int64_t lda, const float* a_scale,
                             const int32_t* a_zp, const int32_t* a_rowsum, const uint8_t* w, int64_t N, int64_t ldw,
                             const float* w_scale, const int32_t* w_zp, const int32_t* w_rowsum, const float* bias,
                             const float* row_weight, const int32_t* group_offsets, int num_groups, int epilogue,
                             void* out, int out_dtype, int64_t ldo, int32_t* acc_out, int64_t ld_acc,
                             const float* next_smooth_recip_f32, int64_t next_ld, unsigned long long* row_ext,
                             void* const* out_tab, const int32_t* out_rank, const int32_t* out_row,
                             moe_stream_t stream, const GemmArgs* fq = nullptr, const GemmArgs* cb = nullptr) {
  MOE_REQUIRE(a && w && a_zp && w_zp && a_rowsum && w_rowsum, "w8a8_gemm: null operand");
  const bool w_corr = (epilogue & MOE_EPI_FLAG_WCORR) != 0;
  const bool ext_ready = (epilogue & MOE_EPI_FLAG_EXT_READY) != 0;
  epilogue &= 0xFF;
  if (row_ext) {
    MOE_REQUIRE(epilogue == MOE_EPI_SWIGLU, "w8a8_gemm: row_ext is produced by the SwiGLU epilogue");
    MOE_REQUIRE(next_smooth_recip_f32 && next_ld >= N / 2 && next_ld % 4 == 0,
                "w8a8_gemm: row_ext needs the next float32 reciprocal smoothing table");
  }
  MOE_REQUIRE(M >= 1 && N >= 1 && K >= 1, "w8a8_gemm: empty problem");
  MOE_REQUIRE(lda >= K && ldw >= K, "w8a8_gemm: bad leading dimension");
  MOE_REQUIRE(M < (1LL << 31) && N < (1LL << 31) && K <= 33025, "w8a8_gemm: K too large for exact int32");
  MOE_REQUIRE(num_groups >= 1 && num_groups <= kMaxGroups, "w8a8_gemm: 1..64 groups");
  MOE_REQUIRE(num_groups == 1 || group_offsets, "w8a8_gemm: grouped GEMM needs offsets");
  MOE_REQUIRE(epilogue >= 0 && epilogue <= 2, "w8a8_gemm: unknown epilogue");
  if (epilogue == MOE_EPI_ACC_I32) {
    MOE_REQUIRE(acc_out && ld_acc >= N, "w8a8_gemm: ACC_I32 needs acc_out");
  } else {
    MOE_REQUIRE(out && a_scale && w_scale, "w8a8_gemm: dequant epilogue needs out and scales");
    MOE_REQUIRE(out_dtype == MOE_DT_F32 || out_dtype == MOE_DT_BF16, "w8a8_gemm: out dtype f32|bf16");
    MOE_REQUIRE(ldo >= (epilogue == MOE_EPI_SWIGLU ? N / 2 : N), "w8a8_gemm: bad ldo");
  }
  if (epilogue == MOE_EPI_SWIGLU) MOE_REQUIRE(N % 256 == 0, "w8a8_gemm: SwiGLU needs N % 256 == 0");

  GemmArgs p{};
  p.M = (int)M;
  p.N = (int)N;
  p.K = (int)K;
  p.Kc = w_corr ? 0 : (int)K;
  p.G = num_groups;
  p.offsets = group_offsets;
  p.a_scale = a_scale;
  p.a_zp = a_zp;
  p.a_rowsum = a_rowsum;
  p.w_scale = w_scale;
  p.w_zp = w_zp;
  p.w_rowsum = w_rowsum;
  p.bias = bias;
  p.row_weight = row_weight;
  p.out = out;
  p.ldo = ldo;
  p.acc_out = acc_out;
  p.ld_acc = ld_acc;
  p.ns_rs32 = next_smooth_recip_f32;
  p.ns_ld = next_ld;
  p.row_ext = row_ext;
  p.out_tab = out_tab;
  p.out_rank = out_rank;
  p.out_row = out_row;
  if (cb) {
    p.comb_src = cb->comb_src;
    p.comb_pos = cb->comb_pos;
    p.comb_cnt = cb->comb_cnt;
    p.comb_chunks = cb->comb_chunks;
    p.comb_out = cb->comb_out;
    p.comb_ldo = cb->comb_ldo;
  }
  if (fq) {
    p.fq = 1;
    p.qa = fq->qa;
    p.q_rs32 = fq->q_rs32;
    p.q_ext = fq->q_ext;
    p.q_codes = fq->q_codes;
    p.q_ldc = fq->q_ldc;
    p.q_scale = fq->q_scale;
    p.q_next = fq->q_next;
    p.q_blk = fq->q_blk;
  }
  const int esz = out_dtype == MOE_DT_BF16 ? 2 : 4;
  p.vec_ok = out && ((reinterpret_cast<uintptr_t>(out) & 15) == 0) && ((ldo * esz) % 16 == 0);
  p.acc_vec_ok = acc_out && ((reinterpret_cast<uintptr_t>(acc_out) & 15) == 0) && (ld_acc % 4 == 0) &&
                 ((reinterpret_cast<uintptr_t>(w_zp) & 15) == 0) && ((reinterpret_cast<uintptr_t>(w_rowsum) & 15) == 0) &&
                 (N % 4 == 0);
  p.param_vec_ok = ((reinterpret_cast<uintptr_t>(w_zp) & 15) == 0) && ((reinterpret_cast<uintptr_t>(w_rowsum) & 15) == 0) &&
                   (!w_scale || (reinterpret_cast<uintptr_t>(w_scale) & 15) == 0) && (N % 4 == 0);
  cudaStream_t s = as_stream(stream);
  if (row_ext && !ext_ready) {
    rowext_init_kernel<<<(unsigned)std::min<int64_t>((M + 255) / 256, 4 * num_sms()), 256, 0, s>>>(row_ext, M);
    ::moe::count_launch();
  }
  const bool bf16 = out_dtype == MOE_DT_BF16;

  const bool tc_ok = (K % 16 == 0) && K >= kBK && (lda % 16 == 0) && (ldw % 16 == 0) &&
                     ((reinterpret_cast<uintptr_t>(a) & 15) == 0) && ((reinterpret_cast<uintptr_t>(w) & 15) == 0);
  MOE_REQUIRE(tc_ok || !row_ext, "w8a8_gemm: row_ext needs the tensor-core path (K % 16 == 0, K >= 128)");
  MOE_REQUIRE(tc_ok || !fq, "w8a8_gemm: fused A quantization needs the tensor-core path");
  MOE_REQUIRE(tc_ok || !cb, "w8a8_gemm: fused combine needs the tensor-core path");
  if (tc_ok) {
    // CTA pairs once there are enough 256-row tiles to fill the machine
    const bool pair = M >= 256 * 8 && getenv("MOE_B200_NO_PAIR") == nullptr;
    return pair ? dispatch_tc<2>(a, M, K, lda, w, N, ldw, num_groups, epilogue, bf16, p, s)
                : dispatch_tc<1>(a, M, K, lda, w, N, ldw, num_groups, epilogue, bf16, p, s);
  }
  const int64_t total = M * (epilogue == MOE_EPI_SWIGLU ? N / 2 : N);
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)num_sms() * 32) blocks = (int64_t)num_sms() * 32;
  if (bf16) gemm_i8_simt_kernel<true><<<(unsigned)blocks, 256, 0, s>>>(a, lda, w, ldw, p, epilogue);
  else gemm_i8_simt_kernel<false><<<(unsigned)blocks, 256, 0, s>>>(a, lda, w, ldw, p, epilogue);
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_w8a8_gemm(const uint8_t* a, int64_t M, int64_t K, int64_t lda, const float* a_scale,
                                    const int32_t* a_zp, const int32_t* a_rowsum, const uint8_t* w, int64_t N,
                                    int64_t ldw, const float* w_scale, const int32_t* w_zp,
                                    const int32_t* w_rowsum, const float* bias, const float* row_weight,
                                    const int32_t* group_offsets, int num_groups, int epilogue, void* out,
                                    int out_dtype, int64_t ldo, int32_t* acc_out, int64_t ld_acc,
                                    const float* next_smooth_recip_f32, int64_t next_ld, unsigned long long* row_ext,
                                    moe_stream_t stream) {
  return gemm_entry(a, M, K, lda, a_scale, a_zp, a_rowsum, w, N, ldw, w_scale, w_zp, w_rowsum, bias, row_weight,
                    group_offsets, num_groups, epilogue, out, out_dtype, ldo, acc_out, ld_acc, next_smooth_recip_f32,
                    next_ld, row_ext, nullptr, nullptr, nullptr, stream);
}

extern "C" moe_status moe_w8a8_gemm_scatter(const uint8_t* a, int64_t M, int64_t K, int64_t lda,
                                            const float* a_scale, const int32_t* a_zp, const int32_t* a_rowsum,
                                            const uint8_t* w, int64_t N, int64_t ldw, const float* w_scale,
                                            const int32_t* w_zp, const int32_t* w_rowsum, const float* bias,
                                            const float* row_weight, const int32_t* group_offsets, int num_groups,
                                            int epilogue, void* const* out_tab, const int32_t* out_rank,
                                            const int32_t* out_row, int out_dtype, int64_t ldo, moe_stream_t stream) {
  MOE_REQUIRE(out_tab && out_rank && out_row, "w8a8_gemm_scatter: null output table");
  MOE_REQUIRE((epilogue & 0xFF) == MOE_EPI_DEQUANT, "w8a8_gemm_scatter: dequant epilogue only");
  // the vector-store check inspects `out`: the table's buffers share the allocation granularity
  return gemm_entry(a, M, K, lda, a_scale, a_zp, a_rowsum, w, N, ldw, w_scale, w_zp, w_rowsum, bias, row_weight,
                    group_offsets, num_groups, epilogue, const_cast<void*>(reinterpret_cast<const void*>(out_tab)),
                    out_dtype, ldo, nullptr, 0, nullptr, 0, nullptr, out_tab, out_rank, out_row, stream);
}

extern "C" int64_t moe_w8a8_gemm_quant_a_workspace(int64_t M) { return 4 * (1 + (M + 31) / 32); }

extern "C" moe_status moe_w8a8_gemm_quant_a(
    const void* x, int64_t ldx, const double* smooth, const double* smooth_recip, const float* smooth_recip_f32,
    const int32_t* row_group, const unsigned long long* row_ext, uint8_t* a, int64_t lda, double* a_scale64,
    float* a_scale, int32_t* a_zp, int32_t* a_rowsum, int64_t M, int64_t K, const uint8_t* w, int64_t N, int64_t ldw,
    const float* w_scale, const int32_t* w_zp, const int32_t* w_rowsum, const float* bias, const float* row_weight,
    const int32_t* group_offsets, int num_groups, int epilogue, void* out, int out_dtype, int64_t ldo,
    void* workspace, int64_t workspace_bytes, moe_stream_t stream) {
  MOE_REQUIRE(x && smooth && smooth_recip && smooth_recip_f32 && row_ext && a && a_scale64 && a_scale && a_zp &&
                  a_rowsum,
              "w8a8_gemm_quant_a: null operand");
  MOE_REQUIRE((epilogue & 0xFF) == MOE_EPI_DEQUANT, "w8a8_gemm_quant_a: dequant epilogue only");
  MOE_REQUIRE(M >= 1 && K % 8 == 0 && ldx % 8 == 0 && lda >= K && (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(a) & 7) == 0 && lda % 8 == 0,
              "w8a8_gemm_quant_a: bf16 rows with K % 8 == 0, 16-byte aligned");
  MOE_REQUIRE(workspace && workspace_bytes >= moe_w8a8_gemm_quant_a_workspace(M), "w8a8_gemm_quant_a: workspace");
  GemmArgs fq{};
  fq.qa = RowArgs{x, MOE_DT_BF16, M, K, ldx, nullptr, row_group, SmoothArgs{smooth, smooth_recip, MOE_SMOOTH_DIVIDE, K}};
  fq.q_rs32 = smooth_recip_f32;
  fq.q_ext = row_ext;
  fq.q_codes = a;
  fq.q_ldc = lda;
  fq.q_scale = a_scale64;
  fq.q_next = static_cast<int*>(workspace);
  fq.q_blk = fq.q_next + 1;
  MOE_CUDA_TRY(cudaMemsetAsync(workspace, 0, (size_t)moe_w8a8_gemm_quant_a_workspace(M), as_stream(stream)));
  return gemm_entry(a, M, K, lda, a_scale, a_zp, a_rowsum, w, N, ldw, w_scale, w_zp, w_rowsum, bias, row_weight,
                    group_offsets, num_groups, epilogue, out, out_dtype, ldo, nullptr, 0, nullptr, 0, nullptr, nullptr,
                    nullptr, nullptr, stream, &fq);
}

extern "C" int64_t moe_w8a8_gemm_combine_workspace(int64_t T, int64_t N) { return 4 * T * ((N + 31) / 32); }

namespace moe {
__global__ void step_init_kernel(uint4* zero, int64_t n16, unsigned long long* re, int64_t rows) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += stride)
    zero[i] = make_uint4(0u, 0u, 0u, 0u);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows; i += stride) {
    re[2 * i] = ~0ull;     // min record
    re[2 * i + 1] = 0ull;  // max record
  }
}
}  // namespace moe

extern "C" moe_status moe_step_init(void* zero, int64_t zero_bytes, unsigned long long* row_ext, int64_t rows,
                                    moe_stream_t stream) {
  MOE_REQUIRE(zero_bytes >= 0 && rows >= 0, "step_init: negative sizes");
  MOE_REQUIRE(!zero_bytes || (zero && zero_bytes % 16 == 0 && (reinterpret_cast<uintptr_t>(zero) & 15) == 0),
              "step_init: zero buffer must be 16-byte aligned and sized");
  MOE_REQUIRE(!rows || row_ext, "step_init: null row_ext");
  const int64_t work = std::max<int64_t>(zero_bytes / 16, rows);
  if (work == 0) return MOE_OK;
  const unsigned blocks = (unsigned)std::min<int64_t>((work + 255) / 256, (int64_t)num_sms() * 8);
  step_init_kernel<<<blocks, 256, 0, as_stream(stream)>>>(static_cast<uint4*>(zero), zero_bytes / 16, row_ext, rows);
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_w8a8_gemm_combine(const uint8_t* a, int64_t M, int64_t K, int64_t lda, const float* a_scale,
                                            const int32_t* a_zp, const int32_t* a_rowsum, const uint8_t* w, int64_t N,
                                            int64_t ldw, const float* w_scale, const int32_t* w_zp,
                                            const int32_t* w_rowsum, const float* row_weight,
                                            const int32_t* group_offsets, int num_groups, int epilogue, void* y,
                                            int64_t ldy, const int32_t* src_token, const int32_t* token_pos,
                                            int64_t T, void* out, int64_t ldo, void* workspace,
                                            int64_t workspace_bytes, moe_stream_t stream) {
  MOE_REQUIRE(y && out && src_token && token_pos, "w8a8_gemm_combine: null pointer");
  MOE_REQUIRE((epilogue & 0xFF) == MOE_EPI_DEQUANT, "w8a8_gemm_combine: dequant epilogue only");
  MOE_REQUIRE(M == 2 * T, "w8a8_gemm_combine: top-2 routing (M == 2 T)");
  MOE_REQUIRE(N % 32 == 0 && ldy % 8 == 0 && ldo % 8 == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(out) & 15) == 0,
              "w8a8_gemm_combine: N % 32 == 0 and 16-byte aligned bf16 rows");
  MOE_REQUIRE(workspace && workspace_bytes >= moe_w8a8_gemm_combine_workspace(T, N),
              "w8a8_gemm_combine: workspace");
  GemmArgs cb{};
  cb.comb_src = src_token;
  cb.comb_pos = token_pos;
  cb.comb_cnt = static_cast<int*>(workspace);
  cb.comb_chunks = (int)(N / 32);
  cb.comb_out = static_cast<__nv_bfloat16*>(out);
  cb.comb_ldo = ldo;
  if (!(epilogue & MOE_EPI_FLAG_WS_ZEROED))
    MOE_CUDA_TRY(cudaMemsetAsync(workspace, 0, (size_t)moe_w8a8_gemm_combine_workspace(T, N), as_stream(stream)));
  return gemm_entry(a, M, K, lda, a_scale, a_zp, a_rowsum, w, N, ldw, w_scale, w_zp, w_rowsum, nullptr, row_weight,
                    group_offsets, num_groups, epilogue & ~MOE_EPI_FLAG_WS_ZEROED, y, MOE_DT_BF16, ldy, nullptr, 0,
                    nullptr, 0, nullptr, nullptr, nullptr, nullptr, stream, nullptr, &cb);
}

#if MOE_GEMM_PROFILE
extern "C" int moe_debug_gemm_waits(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_gemm_waits, sizeof(g_gemm_waits));
  if (reset) {
    static unsigned long long zeros[1024][6] = {};
    cudaMemcpyToSymbol(g_gemm_waits, zeros, sizeof(zeros));
  }
  return (int)cudaGetLastError();
}
#endif
