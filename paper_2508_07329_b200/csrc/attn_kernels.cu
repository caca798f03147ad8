// Attention-block glue of the 32-layer token path:
// rotary position embedding applied in place to the q / k heads of the
// fused W8A8 QKV projection's bf16 output. The attention itself is the
// library's SDPA (cuDNN / flash) on bf16; the projections are the W8A8
// linear (K1 + K2).
//
// Rotate-half convention (Llama / Mixtral): for pair (i, i + hd/2) of a head,
//   out_i        = x_i * cos(p w_i) - x_{i+hd/2} * sin(p w_i)
//   out_{i+hd/2} = x_{i+hd/2} * cos(p w_i) + x_i * sin(p w_i)
// with w_i = theta^(-2i/hd); cos / sin come from a float32 table
// [max_pos, hd/2] built once in float64 by the host layer, the products in
// float32, one bf16 rounding per output. HBM-bound: one read and one write
// of the q / k part of each row.
#include <algorithm>

#include "common.cuh"

namespace moe {

// one thread = 8 consecutive pair indices i of one (token, head)
__global__ void rope_bf16_kernel(__nv_bfloat16* x, int64_t T, int heads, int hd, int64_t ld, const int32_t* pos,
                                 const float* cos_tab, const float* sin_tab) {
  const int half = hd / 2, groups = half / 8;
  const int64_t n = T * heads * groups;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int g = (int)(i % groups);
    const int64_t th = i / groups;
    const int h = (int)(th % heads);
    const int64_t t = th / heads;
    __nv_bfloat16* row = x + t * ld + (int64_t)h * hd;
    const int64_t p = pos ? pos[t] : t;
    const float* ct = cos_tab + p * half + g * 8;
    const float* st = sin_tab + p * half + g * 8;
    uint4 a = *reinterpret_cast<const uint4*>(row + g * 8);
    uint4 b = *reinterpret_cast<const uint4*>(row + half + g * 8);
    __nv_bfloat162* pa = reinterpret_cast<__nv_bfloat162*>(&a);
    __nv_bfloat162* pb = reinterpret_cast<__nv_bfloat162*>(&b);
    const float4 c0 = *reinterpret_cast<const float4*>(ct), c1 = *reinterpret_cast<const float4*>(ct + 4);
    const float4 s0 = *reinterpret_cast<const float4*>(st), s1 = *reinterpret_cast<const float4*>(st + 4);
    const float cs[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
    const float sn[8] = {s0.x, s0.y, s0.z, s0.w, s1.x, s1.y, s1.z, s1.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 xa = __bfloat1622float2(pa[q]), xb = __bfloat1622float2(pb[q]);
      const float2 oa = make_float2(fmaf(xa.x, cs[2 * q], -xb.x * sn[2 * q]),
                                    fmaf(xa.y, cs[2 * q + 1], -xb.y * sn[2 * q + 1]));
      const float2 ob = make_float2(fmaf(xb.x, cs[2 * q], xa.x * sn[2 * q]),
                                    fmaf(xb.y, cs[2 * q + 1], xa.y * sn[2 * q + 1]));
      pa[q] = __float22bfloat162_rn(oa);
      pb[q] = __float22bfloat162_rn(ob);
    }
    *reinterpret_cast<uint4*>(row + g * 8) = a;
    *reinterpret_cast<uint4*>(row + half + g * 8) = b;
  }
}

}  // namespace moe

using namespace moe;

extern "C" moe_status moe_rope_bf16(void* x, int64_t T, int heads, int head_dim, int64_t ld, const int32_t* positions,
                                    const float* cos_tab, const float* sin_tab, moe_stream_t stream) {
  MOE_REQUIRE(x && cos_tab && sin_tab && T >= 1 && heads >= 1, "rope_bf16: bad arguments");
  MOE_REQUIRE(head_dim % 16 == 0 && ld % 8 == 0 && ld >= (int64_t)heads * head_dim &&
                  (reinterpret_cast<uintptr_t>(x) & 15) == 0,
              "rope_bf16: head_dim % 16 == 0, 16-byte aligned rows");
  const int64_t n = T * heads * (head_dim / 16);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 8 * (int64_t)num_sms()));
  rope_bf16_kernel<<<blocks, 256, 0, as_stream(stream)>>>(static_cast<__nv_bfloat16*>(x), T, heads, head_dim, ld,
                                                          positions, cos_tab, sin_tab);
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}
