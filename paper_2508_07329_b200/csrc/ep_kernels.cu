// Expert-parallel plumbing kernels: the data movement either
// side of the two NCCL all-to-all exchanges of an EP MoE forward.
//
//   sender:   route keys (dest rank, expert) -> route_permute -> K1 codes
//             + packed per-row params [scale_f32 | zp | rowsum | weight]
//   receiver: gather the received rows into expert-contiguous order (codes
//             and SoA params for the grouped GEMM), and after GEMM2 gather
//             the output rows back into receive order for the return trip.
//
// All of it is HBM-bound row copying: one warp per row, 16-byte vectors.
#include <algorithm>

#include "common.cuh"

namespace moe {

__global__ void route_keys_kernel(const int32_t* idx, int64_t n, const int32_t* dest, int E, int32_t* keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int e = idx[i];
    keys[i] = dest[e] * E + e;
  }
}

template <typename V>
__global__ void gather_rows_kernel(const uint8_t* src, int64_t src_ld, const int32_t* index, int64_t n,
                                   int64_t nvec, uint8_t* dst, int64_t dst_ld) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
    const int64_t s = index ? index[r] : r;
    const V* sp = reinterpret_cast<const V*>(src + s * src_ld);
    V* dp = reinterpret_cast<V*>(dst + r * dst_ld);
    for (int64_t c = lane; c < nvec; c += 32) dp[c] = __ldcs(sp + c);
  }
}

__global__ void pack_params_kernel(const float* scale, const int32_t* zp, const int32_t* rowsum, const float* weight,
                                   int64_t n, int4* params) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    params[i] = make_int4(__float_as_int(scale[i]), zp[i], rowsum[i], weight ? __float_as_int(weight[i]) : 0x3F800000);
}

__global__ void unpack_params_kernel(const int4* params, const int32_t* index, int64_t n, float* scale, int32_t* zp,
                                     int32_t* rowsum, float* weight) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 p = params[index ? index[i] : i];
    scale[i] = __int_as_float(p.x);
    zp[i] = p.y;
    rowsum[i] = p.z;
    if (weight) weight[i] = __int_as_float(p.w);
  }
}

// rows grouped in contiguous blocks [start[b], start[b+1]): out0[i] = val0[b],
// out1[i] = val1[b] + (i - start[b])   (binary search over nb blocks)
__global__ void block_map_kernel(int64_t n, int nb, const int32_t* start, const int32_t* val0, const int32_t* val1,
                                 int32_t* out0, int32_t* out1) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = nb;   // last b with start[b] <= i
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (start[mid] <= i) lo = mid;
      else hi = mid;
    }
    out0[i] = val0[lo];
    out1[i] = val1[lo] + (int32_t)(i - start[lo]);
  }
}

static unsigned grid_for(int64_t n, int per_block) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + per_block - 1) / per_block, 8 * (int64_t)num_sms()));
}

}  // namespace moe

using namespace moe;

extern "C" moe_status moe_route_keys(const int32_t* topk_idx, int64_t n, const int32_t* dest_rank, int E,
                                     int32_t* keys, moe_stream_t stream) {
  MOE_REQUIRE(topk_idx && dest_rank && keys && n >= 1 && E >= 1, "route_keys: bad arguments");
  route_keys_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(topk_idx, n, dest_rank, E, keys);
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_gather_rows(const void* src, int64_t src_ld_bytes, const int32_t* index, int64_t n,
                                      int64_t row_bytes, void* dst, int64_t dst_ld_bytes, moe_stream_t stream) {
  MOE_REQUIRE(src && dst && row_bytes >= 1 && n >= 0, "gather_rows: bad arguments");
  MOE_REQUIRE(src_ld_bytes >= row_bytes && dst_ld_bytes >= row_bytes, "gather_rows: bad leading dimension");
  if (n == 0) return MOE_OK;
  cudaStream_t s = as_stream(stream);
  const uint8_t* sp = static_cast<const uint8_t*>(src);
  uint8_t* dp = static_cast<uint8_t*>(dst);
  const bool v16 = row_bytes % 16 == 0 && src_ld_bytes % 16 == 0 && dst_ld_bytes % 16 == 0 &&
                   (reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  const bool v4 = row_bytes % 4 == 0 && src_ld_bytes % 4 == 0 && dst_ld_bytes % 4 == 0 &&
                  (reinterpret_cast<uintptr_t>(src) & 3) == 0 && (reinterpret_cast<uintptr_t>(dst) & 3) == 0;
  const unsigned grid = grid_for(n, 8);
  if (v16)
    gather_rows_kernel<uint4><<<grid, 256, 0, s>>>(sp, src_ld_bytes, index, n, row_bytes / 16, dp, dst_ld_bytes);
  else if (v4)
    gather_rows_kernel<uint32_t><<<grid, 256, 0, s>>>(sp, src_ld_bytes, index, n, row_bytes / 4, dp, dst_ld_bytes);
  else
    gather_rows_kernel<uint8_t><<<grid, 256, 0, s>>>(sp, src_ld_bytes, index, n, row_bytes, dp, dst_ld_bytes);
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_ep_pack_params(const float* scale_f32, const int32_t* zp, const int32_t* rowsum,
                                         const float* weight, int64_t n, int32_t* params, moe_stream_t stream) {
  MOE_REQUIRE(scale_f32 && zp && rowsum && params && n >= 0, "ep_pack_params: bad arguments");
  MOE_REQUIRE((reinterpret_cast<uintptr_t>(params) & 15) == 0, "ep_pack_params: params must be 16-byte aligned");
  if (n == 0) return MOE_OK;
  pack_params_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(scale_f32, zp, rowsum, weight, n,
                                                                       reinterpret_cast<int4*>(params));
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_ep_unpack_params(const int32_t* params, const int32_t* index, int64_t n, float* scale_f32,
                                           int32_t* zp, int32_t* rowsum, float* weight, moe_stream_t stream) {
  MOE_REQUIRE(params && scale_f32 && zp && rowsum && n >= 0, "ep_unpack_params: bad arguments");
  MOE_REQUIRE((reinterpret_cast<uintptr_t>(params) & 15) == 0, "ep_unpack_params: params must be 16-byte aligned");
  if (n == 0) return MOE_OK;
  unpack_params_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(reinterpret_cast<const int4*>(params), index,
                                                                         n, scale_f32, zp, rowsum, weight);
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_block_map(int64_t n, int nblocks, const int32_t* block_start, const int32_t* val0,
                                    const int32_t* val1, int32_t* out0, int32_t* out1, moe_stream_t stream) {
  MOE_REQUIRE(n >= 0 && nblocks >= 1 && block_start && val0 && val1 && out0 && out1, "block_map: bad arguments");
  if (n == 0) return MOE_OK;
  block_map_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, nblocks, block_start, val0, val1, out0, out1);
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}
