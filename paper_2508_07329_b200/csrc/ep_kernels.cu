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

__global__ void unpack_params_kernel(const int4* params, const int32_t* index, int64_t n, const int32_t* n_dev,
                                     float* scale, int32_t* zp, int32_t* rowsum, float* weight) {
  if (n_dev) n = min(n, (int64_t)*n_dev);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 p = params[index ? index[i] : i];
    scale[i] = __int_as_float(p.x);
    zp[i] = p.y;
    rowsum[i] = p.z;
    if (weight) weight[i] = __int_as_float(p.w);
  }
}

// rows grouped in contiguous blocks [start[b], start[b+1]): out0[i] = val0[b],
// out1[i] = val1[b] + (i - start[b]), out2[i] = val2[b] (optional), for
// i < n (or i < *n_dev when given; binary search over nb blocks). With
// `valid` given and *valid == 0 every out0 is -1 (a refused exchange plan:
// consumers skip such rows instead of writing anywhere).
constexpr int kMapSmemBlocks = 4096;   // block tables up to this size are staged in shared memory

__global__ void block_map_kernel(int64_t n, const int32_t* n_dev, int nb, const int32_t* start, const int32_t* val0,
                                 const int32_t* val1, const int32_t* val2, const int32_t* valid, int32_t* out0,
                                 int32_t* out1, int32_t* out2) {
  __shared__ int32_t s_start[kMapSmemBlocks];
  if (n_dev) n = min(n, (int64_t)*n_dev);
  const bool ok = !valid || *valid != 0;
  // the binary search runs over a shared-memory copy of the block starts
  // (a chain of dependent global loads per row otherwise)
  const bool staged = nb <= kMapSmemBlocks;
  if (staged)
    for (int b = threadIdx.x; b < nb; b += blockDim.x) s_start[b] = start[b];
  __syncthreads();
  const int32_t* st = staged ? s_start : start;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = nb;   // last b with start[b] <= i
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (st[mid] <= i) lo = mid;
      else hi = mid;
    }
    out0[i] = ok ? val0[lo] : -1;
    out1[i] = val1[lo] + (int32_t)(i - st[lo]);
    if (out2) out2[i] = val2[lo];
  }
}

// ── device-side exchange plan of the peer-memory EP forward ───────────────
// offs[s] = rank s's route_permute offsets over its W*E sort keys (key
// r*E + e = rows of s for expert e served by rank r), gathered from every
// rank: C[s][r][e] = offs[s][key+1] - offs[s][key]. Every receive buffer is
// expert-major, sender-minor. Writes (int32):
//   plan[0]            1 = plan valid, 0 = refused (buffer overflow or rows
//                      for an expert this rank does not hold)
//   plan[1]            R = rows this rank receives
//   send_base[W*E]     first receive-buffer row of this rank's block for key
//   starts[G*W+1], ranks[G*W], homes[G*W], group[G*W]: receive blocks
//                      (local expert g ascending, sender s), each block's
//                      home rank / first home row / local expert index
//   goff[G+1]          grouped-GEMM offsets of the local experts
// Single CTA; W*E <= 4096 keys.
__global__ void ep_peer_plan_kernel(const int32_t* offs, int W, int E, int me, const int32_t* local, int G,
                                    int64_t cap, int64_t cap_home, int32_t* plan, volatile int32_t* host_flag) {
  __shared__ int bad;
  __shared__ int32_t s_offs[3072];   // every rank's offsets, when they fit (W * (W*E + 1) ints)
  const int KE = W * E, ld = KE + 1;
  const bool staged = W * ld <= 3072;
  if (staged)
    for (int i = threadIdx.x; i < W * ld; i += blockDim.x) s_offs[i] = offs[i];
  __syncthreads();
  const int32_t* o = staged ? s_offs : offs;
  auto C = [&](int s, int r, int e) { return o[s * ld + r * E + e + 1] - o[s * ld + r * E + e]; };
  int32_t* send_base = plan + 2;
  int32_t* starts = send_base + KE;
  int32_t* ranks = starts + G * W + 1;
  int32_t* homes = ranks + G * W;
  int32_t* group = homes + G * W;
  int32_t* goff = group + G * W;
  __shared__ int32_t tot[4096];   // rows of all senders for key (r, e)
  __shared__ int32_t pre[4096];   // rows of senders before `me` for key (r, e)
  if (threadIdx.x == 0) bad = 0;
  for (int key = threadIdx.x; key < KE; key += blockDim.x) {
    const int r = key / E, e = key % E;
    int32_t t = 0, b = 0;
    for (int s = 0; s < W; ++s) {
      const int32_t c = C(s, r, e);
      t += c;
      if (s < me) b += c;
    }
    tot[key] = t;
    pre[key] = b;
  }
  __syncthreads();
  // sender side: receiver r's buffer is expert-major, sender-minor
  for (int r = threadIdx.x; r < W; r += blockDim.x) {
    int32_t run = 0;
    for (int e = 0; e < E; ++e) {
      send_base[r * E + e] = run + pre[r * E + e];
      run += tot[r * E + e];
    }
  }
  // capacity checks (every rank evaluates the same global counts)
  for (int r = threadIdx.x; r < W; r += blockDim.x) {
    int64_t recv = 0, home = 0;
    for (int s = 0; s < W; ++s)
      for (int e = 0; e < E; ++e) recv += C(s, r, e);
    home = o[r * ld + KE] - o[r * ld];
    if (recv > cap || home > cap_home) atomicOr(&bad, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // rows for an expert this rank does not hold
    for (int e = 0; e < E; ++e) {
      bool mine = false;
      for (int g = 0; g < G; ++g) mine |= local[g] == e;
      if (!mine)
        for (int s = 0; s < W; ++s) if (C(s, me, e) != 0) bad = 1;
    }
    int64_t pos = 0;
    for (int g = 0; g < G; ++g) {
      goff[g] = (int32_t)pos;
      const int e = local[g];
      for (int s = 0; s < W; ++s) {
        const int b = g * W + s;
        starts[b] = (int32_t)pos;
        ranks[b] = s;
        homes[b] = o[s * ld + me * E + e];
        group[b] = g;
        pos += C(s, me, e);
      }
    }
    if (bad) pos = 0;
    starts[G * W] = (int32_t)pos;
    goff[G] = (int32_t)pos;
    if (bad) for (int g = 0; g < G; ++g) goff[g] = 0;
    plan[0] = bad ? 0 : 1;
    plan[1] = (int32_t)pos;
    if (host_flag) *host_flag = bad ? 0 : 1;   // mapped pinned memory: no copy-engine transfer
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

extern "C" moe_status moe_ep_unpack_params(const int32_t* params, const int32_t* index, int64_t n, const int32_t* n_dev,
                                           float* scale_f32, int32_t* zp, int32_t* rowsum, float* weight,
                                           moe_stream_t stream) {
  MOE_REQUIRE(params && scale_f32 && zp && rowsum && n >= 0, "ep_unpack_params: bad arguments");
  MOE_REQUIRE((reinterpret_cast<uintptr_t>(params) & 15) == 0, "ep_unpack_params: params must be 16-byte aligned");
  if (n == 0) return MOE_OK;
  unpack_params_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(reinterpret_cast<const int4*>(params), index,
                                                                         n, n_dev, scale_f32, zp, rowsum, weight);
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" int64_t moe_ep_peer_plan_size(int W, int E, int G) {
  return 2 + (int64_t)W * E + 4 * (int64_t)G * W + 1 + G + 1;
}

extern "C" moe_status moe_ep_peer_plan(const int32_t* offsets_all, int W, int E, int me, const int32_t* local,
                                       int G, int64_t cap, int64_t cap_home, int32_t* plan, int32_t* host_flag,
                                       moe_stream_t stream) {
  MOE_REQUIRE(offsets_all && plan && (local || G == 0), "ep_peer_plan: null pointer");
  MOE_REQUIRE(W >= 1 && E >= 1 && W * E <= 4096 && me >= 0 && me < W && G >= 0 && G <= E,
              "ep_peer_plan: bad sizes");
  int32_t* hflag = nullptr;
  if (host_flag) {
    void* dp = nullptr;
    MOE_REQUIRE(cudaHostGetDevicePointer(&dp, host_flag, 0) == cudaSuccess,
                "ep_peer_plan: host_flag must be pinned (mapped) host memory");
    hflag = static_cast<int32_t*>(dp);
  }
  ep_peer_plan_kernel<<<1, 256, 0, as_stream(stream)>>>(offsets_all, W, E, me, local, G, cap, cap_home, plan, hflag);
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_block_map(int64_t n, const int32_t* n_dev, int nblocks, const int32_t* block_start,
                                    const int32_t* val0, const int32_t* val1, const int32_t* val2,
                                    const int32_t* valid, int32_t* out0, int32_t* out1, int32_t* out2,
                                    moe_stream_t stream) {
  MOE_REQUIRE(n >= 0 && nblocks >= 1 && block_start && val0 && val1 && out0 && out1, "block_map: bad arguments");
  MOE_REQUIRE(!out2 || val2, "block_map: out2 needs val2");
  if (n == 0) return MOE_OK;
  block_map_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(n, n_dev, nblocks, block_start, val0, val1, val2,
                                                                     valid, out0, out1, out2);
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}
