// Library-level C ABI: thread-local error text, ABI version, device check.
#include "common.cuh"

#include <atomic>

namespace moe {
static thread_local std::string g_last_error;
static std::atomic<unsigned long long> g_launches{0};
void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static std::atomic<int64_t> g_k1_small_rows{[] {
  const char* env = getenv("MOE_B200_K1_SMALL");
  return env ? (int64_t)atoll(env) : (int64_t)256;
}()};
int64_t k1_small_rows() { return g_k1_small_rows.load(std::memory_order_relaxed); }
static std::atomic<int64_t> g_router_cluster_tiles{64};   // tools/router_bench.py crossover
int64_t router_cluster_tiles() { return g_router_cluster_tiles.load(std::memory_order_relaxed); }
static std::atomic<int64_t> g_fused_quant{0};
static std::atomic<int64_t> g_fused_combine{1};
}  // namespace moe

extern "C" moe_status moe_tune(int key, int64_t value, int64_t* old) {
  switch (key) {
    case MOE_TUNE_K1_SMALL_ROWS: {
      const int64_t prev = value < 0 ? moe::g_k1_small_rows.load() : moe::g_k1_small_rows.exchange(value);
      if (old) *old = prev;
      return MOE_OK;
    }
    case MOE_TUNE_ROUTER_CLUSTER_TILES: {
      const int64_t prev =
          value < 0 ? moe::g_router_cluster_tiles.load() : moe::g_router_cluster_tiles.exchange(value);
      if (old) *old = prev;
      return MOE_OK;
    }
    case MOE_TUNE_FUSED_QUANT: {
      const int64_t prev = value < 0 ? moe::g_fused_quant.load() : moe::g_fused_quant.exchange(value);
      if (old) *old = prev;
      return MOE_OK;
    }
    case MOE_TUNE_FUSED_COMBINE: {
      const int64_t prev = value < 0 ? moe::g_fused_combine.load() : moe::g_fused_combine.exchange(value);
      if (old) *old = prev;
      return MOE_OK;
    }
    default:
      moe::set_error("moe_tune: unknown key " + std::to_string(key));
      return MOE_EINVAL;
  }
}

extern "C" const char* moe_last_error(void) { return moe::g_last_error.c_str(); }

extern "C" uint64_t moe_launch_count(void) { return moe::g_launches.load(); }

extern "C" int moe_abi_version(void) { return 1; }

extern "C" moe_status moe_device_check(int dev) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count <= dev) {
    moe::set_error(std::string("no CUDA device: ") + cudaGetErrorString(e));
    return MOE_ECUDA;
  }
  cudaDeviceProp prop;
  MOE_CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10 || prop.minor != 0) {
    moe::set_error("kernels are built for sm_100a; device is sm_" + std::to_string(prop.major) +
                   std::to_string(prop.minor));
    return MOE_EUNSUPPORTED;
  }
  return MOE_OK;
}
