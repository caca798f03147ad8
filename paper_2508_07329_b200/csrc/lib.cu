// Library-level C ABI: thread-local error text, ABI version, device check.
#include "common.cuh"

#include <atomic>

namespace moe {
static thread_local std::string g_last_error;
static thread_local int64_t g_err_pivot = -1;
static thread_local double g_err_value = 0.0;
void set_error_detail(int64_t pivot, double value) {
  g_err_pivot = pivot;
  g_err_value = value;
}
static std::atomic<unsigned long long> g_launches{0};
void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// process-wide knobs (MOE_TUNE_*), indexed by key
static std::atomic<int64_t> g_tune[MOE_TUNE_COUNT] = {
    {0},
    {[] {
      const char* env = getenv("MOE_B200_K1_SMALL");
      return env ? (int64_t)atoll(env) : (int64_t)256;
    }()},
    {64},   // router cluster tiles: tools/router_bench.py crossover
    {0},    // fused K1 in GEMM2 (off)
    {1},    // fused top-2 combine (on)
    {2},    // K1 on x: 2 token-major walk of the row kernel (146 us), 1 token kernel (182 us), 0 gathered rows
    {0},    // GPTQ lanes per row (0: automatic)
    {[] {
      const char* env = getenv("MOE_B200_BAND_MB");
      return env ? (int64_t)atoll(env) : (int64_t)24;
    }()},   // grouped-GEMM raster band budget (MB of A rows kept L2-resident)
};
int64_t tune_value(int key) { return g_tune[key].load(std::memory_order_relaxed); }
int64_t k1_small_rows() { return tune_value(MOE_TUNE_K1_SMALL_ROWS); }
int64_t router_cluster_tiles() { return tune_value(MOE_TUNE_ROUTER_CLUSTER_TILES); }
}  // namespace moe

extern "C" moe_status moe_tune(int key, int64_t value, int64_t* old) {
  if (key <= 0 || key >= MOE_TUNE_COUNT) {
    moe::set_error("moe_tune: unknown key " + std::to_string(key));
    return MOE_EINVAL;
  }
  const int64_t prev = value < 0 ? moe::g_tune[key].load() : moe::g_tune[key].exchange(value);
  if (old) *old = prev;
  return MOE_OK;
}

extern "C" const char* moe_last_error(void) { return moe::g_last_error.c_str(); }

extern "C" moe_status moe_last_error_detail(int64_t* pivot, double* value) {
  if (pivot) *pivot = moe::g_err_pivot;
  if (value) *value = moe::g_err_value;
  return MOE_OK;
}

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
