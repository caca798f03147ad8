// Library-level C ABI: thread-local error text, ABI version, device check.
#include "common.cuh"

#include <atomic>

namespace moe {
static thread_local std::string g_last_error;
static std::atomic<unsigned long long> g_launches{0};
void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace moe

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
