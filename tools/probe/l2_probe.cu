// L2 sharing probe: pass 1, CTA b reads slice b of the buffer; pass 2, CTA b
// reads slice (b + shift) % nb — i.e. data first pulled through L2 by other
// SMs. With one memory-side L2 (each line cached once, at its home die) the
// second pass hits L2 for buffers that fit 126 MB; if each die caches what
// its own SMs read, the second pass misses for every slice first read on
// the other die. ncu dram__bytes_read of pass 2 tells which.
#include <cstdint>
#include <cuda_runtime.h>

__global__ void probe_pass(const uint4* __restrict__ buf, int64_t slice_vec, int shift, unsigned long long* sink) {
  const int nb = gridDim.x;
  const int b = (blockIdx.x + shift) % nb;
  const uint4* s = buf + (int64_t)b * slice_vec;
  uint32_t acc = 0;
  for (int64_t i = threadIdx.x; i < slice_vec; i += blockDim.x) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(s + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

extern "C" int l2_probe(const void* buf, int64_t bytes, int blocks, int shift, void* sink) {
  const int64_t slice_vec = bytes / 16 / blocks;
  probe_pass<<<blocks, 512>>>(static_cast<const uint4*>(buf), slice_vec, shift,
                              static_cast<unsigned long long*>(sink));
  return (int)cudaGetLastError();
}
