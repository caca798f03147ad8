// Calibration kernels: K7 Hessian accumulation (build_hessian,
// quant.py:327-343), K8 the compensated column loop of hessian_quantize
// (quant.py:415-434) in strict reference order, and the Frobenius-loss
// reduction used by quant_loss / search_smoothing (quant.py:267-311).
#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace moe {

// ── K7: H += 2 * xs^T xs (upper-triangle tiles, float64 SIMT) ──────────────
constexpr int kHT = 64;  // output tile
constexpr int kHK = 16;  // tokens per smem stage

__global__ void __launch_bounds__(256) hessian_accum_kernel(const void* x, int dt, int64_t T, int64_t n,
                                                            int64_t ldx, const double* s, const double* rs,
                                                            double* H, unsigned long long* nonzero) {
  // map the linear block id onto an upper-triangle tile (bi <= bj)
  const int nt = (int)((n + kHT - 1) / kHT);
  int b = blockIdx.x, bi = 0;
  while (b >= nt - bi) {
    b -= nt - bi;
    ++bi;
  }
  const int bj = bi + b;
  __shared__ double xa[kHK][kHT + 1];
  __shared__ double xb[kHK][kHT + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // 16x16 threads, 4x4 outputs each
  double acc[4][4] = {};
  unsigned long long nz = 0;
  for (int64_t t0 = 0; t0 < T; t0 += kHK) {
    for (int i = threadIdx.x; i < kHK * kHT; i += blockDim.x) {
      const int tt = i / kHT, c = i % kHT;
      const int64_t t = t0 + tt;
      const int64_t ca = (int64_t)bi * kHT + c, cb = (int64_t)bj * kHT + c;
      double va = 0.0, vb = 0.0;
      if (t < T && ca < n) {
        va = load_as_f64(x, t * ldx + ca, dt);
        if (s) va = rs ? div_rcp(va, s[ca], rs[ca]) : __ddiv_rn(va, s[ca]);
        if (bi == bj) nz += (va != 0.0);
      }
      if (t < T && cb < n) {
        vb = load_as_f64(x, t * ldx + cb, dt);
        if (s) vb = rs ? div_rcp(vb, s[cb], rs[cb]) : __ddiv_rn(vb, s[cb]);
      }
      xa[tt][c] = va;
      xb[tt][c] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kHK; ++k) {
      double a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = xa[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = xb[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = (int64_t)bi * kHT + ty * 4 + i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = (int64_t)bj * kHT + tx * 4 + j;
      if (r < n && c < n && (bi != bj || c >= r)) H[r * n + c] += 2.0 * acc[i][j];
    }
  }
  if (nonzero && nz) atomicAdd(nonzero, nz);
}

// ── K7 on the FP64 tensor cores (DMMA m8n8k4) ───────────────────────────────
// 128 x 128 upper-triangle tiles of H, 8 warps as 4 (rows) x 2 (columns),
// each warp 32 x 64 = 4 x 8 DMMA tiles (64 float64 accumulators per
// thread). Tokens stream through double-buffered shared-memory stages of 16
// (x / s applied on the load, exactly as the SIMT kernel does); rows of a
// stage are padded to 136 doubles so the fragment loads of a warp (4 token
// rows x 8 channels) take the minimum two wavefronts.
constexpr int kHD = 128;           // output tile
constexpr int kHDK = 16;           // tokens per stage
constexpr int kHDLd = kHD + 8;     // padded row (doubles)
constexpr int kHDSmem = 2 * 2 * kHDK * kHDLd * (int)sizeof(double);   // 2 stages x (a, b)

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) hessian_dmma_kernel(const void* x, int dt, int64_t T, int64_t n, int64_t ldx,
                                                           const double* s, const double* rs, double* H,
                                                           unsigned long long* nonzero) {
  extern __shared__ __align__(16) double hsm[];
  const int nt = (int)((n + kHD - 1) / kHD);
  int b = blockIdx.x, bi = 0;
  while (b >= nt - bi) {
    b -= nt - bi;
    ++bi;
  }
  const int bj = bi + b;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp >> 1, wn = warp & 1;             // 4 x 2 warps: rows 32 wm.., cols 64 wn..
  const int gid = lane >> 2, tig = lane & 3;
  double acc[4][8][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  unsigned long long nz = 0;
  auto stage_a = [&](int st) { return hsm + (size_t)st * 2 * kHDK * kHDLd; };
  auto stage_b = [&](int st) { return hsm + (size_t)st * 2 * kHDK * kHDLd + kHDK * kHDLd; };
  // a stage's elements go through registers: the global loads of stage
  // ks + 1 are issued before the DMMAs of stage ks and only consumed
  // (smoothing division, shared-memory store) after them
  constexpr int kPer = kHDK * kHD / 256;               // elements per thread per operand
  double ra[kPer], rb[kPer];
  auto fetch = [&](int64_t t0) {
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int i = threadIdx.x + q * 256;
      const int tt = i / kHD, c = i % kHD;
      const int64_t t = t0 + tt;
      const int64_t ca = (int64_t)bi * kHD + c, cb = (int64_t)bj * kHD + c;
      ra[q] = (t < T && ca < n) ? load_as_f64(x, t * ldx + ca, dt) : 0.0;
      rb[q] = (bi != bj && t < T && cb < n) ? load_as_f64(x, t * ldx + cb, dt) : 0.0;
    }
  };
  auto commit = [&](int st) {
    double* xa = stage_a(st);
    double* xb = stage_b(st);
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int i = threadIdx.x + q * 256;
      const int tt = i / kHD, c = i % kHD;
      const int64_t ca = (int64_t)bi * kHD + c, cb = (int64_t)bj * kHD + c;
      double va = ra[q], vb = rb[q];
      if (s && ca < n) va = rs ? div_rcp(va, s[ca], rs[ca]) : __ddiv_rn(va, s[ca]);
      if (bi == bj) {
        nz += (va != 0.0);
        vb = va;
      } else if (s && cb < n) {
        vb = rs ? div_rcp(vb, s[cb], rs[cb]) : __ddiv_rn(vb, s[cb]);
      }
      xa[tt * kHDLd + c] = va;
      xb[tt * kHDLd + c] = vb;
    }
  };
  const int nst = (int)((T + kHDK - 1) / kHDK);
  fetch(0);
  commit(0);
  __syncthreads();
  for (int ks = 0; ks < nst; ++ks) {
    const int cur = ks & 1;
    if (ks + 1 < nst) fetch((int64_t)(ks + 1) * kHDK);
    const double* xa = stage_a(cur);
    const double* xb = stage_b(cur);
#pragma unroll
    for (int k0 = 0; k0 < kHDK; k0 += 4) {
      double af[4], bf[8];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = xa[(k0 + tig) * kHDLd + wm * 32 + i * 8 + gid];
#pragma unroll
      for (int j = 0; j < 8; ++j) bf[j] = xb[(k0 + tig) * kHDLd + wn * 64 + j * 8 + gid];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (ks + 1 < nst) commit(cur ^ 1);
    __syncthreads();
  }
  // D fragment: element (gid, 2 tig + e) of each 8 x 8 tile
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = (int64_t)bi * kHD + wm * 32 + i * 8 + gid;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t c = (int64_t)bj * kHD + wn * 64 + j * 8 + 2 * tig + e;
        if (r < n && c < n && (bi != bj || c >= r)) H[r * n + c] += 2.0 * acc[i][j][e];
      }
    }
  }
  if (nonzero && nz) atomicAdd(nonzero, nz);
}

// mirror the upper triangle, add damping * mean(diag) (deterministic mean)
__global__ void hessian_diag_mean_kernel(const double* H, int64_t n, double* mean_out) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += H[i * n + i];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if ((int)threadIdx.x < st) sh[threadIdx.x] += sh[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) *mean_out = sh[0] / (double)n;
}

__global__ void hessian_finalize_kernel(double* H, int64_t n, double damping, const double* mean) {
  const double lam = damping * (*mean);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / n, c = i % n;
    if (r > c) H[i] = H[c * n + r];
    else if (r == c) H[i] += lam;
  }
}

// ── K8: left-looking strict-order GPTQ column loop ─────────────────────────
// Each weight row is owned by kGP lanes (below). For column tile [J, J+32):
// start from the original weights, apply the updates of columns i < J in
// ascending i (err_i read from the workspace, U[i, J:J+32] staged in shared
// memory), then run the in-tile sequential loop. Per element the subtractions happen in
// exactly the reference's order, so codes are bit-identical.
constexpr int kGT = 32;      // columns per tile
#ifndef MOE_GPTQ_STAGE
#define MOE_GPTQ_STAGE 32
#endif
constexpr int kGStage = MOE_GPTQ_STAGE;   // U rows per shared-memory stage (double-buffered)

// Each row is owned by kGP adjacent lanes, lane p holding the contiguous
// tile columns [p * kGQ, (p + 1) * kGQ): the left-looking updates of a tile
// are split kGP ways, and in the in-tile sequential part the owner of column
// i computes its code and error and shuffles the error to the row's other
// lanes. Every element still receives its updates one at a time, separate
// multiply and subtract, in ascending column order (quant.py:425-430), so
// the codes equal the reference's bit for bit.

__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// lanes per row kGP (lane p owns tile columns [p * kGQ, (p + 1) * kGQ)), staged
// U rows kGS, threads per CTA NT (rows per CTA = NT / kGP share every staged U chunk)
template <int kGP, int kGS, int NT>
__global__ void __launch_bounds__(NT) gptq_columns_kernel(const double* W, int64_t R, int64_t n, int64_t ldw,
                                                                  const int32_t* order, const double* U,
                                                                  const double* scale, const int32_t* zp, int qmax,
                                                                  uint8_t* codes, int64_t ldc, double* err) {
  constexpr int kGRowsCta = NT / kGP;                    // rows per CTA
  constexpr int kGQ = kGT / kGP;                         // tile columns per lane
  constexpr int kGU = kGS;
  extern __shared__ __align__(16) double gsm[];
  auto us = reinterpret_cast<double (*)[kGU][kGT]>(gsm);                        // [2][kGU][kGT] U rows (double-buffered)
  auto es = reinterpret_cast<double (*)[kGU][kGRowsCta]>(gsm + 2 * kGU * kGT);  // [2][kGU][rows] errors
  auto ut = reinterpret_cast<double (*)[kGT + 1]>(gsm + 2 * kGU * kGT + 2 * kGU * kGRowsCta);
  const int lane = threadIdx.x & 31;
  const int p = threadIdx.x % kGP;                       // column block of this lane
  const int rl = threadIdx.x / kGP;                      // row within the CTA
  const int64_t r0 = (int64_t)blockIdx.x * kGRowsCta;
  const int64_t r = r0 + rl;
  const unsigned group = (lane / kGP) * kGP;             // first lane of this row's group
  const bool valid = r < R;
  const double sc = valid ? scale[r] : 1.0;
  const double rsc = __drcp_rn(sc);
  const int z = valid ? zp[r] : 0;
  for (int64_t J = 0; J < n; J += kGT) {
    const int tw = (int)((n - J) < kGT ? (n - J) : kGT);
    double w[kGQ];
#pragma unroll
    for (int q = 0; q < kGQ; ++q) {
      const int j = p * kGQ + q;
      const int64_t col = J + j;
      w[q] = (valid && j < tw) ? W[r * ldw + (order ? (int64_t)order[col] : col)] : 0.0;
    }
    // updates from all previous columns, ascending; the next chunk of U rows
    // and errors streams in (cp.async) while this one is applied
    auto stage = [&](int64_t i0, int buf) {
      const int ni = (int)((J - i0) < kGU ? (J - i0) : kGU);
      for (int t = threadIdx.x; t < kGU * kGT; t += NT) {
        const int ii = t / kGT, jj = t % kGT;
        const bool ok = ii < ni && jj < tw;
        cp_async8(&us[buf][ii][jj], ok ? U + (i0 + ii) * n + J + jj : U, ok);
      }
      for (int t = threadIdx.x; t < kGU * kGRowsCta; t += NT) {
        const int ii = t / kGRowsCta, rr = t % kGRowsCta;
        const bool ok = ii < ni && r0 + rr < R;
        cp_async8(&es[buf][ii][rr], ok ? err + (i0 + ii) * R + r0 + rr : err, ok);
      }
      cp_async_commit();
    };
    if (J > 0) stage(0, 0);
    int buf = 0;
    for (int64_t i0 = 0; i0 < J; i0 += kGU, buf ^= 1) {
      const int ni = (int)((J - i0) < kGU ? (J - i0) : kGU);
      if (i0 + kGU < J) {
        stage(i0 + kGU, buf ^ 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
#pragma unroll 4
      for (int ii = 0; ii < ni; ++ii) {
        const double e = es[buf][ii][rl];
        const double* u = &us[buf][ii][p * kGQ];
        if constexpr (kGQ % 2 == 0) {
#pragma unroll
          for (int q = 0; q < kGQ; q += 2) {
            const double2 v = *reinterpret_cast<const double2*>(u + q);
            w[q] = __dsub_rn(w[q], __dmul_rn(e, v.x));
            w[q + 1] = __dsub_rn(w[q + 1], __dmul_rn(e, v.y));
          }
        } else {
#pragma unroll
          for (int q = 0; q < kGQ; ++q) w[q] = __dsub_rn(w[q], __dmul_rn(e, u[q]));
        }
      }
      __syncthreads();   // this buffer is restaged two chunks later
    }
    // in-tile sequential part
    for (int t = threadIdx.x; t < kGT * kGT; t += NT) {
      const int ii = t / kGT, jj = t % kGT;
      ut[ii][jj] = (ii < tw && jj < tw) ? U[(J + ii) * n + J + jj] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kGT; ++i) {
      if (i < tw) {
        const int owner = i / kGQ, qi = i % kGQ;
        double e = 0.0;
        if (p == owner) {
          const int c = encode_code(w[qi], sc, rsc, z, qmax);
          const double deq = __dmul_rn((double)(c - z), sc);
          e = __ddiv_rn(__dsub_rn(w[qi], deq), ut[i][i]);
          if (valid) {
            err[(J + i) * R + r] = e;
            const int64_t col = J + i;
            codes[r * ldc + (order ? (int64_t)order[col] : col)] = (uint8_t)c;
          }
        }
        e = __shfl_sync(0xffffffffu, e, (int)group + owner);
#pragma unroll
        for (int q = 0; q < kGQ; ++q) {
          const int j = p * kGQ + q;
          if (j > i) w[q] = __dsub_rn(w[q], __dmul_rn(e, ut[i][j]));
        }
      }
    }
    __syncthreads();   // ut and the error columns of this tile are complete before the next tile
  }
}

// ── Frobenius loss on exact accumulators ───────────────────────────────────
__global__ void __launch_bounds__(256) sq_error_partial_kernel(const int32_t* acc, int64_t M, int64_t N,
                                                               const double* sa, int sa_stride, const double* sw,
                                                               const double* ref, double* partial) {
  __shared__ double sh[256];
  double s = 0.0;
  const int64_t total = M * N;
  const int64_t per = (total + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * per, hi = min(total, lo + per);
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const int64_t m = i / N, c = i % N;
    const double y = __dmul_rn(__dmul_rn(sa[m * sa_stride], sw[c]), (double)acc[i]);
    const double d = __dsub_rn(y, ref[i]);
    s = fma(d, d, s);
  }
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if ((int)threadIdx.x < st) sh[threadIdx.x] += sh[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

__global__ void sq_error_final_kernel(const double* partial, int nparts, double* out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < nparts; ++i) s += partial[i];
    *out = s;
  }
}

constexpr int kSqParts = 512;

}  // namespace moe

using namespace moe;

extern "C" moe_status moe_hessian_accum(const void* x, int x_dtype, int64_t T, int64_t n, int64_t ldx,
                                        const double* smooth, const double* smooth_recip, double* H,
                                        unsigned long long* nonzero_count, moe_stream_t stream) {
  MOE_REQUIRE(x && H && T >= 1 && n >= 1 && ldx >= n, "hessian_accum: bad arguments");
  static const bool simt = getenv("MOE_B200_K7_SIMT") != nullptr;   // A/B against the SIMT kernel
  if (!simt && n >= 256) {
    const int64_t nt = (n + kHD - 1) / kHD;
    const int64_t blocks = nt * (nt + 1) / 2;
    MOE_REQUIRE(blocks < (1LL << 31), "hessian_accum: n too large");
    MOE_CUDA_TRY(set_max_smem_once(reinterpret_cast<const void*>(hessian_dmma_kernel), kHDSmem));
    hessian_dmma_kernel<<<(unsigned)blocks, 256, kHDSmem, as_stream(stream)>>>(x, x_dtype, T, n, ldx, smooth,
                                                                                smooth_recip, H, nonzero_count);
    ::moe::count_launch();
    MOE_LAUNCH_CHECK();
    return MOE_OK;
  }
  const int64_t nt = (n + kHT - 1) / kHT;
  const int64_t blocks = nt * (nt + 1) / 2;
  MOE_REQUIRE(blocks < (1LL << 31), "hessian_accum: n too large");
  hessian_accum_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(x, x_dtype, T, n, ldx, smooth, smooth_recip,
                                                                         H, nonzero_count); ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" moe_status moe_hessian_finalize(double* H, int64_t n, double damping_fraction,
                                           const unsigned long long* nonzero_count, moe_stream_t stream) {
  MOE_REQUIRE(H && n >= 1, "hessian_finalize: bad arguments");
  MOE_REQUIRE(damping_fraction >= 0.0, "damping_fraction must be >= 0");
  cudaStream_t s = as_stream(stream);
  if (nonzero_count) {
    unsigned long long nz = 0;
    MOE_CUDA_TRY(cudaMemcpyAsync(&nz, nonzero_count, sizeof(nz), cudaMemcpyDeviceToHost, s));
    MOE_CUDA_TRY(cudaStreamSynchronize(s));
    if (nz == 0) {
      set_error("calibration activations are all zero");
      return MOE_EDEGENERATE;
    }
  }
  double* mean = nullptr;
  MOE_CUDA_TRY(cudaMallocAsync(&mean, sizeof(double), s));
  hessian_diag_mean_kernel<<<1, 256, 0, s>>>(H, n, mean); ::moe::count_launch();
  int64_t blocks = (n * n + 255) / 256;
  if (blocks > num_sms() * 32) blocks = num_sms() * 32;
  hessian_finalize_kernel<<<(unsigned)blocks, 256, 0, s>>>(H, n, damping_fraction, mean); ::moe::count_launch();
  MOE_CUDA_TRY(cudaFreeAsync(mean, s));
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

// first column i whose factor diagonal U[i, i] is not a positive finite
// number (a U that did not come from a successful Cholesky)
__global__ void factor_diag_check_kernel(const double* U, int64_t n, unsigned long long* first) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = U[i * n + i];
    if (!(d > 0.0) || isinf(d)) atomicMin(first, (unsigned long long)i);
  }
}

extern "C" int64_t moe_gptq_workspace(int64_t R, int64_t n) { return R * n * (int64_t)sizeof(double); }

extern "C" moe_status moe_gptq_columns(const double* W, int64_t R, int64_t n, int64_t ldw, const int32_t* order,
                                       const double* U, const double* scale, const int32_t* zp, int bits,
                                       uint8_t* codes, int64_t ldc, void* err_ws, int64_t err_ws_bytes,
                                       moe_stream_t stream) {
  MOE_REQUIRE(W && U && scale && zp && codes && err_ws, "gptq_columns: null pointer");
  MOE_REQUIRE(R >= 1 && n >= 1 && ldw >= n && ldc >= n, "gptq_columns: bad shape");
  MOE_REQUIRE(bits >= 2 && bits <= 8, "bits must be in [2, 8]");
  MOE_REQUIRE(err_ws_bytes >= moe_gptq_workspace(R, n), "gptq_columns: workspace too small");
  {
    // the column loop divides by U[i, i] (quant.py:428): a factor with a
    // non-positive diagonal is reported as numkit.cholesky would report it
    // (NotPositiveDefiniteError(pivot, value), numkit.py:89-90)
    cudaStream_t s0 = as_stream(stream);
    unsigned long long* first = nullptr;
    MOE_CUDA_TRY(cudaMallocAsync(&first, sizeof(unsigned long long), s0));
    MOE_CUDA_TRY(cudaMemsetAsync(first, 0xFF, sizeof(unsigned long long), s0));
    factor_diag_check_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 256), 256, 0, s0>>>(U, n, first);
    ::moe::count_launch();
    unsigned long long bad = 0;
    MOE_CUDA_TRY(cudaMemcpyAsync(&bad, first, sizeof(bad), cudaMemcpyDeviceToHost, s0));
    MOE_CUDA_TRY(cudaFreeAsync(first, s0));
    MOE_CUDA_TRY(cudaStreamSynchronize(s0));
    if (bad != ~0ull) {
      double v = 0.0;
      MOE_CUDA_TRY(cudaMemcpy(&v, U + (int64_t)bad * n + (int64_t)bad, sizeof(double), cudaMemcpyDeviceToHost));
      set_error_detail((int64_t)bad, v);
      set_error("gptq_columns: factor diagonal U[" + std::to_string(bad) + ", " + std::to_string(bad) +
                "] is not positive");
      return MOE_ENOTPD;
    }
  }
  static const int env_p = getenv("MOE_B200_GPTQ_P") ? atoi(getenv("MOE_B200_GPTQ_P")) : 0;
  const int64_t knob = tune_value(MOE_TUNE_GPTQ_LANES);
  const int forced = knob ? (int)knob : env_p;
  MOE_REQUIRE(forced == 0 || forced == 8 || forced == 16 || forced == 32,
              "gptq_columns: lanes per row must be 8, 16 or 32");
  // 16 lanes per row (2 columns each) and 256-thread CTAs (16 rows share every
  // staged U chunk). tools/k8_ab.py, seeded, best of 3: stacked W1||W3
  // [28672, 4096] 94-99 ms (8 lanes 137-160, 32 lanes 120-135); W2
  // [4096, 14336] 184-186 ms (32 lanes 221-257, 8 lanes 293-527); 128- and
  // 512-thread CTAs within 10 %.
  const int P = forced ? forced : 16;
  static const int env_nt = getenv("MOE_B200_GPTQ_NT") ? atoi(getenv("MOE_B200_GPTQ_NT")) : 0;
  const int NT = env_nt == 128 || env_nt == 256 || env_nt == 512 ? env_nt : 256;
  auto launch = [&](auto kern, int threads, int rows_cta) -> cudaError_t {
    const unsigned blocks = (unsigned)((R + rows_cta - 1) / rows_cta);
    const int smem = (int)sizeof(double) * (2 * kGStage * kGT + 2 * kGStage * rows_cta + kGT * (kGT + 1));
    const cudaError_t e = set_max_smem_once(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    kern<<<blocks, threads, smem, as_stream(stream)>>>(W, R, n, ldw, order, U, scale, zp, (1 << bits) - 1, codes, ldc,
                                                       static_cast<double*>(err_ws));
    return cudaGetLastError();
  };
  auto go = [&](auto nt) -> cudaError_t {
    constexpr int T_ = decltype(nt)::value;
    return P == 32   ? launch(gptq_columns_kernel<32, kGStage, T_>, T_, T_ / 32)
           : P == 16 ? launch(gptq_columns_kernel<16, kGStage, T_>, T_, T_ / 16)
                     : launch(gptq_columns_kernel<8, kGStage, T_>, T_, T_ / 8);
  };
  MOE_CUDA_TRY(NT == 512 ? go(std::integral_constant<int, 512>{})
               : NT == 256 ? go(std::integral_constant<int, 256>{})
                           : go(std::integral_constant<int, 128>{}));
  ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}

extern "C" int64_t moe_quant_sq_error_workspace(int64_t M, int64_t N) {
  (void)M;
  (void)N;
  return kSqParts * (int64_t)sizeof(double);
}

extern "C" moe_status moe_quant_sq_error(const int32_t* acc, int64_t M, int64_t N, const double* a_scale,
                                         int a_scale_stride, const double* w_scale, const double* ref, double* out,
                                         void* workspace, int64_t workspace_bytes, moe_stream_t stream) {
  MOE_REQUIRE(acc && a_scale && w_scale && ref && out && M >= 1 && N >= 1, "quant_sq_error: bad arguments");
  MOE_REQUIRE(workspace && workspace_bytes >= moe_quant_sq_error_workspace(M, N), "quant_sq_error: workspace");
  cudaStream_t s = as_stream(stream);
  double* part = static_cast<double*>(workspace);
  sq_error_partial_kernel<<<kSqParts, 256, 0, s>>>(acc, M, N, a_scale, a_scale_stride, w_scale, ref, part); ::moe::count_launch();
  sq_error_final_kernel<<<1, 32, 0, s>>>(part, kSqParts, out); ::moe::count_launch();
  MOE_LAUNCH_CHECK();
  return MOE_OK;
}
