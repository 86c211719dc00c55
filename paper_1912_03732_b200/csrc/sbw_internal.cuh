// Internal helpers shared by the sm_100a kernels of libsbw.
//
// Domain vocabulary follows the reference package `sboxeval`:
//   n, m        S-box input / output widths (pkg/src/sboxeval/sbox.py:51-76)
//   v           output mask, 1 <= v < 2^m (component g_v = parity(v & S(x)))
//   x / u       input index / spectrum index, 0 <= x,u < 2^n
//   W(u, v)     Walsh coefficient sum_x (-1)^{g_v(x) ^ <u,x>}  (walsh.py:56-70)
//   max|W|      per-component maximum over ALL u including u = 0 (walsh.py:101-102)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/sbw.h"

namespace sbw {

// --- error plumbing (sbw_capi.cpp owns the thread-local message) -----------
int set_error(int code, const char* fmt, ...);
int cuda_error(cudaError_t e, const char* what);
void count_launch(uint64_t k = 1);

#define SBW_CUDA_CHECK(expr)                                  \
  do {                                                        \
    cudaError_t _e = (expr);                                  \
    if (_e != cudaSuccess) return ::sbw::cuda_error(_e, #expr); \
  } while (0)

#define SBW_LAUNCH_CHECK(what)                                \
  do {                                                        \
    cudaError_t _e = cudaGetLastError();                      \
    if (_e != cudaSuccess) return ::sbw::cuda_error(_e, what); \
    ::sbw::count_launch();                                    \
  } while (0)

struct DeviceProps {
  int device;
  int sm_count;
  size_t smem_optin;
  size_t l2_bytes;
};
int device_props(DeviceProps* out);  // current device, cached

// --- device helpers -------------------------------------------------------

// (-1)^{popc(v & s)}: the +/-1 polarity of component g_v at one input
// (sbox.py:114-116 `_mask_parity`, sbox.py:145-152 `polarity_row`).
__device__ __forceinline__ int polarity(uint32_t s, uint32_t v) {
  return 1 - 2 * int(__popc(s & v) & 1u);
}

// numpy int32 |x| wraps INT_MIN to INT_MIN; keep that semantics for the
// generic column kernel (walsh.py:102 `np.abs(lo).max()` on int32).
__device__ __forceinline__ int wrap_abs(int x) { return x < 0 ? int(0u - uint32_t(x)) : x; }

// Packed key for "largest max|W|, ties -> smallest v" so one atomicMax picks
// the reference's first-argmin component (nonlinearity.py:44, :55).
__device__ __forceinline__ unsigned long long nl_key(int max_abs, uint32_t v) {
  return (static_cast<unsigned long long>(static_cast<uint32_t>(max_abs)) << 32) |
         static_cast<unsigned long long>(0xFFFFFFFFu - v);
}

// In-register Walsh-Hadamard butterflies over e[0..LEN) for strides
// S0, 2*S0, ..., < LEN (natural order, unnormalised; walsh.py:91-100).
template <int LEN, int S0>
__device__ __forceinline__ void fwht_regs(int (&e)[LEN]) {
#pragma unroll
  for (int s = S0; s < LEN; s <<= 1) {
#pragma unroll
    for (int i = 0; i < LEN; ++i) {
      if ((i & s) == 0) {
        const int a = e[i], b = e[i + s];
        e[i] = a + b;
        e[i + s] = a - b;
      }
    }
  }
}

// Same, but stops before the stride `SEND` (exclusive).
template <int LEN, int S0, int SEND>
__device__ __forceinline__ void fwht_regs_until(int (&e)[LEN]) {
#pragma unroll
  for (int s = S0; s < SEND; s <<= 1) {
#pragma unroll
    for (int i = 0; i < LEN; ++i) {
      if ((i & s) == 0) {
        const int a = e[i], b = e[i + s];
        e[i] = a + b;
        e[i + s] = a - b;
      }
    }
  }
}

__device__ __forceinline__ int warp_max(int x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

}  // namespace sbw
