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

// --- L2 ring hand-off between concurrently running pass A / pass B (K3) ---
// Counters live in global memory; producers release with a gpu-scope fence
// before a relaxed atomicAdd, consumers poll with ld.acquire.gpu.  A wait
// that exceeds ~4 s (the two kernels were not co-resident) raises *err and
// gives up instead of hanging the device; the host turns *err into poisoned
// results (odd gap -> AssertionError in the NL conversion).
//
// Ring layout: batch k = components [k Bc, (k + 1) Bc) of the ring run lives
// in slot k mod R (R slots of Bc components).  Pass A CTA j = r * T + bp owns
// 2^16-block pair bp and components [r L, (r + 1) L) of every batch
// (Bc = q L, q = NA / T); each of its 8 transform warps arrives on ready[k]
// after its last item of batch k.  Pass B CTA j owns items
// [I j / NB, I (j + 1) / NB) of every batch (I = Bc x items per component)
// and arrives on freed[k] once its last TMA load of batch k has landed.
struct RingArgs {
  int on;              // 0: batch mode (no ring)
  int R, L, q, log_t;  // slots, components per pass-A CTA per batch, CTAs per block pair, log2 block pairs
  int64_t batches;     // full batches in the ring run
  int bc;              // components per batch (q L)
  uint32_t na, nb;     // pass A / pass B CTAs
  uint32_t* ready;     // [batches]: pass-A transform-warp arrivals (target 8 na)
  uint32_t* freed;     // [batches]: pass-B CTA arrivals (target nb)
  uint32_t* err;       // co-residency timeout flag
  unsigned long long* wait_ns;  // [2] optional (SBW_K3_TRACE): ns spent waiting in pass A / pass B
  int nowait;          // timing experiments only (SBW_K3_RING_NOWAIT): skip every wait (results invalid)
};

// Mask at natural position q of [v_lo, v_hi): Gray order inside every aligned
// block of 256 masks that lies in the range (consecutive positions differ in
// one mask bit, so generation is one plane XOR), natural order elsewhere.
__device__ __forceinline__ uint32_t mask_at(int64_t q, uint32_t v_lo, uint32_t v_hi) {
  const int64_t b = q & ~int64_t(255);
  if (b >= int64_t(v_lo) && b + 256 <= int64_t(v_hi)) {
    const uint32_t k = uint32_t(q) & 255u;
    return uint32_t(b) | (k ^ (k >> 1));
  }
  return uint32_t(q);
}

// Ring position -> mask.  Pass-A CTA row r walks positions [r K L, (r + 1) K L)
// (K = batches) in order, so its consecutive components are consecutive in
// Gray order; slot r L + l of batch k holds position r K L + k L + l.
__device__ __forceinline__ uint32_t ring_mask(const RingArgs& r, uint32_t v_first, int64_t pos) {
  return mask_at(int64_t(v_first) + pos, v_first, uint32_t(int64_t(v_first) + r.batches * r.bc));
}
__device__ __forceinline__ int64_t ring_pos(const RingArgs& r, int64_t k, int64_t slot_comp) {
  const int64_t row = slot_comp / r.L;
  return row * r.batches * r.L + k * r.L + (slot_comp - row * r.L);
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void ring_wait_geq(const uint32_t* p, uint32_t target, uint32_t* err,
                                              unsigned long long* wait_ns = nullptr) {
  if (ld_acquire_gpu(p) >= target) return;
  const uint64_t t0 = globaltimer_ns();
  uint64_t t = t0;
  while (ld_acquire_gpu(p) < target) {
    if (ld_acquire_gpu(err) != 0u) break;
    t = globaltimer_ns();
    if (t - t0 > 4000000000ull) {
      atomicExch(err, 1u);
      break;
    }
  }
  if (wait_ns) atomicAdd(wait_ns, static_cast<unsigned long long>(t - t0));
}
__device__ __forceinline__ void ring_signal(uint32_t* p) {
  __threadfence();
  atomicAdd(p, 1u);
}

}  // namespace sbw
