// Multi-pass path for n = 17..24 ("K3"), pass B.
//
// Pass A (k_tile_simd<15, MODE_EMIT>) leaves, for every component of the
// current batch, 2^(n-15) blocks of 2^15 partial transforms (x bits 0..14
// done) in an L2-sized scratch buffer, each as the biased u16
// s = (v + 2^15) / 2 in [0, 2^15]; pass B works on v / 2 = s - 2^14 in int32.  Pass B runs the
// remaining H = n - 15 stages over x bits 15..n-1, i.e. across blocks, and
// fuses max|W| into the top stage exactly like the on-chip kernel.  The
// reference does all n stages on one numpy array per mask (walsh.py:91-103);
// stage order is free because the butterflies of different bits commute.
//
//   H <= 5: registers only; a thread owns one int16 pair column of 2^H rows.
//   H  > 5: a CTA stages a [2^H rows x 64 x] int32 tile in shared memory and
//           runs two register passes over it.
#pragma once

#include "sbw_tile_simd.cuh"

namespace sbw {

struct PassBArgs {
  const uint32_t* scratch;   // int16 pairs: [comp][2^n] halved values
  int n;
  int64_t n_comp;            // components in this batch
  int64_t out_row0;          // index of this batch's first component in max_abs / out
  uint32_t v_first;          // mask of this batch's first component
  int32_t* max_abs;          // zero-initialised by the host for the batch
  unsigned long long* key;
  int32_t* out;              // materialised rows (may be null)
  int64_t ld;
};

constexpr int kPassBThreads = 256;

__device__ __forceinline__ int lo_half(uint32_t u) { return int(u & 0xFFFFu) - 16384; }
__device__ __forceinline__ int hi_half(uint32_t u) { return int(u >> 16) - 16384; }

// Reduce a per-thread partial max over the CTA and publish it (all threads of
// a CTA belong to the same component by construction).
__device__ __forceinline__ void cta_publish_max(int mx, int* s_red, int32_t* slot,
                                                unsigned long long* key, uint32_t v) {
  mx = warp_max(mx);
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) s_red[warp] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    int m = 0;
    for (int w = 0; w < nw; ++w) m = max(m, s_red[w]);
    atomicMax(slot, m);
    if (key) atomicMax(key, nl_key(m, v));
  }
  __syncthreads();
}

// H <= 5.  Grid: one CTA per (component, chunk of 256 pair-columns).
template <int H, int MODE>
__global__ void __launch_bounds__(kPassBThreads) k_passb_regs(PassBArgs a) {
  constexpr int NI = 1 << H;
  __shared__ int s_red[kPassBThreads / 32];
  const int64_t cols = int64_t(1) << 14;                   // pair-columns per component
  const int64_t chunks = cols / kPassBThreads;
  for (int64_t b = blockIdx.x; b < a.n_comp * chunks; b += gridDim.x) {
    const int64_t comp = b / chunks;
    const int64_t col = (b % chunks) * kPassBThreads + threadIdx.x;
    const uint32_t* src = a.scratch + (comp << (a.n - 1)) + col;
    int e[2 * NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const uint32_t u = __ldcs(src + (int64_t(i) << 14));
      e[2 * i] = lo_half(u);
      e[2 * i + 1] = hi_half(u);
    }
    fwht_regs_until<2 * NI, 2, NI>(e);
    int mx = 0;
    if constexpr (MODE == MODE_NL) {
#pragma unroll
      for (int k = 0; k < NI; ++k) mx = max(mx, abs(e[k]) + abs(e[k + NI]));
      mx *= 2;  // values are halved
    } else {
#pragma unroll
      for (int k = 0; k < NI; ++k) {
        const int p = e[k], q = e[k + NI];
        e[k] = 2 * (p + q);
        e[k + NI] = 2 * (p - q);
        mx = max(mx, max(abs(e[k]), abs(e[k + NI])));
      }
      int32_t* dst = a.out + (a.out_row0 + comp) * a.ld + 2 * col;
#pragma unroll
      for (int i = 0; i < NI; ++i) {
        dst[int64_t(i) << 15] = e[2 * i];
        dst[(int64_t(i) << 15) + 1] = e[2 * i + 1];
      }
    }
    cta_publish_max(mx, s_red, a.max_abs + a.out_row0 + comp, a.key,
                    a.v_first + uint32_t(comp));
  }
}

// H = 6..9.  A CTA owns (component, 32 pair-columns) x 2^H rows.  Pass B1
// reads row bits 0..4 straight from the scratch (32 independent coalesced
// loads in flight per thread), runs those 5 stages and parks int32 pairs in
// shared memory; pass B2 runs row bits 5..H-1 with the fused top stage.
template <int H, int MODE>
__global__ void __launch_bounds__(512, 1) k_passb_smem(PassBArgs a) {
  constexpr int H2 = H - 5;
  constexpr int N2 = 1 << H2;
  extern __shared__ int2 tile[];       // [2^H rows][32 columns] int32 pairs
  __shared__ int s_red[16];
  const int64_t chunks = (int64_t(1) << 14) / 32;
  for (int64_t b = blockIdx.x; b < a.n_comp * chunks; b += gridDim.x) {
    const int64_t comp = b / chunks;
    const int64_t col0 = (b % chunks) * 32;
    const uint32_t* src = a.scratch + (comp << (a.n - 1)) + col0;
    // B1: task = (column c, row-high rh); rows (rh << 5) | i
    for (int task = threadIdx.x; task < 32 * N2; task += blockDim.x) {
      const int c = task & 31, rh = task >> 5;
      uint32_t u[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) u[i] = __ldcs(src + (int64_t((rh << 5) | i) << 14) + c);
      int e[64];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        e[2 * i] = lo_half(u[i]);
        e[2 * i + 1] = hi_half(u[i]);
      }
      fwht_regs<64, 2>(e);
#pragma unroll
      for (int i = 0; i < 32; ++i) tile[((rh << 5) | i) * 32 + c] = make_int2(e[2 * i], e[2 * i + 1]);
    }
    __syncthreads();
    // B2: row bits 5..H-1, fused top stage
    int mx = 0;
    for (int task = threadIdx.x; task < 32 * 32; task += blockDim.x) {
      const int c = task & 31, rl = task >> 5;
      int e[2 * N2];
#pragma unroll
      for (int i = 0; i < N2; ++i) {
        const int2 p = tile[((i << 5) | rl) * 32 + c];
        e[2 * i] = p.x;
        e[2 * i + 1] = p.y;
      }
      fwht_regs_until<2 * N2, 2, N2>(e);
      if constexpr (MODE == MODE_NL) {
        int m2 = 0;
#pragma unroll
        for (int k = 0; k < N2; ++k) m2 = max(m2, abs(e[k]) + abs(e[k + N2]));
        mx = max(mx, 2 * m2);
      } else {
#pragma unroll
        for (int k = 0; k < N2; ++k) {
          const int p = e[k], q = e[k + N2];
          e[k] = 2 * (p + q);
          e[k + N2] = 2 * (p - q);
          mx = max(mx, max(abs(e[k]), abs(e[k + N2])));
        }
        int32_t* dst = a.out + (a.out_row0 + comp) * a.ld + 2 * (col0 + c);
#pragma unroll
        for (int i = 0; i < N2; ++i) {
          const int64_t row = (int64_t(i) << 5) | rl;
          dst[row << 15] = e[2 * i];
          dst[(row << 15) + 1] = e[2 * i + 1];
        }
      }
    }
    cta_publish_max(mx, s_red, a.max_abs + a.out_row0 + comp, a.key,
                    a.v_first + uint32_t(comp));
  }
}

}  // namespace sbw
