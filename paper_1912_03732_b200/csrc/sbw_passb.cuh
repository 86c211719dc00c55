// Multi-pass path for n = 17..24 ("K3"), pass B.
//
// Pass A (k_tile_simd<15, MODE_EMIT>, one 1024-thread launch per batch of
// components) leaves, for every component of the batch, 2^(n-15) blocks of
// 2^15 partial transforms (x bits 0..14 done), each as the biased u16
// s = (v + 2^15) / 2 in [0, 2^15].  Pass B runs the remaining H = n - 15
// stages over x bits 15..n-1, i.e. across blocks, on v / 2 = s - 2^14 in
// int32, and fuses max|W| into the top stage like the on-chip kernel.  The
// reference does all n stages on one numpy array per mask (walsh.py:91-103);
// stage order is free because the butterflies of different bits commute.
//
//   H <= 5: k_passb_regs   -- registers only, one thread per pair-column.
//   H >= 6: k_passb_staged -- cp.async-staged [2^H rows x 32 pair-columns]
//           chunks, two register passes through a 128 KiB int32 tile, the
//           next chunk prefetched while the current one computes.
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

// ---- pass-B chunk bodies (called by every thread of the CTA) --------------
// A chunk's u16-pair words are first staged in shared memory by cp.async.cg
// (16-byte pieces, L2 only: the persistent kernel reuses ring slots, so an
// SM's L1 may hold lines of an older component).  Staging is asynchronous, so
// the copy of chunk i+1 overlaps the arithmetic of chunk i.

template <int H, int THREADS>
struct ChunkShape {
  static constexpr int R = 1 << H;                 // rows (x bits 15..n-1)
  static constexpr int CW = H <= 5 ? THREADS : 32; // pair-columns (words) per chunk
  static constexpr int64_t PER_COMP = (int64_t(1) << 14) / CW;
  static constexpr int PIECES = R * CW / 4;        // 16-byte pieces
};

// Issue (not wait for) the copies of chunk `chunk` of a component whose
// scratch starts at `comp_base` into `stg` ([R][CW] words).
template <int H, int THREADS>
__device__ __forceinline__ void stage_chunk(const uint32_t* comp_base, int64_t chunk, uint32_t* stg) {
  using S = ChunkShape<H, THREADS>;
  constexpr int PR = S::CW / 4;  // pieces per row
  const int64_t col0 = chunk * S::CW;
  for (int p = threadIdx.x; p < S::PIECES; p += THREADS) {
    const int r = p / PR, q = p - (p / PR) * PR;
    const uint32_t* g = comp_base + (int64_t(r) << 14) + col0 + 4 * q;
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(stg + r * S::CW + 4 * q));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ __forceinline__ void stage_wait() {
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
}

// H = 6..9: 32 pair-columns x 2^H rows.  B1 runs row bits 0..4 from the
// staging buffer and parks int32 pairs in `tile`; B2 runs row bits 5..H-1
// with the fused top stage.
template <int H, int MODE, typename AfterRead>
__device__ __forceinline__ void passb_smem_chunk(const PassBArgs& a, int64_t comp, int64_t chunk,
                                                 const uint32_t* stg, int2* tile, int* s_red,
                                                 AfterRead after_read) {
  constexpr int H2 = H - 5;
  constexpr int N2 = 1 << H2;
  const int64_t col0 = chunk * 32;
  for (int task = threadIdx.x; task < 32 * N2; task += blockDim.x) {
    const int c = task & 31, rh = task >> 5;
    int e[64];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const uint32_t u = stg[((rh << 5) | i) * 32 + c];
      e[2 * i] = lo_half(u);
      e[2 * i + 1] = hi_half(u);
    }
    fwht_regs<64, 2>(e);
#pragma unroll
    for (int i = 0; i < 32; ++i) tile[((rh << 5) | i) * 32 + c] = make_int2(e[2 * i], e[2 * i + 1]);
  }
  __syncthreads();
  after_read();
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
        *reinterpret_cast<int2*>(dst + (row << 15)) = make_int2(e[2 * i], e[2 * i + 1]);
      }
    }
  }
  cta_publish_max(mx, s_red, a.max_abs + a.out_row0 + comp, a.key, a.v_first + uint32_t(comp));
}

// ---- batched path for H <= 5 (n = 17..20) -----------------------------------
// Pass A runs as standalone 1024-thread EMIT tile launches over a batch of
// components; this kernel then runs the remaining H stages.  One thread owns
// one pair-column (2^H rows, 2^(H+1) ints), 256-thread CTAs at high occupancy.
// Launch boundaries invalidate L1, so plain (evict-first) loads are safe.
constexpr int kPassBThreads = 256;

template <int H, int MODE>
__global__ void __launch_bounds__(kPassBThreads) k_passb_regs(PassBArgs a) {
  constexpr int NI = 1 << H;
  __shared__ int s_red[kPassBThreads / 32];
  const int64_t chunks = (int64_t(1) << 14) / kPassBThreads;  // per component
  for (int64_t b = blockIdx.x; b < a.n_comp * chunks; b += gridDim.x) {
    const int64_t comp = b / chunks;
    const int64_t col = (b % chunks) * kPassBThreads + threadIdx.x;
    const uint32_t* src = a.scratch + (comp << (a.n - 1)) + col;
    uint32_t u[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) u[i] = __ldcs(src + (int64_t(i) << 14));
    int e[2 * NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      e[2 * i] = lo_half(u[i]);
      e[2 * i + 1] = hi_half(u[i]);
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
      for (int i = 0; i < NI; ++i)
        *reinterpret_cast<int2*>(dst + (int64_t(i) << 15)) = make_int2(e[2 * i], e[2 * i + 1]);
    }
    cta_publish_max(mx, s_red, a.max_abs + a.out_row0 + comp, a.key, a.v_first + uint32_t(comp));
  }
}

// H = 6..9 standalone pass B for the batched path: grid-stride over
// (component, chunk) items; each item's u16 rows are staged with cp.async and
// the CTA's next item is prefetched as soon as the current staging is consumed.
constexpr size_t kPassBSmem = size_t(kTileWords) * sizeof(uint32_t) + (size_t(64) << 10);

template <int H, int MODE>
__global__ void __launch_bounds__(512, 1) k_passb_staged(PassBArgs a) {
  constexpr int THREADS = 512;
  using S = ChunkShape<H, THREADS>;
  extern __shared__ uint4 smem4[];  // [128 KiB int32 tile][64 KiB staging]
  uint32_t* stg = reinterpret_cast<uint32_t*>(smem4) + kTileWords;
  __shared__ int s_red[THREADS / 32];
  const int64_t items = a.n_comp * S::PER_COMP;
  const int64_t comp_words = int64_t(1) << (a.n - 1);
  int64_t b = blockIdx.x;
  if (b < items) stage_chunk<H, THREADS>(a.scratch + (b / S::PER_COMP) * comp_words,
                                         b % S::PER_COMP, stg);
  for (; b < items; b += gridDim.x) {
    stage_wait();
    const int64_t nxt = b + gridDim.x;
    auto prefetch = [&]() {
      if (nxt < items)
        stage_chunk<H, THREADS>(a.scratch + (nxt / S::PER_COMP) * comp_words,
                                nxt % S::PER_COMP, stg);
    };
    passb_smem_chunk<H, MODE>(a, b / S::PER_COMP, b % S::PER_COMP, stg,
                              reinterpret_cast<int2*>(smem4), s_red, prefetch);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

}  // namespace sbw
