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
//   H <= 5: registers only; a thread owns one pair column of 2^H rows.
//   H  > 5: a CTA stages a [2^H rows x 32 pair-columns] int32 tile in shared
//           memory and runs two register passes over it.
// Both run inside the persistent k3_persistent kernel below, interleaved with
// pass A so the scratch of in-flight components stays L2-resident.
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
// Scratch reads use ld.global.cg: the persistent kernel reuses ring slots, so
// an SM's L1 may hold lines of an older component.

// H <= 5: THREADS pair-columns of one component, 2^H rows each, in registers.
template <int H, int MODE, int THREADS>
__device__ __forceinline__ void passb_regs_chunk(const PassBArgs& a, int64_t comp, int64_t chunk,
                                                 int* s_red) {
  constexpr int NI = 1 << H;
  const int64_t col = chunk * THREADS + threadIdx.x;
  const uint32_t* src = a.scratch + (comp << (a.n - 1)) + col;
  uint32_t u[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) u[i] = __ldcg(src + (int64_t(i) << 14));
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

// H = 6..9: 32 pair-columns x 2^H rows.  B1 reads row bits 0..4 straight from
// the scratch (32 independent loads in flight per task) and parks int32 pairs
// in shared memory; B2 runs row bits 5..H-1 with the fused top stage.
template <int H, int MODE>
__device__ __forceinline__ void passb_smem_chunk(const PassBArgs& a, int64_t comp, int64_t chunk,
                                                 int2* tile, int* s_red) {
  constexpr int H2 = H - 5;
  constexpr int N2 = 1 << H2;
  const int64_t col0 = chunk * 32;
  const uint32_t* src = a.scratch + (comp << (a.n - 1)) + col0;
  for (int task = threadIdx.x; task < 32 * N2; task += blockDim.x) {
    const int c = task & 31, rh = task >> 5;
    uint32_t u[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) u[i] = __ldcg(src + (int64_t((rh << 5) | i) << 14) + c);
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

// ---- persistent multi-pass kernel ------------------------------------------
// One CTA per SM pulls work items from a global counter in a fixed order:
//   A(0) .. A(D-1) | A(D) B(0) | A(D+1) B(1) | ... | B(C-D) .. B(C-1)
// where A(c) = the 2^(n-16) pass-A tiles of component c and B(c) = its pass-B
// chunks, and the lookahead D puts several waves of items between A(c) and
// B(c).  B(c) waits (acquire) until all A(c) tiles are published; A(c) waits
// until B(c - R) (R > D) has released ring slot c % R.  Every item waits only
// on items dequeued before it by running CTAs, so progress is guaranteed, and
// at most R components of scratch are live, which keeps them in L2.
struct K3Args {
  TileArgs ta;              // planes etc.; EMIT fields are set per item
  PassBArgs pb;             // n, max_abs, key, out, ld; per-item fields set per item
  uint32_t v_lo;
  int64_t ncomp;
  uint32_t* ring;           // R slots of 2^(n-1) u16-pair words
  int ring_slots;
  int64_t lookahead;        // D: B(c) is queued after A(c + D); 1 <= D < R, D <= ncomp
  unsigned int* counters;   // [0] = queue head, [1 + c] = A done, [1 + ncomp + c] = B done
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void wait_counter(const unsigned* p, unsigned target) {
  if (threadIdx.x == 0) {
    while (ld_acquire(p) < target) __nanosleep(256);
  }
  __syncthreads();
}

// bar.sync orders every thread's writes before thread 0's release-add (PTX
// release is cumulative), so one fence-carrying atomic publishes the CTA's work.
__device__ __forceinline__ void release_counter(unsigned* p) {
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

template <int H, int MODE>
__global__ void __launch_bounds__(512, 1) k3_persistent(K3Args a) {
  constexpr int THREADS = 512;
  constexpr int64_t NA = int64_t(1) << (H - 1);        // pass-A tiles per component
  constexpr int64_t NB = H <= 5 ? (int64_t(1) << 14) / THREADS : (int64_t(1) << 14) / 32;
  extern __shared__ uint4 smem4[];
  __shared__ int s_max[2];
  __shared__ int s_red[THREADS / 32];
  __shared__ long long s_item[2];  // current / next queue item (prefetched by thread 0)
  const int64_t total = a.ncomp * (NA + NB);
  unsigned* head = a.counters;
  unsigned* done_a = a.counters + 1;
  unsigned* done_b = a.counters + 1 + a.ncomp;
  const int64_t slot_words = int64_t(1) << (a.pb.n - 1);
  GenState<1024 / THREADS> gs;
  gs.reset();
  if (threadIdx.x == 0) s_item[0] = atomicAdd(head, 1u);
  __syncthreads();
  for (int it = 0;; it ^= 1) {
    const int64_t item = s_item[it];
    if (item >= total) break;
    // fetch the next item now; every item body ends with a barrier, which
    // publishes s_item[it ^ 1] before the next iteration reads it
    if (threadIdx.x == 0) s_item[it ^ 1] = atomicAdd(head, 1u);
    // decode the item (see the sequence above)
    const int64_t D = a.lookahead, C = a.ncomp;
    int64_t c, k;
    bool is_a;
    if (item < D * NA) {
      c = item / NA, k = item - c * NA, is_a = true;
    } else if (item - D * NA < (C - D) * (NA + NB)) {
      const int64_t r = item - D * NA;
      const int64_t j = D + r / (NA + NB), off = r - (j - D) * (NA + NB);
      is_a = off < NA;
      c = is_a ? j : j - D;
      k = is_a ? off : off - NA;
    } else {
      const int64_t r = item - D * NA - (C - D) * (NA + NB);
      c = C - D + r / NB, k = r - (c - (C - D)) * NB, is_a = false;
    }
    uint32_t* slot = a.ring + (c % a.ring_slots) * slot_words;
    if (is_a) {
      if (c >= a.ring_slots) wait_counter(done_b + (c - a.ring_slots), unsigned(NB));
      TileArgs ta = a.ta;
      ta.v_first = a.v_lo + uint32_t(c);
      ta.n_comp = 1;
      ta.emit = slot;
      tile_body<15, MODE_EMIT, THREADS>(ta, k, smem4, s_max, gs);
      release_counter(done_a + c);
    } else {
      wait_counter(done_a + c, unsigned(NA));
      PassBArgs pb = a.pb;
      pb.scratch = slot;
      pb.n_comp = 1;
      pb.out_row0 = c;
      pb.v_first = a.v_lo + uint32_t(c);
      if constexpr (H <= 5) {
        passb_regs_chunk<H, MODE, THREADS>(pb, 0, k, s_red);
      } else {
        passb_smem_chunk<H, MODE>(pb, 0, k, reinterpret_cast<int2*>(smem4), s_red);
      }
      release_counter(done_b + c);
    }
  }
}

}  // namespace sbw
