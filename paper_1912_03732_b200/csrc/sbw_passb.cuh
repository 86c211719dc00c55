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

// H <= 5: THREADS pair-columns, 2^H rows each, in registers.  `after_read`
// runs (by every thread) once the staging buffer is no longer needed.
template <int H, int MODE, int THREADS, typename AfterRead>
__device__ __forceinline__ void passb_regs_chunk(const PassBArgs& a, int64_t comp, int64_t chunk,
                                                 const uint32_t* stg, int* s_red,
                                                 AfterRead after_read) {
  constexpr int NI = 1 << H;
  const int64_t col = chunk * THREADS + threadIdx.x;
  uint32_t u[NI];
#pragma unroll
  for (int i = 0; i < NI; ++i) u[i] = stg[i * THREADS + threadIdx.x];
  __syncthreads();
  after_read();
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
  unsigned long long* prof; // optional (debug): cycle accounting, see k3_persistent
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Non-blocking, CTA-uniform check (one barrier).
__device__ __forceinline__ bool counter_reached(const unsigned* p, unsigned target, int* flag) {
  if (threadIdx.x == 0) *flag = ld_acquire(p) >= target;
  __syncthreads();
  const bool r = *flag != 0;
  __syncthreads();
  return r;
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

struct K3Item {
  int64_t c, k;
  bool is_a;
};

// Decode a queue index (see the sequence above).
template <int64_t NA, int64_t NB>
__device__ __forceinline__ K3Item k3_decode(int64_t item, int64_t D, int64_t C) {
  K3Item r;
  if (item < D * NA) {
    r.c = item / NA, r.k = item - r.c * NA, r.is_a = true;
  } else if (item - D * NA < (C - D) * (NA + NB)) {
    const int64_t q = item - D * NA;
    const int64_t j = D + q / (NA + NB), off = q - (j - D) * (NA + NB);
    r.is_a = off < NA;
    r.c = r.is_a ? j : j - D;
    r.k = r.is_a ? off : off - NA;
  } else {
    const int64_t q = item - D * NA - (C - D) * (NA + NB);
    r.c = C - D + q / NB, r.k = q - (r.c - (C - D)) * NB, r.is_a = false;
  }
  return r;
}

constexpr int kStageWords = 24 * 1024;     // 96 KiB staging: a pass-B chunk or A-tile planes
constexpr int kStagedPlanesMax = kStageWords / 2048;  // 12 plane segments of 8 KiB
constexpr size_t kK3Smem = size_t(kTileWords) * sizeof(uint32_t) + size_t(kStageWords) * 4;

// Issue (not wait for) the copies of the plane segments an A tile needs: the
// first `count` set bits of v, each 2048 words starting at `base_word`.
template <int THREADS>
__device__ __forceinline__ void stage_planes(const uint32_t* planes, int64_t pw, uint32_t v,
                                             int64_t base_word, int count, uint32_t* stg) {
  int j = 0;
  for (uint32_t d = v; d && j < count; d &= d - 1, ++j) {
    const uint32_t* g = planes + int64_t(__ffs(d) - 1) * pw + base_word;
    for (int p = threadIdx.x; p < 512; p += THREADS) {
      const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(stg + j * 2048 + 4 * p));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g + 4 * p) : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int H, int MODE>
__global__ void __launch_bounds__(512, 1) k3_persistent(K3Args a) {
  constexpr int THREADS = 512;
  using S = ChunkShape<H, THREADS>;
  constexpr int64_t NA = int64_t(1) << (H - 1);  // pass-A tiles per component
  constexpr int64_t NB = S::PER_COMP;            // pass-B chunks per component
  extern __shared__ uint4 smem4[];               // [128 KiB tile / int32 rows][96 KiB staging]
  uint32_t* stg = reinterpret_cast<uint32_t*>(smem4) + kTileWords;
  __shared__ int s_max[2];
  __shared__ int s_red[THREADS / 32];
  __shared__ long long s_item[2];  // current / next queue item (prefetched by thread 0)
  __shared__ int s_flag;
  const int64_t total = a.ncomp * (NA + NB);
  unsigned* head = a.counters;
  unsigned* done_a = a.counters + 1;
  unsigned* done_b = a.counters + 1 + a.ncomp;
  const int64_t slot_words = int64_t(1) << (a.pb.n - 1);
  GenState<1024 / THREADS> gs;
  gs.reset();
  int64_t staged = -1;  // queue item whose chunk / planes are in (or in flight to) `stg`
  // Counters only grow, so a condition this CTA has seen satisfied stays
  // satisfied: skip the acquire round trip (and its barrier) when possible.
  int64_t seen_a = -1;  // largest c with done_a[c] == NA observed
  int64_t seen_b = -1;  // component c whose done_b[c] == NB was observed
  if (threadIdx.x == 0) s_item[0] = atomicAdd(head, 1u);
  __syncthreads();
  for (int it = 0;; it ^= 1) {
    const int64_t item = s_item[it];
    if (item >= total) break;
    // fetch the next item now; every item body ends with a barrier, which
    // publishes s_item[it ^ 1] before the next iteration reads it
    if (threadIdx.x == 0) s_item[it ^ 1] = atomicAdd(head, 1u);
    const K3Item cur = k3_decode<NA, NB>(item, a.lookahead, a.ncomp);
    uint32_t* slot = a.ring + (cur.c % a.ring_slots) * slot_words;
    // Start copying the next item's inputs into `stg` once this item no
    // longer reads it: the plane segments of an A tile (always ready) or a
    // pass-B chunk whose tiles are all published (never blocks: this CTA
    // still holds `item`, which A tiles may be waiting on via ring reuse).
    auto prefetch_next = [&]() {
      staged = -1;
      const int64_t nxt = s_item[it ^ 1];
      if (nxt >= total) return;
      const K3Item n = k3_decode<NA, NB>(nxt, a.lookahead, a.ncomp);
      if (n.is_a) {
        const uint32_t vn = a.v_lo + uint32_t(n.c);
        stage_planes<THREADS>(a.ta.planes, a.ta.plane_words, vn, n.k * 2048,
                              min(__popc(vn), kStagedPlanesMax), stg);
        staged = nxt;
        return;
      }
      if (seen_a != n.c) {
        if (!counter_reached(done_a + n.c, unsigned(NA), &s_flag)) return;
        seen_a = n.c;
      }
      stage_chunk<H, THREADS>(a.ring + (n.c % a.ring_slots) * slot_words, n.k, stg);
      staged = nxt;
    };
    const long long t0 = clock64();
    if (cur.is_a) {
      if (cur.c >= a.ring_slots && seen_b != cur.c - a.ring_slots) {
        wait_counter(done_b + (cur.c - a.ring_slots), unsigned(NB));
        seen_b = cur.c - a.ring_slots;
      }
      const long long t1 = clock64();
      TileArgs ta = a.ta;
      ta.v_first = a.v_lo + uint32_t(cur.c);
      ta.n_comp = 1;
      ta.emit = slot;
      StagedPlanes sp;
      if (staged == item) {
        stage_wait();
        sp.words = stg;
        sp.count = min(__popc(ta.v_first), kStagedPlanesMax);
        sp.base_word = cur.k * 2048;
      }
      tile_body<15, MODE_EMIT, THREADS>(ta, cur.k, smem4, s_max, gs, sp, prefetch_next);
      release_counter(done_a + cur.c);
      if (a.prof && threadIdx.x == 0) {
        atomicAdd(a.prof + 0, (unsigned long long)(clock64() - t0));
        atomicAdd(a.prof + 1, (unsigned long long)(t1 - t0));
        atomicAdd(a.prof + 5, 1ull);
      }
    } else {
      if (staged != item) {
        if (seen_a != cur.c) {
          wait_counter(done_a + cur.c, unsigned(NA));
          seen_a = cur.c;
        }
        stage_chunk<H, THREADS>(slot, cur.k, stg);
      }
      const long long t1 = clock64();
      stage_wait();
      const long long t2 = clock64();
      PassBArgs pb = a.pb;
      pb.scratch = slot;
      pb.n_comp = 1;
      pb.out_row0 = cur.c;
      pb.v_first = a.v_lo + uint32_t(cur.c);
      if constexpr (H <= 5) {
        passb_regs_chunk<H, MODE, THREADS>(pb, 0, cur.k, stg, s_red, prefetch_next);
      } else {
        passb_smem_chunk<H, MODE>(pb, 0, cur.k, stg, reinterpret_cast<int2*>(smem4), s_red,
                                  prefetch_next);
      }
      release_counter(done_b + cur.c);
      if (a.prof && threadIdx.x == 0) {
        atomicAdd(a.prof + 2, (unsigned long long)(clock64() - t0));
        atomicAdd(a.prof + 3, (unsigned long long)(t1 - t0));
        atomicAdd(a.prof + 4, (unsigned long long)(t2 - t1));
        atomicAdd(a.prof + 6, 1ull);
        atomicAdd(a.prof + 7, staged >= 0 ? 1ull : 0ull);
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

}  // namespace sbw
