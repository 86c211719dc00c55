// Fused "generate -> FWHT -> max|W|" tile kernel, packed-integer (SIMD) form.
//
// Replaces, per output mask v, polarity_row (sbox.py:145-152) +
// fwht_column_in_place (walsh.py:73-104) + column_nonlinearity (:107-114).
//
// Representation.  After k butterfly stages an element's true value v lies in
// [-2^k, 2^k] with v = 2^k (mod 2); we store s = (v + 2^k) / 2 in [0, 2^k].
// A stage k -> k+1 on a pair (a, b) is then
//     sum  = s_a + s_b            (the bias doubles by itself)
//     diff = s_a - s_b + 2^k      (one 3-input add with a per-lane constant)
// and every lane stays inside [0, 2^(k+1)], so lanes packed into one 32-bit
// register never carry into each other: 4 byte lanes while k+1 <= 7, two
// 16-bit lanes while k+1 <= 15.  Only the n = 16 top stage can reach 2^16;
// there a per-lane modular add (VIADD.16x2) folds +2^16 onto -2^16, which has
// the same |W|.  max|W| = 2 * max |s' - 2^(n-1)| comes from per-lane
// max/min tracking (VIMNMX3.U16x2).
//
// Generation.  plane_i is the bit-sliced i-th output bit of the S-box
// (bit x of plane_i = bit i of S(x)), so the 32 component bits
// g_v(32w..32w+31) are the XOR of plane_i[w] over the set bits i of v.  A
// thread keeps the bits of its 64 inputs for its previous mask and XORs only
// the planes of (v ^ v_prev): for consecutive masks ~2 coalesced 8-byte loads
// per 64 elements replace 64 table reads + 64 POPCs.
//
// Tile: a CTA owns 2^16 elements (C = 2^(16-n) components, or two 2^15 blocks
// in EMIT mode) in 128 KiB of shared memory as 16-bit lane pairs (x, x^1).
//   pass 1: x bits 0..5  -- generation, 4 byte stages (bits 0,1,2,5; byte
//           lanes = bits 3,4), unpack to 16-bit lanes (lane = bit 0),
//           2 stages (bits 3,4), one STS.128 per 8 elements;
//   pass 2: x bits 6..10 (5 stages), pass 3: x bits 11..n-1 (n >= 12);
// the last pass fuses the top stage with the max|W| fold.
#pragma once

#include "sbw_fused.cuh"

// Per-phase cycle stamps of tile_body (debug builds: make EXTRA=-DSBW_PHASE_PROF=1).
#ifndef SBW_PHASE_PROF
#define SBW_PHASE_PROF 0
#endif



namespace sbw {

struct TileArgs {
  const uint32_t* planes;  // [m][2^n / 32] bit planes
  int64_t plane_words;     // 2^n / 32
  int m;
  // NL / SPEC: tiles over masks; tile T holds masks T*C + c, valid in [v_lo, v_hi)
  uint32_t v_lo, v_hi;
  int64_t t_begin, t_count;
  int32_t* max_abs;        // [v - v_lo]
  unsigned long long* key;
  int32_t* out;            // SPEC rows [v - v_lo][x]
  int64_t ld;
  // EMIT (multi-pass pass A): components [v_first, v_first + n_comp), blocks of 2^15
  uint32_t v_first;
  int64_t n_comp;
  int n_full;              // n of the S-box (EMIT: 17..24)
  uint32_t* emit;          // u16 pairs, [comp][2^n_full]
  unsigned long long* phase_prof;  // optional (debug): cycles in pass 1 / 2 / 3 (thread 0)
};

// packed stage helpers -------------------------------------------------------
template <int K>
__device__ __forceinline__ void bfly8(uint32_t& a, uint32_t& b) {
  const uint32_t x = a, y = b;
  a = x + y;
  b = x - y + (uint32_t(1u << K) * 0x01010101u);
}
template <int K>
__device__ __forceinline__ void bfly16(uint32_t& a, uint32_t& b) {
  const uint32_t x = a, y = b;
  a = x + y;
  b = x - y + (uint32_t(1u << K) * 0x00010001u);
}

// stages over register-index bits [SB, SE) of R[0..L), first stage index K0
template <int L, int SB, int SE, int K0>
__device__ __forceinline__ void stages16(uint32_t (&R)[L]) {
#pragma unroll
  for (int sb = SB; sb < SE; ++sb) {
#pragma unroll
    for (int i = 0; i < L; ++i) {
      if ((i & (1 << sb)) == 0) {
        // stage index K0 + (sb - SB) is a compile-time constant after unrolling
        const uint32_t x = R[i], y = R[i | (1 << sb)];
        R[i] = x + y;
        R[i | (1 << sb)] = x - y + ((1u << (K0 + sb - SB)) * 0x00010001u);
      }
    }
  }
}


__device__ __forceinline__ int phys_word(int w) { return w ^ (((w >> 5) & 7) << 2); }

// XOR into (w0, w1) the planes of every set bit of `delta` at plane word `cw`.
__device__ __forceinline__ void apply_planes(const uint32_t* __restrict__ planes, int64_t pw,
                                             uint32_t delta, int64_t cw, uint32_t& w0,
                                             uint32_t& w1) {
  while (delta) {
    const int i = __ffs(delta) - 1;
    delta &= delta - 1;
    const uint2 p = __ldg(reinterpret_cast<const uint2*>(planes + int64_t(i) * pw + cw));
    w0 ^= p.x;
    w1 ^= p.y;
  }
}

// Full recompute (the task moved to a new input range): XOR the planes of
// every set bit of v.  Unrolled and predicated so all loads are in flight at
// once -- a data-dependent loop would serialise up to 24 memory latencies.
__device__ __forceinline__ void planes_full(const uint32_t* __restrict__ planes, int64_t pw,
                                            uint32_t v, int64_t cw, uint32_t& w0, uint32_t& w1) {
  uint2 p[24];
#pragma unroll
  for (int i = 0; i < 24; ++i) {
    p[i] = make_uint2(0u, 0u);
    if ((v >> i) & 1u) p[i] = __ldg(reinterpret_cast<const uint2*>(planes + int64_t(i) * pw + cw));
  }
  uint32_t a = 0, b = 0;
#pragma unroll
  for (int i = 0; i < 24; ++i) {
    a ^= p[i].x;
    b ^= p[i].y;
  }
  w0 = a;
  w1 = b;
}

// max|W| of a task from its packed max/min trackers (top stage index N)
template <int N>
__device__ __forceinline__ int lanes_maxabs(uint32_t mx, uint32_t mn) {
  const int c = 1 << (N - 1);
  const int hi = max(int(mx & 0xFFFFu), int(mx >> 16));
  const int lo = min(int(mn & 0xFFFFu), int(mn >> 16));
  return 2 * max(hi - c, c - lo);
}


__device__ __forceinline__ uint32_t prmt(uint32_t x, uint32_t y, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(y), "r"(sel));
  return r;
}

// Last pass of a tile task: E[NI] 16-bit lane pairs whose register index i
// maps to x bits K0.. (word bit SH..).  Runs the remaining stages, fuses the
// top one with the max|W| fold (NL), the int32 materialisation (SPEC) or the
// u16 emit for the multi-pass path (EMIT).
template <int N, int MODE, int NI, int SH, int K0>
__device__ __forceinline__ void tile_last_pass(const TileArgs& a, uint32_t (&E)[NI], int wb,
                                               int64_t t, int* s_max) {
  constexpr int LOGI = (NI == 1) ? 0 : (NI == 2 ? 1 : (NI == 4 ? 2 : (NI == 8 ? 3 : (NI == 16 ? 4 : 5))));
  static_assert(K0 + LOGI == N, "last pass must end at stage N");
  constexpr int HALF = NI / 2;
  constexpr int C = 1 << (16 - N);
  constexpr int XMASK = (1 << N) - 1;
  stages16<NI, 0, LOGI - 1, K0>(E);
  const int slot = (wb << 1) >> N;
  if constexpr (MODE == MODE_NL) {
    uint32_t mx = 0u, mn = 0xFFFFFFFFu;
#pragma unroll
    for (int k = 0; k < HALF; ++k) {
      const uint32_t x = E[k], y = E[k + HALF];
      // Plain 32-bit adds.  For N < 16 every lane stays in [0, 2^N] (no carry).
      // For N = 16 a low lane reaches 2^16 only when |W| = 2^16, the largest
      // value possible: it wraps to 0 (same |W|) and carries +1 into the high
      // lane, which then reads some |W'| <= 2^16 -- the component max is 2^16
      // either way, so max|W| stays exact without per-lane modular adds.
      const uint32_t S = x + y;
      const uint32_t D = x - y + ((1u << (N - 1)) * 0x00010001u);
      mx = __vimax3_u16x2(mx, S, D);
      mn = __vimin3_u16x2(mn, S, D);
    }
    int m = lanes_maxabs<N>(mx, mn);
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) atomicMax(&s_max[slot], m);
  } else if constexpr (MODE == MODE_SPEC) {
    const int64_t vv = t * C + slot;
    const bool ok = vv >= a.v_lo && vv < a.v_hi;
    int m = 0;
    int32_t* row = a.out + (ok ? (vv - a.v_lo) : 0) * a.ld;
#pragma unroll
    for (int k = 0; k < HALF; ++k) {
      const uint32_t x = E[k], y = E[k + HALF];
      const int xa0 = int(x & 0xFFFFu), xa1 = int(x >> 16);
      const int yb0 = int(y & 0xFFFFu), yb1 = int(y >> 16);
      const int s0 = 2 * (xa0 + yb0) - (1 << N), s1 = 2 * (xa1 + yb1) - (1 << N);
      const int d0 = 2 * (xa0 - yb0), d1 = 2 * (xa1 - yb1);
      m = max(m, max(max(abs(s0), abs(s1)), max(abs(d0), abs(d1))));
      if (ok) {
        const int xs = ((wb | (k << SH)) << 1) & XMASK;
        const int xd = ((wb | ((k + HALF) << SH)) << 1) & XMASK;
        *reinterpret_cast<int2*>(row + xs) = make_int2(s0, s1);
        *reinterpret_cast<int2*>(row + xd) = make_int2(d0, d1);
      }
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) atomicMax(&s_max[slot], m);
  } else {  // MODE_EMIT: s after 15 stages, u16 in [0, 2^15]
    const int64_t bp = t / a.n_comp, ci = t - bp * a.n_comp;
    const int64_t block = 2 * bp + slot;
    uint32_t* dst = a.emit + (ci << (a.n_full - 1)) + (block << 14);
#pragma unroll
    for (int k = 0; k < HALF; ++k) {
      const uint32_t x = E[k], y = E[k + HALF];
      dst[(wb | (k << SH)) & 0x3FFF] = x + y;
      dst[(wb | ((k + HALF) << SH)) & 0x3FFF] = x - y + ((1u << (N - 1)) * 0x00010001u);
    }
  }
}

// Per-thread generation state of the pass-1 tasks (bits of the previous mask).
template <int ROUNDS>
struct GenState {
  uint32_t v[ROUNDS], w0[ROUNDS], w1[ROUNDS];
  int64_t cw[ROUNDS];
  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int r = 0; r < ROUNDS; ++r) {
      v[r] = w0[r] = w1[r] = 0;
      cw[r] = -1;
    }
  }
};

// One tile t (see the file comment): three passes over the shared-memory
// tile, result published per component (NL / SPEC) or emitted (EMIT).  Must be
// called by all THREADS threads of the CTA.
template <int N, int MODE, int THREADS>
__device__ __forceinline__ void tile_body(const TileArgs& a, int64_t t, uint4* smem4, int* s_max,
                                          GenState<1024 / THREADS>& gs) {
  constexpr int ROUNDS = 1024 / THREADS;         // pass-1 tasks per thread
  static_assert(N >= 7 && N <= 16, "tile kernel covers n = 7..16");
  static_assert(MODE != MODE_EMIT || N == 15, "EMIT works on 2^15 blocks");
  constexpr int J = 16 - N;
  constexpr int C = 1 << J;                      // items per tile
  constexpr int B2 = (N - 6) < 5 ? (N - 6) : 5;  // x bits in pass 2
  constexpr int B3 = N > 11 ? N - 11 : 0;        // x bits in pass 3
  constexpr int XMASK = (1 << N) - 1;
  uint32_t* sm = reinterpret_cast<uint32_t*>(smem4);
  const int tid = threadIdx.x;
#if SBW_PHASE_PROF
  const long long ph0 = clock64();
#endif
  uint32_t* g_v = gs.v;
  uint32_t* g_w0 = gs.w0;
  uint32_t* g_w1 = gs.w1;
  int64_t* g_cw = gs.cw;

  // ---------------- pass 1: generation + x bits 0..5 ---------------------
#pragma unroll
  for (int r = 0; r < ROUNDS; ++r) {
    const int task = r * THREADS + tid;
    const int p0 = task << 6;
    const int slot = p0 >> N;
    const int x0 = p0 & XMASK;
    uint32_t v = 0;
    int64_t cw = 0;
    bool valid;
    if constexpr (MODE == MODE_EMIT) {
      const int64_t bp = t / a.n_comp, ci = t - bp * a.n_comp;
      v = a.v_first + uint32_t(ci);
      cw = ((2 * bp + slot) * (int64_t(1) << 15) + x0) >> 5;
      valid = true;
    } else {
      const int64_t vv = t * C + slot;
      v = uint32_t(vv);
      cw = x0 >> 5;
      valid = vv >= a.v_lo && vv < a.v_hi;
    }
    uint32_t w0 = 0, w1 = 0;
    if (valid) {
      if (cw == g_cw[r]) {
        w0 = g_w0[r];
        w1 = g_w1[r];
        apply_planes(a.planes, a.plane_words, v ^ g_v[r], cw, w0, w1);
      } else {
        planes_full(a.planes, a.plane_words, v, cw, w0, w1);
      }
      g_v[r] = v;
      g_w0[r] = w0;
      g_w1[r] = w1;
      g_cw[r] = cw;
    }
    // bytes: R[h*8 + r'] lane l <- 1 - g(x), x = 32h + 8l + r'  (s at k = 0)
    uint32_t R[16];
    const uint32_t n0 = ~w0, n1 = ~w1;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      // w >> q as a high multiply (FMA pipe) instead of SHF (ALU pipe)
      R[q] = (q ? __umulhi(n0, 1u << (32 - q)) : n0) & 0x01010101u;
      R[8 + q] = (q ? __umulhi(n1, 1u << (32 - q)) : n1) & 0x01010101u;
    }
    // byte stages on register bits (x bits 0,1,2,5), k = 0..3
#pragma unroll
    for (int i = 0; i < 16; ++i) if (!(i & 1)) bfly8<0>(R[i], R[i | 1]);
#pragma unroll
    for (int i = 0; i < 16; ++i) if (!(i & 2)) bfly8<1>(R[i], R[i | 2]);
#pragma unroll
    for (int i = 0; i < 16; ++i) if (!(i & 4)) bfly8<2>(R[i], R[i | 4]);
#pragma unroll
    for (int i = 0; i < 16; ++i) if (!(i & 8)) bfly8<3>(R[i], R[i | 8]);
    // unpack: H[q], q = (x1, x2, x3, x4, x5) bits 0..4; 16-bit lane = x0.
    // source bytes: R[(x5 << 3) | (x2 << 2) | (x1 << 1) | x0], byte lane (x4 << 1) | x3.
    // Values are <= 16 after 4 stages, so PRMT sign-replicate yields 0x00.
    uint32_t H[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      const int x1 = q & 1, x2 = (q >> 1) & 1, l = (q >> 2) & 3, x5 = (q >> 4) & 1;
      const int i0 = (x5 << 3) | (x2 << 2) | (x1 << 1);
      const uint32_t sel = uint32_t(l) | (uint32_t(8 | l) << 4) | (uint32_t(4 + l) << 8) |
                           (uint32_t(8 | (4 + l)) << 12);
      H[q] = prmt(R[i0], R[i0 | 1], sel);
    }
    // 16-bit stages on x3 (H bit 2) and x4 (H bit 3), k = 4, 5
    stages16<32, 2, 4, 4>(H);
    // store: task's 32 words as 8 x 16 B, chunk-swizzled
    uint4* dst = smem4 + (task << 3);
#pragma unroll
    for (int c4 = 0; c4 < 8; ++c4)
      dst[c4 ^ (task & 7)] = make_uint4(H[4 * c4], H[4 * c4 + 1], H[4 * c4 + 2], H[4 * c4 + 3]);
  }
  __syncthreads();
#if SBW_PHASE_PROF
  const long long ph1 = clock64();
#endif

  // ---------------- pass 2: x bits 6 .. 6+B2-1 ---------------------------
  {
    constexpr int NI = 1 << B2;
    constexpr int NT = kTileWords >> B2;
    constexpr bool LAST = (B3 == 0);
    // two tasks per thread in flight when there are enough of them: all loads
    // of both issue before either's arithmetic (hides the LDS latency with
    // few warps, e.g. the 512-thread multi-pass kernel)
    constexpr int IL = (!LAST && THREADS <= 512 && NT >= 2 * THREADS) ? 2 : 1;
    for (int task0 = tid; IL == 2 && task0 < NT; task0 += 2 * THREADS) {
      uint32_t E[2][NI];
      int P[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int task = task0 + q * THREADS;
        P[q] = phys_word(((task >> 5) << (5 + B2)) | (task & 31));
#pragma unroll
        for (int i = 0; i < NI; ++i) E[q][i] = sm[(P[q] ^ ((i & 7) << 2)) + (i << 5)];
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) stages16<NI, 0, B2, 6>(E[q]);
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int i = 0; i < NI; ++i) sm[(P[q] ^ ((i & 7) << 2)) + (i << 5)] = E[q][i];
    }
    for (int task = tid; IL == 1 && task < NT; task += THREADS) {
      const int lo = task & 31, hi = task >> 5;
      const int wb = (hi << (5 + B2)) | lo;
      // phys(wb | i << 5) = (P ^ ((i & 7) << 2)) + (i << 5), P = phys(wb):
      // at most 8 base pointers, the rest are immediate offsets
      const int P = phys_word(wb);
      uint32_t E[NI];
#pragma unroll
      for (int i = 0; i < NI; ++i) E[i] = sm[(P ^ ((i & 7) << 2)) + (i << 5)];
      if constexpr (!LAST) {
        stages16<NI, 0, B2, 6>(E);
#pragma unroll
        for (int i = 0; i < NI; ++i) sm[(P ^ ((i & 7) << 2)) + (i << 5)] = E[i];
      } else {
        tile_last_pass<N, MODE, NI, 5, 6>(a, E, wb, t, s_max);
      }
    }
  }
  __syncthreads();
#if SBW_PHASE_PROF
  const long long ph2 = clock64();
#endif

  // ---------------- pass 3: x bits 11 .. N-1 ------------------------------
  if constexpr (B3 > 0) {
    constexpr int NI = 1 << B3;
    constexpr int NT = kTileWords >> B3;
    // the swizzle depends on word bits 5..7 only, so phys(wb | i << 10) = phys(wb) + (i << 10).
    constexpr int IL = 1;  // a 2-task interleave here measured slower (5.2K vs 4.6K cyc)
    for (int task0 = tid; task0 < NT; task0 += IL * THREADS) {
      uint32_t E[IL][NI];
      int wb[IL];
#pragma unroll
      for (int q = 0; q < IL; ++q) {
        const int task = task0 + q * THREADS;
        wb[q] = ((task >> 10) << (10 + B3)) | (task & 1023);
        const uint32_t* base = sm + phys_word(wb[q]);
#pragma unroll
        for (int i = 0; i < NI; ++i) E[q][i] = base[i << 10];
      }
#pragma unroll
      for (int q = 0; q < IL; ++q) tile_last_pass<N, MODE, NI, 10, 11>(a, E[q], wb[q], t, s_max);
    }
    __syncthreads();
  }

#if SBW_PHASE_PROF
  if (a.phase_prof && threadIdx.x == 0) {
    const long long ph3 = clock64();
    atomicAdd(a.phase_prof + 0, (unsigned long long)(ph1 - ph0));
    atomicAdd(a.phase_prof + 1, (unsigned long long)(ph2 - ph1));
    atomicAdd(a.phase_prof + 2, (unsigned long long)(ph3 - ph2));
  }
#endif
}

// Publish tile t's per-component maxima and clear its slots.  Called right
// after tile_body (whose last barrier orders every atomicMax before this);
// the caller alternates two s_max buffers so no extra barrier is needed.
template <int N>
__device__ __forceinline__ void tile_publish(const TileArgs& a, int64_t t, int* s_max) {
  constexpr int C = 1 << (16 - N);
  if (threadIdx.x < C) {
    const int64_t vv = t * C + threadIdx.x;
    if (vv >= a.v_lo && vv < a.v_hi) {
      const int mx = s_max[threadIdx.x];
      a.max_abs[vv - a.v_lo] = mx;
      if (a.key) atomicMax(a.key, nl_key(mx, uint32_t(vv)));
    }
    s_max[threadIdx.x] = 0;
  }
}

template <int N, int MODE, int THREADS = kTileThreads>
__global__ void __launch_bounds__(THREADS, 1) k_tile_simd(TileArgs a) {
  constexpr int C = 1 << (16 - N);
  extern __shared__ uint4 smem4[];
  __shared__ int s_max[2][C];  // per-component max, double-buffered by tile parity
  const int64_t t_lo = a.t_begin + (a.t_count * blockIdx.x) / gridDim.x;
  const int64_t t_hi = a.t_begin + (a.t_count * (blockIdx.x + 1)) / gridDim.x;
  if (threadIdx.x < C) s_max[0][threadIdx.x] = s_max[1][threadIdx.x] = 0;
  __syncthreads();
  GenState<1024 / THREADS> gs;
  gs.reset();
  int par = 0;
  for (int64_t t = t_lo; t < t_hi; ++t, par ^= 1) {
    tile_body<N, MODE, THREADS>(a, t, smem4, s_max[par], gs);
    if constexpr (MODE != MODE_EMIT) tile_publish<N>(a, t, s_max[par]);
  }
}

}  // namespace sbw
