// Fused "generate component -> FWHT -> max|W| (or materialise)" kernels.
//
// Replaces, per output mask v, the reference's
//   polarity_row            pkg/src/sboxeval/sbox.py:145-152
//   fwht_column_in_place    pkg/src/sboxeval/walsh.py:73-104
//   column_nonlinearity     pkg/src/sboxeval/walsh.py:107-114
// driven by fwht_fused / fwht_parallel (walsh.py:204-248, parallel.py:64-133).
//
// Tile kernel (n = 7..16, "K1"): a CTA owns a tile of 2^16 elements = C =
// 2^(16-n) components resident in shared memory as int16 pairs (128 KiB).
// Three register passes cover the 16 index bits:
//   pass 1: x bits 0..5   (generation from the S-box table + 6 stages),
//   pass 2: x bits 6..10  (5 stages),
//   pass 3: x bits 11..15 (5 stages, n >= 12 only),
// each pass exchanging through a bank-swizzled int16-pair buffer.  Stored
// values have seen <= 11 stages, so |value| <= 2^11 fits int16 exactly; the
// last pass computes in int32 and folds max(|a+b|,|a-b|) = |a|+|b| on its final
// stage, so the spectrum never leaves the SM unless materialised.
// The same kernel with MODE_EMIT is pass A of the multi-pass path (n >= 17):
// 15 stages over a 2^15-element block, halved int16 results to global.
#pragma once

#include <type_traits>

#include "sbw_internal.cuh"

namespace sbw {

constexpr int kTileThreads = 512;
constexpr int kTileWords = 1 << 15;  // 2^16 int16 elements as 32-bit pairs

enum FusedMode { MODE_NL = 0, MODE_SPEC = 1, MODE_EMIT = 2 };

struct FusedArgs {
  const void* table;
  uint32_t v_first;       // mask of item 0
  int nbl;                // log2(blocks per component); 0 unless MODE_EMIT
  int64_t n_items;        // (component, block) items
  int32_t* max_abs;       // [item] for NL / SPEC
  unsigned long long* key;
  int32_t* out;           // SPEC: out[item * ld + x]
  int64_t ld;
  uint32_t* emit;         // EMIT: int16 pairs, component stride 2^(N + nbl) elements
};

__device__ __forceinline__ int swz(int w) { return w ^ ((w >> 5) & 31); }

// Load 64 consecutive table entries and turn them into +/-1 polarities.
template <typename TT>
__device__ __forceinline__ void gen64(const TT* __restrict__ p, uint32_t v, int (&e)[64]) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  constexpr int PER = 16 / int(sizeof(TT));
#pragma unroll
  for (int k = 0; k < 64 / PER; ++k) {
    const uint4 r = __ldg(q + k);
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      uint32_t s;
      if constexpr (sizeof(TT) == 4) {
        s = w[j];
      } else {
        s = (w[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
      }
      e[k * PER + j] = polarity(s, v);
    }
  }
}

// Final stage of a register group e[0..2*NI): pairs at stride NI (the top
// i-bit).  Returns the partial max|W| of the group; materialises if asked.
template <int NI, int MODE>
__device__ __forceinline__ int final_stage(int (&e)[2 * NI]) {
  int mx = 0;
  if constexpr (MODE == MODE_NL) {
#pragma unroll
    for (int k = 0; k < NI; ++k) mx = max(mx, abs(e[k]) + abs(e[k + NI]));
  } else {
#pragma unroll
    for (int k = 0; k < NI; ++k) {
      const int a = e[k], b = e[k + NI];
      e[k] = a + b;
      e[k + NI] = a - b;
      mx = max(mx, max(abs(e[k]), abs(e[k + NI])));
    }
  }
  return mx;
}

template <int N, typename TT, int MODE>
__global__ void __launch_bounds__(kTileThreads, 1) k_fused_tile(FusedArgs a) {
  static_assert(N >= 7 && N <= 16, "tile kernel covers n = 7..16");
  constexpr int C = 1 << (16 - N);              // items per tile
  constexpr int B2 = (N - 6) < 5 ? (N - 6) : 5; // x bits in pass 2
  constexpr int B3 = N > 11 ? N - 11 : 0;       // x bits in pass 3
  constexpr int XMASK = (1 << N) - 1;
  extern __shared__ uint32_t sm[];
  __shared__ int s_max[C];

  const int tid = threadIdx.x;
  const TT* __restrict__ table = static_cast<const TT*>(a.table);
  const int64_t ntiles = (a.n_items + C - 1) / C;
  const int64_t bmask = (int64_t(1) << a.nbl) - 1;

  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t item0 = t * C;
    if (tid < C) s_max[tid] = 0;

    // ---- pass 1: generate 64 consecutive x and butterfly x bits 0..5 ----
    for (int task = tid; task < 1024; task += kTileThreads) {
      const int p0 = task << 6;
      const int64_t g = item0 + (p0 >> N);
      int e[64];
      if (g < a.n_items) {
        const uint32_t v = a.v_first + uint32_t(g >> a.nbl);
        const int64_t x0 = ((g & bmask) << N) + (p0 & XMASK);
        gen64<TT>(table + x0, v, e);
      } else {
#pragma unroll
        for (int i = 0; i < 64; ++i) e[i] = 0;
      }
      fwht_regs<64, 1>(e);
      const int wb = task << 5;
#pragma unroll
      for (int j = 0; j < 32; ++j) sm[wb | (j ^ (task & 31))] = pack2(e[2 * j], e[2 * j + 1]);
    }
    __syncthreads();

    // ---- pass 2 (x bits 6..6+B2-1) and pass 3 (x bits 11..N-1) ----------
#pragma unroll
    for (int pass = 2; pass <= 3; ++pass) {
      if (pass == 3 && B3 == 0) break;
      const bool last = (pass == 3) || (B3 == 0);
      // Both passes are instantiated through the same generic lambda below.
      auto run = [&](auto BI_c, auto SH_c) {
        constexpr int BI = decltype(BI_c)::value;   // bits handled
        constexpr int SH = decltype(SH_c)::value;   // word-bit offset of i
        constexpr int NI = 1 << BI;
        constexpr int LOW = (1 << SH) - 1;
        constexpr int NT = kTileWords >> BI;
        for (int task = tid; task < NT; task += kTileThreads) {
          const int lo = task & LOW;
          const int hi = task >> SH;
          const int wb = (hi << (SH + BI)) | lo;
          int e[2 * NI];
#pragma unroll
          for (int i = 0; i < NI; ++i) {
            const uint32_t u = sm[swz(wb | (i << SH))];
            e[2 * i] = lo16(u);
            e[2 * i + 1] = hi16(u);
          }
          if (!last) {
            fwht_regs<2 * NI, 2>(e);
#pragma unroll
            for (int i = 0; i < NI; ++i) sm[swz(wb | (i << SH))] = pack2(e[2 * i], e[2 * i + 1]);
            continue;
          }
          // last pass: every stage but the top one, then the fused top stage
          fwht_regs_until<2 * NI, 2, NI>(e);
          const int slot = (wb << 1) >> N;            // component slot in tile
          const int64_t g = item0 + slot;
          const int xw = (wb << 1) & XMASK;           // x of element (i=0, j=0)
          if constexpr (MODE == MODE_EMIT) {
#pragma unroll
            for (int k = 0; k < NI; ++k) {
              const int p = e[k], q = e[k + NI];
              e[k] = (p + q) >> 1;                    // values are even after >= 1 stage
              e[k + NI] = (p - q) >> 1;
            }
            if (g < a.n_items) {
              const int64_t comp = g >> a.nbl;
              const int64_t base = (comp << (N + a.nbl)) + ((g & bmask) << N) + xw;
              uint32_t* dst = a.emit + (base >> 1);
#pragma unroll
              for (int i = 0; i < NI; ++i) dst[i << SH] = pack2(e[2 * i], e[2 * i + 1]);
            }
          } else {
            int mx = final_stage<NI, MODE>(e);
            if constexpr (MODE == MODE_SPEC) {
              if (g < a.n_items) {
                int32_t* dst = a.out + g * a.ld + xw;
#pragma unroll
                for (int i = 0; i < NI; ++i) {
                  dst[(i << (SH + 1))] = e[2 * i];
                  dst[(i << (SH + 1)) + 1] = e[2 * i + 1];
                }
              }
            }
            mx = warp_max(mx);
            if ((tid & 31) == 0) atomicMax(&s_max[slot], mx);
          }
        }
      };
      if (pass == 2) {
        run(std::integral_constant<int, B2>{}, std::integral_constant<int, 5>{});
      } else {
        run(std::integral_constant<int, (B3 > 0 ? B3 : 1)>{}, std::integral_constant<int, 10>{});
      }
      __syncthreads();
    }

    if constexpr (MODE != MODE_EMIT) {
      if (tid < C) {
        const int64_t g = item0 + tid;
        if (g < a.n_items) {
          const int mx = s_max[tid];
          a.max_abs[g] = mx;
          if (a.key) atomicMax(a.key, nl_key(mx, a.v_first + uint32_t(g)));
        }
      }
      __syncthreads();
    }
  }
}

// n = 1..6: one thread owns one whole component in registers.
template <int N, typename TT, int MODE>
__global__ void __launch_bounds__(256) k_fused_small(FusedArgs a) {
  constexpr int L = 1 << N;
  const TT* __restrict__ table = static_cast<const TT*>(a.table);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < a.n_items; base += stride) {
    const int64_t g = base + threadIdx.x;
    const bool ok = g < a.n_items;
    const uint32_t v = a.v_first + uint32_t(ok ? g : 0);
    int e[L];
#pragma unroll
    for (int x = 0; x < L; ++x) e[x] = polarity(uint32_t(__ldg(table + x)), v);
    fwht_regs<L, 1>(e);
    int mx = 0;
#pragma unroll
    for (int x = 0; x < L; ++x) mx = max(mx, abs(e[x]));
    if (ok) {
      a.max_abs[g] = mx;
      if constexpr (MODE == MODE_SPEC) {
        int32_t* dst = a.out + g * a.ld;
#pragma unroll
        for (int x = 0; x < L; ++x) dst[x] = e[x];
      }
    }
    if (a.key) {
      // warp-aggregate the (max, smallest v) key before one atomic
      const unsigned mask = __ballot_sync(0xffffffffu, ok);
      if (ok) {
        const int wmx = __reduce_max_sync(mask, mx);
        const unsigned vmin = __reduce_min_sync(mask, mx == wmx ? v : 0xFFFFFFFFu);
        if (v == vmin && mx == wmx) atomicMax(a.key, nl_key(wmx, vmin));
      }
    }
  }
}

}  // namespace sbw
