// Fused "generate component -> FWHT -> max|W| (or materialise)" kernels.
//
// Replaces, per output mask v, the reference's
//   polarity_row            pkg/src/sboxeval/sbox.py:145-152
//   fwht_column_in_place    pkg/src/sboxeval/walsh.py:73-104
//   column_nonlinearity     pkg/src/sboxeval/walsh.py:107-114
// driven by fwht_fused / fwht_parallel (walsh.py:204-248, parallel.py:64-133).
//
// This header holds the shared mode/argument definitions and the n <= 6
// kernel (one thread per component, popcount generation); the n = 7..16
// tile kernel is in sbw_tile_simd.cuh and the n >= 17 pass B in sbw_passb.cuh.
#pragma once

#include <type_traits>

#include "sbw_internal.cuh"

namespace sbw {

constexpr int kTileThreads = 1024;
constexpr int kTileWords = 1 << 15;  // 2^16 int16 elements as 32-bit pairs

enum FusedMode { MODE_NL = 0, MODE_SPEC = 1, MODE_EMIT = 2 };

struct FusedArgs {
  const void* table;
  uint32_t v_first;       // mask of item 0
  int64_t n_items;        // (component, block) items
  int32_t* max_abs;       // [item] for NL / SPEC
  unsigned long long* key;
  int32_t* out;           // SPEC: out[item * ld + x]
  int64_t ld;
};

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
