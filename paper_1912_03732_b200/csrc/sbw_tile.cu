// Instantiation and dispatch of the fused on-chip kernels (n = 1..16) and of
// pass A of the multi-pass path.  See sbw_fused.cuh for the algorithm.
#include "sbw_fused.cuh"
#include "sbw_launch.h"

namespace sbw {

namespace {

constexpr size_t kTileSmem = size_t(kTileWords) * sizeof(uint32_t);  // 128 KiB

template <int N, typename TT, int MODE>
int run_tile(const FusedArgs& a, cudaStream_t st) {
  auto kern = k_fused_tile<N, TT, MODE>;
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  // per (instantiation, device); the attribute call is idempotent, so a race is benign
  static unsigned long long attr_done = 0;
  if (!(attr_done >> (dp.device & 63) & 1ull)) {
    SBW_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(kTileSmem)));
    attr_done |= 1ull << (dp.device & 63);
  }
  constexpr int C = 1 << (16 - N);
  const int64_t ntiles = (a.n_items + C - 1) / C;
  const int grid = int(ntiles < dp.sm_count ? ntiles : dp.sm_count);
  if (grid == 0) return SBW_OK;
  kern<<<grid, kTileThreads, kTileSmem, st>>>(a);
  SBW_LAUNCH_CHECK("k_fused_tile");
  return SBW_OK;
}

template <int N, typename TT, int MODE>
int run_small(const FusedArgs& a, cudaStream_t st) {
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  int64_t blocks = (a.n_items + 255) / 256;
  const int64_t cap = int64_t(dp.sm_count) * 8;
  if (blocks > cap) blocks = cap;
  if (blocks == 0) return SBW_OK;
  k_fused_small<N, TT, MODE><<<int(blocks), 256, 0, st>>>(a);
  SBW_LAUNCH_CHECK("k_fused_small");
  return SBW_OK;
}

template <typename TT, int MODE>
int dispatch_n(int n, const FusedArgs& a, cudaStream_t st) {
  switch (n) {
    case 1: return run_small<1, TT, MODE>(a, st);
    case 2: return run_small<2, TT, MODE>(a, st);
    case 3: return run_small<3, TT, MODE>(a, st);
    case 4: return run_small<4, TT, MODE>(a, st);
    case 5: return run_small<5, TT, MODE>(a, st);
    case 6: return run_small<6, TT, MODE>(a, st);
    case 7: return run_tile<7, TT, MODE>(a, st);
    case 8: return run_tile<8, TT, MODE>(a, st);
    case 9: return run_tile<9, TT, MODE>(a, st);
    case 10: return run_tile<10, TT, MODE>(a, st);
    case 11: return run_tile<11, TT, MODE>(a, st);
    case 12: return run_tile<12, TT, MODE>(a, st);
    case 13: return run_tile<13, TT, MODE>(a, st);
    case 14: return run_tile<14, TT, MODE>(a, st);
    case 15: return run_tile<15, TT, MODE>(a, st);
    case 16: return run_tile<16, TT, MODE>(a, st);
    default: return set_error(SBW_EINVAL, "on-chip path needs n in 1..16, got %d", n);
  }
}

}  // namespace

int launch_fused_onchip(const void* table, int tbytes, int n, uint32_t v_lo, uint32_t v_hi,
                        int32_t* max_abs, unsigned long long* key, int32_t* out, int64_t ld,
                        cudaStream_t st) {
  FusedArgs a{};
  a.table = table;
  a.v_first = v_lo;
  a.nbl = 0;
  a.n_items = int64_t(v_hi) - int64_t(v_lo);
  a.max_abs = max_abs;
  a.key = key;
  a.out = out;
  a.ld = ld;
  a.emit = nullptr;
  if (a.n_items <= 0) return SBW_OK;
  if (out) {
    return tbytes == 2 ? dispatch_n<uint16_t, MODE_SPEC>(n, a, st)
                       : dispatch_n<uint32_t, MODE_SPEC>(n, a, st);
  }
  return tbytes == 2 ? dispatch_n<uint16_t, MODE_NL>(n, a, st)
                     : dispatch_n<uint32_t, MODE_NL>(n, a, st);
}

int launch_emit_tile(const void* table, int tbytes, int n, uint32_t v_first, int64_t n_comp,
                     uint32_t* emit, cudaStream_t st) {
  FusedArgs a{};
  a.table = table;
  a.v_first = v_first;
  a.nbl = n - 15;
  a.n_items = n_comp << (n - 15);
  a.emit = emit;
  return tbytes == 2 ? run_tile<15, uint16_t, MODE_EMIT>(a, st)
                     : run_tile<15, uint32_t, MODE_EMIT>(a, st);
}

}  // namespace sbw
