// Dispatch of the fused on-chip kernels (n = 1..16) and of pass A of the
// multi-pass path; bit-plane construction.  See sbw_tile_simd.cuh.
#include <cstdio>
#include <cstdlib>

#include "sbw_launch.h"
#include "sbw_tile_simd.cuh"

namespace sbw {

namespace {

constexpr size_t kTileSmem = size_t(kTileWords) * sizeof(uint32_t);  // 128 KiB

// planes[i][w] bit b = bit i of S(32 w + b): one warp per 32 inputs, a ballot per plane.
template <typename TT>
__global__ void __launch_bounds__(256) k_build_planes(const TT* __restrict__ table, int n, int m,
                                                      uint32_t* __restrict__ planes) {
  const int64_t words = (int64_t(1) << n) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < words; w += warps) {
    const uint32_t s = uint32_t(table[(w << 5) + lane]);
    for (int i = 0; i < m; ++i) {
      const uint32_t b = __ballot_sync(0xffffffffu, (s >> i) & 1u);
      if (lane == 0) planes[int64_t(i) * words + w] = b;
    }
  }
}

template <int N, int MODE>
int run_tile(const TileArgs& a, int64_t ntiles, cudaStream_t st) {
  // materialising (SPEC) tiles are store-bound and need more registers for
  // the int32 epilogue: 512 threads; fused NL tiles: 1024 threads
  constexpr int THREADS = MODE == MODE_SPEC ? 512 : kTileThreads;
  auto kern = k_tile_simd<N, MODE, THREADS>;
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  // per (instantiation, device); the attribute call is idempotent, so a race is benign
  static unsigned long long attr_done = 0;
  if (!(attr_done >> (dp.device & 63) & 1ull)) {
    SBW_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(kTileSmem)));
    attr_done |= 1ull << (dp.device & 63);
  }
  const int grid = int(ntiles < dp.sm_count ? ntiles : dp.sm_count);
  if (grid <= 0) return SBW_OK;
  kern<<<grid, THREADS, kTileSmem, st>>>(a);
  SBW_LAUNCH_CHECK("k_tile_simd");
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
int dispatch_small(int n, const FusedArgs& a, cudaStream_t st) {
  switch (n) {
    case 1: return run_small<1, TT, MODE>(a, st);
    case 2: return run_small<2, TT, MODE>(a, st);
    case 3: return run_small<3, TT, MODE>(a, st);
    case 4: return run_small<4, TT, MODE>(a, st);
    case 5: return run_small<5, TT, MODE>(a, st);
    case 6: return run_small<6, TT, MODE>(a, st);
    default: return set_error(SBW_EINVAL, "small path needs n in 1..6, got %d", n);
  }
}

template <int MODE>
int dispatch_tile(int n, const TileArgs& a, int64_t nt, cudaStream_t st) {
  switch (n) {
    case 7: return run_tile<7, MODE>(a, nt, st);
    case 8: return run_tile<8, MODE>(a, nt, st);
    case 9: return run_tile<9, MODE>(a, nt, st);
    case 10: return run_tile<10, MODE>(a, nt, st);
    case 11: return run_tile<11, MODE>(a, nt, st);
    case 12: return run_tile<12, MODE>(a, nt, st);
    case 13: return run_tile<13, MODE>(a, nt, st);
    case 14: return run_tile<14, MODE>(a, nt, st);
    case 15: return run_tile<15, MODE>(a, nt, st);
    case 16: return run_tile<16, MODE>(a, nt, st);
    default: return set_error(SBW_EINVAL, "tile path needs n in 7..16, got %d", n);
  }
}

}  // namespace

size_t planes_bytes(int n, int m) {
  if (n < 7) return 0;
  const size_t b = size_t(m) * ((size_t(1) << n) / 8);
  return (b + 255) & ~size_t(255);
}

int build_planes(const void* table, int tbytes, int n, int m, uint32_t* planes, cudaStream_t st) {
  if (n < 5) return set_error(SBW_EINVAL, "bit planes need n >= 5");
  const int64_t words = (int64_t(1) << n) >> 5;
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  int64_t blocks = (words + 7) / 8;
  if (blocks > int64_t(dp.sm_count) * 16) blocks = int64_t(dp.sm_count) * 16;
  if (tbytes == 2)
    k_build_planes<uint16_t><<<int(blocks), 256, 0, st>>>(static_cast<const uint16_t*>(table), n,
                                                          m, planes);
  else
    k_build_planes<uint32_t><<<int(blocks), 256, 0, st>>>(static_cast<const uint32_t*>(table), n,
                                                          m, planes);
  SBW_LAUNCH_CHECK("k_build_planes");
  return SBW_OK;
}

int launch_fused_onchip(const void* table, int tbytes, int n, int m, uint32_t v_lo, uint32_t v_hi,
                        int32_t* max_abs, unsigned long long* key, int32_t* out, int64_t ld,
                        void* scratch, cudaStream_t st) {
  if (v_hi <= v_lo) return SBW_OK;
  if (n <= 6) {
    FusedArgs a{};
    a.table = table;
    a.v_first = v_lo;
    a.n_items = int64_t(v_hi) - int64_t(v_lo);
    a.max_abs = max_abs;
    a.key = key;
    a.out = out;
    a.ld = ld;
    if (out)
      return tbytes == 2 ? dispatch_small<uint16_t, MODE_SPEC>(n, a, st)
                         : dispatch_small<uint32_t, MODE_SPEC>(n, a, st);
    return tbytes == 2 ? dispatch_small<uint16_t, MODE_NL>(n, a, st)
                       : dispatch_small<uint32_t, MODE_NL>(n, a, st);
  }
  uint32_t* planes = static_cast<uint32_t*>(scratch);
  if (int rc = build_planes(table, tbytes, n, m, planes, st)) return rc;
  if (n >= tc_min_small_n() && n <= 15 && m >= 16 - n && tc_path_enabled())
    return out == nullptr ? launch_tc_nl_small(planes, n, v_lo, v_hi, max_abs, key, st)
                          : launch_tc_spec_small(planes, n, v_lo, v_hi, max_abs, out, ld, st);
  if (n == 16 && tc_path_enabled())
    return out == nullptr ? launch_tc16_nl(planes, v_lo, v_hi, max_abs, key, st)
                          : launch_tc16_spec(planes, v_lo, v_hi, max_abs, out, ld, st);
  TileArgs a{};
  a.planes = planes;
  a.plane_words = (int64_t(1) << n) >> 5;
  a.m = m;
  a.v_lo = v_lo;
  a.v_hi = v_hi;
  const int j = 16 - n;
  a.t_begin = int64_t(v_lo) >> j;
  a.t_count = ((int64_t(v_hi) - 1) >> j) + 1 - a.t_begin;
  a.max_abs = max_abs;
  a.key = key;
  a.out = out;
  a.ld = ld;
#if SBW_PHASE_PROF
  // debug builds: per-phase cycle accounting of the on-chip tiles (SBW_K3_PROF=1)
  unsigned long long* dprof = nullptr;
  if (getenv("SBW_K3_PROF")) {
    SBW_CUDA_CHECK(cudaMallocAsync(&dprof, 4 * sizeof(unsigned long long), st));
    SBW_CUDA_CHECK(cudaMemsetAsync(dprof, 0, 4 * sizeof(unsigned long long), st));
    a.phase_prof = dprof;
  }
#endif
  const int rc = out ? dispatch_tile<MODE_SPEC>(n, a, a.t_count, st)
                     : dispatch_tile<MODE_NL>(n, a, a.t_count, st);
#if SBW_PHASE_PROF
  if (dprof) {
    unsigned long long h[4];
    SBW_CUDA_CHECK(cudaMemcpyAsync(h, dprof, sizeof(h), cudaMemcpyDeviceToHost, st));
    SBW_CUDA_CHECK(cudaStreamSynchronize(st));
    cudaFreeAsync(dprof, st);
    const double nt = double(a.t_count);
    fprintf(stderr, "[tile prof] n=%d tiles=%lld pass1 %.0f pass2 %.0f pass3 %.0f cyc/tile\n", n,
            (long long)a.t_count, h[0] / nt, h[1] / nt, h[2] / nt);
  }
#endif
  return rc;
}

int launch_emit_tiles(const uint32_t* planes, int n, int m, uint32_t v_first, int64_t n_comp,
                      uint32_t* emit, cudaStream_t st) {
  TileArgs a{};
  a.planes = planes;
  a.plane_words = (int64_t(1) << n) >> 5;
  a.m = m;
  a.v_first = v_first;
  a.n_comp = n_comp;
  a.n_full = n;
  a.emit = emit;
  a.t_begin = 0;
  a.t_count = n_comp << (n - 16);  // (block pair, component) tiles, component fastest
  return run_tile<15, MODE_EMIT>(a, a.t_count, st);
}

}  // namespace sbw
