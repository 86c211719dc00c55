// Multi-pass driver for n = 17..24: per batch of components, pass A
// (generation + 15 on-chip stages, halved int16 to an L2-sized scratch) then
// pass B (stages 15..n-1 + fused max|W|).  Batches are sized so that the
// scratch of one batch stays resident in the 126 MB L2 between the two
// launches.
#include "sbw_passb.cuh"
#include "sbw_launch.h"

namespace sbw {

namespace {

constexpr size_t kL2Budget = size_t(64) << 20;  // bytes of scratch per batch

int64_t batch_components(int n, uint32_t v_lo, uint32_t v_hi) {
  const int64_t per = int64_t(2) << n;  // int16 bytes per component
  int64_t bb = int64_t(kL2Budget) / per;
  if (bb < 1) bb = 1;
  const int64_t total = int64_t(v_hi) - int64_t(v_lo);
  return bb < total ? bb : total;
}

template <int H, int MODE>
int run_passb(const PassBArgs& a, cudaStream_t st) {
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  if constexpr (H <= 5) {
    const int64_t ctas = a.n_comp * ((int64_t(1) << 14) / kPassBThreads);
    const int64_t cap = int64_t(dp.sm_count) * 8;
    const int grid = int(ctas < cap ? ctas : cap);
    k_passb_regs<H, MODE><<<grid, kPassBThreads, 0, st>>>(a);
    SBW_LAUNCH_CHECK("k_passb_regs");
  } else {
    auto kern = k_passb_smem<H, MODE>;
    const size_t smem = size_t(1) << (H + 5 + 3);  // 2^H rows x 32 int2
    static unsigned long long attr_done = 0;
    if (!(attr_done >> (dp.device & 63) & 1ull)) {
      SBW_CUDA_CHECK(
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
      attr_done |= 1ull << (dp.device & 63);
    }
    const int64_t ctas = a.n_comp * ((int64_t(1) << 14) / 32);
    const int64_t cap = int64_t(dp.sm_count) * (smem > (size_t(96) << 10) ? 1 : 2);
    const int grid = int(ctas < cap ? ctas : cap);
    kern<<<grid, 512, smem, st>>>(a);
    SBW_LAUNCH_CHECK("k_passb_smem");
  }
  return SBW_OK;
}

template <int MODE>
int dispatch_h(int h, const PassBArgs& a, cudaStream_t st) {
  switch (h) {
    case 2: return run_passb<2, MODE>(a, st);
    case 3: return run_passb<3, MODE>(a, st);
    case 4: return run_passb<4, MODE>(a, st);
    case 5: return run_passb<5, MODE>(a, st);
    case 6: return run_passb<6, MODE>(a, st);
    case 7: return run_passb<7, MODE>(a, st);
    case 8: return run_passb<8, MODE>(a, st);
    case 9: return run_passb<9, MODE>(a, st);
    default: return set_error(SBW_EINVAL, "multi-pass path needs n in 17..24");
  }
}

}  // namespace

size_t k3_scratch_bytes(int n, int m, uint32_t v_lo, uint32_t v_hi) {
  if (n < 17) return 0;
  return planes_bytes(n, m) + size_t(batch_components(n, v_lo, v_hi)) * (size_t(2) << n);
}

int launch_k3(const void* table, int tbytes, int n, int m, uint32_t v_lo, uint32_t v_hi,
              int32_t* max_abs, unsigned long long* key, int32_t* out, int64_t ld, void* scratch,
              size_t scratch_bytes, cudaStream_t st) {
  if (n < 17 || n > 24) return set_error(SBW_EINVAL, "multi-pass path needs n in 17..24");
  if (v_hi <= v_lo) return SBW_OK;
  const int64_t bb = batch_components(n, v_lo, v_hi);
  const size_t need = k3_scratch_bytes(n, m, v_lo, v_hi);
  if (scratch == nullptr || scratch_bytes < need)
    return set_error(SBW_EINVAL, "n=%d needs a scratch workspace of %zu bytes, got %zu", n, need,
                     scratch_bytes);
  uint32_t* planes = static_cast<uint32_t*>(scratch);
  uint32_t* emit = reinterpret_cast<uint32_t*>(static_cast<char*>(scratch) + planes_bytes(n, m));
  if (int rc = build_planes(table, tbytes, n, m, planes, st)) return rc;
  SBW_CUDA_CHECK(cudaMemsetAsync(max_abs, 0, sizeof(int32_t) * (size_t(v_hi) - v_lo), st));
  for (int64_t c0 = 0; c0 < int64_t(v_hi) - int64_t(v_lo); c0 += bb) {
    const int64_t nc = (int64_t(v_hi) - int64_t(v_lo) - c0) < bb
                           ? (int64_t(v_hi) - int64_t(v_lo) - c0)
                           : bb;
    const uint32_t vf = v_lo + uint32_t(c0);
    if (int rc = launch_emit_tile(planes, n, m, vf, nc, emit, st)) return rc;
    PassBArgs a{};
    a.scratch = emit;
    a.n = n;
    a.n_comp = nc;
    a.out_row0 = c0;
    a.v_first = vf;
    a.max_abs = max_abs;
    a.key = key;
    a.out = out;
    a.ld = ld;
    const int rc = out ? dispatch_h<MODE_SPEC>(n - 15, a, st) : dispatch_h<MODE_NL>(n - 15, a, st);
    if (rc) return rc;
  }
  return SBW_OK;
}

}  // namespace sbw
