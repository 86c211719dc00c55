// Multi-pass driver for n = 17..24: per batch of components, pass A
// (generation + 15 on-chip stages, halved int16 to an L2-sized scratch) then
// pass B (stages 15..n-1 + fused max|W|).  Batches are sized so that the
// scratch of one batch stays resident in the 126 MB L2 between the two
// launches.
#include "sbw_passb.cuh"
#include "sbw_launch.h"

#include <cstdlib>
#include <mutex>

namespace sbw {

namespace {

// Scratch of BOTH in-flight batches (double buffer) stays within this many
// bytes so pass B reads what pass A just wrote from the 126 MB L2.
constexpr size_t kL2Budget = size_t(96) << 20;

int64_t batch_components(int n, uint32_t v_lo, uint32_t v_hi) {
  const int64_t per = int64_t(2) << n;  // u16 bytes per component
  int64_t bb = int64_t(kL2Budget / 2) / per;
  if (bb < 1) bb = 1;
  const int64_t total = int64_t(v_hi) - int64_t(v_lo);
  return bb < total ? bb : total;
}

// Two auxiliary streams per device: pass A of batch b+1 runs beside pass B of
// batch b, filling the SMs that each launch's tail leaves idle.
struct K3Streams {
  cudaStream_t a = nullptr, b = nullptr;
  cudaEvent_t fork = nullptr, done_a[2] = {nullptr, nullptr}, done_b[2] = {nullptr, nullptr};
};
K3Streams g_k3[64];
std::mutex g_k3_mu;
std::mutex g_k3_launch_mu[64];  // one enqueue at a time per device (shared events)

int k3_streams(int dev, K3Streams** out) {
  std::lock_guard<std::mutex> lk(g_k3_mu);
  K3Streams& s = g_k3[dev & 63];
  if (!s.a) {
    SBW_CUDA_CHECK(cudaStreamCreateWithFlags(&s.a, cudaStreamNonBlocking));
    SBW_CUDA_CHECK(cudaStreamCreateWithFlags(&s.b, cudaStreamNonBlocking));
    SBW_CUDA_CHECK(cudaEventCreateWithFlags(&s.fork, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      SBW_CUDA_CHECK(cudaEventCreateWithFlags(&s.done_a[i], cudaEventDisableTiming));
      SBW_CUDA_CHECK(cudaEventCreateWithFlags(&s.done_b[i], cudaEventDisableTiming));
    }
  }
  *out = &s;
  return SBW_OK;
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
  return planes_bytes(n, m) + 2 * size_t(batch_components(n, v_lo, v_hi)) * (size_t(2) << n);
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
  uint32_t* emit0 = reinterpret_cast<uint32_t*>(static_cast<char*>(scratch) + planes_bytes(n, m));
  uint32_t* emit[2] = {emit0, emit0 + size_t(bb) * (size_t(1) << (n - 1))};
  if (int rc = build_planes(table, tbytes, n, m, planes, st)) return rc;
  SBW_CUDA_CHECK(cudaMemsetAsync(max_abs, 0, sizeof(int32_t) * (size_t(v_hi) - v_lo), st));
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  K3Streams* ks = nullptr;
  if (int rc = k3_streams(dp.device, &ks)) return rc;
  std::lock_guard<std::mutex> launch_lock(g_k3_launch_mu[dp.device & 63]);
  static const bool single = getenv("SBW_K3_SINGLE_STREAM") != nullptr;  // debugging aid
  K3Streams one = *ks;
  if (single) {
    one.a = st;
    one.b = st;
    ks = &one;
  }
  // fork: both aux streams start after everything already queued on `st`
  SBW_CUDA_CHECK(cudaEventRecord(ks->fork, st));
  SBW_CUDA_CHECK(cudaStreamWaitEvent(ks->a, ks->fork, 0));
  SBW_CUDA_CHECK(cudaStreamWaitEvent(ks->b, ks->fork, 0));
  const int64_t total = int64_t(v_hi) - int64_t(v_lo);
  int64_t nb = 0;
  for (int64_t c0 = 0; c0 < total; c0 += bb, ++nb) {
    const int64_t nc = (total - c0) < bb ? (total - c0) : bb;
    const uint32_t vf = v_lo + uint32_t(c0);
    const int buf = int(nb & 1);
    if (nb >= 2) SBW_CUDA_CHECK(cudaStreamWaitEvent(ks->a, ks->done_b[buf], 0));  // buffer free
    if (int rc = launch_emit_tile(planes, n, m, vf, nc, emit[buf], ks->a)) return rc;
    SBW_CUDA_CHECK(cudaEventRecord(ks->done_a[buf], ks->a));
    SBW_CUDA_CHECK(cudaStreamWaitEvent(ks->b, ks->done_a[buf], 0));
    PassBArgs a{};
    a.scratch = emit[buf];
    a.n = n;
    a.n_comp = nc;
    a.out_row0 = c0;
    a.v_first = vf;
    a.max_abs = max_abs;
    a.key = key;
    a.out = out;
    a.ld = ld;
    const int rc = out ? dispatch_h<MODE_SPEC>(n - 15, a, ks->b) : dispatch_h<MODE_NL>(n - 15, a, ks->b);
    if (rc) return rc;
    SBW_CUDA_CHECK(cudaEventRecord(ks->done_b[buf], ks->b));
  }
  // join: `st` continues after the last pass B (which follows every pass A)
  SBW_CUDA_CHECK(cudaEventRecord(ks->fork, ks->b));
  SBW_CUDA_CHECK(cudaStreamWaitEvent(st, ks->fork, 0));
  return SBW_OK;
}

}  // namespace sbw
