// Multi-pass driver for n = 17..24: bit planes, then per batch of components
// one pass-A launch (generation + 15 on-chip stages, biased u16 out) and one
// pass-B launch (stages 15..n-1 + fused max|W|).  Batch b+1's pass A runs on
// one stream beside batch b's pass B on another (double-buffered scratch).
// Measured: ~1 GiB batches beat L2-sized ones and a persistent
// work-queue kernel, because launches are few and both passes run at full
// occupancy; the scratch traffic (4 B / element) streams through HBM.
#include <cstdio>
#include <cstdlib>

#include "sbw_launch.h"
#include "sbw_passb.cuh"

#include <mutex>

namespace sbw {

namespace {

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// ---- batched two-kernel path for n = 17..24 ---------------------------------
// Two scratch buffers of `bb` components (~4 GiB each): pass A of batch b+1
// runs on one stream beside pass B of batch b on another.  Each batch pays a
// fixed ~20-30 us (kernel prologues, pipeline fill, launch gaps), so bigger
// batches win: 24x16 full NL 1000 / 938 / 906 / 896 ms at 0.5 / 1 / 2 / 4 GiB,
// 20x20 860 / 843 / 836 / 830 ms (SBW_K3_BATCH sweep).
constexpr size_t kBatchBytes = size_t(4) << 30;  // per buffer

// Smallest n whose NL pass B runs on the tensor cores (SBW_PASSB_TC_MIN_N
// overrides).  Below n = 21 the GEMM is block-diagonal (H_(2^H) (x) I_P) and
// does P times the useful MACs: at 20x20 the kernel alone is 4 % faster than
// k_passb_regs (689 vs 717 us per 4 GiB batch, both HBM-bound) but the full
// run is 5 % slower (870 vs 830 ms; the tensor work lowers the clock under
// the power cap), so n <= 20 keeps the fp32 register kernel.
const int kPassBTcMinN = [] {
  const char* e = getenv("SBW_PASSB_TC_MIN_N");
  return e ? atoi(e) : 21;
}();

int64_t batch_components(int n, int64_t total) {
  static const char* env = getenv("SBW_K3_BATCH");  // tuning aid: components per batch
  int64_t bb = env ? atoll(env) : int64_t(kBatchBytes / (size_t(2) << n));
  if (bb < 1) bb = 1;
  return bb < total ? bb : total;
}

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
int run_passb_regs(const PassBArgs& a, cudaStream_t st) {
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  // one resident wave: each CTA owns a contiguous item range
  static int per_sm[64][10][2] = {};
  int& occ = per_sm[dp.device & 63][H][MODE == MODE_NL ? 0 : 1];
  if (occ == 0)
    SBW_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_passb_regs<H, MODE>,
                                                                 kPassBThreads, 0));
  const int64_t ctas = a.n_comp * ((int64_t(1) << 14) / kPassBThreads);
  const int64_t cap = int64_t(dp.sm_count) * (occ > 0 ? occ : 1);
  k_passb_regs<H, MODE><<<int(ctas < cap ? ctas : cap), kPassBThreads, 0, st>>>(a);
  SBW_LAUNCH_CHECK("k_passb_regs");
  return SBW_OK;
}

template <int H, int MODE>
int run_passb_staged(const PassBArgs& a, cudaStream_t st) {
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  auto kern = k_passb_staged<H, MODE>;
  static unsigned long long attr_done = 0;
  if (!(attr_done >> (dp.device & 63) & 1ull)) {
    SBW_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(kStagedSmem)));
    attr_done |= 1ull << (dp.device & 63);
  }
  const int64_t items = a.n_comp * StagedShape<H>::PER_COMP;
  const int64_t slots = 2 * int64_t(dp.sm_count);  // two CTAs per SM
  const int grid = int(items < slots ? items : slots);
  kern<<<grid, kStagedThreads, kStagedSmem, st>>>(a);
  SBW_LAUNCH_CHECK("k_passb_staged");
  return SBW_OK;
}

template <int MODE>
int dispatch_passb_regs(int h, const PassBArgs& a, cudaStream_t st) {
  switch (h) {
    case 2: return run_passb_regs<2, MODE>(a, st);
    case 3: return run_passb_regs<3, MODE>(a, st);
    case 4: return run_passb_regs<4, MODE>(a, st);
    case 5: return run_passb_regs<5, MODE>(a, st);
    case 6: return run_passb_staged<6, MODE>(a, st);
    case 7: return run_passb_staged<7, MODE>(a, st);
    case 8: return run_passb_staged<8, MODE>(a, st);
    case 9: return run_passb_staged<9, MODE>(a, st);
    default: return set_error(SBW_EINVAL, "batched path needs n in 17..24");
  }
}

int launch_k3_batched(const uint32_t* planes, int n, int m, uint32_t v_lo, uint32_t v_hi,
                      int32_t* max_abs, unsigned long long* key, int32_t* out, int64_t ld,
                      uint32_t* bufs, cudaStream_t st) {
  const int64_t total = int64_t(v_hi) - int64_t(v_lo);
  const int64_t bb = batch_components(n, total);
  uint32_t* emit[2] = {bufs, bufs + size_t(bb) * (size_t(1) << (n - 1))};
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  K3Streams* ks = nullptr;
  if (int rc = k3_streams(dp.device, &ks)) return rc;
  std::lock_guard<std::mutex> launch_lock(g_k3_launch_mu[dp.device & 63]);
  // fork: both aux streams start after everything already queued on `st`
  SBW_CUDA_CHECK(cudaEventRecord(ks->fork, st));
  SBW_CUDA_CHECK(cudaStreamWaitEvent(ks->a, ks->fork, 0));
  SBW_CUDA_CHECK(cudaStreamWaitEvent(ks->b, ks->fork, 0));
  int64_t nb = 0;
  for (int64_t c0 = 0; c0 < total; c0 += bb, ++nb) {
    const int64_t nc = (total - c0) < bb ? (total - c0) : bb;
    const uint32_t vf = v_lo + uint32_t(c0);
    const int buf = int(nb & 1);
    if (nb >= 2) SBW_CUDA_CHECK(cudaStreamWaitEvent(ks->a, ks->done_b[buf], 0));  // buffer free
    if (int rc = (out == nullptr && tc_path_enabled())
                     ? launch_tc_emit(planes, n, vf, nc, emit[buf], ks->a)
                     : launch_emit_tiles(planes, n, m, vf, nc, emit[buf], ks->a))
      return rc;
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
    const int rc = out ? dispatch_passb_regs<MODE_SPEC>(n - 15, a, ks->b)
                       : (n >= kPassBTcMinN && passb_tc_enabled()) ? launch_passb_tc(a, ks->b)
                                                         : dispatch_passb_regs<MODE_NL>(n - 15, a, ks->b);
    if (rc) return rc;
    SBW_CUDA_CHECK(cudaEventRecord(ks->done_b[buf], ks->b));
  }
  // join: `st` continues after the last pass B (which follows every pass A)
  SBW_CUDA_CHECK(cudaEventRecord(ks->fork, ks->b));
  SBW_CUDA_CHECK(cudaStreamWaitEvent(st, ks->fork, 0));
  return SBW_OK;
}

}  // namespace

size_t k3_scratch_bytes(int n, int m, uint32_t v_lo, uint32_t v_hi) {
  if (n < 17) return 0;
  const int64_t ncomp = int64_t(v_hi) - int64_t(v_lo);
  // bit planes + two batch buffers of biased u16 partial transforms
  return planes_bytes(n, m) +
         align256(2 * size_t(batch_components(n, ncomp > 0 ? ncomp : 1)) * (size_t(2) << n));
}

int launch_k3(const void* table, int tbytes, int n, int m, uint32_t v_lo, uint32_t v_hi,
              int32_t* max_abs, unsigned long long* key, int32_t* out, int64_t ld, void* scratch,
              size_t scratch_bytes, cudaStream_t st) {
  if (n < 17 || n > 24) return set_error(SBW_EINVAL, "multi-pass path needs n in 17..24");
  if (v_hi <= v_lo) return SBW_OK;
  const size_t need = k3_scratch_bytes(n, m, v_lo, v_hi);
  if (scratch == nullptr || scratch_bytes < need)
    return set_error(SBW_EINVAL, "n=%d needs a scratch workspace of %zu bytes, got %zu", n, need,
                     scratch_bytes);
  char* base = static_cast<char*>(scratch);
  uint32_t* planes = reinterpret_cast<uint32_t*>(base);
  uint32_t* bufs = reinterpret_cast<uint32_t*>(base + planes_bytes(n, m));
  if (int rc = build_planes(table, tbytes, n, m, planes, st)) return rc;
  SBW_CUDA_CHECK(cudaMemsetAsync(max_abs, 0, sizeof(int32_t) * (size_t(v_hi) - v_lo), st));
  return launch_k3_batched(planes, n, m, v_lo, v_hi, max_abs, key, out, ld, bufs, st);
}

}  // namespace sbw
