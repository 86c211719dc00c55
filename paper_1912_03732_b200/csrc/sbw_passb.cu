// Multi-pass driver for n = 17..24: bit planes, then one persistent kernel
// that interleaves pass A (generation + 15 on-chip stages, biased u16 to an
// L2-resident ring of scratch slots) and pass B (stages 15..n-1 + fused
// max|W|) through an ordered work queue.  See sbw_passb.cuh.
#include <cstdio>
#include <cstdlib>

#include "sbw_launch.h"
#include "sbw_passb.cuh"

namespace sbw {

namespace {

// Ring of component scratch slots kept within this budget so that pass B
// reads what pass A just wrote from the 126 MB L2.
constexpr size_t kRingBudget = size_t(64) << 20;

// Lookahead D (components) so that >= ~3 waves of queue items separate A(c)
// from B(c): B(c) then rarely waits for its tiles.
int64_t lookahead(int n, int64_t ncomp) {
  const int64_t na = int64_t(1) << (n - 16);
  const int64_t nb = (n - 15) <= 5 ? (int64_t(1) << 14) / 512 : (int64_t(1) << 14) / 32;
  int64_t d = (3 * 148 + na + nb - 1) / (na + nb);
  if (d < 1) d = 1;
  if (d > ncomp) d = ncomp;
  return d;
}

int ring_slots(int n, int64_t ncomp) {
  const size_t per = size_t(2) << n;  // u16 bytes per component
  int64_t r = int64_t(kRingBudget / per);
  const int64_t need = lookahead(n, ncomp) + 2;  // R > D, plus one slot of slack (R = D + 1 measured slower)
  if (r < need) r = need;
  return int(r);
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

template <int H, int MODE>
int run_persistent(const K3Args& a, cudaStream_t st) {
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  auto kern = k3_persistent<H, MODE>;
  constexpr size_t kSmem = kK3Smem;  // 128 KiB tile / pass-B rows + 64 KiB staging
  static unsigned long long attr_done = 0;
  if (!(attr_done >> (dp.device & 63) & 1ull)) {
    SBW_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(kSmem)));
    attr_done |= 1ull << (dp.device & 63);
  }
  kern<<<dp.sm_count, 512, kSmem, st>>>(a);
  SBW_LAUNCH_CHECK("k3_persistent");
  return SBW_OK;
}

template <int MODE>
int dispatch_h(int h, const K3Args& a, cudaStream_t st) {
  switch (h) {
    case 2: return run_persistent<2, MODE>(a, st);
    case 3: return run_persistent<3, MODE>(a, st);
    case 4: return run_persistent<4, MODE>(a, st);
    case 5: return run_persistent<5, MODE>(a, st);
    case 6: return run_persistent<6, MODE>(a, st);
    case 7: return run_persistent<7, MODE>(a, st);
    case 8: return run_persistent<8, MODE>(a, st);
    case 9: return run_persistent<9, MODE>(a, st);
    default: return set_error(SBW_EINVAL, "multi-pass path needs n in 17..24");
  }
}

}  // namespace

size_t k3_scratch_bytes(int n, int m, uint32_t v_lo, uint32_t v_hi) {
  if (n < 17) return 0;
  const int64_t ncomp = int64_t(v_hi) - int64_t(v_lo);
  const size_t ring = size_t(ring_slots(n, ncomp)) * (size_t(2) << n);
  const size_t counters = sizeof(unsigned) * (1 + 2 * size_t(ncomp > 0 ? ncomp : 0));
  return planes_bytes(n, m) + align256(ring) + align256(counters);
}

int launch_k3(const void* table, int tbytes, int n, int m, uint32_t v_lo, uint32_t v_hi,
              int32_t* max_abs, unsigned long long* key, int32_t* out, int64_t ld, void* scratch,
              size_t scratch_bytes, cudaStream_t st) {
  if (n < 17 || n > 24) return set_error(SBW_EINVAL, "multi-pass path needs n in 17..24");
  if (v_hi <= v_lo) return SBW_OK;
  const int64_t ncomp = int64_t(v_hi) - int64_t(v_lo);
  const size_t need = k3_scratch_bytes(n, m, v_lo, v_hi);
  if (scratch == nullptr || scratch_bytes < need)
    return set_error(SBW_EINVAL, "n=%d needs a scratch workspace of %zu bytes, got %zu", n, need,
                     scratch_bytes);
  const int R = ring_slots(n, ncomp);
  char* base = static_cast<char*>(scratch);
  uint32_t* planes = reinterpret_cast<uint32_t*>(base);
  uint32_t* ring = reinterpret_cast<uint32_t*>(base + planes_bytes(n, m));
  unsigned* counters = reinterpret_cast<unsigned*>(base + planes_bytes(n, m) +
                                                   align256(size_t(R) * (size_t(2) << n)));
  if (int rc = build_planes(table, tbytes, n, m, planes, st)) return rc;
  SBW_CUDA_CHECK(cudaMemsetAsync(max_abs, 0, sizeof(int32_t) * size_t(ncomp), st));
  SBW_CUDA_CHECK(cudaMemsetAsync(counters, 0, sizeof(unsigned) * (1 + 2 * size_t(ncomp)), st));
  K3Args a{};
  a.ta.planes = planes;
  a.ta.plane_words = (int64_t(1) << n) >> 5;
  a.ta.m = m;
  a.ta.n_full = n;
  a.pb.n = n;
  a.pb.max_abs = max_abs;
  a.pb.key = key;
  a.pb.out = out;
  a.pb.ld = ld;
  a.v_lo = v_lo;
  a.ncomp = ncomp;
  a.ring = ring;
  a.ring_slots = R;
  a.lookahead = lookahead(n, ncomp);
  a.counters = counters;
  // SBW_K3_PROF=1 (debugging aid): per-item cycle accounting printed to stderr
  static const bool prof = getenv("SBW_K3_PROF") != nullptr;
  unsigned long long* dprof = nullptr;
  if (prof) {
    SBW_CUDA_CHECK(cudaMallocAsync(&dprof, 16 * sizeof(unsigned long long), st));
    SBW_CUDA_CHECK(cudaMemsetAsync(dprof, 0, 16 * sizeof(unsigned long long), st));
    a.prof = dprof;
    a.ta.phase_prof = dprof + 8;
  }
  const int rc = out ? dispatch_h<MODE_SPEC>(n - 15, a, st) : dispatch_h<MODE_NL>(n - 15, a, st);
  if (prof) {
    unsigned long long h[16];
    SBW_CUDA_CHECK(cudaMemcpyAsync(h, dprof, sizeof(h), cudaMemcpyDeviceToHost, st));
    SBW_CUDA_CHECK(cudaStreamSynchronize(st));
    cudaFreeAsync(dprof, st);
    fprintf(stderr,
            "[k3 prof] n=%d comps=%lld R=%d D=%lld | A items %llu avg %.0f cyc (wait %.0f) | "
            "B items %llu avg %.0f cyc (counter wait %.0f, stage wait %.0f, prefetched %llu)\n",
            n, (long long)ncomp, R, (long long)a.lookahead, h[5], h[5] ? double(h[0]) / h[5] : 0.0,
            h[5] ? double(h[1]) / h[5] : 0.0, h[6], h[6] ? double(h[2]) / h[6] : 0.0,
            h[6] ? double(h[3]) / h[6] : 0.0, h[6] ? double(h[4]) / h[6] : 0.0, h[7]);
    if (h[5])
      fprintf(stderr, "[k3 prof]   A tile phases: pass1 %.0f  pass2 %.0f  pass3+emit %.0f cyc\n",
              double(h[8]) / h[5], double(h[9]) / h[5], double(h[10]) / h[5]);
  }
  return rc;
}

}  // namespace sbw
