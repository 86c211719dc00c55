// Multi-pass driver for n = 17..24: bit planes, then per batch of components
// one pass-A launch (generation + 15 on-chip stages, biased u16 out) and one
// pass-B launch (stages 15..n-1 + fused max|W|).  Batch b+1's pass A runs on
// one stream beside batch b's pass B on another (double-buffered scratch).
// Measured: ~1 GiB batches beat L2-sized ones and a persistent
// work-queue kernel, because launches are few and both passes run at full
// occupancy; the scratch traffic (4 B / element) streams through HBM.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "sbw_internal.cuh"
#include "sbw_launch.h"
#include "sbw_passb.cuh"

#include <mutex>
#include <vector>

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

// ---- L2 ring (n = 17..21, NL; SBW_K3_RING=1, off by default) ---------------
// Pass A and pass B run concurrently on disjoint SMs (pass B launched first
// with NB CTAs, pass A with NA; one CTA per SM each, NA + NB <= SMs, so both
// are resident) and hand batches of Bc components through R slots of scratch
// that stay in L2 instead of streaming 4 B / element through HBM (RingArgs,
// sbw_internal.cuh).  Bit-exact, but measured slower than the batched path
// (20x20, 32768 masks: 28.2 vs 25.9 ms at the best split NA = 64, L = 4,
// R = 3): an SM writes to L2 at ~32 B/clk (tools/micro/l2_bw.cu: 62 GB/s per
// SM), so pass A's 128 KiB per item costs as much as its arithmetic, and pass
// B's ~0.9 us per 32 KiB item is its own compute/issue limit, so the SMs
// split between the two passes do no better than all SMs alternating.
struct RingPlan {
  bool on = false;
  RingArgs r{};
  size_t ring_bytes = 0, counter_bytes = 0;
};

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

RingPlan ring_plan(int n, int64_t total, int sm_count) {
  RingPlan p;
  const int enabled = env_int("SBW_K3_RING", 0);  // read per call (A/B runs)
  if (!enabled || n < 17 || n > 21 || !tc_path_enabled() || !passb_tc_enabled()) return p;
  const int log_t = n - 16, T = 1 << log_t;
  const int q = std::max(1, env_int("SBW_K3_NA", 64) / T);
  const int na = q * T;
  const int nb = std::min(env_int("SBW_K3_NB", sm_count - na), sm_count - na);
  if (nb < 1) return p;
  const int L = std::max(1, env_int("SBW_K3_RING_L", 4));
  const int R = std::max(2, env_int("SBW_K3_RING_R", 3));
  const int bc = q * L;
  const int64_t batches = total / bc;
  const int64_t per_comp_b = int64_t(2) << (n - 15);  // k_passb_tc items per component (H <= 7)
  if (batches < 2 * R || int64_t(bc) * per_comp_b < nb) return p;
  p.on = true;
  p.r.on = 1;
  p.r.R = R;
  p.r.L = L;
  p.r.q = q;
  p.r.log_t = log_t;
  p.r.batches = batches;
  p.r.bc = bc;
  p.r.na = uint32_t(na);
  p.r.nb = uint32_t(nb);
  p.ring_bytes = align256(size_t(R) * bc * (size_t(2) << n));
  p.counter_bytes = align256(sizeof(uint32_t) * (2 * size_t(batches) + 1)) + 256;  // + wait_ns[2]
  return p;
}

__global__ void k_ring_poison(const uint32_t* err, int32_t* max_abs, int64_t count) {
  if (*err == 0u) return;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
    max_abs[i] = -1;  // odd gap: the NL conversion reports the failure
}

int64_t batch_components(int n, int64_t total) {
  static const char* env = getenv("SBW_K3_BATCH");  // tuning aid: components per batch
  int64_t bb = env ? atoll(env) : int64_t(kBatchBytes / (size_t(2) << n));
  if (bb < 1) bb = 1;
  return bb < total ? bb : total;
}

struct K3Streams {
  cudaStream_t a = nullptr, b = nullptr;
  cudaEvent_t fork = nullptr, done_a[2] = {nullptr, nullptr}, done_b[2] = {nullptr, nullptr};
  int* flags = nullptr;  // [2]: per scratch buffer, "a tile of this batch wrapped at stage 16"
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
    SBW_CUDA_CHECK(cudaMalloc(&s.flags, 2 * sizeof(int)));
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

// SBW_PASSB_BULK=0 keeps k_passb_regs for the H <= 5 NL pass B.
bool passb_bulk_enabled() {
  static const bool on = [] {
    const char* e = getenv("SBW_PASSB_BULK");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int H>
int run_passb_bulk(const PassBArgs& a, cudaStream_t st) {
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  constexpr int smem = bulk_smem_bytes<H>();
  static int occ_dev[64] = {};
  int& occ = occ_dev[dp.device & 63];
  if (occ == 0) {
    SBW_CUDA_CHECK(cudaFuncSetAttribute(k_passb_bulk<H>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    SBW_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_passb_bulk<H>, kBulkThreads, smem));
  }
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(tma_encode_ptr());
  if (!enc) return set_error(SBW_ECUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  const cuuint64_t dims[2] = {cuuint64_t(1) << (14 + a.e16), cuuint64_t(a.n_comp) << H};
  const cuuint64_t strides[1] = {cuuint64_t(4) << (14 + a.e16)};
  const cuuint32_t box[2] = {cuuint32_t(kBulkThreads), cuuint32_t(1 << H)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(a.scratch), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(SBW_ECUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  const int64_t ctas = a.n_comp * ((int64_t(1) << (14 + a.e16)) / kBulkThreads);
  const int64_t cap = int64_t(dp.sm_count) * (occ > 0 ? occ : 1);
  k_passb_bulk<H><<<int(ctas < cap ? ctas : cap), kBulkThreads, smem, st>>>(map, a);
  SBW_LAUNCH_CHECK("k_passb_bulk");
  return SBW_OK;
}

template <int MODE>
int dispatch_passb_regs(int h, const PassBArgs& a, cudaStream_t st) {
  if (MODE == MODE_NL && h <= 5 && passb_bulk_enabled()) {
    switch (h) {
      case 2: return run_passb_bulk<2>(a, st);
      case 3: return run_passb_bulk<3>(a, st);
      case 4: return run_passb_bulk<4>(a, st);
      case 5: return run_passb_bulk<5>(a, st);
      default: break;
    }
  }
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
  // SBW_K3_TRACE=1 (development aid): timing events around every pass A /
  // pass B launch, synchronised and summarised on stderr at the end.
  static const bool trace = getenv("SBW_K3_TRACE") != nullptr;
  std::vector<cudaEvent_t> ev;
  auto mark = [&](cudaStream_t s) {
    if (!trace) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, s);
    ev.push_back(e);
  };
  // NL with the tensor-core pass A: Gray-ordered components (PassBArgs::gray)
  const bool gray = out == nullptr && tc_path_enabled();
  // 16 stages in pass A (n >= 18; pass B k_passb_regs for n <= 20, k_passb_tc
  // above): pass B does one stage less.  A batch in which some tile wrapped
  // at stage 16 (|W_16| = 2^16: the component is affine on that tile) is
  // redone by gated 15-stage launches; the gates read a device flag, so no
  // host synchronisation is needed.  Off by default (SBW_K3_EMIT16=1 enables
  // it): bit-identical, but measured no faster -- 20x20 928 vs 927 ms, 24x16
  // 978 vs 956 ms, 18x18 67 vs 57 ms -- the extra stage and wrap check cost
  // pass A what pass B saves, plus two gated launches per batch.
  const bool tc_b = n >= kPassBTcMinN && passb_tc_enabled();
  const bool e16 = gray && n >= 18 && (tc_b || n <= 20) && env_int("SBW_K3_EMIT16", 0) != 0;
  // SBW_K3_SERIAL=1: pass A of batch b+1 waits for pass B of batch b (no
  // overlap between the HBM-bound passes)
  const bool serial = env_int("SBW_K3_SERIAL", 0) != 0;
  int64_t nb = 0;
  for (int64_t c0 = 0; c0 < total; c0 += bb, ++nb) {
    const int64_t nc = (total - c0) < bb ? (total - c0) : bb;
    const uint32_t vf = v_lo + uint32_t(c0);
    const int buf = int(nb & 1);
    if (nb >= 2) SBW_CUDA_CHECK(cudaStreamWaitEvent(ks->a, ks->done_b[buf], 0));  // buffer free
    if (serial && nb >= 1) SBW_CUDA_CHECK(cudaStreamWaitEvent(ks->a, ks->done_b[buf ^ 1], 0));
    mark(ks->a);
    int* flag = ks->flags + buf;
    if (e16) SBW_CUDA_CHECK(cudaMemsetAsync(flag, 0, sizeof(int), ks->a));
    if (int rc = gray ? launch_tc_emit(planes, n, vf, nc, emit[buf], v_lo, v_hi, ks->a, e16 ? 1 : 0, flag)
                     : launch_emit_tiles(planes, n, m, vf, nc, emit[buf], ks->a))
      return rc;
    mark(ks->a);
    SBW_CUDA_CHECK(cudaEventRecord(ks->done_a[buf], ks->a));
    SBW_CUDA_CHECK(cudaStreamWaitEvent(ks->b, ks->done_a[buf], 0));
    mark(ks->b);
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
    a.gray = gray ? 1 : 0;
    a.run_lo = v_lo;
    a.run_hi = v_hi;
    auto run_b = [&](const PassBArgs& x) {
      return out ? dispatch_passb_regs<MODE_SPEC>(n - 15, x, ks->b)
                 : tc_b ? launch_passb_tc(x, ks->b) : dispatch_passb_regs<MODE_NL>(n - 15 - x.e16, x, ks->b);
    };
    if (e16) {
      PassBArgs a16 = a;  // the 16-stage batch, unless a tile wrapped
      a16.e16 = 1;
      a16.gate = flag;
      a16.gate_on = 0;
      if (int rc = run_b(a16)) return rc;
      // fallback, only if a tile wrapped: the same batch with 15 stages
      if (int rc = launch_tc_emit(planes, n, vf, nc, emit[buf], v_lo, v_hi, ks->b, 0, nullptr, flag, 1)) return rc;
      a.gate = flag;
      a.gate_on = 1;
    }
    if (int rc = run_b(a)) return rc;
    mark(ks->b);
    SBW_CUDA_CHECK(cudaEventRecord(ks->done_b[buf], ks->b));
  }
  if (trace && !ev.empty()) {
    // per batch: [A start, A end, B start, B end]
    SBW_CUDA_CHECK(cudaEventSynchronize(ev.back()));
    double sa = 0, sb = 0, span = 0, gap_ab = 0;
    float t;
    for (size_t i = 0; i + 3 < ev.size(); i += 4) {
      cudaEventElapsedTime(&t, ev[i], ev[i + 1]); sa += t;
      cudaEventElapsedTime(&t, ev[i + 2], ev[i + 3]); sb += t;
      cudaEventElapsedTime(&t, ev[i + 1], ev[i + 2]); gap_ab += t;
    }
    cudaEventElapsedTime(&t, ev.front(), ev.back()); span = t;
    fprintf(stderr, "[k3 trace] n=%d batches=%lld comps/batch=%lld span %.3f ms, sum passA %.3f ms, sum passB %.3f ms, "
            "sum(A end -> B start) %.3f ms\n", n, (long long)nb, (long long)bb, span, sa, sb, gap_ab);
    for (size_t i = 0; i + 3 < ev.size() && i < 16; i += 4) {
      float a0, a1, b0, b1;
      cudaEventElapsedTime(&a0, ev.front(), ev[i]); cudaEventElapsedTime(&a1, ev.front(), ev[i + 1]);
      cudaEventElapsedTime(&b0, ev.front(), ev[i + 2]); cudaEventElapsedTime(&b1, ev.front(), ev[i + 3]);
      fprintf(stderr, "[k3 trace]   batch %zu: A %.3f..%.3f  B %.3f..%.3f\n", i / 4, a0, a1, b0, b1);
    }
    for (auto e : ev) cudaEventDestroy(e);
  }
  // join: `st` continues after the last pass B (which follows every pass A)
  SBW_CUDA_CHECK(cudaEventRecord(ks->fork, ks->b));
  SBW_CUDA_CHECK(cudaStreamWaitEvent(st, ks->fork, 0));
  return SBW_OK;
}

// Ring run over the first p.r.batches * p.r.bc components of [v_lo, ...):
// pass B (k_passb_tc, NB CTAs) is enqueued before pass A (k_tc_hybrid<EMIT>,
// NA CTAs) on the two K3 streams; `st` continues after both.
int launch_k3_ring(const uint32_t* planes, int n, uint32_t v_lo, const RingPlan& p, int32_t* max_abs,
                   unsigned long long* key, uint32_t* ring_buf, uint32_t* counters, cudaStream_t st) {
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  K3Streams* ks = nullptr;
  if (int rc = k3_streams(dp.device, &ks)) return rc;
  std::lock_guard<std::mutex> launch_lock(g_k3_launch_mu[dp.device & 63]);
  RingArgs r = p.r;
  r.ready = counters;
  r.freed = counters + r.batches;
  r.err = counters + 2 * r.batches;
  r.nowait = env_int("SBW_K3_RING_NOWAIT", 0);
  static const bool trace = getenv("SBW_K3_TRACE") != nullptr;
  r.wait_ns = trace ? reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(counters) + p.counter_bytes - 256)
                    : nullptr;
  SBW_CUDA_CHECK(cudaMemsetAsync(counters, 0, p.counter_bytes, st));
  SBW_CUDA_CHECK(cudaEventRecord(ks->fork, st));
  SBW_CUDA_CHECK(cudaStreamWaitEvent(ks->a, ks->fork, 0));
  SBW_CUDA_CHECK(cudaStreamWaitEvent(ks->b, ks->fork, 0));
  cudaEvent_t ev[4] = {};
  if (trace)
    for (auto& e : ev) cudaEventCreate(&e);
  PassBArgs b{};
  b.scratch = ring_buf;
  b.n = n;
  b.n_comp = int64_t(r.R) * r.bc;  // extent of the tensor map: the R slots
  b.out_row0 = 0;
  b.v_first = v_lo;
  b.max_abs = max_abs;
  b.key = key;
  b.ring = r;
  if (trace) cudaEventRecord(ev[0], ks->b);
  if (int rc = launch_passb_tc(b, ks->b)) return rc;
  if (trace) cudaEventRecord(ev[1], ks->b);
  if (trace) cudaEventRecord(ev[2], ks->a);
  if (int rc = launch_tc_emit_ring(planes, n, v_lo, r, ring_buf, ks->a)) return rc;
  if (trace) cudaEventRecord(ev[3], ks->a);
  SBW_CUDA_CHECK(cudaEventRecord(ks->done_a[0], ks->a));
  SBW_CUDA_CHECK(cudaEventRecord(ks->done_b[0], ks->b));
  SBW_CUDA_CHECK(cudaStreamWaitEvent(st, ks->done_a[0], 0));
  SBW_CUDA_CHECK(cudaStreamWaitEvent(st, ks->done_b[0], 0));
  k_ring_poison<<<64, 256, 0, st>>>(r.err, max_abs, r.batches * r.bc);
  SBW_LAUNCH_CHECK("k_ring_poison");
  if (trace) {
    cudaEventSynchronize(ev[3]);
    cudaEventSynchronize(ev[1]);
    float tb = 0, ta = 0, d = 0;
    cudaEventElapsedTime(&tb, ev[0], ev[1]);
    cudaEventElapsedTime(&ta, ev[2], ev[3]);
    cudaEventElapsedTime(&d, ev[0], ev[2]);
    uint32_t err = 0;
    unsigned long long w[2] = {0, 0};
    cudaMemcpy(&err, r.err, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(w, r.wait_ns, sizeof(w), cudaMemcpyDeviceToHost);
    fprintf(stderr, "[k3 ring] n=%d NA=%u NB=%u L=%d R=%d Bc=%d batches=%lld: pass B %.3f ms, pass A %.3f ms (A starts %.3f ms after B), "
            "waits: pass A warps avg %.3f ms, pass B producers avg %.3f ms, err=%u\n",
            n, r.na, r.nb, r.L, r.R, r.bc, (long long)r.batches, tb, ta, d, w[0] * 1e-6 / (8.0 * r.na),
            w[1] * 1e-6 / r.nb, err);
    for (auto e : ev) cudaEventDestroy(e);
  }
  return SBW_OK;
}

}  // namespace

size_t k3_scratch_bytes(int n, int m, uint32_t v_lo, uint32_t v_hi) {
  if (n < 17) return 0;
  const int64_t ncomp = int64_t(v_hi) - int64_t(v_lo);
  // bit planes + two batch buffers of biased u16 partial transforms (or the
  // L2 ring + its counters, whichever is larger)
  size_t bufs = align256(2 * size_t(batch_components(n, ncomp > 0 ? ncomp : 1)) * (size_t(2) << n));
  DeviceProps dp;
  if (device_props(&dp) == SBW_OK) {
    const RingPlan p = ring_plan(n, ncomp, dp.sm_count);
    if (p.on) bufs = std::max(bufs, p.ring_bytes + p.counter_bytes);
  }
  return planes_bytes(n, m) + bufs;
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
  if (out == nullptr) {
    DeviceProps dp;
    if (int rc = device_props(&dp)) return rc;
    const RingPlan p = ring_plan(n, int64_t(v_hi) - v_lo, dp.sm_count);
    if (p.on && planes_bytes(n, m) + p.ring_bytes + p.counter_bytes <= scratch_bytes) {
      uint32_t* counters = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(bufs) + p.ring_bytes);
      if (int rc = launch_k3_ring(planes, n, v_lo, p, max_abs, key, bufs, counters, st)) return rc;
      const int64_t done = p.r.batches * p.r.bc;
      if (v_lo + done >= v_hi) return SBW_OK;
      return launch_k3_batched(planes, n, m, v_lo + uint32_t(done), v_hi, max_abs + done, key, nullptr, 0, bufs,
                               st);
    }
  }
  return launch_k3_batched(planes, n, m, v_lo, v_hi, max_abs, key, out, ld, bufs, st);
}

}  // namespace sbw
