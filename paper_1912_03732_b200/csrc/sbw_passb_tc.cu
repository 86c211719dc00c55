// K3 pass B on the tensor cores: n = 17..24 (H = n - 15 = 2..9), NL only.
//
// Pass A leaves, per component, 2^H rows (x bits 15..n-1) of 2^15 biased u16
// s = h + 2^14 (h = W_15 / 2, sbw_passb.cuh).  Up to 7 row stages are one
// int8 GEMM per 128-row block g:
//
//   D_g[r'][c] = sum_r A[r'][r] * B_g[r][c],   B_g = the u16 rows of block g
//                read as a u8 matrix (column 2e = low byte of element e,
//                column 2e+1 = high byte),
//
// so A (s8 +/-1: H_128, or I_P (x) H_(2^H) for H < 7, see PbShape) times the
// raw scratch bytes (u8, the B operand, MN-major exactly as they lie in HBM)
// gives W_g = D_g[2e] + 256 D_g[2e+1] = A s, exact in s32 (|D| <= 128 * 255).
// The bias 2^14 of s adds 2^14 * 2^h to row u = 0 of every 2^h block only
// (H_(2^h) * 1 = 2^h e_0).  The remaining H - 7 stages (across the
// G = 2^(H-7) blocks) and the max|W| fold run on the ALU from TMEM: ~4
// instructions per element instead of ~13 for the fp32 pass
// (k_passb_staged), so the kernel is bound by the HBM read.
//
// Data path: TMA (3D tensor map [rows][chunks][64 B] over the batch scratch,
// SWIZZLE_64B boxes of 64 B x P chunks x <= 256 rows) -> 4-stage ring -> tcgen05.mma
// kind::i8 (M128 N64 K32, B MN-major SW64) -> double-buffered TMEM ->
// tcgen05.ld by 8 epilogue warps.  One item = one component x 32 KiB: 32 P CG
// elements (P CG adjacent 64-byte chunks) of every row.  The reference runs all n
// stages per mask in numpy (walsh.py:91-103); stage order is free because
// butterflies commute.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <cstdlib>

#include "sbw_internal.cuh"
#include "sbw_launch.h"
#include "sbw_passb.cuh"
#include "sbw_tc.cuh"

namespace sbw {
namespace {

constexpr int kPbThreads = 64 + 256;  // warp 0 TMA producer, warp 1 MMA issuer, 8 epilogue warps
constexpr int kPbAOff = 0;            // H_128, s8, K-major no-swizzle (16 KiB)
constexpr int kPbBOff = 16384;        // stage ring, 1024-aligned
constexpr int kPbRingBytes = 4 * 32768;
constexpr size_t kPbSmem = size_t(kPbBOff) + kPbRingBytes + 1024;  // + alignment slack

__device__ __forceinline__ void mbar_arrive_pb(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(tc::smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(tc::smem_u32(bar))
      : "memory");
}
// MN-major SWIZZLE_64B descriptor: 8 K-rows x 64 B atoms (512 B, 512-aligned),
// 16-byte chunk c of K-row i at chunk c ^ ((i >> 1) & 3); SBO = distance
// between 8-row atoms along K; one atom spans the whole N = 64 extent, so LBO
// is unused.
__device__ __forceinline__ uint64_t sdesc_mn_sw64(uint32_t saddr, uint32_t sbo) {
  return uint64_t((saddr & 0x3FFFFu) >> 4) | (uint64_t(1) << 16) | (uint64_t((sbo >> 4) & 0x3FFFu) << 32) |
         (uint64_t(1) << 46) | (uint64_t(4) << 61);
}
__device__ __forceinline__ void wait_ld_tied32(uint32_t (&r)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
                 "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
                 "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]),
                 "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]),
                 "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

// H >= 7: G = 2^(H-7) blocks of 128 rows, A = H_128, the last H - 7 stages on
// the ALU.  H <= 6: all H stages in the GEMM; P = 128 / 2^H adjacent 64-byte
// column chunks of one component are interleaved along K (K index = row P + p,
// exactly how one TMA box {64 B, P chunks, 2^H rows} lands) and A =
// H_(2^H) (x) I_P, so output row r' = u P + p is coefficient u of chunk p.
//
// An item is CG = 4 / G column groups (32 P elements each) so that every item
// moves 32 KiB: small items pay the per-item handshakes (mbarrier waits, TMEM
// loads) too often to keep up with HBM.
template <int H>
struct PbShape {
  static constexpr int h = H < 7 ? H : 7;                   // stages in the GEMM
  static constexpr int G = 1 << (H - h);                    // 128-row blocks
  static constexpr int LP = 7 - h, P = 1 << LP;             // chunks interleaved along K
  static constexpr int CG = 4 / G;                          // column groups per item
  static constexpr int LCG = CG == 4 ? 2 : (CG == 2 ? 1 : 0);
  static constexpr int ROWS = 1 << H;
  static constexpr int SUB_BYTES = G * 128 * 64;            // one column group
  static constexpr int ITEM_BYTES = CG * SUB_BYTES;         // 32 KiB
  static constexpr int BOX_ROWS = ROWS < 256 ? ROWS : 256;  // TMA box {64 B, P, BOX_ROWS}
  static constexpr int BOXES = ROWS / BOX_ROWS;             // per column group
  static constexpr int STAGES = kPbRingBytes / ITEM_BYTES;  // 4
  static constexpr int TCOLS = CG * G * 64;                 // TMEM columns per buffer (256)
  static constexpr int TBUF = 512 / TCOLS;                  // 2
  static constexpr int TALLOC = 512;
  static constexpr int LPC = 10 - LP - LCG;                 // log2 items per component
  static constexpr int64_t PER_COMP = int64_t(1) << LPC;
};

template <int H>
__global__ void __launch_bounds__(kPbThreads, 1) k_passb_tc(const __grid_constant__ CUtensorMap tmap, PassBArgs a) {
  using S = PbShape<H>;
  constexpr uint32_t kIdesc = tc::idesc_i8(128, 64, true, false) | (1u << 16);  // B MN-major
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t full[S::STAGES], empty[S::STAGES], tfull[S::TBUF], tempty[S::TBUF];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (passb_gated_off(a)) return;  // CTA-uniform, before any setup
  // e16: rows are twice as wide (2^16 u16), so a component has twice the items
  const int64_t per_comp = S::PER_COMP << a.e16;
  const int lpc = S::LPC + a.e16;
  const bool ring = a.ring.on != 0;
  int64_t b0 = 0, n_pb = 1, ib_off = 0, I = 0;
  int n_my = 0;
  if (ring) {  // this CTA's share [I j / NB, I (j + 1) / NB) of every batch
    I = int64_t(a.ring.bc) * S::PER_COMP;
    ib_off = I * blockIdx.x / gridDim.x;
    n_pb = I * (blockIdx.x + 1) / gridDim.x - ib_off;
    n_my = n_pb > 0 ? int(a.ring.batches * n_pb) : 0;
  } else {
    const int64_t items = a.n_comp * per_comp;
    const int64_t per_cta = (items + gridDim.x - 1) / gridDim.x;
    b0 = blockIdx.x * per_cta;
    const int64_t b1 = b0 + per_cta < items ? b0 + per_cta : items;
    n_my = b0 < b1 ? int(b1 - b0) : 0;
  }
  // i-th item of this CTA -> item index (component-major) within the launch
  auto item_b = [&](int i) -> int64_t {
    if (!ring) return b0 + i;
    const int64_t k = i / n_pb;
    return k * I + ib_off + (i - k * n_pb);
  };

  // A = H_(2^h) (x) I_P: core matrix (row group rg, 16-byte K chunk kc) at
  // (rg * 8 + kc) * 128, row r & 7 at + 16 (r & 7)
  for (int e = tid; e < 128 * 32; e += kPbThreads) {
    const int r = e >> 5, k4 = (e & 31) * 4;
    uint32_t w = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = k4 + j;
      const uint32_t v = ((r ^ k) & (S::P - 1)) ? 0u : ((__popc((r >> S::LP) & (k >> S::LP)) & 1) ? 0xFFu : 0x01u);
      w |= v << (8 * j);
    }
    *reinterpret_cast<uint32_t*>(smem + kPbAOff + ((r >> 3) * 8 + (k4 >> 4)) * 128 + (r & 7) * 16 + (k4 & 15)) = w;
  }
  if (warp == 0) tc::tmem_alloc(&tmem_slot, S::TALLOC);
  if (tid == 0) {
    for (int s = 0; s < S::STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < S::TBUF; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], 256);
    }
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (one thread) ----------------
    if (lane == 0) {
      for (int i = 0; i < n_my; ++i) {
        const int s = i % S::STAGES;
        if (i >= S::STAGES) tc::mbar_wait(&empty[s], uint32_t((i / S::STAGES - 1) & 1));
        const int64_t b = item_b(i);
        int comp = int(b >> lpc);
        const int q = int(b & (per_comp - 1));
        if (ring) {
          // batch k sits in slot k mod R; its first item waits for every
          // pass-A warp's arrival, then orders the TMA reads after the acquire
          const int64_t k = i / n_pb;
          if (i - k * n_pb == 0 && !a.ring.nowait) {
            ring_wait_geq(a.ring.ready + k, 8u * a.ring.na, a.ring.err, a.ring.wait_ns ? a.ring.wait_ns + 1 : nullptr);
            asm volatile("fence.proxy.async.global;" ::: "memory");
          }
          comp = int((k % a.ring.R) * a.ring.bc + (int64_t(comp) - k * a.ring.bc));
        }
        mbar_expect_tx(&full[s], S::ITEM_BYTES);
#pragma unroll
        for (int c = 0; c < S::CG; ++c)
#pragma unroll
          for (int bx = 0; bx < S::BOXES; ++bx)
            tma_load_3d(smem + kPbBOff + s * S::ITEM_BYTES + c * S::SUB_BYTES + bx * S::BOX_ROWS * 64, &tmap, 0,
                        (q * S::CG + c) * S::P, comp * S::ROWS + bx * S::BOX_ROWS, &full[s]);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t a_base = tc::smem_u32(smem + kPbAOff);
    for (int i = 0; i < n_my; ++i) {
      const int s = i % S::STAGES, buf = i % S::TBUF;
      tc::mbar_wait(&full[s], uint32_t((i / S::STAGES) & 1));
      // ring: the last load of this CTA's share of a batch has landed -> the
      // slot may be overwritten as far as this CTA is concerned
      if (ring && lane == 0 && (i % n_pb) == n_pb - 1) ring_signal(a.ring.freed + i / n_pb);
      __syncwarp();
      if (i >= S::TBUF) tc::mbar_wait(&tempty[buf], uint32_t((i / S::TBUF - 1) & 1));
      tc::fence_after();
      const uint32_t b_base = tc::smem_u32(smem + kPbBOff + s * S::ITEM_BYTES);
#pragma unroll
      for (int c = 0; c < S::CG; ++c)
#pragma unroll
        for (int g = 0; g < S::G; ++g)
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc::mma_i8_elect(tmem + buf * S::TCOLS + (c * S::G + g) * 64, tc::sdesc(a_base + k * 256, 128, 1024),
                             sdesc_mn_sw64(b_base + c * S::SUB_BYTES + (g * 128 + 32 * k) * 64, 512), kIdesc,
                             k > 0 ? 1u : 0u);
      tc::mma_commit_elect(&empty[s]);
      tc::mma_commit_elect(&tfull[buf]);
      __syncwarp();
    }
  } else {
    // ---------------- epilogue: 8 warps, lane quarter warp & 3 ----------------
    // Both warpgroups read every item: CG >= 2 -> column groups split between
    // them; CG = 1 (G = 4) -> one column half each.
    const int quarter = warp & 3, wg = (warp - 2) >> 2;
    const int rr = quarter * 32 + lane;  // output row r' = TMEM lane
    // row u = 0 of every 2^h block carries 2^14 * 2^h from the bias of s
    // (twice that after the first ALU stage when G >= 2)
    const int corr = rr < S::P ? -(S::G == 1 ? (1 << (14 + a.e16 + S::h)) : (1 << (22 + a.e16))) : 0;
    const uint32_t t_lane = uint32_t(quarter * 32) << 16;
    int run = 0;
    for (int i = 0; i < n_my; ++i) {
      const int buf = i % S::TBUF;
      const uint32_t tb = tmem + t_lane + buf * S::TCOLS;
      tc::mbar_wait(&tfull[buf], uint32_t((i / S::TBUF) & 1));
      tc::fence_after();
      int m = 0;
      if constexpr (S::G == 1) {
        // CG = 4: two column groups per warpgroup, 32 elements each
        int mx = INT_MIN, mn = INT_MAX;
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          uint32_t d[64];
          tc::tmem_ld_x64(tb + (2 * wg + cc) * 64, d);
          tc::wait_ld_tied(d);
          if (cc == 1) {
            tc::fence_before();
            mbar_arrive_pb(&tempty[buf]);
          }
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const int w0 = int(d[2 * e + 1]) * 256 + int(d[2 * e]);
            const int w1 = int(d[2 * e + 3]) * 256 + int(d[2 * e + 2]);
            mx = __vimax3_s32(mx, w0, w1);
            mn = __vimin3_s32(mn, w0, w1);
          }
        }
        m = max(mx + corr, -(mn + corr));
      } else if constexpr (S::G == 2) {
        // CG = 2: one column group per warpgroup, both blocks, then the top stage
        uint32_t d0[64], d1[64];
        tc::tmem_ld_x64(tb + (wg * 2) * 64, d0);
        tc::tmem_ld_x64(tb + (wg * 2 + 1) * 64, d1);
        tc::wait_ld_tied(d0);
        tc::wait_ld_tied(d1);
        tc::fence_before();
        mbar_arrive_pb(&tempty[buf]);
        int mx = INT_MIN, mn = INT_MAX;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int w0 = int(d0[2 * e + 1]) * 256 + int(d0[2 * e]);
          const int w1 = int(d1[2 * e + 1]) * 256 + int(d1[2 * e]);
          mx = __vimax3_s32(mx, w0 + w1 + corr, w0 - w1);
          mn = __vimin3_s32(mn, w0 + w1 + corr, w0 - w1);
        }
        m = max(mx, -mn);
      } else {
        // CG = 1, G = 4: one column half per warpgroup
        uint32_t d[S::G][32];
#pragma unroll
        for (int g = 0; g < S::G; ++g) tc::tmem_ld_x32(tb + g * 64 + wg * 32, d[g]);
#pragma unroll
        for (int g = 0; g < S::G; ++g) wait_ld_tied32(d[g]);
        tc::fence_before();
        mbar_arrive_pb(&tempty[buf]);
#pragma unroll
        for (int e = 0; e < 16; ++e) {
          int w[S::G];
#pragma unroll
          for (int g = 0; g < S::G; ++g) w[g] = int(d[g][2 * e + 1]) * 256 + int(d[g][2 * e]);
          // stage over block bit 0, then the top stage fused with the fold
          const int s01 = w[0] + w[1] + corr, d01 = w[0] - w[1];
          const int s23 = w[2] + w[3] + corr, d23 = w[2] - w[3];
          m = __vimax3_s32(m, abs(s01) + abs(s23), abs(d01) + abs(d23));
        }
      }
      run = max(run, 2 * m);  // values are W / 2
      const int64_t comp = item_b(i) >> lpc;
      if (i + 1 >= n_my || (item_b(i + 1) >> lpc) != comp) {
        if (ring) {  // batch k, slot component cb -> its ring position's mask
          const int64_t k = comp / a.ring.bc;
          const uint32_t v = ring_mask(a.ring, a.v_first, ring_pos(a.ring, k, comp - k * a.ring.bc));
          warp_publish_max(run, a.max_abs + (v - a.v_first), a.key, v);
        } else {
          publish_comp(a, comp, run);
        }
        run = 0;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    tc::fence_after();
    tc::tmem_dealloc(tmem, S::TALLOC);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

template <int H>
int run_passb_tc(const PassBArgs& a, cudaStream_t st) {
  using S = PbShape<H>;
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  auto enc = encode_fn();
  if (!enc) return set_error(SBW_ECUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap map;
  // [rows][1024 (e16: 2048) chunks][64 B]: box {64 B, P chunks, BOX_ROWS rows}
  const cuuint64_t dims[3] = {64, cuuint64_t(1024) << a.e16, cuuint64_t(a.n_comp) << H};
  const cuuint64_t strides[2] = {64, cuuint64_t(1) << (16 + a.e16)};
  const cuuint32_t box[3] = {64, cuuint32_t(S::P), cuuint32_t(S::BOX_ROWS)};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint32_t*>(a.scratch), dims, strides, box,
                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(SBW_ECUDA, "cuTensorMapEncodeTiled failed (%d)", int(r));
  static unsigned long long attr_done = 0;
  if (!(attr_done >> (dp.device & 63) & 1ull)) {
    SBW_CUDA_CHECK(cudaFuncSetAttribute(k_passb_tc<H>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kPbSmem)));
    attr_done |= 1ull << (dp.device & 63);
  }
  const int64_t items = a.n_comp * (S::PER_COMP << a.e16);
  const int grid = a.ring.on ? int(a.ring.nb) : int(items < dp.sm_count ? items : dp.sm_count);
  k_passb_tc<H><<<grid, kPbThreads, kPbSmem, st>>>(map, a);
  SBW_LAUNCH_CHECK("k_passb_tc");
  return SBW_OK;
}

}  // namespace

void* tma_encode_ptr() { return reinterpret_cast<void*>(encode_fn()); }

bool passb_tc_enabled() {
  static const bool on = [] {
    const char* e = getenv("SBW_PASSB_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

int launch_passb_tc(const PassBArgs& a, cudaStream_t st) {
  switch (a.n - 15 - a.e16) {
    case 2: return run_passb_tc<2>(a, st);
    case 3: return run_passb_tc<3>(a, st);
    case 4: return run_passb_tc<4>(a, st);
    case 5: return run_passb_tc<5>(a, st);
    case 6: return run_passb_tc<6>(a, st);
    case 7: return run_passb_tc<7>(a, st);
    case 8: return run_passb_tc<8>(a, st);
    case 9: return run_passb_tc<9>(a, st);
    default: return set_error(SBW_EINVAL, "tensor-core pass B needs n in 17..24");
  }
}

}  // namespace sbw
