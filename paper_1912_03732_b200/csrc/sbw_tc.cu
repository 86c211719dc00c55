// Tensor-core + packed-integer hybrid kernel for the n = 16 nonlinearity path.
//
// Replaces, per output mask v, polarity_row (sbox.py:145-152) +
// fwht_column_in_place (walsh.py:73-104) + column_nonlinearity
// (walsh.py:107-114), like k_tile_simd, but splits the 16 butterfly stages:
//
//   x = c * 256 + r  (r = x bits 0..7, c = x bits 8..15).
//
//   Stages over r (8 of them) are one int8 GEMM on the 5th-gen tensor cores:
//     s[u][c] = 128 + 128 [u == 0] - sum_r H[u][r] * B[c][r]
//   with B[c][r] = g_v(c * 256 + r) in {0, 1} (u8, generated from bit planes
//   straight into shared memory) and A = -H_256 (s8).  Because the polarity
//   is 1 - 2 B, s is exactly the biased value (W_8 + 2^8) / 2 in [0, 256]
//   that the packed SIMD stages below expect (see sbw_tile_simd.cuh).  The
//   bias rides along as a 9th K block of the same MMA chain.
//   Accumulators: 256 rows (u) x 256 columns (c) of s32 = all 512 TMEM columns.
//
//   Stages over c (8 of them) run on the integer pipes, one TMEM lane (one u)
//   per thread, 256 values in registers: the c-bit-0 stage is fused into the
//   TMEM -> u16x2 packing (two IMADs per pair), c bits 1..6 are packed 16-bit
//   stages, c bit 7 is the top stage fused with the max/min fold.
//
// Pipeline per CTA (persistent over a contiguous range of masks; one CTA/SM):
//   wait MMA(i) -> TMEM -> registers -> barrier -> issue MMA(i+1) ->
//   FWHT(i) on the ALUs while the tensor core runs MMA(i+1) -> generate the
//   B operand of i+2 into the buffer MMA(i) just released.
// Masks are visited in Gray-code order inside every aligned block of 256 that
// lies in [v_lo, v_hi), so consecutive masks differ in one bit and the bit
// rows are updated with a single plane XOR.
#include <cstdio>
#include <cstdlib>

#include "sbw_internal.cuh"
#include "sbw_launch.h"
#include "sbw_tc.cuh"
#include "sbw_tile_simd.cuh"

namespace sbw {
namespace {

constexpr int kTcThreads = 256;
constexpr int kKA = 288;                       // K of A: 256 (r) + 32 (bias block)
constexpr int kAHalf = 128 * kKA;              // one M = 128 half of A (36 KiB)
constexpr int kAOff = 0;
constexpr int kBbOff = kAOff + 2 * kAHalf;     // bias block of B: 256 x 32
constexpr int kBOff = kBbOff + 256 * 32;       // 2 x (256 x 256) generated B operands
constexpr int kBBytes = 256 * 256;
constexpr int kTcSmem = kBOff + 2 * kBBytes;   // 212992 bytes
constexpr uint32_t kIdesc = tc::idesc_i8(128, 256, /*A s8*/ true, /*B u8*/ false);

// K position of bit r inside its 32-bit plane word after the byte expansion
// (w >> k) & 0x01010101 (k = 0..7): element r = 32 j + 8 jb + k lands at
// byte 32 j + 4 k + jb.  A's columns carry the same permutation.
__device__ __forceinline__ int r_of_p(int p) { return (p & ~31) | ((p & 3) << 3) | ((p >> 2) & 7); }

__device__ __forceinline__ int8_t a_value(int u, int p) {
  if (p < 256) return (__popc(u & r_of_p(p)) & 1) ? int8_t(1) : int8_t(-1);  // -H[u][r]
  const int k = p - 256;  // bias block: +128 everywhere, +256 on row u = 0
  if (k < 2) return 64;
  if (k == 2) return u == 0 ? 127 : 0;
  if (k == 3) return u == 0 ? 1 : 0;
  return 0;
}

__device__ __forceinline__ uint32_t mask_at(int64_t q, uint32_t v_lo, uint32_t v_hi) {
  const int64_t b = q & ~int64_t(255);
  if (b >= int64_t(v_lo) && b + 256 <= int64_t(v_hi)) {
    const uint32_t k = uint32_t(q) & 255u;
    return uint32_t(b) | (k ^ (k >> 1));
  }
  return uint32_t(q);
}

// Bits g_v(c*256 .. c*256+255) of this thread's row c: update by the planes of
// (v ^ vcur) and expand into the u8 B operand (K-major core-matrix layout).
__device__ __forceinline__ void gen_row(const uint32_t* __restrict__ planes, uint32_t& vcur,
                                        uint32_t vnew, uint32_t (&g)[8], uint8_t* bbuf, int c) {
  uint32_t d = vcur ^ vnew;
  vcur = vnew;
  while (d) {
    const int i = __ffs(d) - 1;
    d &= d - 1;
    const uint4* p = reinterpret_cast<const uint4*>(planes + (int64_t(i) << 11) + c * 8);
    const uint4 a = __ldg(p), b = __ldg(p + 1);
    g[0] ^= a.x; g[1] ^= a.y; g[2] ^= a.z; g[3] ^= a.w;
    g[4] ^= b.x; g[5] ^= b.y; g[6] ^= b.z; g[7] ^= b.w;
  }
  uint8_t* row = bbuf + (c >> 3) * 2048 + (c & 7) * 16;
  constexpr uint32_t M = 0x01010101u;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t w = g[j];
    *reinterpret_cast<uint4*>(row + (2 * j) * 128) =
        make_uint4(w & M, (w >> 1) & M, (w >> 2) & M, (w >> 3) & M);
    *reinterpret_cast<uint4*>(row + (2 * j + 1) * 128) =
        make_uint4((w >> 4) & M, (w >> 5) & M, (w >> 6) & M, (w >> 7) & M);
  }
}

__device__ __forceinline__ void issue_mma(uint32_t tmem, const uint8_t* smem, int buf, uint64_t* bar) {
  const uint32_t a0 = tc::smem_u32(smem + kAOff);
  const uint32_t bb = tc::smem_u32(smem + kBbOff);
  const uint32_t b0 = tc::smem_u32(smem + kBOff + buf * kBBytes);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int kb = 0; kb < 9; ++kb) {
      const uint64_t da = tc::sdesc(a0 + h * kAHalf + kb * 256, 128, kKA / 16 * 128);
      const uint64_t db = kb < 8 ? tc::sdesc(b0 + kb * 256, 128, 2048) : tc::sdesc(bb, 128, 256);
      tc::mma_i8(tmem + h * 256, da, db, kIdesc, kb > 0 ? 1u : 0u);
    }
  }
  tc::mma_commit(bar);
}

__global__ void __launch_bounds__(kTcThreads, 1)
    k_tc16_nl(const uint32_t* __restrict__ planes, uint32_t v_lo, uint32_t v_hi,
              int32_t* __restrict__ max_abs, unsigned long long* key) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_slot;
  __shared__ int s_max[2];
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t total = int64_t(v_hi) - v_lo;
  const int64_t q_lo = v_lo + total * blockIdx.x / gridDim.x;
  const int n_my = int(v_lo + total * (blockIdx.x + 1) / gridDim.x - q_lo);

  // constant operands: A = -H_256 (+ bias block), B bias block
  for (int e = tid; e < 256 * (kKA / 16); e += kTcThreads) {
    const int u = e / (kKA / 16), pc = e % (kKA / 16);
    uint32_t wv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t x = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) x |= uint32_t(uint8_t(a_value(u, pc * 16 + q * 4 + b))) << (8 * b);
      wv[q] = x;
    }
    *reinterpret_cast<uint4*>(smem + kAOff + ((u >> 3) * (kKA / 16) + pc) * 128 + (u & 7) * 16) =
        make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
  {
    const int c = tid;  // 256 rows of the bias block: K bytes 0..3 = 1
    uint8_t* row = smem + kBbOff + (c >> 3) * 256 + (c & 7) * 16;
    *reinterpret_cast<uint4*>(row) = make_uint4(0x01010101u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(row + 128) = make_uint4(0u, 0u, 0u, 0u);
  }
  if (warp == 0) tc::tmem_alloc(&tmem_slot, 512);
  if (tid == 0) tc::mbar_init(&mbar, 1);
  if (tid < 2) s_max[tid] = 0;

  uint32_t g[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  uint32_t vcur = 0;
  if (n_my > 0) gen_row(planes, vcur, mask_at(q_lo, v_lo, v_hi), g, smem + kBOff, tid);
  if (n_my > 1) gen_row(planes, vcur, mask_at(q_lo + 1, v_lo, v_hi), g, smem + kBOff + kBBytes, tid);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_slot;
  if (tid == 0 && n_my > 0) issue_mma(tmem, smem, 0, &mbar);

  // this thread's TMEM lane: u = 128 * (warp >> 2) + 32 * (warp & 3) + lane
  const uint32_t tbase = tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t(warp >> 2) * 256;
  for (int i = 0; i < n_my; ++i) {
    tc::mbar_wait(&mbar, uint32_t(i & 1));
    tc::fence_after();
    uint32_t R[128];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      uint32_t t[32];
      tc::tmem_ld_x32(tbase + cc * 32, t);
      tc::wait_ld();
      // c bit 0 stage + packing: (a, b) -> lanes (a + b, a - b + 256)
#pragma unroll
      for (int j = 0; j < 16; ++j)
        R[cc * 16 + j] = t[2 * j] * 65537u + t[2 * j + 1] * 0xFFFF0001u + 0x01000000u;
    }
    tc::fence_before();
    __syncthreads();
    if (tid == 0) {
      if (i + 1 < n_my) issue_mma(tmem, smem, (i + 1) & 1, &mbar);
      if (i > 0) {
        const uint32_t vp = mask_at(q_lo + i - 1, v_lo, v_hi);
        const int mx = s_max[(i - 1) & 1];
        max_abs[vp - v_lo] = mx;
        if (key) atomicMax(key, nl_key(mx, vp));
        s_max[(i - 1) & 1] = 0;
      }
    }
    // c bits 1..6 (stages 9..14), then c bit 7 fused with the max/min fold
    stages16<128, 0, 6, 9>(R);
    uint32_t mx = 0u, mn = 0xFFFFFFFFu;
#pragma unroll
    for (int k = 0; k < 64; ++k) {
      const uint32_t x = R[k], y = R[k + 64];
      const uint32_t S = x + y;  // carry argument: see tile_last_pass
      const uint32_t D = x - y + 0x80008000u;
      mx = __vimax3_u16x2(mx, S, D);
      mn = __vimin3_u16x2(mn, S, D);
    }
    int m = lanes_maxabs<16>(mx, mn);
    m = warp_max(m);
    if ((tid & 31) == 0) atomicMax(&s_max[i & 1], m);
    if (i + 2 < n_my) {
      gen_row(planes, vcur, mask_at(q_lo + i + 2, v_lo, v_hi), g, smem + kBOff + (i & 1) * kBBytes, tid);
      tc::fence_proxy_async();
    }
  }
  tc::fence_before();
  __syncthreads();
  if (tid == 0 && n_my > 0) {
    const uint32_t vp = mask_at(q_lo + n_my - 1, v_lo, v_hi);
    const int mx = s_max[(n_my - 1) & 1];
    max_abs[vp - v_lo] = mx;
    if (key) atomicMax(key, nl_key(mx, vp));
  }
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

}  // namespace

// SBW_TC=0 selects the all-ALU tile kernel instead (A/B experiments only).
bool tc_path_enabled() {
  static const bool on = [] {
    const char* e = getenv("SBW_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

int launch_tc16_nl(const uint32_t* planes, uint32_t v_lo, uint32_t v_hi, int32_t* max_abs,
                   unsigned long long* key, cudaStream_t st) {
  if (v_hi <= v_lo) return SBW_OK;
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  static unsigned long long attr_done = 0;
  if (!(attr_done >> (dp.device & 63) & 1ull)) {
    SBW_CUDA_CHECK(cudaFuncSetAttribute(k_tc16_nl, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem));
    attr_done |= 1ull << (dp.device & 63);
  }
  const int64_t count = int64_t(v_hi) - v_lo;
  const int grid = int(count < dp.sm_count ? count : dp.sm_count);
  k_tc16_nl<<<grid, kTcThreads, kTcSmem, st>>>(planes, v_lo, v_hi, max_abs, key);
  SBW_LAUNCH_CHECK("k_tc16_nl");
  return SBW_OK;
}

}  // namespace sbw
