// k_tc_lut: the n = 16 nonlinearity kernel with the GEMM contracting over the
// HIGH input bits and a table-lookup generation (K2L in DESIGN.md).
//
// Same job as k_tc_hybrid<NL, 16> (sbw_tc.cu): per output mask v,
// polarity_row (sbox.py:145-152) + fwht_column_in_place (walsh.py:73-104) +
// column_nonlinearity (walsh.py:107-114), all 16 butterfly stages of the
// 2^16-point transform, only max|W| leaves the chip.  The split x = c * 256 + r
// (r = x bits 0..7, c = bits 8..15) is used the other way round:
//
//   Generation (r bits 0..4, 5 stages, no bit expansion).  The 32 component
//   bits of one plane word are 4 bytes; a 256-entry shared-memory table maps
//   a byte straight to the biased 8-point WHT of its 8 bits (8 output bytes,
//   LDS.64), and two byte-lane butterfly stages across the 4 lookups finish
//   the 32-point WHT of the word: U[c][32 ks + e5] in [0, 32], offset 16 on
//   all but e5 = 0.  The (w >> k) & 0x01010101 expansion and three of the
//   byte stages of k_tc_hybrid (0.5 + 0.375 ALU instructions per element)
//   become one PRMT + one LDS.64 per 8 elements.
//
//   GEMM (c bits 0..7, 8 stages).  D[u_c][n] = sum_c A[u_c][c] U[c][n],
//   A = -H_256 (s8), U the B operand (u8, MN-major SWIZZLE_128B: the 32 bytes
//   a thread produces for one (c, word) are contiguous), plus the bias K block
//   of the 32-row form: +4096 on every entry and +4096 more on row u_c = 0, so
//   D = W_13 / 2 + 2^12 in [0, 2^13] exactly (the biased s form).
//
//   Integer stages (r bits 5..7 = column bits 5..7).  tcgen05.ld .pack::16b,
//   two packed int16 stages, the top stage fused with the VIMNMX3 fold.
//
// Output positions are permuted relative to k_tc_hybrid (TMEM lane = u_c, not
// u_r), which the max does not see; the materialising modes keep k_tc_hybrid.
// Pipeline, warp roles, Gray mask order and publishing are those of
// k_tc_hybrid (one MMA-issuing warp, 8 transform warps, mbarriers only).
#include <cstdlib>
#include <mutex>

#include "sbw_internal.cuh"
#include "sbw_launch.h"
#include "sbw_tc.cuh"
#include "sbw_tile_simd.cuh"

namespace sbw {
namespace {

#ifndef SBW_LUT_COPIES
#define SBW_LUT_COPIES 16  // table replicas (lane & 15 picks one): LDS.64 without bank conflicts
#endif
constexpr int kCopies = SBW_LUT_COPIES;
#ifndef SBW_LUT_HALVES
#define SBW_LUT_HALVES 1  // the two M = 128 halves of a component complete and are consumed separately
#endif
constexpr bool kHalves = SBW_LUT_HALVES;
#ifndef SBW_LUT_WARPS_DEFAULT
#define SBW_LUT_WARPS_DEFAULT 16  // transform warps: 8 (k_tc_lut) or 16 (k_tc_lut16); SBW_LUT_WARPS overrides
#endif
#ifndef SBW_LUT_GEN7
#define SBW_LUT_GEN7 1  // r bits 5, 6 as two more byte-lane stages across a thread's 4 words (else int16 stages)
#endif
constexpr int kGenStages = SBW_LUT_GEN7 ? 7 : 5;  // r stages before the GEMM
constexpr int kMathWarps = 8;
// A = -H_256 needs only two 128 x 128 blocks: with Hs = -H_128,
//   rows u < 128 : A[u][c] = Hs[u][c & 127]
//   rows u >= 128: A[u][c] = Hs[u & 127][c & 127] for c < 128, -Hs[..] for c >= 128,
// so both M = 128 halves read Hs for K blocks 0..3 and Hs / -Hs for K blocks
// 4..7 (32 KiB instead of 64 KiB; the space holds the lookup table replicas).
constexpr int kHsOff = 0;                       // Hs, 128 x 128 s8, K-major core matrices
constexpr int kNegOff = kHsOff + 128 * 128;     // -Hs
constexpr int kAbOff = kNegOff + 128 * 128;     // A's bias K block, 2 halves x (128 x 32)
constexpr int kBbOff = kAbOff + 2 * 128 * 32;   // B's bias block, 256 x 32, K-major
constexpr int kBOff = kBbOff + 256 * 32;        // 2 x (256 x 256) generated B, MN-major SW128
constexpr int kBBytes = 256 * 256;
constexpr int kLutOff = kBOff + 2 * kBBytes;    // kCopies x 256 x 8 bytes
constexpr int kLutBytes = kCopies * 2048;
constexpr int kSmem = kLutOff + kLutBytes;
constexpr int kImgBytes = kBOff + kLutBytes;    // constant image: Hs | -Hs | A bias | Bb | LUT
static_assert(kBOff % 1024 == 0, "SW128 atoms need 1024-byte alignment");
static_assert(kSmem <= 227 * 1024 - 1024, "k_tc_lut shared memory");
// bias (the 32-row form of sbw_tc.cu): 4096 per D entry as 9 columns of
// 127, ..., 8 against B columns of 4; twice on row u_c = 0
constexpr int kBiasT = 1 << (kGenStages + 7), kBiasB = 1 << (kGenStages - 3);
constexpr int kBiasCols = (kBiasT / kBiasB + 126) / 127;
static_assert(2 * kBiasCols <= 32, "bias block is one K block");
constexpr uint32_t kIdescK = tc::idesc_i8(128, 256, /*A s8*/ true, /*B u8*/ false);
constexpr uint32_t kIdescMN = kIdescK | (1u << 16);  // B MN-major
constexpr int kIssuerRegs = 32, kMathRegs = 232;
constexpr int kAllThreads = 128 + kMathWarps * 32;

// MN-major SWIZZLE_128B descriptor (u8): atoms of 8 K-rows x 128 bytes of N
// (1024 B, 1024-aligned), 16-byte chunk j of K-row i at chunk j ^ i; LBO = the
// distance between atoms along N, SBO = between 8-row groups along K.
__device__ __forceinline__ uint64_t sdesc_mn_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr & 0x3FFFFu) >> 4) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (uint64_t(1) << 46) | (uint64_t(2) << 61);
}

// bias K block of A (against B's columns of kBiasB): +4096 on every row, +4096 more on u = 0
__device__ __forceinline__ int a_bias_value(int u, int k) {
  const int col = k % kBiasCols, last = kBiasT / kBiasB - 127 * (kBiasCols - 1);
  if (k < kBiasCols) return col < kBiasCols - 1 ? 127 : last;
  if (k < 2 * kBiasCols) return u == 0 ? (col < kBiasCols - 1 ? 127 : last) : 0;
  return 0;
}

// constant image: Hs, -Hs and A's bias block (K-major core matrices), B's
// bias block, the lookup table
// EMIT (pass A of the multi-pass path): 14 stages in front of the top int16
// stage (x bit 15 is left out of the GEMM), bias 2^13 per entry and 2^13 more on
// row u = 0 of EACH M half
constexpr int kBiasTE = kBiasT / 2;
constexpr int kBiasColsE = (kBiasTE / kBiasB + 126) / 127;
__device__ __forceinline__ int a_bias_value_emit(int ul, int k) {
  const int col = k % kBiasColsE, last = kBiasTE / kBiasB - 127 * (kBiasColsE - 1);
  if (k < kBiasColsE) return col < kBiasColsE - 1 ? 127 : last;
  if (k < 2 * kBiasColsE) return ul == 0 ? (col < kBiasColsE - 1 ? 127 : last) : 0;
  return 0;
}

__global__ void k_lut_consts(uint8_t* img, int emit) {
  const int t0 = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  for (int e = t0; e < 128 * 128; e += nt) {
    const int u = e >> 7, p = e & 127;
    const int v = (__popc(u & p) & 1) ? 1 : -1;  // -H_128
    const int off = ((u >> 3) * 8 + (p >> 4)) * 128 + (u & 7) * 16 + (p & 15);
    img[kHsOff + off] = uint8_t(v);
    img[kNegOff + off] = uint8_t(-v);
  }
  for (int e = t0; e < 256 * 32; e += nt) {
    const int u = e >> 5, k = e & 31, ul = u & 127;
    img[kAbOff + (u >> 7) * 4096 + ((ul >> 3) * 2 + (k >> 4)) * 128 + (ul & 7) * 16 + (k & 15)] =
        uint8_t(emit ? a_bias_value_emit(ul, k) : a_bias_value(u, k));
  }
  for (int e = t0; e < 256 * 32; e += nt) {
    const int n = e >> 5, k = e & 31;
    img[kBbOff + ((n >> 3) * 2 + (k >> 4)) * 128 + (n & 7) * 16 + (k & 15)] = k < 2 * kBiasCols ? kBiasB : 0;
  }
  // table: byte b -> 8-point WHT of its bits, +4 on outputs e != 0 (every byte in [0, 8])
  for (int e = t0; e < 256 * kCopies * 8; e += nt) {
    const int oe = e & 7, cp = (e >> 3) % kCopies, b = e / (8 * kCopies);
    int s = oe ? 4 : 0;
    for (int j = 0; j < 8; ++j)
      if ((b >> j) & 1) s += (__popc(oe & j) & 1) ? -1 : 1;
    img[kBOff + (b * kCopies + cp) * 8 + oe] = uint8_t(s);
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

__device__ __forceinline__ uint2 lds64(uint32_t saddr) {
  uint2 r;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "r"(saddr));
  return r;
}

struct LutArgs {
  const uint8_t* consts;
  const uint32_t* planes;  // [16][2048]
  uint32_t v_lo, v_hi;
  int32_t* max_abs;
  unsigned long long* key;
};

__device__ __forceinline__ void publish(const uint32_t* wmax, uint32_t v, const LutArgs& a) {
  const uint4 x = *reinterpret_cast<const uint4*>(wmax);
  const uint4 y = *reinterpret_cast<const uint4*>(wmax + 4);
  const int m = int(max(max(max(x.x, x.y), max(x.z, x.w)), max(max(y.x, y.y), max(y.z, y.w))));
  a.max_abs[v - a.v_lo] = m;
  if (a.key) atomicMax(a.key, nl_key(m, v));
}

// MMA chain of one M = 128 half of a mask: 8 K blocks of generated B + the bias block
__device__ __forceinline__ void issue_mma_half(uint32_t tmem, const uint8_t* smem, int buf, int h, uint64_t* bar) {
  const uint64_t dhs = tc::sdesc(tc::smem_u32(smem + kHsOff), 128, 1024);
  const uint64_t dab = tc::sdesc(tc::smem_u32(smem + kAbOff), 128, 256);
  const uint64_t db0 = sdesc_mn_sw128(tc::smem_u32(smem + kBOff + buf * kBBytes), 1024, 2048);
  const uint64_t dbb = tc::sdesc(tc::smem_u32(smem + kBbOff), 128, 256);
#pragma unroll
  for (int kb = 0; kb < 9; ++kb) {
    // A: K block kb of half h = block kb & 3 of Hs (-Hs for h = 1, kb >= 4)
    const uint64_t da = kb == 8 ? dab + uint64_t((h * 4096) >> 4)
                                : dhs + uint64_t((((h == 1 && kb >= 4) ? kNegOff - kHsOff : 0) + (kb & 3) * 256) >> 4);
    // B: K block kb = 32 K-rows = 4 groups of 8 (2048 B each)
    const uint64_t db = kb == 8 ? dbb : db0 + uint64_t((kb * 8192) >> 4);
    tc::mma_i8_elect(tmem + h * 256, da, db, kb == 8 ? kIdescK : kIdescMN, kb > 0 ? 1u : 0u);
  }
  if (bar) tc::mma_commit_elect(bar);
}

// One plane word (32 component bits of row c, r = 32 ks ..) -> the 32 bytes
// U[c][32 ks .. 32 ks + 31]: four table lookups (r bits 0..2; byte i -> table
// address by one PRMT on the ALU pipe + one IMAD on the FMA pipe) ...
__device__ __forceinline__ void word_lookup(uint32_t w, uint32_t lut, uint4& lo, uint4& hi) {
  const uint2 l0 = lds64(__byte_perm(w, 0u, 0x4440u) * uint32_t(8 * kCopies) + lut);
  const uint2 l1 = lds64(__byte_perm(w, 0u, 0x4441u) * uint32_t(8 * kCopies) + lut);
  const uint2 l2 = lds64(__byte_perm(w, 0u, 0x4442u) * uint32_t(8 * kCopies) + lut);
  const uint2 l3 = lds64(__byte_perm(w, 0u, 0x4443u) * uint32_t(8 * kCopies) + lut);
  lo = make_uint4(l0.x, l0.y, l1.x, l1.y);
  hi = make_uint4(l2.x, l2.y, l3.x, l3.y);
}
// ... and two byte-lane stages across them (r bits 3, 4; diff + 2^t per byte,
// so every byte stays in [0, 2^(t+1)]), in place.
__device__ __forceinline__ void word_stages(uint4& lo, uint4& hi) {
  constexpr uint32_t M = 0x01010101u;
  // stage r bit 3: (l0, l1), (l2, l3); bias 8
  const uint32_t s0x = lo.x + lo.z, s0y = lo.y + lo.w, d0x = lo.x - lo.z + (M << 3), d0y = lo.y - lo.w + (M << 3);
  const uint32_t s1x = hi.x + hi.z, s1y = hi.y + hi.w, d1x = hi.x - hi.z + (M << 3), d1y = hi.y - hi.w + (M << 3);
  // stage r bit 4: (s0, s1), (d0, d1); bias 16.  Output index e5 = 8 i + e3, i = (bit 4, bit 3)
  lo = make_uint4(s0x + s1x, s0y + s1y, d0x + d1x, d0y + d1y);                                    // i = 0, 1
  hi = make_uint4(s0x - s1x + (M << 4), s0y - s1y + (M << 4), d0x - d1x + (M << 4), d0y - d1y + (M << 4));  // i = 2, 3
}

__global__ void __launch_bounds__(kAllThreads, 1) k_tc_lut(LutArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // full[h]: MMA(i) half h done (kHalves; else full[0] = both).  tmem_empty[h]:
  // D(i) half h read.  kHalves: warps 0-3 (half 0) also arrive on tmem_empty[1]
  // once they have seen full[1](i), so full[1] never runs two phases ahead of
  // their parity wait.  bfull[b]: every transform thread stored B into buffer b.
  __shared__ uint64_t bar_full[2], bar_tmem_empty[2], bar_bfull[2], bar_done;
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(16) uint32_t s_wmax[4][kMathWarps];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t total = int64_t(a.v_hi) - a.v_lo;
  const int64_t t_lo = total * blockIdx.x / gridDim.x;
  const int n_my = int(total * (blockIdx.x + 1) / gridDim.x - t_lo);

  for (int e = tid; e < kBOff / 16; e += kAllThreads)
    reinterpret_cast<uint4*>(smem)[e] = __ldg(reinterpret_cast<const uint4*>(a.consts) + e);
  for (int e = tid; e < kLutBytes / 16; e += kAllThreads)
    reinterpret_cast<uint4*>(smem + kLutOff)[e] = __ldg(reinterpret_cast<const uint4*>(a.consts + kBOff) + e);
  if (warp == 0) tc::tmem_alloc(&tmem_slot, 512);
  if (tid == 0) {
    tc::mbar_init(&bar_full[0], 1);
    tc::mbar_init(&bar_full[1], 1);
    tc::mbar_init(&bar_tmem_empty[0], kHalves ? kMathWarps * 16 : kMathWarps * 32);
    tc::mbar_init(&bar_tmem_empty[1], kMathWarps * 32);
    tc::mbar_init(&bar_bfull[0], kMathWarps * 32);
    tc::mbar_init(&bar_bfull[1], kMathWarps * 32);
    tc::mbar_init(&bar_done, kMathWarps * 32);
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp < 4) {
    // ---------------- issuer warpgroup ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kIssuerRegs));
    if (warp == 0) {
      for (int i = 0; i < n_my; ++i) {
        tc::mbar_wait(&bar_bfull[i & 1], uint32_t((i >> 1) & 1));
        if constexpr (kHalves) {
          // half h of D(i-1) read -> MMA(i) half h; the halves commit separately
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (i > 0) tc::mbar_wait(&bar_tmem_empty[h], uint32_t((i - 1) & 1));
            tc::fence_after();
            issue_mma_half(tmem, smem, i & 1, h, &bar_full[h]);
          }
        } else {
          if (i > 0) tc::mbar_wait(&bar_tmem_empty[0], uint32_t((i - 1) & 1));
          tc::fence_after();
          issue_mma_half(tmem, smem, i & 1, 0, nullptr);
          issue_mma_half(tmem, smem, i & 1, 1, &bar_full[0]);
        }
        // tmem_empty(i-1) follows every thread's store of its maxima of item i - 2
        if (i >= 2 && lane == 0)
          publish(s_wmax[(i - 2) & 3], mask_at(int64_t(a.v_lo) + t_lo + i - 2, a.v_lo, a.v_hi), a);
      }
      tc::mbar_wait(&bar_done, 0u);
      tc::fence_after();
      if (lane == 0)
        for (int i = n_my - 2 < 0 ? 0 : n_my - 2; i < n_my; ++i)
          publish(s_wmax[i & 3], mask_at(int64_t(a.v_lo) + t_lo + i, a.v_lo, a.v_hi), a);
      __syncwarp();
      tc::tmem_dealloc(tmem, 512);
    }
  } else {
    // ---------------- transform warps ----------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kMathRegs));
    const int mt = tid - 128, mw = mt >> 5;
    // generation: rows cA = 16 mw + (lane & 7) + 8 (lane >> 4) and cA + 128, plane
    // words 4 q .. 4 q + 3 of each (q = lane bit 3).  A quarter-warp (one STS.128
    // phase) is 8 consecutive rows of one q: chunk positions j ^ (c & 7) all differ.
    const int q = (lane >> 3) & 1;
    const int cA = 16 * mw + (lane & 7) + 8 * (lane >> 4);
    const uint32_t* __restrict__ planes = a.planes;
    const uint32_t lut = tc::smem_u32(smem + kLutOff) + uint32_t(lane & (kCopies - 1)) * 8u;
    uint32_t g[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) g[k] = 0;
    uint32_t vcur = 0;
    auto load_pl = [&](int i, uint4 (&x)[2]) {
      const uint32_t* p = planes + int64_t(i) * 2048 + cA * 8 + 4 * q;
      x[0] = __ldg(reinterpret_cast<const uint4*>(p));
      x[1] = __ldg(reinterpret_cast<const uint4*>(p + 128 * 8));
    };
    auto xor_pl = [&](const uint4 (&x)[2]) {
      g[0] ^= x[0].x; g[1] ^= x[0].y; g[2] ^= x[0].z; g[3] ^= x[0].w;
      g[4] ^= x[1].x; g[5] ^= x[1].y; g[6] ^= x[1].z; g[7] ^= x[1].w;
    };
    auto xor_all = [&](uint32_t d) {
      while (d) {
        const int i = __ffs(d) - 1;
        d &= d - 1;
        uint4 x[2];
        load_pl(i, x);
        xor_pl(x);
      }
    };
    // B rows of one item: the table lookups and byte stages run into registers
    // (o[]) while no TMEM values are live, so all 32 lookups of a thread are in
    // flight together; the stores follow once MMA(i) has released the buffer.
    uint4 o[16];
    auto gen_lookup = [&]() {
#pragma unroll
      for (int k = 0; k < 8; ++k) word_lookup(g[k], lut, o[2 * k], o[2 * k + 1]);
    };
    auto gen_stages = [&]() {
#pragma unroll
      for (int k = 0; k < 8; ++k) word_stages(o[2 * k], o[2 * k + 1]);
      if constexpr (kGenStages == 7) {
        // r bits 5, 6: across the 4 words of each row (diff + 32, + 64 per byte: every byte in [0, 128])
        auto bfly = [](uint4& x, uint4& y, uint32_t b) {
          const uint4 s4 = make_uint4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
          y = make_uint4(x.x - y.x + b, x.y - y.y + b, x.z - y.z + b, x.w - y.w + b);
          x = s4;
        };
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {  // lo / hi chunk of every word
            bfly(o[8 * h + j], o[8 * h + 2 + j], 0x20202020u);
            bfly(o[8 * h + 4 + j], o[8 * h + 6 + j], 0x20202020u);
            bfly(o[8 * h + j], o[8 * h + 4 + j], 0x40404040u);
            bfly(o[8 * h + 2 + j], o[8 * h + 6 + j], 0x40404040u);
          }
        }
      }
    };
    auto gen_compute = [&]() {
      gen_lookup();
      gen_stages();
    };
    auto gen_sts = [&](int buf) {
      uint8_t* bb = smem + kBOff + buf * kBBytes;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int c = cA + 128 * half;
        uint8_t* row = bb + (c >> 3) * 2048 + q * 1024 + (c & 7) * 128;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          *reinterpret_cast<uint4*>(row + (((2 * w) ^ (c & 7)) << 4)) = o[2 * (4 * half + w)];
          *reinterpret_cast<uint4*>(row + (((2 * w + 1) ^ (c & 7)) << 4)) = o[2 * (4 * half + w) + 1];
        }
      }
    };
    auto gen_done = [&](int buf) {  // generic-proxy stores -> visible to the tensor core, then bfull
      tc::fence_proxy_async();
      mbar_arrive(&bar_bfull[buf]);
    };
    for (int k = 0; k < 3 && k < n_my; ++k) {
      const uint32_t vn = mask_at(int64_t(a.v_lo) + t_lo + k, a.v_lo, a.v_hi);
      xor_all(vcur ^ vn);
      vcur = vn;
      gen_compute();
      if (k < 2) {  // item 2 stays in o[] until MMA(0) has released buffer 0
        gen_sts(k);
        gen_done(k);
      }
    }
    // TMEM lane of this thread (warp w may only touch lanes 32 (w % 4) .. + 31)
    const uint32_t tbase = tmem + (uint32_t((mw & 3) * 32) << 16) + uint32_t(mw >> 2) * 256;
    const int hg = kHalves ? (mw >> 2) : 0;  // which M half this warp reads
    for (int i = 0; i < n_my; ++i) {
      // prefetch the first changed plane of the item three steps ahead
      const bool gen = i + 3 < n_my;
      uint32_t vn = 0, d = 0;
      uint4 pa[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
      if (gen) {
        vn = mask_at(int64_t(a.v_lo) + t_lo + i + 3, a.v_lo, a.v_hi);
        d = vcur ^ vn;
        if (d) {
          load_pl(__ffs(d) - 1, pa);
          d &= d - 1;
        }
      }
      tc::mbar_wait(&bar_full[hg], uint32_t(i & 1));
      tc::fence_after();
      uint32_t R[128];
      uint32_t(&R0)[64] = *reinterpret_cast<uint32_t(*)[64]>(&R[0]);
      uint32_t(&R1)[64] = *reinterpret_cast<uint32_t(*)[64]>(&R[64]);
      tc::tmem_ld_x64_p16(tbase, R0);
      tc::tmem_ld_x64_p16(tbase + 128, R1);
      tc::wait_ld_tied(R0);
      tc::wait_ld_tied(R1);
      tc::fence_before();
      // MMA(i+1) (this half) may start: no fence or store sits in that gap.
      // (B stores issued under the TMEM loads: 1.11 vs 0.86 ms; the proxy fence
      // and bfull arrive moved behind the fold: 0.864 vs 0.862 ms.)
      mbar_arrive(&bar_tmem_empty[hg]);
      // B(i+2) from o[] into the buffer MMA(i) released; then B(i+3): plane XOR
      // and the 32 lookups, in flight under the fold
      auto next_b = [&]() {
        if (i + 2 < n_my) {
          gen_sts(i & 1);
          gen_done(i & 1);
        }
        if (gen) {
          xor_pl(pa);
          if (d) xor_all(d);  // rare: more than one changed bit
          vcur = vn;
          gen_lookup();
        }
      };
      // R[j] = columns (2j, 2j + 1), D = W_15 / 2 + 2^14; register bit 6 = column
      // bit 7 = r bit 7: the top stage, fused with the max / min fold
      auto fold = [&]() {
#pragma unroll
        for (int sb = 4; sb < (kGenStages == 7 ? 4 : 6); ++sb)  // 5-stage generation: r bits 5, 6 here
#pragma unroll
          for (int k = 0; k < 128; ++k)
            if ((k & (1 << sb)) == 0) {
              const uint32_t x = R[k], y = R[k | (1 << sb)];
              R[k] = x + y;
              R[k | (1 << sb)] = x - y + (0x02000200u << sb);
            }
        uint32_t mx = 0u, mn = 0xFFFFFFFFu;
#pragma unroll
        for (int k = 0; k < 64; ++k) {
          const uint32_t x = R[k], y = R[k + 64];
          const uint32_t S = x + y;
          const uint32_t D = x - y + 0x80008000u;
          mx = __vimax3_u16x2(mx, S, D);
          mn = __vimin3_u16x2(mn, S, D);
        }
        const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, uint32_t(lanes_maxabs<16>(mx, mn)));
        if (lane == 0) s_wmax[i & 3][mw] = m;
      };
      if (kHalves && hg == 0) {
        // half 0 is ready half a GEMM before MMA(i) has released B(i)'s buffer:
        // fold first, store afterwards
        fold();
        tc::mbar_wait(&bar_full[1], uint32_t(i & 1));
        tc::fence_after();
        mbar_arrive(&bar_tmem_empty[1]);
        next_b();
      } else {
        next_b();
        fold();
      }
      if (gen) gen_stages();
    }
    tc::fence_before();
    mbar_arrive(&bar_done);
  }
}

// One generation unit of the 16-warp kernels: the 4 plane words g of one
// (row, word quad) -> 128 B of B (o[2 w], o[2 w + 1] = word w): 16 lookups, two
// byte-lane stages inside each word (r bits 3, 4) and two across the 4 words
// (r bits 5, 6; diff + 32, + 64 per byte: every byte in [0, 128])
__device__ __forceinline__ void gen_unit(const uint4& g, uint32_t lut, uint4 (&o)[8]) {
  word_lookup(g.x, lut, o[0], o[1]);
  word_lookup(g.y, lut, o[2], o[3]);
  word_lookup(g.z, lut, o[4], o[5]);
  word_lookup(g.w, lut, o[6], o[7]);
#pragma unroll
  for (int k = 0; k < 4; ++k) word_stages(o[2 * k], o[2 * k + 1]);
  auto bfly = [](uint4& x, uint4& y, uint32_t b) {
    const uint4 s4 = make_uint4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w);
    y = make_uint4(x.x - y.x + b, x.y - y.y + b, x.z - y.z + b, x.w - y.w + b);
    x = s4;
  };
#pragma unroll
  for (int j = 0; j < 2; ++j) {  // lo / hi chunk of every word
    bfly(o[j], o[2 + j], 0x20202020u);
    bfly(o[4 + j], o[6 + j], 0x20202020u);
    bfly(o[j], o[4 + j], 0x40404040u);
    bfly(o[2 + j], o[6 + j], 0x40404040u);
  }
}
// ... and its 8 conflict-free STS.128 into the MN-major SW128 buffer (row = the
// unit's 128-byte row, sw = (c & 7) << 4 the row's chunk swizzle)
__device__ __forceinline__ void sts_unit(uint8_t* row, uint32_t sw, const uint4 (&o)[8]) {
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    *reinterpret_cast<uint4*>(row + (uint32_t(32 * w) ^ sw)) = o[2 * w];
    *reinterpret_cast<uint4*>(row + (uint32_t(32 * w + 16) ^ sw)) = o[2 * w + 1];
  }
}

// ---------------------------------------------------------------------------
// k_tc_lut16: the same job with 16 transform warps (4 per SM sub-partition
// instead of 2, so one warp's TMEM / table-lookup latency hides behind three
// others).  Warp mw = (column half ch, M half h, lane quarter): it reads the 128
// TMEM columns {64 ch .. + 63} u {128 + 64 ch .. + 63} of its lanes (the top
// stage pairs column n with n + 128) into 64 packed registers, and generates
// one (row c, word quad q) unit of B: 4 plane words, 16 lookups, 32 output
// registers.  Every warp runs: wait full[h](i) -> read D -> tmem_empty[h] ->
// fold -> B(i+2) into registers -> (half 0: wait full[1](i), tmem_empty[1]) ->
// store B(i+2) -> bfull, so TMEM values and B bytes are never live together
// (112 registers per transform thread: 640 threads x 96 at launch, the issuer
// warpgroup drops to 24).
#ifndef SBW_LUT16_PIN
#define SBW_LUT16_PIN 1
#endif
#ifndef SBW_LUT16_TWO_LOADS
#define SBW_LUT16_TWO_LOADS 1
#endif
constexpr int kW16 = 16;
constexpr int kThreads16 = 128 + kW16 * 32;
constexpr int kIssuerRegs16 = 24, kMathRegs16 = 112;
static_assert(4 * 32 * kIssuerRegs16 + kW16 * 32 * kMathRegs16 <= kThreads16 * 96,
              "setmaxnreg split must fit the CTA's launch allocation (640 x 96 registers)");

__global__ void __launch_bounds__(kThreads16, 1) k_tc_lut16(LutArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_full[2], bar_tmem_empty[2], bar_bfull[2], bar_done;
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(16) uint32_t s_wmax[4][kW16];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t total = int64_t(a.v_hi) - a.v_lo;
  const int64_t t_lo64 = total * blockIdx.x / gridDim.x;
  const int n_my = int(total * (blockIdx.x + 1) / gridDim.x - t_lo64);
  const uint32_t q_lo = a.v_lo + uint32_t(t_lo64);  // natural position of this CTA's first mask (< 2^24)
  // mask_at in 32-bit arithmetic (positions and masks are below 2^24)
  auto mask32 = [&](uint32_t qpos) -> uint32_t {
    const uint32_t b = qpos & ~255u;
    if (b >= a.v_lo && b + 256u <= a.v_hi) {
      const uint32_t kk = qpos & 255u;
      return b | (kk ^ (kk >> 1));
    }
    return qpos;
  };

  for (int e = tid; e < kBOff / 16; e += kThreads16)
    reinterpret_cast<uint4*>(smem)[e] = __ldg(reinterpret_cast<const uint4*>(a.consts) + e);
  for (int e = tid; e < kLutBytes / 16; e += kThreads16)
    reinterpret_cast<uint4*>(smem + kLutOff)[e] = __ldg(reinterpret_cast<const uint4*>(a.consts + kBOff) + e);
  if (warp == 0) tc::tmem_alloc(&tmem_slot, 512);
  if (tid == 0) {
    tc::mbar_init(&bar_full[0], 1);
    tc::mbar_init(&bar_full[1], 1);
    tc::mbar_init(&bar_tmem_empty[0], kW16 * 16);  // the half-0 warps
    tc::mbar_init(&bar_tmem_empty[1], kW16 * 32);  // the half-1 warps + the half-0 warps after full[1]
    tc::mbar_init(&bar_bfull[0], kW16 * 32);
    tc::mbar_init(&bar_bfull[1], kW16 * 32);
    tc::mbar_init(&bar_done, kW16 * 32);
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kIssuerRegs16));
    if (warp == 0) {
      auto publish16 = [&](int i) {
        const uint32_t* w = s_wmax[i & 3];
        uint32_t m = 0;
#pragma unroll
        for (int k = 0; k < kW16; ++k) m = max(m, w[k]);
        const uint32_t v = mask32(q_lo + uint32_t(i));
        a.max_abs[v - a.v_lo] = int(m);
        if (a.key) atomicMax(a.key, nl_key(int(m), v));
      };
      for (int i = 0; i < n_my; ++i) {
        tc::mbar_wait(&bar_bfull[i & 1], uint32_t((i >> 1) & 1));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (i > 0) tc::mbar_wait(&bar_tmem_empty[h], uint32_t((i - 1) & 1));
          tc::fence_after();
          issue_mma_half(tmem, smem, i & 1, h, &bar_full[h]);
        }
        if (i >= 2 && lane == 0) publish16(i - 2);
      }
      tc::mbar_wait(&bar_done, 0u);
      tc::fence_after();
      if (lane == 0)
        for (int i = n_my - 2 < 0 ? 0 : n_my - 2; i < n_my; ++i) publish16(i);
      __syncwarp();
      tc::tmem_dealloc(tmem, 512);
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kMathRegs16));
    const int mt = tid - 128, mw = mt >> 5;
    const int hg = (mw >> 2) & 1, ch = mw >> 3;
    // generation unit: row c = 16 mw + (lane & 7) + 8 (lane >> 4), word quad q = lane bit 3
    const int q = (lane >> 3) & 1;
    const int c = 16 * mw + (lane & 7) + 8 * (lane >> 4);
#if SBW_LUT16_PIN
    // thread constants as opaque register values (ptxas otherwise re-derives them from
    // S2R SR_TID.X in every iteration)
    uint32_t pl_off = uint32_t(c * 8 + 4 * q);
    uint32_t lut = tc::smem_u32(smem + kLutOff) + uint32_t(lane & (kCopies - 1)) * 8u;
    uint32_t row_off = uint32_t(kBOff + (c >> 3) * 2048 + q * 1024 + (c & 7) * 128);
    uint32_t sw = uint32_t(c & 7) << 4;
    asm volatile("mov.b32 %0, %0;" : "+r"(pl_off));
    asm volatile("mov.b32 %0, %0;" : "+r"(lut));
    asm volatile("mov.b32 %0, %0;" : "+r"(row_off));
    asm volatile("mov.b32 %0, %0;" : "+r"(sw));
    const uint32_t* __restrict__ pl = a.planes + pl_off;
#else
    const uint32_t* __restrict__ pl = a.planes + c * 8 + 4 * q;
    const uint32_t lut = tc::smem_u32(smem + kLutOff) + uint32_t(lane & (kCopies - 1)) * 8u;
    const uint32_t row_off = uint32_t(kBOff + (c >> 3) * 2048 + q * 1024 + (c & 7) * 128);
    const uint32_t sw = uint32_t(c & 7) << 4;  // swizzle XOR of this row's chunk offsets
#endif
    // (pinning these thread constants in registers, so ptxas cannot re-derive them
    // from S2R SR_TID.X every iteration, was slower: 0.725 vs 0.711 ms at 112 registers)
    uint4 g = make_uint4(0, 0, 0, 0);
    uint32_t vcur = 0;
    auto xor_all = [&](uint32_t d) {
      while (d) {
        const int i = __ffs(d) - 1;
        d &= d - 1;
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(pl + int64_t(i) * 2048));
        g.x ^= x.x; g.y ^= x.y; g.z ^= x.z; g.w ^= x.w;
      }
    };
    uint4 o[8];
    auto gen_compute = [&]() { gen_unit(g, lut, o); };
    auto gen_sts = [&](int buf) {
      sts_unit(smem + row_off + buf * kBBytes, sw, o);
      tc::fence_proxy_async();
      mbar_arrive(&bar_bfull[buf]);
    };
    for (int k = 0; k < 2 && k < n_my; ++k) {
      const uint32_t vn = mask32(q_lo + uint32_t(k));
      xor_all(vcur ^ vn);
      vcur = vn;
      gen_compute();
      gen_sts(k);
    }
    const uint32_t tbase = tmem + (uint32_t((mw & 3) * 32) << 16) + uint32_t(hg) * 256 + uint32_t(ch) * 64;

    for (int i = 0; i < n_my; ++i) {
      // prefetch the first changed plane of the item two steps ahead
      const bool gen = i + 2 < n_my;
      uint32_t vn = 0, d = 0;
      uint4 pa = make_uint4(0, 0, 0, 0);
      if (gen) {
        vn = mask32(q_lo + uint32_t(i) + 2u);
        d = vcur ^ vn;
        if (d) {
          pa = __ldg(reinterpret_cast<const uint4*>(pl + int64_t(__ffs(d) - 1) * 2048));
          d &= d - 1;
        }
      }
      tc::mbar_wait(&bar_full[hg], uint32_t(i & 1));
      tc::fence_after();
#if SBW_LUT16_TWO_LOADS
      {
        // two rounds of 32 + 32 columns: 32 TMEM registers live instead of 64 (at 112
        // registers the one-shot read made ptxas spill and re-derive thread constants
        // every iteration); MMA(i+1) of this half is >= half a GEMM away, so the later
        // tmem_empty costs nothing
        uint32_t mx = 0u, mn = 0xFFFFFFFFu;
#pragma unroll
        for (int r2 = 0; r2 < 2; ++r2) {
          uint32_t X[16], Y[16];  // columns 64 ch + 32 r2 + (2j, 2j+1) and the same + 128
          tc::tmem_ld_x16_p16(tbase + 32 * r2, X);
          tc::tmem_ld_x16_p16(tbase + 32 * r2 + 128, Y);
          tc::wait_ld_tied(X);
          tc::wait_ld_tied(Y);
          if (r2 == 1) {
            tc::fence_before();
            mbar_arrive(&bar_tmem_empty[hg]);
          }
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const uint32_t S = X[k] + Y[k];
            const uint32_t D = X[k] - Y[k] + 0x80008000u;
            mx = __vimax3_u16x2(mx, S, D);
            mn = __vimin3_u16x2(mn, S, D);
          }
        }
        const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, uint32_t(lanes_maxabs<16>(mx, mn)));
        if (lane == 0) s_wmax[i & 3][mw] = m;
      }
#else
      {
        uint32_t X[32], Y[32];  // columns 64 ch + (2j, 2j+1) and the same + 128
        tc::tmem_ld_x32_p16(tbase, X);
        tc::tmem_ld_x32_p16(tbase + 128, Y);
        tc::wait_ld_tied(X);
        tc::wait_ld_tied(Y);
        tc::fence_before();
        mbar_arrive(&bar_tmem_empty[hg]);
        uint32_t mx = 0u, mn = 0xFFFFFFFFu;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const uint32_t S = X[k] + Y[k];
          const uint32_t D = X[k] - Y[k] + 0x80008000u;
          mx = __vimax3_u16x2(mx, S, D);
          mn = __vimin3_u16x2(mn, S, D);
        }
        const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, uint32_t(lanes_maxabs<16>(mx, mn)));
        if (lane == 0) s_wmax[i & 3][mw] = m;
      }
#endif
      if (gen) {
        g.x ^= pa.x; g.y ^= pa.y; g.z ^= pa.z; g.w ^= pa.w;
        if (d) xor_all(d);  // rare: more than one changed bit
        vcur = vn;
        gen_compute();
      }
      if (hg == 0) {  // B(i)'s buffer is free once MMA(i) half 1 is done too
        tc::mbar_wait(&bar_full[1], uint32_t(i & 1));
        tc::fence_after();
        mbar_arrive(&bar_tmem_empty[1]);
      }
      if (gen) gen_sts(i & 1);
    }
    tc::fence_before();
    mbar_arrive(&bar_done);
  }
}

// ---------------------------------------------------------------------------
// k_tc_lut_emit: pass A of the multi-pass path (n = 17..24) with the same
// table-lookup generation.  An item is one component x one 2^16 block pair bp;
// x bit 15 (the pair's block parity = c bit 7 = the M half) stays out of the
// GEMM -- half h multiplies Hs (128 x 128) with B rows 128 h .. 128 h + 127 only:
// 2 x (4 + 1) MMAs per item instead of 18 -- so D = W_14 / 2 + 2^13 for x bits
// 0..6 and 8..14, the int16 stage adds x bit 7, and the thread writes the
// biased u16 s = W_15 / 2 + 2^14 of block 2 bp + h in a block-internal word order
// of its own: word ((ch 16 + jj) 128 + u7) 4 + (0..3) for its jj-th uint4 (pass B
// only pairs equal word positions across blocks, sbw_passb.cuh).  Replaces
// k_tc_hybrid<EMIT> (7 int16 stages per item on the ALUs).
struct LutEmitArgs {
  const uint8_t* consts;
  const uint32_t* planes;
  int64_t plane_words;  // 2^n / 32
  uint32_t v_first;     // batch position j holds mask mask_at(v_first + j, run_lo, run_hi)
  uint32_t run_lo, run_hi;
  int64_t n_comp, n_items;
  int n_full;
  uint32_t* emit;
  const int* gate;  // run only if (*gate != 0) == gate_on (gate may be null)
  int gate_on;
};

__device__ __forceinline__ void issue_mma_half_emit(uint32_t tmem, const uint8_t* smem, int buf, int h,
                                                    uint64_t* bar) {
  const uint64_t dhs = tc::sdesc(tc::smem_u32(smem + kHsOff), 128, 1024);
  const uint64_t dab = tc::sdesc(tc::smem_u32(smem + kAbOff), 128, 256);
  const uint64_t db0 = sdesc_mn_sw128(tc::smem_u32(smem + kBOff + buf * kBBytes), 1024, 2048);
  const uint64_t dbb = tc::sdesc(tc::smem_u32(smem + kBbOff), 128, 256);
#pragma unroll
  for (int kb = 0; kb < 5; ++kb) {
    const uint64_t da = kb == 4 ? dab + uint64_t((h * 4096) >> 4) : dhs + uint64_t((kb * 256) >> 4);
    const uint64_t db = kb == 4 ? dbb : db0 + uint64_t(((4 * h + kb) * 8192) >> 4);
    tc::mma_i8_elect(tmem + h * 256, da, db, kb == 4 ? kIdescK : kIdescMN, kb > 0 ? 1u : 0u);
  }
  tc::mma_commit_elect(bar);
}

__global__ void __launch_bounds__(kThreads16, 1) k_tc_lut_emit(LutEmitArgs a) {
  static_assert(kGenStages == 7, "k_tc_lut_emit assumes the 7-stage generation");
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar_full[2], bar_tmem_empty[2], bar_bfull[2], bar_done;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (a.gate && ((*a.gate != 0) != (a.gate_on != 0))) return;  // CTA-uniform, before any setup
  const int64_t t_lo = a.n_items * blockIdx.x / gridDim.x;
  const int n_my = int(a.n_items * (blockIdx.x + 1) / gridDim.x - t_lo);

  for (int e = tid; e < kBOff / 16; e += kThreads16)
    reinterpret_cast<uint4*>(smem)[e] = __ldg(reinterpret_cast<const uint4*>(a.consts) + e);
  for (int e = tid; e < kLutBytes / 16; e += kThreads16)
    reinterpret_cast<uint4*>(smem + kLutOff)[e] = __ldg(reinterpret_cast<const uint4*>(a.consts + kBOff) + e);
  if (warp == 0) tc::tmem_alloc(&tmem_slot, 512);
  if (tid == 0) {
    tc::mbar_init(&bar_full[0], 1);
    tc::mbar_init(&bar_full[1], 1);
    tc::mbar_init(&bar_tmem_empty[0], kW16 * 16);
    tc::mbar_init(&bar_tmem_empty[1], kW16 * 32);
    tc::mbar_init(&bar_bfull[0], kW16 * 32);
    tc::mbar_init(&bar_bfull[1], kW16 * 32);
    tc::mbar_init(&bar_done, kW16 * 32);
  }
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_slot;

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kIssuerRegs16));
    if (warp == 0) {
      for (int i = 0; i < n_my; ++i) {
        tc::mbar_wait(&bar_bfull[i & 1], uint32_t((i >> 1) & 1));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (i > 0) tc::mbar_wait(&bar_tmem_empty[h], uint32_t((i - 1) & 1));
          tc::fence_after();
          issue_mma_half_emit(tmem, smem, i & 1, h, &bar_full[h]);
        }
      }
      tc::mbar_wait(&bar_done, 0u);
      tc::fence_after();
      __syncwarp();
      tc::tmem_dealloc(tmem, 512);
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kMathRegs16));
    const int mt = tid - 128, mw = mt >> 5;
    const int hg = (mw >> 2) & 1, ch = mw >> 3;
    const int q = (lane >> 3) & 1;
    const int c = 16 * mw + (lane & 7) + 8 * (lane >> 4);
    const uint32_t* __restrict__ pl = a.planes + c * 8 + 4 * q;
    const uint32_t lut = tc::smem_u32(smem + kLutOff) + uint32_t(lane & (kCopies - 1)) * 8u;
    const uint32_t row_off = uint32_t(kBOff + (c >> 3) * 2048 + q * 1024 + (c & 7) * 128);
    const uint32_t sw = uint32_t(c & 7) << 4;
    uint4 g = make_uint4(0, 0, 0, 0);
    uint32_t vcur = 0, bpcur = 0;
    // items of a CTA are consecutive: (block pair bp, batch position pos) cursors
    // stepped incrementally (one 64-bit division at the start, none in the loop)
    const uint32_t ncomp = uint32_t(a.n_comp);
    auto mask32 = [&](uint32_t qpos) -> uint32_t {  // mask_at in 32-bit arithmetic (masks < 2^24)
      const uint32_t b = qpos & ~255u;
      if (b >= a.run_lo && b + 256u <= a.run_hi) {
        const uint32_t kk = qpos & 255u;
        return b | (kk ^ (kk >> 1));
      }
      return qpos;
    };
    auto step = [&](uint32_t& bp, uint32_t& pos) {
      if (++pos == ncomp) {
        pos = 0;
        ++bp;
      }
    };
    uint32_t bp_i = uint32_t(t_lo / a.n_comp), pos_i = uint32_t(t_lo - int64_t(bp_i) * a.n_comp);  // item i
    uint32_t bp_g = bp_i, pos_g = pos_i;                                                            // item generated next
    auto xor_all = [&](uint32_t d, uint32_t bp) {
      while (d) {
        const int i = __ffs(d) - 1;
        d &= d - 1;
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(pl + int64_t(i) * a.plane_words + int64_t(bp) * 2048));
        g.x ^= x.x; g.y ^= x.y; g.z ^= x.z; g.w ^= x.w;
      }
    };
    uint4 o[8];
    auto gen_compute = [&]() { gen_unit(g, lut, o); };
    auto gen_sts = [&](int buf) {
      sts_unit(smem + row_off + buf * kBBytes, sw, o);
      tc::fence_proxy_async();
      mbar_arrive(&bar_bfull[buf]);
    };
    auto advance = [&](uint32_t vn, uint32_t bpn, uint4 pa, uint32_t d, bool reset) {
      if (reset) {
        g = make_uint4(0, 0, 0, 0);
        bpcur = bpn;
      }
      g.x ^= pa.x; g.y ^= pa.y; g.z ^= pa.z; g.w ^= pa.w;
      if (d) xor_all(d, bpn);
      vcur = vn;
    };
    for (int k = 0; k < 2 && k < n_my; ++k) {
      const uint32_t vn = mask32(a.v_first + pos_g), bpn = bp_g;
      step(bp_g, pos_g);
      const bool reset = bpn != bpcur;
      advance(vn, bpn, make_uint4(0, 0, 0, 0), reset ? vn : (vcur ^ vn), reset);
      gen_compute();
      gen_sts(k);
    }
    const uint32_t tbase = tmem + (uint32_t((mw & 3) * 32) << 16) + uint32_t(hg) * 256 + uint32_t(ch) * 64;
    const int u7 = 32 * (mw & 3) + lane;
    for (int i = 0; i < n_my; ++i) {
      // prefetch the first changed plane of the item two steps ahead
      const bool gen = i + 2 < n_my;
      uint32_t vn = 0, bpn = 0, d = 0;
      bool reset = false;
      uint4 pa = make_uint4(0, 0, 0, 0);
      if (gen) {
        vn = mask32(a.v_first + pos_g);
        bpn = bp_g;
        step(bp_g, pos_g);
        reset = bpn != bpcur;
        d = reset ? vn : (vcur ^ vn);
        if (d) {
          pa = __ldg(reinterpret_cast<const uint4*>(pl + int64_t(__ffs(d) - 1) * a.plane_words + int64_t(bpn) * 2048));
          d &= d - 1;
        }
      }
      // where this thread's words of item i go: component slot pos_i of the batch, block 2 bp + h
      uint32_t* dst = a.emit + (int64_t(pos_i) << (a.n_full - 1)) + (int64_t(2 * bp_i + hg) << 14) +
                      (int64_t(ch) * 16 * 128 + u7) * 4;
      step(bp_i, pos_i);
      tc::mbar_wait(&bar_full[hg], uint32_t(i & 1));
      tc::fence_after();
      {
        uint32_t X[32], Y[32];  // columns 64 ch + (2j, 2j+1) and the same + 128 (x bit 7)
        tc::tmem_ld_x32_p16(tbase, X);
        tc::tmem_ld_x32_p16(tbase + 128, Y);
        tc::wait_ld_tied(X);
        tc::wait_ld_tied(Y);
        tc::fence_before();
        mbar_arrive(&bar_tmem_empty[hg]);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const uint32_t x = X[k], y = Y[k];
          X[k] = x + y;
          Y[k] = x - y + 0x40004000u;
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          __stcs(reinterpret_cast<uint4*>(dst + jj * 512), make_uint4(X[4 * jj], X[4 * jj + 1], X[4 * jj + 2], X[4 * jj + 3]));
          __stcs(reinterpret_cast<uint4*>(dst + (8 + jj) * 512),
                 make_uint4(Y[4 * jj], Y[4 * jj + 1], Y[4 * jj + 2], Y[4 * jj + 3]));
        }
      }
      if (gen) {
        advance(vn, bpn, pa, d, reset);
        gen_compute();
      }
      if (hg == 0) {  // B(i)'s buffer is free once MMA(i) half 1 is done too
        tc::mbar_wait(&bar_full[1], uint32_t(i & 1));
        tc::fence_after();
        mbar_arrive(&bar_tmem_empty[1]);
      }
      if (gen) gen_sts(i & 1);
    }
    tc::fence_before();
    mbar_arrive(&bar_done);
  }
}

std::mutex g_lut_mu;
uint8_t* g_lut_consts[2][64] = {};
int lut_consts(int dev, cudaStream_t st, const uint8_t** out, int emit = 0) {
  std::lock_guard<std::mutex> lk(g_lut_mu);
  if (!g_lut_consts[emit][dev & 63]) {
    uint8_t* p = nullptr;
    SBW_CUDA_CHECK(cudaMalloc(&p, kImgBytes));
    k_lut_consts<<<64, 256, 0, st>>>(p, emit);
    SBW_LAUNCH_CHECK("k_lut_consts");
    SBW_CUDA_CHECK(cudaStreamSynchronize(st));
    g_lut_consts[emit][dev & 63] = p;
  }
  *out = g_lut_consts[emit][dev & 63];
  return SBW_OK;
}

}  // namespace

// SBW_TC_LUT=0 keeps k_tc_hybrid<NL, 16> for the n = 16 NL path (A/B runs)
bool tc_lut_enabled() {
  static const bool on = [] {
    const char* e = getenv("SBW_TC_LUT");
    return !(e && e[0] == '0');
  }();
  return on;
}

int launch_tc16_nl_lut(const uint32_t* planes, uint32_t v_lo, uint32_t v_hi, int32_t* max_abs,
                       unsigned long long* key, cudaStream_t st) {
  const int64_t items = int64_t(v_hi) - v_lo;
  if (items <= 0) return SBW_OK;
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  static unsigned long long attr_done = 0;
  if (!(attr_done >> (dp.device & 63) & 1ull)) {
    SBW_CUDA_CHECK(cudaFuncSetAttribute(k_tc_lut, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    SBW_CUDA_CHECK(cudaFuncSetAttribute(k_tc_lut16, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr_done |= 1ull << (dp.device & 63);
  }
  LutArgs a{};
  if (int rc = lut_consts(dp.device, st, &a.consts)) return rc;
  a.planes = planes;
  a.v_lo = v_lo;
  a.v_hi = v_hi;
  a.max_abs = max_abs;
  a.key = key;
  const int grid = int(items < dp.sm_count ? items : dp.sm_count);
  static const int warps = getenv("SBW_LUT_WARPS") ? atoi(getenv("SBW_LUT_WARPS")) : SBW_LUT_WARPS_DEFAULT;
  if (warps == 16) {
    k_tc_lut16<<<grid, kThreads16, kSmem, st>>>(a);
    SBW_LAUNCH_CHECK("k_tc_lut16");
    return SBW_OK;
  }
  k_tc_lut<<<grid, kAllThreads, kSmem, st>>>(a);
  SBW_LAUNCH_CHECK("k_tc_lut");
  return SBW_OK;
}

// Off by default (SBW_TC_LUT_EMIT=1 selects it): exact, but pass A is bound by the
// 128 KiB an SM must write per item, not by its arithmetic, and the full runs
// measured 852 vs 814 ms (20x20) and 954 vs 919 ms (24x16) against k_tc_hybrid<EMIT>.
bool tc_lut_emit_enabled() {
  static const bool on = [] {
    const char* e = getenv("SBW_TC_LUT_EMIT");
    return e && e[0] == '1';
  }();
  return on;
}

int launch_tc_emit_lut(const uint32_t* planes, int n, uint32_t v_first, int64_t n_comp, uint32_t* emit,
                       uint32_t run_lo, uint32_t run_hi, cudaStream_t st, const int* gate, int gate_on) {
  LutEmitArgs a{};
  a.planes = planes;
  a.plane_words = (int64_t(1) << n) >> 5;
  a.v_first = v_first;
  a.run_lo = run_lo;
  a.run_hi = run_hi;
  a.n_comp = n_comp;
  a.n_items = n_comp << (n - 16);
  a.n_full = n;
  a.emit = emit;
  a.gate = gate;
  a.gate_on = gate_on;
  if (a.n_items <= 0) return SBW_OK;
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  static unsigned long long attr_done = 0;
  if (!(attr_done >> (dp.device & 63) & 1ull)) {
    SBW_CUDA_CHECK(cudaFuncSetAttribute(k_tc_lut_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr_done |= 1ull << (dp.device & 63);
  }
  if (int rc = lut_consts(dp.device, st, &a.consts, 1)) return rc;
  const int grid = int(a.n_items < dp.sm_count ? a.n_items : dp.sm_count);
  k_tc_lut_emit<<<grid, kThreads16, kSmem, st>>>(a);
  SBW_LAUNCH_CHECK("k_tc_lut_emit");
  return SBW_OK;
}

}  // namespace sbw
