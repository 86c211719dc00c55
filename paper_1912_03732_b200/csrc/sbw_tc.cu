// Tensor-core + packed-integer hybrid kernel k_tc_hybrid<EMIT>:
//   EMIT = false: the n = 16 nonlinearity path (sbw_nl), K2 in DESIGN.md;
//   EMIT = true : pass A of the multi-pass path (n = 17..24), 15 stages per
//                 2^15 block, biased u16 out for pass B (sbw_passb.cuh).
//
// Replaces, per output mask v, polarity_row (sbox.py:145-152) +
// fwht_column_in_place (walsh.py:73-104) + column_nonlinearity
// (walsh.py:107-114), like k_tile_simd, with the 16 butterfly stages of a
// 2^16-element item split as x = c * 256 + r (r = x bits 0..7, c = bits 8..15,
// c = 2 j + c0):
//
//   GEMM (stages over r and c bits 0..2).  With b_c[r] = g_v(c * 256 + r)
//   in {0, 1} (bit planes -> bytes, straight into shared memory), the B
//   operand (u8) holds, for each group of 8 consecutive c, the 8-point WHT of
//   their bit rows (biased butterflies, every byte in [0, 8]), A = -H_256
//   (s8), and a 9th K block adds a bias against constant all-ones B columns,
//   so that
//     D[u][8 j + e] = W_11 / 2 + 2^10   in [0, 2^11]
//   exactly -- the biased "s = W/2 + 2^(k-1) after k stages" form of
//   sbw_tile_simd.cuh, row u = 0 included.  (SBW_TC_ROWS = 2 builds the
//   pair form: c bit 0 only, D = W_9 / 2 + 2^8.)  tcgen05.mma.kind::i8, M = 128,
//   N = 256, K = 32; 2 M-halves x 9 K blocks; s32 accumulators fill all 512
//   TMEM columns.  B is K-major SWIZZLE_128B; A and B's bias block are
//   K-major without swizzle (layouts validated in tools/micro/tc_probe.cu).
//
//   Integer stages (c bits 3..7).  One TMEM lane (one u) per transform
//   thread: tcgen05.ld .pack::16b returns columns (2j, 2j+1) as the 16-bit
//   lanes of register j, so the 256 values arrive packed in 128 registers.
//   c bits 3..6 are packed biased stages (sum IMAD.IADD, diff IADD3 with the
//   lane bias); c bit 7 is fused with the VIMNMX3 max/min fold (NL) or left
//   to pass B (EMIT, which writes the stage-15 lanes).
//
// Warp roles (one persistent CTA per SM over a contiguous range of items):
// warpgroup 0 = one MMA-issuing warp (tcgen05.mma blocks its thread while the
// tensor core queue is full; the other 3 warps exit), warpgroups 1-2 = 8
// transform warps; setmaxnreg gives them 232 registers and the issuer 32.
// mbarriers: full (MMA(i) done) -> transform warps read D(i) -> tmem_empty ->
// issuer starts MMA(i+1) once bfull says B(i+1) is ready; meanwhile the
// transform warps generate B(i+2) into the buffer MMA(i) released and run
// the integer stages of item i.  In NL mode masks are visited in Gray-code
// order inside every aligned block of 256 that lies in [v_lo, v_hi), so
// consecutive masks differ in one bit: one (prefetched) plane XOR per row.
// SBW_TC_ROWS=1 builds the earliest form (plain bit rows, c0 packed on the
// FMA pipe with two IMADs per pair), kept for A/B measurements.
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "sbw_internal.cuh"
#include "sbw_launch.h"
#include "sbw_tc.cuh"
#include "sbw_tile_simd.cuh"

namespace sbw {
namespace {

#ifndef SBW_TC_ROWS
#define SBW_TC_ROWS 16
#endif
// SBW_TC_ROWS = R: the B operand rows come in groups of R = 2^L consecutive c
// holding the R-point WHT of their bit rows (unsigned, offset R/2 on all but
// the first), so the GEMM also runs c bits 0..L-1; a bias K block and
// .pack::16b loads deliver the biased lanes.  R = 1: plain bit rows, the
// transform warps pack c0 with IMADs (the earlier form, kept for A/B).
constexpr int kRows = SBW_TC_ROWS;
// EMIT store order: 1 = per 16-register network as soon as it is final (5 %
// faster pass A in the L2 ring, 1 % slower in the HBM-bound batched path),
// 0 = all stores after the stages (default).
#ifndef SBW_R16_LATE
#define SBW_R16_LATE 0  // 1: R = 16 stores B(i+2) after the item's stages (measured 2 % slower)
#endif
constexpr bool kLateB = (SBW_TC_ROWS == 16 && SBW_R16_LATE) || SBW_TC_ROWS == 32;  // R = 32 cannot hold both
#ifndef SBW_EMIT_NET
#define SBW_EMIT_NET 0
#endif
static_assert(kRows == 1 || kRows == 2 || kRows == 8 || kRows == 16 || kRows == 32,
              "SBW_TC_ROWS must be 1, 2, 8, 16 or 32");
constexpr int kLogRows = kRows == 32 ? 5 : (kRows == 16 ? 4 : (kRows == 8 ? 3 : (kRows == 2 ? 1 : 0)));
constexpr bool kC0Mma = kRows > 1;
// bias per D entry: 128 R on every row, 128 R more on row u = 0, as columns of
// 127 (plus a remainder) against B columns of kBiasB (2 for R = 16, so both
// bias column sets fit one 32-wide K block)
constexpr int kBiasT = 128 * kRows;
constexpr int kBiasB = kRows >= 16 ? kRows / 8 : 1;
constexpr int kBiasCols = (kBiasT / kBiasB + 126) / 127;
// generation state: plane words per transform thread (R = 16: word ks of 16 rows)
constexpr int kGW = kRows >= 16 ? kRows : 8;
constexpr int kMathWarps = 8;
constexpr int kKA = kC0Mma ? 288 : 256;        // K of A: 256 (r) [+ 32 bias block]
constexpr int kAHalf = 128 * kKA;              // one M = 128 half of A
constexpr int kAOff = 0;                       // A = -H_256 [| bias], 256 x kKA s8
constexpr int kBbOff = kAOff + 2 * kAHalf;     // bias block of B (C0MMA), 256 x 32
constexpr int kBOff = kBbOff + (kC0Mma ? 256 * 32 : 0);  // 2 x (256 x 256) generated B
constexpr int kBBytes = 256 * 256;
constexpr int kTcSmem = kBOff + 2 * kBBytes;   // 212992 (C0MMA) / 196608 bytes
constexpr uint32_t kIdesc = tc::idesc_i8(128, 256, /*A s8*/ true, /*B u8*/ false);
static_assert(kBOff % 1024 == 0, "SW128 B atoms need 1024-byte alignment");

// K position of bit r inside its 32-bit plane word after the byte expansion
// (w >> k) & 0x01010101 (k = 0..7): element r = 32 j + 8 jb + k lands at
// byte 32 j + 4 k + jb.  A's columns carry the same permutation.
__device__ __forceinline__ int r_of_p(int p) { return (p & ~31) | ((p & 3) << 3) | ((p >> 2) & 7); }

// A[u][p]: -H[u][r(p)] for p < 256.  Bias block (against B's all-ones bias
// columns): +128 R on every row and +128 R more on row u = 0.  That makes
// every D entry the biased s = W_(8+L)/2 + 2^(7+L): the polarity 1 - 2b puts
// +128 R on row 0's first row of each group, and the unsigned offset R/2 of
// the other rows costs -(R/2) sum_r H[u][r] = -128 R [u = 0].
__device__ __forceinline__ int a_value(int u, int p) {
  if (p < 256) return (__popc(u & r_of_p(p)) & 1) ? 1 : -1;
  const int k = p - 256;
  const int col = k % kBiasCols, last = kBiasT / kBiasB - 127 * (kBiasCols - 1);
  if (k < kBiasCols) return col < kBiasCols - 1 ? 127 : last;
  if (k < 2 * kBiasCols) return u == 0 ? (col < kBiasCols - 1 ? 127 : last) : 0;
  return 0;
}


__device__ __forceinline__ void xor_plane(uint32_t (&g)[kGW], const uint4 (&p)[kGW / 4]) {
#pragma unroll
  for (int q = 0; q < kGW / 4; ++q) {
    g[4 * q] ^= p[q].x; g[4 * q + 1] ^= p[q].y; g[4 * q + 2] ^= p[q].z; g[4 * q + 3] ^= p[q].w;
  }
}

// Expand the 256 bits of row c into the u8 B operand (K-major core matrices).
[[maybe_unused]] __device__ __forceinline__ void store_row(const uint32_t* g, uint8_t* bbuf, int c) {
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

// C0MMA generation: thread (j, kh) owns K half kh (= SW128 atom column kh)
// of rows 2j and 2j+1: g[0..3] = row 2j's plane words 4kh..4kh+3, g[4..7] =
// row 2j+1's.  Sum row 2j: b0 + b1; diff row 2j+1: b0 - b1 + 1 (u8).
// SW128 layout: atom (kh, g8 = n >> 3) at (kh * 32 + g8) * 1024, row i = n & 7
// at i * 128, logical chunk c at chunk c ^ i.  The two K halves of a row pair
// write chunks 2w + kh first and 2w + 1 - kh second, so the 8 threads of a
// store phase hit 8 different 16-byte bank groups.
[[maybe_unused]] __device__ __forceinline__ void store_rows_sw128(const uint32_t* g, uint8_t* bbuf, int j, int kh) {
  const int i0 = (2 * j) & 7;
  uint8_t* a0 = bbuf + (kh * 32 + (j >> 2)) * 1024 + i0 * 128;  // row 2j (sum)
  uint8_t* a1 = a0 + 128;                                          // row 2j+1 (diff)
  constexpr uint32_t M = 0x01010101u;
  const int s4 = 4 * kh;  // first chunk holds bits 0..3 (kh = 0) or 4..7 (kh = 1)
#pragma unroll
  for (int w = 0; w < 4; ++w) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint32_t sv[4], dv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = (4 * half + q) ^ s4;
        const uint32_t b0 = (g[w] >> k) & M, b1 = (g[4 + w] >> k) & M;
        sv[q] = b0 + b1;
        dv[q] = b0 + M - b1;  // per byte in {0, 1, 2}: no borrow
      }
      const int c = 2 * w + (half ^ kh);  // logical chunk of this store
      *reinterpret_cast<uint4*>(a0 + ((c ^ i0) << 4)) = make_uint4(sv[0], sv[1], sv[2], sv[3]);
      *reinterpret_cast<uint4*>(a1 + ((c ^ (i0 + 1)) << 4)) = make_uint4(dv[0], dv[1], dv[2], dv[3]);
    }
  }
}

// R = 8 generation: thread (j, ks) owns plane word ks (K positions
// 32 ks .. 32 ks + 31 = SW128 atom column ks >> 2, chunks 2 (ks & 3) + 0/1)
// of the 8 rows 8j .. 8j+7 (g[e] = row 8j + e).  Per bit k the 8 byte
// vectors b_e run through a biased 8-point WHT (diff + 2^t at stage t, so
// every output is in [0, 8]); output e goes to row 8j + e.  Threads with
// ks >= 4 store their second chunk first, so a store phase (8 threads, one
// row e, ks = 0..7) covers all 8 chunk positions c ^ e: no bank conflicts.
[[maybe_unused]] __device__ __forceinline__ void store_rows8_sw128(const uint32_t* g, uint8_t* bbuf, int j, int ks) {
  uint8_t* base = bbuf + ((ks >> 2) * 32 + j) * 1024;
  constexpr uint32_t M = 0x01010101u;
  const int s4 = 4 * (ks >> 2);
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    uint32_t o[8][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = (4 * half + q) ^ s4;
      uint32_t b[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) b[e] = (g[e] >> k) & M;
#pragma unroll
      for (int t = 0; t < 3; ++t)
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if ((e & (1 << t)) == 0) {
            const uint32_t x = b[e], y = b[e | (1 << t)];
            b[e] = x + y;
            b[e | (1 << t)] = x - y + (M << t);  // per byte in [0, 2^(t+1)]: no borrow
          }
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e][q] = b[e];
    }
    const int c = 2 * (ks & 3) + (half ^ (ks >> 2));  // logical chunk of this store
#pragma unroll
    for (int e = 0; e < 8; ++e)
      *reinterpret_cast<uint4*>(base + e * 128 + ((c ^ e) << 4)) = make_uint4(o[e][0], o[e][1], o[e][2], o[e][3]);
  }
}

// R = 16 generation: thread (j, ks, kq) owns plane word ks of the 16 rows
// 16 j .. 16 j + 15 (g[e] = row 16 j + e) and the bit positions k = 4 kq ..
// 4 kq + 3 of its bytes, i.e. one 16-byte chunk (2 (ks & 3) + kq of SW128
// atom column ks >> 2) of every row.  Per k the 16 byte vectors run through
// a biased 16-point WHT (every output in [0, 16]).  A store phase (8 threads:
// ks = 0..3 or 4..7, kq = 0, 1) covers the 8 chunk positions of one atom
// row: no bank conflicts.
[[maybe_unused]] __device__ __forceinline__ void store_rows16_sw128(const uint32_t* g, uint8_t* bbuf, int j,
                                                                    int ks, int kq) {
  uint8_t* base = bbuf + ((ks >> 2) * 32 + 2 * j) * 1024;
  constexpr uint32_t M = 0x01010101u;
  uint32_t o[16][4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int k = 4 * kq + q;
    uint32_t b[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) b[e] = (g[e] >> k) & M;
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if ((e & (1 << t)) == 0) {
          const uint32_t x = b[e], y = b[e | (1 << t)];
          b[e] = x + y;
          b[e | (1 << t)] = x - y + (M << t);  // per byte in [0, 2^(t+1)]: no borrow
        }
#pragma unroll
    for (int e = 0; e < 16; ++e) o[e][q] = b[e];
  }
  const int c = 2 * (ks & 3) + kq;  // logical chunk of this thread in every row
#pragma unroll
  for (int e = 0; e < 16; ++e)
    *reinterpret_cast<uint4*>(base + (e >> 3) * 1024 + (e & 7) * 128 + ((c ^ (e & 7)) << 4)) =
        make_uint4(o[e][0], o[e][1], o[e][2], o[e][3]);
}

// Pass-A scratch store (SBW_EMIT_CS=1: streaming st.global.cs, evict-first)
#ifndef SBW_EMIT_CS
#define SBW_EMIT_CS 1  // 24x16: 945 vs 956 ms (plain stores); 20x20 unchanged
#endif
__device__ __forceinline__ void emit_store(uint4* p, uint4 v) {
  if (SBW_EMIT_CS)
    __stcs(p, v);
  else
    *p = v;
}

// R = 32 generation: thread (j, ks, kq) owns plane word ks of the 32 rows
// 32 j .. 32 j + 31 and the bit positions k = 2 kq, 2 kq + 1: 8 bytes (half a
// 16-byte SW128 chunk) of every row.  Biased 32-point WHT, outputs in [0, 32].
[[maybe_unused]] __device__ __forceinline__ void store_rows32_sw128(const uint32_t* g, uint8_t* bbuf, int j,
                                                                    int ks, int kq) {
  uint8_t* base = bbuf + ((ks >> 2) * 32 + 4 * j) * 1024;
  constexpr uint32_t M = 0x01010101u;
  uint32_t o[32][2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int k = 2 * kq + q;
    uint32_t b[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) b[e] = (g[e] >> k) & M;
#pragma unroll
    for (int t = 0; t < 5; ++t)
#pragma unroll
      for (int e = 0; e < 32; ++e)
        if ((e & (1 << t)) == 0) {
          const uint32_t x = b[e], y = b[e | (1 << t)];
          b[e] = x + y;
          b[e | (1 << t)] = x - y + (M << t);  // per byte in [0, 2^(t+1)]: no borrow
        }
#pragma unroll
    for (int e = 0; e < 32; ++e) o[e][q] = b[e];
  }
  const int c = 2 * (ks & 3) + (kq >> 1);  // logical chunk; this thread's 8 bytes at half kq & 1
#pragma unroll
  for (int e = 0; e < 32; ++e)
    *reinterpret_cast<uint2*>(base + (e >> 3) * 1024 + (e & 7) * 128 + ((c ^ (e & 7)) << 4) + 8 * (kq & 1)) =
        make_uint2(o[e][0], o[e][1]);
}

__device__ __forceinline__ void publish(const uint32_t* wmax, uint32_t v, uint32_t v_lo,
                                        int32_t* max_abs, unsigned long long* key) {
  const uint4 a = *reinterpret_cast<const uint4*>(wmax);
  const uint4 b = *reinterpret_cast<const uint4*>(wmax + 4);
  const int m = int(max(max(max(a.x, a.y), max(a.z, a.w)), max(max(b.x, b.y), max(b.z, b.w))));
  max_abs[v - v_lo] = m;
  if (key) atomicMax(key, nl_key(m, v));
}

// MMA chain of one mask (2 M-halves x 8 (+1 bias) K blocks), issued by a
// converged warp.  Descriptors differ only in the start-address field (bits
// 0..13, smem < 256 KiB, no carry): one base plus a compile-time offset each.
__device__ __forceinline__ void issue_mma_warp(uint32_t tmem, const uint8_t* smem, int buf, uint64_t* bar) {
  const uint64_t da0 = tc::sdesc(tc::smem_u32(smem + kAOff), 128, kKA / 16 * 128);
  const uint32_t b0 = tc::smem_u32(smem + kBOff + buf * kBBytes);
  const uint64_t db0 = kC0Mma ? tc::sdesc_sw128(b0, 1024) : tc::sdesc(b0, 128, 2048);
  const uint64_t dbb = tc::sdesc(tc::smem_u32(smem + kBbOff), 128, 256);
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int kb = 0; kb < (kC0Mma ? 9 : 8); ++kb) {
      // SW128: K block kb = atom column kb >> 2 (32 KiB apart), 32 B steps inside
      const uint64_t db = kb == 8 ? dbb
                                  : db0 + uint64_t(kC0Mma ? ((kb >> 2) * 32768 + (kb & 3) * 32) >> 4 : kb * 16);
      tc::mma_i8_elect(tmem + h * 256, da0 + uint64_t((h * kAHalf + kb * 256) >> 4), db, kIdesc,
                       kb > 0 ? 1u : 0u);
    }
  tc::mma_commit_elect(bar);
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

// Warp roles.  tcgen05.mma blocks its issuing thread while the tensor core's
// queue is full (~one MMA per 128 cycles here), so the 16 MMAs of a mask
// would stall a transform warp for ~2K cycles; they get their own warp.
// setmaxnreg moves the registers: the issuer warpgroup keeps 32 per thread,
// the two transform warpgroups get 232 (3 warps per SM sub-partition:
// 32 + 232 + 232 = 496 of the 512 registers per lane of a sub-partition;
// an exact 512 fit hung setmaxnreg.inc on B200).
#ifndef SBW_ISSUER_REGS
#define SBW_ISSUER_REGS 32
#endif
#ifndef SBW_MATH_REGS
#define SBW_MATH_REGS 232
#endif
constexpr int kIssuerRegs = SBW_ISSUER_REGS;
constexpr int kMathRegs = SBW_MATH_REGS;
// (an exact 512 fit -- e.g. 48 + 2 x 232 -- hangs setmaxnreg.inc on B200;
// 40 + 2 x 232 spills the transform warps and runs 6 % slower)
static_assert(kIssuerRegs + 2 * kMathRegs < 512 && kIssuerRegs % 8 == 0 && kMathRegs % 8 == 0,
              "setmaxnreg split of a sub-partition's 512 registers per lane");
constexpr int kAllThreads = 128 + kMathWarps * 32;  // warpgroup 0: issuer (+3 idle warps)

struct TcArgs {
  const uint8_t* consts;  // smem image of A and B's bias block (kBOff bytes), k_tc_consts
  const uint32_t* planes;
  int64_t plane_words;  // 2^n / 32
  // NL (n = 16): masks [v_lo, v_hi), Gray order inside aligned 256-blocks
  uint32_t v_lo, v_hi;
  int32_t* max_abs;
  unsigned long long* key;
  // EMIT (pass A of the multi-pass path, n = 17..24): item t = (component
  // v_first + t % n_comp, 2^16-block bp = t / n_comp); 15 stages per 2^15 block
  uint32_t v_first;
  int64_t n_comp, n_items;
  int n_full;
  uint32_t* emit;
  uint32_t run_lo, run_hi;  // position v_first + j holds mask mask_at(., run_lo, run_hi)
  // SPEC (n = 16 materialised spectrum, mask-major): out[(v - v_lo) * ld + u]
  int32_t* out;
  int64_t ld;
  // kTcSpecSt only: element (v, z) goes to out[(v - v_lo) * ld + z - zoff + goff]
  // and z < zoff is dropped.  zoff = 0, goff = 0: the mask-major rows
  // (ld % 4 == 0).  zoff = 1: the reference's x-major store of a bijective
  // box S from its inverse T = S^-1 (W_S(u, v) = W_T(v, u): item mask = x-major
  // row u, z = v, pitch 2^n - 1 odd), out 16-byte aligned and goff < 4 the
  // caller pointer's offset from it.
  int zoff;
  int64_t goff;
  // EMIT into the L2 ring shared with a concurrent pass B (sbw_internal.cuh)
  RingArgs ring;
  // MODE kTcEmit16 runs the 16th stage (x bit 15) too and writes the
  // wrapped u16 s = W_16 / 2 + 2^15 (h = 0: u bit 15 = 0, h = 1: = 1); a lane
  // that wraps (|W_16| = 2^16, an affine tile) raises *flag, and the host's
  // gated launches redo the batch with the 15-stage form (sbw_passb.cu).
  int* flag;  // kTcEmit16
  // run only if (*gate != 0) == gate_on (gate may be null)
  const int* gate;
  int gate_on;
};

constexpr int kTcNL = 0, kTcEmit = 1, kTcSpec = 2, kTcEmit16 = 3;  // kTcEmit16: EMIT + stage 16
// kTcSpecSt: n = 16 spectrum with the staged epilogue.  The exact W rows go
// to a shared-memory ring of 8 KiB slots (8 u_c rows x 256 u_r: 8 KiB of one
// contiguous mask-major row) and the three otherwise idle warps of the issuer
// warpgroup copy each slot to global memory (STG.128, streaming).  The
// transform warps no longer stall on the store queue before they can start
// the next item, so the ~2 us of generation + stages per item overlaps the
// ~6 us the SM needs to write 256 KiB (tools/micro/stg_width: 6.4 TB/s is
// reachable with either store width).  The ring needs the smem of the second
// B buffer: this mode generates B(i+1) into the single buffer after MMA(i).
constexpr int kTcSpecSt = 4;
// kTcSpecStX: the same staged epilogue writing shifted rows (TcArgs::zoff = 1),
// the x-major store of a bijective box from its inverse
constexpr int kTcSpecStX = 5;
__host__ __device__ constexpr bool is_emit(int mode) { return mode == kTcEmit || mode == kTcEmit16; }
__host__ __device__ constexpr bool is_staged(int mode) { return mode == kTcSpecSt || mode == kTcSpecStX; }
__host__ __device__ constexpr bool is_spec(int mode) { return mode == kTcSpec || is_staged(mode); }
constexpr int kStSlotBytes = 8192;  // 8 u_c rows x 256 u_r of int32
#ifndef SBW_ST_SLOTS
#define SBW_ST_SLOTS 10
#endif
constexpr int kStSlots = SBW_ST_SLOTS;
constexpr int kStOff = kBOff + kBBytes;  // after the single B buffer
constexpr int kTcSmemSt = kStOff + kStSlots * kStSlotBytes;
static_assert(kTcSmemSt <= 230 * 1024, "staged spectrum ring exceeds shared memory");
#ifndef SBW_ST_INFLIGHT
#define SBW_ST_INFLIGHT 3
#endif
constexpr int kStInflight = SBW_ST_INFLIGHT;  // bulk copies in flight before a slot is recycled
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(tc::smem_u32(ssrc)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

// NL items for an n = NB <= 16 box: one 2^16 tile holds C = 2^(16 - NB)
// components (slots); item t covers masks (base << log2 C) | slot, with base
// running over [v_lo >> log2 C, ceil(v_hi / C)) in Gray order inside aligned
// blocks of 256.  NB = 16: one slot, item = mask.
template <int MODE, int NB>
__device__ __forceinline__ int64_t items_total(const TcArgs& a) {
  constexpr int LC = 16 - NB;
  if constexpr (is_emit(MODE)) return a.n_items;
  return ((int64_t(a.v_hi) - 1) >> LC) + 1 - (int64_t(a.v_lo) >> LC);
}
// item t of the launch -> (mask v of slot 0, 2^16-block index bp)
template <int MODE, int NB>
__device__ __forceinline__ void item_at(const TcArgs& a, int64_t t, uint32_t& v, uint32_t& bp) {
  if constexpr (is_emit(MODE)) {
    if (a.ring.on) {  // CTA (r, bp): ring position r K L + t (slot r L + t mod L of batch t / L)
      bp = blockIdx.x & ((1u << a.ring.log_t) - 1u);
      v = ring_mask(a.ring, a.v_first, int64_t(blockIdx.x >> a.ring.log_t) * a.ring.batches * a.ring.L + t);
      return;
    }
    bp = uint32_t(t / a.n_comp);
    v = mask_at(int64_t(a.v_first) + (t - int64_t(bp) * a.n_comp), a.run_lo, a.run_hi);
  } else {
    constexpr int LC = 16 - NB;
    const uint32_t b0 = a.v_lo >> LC, b1 = uint32_t(((int64_t(a.v_hi) - 1) >> LC) + 1);
    bp = 0;
    v = mask_at(b0 + t, b0, b1) << LC;
  }
}

// Generation state of one transform thread: row c's 8 plane words for mask
// vcur in block bpcur.
struct GenState16 {
  uint32_t g[kGW];
  uint32_t vcur, bpcur;
};

// Shared-memory image of the constant operands: A = -H_256 with the K
// permutation of the byte expansion (+ the bias block columns) and, for
// C0MMA, B's bias block (columns 0 .. 2 kBiasCols - 1 = 1 on every row).
__global__ void k_tc_consts(uint8_t* img) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 256 * (kKA / 16); e += gridDim.x * blockDim.x) {
    const int uu = e / (kKA / 16), pc = e % (kKA / 16);
    uint32_t wv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t x = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) x |= uint32_t(uint8_t(a_value(uu, pc * 16 + q * 4 + b))) << (8 * b);
      wv[q] = x;
    }
    *reinterpret_cast<uint4*>(img + kAOff + ((uu >> 3) * (kKA / 16) + pc) * 128 + (uu & 7) * 16) =
        make_uint4(wv[0], wv[1], wv[2], wv[3]);
  }
  if constexpr (kC0Mma) {
    static_assert(2 * kBiasCols <= 32, "bias block is one K block");
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 256 * 32; e += gridDim.x * blockDim.x) {
      const int n = e >> 5, k = e & 31;
      img[kBbOff + ((n >> 3) * 2 + (k >> 4)) * 128 + (n & 7) * 16 + (k & 15)] = k < 2 * kBiasCols ? kBiasB : 0;
    }
  }
}

// publish slot `slot` of NL item t (masks outside [v_lo, v_hi) are skipped)
template <int NB>
__device__ __forceinline__ void publish_item(const TcArgs& a, const uint32_t* wmax, int64_t t, int slot) {
  uint32_t v, bp;
  item_at<kTcNL, NB>(a, t, v, bp);
  v |= uint32_t(slot);
  if (v >= a.v_lo && v < a.v_hi) publish(wmax, v, a.v_lo, a.max_abs, a.key);
}

template <int MODE, int NB = 16>
__global__ void __launch_bounds__(kAllThreads, 1) k_tc_hybrid(TcArgs a) {
  constexpr bool EMIT = is_emit(MODE);
  static_assert(NB == 16 || ((MODE == kTcNL || is_spec(MODE)) && NB >= 8 + kLogRows && kRows >= 8),
                "n < 16: NL / SPEC with 8/16-row groups");
  constexpr int kSlots = 1 << (16 - NB);  // components per 2^16 tile
  static_assert(!is_spec(MODE) || kC0Mma, "exact SPEC output needs the bias-block GEMM");
  static_assert(!is_staged(MODE) || (NB >= 12 && kRows == 16), "staged spectrum: n = 12..16, 16-row generation");
  constexpr bool kStaged = is_staged(MODE);
  constexpr bool kShift = MODE == kTcSpecStX;
  constexpr int kNBuf = kStaged ? 1 : 2;  // B operand buffers (generation runs kNBuf items ahead)
  extern __shared__ __align__(1024) uint8_t smem[];
  // full: MMA(i) done.  tmem_empty: all transform threads read D(i).
  // bfull[b]: all transform threads generated the B operand in buffer b.
  __shared__ uint64_t bar_full, bar_tmem_empty, bar_bfull[2], bar_done;
  __shared__ uint64_t bar_st_full[kStaged ? kStSlots : 1], bar_st_empty[kStaged ? kStSlots : 1];
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(16) uint32_t s_wmax[4][kSlots][kMathWarps];  // per-warp max|W| [item & 3][slot]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (EMIT && a.gate && ((*a.gate != 0) != (a.gate_on != 0))) return;  // CTA-uniform, before any setup
  const int64_t total = items_total<MODE, NB>(a);
  const bool ring = EMIT && a.ring.on;
  const int64_t t_lo = ring ? 0 : total * blockIdx.x / gridDim.x;
  const int n_my = ring ? int(a.ring.batches * a.ring.L) : int(total * (blockIdx.x + 1) / gridDim.x - t_lo);

  // constant operands (A and B's bias block): one coalesced copy of the
  // image k_tc_consts built once per device
  for (int e = tid; e < kBOff / 16; e += kAllThreads)
    reinterpret_cast<uint4*>(smem)[e] = __ldg(reinterpret_cast<const uint4*>(a.consts) + e);
  if (warp == 0) tc::tmem_alloc(&tmem_slot, 512);
  if (tid == 0) {
    tc::mbar_init(&bar_full, 1);
    tc::mbar_init(&bar_tmem_empty, kMathWarps * 32);
    tc::mbar_init(&bar_bfull[0], kMathWarps * 32);
    tc::mbar_init(&bar_bfull[1], kMathWarps * 32);
    tc::mbar_init(&bar_done, kMathWarps * 32);
    if constexpr (kStaged)
      for (int q = 0; q < kStSlots; ++q) {
        tc::mbar_init(&bar_st_full[q], kMathWarps * 32);
        tc::mbar_init(&bar_st_empty[q], 1);
      }
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
        tc::mbar_wait(&bar_bfull[i % kNBuf], uint32_t((i / kNBuf) & 1));
        if (i > 0) tc::mbar_wait(&bar_tmem_empty, uint32_t((i - 1) & 1));
        tc::fence_after();
        int ibuf = i % kNBuf;
        if constexpr (kNBuf == 1) asm volatile("mov.b32 %0, %0;" : "+r"(ibuf));  // keep descriptors in the loop
        issue_mma_warp(tmem, smem, ibuf, &bar_full);
        if constexpr (!EMIT) {
          // bfull for item i (i >= 2) is produced after each thread stored
          // its maxima of item i - 2
          if (i >= 2 && lane < kSlots) publish_item<NB>(a, s_wmax[(i - 2) & 3][lane], t_lo + i - 2, lane);
        }
      }
      // every transform thread has read D(last) and stored its last max
      tc::mbar_wait(&bar_done, 0u);
      tc::fence_after();
      if constexpr (!EMIT) {
        if (lane < kSlots)
          for (int i = n_my - 2 < 0 ? 0 : n_my - 2; i < n_my; ++i)
            publish_item<NB>(a, s_wmax[i & 3][lane], t_lo + i, lane);
      }
      __syncwarp();
      tc::tmem_dealloc(tmem, 512);
    } else if (kStaged && warp == 1 && lane == 0) {
      // slot writer: ring position p = 32 i + j holds 8 KiB of item i's row
      // (u_c rows 8 q .. 8 q + 7, q = j / 2 (+ 16 for odd j)), written by one
      // bulk copy (TMA engine, async); a slot is released once the copy
      // kStInflight positions later has been issued and its read completed
      constexpr int P = 1 << (NB - 9);  // registers (2 P u_c rows) per component
      int q = 0, qr = 0;
      uint32_t ph = 0;
      int64_t issued = 0;
#pragma unroll 1
      for (int il = 0; il < n_my; ++il) {
        uint32_t vi, bp;
        item_at<MODE, NB>(a, t_lo + il, vi, bp);
#pragma unroll 1
        for (int j = 0; j < 32; ++j) {
          // position j: component slot sl, u_c rows half * P + 8 q8 .. + 7
          const int sl = j / (P / 4), r = j % (P / 4);
          const uint32_t v = vi | uint32_t(sl);
          tc::mbar_wait(&bar_st_full[q], ph);
          if (v >= a.v_lo && v < a.v_hi) {
            // the aligned chunks [A, B) of the slot's z0 .. z0 + 2047 go by bulk
            // copy (the slot holds word g at g - A); the < 4 words at either
            // end (shared with the neighbouring slot / row) were stored per lane
            const int z0 = ((r & 1) * P + 8 * (r >> 1)) * 256;
            const int64_t g0 = int64_t(v - a.v_lo) * a.ld + z0 - (kShift ? 1 : 0) + (kShift ? a.goff : 0);
            const int sh = kShift ? int(g0 & 3) : 0;
            const int h = kShift ? ((z0 == 0 && sh == 0) ? 4 : ((4 - sh) & 3)) : 0;
            const int64_t A = g0 + h, B = (g0 + 2048) & ~int64_t(3);
            const int off = kShift ? (sh ? sh - 4 : 0) : 0;  // slot word of z0 + p is p + off
            bulk_store(a.out + A, smem + kStOff + q * kStSlotBytes + 4 * (h + off), uint32_t(4 * (B - A)));
          } else
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");  // empty group: FIFO release order
          if (++issued > kStInflight) {
            bulk_wait_read<kStInflight>();
            mbar_arrive(&bar_st_empty[qr]);
            if (++qr == kStSlots) qr = 0;
          }
          if (++q == kStSlots) {
            q = 0;
            ph ^= 1u;
          }
        }
      }
      bulk_wait_read<0>();
      for (int64_t k = 0; k < (issued < kStInflight ? issued : kStInflight); ++k) {
        mbar_arrive(&bar_st_empty[qr]);
        if (++qr == kStSlots) qr = 0;
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // writes complete before exit
    }
  } else {
    // ---------------- transform warps ----------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kMathRegs));
    const int mt = tid - 128, mw = mt >> 5;  // transform thread / warp index
    const int c = mt;                        // generation row (plain B rows)
    const int gj = kRows == 32 ? mt >> 5 : (kRows == 16 ? mt >> 4 : (kRows == 8 ? mt >> 3 : mt >> 1));  // C0MMA: row group
    // C0MMA: plane word (R = 8, 16) / K half (R = 2); R = 16 also splits the
    // bit positions of the bytes: gkq = k half
    const int gkh = kRows == 32 ? (mt >> 2) & 7 : (kRows == 16 ? (mt >> 1) & 7 : (kRows == 8 ? mt & 7 : mt & 1));
    const int gkq = kRows == 32 ? mt & 3 : mt & 1;
    const uint32_t* __restrict__ planes = a.planes;
    const int64_t pw = EMIT ? a.plane_words : (int64_t(1) << NB) >> 5;
    // NB < 16: this thread's 8 rows belong to slot gslot; its rows within the
    // component start at row group gj mod 2^(NB - 11)
    constexpr int kGrpLog = NB - 8 - kLogRows;  // log2 row groups per component (NB < 16)
    const uint32_t gslot = NB < 16 ? uint32_t(gj >> kGrpLog) : 0u;
    const int gjc = NB < 16 ? (gj & ((1 << kGrpLog) - 1)) : gj;
    GenState16 gs;
#pragma unroll
    for (int k = 0; k < kGW; ++k) gs.g[k] = 0;
    gs.vcur = 0;
    gs.bpcur = 0;
    // plane words of this thread's generation state in block bp: row c's 8
    // words at bp * 2048 + 8 c, or (C0MMA) 4 words of row 2j and 4 of row
    // 2j+1 at bp * 2048 + 16 j + 4 kh (+ 8)
    auto row_off = [&](uint32_t bp) {
      return int64_t(bp) * 2048 +
             (kRows >= 8 ? 8 * kRows * gjc + gkh : (kRows == 2 ? 16 * gj + 4 * gkh : c * 8));
    };
    auto load_pl = [&](int i, uint32_t bp, uint4 (&x)[kGW / 4]) {
      const uint32_t* p = planes + int64_t(i) * pw + row_off(bp);
      if constexpr (kRows >= 8) {  // word gkh of rows R j + e: stride 8 words
#pragma unroll
        for (int q = 0; q < kGW / 4; ++q)
          x[q] = make_uint4(__ldg(p + 32 * q), __ldg(p + 32 * q + 8), __ldg(p + 32 * q + 16), __ldg(p + 32 * q + 24));
      } else {
        x[0] = __ldg(reinterpret_cast<const uint4*>(p));
        x[1] = __ldg(reinterpret_cast<const uint4*>(p) + (kC0Mma ? 2 : 1));
      }
    };
    auto xor_all = [&](uint32_t d, uint32_t bp) {
      while (d) {
        const int i = __ffs(d) - 1;
        d &= d - 1;
        uint4 x[kGW / 4];
        load_pl(i, bp, x);
        xor_plane(gs.g, x);
      }
    };
    // full recompute (first items): the planes of all set bits of d, 8 at a
    // time with every load in flight, instead of one serialized load per bit
    auto xor_full = [&](uint32_t d, uint32_t bp) {
      constexpr int kXB = kGW >= 32 ? 2 : 8;  // planes per batch (R = 32: 32 words each)
#pragma unroll 1
      for (int i0 = 0; i0 < 32 && (d >> i0); i0 += kXB) {
        uint4 x[kXB][kGW / 4];
#pragma unroll
        for (int q = 0; q < kXB; ++q) {
#pragma unroll
          for (int h = 0; h < kGW / 4; ++h) x[q][h] = make_uint4(0, 0, 0, 0);
          if ((d >> (i0 + q)) & 1u) load_pl(i0 + q, bp, x[q]);
        }
#pragma unroll
        for (int q = 0; q < kXB; ++q) xor_plane(gs.g, x[q]);
      }
    };
    auto store_b = [&](int buf) {
      if constexpr (kRows == 32)
        store_rows32_sw128(gs.g, smem + kBOff + buf * kBBytes, gj, gkh, gkq);
      else if constexpr (kRows == 16)
        store_rows16_sw128(gs.g, smem + kBOff + buf * kBBytes, gj, gkh, gkq);
      else if constexpr (kRows == 8)
        store_rows8_sw128(gs.g, smem + kBOff + buf * kBBytes, gj, gkh);
      else if constexpr (kRows == 2)
        store_rows_sw128(gs.g, smem + kBOff + buf * kBBytes, gj, gkh);
      else
        store_row(gs.g, smem + kBOff + buf * kBBytes, c);
    };
    for (int k = 0; k < kNBuf && k < n_my; ++k) {
      uint32_t vn, bpn;
      item_at<MODE, NB>(a, t_lo + k, vn, bpn);
      vn |= gslot;
      if (EMIT && bpn != gs.bpcur) {
#pragma unroll
        for (int q = 0; q < kGW; ++q) gs.g[q] = 0;
        gs.vcur = 0;
        gs.bpcur = bpn;
      }
      xor_full(gs.vcur ^ vn, bpn);
      gs.vcur = vn;
      store_b(k);
      tc::fence_proxy_async();
      mbar_arrive(&bar_bfull[k]);
    }
    // this thread's TMEM lane: u = 128 * (mw >> 2) + 32 * (mw & 3) + lane
    // (warp w may only touch lanes 32 * (w % 4) .. +31; here w % 4 == mw % 4)
    const int u = 128 * (mw >> 2) + 32 * (mw & 3) + lane;
    const uint32_t tbase = tmem + (uint32_t((mw & 3) * 32) << 16) + uint32_t(mw >> 2) * 256;
    // EMIT: where this thread's words of item i go.  Batched: component slot
    // = batch position.  Ring: slot r L + l of batch k's ring slot, after
    // waiting (first item of a batch) until pass B has loaded batch k - R.
    auto emit_dst = [&](int i) -> uint32_t* {
      uint32_t vi, bpi;
      item_at<MODE, NB>(a, t_lo + i, vi, bpi);
      int64_t slot_comp = (t_lo + i) - int64_t(bpi) * a.n_comp;
      if (ring) {
        const int64_t rk = i / a.ring.L;
        const int rl = int(i - rk * a.ring.L);
        slot_comp = (rk % a.ring.R) * a.ring.bc + int64_t(blockIdx.x >> a.ring.log_t) * a.ring.L + rl;
        if (rl == 0 && rk >= a.ring.R && !a.ring.nowait) {
          if (lane == 0) ring_wait_geq(a.ring.freed + (rk - a.ring.R), a.ring.nb, a.ring.err, a.ring.wait_ns);
          __syncwarp();
        }
      }
      return a.emit + (slot_comp << (a.n_full - 1)) + (int64_t(2 * bpi) << 14) + 4 * u;
    };
    // Ring: this warp's part of batch k is stored after its last item of k.
    auto emit_done = [&](int i) {
      if (ring && (i + 1) % a.ring.L == 0) {
        __syncwarp();
        if (lane == 0) ring_signal(a.ring.ready + i / a.ring.L);
      }
    };
    int st_q = 0;  // kTcSpecSt: next ring slot, its phase, and whether the ring wrapped
    uint32_t st_ph = 0;
    bool st_round = false;
    (void)st_q; (void)st_ph; (void)st_round;
    for (int i = 0; i < n_my; ++i) {
      // prefetch the first plane of the item two steps ahead
      const bool gen = i + kNBuf < n_my;
      uint32_t vn = 0, bpn = 0, d = 0;
      bool reset = false;
      uint4 pa[kGW / 4];
#pragma unroll
      for (int h = 0; h < kGW / 4; ++h) pa[h] = make_uint4(0, 0, 0, 0);
      if (gen) {
        item_at<MODE, NB>(a, t_lo + i + kNBuf, vn, bpn);
        vn |= gslot;
        reset = EMIT && bpn != gs.bpcur;
        d = reset ? vn : (gs.vcur ^ vn);
        if (d) {
          load_pl(__ffs(d) - 1, bpn, pa);
          d &= d - 1;
        }
      }
      tc::mbar_wait(&bar_full, uint32_t(i & 1));
      tc::fence_after();
      uint32_t R[128];
      auto gen_update = [&]() {
        if (gen) {
          if (reset) {
#pragma unroll
            for (int q = 0; q < kGW; ++q) gs.g[q] = 0;
            gs.bpcur = bpn;
          }
          xor_plane(gs.g, pa);
          if (d) xor_all(d, bpn);  // rare: more than one changed bit
          gs.vcur = vn;
        }
      };
      auto gen_store = [&]() {
        if (gen) {
          store_b(i % kNBuf);  // buffer i % kNBuf was released by MMA(i)
          tc::fence_proxy_async();
          mbar_arrive(&bar_bfull[i % kNBuf]);
        }
      };
      if constexpr (kC0Mma) {
        // TMEM -> registers already packed: R[j] = lanes (columns 2j, 2j+1),
        // biased s = W_(8+L) / 2 + 2^(7+L) straight from the GEMM
        uint32_t(&R0)[64] = *reinterpret_cast<uint32_t(*)[64]>(&R[0]);
        uint32_t(&R1)[64] = *reinterpret_cast<uint32_t(*)[64]>(&R[64]);
        if constexpr (kLateB) gen_update();  // before R is live (register pressure)
        tc::tmem_ld_x64_p16(tbase, R0);
        tc::tmem_ld_x64_p16(tbase + 128, R1);
        tc::wait_ld_tied(R0);
        tc::wait_ld_tied(R1);
        tc::fence_before();
        mbar_arrive(&bar_tmem_empty);
        if constexpr (!kLateB) gen_update();
        // R = 16: the 16-row generation needs 64 output registers, so B(i+2)
        // is stored after this item's stages (R dead); MMA(i+2) still only
        // waits for item i+1's TMEM read
        if constexpr (!kLateB) gen_store();
      } else {
        // TMEM -> registers: two pairs of 64-column loads, two waits; TMEM is
        // released before any of the stages run.  R[j] holds c = 2j, 2j+1.
        {
          uint32_t t0[64], t1[64];
          tc::tmem_ld_x64(tbase, t0);
          tc::tmem_ld_x64(tbase + 64, t1);
          tc::wait_ld_tied(t0);
          tc::wait_ld_tied(t1);
          // c bit 0 stage + packing: biased lanes (a + b + 256, a - b + 256)
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            R[j] = t0[2 * j] * 0x10001u + t0[2 * j + 1] * 0xFFFF0001u + 0x01000100u;
            R[32 + j] = t1[2 * j] * 0x10001u + t1[2 * j + 1] * 0xFFFF0001u + 0x01000100u;
          }
        }
        uint32_t t2[64], t3[64];
        tc::tmem_ld_x64(tbase + 128, t2);
        tc::tmem_ld_x64(tbase + 192, t3);
        tc::wait_ld_tied(t2);
        tc::wait_ld_tied(t3);
        tc::fence_before();
        mbar_arrive(&bar_tmem_empty);
        // The second packing (IMAD, FMA pipe) shares its basic block with the
        // byte expansion of item i+2 (LOP3/SHF, ALU pipe), so the two
        // half-rate streams interleave.
        gen_update();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          R[64 + j] = t2[2 * j] * 0x10001u + t2[2 * j + 1] * 0xFFFF0001u + 0x01000100u;
          R[96 + j] = t3[2 * j] * 0x10001u + t3[2 * j + 1] * 0xFFFF0001u + 0x01000100u;
        }
        gen_store();
      }
      if constexpr (EMIT && kRows == 8 && SBW_EMIT_NET) {
        // 15 stages per 2^15 block (c bit 7 = the block's parity, register
        // bit 6, is left to pass B); lanes are s = W_15 / 2 + 2^14.  The
        // remaining ALU stages (register bits 2..5) run one 16-register
        // network (fixed bits 0, 1, 6) at a time and each network is stored
        // as soon as it is final, so the 128 KiB of stores per item spread
        // over the stage arithmetic instead of queueing behind it.  Block word
        // layout (pass B only pairs equal positions across blocks):
        //   network (h, b = bits 0..1), group g = bits 4..5 ->
        //   words (4 b + g) * 1024 + 4 u + (0..3) <- R[64 h + b + 4 (4 g + 0..3)]
        uint32_t* dst = emit_dst(i);
#pragma unroll
        for (int net = 0; net < 8; ++net) {
          const int base = (net >> 2) * 64 + (net & 3);  // h = net >> 2, b = net & 3
#pragma unroll
          for (int sb = 2; sb < 6; ++sb)
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if ((j & (1 << (sb - 2))) == 0) {
                const int k0 = base + 4 * j, k1 = base + 4 * (j | (1 << (sb - 2)));
                const uint32_t x = R[k0], y = R[k1];
                R[k0] = x + y;
                R[k1] = x - y + (0x02000200u << sb);
              }
#pragma unroll
          for (int g = 0; g < 4; ++g)
            *reinterpret_cast<uint4*>(dst + ((net >> 2) << 14) + (4 * (net & 3) + g) * 1024) =
                make_uint4(R[base + 16 * g], R[base + 16 * g + 4], R[base + 16 * g + 8], R[base + 16 * g + 12]);
        }
        emit_done(i);
      } else {
        // c bits L..6 (register bits L-1..5, stages 8+L..14); register bit b is
        // c bit b+1, stage 9+b, diff bias 2^(9+b) per lane
#pragma unroll
        for (int sb = (kLogRows > 0 ? kLogRows - 1 : 0); sb < NB - 10; ++sb)
#pragma unroll
          for (int k = 0; k < 128; ++k)
            if ((k & (1 << sb)) == 0) {
              const uint32_t x = R[k], y = R[k | (1 << sb)];
              R[k] = x + y;
              R[k | (1 << sb)] = x - y + (0x02000200u << sb);
            }
        if constexpr (EMIT) {
          // natural block word layout (default, and SBW_TC_ROWS < 8 builds):
          //   word (j >> 2) * 1024 + 4 u + (j & 3)  <-  R[64 h + j]
          static_assert(!EMIT || NB == 16, "EMIT covers one 2^16 tile");
          if (!kC0Mma && u == 0) {
            R[0] += 0x4000u;
            R[64] += 0x4000u;
          }
          uint32_t* dst = emit_dst(i);
          if constexpr (MODE == kTcEmit16) {
            // stage 16 (register bit 6): S = x + y -> h = 0, D = x - y + 2^15 -> h = 1,
            // lanes = W_16 / 2 + 2^15 mod 2^16; a lane at 0 is W_16 = +-2^16
            uint32_t mn = 0xFFFFFFFFu;
#pragma unroll
            for (int k = 0; k < 64; ++k) {
              const uint32_t x = R[k], y = R[k + 64];
              R[k] = x + y;
              R[k + 64] = x - y + 0x80008000u;
              mn = __vimin3_u16x2(mn, R[k], R[k + 64]);
            }
            if (__any_sync(0xFFFFFFFFu, (mn & 0xFFFFu) == 0u || (mn >> 16) == 0u) && lane == 0) atomicOr(a.flag, 1);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int q = 0; q < 16; ++q)
              emit_store(reinterpret_cast<uint4*>(dst + (h << 14) + q * 1024),
                         make_uint4(R[64 * h + 4 * q], R[64 * h + 4 * q + 1], R[64 * h + 4 * q + 2],
                                    R[64 * h + 4 * q + 3]));
          emit_done(i);
          if constexpr (kLateB) gen_store();
          continue;
        }
        // top stage (c bit NB-9 = register bit NB-10) fused with the max/min
        // fold, per slot (register bits NB-9..6; carry argument of
        // tile_last_pass for NB = 16).  NB = 11 has no ALU stage left: the
        // fold runs on the GEMM output directly.  The row u = 0 offset of the
        // R = 1 form reaches only S of register 0.
        const uint32_t corr0 = (!kC0Mma && u == 0) ? 0x8000u : 0u;
        constexpr int kTop = NB - 10;         // register bit of the top stage (NB >= 12)
        constexpr int kPerSlot = 1 << (NB - 9);
#pragma unroll
        for (int sl = 0; sl < kSlots; ++sl) {
          uint32_t mx = 0u, mn = 0xFFFFFFFFu;
          if constexpr (NB >= 9 + kLogRows) {  // an ALU top stage is left
#pragma unroll
            for (int kk = 0; kk < kPerSlot / 2; ++kk) {
              const int k = sl * kPerSlot + (kk & ((1 << kTop) - 1)) + ((kk >> kTop) << (kTop + 1));
              const uint32_t x = R[k], y = R[k + (1 << kTop)];
              const uint32_t S = x + y + (k == 0 ? corr0 : 0u);
              const uint32_t D = x - y + ((1u << (NB - 1)) * 0x00010001u);
              mx = __vimax3_u16x2(mx, S, D);
              mn = __vimin3_u16x2(mn, S, D);
            }
          } else {
#pragma unroll
            for (int k = 0; k < kPerSlot; k += 2) {
              mx = __vimax3_u16x2(mx, R[sl * kPerSlot + k], R[sl * kPerSlot + k + 1]);
              mn = __vimin3_u16x2(mn, R[sl * kPerSlot + k], R[sl * kPerSlot + k + 1]);
            }
          }
          const uint32_t m = __reduce_max_sync(0xFFFFFFFFu, uint32_t(lanes_maxabs<NB>(mx, mn)));
          if (lane == 0) s_wmax[i & 3][sl][mw] = m;
        }
        if constexpr (MODE == kTcSpec && NB < 16) {
          // n < 16: per slot (component v = vi | slot) the exact W of every
          // lane, W = 2 s - 2^NB for the biased s; no lane can wrap (|W| <=
          // 2^NB <= 2^15).  u = u_c * 256 + u_r, u_c from the register index
          // and lane inside the slot (natural order); 32 consecutive u_r per
          // warp store.
          uint32_t vi, bpi;
          item_at<MODE, NB>(a, t_lo + i, vi, bpi);
          constexpr int kPerSlot = 1 << (NB - 9);  // registers per slot
#pragma unroll
          for (int sl = 0; sl < kSlots; ++sl) {
            const uint32_t v = vi | uint32_t(sl);
            if (v < a.v_lo || v >= a.v_hi) continue;
            int32_t* row = a.out + int64_t(v - a.v_lo) * a.ld + u;
            if constexpr (NB >= 9 + kLogRows) {  // the top stage pairs k, k + kPerSlot / 2
#pragma unroll
              for (int kk = 0; kk < kPerSlot / 2; ++kk) {
                const uint32_t x = R[sl * kPerSlot + kk], y = R[sl * kPerSlot + kk + kPerSlot / 2];
                const int x0 = int(x & 0xFFFFu), x1 = int(x >> 16), y0 = int(y & 0xFFFFu), y1 = int(y >> 16);
                __stcs(row + (2 * kk) * 256, 2 * (x0 + y0) - (1 << NB));
                __stcs(row + (2 * kk + 1) * 256, 2 * (x1 + y1) - (1 << NB));
                __stcs(row + (2 * kk + kPerSlot) * 256, 2 * (x0 - y0));
                __stcs(row + (2 * kk + 1 + kPerSlot) * 256, 2 * (x1 - y1));
              }
            } else {  // the GEMM output is final
#pragma unroll
              for (int kk = 0; kk < kPerSlot; ++kk) {
                const uint32_t x = R[sl * kPerSlot + kk];
                __stcs(row + (2 * kk) * 256, 2 * int(x & 0xFFFFu) - (1 << NB));
                __stcs(row + (2 * kk + 1) * 256, 2 * int(x >> 16) - (1 << NB));
              }
            }
          }
        }
        if constexpr (kStaged) {
          // exact W per lane into the slot ring.  Per component (slot sl,
          // P = 2^(NB-9) registers, u_c = 2 k, 2 k + 1 for register k of the
          // slot), steps of 4 register pairs (k, k + P/2) give 8 u_c rows of
          // the top stage's sum half and 8 of its difference half: 32 ring
          // positions per item for every NB; row-major 256 u_r per u_c row
          // (each warp store is 128 contiguous bytes: no bank conflicts)
          constexpr int P = 1 << (NB - 9);
          uint32_t st_vi = 0, st_bp;
          if constexpr (kShift) item_at<MODE, NB>(a, t_lo + i, st_vi, st_bp);
#pragma unroll
          for (int qq = 0; qq < 16; ++qq) {
            const int sl = qq / (P / 8), q8 = qq % (P / 8);
            uint32_t lo[8], hi[8];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t x = R[sl * P + 4 * q8 + kk], y = R[sl * P + 4 * q8 + kk + P / 2];
              const int x0 = int(x & 0xFFFFu), x1 = int(x >> 16), y0 = int(y & 0xFFFFu), y1 = int(y >> 16);
              if constexpr (NB >= 9 + kLogRows) {  // the top stage (register k with k + P/2)
                lo[2 * kk] = uint32_t(2 * (x0 + y0) - (1 << NB));
                lo[2 * kk + 1] = uint32_t(2 * (x1 + y1) - (1 << NB));
                hi[2 * kk] = uint32_t(2 * (x0 - y0));
                hi[2 * kk + 1] = uint32_t(2 * (x1 - y1));
              } else {  // n = 12: the GEMM output is final (u_c 2k, 2k+1 of register k)
                lo[2 * kk] = uint32_t(2 * x0 - (1 << NB));
                lo[2 * kk + 1] = uint32_t(2 * x1 - (1 << NB));
                hi[2 * kk] = uint32_t(2 * y0 - (1 << NB));
                hi[2 * kk + 1] = uint32_t(2 * y1 - (1 << NB));
              }
            }
#pragma unroll
            for (int half = 0; half < 2; ++half) {
              if (st_round) tc::mbar_wait(&bar_st_empty[st_q], st_ph ^ 1u);
              int off = 0;  // shifted rows: slot word of element p is p + off (off in -3..0)
              if constexpr (kShift) {  // shifted rows: this position's word shift and its end words
                const uint32_t v = st_vi | uint32_t(sl);
                const int z0 = (half * P + 8 * q8) * 256;
                const int64_t g0 = int64_t(v - a.v_lo) * a.ld + z0 - 1 + a.goff;
                const int sh = int(g0 & 3);
                off = sh ? sh - 4 : 0;
                if (v >= a.v_lo && v < a.v_hi) {
                  const int h = (z0 == 0 && sh == 0) ? 4 : ((4 - sh) & 3);
                  if (u < h && !(z0 == 0 && u == 0)) __stcs(a.out + g0 + u, int(half ? hi[0] : lo[0]));
                  if (u >= 256 - sh) __stcs(a.out + g0 + 1792 + u, int(half ? hi[7] : lo[7]));
                }
              }
              uint32_t* slot = reinterpret_cast<uint32_t*>(smem + kStOff + st_q * kStSlotBytes) + u + off;
#pragma unroll
              for (int e = 0; e < 8; ++e)
                if (!kShift || e > 0 || u + off >= 0) slot[e * 256] = half ? hi[e] : lo[e];
              tc::fence_proxy_async();  // generic-proxy writes -> the bulk copy (async proxy)
              mbar_arrive(&bar_st_full[st_q]);
              if (++st_q == kStSlots) {
                st_q = 0;
                st_ph ^= 1u;
                st_round = true;
              }
            }
          }
        }
        if constexpr (MODE == kTcSpec && NB == 16) {
          // exact W of the top stage per lane (the packed S / D above may wrap
          // at |W| = 2^16), stored at u = u_c * 256 + u_r with
          // u_c = lane + 2 k (+ 128 for the diff) -- 32 consecutive u_r per
          // warp store, 128 B coalesced
          uint32_t vi, bpi;
          item_at<MODE, NB>(a, t_lo + i, vi, bpi);
          int32_t* row = a.out + int64_t(vi - a.v_lo) * a.ld + u;
#pragma unroll
          for (int k = 0; k < 64; ++k) {
            const int x0 = int(R[k] & 0xFFFFu), x1 = int(R[k] >> 16);
            const int y0 = int(R[k + 64] & 0xFFFFu), y1 = int(R[k + 64] >> 16);
            __stcs(row + (2 * k) * 256, 2 * (x0 + y0) - 65536);
            __stcs(row + (2 * k + 1) * 256, 2 * (x1 + y1) - 65536);
            __stcs(row + (2 * k + 128) * 256, 2 * (x0 - y0));
            __stcs(row + (2 * k + 129) * 256, 2 * (x1 - y1));
          }
        }
      }
      if constexpr (kLateB) gen_store();
    }
    tc::fence_before();
    mbar_arrive(&bar_done);
  }
}

// int8 MMA peak: one CTA per SM, one thread issues `reps` chains of 8
// accumulating 128x256x32 MMAs on fixed smem operands (A 32 KiB, B 64 KiB).
// mn = 1: B as an MN-major SWIZZLE_128B operand (probe: SBW_PEAK_MN=1), mn = 2: A reused from one 32 KiB block
__global__ void __launch_bounds__(128, 1) k_int8_mma_peak(int reps, int* sink, int mn) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 96 * 1024 / 16; i += 128) reinterpret_cast<uint4*>(smem)[i] = make_uint4(i, 3 * i, 5, 7);
  if (warp == 0) tc::tmem_alloc(&slot, 256);
  if (tid == 0) tc::mbar_init(&bar, 1);
  tc::fence_proxy_async();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {
    const uint64_t da = tc::sdesc(tc::smem_u32(smem), 128, 2048);
    const uint64_t db = tc::sdesc(tc::smem_u32(smem + 32768), 128, 2048);
    if (mn == 1) {
      const uint32_t b0 = tc::smem_u32(smem + 32768);
      const uint64_t dmn = uint64_t((b0 & 0x3FFFFu) >> 4) | (uint64_t(1024 >> 4) << 16) | (uint64_t(2048 >> 4) << 32) |
                           (uint64_t(1) << 46) | (uint64_t(2) << 61);
      for (int r = 0; r < reps; ++r)
#pragma unroll
        for (int kb = 0; kb < 8; ++kb)
          tc::mma_i8_elect(tmem, da + uint64_t(kb * 16), dmn + uint64_t((kb * 8192) >> 4), kIdesc | (1u << 16),
                           (r | kb) ? 1u : 0u);
    } else
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int kb = 0; kb < 8; ++kb)
        tc::mma_i8_elect(tmem, da + uint64_t(kb * 16), db + uint64_t(kb * 16), kIdesc, (r | kb) ? 1u : 0u);
    tc::mma_commit_elect(&bar);
    tc::mbar_wait(&bar, 0u);
    tc::fence_after();
    uint32_t t[32];
    tc::tmem_ld_x32(tmem, t);
    tc::wait_ld();
    if (t[0] == 0x12345678u) sink[0] = 1;  // keeps the chain observable
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

}  // namespace

int run_int8_mma_peak(double* ops_per_s, double* ms_out, cudaStream_t st) {
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  const int smem = 96 * 1024;
  SBW_CUDA_CHECK(cudaFuncSetAttribute(k_int8_mma_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int* sink = nullptr;
  SBW_CUDA_CHECK(cudaMallocAsync(&sink, sizeof(int), st));
  cudaEvent_t e0, e1;
  SBW_CUDA_CHECK(cudaEventCreate(&e0));
  SBW_CUDA_CHECK(cudaEventCreate(&e1));
  const int reps = 2048;
  double best = 0, best_ms = 0;
  for (int rep = 0; rep < 4; ++rep) {
    SBW_CUDA_CHECK(cudaEventRecord(e0, st));
    static const int mn = getenv("SBW_PEAK_MN") ? atoi(getenv("SBW_PEAK_MN")) : 0;
    k_int8_mma_peak<<<dp.sm_count, 128, smem, st>>>(reps, sink, mn);
    SBW_LAUNCH_CHECK("k_int8_mma_peak");
    SBW_CUDA_CHECK(cudaEventRecord(e1, st));
    SBW_CUDA_CHECK(cudaEventSynchronize(e1));
    float ms = 0;
    SBW_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    const double ops = 2.0 * dp.sm_count * double(reps) * 8 * 128 * 256 * 32;
    if (rep > 0 && ops / (ms * 1e-3) > best) {
      best = ops / (ms * 1e-3);
      best_ms = ms;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  SBW_CUDA_CHECK(cudaFreeAsync(sink, st));
  *ops_per_s = best;
  if (ms_out) *ms_out = best_ms;
  return SBW_OK;
}

// SBW_TC=0 selects the all-ALU tile kernel instead (A/B experiments only).
bool tc_path_enabled() {
  static const bool on = [] {
    const char* e = getenv("SBW_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

namespace {
// per-device constant-operand image, built on first use (kept for the
// process lifetime, like the library's other per-device state)
std::mutex g_consts_mu;
uint8_t* g_consts[64] = {};
int tc_consts(int dev, cudaStream_t st, const uint8_t** out) {
  std::lock_guard<std::mutex> lk(g_consts_mu);
  if (!g_consts[dev & 63]) {
    uint8_t* p = nullptr;
    SBW_CUDA_CHECK(cudaMalloc(&p, kBOff));
    k_tc_consts<<<64, 256, 0, st>>>(p);
    SBW_LAUNCH_CHECK("k_tc_consts");
    SBW_CUDA_CHECK(cudaStreamSynchronize(st));  // later launches may use other streams
    g_consts[dev & 63] = p;
  }
  *out = g_consts[dev & 63];
  return SBW_OK;
}

template <int MODE, int NB = 16>
int run_tc_hybrid(const TcArgs& a, int64_t items, cudaStream_t st, int grid_override = 0) {
  if (items <= 0) return SBW_OK;
  DeviceProps dp;
  if (int rc = device_props(&dp)) return rc;
  static unsigned long long attr_done = 0;  // per device; the call is idempotent
  if (!(attr_done >> (dp.device & 63) & 1ull)) {
    SBW_CUDA_CHECK(cudaFuncSetAttribute(k_tc_hybrid<MODE, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        is_staged(MODE) ? kTcSmemSt : kTcSmem));
    attr_done |= 1ull << (dp.device & 63);
  }
  TcArgs args = a;
  if (int rc = tc_consts(dp.device, st, &args.consts)) return rc;
  const int grid = grid_override > 0 ? grid_override : int(items < dp.sm_count ? items : dp.sm_count);
  k_tc_hybrid<MODE, NB><<<grid, kAllThreads, is_staged(MODE) ? kTcSmemSt : kTcSmem, st>>>(args);
  SBW_LAUNCH_CHECK(is_emit(MODE) ? "k_tc_hybrid<emit>" : (is_spec(MODE) ? "k_tc_hybrid<spec>" : "k_tc_hybrid<nl>"));
  return SBW_OK;
}
}  // namespace

int launch_tc16_nl(const uint32_t* planes, uint32_t v_lo, uint32_t v_hi, int32_t* max_abs,
                   unsigned long long* key, cudaStream_t st) {
  if (tc_lut_enabled()) return launch_tc16_nl_lut(planes, v_lo, v_hi, max_abs, key, st);
  TcArgs a{};
  a.planes = planes;
  a.plane_words = 2048;
  a.v_lo = v_lo;
  a.v_hi = v_hi;
  a.max_abs = max_abs;
  a.key = key;
  return run_tc_hybrid<kTcNL>(a, int64_t(v_hi) - v_lo, st);
}

int tc_min_small_n() { return 8 + kLogRows; }

int launch_tc_nl_small(const uint32_t* planes, int n, uint32_t v_lo, uint32_t v_hi, int32_t* max_abs,
                       unsigned long long* key, cudaStream_t st) {
  TcArgs a{};
  a.planes = planes;
  a.plane_words = (int64_t(1) << n) >> 5;
  a.v_lo = v_lo;
  a.v_hi = v_hi;
  a.max_abs = max_abs;
  a.key = key;
  const int lc = 16 - n;
  const int64_t items = ((int64_t(v_hi) - 1) >> lc) + 1 - (int64_t(v_lo) >> lc);
  switch (n) {
#define SBW_TC_SMALL_CASE(N)                                         \
    case N:                                                          \
      if constexpr (8 + kLogRows <= N) return run_tc_hybrid<kTcNL, N>(a, items, st); \
      return set_error(SBW_EINVAL, "row-group generation needs n >= %d", 8 + kLogRows);
    SBW_TC_SMALL_CASE(11)
    SBW_TC_SMALL_CASE(12)
    SBW_TC_SMALL_CASE(13)
    SBW_TC_SMALL_CASE(14)
    SBW_TC_SMALL_CASE(15)
#undef SBW_TC_SMALL_CASE
    default: return set_error(SBW_EINVAL, "tensor-core NL for n < 16 needs n in 11..15");
  }
}

// staged spectrum epilogue (bulk copies of 8 KiB slots) when the rows are
// 16-byte aligned; SBW_SPEC_STAGE=0 keeps the per-lane store epilogue (A/B)
bool spec_staged_ok(const int32_t* out, int64_t ld) {
  static const bool on = !(getenv("SBW_SPEC_STAGE") && atoi(getenv("SBW_SPEC_STAGE")) == 0);
  return on && (reinterpret_cast<uintptr_t>(out) & 15) == 0 && (ld & 3) == 0;
}

int launch_tc_spec_small(const uint32_t* planes, int n, uint32_t v_lo, uint32_t v_hi, int32_t* max_abs,
                         int32_t* out, int64_t ld, cudaStream_t st) {
  TcArgs a{};
  a.planes = planes;
  a.plane_words = (int64_t(1) << n) >> 5;
  a.v_lo = v_lo;
  a.v_hi = v_hi;
  a.max_abs = max_abs;
  a.out = out;
  a.ld = ld;
  const int lc = 16 - n;
  const int64_t items = ((int64_t(v_hi) - 1) >> lc) + 1 - (int64_t(v_lo) >> lc);
  switch (n) {
#define SBW_TC_SPEC_CASE(N)                                                             \
    case N:                                                                             \
      if constexpr (8 + kLogRows <= N) {                                                \
        if constexpr (kRows == 16 && N >= 12)                                           \
          if (spec_staged_ok(out, ld)) return run_tc_hybrid<kTcSpecSt, N>(a, items, st); \
        return run_tc_hybrid<kTcSpec, N>(a, items, st);                                 \
      }                                                                                 \
      return set_error(SBW_EINVAL, "row-group generation needs n >= %d", 8 + kLogRows);
    SBW_TC_SPEC_CASE(11)
    SBW_TC_SPEC_CASE(12)
    SBW_TC_SPEC_CASE(13)
    SBW_TC_SPEC_CASE(14)
    SBW_TC_SPEC_CASE(15)
#undef SBW_TC_SPEC_CASE
    default: return set_error(SBW_EINVAL, "tensor-core spectrum for n < 16 needs n in 11..15");
  }
}

int launch_tc16_spec(const uint32_t* planes, uint32_t v_lo, uint32_t v_hi, int32_t* max_abs,
                     int32_t* out, int64_t ld, cudaStream_t st) {
  if (!kC0Mma) return set_error(SBW_EINVAL, "tensor-core spectrum needs SBW_TC_ROWS >= 2");
  TcArgs a{};
  a.planes = planes;
  a.plane_words = 2048;
  a.v_lo = v_lo;
  a.v_hi = v_hi;
  a.max_abs = max_abs;
  a.out = out;
  a.ld = ld;
  if (kRows == 16 && spec_staged_ok(out, ld)) return run_tc_hybrid<kTcSpecSt>(a, int64_t(v_hi) - v_lo, st);
  return run_tc_hybrid<kTcSpec>(a, int64_t(v_hi) - v_lo, st);
}

// x-major rows of a bijective box from its inverse's planes (kTcSpecSt with
// zoff = 1): row u in [u_lo, u_hi) of wt[u][v - 1] at out + (u - u_lo) * ld
int launch_tc_xmajor_inverse(const uint32_t* inv_planes, int n, uint32_t u_lo, uint32_t u_hi,
                             int32_t* max_scratch, int32_t* out, int64_t ld, cudaStream_t st) {
  if (kRows != 16) return set_error(SBW_EINVAL, "x-major from the inverse needs SBW_TC_ROWS = 16");
  if (n < 12 || n > 16) return set_error(SBW_EINVAL, "x-major from the inverse needs n in 12..16");
  if (reinterpret_cast<uintptr_t>(out) & 3) return set_error(SBW_EINVAL, "output not 4-byte aligned");
  TcArgs a{};
  a.planes = inv_planes;
  a.plane_words = (int64_t(1) << n) >> 5;
  a.v_lo = u_lo;
  a.v_hi = u_hi;
  a.max_abs = max_scratch;
  a.goff = int64_t((reinterpret_cast<uintptr_t>(out) & 15) >> 2);
  a.out = reinterpret_cast<int32_t*>(reinterpret_cast<uintptr_t>(out) & ~uintptr_t(15));
  a.ld = ld;
  a.zoff = 1;  // (kTcSpecStX; recorded for readers of TcArgs)
  const int lc = 16 - n;
  const int64_t items = ((int64_t(u_hi) - 1) >> lc) + 1 - (int64_t(u_lo) >> lc);
  if constexpr (kRows == 16) {
    switch (n) {
      case 12: return run_tc_hybrid<kTcSpecStX, 12>(a, items, st);
      case 13: return run_tc_hybrid<kTcSpecStX, 13>(a, items, st);
      case 14: return run_tc_hybrid<kTcSpecStX, 14>(a, items, st);
      case 15: return run_tc_hybrid<kTcSpecStX, 15>(a, items, st);
      default: return run_tc_hybrid<kTcSpecStX, 16>(a, items, st);
    }
  }
  return SBW_OK;
}

int launch_tc_emit(const uint32_t* planes, int n, uint32_t v_first, int64_t n_comp, uint32_t* emit,
                   uint32_t run_lo, uint32_t run_hi, cudaStream_t st, int emit16, int* flag, const int* gate,
                   int gate_on) {
  if (!emit16 && tc_lut_emit_enabled())
    return launch_tc_emit_lut(planes, n, v_first, n_comp, emit, run_lo, run_hi, st, gate, gate_on);
  TcArgs a{};
  a.run_lo = run_lo;
  a.run_hi = run_hi;

  a.flag = flag;
  a.gate = gate;
  a.gate_on = gate_on;
  a.planes = planes;
  a.plane_words = (int64_t(1) << n) >> 5;
  a.v_first = v_first;
  a.n_comp = n_comp;
  a.n_items = n_comp << (n - 16);
  a.n_full = n;
  a.emit = emit;
  return emit16 ? run_tc_hybrid<kTcEmit16>(a, a.n_items, st) : run_tc_hybrid<kTcEmit>(a, a.n_items, st);
}

int launch_tc_emit_ring(const uint32_t* planes, int n, uint32_t v_first, const RingArgs& ring, uint32_t* emit,
                        cudaStream_t st) {
  TcArgs a{};
  a.planes = planes;
  a.plane_words = (int64_t(1) << n) >> 5;
  a.v_first = v_first;
  a.n_comp = ring.batches * ring.bc;
  a.n_items = a.n_comp << (n - 16);
  a.n_full = n;
  a.emit = emit;
  a.ring = ring;
  return run_tc_hybrid<kTcEmit>(a, a.n_items, st, int(ring.na));
}

}  // namespace sbw
