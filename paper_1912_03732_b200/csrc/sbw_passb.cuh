// Multi-pass path for n = 17..24 ("K3"), pass B.
//
// Pass A (k_tc_hybrid<kTcEmit> in sbw_tc.cu, or k_tile_simd<15, MODE_EMIT>
// with SBW_TC=0; one launch per batch of components) leaves, for every
// component of the batch, 2^(n-15) blocks of 2^15 partial transforms (x bits
// 0..14 done), each as the biased u16 s = (v + 2^15) / 2 in [0, 2^15].  Pass
// B runs the remaining H = n - 15 stages over x bits 15..n-1, i.e. across
// blocks, on v / 2 = s - 2^14 in exact fp32, and fuses max|W| into the top
// stage like the on-chip kernel.  The reference does all n stages on one
// numpy array per mask (walsh.py:91-103); stage order is free because the
// butterflies of different bits commute.
//
//   H <= 5: k_passb_regs   -- registers only, one thread per pair-column,
//           barrier-free.
//   H >= 6: k_passb_staged -- cp.async-staged [2^H rows x 2^(13-H) pair-columns]
//           chunks, two register passes through a 64 KiB fp32 tile, the next
//           chunk prefetched while the current one computes.
#pragma once

#include <cuda.h>

#include "sbw_tile_simd.cuh"

namespace sbw {

struct PassBArgs {
  const uint32_t* scratch;   // int16 pairs: [comp][2^n] halved values
  int n;
  int64_t n_comp;            // components in this batch
  int64_t out_row0;          // index of this batch's first component in max_abs / out
  uint32_t v_first;          // mask of this batch's first component
  int32_t* max_abs;          // zero-initialised by the host for the batch
  unsigned long long* key;
  int32_t* out;              // materialised rows (may be null)
  int64_t ld;
  RingArgs ring;             // k_passb_tc only: L2 ring mode (scratch = the ring slots)
  // gray != 0 (NL after the tensor-core pass A): batch position p = v_first +
  // comp holds mask mask_at(p, run_lo, run_hi) (Gray order inside aligned
  // 256-blocks of the run, so pass A's generation is one plane XOR per
  // component); max_abs is indexed by mask - run_lo.
  int gray;
  uint32_t run_lo, run_hi;
  // e16 = 1: the scratch holds pass A's 16-stage output (rows = x bits
  // 16..n-1 of 2^16 biased u16 s = W_16 / 2 + 2^15, k_passb_regs /
  // k_passb_tc only); 0: 15-stage (rows = x bits 15..n-1, 2^15 u16, bias 2^14)
  int e16;
  // run only if (*gate != 0) == gate_on (gate may be null)
  const int* gate;
  int gate_on;
};

__device__ __forceinline__ bool passb_gated_off(const PassBArgs& a) {
  return a.gate && ((*a.gate != 0) != (a.gate_on != 0));
}

// Publish a component's max: natural order (mask v_first + comp, row
// out_row0 + comp) or the Gray order of the tensor-core pass A.
__device__ __forceinline__ void publish_comp(const PassBArgs& a, int64_t comp, int run);

// Pass B of max|W| runs its butterflies in fp32 on the FMA pipe (FADD at 4
// warp-instr/clk/SM, twice the IADD3 rate).  Every intermediate is an integer
// with |h| <= 2^(n-1) <= 2^23, which fp32 represents exactly, and the sum of
// two such values is rounded only above 2^24, so the arithmetic is bit-exact
// (K3).  The u16 s = h + 2^14 enters by PRMT under the exponent of
// 2^23 (0x4B000000 | s is the float 2^23 + s), and the first row stage absorbs
// the bias: with A = 2^23 + s_a, B = 2^23 + s_b, h_a - h_b = A - B and
// h_a + h_b = (A - (2^24 + 2^15)) + B, every partial an integer below 2^24 --
// three FADDs per lane pair.  Rows ua (even) / ub (odd) -> e[0..3].
// (e16: s = h + 2^15, so the pair's bias is 2^24 + 2^16.)
__device__ __forceinline__ void load_rows_stage1(uint32_t ua, uint32_t ub, float* e, float bias2 = 16809984.0f) {
  const float al = __int_as_float(int(__byte_perm(ua, 0x4B000000u, 0x7610)));
  const float ah = __int_as_float(int(__byte_perm(ua, 0x4B000000u, 0x7632)));
  const float bl = __int_as_float(int(__byte_perm(ub, 0x4B000000u, 0x7610)));
  const float bh = __int_as_float(int(__byte_perm(ub, 0x4B000000u, 0x7632)));
  e[0] = __fadd_rn(__fsub_rn(al, bias2), bl);
  e[1] = __fadd_rn(__fsub_rn(ah, bias2), bh);
  e[2] = __fsub_rn(al, bl);
  e[3] = __fsub_rn(ah, bh);
}

template <int LEN, int S0, int SEND>
__device__ __forceinline__ void fwht_regs_f(float (&e)[LEN]) {
#pragma unroll
  for (int s = S0; s < SEND; s <<= 1) {
#pragma unroll
    for (int i = 0; i < LEN; ++i) {
      if ((i & s) == 0) {
        const float a = e[i], b = e[i + s];
        e[i] = __fadd_rn(a, b);
        e[i + s] = __fsub_rn(a, b);
      }
    }
  }
}

// ---- H = 6..9: staged chunks ---------------------------------------------
// A chunk is 2^H rows (x bits 15..n-1) x CW = 2^(13-H) pair-columns: 8192
// u16-pair words.  Its words are first staged in shared memory by cp.async.cg
// (16-byte pieces, L2 only: the persistent kernel reuses its staging buffer, so
// an SM's L1 may hold lines of an older component); the copy of the CTA's next
// chunk overlaps the arithmetic of the current one.  B1 runs row bits
// H2..H-1 from the staging buffer into a 64 KiB fp32-pair tile, B2 runs row
// bits 0..H2-1 with the fused top stage.  96 KiB per CTA, two 256-thread CTAs
// per SM, so one CTA's barriers and staging waits overlap the other's
// arithmetic.  Every warp access is 32 consecutive words (B1, staging) or two
// contiguous 128-byte half-warp rows (tile), so shared memory is conflict-free.
constexpr int kStagedThreads = 256;

template <int H>
struct StagedShape {
  static constexpr int LCW = 13 - H;               // log2 pair-columns per chunk
  static constexpr int CW = 1 << LCW;
  static constexpr int H1 = (H + 1) / 2;           // B1 stages (row bits H2..H-1)
  static constexpr int H2 = H - H1;                // B2 stages (row bits 0..H2-1)
  static constexpr int64_t PER_COMP = (int64_t(1) << 14) >> LCW;
  static constexpr int WORDS = CW << H;            // 8192
};
constexpr size_t kStagedSmem = size_t(8192) * 4 + size_t(8192) * 8;  // staging + tile

// Issue (not wait for) the copies of chunk `chunk` of a component whose
// scratch starts at `comp_base` into `stg` ([2^H][CW] words).
template <int H>
__device__ __forceinline__ void stage_chunk(const uint32_t* comp_base, int64_t chunk, uint32_t* stg) {
  using S = StagedShape<H>;
  constexpr int PR = S::CW / 4;  // 16-byte pieces per row
  const uint32_t* g0 = comp_base + chunk * S::CW;
#pragma unroll
  for (int k = 0; k < S::WORDS / 4 / kStagedThreads; ++k) {
    const int p = threadIdx.x + k * kStagedThreads;
    const int r = p / PR, q = p % PR;
    const uint32_t* g = g0 + (int64_t(r) << 14) + 4 * q;
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(stg + 4 * p));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(g) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__device__ __forceinline__ void stage_wait() {
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
}

// Returns this thread's max|W| over the chunk.
template <int H, int MODE, typename AfterRead>
__device__ __forceinline__ int passb_staged_chunk(const PassBArgs& a, int64_t comp, int64_t chunk,
                                                  const uint32_t* stg, float2* tile,
                                                  AfterRead after_read) {
  using S = StagedShape<H>;
  constexpr int N1 = 1 << S::H1, N2 = 1 << S::H2;
#pragma unroll 1
  for (int task = threadIdx.x; task < (S::CW << S::H2); task += kStagedThreads) {
    const int c = task & (S::CW - 1), rb = task >> S::LCW;
    float e[2 * N1];
#pragma unroll
    for (int i = 0; i < N1; i += 2)
      load_rows_stage1(stg[(rb + (i << S::H2)) * S::CW + c], stg[(rb + ((i + 1) << S::H2)) * S::CW + c],
                       e + 2 * i);
    fwht_regs_f<2 * N1, 4, 2 * N1>(e);
#pragma unroll
    for (int i = 0; i < N1; ++i)
      tile[(rb + (i << S::H2)) * S::CW + c] = make_float2(e[2 * i], e[2 * i + 1]);
  }
  __syncthreads();
  after_read();
  float mf = 0.f;
  int mx = 0;
#pragma unroll 1
  for (int task = threadIdx.x; task < (S::CW << S::H1); task += kStagedThreads) {
    const int c = task & (S::CW - 1), g = task >> S::LCW;
    float e[2 * N2];
#pragma unroll
    for (int j = 0; j < N2; ++j) {
      const float2 p = tile[((g << S::H2) + j) * S::CW + c];
      e[2 * j] = p.x;
      e[2 * j + 1] = p.y;
    }
    fwht_regs_f<2 * N2, 2, N2>(e);
    if constexpr (MODE == MODE_NL) {
#pragma unroll
      for (int k = 0; k < N2; ++k) mf = fmaxf(mf, __fadd_rn(fabsf(e[k]), fabsf(e[k + N2])));
    } else {
      int w[2 * N2];
#pragma unroll
      for (int k = 0; k < N2; ++k) {
        const float p = e[k], q = e[k + N2];  // W / 2, exact below 2^24
        w[k] = 2 * __float2int_rn(__fadd_rn(p, q));
        w[k + N2] = 2 * __float2int_rn(__fsub_rn(p, q));
        mx = max(mx, max(abs(w[k]), abs(w[k + N2])));
      }
      int32_t* dst = a.out + (a.out_row0 + comp) * a.ld + 2 * (chunk * S::CW + c);
#pragma unroll
      for (int j = 0; j < N2; ++j) {
        const int64_t row = (int64_t(g) << S::H2) + j;
        __stcs(reinterpret_cast<int2*>(dst + (row << 15)), make_int2(w[2 * j], w[2 * j + 1]));
      }
    }
  }
  if constexpr (MODE == MODE_NL) mx = 2 * __float2int_rn(mf);
  return mx;
}

// Per-warp publish of a component's running max (no CTA barrier).
__device__ __forceinline__ void warp_publish_max(int mx, int32_t* slot, unsigned long long* key,
                                                 uint32_t v) {
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) {
    atomicMax(slot, mx);
    if (key) atomicMax(key, nl_key(mx, v));
  }
}

__device__ __forceinline__ void publish_comp(const PassBArgs& a, int64_t comp, int run) {
  if (a.gray) {
    const uint32_t v = mask_at(int64_t(a.v_first) + comp, a.run_lo, a.run_hi);
    warp_publish_max(run, a.max_abs + (v - a.run_lo), a.key, v);
  } else {
    warp_publish_max(run, a.max_abs + a.out_row0 + comp, a.key, a.v_first + uint32_t(comp));
  }
}

// ---- batched path for H <= 5 (n = 17..20) -----------------------------------
// Pass A runs as standalone EMIT tile launches over a batch of components;
// this kernel then runs the remaining H stages.  One thread owns one
// pair-column (2^H rows, 2^(H+1) fp32 values, exact as in pass B staged),
// 256-thread CTAs at high occupancy, each CTA one contiguous range of
// (component, 256-column) items with no barrier: warps drift apart, so one
// warp's loads overlap another's arithmetic.  Launch boundaries invalidate L1,
// so plain (evict-first) loads are safe.
constexpr int kPassBThreads = 256;

template <int H, int MODE>
__global__ void __launch_bounds__(kPassBThreads) k_passb_regs(PassBArgs a) {
  constexpr int NI = 1 << H;
  if (passb_gated_off(a)) return;
  const int row_log = 14 + a.e16;                                   // u32 words per row
  const int64_t chunks = (int64_t(1) << row_log) / kPassBThreads;  // per component
  const float bias2 = a.e16 ? 16842752.0f : 16809984.0f;           // 2^24 + 2^16 / 2^24 + 2^15
  const int64_t items = a.n_comp * chunks;
  const int64_t per_cta = (items + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per_cta;
  const int64_t b1 = b0 + per_cta < items ? b0 + per_cta : items;
  int run = 0;
  for (int64_t b = b0; b < b1; ++b) {
    const int64_t comp = b / chunks;
    const int64_t col = (b % chunks) * kPassBThreads + threadIdx.x;
    const uint32_t* src = a.scratch + (comp << (a.n - 1)) + col;
    uint32_t u[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) u[i] = __ldcs(src + (int64_t(i) << row_log));
    float e[2 * NI];
#pragma unroll
    for (int i = 0; i < NI; i += 2) load_rows_stage1(u[i], u[i + 1], e + 2 * i, bias2);
    fwht_regs_f<2 * NI, 4, NI>(e);
    if constexpr (MODE == MODE_NL) {
      float mf = 0.f;
#pragma unroll
      for (int k = 0; k < NI; ++k) mf = fmaxf(mf, __fadd_rn(fabsf(e[k]), fabsf(e[k + NI])));
      run = max(run, 2 * __float2int_rn(mf));  // values are halved
    } else {
      int w[2 * NI];
#pragma unroll
      for (int k = 0; k < NI; ++k) {
        const float p = e[k], q = e[k + NI];
        w[k] = 2 * __float2int_rn(__fadd_rn(p, q));
        w[k + NI] = 2 * __float2int_rn(__fsub_rn(p, q));
        run = max(run, max(abs(w[k]), abs(w[k + NI])));
      }
      int32_t* dst = a.out + (a.out_row0 + comp) * a.ld + 2 * col;
#pragma unroll
      for (int i = 0; i < NI; ++i)
        __stcs(reinterpret_cast<int2*>(dst + (int64_t(i) << 15)), make_int2(w[2 * i], w[2 * i + 1]));
    }
    if (b + 1 >= b1 || (b + 1) / chunks != comp) {  // CTA-uniform
      publish_comp(a, comp, run);
      run = 0;
    }
  }
}

// ---- H <= 5 (n = 17..20) NL pass B fed by bulk copies ------------------------
// The same per-column arithmetic as k_passb_regs, but an item's 2^H rows of
// 256 words (1 KiB each) reach shared memory by TMA (completion on an
// mbarrier), kBulkStages items ahead of
// the one being computed, one 2D TMA load per item.  k_passb_regs keeps 2^H
// 4-byte loads per thread in flight and is latency-bound near 5 TB/s; here
// one thread per CTA keeps kBulkStages x 2^H KiB in flight.
#ifndef SBW_BULK_THREADS
#define SBW_BULK_THREADS 256
#endif
constexpr int kBulkThreads = SBW_BULK_THREADS;
#ifndef SBW_BULK_STAGES
#define SBW_BULK_STAGES 2
#endif
constexpr int kBulkStages = SBW_BULK_STAGES;
template <int H>
constexpr int bulk_smem_bytes() { return kBulkStages * (1 << H) * kBulkThreads * 4; }

__device__ __forceinline__ void tma_load_2d_u32(uint32_t* dst, const void* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y),
      "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
      : "memory");
}

__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tSBW_BULK_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra SBW_BULK_DONE;\n\tbra SBW_BULK_WAIT;\n\tSBW_BULK_DONE:\n\t}\n" ::"r"(
          static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
      "r"(parity)
      : "memory");
}

// tmap: 2D tensor map over the batch scratch, dims {2^(14 + e16) words of a
// row, n_comp * 2^H rows}, box {256 words, 2^H rows}: one TMA load per item.
template <int H>
__global__ void __launch_bounds__(kBulkThreads) k_passb_bulk(const __grid_constant__ CUtensorMap tmap, PassBArgs a) {
  constexpr int NI = 1 << H;
  constexpr uint32_t kRowBytes = kBulkThreads * 4;
  extern __shared__ __align__(128) uint32_t bsm[];  // [kBulkStages][NI][256] words
  __shared__ __align__(8) uint64_t full[kBulkStages];
  if (passb_gated_off(a)) return;
  const int row_log = 14 + a.e16;  // u32 words per row
  const int64_t chunks = (int64_t(1) << row_log) / kBulkThreads;
  const float bias2 = a.e16 ? 16842752.0f : 16809984.0f;
  const int64_t items = a.n_comp * chunks;
  const int64_t per_cta = (items + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per_cta;
  const int64_t b1 = b0 + per_cta < items ? b0 + per_cta : items;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kBulkStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(
                       static_cast<uint32_t>(__cvta_generic_to_shared(&full[s])))
                   : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // thread 0: load item b's rows into stage s
  auto issue = [&](int64_t b, int s) {
    const int64_t comp = b / chunks, ch = b - comp * chunks;
    bar_expect_tx(&full[s], NI * kRowBytes);
    tma_load_2d_u32(bsm + s * (NI * kBulkThreads), &tmap, int(ch * kBulkThreads), int(comp * NI), &full[s]);
  };
  if (tid == 0)
    for (int k = 0; k < kBulkStages && b0 + k < b1; ++k) issue(b0 + k, k);
  int run = 0;
  int64_t it = 0;
  for (int64_t b = b0; b < b1; ++b, ++it) {
    const int s = int(it % kBulkStages);
    bar_wait_parity(&full[s], uint32_t((it / kBulkStages) & 1));
    uint32_t u[NI];
    const uint32_t* stg = bsm + s * (NI * kBulkThreads) + tid;
#pragma unroll
    for (int r = 0; r < NI; ++r) u[r] = stg[r * kBulkThreads];
    __syncthreads();  // stage s fully read: refill it
    if (tid == 0 && b + kBulkStages < b1) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(b + kBulkStages, s);
    }
    float e[2 * NI];
#pragma unroll
    for (int i = 0; i < NI; i += 2) load_rows_stage1(u[i], u[i + 1], e + 2 * i, bias2);
    fwht_regs_f<2 * NI, 4, NI>(e);
    float mf = 0.f;
#pragma unroll
    for (int k = 0; k < NI; ++k) mf = fmaxf(mf, __fadd_rn(fabsf(e[k]), fabsf(e[k + NI])));
    run = max(run, 2 * __float2int_rn(mf));  // values are halved
    const int64_t comp = b / chunks;
    if (b + 1 >= b1 || (b + 1) / chunks != comp) {  // CTA-uniform
      publish_comp(a, comp, run);
      run = 0;
    }
  }
}

// H = 6..9 standalone pass B over (component, chunk) items; each item's u16 rows are staged with cp.async and the CTA's next item is
// prefetched as soon as B1 has consumed the current staging.
template <int H, int MODE>
__global__ void __launch_bounds__(kStagedThreads, 2) k_passb_staged(PassBArgs a) {
  using S = StagedShape<H>;
  if (passb_gated_off(a)) return;  // (15-stage layout only: e16 is never set here)
  extern __shared__ uint4 smem4[];  // [32 KiB staging][64 KiB fp32-pair tile]
  uint32_t* stg = reinterpret_cast<uint32_t*>(smem4);
  float2* tile = reinterpret_cast<float2*>(stg + S::WORDS);
  // Each CTA owns one contiguous range of items, so it meets few component
  // boundaries and publishes (per warp, no barrier) only at those.
  const int64_t items = a.n_comp * S::PER_COMP;
  const int64_t per_cta = (items + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per_cta;
  const int64_t b1 = b0 + per_cta < items ? b0 + per_cta : items;
  const int64_t comp_words = int64_t(1) << (a.n - 1);
  if (b0 < b1) stage_chunk<H>(a.scratch + (b0 / S::PER_COMP) * comp_words, b0 % S::PER_COMP, stg);
  int run = 0;  // running max over this CTA's chunks of the current component
  for (int64_t b = b0; b < b1; ++b) {
    stage_wait();  // also orders the previous chunk's B2 tile reads before this B1
    const int64_t comp = b / S::PER_COMP, nxt = b + 1;
    auto prefetch = [&]() {
      if (nxt < b1)
        stage_chunk<H>(a.scratch + (nxt / S::PER_COMP) * comp_words, nxt % S::PER_COMP, stg);
    };
    run = max(run, passb_staged_chunk<H, MODE>(a, comp, b % S::PER_COMP, stg, tile, prefetch));
    if (nxt >= b1 || nxt / S::PER_COMP != comp) {  // CTA-uniform
      publish_comp(a, comp, run);
      run = 0;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
}

}  // namespace sbw
