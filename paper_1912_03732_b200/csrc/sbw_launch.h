// Host-side launchers shared between the libsbw translation units.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace sbw {

// Bit planes of the S-box (bit x of plane i = bit i of S(x)), n >= 7.
size_t planes_bytes(int n, int m);
int build_planes(const void* table, int tbytes, int n, int m, uint32_t* planes, cudaStream_t st);

// Fused on-chip path (n <= 16): NL (out == nullptr) or mask-major SPEC rows.
// `scratch` holds the bit planes (planes_bytes(n, m)) for n >= 7.
int launch_fused_onchip(const void* table, int tbytes, int n, int m, uint32_t v_lo, uint32_t v_hi,
                        int32_t* max_abs, unsigned long long* key, int32_t* out, int64_t ld,
                        void* scratch, cudaStream_t st);

// Tensor-core hybrid for n = 16 NL (planes already built): int8 MMA for x bits
// 0..7, packed integer stages for bits 8..15 (sbw_tc.cu).
int launch_tc16_nl(const uint32_t* planes, uint32_t v_lo, uint32_t v_hi, int32_t* max_abs,
                   unsigned long long* key, cudaStream_t st);
bool tc_path_enabled();
// Tensor-core NL for n = 11..15 (2^(16-n) components per 2^16 tile); needs
// m >= 16 - n so every slot's mask is a valid mask.
// k_tc_lut (sbw_tc_lut.cu): the same n = 16 NL job with the GEMM over x bits
// 8..15 and a table-lookup generation; launch_tc16_nl takes it unless SBW_TC_LUT=0
bool tc_lut_enabled();
int launch_tc16_nl_lut(const uint32_t* planes, uint32_t v_lo, uint32_t v_hi, int32_t* max_abs,
                       unsigned long long* key, cudaStream_t st);
// k_tc_lut_emit: pass A of the multi-pass path with the table-lookup generation
// (exact but measured slower; launch_tc_emit takes it only with SBW_TC_LUT_EMIT=1)
bool tc_lut_emit_enabled();
int launch_tc_emit_lut(const uint32_t* planes, int n, uint32_t v_first, int64_t n_comp, uint32_t* emit,
                       uint32_t run_lo, uint32_t run_hi, cudaStream_t st, const int* gate, int gate_on);
int tc_min_small_n();  // smallest n of launch_tc_nl_small (11, or 12 for 16-row generation builds)
int launch_tc_nl_small(const uint32_t* planes, int n, uint32_t v_lo, uint32_t v_hi, int32_t* max_abs,
                       unsigned long long* key, cudaStream_t st);
// Tensor-core n = tc_min_small_n()..15 materialised spectrum (m >= 16 - n), mask-major rows.
int launch_tc_spec_small(const uint32_t* planes, int n, uint32_t v_lo, uint32_t v_hi, int32_t* max_abs,
                         int32_t* out, int64_t ld, cudaStream_t st);
// Tensor-core n = 16 materialised spectrum, mask-major rows out[(v - v_lo) * ld + u].
int launch_tc16_spec(const uint32_t* planes, uint32_t v_lo, uint32_t v_hi, int32_t* max_abs,
                     int32_t* out, int64_t ld, cudaStream_t st);
// The reference's x-major store (wt[u][v - 1], any pitch ld) of a bijective
// n x n box, rows u in [u_lo, u_hi), from its inverse's bit planes: the
// staged spectrum kernel with rows shifted by one (W_S(u, v) = W_T(v, u),
// T = S^-1).  n = 12..16; max_scratch gets T's per-row maxima (discarded).
int launch_tc_xmajor_inverse(const uint32_t* inv_planes, int n, uint32_t u_lo, uint32_t u_hi,
                             int32_t* max_scratch, int32_t* out, int64_t ld, cudaStream_t st);
// Tensor-core pass A of the multi-pass NL path (n = 17..24): 15 stages per
// 2^15 block, biased u16 out in a block-internal word order of its own
// (pass B pairs equal word positions across blocks only, so any fixed order
// works for NL; SPEC keeps launch_emit_tiles).
// Components are taken in the Gray order mask_at(position, run_lo, run_hi)
// of the whole run [run_lo, run_hi) (pass B publishes with the same map).
// emit16 = 1: 16 stages, wrapped u16 out (an affine tile raises *flag);
// gate: run only if (*gate != 0) == gate_on (null: always).
int launch_tc_emit(const uint32_t* planes, int n, uint32_t v_first, int64_t n_comp, uint32_t* emit,
                   uint32_t run_lo, uint32_t run_hi, cudaStream_t st, int emit16 = 0, int* flag = nullptr,
                   const int* gate = nullptr, int gate_on = 0);

// The same pass A streaming into the L2 ring of a concurrently running
// k_passb_tc (RingArgs in sbw_internal.cuh); grid = ring.na CTAs.
struct RingArgs;
int launch_tc_emit_ring(const uint32_t* planes, int n, uint32_t v_first, const RingArgs& ring, uint32_t* emit,
                        cudaStream_t st);

// Multi-pass path (n >= 17): planes, then pass A (emit) + pass B per L2-sized batch.
size_t k3_scratch_bytes(int n, int m, uint32_t v_lo, uint32_t v_hi);
// K3 pass B on the tensor cores (n = 22..24, NL only), sbw_passb_tc.cu;
// SBW_PASSB_TC=0 keeps the fp32 k_passb_staged kernel.
struct PassBArgs;
bool passb_tc_enabled();
// cuTensorMapEncodeTiled through the runtime's driver entry point (null if unavailable)
void* tma_encode_ptr();
int launch_passb_tc(const PassBArgs& a, cudaStream_t st);
int launch_k3(const void* table, int tbytes, int n, int m, uint32_t v_lo, uint32_t v_hi,
              int32_t* max_abs, unsigned long long* key, int32_t* out, int64_t ld, void* scratch,
              size_t scratch_bytes, cudaStream_t st);


// Pass-A tiles (generation + 15 stages, biased u16 out) for components
// [v_first, v_first + n_comp), used by the batched multi-pass path.
int launch_emit_tiles(const uint32_t* planes, int n, int m, uint32_t v_first, int64_t n_comp,
                      uint32_t* emit, cudaStream_t st);

// Total workspace of sbw_nl (planes + multi-pass scratch).
inline size_t nl_scratch_bytes(int n, int m, uint32_t v_lo, uint32_t v_hi) {
  return n >= 17 ? k3_scratch_bytes(n, m, v_lo, v_hi) : planes_bytes(n, m);
}

// Misc kernels.
int launch_transpose_i32(const int32_t* in, int64_t rows, int64_t cols, int64_t ld_in,
                         int32_t* out, int64_t ld_out, cudaStream_t st);
int launch_fill_i32(int32_t* p, int64_t count, int32_t value, cudaStream_t st);
int inplace_fwht(int32_t* d, int k, int64_t count, long long* max_abs, cudaStream_t st);
// Any integer dtype (SBW_ELEM_*), any strides (sbw_inplace.cu).
int inplace_fwht_strided(void* data, int elem, int k, int64_t count, int64_t col_stride,
                         int64_t elem_stride, long long* max_abs, cudaStream_t st);
int launch_polarity(const void* table, int tbytes, int n, uint32_t v_lo, uint32_t v_hi,
                    int layout, int32_t* out, int64_t ld, cudaStream_t st);
int launch_maxabs_to_nl(const int32_t* mx, int64_t count, int n, long long* nl, long long* bad,
                        cudaStream_t st);
int launch_maxabs64_to_nl(const long long* mx, int64_t count, long long pw, long long* nl,
                          long long* bad, cudaStream_t st);
int launch_row_maxabs(const int32_t* rows, int64_t nrows, int64_t cols, int64_t ld,
                      long long* row_max, unsigned long long* key, cudaStream_t st);
int launch_walsh_direct(const void* table, int tbytes, int n, const uint32_t* u,
                        const uint32_t* v, int64_t count, int32_t* out, cudaStream_t st);
int launch_bruteforce(const void* table, int tbytes, int n, int m, int32_t* best,
                      cudaStream_t st);
// *dst = max(*dst, *src) with a system-scope atomic (dst may be peer memory).
int launch_key_merge(const unsigned long long* src, unsigned long long* dst, cudaStream_t st);
int run_int32_peak(double* ops_per_s, double* ms_out, cudaStream_t st);
int run_int8_mma_peak(double* ops_per_s, double* ms_out, cudaStream_t st);

}  // namespace sbw
