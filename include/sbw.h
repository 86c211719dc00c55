/*
 * sbw.h -- C ABI of libsbw, the sm_100a (B200) S-box Walsh-spectrum and
 * nonlinearity engine.  No torch types cross this boundary: plain pointers,
 * sizes and a cudaStream_t passed as void*.
 *
 * The reference (`sboxeval`, pure Python + numpy, under /root/reference) has
 * no native code; each entry point below names the reference function whose
 * hot loop it replaces.  INTEGRATION.md shows the ctypes binding a
 * maintainer would add to the reference package.
 *
 * Conventions (identical to the reference):
 *   - masks v run over [v_lo, v_hi) with 1 <= v_lo <= v_hi <= 2^m; the v = 0
 *     row is never stored (sbox.py:155-159);
 *   - spectra are int32 in natural (Sylvester) order, unnormalised:
 *     W(u,v) = sum_x (-1)^{popc(v & S(x)) + popc(u & x)} (walsh.py:56-70);
 *   - per-component maxima are max over ALL u (u = 0 included) of |W(u,v)|
 *     (walsh.py:101-102); NL_v = (2^n - max|W|) / 2 (walsh.py:107-114);
 *   - the "key" is the 64-bit value (max|W| << 32) | (0xFFFFFFFF - v),
 *     so an atomicMax picks the largest max|W| with ties to the SMALLEST v,
 *     i.e. the reference's first-argmin (nonlinearity.py:44, :55).
 *
 * Device pointers are caller-owned and never freed by the library.  Calls
 * are asynchronous on `stream` (NULL = legacy default stream) unless the
 * name ends in _host.  Table entries are `table_bytes` wide (2 or 4):
 * the host narrows SBox.table (uint32, sbox.py:64) to uint16 when m <= 16.
 *
 * Return codes: 0 = ok, < 0 = error; sbw_last_error() gives the message of
 * the last failing call on the calling thread.
 */
#ifndef SBW_H_
#define SBW_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SBW_ABI_VERSION 1

#define SBW_OK 0
#define SBW_EINVAL -1  /* ValueError in the reference (walsh.py:86-87, :216-217) */
#define SBW_ECUDA -2   /* CUDA runtime failure (no reference analogue)          */
#define SBW_EPARITY -3 /* AssertionError: odd spectrum gap (walsh.py:110-113)   */
#define SBW_ERANGE -4  /* IndexError: mask / input out of range (walsh.py:63-66) */

#define SBW_LAYOUT_MASK_MAJOR 0 /* out[(v - v_lo) * ld + u]  (WalshSpectrum.rows, walsh.py:32-44) */
#define SBW_LAYOUT_X_MAJOR 1    /* out[u * ld + (v - v_lo)]  (build_polarity_xmajor, walsh.py:117-131) */

/* Element types of sbw_fwht_inplace_strided (numpy dtypes of the column). */
#define SBW_ELEM_I8 1
#define SBW_ELEM_U8 2
#define SBW_ELEM_I16 3
#define SBW_ELEM_U16 4
#define SBW_ELEM_I32 5
#define SBW_ELEM_U32 6
#define SBW_ELEM_I64 7
#define SBW_ELEM_U64 8

typedef struct sbw_device_info {
  int device;
  int sm_count;
  int cc_major;
  int cc_minor;
  int64_t smem_optin_bytes;
  int64_t l2_bytes;
  int64_t global_mem_bytes;
  char name[128];
} sbw_device_info_t;

int sbw_abi_version(void);
const char* sbw_last_error(void);
int sbw_device_info(int device, sbw_device_info_t* out);
/* Number of libsbw kernels launched by this process so far. */
uint64_t sbw_launch_count(void);

/*
 * Fused component generation -> FWHT -> max|W|, spectrum never stored.
 * Replaces the stream loop of fwht_fused (walsh.py:230-244) and the worker
 * body of fwht_parallel (parallel.py:99-115): polarity_row (sbox.py:145-152)
 * + fwht_column_in_place (walsh.py:73-104) + column_nonlinearity (:107-114).
 *   d_max_abs[v - v_lo] <- max_u |W(u,v)|               (int32, device)
 *   *d_key              <- atomicMax(key) over the range (device, may be NULL;
 *                          caller initialises it, e.g. to 0)
 * n, m in 1..24.  `scratch`/`scratch_bytes` is a device workspace of at
 * least sbw_nl_scratch_bytes(n, m, v_lo, v_hi) bytes: the S-box bit planes
 * for n = 7..16, plus the multi-pass batch buffers for n >= 17.  Only when
 * that size is 0 (n <= 6) may it be NULL/0.
 *
 * Device selection (every entry point taking a stream): the call runs on
 * the stream's device, or -- for the NULL/legacy stream -- on the device
 * that owns the first device pointer argument (the table here); the
 * caller's current device is restored before returning.
 */
int sbw_nl(const void* d_table, int table_bytes, int n, int m, uint32_t v_lo, uint32_t v_hi,
           int32_t* d_max_abs, unsigned long long* d_key, void* scratch, size_t scratch_bytes,
           void* stream);
size_t sbw_nl_scratch_bytes(int n, int m, uint32_t v_lo, uint32_t v_hi);

/*
 * Materialised spectrum rows for masks [v_lo, v_hi) in either layout, plus
 * the per-component max|W| (d_max_abs may be NULL).  Replaces
 * fwht_transposed (walsh.py:183-201), fwht_rowmajor (walsh.py:155-180) and
 * fwht_fused(mode="retain") (walsh.py:220-229).  `ld` is the row pitch in
 * elements (>= 2^n for mask-major, >= v_hi - v_lo for x-major).  The x-major
 * layout needs a workspace of sbw_spectrum_scratch_bytes(...) bytes.
 */
int sbw_spectrum(const void* d_table, int table_bytes, int n, int m, uint32_t v_lo,
                 uint32_t v_hi, int layout, int32_t* d_out, int64_t ld, int32_t* d_max_abs,
                 void* scratch, size_t scratch_bytes, void* stream);
size_t sbw_spectrum_scratch_bytes(int n, int m, uint32_t v_lo, uint32_t v_hi, int layout);

/*
 * The x-major store wt[u][v - 1] (v = 1 .. 2^n - 1) of a BIJECTIVE n x n
 * S-box S, rows u in [u_lo, u_hi) (1 <= u_lo, u_hi <= 2^n) at
 * d_out + (u - u_lo) * ld, ld >= 2^n - 1 (the reference's dense pitch
 * 2^m - 1 included), computed from the inverse table T = S^-1 passed as
 * d_inv_table: W_S(u, v) = W_T(v, u), so row u is T's mask-major spectrum
 * row u without its v = 0 entry, written straight to the odd pitch (no
 * transpose, no full-size scratch).  Row u = 0 (all zeros for a bijective S)
 * is the caller's.  n = 12..16; d_out 4-byte aligned.  Replaces the x-major
 * materialisation inside fwht_rowmajor (walsh.py:155-180: build_polarity_xmajor
 * + transform_xmajor_in_place, walsh.py:117-137) for full-range bijective
 * boxes; a non-bijective table gives the x-major store of some other box
 * (the caller checks bijectivity when it builds T).
 */
int sbw_xmajor_from_inverse(const void* d_inv_table, int table_bytes, int n, uint32_t u_lo,
                            uint32_t u_hi, int32_t* d_out, int64_t ld, void* scratch,
                            size_t scratch_bytes, void* stream);
size_t sbw_xmajor_inverse_scratch_bytes(int n, uint32_t u_lo, uint32_t u_hi);

/*
 * Polarity truth table (-1)^{g_v(x)} as int32, either layout.  Replaces
 * polarity_row / polarity_truth_table (sbox.py:145-162) and
 * build_polarity_xmajor (walsh.py:117-131).  Unlike the spectrum calls the
 * range may start at v = 0 (the constant +1 row).
 */
int sbw_polarity(const void* d_table, int table_bytes, int n, int m, uint32_t v_lo,
                 uint32_t v_hi, int layout, int32_t* d_out, int64_t ld, void* stream);

/*
 * Generic in-place int32 FWHT of `count` contiguous columns of length 2^k
 * (k in 0..24), int32 wrap-around arithmetic exactly like numpy.  Replaces
 * fwht_column_in_place (walsh.py:73-104) and transform_rows_in_place
 * (walsh.py:140-152).  d_max_abs[c] (int64, may be NULL) receives the
 * column's max of numpy-int32 |x| (k >= 1) or |x| (k == 0).
 */
int sbw_fwht_inplace(int32_t* d_data, int k, int64_t count, int64_t* d_max_abs, void* stream);

/*
 * The same butterfly on any integer dtype and any strides, in place:
 * fwht_column_in_place on non-int32 / strided numpy columns (walsh.py:73-104,
 * "Accepts any uniformly strided 1-D view") and transform_xmajor_in_place
 * (walsh.py:134-137: col_stride 1, elem_stride = the x-major row pitch).
 * Column c starts at d_data + c * col_stride and its element i sits at
 * + i * elem_stride (strides in elements, may be negative).  Arithmetic wraps
 * modulo 2^(8 * sizeof(elem)) exactly as numpy's in-place ufuncs do, and
 * d_max_abs[c] (may be NULL) receives np.abs(column).max() in that dtype
 * (np.abs(MIN) == MIN for signed types; uint64 results are uint64 bits),
 * or abs(int(col[0])) as uint64 bits when k == 0.
 */
int sbw_fwht_inplace_strided(void* d_data, int elem_type, int k, int64_t count, int64_t col_stride,
                             int64_t elem_stride, int64_t* d_max_abs, void* stream);

/*
 * Per-component max|W| -> NL_v = (2^n - max|W|) >> 1 as int64 (ColumnMaxima
 * values, walsh.py:47-53 / :107-114).  *d_bad (device int64) receives the
 * smallest index with an odd gap, or stays INT64_MAX (the library
 * initialises it on `stream`).
 */
int sbw_maxabs_to_nl(const int32_t* d_max_abs, int64_t count, int n, int64_t* d_nl,
                     int64_t* d_bad, void* stream);
/* int64 variant for sbw_fwht_inplace maxima (transform_rows_in_place, walsh.py:148-152). */
int sbw_maxabs64_to_nl(const int64_t* d_max_abs, int64_t count, int64_t pw, int64_t* d_nl,
                       int64_t* d_bad, void* stream);

/*
 * Spectrum scan (nonlinearity_from_spectrum, nonlinearity.py:36-48):
 * d_row_max[r] = max(rows[r].max(), -rows[r].min()) as int64, and
 * atomicMax of the (row_max, smallest row) key into *d_key (may be NULL).
 */
int sbw_row_maxabs(const int32_t* d_rows, int64_t rows, int64_t cols, int64_t ld,
                   int64_t* d_row_max, unsigned long long* d_key, void* stream);

/* Direct evaluation W(u_i, v_i) of the defining sum (walsh_direct, walsh.py:56-70). */
int sbw_walsh_direct(const void* d_table, int table_bytes, int n, int m, const uint32_t* d_u,
                     const uint32_t* d_v, int64_t count, int32_t* d_out, void* stream);

/*
 * Affine-distance brute force (nonlinearity_bruteforce, nonlinearity.py:59-86),
 * n, m <= 8: d_best[v - 1] = min over affine functions of the Hamming
 * distance to g_v, for v in [1, 2^m).
 */
int sbw_nl_bruteforce(const void* d_table, int table_bytes, int n, int m, int32_t* d_best,
                      void* stream);

/*
 * Host-buffer end-to-end call (what a plugin binding makes): copies the
 * uint32 table host->device, runs sbw_nl over [v_lo, v_hi) on `device`,
 * copies per-component NL (int64) device->host and returns
 * out3 = {NL value, argmin_v, max|W|}.  Synchronous.  Page-locked h_table /
 * h_nl (cudaHostRegister, cudaMallocHost) are DMA'd directly; pageable ones
 * are staged through an internal pinned buffer.  The caller's current device
 * is restored on return.
 */
int sbw_nl_host(const uint32_t* h_table, int n, int m, uint32_t v_lo, uint32_t v_hi,
                int64_t* h_nl, int64_t* out3, int device);

/*
 * INT32 ALU peak microbenchmark on the current device: independent
 * add/sub chains (IADD3 on the ALU pipe mixed with IMAD on the FMA pipe).
 * Writes lane-ops per second and the kernel time.
 */
int sbw_int32_peak(double* ops_per_s, double* ms, void* stream);

/*
 * Dense int8 tensor-core peak microbenchmark on the current device: one CTA
 * per SM issues back-to-back tcgen05.mma.kind::i8 (M=128, N=256, K=32, s32
 * accumulators in TMEM) from shared-memory operands.  Writes int8 ops per
 * second (2 per multiply-add) and the kernel time.
 */
int sbw_int8_mma_peak(double* ops_per_s, double* ms, void* stream);

/*
 * Multi-GPU exchange over peer memory (NVLink), no collective library on the
 * data path.  Replaces the all-reduce / all-gather of the per-worker results
 * in fwht_parallel (parallel.py:118-126) when the workers are processes on
 * different GPUs: the root allocates the result buffers with sbw_ipc_alloc,
 * the other ranks map them with sbw_ipc_open, and every rank's sbw_nl writes
 * its component maxima straight into the root's array (d_max_abs = the mapped
 * pointer + (v_lo - 1)); sbw_key_merge then folds the rank's key into the
 * root's with one system-scope atomicMax.
 *   sbw_ipc_alloc: cudaMalloc(bytes) zeroed on the current device + its
 *                  64-byte cudaIpcMemHandle in handle_out.
 *   sbw_ipc_open:  map a handle from another process (any device with peer
 *                  access to the owner, or the owner's device itself).
 *   sbw_ipc_close / sbw_ipc_free: unmap / free.
 */
int sbw_ipc_alloc(size_t bytes, void** d_ptr_out, void* handle_out);
int sbw_ipc_open(const void* handle, void** d_ptr_out);
int sbw_ipc_close(void* d_ptr);
int sbw_ipc_free(void* d_ptr);
int sbw_key_merge(const unsigned long long* d_key, unsigned long long* d_dst_key, void* stream);
/* Copy `bytes` between any two device (or mapped peer) addresses, async on `stream`. */
int sbw_peer_copy(void* d_dst, const void* d_src, size_t bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SBW_H_ */
