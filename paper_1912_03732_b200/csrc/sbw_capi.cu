// extern "C" boundary of libsbw (declared in include/sbw.h).
//
// Argument validation mirrors the reference's exceptions: n, m in 1..24
// (sbox.py:18, :60-63), mask ranges within [1, 2^m) (sbox.py:155-159),
// power-of-two columns (walsh.py:86-87).  Budget checks (memory.py:66-68) stay
// in the host package, before any launch.
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>

#include "sbw_internal.cuh"
#include "sbw_launch.h"

namespace sbw {

namespace {
thread_local char g_err[512] = "";
std::atomic<uint64_t> g_launches{0};

struct PropsCache {
  std::mutex mu;
  bool valid[64] = {};
  DeviceProps p[64];
} g_props;
}  // namespace

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_error(cudaError_t e, const char* what) {
  return set_error(SBW_ECUDA, "CUDA error %s (%s) in %s", cudaGetErrorName(e),
                   cudaGetErrorString(e), what);
}

void count_launch(uint64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

int device_props(DeviceProps* out) {
  int dev = 0;
  SBW_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return set_error(SBW_EINVAL, "device index %d unsupported", dev);
  std::lock_guard<std::mutex> lk(g_props.mu);
  if (!g_props.valid[dev]) {
    DeviceProps p{};
    p.device = dev;
    int v = 0;
    SBW_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    p.sm_count = v;
    SBW_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    p.smem_optin = size_t(v);
    SBW_CUDA_CHECK(cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev));
    p.l2_bytes = size_t(v);
    g_props.p[dev] = p;
    g_props.valid[dev] = true;
  }
  *out = g_props.p[dev];
  return SBW_OK;
}

}  // namespace sbw

using namespace sbw;

namespace {

int check_nm(int n, int m) {
  if (n < 1 || n > 24) return set_error(SBW_EINVAL, "n must be in 1..24, got %d", n);
  if (m < 1 || m > 24) return set_error(SBW_EINVAL, "m must be in 1..24, got %d", m);
  return SBW_OK;
}

int check_table(const void* t, int tbytes, int m) {
  if (t == nullptr) return set_error(SBW_EINVAL, "null table pointer");
  if (tbytes != 2 && tbytes != 4)
    return set_error(SBW_EINVAL, "table entries must be 2 or 4 bytes, got %d", tbytes);
  if (tbytes == 2 && m > 16)
    return set_error(SBW_EINVAL, "m = %d needs a 4-byte table", m);
  if ((reinterpret_cast<uintptr_t>(t) & 15u) != 0)
    return set_error(SBW_EINVAL, "table pointer must be 16-byte aligned");
  return SBW_OK;
}

int check_range(int m, uint32_t v_lo, uint32_t v_hi) {
  const uint64_t top = uint64_t(1) << m;
  if (v_lo < 1 || v_lo > v_hi || uint64_t(v_hi) > top)
    return set_error(SBW_ERANGE, "mask range [%u, %u) outside [1, %llu)", v_lo, v_hi,
                     (unsigned long long)top);
  return SBW_OK;
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Every entry point runs on the device that owns its work: the stream's
// device (cudaStreamGetDevice) for a created stream, else (NULL / legacy
// stream, or a stream being captured into a CUDA graph) the device of the
// data pointer (the NULL stream belongs to whatever device is current, which
// need not be where the caller's buffers live).  The caller's
// current device is restored on return, and the per-device caches inside
// libsbw (device_props, tensor-core constants, K3 streams) key off the
// device selected here.
class DeviceScope {
 public:
  DeviceScope(void* stream, const void* ptr) {
    int want = -1;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (st != nullptr && st != cudaStreamLegacy && st != cudaStreamPerThread) {
      // cudaStreamGetDevice is not allowed while the stream is being
      // captured into a CUDA graph (it invalidates the capture); a capturing
      // caller gets the pointer's device below
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone) {
        if (cudaStreamGetDevice(st, &want) != cudaSuccess) {
          cudaGetLastError();
          want = -1;
        }
      } else {
        cudaGetLastError();
      }
    }
    if (want < 0 && ptr != nullptr) {
      cudaPointerAttributes at{};
      if (cudaPointerGetAttributes(&at, ptr) == cudaSuccess &&
          (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged))
        want = at.device;
      else
        cudaGetLastError();
    }
    if (want >= 0 && cudaGetDevice(&prev_) == cudaSuccess && prev_ != want) {
      if (cudaSetDevice(want) == cudaSuccess) switched_ = true;
      else cudaGetLastError();
    }
  }
  ~DeviceScope() {
    if (switched_) cudaSetDevice(prev_);
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;

 private:
  int prev_ = -1;
  bool switched_ = false;
};

// Restores the caller's current device (sbw_nl_host selects `device` itself).
class DeviceRestore {
 public:
  DeviceRestore() {
    if (cudaGetDevice(&prev_) != cudaSuccess) prev_ = -1;
  }
  ~DeviceRestore() {
    if (prev_ >= 0) cudaSetDevice(prev_);
  }

 private:
  int prev_ = -1;
};

}  // namespace

extern "C" {

int sbw_abi_version(void) { return SBW_ABI_VERSION; }

const char* sbw_last_error(void) { return g_err; }

uint64_t sbw_launch_count(void) { return g_launches.load(); }

int sbw_device_info(int device, sbw_device_info_t* out) {
  if (!out) return set_error(SBW_EINVAL, "null output");
  cudaDeviceProp p;
  SBW_CUDA_CHECK(cudaGetDeviceProperties(&p, device));
  memset(out, 0, sizeof(*out));
  out->device = device;
  out->sm_count = p.multiProcessorCount;
  out->cc_major = p.major;
  out->cc_minor = p.minor;
  out->smem_optin_bytes = int64_t(p.sharedMemPerBlockOptin);
  out->l2_bytes = int64_t(p.l2CacheSize);
  out->global_mem_bytes = int64_t(p.totalGlobalMem);
  snprintf(out->name, sizeof(out->name), "%.127s", p.name);
  return SBW_OK;
}

size_t sbw_nl_scratch_bytes(int n, int m, uint32_t v_lo, uint32_t v_hi) {
  return nl_scratch_bytes(n, m, v_lo, v_hi);
}

int sbw_nl(const void* d_table, int table_bytes, int n, int m, uint32_t v_lo, uint32_t v_hi,
           int32_t* d_max_abs, unsigned long long* d_key, void* scratch, size_t scratch_bytes,
           void* stream) {
  DeviceScope dev_scope(stream, d_table);
  if (int rc = check_nm(n, m)) return rc;
  if (int rc = check_table(d_table, table_bytes, m)) return rc;
  if (int rc = check_range(m, v_lo, v_hi)) return rc;
  if (!d_max_abs) return set_error(SBW_EINVAL, "null max_abs output");
  const size_t need = nl_scratch_bytes(n, m, v_lo, v_hi);
  if (need && (scratch == nullptr || scratch_bytes < need))
    return set_error(SBW_EINVAL, "sbw_nl(n=%d, m=%d) needs %zu scratch bytes, got %zu", n, m, need,
                     scratch_bytes);
  if (n <= 16)
    return launch_fused_onchip(d_table, table_bytes, n, m, v_lo, v_hi, d_max_abs, d_key, nullptr,
                               0, scratch, as_stream(stream));
  return launch_k3(d_table, table_bytes, n, m, v_lo, v_hi, d_max_abs, d_key, nullptr, 0, scratch,
                   scratch_bytes, as_stream(stream));
}

size_t sbw_spectrum_scratch_bytes(int n, int m, uint32_t v_lo, uint32_t v_hi, int layout) {
  size_t s = nl_scratch_bytes(n, m, v_lo, v_hi);
  if (layout == SBW_LAYOUT_X_MAJOR) s += (size_t(v_hi) - v_lo) * (size_t(4) << n);
  return s;
}

int sbw_spectrum(const void* d_table, int table_bytes, int n, int m, uint32_t v_lo,
                 uint32_t v_hi, int layout, int32_t* d_out, int64_t ld, int32_t* d_max_abs,
                 void* scratch, size_t scratch_bytes, void* stream) {
  DeviceScope dev_scope(stream, d_table);
  if (int rc = check_nm(n, m)) return rc;
  if (int rc = check_table(d_table, table_bytes, m)) return rc;
  if (int rc = check_range(m, v_lo, v_hi)) return rc;
  if (!d_out) return set_error(SBW_EINVAL, "null output");
  const int64_t rows = int64_t(v_hi) - int64_t(v_lo), cols = int64_t(1) << n;
  cudaStream_t st = as_stream(stream);
  int32_t* mx = d_max_abs;
  if (rows == 0) return SBW_OK;
  if (layout != SBW_LAYOUT_MASK_MAJOR && layout != SBW_LAYOUT_X_MAJOR)
    return set_error(SBW_EINVAL, "layout must be 0 (mask-major) or 1 (x-major)");
  if (layout == SBW_LAYOUT_MASK_MAJOR && ld < cols)
    return set_error(SBW_EINVAL, "ld %lld < 2^n", (long long)ld);
  if (layout == SBW_LAYOUT_MASK_MAJOR && n >= 7 &&
      ((ld & 1) || (reinterpret_cast<uintptr_t>(d_out) & 7)))
    return set_error(SBW_EINVAL, "mask-major output needs an even ld and 8-byte alignment");
  if (layout == SBW_LAYOUT_X_MAJOR && ld < rows)
    return set_error(SBW_EINVAL, "ld %lld < number of masks", (long long)ld);
  const size_t k3 = nl_scratch_bytes(n, m, v_lo, v_hi);
  const size_t need = sbw_spectrum_scratch_bytes(n, m, v_lo, v_hi, layout);
  if (need && (scratch == nullptr || scratch_bytes < need))
    return set_error(SBW_EINVAL, "spectrum needs %zu scratch bytes, got %zu", need, scratch_bytes);
  int32_t* own_mx = nullptr;
  if (mx == nullptr) {
    SBW_CUDA_CHECK(cudaMallocAsync(&own_mx, sizeof(int32_t) * rows, st));
    mx = own_mx;
  }
  int32_t* rows_out = d_out;
  int64_t rows_ld = ld;
  if (layout == SBW_LAYOUT_X_MAJOR) {
    rows_out = reinterpret_cast<int32_t*>(static_cast<char*>(scratch) + k3);
    rows_ld = cols;
  }
  int rc;
  if (n <= 16)
    rc = launch_fused_onchip(d_table, table_bytes, n, m, v_lo, v_hi, mx, nullptr, rows_out,
                             rows_ld, scratch, st);
  else
    rc = launch_k3(d_table, table_bytes, n, m, v_lo, v_hi, mx, nullptr, rows_out, rows_ld, scratch,
                   k3, st);
  if (rc == SBW_OK && layout == SBW_LAYOUT_X_MAJOR)
    rc = launch_transpose_i32(rows_out, rows, cols, cols, d_out, ld, st);
  if (own_mx) cudaFreeAsync(own_mx, st);
  return rc;
}

size_t sbw_xmajor_inverse_scratch_bytes(int n, uint32_t u_lo, uint32_t u_hi) {
  if (n < 1 || n > 16 || u_hi < u_lo) return 0;
  return ((planes_bytes(n, n) + 255) & ~size_t(255)) + 4 * (size_t(u_hi) - u_lo);
}

int sbw_xmajor_from_inverse(const void* d_inv_table, int table_bytes, int n, uint32_t u_lo,
                            uint32_t u_hi, int32_t* d_out, int64_t ld, void* scratch,
                            size_t scratch_bytes, void* stream) {
  DeviceScope dev_scope(stream, d_inv_table);
  if (n < 12 || n > 16) return set_error(SBW_EINVAL, "x-major from the inverse needs n in 12..16, got %d", n);
  if (int rc = check_table(d_inv_table, table_bytes, n)) return rc;
  if (u_lo < 1 || u_hi < u_lo || uint64_t(u_hi) > (uint64_t(1) << n))
    return set_error(SBW_ERANGE, "row range [%u, %u) outside [1, 2^%d]", u_lo, u_hi, n);
  if (u_hi == u_lo) return SBW_OK;
  if (!d_out) return set_error(SBW_EINVAL, "null output");
  if (reinterpret_cast<uintptr_t>(d_out) & 3) return set_error(SBW_EINVAL, "output not 4-byte aligned");
  if (ld < (int64_t(1) << n) - 1) return set_error(SBW_EINVAL, "ld %lld < 2^n - 1", (long long)ld);
  const size_t need = sbw_xmajor_inverse_scratch_bytes(n, u_lo, u_hi);
  if (scratch == nullptr || scratch_bytes < need)
    return set_error(SBW_EINVAL, "x-major from the inverse needs %zu scratch bytes, got %zu", need,
                     scratch_bytes);
  cudaStream_t st = as_stream(stream);
  uint32_t* planes = static_cast<uint32_t*>(scratch);
  int32_t* mx = reinterpret_cast<int32_t*>(static_cast<char*>(scratch) +
                                           ((planes_bytes(n, n) + 255) & ~size_t(255)));
  if (int rc = build_planes(d_inv_table, table_bytes, n, n, planes, st)) return rc;
  return launch_tc_xmajor_inverse(planes, n, u_lo, u_hi, mx, d_out, ld, st);
}

int sbw_polarity(const void* d_table, int table_bytes, int n, int m, uint32_t v_lo,
                 uint32_t v_hi, int layout, int32_t* d_out, int64_t ld, void* stream) {
  DeviceScope dev_scope(stream, d_table);
  if (int rc = check_nm(n, m)) return rc;
  if (int rc = check_table(d_table, table_bytes, m)) return rc;
  // polarity rows may include the constant v = 0 row (polarity_row(s, 0))
  if (v_lo > v_hi || uint64_t(v_hi) > (uint64_t(1) << m))
    return set_error(SBW_ERANGE, "mask range [%u, %u) outside [0, 2^%d)", v_lo, v_hi, m);
  if (!d_out) return set_error(SBW_EINVAL, "null output");
  if (layout != SBW_LAYOUT_MASK_MAJOR && layout != SBW_LAYOUT_X_MAJOR)
    return set_error(SBW_EINVAL, "layout must be 0 (mask-major) or 1 (x-major)");
  return launch_polarity(d_table, table_bytes, n, v_lo, v_hi, layout, d_out, ld,
                         as_stream(stream));
}

int sbw_fwht_inplace(int32_t* d_data, int k, int64_t count, int64_t* d_max_abs, void* stream) {
  DeviceScope dev_scope(stream, d_data);
  if (k < 0 || k > 30) return set_error(SBW_EINVAL, "column length must be 2^k, k in 0..30");
  if (count < 0) return set_error(SBW_EINVAL, "negative column count");
  if (count > 0 && !d_data) return set_error(SBW_EINVAL, "null data");
  return inplace_fwht(d_data, k, count, reinterpret_cast<long long*>(d_max_abs),
                      as_stream(stream));
}

int sbw_fwht_inplace_strided(void* d_data, int elem_type, int k, int64_t count, int64_t col_stride,
                             int64_t elem_stride, int64_t* d_max_abs, void* stream) {
  DeviceScope dev_scope(stream, d_data);
  if (k < 0 || k > 30) return set_error(SBW_EINVAL, "column length must be 2^k, k in 0..30");
  if (count < 0) return set_error(SBW_EINVAL, "negative column count");
  if (elem_type < SBW_ELEM_I8 || elem_type > SBW_ELEM_U64)
    return set_error(SBW_EINVAL, "unknown element type %d", elem_type);
  if (count > 0 && !d_data) return set_error(SBW_EINVAL, "null data");
  if (k > 0 && elem_stride == 0) return set_error(SBW_EINVAL, "zero element stride");
  return inplace_fwht_strided(d_data, elem_type, k, count, col_stride, elem_stride,
                              reinterpret_cast<long long*>(d_max_abs), as_stream(stream));
}

__global__ void k_fill_ll(long long* p, long long v) { *p = v; }

int sbw_maxabs_to_nl(const int32_t* d_max_abs, int64_t count, int n, int64_t* d_nl,
                     int64_t* d_bad, void* stream) {
  DeviceScope dev_scope(stream, d_nl);
  if (n < 0 || n > 30) return set_error(SBW_EINVAL, "bad n");
  cudaStream_t st = as_stream(stream);
  k_fill_ll<<<1, 1, 0, st>>>(reinterpret_cast<long long*>(d_bad), LLONG_MAX);
  SBW_LAUNCH_CHECK("k_fill_ll");
  return launch_maxabs_to_nl(d_max_abs, count, n, reinterpret_cast<long long*>(d_nl),
                             reinterpret_cast<long long*>(d_bad), st);
}

int sbw_maxabs64_to_nl(const int64_t* d_max_abs, int64_t count, int64_t pw, int64_t* d_nl,
                       int64_t* d_bad, void* stream) {
  DeviceScope dev_scope(stream, d_nl);
  cudaStream_t st = as_stream(stream);
  k_fill_ll<<<1, 1, 0, st>>>(reinterpret_cast<long long*>(d_bad), LLONG_MAX);
  SBW_LAUNCH_CHECK("k_fill_ll");
  return launch_maxabs64_to_nl(reinterpret_cast<const long long*>(d_max_abs), count, pw,
                               reinterpret_cast<long long*>(d_nl),
                               reinterpret_cast<long long*>(d_bad), st);
}

int sbw_row_maxabs(const int32_t* d_rows, int64_t rows, int64_t cols, int64_t ld,
                   int64_t* d_row_max, unsigned long long* d_key, void* stream) {
  DeviceScope dev_scope(stream, d_rows);
  if (rows < 0 || cols < 1 || ld < cols) return set_error(SBW_EINVAL, "bad spectrum shape");
  return launch_row_maxabs(d_rows, rows, cols, ld, reinterpret_cast<long long*>(d_row_max), d_key,
                           as_stream(stream));
}

int sbw_walsh_direct(const void* d_table, int table_bytes, int n, int m, const uint32_t* d_u,
                     const uint32_t* d_v, int64_t count, int32_t* d_out, void* stream) {
  DeviceScope dev_scope(stream, d_table);
  if (int rc = check_nm(n, m)) return rc;
  if (int rc = check_table(d_table, table_bytes, m)) return rc;
  return launch_walsh_direct(d_table, table_bytes, n, d_u, d_v, count, d_out, as_stream(stream));
}

int sbw_nl_bruteforce(const void* d_table, int table_bytes, int n, int m, int32_t* d_best,
                      void* stream) {
  DeviceScope dev_scope(stream, d_table);
  if (int rc = check_nm(n, m)) return rc;
  if (n > 8 || m > 8) return set_error(SBW_EINVAL, "brute force capped at 8 bits, got %dx%d", n, m);
  if (int rc = check_table(d_table, table_bytes, m)) return rc;
  return launch_bruteforce(d_table, table_bytes, n, m, d_best, as_stream(stream));
}

namespace {
// Per-device cached workspace for the host-buffer entry point, so repeated
// calls pay only the copies and the kernels (not allocation).
struct HostCallWs {
  std::mutex mu;
  cudaStream_t st = nullptr;
  void* h_stage = nullptr;   // pinned: narrowed table in, NL out
  size_t h_bytes = 0;
  void* d_buf = nullptr;     // table | max_abs | nl | bad | key | scratch
  size_t d_bytes = 0;
};
HostCallWs g_host_ws[64];

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }
}  // namespace

int sbw_nl_host(const uint32_t* h_table, int n, int m, uint32_t v_lo, uint32_t v_hi,
                int64_t* h_nl, int64_t* out3, int device) {
  DeviceRestore dev_restore;
  if (int rc = check_nm(n, m)) return rc;
  if (int rc = check_range(m, v_lo, v_hi)) return rc;
  if (!h_table) return set_error(SBW_EINVAL, "null host table");
  if (device < 0 || device >= 64) return set_error(SBW_EINVAL, "bad device %d", device);
  SBW_CUDA_CHECK(cudaSetDevice(device));
  HostCallWs& ws = g_host_ws[device];
  std::lock_guard<std::mutex> lk(ws.mu);
  if (!ws.st) SBW_CUDA_CHECK(cudaStreamCreateWithFlags(&ws.st, cudaStreamNonBlocking));
  cudaStream_t st = ws.st;
  const int64_t nx = int64_t(1) << n, nv = int64_t(v_hi) - int64_t(v_lo);
  const int tb = m <= 16 ? 2 : 4;
  const size_t tbl = align_up(size_t(nx) * 4), mxb = align_up(sizeof(int32_t) * nv),
               nlb = align_up(sizeof(int64_t) * nv), small = 256;
  const size_t sb = nl_scratch_bytes(n, m, v_lo, v_hi);
  const size_t dneed = tbl + mxb + nlb + 2 * small + sb;
  const size_t hneed = (tbl > nlb ? tbl : nlb) + 2 * small;
  if (ws.h_bytes < hneed) {
    if (ws.h_stage) cudaFreeHost(ws.h_stage);
    ws.h_stage = nullptr;
    ws.h_bytes = 0;
    SBW_CUDA_CHECK(cudaMallocHost(&ws.h_stage, hneed));
    ws.h_bytes = hneed;
  }
  if (ws.d_bytes < dneed) {
    if (ws.d_buf) cudaFree(ws.d_buf);
    ws.d_buf = nullptr;
    ws.d_bytes = 0;
    SBW_CUDA_CHECK(cudaMalloc(&ws.d_buf, dneed));
    ws.d_bytes = dneed;
  }
  char* d = static_cast<char*>(ws.d_buf);
  void* d_table = d;
  int32_t* d_mx = reinterpret_cast<int32_t*>(d + tbl);
  int64_t* d_nl = reinterpret_cast<int64_t*>(d + tbl + mxb);
  int64_t* d_bad = reinterpret_cast<int64_t*>(d + tbl + mxb + nlb);
  unsigned long long* d_key = reinterpret_cast<unsigned long long*>(d + tbl + mxb + nlb + small);
  void* scratch = sb ? d + tbl + mxb + nlb + 2 * small : nullptr;
  char* h = static_cast<char*>(ws.h_stage);
  long long* h_bad = reinterpret_cast<long long*>(h + (tbl > nlb ? tbl : nlb));
  unsigned long long* h_key = reinterpret_cast<unsigned long long*>(h_bad + 32);
  // Page-locked caller buffers (cudaHostRegister / cudaMallocHost) are
  // copied to and from directly; pageable ones go through the pinned staging.
  auto pinned = [](const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();  // clear the sticky-free error of an unknown pointer
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  const bool tbl_pinned = pinned(h_table), nl_pinned = h_nl != nullptr && pinned(h_nl);
  int tbw = tb;
  if (tbl_pinned) {
    // uint32 straight from the caller; sbw_nl reads 4-byte tables too
    tbw = 4;
    if (size_t(nx) * 4 > tbl) return set_error(SBW_EINVAL, "table workspace too small");
    SBW_CUDA_CHECK(cudaMemcpyAsync(d_table, h_table, size_t(nx) * 4, cudaMemcpyHostToDevice, st));
  } else if (tb == 2) {
    // narrow the caller's uint32 table into pinned staging, then one H2D copy
    uint16_t* s16 = reinterpret_cast<uint16_t*>(h);
    for (int64_t i = 0; i < nx; ++i) s16[i] = uint16_t(h_table[i]);
    SBW_CUDA_CHECK(cudaMemcpyAsync(d_table, h, size_t(nx) * tb, cudaMemcpyHostToDevice, st));
  } else {
    memcpy(h, h_table, size_t(nx) * 4);
    SBW_CUDA_CHECK(cudaMemcpyAsync(d_table, h, size_t(nx) * tb, cudaMemcpyHostToDevice, st));
  }
  SBW_CUDA_CHECK(cudaMemsetAsync(d_key, 0, sizeof(unsigned long long), st));
  if (int rc = sbw_nl(d_table, tbw, n, m, v_lo, v_hi, d_mx, d_key, scratch, sb, st)) return rc;
  if (int rc = sbw_maxabs_to_nl(d_mx, nv, n, d_nl, d_bad, st)) return rc;
  // the staging buffer is reused for the results once the table copy is done
  int64_t* nl_dst = nl_pinned ? h_nl : reinterpret_cast<int64_t*>(h);
  SBW_CUDA_CHECK(cudaMemcpyAsync(nl_dst, d_nl, sizeof(int64_t) * nv, cudaMemcpyDeviceToHost, st));
  SBW_CUDA_CHECK(cudaMemcpyAsync(h_bad, d_bad, sizeof(long long), cudaMemcpyDeviceToHost, st));
  SBW_CUDA_CHECK(cudaMemcpyAsync(h_key, d_key, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  SBW_CUDA_CHECK(cudaStreamSynchronize(st));
  if (*h_bad != LLONG_MAX)
    return set_error(SBW_EPARITY, "odd spectrum gap at mask %lld", (long long)(v_lo + *h_bad));
  if (h_nl && !nl_pinned) memcpy(h_nl, h, sizeof(int64_t) * nv);
  if (out3) {
    const int64_t mxw = int64_t(*h_key >> 32);
    out3[0] = (nx - mxw) >> 1;
    out3[1] = int64_t(0xFFFFFFFFull - (*h_key & 0xFFFFFFFFull));
    out3[2] = mxw;
  }
  return SBW_OK;
}

int sbw_int32_peak(double* ops_per_s, double* ms, void* stream) {
  DeviceScope dev_scope(stream, nullptr);
  if (!ops_per_s) return set_error(SBW_EINVAL, "null output");
  return run_int32_peak(ops_per_s, ms, as_stream(stream));
}

int sbw_int8_mma_peak(double* ops_per_s, double* ms, void* stream) {
  DeviceScope dev_scope(stream, nullptr);
  if (!ops_per_s) return set_error(SBW_EINVAL, "null output");
  return run_int8_mma_peak(ops_per_s, ms, as_stream(stream));
}

int sbw_ipc_alloc(size_t bytes, void** d_ptr_out, void* handle_out) {
  if (!d_ptr_out || !handle_out || bytes == 0) return set_error(SBW_EINVAL, "sbw_ipc_alloc: bad arguments");
  void* p = nullptr;
  SBW_CUDA_CHECK(cudaMalloc(&p, bytes));
  SBW_CUDA_CHECK(cudaMemset(p, 0, bytes));
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_error(e, "cudaIpcGetMemHandle");
  }
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle_out, &h, sizeof(h));
  *d_ptr_out = p;
  return SBW_OK;
}

int sbw_ipc_open(const void* handle, void** d_ptr_out) {
  if (!handle || !d_ptr_out) return set_error(SBW_EINVAL, "sbw_ipc_open: bad arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  SBW_CUDA_CHECK(cudaIpcOpenMemHandle(d_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return SBW_OK;
}

int sbw_ipc_close(void* d_ptr) {
  SBW_CUDA_CHECK(cudaIpcCloseMemHandle(d_ptr));
  return SBW_OK;
}

int sbw_ipc_free(void* d_ptr) {
  SBW_CUDA_CHECK(cudaFree(d_ptr));
  return SBW_OK;
}

int sbw_key_merge(const unsigned long long* d_key, unsigned long long* d_dst_key, void* stream) {
  DeviceScope dev_scope(stream, d_key);
  if (!d_key || !d_dst_key) return set_error(SBW_EINVAL, "sbw_key_merge: null key");
  return launch_key_merge(d_key, d_dst_key, as_stream(stream));
}

int sbw_peer_copy(void* d_dst, const void* d_src, size_t bytes, void* stream) {
  DeviceScope dev_scope(stream, d_dst);
  if (bytes == 0) return SBW_OK;
  if (!d_dst || !d_src) return set_error(SBW_EINVAL, "sbw_peer_copy: null pointer");
  SBW_CUDA_CHECK(cudaMemcpyAsync(d_dst, d_src, bytes, cudaMemcpyDefault, as_stream(stream)));
  return SBW_OK;
}

}  // extern "C"
