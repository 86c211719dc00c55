// Strided, any-integer-dtype in-place FWHT: the general form of
// fwht_column_in_place (walsh.py:73-104) and transform_xmajor_in_place
// (walsh.py:134-137).
//
// The reference's butterfly runs numpy ufuncs on whatever integer dtype the
// caller's column has, so its arithmetic wraps modulo 2^(8*sizeof(T)) and
// its max is np.abs(...).max() in that dtype (np.abs(INT_MIN) == INT_MIN).
// This kernel does the same arithmetic on the caller's dtype in place: the
// adds/subtracts run on the unsigned type of the same width (well-defined
// wrap-around), and the last pass folds numpy's |.| into one max per
// column.  Columns live at base + c * col_stride, element i of a column at
// + i * elem_stride (both in elements), so one kernel serves contiguous
// mask-major rows, x-major stores (col_stride 1, elem_stride = row pitch)
// and arbitrary numpy views.  The int32 contiguous case keeps its
// shared-memory tile kernel (sbw_misc.cu); this one handles the rest.
#include <climits>
#include <cstdint>
#include <type_traits>

#include "sbw_internal.cuh"
#include "sbw_launch.h"

namespace sbw {

namespace {

// numpy's np.abs(x) in dtype T, widened to the 64-bit fold type
// (signed T: long long, MIN stays negative; unsigned T: the value).
template <typename T>
__device__ __forceinline__ long long np_abs_fold(T x) {
  if constexpr (std::is_signed<T>::value) {
    using U = typename std::make_unsigned<T>::type;
    const T a = x < 0 ? T(U(0) - U(x)) : x;
    return (long long)a;
  } else {
    return (long long)(unsigned long long)x;
  }
}

template <typename T, int NB>
__global__ void __launch_bounds__(256) k_inplace_gen(T* __restrict__ base, int k, int b0, int64_t count,
                                                     int64_t col_stride, int64_t elem_stride, int col_fast,
                                                     long long* max_abs) {
  using U = typename std::make_unsigned<T>::type;
  constexpr int L = 1 << NB;
  const int64_t per_col = int64_t(1) << (k - NB);
  const int64_t total = count * per_col;
  const int64_t lo_mask = (int64_t(1) << b0) - 1;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += int64_t(gridDim.x) * blockDim.x) {
    int64_t col, r;
    if (col_fast) {  // neighbouring threads -> neighbouring columns (x-major: coalesced)
      col = t % count;
      r = t / count;
    } else {         // neighbouring threads -> neighbouring elements of one column
      col = t / per_col;
      r = t - col * per_col;
    }
    const int64_t e0 = ((r >> b0) << (b0 + NB)) + (r & lo_mask);
    T* p = base + col * col_stride + e0 * elem_stride;
    const int64_t step = (int64_t(1) << b0) * elem_stride;
    U e[L];
#pragma unroll
    for (int i = 0; i < L; ++i) e[i] = U(p[i * step]);
#pragma unroll
    for (int s = 1; s < L; s <<= 1)
#pragma unroll
      for (int i = 0; i < L; ++i)
        if ((i & s) == 0) {
          const U a = e[i], b = e[i + s];
          e[i] = U(a + b);
          e[i + s] = U(a - b);
        }
    constexpr bool kU64 = std::is_same<T, uint64_t>::value;
    long long mx = LLONG_MIN;   // signed fold (every T but uint64)
    unsigned long long umx = 0;  // uint64 fold
#pragma unroll
    for (int i = 0; i < L; ++i) {
      p[i * step] = T(e[i]);
      if constexpr (kU64) {
        umx = (unsigned long long)e[i] > umx ? (unsigned long long)e[i] : umx;
      } else {
        const long long f = np_abs_fold<T>(T(e[i]));
        mx = f > mx ? f : mx;
      }
    }
    if (max_abs) {
      if constexpr (kU64)
        atomicMax(reinterpret_cast<unsigned long long*>(max_abs) + col, umx);
      else
        atomicMax(max_abs + col, mx);
    }
  }
}

// length-1 columns: the reference returns abs(int(col[0])) as a Python int
// (walsh.py:88-89), the true absolute value, written as uint64 bits.
template <typename T>
__global__ void k_len1_gen(const T* base, int64_t count, int64_t col_stride, long long* max_abs) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    const T x = base[i * col_stride];
    unsigned long long a;
    if constexpr (std::is_signed<T>::value)
      a = x < 0 ? 0ull - (unsigned long long)(long long)x : (unsigned long long)x;
    else
      a = (unsigned long long)x;
    max_abs[i] = (long long)a;
  }
}

template <typename T>
__global__ void k_init_gen(long long* p, int64_t count) {
  const long long v = std::is_same<T, uint64_t>::value ? 0 : LLONG_MIN;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = v;
}

int grid_cap(int64_t work) {
  DeviceProps dp;
  if (device_props(&dp)) return 1;
  int64_t g = (work + 255) / 256;
  const int64_t cap = int64_t(dp.sm_count) * 8;
  return int(g < 1 ? 1 : (g > cap ? cap : g));
}

template <typename T>
int run_gen(void* data, int k, int64_t count, int64_t col_stride, int64_t elem_stride,
            long long* max_abs, cudaStream_t st) {
  T* d = static_cast<T*>(data);
  if (k == 0) {
    if (max_abs) {
      k_len1_gen<T><<<grid_cap(count), 256, 0, st>>>(d, count, col_stride, max_abs);
      SBW_LAUNCH_CHECK("k_len1_gen");
    }
    return SBW_OK;
  }
  if (max_abs) {
    k_init_gen<T><<<grid_cap(count), 256, 0, st>>>(max_abs, count);
    SBW_LAUNCH_CHECK("k_init_gen");
  }
  // the unit-stride dimension varies fastest across threads
  const int col_fast = (col_stride == 1 && elem_stride != 1) ? 1 : 0;
  int b0 = 0;
  while (b0 < k) {
    constexpr int kMaxNb = sizeof(T) == 8 ? 4 : 6;  // 2^NB elements in registers (64-bit: no spills)
    const int nb = (k - b0) < kMaxNb ? (k - b0) : kMaxNb;
    long long* mx = (b0 + nb == k) ? max_abs : nullptr;
    const int grid = grid_cap(count << (k - nb));
    switch (nb) {
      case 1: k_inplace_gen<T, 1><<<grid, 256, 0, st>>>(d, k, b0, count, col_stride, elem_stride, col_fast, mx); break;
      case 2: k_inplace_gen<T, 2><<<grid, 256, 0, st>>>(d, k, b0, count, col_stride, elem_stride, col_fast, mx); break;
      case 3: k_inplace_gen<T, 3><<<grid, 256, 0, st>>>(d, k, b0, count, col_stride, elem_stride, col_fast, mx); break;
      case 4: k_inplace_gen<T, 4><<<grid, 256, 0, st>>>(d, k, b0, count, col_stride, elem_stride, col_fast, mx); break;
      case 5: k_inplace_gen<T, 5><<<grid, 256, 0, st>>>(d, k, b0, count, col_stride, elem_stride, col_fast, mx); break;
      default:
        if constexpr (kMaxNb >= 6)
          k_inplace_gen<T, 6><<<grid, 256, 0, st>>>(d, k, b0, count, col_stride, elem_stride, col_fast, mx);
        break;
    }
    SBW_LAUNCH_CHECK("k_inplace_gen");
    b0 += nb;
  }
  return SBW_OK;
}

}  // namespace

int inplace_fwht_strided(void* data, int elem, int k, int64_t count, int64_t col_stride,
                         int64_t elem_stride, long long* max_abs, cudaStream_t st) {
  if (count <= 0) return SBW_OK;
  switch (elem) {
    case SBW_ELEM_I8: return run_gen<int8_t>(data, k, count, col_stride, elem_stride, max_abs, st);
    case SBW_ELEM_U8: return run_gen<uint8_t>(data, k, count, col_stride, elem_stride, max_abs, st);
    case SBW_ELEM_I16: return run_gen<int16_t>(data, k, count, col_stride, elem_stride, max_abs, st);
    case SBW_ELEM_U16: return run_gen<uint16_t>(data, k, count, col_stride, elem_stride, max_abs, st);
    case SBW_ELEM_I32: return run_gen<int32_t>(data, k, count, col_stride, elem_stride, max_abs, st);
    case SBW_ELEM_U32: return run_gen<uint32_t>(data, k, count, col_stride, elem_stride, max_abs, st);
    case SBW_ELEM_I64: return run_gen<int64_t>(data, k, count, col_stride, elem_stride, max_abs, st);
    case SBW_ELEM_U64: return run_gen<uint64_t>(data, k, count, col_stride, elem_stride, max_abs, st);
    default: return set_error(SBW_EINVAL, "unknown element type %d", elem);
  }
}

}  // namespace sbw
