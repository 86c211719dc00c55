// HBM write rate of the spectrum epilogue's store pattern vs wider stores:
// 148 CTAs x 256 threads; every CTA writes consecutive 256 KiB "items" (one
// 2^16 int32 spectrum row each), thread t owning u_r = t and looping over the
// 256 u_c (address u_c * 256 + u_r): mode 0 = STG.32 (st.global.cs, the
// shipped K2 SPEC epilogue), mode 1 = STG.32 plain, mode 2 = STG.128 over the
// same 256 KiB (thread t writes 16 consecutive bytes per step), mode 3 =
// STG.128 .cs.  Prints GB/s over `gib` GiB.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stg_width stg_width.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) k(int* out, long items_per_cta) {
  const int t = threadIdx.x;
  for (long it = 0; it < items_per_cta; ++it) {
    int* row = out + ((long)blockIdx.x * items_per_cta + it) * 65536;
    if (MODE <= 1) {
#pragma unroll 8
      for (int c = 0; c < 256; ++c) {
        if (MODE == 0) __stcs(row + c * 256 + t, c ^ t);
        else row[c * 256 + t] = c ^ t;
      }
    } else {
      int4* r4 = reinterpret_cast<int4*>(row);
#pragma unroll 8
      for (int c = 0; c < 64; ++c) {
        int4 v = make_int4(c, t, c ^ t, 1);
        if (MODE == 3) __stcs(r4 + c * 256 + t, v);
        else r4[c * 256 + t] = v;
      }
    }
  }
}

int main(int argc, char** argv) {
  const int gib = argc > 1 ? atoi(argv[1]) : 4;
  const long items = (long(gib) << 30) / (65536L * 4) / 148;
  int* buf;
  cudaMalloc(&buf, size_t(items) * 148 * 65536 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 4; ++mode)
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<148, 256>>>(buf, items);
      if (mode == 1) k<1><<<148, 256>>>(buf, items);
      if (mode == 2) k<2><<<148, 256>>>(buf, items);
      if (mode == 3) k<3><<<148, 256>>>(buf, items);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("mode %d (%s): %.3f ms, %.0f GB/s\n", mode,
                      mode == 0 ? "STG.32 .cs" : mode == 1 ? "STG.32" : mode == 2 ? "STG.128" : "STG.128 .cs", ms,
                      double(items) * 148 * 65536 * 4 / (ms * 1e-3) / 1e9);
    }
  return 0;
}
