// Integer pipe throughput on B200: independent chains of one opcode class,
// 2 or 8 warps per SM sub-partition.  Reports warp-instructions / clk / SM.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pipe_probe pipe_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

template <int MODE>
__global__ void k(int iters, uint32_t* out, unsigned long long* cyc) {
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = threadIdx.x * (i + 3) + i;
  const uint32_t c1 = out[1023] | 0x10001u, c2 = out[1022] | 0x20002u;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      uint32_t x = r[i];
      if (MODE == 0) asm volatile("add.u32 %0, %0, %1;" : "+r"(x) : "r"(c1));                    // IADD3 or IMAD.IADD
      if (MODE == 1) asm volatile("sub.u32 %0, %0, %1;\n\tadd.u32 %0, %0, 0x200020;" : "+r"(x) : "r"(c2));  // IADD3 3-input
      if (MODE == 2) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x) : "r"(c1), "r"(c2));     // IMAD
      if (MODE == 3) asm volatile("xor.b32 %0, %0, %1;" : "+r"(x) : "r"(c1));                    // LOP3
      if (MODE == 4) asm volatile("sub.u32 %0, %0, %1;" : "+r"(x) : "r"(c1));                    // 2-input sub
      r[i] = x;
    }
    if (MODE == 5) {  // butterfly network, bias-free: 8 pairs per iteration
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t a = r[i], b = r[i + 8];
        uint32_t s_, d_;
        asm volatile("add.u32 %0, %1, %2;" : "=r"(s_) : "r"(a), "r"(b));
        asm volatile("sub.u32 %0, %1, %2;" : "=r"(d_) : "r"(a), "r"(b));
        r[i] = s_;
        r[i + 8] = d_;
      }
    }
    if (MODE == 6) {  // butterfly, biased diff
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t a = r[i], b = r[i + 8];
        uint32_t s_, d_;
        asm volatile("add.u32 %0, %1, %2;" : "=r"(s_) : "r"(a), "r"(b));
        asm volatile("{.reg .u32 t; sub.u32 t, %1, %2; add.u32 %0, t, 0x2000200;}" : "=r"(d_) : "r"(a), "r"(b));
        r[i] = s_;
        r[i + 8] = d_;
      }
    }
    if (MODE == 7) {  // vimax3 u16x2 fold
#pragma unroll
      for (int i = 0; i < 8; ++i) r[i] = __vimax3_u16x2(r[i], r[i + 8], c1);
    }
  }
  const unsigned long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  uint32_t* out; unsigned long long* cyc;
  CK(cudaMalloc(&out, 64 << 20)); CK(cudaMemset(out, 0, 64 << 20));
  CK(cudaMalloc(&cyc, 8 * 4096));
  unsigned long long h[4096];
  const char* names[] = {"add.u32", "sub+add(imm)", "mad.lo", "xor", "sub.u32", "bfly", "bfly+bias", "vimax3"};
  for (int mode = 0; mode < 8; ++mode)
    for (int warps : {8, 16, 32}) {
      const int iters = 2048;
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k<0><<<148, warps * 32>>>(iters, out, cyc);
        if (mode == 1) k<1><<<148, warps * 32>>>(iters, out, cyc);
        if (mode == 2) k<2><<<148, warps * 32>>>(iters, out, cyc);
        if (mode == 3) k<3><<<148, warps * 32>>>(iters, out, cyc);
        if (mode == 4) k<4><<<148, warps * 32>>>(iters, out, cyc);
        if (mode == 5) k<5><<<148, warps * 32>>>(iters, out, cyc);
        if (mode == 6) k<6><<<148, warps * 32>>>(iters, out, cyc);
        if (mode == 7) k<7><<<148, warps * 32>>>(iters, out, cyc);
        CK(cudaDeviceSynchronize());
      }
      CK(cudaMemcpy(h, cyc, 8 * 148, cudaMemcpyDeviceToHost));
      double avg = 0; for (int i = 0; i < 148; ++i) avg += double(h[i]) / 148;
      const double per = (mode == 1 ? 1.0 : (mode == 7 ? 0.5 : 1.0));
      printf("%-14s warps/SM=%2d: %.2f warp-instr/clk/SM\n", names[mode], warps, per * warps * iters * 16 / avg);
    }
  return 0;
}
