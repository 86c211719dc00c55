// Integer pipe rates on B200, SASS-verified opcode classes.  Each mode runs
// 16 independent dependency chains per thread (plenty of ILP) with 8 warps per
// SM (2 per sub-partition, like the tensor-core kernel) and with 32 warps.
// Reports warp-instructions per clock per SM of the named opcode.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o pipe_probe2 pipe_probe2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(int iters, const uint32_t* in, uint32_t* out, unsigned long long* cyc) {
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = in[threadIdx.x + i];
  const uint32_t a = in[100], b = in[101];
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t n[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint32_t x = r[i], y = r[(i + 1) & 15], z = r[(i + 5) & 15];
      uint32_t o;
      // one instruction of the class per element; operands from other chains
      if (MODE == 0) o = x + y + z;                       // IADD3 (3 regs)
      if (MODE == 1) o = x + y;                           // 2-input add
      if (MODE == 2) o = (x ^ y) & z;                     // LOP3
      if (MODE == 3) o = __funnelshift_r(x, y, z);        // SHF
      if (MODE == 4) o = __vimax3_u16x2(x, y, z);         // VIMNMX3
      if (MODE == 5) o = x * y + z;                       // IMAD
      if (MODE == 6) o = __byte_perm(x, y, z);            // PRMT
      if (MODE == 7) o = (i & 1) ? x + y + z : x + y;     // IADD3 / 2-input add 50:50
      if (MODE == 8) o = (i & 1) ? x - y + 0x02000200u : x + y;  // butterfly-like mix
      if (MODE == 9) o = (i & 1) ? x - y : x + y;                // bias-free butterfly
      if (MODE == 10) o = x - y;                                // 2-input sub
      n[i] = o;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) r[i] = n[i];
  }
  const unsigned long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= r[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  uint32_t *in, *out;
  unsigned long long* cyc;
  cudaMalloc(&in, 1 << 20);
  cudaMemset(in, 0x5a, 1 << 20);
  cudaMalloc(&out, 64 << 20);
  cudaMalloc(&cyc, 8 * 4096);
  unsigned long long h[4096];
  const char* names[] = {"IADD3 (3 reg)", "add 2-input", "LOP3", "SHF", "VIMNMX3.U16x2", "IMAD", "PRMT", "IADD3/add 50:50", "x-y+imm / x+y", "x-y / x+y", "sub 2-input"};
  for (int mode = 0; mode < 11; ++mode)
    for (int warps : {8, 32}) {
      const int iters = 2048;
      for (int rep = 0; rep < 2; ++rep) {
        switch (mode) {
          case 0: k<0><<<148, warps * 32>>>(iters, in, out, cyc); break;
          case 1: k<1><<<148, warps * 32>>>(iters, in, out, cyc); break;
          case 2: k<2><<<148, warps * 32>>>(iters, in, out, cyc); break;
          case 3: k<3><<<148, warps * 32>>>(iters, in, out, cyc); break;
          case 4: k<4><<<148, warps * 32>>>(iters, in, out, cyc); break;
          case 5: k<5><<<148, warps * 32>>>(iters, in, out, cyc); break;
          case 6: k<6><<<148, warps * 32>>>(iters, in, out, cyc); break;
          case 7: k<7><<<148, warps * 32>>>(iters, in, out, cyc); break;
          case 8: k<8><<<148, warps * 32>>>(iters, in, out, cyc); break;
          case 9: k<9><<<148, warps * 32>>>(iters, in, out, cyc); break;
          case 10: k<10><<<148, warps * 32>>>(iters, in, out, cyc); break;
        }
        cudaDeviceSynchronize();
      }
      cudaMemcpy(h, cyc, 8 * 148, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += double(h[i]) / 148;
      printf("%-16s warps/SM=%2d: %.2f warp-instr/clk/SM\n", names[mode], warps, double(warps) * iters * 16 / avg);
    }
  return 0;
}
