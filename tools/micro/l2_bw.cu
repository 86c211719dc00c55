// Per-SM L2 bandwidth probe: `ctas` CTAs (one per SM) of 256 threads stream
// STG.128 (write) or LDG.128 (read) over a buffer of `mib` MiB (L2-resident
// when small), `reps` passes; prints aggregate and per-SM GB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_bw l2_bw.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k_write(uint4* buf, size_t n16, int reps) {
  const size_t per = n16 / gridDim.x;
  uint4* p = buf + per * blockIdx.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = threadIdx.x; i < per; i += blockDim.x) p[i] = make_uint4(r, i, 1, 2);
}
__global__ void k_read(const uint4* buf, size_t n16, int reps, unsigned* sink) {
  const size_t per = n16 / gridDim.x;
  const uint4* p = buf + per * blockIdx.x;
  unsigned acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = threadIdx.x; i < per; i += blockDim.x) {
      uint4 v = __ldcg(p + i);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  if (acc == 0x12345u) sink[0] = acc;
}

int main(int argc, char** argv) {
  const int mib = argc > 1 ? atoi(argv[1]) : 32;
  const size_t bytes = size_t(mib) << 20, n16 = bytes / 16;
  uint4* buf;
  unsigned* sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 0, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int ctas_list[] = {8, 16, 32, 64, 96, 148};
  for (int threads : {256, 1024})
    for (int ctas : ctas_list) {
      const int reps = 20;
      for (int mode = 0; mode < 2; ++mode) {
        auto run = [&]() {
          if (mode == 0) k_write<<<ctas, threads>>>(buf, n16, reps);
          else k_read<<<ctas, threads>>>(buf, n16, reps, sink);
        };
        run();
        cudaEventRecord(e0);
        run();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double gbs = double(bytes / ctas * ctas) * reps / (ms * 1e-3) / 1e9;
        printf("%s %4d thr %3d CTAs, %d MiB: %8.1f GB/s total, %6.1f GB/s per SM\n", mode ? "read " : "write", threads,
               ctas, mib, gbs, gbs / ctas);
      }
    }
  return 0;
}
