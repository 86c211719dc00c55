// DSMEM read-bandwidth probe: clusters of C CTAs (1 per SM, 128 KiB smem
// each); every CTA repeatedly reads the shared tiles of all other CTAs in its
// cluster (coalesced 32-bit loads, like the planned pass B).
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(1024, 1) k_dsmem(int reps, uint32_t* sink) {
  extern __shared__ uint32_t sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int C = cl.num_blocks(), r = cl.block_rank();
  for (int i = threadIdx.x; i < 32768; i += blockDim.x) sm[i] = i * 2654435761u + r;
  cl.sync();
  uint32_t acc = 0;
  for (int it = 0; it < reps; ++it) {
    // each thread: 32 words, rows spread over the cluster (remote-heavy, like pass B)
    for (int k = 0; k < 32; ++k) {
      const int src = (r + 1 + k) % C;
      const uint32_t* rem = cl.map_shared_rank(sm, src);
      acc += rem[((k * 1024) + threadIdx.x + it * 97) & 32767];
    }
  }
  cl.sync();
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  uint32_t* sink;
  cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int C : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = 131072;
    int maxc = 0;
    cfg.gridDim = dim3(C);
    cudaOccupancyMaxActiveClusters(&maxc, k_dsmem, &cfg);
    cfg.gridDim = dim3(maxc * C);
    int reps = 200;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, k_dsmem, reps, sink);
    cudaEventRecord(e0);
    cudaLaunchKernelEx(&cfg, k_dsmem, reps, sink);
    cudaEventRecord(e1);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    double bytes = double(maxc) * C * 1024.0 * 32 * 4 * reps;
    printf("cluster %2d: max active clusters %d (%d SMs)  %s  %.3f ms  %.1f GB/s total  %.1f B/clk/SM @1.95GHz\n",
           C, maxc, maxc * C, cudaGetErrorString(err), ms, bytes / ms / 1e6,
           bytes / (ms * 1e-3) / (maxc * C) / 1.95e9);
  }
  return 0;
}
