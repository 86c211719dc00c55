// Which runtime calls invalidate a stream capture on this driver (development probe).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k() {}
static void probe(const char* name, int which, void* ptr) {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
  cudaError_t e = cudaSuccess;
  int dev = -1;
  cudaPointerAttributes at{};
  if (which == 0) e = cudaStreamGetDevice(st, &dev);
  if (which == 1) e = cudaPointerGetAttributes(&at, ptr);
  if (which == 2) e = cudaGetDevice(&dev);
  k<<<1, 1, 0, st>>>();
  cudaError_t le = cudaGetLastError();
  cudaGraph_t g;
  cudaError_t ee = cudaStreamEndCapture(st, &g);
  printf("%-28s call=%s launch=%s end=%s\n", name, cudaGetErrorName(e), cudaGetErrorName(le), cudaGetErrorName(ee));
  cudaGetLastError();
  cudaStreamDestroy(st);
}
int main() {
  void* p;
  cudaMalloc(&p, 256);
  probe("cudaStreamGetDevice", 0, p);
  probe("cudaPointerGetAttributes", 1, p);
  probe("cudaGetDevice", 2, p);
  return 0;
}
