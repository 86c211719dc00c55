// Probe: tcgen05.mma.kind::i8 with the A operand in TENSOR MEMORY (written by
// tcgen05.st), B in shared memory (K-major, no swizzle), D in TMEM.  Checks the
// A-in-TMEM data layout (lane = row, 4 consecutive K bytes per 32-bit column) against
// a CPU GEMM and times a chain of such MMAs against the A-in-smem form.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tc_probe_atmem tc_probe_atmem.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr & 0x3FFFFu) >> 4) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) | (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (uint64_t(1) << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool as, bool bs) {
  return (2u << 4) | (uint32_t(as) << 7) | (uint32_t(bs) << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ uint32_t kmaj_off(int row, int k, int kchunks) {  // K-major core matrices
  return uint32_t(((row >> 3) * kchunks + (k >> 4)) * 128 + (row & 7) * 16 + (k & 15));
}
// mode 0: A from TMEM, mode 1: A from smem.  K = 32 * kblocks (<= 128)
__global__ void __launch_bounds__(128) k_probe(const int8_t* A, const uint8_t* B, int32_t* D, int kblocks, int mode,
                                               int reps, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;              // 128 x 128
  uint8_t* sB = sm + 16384;      // 128 (N) x 128 (K)
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = 32 * kblocks;
  for (int i = tid; i < 128 * 128; i += 128) sA[kmaj_off(i >> 7, i & 127, 8)] = (i & 127) < K ? uint8_t(A[(i >> 7) * K + (i & 127)]) : 0;
  for (int i = tid; i < 128 * 128; i += 128) sB[kmaj_off(i >> 7, i & 127, 8)] = (i & 127) < K ? B[(i >> 7) * K + (i & 127)] : 0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = slot;
  const uint32_t tmD = tm, tmA = tm + 128;  // D: columns 0..127, A: columns 128..159
  // A row (lane) -> TMEM: column j holds K bytes 4j .. 4j+3 (little endian)
  {
    const int row = warp * 32 + lane;
    uint32_t w[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      uint32_t x = 0;
      for (int b = 0; b < 4; ++b) {
        const int k = 4 * j + b;
        x |= uint32_t(k < K ? uint8_t(A[row * K + k]) : 0) << (8 * b);
      }
      w[j] = x;
    }
    const uint32_t ta = tmA + (uint32_t(warp * 32) << 16);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
        "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(ta),
        "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]),
        "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]),
        "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]),
        "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31])
        : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t idesc = idesc_i8(128, 128, true, false);
  unsigned long long t0 = clock64();
  if (tid == 0) {
    for (int r = 0; r < reps; ++r)
      for (int kb = 0; kb < kblocks; ++kb) {
        const uint64_t db = sdesc(smem_u32(sB) + kb * 256, 128, 1024);
        const uint32_t acc = (r | kb) ? 1u : 0u;
        if (mode == 0) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmD),
              "r"(tmA + kb * 8), "l"(db), "r"(idesc), "r"(acc));
        } else {
          const uint64_t da = sdesc(smem_u32(sA) + kb * 256, 128, 1024);
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmD),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
      }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  __syncwarp();
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra Dn;\n\tbra W;\n\tDn:\n\t}\n" ::"r"(smem_u32(&bar)), "r"(0));
  unsigned long long t1 = clock64();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) cyc[0] = t1 - t0;
  const uint32_t lane_off = uint32_t(warp * 32) << 16;
  for (int c = 0; c < 128; c += 32) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
        "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tmD + lane_off + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * 128 + c + j] = int32_t(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

int main() {
  for (int kblocks : {1, 4}) {
    const int K = 32 * kblocks;
    std::vector<int8_t> A(128 * K);
    std::vector<uint8_t> B(128 * K);
    srand(7);
    for (auto& x : A) x = int8_t(rand() % 255 - 127);
    for (auto& x : B) x = uint8_t(rand() % 129);
    std::vector<int32_t> want(128 * 128);
    for (int i = 0; i < 128; ++i)
      for (int n = 0; n < 128; ++n) {
        int s = 0;
        for (int k = 0; k < K; ++k) s += int(A[i * K + k]) * int(B[n * K + k]);
        want[i * 128 + n] = s;
      }
    int8_t* dA; uint8_t* dB; int32_t* dD; unsigned long long* dc;
    CK(cudaMalloc(&dA, A.size())); CK(cudaMalloc(&dB, B.size())); CK(cudaMalloc(&dD, want.size() * 4)); CK(cudaMalloc(&dc, 8));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
    CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024));
    for (int mode : {0, 1}) {
      CK(cudaMemset(dD, 0xFF, want.size() * 4));
      k_probe<<<1, 128, 40 * 1024>>>(dA, dB, dD, kblocks, mode, 1, dc);
      CK(cudaDeviceSynchronize());
      std::vector<int32_t> got(want.size());
      CK(cudaMemcpy(got.data(), dD, got.size() * 4, cudaMemcpyDeviceToHost));
      int bad = 0;
      for (size_t i = 0; i < got.size(); ++i) bad += got[i] != want[i];
      printf("K=%d mode=%s: %d mismatches of %zu (got[0]=%d want[0]=%d, got[129]=%d want[129]=%d)\n", K,
             mode == 0 ? "A in TMEM" : "A in smem", bad, got.size(), got[0], want[0], got[129], want[129]);
      unsigned long long c;
      k_probe<<<1, 128, 40 * 1024>>>(dA, dB, dD, kblocks, mode, 2048, dc);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost));
      printf("   chain of %d MMAs (M128 N128 K32): %.1f cycles per MMA\n", 2048 * kblocks, double(c) / (2048.0 * kblocks));
    }
    cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
  }
  return 0;
}
