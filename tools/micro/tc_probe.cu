// Microbenchmarks for the tensor-core FWHT experiment (not part of libsbw):
//   1. TMEM read throughput of tcgen05.ld 32x32b (plain / .pack::16b)
//   2. correctness of a hand-built kind::i8 MMA (s8 A, u8 B, s32 D in TMEM,
//      K-major SWIZZLE_NONE canonical smem layouts)
//   3. MMA issue throughput for M=128, N=256, K=32 i8 instructions
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tc_probe tc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#include "tmem_ld.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d: %s\n", cudaGetErrorString(e), __FILE__, __LINE__, #x); exit(1);} } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- 1. TMEM read
template <int PACK>
__global__ void k_tmem_read(int iters, unsigned long long* cycles, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t base = slot;
  const uint32_t lane_off = uint32_t((warp & 3) * 32) << 16;
  const int nq = blockDim.x >> 7;  // warps per lane quarter
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const uint32_t col = uint32_t(((i * nq + (warp >> 2)) * (PACK ? 128 : 64)) & 511);
    if constexpr (PACK) {
      uint32_t r[64];
      tmem_ld_x64_p16(base + lane_off + col, r);
      tmem_wait_ld();
      acc ^= r[0] ^ r[63];
    } else {
      uint32_t r[64];
      tmem_ld_x64(base + lane_off + col, r);
      tmem_wait_ld();
      acc ^= r[0] ^ r[63];
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(base, 512);
}

// ---------------------------------------------------------------- 2/3. MMA
// K-major, no swizzle: core matrix = 8 rows x 16 bytes (128 B contiguous).
// Layout used here for an R x 256 operand: byte (row, k) at
//   ((row / 8) * 16 + k / 16) * 128 + (row % 8) * 16 + k % 16
// => LBO (next 16-byte K chunk) = 128 B, SBO (next 8-row group) = 2048 B.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr & 0x3FFFF) >> 4);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // sm100 descriptor version
  return d;
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int a_signed, int b_signed) {
  return (2u << 4) | (uint32_t(a_signed) << 7) | (uint32_t(b_signed) << 10) |
         (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}\n" ::"r"(smem_u32(bar)), "r"(phase));
}

__device__ __forceinline__ uint32_t kmaj_off(int row, int k) {
  return uint32_t(((row >> 3) * 16 + (k >> 4)) * 128 + (row & 7) * 16 + (k & 15));
}

// A: 128 x 256 s8 (row-major in global), B: 256(N) x 256(K) u8 (row-major, K contiguous)
// D: 128 x 256 s32 -> global row-major. reps: MMA chains repeated for timing.
__global__ void __launch_bounds__(128) k_mma_i8(const int8_t* A, const uint8_t* B, int32_t* D, int reps,
                                                unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;                  // 32 KiB
  uint8_t* sB = sm + 128 * 256;      // 64 KiB
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 256; i += 128) sA[kmaj_off(i >> 8, i & 255)] = uint8_t(A[i]);
  for (int i = tid; i < 256 * 256; i += 128) sB[kmaj_off(i >> 8, i & 255)] = B[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc(&slot, 256);
  if (tid == 0) mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  const uint32_t idesc = idesc_i8(128, 256, 1, 0);
  unsigned long long t0 = clock64();
  if (tid == 0) {
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kb = 0; kb < 8; ++kb) {
        const uint64_t da = sdesc(smem_u32(sA) + kb * 256, 128, 2048);
        const uint64_t db = sdesc(smem_u32(sB) + kb * 256, 128, 2048);
        mma_i8(tm, da, db, idesc, (r | kb) ? 1u : 0u);
      }
    }
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  unsigned long long t1 = clock64();
  tc_fence_after();
  if (tid == 0) cycles[blockIdx.x] = t1 - t0;
  // each warp reads its 32 lanes, 256 columns
  const uint32_t lane_off = uint32_t(warp * 32) << 16;
  for (int c = 0; c < 256; c += 64) {
    uint32_t r[64];
    tmem_ld_x64(tm + lane_off + c, r);
    tmem_wait_ld();
    if (blockIdx.x == 0)
      for (int j = 0; j < 64; ++j) D[(warp * 32 + (tid & 31)) * 256 + c + j] = int32_t(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 256);
}

// B operand in K-major SWIZZLE_128B layout: atoms of 8 rows x 128 B,
// chunk c of row i at c ^ i; atom (ka, g) at (ka * 32 + g) * 1024.
__device__ __forceinline__ uint32_t sw128_off(int n, int k) {
  const int ka = k >> 7, g = n >> 3, i = n & 7, c = (k & 127) >> 4;
  return uint32_t((ka * 32 + g) * 1024 + i * 128 + ((c ^ i) << 4) + (k & 15));
}
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t sbo) {
  return uint64_t((saddr & 0x3FFFFu) >> 4) | (uint64_t(1) << 16) | (uint64_t((sbo >> 4) & 0x3FFFu) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
__global__ void __launch_bounds__(128) k_mma_i8_sw128(const int8_t* A, const uint8_t* B, int32_t* D) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;                  // 32 KiB, no swizzle
  uint8_t* sB = sm + 32768;          // 64 KiB, SW128 (1024-aligned)
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 256; i += 128) sA[kmaj_off(i >> 8, i & 255)] = uint8_t(A[i]);
  for (int i = tid; i < 256 * 256; i += 128) sB[sw128_off(i >> 8, i & 255)] = B[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc(&slot, 256);
  if (tid == 0) mbar_init(&bar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  if (tid == 0) {
#pragma unroll
    for (int kb = 0; kb < 8; ++kb)
      mma_i8(tm, sdesc(smem_u32(sA) + kb * 256, 128, 2048),
             sdesc_sw128(smem_u32(sB) + (kb >> 2) * 32768 + (kb & 3) * 32, 1024), idesc_i8(128, 256, 1, 0),
             kb ? 1u : 0u);
    mma_commit(&bar);
  }
  __syncwarp();
  mbar_wait(&bar, 0);
  tc_fence_after();
  const uint32_t lane_off = uint32_t(warp * 32) << 16;
  for (int c = 0; c < 256; c += 64) {
    uint32_t r[64];
    tmem_ld_x64(tm + lane_off + c, r);
    tmem_wait_ld();
    for (int j = 0; j < 64; ++j) D[(warp * 32 + (tid & 31)) * 256 + c + j] = int32_t(r[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 256);
}

// MMA chain time while other warps stream STS.128 (MODE 1) / LDS.128 (MODE 2) / nothing (0)
template <int MODE>
__global__ void __launch_bounds__(256) k_mma_contention(int reps, unsigned long long* cycles, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sA = sm;
  uint8_t* sB = sm + 128 * 256;
  uint4* sX = reinterpret_cast<uint4*>(sm + 96 * 1024);  // 64 KiB scratch
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 96 * 1024 / 16; i += 256) reinterpret_cast<uint4*>(sm)[i] = make_uint4(i, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc(&slot, 256);
  if (tid == 0) { mbar_init(&bar, 1); done = 0; }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  const uint32_t idesc = idesc_i8(128, 256, 1, 0);
  if (warp == 0) {
    if (tid == 0) {
      const unsigned long long t0 = clock64();
      for (int r = 0; r < reps; ++r)
#pragma unroll
        for (int kb = 0; kb < 8; ++kb)
          mma_i8(tm, sdesc(smem_u32(sA) + kb * 256, 128, 2048), sdesc(smem_u32(sB) + kb * 256, 128, 2048), idesc,
                 (r | kb) ? 1u : 0u);
      const unsigned long long t1 = clock64();
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      cycles[blockIdx.x] = clock64() - t0;
      cycles[512 + blockIdx.x] = t1 - t0;
      done = 1;
    }
    __syncwarp();
  } else {
    uint32_t acc = 0;
    int it = 0;
    while (!done) {
      for (int k = 0; k < 64; ++k) {
        const int idx = ((it * 64 + k) * 224 + (tid - 32)) & 4095;
        if (MODE == 1) sX[idx] = make_uint4(k, it, tid, acc);
        if (MODE == 2) { const uint4 v = sX[idx]; acc ^= v.x ^ v.w; }
      }
      ++it;
    }
    sink[blockIdx.x * 256 + tid] = acc + it;
    if (tid == 32) cycles[1024 + blockIdx.x] = it;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 256);
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  unsigned long long* d_cyc;
  uint32_t* d_sink;
  CK(cudaMalloc(&d_cyc, sizeof(unsigned long long) * 2048));
  CK(cudaMalloc(&d_sink, 1 << 24));
  std::vector<unsigned long long> cyc(1024);

  // 1. TMEM read throughput
  for (int pack = 0; pack < 2; ++pack)
    for (int warps : {4, 8, 16}) {
      const int iters = 4096;
      for (int rep = 0; rep < 2; ++rep) {
        if (pack) k_tmem_read<1><<<sms, warps * 32>>>(iters, d_cyc, d_sink);
        else k_tmem_read<0><<<sms, warps * 32>>>(iters, d_cyc, d_sink);
        CK(cudaDeviceSynchronize());
      }
      CK(cudaMemcpy(cyc.data(), d_cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost));
      double avg = 0;
      for (int i = 0; i < sms; ++i) avg += double(cyc[i]) / sms;
      const double cols = double(warps) * iters * (pack ? 128 : 64);  // columns x 32 lanes per warp-load
      printf("tmem_read pack=%d warps=%2d: %.1f B/clk/SM (TMEM cells), %.1f reg-B/clk/SM\n", pack, warps,
             cols * 32 * 4 / avg, cols * 32 * 4 / avg / (pack ? 2 : 1));
    }

  // 2. MMA correctness
  std::vector<int8_t> A(128 * 256);
  std::vector<uint8_t> B(256 * 256);
  srand(1);
  for (auto& a : A) a = int8_t((rand() % 255) - 127);
  for (auto& b : B) b = uint8_t(rand() % 256);
  int8_t* dA; uint8_t* dB; int32_t* dD;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dD, 128 * 256 * 4));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  const int smem = 96 * 1024;
  CK(cudaFuncSetAttribute(k_mma_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  k_mma_i8<<<1, 128, smem>>>(dA, dB, dD, 1, d_cyc);
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> D(128 * 256);
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 256; ++n) {
      int32_t ref = 0;
      for (int k = 0; k < 256; ++k) ref += int32_t(A[m * 256 + k]) * int32_t(B[n * 256 + k]);
      if (ref != D[m * 256 + n]) {
        if (bad < 5) printf("  mismatch m=%d n=%d got %d want %d\n", m, n, D[m * 256 + n], ref);
        ++bad;
      }
    }
  printf("mma_i8 128x256x256 correctness: %ld mismatches\n", bad);

  // 2b. SW128 B operand
  CK(cudaFuncSetAttribute(k_mma_i8_sw128, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaMemset(dD, 0, 128 * 256 * 4));
  k_mma_i8_sw128<<<1, 128, smem>>>(dA, dB, dD);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 256; ++n) {
      int32_t ref = 0;
      for (int k = 0; k < 256; ++k) ref += int32_t(A[m * 256 + k]) * int32_t(B[n * 256 + k]);
      if (ref != D[m * 256 + n]) ++bad;
    }
  printf("mma_i8 SW128 B correctness: %ld mismatches\n", bad);

  // 3. MMA throughput: all SMs, reps chains of 8 K=32 MMAs
  for (int reps : {64, 512}) {
    k_mma_i8<<<sms, 128, smem>>>(dA, dB, dD, reps, d_cyc);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(cyc.data(), d_cyc, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost));
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += double(cyc[i]) / sms;
    const double macs = double(reps) * 8 * 128 * 256 * 32;
    printf("mma_i8 reps=%d: %.1f cyc/instr, %.0f MAC/clk/SM, chip %.2f POPS at %d MHz\n", reps,
           avg / (reps * 8), macs / avg, 2 * macs / avg * sms * clk_khz * 1e3 / 1e15, clk_khz / 1000);
  }
  // 4. MMA chain under smem contention
  const int smem2 = 160 * 1024;
  CK(cudaFuncSetAttribute(k_mma_contention<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
  CK(cudaFuncSetAttribute(k_mma_contention<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
  CK(cudaFuncSetAttribute(k_mma_contention<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2));
  std::vector<unsigned long long> c2(2048);
  for (int mode = 0; mode < 3; ++mode) {
    const int reps = 2;
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) k_mma_contention<0><<<sms, 256, smem2>>>(reps, d_cyc, d_sink);
      if (mode == 1) k_mma_contention<1><<<sms, 256, smem2>>>(reps, d_cyc, d_sink);
      if (mode == 2) k_mma_contention<2><<<sms, 256, smem2>>>(reps, d_cyc, d_sink);
      CK(cudaDeviceSynchronize());
    }
    CK(cudaMemcpy(c2.data(), d_cyc, sizeof(unsigned long long) * 2048, cudaMemcpyDeviceToHost));
    double avg = 0, its = 0, iss = 0;
    for (int i = 0; i < sms; ++i) { avg += double(c2[i]) / sms; its += double(c2[1024 + i]) / sms; iss += double(c2[512 + i]) / sms; }
    printf("  issue-only %.1f cyc/instr\n", iss / (reps * 8));
    const double bytes = its * 64 * 16 * 224;
    printf("mma under contention mode=%d: %.1f cyc/instr, other warps moved %.1f B/clk\n", mode,
           avg / (reps * 8), bytes / avg);
  }
  return 0;
}
