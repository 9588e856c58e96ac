// Microbenchmark: issue rate of tcgen05.mma (kind::f16, bf16 -> fp32) for
// A in TMEM (TS) vs A in smem (SS), N = 64 / 128 / 256, M = 128, K = 16.
// One CTA, one thread issues `iters` MMAs into 2 alternating accumulators;
// cycles per MMA printed.  Operand contents are garbage (timing only).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2409_07704_b200/csrc/mas_ptx.cuh"
#include "../../paper_2409_07704_b200/csrc/mas_umma.cuh"
using namespace mas;

__device__ __forceinline__ uint32_t idesc(int M, int N) { return umma::idesc_bf16_f32(M, N); }

__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, bool acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b),
               "r"(id), "r"(acc ? 1u : 0u) : "memory");
}

template <bool TS>
__global__ void k(int N, int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ alignas(8) uint64_t bar;
  const uint32_t base = (smem_addr(sm) + 1023u) & ~1023u;
  if (threadIdx.x < 32) umma::tmem_alloc(smem_addr(&slot), 512);
  if (threadIdx.x == 0) { mbar_init(smem_addr(&bar), 1); fence_mbar_init(); }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(128, N);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint64_t bd = umma::sdesc_kmajor_sw128(base + 65536 + (i & 3) * 32);
      const uint32_t d = tmem + 256 + (i & 1) * 0;  // one accumulator region
      if (TS) umma::mma_ts(d, tmem + (i & 3) * 8, bd, id, (i & 7) != 0);
      else mma_ss(d, umma::sdesc_kmajor_sw128(base + (i & 3) * 32), bd, id, (i & 7) != 0);
    }
    umma::mma_commit(smem_addr(&bar));
    long long t1 = clock64();
    mbar_wait(smem_addr(&bar), 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  umma::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) umma::tmem_dealloc(tmem, 512);
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  long long h[2];
  cudaFuncSetAttribute(k<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int ts = 1; ts >= 0; --ts)
    for (int N : {32, 64, 128, 256}) {
      const int iters = 4096;
      for (int rep = 0; rep < 2; ++rep) {
        if (ts) k<true><<<1, 128, 200 * 1024>>>(N, iters, d);
        else k<false><<<1, 128, 200 * 1024>>>(N, iters, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      }
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("%s N=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma (%.0f flop/cyc)\n", ts ? "TS" : "SS", N,
             double(h[0]) / iters, double(h[1]) / iters, 2.0 * 128 * N * 16 * iters / double(h[1]));
    }
  return 0;
}
