// Pure TMA streaming of q in the forward kernel's access pattern (no DP):
// each warp walks its ROWS rows across all S columns in stages of COLS
// columns (COLS/32 boxes of {32 cols, 32 rows-groups, ROWS/32 residues}),
// NSTAGE-deep ring, lane 0 issues, all lanes wait.  Reports GB/s.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c)); }
__device__ __forceinline__ void expect(uint32_t bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b) : "memory"); }
__device__ __forceinline__ bool tryw(uint32_t bar, uint32_t p) { uint32_t ok; asm volatile("{.reg .pred q; mbarrier.try_wait.parity.shared::cta.b64 q, [%1], %2; selp.u32 %0,1,0,q;}" : "=r"(ok) : "r"(bar), "r"(p) : "memory"); return ok; }
__device__ __forceinline__ void load3(uint32_t dst, const CUtensorMap* m, int c0, int c1, int c2, uint32_t bar) {
  asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst), "l"((uint64_t)m), "r"(c0), "r"(c1), "r"(c2), "r"(bar) : "memory");
}
template <int ROWS, int COLS, int NST>
__global__ void k(const __grid_constant__ CUtensorMap tm, int S, int T, int W) {
  extern __shared__ uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int RES = ROWS / 32;
  constexpr int STAGE = ROWS * COLS * 4;
  uint32_t base = ((uint32_t)__cvta_generic_to_shared(sm) + 1023) & ~1023u;
  uint32_t ring = base + warp * NST * STAGE;
  uint32_t bars = base + W * NST * STAGE + warp * NST * 8;
  if (lane == 0) for (int s = 0; s < NST; ++s) mbar_init(bars + 8 * s, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int gwarp = blockIdx.x * W + warp;
  const int group0 = gwarp * 32;  // 32 groups of RES rows
  const int nit = S / COLS;
  if (lane == 0)
    for (int it = 0; it < NST - 1 && it < nit; ++it) {
      expect(bars + 8 * it, STAGE);
      for (int c = 0; c < COLS / 32; ++c) load3(ring + it * STAGE + c * (ROWS * 128), &tm, it * COLS + 32 * c, group0, 0, bars + 8 * it);
    }
  int slot = 0; uint32_t par = 0;
  for (int m = 0; m < nit; ++m) {
    int nxt = m + NST - 1;
    if (nxt < nit && lane == 0) {
      int fs = nxt % NST;
      expect(bars + 8 * fs, STAGE);
      for (int c = 0; c < COLS / 32; ++c) load3(ring + fs * STAGE + c * (ROWS * 128), &tm, nxt * COLS + 32 * c, group0, 0, bars + 8 * fs);
    }
    while (!tryw(bars + 8 * slot, par)) {}
    __syncwarp();
    slot = slot + 1 == NST ? 0 : slot + 1; if (slot == 0) par ^= 1;
  }
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
template <int ROWS, int COLS, int NST>
void run(float* q, int B, int T, int S, int W) {
  void* p; cudaDriverEntryPointQueryResult qr; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr);
  Enc enc = (Enc)p; CUtensorMap tm;
  constexpr int RES = ROWS / 32;
  cuuint64_t dims[3] = {(cuuint64_t)S, (cuuint64_t)B * T / RES, RES};
  cuuint64_t str[2] = {(cuuint64_t)RES * S * 4, (cuuint64_t)S * 4};
  cuuint32_t box[3] = {32, 32, RES}; cuuint32_t es[3] = {1, 1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, q, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int warps = B * T / ROWS; int ctas = warps / W;
  size_t smem = (size_t)W * NST * ROWS * COLS * 4 + W * NST * 8 + 1024;
  cudaFuncSetAttribute(k<ROWS, COLS, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k<ROWS, COLS, NST><<<ctas, W * 32, smem>>>(tm, S, T, W);
  cudaEventRecord(a);
  for (int i = 0; i < 5; ++i) k<ROWS, COLS, NST><<<ctas, W * 32, smem>>>(tm, S, T, W);
  cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
  printf("rows/warp %3d cols/stage %3d stages %d W %d ctas %4d smem %6zu: %.1f us  %.0f GB/s  (%s)\n", ROWS, COLS, NST, W, ctas, smem, ms * 1e3, (double)B * T * S * 4 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  int B = 32, T = 1024, S = 8192; float* q; cudaMalloc(&q, (size_t)B * T * S * 4); cudaMemset(q, 0, (size_t)B * T * S * 4);
  run<64, 32, 4>(q, B, T, S, 4);
  run<64, 64, 3>(q, B, T, S, 4);
  run<64, 128, 3>(q, B, T, S, 2);
  run<128, 32, 4>(q, B, T, S, 2);
  run<128, 32, 3>(q, B, T, S, 4);
  run<128, 64, 3>(q, B, T, S, 2);
  run<128, 64, 2>(q, B, T, S, 2);
  run<128, 128, 2>(q, B, T, S, 1);
  run<32, 128, 3>(q, B, T, S, 4);
  return 0;
}
