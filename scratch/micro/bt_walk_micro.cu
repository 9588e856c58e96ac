// Micro: the walker's word loop on synthetic smem words, one thread.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t lds32(uint32_t a) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory"); return v; }

template <int VARIANT>
__global__ void k(const uint32_t* g, long long* out, int R, int words) {
  extern __shared__ uint32_t sm[];
  __shared__ int rec_y[512];
  __shared__ uint32_t rec_ex[512];
  // window: [words][R] rows, random bits density ~1/8 per (row, position)
  for (int i = threadIdx.x; i < words * R + 64; i += blockDim.x) sm[i] = g[i % 8192];
  __syncthreads();
  if (threadIdx.x) return;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + 64 * 4;
  const uint32_t wstride = R * 4;
  int y = R - 1;
  int ml = words - 1;
  uint32_t pw = base + (ml * R + y) * 4;
  uint32_t x = lds32(pw);
  long long t0 = clock64();
  int nw = 0;
  while (true) {
    uint32_t q1 = lds32(pw - 4), q2 = lds32(pw - 8), q3 = lds32(pw - 12), q4 = lds32(pw - 16);
    uint32_t pb = pw, exw = 0;
#define STEP(Q, OFF) { const uint32_t d = x - 1u; exw |= x & ~d; x = (Q) & ~(x ^ d); (Q) = lds32(pb - (OFF)); }
    while (true) {
      STEP(q1, 20u) STEP(q2, 24u) STEP(q3, 28u) STEP(q4, 32u)
      pb -= 16u;
      if ((x & 0x7fffffffu) == 0u) break;
    }
    exw |= x;
    if (VARIANT >= 1) rec_ex[ml] = exw;
    const int ex = __popc(exw);
    y -= ex;
    --ml; ++nw;
    if (y <= 40 || ml < 0) break;
    pw -= (uint32_t)(ex * 4) + wstride;
    if (VARIANT >= 2) rec_y[ml] = y;
    x = lds32(pw);
  }
  long long t1 = clock64();
  out[0] = t1 - t0; out[1] = nw; out[2] = R - 1 - y;
}
int main() {
  uint32_t* g; long long* o; cudaMalloc(&g, 8192 * 4); cudaMalloc(&o, 24);
  static uint32_t h[8192]; uint64_t st = 7;
  for (int i = 0; i < 8192; ++i) { uint32_t v = 0; for (int b = 0; b < 32; ++b) { st = st * 6364136223846793005ull + 1442695040888963407ull; if ((st >> 40) % 8 == 0) v |= 1u << b; } h[i] = v; }
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  int R = 256, words = 200;
  size_t smem = (words * R + 64) * 4;
#define RUN(V) cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
  k<V><<<1, 32, smem>>>(g, o, R, words); k<V><<<1, 32, smem>>>(g, o, R, words); \
  { long long c[3]; cudaMemcpy(c, o, 24, cudaMemcpyDeviceToHost); printf("variant %d: %lld cycles, %lld words, %lld exits -> %.1f cyc/word, %.2f exits/word  (%s)\n", V, c[0], c[1], c[2], (double)c[0] / c[1], (double)c[2] / c[1], cudaGetErrorString(cudaGetLastError())); }
  RUN(0) RUN(1) RUN(2)
  return 0;
}
