// Microbenchmark: single-thread latency of the backtrack walker's building blocks.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t lds32(uint32_t a) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory"); return v; }
__device__ __forceinline__ uint32_t lds32v(uint32_t a) { uint32_t v; asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory"); return v; }

__global__ void k(const uint32_t* g, long long* out, int mode) {
  __shared__ uint32_t W[8192 + 64];
  for (int i = threadIdx.x; i < 8192 + 64; i += blockDim.x) W[i] = g[i];
  __syncthreads();
  if (threadIdx.x) return;
  uint32_t base = (uint32_t)__cvta_generic_to_shared(W) + 64 * 4;
  uint32_t x = W[5000], acc = 0;
  long long t0 = clock64();
  if (mode == 0) {  // dependent ALU chain IADD->LOP3, 4096 pairs
    for (int i = 0; i < 4096; ++i) { uint32_t d = x - 1u; x = W[i & 7] & ~(x ^ d); acc += x; }
  } else if (mode == 1) {  // dependent LDS chain
    uint32_t a = base;
    for (int i = 0; i < 4096; ++i) { uint32_t v = lds32(a); a = base + (v & 0x3ffc); }
    acc = a;
  } else if (mode == 2) {  // block-of-4 walker over synthetic words
    uint32_t pb = base + 8000 * 4;
    uint32_t q1 = lds32(pb - 4), q2 = lds32(pb - 8), q3 = lds32(pb - 12), q4 = lds32(pb - 16);
    uint32_t exw = 0;
    for (int i = 0; i < 1024; ++i) {
      uint32_t d;
      d = x - 1u; exw |= x & ~d; x = q1 & ~(x ^ d) | 1u; q1 = lds32v(pb - 20);
      d = x - 1u; exw |= x & ~d; x = q2 & ~(x ^ d) | 1u; q2 = lds32v(pb - 24);
      d = x - 1u; exw |= x & ~d; x = q3 & ~(x ^ d) | 1u; q3 = lds32v(pb - 28);
      d = x - 1u; exw |= x & ~d; x = q4 & ~(x ^ d) | 1u; q4 = lds32v(pb - 32);
      pb -= 16u; if (pb < base + 64) pb = base + 8000 * 4;
      if ((x & 0x7fffffffu) == 0u) break;
    }
    acc = exw + x;
  } else if (mode == 3) {  // same with non-volatile loads
    uint32_t pb = base + 8000 * 4;
    uint32_t q1 = lds32(pb - 4), q2 = lds32(pb - 8), q3 = lds32(pb - 12), q4 = lds32(pb - 16);
    uint32_t exw = 0;
    for (int i = 0; i < 1024; ++i) {
      uint32_t d;
      d = x - 1u; exw |= x & ~d; x = q1 & ~(x ^ d) | 1u; q1 = lds32(pb - 20);
      d = x - 1u; exw |= x & ~d; x = q2 & ~(x ^ d) | 1u; q2 = lds32(pb - 24);
      d = x - 1u; exw |= x & ~d; x = q3 & ~(x ^ d) | 1u; q3 = lds32(pb - 28);
      d = x - 1u; exw |= x & ~d; x = q4 & ~(x ^ d) | 1u; q4 = lds32(pb - 32);
      pb -= 16u; if (pb < base + 64) pb = base + 8000 * 4;
      if ((x & 0x7fffffffu) == 0u) break;
    }
    acc = exw + x;
  } else if (mode == 4) {  // word-change-like: dependent LDS + popc + address
    uint32_t pw = base + 8000 * 4;
    for (int i = 0; i < 1024; ++i) {
      uint32_t v = lds32(pw);
      int ex = __popc(v);
      pw -= (uint32_t)(ex * 4) + 64u;
      if (pw < base + 256) pw = base + 8000 * 4;
      acc += v;
    }
  }
  long long t1 = clock64();
  out[0] = t1 - t0; out[1] = acc;
}
int main() {
  uint32_t* g; long long* o; cudaMalloc(&g, 8256 * 4); cudaMalloc(&o, 16);
  uint32_t h[8256]; uint64_t st = 1; for (int i = 0; i < 8256; ++i) { st = st * 6364136223846793005ull + 1442695040888963407ull; h[i] = (uint32_t)(st >> 32) & (uint32_t)(st >> 13) & (uint32_t)(st>>7); }
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  const char* names[] = {"ALU chain (per IADD+LOP3 pair)", "LDS chain (per load)", "walker block volatile (per step)", "walker block (per step)", "word change sim (per word)"};
  const double div[] = {4096, 4096, 4096, 4096, 1024};
  for (int m = 0; m < 5; ++m) {
    long long c[2];
    k<<<1, 128>>>(g, o, m); k<<<1, 128>>>(g, o, m);
    cudaMemcpy(c, o, 16, cudaMemcpyDeviceToHost);
    printf("%-36s %.1f cycles\n", names[m], c[0] / div[m]);
  }
  return 0;
}
