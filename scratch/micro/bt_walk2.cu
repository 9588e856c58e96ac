// Micro: variants of the backtrack walker's word loop on synthetic smem
// words (density 1/8 -> ~4 exits per 32-bit word), one thread.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t lds32(uint32_t a) { uint32_t v; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory"); return v; }

template <int V>
__global__ void k(const uint32_t* g, long long* out, int R, int words) {
  extern __shared__ uint32_t sm[];
  __shared__ int rec_y[512];
  __shared__ uint32_t rec_ex[512];
  for (int i = threadIdx.x; i < words * R + 512; i += blockDim.x) sm[i] = g[i % 8192];
  __syncthreads();
  if (threadIdx.x) return;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + 512 * 4;
  const uint32_t wstride = R * 4;
  int y = R - 1, ml = words - 1, nw = 0;
  uint32_t pw = base + (ml * R + y) * 4;
  uint32_t x = lds32(pw);
  uint32_t q1 = lds32(pw - 4), q2 = lds32(pw - 8), q3 = lds32(pw - 12), q4 = lds32(pw - 16);
  long long t0 = clock64();
  while (true) {
    uint32_t pb = pw, ps = pw, exw = 0;
    if (V == 0) {  // current kernel: ps tracked per step
#define STEP(Q, OFF) { const uint32_t d = x - 1u; exw |= x & ~d; ps -= x != 0u ? 4u : 0u; x = (Q) & ~(x ^ d); (Q) = lds32(pb - (OFF)); }
      while (true) { STEP(q1, 20u) STEP(q2, 24u) STEP(q3, 28u) STEP(q4, 32u) pb -= 16u; if ((x & 0x7fffffffu) == 0u) break; }
#undef STEP
    } else if (V == 1) {  // no ps: popc at the end
#define STEP(Q, OFF) { const uint32_t d = x - 1u; exw |= x & ~d; x = (Q) & ~(x ^ d); (Q) = lds32(pb - (OFF)); }
      while (true) { STEP(q1, 20u) STEP(q2, 24u) STEP(q3, 28u) STEP(q4, 32u) pb -= 16u; if ((x & 0x7fffffffu) == 0u) break; }
#undef STEP
      ps = pw - 4u * __popc(exw);
    } else if (V == 2) {  // 2-step blocks
#define STEP(Q, OFF) { const uint32_t d = x - 1u; exw |= x & ~d; x = (Q) & ~(x ^ d); (Q) = lds32(pb - (OFF)); }
      uint32_t q5 = 0, q6 = 0;
      while (true) { STEP(q1, 20u) STEP(q2, 24u) pb -= 8u; if ((x & 0x7fffffffu) == 0u) break; STEP(q3, 20u) STEP(q4, 24u) pb -= 8u; if ((x & 0x7fffffffu) == 0u) break; }
#undef STEP
      ps = pw - 4u * __popc(exw);
    }
    if (V == 3) {  // 64-bit pairs: lo = word ml, hi = word ml-1
      uint64_t X = (uint64_t)x | ((uint64_t)lds32(pw - wstride) << 32);
      uint64_t Q1 = (uint64_t)q1 | ((uint64_t)lds32(pw - 4 - wstride) << 32);
      uint64_t Q2 = (uint64_t)q2 | ((uint64_t)lds32(pw - 8 - wstride) << 32);
      uint64_t Q3 = (uint64_t)q3 | ((uint64_t)lds32(pw - 12 - wstride) << 32);
      uint64_t Q4 = (uint64_t)q4 | ((uint64_t)lds32(pw - 16 - wstride) << 32);
      uint64_t E = 0;
#define STEP(Q, OFF) { const uint64_t d = X - 1ull; E |= X & ~d; X = (Q) & ~(X ^ d); (Q) = (uint64_t)lds32(pb - (OFF)) | ((uint64_t)lds32(pb - (OFF) - wstride) << 32); }
      while (true) { STEP(Q1, 20u) STEP(Q2, 24u) STEP(Q3, 28u) STEP(Q4, 32u) pb -= 16u; if ((X & 0x7fffffffffffffffull) == 0ull) break; }
#undef STEP
      const uint64_t lastX = X;
      const int ex = __popcll(E | lastX);
      ps = pw - 4u * ex;
      const uint32_t pn = ps - 2 * wstride;
      x = lds32(pn); q1 = lds32(pn - 4); q2 = lds32(pn - 8); q3 = lds32(pn - 12); q4 = lds32(pn - 16);
      rec_ex[ml & 511] = (uint32_t)E;
      rec_ex[(ml - 1) & 511] = (uint32_t)((E | lastX) >> 32);
      y -= ex;
      ml -= 2; nw += 2;
      if (y <= 80 || ml < 1) break;
      pw = pn;
      rec_y[ml & 511] = y;
      continue;
    }
    const uint32_t last = x;
    if (V == 0) ps -= last != 0u ? 4u : 0u; else ps -= last != 0u ? 4u : 0u;
    const uint32_t pn = ps - wstride;
    x = lds32(pn); q1 = lds32(pn - 4); q2 = lds32(pn - 8); q3 = lds32(pn - 12); q4 = lds32(pn - 16);
    rec_ex[ml & 511] = exw | last;
    y -= (int)((pw - ps) >> 2);
    --ml; ++nw;
    if (y <= 48 || ml < 0) break;
    pw = pn;
    rec_y[ml & 511] = y;
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
  size_t smem = (words * R + 512) * 4;
#define RUN(V) cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
  k<V><<<1, 32, smem>>>(g, o, R, words); k<V><<<1, 32, smem>>>(g, o, R, words); \
  { long long c[3]; cudaMemcpy(c, o, 24, cudaMemcpyDeviceToHost); printf("variant %d: %lld cycles, %lld words, %lld exits -> %.1f cyc/word, %.2f exits/word (%s)\n", V, c[0], c[1], c[2], (double)c[0] / c[1], (double)c[2] / c[1], cudaGetErrorString(cudaGetLastError())); }
  RUN(0) RUN(1) RUN(2) RUN(3)
  return 0;
}
