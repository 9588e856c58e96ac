// Microbenchmark: cycles per DP step for one warp -- pipe-balanced variants.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void fold3(float& acc, float a, float b) { asm("max.NaN.f32 %0, %0, %1, %2;" : "+f"(acc) : "f"(fabsf(a)), "f"(fabsf(b))); }
// bit via predicated IMAD (fma pipe): if (a > b) w += one * imm
__device__ __forceinline__ void bit_imad(uint32_t& w, float a, float b, uint32_t one, uint32_t bitv) {
  asm("{ .reg .pred q; setp.gt.f32 q, %1, %2; @q mad.lo.u32 %0, %3, %4, %0; }" : "+r"(w) : "f"(a), "f"(b), "r"(one), "r"(bitv));
}
__device__ __forceinline__ void bit_sel(uint32_t& w, float a, float b, int u) {
  uint32_t d; asm("set.gt.u32.f32 %0, %1, %2;" : "=r"(d) : "f"(a), "f"(b)); w |= d & (1u << u);
}

template <int R, int BITS, int FIN>
__global__ void k(const float* qg, float* out, int steps, long long* cyc, const uint32_t* ones) {
  int lane = threadIdx.x;
  float q[R][8];
  for (int r = 0; r < R; ++r) for (int e = 0; e < 8; ++e) q[r][e] = qg[(lane * R + r) * 8 + e];
  float o[R]; for (int r = 0; r < R; ++r) o[r] = 0.f;
  float acc = 0.f; uint32_t w[R]; for (int r = 0; r < R; ++r) w[r] = 0;
  uint32_t one = ones[0]; float zero = __int_as_float(ones[1]);
  uint32_t bitv[32]; for (int u = 0; u < 32; ++u) bitv[u] = ones[2 + u];
  bool is31 = lane == 31; int src = (lane + 31) & 31; float bnd = qg[1000];
  long long t0 = clock64();
  for (int it = 0; it < steps / 32; ++it) {
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      float send = is31 ? bnd : o[R-1];
      float up = __shfl_sync(0xffffffffu, send, src);
      float n[R];
      float prev = up;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (BITS == 0) bit_sel(w[r], prev, o[r], u); else bit_imad(w[r], prev, o[r], one, bitv[u]);
        n[r] = q[r][u & 7] + fmaxf(prev, o[r]);
        prev = o[r];
      }
      if (FIN == 0) {
#pragma unroll
        for (int r = 0; r < R; r += 2) fold3(acc, q[r][u&7], q[r+1][u&7]);
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) acc = __fmaf_rn(q[r][u&7], zero, acc);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) o[r] = n[r];
    }
  }
  long long t1 = clock64();
  float s = acc; for (int r = 0; r < R; ++r) s += o[r] + (float)w[r];
  out[lane] = s;
  if (lane == 0) *cyc = t1 - t0;
}
int main() {
  float* q; float* o; long long* c; uint32_t* ones; cudaMalloc(&q, 1 << 20); cudaMalloc(&o, 4096); cudaMalloc(&c, 8); cudaMalloc(&ones, 256);
  cudaMemset(q, 0, 1 << 20);
  uint32_t h[34]; h[0] = 1; h[1] = 0; for (int u = 0; u < 32; ++u) h[2+u] = 1u << u; cudaMemcpy(ones, h, sizeof(h), cudaMemcpyHostToDevice);
  int steps = 1 << 16; long long cy;
#define RUN(R, B, F) k<R, B, F><<<1, 32>>>(q, o, steps, c, ones); k<R, B, F><<<1, 32>>>(q, o, steps, c, ones); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("R=%d bits=%s fin=%s: %.2f cycles/step, %.2f per row-step\n", R, B ? "imad" : "sel ", F ? "ffma" : "mnmx3", (double)cy / steps, (double)cy / steps / R);
  RUN(2,0,0) RUN(2,1,0) RUN(2,1,1) RUN(4,0,0) RUN(4,1,0) RUN(4,1,1) RUN(8,1,0) RUN(8,1,1)
  return 0;
}
