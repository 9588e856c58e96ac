// Microbenchmark: cycles per DP step for one warp (no memory traffic).
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t gt_mask(float a, float b) { uint32_t d; asm("set.gt.u32.f32 %0, %1, %2;" : "=r"(d) : "f"(a), "f"(b)); return d; }
__device__ __forceinline__ void fold(float& acc, float a, float b) { asm("max.NaN.f32 %0, %0, %1, %2;" : "+f"(acc) : "f"(fabsf(a)), "f"(fabsf(b))); }

template <int R, bool SHFL>
__global__ void k(const float* qg, float* out, int steps, long long* cyc) {
  int lane = threadIdx.x;
  float q[R][8];
  for (int r = 0; r < R; ++r) for (int e = 0; e < 8; ++e) q[r][e] = qg[(lane * R + r) * 8 + e];
  float o[R]; for (int r = 0; r < R; ++r) o[r] = 0.f;
  float acc = 0.f; uint32_t w[R]; for (int r = 0; r < R; ++r) w[r] = 0;
  bool is31 = lane == 31; int src = (lane + 31) & 31; float bnd = qg[1000];
  long long t0 = clock64();
  for (int it = 0; it < steps / 32; ++it) {
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      float send = is31 ? bnd : o[R-1];
      float up = SHFL ? __shfl_sync(0xffffffffu, send, src) : send;
      float n[R];
      float prev = up;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        w[r] |= gt_mask(prev, o[r]) & (1u << u);
        n[r] = q[r][u & 7] + fmaxf(prev, o[r]);
        prev = o[r];
      }
#pragma unroll
      for (int r = 0; r < R; r += 2) fold(acc, q[r][u&7], q[r+1][u&7]);
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
  float* q; float* o; long long* c; cudaMalloc(&q, 1 << 20); cudaMalloc(&o, 4096); cudaMalloc(&c, 8);
  cudaMemset(q, 0, 1 << 20);
  int steps = 1 << 16; long long cy;
#define RUN(R, S) k<R, S><<<1, 32>>>(q, o, steps, c); k<R, S><<<1, 32>>>(q, o, steps, c); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("R=%d shfl=%d: %.2f cycles/step, %.2f per row-step\n", R, (int)S, (double)cy / steps, (double)cy / steps / R);
  RUN(2, true) RUN(2, false) RUN(4, true) RUN(4, false) RUN(8, true)
  // 4 warps per SM sub-partition contention check: launch 4 warps in 1 block
  return 0;
}
