// Microbenchmark: cycles per DP column for one warp, current kernel's op mix
// (FSET+FFMA bits, FMNMX3 fold, SEL send, SHFL) and variants.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void fold3(float& acc, float a, float b) {
  asm("max.NaN.f32 %0, %0, %1, %2;" : "+f"(acc) : "f"(fabsf(a)), "f"(fabsf(b)));
}
template <int BIT>
__device__ __forceinline__ void bitf(float& wf, float a, float b) {
  constexpr float kB = static_cast<float>(1u << BIT);
  asm("{ .reg .f32 t; set.gt.f32.f32 t, %1, %2; fma.rn.f32 %0, t, %3, %0; }" : "+f"(wf) : "f"(a), "f"(b), "f"(kB));
}
__device__ __forceinline__ float add_ffma(float m, float q) {
  float r;
  asm("fma.rn.f32 %0, %1, 0f3F800000, %2;" : "=f"(r) : "f"(m), "f"(q));
  return r;
}

// FLAGS: 1 shfl, 2 bits, 4 fold, 8 ffma-add, 16 sel
template <int R, int FLAGS>
__global__ void k(const float* qg, float* out, int steps, long long* cyc) {
  int lane = threadIdx.x & 31;
  float q[R][4];
  for (int r = 0; r < R; ++r) for (int e = 0; e < 4; ++e) q[r][e] = qg[(lane * R + r) * 4 + e];
  float o[R]; for (int r = 0; r < R; ++r) o[r] = 0.f;
  float acc = 0.f; float wf[R]; for (int r = 0; r < R; ++r) wf[r] = 8388608.0f;
  bool is31 = lane == 31; int src = (lane + 31) & 31; float bnd = qg[1000 + lane];
  const float s31 = is31 ? 0.0f : 1.0f;
  float sendf = 0.f;
  float upp = 0.f;
  __syncwarp();
  long long t0 = clock64();
  for (int it = 0; it < steps / 16; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      float send = (FLAGS & 16) ? (is31 ? bnd : o[R - 1]) : o[R - 1];
      if (FLAGS & 64) send = sendf;  // computed with the previous column's n[R-1]
      float up = (FLAGS & 1) ? __shfl_sync(0xffffffffu, send, src) : send + bnd;
      if (FLAGS & 32) up = lane == 0 ? bnd : up;
      if (FLAGS & 128) {  // skewed lanes: the value shuffled one column earlier
        const float u2 = lane == 0 ? bnd : upp;
        upp = __shfl_sync(0xffffffffu, o[R - 1], src);
        up = u2;
      }
      float n[R];
      float prev = up;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (FLAGS & 2) {
          switch (u) {
#define B(U) case U: bitf<15 - U>(wf[r], prev, o[r]); break;
            B(0) B(1) B(2) B(3) B(4) B(5) B(6) B(7) B(8) B(9) B(10) B(11) B(12) B(13) B(14) B(15)
#undef B
          }
        }
        const float m = fmaxf(prev, o[r]);
        n[r] = (FLAGS & 8) ? add_ffma(m, q[r][u & 3]) : q[r][u & 3] + m;
        if ((FLAGS & 64) && r == R - 1) sendf = __fmaf_rn(m, s31, is31 ? bnd : q[r][u & 3]);
        prev = o[r];
      }
      if (FLAGS & 4) {
#pragma unroll
        for (int r = 0; r + 1 < R; r += 2) fold3(acc, q[r][u & 3], q[r + 1][u & 3]);
        if (R == 1) fold3(acc, q[0][u & 3], q[0][u & 3]);
      }
#pragma unroll
      for (int r = 0; r < R; ++r) o[r] = n[r];
    }
    if (FLAGS & 2) {
#pragma unroll
      for (int r = 0; r < R; ++r) { acc += wf[r]; wf[r] = 8388608.0f; }
    }
  }
  long long t1 = clock64();
  float s = acc; for (int r = 0; r < R; ++r) s += o[r] + wf[r];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void shfl_chain(float* out, int n, long long* cyc) {
  float v = threadIdx.x;
  int src = (threadIdx.x + 31) & 31;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) v = __shfl_sync(0xffffffffu, v, src);
  long long t1 = clock64();
  out[threadIdx.x] = v;
  if (threadIdx.x == 0) *cyc = (t1 - t0);
}

int main() {
  float *q, *o; long long* c;
  cudaMalloc(&q, 1 << 20); cudaMalloc(&o, 1 << 16); cudaMalloc(&c, 8);
  cudaMemset(q, 0, 1 << 20);
  int steps = 1 << 16; long long cy;
  shfl_chain<<<1, 32>>>(o, 4096, c); shfl_chain<<<1, 32>>>(o, 4096, c);
  cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
  printf("dependent SHFL latency: %.2f cycles\n", (double)cy / 4096);
#define RUN(R, F, WARPS)                                                                       \
  k<R, F><<<1, 32 * WARPS>>>(q, o, steps, c); k<R, F><<<1, 32 * WARPS>>>(q, o, steps, c);      \
  cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);                                               \
  printf("R=%d flags=%2d (shfl%d bits%d fold%d ffma%d sel%d) warps=%d: %6.2f cycles/col, %5.2f per cell\n", R, F, \
         !!(F & 1), !!(F & 2), !!(F & 4), !!(F & 8), !!(F & 16), WARPS, (double)cy / steps,     \
         (double)cy / steps / R);
  RUN(4, 6, 1) RUN(4, 23, 1) RUN(4, 134, 1) RUN(4, 142, 1) RUN(4, 132, 1) RUN(4, 128, 1)
  RUN(2, 23, 1) RUN(2, 134, 1) RUN(1, 134, 1) RUN(8, 23, 1) RUN(8, 134, 1) RUN(4, 134, 4) RUN(2, 134, 4) RUN(2, 134, 8)
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
