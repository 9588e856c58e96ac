// Microbenchmark: single-warp issue rate of the DP's instructions (8
// independent chains each), to find the per-op reciprocal throughput.
#include <cstdio>
#include <cstdint>

template <int OP>
__global__ void k(const float* in, float* out, int n, long long* cyc) {
  float a[8], b[8];
  for (int i = 0; i < 8; ++i) { a[i] = in[threadIdx.x + i]; b[i] = in[threadIdx.x + 64 + i]; }
  const bool p = threadIdx.x & 1;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("set.gt.f32.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i]));
      if (OP == 1) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i]));
      if (OP == 2) asm volatile("max.NaN.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b[i]), "f"(b[(i + 1) & 7]));
      if (OP == 3) asm volatile("add.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i]));
      if (OP == 4) asm volatile("fma.rn.f32 %0, %1, 0f46000000, %0;" : "+f"(a[i]) : "f"(b[i]));
      if (OP == 5) asm volatile("{.reg .pred q; setp.ne.b32 q, %2, 0; selp.f32 %0, %1, %0, q;}" : "+f"(a[i]) : "f"(b[i]), "r"((int)p));
      if (OP == 6) asm volatile("{.reg .pred q; setp.gt.f32 q, %0, %1; @q add.f32 %0, %0, 0f3F800000;}" : "+f"(a[i]) : "f"(b[i]));
      if (OP == 7) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(a[i]) : "f"(b[i]), "f"(b[(i + 3) & 7]));
      if (OP == 8) {  // FMNMX + FADD pair (the DP core)
        asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[i]));
        asm volatile("add.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b[(i + 2) & 7]));
      }
      if (OP == 9) {  // FSET + FFMA pair (a bit)
        float t;
        asm volatile("set.gt.f32.f32 %0, %1, %2;" : "=f"(t) : "f"(a[i]), "f"(b[i]));
        asm volatile("fma.rn.f32 %0, %1, 0f46000000, %0;" : "+f"(b[i]) : "f"(t));
      }
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + b[i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  float *in, *out; long long* c; cudaMalloc(&in, 4096); cudaMalloc(&out, 4096); cudaMalloc(&c, 8);
  cudaMemset(in, 0, 4096);
  const char* names[] = {"FSET.BF", "FMNMX", "FMNMX3.NAN", "FADD", "FFMA imm", "SEL(pred)", "FSETP+@FADD", "FFMA reg", "FMNMX+FADD", "FSET+FFMA"};
  int n = 4096; long long cy;
#define RUN(OP)                                                            \
  for (int w = 1; w <= 4; w *= 4) {                                        \
    k<OP><<<1, 32 * w>>>(in, out, n, c); k<OP><<<1, 32 * w>>>(in, out, n, c); \
    cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);                        \
    printf("%-12s warps=%d: %.2f cycles per warp-instr (per SMSP)\n", names[OP], w, (double)cy / (n * 8.0) / ((OP >= 8) ? 2 : 1)); \
  }
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7) RUN(8) RUN(9)
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
