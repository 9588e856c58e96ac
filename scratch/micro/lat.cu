// Dependent-latency microbenchmark: chains of FMNMX/FADD/FSEL/SHFL (1 warp).
#include <cstdio>
template <int OP>
__global__ void k(float* out, int n, long long* cyc, float b) {
  float a = threadIdx.x, c = b * 2.f;
  const bool p = threadIdx.x & 1;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (OP == 0) asm volatile("max.f32 %0, %0, %1;" : "+f"(a) : "f"(c));
      if (OP == 1) asm volatile("add.f32 %0, %0, %1;" : "+f"(a) : "f"(c));
      if (OP == 2) { asm volatile("max.f32 %0, %0, %1;" : "+f"(a) : "f"(c)); asm volatile("add.f32 %0, %0, %1;" : "+f"(a) : "f"(c)); }
      if (OP == 3) asm volatile("{.reg .pred q; setp.ne.b32 q, %2, 0; selp.f32 %0, %1, %0, q;}" : "+f"(a) : "f"(c), "r"((int)p));
      if (OP == 4) { asm volatile("{.reg .pred q; setp.ne.b32 q, %2, 0; selp.f32 %0, %1, %0, q;}" : "+f"(a) : "f"(c), "r"((int)p)); asm volatile("max.f32 %0, %0, %1;" : "+f"(a) : "f"(c)); asm volatile("add.f32 %0, %0, %1;" : "+f"(a) : "f"(c)); }
      if (OP == 5) asm volatile("fma.rn.f32 %0, %0, 0f3F800000, %1;" : "+f"(a) : "f"(c));
      if (OP == 6) { asm volatile("max.f32 %0, %0, %1;" : "+f"(a) : "f"(c)); asm volatile("fma.rn.f32 %0, %0, 0f3F800000, %1;" : "+f"(a) : "f"(c)); }
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 8);
  const char* nm[] = {"FMNMX", "FADD", "FMNMX+FADD", "SEL", "SEL+FMNMX+FADD", "FFMA", "FMNMX+FFMA"};
  int n = 4096; long long cy;
#define R(OP) k<OP><<<1,32>>>(o, n, c, 0.5f); k<OP><<<1,32>>>(o, n, c, 0.5f); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost); printf("%-16s %.2f cycles per chain link\n", nm[OP], (double)cy / (n * 8.0));
  R(0) R(1) R(2) R(3) R(4) R(5) R(6)
  return 0;
}
