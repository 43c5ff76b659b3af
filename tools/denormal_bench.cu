// Throughput of FADD2 / FMUL / FFMA2 chains on normal vs subnormal operands.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f2;
__device__ __forceinline__ f2 add2(f2 a, f2 b) { f2 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { f2 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__global__ void k_add2(f2* out, f2 a, f2 b, int n) {
  f2 x0 = a, x1 = a ^ 1, x2 = a ^ 2, x3 = a ^ 3;
  for (int i = 0; i < n; ++i) { x0 = add2(x0, b); x1 = add2(x1, b); x2 = add2(x2, b); x3 = add2(x3, b); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 ^ x1 ^ x2 ^ x3;
}
__global__ void k_fmul(float* out, float a, float b, int n) {
  float x0 = a, x1 = a * 1.0001f, x2 = a * 1.0002f, x3 = a * 1.0003f;
  for (int i = 0; i < n; ++i) { x0 = __fmul_rn(x0, b); x1 = __fmul_rn(x1, b); x2 = __fmul_rn(x2, b); x3 = __fmul_rn(x3, b); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
__global__ void k_fma2(f2* out, f2 a, f2 b, f2 c, int n) {
  f2 x0 = a, x1 = a ^ 1, x2 = a ^ 2, x3 = a ^ 3;
  for (int i = 0; i < n; ++i) { x0 = fma2(x0, b, c); x1 = fma2(x1, b, c); x2 = fma2(x2, b, c); x3 = fma2(x3, b, c); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 ^ x1 ^ x2 ^ x3;
}
static f2 pk(float x) { unsigned u; memcpy(&u, &x, 4); return ((f2)u << 32) | u; }
int main() {
  f2* d; cudaMalloc(&d, 148 * 8 * 256 * 8);
  cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
  const int n = 4096, blocks = 148 * 8, thr = 256;
  struct { const char* name; float a, b; } cases[] = {
      {"normal", 1.5f, 0.0f}, {"subnormal-in", 1e-40f, 0.0f}, {"subnormal-both", 1e-40f, 1e-41f}};
  for (auto& c : cases) {
    float ms;
    k_add2<<<blocks, thr>>>(d, pk(c.a), pk(c.b), n);
    cudaEventRecord(s); k_add2<<<blocks, thr>>>(d, pk(c.a), pk(c.b), n); cudaEventRecord(e); cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    double ops = 2.0 * 4 * n * blocks * thr;
    printf("FADD2 %-15s %.3f ms  %.1f Gop/s\n", c.name, ms, ops / ms / 1e6);
    cudaEventRecord(s); k_fma2<<<blocks, thr>>>(d, pk(c.a), pk(1.0f), pk(c.b), n); cudaEventRecord(e); cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    printf("FFMA2 %-15s %.3f ms  %.1f Gop/s\n", c.name, ms, ops / ms / 1e6);
    cudaEventRecord(s); k_fmul<<<blocks, thr>>>((float*)d, c.a, c.name[0] == 'n' ? 1.0f : 0.9999f, n); cudaEventRecord(e); cudaEventSynchronize(e);
    cudaEventElapsedTime(&ms, s, e);
    printf("FMUL  %-15s %.3f ms  %.1f Gop/s\n", c.name, ms, ops / 2 / ms / 1e6);
  }
  return 0;
}
