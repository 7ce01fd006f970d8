// Microbenchmark: per-SM throughput of MUFU.EX2, F2FP (cvt.rn.bf16x2.f32), FFMA2, FFMA on B200.
// One CTA per SM, W warps; each thread runs N iterations of 16 independent ops.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(float* out, int iters, long long* clk) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  uint32_t u[16];
  unsigned long long v2[16];
  for (int i = 0; i < 16; ++i) v2[i] = ((unsigned long long)__float_as_uint(a[i]) << 32) | __float_as_uint(a[i]);
  for (int i = 0; i < 16; ++i) u[i] = i;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[i])); a[i] = __uint_as_float(r); }
      if (OP == 4) { uint32_t r; asm volatile("{.reg .b32 t0, t1;\n\tadd.u32 t0, %1, 0x8000;\n\tadd.u32 t1, %2, 0x8000;\n\tprmt.b32 %0, t0, t1, 0x7632;}" : "=r"(r) : "r"(__float_as_uint(a[i])), "r"(u[i])); a[i] = __uint_as_float(r); }
      if (OP == 5) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i])); uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[(i + 8) & 15]), "f"(a[(i + 8) & 15])); u[i] ^= r; a[(i + 8) & 15] += __uint_as_float(r) * 0.f; }
      if (OP == 2) asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(v2[i]));
      if (OP == 6) asm volatile("add.rn.f32x2 %0, %0, %0;" : "+l"(v2[i]));
      if (OP == 7) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i])); asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(v2[i])); }
      if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
      if (OP == 8) { uint32_t r; asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(__float_as_uint(a[i])), "r"(u[i])); a[i] = __uint_as_float(r); }
      if (OP == 9) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i])); uint32_t r; asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(u[(i + 8) & 15]), "r"(u[i])); u[i] ^= r; }
    }
  }
  unsigned long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i] + u[i] + __uint_as_float((uint32_t)v2[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
template <int OP> void run(const char* name, int warps) {
  float* o; long long* c; int sms = 148, iters = 2000;
  cudaMalloc(&o, sms * warps * 32 * 4); cudaMalloc(&c, sms * 8);
  k<OP><<<sms, warps * 32>>>(o, iters, c); cudaDeviceSynchronize();
  k<OP><<<sms, warps * 32>>>(o, iters, c); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  double ops = (double)iters * 16 * warps * 32;  // lane-ops per SM (OP 2 counts pairs)
  printf("%-6s warps/SM %2d: %.2f lane-ops/clk/SM  (%.2f clk per warp-instr per SMSP)\n", name, warps, ops / h,
         (double)h / (iters * 16.0 * warps / 4));
  cudaFree(o); cudaFree(c);
}
int main() {
  for (int w : {4, 8, 16}) { run<0>("ex2", w); run<1>("f2fp", w); run<5>("ex2+f2fp", w); run<8>("prmt", w); run<9>("ex2+prmt", w); run<2>("ffma2", w); run<7>("ex2+ffma2", w); }
  return 0;
}
