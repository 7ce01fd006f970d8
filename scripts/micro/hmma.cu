// Microbenchmark: legacy tensor path (mma.sync m16n8k16 bf16 -> f32, SASS HMMA.16816) and
// ldmatrix.x4 throughput per SM on B200.  One CTA per SM, W warps, 8 independent accumulator
// chains per warp (OP 0), or ldmatrix.x4 from a conflict-free swizzled tile (OP 1).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro/hmma.bin scripts/micro/hmma.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(float* out, int iters, long long* clk) {
  __shared__ __align__(1024) uint8_t sm[16384];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float d[8][4] = {};
  uint32_t a0 = lane, a1 = lane * 3, a2 = lane * 5, a3 = lane * 7, b0 = lane * 11, b1 = lane * 13;
  uint32_t acc = 0;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(sm) + (threadIdx.x >> 5) * 1024 % 16384;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (OP == 0) {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int row = lane & 7, mat = lane >> 3;
        const uint32_t addr = base + (c * 2 + (mat & 1)) * 128 * 4 % 8192 + row * 128 + (((mat >> 1) ^ row) << 4);
        uint32_t r0, r1, r2, r3;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];" : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
        acc ^= r0 ^ r1 ^ r2 ^ r3;
      }
    }
  }
  unsigned long long t1 = clock64();
  float s = acc;
  for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
template <int OP>
void run(const char* name, int warps) {
  float* o;
  long long* c;
  int sms = 148, iters = 4000;
  cudaMalloc(&o, sms * warps * 32 * 4);
  cudaMalloc(&c, sms * 8);
  k<OP><<<sms, warps * 32>>>(o, iters, c);
  cudaDeviceSynchronize();
  k<OP><<<sms, warps * 32>>>(o, iters, c);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double n = (double)iters * 8 * warps;  // warp-instructions per SM
  if (OP == 0)
    printf("%-9s warps/SM %2d: %.1f clk per warp-mma per SM, %.0f flop/clk/SM\n", name, warps, h / n, n * 4096 * 2 / h);
  else
    printf("%-9s warps/SM %2d: %.2f clk per ldmatrix.x4 per SM, %.0f B/clk/SM\n", name, warps, h / n, n * 512 / h);
}
int main() {
  for (int w : {1, 2, 4, 8, 16}) run<0>("hmma16816", w);
  for (int w : {1, 4, 8, 16}) run<1>("ldsm.x4", w);
  return 0;
}
