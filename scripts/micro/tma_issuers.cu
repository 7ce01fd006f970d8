// Microbenchmark: per-SM rate of 4 KB TMA boxes (K2 / K1's unit: 16 keys x 1 head of a paged
// NHD cache) vs the number of issuing warps.  One CTA per SM; warp w's lane 0 keeps its own
// `per` ring slots (4 KB each) in flight; random blocks of a 2 GiB cache.  Shows whether the
// ~26 GB/s/SM of one issuing thread is the thread's issue loop or the SM's TMA unit.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/micro/tma_issuers.bin scripts/micro/tma_issuers.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void stream(const __grid_constant__ CUtensorMap tm, int nblk, int loads, int per, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nw * per; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (lane != 0) return;
  unsigned long long t0 = clock64();
  uint32_t seed = blockIdx.x * 7919u + warp * 104729u + 13u;
  for (int i = 0; i < loads; ++i) {
    const int slot = warp * per + i % per;
    if (i >= per)
      asm volatile("{\n.reg .pred P;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}" ::"r"(
                       sa(&bar[slot])),
                   "r"(((i / per) - 1) & 1)
                   : "memory");
    seed = seed * 1664525u + 1013904223u;
    const int blk = (int)((seed >> 8) % (uint32_t)nblk), head = (seed >> 3) & 7;
    const uint32_t b = sa(&bar[slot]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(4096) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, "
        "%7}], [%2];" ::"r"(sa(s + (size_t)slot * 4096)),
        "l"(&tm), "r"(b), "r"(0), "r"(0), "r"(0), "r"(head), "r"(blk)
        : "memory");
  }
  for (int i = loads - per; i < loads; ++i)
    asm volatile("{\n.reg .pred P;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}" ::"r"(
                     sa(&bar[warp * per + i % per])),
                 "r"((i / per) & 1)
                 : "memory");
  if (warp == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  const int NB = 65536, BS = 16, H = 8, D = 128;
  uint8_t* d;
  if (cudaMalloc(&d, (size_t)NB * BS * H * D * 2) != cudaSuccess) return 1;
  cudaMemset(d, 0, (size_t)NB * BS * H * D * 2);
  unsigned long long* dout;
  cudaMalloc(&dout, 148 * 8);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap tm;
  cuuint64_t dims[5] = {64, (cuuint64_t)BS, 2, (cuuint64_t)H, (cuuint64_t)NB};
  cuuint64_t str[4] = {(cuuint64_t)H * D * 2, 128, (cuuint64_t)D * 2, (cuuint64_t)BS * H * D * 2};
  cuuint32_t box[5] = {64, 16, 2, 1, 1}, es[5] = {1, 1, 1, 1, 1};
  if (fn(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
    return 2;
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int grid : {36, 148}) {
    for (int warps : {1, 2, 4, 8, 16}) {
      const int per = 48 / warps;  // 192 KB in flight in total
      const int loads = 2048;
      stream<<<grid, warps * 32, 200 * 1024>>>(tm, NB, per * 2, per, dout);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      stream<<<grid, warps * 32, 200 * 1024>>>(tm, NB, loads / warps, per, dout);
      cudaEventRecord(e1);
      cudaError_t e = cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)grid * (loads / warps) * warps * 4096;
      printf("grid %3d issuing warps %2d (%2d slots each): %s %7.1f GB/s/SM, %.0f ns per box per SM\n", grid, warps, per,
             cudaGetErrorString(e), bytes / ms / 1e6 / grid, ms * 1e6 / ((double)(loads / warps) * warps));
    }
  }
  return 0;
}
