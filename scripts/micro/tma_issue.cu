// Microbenchmark: TMA issue cost / per-SM throughput for KV-cache-like boxes.
// One CTA per SM streams `rounds` x `per_round` boxes of {64 d, 16 slots, 2 halves} (4 KB,
// 5-D view of an NHD paged cache, random blocks) into shared memory.  Issuers: `lanes`
// lanes in each of `warps` warps, each issuing per_round/(lanes*warps) boxes per round.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void stream(const __grid_constant__ CUtensorMap tm, const int* blocks, int nblk, int rounds, int per_round,
                       int lanes, int warps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sa(&bar[0])));
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sa(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int issuers = lanes * warps;
  const int per = per_round / issuers;
  const bool me = warp < warps && lane < lanes;
  const int id = warp * lanes + lane;
  unsigned long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    uint32_t b = sa(&bar[r & 1]);
    if (threadIdx.x == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(per_round * 4096));
    __syncthreads();
    if (me) {
      for (int i = 0; i < per; ++i) {
        const int k = id * per + i;
        const int blk = blocks[(blockIdx.x * 7919 + r * per_round + k) % nblk];
        const uint32_t dst = sa(s) + (uint32_t)(k % 32) * 4096u;
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, "
            "%7}], [%2];" ::"r"(dst),
            "l"(&tm), "r"(b), "r"(0), "r"(0), "r"(0), "r"(k % 8), "r"(blk)
            : "memory");
      }
    }
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(b),
                 "r"((r >> 1) & 1));
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main(int argc, char** argv) {
  const int NB = 65536, BS = 16, H = 8, D = 128;  // 1 GiB of K
  size_t n = (size_t)NB * BS * H * D;
  void* d;
  if (cudaMalloc(&d, n * 2) != cudaSuccess) return 1;
  cudaMemset(d, 0, n * 2);
  std::vector<int> hb(NB);
  srand(1);
  for (int i = 0; i < NB; ++i) hb[i] = rand() % NB;
  int* db;
  cudaMalloc(&db, NB * 4);
  cudaMemcpy(db, hb.data(), NB * 4, cudaMemcpyHostToDevice);
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
         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return 2;
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  int cfg[][4] = {{16, 1, 1, 16}, {32, 1, 1, 16}, {16, 8, 1, 16}, {32, 32, 1, 16}, {32, 1, 4, 16}, {32, 8, 4, 16},
                  {16, 1, 1, 148}, {32, 1, 1, 148}, {32, 8, 1, 148}, {32, 1, 4, 148}, {32, 32, 1, 148}};
  for (auto& c : cfg) {
    int per_round = c[0], lanes = c[1], warps = c[2], grid = c[3];
    int rounds = 4096 / per_round * 4;
    stream<<<grid, 128, 140 * 1024>>>(tm, db, NB, 4, per_round, lanes, warps, dout);  // warm
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    stream<<<grid, 128, 140 * 1024>>>(tm, db, NB, rounds, per_round, lanes, warps, dout);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double bytes = (double)grid * rounds * per_round * 4096;
    std::vector<unsigned long long> h(grid);
    cudaMemcpy(h.data(), dout, grid * 8, cudaMemcpyDeviceToHost);
    double clk = 0;
    for (auto v : h) clk += v;
    clk /= grid;
    printf("in-flight %2d KB lanes %2d warps %d grid %3d: %s  %.1f GB/s total, %.1f GB/s/SM, %.1f B/clk/SM, %.0f clk/box\n",
           per_round * 4, lanes, warps, grid, cudaGetErrorString(e), bytes / ms / 1e6, bytes / ms / 1e6 / grid,
           bytes / grid / clk, clk / (rounds * (double)per_round));
  }
  return 0;
}
