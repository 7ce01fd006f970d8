// Microbenchmark: per-SM streaming rate of paged-KV-like loads into shared memory (no
// consumers): how fast can ONE SM pull K/V from HBM with each load shape, at a given depth of
// bytes in flight?  One CTA per SM, thread 0 keeps `depth` ring slots in flight (mbarrier per
// slot), random 32 KB blocks out of a 2 GiB NHD cache [block][16 slots][8 heads][128 d] bf16.
//   shape 0: 5-D TMA box {64 d, 16 slots, 2 halves, 1 head, 1 block} = 4 KB (K2 today)
//   shape 1: 4-D TMA box {64 d, 2 halves, 8 heads, 16 slots} of one block = 32 KB (all heads)
//   shape 2: 1-D cp.async.bulk of the whole 32 KB block (contiguous in NHD)
//   shape 3: 1-D cp.async.bulk of 4 KB (one head's 16 slots in an HND layout: contiguous)
//   shape 4: the shape-0 map with box {64 d, 16 slots, 2 halves, 8 heads, 1 block} = 32 KB
//            (lands as 8 head-major copies of the shape-0 layout)
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/kv_stream scripts/micro/kv_stream.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t par) {
  asm volatile("{\n.reg .pred P;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}" ::"r"(bar),
               "r"(par)
               : "memory");
}

__global__ void stream(const __grid_constant__ CUtensorMap tm5, const __grid_constant__ CUtensorMap tm4,
                       const __grid_constant__ CUtensorMap tm5w,
                       const uint8_t* base, const int* blocks, int nblk, int shape, int loads, int depth,
                       unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar[64];
  const uint32_t bytes = (shape == 0 || shape == 3) ? 4096u : 32768u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned long long t0 = clock64();
  uint32_t seed = blockIdx.x * 7919u + 13u;
  for (int i = 0; i < loads; ++i) {
    const int slot = i % depth;
    if (i >= depth) wait(sa(&bar[slot]), ((i / depth) - 1) & 1);
    seed = seed * 1664525u + 1013904223u;
    const int blk = (int)((seed >> 8) % (uint32_t)nblk);  // no dependent table load on the issue path
    const uint32_t dst = sa(s + (size_t)slot * bytes), b = sa(&bar[slot]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    if (shape == 0) {
      const int head = (seed >> 3) & 7;
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
          "%6, %7}], [%2];" ::"r"(dst),
          "l"(&tm5), "r"(b), "r"(0), "r"(0), "r"(0), "r"(head), "r"(blk)
          : "memory");
    } else if (shape == 4) {
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
          "%6, %7}], [%2];" ::"r"(dst),
          "l"(&tm5w), "r"(b), "r"(0), "r"(0), "r"(0), "r"(0), "r"(blk)
          : "memory");
    } else if (shape == 1) {
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
          "%6, %7}], [%2];" ::"r"(dst),
          "l"(&tm4), "r"(b), "r"(0), "r"(0), "r"(0), "r"(0), "r"(blk)
          : "memory");
    } else {
      const uint8_t* src = base + (size_t)blk * 32768u + (shape == 3 ? ((seed >> 3) & 7) * 4096u : 0u);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                   "l"(src), "r"(bytes), "r"(b)
                   : "memory");
    }
  }
  for (int i = loads - depth; i < loads; ++i) wait(sa(&bar[i % depth]), (i / depth) & 1);
  out[blockIdx.x] = clock64() - t0;
}

int main() {
  const int NB = 65536, BS = 16, H = 8, D = 128;  // 2 GiB
  const size_t n = (size_t)NB * BS * H * D;
  uint8_t* d;
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
  CUtensorMap tm5, tm4, tm5w;
  {  // {d_lo 64, slot, d_hi 2, head, block}
    cuuint64_t dims[5] = {64, (cuuint64_t)BS, 2, (cuuint64_t)H, (cuuint64_t)NB};
    cuuint64_t str[4] = {(cuuint64_t)H * D * 2, 128, (cuuint64_t)D * 2, (cuuint64_t)BS * H * D * 2};
    cuuint32_t box[5] = {64, 16, 2, 1, 1}, es[5] = {1, 1, 1, 1, 1};
    if (fn(&tm5, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
      return 2;
    cuuint32_t boxw[5] = {64, 16, 2, (cuuint32_t)H, 1};
    if (fn(&tm5w, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, d, dims, str, boxw, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
      return 4;
  }
  {  // {d_lo 64, d_hi 2, head 8, slot 16, block}: the whole block in one box
    cuuint64_t dims[5] = {64, 2, (cuuint64_t)H, (cuuint64_t)BS, (cuuint64_t)NB};
    cuuint64_t str[4] = {128, (cuuint64_t)D * 2, (cuuint64_t)H * D * 2, (cuuint64_t)BS * H * D * 2};
    cuuint32_t box[5] = {64, 2, (cuuint32_t)H, (cuuint32_t)BS, 1}, es[5] = {1, 1, 1, 1, 1};
    CUresult r = fn(&tm4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) {
      printf("encode all-heads box failed %d\n", (int)r);
      return 3;
    }
  }
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[5] = {"tma5d 4KB/head", "tma 32KB/block", "bulk 32KB", "bulk 4KB", "tma5d 8 heads"};
  for (int grid : {1, 36, 148}) {
    for (int shape = 0; shape < 5; ++shape) {
      const int kb = (shape == 0 || shape == 3) ? 4 : 32;
      for (int inflight : {32, 64, 128, 192}) {
        const int depth = inflight / kb;
        if (depth < 1 || depth > 64) continue;
        const int loads = (grid == 148 ? 2048 : 8192) * 4 / kb;
        stream<<<grid, 32, 200 * 1024>>>(tm5, tm4, tm5w, d, db, NB, shape, depth * 2, depth, dout);  // warm
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        stream<<<grid, 32, 200 * 1024>>>(tm5, tm4, tm5w, d, db, NB, shape, loads, depth, dout);
        cudaEventRecord(e1);
        cudaError_t e = cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = (double)grid * loads * kb * 1024;
        printf("grid %3d %-15s in-flight %3d KB: %s %8.1f GB/s total %6.1f GB/s/SM\n", grid, names[shape], inflight,
               cudaGetErrorString(e), bytes / ms / 1e6, bytes / ms / 1e6 / grid);
      }
    }
  }
  return 0;
}
