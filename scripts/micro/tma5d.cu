// Probe: does cuTensorMapEncodeTiled accept a 5-D KV view with a non-monotonic stride order
// {d_lo 64, slot 16, d_hi 2, head, block} (one box = K of one 16-key sub-block, both d-halves)?
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap tm, int head, int blk, unsigned short* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint32_t sb = (uint32_t)__cvta_generic_to_shared(s), bb = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bb));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bb), "r"(4096));
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
                 ::"r"(sb), "l"(&tm), "r"(bb), "r"(0), "r"(0), "r"(0), "r"(head), "r"(blk) : "memory");
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"(bb));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) {
    int row = i / 64, e = i % 64;  // row = half*16 + slot
    int ch = (e / 8) ^ (row & 7);
    out[i] = *reinterpret_cast<unsigned short*>(s + row * 128 + ch * 16 + (e % 8) * 2);
  }
}

int main() {
  const int NB = 4, BS = 16, H = 8, D = 128;
  std::vector<unsigned short> h((size_t)NB * BS * H * D);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (unsigned short)(i & 0xffff);
  unsigned short *d, *o;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&o, 4096);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap tm;
  cuuint64_t dims[5] = {64, (cuuint64_t)BS, 2, (cuuint64_t)H, (cuuint64_t)NB};
  cuuint64_t str[4] = {(cuuint64_t)H * D * 2, 128, (cuuint64_t)D * 2, (cuuint64_t)BS * H * D * 2};
  cuuint32_t box[5] = {64, 16, 2, 1, 1}, es[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode 5d non-monotonic: %d\n", (int)r);
  if (r != CUDA_SUCCESS) return 1;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  probe<<<1, 128, 8192>>>(tm, 3, 2, o);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<unsigned short> g(2048);
  cudaMemcpy(g.data(), o, 4096, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 2048; ++i) {
    int row = i / 64, e2 = i % 64, half = row / 16, slot = row % 16;
    size_t src = (((size_t)2 * BS + slot) * H + 3) * D + half * 64 + e2;
    if (g[i] != h[src]) ++bad;
  }
  printf("kernel %s, mismatches %d / 2048\n", cudaGetErrorString(e), bad);
  return bad != 0;
}
