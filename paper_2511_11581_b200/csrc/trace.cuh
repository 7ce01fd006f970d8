// Debug-only timeline instrumentation (build with make EXTRA=-DPATTN_TRACE; never in the
// product build).  Each kernel file defines its own device buffers (no -rdc):
//   PATTN_CTA_TRACE_DEFINE(name)  -> per-CTA {start ns, end ns, smid, items} for the last
//                                    launch and an exported reader pattn_debug_<name>_cta
//   PATTN_EV_TRACE_DEFINE(name)   -> 8 event types x 4096 slots of clock64 stamps of CTA 0
//                                    and an exported reader pattn_debug_<name>_ev
#pragma once
#ifdef PATTN_TRACE
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pattn_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned pattn_smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}

#define PATTN_CTA_TRACE_DEFINE(name)                                                                      \
  __device__ unsigned long long g_##name##_cta[2048][4];                                                  \
  extern "C" __attribute__((visibility("default"))) int pattn_debug_##name##_cta(unsigned long long* host, \
                                                                                 int cap) {               \
    static unsigned long long tmp[2048][4];                                                                \
    cudaMemcpyFromSymbol(tmp, g_##name##_cta, sizeof(tmp));                                                \
    int n = cap < 2048 ? cap : 2048;                                                                       \
    for (int i = 0; i < n; ++i)                                                                            \
      for (int j = 0; j < 4; ++j) host[4 * i + j] = tmp[i][j];                                             \
    return n;                                                                                              \
  }
#define PATTN_CTA_BEGIN(name) const unsigned long long pattn_t_begin = pattn_globaltimer()
#define PATTN_CTA_END(name, items)                                       \
  do {                                                                   \
    if (blockIdx.x < 2048) {                                             \
      g_##name##_cta[blockIdx.x][0] = pattn_t_begin;                     \
      g_##name##_cta[blockIdx.x][1] = pattn_globaltimer();               \
      g_##name##_cta[blockIdx.x][2] = pattn_smid();                      \
      g_##name##_cta[blockIdx.x][3] = (unsigned long long)(items);       \
    }                                                                    \
  } while (0)

#define PATTN_EV_TRACE_DEFINE(name)                                                                       \
  __device__ unsigned long long g_##name##_ev[8][4096];                                                   \
  extern "C" __attribute__((visibility("default"))) int pattn_debug_##name##_ev(unsigned long long* host,  \
                                                                                int cap, int reset) {     \
    static unsigned long long tmp[8][4096];                                                                \
    cudaMemcpyFromSymbol(tmp, g_##name##_ev, sizeof(tmp));                                                 \
    int k = 0;                                                                                             \
    for (int t = 0; t < 8; ++t)                                                                            \
      for (int i = 0; i < 4096 && k < cap; ++i, ++k) host[k] = tmp[t][i];                                  \
    if (reset) {                                                                                           \
      static unsigned long long z[8][4096];                                                                \
      cudaMemcpyToSymbol(g_##name##_ev, z, sizeof(z));                                                     \
    }                                                                                                      \
    return k;                                                                                              \
  }
// event slot [type][idx] of CTA 0 := clock64 (store only: no atomics on the traced path)
#define PATTN_EV(name, type, idx)                                    \
  do {                                                               \
    if (blockIdx.x == 0 && (unsigned)(idx) < 4096u)                  \
      g_##name##_ev[(type)][(idx)] = clock64();                      \
  } while (0)
#else
#define PATTN_CTA_TRACE_DEFINE(name)
#define PATTN_EV_TRACE_DEFINE(name)
#define PATTN_CTA_BEGIN(name) \
  do {                        \
  } while (0)
#define PATTN_CTA_END(name, items) \
  do {                             \
  } while (0)
#define PATTN_EV(name, type, idx) \
  do {                            \
  } while (0)
#endif
