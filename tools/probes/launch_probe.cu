// launch_probe.cu -- fixed costs of the elementwise pipeline's launch shape on
// B200: empty CTAs with large dynamic smem, a CLC (cluster launch control)
// work-stealing loop with no work, a plain large grid; each launch preceded by
// a 2 x L2 read flush, CUDA events around the probe kernel only, median of 20.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void read_sum(const uint4 *a, size_t n, uint32_t *out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = a[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *out = acc;
}
__global__ void k_empty(int *out) {
  extern __shared__ int sm[];
  if (threadIdx.x == 1023) out[0] = sm[0];
}
__global__ void k_bar_init(int *out) {
  extern __shared__ __align__(16) uint64_t smb[];
  if (threadIdx.x == 0) {
    for (int s = 0; s < 9; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&smb[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 1023) out[0] = 1;
}
__global__ void k_clc(int *out) {
  extern __shared__ __align__(16) uint64_t smb[];
  __shared__ __align__(16) uint4 resp;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&smb[0])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t ph = 0;
  int n = 0;
  while (true) {
    uint32_t bar = (uint32_t)__cvta_generic_to_shared(&smb[0]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" ::"r"(bar) : "memory");
    asm volatile("clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&resp)), "r"(bar) : "memory");
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(bar), "r"(ph) : "memory");
    ph ^= 1;
    uint32_t ok;
    asm volatile("{\n.reg .b128 r;\n.reg .pred p;\nld.shared.b128 r, [%1];\nclusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, r;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(&resp)) : "memory");
    if (!ok) break;
    ++n;
  }
  if (n == 123456789) out[0] = n;
}

int main() {
  int sms = 0, l2 = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
  const size_t FL = std::max((size_t)2 * l2, (size_t)256 << 20);
  char *fl; uint32_t *sink; int *out;
  CK(cudaMalloc(&fl, FL)); CK(cudaMalloc(&sink, 4)); CK(cudaMalloc(&out, 4));
  CK(cudaMemset(fl, 0, FL));
  CK(cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(k_bar_init, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(k_clc, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto timeit = [&](const char *name, bool flush, auto launch) {
    std::vector<float> t;
    for (int it = 0; it < 23; ++it) {
      if (flush) read_sum<<<sms * 8, 256>>>((const uint4 *)fl, FL / 16, sink);
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      if (it >= 3) t.push_back(ms);
    }
    CK(cudaGetLastError());
    std::sort(t.begin(), t.end());
    printf("{\"probe\": \"%s\", \"flush\": %d, \"us\": %.2f}\n", name, (int)flush, t[t.size() / 2] * 1e3);
  };
  for (int fl_ : {1, 0}) {
    timeit("events only", fl_, [&] {});
    timeit("empty 296x544 smem0", fl_, [&] { k_empty<<<2 * sms, 544, 0>>>(out); });
    timeit("empty 296x544 smem70K", fl_, [&] { k_empty<<<2 * sms, 544, 70 * 1024>>>(out); });
    timeit("empty 148x544 smem200K", fl_, [&] { k_empty<<<sms, 544, 200 * 1024>>>(out); });
    timeit("bar_init 296x544 smem70K", fl_, [&] { k_bar_init<<<2 * sms, 544, 70 * 1024>>>(out); });
    timeit("empty grid 11000x544 smem70K", fl_, [&] { k_empty<<<11000, 544, 70 * 1024>>>(out); });
    timeit("clc grid 11000x544 smem70K", fl_, [&] { k_clc<<<11000, 544, 70 * 1024>>>(out); });
    timeit("clc grid 296x544 smem70K", fl_, [&] { k_clc<<<296, 544, 70 * 1024>>>(out); });
    timeit("clc grid 2400x544 smem70K", fl_, [&] { k_clc<<<2400, 544, 70 * 1024>>>(out); });
    timeit("empty grid 2400x544 smem70K", fl_, [&] { k_empty<<<2400, 544, 70 * 1024>>>(out); });
  }
  return 0;
}
