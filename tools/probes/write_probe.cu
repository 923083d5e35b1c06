// write_probe.cu -- HBM write-path probe on B200: st.global.v4 vs .v8 vs
// TMA bulk store (cp.async.bulk.global.shared::cta), fills and copies, with
// L2 flushed (read of 2 x L2) before every launch, CUDA events, median of 15.
// Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o wp write_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void fill_v4(uint4 *p, size_t n) {
  uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__global__ void fill_v4_na(uint4 *p, size_t n) {
  uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__global__ void fill_v4_cs(uint4 *p, size_t n) {
  uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__global__ void fill_v8(uint4 *p, size_t n) {  // n in 16-byte units, 32-byte stores
  uint32_t a = threadIdx.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; 2 * i < n; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(p + 2 * i), "r"(a) : "memory");
}
__global__ void fill_v4_ef(uint4 *p, size_t n) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol) : "memory");
}
// TMA bulk store: one elected thread per CTA streams CHUNK-byte pieces from a
// smem buffer to global, keeping up to DEPTH bulk groups in flight.
template <int CHUNK, int DEPTH>
__global__ void fill_tma(char *p, size_t bytes) {
  extern __shared__ __align__(128) char sm[];
  for (int i = threadIdx.x; i < CHUNK / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t nchunks = bytes / CHUNK;
  int inflight = 0;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + c * CHUNK),
                 "r"((uint32_t)__cvta_generic_to_shared(sm)), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    ++inflight;
    if (inflight >= DEPTH) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(DEPTH - 1) : "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__global__ void copy_v4(const uint4 *a, uint4 *b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a + i));
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(b + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  }
}
__global__ void copy_v4_u4(const uint4 *a, uint4 *b, size_t n) {  // 4 loads in flight per thread
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += 4 * stride) {
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (i + j * stride < n)
        asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[j].x), "=r"(v[j].y), "=r"(v[j].z), "=r"(v[j].w) : "l"(a + i + j * stride));
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (i + j * stride < n)
        asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(b + i + j * stride), "r"(v[j].x), "r"(v[j].y), "r"(v[j].z), "r"(v[j].w) : "memory");
  }
}
// TMA copy: load CHUNK into a smem ring slot (mbarrier), store it back out with a bulk store.
template <int CHUNK, int S>
__global__ void copy_tma(const char *a, char *b, size_t bytes) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bar[S];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t nchunks = bytes / CHUNK;
  size_t mine[64];
  int cnt = 0;
  // issue loads for the first S chunks, then loop: wait load k, store k, (after its read completes) reload slot
  uint32_t ph[S];
  for (int s = 0; s < S; ++s) ph[s] = 0;
  size_t c = blockIdx.x;
  int k = 0;
  auto load = [&](size_t ch, int s) {
    uint32_t bs = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bs), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(sm + s * CHUNK)), "l"(a + ch * CHUNK), "r"(CHUNK), "r"(bs) : "memory");
  };
  size_t pend[S];
  int np = 0;
  for (int s = 0; s < S && c < nchunks; ++s, c += gridDim.x) { load(c, s); pend[s] = c; ++np; }
  (void)mine; (void)cnt;
  int s = 0;
  while (np > 0) {
    uint32_t bs = (uint32_t)__cvta_generic_to_shared(&bar[s]);
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(bs), "r"(ph[s]) : "memory");
    ph[s] ^= 1;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(b + pend[s] * CHUNK),
                 "r"((uint32_t)__cvta_generic_to_shared(sm + s * CHUNK)), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // slot free again
    --np;
    if (c < nchunks) { load(c, s); pend[s] = c; ++np; c += gridDim.x; }
    s = (s + 1) % S;
    ++k;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__global__ void read_sum(const uint4 *a, size_t n, uint32_t *out) {
  uint32_t acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(a + i));
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *out = acc;
}

int main(int argc, char **argv) {
  const size_t BYTES = (size_t)1 << 30;
  const size_t n = BYTES / 16;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int l2 = 0;
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0));
  char *a, *b, *fl;
  uint32_t *sink;
  CK(cudaMalloc(&a, BYTES));
  CK(cudaMalloc(&b, BYTES));
  const size_t FL = std::max((size_t)2 * l2, (size_t)256 << 20);
  CK(cudaMalloc(&fl, FL));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(a, 1, BYTES));
  CK(cudaMemset(fl, 0, FL));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto flush = [&]() { read_sum<<<sms * 8, 256>>>((const uint4 *)fl, FL / 16, sink); };
  auto timeit = [&](const char *name, double bytes_moved, auto launch) {
    std::vector<float> t;
    for (int it = 0; it < 18; ++it) {
      flush();
      CK(cudaEventRecord(e0));
      launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (it >= 3) t.push_back(ms);
    }
    CK(cudaGetLastError());
    std::sort(t.begin(), t.end());
    float med = t[t.size() / 2];
    printf("{\"probe\": \"%s\", \"us\": %.2f, \"GB/s\": %.1f}\n", name, med * 1e3, bytes_moved / (med * 1e-3) / 1e9);
  };
  for (int g : {1, 2, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "fill_v4 grid=%dxSM", g);
    timeit(nm, BYTES, [&] { fill_v4<<<sms * g, 512>>>((uint4 *)b, n); });
  }
  timeit("fill_v4_noalloc 4xSM", BYTES, [&] { fill_v4_na<<<sms * 4, 512>>>((uint4 *)b, n); });
  timeit("fill_v4_cs 4xSM", BYTES, [&] { fill_v4_cs<<<sms * 4, 512>>>((uint4 *)b, n); });
  timeit("fill_v4_evict_first 4xSM", BYTES, [&] { fill_v4_ef<<<sms * 4, 512>>>((uint4 *)b, n); });
  timeit("fill_v8 4xSM", BYTES, [&] { fill_v8<<<sms * 4, 512>>>((uint4 *)b, n); });
  timeit("memset", BYTES, [&] { cudaMemsetAsync(b, 0, BYTES); });
  {
    auto k1 = fill_tma<16384, 4>;
    CK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
    for (int g : {1, 2, 4}) {
      char nm[64];
      snprintf(nm, 64, "fill_tma 16KB d4 grid=%dxSM", g);
      timeit(nm, BYTES, [&] { k1<<<sms * g, 128, 16384>>>(b, BYTES); });
    }
    auto k2 = fill_tma<32768, 8>;
    CK(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768));
    timeit("fill_tma 32KB d8 grid=2xSM", BYTES, [&] { k2<<<sms * 2, 128, 32768>>>(b, BYTES); });
    auto k3 = fill_tma<4096, 16>;
    CK(cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096));
    timeit("fill_tma 4KB d16 grid=4xSM", BYTES, [&] { k3<<<sms * 4, 128, 4096>>>(b, BYTES); });
  }
  timeit("read 4xSM", BYTES, [&] { read_sum<<<sms * 4, 512>>>((const uint4 *)a, n, sink); });
  timeit("copy_v4 4xSM", 2.0 * BYTES, [&] { copy_v4<<<sms * 4, 512>>>((const uint4 *)a, (uint4 *)b, n); });
  timeit("copy_v4_u4 4xSM", 2.0 * BYTES, [&] { copy_v4_u4<<<sms * 4, 512>>>((const uint4 *)a, (uint4 *)b, n); });
  timeit("cudaMemcpy D2D", 2.0 * BYTES, [&] { cudaMemcpyAsync(b, a, BYTES, cudaMemcpyDeviceToDevice); });
  {
    auto k = copy_tma<16384, 4>;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384));
    for (int g : {1, 2, 3}) {
      char nm[64];
      snprintf(nm, 64, "copy_tma 16KBx4 grid=%dxSM", g);
      timeit(nm, 2.0 * BYTES, [&] { k<<<sms * g, 32, 4 * 16384>>>(a, b, BYTES); });
    }
    auto k8 = copy_tma<16384, 8>;
    CK(cudaFuncSetAttribute(k8, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384));
    timeit("copy_tma 16KBx8 grid=1xSM", 2.0 * BYTES, [&] { k8<<<sms, 32, 8 * 16384>>>(a, b, BYTES); });
  }
  return 0;
}
