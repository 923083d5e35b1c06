// common.cuh -- shared device helpers for the lmbp kernels (sm_100a).
// Product code: nothing here is shared with oracle/.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <type_traits>
#include <utility>

#include "constants.cuh"

namespace lmbp {

// ---------------------------------------------------------------------------
// Storage-type traits.  One 16-byte vector holds kVec elements.
// ---------------------------------------------------------------------------
template <typename T> struct Traits;
template <> struct Traits<float> {
  static constexpr int kVec = 4;
};
template <> struct Traits<__nv_bfloat16> {
  static constexpr int kVec = 8;
};
template <> struct Traits<__half> {
  static constexpr int kVec = 8;
};

__device__ __forceinline__ float bits_f32(uint32_t b) { return __uint_as_float(b); }

// ---------------------------------------------------------------------------
// Global memory: 128-bit streaming loads/stores.  Plain ld.global (no .nc) so
// exact aliasing (y == x, dx == dy) stays well defined; L1::no_allocate keeps
// streamed data from displacing anything in L1.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(uint4 *p, const uint4 &v) {
#ifdef LMBP_ST_CS
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
#else
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
#endif
}

// 32 contiguous bytes per thread in one 256-bit access (sm_100 .v8.b32): a
// warp instruction then covers 1 KB of whole sectors, where two 16-byte
// accesses at a 32-byte stride each touch every sector half.  p must be
// 32-byte aligned.
#ifndef LMBP_NO_V8
constexpr bool kUseV8 = true;
#else
constexpr bool kUseV8 = false;  // tuning knob: pairs of 16-byte accesses instead
#endif
__device__ __forceinline__ void st_stream32(uint4 *p, const uint4 &a, const uint4 &b) {
  asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(a.x),
               "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}
__device__ __forceinline__ void ld_stream32(const uint4 *p, uint4 &a, uint4 &b) {
  asm volatile("ld.global.L1::no_allocate.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
               : "l"(p));
}

// ---------------------------------------------------------------------------
// Element conversions (round-to-nearest-even, no FTZ).
// ---------------------------------------------------------------------------
template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
template <> __device__ __forceinline__ float to_f32<__half>(__half v) { return __half2float(v); }

template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
template <> __device__ __forceinline__ __half from_f32<__half>(float v) { return __float2half_rn(v); }

// 16-byte vector <-> kVec floats.
template <typename T> struct Vec;

template <> struct Vec<float> {
  __device__ __forceinline__ static void unpack(const uint4 &r, float *f) {
    f[0] = __uint_as_float(r.x);
    f[1] = __uint_as_float(r.y);
    f[2] = __uint_as_float(r.z);
    f[3] = __uint_as_float(r.w);
  }
  __device__ __forceinline__ static uint4 pack(const float *f) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                      __float_as_uint(f[3]));
  }
};

__device__ __forceinline__ void bf2_unpack(uint32_t w, float &lo, float &hi) {
  lo = __uint_as_float(w << 16);
  hi = __uint_as_float(w & 0xffff0000u);
}
__device__ __forceinline__ uint32_t bf2_pack(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);  // F2FP.BF16.F32.PACK_AB, RNE
  return *reinterpret_cast<uint32_t *>(&h);
}

template <> struct Vec<__nv_bfloat16> {
  __device__ __forceinline__ static void unpack(const uint4 &r, float *f) {
    bf2_unpack(r.x, f[0], f[1]);
    bf2_unpack(r.y, f[2], f[3]);
    bf2_unpack(r.z, f[4], f[5]);
    bf2_unpack(r.w, f[6], f[7]);
  }
  __device__ __forceinline__ static uint4 pack(const float *f) {
    return make_uint4(bf2_pack(f[0], f[1]), bf2_pack(f[2], f[3]), bf2_pack(f[4], f[5]),
                      bf2_pack(f[6], f[7]));
  }
};

__device__ __forceinline__ void h2_unpack(uint32_t w, float &lo, float &hi) {
  __half2 h = *reinterpret_cast<__half2 *>(&w);
  float2 f = __half22float2(h);
  lo = f.x;
  hi = f.y;
}
__device__ __forceinline__ uint32_t h2_pack(float lo, float hi) {
  __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&h);
}

template <> struct Vec<__half> {
  __device__ __forceinline__ static void unpack(const uint4 &r, float *f) {
    h2_unpack(r.x, f[0], f[1]);
    h2_unpack(r.y, f[2], f[3]);
    h2_unpack(r.z, f[4], f[5]);
    h2_unpack(r.w, f[6], f[7]);
  }
  __device__ __forceinline__ static uint4 pack(const float *f) {
    return make_uint4(h2_pack(f[0], f[1]), h2_pack(f[2], f[3]), h2_pack(f[4], f[5]),
                      h2_pack(f[6], f[7]));
  }
};

// ---------------------------------------------------------------------------
// MUFU wrappers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float ex2_approx(float x) {  // 2^x, FTZ
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {  // 1/x, FTZ
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ---------------------------------------------------------------------------
// Reductions (fixed order -> deterministic).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float2 warp_sum2(float2 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

// Runtime step table for the k-bit activations (stepact.cu): binary32
// thresholds rounded toward -inf and binary32 levels, k in {1, 2, 4}.
struct StepTable {
  float thr[15];
  float lvl[16];
  uint32_t thr2[15];  // bf16 / fp16 launches: RD_T(thr) duplicated into both halves (packed compares)
  int k;
};

// Device attribute helpers (host side).
int sm_count();

// ---------------------------------------------------------------------------
// Programmatic dependent launch (sm_90+).  Every hot-path kernel is launched
// with programmatic stream serialization, so when it follows another kernel
// on the stream its CTAs may be scheduled before that kernel has finished
// (once every CTA of it has executed launch_dependents or exited) and run
// their prologue -- launch, barrier init, the 128 KB table copy -- under the
// previous kernel's drain.  pdl_wait() (griddepcontrol.wait) then blocks
// until the previous grid has COMPLETED and its memory is visible, so it sits
// before the first global access that could depend on it: every load of an
// input and every store of an output (a store could race a read of the
// previous kernel: WAR).  Only immutable data (the module's constant tables,
// kernel parameters) is touched before it.  Launched without the attribute
// (LMBP_PDL=0, or after a non-kernel stream operation) both instructions are
// no-ops and the stream serialises as usual.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Entry of a kernel with no prologue worth overlapping.
__device__ __forceinline__ void pdl_enter() {
  pdl_wait();
  pdl_trigger();
}

bool pdl_enabled();  // abi.cu: LMBP_PDL environment variable, read once (default on)

// Launch `kernel` on `s` with programmatic stream serialization (when
// enabled).  Like <<<>>>, a failed launch leaves its error in the runtime's
// last-error slot: callers return cudaGetLastError().
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Opt a kernel into `bytes` of dynamic shared memory on the current device,
// once per (kernel instantiation, device).  Function attributes are per
// device, so a process driving several GPUs sets it on each.  `mask` is the
// caller's per-instantiation bitmask (devices 0..63); racing threads at worst
// set the same attribute twice.
template <typename K>
inline cudaError_t ensure_dyn_smem(K kernel, size_t bytes, std::atomic<unsigned long long> &mask) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cudaErrorInvalidDevice;
  const unsigned long long bit = 1ull << (dev & 63);
  if (mask.load(std::memory_order_acquire) & bit) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) mask.fetch_or(bit, std::memory_order_release);
  return e;
}

}  // namespace lmbp

namespace lmbp {
// ---------------------------------------------------------------------------
// mbarrier + bulk-async copy (TMA engine, non-tensor form) helpers, sm_90+.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LMBP_WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LMBP_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// global -> shared bulk copy (TMA engine), completion signalled on `bar`
// (bytes % 16 == 0, both addresses 16-byte aligned).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Cluster launch control (sm_100): ask the hardware to cancel a CTA of this
// grid that has not started yet; the response (16 bytes in shared memory)
// arrives on `bar` with complete_tx.  Hardware work stealing without any
// global counter (the library keeps no mutable global state).
__device__ __forceinline__ void clc_try_cancel(void *resp, uint64_t *bar) {
  asm volatile(
      "clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];" ::"r"(
          smem_u32(resp)),
      "r"(smem_u32(bar))
      : "memory");
}
// Returns the x index of the cancelled CTA, or -1 when nothing was cancelled.
__device__ __forceinline__ int clc_query(const void *resp) {
  uint32_t ok, cx;
  asm volatile(
      "{\n"
      ".reg .b128 r;\n"
      ".reg .pred p;\n"
      "ld.shared.b128 r, [%2];\n"
      "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, r;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %1, r;\n"
      "}\n"
      : "=r"(ok), "=r"(cx)
      : "r"(smem_u32(resp))
      : "memory");
  return ok ? (int)cx : -1;
}

__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint4 lds128(const void *p) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_u32(p)));
  return r;
}

// Row blocks of the warp-team kernels scheduled by cluster launch control:
// the grid has one CTA per block of `teams` rows, and a running CTA takes
// over the blocks of CTAs that have not started yet (hardware work stealing,
// as in ew_pipeline.cuh).  Unlike a persistent grid-stride loop, a CTA that
// starts late -- e.g. under programmatic dependent launch, once the previous
// kernel's CTAs have left its SM -- simply ends up with fewer blocks.
template <typename F>
__device__ __forceinline__ void clc_row_blocks(int64_t rows, int teams, int team_id, F &&body) {
  __shared__ __align__(16) uint4 resp;
  __shared__ uint64_t bar;
  __shared__ int next[2];
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  int64_t blk = blockIdx.x;
  for (uint32_t ph = 0;; ph ^= 1u) {
    if (threadIdx.x == 0) {  // ask for the next block now; the answer arrives while this one runs
      mbar_arrive_expect_tx(&bar, 16);
      clc_try_cancel(&resp, &bar);
    }
    const int64_t row = blk * teams + team_id;
    if (row < rows) body(row);
    if (threadIdx.x == 0) {
      mbar_wait(&bar, ph);
      next[ph] = clc_query(&resp);
    }
    __syncthreads();
    blk = next[ph];  // thread 0 rewrites next[ph] two iterations on, after a barrier every thread
                     // reaches only once it has read it here
    if (blk < 0) break;
  }
}

}  // namespace lmbp
