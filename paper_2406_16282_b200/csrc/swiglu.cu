// swiglu.cu -- fused ReSwiGLU2: the LLaMA MLP gate h = SiLU(gate) * up with
// ReSiLU2's 2-bit backward.
//
// LLaMA uses SwiGLU; the paper replaces its SiLU by ReSiLU2
// (P:L413-416).  Unfused, that is three kernels (ReSiLU2 fwd, mul fwd; mul
// bwd, ReSiLU2 bwd) and an extra round trip of an [R, F] tensor each way.
// Fused, with the exact composition semantics of the unfused ops:
//   forward : a = RN_T(SiLU(gate)), h = RN_T(a * up), code = #{i : gate > c_i}
//             saved for backward: codes (2 bits), a and up (the mul's inputs)
//   backward: dup   = RN_T(dh * a)
//             da    = RN_T(dh * up)                  (the mul's grad wrt a)
//             dgate = RN_T(RN32(da * RN32(s[code])))  (ReSiLU2 backward, reading R5)
// Bytes per element: forward 4b + 1/4 (read gate, up; write h, a, codes),
// backward 5b + 1/4 (read dh, up, a, codes; write dgate, dup).
#include "act_math.cuh"
#include "common.cuh"
#include "ew_pipeline.cuh"
#include "kernels.h"

// Pipeline shapes (tools/sweep.py knobs): consumer warps x vectors per lane x stages.
#ifndef LMBP_SWF_W
#define LMBP_SWF_W 16
#define LMBP_SWF_U 2
#define LMBP_SWF_S 3
#endif
#ifndef LMBP_SWB_W
#define LMBP_SWB_W 12
#define LMBP_SWB_U 2
#define LMBP_SWB_S 3
#endif

namespace lmbp {

template <typename T, bool kPrecise>
__device__ __forceinline__ void swiglu_fwd_elem(float g, float u, T &h, T &a) {
  const T aT = from_f32<T>(silu_f<kPrecise>(g));
  a = aT;
  h = from_f32<T>(__fmul_rn(to_f32<T>(aT), u));
}

template <typename T>
__device__ __forceinline__ void swiglu_bwd_elem(float dh, float u, float a, uint32_t c, T &dg, T &du) {
  du = from_f32<T>(__fmul_rn(dh, a));
  const float da = to_f32<T>(from_f32<T>(__fmul_rn(dh, u)));
  dg = from_f32<T>(__fmul_rn(da, level<kActSilu>(c)));
}

template <typename T, bool kPrecise>
struct SwiGluFwdOp {
  static constexpr int W = LMBP_SWF_W, U = LMBP_SWF_U, S = LMBP_SWF_S, kIn = 2, kCodeIn = 0,
                       kCodeOut = Traits<T>::kVec / 4;
  __device__ static uint32_t apply(const uint4 (&v)[2], uint32_t, int64_t i, const EwParams &p) {
    constexpr int kVec = Traits<T>::kVec;
    float g[kVec], u[kVec], a[kVec];
    Vec<T>::unpack(v[0], g);
    Vec<T>::unpack(v[1], u);
    uint32_t c;
    if constexpr (kVec == 4) c = codes_vec_f32<kActSilu>(g);
    else c = codes_vec_16<T, kActSilu>(v[0]);
#pragma unroll
    for (int k = 0; k < kVec; k += 2) {
      const float2 r = act2_f<kActSilu, kPrecise>(make_float2(g[k], g[k + 1]));
      a[k] = r.x;
      a[k + 1] = r.y;
    }
    const uint4 aT = Vec<T>::pack(a);
    Vec<T>::unpack(aT, a);  // the stored (rounded) a is the mul's operand
#pragma unroll
    for (int k = 0; k < kVec; ++k) a[k] = __fmul_rn(a[k], u[k]);
    st_stream(p.out[0] + i, Vec<T>::pack(a));
    st_stream(p.out[1] + i, aT);
    return c;
  }
  __device__ static void tail(const EwParams &p) {
    const T *g = reinterpret_cast<const T *>(p.in[0]);
    const T *u = reinterpret_cast<const T *>(p.in[1]);
    T *h = reinterpret_cast<T *>(p.out[0]);
    T *a = reinterpret_cast<T *>(p.out[1]);
    for (int64_t b = (p.nvec * Traits<T>::kVec) >> 2; 4 * b < p.n; ++b) {
      uint32_t byte = 0;
      for (int k = 0; k < 4 && 4 * b + k < p.n; ++k) {
        const int64_t j = 4 * b + k;
        const float gj = to_f32<T>(g[j]);
        const float uj = to_f32<T>(u[j]);
        swiglu_fwd_elem<T, kPrecise>(gj, uj, h[j], a[j]);
        byte |= code_f32<kActSilu>(gj) << (2 * k);
      }
      p.codes_out[b] = (uint8_t)byte;
    }
  }
};

template <typename T>
struct SwiGluBwdOp {
  static constexpr int W = LMBP_SWB_W, U = LMBP_SWB_U, S = LMBP_SWB_S, kIn = 3, kCodeIn = Traits<T>::kVec / 4,
                       kCodeOut = 0;
  __device__ static uint32_t apply(const uint4 (&v)[3], uint32_t c, int64_t i, const EwParams &p) {
    constexpr int kVec = Traits<T>::kVec;
    float dh[kVec], u[kVec], a[kVec];
    Vec<T>::unpack(v[0], dh);
    Vec<T>::unpack(v[1], u);
    Vec<T>::unpack(v[2], a);
#pragma unroll
    for (int k = 0; k < kVec; ++k) {
      a[k] = __fmul_rn(dh[k], a[k]);  // dup
      u[k] = __fmul_rn(dh[k], u[k]);  // da (rounded to T below)
    }
    st_stream(p.out[1] + i, Vec<T>::pack(a));
    Vec<T>::unpack(Vec<T>::pack(u), u);
#pragma unroll
    for (int k = 0; k < kVec; ++k) u[k] = __fmul_rn(u[k], level<kActSilu>((c >> (2 * k)) & 3u));
    st_stream(p.out[0] + i, Vec<T>::pack(u));
    return 0u;
  }
  __device__ static void tail(const EwParams &p) {
    const T *dh = reinterpret_cast<const T *>(p.in[0]);
    const T *u = reinterpret_cast<const T *>(p.in[1]);
    const T *a = reinterpret_cast<const T *>(p.in[2]);
    T *dg = reinterpret_cast<T *>(p.out[0]);
    T *du = reinterpret_cast<T *>(p.out[1]);
    for (int64_t j = p.nvec * Traits<T>::kVec; j < p.n; ++j) {
      const uint32_t cj = (p.codes_in[j >> 2] >> (2 * (j & 3))) & 3u;
      swiglu_bwd_elem<T>(to_f32<T>(dh[j]), to_f32<T>(u[j]), to_f32<T>(a[j]), cj, dg[j], du[j]);
    }
  }
};

// Scalar fallbacks (any alignment): one code byte (4 elements) per thread.
template <typename T, bool kPrecise>
__global__ void __launch_bounds__(256) swiglu_fwd_scalar(const T *g, const T *u, T *h, T *a, uint8_t *codes,
                                                         int64_t n) {
  pdl_enter();
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < (n + 3) / 4;
       b += (int64_t)gridDim.x * blockDim.x) {
    uint32_t byte = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t j = 4 * b + k;
      if (j < n) {
        const float gj = to_f32<T>(g[j]);
        const float uj = to_f32<T>(u[j]);
        swiglu_fwd_elem<T, kPrecise>(gj, uj, h[j], a[j]);
        byte |= code_f32<kActSilu>(gj) << (2 * k);
      }
    }
    codes[b] = (uint8_t)byte;
  }
}

template <typename T>
__global__ void __launch_bounds__(256) swiglu_bwd_scalar(const T *dh, const T *u, const T *a, const uint8_t *codes,
                                                         T *dg, T *du, int64_t n) {
  pdl_enter();
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t cj = (codes[j >> 2] >> (2 * (j & 3))) & 3u;
    swiglu_bwd_elem<T>(to_f32<T>(dh[j]), to_f32<T>(u[j]), to_f32<T>(a[j]), cj, dg[j], du[j]);
  }
}

static bool al16(const void *p) { return (uintptr_t)p % 16 == 0; }

static int scalar_grid(int64_t work) {
  const int64_t want = (work + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count() * 8));
}

template <typename T>
static cudaError_t swiglu_fwd_t(const void *g, const void *u, void *h, void *a, uint8_t *codes, int64_t n,
                                cudaStream_t s) {
  constexpr int kVec = Traits<T>::kVec;
  constexpr bool kPrecise = std::is_same<T, float>::value;
  if (al16(g) && al16(u) && al16(h) && al16(a) && al16(codes)) {
    EwParams p{};
    p.in[0] = reinterpret_cast<const uint4 *>(g);
    p.in[1] = reinterpret_cast<const uint4 *>(u);
    p.out[0] = reinterpret_cast<uint4 *>(h);
    p.out[1] = reinterpret_cast<uint4 *>(a);
    p.codes_out = codes;
    p.nvec = n / kVec;
    p.n = n;
    return launch_ew<SwiGluFwdOp<T, kPrecise>>(p, s);
  }
  launch_k(swiglu_fwd_scalar<T, kPrecise>, scalar_grid((n + 3) / 4), 256, 0, s,
           reinterpret_cast<const T *>(g), reinterpret_cast<const T *>(u), reinterpret_cast<T *>(h),
           reinterpret_cast<T *>(a), codes, n);
  return cudaGetLastError();
}

template <typename T>
static cudaError_t swiglu_bwd_t(const void *dh, const void *u, const void *a, const uint8_t *codes, void *dg,
                                void *du, int64_t n, cudaStream_t s) {
  constexpr int kVec = Traits<T>::kVec;
  if (al16(dh) && al16(u) && al16(a) && al16(dg) && al16(du) && al16(codes)) {
    EwParams p{};
    p.in[0] = reinterpret_cast<const uint4 *>(dh);
    p.in[1] = reinterpret_cast<const uint4 *>(u);
    p.in[2] = reinterpret_cast<const uint4 *>(a);
    p.codes_in = codes;
    p.out[0] = reinterpret_cast<uint4 *>(dg);
    p.out[1] = reinterpret_cast<uint4 *>(du);
    p.nvec = n / kVec;
    p.n = n;
    return launch_ew<SwiGluBwdOp<T>>(p, s);
  }
  launch_k(swiglu_bwd_scalar<T>, scalar_grid(n), 256, 0, s, reinterpret_cast<const T *>(dh), reinterpret_cast<const T *>(u),
           reinterpret_cast<const T *>(a), codes, reinterpret_cast<T *>(dg),
           reinterpret_cast<T *>(du), n);
  return cudaGetLastError();
}

cudaError_t swiglu_fwd(int dtype, const void *g, const void *u, void *h, void *a, uint8_t *codes, int64_t n,
                       cudaStream_t s) {
  if (dtype == 0) return swiglu_fwd_t<float>(g, u, h, a, codes, n, s);
  if (dtype == 1) return swiglu_fwd_t<__nv_bfloat16>(g, u, h, a, codes, n, s);
  return swiglu_fwd_t<__half>(g, u, h, a, codes, n, s);
}

cudaError_t swiglu_bwd(int dtype, const void *dh, const void *u, const void *a, const uint8_t *codes, void *dg,
                       void *du, int64_t n, cudaStream_t s) {
  if (dtype == 0) return swiglu_bwd_t<float>(dh, u, a, codes, dg, du, n, s);
  if (dtype == 1) return swiglu_bwd_t<__nv_bfloat16>(dh, u, a, codes, dg, du, n, s);
  return swiglu_bwd_t<__half>(dh, u, a, codes, dg, du, n, s);
}

}  // namespace lmbp
