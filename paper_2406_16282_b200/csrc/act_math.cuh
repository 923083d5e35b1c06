// act_math.cuh -- element math of ReGELU2 / ReSiLU2 shared by the activation
// kernels (act.cu) and the fused ReSwiGLU2 kernels (swiglu.cu).
//   forward : y = GELU(x) or SiLU(x), unchanged;
//             code = #{i : x > c_i}, 2 bits per element.
//   backward: dx = dy * s[code], s = (0, a1, a1 + a2, 1).
// GELU is evaluated branch-free as max(x,-0) - |x| e^{-x^2/2} G(|x|),
// G(u) = Phi(-u) e^{u^2/2} ~= t P6(t), t = 1/(1 + k u); SiLU as
// max(x,-0) - u e^{-u} / (1 + e^{-u}) with e^{-u} = (e^{-u/2})^2.  fp32 outputs
// add an exact split of the exponent argument ("precise").  The relu term is
// max(x, -0), so a negative x whose product underflows returns -0, the sign
// of the exact value (x Phi(x), x sigma(x) < 0), and x = +-0 returns +-0.
#pragma once
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace lmbp {

template <int A> struct Tab;
template <> struct Tab<kActGelu> {
  static constexpr uint32_t t0 = kGELU_THR_F32[0], t1 = kGELU_THR_F32[1], t2 = kGELU_THR_F32[2];
  static constexpr uint16_t b0 = kGELU_THR_BF16[0], b1 = kGELU_THR_BF16[1], b2 = kGELU_THR_BF16[2];
  static constexpr uint16_t h0 = kGELU_THR_F16[0], h1 = kGELU_THR_F16[1], h2 = kGELU_THR_F16[2];
  static constexpr uint32_t s1 = kGELU_LVL_F32[1], s2 = kGELU_LVL_F32[2];
};
template <> struct Tab<kActSilu> {
  static constexpr uint32_t t0 = kSILU_THR_F32[0], t1 = kSILU_THR_F32[1], t2 = kSILU_THR_F32[2];
  static constexpr uint16_t b0 = kSILU_THR_BF16[0], b1 = kSILU_THR_BF16[1], b2 = kSILU_THR_BF16[2];
  static constexpr uint16_t h0 = kSILU_THR_F16[0], h1 = kSILU_THR_F16[1], h2 = kSILU_THR_F16[2];
  static constexpr uint32_t s1 = kSILU_LVL_F32[1], s2 = kSILU_LVL_F32[2];
};

struct GeluPoly {  // degree 6 (tools/gen_kernel_constants.py: max rel. error 7.9e-7 on [0, 13.5])
  static_assert(kGeluDeg == 6, "Horner below is written for degree 6");
  static constexpr uint32_t p0 = kGeluP[0], p1 = kGeluP[1], p2 = kGeluP[2], p3 = kGeluP[3], p4 = kGeluP[4],
                            p5 = kGeluP[5], p6 = kGeluP[6];
};

// ---------------------------------------------------------------------------
// Element math.  Every multiply is an explicit __fmul_rn / fmaf so the
// vector, scalar and tail paths execute the identical rounding sequence.
// ---------------------------------------------------------------------------
template <bool kPrecise>
__device__ __forceinline__ float exp_neg_half(float v) {  // e^{-v/2}, v >= 0
  const float KH = __uint_as_float(kExpKH);
  if constexpr (kPrecise) {
    const float KL = __uint_as_float(kExpKL);
    float bh = __fmul_rn(v, KH);
    float bl = fmaf(v, KH, -bh);  // exact residual of the product
    bl = fmaf(v, KL, bl);         // + the part of -log2(e)/2 below binary32
    float e0 = ex2_approx(bh);
    return fmaf(e0, __fmul_rn(bl, __uint_as_float(kLn2)), e0);  // 2^(bh+bl) ~= 2^bh (1 + bl ln2)
  } else {
    return ex2_approx(__fmul_rn(v, KH));
  }
}

// GELU(x) = x Phi(x) = max(x,0) - u Phi(-u), u = |x|; Phi(-u) = e^{-u^2/2} G(u).
template <bool kPrecise>
__device__ __forceinline__ float gelu_f(float x) {
  const float u = fabsf(x);
  const float t = rcp_approx(fmaf(kGeluK, u, 1.0f));
  float p = __uint_as_float(GeluPoly::p0);  // Horner, degree 6
  p = fmaf(p, t, __uint_as_float(GeluPoly::p1));
  p = fmaf(p, t, __uint_as_float(GeluPoly::p2));
  p = fmaf(p, t, __uint_as_float(GeluPoly::p3));
  p = fmaf(p, t, __uint_as_float(GeluPoly::p4));
  p = fmaf(p, t, __uint_as_float(GeluPoly::p5));
  p = fmaf(p, t, __uint_as_float(GeluPoly::p6));
  const float q = __fmul_rn(u, __fmul_rn(t, p));  // u G(u)
  float e;
  if constexpr (kPrecise) {
    // e^{-u^2/2} with u^2 split exactly: u^2 = ah + al.
    const float uc = fminf(u, 16.0f);  // e^{-128} is 0 in binary32 anyway
    const float ah = __fmul_rn(uc, uc);
    const float al = fmaf(uc, uc, -ah);
    const float KH = __uint_as_float(kExpKH), KL = __uint_as_float(kExpKL);
    const float bh = __fmul_rn(ah, KH);
    float bl = fmaf(ah, KH, -bh);
    bl = fmaf(ah, KL, bl);
    bl = fmaf(al, KH, bl);
    const float e0 = ex2_approx(bh);
    e = fmaf(e0, __fmul_rn(bl, __uint_as_float(kLn2)), e0);
  } else {
    e = ex2_approx(__fmul_rn(__fmul_rn(u, u), __uint_as_float(kExpKH)));
  }
  return fmaf(-q, e, fmaxf(x, -0.0f));
}

// SiLU(x) = x sigma(x) = max(x,0) - u sigma(-u) = max(x,0) - u e^{-u} / (1 + e^{-u}).
template <bool kPrecise>
__device__ __forceinline__ float silu_f(float x) {
  const float u = fabsf(x);
  const float eh = exp_neg_half<kPrecise>(u);       // e^{-u/2}, never subnormal for u < 174
  const float s = rcp_approx(fmaf(eh, eh, 1.0f));   // 1 / (1 + e^{-u})
  // max(x,0) - (u eh s) eh with one rounding (an explicit FMA, as in the packed
  // path: ptxas fuses mul.rn.f32x2 + add.rn.f32x2 into FFMA2 regardless of the
  // rounding modifier, so the contract is written as the fused form on both).
  const float nq = __fmul_rn(__fmul_rn(-u, eh), s);
  return fmaf(nq, eh, fmaxf(x, -0.0f));
}

// Packed-pair versions on sm_100's f32x2 FMA pipe (FFMA2 / FMUL2): the same
// IEEE operations in the same order as gelu_f / silu_f, lane by lane, so the
// results are bitwise identical to the scalar path; half the issue slots for
// the polynomial and the products.
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

template <bool kPrecise>
__device__ __forceinline__ float2 gelu2_f(float2 x) {
  if constexpr (kPrecise) {
    return make_float2(gelu_f<true>(x.x), gelu_f<true>(x.y));
  } else {
    const float2 u = make_float2(fabsf(x.x), fabsf(x.y));
    const float2 d = __ffma2_rn(f2(kGeluK), u, f2(1.0f));
    const float2 t = make_float2(rcp_approx(d.x), rcp_approx(d.y));
    float2 p = f2(__uint_as_float(GeluPoly::p0));
    p = __ffma2_rn(p, t, f2(__uint_as_float(GeluPoly::p1)));
    p = __ffma2_rn(p, t, f2(__uint_as_float(GeluPoly::p2)));
    p = __ffma2_rn(p, t, f2(__uint_as_float(GeluPoly::p3)));
    p = __ffma2_rn(p, t, f2(__uint_as_float(GeluPoly::p4)));
    p = __ffma2_rn(p, t, f2(__uint_as_float(GeluPoly::p5)));
    p = __ffma2_rn(p, t, f2(__uint_as_float(GeluPoly::p6)));
    const float2 nu = make_float2(-u.x, -u.y);
    const float2 nq = __fmul2_rn(nu, __fmul2_rn(t, p));  // -u G(u), exact negation of q
    const float2 a = __fmul2_rn(__fmul2_rn(u, u), f2(__uint_as_float(kExpKH)));
    const float2 e = make_float2(ex2_approx(a.x), ex2_approx(a.y));
    return __ffma2_rn(nq, e, make_float2(fmaxf(x.x, -0.0f), fmaxf(x.y, -0.0f)));
  }
}

template <bool kPrecise>
__device__ __forceinline__ float2 silu2_f(float2 x) {
  if constexpr (kPrecise) {
    return make_float2(silu_f<true>(x.x), silu_f<true>(x.y));
  } else {
    const float2 u = make_float2(fabsf(x.x), fabsf(x.y));
    const float2 a = __fmul2_rn(u, f2(__uint_as_float(kExpKH)));
#ifdef LMBP_DIAG_NO_EX2  // diagnostic build knobs: the MUFU ops replaced by FMUL (wrong values; timing only)
    const float2 eh = __fmul2_rn(a, f2(0.25f));
#else
    const float2 eh = make_float2(ex2_approx(a.x), ex2_approx(a.y));
#endif
    const float2 d = __ffma2_rn(eh, eh, f2(1.0f));
#ifdef LMBP_DIAG_NO_RCP
    const float2 s = __fmul2_rn(d, f2(0.75f));
#else
    const float2 s = make_float2(rcp_approx(d.x), rcp_approx(d.y));
#endif
    const float2 nq = __fmul2_rn(__fmul2_rn(make_float2(-u.x, -u.y), eh), s);
    return __ffma2_rn(nq, eh, make_float2(fmaxf(x.x, -0.0f), fmaxf(x.y, -0.0f)));
  }
}

template <int A, bool kPrecise>
__device__ __forceinline__ float2 act2_f(float2 x) {
  if constexpr (A == kActGelu) return gelu2_f<kPrecise>(x);
  else return silu2_f<kPrecise>(x);
}

template <int A, bool kPrecise>
__device__ __forceinline__ float act_f(float x) {
  if constexpr (A == kActGelu) return gelu_f<kPrecise>(x);
  else return silu_f<kPrecise>(x);
}

// Scalar code: exact for any fp32/bf16/fp16 input (thresholds rounded down).
template <int A>
__device__ __forceinline__ uint32_t code_f32(float x) {
  return (uint32_t)(x > __uint_as_float(Tab<A>::t0)) + (uint32_t)(x > __uint_as_float(Tab<A>::t1)) +
         (uint32_t)(x > __uint_as_float(Tab<A>::t2));
}

// From three nested compare masks (m1 >= m2 >= m3 since c1 < c2 < c3):
// code = m1 + m2 + m3 -> bit0 = m1 ^ m2 ^ m3, bit1 = m2.  Interleave both
// bits into every 2-bit field of the word, then the caller keeps one field.
__device__ __forceinline__ uint32_t code_fields(uint32_t m1, uint32_t m2, uint32_t m3) {
  return ((m1 ^ m2 ^ m3) & 0x55555555u) | (m2 & 0xAAAAAAAAu);
}

// 4 fp32 elements -> 8 code bits.
template <int A>
__device__ __forceinline__ uint32_t codes_vec_f32(const float *f) {
  const float T0 = __uint_as_float(Tab<A>::t0), T1 = __uint_as_float(Tab<A>::t1),
              T2 = __uint_as_float(Tab<A>::t2);
  uint32_t W = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t m1 = f[k] > T0 ? 0xffffffffu : 0u;
    const uint32_t m2 = f[k] > T1 ? 0xffffffffu : 0u;
    const uint32_t m3 = f[k] > T2 ? 0xffffffffu : 0u;
    W |= code_fields(m1, m2, m3) & (0x3u << (2 * k));
  }
  return W;
}

// 8 bf16 / fp16 elements (4 packed pairs) -> 16 code bits.  Pair j holds
// element 2j in its low half and 2j+1 in its high half; the compare masks are
// 0xffff per half.  Element 2j's field is taken from bits 4j..4j+1, element
// 2j+1's from bits 16+4j+2..16+4j+3 and folded down by the final shift.
template <typename T, int A>
__device__ __forceinline__ uint32_t codes_vec_16(const uint4 &r) {
  const uint32_t w[4] = {r.x, r.y, r.z, r.w};
  uint32_t W = 0;
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    const __nv_bfloat162 T0 = __halves2bfloat162(__ushort_as_bfloat16(Tab<A>::b0), __ushort_as_bfloat16(Tab<A>::b0));
    const __nv_bfloat162 T1 = __halves2bfloat162(__ushort_as_bfloat16(Tab<A>::b1), __ushort_as_bfloat16(Tab<A>::b1));
    const __nv_bfloat162 T2 = __halves2bfloat162(__ushort_as_bfloat16(Tab<A>::b2), __ushort_as_bfloat16(Tab<A>::b2));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __nv_bfloat162 v = *reinterpret_cast<const __nv_bfloat162 *>(&w[j]);
      const uint32_t z = code_fields(__hgt2_mask(v, T0), __hgt2_mask(v, T1), __hgt2_mask(v, T2));
      W |= z & ((0x3u << (4 * j)) | (0x3u << (18 + 4 * j)));
    }
  } else {
    const __half2 T0 = __halves2half2(__ushort_as_half(Tab<A>::h0), __ushort_as_half(Tab<A>::h0));
    const __half2 T1 = __halves2half2(__ushort_as_half(Tab<A>::h1), __ushort_as_half(Tab<A>::h1));
    const __half2 T2 = __halves2half2(__ushort_as_half(Tab<A>::h2), __ushort_as_half(Tab<A>::h2));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const __half2 v = *reinterpret_cast<const __half2 *>(&w[j]);
      const uint32_t z = code_fields(__hgt2_mask(v, T0), __hgt2_mask(v, T1), __hgt2_mask(v, T2));
      W |= z & ((0x3u << (4 * j)) | (0x3u << (18 + 4 * j)));
    }
  }
  return (W | (W >> 16)) & 0xffffu;
}

template <typename T> using CodeWord = typename std::conditional<Traits<T>::kVec == 8, uint16_t, uint8_t>::type;

// Level s[c] for a 2-bit code (s0 = 0, s3 = 1 exactly).
template <int A>
__device__ __forceinline__ float level(uint32_t c) {
  const float lo = (c & 1u) ? __uint_as_float(Tab<A>::s1) : 0.0f;
  const float hi = (c & 1u) ? 1.0f : __uint_as_float(Tab<A>::s2);
  return (c & 2u) ? hi : lo;
}

}  // namespace lmbp
