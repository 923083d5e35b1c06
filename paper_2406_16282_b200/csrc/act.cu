// act.cu -- ReGELU2 / ReSiLU2 forward and backward kernels (sm_100a).
//
// Method (arXiv 2406.16282, Sec. 4.2; App. E):
//   forward : y = GELU(x) or SiLU(x), unchanged;
//             code = #{i : x > c_i}, 2 bits per element, 4 per byte.
//   backward: dx = dy * s[code], s = (0, a1, a1 + a2, 1) -- the derivative of
//             the ReLU combination of Eq. 14.
//
// B200 design:
//   * HBM-bound streaming: 16-byte vector loads/stores, lane-interleaved so
//     every warp instruction touches 512 contiguous bytes; U vectors per thread
//     in flight; grid = SMs x resident CTAs, grid-stride over tiles.
//   * codes: one 16-bit word per 8 bf16/fp16 elements (one byte per 4 fp32),
//     stored by the lane that owns the 16-byte vector -> 64 (32) contiguous
//     bytes per warp store.  16-bit types compute codes with packed x2
//     compares (HSET2) and a bit-interleave trick, no per-element shifts.
//   * GELU is evaluated branch-free as max(x,0) - |x| e^{-x^2/2} G(|x|),
//     G(u) = Phi(-u) e^{u^2/2} ~= t P7(t), t = 1/(1 + k u): 2 MUFU + ~16 FMA-pipe
//     ops per element; SiLU as max(x,0) - u e^{-u} / (1 + e^{-u}) with the
//     exponential split e^{-u} = (e^{-u/2})^2 so products underflow gradually.
//     fp32 outputs add an exact split of the exponent argument ("precise").
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

struct GeluPoly {
  static constexpr uint32_t p0 = kGeluP[0], p1 = kGeluP[1], p2 = kGeluP[2], p3 = kGeluP[3], p4 = kGeluP[4],
                            p5 = kGeluP[5], p6 = kGeluP[6], p7 = kGeluP[7];
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
  float p = __uint_as_float(GeluPoly::p0);  // Horner, degree 7
  p = fmaf(p, t, __uint_as_float(GeluPoly::p1));
  p = fmaf(p, t, __uint_as_float(GeluPoly::p2));
  p = fmaf(p, t, __uint_as_float(GeluPoly::p3));
  p = fmaf(p, t, __uint_as_float(GeluPoly::p4));
  p = fmaf(p, t, __uint_as_float(GeluPoly::p5));
  p = fmaf(p, t, __uint_as_float(GeluPoly::p6));
  p = fmaf(p, t, __uint_as_float(GeluPoly::p7));
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
  return fmaf(-q, e, fmaxf(x, 0.0f));
}

// SiLU(x) = x sigma(x) = max(x,0) - u sigma(-u) = max(x,0) - u e^{-u} / (1 + e^{-u}).
template <bool kPrecise>
__device__ __forceinline__ float silu_f(float x) {
  const float u = fabsf(x);
  const float eh = exp_neg_half<kPrecise>(u);       // e^{-u/2}, never subnormal for u < 174
  const float s = rcp_approx(fmaf(eh, eh, 1.0f));   // 1 / (1 + e^{-u})
  const float q = __fmul_rn(__fmul_rn(__fmul_rn(u, eh), s), eh);
  return __fsub_rn(fmaxf(x, 0.0f), q);
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
    p = __ffma2_rn(p, t, f2(__uint_as_float(GeluPoly::p7)));
    const float2 nu = make_float2(-u.x, -u.y);
    const float2 nq = __fmul2_rn(nu, __fmul2_rn(t, p));  // -u G(u), exact negation of q
    const float2 a = __fmul2_rn(__fmul2_rn(u, u), f2(__uint_as_float(kExpKH)));
    const float2 e = make_float2(ex2_approx(a.x), ex2_approx(a.y));
    return __ffma2_rn(nq, e, make_float2(fmaxf(x.x, 0.0f), fmaxf(x.y, 0.0f)));
  }
}

template <bool kPrecise>
__device__ __forceinline__ float2 silu2_f(float2 x) {
  if constexpr (kPrecise) {
    return make_float2(silu_f<true>(x.x), silu_f<true>(x.y));
  } else {
    const float2 u = make_float2(fabsf(x.x), fabsf(x.y));
    const float2 a = __fmul2_rn(u, f2(__uint_as_float(kExpKH)));
    const float2 eh = make_float2(ex2_approx(a.x), ex2_approx(a.y));
    const float2 d = __ffma2_rn(eh, eh, f2(1.0f));
    const float2 s = make_float2(rcp_approx(d.x), rcp_approx(d.y));
    const float2 q = __fmul2_rn(__fmul2_rn(__fmul2_rn(u, eh), s), eh);
    return make_float2(__fsub_rn(fmaxf(x.x, 0.0f), q.x), __fsub_rn(fmaxf(x.y, 0.0f), q.y));
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

// Scalar fp32/bf16/fp16 tail: elements [j0, n), j0 a multiple of 4.
template <typename T, int A, bool kPrecise>
__device__ void act_fwd_tail(const T *x, T *y, uint8_t *codes, int64_t j0, int64_t n) {
  for (int64_t b = j0 >> 2; 4 * b < n; ++b) {
    uint32_t byte = 0;
    for (int k = 0; k < 4; ++k) {
      const int64_t j = 4 * b + k;
      if (j >= n) break;
      const float f = to_f32<T>(x[j]);
      y[j] = from_f32<T>(act_f<A, kPrecise>(f));
      byte |= code_f32<A>(f) << (2 * k);
    }
    codes[b] = (uint8_t)byte;
  }
}

// ---------------------------------------------------------------------------
// Forward, vector path.
// ---------------------------------------------------------------------------
template <typename T, int A, bool kPrecise, int U>
__global__ void __launch_bounds__(256) act_fwd_vec(const uint4 *x, uint4 *y, uint8_t *codes, int64_t nvec,
                                                   int64_t n) {
  constexpr int kVec = Traits<T>::kVec;
  CodeWord<T> *cw = reinterpret_cast<CodeWord<T> *>(codes);
  const int64_t tile = (int64_t)blockDim.x * U;
  const int64_t stride = (int64_t)gridDim.x * tile;
  // Register double buffering: the next tile's loads are in flight while the
  // current tile is computed, so every warp always has U x 16 B per lane
  // outstanding (the activation math is long enough to expose DRAM latency).
  int64_t base = (int64_t)blockIdx.x * tile + threadIdx.x;
  uint4 v[U];
#pragma unroll
  for (int j = 0; j < U; ++j) {
    const int64_t i = base + (int64_t)j * blockDim.x;
    if (i < nvec) v[j] = ld_stream(x + i);
  }
  for (; base < nvec; base += stride) {
    uint4 nv[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t i = base + stride + (int64_t)j * blockDim.x;
      if (i < nvec) nv[j] = ld_stream(x + i);
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t i = base + (int64_t)j * blockDim.x;
      if (i < nvec) {
        float f[kVec];
        Vec<T>::unpack(v[j], f);
        uint32_t c;
        if constexpr (kVec == 4) c = codes_vec_f32<A>(f);
        else c = codes_vec_16<T, A>(v[j]);
#pragma unroll
        for (int k = 0; k < kVec; k += 2) {
          const float2 r = act2_f<A, kPrecise>(make_float2(f[k], f[k + 1]));
          f[k] = r.x;
          f[k + 1] = r.y;
        }
        st_stream(y + i, Vec<T>::pack(f));
        cw[i] = (CodeWord<T>)c;
      }
    }
#pragma unroll
    for (int j = 0; j < U; ++j) v[j] = nv[j];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && nvec * kVec < n)
    act_fwd_tail<T, A, kPrecise>(reinterpret_cast<const T *>(x), reinterpret_cast<T *>(y), codes, nvec * kVec, n);
}

// Forward, scalar path (any alignment): one code byte (4 elements) per thread.
template <typename T, int A, bool kPrecise>
__global__ void __launch_bounds__(256) act_fwd_scalar(const T *x, T *y, uint8_t *codes, int64_t n) {
  const int64_t nbytes = (n + 3) >> 2;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nbytes; b += (int64_t)gridDim.x * blockDim.x) {
    uint32_t byte = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t j = 4 * b + k;
      if (j < n) {
        const float f = to_f32<T>(x[j]);
        y[j] = from_f32<T>(act_f<A, kPrecise>(f));
        byte |= code_f32<A>(f) << (2 * k);
      }
    }
    codes[b] = (uint8_t)byte;
  }
}

// ---------------------------------------------------------------------------
// Backward.
// ---------------------------------------------------------------------------
template <typename T, int A, int U>
__global__ void __launch_bounds__(256) act_bwd_vec(const uint4 *dy, const uint8_t *codes, uint4 *dx, int64_t nvec,
                                                   int64_t n) {
  constexpr int kVec = Traits<T>::kVec;
  const CodeWord<T> *cw = reinterpret_cast<const CodeWord<T> *>(codes);
  const int64_t tile = (int64_t)blockDim.x * U;
  const int64_t stride = (int64_t)gridDim.x * tile;
  int64_t base = (int64_t)blockIdx.x * tile + threadIdx.x;
  uint4 v[U];
  uint32_t c[U];
#pragma unroll
  for (int j = 0; j < U; ++j) {
    const int64_t i = base + (int64_t)j * blockDim.x;
    if (i < nvec) {
      v[j] = ld_stream(dy + i);
      c[j] = cw[i];
    }
  }
  for (; base < nvec; base += stride) {
    uint4 nv[U];
    uint32_t nc[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t i = base + stride + (int64_t)j * blockDim.x;
      if (i < nvec) {
        nv[j] = ld_stream(dy + i);
        nc[j] = cw[i];
      }
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int64_t i = base + (int64_t)j * blockDim.x;
      if (i < nvec) {
        float f[kVec];
        Vec<T>::unpack(v[j], f);
#pragma unroll
        for (int k = 0; k < kVec; ++k) f[k] = __fmul_rn(f[k], level<A>((c[j] >> (2 * k)) & 3u));
        st_stream(dx + i, Vec<T>::pack(f));
      }
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      v[j] = nv[j];
      c[j] = nc[j];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const T *dys = reinterpret_cast<const T *>(dy);
    T *dxs = reinterpret_cast<T *>(dx);
    for (int64_t j = nvec * kVec; j < n; ++j) {
      const uint32_t cj = (codes[j >> 2] >> (2 * (j & 3))) & 3u;
      dxs[j] = from_f32<T>(__fmul_rn(to_f32<T>(dys[j]), level<A>(cj)));
    }
  }
}

template <typename T, int A>
__global__ void __launch_bounds__(256) act_bwd_scalar(const T *dy, const uint8_t *codes, T *dx, int64_t n) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t cj = (codes[j >> 2] >> (2 * (j & 3))) & 3u;
    dx[j] = from_f32<T>(__fmul_rn(to_f32<T>(dy[j]), level<A>(cj)));
  }
}

// ---------------------------------------------------------------------------
// TMA-pipelined path (the default for 16-byte aligned tensors).
//
// One producer warp streams 16 KB tiles of the input (x, or dy + codes) into a
// ring of kStages shared-memory stages with cp.async.bulk (the TMA engine, no
// tensor map needed for contiguous data), completion on a per-stage mbarrier.
// Eight consumer warps copy their part of a tile into registers, release the
// stage at once (so the producer refills it while they compute), compute and
// store straight to global with coalesced 16-byte stores.  Loads in flight
// per SM = CTAs x stages x 16 KB, independent of the math latency -- this is
// what the register-prefetch variant could not reach for GELU/SiLU.
// ---------------------------------------------------------------------------
// Pipeline shapes, tuned on B200 (tools/sweep.py; profiles/r01/sweep*.jsonl):
// forward 16 consumer warps x 2 vectors/lane (16 KB tiles) x 4 stages;
// backward 12 warps x 4 vectors/lane (24 KB tiles) x 3 stages.  Plain bulk
// loads (no L2 evict-first hint: it cost 2-3 %).
template <bool kFwd> struct TmaShape;
template <> struct TmaShape<true> {
  static constexpr int W = 16, U = 2, S = 4;
};
template <> struct TmaShape<false> {
  static constexpr int W = 12, U = 4, S = 3;
};
template <bool kFwd> __host__ __device__ constexpr int tile_vec() {
  return TmaShape<kFwd>::W * 32 * TmaShape<kFwd>::U;
}
template <bool kFwd> __host__ __device__ constexpr int tma_threads() { return (TmaShape<kFwd>::W + 1) * 32; }
template <typename T, bool kFwd> __host__ __device__ constexpr int tile_code_bytes() {
  return tile_vec<kFwd>() * Traits<T>::kVec / 4;
}

template <typename T, bool kFwd>
constexpr size_t tma_smem_bytes() {
  return (size_t)TmaShape<kFwd>::S * tile_vec<kFwd>() * 16 +
         (kFwd ? 0 : (size_t)TmaShape<kFwd>::S * tile_code_bytes<T, kFwd>()) + 2 * TmaShape<kFwd>::S * sizeof(uint64_t);
}

template <typename T, int A, bool kPrecise, bool kFwd>
__device__ __forceinline__ void act_vec_op(const uint4 &v, uint32_t c_in, uint4 *out, CodeWord<T> *cw, int64_t i) {
  constexpr int kVec = Traits<T>::kVec;
  float f[kVec];
  Vec<T>::unpack(v, f);
  if constexpr (kFwd) {
    uint32_t c;
    if constexpr (kVec == 4) c = codes_vec_f32<A>(f);
    else c = codes_vec_16<T, A>(v);
#pragma unroll
    for (int k = 0; k < kVec; k += 2) {
      const float2 r = act2_f<A, kPrecise>(make_float2(f[k], f[k + 1]));
      f[k] = r.x;
      f[k + 1] = r.y;
    }
    st_stream(out + i, Vec<T>::pack(f));
    cw[i] = (CodeWord<T>)c;
  } else {
#pragma unroll
    for (int k = 0; k < kVec; ++k) f[k] = __fmul_rn(f[k], level<A>((c_in >> (2 * k)) & 3u));
    st_stream(out + i, Vec<T>::pack(f));
  }
}

template <typename T, int A, bool kPrecise, bool kFwd>
__global__ void __launch_bounds__(tma_threads<kFwd>()) act_tma(const uint4 *in, const uint8_t *codes_in, uint4 *out,
                                                               uint8_t *codes_out, int64_t nvec, int64_t n) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int kVec = Traits<T>::kVec;
  constexpr int kTmaWarps = TmaShape<kFwd>::W, kTmaU = TmaShape<kFwd>::U, kStages = TmaShape<kFwd>::S;
  constexpr int kTileVec = tile_vec<kFwd>();
  constexpr int kCB = tile_code_bytes<T, kFwd>();
  uint4 *buf = reinterpret_cast<uint4 *>(smem);
  uint8_t *cbuf = smem + (size_t)kStages * kTileVec * 16;
  uint64_t *full = reinterpret_cast<uint64_t *>(cbuf + (kFwd ? 0 : (size_t)kStages * kCB));
  uint64_t *empty = full + kStages;
  CodeWord<T> *cw_out = reinterpret_cast<CodeWord<T> *>(codes_out);
  const CodeWord<T> *cw_in = reinterpret_cast<const CodeWord<T> *>(codes_in);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = nvec / kTileVec;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTmaWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == kTmaWarps) {  // producer
    if (lane == 0) {
      int k = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int s = k % kStages;
        const uint32_t ph = (uint32_t)(k / kStages) & 1u;
        mbar_wait(&empty[s], ph ^ 1u);
        mbar_arrive_expect_tx(&full[s], kTileVec * 16 + (kFwd ? 0 : kCB));
        bulk_g2s(buf + (size_t)s * kTileVec, in + t * kTileVec, kTileVec * 16, &full[s]);
        if constexpr (!kFwd) bulk_g2s(cbuf + (size_t)s * kCB, codes_in + t * kCB, kCB, &full[s]);
      }
    }
  } else {  // consumers
    int k = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
      const int s = k % kStages;
      const uint32_t ph = (uint32_t)(k / kStages) & 1u;
      mbar_wait(&full[s], ph);
      uint4 v[kTmaU];
      uint32_t c[kTmaU];
#pragma unroll
      for (int j = 0; j < kTmaU; ++j) {
        const int vi = j * (kTmaWarps * 32) + warp * 32 + lane;
        v[j] = lds128(buf + (size_t)s * kTileVec + vi);
        if constexpr (!kFwd) c[j] = reinterpret_cast<const CodeWord<T> *>(cbuf + (size_t)s * kCB)[vi];
        else c[j] = 0;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // stage may be refilled while we compute
#pragma unroll
      for (int j = 0; j < kTmaU; ++j) {
        const int64_t i = t * kTileVec + j * (kTmaWarps * 32) + warp * 32 + lane;
        act_vec_op<T, A, kPrecise, kFwd>(v[j], c[j], out, cw_out, i);
      }
    }
    // leftover vectors (< one tile) and the ragged scalar tail: CTA 0
    if (blockIdx.x == 0) {
      for (int64_t i = ntiles * kTileVec + threadIdx.x; i < nvec; i += kTmaWarps * 32) {
        const uint4 v = ld_stream(in + i);
        act_vec_op<T, A, kPrecise, kFwd>(v, kFwd ? 0u : (uint32_t)cw_in[i], out, cw_out, i);
      }
      if (threadIdx.x == 0 && nvec * kVec < n) {
        if constexpr (kFwd) {
          act_fwd_tail<T, A, kPrecise>(reinterpret_cast<const T *>(in), reinterpret_cast<T *>(out), codes_out,
                                       nvec * kVec, n);
        } else {
          const T *dys = reinterpret_cast<const T *>(in);
          T *dxs = reinterpret_cast<T *>(out);
          for (int64_t j = nvec * kVec; j < n; ++j) {
            const uint32_t cj = (codes_in[j >> 2] >> (2 * (j & 3))) & 3u;
            dxs[j] = from_f32<T>(__fmul_rn(to_f32<T>(dys[j]), level<A>(cj)));
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Launchers.
// ---------------------------------------------------------------------------
template <typename K>
static int occupancy(K kernel, int threads) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, 0) != cudaSuccess || b < 1) b = 1;
  return b;
}

static inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

constexpr int kActThreads = 256;
constexpr int kActUnroll = 4;

template <typename T, int A>
static cudaError_t act_fwd_t(const void *x, void *y, uint8_t *codes, int64_t n, cudaStream_t s) {
  constexpr int kVec = Traits<T>::kVec;
  constexpr bool kPrecise = std::is_same<T, float>::value;
  const bool aligned = ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0) &&
                       (kVec == 4 || (uintptr_t)codes % 2 == 0);
  const int sms = sm_count();
  if (aligned && n >= (int64_t)tile_vec<true>() * kVec) {
    auto kern = act_tma<T, A, kPrecise, true>;
    constexpr size_t smem = tma_smem_bytes<T, true>();
    constexpr int threads = tma_threads<true>();
    static const int occ = [&] {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int b = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, threads, smem) != cudaSuccess || b < 1) b = 1;
      return b;
    }();
    const int64_t nvec = n / kVec;
    const int64_t want = std::max<int64_t>(1, nvec / tile_vec<true>());
    const int grid = (int)std::min<int64_t>(want, (int64_t)sms * occ);
    kern<<<grid, threads, smem, s>>>(reinterpret_cast<const uint4 *>(x), nullptr, reinterpret_cast<uint4 *>(y),
                                         codes, nvec, n);
  } else if (aligned) {
    auto kern = act_fwd_vec<T, A, kPrecise, kActUnroll>;
    static const int occ = occupancy(kern, kActThreads);
    const int64_t nvec = n / kVec;
    const int64_t want = cdiv(nvec, (int64_t)kActThreads * kActUnroll);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * occ));
    kern<<<grid, kActThreads, 0, s>>>(reinterpret_cast<const uint4 *>(x), reinterpret_cast<uint4 *>(y), codes,
                                      nvec, n);
  } else {
    auto kern = act_fwd_scalar<T, A, kPrecise>;
    static const int occ = occupancy(kern, kActThreads);
    const int64_t want = cdiv(cdiv(n, 4), kActThreads);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * occ));
    kern<<<grid, kActThreads, 0, s>>>(reinterpret_cast<const T *>(x), reinterpret_cast<T *>(y), codes, n);
  }
  return cudaGetLastError();
}

template <typename T, int A>
static cudaError_t act_bwd_t(const void *dy, const uint8_t *codes, void *dx, int64_t n, cudaStream_t s) {
  constexpr int kVec = Traits<T>::kVec;
  const bool aligned = ((uintptr_t)dy % 16 == 0) && ((uintptr_t)dx % 16 == 0) &&
                       (kVec == 4 || (uintptr_t)codes % 2 == 0);
  const int sms = sm_count();
  if (aligned && (uintptr_t)codes % 16 == 0 && n >= (int64_t)tile_vec<false>() * kVec) {
    auto kern = act_tma<T, A, false, false>;
    constexpr size_t smem = tma_smem_bytes<T, false>();
    constexpr int threads = tma_threads<false>();
    static const int occ = [&] {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int b = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, threads, smem) != cudaSuccess || b < 1) b = 1;
      return b;
    }();
    const int64_t nvec = n / kVec;
    const int64_t want = std::max<int64_t>(1, nvec / tile_vec<false>());
    const int grid = (int)std::min<int64_t>(want, (int64_t)sms * occ);
    kern<<<grid, threads, smem, s>>>(reinterpret_cast<const uint4 *>(dy), codes, reinterpret_cast<uint4 *>(dx),
                                         nullptr, nvec, n);
  } else if (aligned) {
    auto kern = act_bwd_vec<T, A, kActUnroll>;
    static const int occ = occupancy(kern, kActThreads);
    const int64_t nvec = n / kVec;
    const int64_t want = cdiv(nvec, (int64_t)kActThreads * kActUnroll);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * occ));
    kern<<<grid, kActThreads, 0, s>>>(reinterpret_cast<const uint4 *>(dy), codes, reinterpret_cast<uint4 *>(dx),
                                      nvec, n);
  } else {
    auto kern = act_bwd_scalar<T, A>;
    static const int occ = occupancy(kern, kActThreads);
    const int64_t want = cdiv(n, kActThreads);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * occ));
    kern<<<grid, kActThreads, 0, s>>>(reinterpret_cast<const T *>(dy), codes, reinterpret_cast<T *>(dx), n);
  }
  return cudaGetLastError();
}

cudaError_t act_fwd(int kind, int dtype, const void *x, void *y, uint8_t *codes, int64_t n, cudaStream_t s) {
  if (kind == kActGelu) {
    if (dtype == 0) return act_fwd_t<float, kActGelu>(x, y, codes, n, s);
    if (dtype == 1) return act_fwd_t<__nv_bfloat16, kActGelu>(x, y, codes, n, s);
    return act_fwd_t<__half, kActGelu>(x, y, codes, n, s);
  }
  if (dtype == 0) return act_fwd_t<float, kActSilu>(x, y, codes, n, s);
  if (dtype == 1) return act_fwd_t<__nv_bfloat16, kActSilu>(x, y, codes, n, s);
  return act_fwd_t<__half, kActSilu>(x, y, codes, n, s);
}

cudaError_t act_bwd(int kind, int dtype, const void *dy, const uint8_t *codes, void *dx, int64_t n, cudaStream_t s) {
  if (kind == kActGelu) {
    if (dtype == 0) return act_bwd_t<float, kActGelu>(dy, codes, dx, n, s);
    if (dtype == 1) return act_bwd_t<__nv_bfloat16, kActGelu>(dy, codes, dx, n, s);
    return act_bwd_t<__half, kActGelu>(dy, codes, dx, n, s);
  }
  if (dtype == 0) return act_bwd_t<float, kActSilu>(dy, codes, dx, n, s);
  if (dtype == 1) return act_bwd_t<__nv_bfloat16, kActSilu>(dy, codes, dx, n, s);
  return act_bwd_t<__half, kActSilu>(dy, codes, dx, n, s);
}

}  // namespace lmbp
