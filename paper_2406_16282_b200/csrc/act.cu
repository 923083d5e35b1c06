// act.cu -- ReGELU2 / ReSiLU2 forward and backward kernels (sm_100a).
//
// Method (arXiv 2406.16282, Sec. 4.2; App. E):
//   forward : y = GELU(x) or SiLU(x), unchanged;
//             code = #{i : x > c_i}, 2 bits per element, 4 per byte.
//   backward: dx = dy * s[code], s = (0, a1, a1 + a2, 1) -- the derivative of
//             the ReLU combination of Eq. 14.
//
// B200 design:
//   * TMA bulk-copy pipeline with cluster-launch-control work stealing
//     (ew_pipeline.cuh): 16 KB (fwd) / 24 KB (bwd) tiles staged in shared
//     memory by a producer warp, consumer warps compute and store with
//     coalesced 16-byte stores; codes staged per warp and written as 16-byte
//     vectors.  Fallbacks: a register-pipelined vector kernel (backward with a
//     codes pointer not 16-byte aligned) and a scalar kernel (misaligned).
//   * 16-bit types compute codes with packed x2 compares (HSET2) and a
//     bit-interleave trick, no per-element shifts.
//   * Element math in act_math.cuh (branch-free GELU via the Mills ratio,
//     SiLU with e^{-u} = (e^{-u/2})^2; packed FFMA2/FMUL2).
#include <type_traits>

#include "common.cuh"
#include "act_math.cuh"
#include "act_lut.cuh"
#include "ew_pipeline.cuh"
#include "kernels.h"

namespace lmbp {

// Scalar fp32/bf16/fp16 tail: elements [j0, n), j0 a multiple of 4.
template <typename T, int A, bool kPrecise>
__device__ void act_fwd_tail(const T *x, T *y, uint8_t *codes, int64_t j0, int64_t n) {
  for (int64_t b = j0 >> 2; 4 * b < n; ++b) {
    uint32_t byte = 0;
    for (int k = 0; k < 4; ++k) {
      const int64_t j = 4 * b + k;
      if (j >= n) break;
      const float f = to_f32<T>(x[j]);
      y[j] = act_y<T, A, kPrecise>(x[j], f);
      byte |= code_f32<A>(f) << (2 * k);
    }
    codes[b] = (uint8_t)byte;
  }
}

// Forward, scalar path (any alignment): one code byte (4 elements) per thread.
template <typename T, int A, bool kPrecise>
__global__ void __launch_bounds__(256) act_fwd_scalar(const T *x, T *y, uint8_t *codes, int64_t n) {
  pdl_enter();
  const int64_t nbytes = (n + 3) >> 2;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nbytes; b += (int64_t)gridDim.x * blockDim.x) {
    uint32_t byte = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t j = 4 * b + k;
      if (j < n) {
        const float f = to_f32<T>(x[j]);
        y[j] = act_y<T, A, kPrecise>(x[j], f);
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
  pdl_enter();
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
  pdl_enter();
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t cj = (codes[j >> 2] >> (2 * (j & 3))) & 3u;
    dx[j] = from_f32<T>(__fmul_rn(to_f32<T>(dy[j]), level<A>(cj)));
  }
}

// ---------------------------------------------------------------------------
// TMA-pipelined path (ew_pipeline.cuh), the default for 16-byte aligned
// tensors.  Shapes tuned on B200 (tools/sweep.py, profiles/r01/sweep*.jsonl):
// forward 16 consumer warps x 2 vectors/lane (16 KB tiles) x 4 stages;
// backward 12 warps x 4 vectors/lane (24 KB tiles + codes) x 3 stages.
// ---------------------------------------------------------------------------
// Returns the code word (forward); the caller stores it.
template <typename T, int A, bool kPrecise, bool kFwd>
__device__ __forceinline__ uint32_t act_vec_op(const uint4 &v, uint32_t c_in, uint4 *out, int64_t i) {
  constexpr int kVec = Traits<T>::kVec;
  float f[kVec];
  Vec<T>::unpack(v, f);
  if constexpr (kFwd) {
    uint32_t c;
    if constexpr (kVec == 4) c = codes_vec_f32<A>(f);
    else c = codes_vec_16<T, A>(v);
#ifndef LMBP_DIAG_NO_MATH  // diagnostic build knob (tools/sweep.py): time the pipeline without the math
#ifdef LMBP_DIAG_SKIP_LO     // diagnostic: no math for vectors [LO, HI) only (start / end transients)
    if (!(i >= (int64_t)LMBP_DIAG_SKIP_LO && i < (int64_t)LMBP_DIAG_SKIP_HI))
#endif
#pragma unroll
    for (int k = 0; k < kVec; k += 2) {
      const float2 r = act2_f<A, kPrecise>(make_float2(f[k], f[k + 1]));
      f[k] = r.x;
      f[k + 1] = r.y;
    }
#endif
    st_stream(out + i, Vec<T>::pack(f));
    return c;
  } else {
#pragma unroll
    for (int k = 0; k < kVec; ++k) f[k] = __fmul_rn(f[k], level<A>((c_in >> (2 * k)) & 3u));
    st_stream(out + i, Vec<T>::pack(f));
    return 0u;
  }
}

// Forward pipeline shape (tools/sweep.py): 16-bit types 16 consumer warps x
// 2 vectors x 4 stages; fp32 8 x 4 x 3 (C3 GELU fp32 67.6 -> 65.7 us,
// profiles/r01/sweep24_fwd_shapes_c2_c3_c4.jsonl; no shape moves the
// instruction-bound bf16 GELU at C2).
#ifndef LMBP_FWD_W
#define LMBP_FWD_W 16
#define LMBP_FWD_U 2
#define LMBP_FWD_S 4
#endif
#ifndef LMBP_FWD32_W
#define LMBP_FWD32_W 8
#define LMBP_FWD32_U 4
#define LMBP_FWD32_S 3
#endif
template <typename T, int A, bool kPrecise>
struct ActFwdOp {
  static constexpr bool k32 = sizeof(T) == 4;
  static constexpr int W = k32 ? LMBP_FWD32_W : LMBP_FWD_W, U = k32 ? LMBP_FWD32_U : LMBP_FWD_U,
                       S = k32 ? LMBP_FWD32_S : LMBP_FWD_S, kIn = 1, kCodeIn = 0;
  static constexpr int kCodeOut = Traits<T>::kVec / 4;
  __device__ static uint32_t apply(const uint4 (&v)[1], uint32_t, int64_t i, const EwParams &p) {
    return act_vec_op<T, A, kPrecise, true>(v[0], 0u, p.out[0], i);
  }
  __device__ static void tail(const EwParams &p) {
    constexpr int kVec = Traits<T>::kVec;
    if (p.nvec * kVec < p.n)
      act_fwd_tail<T, A, kPrecise>(reinterpret_cast<const T *>(p.in[0]), reinterpret_cast<T *>(p.out[0]),
                                   p.codes_out, p.nvec * kVec, p.n);
  }
};

// GELU on 16-bit types (kUseLut): the correctly rounded table (act_lut.cuh)
// copied to shared memory once per CTA; one LDS per element instead of the
// polynomial / MUFU math; codes as before (packed compares).  Tail elements
// read the same table.
#ifndef LMBP_LUT_W
#define LMBP_LUT_W 16
#define LMBP_LUT_U 2
#define LMBP_LUT_S 4
#endif
template <typename T, int A>
struct ActFwdLutOp {
  static_assert(sizeof(T) == 2, "16-bit types only");
  static constexpr bool kTab16 = true;
  static constexpr int W = LMBP_LUT_W, U = LMBP_LUT_U, S = LMBP_LUT_S, kIn = 1, kCodeIn = 0, kCodeOut = 2;
  __device__ static const uint16_t *tab16() { return lut16<T, A>(); }
  __device__ static uint32_t apply(const uint4 (&v)[1], uint32_t, int64_t i, const EwParams &p, Tabs tb) {
    const uint32_t c = codes_vec_16<T, A>(v[0]);
    const uint32_t tab = tb.y;
    st_stream(p.out[0] + i, make_uint4(tab16_pair(tab, v[0].x), tab16_pair(tab, v[0].y), tab16_pair(tab, v[0].z),
                                       tab16_pair(tab, v[0].w)));
    return c;
  }
  __device__ static void tail(const EwParams &p, Tabs tb) {
    const uint32_t tab = tb.y;
    const int64_t j0 = p.nvec * 8;
    if (j0 >= p.n) return;
    const T *x = reinterpret_cast<const T *>(p.in[0]);
    uint16_t *y = reinterpret_cast<uint16_t *>(p.out[0]);
    for (int64_t b = j0 >> 2; 4 * b < p.n; ++b) {
      uint32_t byte = 0;
      for (int k = 0; k < 4; ++k) {
        const int64_t j = 4 * b + k;
        if (j >= p.n) break;
        const uint16_t xb = reinterpret_cast<const uint16_t *>(x)[j];
        y[j] = (uint16_t)lds_u16(tab + 2u * xb);
        byte |= code_f32<A>(to_f32<T>(x[j])) << (2 * k);
      }
      p.codes_out[b] = (uint8_t)byte;
    }
  }
};

template <typename T, int A>
__device__ void act_bwd_tail(const T *dy, const uint8_t *codes, T *dx, int64_t j0, int64_t n) {
  for (int64_t j = j0; j < n; ++j) {
    const uint32_t cj = (codes[j >> 2] >> (2 * (j & 3))) & 3u;
    dx[j] = from_f32<T>(__fmul_rn(to_f32<T>(dy[j]), level<A>(cj)));
  }
}

// Backward shape: 12 consumer warps x 4 vectors (24 KB tiles + codes) x 2
// stages (was 3: C2 26.6 -> 24.6 us, C4/C5 unchanged -- a shallower ring
// leaves less queued work per CTA to drain at the end, profiles/r02/sweep38).
#ifndef LMBP_BWD_W
#define LMBP_BWD_W 12
#define LMBP_BWD_U 4
#define LMBP_BWD_S 2
#endif
template <typename T, int A>
struct ActBwdOp {
  static constexpr int W = LMBP_BWD_W, U = LMBP_BWD_U, S = LMBP_BWD_S, kIn = 1, kCodeIn = Traits<T>::kVec / 4,
                       kCodeOut = 0;
  __device__ static uint32_t apply(const uint4 (&v)[1], uint32_t c, int64_t i, const EwParams &p) {
    return act_vec_op<T, A, false, false>(v[0], c, p.out[0], i);
  }
  __device__ static void tail(const EwParams &p) {
    act_bwd_tail<T, A>(reinterpret_cast<const T *>(p.in[0]), p.codes_in, reinterpret_cast<T *>(p.out[0]),
                       p.nvec * Traits<T>::kVec, p.n);
  }
};

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
  // The TMA path writes each warp's codes as 16-byte vectors: codes must be
  // 16-byte aligned too (any other alignment takes the scalar path).
  const bool aligned = ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0) && ((uintptr_t)codes % 16 == 0);
  const int sms = sm_count();
  if (aligned) {
    EwParams p{};
    p.in[0] = reinterpret_cast<const uint4 *>(x);
    p.out[0] = reinterpret_cast<uint4 *>(y);
    p.codes_out = codes;
    p.nvec = n / kVec;
    p.n = n;
#ifndef LMBP_NO_LUT
    if constexpr (kUseLut<T, A>) return launch_ew<ActFwdLutOp<T, A>>(p, s);
    else
#endif
      return launch_ew<ActFwdOp<T, A, kPrecise>>(p, s);
  } else {
    auto kern = act_fwd_scalar<T, A, kPrecise>;
    static const int occ = occupancy(kern, kActThreads);
    const int64_t want = cdiv(cdiv(n, 4), kActThreads);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * occ));
    launch_k(kern, grid, kActThreads, 0, s, reinterpret_cast<const T *>(x), reinterpret_cast<T *>(y), codes, n);
  }
  return cudaGetLastError();
}

template <typename T, int A>
static cudaError_t act_bwd_t(const void *dy, const uint8_t *codes, void *dx, int64_t n, cudaStream_t s) {
  constexpr int kVec = Traits<T>::kVec;
  const bool aligned = ((uintptr_t)dy % 16 == 0) && ((uintptr_t)dx % 16 == 0) &&
                       (kVec == 4 || (uintptr_t)codes % 2 == 0);
  const int sms = sm_count();
  if (aligned && (uintptr_t)codes % 16 == 0) {
    EwParams p{};
    p.in[0] = reinterpret_cast<const uint4 *>(dy);
    p.codes_in = codes;
    p.out[0] = reinterpret_cast<uint4 *>(dx);
    p.nvec = n / kVec;
    p.n = n;
    return launch_ew<ActBwdOp<T, A>>(p, s);
  } else if (aligned) {
    auto kern = act_bwd_vec<T, A, kActUnroll>;
    static const int occ = occupancy(kern, kActThreads);
    const int64_t nvec = n / kVec;
    const int64_t want = cdiv(nvec, (int64_t)kActThreads * kActUnroll);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * occ));
    launch_k(kern, grid, kActThreads, 0, s, reinterpret_cast<const uint4 *>(dy), codes, reinterpret_cast<uint4 *>(dx),
             nvec, n);
  } else {
    auto kern = act_bwd_scalar<T, A>;
    static const int occ = occupancy(kern, kActThreads);
    const int64_t want = cdiv(n, kActThreads);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * occ));
    launch_k(kern, grid, kActThreads, 0, s, reinterpret_cast<const T *>(dy), codes, reinterpret_cast<T *>(dx), n);
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

#ifdef LMBP_TRACE
// Diagnostic build only: read / reset this translation unit's CTA trace.
extern "C" __attribute__((visibility("default"))) int lmbp_trace_act(unsigned long long *host, int max_records,
                                                                    int reset) {
  unsigned int n = 0;
  if (cudaMemcpyFromSymbol(&n, lmbp::lmbp_trace_n, sizeof(n)) != cudaSuccess) return -1;
  const int m = (int)(n < (unsigned)max_records ? n : (unsigned)max_records);
  if (m > 0 && cudaMemcpyFromSymbol(host, lmbp::lmbp_trace_buf, (size_t)m * 5 * sizeof(unsigned long long)) != cudaSuccess)
    return -1;
  if (reset) {
    const unsigned int z = 0;
    if (cudaMemcpyToSymbol(lmbp::lmbp_trace_n, &z, sizeof(z)) != cudaSuccess) return -1;
    if (cudaMemcpyToSymbol(lmbp::lmbp_trace_un, &z, sizeof(z)) != cudaSuccess) return -1;
  }
  return m;
}

// Diagnostic build only: the (unit, time) pairs of the CLC claims.
extern "C" __attribute__((visibility("default"))) int lmbp_trace_units_act(unsigned long long *host, int max_pairs) {
  unsigned int n = 0;
  if (cudaMemcpyFromSymbol(&n, lmbp::lmbp_trace_un, sizeof(n)) != cudaSuccess) return -1;
  const int m = (int)(n < (unsigned)max_pairs ? n : (unsigned)max_pairs);
  if (m > 0 && cudaMemcpyFromSymbol(host, lmbp::lmbp_trace_units, (size_t)m * 2 * sizeof(unsigned long long)) !=
                   cudaSuccess)
    return -1;
  return m;
}
#endif
