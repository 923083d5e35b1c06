// stepact.cu -- table-driven k-bit step-derivative activations
// (SURVEY.md 8(f) NEXT #3).
//
// Eq. 14 with 2^k - 1 ReLUs: the forward keeps the primitive
// h = GELU or SiLU unchanged, the backward uses the 2^k-segment step function
// dh~ (Prop. 4.1), so k bits per element are stored (P:L362,
// "k is the required bit number").  k = 2 with the published tables is
// ReGELU2 / ReSiLU2 (bitwise identical to regelu2_* / resilu2_*, tested);
// other tables cover ReGELU2-d (App. I) and k = 1 / 3 / 4
// variants ("setting a larger k ... is also feasible").
//
// Packing: element j occupies bits k*j .. k*j + k - 1 of the flat
// LSB-first bit stream.  Any 8 consecutive elements starting at a multiple of
// 8 fill exactly k whole bytes, so a thread (or a 16-byte vector of 8 16-bit
// elements) owns k bytes of codes; for k = 3 a single code may straddle two
// of those bytes (handled by building the group's 24-bit word first).
#include "act_lut.cuh"
#include "act_math.cuh"
#include "common.cuh"
#include "ew_pipeline.cuh"
#include "kernels.h"

// Forward pipeline shape (tools/sweep.py): consumer warps x vectors x stages,
// and for k = 4 the CTAs per SM the register budget must allow.
#ifndef LMBP_STEP_W
#define LMBP_STEP_W 16
#define LMBP_STEP_U 2
#define LMBP_STEP_S 4
#endif
#ifndef LMBP_STEP4_W  // k = 4, 16-bit types
#define LMBP_STEP4_W 12
#endif
#ifndef LMBP_STEP4_S
#define LMBP_STEP4_S 3
#endif
#ifndef LMBP_STEP_MINB4
#define LMBP_STEP_MINB4 3
#endif
#ifndef LMBP_STEP_MINB4_F32
#define LMBP_STEP_MINB4_F32 2
#endif

namespace lmbp {

template <int K>
__device__ __forceinline__ uint32_t step_code(float x, const float *thr) {
  uint32_t c = 0;
#pragma unroll
  for (int i = 0; i < (1 << K) - 1; ++i) c += (uint32_t)(x > thr[i]);
  return c;
}

// Code of element j read from the packed stream, for any k <= 4 (a k = 3
// code straddles a byte boundary when (3 j) % 8 > 5; the second byte exists
// then because the code's bits lie inside the stream).
template <int K>
__device__ __forceinline__ uint32_t code_at(const uint8_t *codes, int64_t j) {
  const int64_t bit = (int64_t)K * j;
  uint32_t w = codes[bit >> 3];
  if ((bit & 7) + K > 8) w |= (uint32_t)codes[(bit >> 3) + 1] << 8;
  return (w >> (bit & 7)) & ((1u << K) - 1u);
}

template <typename T>
__device__ __forceinline__ void load8(const T *p, int64_t g, bool vec, float *f) {
  if (vec) {
    if constexpr (Traits<T>::kVec == 8) {
      Vec<T>::unpack(ld_stream(reinterpret_cast<const uint4 *>(p) + g), f);
    } else if (kUseV8 && ((uintptr_t)p & 31u) == 0) {  // 8 fp32 = one 256-bit access
      uint4 a, b;
      ld_stream32(reinterpret_cast<const uint4 *>(p) + 2 * g, a, b);
      Vec<T>::unpack(a, f);
      Vec<T>::unpack(b, f + 4);
    } else {
      Vec<T>::unpack(ld_stream(reinterpret_cast<const uint4 *>(p) + 2 * g), f);
      Vec<T>::unpack(ld_stream(reinterpret_cast<const uint4 *>(p) + 2 * g + 1), f + 4);
    }
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = to_f32<T>(p[8 * g + e]);
  }
}

template <typename T>
__device__ __forceinline__ void store8(T *p, int64_t g, bool vec, const float *f) {
  if (vec) {
    if constexpr (Traits<T>::kVec == 8) {
      st_stream(reinterpret_cast<uint4 *>(p) + g, Vec<T>::pack(f));
    } else if (kUseV8 && ((uintptr_t)p & 31u) == 0) {
      st_stream32(reinterpret_cast<uint4 *>(p) + 2 * g, Vec<T>::pack(f), Vec<T>::pack(f + 4));
    } else {
      st_stream(reinterpret_cast<uint4 *>(p) + 2 * g, Vec<T>::pack(f));
      st_stream(reinterpret_cast<uint4 *>(p) + 2 * g + 1, Vec<T>::pack(f + 4));
    }
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) p[8 * g + e] = from_f32<T>(f[e]);
  }
}

template <typename T, int A, bool kPrecise, int K>
__global__ void __launch_bounds__(256) stepact_fwd_k(const T *x, T *y, uint8_t *codes, int64_t n, StepTable tab,
                                                     bool vec) {
  pdl_enter();
  const int64_t groups = n / 8;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
    float f[8];
    load8<T>(x, g, vec, f);
    uint32_t w = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) w |= step_code<K>(f[e], tab.thr) << (K * e);
    if constexpr (kUseLut<T, A>) {
#pragma unroll
      for (int e = 0; e < 8; ++e) y[8 * g + e] = act_y<T, A, kPrecise>(from_f32<T>(f[e]), f[e]);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) f[e] = act_f<A, kPrecise>(f[e]);
      store8<T>(y, g, vec, f);
    }
#pragma unroll
    for (int b = 0; b < K; ++b) codes[g * K + b] = (uint8_t)(w >> (8 * b));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && groups * 8 < n) {  // ragged tail, trailing bits 0
    uint32_t w = 0;
    for (int64_t j = groups * 8; j < n; ++j) {
      const float f = to_f32<T>(x[j]);
      w |= step_code<K>(f, tab.thr) << (K * (j - groups * 8));
      y[j] = act_y<T, A, kPrecise>(x[j], f);
    }
    const int nbytes = (int)(((n - groups * 8) * K + 7) / 8);
    for (int b = 0; b < nbytes; ++b) codes[groups * K + b] = (uint8_t)(w >> (8 * b));
  }
}

template <typename T, int K>
__global__ void __launch_bounds__(256) stepact_bwd_k(const T *dy, const uint8_t *codes, T *dx, int64_t n,
                                                     StepTable tab, bool vec) {
  pdl_enter();
  __shared__ float lvl[16];
  if (threadIdx.x < (1 << K)) lvl[threadIdx.x] = tab.lvl[threadIdx.x];
  __syncthreads();
  constexpr uint32_t kMask = (1u << K) - 1u;
  const int64_t groups = n / 8;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
    float f[8];
    load8<T>(dy, g, vec, f);
    uint32_t w = 0;
#pragma unroll
    for (int b = 0; b < K; ++b) w |= (uint32_t)codes[g * K + b] << (8 * b);
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = __fmul_rn(f[e], lvl[(w >> (K * e)) & kMask]);
    store8<T>(dx, g, vec, f);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int64_t j = groups * 8; j < n; ++j)
      dx[j] = from_f32<T>(__fmul_rn(to_f32<T>(dy[j]), lvl[code_at<K>(codes, j)]));
  }
}

// ---------------------------------------------------------------------------
// TMA/CLC pipeline path (ew_pipeline.cuh): one 16-byte vector of kVec
// elements yields kVec k bits = kVec k / 8 whole bytes of codes (needs
// kVec k to be a multiple of 8: every case except fp32 with k = 1 or k = 3,
// which keep the simple kernel).  Same per-element arithmetic as the simple kernel -> bitwise equal.
// ---------------------------------------------------------------------------
struct StepEwParams : EwParams {
  StepTable tab;  // runtime step table
};

// Codes of one 16-byte vector by a branch-free binary search over the sorted
// thresholds, bit by bit from the top: bit b of code = #{i : x > c_i} is
// [x > c_(j 2^b + 2^b)] (1-based) where j holds the bits above b already
// found (thresholds increasing, so the count is the position of x among them).
// The candidate threshold for bit b is picked from 2^(K-1-b) candidates by a
// mux tree on the higher bits' masks.  k compares per element instead of
// 2^k - 1; for 16-bit types the compares are packed (HSET2: two elements per
// instruction, masks 0xffff per half) and the mux is one LOP3 per node on
// both halves at once.
template <int K>
__device__ __forceinline__ uint32_t bsearch_masks_16(uint32_t v, const uint32_t (&t)[15], bool bf16,
                                                     uint32_t (&M)[K]) {
#pragma unroll
  for (int b = K - 1; b >= 0; --b) {
    uint32_t cand[1 << (K - 1)];
#pragma unroll
    for (int j = 0; j < (1 << (K - 1 - b)); ++j) cand[j] = t[(2 * j + 1) * (1 << b) - 1];
#pragma unroll
    for (int q = b + 1, w = 1 << (K - 1 - b); q < K; ++q, w >>= 1) {
#pragma unroll
      for (int j = 0; j < w / 2; ++j) cand[j] = (M[q] & cand[2 * j + 1]) | (~M[q] & cand[2 * j]);
    }
    if (bf16)
      M[b] = __hgt2_mask(*reinterpret_cast<const __nv_bfloat162 *>(&v), *reinterpret_cast<const __nv_bfloat162 *>(&cand[0]));
    else
      M[b] = __hgt2_mask(*reinterpret_cast<const __half2 *>(&v), *reinterpret_cast<const __half2 *>(&cand[0]));
  }
  uint32_t z = 0;
#pragma unroll
  for (int b = 0; b < K; ++b) z |= M[b] & (0x10001u << b);
  return z;  // element 2j's code at bits 0..K-1, element 2j+1's at 16..16+K-1
}

template <int K>
__device__ __forceinline__ uint32_t bsearch_code_f32(float x, const float (&t)[15]) {
  bool M[K];
  uint32_t code = 0;
#pragma unroll
  for (int b = K - 1; b >= 0; --b) {
    float cand[1 << (K - 1)];
#pragma unroll
    for (int j = 0; j < (1 << (K - 1 - b)); ++j) cand[j] = t[(2 * j + 1) * (1 << b) - 1];
#pragma unroll
    for (int q = b + 1, w = 1 << (K - 1 - b); q < K; ++q, w >>= 1) {
#pragma unroll
      for (int j = 0; j < w / 2; ++j) cand[j] = M[q] ? cand[2 * j + 1] : cand[2 * j];
    }
    M[b] = x > cand[0];
    code |= (uint32_t)M[b] << b;
  }
  return code;
}

template <typename T, int K>
__device__ __forceinline__ uint32_t step_codes_vec(const uint4 &r, const float *f, const StepTable &tab) {
  uint32_t W = 0;
  if constexpr (Traits<T>::kVec == 4) {
    float t[15];
#pragma unroll
    for (int i = 0; i < 15; ++i) t[i] = i < (1 << K) - 1 ? tab.thr[i] : 0.0f;
#pragma unroll
    for (int e = 0; e < 4; ++e) W |= bsearch_code_f32<K>(f[e], t) << (K * e);
  } else {
    uint32_t t[15];
#pragma unroll
    for (int i = 0; i < 15; ++i) t[i] = i < (1 << K) - 1 ? tab.thr2[i] : 0u;
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t M[K];
      const uint32_t z = bsearch_masks_16<K>(w[j], t, std::is_same<T, __nv_bfloat16>::value, M);
      W |= ((z & ((1u << K) - 1)) | ((z >> 16) << K)) << (2 * K * j);
    }
  }
  return W;
}

// ---------------------------------------------------------------------------
// Per-CTA code table for k >= 3 on 16-bit types: the code of every 16-bit
// pattern, one byte each (64 KB of shared memory), so an element's code is
// PRMT + IADD + LDS.U8 instead of the k-level compare / mux tree (11 LOP3 per
// pair at k = 4, the ALU-bound part of the forward, DESIGN 5.6).  The table
// depends on the runtime thresholds, so the consumers fill it at CTA start
// (the producer streams the first tiles meanwhile).  Filling walks the two
// monotone halves of the pattern space: for p < 0x8000, x grows with p and
// x > t <=> p > A(t); for p >= 0x8000, x falls with p and x > t <=> p < B(t),
// with A(t) = -1, B(t) = bits(t) for t < 0 and A(t) = bits(t) & 0x7fff,
// B(t) = 0 otherwise (t = RD_T(c), exact, reading R2); NaN patterns get 0.
// Each consumer thread writes 16-byte vectors of the table, their codes found
// by binary search (a linear recount per 64-byte chunk, with boundary chunks
// redone word by word, cost ~10 us more per launch at k = 4, and contiguous
// per-thread runs walked monotonically cost more still -- strided 16-byte
// stores -- profiles/r02/session4/fixed_cost_kbit*.jsonl).
// ---------------------------------------------------------------------------
template <typename T> struct Pat16;
template <> struct Pat16<__nv_bfloat16> { static constexpr int kInf = 0x7F80; };
template <> struct Pat16<__half> { static constexpr int kInf = 0x7C00; };

template <typename T, int K>
__device__ __forceinline__ void fill_code_table(uint8_t *ctab, const StepTable &tab, int tid, int nthr) {
  constexpr int M = (1 << K) - 1;
  __shared__ int sA[16], sB[16];
  if (tid < M) {
    const int tb = (int)(tab.thr2[tid] & 0xffffu);
    const bool negt = (tb & 0x8000) && (tb & 0x7fff);  // strictly negative (-0 acts as +0)
    sA[tid] = negt ? -1 : (tb & 0x7fff);
    sB[tid] = negt ? tb : 0;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
#ifndef LMBP_DIAG_NO_FILL  // diagnostic (timing only): leave the table unwritten
  // code(q) = #{j : sA[j] < q} (q < 0x8000) or #{j : sB[j] > q} (q >= 0x8000).
  // Both predicates hold on a prefix of j (sA is non-decreasing, sB
  // non-increasing: the thresholds are sorted), so the count is a binary
  // search for the prefix length: K dependent shared-memory loads.
  auto code_of = [&](int q) -> uint32_t {
    int lo = 0;
#pragma unroll
    for (int step = 1 << (K - 1); step; step >>= 1) {
      const int j = lo + step - 1;
      if (j < M && (q < 0x8000 ? sA[j] < q : sB[j] > q)) lo += step;
    }
    return (uint32_t)lo;
  };
  // One 16-byte vector of the table (16 patterns, never straddling 0x8000)
  // per step, lane-consecutive (conflict-free stores); the code is monotone
  // within a half, so equal codes at both ends make a constant vector.  Only
  // the ~2^(K+1) vectors holding a threshold (or the NaN boundary) are filled
  // pattern by pattern.  Two vectors per iteration: four independent searches
  // in flight (C4 k = 4: 75.8 -> 69.7 us, k = 3: 71.7 -> 69.8 us).
#pragma unroll 2
  for (int v = tid; v < 65536 / 16; v += nthr) {
    const int p0 = 16 * v;
    const int nan_lo = (p0 >= 0x8000 ? (0x8000 | Pat16<T>::kInf) : Pat16<T>::kInf) + 1;
    const uint32_t c0 = code_of(p0), c1 = code_of(p0 + 15);
    uint32_t w[4];
    if (c0 == c1 && p0 + 15 < nan_lo) {
      w[0] = w[1] = w[2] = w[3] = c0 * 0x01010101u;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        w[e] = 0;
        for (int q = 0; q < 4; ++q) {
          const int pq = p0 + 4 * e + q;
          w[e] |= (pq >= nan_lo ? 0u : code_of(pq)) << (8 * q);
        }
      }
    }
    *reinterpret_cast<uint4 *>(ctab + p0) = make_uint4(w[0], w[1], w[2], w[3]);
  }
#endif
}

// Codes of one 16-byte vector (8 16-bit elements) from the code table.
template <int K>
__device__ __forceinline__ uint32_t ctab_codes_vec(const uint4 &v, uint32_t ctab) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t W = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t lo = lds_u8(ctab + __byte_perm(w[j], 0u, 0x4410));
    const uint32_t hi = lds_u8(ctab + __byte_perm(w[j], 0u, 0x4432));
    W |= (lo | (hi << K)) << (2 * K * j);
  }
  return W;
}

// Shapes with tables: GELU (128 KB y table + 64 KB code table) fits one CTA
// per SM with 8 KB tiles x 3 stages; SiLU (64 KB code table) two CTAs per SM.
#ifndef LMBP_STEPC_W
#define LMBP_STEPC_W 12
#define LMBP_STEPC_U 2
#define LMBP_STEPC_S 3
#endif
#ifndef LMBP_STEPCG_W
#define LMBP_STEPCG_W 16
#define LMBP_STEPCG_U 1
#define LMBP_STEPCG_S 3
#endif

template <typename T, int A, bool kPrecise, int K>
struct StepFwdOp {
  using Params = StepEwParams;
  // k = 4 register budget: the 15 hoisted thresholds would otherwise take the
  // kernel to 72+ registers and fewer warps per SM.  16-bit types: 12
  // consumer warps x 3 stages, 3 CTAs / SM (<= 48 registers) for SiLU; GELU
  // (it would spill at 48) and fp32: 16 x 4, 2 CTAs / SM (profiles/r01/sweep32_*, sweep33_*: C4 96.4 -> 94.3 us,
  // C5 443 -> 429 us; the 16-bit shape costs C3 fp32 +2 %, so fp32 keeps its own).
  static constexpr bool k16 = sizeof(T) == 2 && A == kActSilu;  // GELU's math needs > 48 registers
#ifndef LMBP_NO_LUT
  // y from the correctly rounded table where regelu2_fwd / resilu2_fwd take
  // it (kUseLut: GELU on 16-bit types), so k = 2 with the paper's table stays
  // bitwise equal to them; 128 KB of shared memory -> one CTA per SM.
  static constexpr bool kTab16 = kUseLut<T, A>;
#else
  static constexpr bool kTab16 = false;
#endif
#ifndef LMBP_NO_CTAB
  // the code table where the compare / mux tree is the ALU-bound part: SiLU
  // (GELU on 16-bit types already holds the 128 KB y table; both tables leave
  // one CTA per SM with 8 KB tiles, measured slower, profiles/r02/sweep40)
  static constexpr bool kCtab = sizeof(T) == 2 && K >= 3 && !kTab16;
#else
  static constexpr bool kCtab = false;
#endif
  __device__ static const uint16_t *tab16() {
    if constexpr (kUseLut<T, A>) return lut16<T, A>();
    else return nullptr;
  }
  __device__ static void fill_ctab(uint8_t *ctab, const StepEwParams &p, int tid, int nthr) {
    if constexpr (kCtab) fill_code_table<T, K>(ctab, p.tab, tid, nthr);
  }
  static constexpr int kMinBlocks =
      (kTab16 || kCtab) ? 0 : K == 4 ? (k16 ? LMBP_STEP_MINB4 : LMBP_STEP_MINB4_F32) : 0;
  static constexpr int kVecT = Traits<T>::kVec;
  static constexpr int W = kCtab ? (kTab16 ? LMBP_STEPCG_W : LMBP_STEPC_W)
                                 : kTab16 ? LMBP_STEP_W : K == 4 && k16 ? LMBP_STEP4_W : LMBP_STEP_W,
                       U = kCtab ? (kTab16 ? LMBP_STEPCG_U : LMBP_STEPC_U) : LMBP_STEP_U,
                       S = kCtab ? (kTab16 ? LMBP_STEPCG_S : LMBP_STEPC_S)
                                 : kTab16 ? LMBP_STEP_S : K == 4 && k16 ? LMBP_STEP4_S : LMBP_STEP_S,
                       kIn = 1, kCodeIn = 0, kCodeOut = kVecT * K / 8;
  __device__ static uint32_t apply(const uint4 (&v)[1], uint32_t, int64_t i, const StepEwParams &p) {
    float f[kVecT];
    Vec<T>::unpack(v[0], f);
    const uint32_t w = step_codes_vec<T, K>(v[0], f, p.tab);
#pragma unroll
    for (int e = 0; e < kVecT; e += 2) {
      const float2 r = act2_f<A, kPrecise>(make_float2(f[e], f[e + 1]));
      f[e] = r.x;
      f[e + 1] = r.y;
    }
    st_stream(p.out[0] + i, Vec<T>::pack(f));
    return w;
  }
  // 16-bit types with a y table and/or a code table.
  __device__ static uint32_t apply(const uint4 (&v)[1], uint32_t, int64_t i, const StepEwParams &p, Tabs tb) {
    float f[kVecT];
    uint32_t w;
    if constexpr (kCtab) w = ctab_codes_vec<K>(v[0], tb.code);
    else w = step_codes_vec<T, K>(v[0], f, p.tab);  // (f unused for 16-bit types)
    if constexpr (kTab16) {
      st_stream(p.out[0] + i, make_uint4(tab16_pair(tb.y, v[0].x), tab16_pair(tb.y, v[0].y),
                                         tab16_pair(tb.y, v[0].z), tab16_pair(tb.y, v[0].w)));
    } else {
      Vec<T>::unpack(v[0], f);
#pragma unroll
      for (int e = 0; e < kVecT; e += 2) {
        const float2 r = act2_f<A, kPrecise>(make_float2(f[e], f[e + 1]));
        f[e] = r.x;
        f[e + 1] = r.y;
      }
      st_stream(p.out[0] + i, Vec<T>::pack(f));
    }
    return w;
  }
  __device__ static void tail(const StepEwParams &p, Tabs tb = Tabs{0, 0}) {
    const int64_t j0 = p.nvec * kVecT;
    if (j0 >= p.n) return;
    const T *x = reinterpret_cast<const T *>(p.in[0]);
    T *y = reinterpret_cast<T *>(p.out[0]);
    uint32_t w = 0;
    for (int64_t j = j0; j < p.n; ++j) {
      const float f = to_f32<T>(x[j]);
      w |= step_code<K>(f, p.tab.thr) << (K * (j - j0));
      if constexpr (kTab16) {
        const uint16_t b = (uint16_t)lds_u16(tb.y + 2u * reinterpret_cast<const uint16_t *>(x)[j]);
        y[j] = *reinterpret_cast<const T *>(&b);
      } else {
        y[j] = from_f32<T>(act_f<A, kPrecise>(f));
      }
    }
    const int nbytes = (int)(((p.n - j0) * K + 7) / 8);
    for (int b = 0; b < nbytes; ++b) p.codes_out[j0 * K / 8 + b] = (uint8_t)(w >> (8 * b));
  }
};

template <typename T, int K>
struct StepBwdOp {
  using Params = StepEwParams;
  static constexpr int kVecT = Traits<T>::kVec;
  static constexpr int W = 12, U = 4, S = 3, kIn = 1, kCodeIn = kVecT * K / 8, kCodeOut = 0;
  // Levels in a shared-memory table: one conflict-free LDS per element (16
  // words in 16 banks; equal codes broadcast) instead of a 2^k - 1 select tree.
  static constexpr int kLut = 1 << K;
  __device__ static float lut_entry(const StepEwParams &p, int i) { return p.tab.lvl[i]; }
  __device__ static uint32_t apply(const uint4 (&v)[1], uint32_t c, int64_t i, const StepEwParams &p,
                                   const float *lut) {
    constexpr uint32_t kMask = (1u << K) - 1u;
    float f[kVecT];
    Vec<T>::unpack(v[0], f);
#pragma unroll
    for (int e = 0; e < kVecT; ++e) f[e] = __fmul_rn(f[e], lut[(c >> (K * e)) & kMask]);
    st_stream(p.out[0] + i, Vec<T>::pack(f));
    return 0u;
  }
  __device__ static void tail(const StepEwParams &p) {
    const T *dy = reinterpret_cast<const T *>(p.in[0]);
    T *dx = reinterpret_cast<T *>(p.out[0]);
    for (int64_t j = p.nvec * kVecT; j < p.n; ++j)
      dx[j] = from_f32<T>(__fmul_rn(to_f32<T>(dy[j]), p.tab.lvl[code_at<K>(p.codes_in, j)]));
  }
};

static int step_grid(int64_t groups) {
  const int64_t want = (groups + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count() * 8));
}

template <typename T, int A, int K>
static cudaError_t stepact_fwd_t(const void *x, void *y, uint8_t *codes, int64_t n, const StepTable &tab,
                                 cudaStream_t s) {
  constexpr bool kPrecise = std::is_same<T, float>::value;
  const bool vec = (uintptr_t)x % 16 == 0 && (uintptr_t)y % 16 == 0;
  if constexpr ((Traits<T>::kVec * K) % 8 == 0) {
    if (vec && (uintptr_t)codes % 16 == 0) {
      StepEwParams p{};
      p.in[0] = reinterpret_cast<const uint4 *>(x);
      p.out[0] = reinterpret_cast<uint4 *>(y);
      p.codes_out = codes;
      p.nvec = n / Traits<T>::kVec;
      p.n = n;
      p.tab = tab;
      return launch_ew<StepFwdOp<T, A, kPrecise, K>>(p, s);
    }
  }
  launch_k(stepact_fwd_k<T, A, kPrecise, K>, step_grid(n / 8), 256, 0, s, reinterpret_cast<const T *>(x),
           reinterpret_cast<T *>(y), codes, n, tab, vec);
  return cudaGetLastError();
}

template <typename T, int K>
static cudaError_t stepact_bwd_t(const void *dy, const uint8_t *codes, void *dx, int64_t n, const StepTable &tab,
                                 cudaStream_t s) {
  const bool vec = (uintptr_t)dy % 16 == 0 && (uintptr_t)dx % 16 == 0;
  if constexpr ((Traits<T>::kVec * K) % 8 == 0) {
    if (vec && (uintptr_t)codes % 16 == 0) {
      StepEwParams p{};
      p.in[0] = reinterpret_cast<const uint4 *>(dy);
      p.codes_in = codes;
      p.out[0] = reinterpret_cast<uint4 *>(dx);
      p.nvec = n / Traits<T>::kVec;
      p.n = n;
      p.tab = tab;
      return launch_ew<StepBwdOp<T, K>>(p, s);
    }
  }
  launch_k(stepact_bwd_k<T, K>, step_grid(n / 8), 256, 0, s, reinterpret_cast<const T *>(dy), codes,
           reinterpret_cast<T *>(dx), n, tab, vec);
  return cudaGetLastError();
}

template <typename T, int A>
static cudaError_t fwd_k(int k, const void *x, void *y, uint8_t *codes, int64_t n, const StepTable &t, cudaStream_t s) {
  if (k == 1) return stepact_fwd_t<T, A, 1>(x, y, codes, n, t, s);
  if (k == 2) return stepact_fwd_t<T, A, 2>(x, y, codes, n, t, s);
  if (k == 3) return stepact_fwd_t<T, A, 3>(x, y, codes, n, t, s);
  return stepact_fwd_t<T, A, 4>(x, y, codes, n, t, s);
}

template <typename T>
static cudaError_t bwd_k(int k, const void *dy, const uint8_t *codes, void *dx, int64_t n, const StepTable &t,
                         cudaStream_t s) {
  if (k == 1) return stepact_bwd_t<T, 1>(dy, codes, dx, n, t, s);
  if (k == 2) return stepact_bwd_t<T, 2>(dy, codes, dx, n, t, s);
  if (k == 3) return stepact_bwd_t<T, 3>(dy, codes, dx, n, t, s);
  return stepact_bwd_t<T, 4>(dy, codes, dx, n, t, s);
}

cudaError_t stepact_fwd(int act, int dtype, const StepTable &t, const void *x, void *y, uint8_t *codes, int64_t n,
                        cudaStream_t s) {
  if (act == kActGelu) {
    if (dtype == 0) return fwd_k<float, kActGelu>(t.k, x, y, codes, n, t, s);
    if (dtype == 1) return fwd_k<__nv_bfloat16, kActGelu>(t.k, x, y, codes, n, t, s);
    return fwd_k<__half, kActGelu>(t.k, x, y, codes, n, t, s);
  }
  if (dtype == 0) return fwd_k<float, kActSilu>(t.k, x, y, codes, n, t, s);
  if (dtype == 1) return fwd_k<__nv_bfloat16, kActSilu>(t.k, x, y, codes, n, t, s);
  return fwd_k<__half, kActSilu>(t.k, x, y, codes, n, t, s);
}

cudaError_t stepact_bwd(int dtype, const StepTable &t, const void *dy, const uint8_t *codes, void *dx, int64_t n,
                        cudaStream_t s) {
  if (dtype == 0) return bwd_k<float>(t.k, dy, codes, dx, n, t, s);
  if (dtype == 1) return bwd_k<__nv_bfloat16>(t.k, dy, codes, dx, n, t, s);
  return bwd_k<__half>(t.k, dy, codes, dx, n, t, s);
}

}  // namespace lmbp
