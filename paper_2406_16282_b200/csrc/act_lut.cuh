// act_lut.cuh -- the correctly rounded 16-bit forward tables (generated at
// build time by paper_2406_16282_b200/lut.py into _obj/act_lut.inc): for every
// bf16 / fp16 bit pattern x, RN_T(GELU(x)) / RN_T(SiLU(x)).  Each translation
// unit that includes this keeps its own copy (no relocatable device code).
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "act_lut.inc"
#include "act_math.cuh"

namespace lmbp {

template <typename T, int A> __device__ __forceinline__ const uint16_t *lut16();
// (The SiLU tables are generated and compiled too; kUseLut below selects.)
template <> __device__ __forceinline__ const uint16_t *lut16<__nv_bfloat16, kActGelu>() { return kLutGeluBf16; }
template <> __device__ __forceinline__ const uint16_t *lut16<__nv_bfloat16, kActSilu>() { return kLutSiluBf16; }
template <> __device__ __forceinline__ const uint16_t *lut16<__half, kActGelu>() { return kLutGeluF16; }
template <> __device__ __forceinline__ const uint16_t *lut16<__half, kActSilu>() { return kLutSiluF16; }

// Which forwards read the table: GELU on 16-bit types.  Its math is the
// expensive one (Mills-ratio polynomial + 2 MUFU, issue-bound at C2); the
// table costs 128 KB of shared memory per CTA (one CTA per SM), which measured
// 6 % faster for GELU at C2 but 6 % slower for SiLU at C4, whose cheaper math
// is not the limiter (profiles/r02/sweep37, sweep38).  One definition per
// (activation, type) across every kernel, so all paths return the same bits.
template <typename T, int A>
constexpr bool kUseLut =
#ifndef LMBP_NO_LUT
    sizeof(T) == 2 && A == kActGelu;
#else
    false;
#endif

// y for one element outside the pipeline: the table where kUseLut (so every
// path of such a launch returns the same bits), else the fp32 math.
template <typename T, int A, bool kPrecise>
__device__ __forceinline__ T act_y(T xv, float f) {
#ifndef LMBP_NO_LUT
  if constexpr (kUseLut<T, A>) {
    const uint16_t b = lut16<T, A>()[*reinterpret_cast<const uint16_t *>(&xv)];
    return *reinterpret_cast<const T *>(&b);
  } else
#endif
  {
    return from_f32<T>(act_f<A, kPrecise>(f));
  }
}

}  // namespace lmbp
