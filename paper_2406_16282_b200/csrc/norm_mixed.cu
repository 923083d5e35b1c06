// norm_mixed.cu -- MS-LN / MS-RMSNorm with an fp32 residual stream and a
// 16-bit normalised output (the AMP layout the paper measures: "Layer
// Normalization uses fp32, other operators use fp16" / "RMSNorm uses fp32,
// other operators use bf16", Fig. 5 / Fig. 6 captions).
//
// Memory sharing needs y in the dtype the next linear layer saves (its
// input, Prop. 5.1 condition 3), so under AMP the MS norm reads the
// fp32 residual x and writes the 16-bit y the linear consumes; its backward
// takes the 16-bit dy and y and returns the fp32 dx of the residual stream:
//   fwd : x fp32 -> y = (x - mu) rstd (LN) or x rstd (RMS), RN to bf16 / fp16;
//         rstd fp32 (Alg. 2 / Alg. 3)
//   bwd : dx = rstd (dy - mean(dy) - y mean(dy y)), fp32
// Same arithmetic as norm.cu's register teams (two-pass statistics from
// registers, deterministic fixed-order reductions), on groups of 8 elements:
// 32 bytes of fp32 and 16 bytes of 16-bit data per group.  Rows whose width
// is not a multiple of 8, misaligned pointers or rows wider than the teams
// hold take a scalar CTA-per-row path.
#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace lmbp {
namespace {

template <bool kWarpTeam>
__device__ __forceinline__ float msum(float v, float *buf) {
  v = warp_sum(v);
  if constexpr (kWarpTeam) {
    return v;
  } else {
    const int nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = v;
    __syncthreads();
    float t = 0.0f;
    for (int w = 0; w < nw; ++w) t += buf[w];
    return t;
  }
}

template <bool kWarpTeam>
__device__ __forceinline__ float2 msum2(float2 v, float2 *buf) {
  v = warp_sum2(v);
  if constexpr (kWarpTeam) {
    return v;
  } else {
    const int nw = blockDim.x >> 5;
    if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = v;
    __syncthreads();
    float2 t = make_float2(0.0f, 0.0f);
    for (int w = 0; w < nw; ++w) {
      t.x += buf[w].x;
      t.y += buf[w].y;
    }
    return t;
  }
}

// 8 fp32 <-> two 16-byte vectors
__device__ __forceinline__ void unpack8_f32(const uint4 &a, const uint4 &b, float *f) {
  Vec<float>::unpack(a, f);
  Vec<float>::unpack(b, f + 4);
}

}  // namespace

template <typename TO, int NORM, int V, bool kWarpTeam>
__global__ void __launch_bounds__(kWarpTeam ? 256 : 512) norm_fwd_mixed_vec(const uint4 *x, uint4 *y, float *rstd,
                                                                           int64_t rows, int ngrp, int cols,
                                                                           float eps) {
  pdl_enter();
  __shared__ float red[2][32];
  const int team = kWarpTeam ? 32 : (int)blockDim.x;
  const int tid = kWarpTeam ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
  const int teams = kWarpTeam ? (int)(blockDim.x >> 5) : 1;
  const int team_id = kWarpTeam ? (int)(threadIdx.x >> 5) : 0;
  const float fcols = (float)cols;
  const bool x32 = kUseV8 && ((uintptr_t)x & 31u) == 0;  // fp32 rows are 32 B multiples: whole 256-bit loads
  int it = 0;
  for (int64_t row = (int64_t)blockIdx.x * teams + team_id; row < rows; row += (int64_t)gridDim.x * teams, ++it) {
    const uint4 *xr = x + row * (int64_t)ngrp * 2;
    uint4 ra[V], rb[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int gi = j * team + tid;
      if (gi < ngrp) {
        if (x32) {
          ld_stream32(xr + 2 * gi, ra[j], rb[j]);
        } else {
          ra[j] = ld_stream(xr + 2 * gi);
          rb[j] = ld_stream(xr + 2 * gi + 1);
        }
      } else {
        ra[j] = rb[j] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
    float mean = 0.0f, ss = 0.0f;
    if constexpr (NORM == kNormLN) {
      float s = 0.0f;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        float f[8];
        unpack8_f32(ra[j], rb[j], f);  // zero-filled groups add 0
#pragma unroll
        for (int k = 0; k < 8; ++k) s += f[k];
      }
      mean = __fdiv_rn(msum<kWarpTeam>(s, red[0]), fcols);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        if (j * team + tid < ngrp) {
          float f[8];
          unpack8_f32(ra[j], rb[j], f);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float d = __fsub_rn(f[k], mean);
            ss = fmaf(d, d, ss);
          }
        }
      }
      ss = msum<kWarpTeam>(ss, red[1]);
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        float f[8];
        unpack8_f32(ra[j], rb[j], f);
#pragma unroll
        for (int k = 0; k < 8; ++k) ss = fmaf(f[k], f[k], ss);
      }
      ss = msum<kWarpTeam>(ss, red[it & 1]);
    }
    const float r = rsqrtf(__fadd_rn(__fdiv_rn(ss, fcols), eps));
    uint4 *yr = y + row * (int64_t)ngrp;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int gi = j * team + tid;
      if (gi < ngrp) {
        float f[8];
        unpack8_f32(ra[j], rb[j], f);
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = __fmul_rn(NORM == kNormLN ? __fsub_rn(f[k], mean) : f[k], r);
        st_stream(yr + gi, Vec<TO>::pack(f));
      }
    }
    if (tid == 0) rstd[row] = r;
    if constexpr (!kWarpTeam) __syncthreads();  // red[] is reused by the next row
  }
}

template <typename TO, int NORM, int V, bool kWarpTeam>
__global__ void __launch_bounds__(kWarpTeam ? 256 : 512) norm_bwd_mixed_vec(const uint4 *dy, const uint4 *__restrict__ y,
                                                                           const float *__restrict__ rstd, uint4 *dx,
                                                                           int64_t rows, int ngrp, int cols) {
  pdl_enter();
  __shared__ float2 red[2][32];
  const int team = kWarpTeam ? 32 : (int)blockDim.x;
  const int tid = kWarpTeam ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
  const int teams = kWarpTeam ? (int)(blockDim.x >> 5) : 1;
  const int team_id = kWarpTeam ? (int)(threadIdx.x >> 5) : 0;
  const float fcols = (float)cols;
  const bool dx32 = kUseV8 && ((uintptr_t)dx & 31u) == 0;
  auto body = [&](int64_t row, int it) {
    const uint4 *gr = dy + row * (int64_t)ngrp;
    const uint4 *yr = y + row * (int64_t)ngrp;
    const float r = rstd[row];
    uint4 rg[V], ry[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int gi = j * team + tid;
      if (gi < ngrp) {
        rg[j] = ld_stream(gr + gi);
        ry[j] = ld_stream(yr + gi);
      } else {
        rg[j] = ry[j] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
    float2 acc = make_float2(0.0f, 0.0f);  // (sum dy, sum dy*y)
#pragma unroll
    for (int j = 0; j < V; ++j) {
      float g[8], h[8];
      Vec<TO>::unpack(rg[j], g);
      Vec<TO>::unpack(ry[j], h);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if constexpr (NORM == kNormLN) acc.x += g[k];
        acc.y = fmaf(g[k], h[k], acc.y);
      }
    }
    acc = msum2<kWarpTeam>(acc, red[it & 1]);
    const float m1 = NORM == kNormLN ? __fdiv_rn(acc.x, fcols) : 0.0f;
    const float m2 = __fdiv_rn(acc.y, fcols);
    uint4 *dr = dx + row * (int64_t)ngrp * 2;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int gi = j * team + tid;
      if (gi < ngrp) {
        float g[8], h[8];
        Vec<TO>::unpack(rg[j], g);
        Vec<TO>::unpack(ry[j], h);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float c = NORM == kNormLN ? __fsub_rn(g[k], m1) : g[k];
          g[k] = __fmul_rn(r, fmaf(-h[k], m2, c));
        }
        if (dx32) {
          st_stream32(dr + 2 * gi, Vec<float>::pack(g), Vec<float>::pack(g + 4));
        } else {
          st_stream(dr + 2 * gi, Vec<float>::pack(g));
          st_stream(dr + 2 * gi + 1, Vec<float>::pack(g + 4));
        }
      }
    }
  };
  if constexpr (kWarpTeam) {  // one CTA per 8-row block, work stealing (as norm.cu's backward)
    clc_row_blocks(rows, teams, team_id, [&](int64_t row) { body(row, 0); });
  } else {
    int it = 0;
    for (int64_t row = (int64_t)blockIdx.x * teams + team_id; row < rows; row += (int64_t)gridDim.x * teams, ++it)
      body(row, it);
  }
}

// Scalar fallback: one CTA per row, strided loops, the same arithmetic.
template <typename TO, int NORM>
__global__ void __launch_bounds__(256) norm_fwd_mixed_scalar(const float *x, TO *y, float *rstd, int64_t rows,
                                                             int64_t cols, float eps) {
  pdl_enter();
  __shared__ float red[2][32];
  const float fcols = (float)cols;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const float *xr = x + row * cols;
    float mean = 0.0f, ss = 0.0f;
    if constexpr (NORM == kNormLN) {
      float s = 0.0f;
      for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) s += xr[c];
      mean = __fdiv_rn(msum<false>(s, red[0]), fcols);
      for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
        const float d = __fsub_rn(xr[c], mean);
        ss = fmaf(d, d, ss);
      }
    } else {
      for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) ss = fmaf(xr[c], xr[c], ss);
    }
    ss = msum<false>(ss, red[1]);
    const float r = rsqrtf(__fadd_rn(__fdiv_rn(ss, fcols), eps));
    TO *yr = y + row * cols;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x)
      yr[c] = from_f32<TO>(__fmul_rn(NORM == kNormLN ? __fsub_rn(xr[c], mean) : xr[c], r));
    if (threadIdx.x == 0) rstd[row] = r;
    __syncthreads();
  }
}

template <typename TO, int NORM>
__global__ void __launch_bounds__(256) norm_bwd_mixed_scalar(const TO *dy, const TO *y, const float *rstd, float *dx,
                                                             int64_t rows, int64_t cols) {
  pdl_enter();
  __shared__ float2 red[2][32];
  const float fcols = (float)cols;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const TO *gr = dy + row * cols;
    const TO *yr = y + row * cols;
    float2 acc = make_float2(0.0f, 0.0f);
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
      const float g = to_f32<TO>(gr[c]);
      if constexpr (NORM == kNormLN) acc.x += g;
      acc.y = fmaf(g, to_f32<TO>(yr[c]), acc.y);
    }
    acc = msum2<false>(acc, red[0]);
    const float m1 = NORM == kNormLN ? __fdiv_rn(acc.x, fcols) : 0.0f;
    const float m2 = __fdiv_rn(acc.y, fcols);
    const float r = rstd[row];
    float *dr = dx + row * cols;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
      const float g = to_f32<TO>(gr[c]);
      const float cc = NORM == kNormLN ? __fsub_rn(g, m1) : g;
      dr[c] = __fmul_rn(r, fmaf(-to_f32<TO>(yr[c]), m2, cc));
    }
    __syncthreads();
  }
}

namespace {

struct MixedPlan {
  bool vec;    // vector path possible
  bool warp;   // one warp per row (8 rows per CTA) vs one CTA per row
  int V;       // groups per thread
  int team;    // threads per row (CTA teams)
  int ngrp;
};

#ifndef LMBP_MIX_FWD_V
#define LMBP_MIX_FWD_V 4
#endif
#ifndef LMBP_MIX_BWD_V
#define LMBP_MIX_BWD_V 4
#endif
// vmax: groups per thread of the CTA teams (the kernels are instantiated
// for V = 4; a smaller vmax only widens the team).
MixedPlan plan_mixed(int64_t cols, uintptr_t a, uintptr_t b, uintptr_t c, int vmax) {
  MixedPlan p{false, false, 0, 0, 0};
  if (cols % 8 != 0 || (a | b | c) % 16 != 0 || cols > 8 * 512 * vmax) return p;
  p.ngrp = (int)(cols / 8);
  p.vec = true;
  if (p.ngrp <= 32 * 4) {          // up to 1024 columns: a warp per row
    p.warp = true;
    p.V = (p.ngrp + 31) / 32;
  } else {                         // a CTA of <= 512 threads per row, <= vmax groups per thread
    p.V = 4;
    p.team = 32 * (int)((p.ngrp + vmax * 32 - 1) / (vmax * 32));
  }
  return p;
}

template <typename K>
int occupancy_mixed(K kernel, int threads) {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, 0) != cudaSuccess || b < 1) b = 1;
  return b;
}

template <typename TO, int NORM>
cudaError_t fwd_mixed_t(const float *x, void *y, float *rstd, int64_t rows, int64_t cols, float eps, cudaStream_t s) {
  const MixedPlan p = plan_mixed(cols, (uintptr_t)x, (uintptr_t)y, 0, LMBP_MIX_FWD_V);
  const uint4 *xv = reinterpret_cast<const uint4 *>(x);
  uint4 *yv = reinterpret_cast<uint4 *>(y);
  if (p.vec && p.warp) {
    auto launch = [&](auto kern) {
      static const int occ = occupancy_mixed(kern, 256);
      const int64_t want = (rows + 7) / 8;
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count() * occ));
      launch_k(kern, grid, 256, 0, s, xv, yv, rstd, rows, p.ngrp, (int)cols, eps);
    };
    switch (p.V) {
      case 1: launch(norm_fwd_mixed_vec<TO, NORM, 1, true>); break;
      case 2: launch(norm_fwd_mixed_vec<TO, NORM, 2, true>); break;
      case 3: launch(norm_fwd_mixed_vec<TO, NORM, 3, true>); break;
      default: launch(norm_fwd_mixed_vec<TO, NORM, 4, true>); break;
    }
  } else if (p.vec) {
    const int grid = (int)std::min<int64_t>(rows, 0x7fffffff);  // one CTA per row; the hardware balances
    launch_k(norm_fwd_mixed_vec<TO, NORM, 4, false>, grid, p.team, 0, s, xv, yv, rstd, rows, p.ngrp, (int)cols, eps);
  } else {
    const int grid = (int)std::min<int64_t>(rows, (int64_t)sm_count() * 8);
    launch_k(norm_fwd_mixed_scalar<TO, NORM>, grid, 256, 0, s, x, reinterpret_cast<TO *>(y), rstd, rows, cols, eps);
  }
  return cudaGetLastError();
}

template <typename TO, int NORM>
cudaError_t bwd_mixed_t(const void *dy, const void *y, const float *rstd, float *dx, int64_t rows, int64_t cols,
                        cudaStream_t s) {
  const MixedPlan p = plan_mixed(cols, (uintptr_t)dy, (uintptr_t)y, (uintptr_t)dx, LMBP_MIX_BWD_V);
  const uint4 *gv = reinterpret_cast<const uint4 *>(dy);
  const uint4 *yv = reinterpret_cast<const uint4 *>(y);
  uint4 *dv = reinterpret_cast<uint4 *>(dx);
  if (p.vec && p.warp) {
    auto launch = [&](auto kern) {
      const int64_t want = (rows + 7) / 8;   // every block gets a CTA; running ones steal (CLC)
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, 0x7fffffff));
      launch_k(kern, grid, 256, 0, s, gv, yv, rstd, dv, rows, p.ngrp, (int)cols);
    };
    switch (p.V) {
      case 1: launch(norm_bwd_mixed_vec<TO, NORM, 1, true>); break;
      case 2: launch(norm_bwd_mixed_vec<TO, NORM, 2, true>); break;
      case 3: launch(norm_bwd_mixed_vec<TO, NORM, 3, true>); break;
      default: launch(norm_bwd_mixed_vec<TO, NORM, 4, true>); break;
    }
  } else if (p.vec) {
    const int grid = (int)std::min<int64_t>(rows, 0x7fffffff);
    launch_k(norm_bwd_mixed_vec<TO, NORM, 4, false>, grid, p.team, 0, s, gv, yv, rstd, dv, rows, p.ngrp, (int)cols);
  } else {
    const int grid = (int)std::min<int64_t>(rows, (int64_t)sm_count() * 8);
    launch_k(norm_bwd_mixed_scalar<TO, NORM>, grid, 256, 0, s, reinterpret_cast<const TO *>(dy),
             reinterpret_cast<const TO *>(y), rstd, dx, rows, cols);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t norm_fwd_mixed(int kind, int dtype, const float *x, void *y, float *rstd, int64_t rows, int64_t cols,
                           float eps, cudaStream_t s) {
  if (kind == kNormLN)
    return dtype == 1 ? fwd_mixed_t<__nv_bfloat16, kNormLN>(x, y, rstd, rows, cols, eps, s)
                      : fwd_mixed_t<__half, kNormLN>(x, y, rstd, rows, cols, eps, s);
  return dtype == 1 ? fwd_mixed_t<__nv_bfloat16, kNormRMS>(x, y, rstd, rows, cols, eps, s)
                    : fwd_mixed_t<__half, kNormRMS>(x, y, rstd, rows, cols, eps, s);
}

cudaError_t norm_bwd_mixed(int kind, int dtype, const void *dy, const void *y, const float *rstd, float *dx,
                           int64_t rows, int64_t cols, cudaStream_t s) {
#ifndef LMBP_MIX_NO_ROWS
  // rows of >= 256 16-byte vectors of dy (H >= 2048): the TMA row pipeline
  // of the same-type backward, writing fp32 (C4 49.2 -> see DESIGN 5.9)
  if (cols >= 2048) {
    const cudaError_t e = norm_bwd_mixed_rows(kind, dtype, dy, y, rstd, dx, rows, cols, s);
    if (e != cudaErrorNotSupported) return e;
  }
#endif
  if (kind == kNormLN)
    return dtype == 1 ? bwd_mixed_t<__nv_bfloat16, kNormLN>(dy, y, rstd, dx, rows, cols, s)
                      : bwd_mixed_t<__half, kNormLN>(dy, y, rstd, dx, rows, cols, s);
  return dtype == 1 ? bwd_mixed_t<__nv_bfloat16, kNormRMS>(dy, y, rstd, dx, rows, cols, s)
                    : bwd_mixed_t<__half, kNormRMS>(dy, y, rstd, dx, rows, cols, s);
}

}  // namespace lmbp
