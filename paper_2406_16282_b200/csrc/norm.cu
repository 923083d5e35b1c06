// norm.cu -- MS-LN / MS-RMSNorm forward and backward kernels (sm_100a).
//
// Method (arXiv 2406.16282, Sec. 5.2 Alg. 1; App. F Alg. 2-3,
// P:L1236-1272).  Per row of p = cols elements:
//   MS-LN fwd : mu = mean(x); var = mean((x-mu)^2); rstd = 1/sqrt(var+eps);
//               y = (x - mu) rstd                                    (Alg. 2)
//   MS-LN bwd : dx = rstd (dy - mean(dy) - y mean(dy y))
//   MS-RMS fwd: rstd = 1/sqrt(mean(x^2)+eps); y = x rstd             (Alg. 3)
//   MS-RMS bwd: dx = rstd (dy - y mean(dy y))
// The affine is merged into the next linear layer, so there are
// no parameter reads and no dgamma/dbeta column reductions.
//
// B200 design:
//   * register teams: a row is owned by one warp (8 rows per 256-thread CTA,
//     persistent grid) or one CTA of <= 512 threads (one CTA per row, the
//     hardware block scheduler balances the SMs); each thread holds V <= 8
//     lane-interleaved 16-byte vectors, so every byte is read from HBM once
//     and the two-pass statistics come from registers.  Reductions: warp
//     shuffles, then one fixed-order pass over per-warp partials in shared
//     memory -> deterministic.
//   * per-warp TMA ring (backward rows >= 8 KB, and rows too long for
//     registers): each warp streams its rows through 2-4 shared-memory stages
//     with cp.async.bulk on mbarriers and reduces from shared memory.
//   * misaligned rows, or rows too long for both, take a scalar multi-pass path.
#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace lmbp {

template <bool kWarpTeam>
__device__ __forceinline__ float team_sum(float v, float *buf) {
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
__device__ __forceinline__ float2 team_sum2(float2 v, float2 *buf) {
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

#ifndef LMBP_NORM_NO_CLC
constexpr bool kNormClc = true;
#else
constexpr bool kNormClc = false;  // tuning knob: persistent grid-stride warp teams
#endif
#ifdef LMBP_NORM_FWD_CLC
constexpr bool kNormFwdClc = kNormClc;
#else
constexpr bool kNormFwdClc = false;  // the forward keeps the persistent grid (see fwd_v)
#endif

// ---------------------------------------------------------------------------
// Forward, vector path.
// ---------------------------------------------------------------------------
// Warp teams run in 256-thread CTAs (8 rows in flight per CTA); CTA teams have
// at most 512 threads, so both variants get >= 128 registers per thread.
template <typename T, int NORM, int V, bool kWarpTeam>
__global__ void __launch_bounds__(kWarpTeam ? 256 : 512) norm_fwd_vec(const uint4 *x, uint4 *y, float *rstd,
                                                     int64_t rows, int nvec, int cols, float eps) {
  pdl_enter();
  constexpr int kVec = Traits<T>::kVec;
  __shared__ float red[2][32];
  const int team = kWarpTeam ? 32 : (int)blockDim.x;
  const int tid = kWarpTeam ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
  const int teams = kWarpTeam ? (int)(blockDim.x >> 5) : 1;
  const int team_id = kWarpTeam ? (int)(threadIdx.x >> 5) : 0;
  const float fcols = (float)cols;
  auto body = [&](int64_t row, int it) {
    const uint4 *xr = x + row * nvec;
    uint4 raw[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int vi = j * team + tid;
      if (vi < nvec) raw[j] = ld_stream(xr + vi);
      else raw[j] = make_uint4(0u, 0u, 0u, 0u);
    }
    float mean = 0.0f;
    float ss = 0.0f;
    if constexpr (NORM == kNormLN) {
      float s = 0.0f;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        float f[kVec];
        Vec<T>::unpack(raw[j], f);  // zero-filled slots add 0
#pragma unroll
        for (int k = 0; k < kVec; ++k) s += f[k];
      }
      mean = __fdiv_rn(team_sum<kWarpTeam>(s, red[0]), fcols);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        if (j * team + tid < nvec) {
          float f[kVec];
          Vec<T>::unpack(raw[j], f);
#pragma unroll
          for (int k = 0; k < kVec; ++k) {
            const float d = __fsub_rn(f[k], mean);
            ss = fmaf(d, d, ss);
          }
        }
      }
      ss = team_sum<kWarpTeam>(ss, red[1]);
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        float f[kVec];
        Vec<T>::unpack(raw[j], f);
#pragma unroll
        for (int k = 0; k < kVec; ++k) ss = fmaf(f[k], f[k], ss);
      }
      ss = team_sum<kWarpTeam>(ss, red[it & 1]);
    }
    const float r = rsqrtf(__fadd_rn(__fdiv_rn(ss, fcols), eps));
    uint4 *yr = y + row * nvec;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int vi = j * team + tid;
      if (vi < nvec) {
        float f[kVec];
        Vec<T>::unpack(raw[j], f);
#pragma unroll
        for (int k = 0; k < kVec; ++k) f[k] = __fmul_rn(NORM == kNormLN ? __fsub_rn(f[k], mean) : f[k], r);
        st_stream(yr + vi, Vec<T>::pack(f));
      }
    }
    if (tid == 0) rstd[row] = r;
  };
  if constexpr (kWarpTeam && V <= 4 && kNormFwdClc) {
    clc_row_blocks(rows, teams, team_id, [&](int64_t row) { body(row, 0); });
  } else {
    int it = 0;
    for (int64_t row = (int64_t)blockIdx.x * teams + team_id; row < rows; row += (int64_t)gridDim.x * teams, ++it)
      body(row, it);
  }
}

// ---------------------------------------------------------------------------
// Backward, vector path.
// ---------------------------------------------------------------------------
template <typename T, int NORM, int V, bool kWarpTeam>
__global__ void __launch_bounds__(kWarpTeam ? 256 : 512) norm_bwd_vec(const uint4 *dy, const uint4 *__restrict__ y,
                                                     const float *__restrict__ rstd, uint4 *dx, int64_t rows,
                                                     int nvec, int cols) {
  pdl_enter();
  constexpr int kVec = Traits<T>::kVec;
  __shared__ float2 red[2][32];
  const int team = kWarpTeam ? 32 : (int)blockDim.x;
  const int tid = kWarpTeam ? (int)(threadIdx.x & 31) : (int)threadIdx.x;
  const int teams = kWarpTeam ? (int)(blockDim.x >> 5) : 1;
  const int team_id = kWarpTeam ? (int)(threadIdx.x >> 5) : 0;
  const float fcols = (float)cols;
  auto body = [&](int64_t row, int it) {
    const uint4 *gr = dy + row * nvec;
    const uint4 *yr = y + row * nvec;
    const float r = rstd[row];
    uint4 rg[V], ry[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int vi = j * team + tid;
      if (vi < nvec) {
        rg[j] = ld_stream(gr + vi);
        ry[j] = ld_stream(yr + vi);
      } else {
        rg[j] = make_uint4(0u, 0u, 0u, 0u);
        ry[j] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
    float2 acc = make_float2(0.0f, 0.0f);  // (sum dy, sum dy*y)
#pragma unroll
    for (int j = 0; j < V; ++j) {
      float g[kVec], h[kVec];
      Vec<T>::unpack(rg[j], g);
      Vec<T>::unpack(ry[j], h);
#pragma unroll
      for (int k = 0; k < kVec; ++k) {
        if constexpr (NORM == kNormLN) acc.x += g[k];
        acc.y = fmaf(g[k], h[k], acc.y);
      }
    }
    acc = team_sum2<kWarpTeam>(acc, red[it & 1]);
    const float m1 = NORM == kNormLN ? __fdiv_rn(acc.x, fcols) : 0.0f;
    const float m2 = __fdiv_rn(acc.y, fcols);
    uint4 *dr = dx + row * nvec;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int vi = j * team + tid;
      if (vi < nvec) {
        float g[kVec], h[kVec];
        Vec<T>::unpack(rg[j], g);
        Vec<T>::unpack(ry[j], h);
#pragma unroll
        for (int k = 0; k < kVec; ++k) {
          const float c = NORM == kNormLN ? __fsub_rn(g[k], m1) : g[k];
          g[k] = __fmul_rn(r, fmaf(-h[k], m2, c));
        }
        st_stream(dr + vi, Vec<T>::pack(g));
      }
    }
  };
  if constexpr (kWarpTeam && V <= 4 && kNormClc) {
    clc_row_blocks(rows, teams, team_id, [&](int64_t row) { body(row, 0); });
  } else {
    int it = 0;
    for (int64_t row = (int64_t)blockIdx.x * teams + team_id; row < rows; row += (int64_t)gridDim.x * teams, ++it)
      body(row, it);
  }
}

// ---------------------------------------------------------------------------
// TMA-pipelined path (default for aligned rows that fit the shared-memory
// ring).  Every warp owns rows gw, gw + GW, ... (GW = warps in the grid) and
// streams them through its own ring of S stages: lane 0 issues cp.async.bulk
// copies of the next S rows (x; or dy and y) completing on the stage's
// mbarrier; the warp reduces and writes the current row from shared memory.
// No CTA-level synchronisation at all: reductions are warp butterflies over
// lane partials accumulated in a fixed order -> deterministic.
// ---------------------------------------------------------------------------
template <typename T, int NORM, bool kFwd>
__device__ __forceinline__ void norm_issue(uint8_t *stage, uint64_t *bar, const uint4 *a, const uint4 *b, int64_t row,
                                           int nvec) {
  const uint32_t rowbytes = (uint32_t)nvec * 16u;
  mbar_arrive_expect_tx(bar, kFwd ? rowbytes : 2u * rowbytes);
  bulk_g2s(stage, a + row * nvec, rowbytes, bar);
  if constexpr (!kFwd) bulk_g2s(stage + rowbytes, b + row * nvec, rowbytes, bar);
}

template <typename T, int NORM, bool kFwd>
__global__ void __launch_bounds__(512) norm_tma(const uint4 *a, const uint4 *b, const float *rstd_in, uint4 *out,
                                                float *rstd_out, int64_t rows, int nvec, int cols, float eps,
                                                int stages, int rpw) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int kVec = Traits<T>::kVec;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  const int stage_bytes = nvec * 16 * (kFwd ? 1 : 2);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem) + warp * stages;
  uint8_t *ring = smem + ((W * stages * 8 + 127) & ~127) + (size_t)warp * stages * stage_bytes;
  // rpw > 0: the CTA owns rows [b W rpw, (b + 1) W rpw) (grid = one CTA per
  // such block, balanced by the hardware block scheduler); rpw == 0:
  // persistent grid-stride over all rows.
  int64_t gw, GW, row_end;
  if (rpw > 0) {
    gw = (int64_t)blockIdx.x * W * rpw + warp;
    GW = W;
    row_end = min(rows, (int64_t)(blockIdx.x + 1) * W * rpw);
  } else {
    gw = (int64_t)blockIdx.x * W + warp;
    GW = (int64_t)gridDim.x * W;
    row_end = rows;
  }
  pdl_enter();
  const float fcols = (float)cols;
  if (lane == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
    for (int s = 0; s < stages; ++s) {
      const int64_t row = gw + s * GW;
      if (row < row_end) norm_issue<T, NORM, kFwd>(ring + (size_t)s * stage_bytes, &full[s], a, b, row, nvec);
    }
  }
  __syncwarp();
  int k = 0;
  for (int64_t row = gw; row < row_end; row += GW, ++k) {
    const int s = k % stages;
    mbar_wait(&full[s], (uint32_t)(k / stages) & 1u);
    const uint4 *sa = reinterpret_cast<const uint4 *>(ring + (size_t)s * stage_bytes);
    uint4 *orow = out + row * nvec;
    if constexpr (kFwd) {
      float mean = 0.0f;
      if constexpr (NORM == kNormLN) {
        float s0 = 0.0f, s1 = 0.0f;
        for (int vi = lane; vi < nvec; vi += 32) {
          float f[kVec];
          Vec<T>::unpack(lds128(sa + vi), f);
#pragma unroll
          for (int e = 0; e < kVec; e += 2) {
            s0 += f[e];
            s1 += f[e + 1];
          }
        }
        mean = __fdiv_rn(warp_sum(s0 + s1), fcols);
      }
      float q0 = 0.0f, q1 = 0.0f;
      for (int vi = lane; vi < nvec; vi += 32) {
        float f[kVec];
        Vec<T>::unpack(lds128(sa + vi), f);
#pragma unroll
        for (int e = 0; e < kVec; e += 2) {
          const float d0 = __fsub_rn(f[e], mean), d1 = __fsub_rn(f[e + 1], mean);
          q0 = fmaf(d0, d0, q0);
          q1 = fmaf(d1, d1, q1);
        }
      }
      const float r = rsqrtf(__fadd_rn(__fdiv_rn(warp_sum(q0 + q1), fcols), eps));
      for (int vi = lane; vi < nvec; vi += 32) {
        float f[kVec];
        Vec<T>::unpack(lds128(sa + vi), f);
#pragma unroll
        for (int e = 0; e < kVec; ++e) f[e] = __fmul_rn(__fsub_rn(f[e], mean), r);
        st_stream(orow + vi, Vec<T>::pack(f));
      }
      if (lane == 0) rstd_out[row] = r;
    } else {
      // Packed f32x2 math (FADD2/FFMA2/FMUL2) and four independent
      // accumulator pairs: the ring kernel runs few warps per SM (the ring
      // fills shared memory), so per-warp ILP decides its speed.
      const uint4 *sb = sa + nvec;
      const float r = rstd_in[row];
      const float2 z2 = make_float2(0.0f, 0.0f);
      float2 gs0 = z2, gs1 = z2, ps0 = z2, ps1 = z2;
#pragma unroll 2
      for (int vi = lane; vi < nvec; vi += 32) {
        float g[kVec], h[kVec];
        Vec<T>::unpack(lds128(sa + vi), g);
        Vec<T>::unpack(lds128(sb + vi), h);
#pragma unroll
        for (int e = 0; e < kVec; e += 4) {
          const float2 ga = make_float2(g[e], g[e + 1]), gb = make_float2(g[e + 2], g[e + 3]);
          if constexpr (NORM == kNormLN) {
            gs0 = __fadd2_rn(gs0, ga);
            gs1 = __fadd2_rn(gs1, gb);
          }
          ps0 = __ffma2_rn(ga, make_float2(h[e], h[e + 1]), ps0);
          ps1 = __ffma2_rn(gb, make_float2(h[e + 2], h[e + 3]), ps1);
        }
      }
      const float2 acc = warp_sum2(make_float2((gs0.x + gs0.y) + (gs1.x + gs1.y), (ps0.x + ps0.y) + (ps1.x + ps1.y)));
      const float m1 = NORM == kNormLN ? __fdiv_rn(acc.x, fcols) : 0.0f;
      const float m2 = __fdiv_rn(acc.y, fcols);
      const float2 nm1 = make_float2(-m1, -m1), nm2 = make_float2(-m2, -m2), r2 = make_float2(r, r);
#pragma unroll 2
      for (int vi = lane; vi < nvec; vi += 32) {
        float g[kVec], h[kVec];
        Vec<T>::unpack(lds128(sa + vi), g);
        Vec<T>::unpack(lds128(sb + vi), h);
#pragma unroll
        for (int e = 0; e < kVec; e += 2) {
          float2 c = make_float2(g[e], g[e + 1]);
          if constexpr (NORM == kNormLN) c = __fadd2_rn(c, nm1);
          const float2 o = __fmul2_rn(r2, __ffma2_rn(make_float2(h[e], h[e + 1]), nm2, c));
          g[e] = o.x;
          g[e + 1] = o.y;
        }
        st_stream(orow + vi, Vec<T>::pack(g));
      }
    }
    __syncwarp();  // every lane has finished reading stage s
    if (lane == 0) {
      const int64_t nr = row + (int64_t)stages * GW;
      if (nr < row_end) norm_issue<T, NORM, kFwd>(ring + (size_t)s * stage_bytes, &full[s], a, b, nr, nvec);
    }
  }
}

// ---------------------------------------------------------------------------
// Row pipeline: TMA staging + cluster-launch-control row stealing
// (rows of >= 256 vectors, i.e. the LLaMA shapes).
//
// One producer warp streams whole rows (x; or dy and y) into a ring of S
// shared-memory stages with cp.async.bulk; W consumer warps split each row
// (V lane-interleaved 16-byte vectors per thread, kept in registers), release
// the stage at once, reduce across the W warps through shared memory and one
// named barrier per reduction (the producer warp never joins it), and store.
// The grid has one CTA per row; the producer asks the hardware for
// not-yet-started CTAs (clusterlaunchcontrol.try_cancel) and takes over their
// rows, so rows are balanced dynamically over the SMs while each CTA keeps a
// single pipeline.  The row a stage holds is passed in a per-stage slot.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void consumer_bar(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

#ifndef LMBP_ROW_UNIT
#define LMBP_ROW_UNIT 1
#endif
// kF32Out (backward only): dx is written as fp32 (the mixed-precision
// backward of norm_mixed.cu: 16-bit dy, y -> fp32 residual gradient).
template <typename T, int NORM, bool kFwd, int V, bool kF32Out = false>
__global__ void __launch_bounds__(544) norm_row_tma(const uint4 *a, const uint4 *b, const float *rstd_in, uint4 *out,
                                                    float *rstd_out, int64_t rows, int nvec, int cols, float eps,
                                                    int stages) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int kVec = Traits<T>::kVec;
  constexpr int NIN = kFwd ? 1 : 2;
  const int W = (int)(blockDim.x >> 5) - 1;  // consumer warps
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t row_bytes = (size_t)nvec * 16;
  const size_t stage_bytes = row_bytes * NIN;
  const bool out32 = kUseV8 && ((uintptr_t)out & 31u) == 0;  // fp32 rows are 32 B multiples: whole 256-bit stores
  // layout: stages | clc response (16 B) | full[S] empty[S] clc_bar | slot[S] | red | rslot[S]
  uint4 *clc_resp = reinterpret_cast<uint4 *>(smem + (size_t)stages * stage_bytes);  // 16-byte aligned
  uint64_t *full = reinterpret_cast<uint64_t *>(clc_resp + 1);
  uint64_t *empty = full + stages;
  uint64_t *clc_bar = empty + stages;
  int64_t *slot = reinterpret_cast<int64_t *>(clc_bar + 1);
  float2 *red = reinterpret_cast<float2 *>(slot + stages);     // [2 parities][2 reductions][16 warps]
  float *rslot = reinterpret_cast<float *>(red + 64);          // backward: the stage row's rstd
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], W);
    }
    mbar_init(clc_bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  pdl_enter();

  if (warp == W) {  // producer
    if (lane == 0) {
      // backward: the producer loads the row's rstd (issued a row ahead, so
      // the load's latency hides behind the stage wait) and hands it over in
      // the stage's slot; the consumers never wait on global memory.
      // Work unit u = rows [u R, min(rows, (u + 1) R)), R = LMBP_ROW_UNIT.
      int64_t row = (int64_t)blockIdx.x * LMBP_ROW_UNIT;
      float rnext = 0.0f;
      if constexpr (!kFwd) rnext = rstd_in[row];
      uint32_t ph = 0;
      int k = 0;
      for (;;) {
        mbar_arrive_expect_tx(clc_bar, 16);
        clc_try_cancel(clc_resp, clc_bar);
        const int64_t row_end = min(rows, row + LMBP_ROW_UNIT);
        for (; row < row_end; ++row, ++k) {
          const int s = k % stages;
          mbar_wait(&empty[s], ((uint32_t)(k / stages) & 1u) ^ 1u);
          slot[s] = row;
          if constexpr (!kFwd) {
            rslot[s] = rnext;
            if (row + 1 < row_end) rnext = rstd_in[row + 1];
          }
          mbar_arrive_expect_tx(&full[s], (uint32_t)stage_bytes);
          uint8_t *st = smem + (size_t)s * stage_bytes;
          bulk_g2s(st, a + row * nvec, (uint32_t)row_bytes, &full[s]);
          if constexpr (!kFwd) bulk_g2s(st + row_bytes, b + row * nvec, (uint32_t)row_bytes, &full[s]);
        }
        mbar_wait(clc_bar, ph);
        ph ^= 1u;
        const int next = clc_query(clc_resp);
        if (next < 0) break;
        row = (int64_t)next * LMBP_ROW_UNIT;
        if constexpr (!kFwd) rnext = rstd_in[row];
      }
      const int s = k % stages;
      mbar_wait(&empty[s], ((uint32_t)(k / stages) & 1u) ^ 1u);
      slot[s] = -1;
      mbar_arrive(&full[s]);
    }
    return;
  }

  const int nthreads = W * 32;
  const int tid = threadIdx.x;
  const float fcols = (float)cols;
  for (int k = 0;; ++k) {
    const int s = k % stages;
    mbar_wait(&full[s], (uint32_t)(k / stages) & 1u);
    const int64_t row = slot[s];
    if (row < 0) break;
    float r_row = 0.0f;
    if constexpr (!kFwd) r_row = rslot[s];  // read before the stage is released
    const uint8_t *st = smem + (size_t)s * stage_bytes;
    uint4 ra[V], rb[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int vi = j * nthreads + tid;
      if (vi < nvec) {
        ra[j] = lds128(st + (size_t)vi * 16);
        if constexpr (!kFwd) rb[j] = lds128(st + row_bytes + (size_t)vi * 16);
      } else {
        ra[j] = make_uint4(0u, 0u, 0u, 0u);
        if constexpr (!kFwd) rb[j] = make_uint4(0u, 0u, 0u, 0u);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // row is in registers: the stage may be refilled
    float2 *rk = red + (k & 1) * 32;
    uint4 *orow = out + row * nvec;
    if constexpr (kFwd) {
      float mean = 0.0f;
      if constexpr (NORM == kNormLN) {
        float sm = 0.0f;
#pragma unroll
        for (int j = 0; j < V; ++j) {
          float f[kVec];
          Vec<T>::unpack(ra[j], f);
#pragma unroll
          for (int e = 0; e < kVec; ++e) sm += f[e];
        }
        sm = warp_sum(sm);
        if (lane == 0) rk[warp].x = sm;
        consumer_bar(nthreads);
        float t = 0.0f;
        for (int w = 0; w < W; ++w) t += rk[w].x;
        mean = __fdiv_rn(t, fcols);
      }
      float ss = 0.0f;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        if (j * nthreads + tid < nvec) {
          float f[kVec];
          Vec<T>::unpack(ra[j], f);
#pragma unroll
          for (int e = 0; e < kVec; ++e) {
            const float d = NORM == kNormLN ? __fsub_rn(f[e], mean) : f[e];
            ss = fmaf(d, d, ss);
          }
        }
      }
      ss = warp_sum(ss);
      if (lane == 0) rk[16 + warp].x = ss;
      consumer_bar(nthreads);
      float t = 0.0f;
      for (int w = 0; w < W; ++w) t += rk[16 + w].x;
      const float r = rsqrtf(__fadd_rn(__fdiv_rn(t, fcols), eps));
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int vi = j * nthreads + tid;
        if (vi < nvec) {
          float f[kVec];
          Vec<T>::unpack(ra[j], f);
#pragma unroll
          for (int e = 0; e < kVec; ++e) f[e] = __fmul_rn(NORM == kNormLN ? __fsub_rn(f[e], mean) : f[e], r);
          st_stream(orow + vi, Vec<T>::pack(f));
        }
      }
      if (tid == 0) rstd_out[row] = r;
    } else {
      const float r = r_row;
      float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        float g[kVec], h[kVec];
        Vec<T>::unpack(ra[j], g);
        Vec<T>::unpack(rb[j], h);
#pragma unroll
        for (int e = 0; e < kVec; ++e) {
          if constexpr (NORM == kNormLN) acc.x += g[e];
          acc.y = fmaf(g[e], h[e], acc.y);
        }
      }
      acc = warp_sum2(acc);
      if (lane == 0) rk[warp] = acc;
      consumer_bar(nthreads);
      float2 t = make_float2(0.0f, 0.0f);
      for (int w = 0; w < W; ++w) {
        t.x += rk[w].x;
        t.y += rk[w].y;
      }
      const float m1 = NORM == kNormLN ? __fdiv_rn(t.x, fcols) : 0.0f;
      const float m2 = __fdiv_rn(t.y, fcols);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int vi = j * nthreads + tid;
        if (vi < nvec) {
          float g[kVec], h[kVec];
          Vec<T>::unpack(ra[j], g);
          Vec<T>::unpack(rb[j], h);
#pragma unroll
          for (int e = 0; e < kVec; ++e) {
            const float c = NORM == kNormLN ? __fsub_rn(g[e], m1) : g[e];
            g[e] = __fmul_rn(r, fmaf(-h[e], m2, c));
          }
          if constexpr (kF32Out) {
            uint4 *o32 = out + row * (int64_t)nvec * 2;
            if (out32) {
              st_stream32(o32 + 2 * vi, Vec<float>::pack(g), Vec<float>::pack(g + 4));
            } else {
              st_stream(o32 + 2 * vi, Vec<float>::pack(g));
              st_stream(o32 + 2 * vi + 1, Vec<float>::pack(g + 4));
            }
          } else {
            st_stream(orow + vi, Vec<T>::pack(g));
          }
        }
      }
    }
  }
}

struct RowTmaPlan {
  bool ok;
  int warps;   // consumer warps
  int V;       // vectors per thread
  int stages;
  size_t smem;
};

static RowTmaPlan plan_row_tma(int64_t nvec, bool fwd) {
  RowTmaPlan p{false, 0, 0, 0, 0};
  if (nvec < 256 || nvec > 16 * 32 * 4) return p;
#ifndef LMBP_ROW_VAIM
#define LMBP_ROW_VAIM 4
#endif
#ifndef LMBP_ROW_STAGE_KB
#define LMBP_ROW_STAGE_KB 96
#endif
  int warps = (int)((nvec + LMBP_ROW_VAIM * 32 - 1) / (LMBP_ROW_VAIM * 32));  // aim for 4 vectors per thread
  if (warps > 16) warps = 16;
  const int V = (int)((nvec + warps * 32 - 1) / (warps * 32));
  // 17 warps under __launch_bounds__(544) leave ~120 registers per thread:
  // V > 4 would spill (ptxas), so wider rows (> 2048 vectors, H > 16384 at
  // 16 bits) take the per-warp ring instead.
  if (V > 4) return p;
  const size_t stage = (size_t)nvec * 16 * (fwd ? 1 : 2);
#ifndef LMBP_ROW_MAXST
#define LMBP_ROW_MAXST 4
#endif
  int stages = (int)std::min<size_t>(LMBP_ROW_MAXST, (size_t)(LMBP_ROW_STAGE_KB * 1024) / stage);
  if (stages < 2) stages = 2;
  const size_t tail = 16 + (2 * (size_t)stages + 1) * 8 + (size_t)stages * 8 + 64 * sizeof(float2) +
                      (size_t)stages * sizeof(float);
  p.smem = (size_t)stages * stage + tail;
  if (p.smem > 227 * 1024) return p;
  p.ok = true;
  p.warps = warps;
  p.V = V;
  p.stages = stages;
  return p;
}

template <typename T, int NORM, bool kFwd, int V, bool kF32Out = false>
static cudaError_t launch_row_tma_v(const RowTmaPlan &rp, const void *a, const void *b, const float *rstd_in,
                                    void *out, float *rstd_out, int64_t rows, int nvec, int64_t cols, float eps,
                                    cudaStream_t s) {
  auto kern = norm_row_tma<T, NORM, kFwd, V, kF32Out>;
  static std::atomic<unsigned long long> smem_set{0};
  const cudaError_t e = ensure_dyn_smem(kern, 227 * 1024, smem_set);
  if (e != cudaSuccess) return e;
  const int64_t units = (rows + LMBP_ROW_UNIT - 1) / LMBP_ROW_UNIT;
  if (units > 0x7fffffff) return cudaErrorInvalidValue;
  launch_k(kern, (int)units, (rp.warps + 1) * 32, rp.smem, s, reinterpret_cast<const uint4 *>(a),
           reinterpret_cast<const uint4 *>(b), rstd_in,
           reinterpret_cast<uint4 *>(out), rstd_out, rows, nvec,
           (int)cols, eps, rp.stages);
  return cudaGetLastError();
}

template <typename T, int NORM, bool kFwd, bool kF32Out = false>
static cudaError_t launch_row_tma(const RowTmaPlan &rp, const void *a, const void *b, const float *rstd_in, void *out,
                                  float *rstd_out, int64_t rows, int nvec, int64_t cols, float eps, cudaStream_t s) {
  switch (rp.V) {
    case 1: return launch_row_tma_v<T, NORM, kFwd, 1, kF32Out>(rp, a, b, rstd_in, out, rstd_out, rows, nvec, cols, eps, s);
    case 2: return launch_row_tma_v<T, NORM, kFwd, 2, kF32Out>(rp, a, b, rstd_in, out, rstd_out, rows, nvec, cols, eps, s);
    case 3: return launch_row_tma_v<T, NORM, kFwd, 3, kF32Out>(rp, a, b, rstd_in, out, rstd_out, rows, nvec, cols, eps, s);
    default: return launch_row_tma_v<T, NORM, kFwd, 4, kF32Out>(rp, a, b, rstd_in, out, rstd_out, rows, nvec, cols, eps, s);
  }
}

struct TmaPlan {
  bool ok;
  int warps, stages;
  size_t smem;
};

// Shared-memory budget per CTA for the ring (B200: 227 KB opt-in per CTA,
// minus the barriers).  More rings per SM = finer row granularity: at C4
// (16 KB row pairs) 7 rings of 2 stages would fit in 224 KB; measured no gain.
#ifndef LMBP_NORM_SMEM_KB
#define LMBP_NORM_SMEM_KB 200
#endif
constexpr size_t kNormSmemBudget = LMBP_NORM_SMEM_KB * 1024;

static TmaPlan plan_tma(int nvec, bool fwd) {
  const size_t stage = (size_t)nvec * 16 * (fwd ? 1 : 2);
  TmaPlan p{false, 0, 0, 0};
  int stages = stage <= 4096 ? 4 : (stage <= 12288 ? 3 : 2);
  int warps = (int)std::min<size_t>(16, kNormSmemBudget / (stages * stage));
  while (warps < 1 && stages > 2) {
    --stages;
    warps = (int)std::min<size_t>(16, kNormSmemBudget / (stages * stage));
  }
  if (warps < 1) return p;
  p.ok = true;
  p.warps = warps;
  p.stages = stages;
  p.smem = ((size_t)warps * stages * 8 + 127) / 128 * 128 + (size_t)warps * stages * stage;
  return p;
}

template <typename T, int NORM, bool kFwd>
static cudaError_t launch_norm_tma(const TmaPlan &tp, const void *a, const void *b, const float *rstd_in, void *out,
                            float *rstd_out, int64_t rows, int nvec, int64_t cols, float eps, cudaStream_t s) {
  auto kern = norm_tma<T, NORM, kFwd>;
  static std::atomic<unsigned long long> smem_set{0};
  const cudaError_t e = ensure_dyn_smem(kern, 227 * 1024, smem_set);
  if (e != cudaSuccess) return e;
  const int threads = tp.warps * 32;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, tp.smem) != cudaSuccess || occ < 1) occ = 1;
#ifndef LMBP_NORM_RPW
#define LMBP_NORM_RPW 0
#endif
  const int rpw = LMBP_NORM_RPW;
  const int64_t want = (rows + tp.warps - 1) / tp.warps;
  const int grid = rpw > 0 ? (int)std::max<int64_t>(1, (rows + (int64_t)tp.warps * rpw - 1) / ((int64_t)tp.warps * rpw))
                           : (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count() * occ));
  launch_k(kern, grid, threads, tp.smem, s, reinterpret_cast<const uint4 *>(a), reinterpret_cast<const uint4 *>(b), rstd_in,
           reinterpret_cast<uint4 *>(out), rstd_out, rows, nvec, (int)cols, eps, tp.stages,
           rpw);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Scalar multi-pass fallback (any alignment / any length): one CTA per row.
// ---------------------------------------------------------------------------
template <typename T, int NORM>
__global__ void __launch_bounds__(256) norm_fwd_scalar(const T *x, T *y, float *rstd, int64_t rows, int64_t cols,
                                                       float eps) {
  pdl_enter();
  __shared__ float red[2][32];
  const float fcols = (float)cols;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const T *xr = x + row * cols;
    float mean = 0.0f;
    if constexpr (NORM == kNormLN) {
      float s = 0.0f;
      for (int64_t i = threadIdx.x; i < cols; i += blockDim.x) s += to_f32<T>(xr[i]);
      mean = __fdiv_rn(team_sum<false>(s, red[0]), fcols);
    }
    float ss = 0.0f;
    for (int64_t i = threadIdx.x; i < cols; i += blockDim.x) {
      const float d = __fsub_rn(to_f32<T>(xr[i]), mean);
      ss = fmaf(d, d, ss);
    }
    ss = team_sum<false>(ss, red[1]);
    const float r = rsqrtf(__fadd_rn(__fdiv_rn(ss, fcols), eps));
    __syncthreads();  // every thread has read x before any y store (y may alias x)
    T *yr = y + row * cols;
    for (int64_t i = threadIdx.x; i < cols; i += blockDim.x)
      yr[i] = from_f32<T>(__fmul_rn(__fsub_rn(to_f32<T>(xr[i]), mean), r));
    if (threadIdx.x == 0) rstd[row] = r;
    __syncthreads();
  }
}

template <typename T, int NORM>
__global__ void __launch_bounds__(256) norm_bwd_scalar(const T *dy, const T *y, const float *rstd, T *dx,
                                                       int64_t rows, int64_t cols) {
  pdl_enter();
  __shared__ float2 red[2][32];
  const float fcols = (float)cols;
  int it = 0;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x, ++it) {
    const T *gr = dy + row * cols;
    const T *yr = y + row * cols;
    float2 acc = make_float2(0.0f, 0.0f);
    for (int64_t i = threadIdx.x; i < cols; i += blockDim.x) {
      const float g = to_f32<T>(gr[i]);
      if constexpr (NORM == kNormLN) acc.x += g;
      acc.y = fmaf(g, to_f32<T>(yr[i]), acc.y);
    }
    acc = team_sum2<false>(acc, red[it & 1]);
    const float m1 = NORM == kNormLN ? __fdiv_rn(acc.x, fcols) : 0.0f;
    const float m2 = __fdiv_rn(acc.y, fcols);
    const float r = rstd[row];
    __syncthreads();  // dx may alias dy
    T *dr = dx + row * cols;
    for (int64_t i = threadIdx.x; i < cols; i += blockDim.x) {
      const float g = to_f32<T>(gr[i]);
      const float c = NORM == kNormLN ? __fsub_rn(g, m1) : g;
      dr[i] = from_f32<T>(__fmul_rn(r, fmaf(-to_f32<T>(yr[i]), m2, c)));
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Launch configuration.
// ---------------------------------------------------------------------------
// Warp teams: the forward takes rows up to 8 vectors per lane (fp32 H = 768:
// C3 18.4 -> 17.2 us, faster than a torch copy of its bytes), the backward up
// to 4 (a 6-vector warp team measured slower there than the 64-thread CTA
// team); profiles/r01/sweep25_norm_small_rows.jsonl.
constexpr int kWarpVmaxFwd = 8, kWarpVmaxBwd = 4;

struct RowPlan {
  bool vec;
  bool warp_team;
  int team;  // threads per row
  int V;     // vectors per thread
  int nvec;  // vectors per row
};

template <typename T>
static RowPlan plan_rows(int64_t cols, const void *a, const void *b, const void *c, int warp_vmax) {
  constexpr int kVec = Traits<T>::kVec;
  RowPlan p{false, false, 0, 0, 0};
  const bool aligned = ((uintptr_t)a % 16 == 0) && ((uintptr_t)b % 16 == 0) && ((uintptr_t)c % 16 == 0) &&
                       (cols % kVec == 0);
  if (!aligned) return p;
  const int64_t nvec = cols / kVec;
  if (nvec > 8 * 512) return p;
  p.nvec = (int)nvec;
  if (nvec <= warp_vmax * 32) {  // one warp per row, up to warp_vmax vectors per lane
    p.warp_team = true;
    p.team = 32;
    p.V = (int)((nvec + 31) / 32);
  } else {
#ifndef LMBP_NORM_VAIM
#define LMBP_NORM_VAIM 4
#endif
    const int64_t want = (nvec + LMBP_NORM_VAIM - 1) / LMBP_NORM_VAIM;  // aim for 4 vectors per thread
    int64_t team = ((want + 31) / 32) * 32;
    if (team > 512) team = 512;
    p.team = (int)team;
    p.V = (int)((nvec + team - 1) / team);
  }
  p.vec = p.V >= 1 && p.V <= (p.warp_team ? warp_vmax : 8);
  return p;
}

// Resident CTAs per SM for (kernel, threads).  The kernel is a template
// argument, so every kernel instantiation has its own cache, slotted by block
// size (a benign race: every writer stores the same value).
template <auto Kern>
static int occupancy_of(int threads) {
  static std::atomic<int> cache[33];  // zero-initialised (static storage)
  const auto kernel = Kern;
  const int slot = threads >> 5;
  if (slot < 33) {
    const int c = cache[slot].load(std::memory_order_relaxed);
    if (c > 0) return c;
  }
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, 0) != cudaSuccess || b < 1) b = 1;
  if (slot < 33) cache[slot].store(b, std::memory_order_relaxed);
  return b;
}

// Grid for the register-team kernels.  CTA teams (one row per CTA) launch one
// CTA per row and let the hardware block scheduler balance the SMs (measured
// C4 MS-RMSNorm fwd 22.4 -> 20.5 us, C3 MS-LN bwd 24.6 -> 22.5 us); warp teams
// (8 short rows per CTA) of up to 4 vectors per lane keep a persistent grid,
// which measured faster there (C2 bwd 14.4 vs 16.4 us); longer warp rows
// (V > 4, the fp32 H = 768 forward) launch every CTA (C3 fwd 17.2 vs 18.4 us).
template <typename K, typename... Args>
static void launch_rows(K kernel, int64_t rows, int rows_per_block, int threads, cudaStream_t s, int occ,
                        bool persistent, Args... args) {
  const int64_t want = (rows + rows_per_block - 1) / rows_per_block;
#ifdef LMBP_NORM_NO_PERSIST  // tuning knob (tools/gpu_stream_ab.sh): warp teams launch every CTA too
  persistent = false;
#endif
  const int64_t cap = (rows_per_block == 1 || !persistent) ? (int64_t)0x7fffffff : (int64_t)sm_count() * occ;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, cap));
  launch_k(kernel, grid, threads, 0, s, args...);
}

template <typename T, int NORM, int V, bool W>
static void fwd_v(const RowPlan &p, const void *x, void *y, float *rstd, int64_t rows, int64_t cols, float eps,
                  cudaStream_t s) {
  auto k = norm_fwd_vec<T, NORM, V, W>;
  const int threads = W ? 256 : p.team;
  const int occ = occupancy_of<norm_fwd_vec<T, NORM, V, W>>(threads);
  launch_rows(k, rows, W ? threads / 32 : 1, threads, s, occ, V <= 4 && !(W && kNormFwdClc), reinterpret_cast<const uint4 *>(x),
              reinterpret_cast<uint4 *>(y), rstd, rows, p.nvec, (int)cols, eps);
}

template <typename T, int NORM, int V, bool W>
static void bwd_v(const RowPlan &p, const void *dy, const void *y, const float *rstd, void *dx, int64_t rows,
                  int64_t cols, cudaStream_t s) {
  auto k = norm_bwd_vec<T, NORM, V, W>;
  const int threads = W ? 256 : p.team;
  const int occ = occupancy_of<norm_bwd_vec<T, NORM, V, W>>(threads);
  launch_rows(k, rows, W ? threads / 32 : 1, threads, s, occ, !(W && V <= 4 && kNormClc), reinterpret_cast<const uint4 *>(dy),
              reinterpret_cast<const uint4 *>(y), rstd, reinterpret_cast<uint4 *>(dx), rows, p.nvec, (int)cols);
}

template <typename T, int NORM>
static cudaError_t norm_fwd_t(const void *x, void *y, float *rstd, int64_t rows, int64_t cols, float eps,
                              cudaStream_t s) {
  const RowPlan p = plan_rows<T>(cols, x, y, y, kWarpVmaxFwd);
#ifdef LMBP_ROW_TMA_FWD  // measured slower than the register teams for the forward (C4 24.6 vs 20.5 us)
  if (p.vec && rows > 0) {
    const RowTmaPlan rp = plan_row_tma(p.nvec, true);
    if (rp.ok) return launch_row_tma<T, NORM, true>(rp, x, nullptr, nullptr, y, rstd, rows, p.nvec, cols, eps, s);
  }
#endif
  // Forward: the register-resident team kernel measured faster than the TMA
  // ring at every BASELINE shape (C4 21.9 vs 23.5 us, C5 104 vs 117 us), so
  // the ring is only used where registers cannot hold a row.
  if (!p.vec) {
    const int64_t nv = cols / Traits<T>::kVec;
    const bool ok16 = cols % Traits<T>::kVec == 0 && (uintptr_t)x % 16 == 0 && (uintptr_t)y % 16 == 0;
    const TmaPlan tp = ok16 && nv < (1 << 26) ? plan_tma((int)nv, true) : TmaPlan{false, 0, 0, 0};
    if (tp.ok) {
      return launch_norm_tma<T, NORM, true>(tp, x, nullptr, nullptr, y, rstd, rows, (int)nv, cols, eps, s);
    }
  }
  if (!p.vec) {
    auto k = norm_fwd_scalar<T, NORM>;
    launch_rows(k, rows, 1, 256, s, occupancy_of<norm_fwd_scalar<T, NORM>>(256), true, reinterpret_cast<const T *>(x), reinterpret_cast<T *>(y),
                rstd, rows, cols, eps);
    return cudaGetLastError();
  }
#define LMBP_FWD_CASE(VV)                                                                   \
  case VV:                                                                                  \
    if constexpr (VV <= kWarpVmaxFwd) {                                                     \
      if (p.warp_team) {                                                                    \
        fwd_v<T, NORM, (VV <= kWarpVmaxFwd ? VV : 1), true>(p, x, y, rstd, rows, cols, eps, s);        \
        break;                                                                              \
      }                                                                                     \
    }                                                                                       \
    fwd_v<T, NORM, VV, false>(p, x, y, rstd, rows, cols, eps, s);                           \
    break;
  switch (p.V) {
    LMBP_FWD_CASE(1) LMBP_FWD_CASE(2) LMBP_FWD_CASE(3) LMBP_FWD_CASE(4)
    LMBP_FWD_CASE(5) LMBP_FWD_CASE(6) LMBP_FWD_CASE(7) LMBP_FWD_CASE(8)
    default: break;
  }
#undef LMBP_FWD_CASE
  return cudaGetLastError();
}

template <typename T, int NORM>
static cudaError_t norm_bwd_t(const void *dy, const void *y, const float *rstd, void *dx, int64_t rows,
                              int64_t cols, cudaStream_t s) {
  const RowPlan p = plan_rows<T>(cols, dy, y, dx, kWarpVmaxBwd);
#ifndef LMBP_NO_ROW_TMA  // backward rows >= 256 vectors: row pipeline (C5 160 -> 147 us; C4 equal)
  if (p.vec && rows > 0) {
    const RowTmaPlan rp = plan_row_tma(p.nvec, false);
    if (rp.ok) return launch_row_tma<T, NORM, false>(rp, dy, y, rstd, dx, nullptr, rows, p.nvec, cols, 0.0f, s);
  }
#endif
  // Backward: the TMA ring wins once a row pair (dy, y) is >= 8 KB (C4: 32.8
  // vs 34.6 us, C5: 160 vs 172 us); short rows (H = 768) stay on the register
  // team kernel (C2/C3 measured faster there).  Rows too long for registers
  // also take the ring when it fits.
  {
    const int64_t nv = cols / Traits<T>::kVec;
    const bool ok16 = cols % Traits<T>::kVec == 0 && (uintptr_t)dy % 16 == 0 && (uintptr_t)y % 16 == 0 &&
                      (uintptr_t)dx % 16 == 0;
#ifdef LMBP_NORM_NO_TMA
    const bool want = ok16 && !p.vec && nv < (1 << 26);
#else
    const bool want = ok16 && (!p.vec || nv * 32 >= 8192) && nv < (1 << 26);
#endif
    const TmaPlan tp = want ? plan_tma((int)nv, false) : TmaPlan{false, 0, 0, 0};
    if (tp.ok) {
      return launch_norm_tma<T, NORM, false>(tp, dy, y, rstd, dx, nullptr, rows, (int)nv, cols, 0.0f, s);
    }
  }
  if (!p.vec) {
    auto k = norm_bwd_scalar<T, NORM>;
    launch_rows(k, rows, 1, 256, s, occupancy_of<norm_bwd_scalar<T, NORM>>(256), true, reinterpret_cast<const T *>(dy),
                reinterpret_cast<const T *>(y), rstd, reinterpret_cast<T *>(dx), rows, cols);
    return cudaGetLastError();
  }
#define LMBP_BWD_CASE(VV)                                                                   \
  case VV:                                                                                  \
    if constexpr (VV <= kWarpVmaxBwd) {                                                     \
      if (p.warp_team) {                                                                    \
        bwd_v<T, NORM, (VV <= kWarpVmaxBwd ? VV : 1), true>(p, dy, y, rstd, dx, rows, cols, s);        \
        break;                                                                              \
      }                                                                                     \
    }                                                                                       \
    bwd_v<T, NORM, VV, false>(p, dy, y, rstd, dx, rows, cols, s);                           \
    break;
  switch (p.V) {
    LMBP_BWD_CASE(1) LMBP_BWD_CASE(2) LMBP_BWD_CASE(3) LMBP_BWD_CASE(4)
    LMBP_BWD_CASE(5) LMBP_BWD_CASE(6) LMBP_BWD_CASE(7) LMBP_BWD_CASE(8)
    default: break;
  }
#undef LMBP_BWD_CASE
  return cudaGetLastError();
}

// Mixed-precision backward on the row pipeline (norm_mixed.cu): 16-bit dy, y
// (dtype 1 / 2) -> fp32 dx, for rows the ring holds (>= 256 vectors, as the
// same-type backward); cudaErrorNotSupported otherwise (the caller falls back).
cudaError_t norm_bwd_mixed_rows(int kind, int dtype, const void *dy, const void *y, const float *rstd, float *dx,
                                int64_t rows, int64_t cols, cudaStream_t s) {
  if (cols % 8 != 0 || ((uintptr_t)dy | (uintptr_t)y | (uintptr_t)dx) % 16 != 0 || rows <= 0)
    return cudaErrorNotSupported;
  const int64_t nvec = cols / 8;
  const RowTmaPlan rp = plan_row_tma(nvec, false);
  if (!rp.ok) return cudaErrorNotSupported;
  if (kind == kNormLN)
    return dtype == 1 ? launch_row_tma<__nv_bfloat16, kNormLN, false, true>(rp, dy, y, rstd, dx, nullptr, rows, (int)nvec, cols, 0.0f, s)
                      : launch_row_tma<__half, kNormLN, false, true>(rp, dy, y, rstd, dx, nullptr, rows, (int)nvec, cols, 0.0f, s);
  return dtype == 1 ? launch_row_tma<__nv_bfloat16, kNormRMS, false, true>(rp, dy, y, rstd, dx, nullptr, rows, (int)nvec, cols, 0.0f, s)
                    : launch_row_tma<__half, kNormRMS, false, true>(rp, dy, y, rstd, dx, nullptr, rows, (int)nvec, cols, 0.0f, s);
}

cudaError_t norm_fwd(int kind, int dtype, const void *x, void *y, float *rstd, int64_t rows, int64_t cols, float eps,
                     cudaStream_t s) {
  if (kind == kNormLN) {
    if (dtype == 0) return norm_fwd_t<float, kNormLN>(x, y, rstd, rows, cols, eps, s);
    if (dtype == 1) return norm_fwd_t<__nv_bfloat16, kNormLN>(x, y, rstd, rows, cols, eps, s);
    return norm_fwd_t<__half, kNormLN>(x, y, rstd, rows, cols, eps, s);
  }
  if (dtype == 0) return norm_fwd_t<float, kNormRMS>(x, y, rstd, rows, cols, eps, s);
  if (dtype == 1) return norm_fwd_t<__nv_bfloat16, kNormRMS>(x, y, rstd, rows, cols, eps, s);
  return norm_fwd_t<__half, kNormRMS>(x, y, rstd, rows, cols, eps, s);
}

cudaError_t norm_bwd(int kind, int dtype, const void *dy, const void *y, const float *rstd, void *dx, int64_t rows,
                     int64_t cols, cudaStream_t s) {
  if (kind == kNormLN) {
    if (dtype == 0) return norm_bwd_t<float, kNormLN>(dy, y, rstd, dx, rows, cols, s);
    if (dtype == 1) return norm_bwd_t<__nv_bfloat16, kNormLN>(dy, y, rstd, dx, rows, cols, s);
    return norm_bwd_t<__half, kNormLN>(dy, y, rstd, dx, rows, cols, s);
  }
  if (dtype == 0) return norm_bwd_t<float, kNormRMS>(dy, y, rstd, dx, rows, cols, s);
  if (dtype == 1) return norm_bwd_t<__nv_bfloat16, kNormRMS>(dy, y, rstd, dx, rows, cols, s);
  return norm_bwd_t<__half, kNormRMS>(dy, y, rstd, dx, rows, cols, s);
}

}  // namespace lmbp
