// ew_pipeline.cuh -- generic TMA bulk-copy pipeline for elementwise kernels
// over up to three 16-byte-vector input streams (+ optional packed codes).
//
// One producer warp (one elected lane) streams tiles of every input into a
// ring of S shared-memory stages with cp.async.bulk (the TMA engine; the data
// is contiguous, so no tensor map), completion on a per-stage mbarrier with
// expect_tx.  W consumer warps copy their slice of a tile into registers,
// release the stage at once (one mbarrier arrive per warp) so the producer
// refills it while they compute, and store their outputs straight to global
// memory with coalesced 16-byte stores.  Loads in flight per SM = resident
// CTAs x S x stage bytes, independent of the per-element math latency.
//
// An Op supplies the shape and the per-vector work:
//   static constexpr int W, U, S;   consumer warps, vectors per lane per tile, stages
//   static constexpr int kIn;       input streams (1..3)
//   static constexpr int kCodeIn;   bytes of packed codes read per vector (0, 1, 2)
//   __device__ static void apply(const uint4 (&v)[kIn], uint32_t code, int64_t i, const EwParams &p);
//   __device__ static void tail(const EwParams &p);   elements [nvec * kVec, n), one thread
#pragma once

#include "common.cuh"

namespace lmbp {

struct EwParams {
  const uint4 *in[3];        // input streams, nvec 16-byte vectors each
  const uint8_t *codes_in;   // packed codes (backward ops): vector i's code word is word i
  uint4 *out[2];             // output streams
  uint8_t *codes_out;        // packed codes written by forward ops
  int64_t nvec;              // whole 16-byte vectors
  int64_t n;                 // elements
};

template <class Op> struct EwShape {
  static constexpr int kTile = Op::W * 32 * Op::U;  // vectors per tile
  static constexpr int kThreads = (Op::W + 1) * 32;
  static constexpr size_t kStageBytes = (size_t)Op::kIn * kTile * 16 + (size_t)Op::kCodeIn * kTile;
  static constexpr size_t kSmem = (size_t)Op::S * kStageBytes + 2 * (size_t)Op::S * sizeof(uint64_t);
  static_assert(kStageBytes % 16 == 0, "stage must stay 16-byte aligned");
};

template <int kCodeIn>
__device__ __forceinline__ uint32_t code_word(const uint8_t *base, int64_t i) {
  if constexpr (kCodeIn == 2) return reinterpret_cast<const uint16_t *>(base)[i];
  else if constexpr (kCodeIn == 1) return base[i];
  else return 0u;
}

template <class Op>
__global__ void __launch_bounds__(EwShape<Op>::kThreads) ew_tma(const EwParams p) {
  extern __shared__ __align__(128) uint8_t smem[];
  using Sh = EwShape<Op>;
  constexpr int W = Op::W, U = Op::U, S = Op::S, NIN = Op::kIn, TILE = Sh::kTile;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)S * Sh::kStageBytes);
  uint64_t *empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = p.nvec / TILE;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], W);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == W) {  // producer
    if (lane == 0) {
      int k = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int s = k % S;
        mbar_wait(&empty[s], ((uint32_t)(k / S) & 1u) ^ 1u);
        mbar_arrive_expect_tx(&full[s], (uint32_t)Sh::kStageBytes);
        uint8_t *st = smem + (size_t)s * Sh::kStageBytes;
#pragma unroll
        for (int m = 0; m < NIN; ++m) bulk_g2s(st + (size_t)m * TILE * 16, p.in[m] + t * TILE, TILE * 16, &full[s]);
        if constexpr (Op::kCodeIn > 0)
          bulk_g2s(st + (size_t)NIN * TILE * 16, p.codes_in + t * TILE * Op::kCodeIn, TILE * Op::kCodeIn, &full[s]);
      }
    }
    return;
  }

  int k = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % S;
    mbar_wait(&full[s], (uint32_t)(k / S) & 1u);
    const uint8_t *st = smem + (size_t)s * Sh::kStageBytes;
    uint4 v[U][NIN];
    uint32_t c[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int vi = j * (W * 32) + warp * 32 + lane;
#pragma unroll
      for (int m = 0; m < NIN; ++m) v[j][m] = lds128(st + ((size_t)m * TILE + vi) * 16);
      c[j] = code_word<Op::kCodeIn>(st + (size_t)NIN * TILE * 16, vi);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // the stage may be refilled while we compute
#pragma unroll
    for (int j = 0; j < U; ++j) Op::apply(v[j], c[j], t * TILE + j * (W * 32) + warp * 32 + lane, p);
  }

  if (blockIdx.x == 0) {  // leftover vectors (< one tile), then the ragged element tail
    for (int64_t i = ntiles * TILE + threadIdx.x; i < p.nvec; i += W * 32) {
      uint4 v[NIN];
#pragma unroll
      for (int m = 0; m < NIN; ++m) v[m] = ld_stream(p.in[m] + i);
      Op::apply(v, code_word<Op::kCodeIn>(p.codes_in, i), i, p);
    }
    if (threadIdx.x == 0) Op::tail(p);
  }
}

// Launch on a persistent grid of SMs x resident CTAs (at most one CTA per tile).
template <class Op>
cudaError_t launch_ew(const EwParams &p, cudaStream_t stream) {
  using Sh = EwShape<Op>;
  auto kern = ew_tma<Op>;
  static const int occ = [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Sh::kSmem);
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, Sh::kThreads, Sh::kSmem) != cudaSuccess || b < 1)
      b = 1;
    return b;
  }();
  const int64_t tiles = p.nvec / Sh::kTile;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sm_count() * occ));
  kern<<<grid, Sh::kThreads, Sh::kSmem, stream>>>(p);
  return cudaGetLastError();
}

}  // namespace lmbp
