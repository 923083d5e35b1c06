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
//   static constexpr int kCodeIn;   bytes of packed codes read per vector (0 .. 4)
//   static constexpr int kCodeOut;  bytes of packed codes written per vector (0 .. 4; 3 = k = 3
//                                   codes of 8 16-bit elements, written / read as single bytes)
//   using Params = ...;            optional, a struct derived from EwParams (default EwParams)
//   __device__ static uint32_t apply(const uint4 (&v)[kIn], uint32_t code, int64_t i, const Params &p);
//       -> the code word of vector i (ignored when kCodeOut == 0)
//   __device__ static void tail(const Params &p);   elements [nvec * kVec, n), one thread
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

// An Op may extend the parameters (`using Params = ...;`, derived from
// EwParams); the kernel takes that type by value, so only the ops that need
// extra data pay for a larger parameter block (a 128-byte step table in every
// op's parameters cost the fp32 SwiGLU backward a register spill).
template <class Op, class = void> struct ParamsOf { using type = EwParams; };
template <class Op> struct ParamsOf<Op, std::void_t<typename Op::Params>> { using type = typename Op::Params; };

// Optional `static constexpr int kMinBlocks` (CTAs that must fit per SM;
// default: no register cap beyond the CTA size).
template <class Op, class = void> struct MinBlocksOf { static constexpr int value = 0; };
template <class Op> struct MinBlocksOf<Op, std::void_t<decltype(Op::kMinBlocks)>> {
  static constexpr int value = Op::kMinBlocks;
};

// Optional 16-bit lookup table (the ReGELU2 / ReSiLU2 forward of 16-bit
// types, lut.py): an Op with `static constexpr bool kTab16 = true` and
// `__device__ static const uint16_t *tab16()` (a 65536-entry table in global
// memory) gets it copied once per CTA into the first 128 KB of shared memory
// (bulk copies on their own mbarrier, issued by the producer before the first
// tile) and receives its shared-window address as a trailing `uint32_t`
// argument of apply().
template <class Op, class = void> struct Tab16Of { static constexpr bool value = false; };
template <class Op> struct Tab16Of<Op, std::void_t<decltype(Op::kTab16)>> { static constexpr bool value = Op::kTab16; };
constexpr uint32_t kTab16Bytes = 65536 * 2;

// Optional per-CTA code table (the k-bit step forwards, stepact.cu): an Op
// with `static constexpr bool kCtab = true` gets 64 KB of shared memory after
// the 16-bit table, which its consumer threads fill at CTA start through
// `__device__ static void fill_ctab(uint8_t *ctab, const Params &, int tid,
// int nthreads)` (a named barrier among the consumers follows; the producer
// starts streaming tiles meanwhile).
template <class Op, class = void> struct CtabOf { static constexpr bool value = false; };
template <class Op> struct CtabOf<Op, std::void_t<decltype(Op::kCtab)>> { static constexpr bool value = Op::kCtab; };
constexpr uint32_t kCtabBytes = 65536;

// Shared-window addresses of the tables an Op's apply() / tail() receive.
struct Tabs {
  uint32_t y;     // 16-bit output table (Tab16Of)
  uint32_t code;  // byte-per-pattern code table (CtabOf)
};

template <class Op> struct EwShape {
  static constexpr size_t kTabBytes = (Tab16Of<Op>::value ? kTab16Bytes : 0) + (CtabOf<Op>::value ? kCtabBytes : 0);
  static constexpr int kTile = Op::W * 32 * Op::U;  // vectors per tile
  static constexpr int kThreads = (Op::W + 1) * 32;
  static constexpr size_t kStageBytes = (size_t)Op::kIn * kTile * 16 + (size_t)Op::kCodeIn * kTile;
  // per-warp staging of the codes a warp writes for one tile (32 U words)
  static constexpr size_t kWarpCodeBytes = (size_t)32 * Op::U * Op::kCodeOut;
  static constexpr size_t kCodeStage = (size_t)Op::W * kWarpCodeBytes;
  // [table] | stages | code staging | full[S] empty[S] clc_bar tab_bar | slot[S+1] | clc response (16 B)
  static constexpr size_t kBarBytes = (2 * (size_t)Op::S + 2) * sizeof(uint64_t);
  static constexpr size_t kSlotBytes = (((size_t)Op::S + 1) * sizeof(int64_t) + 15) / 16 * 16;
  static constexpr size_t kSmemUsed = kTabBytes + (size_t)Op::S * kStageBytes + kCodeStage + kBarBytes + kSlotBytes + 16;
#ifdef LMBP_EW_ONE_CTA  // tuning knob: request > half the SM's shared memory so one CTA runs per SM
  static constexpr size_t kSmem = kSmemUsed > 116 * 1024 ? kSmemUsed : 116 * 1024;
#else
  static constexpr size_t kSmem = kSmemUsed;
#endif
  static_assert(kStageBytes % 16 == 0, "stage must stay 16-byte aligned");
  static_assert(kWarpCodeBytes % 16 == 0, "code staging must stay 16-byte aligned");
};

template <int kCodeOut>
__device__ __forceinline__ void put_code(uint8_t *base, int64_t i, uint32_t c) {
  if constexpr (kCodeOut == 4) reinterpret_cast<uint32_t *>(base)[i] = c;
  else if constexpr (kCodeOut == 3) {
    base[3 * i] = (uint8_t)c;
    base[3 * i + 1] = (uint8_t)(c >> 8);
    base[3 * i + 2] = (uint8_t)(c >> 16);
  } else if constexpr (kCodeOut == 2) reinterpret_cast<uint16_t *>(base)[i] = (uint16_t)c;
  else if constexpr (kCodeOut == 1) base[i] = (uint8_t)c;
}

template <int kCodeIn>
__device__ __forceinline__ uint32_t code_word(const uint8_t *base, int64_t i) {
  if constexpr (kCodeIn == 4) return reinterpret_cast<const uint32_t *>(base)[i];
  else if constexpr (kCodeIn == 3)
    return (uint32_t)base[3 * i] | ((uint32_t)base[3 * i + 1] << 8) | ((uint32_t)base[3 * i + 2] << 16);
  else if constexpr (kCodeIn == 2) return reinterpret_cast<const uint16_t *>(base)[i];
  else if constexpr (kCodeIn == 1) return base[i];
  else return 0u;
}

// Tile schedule: hardware work stealing with cluster launch control.  The
// grid has one CTA per work unit of kUnit consecutive tiles (+ one pseudo-tile
// index == ntiles that stands for the leftover vectors and the ragged tail).
// Each running CTA's producer lane asks the hardware (clusterlaunchcontrol.
// try_cancel) for a not-yet-started CTA of the grid and takes over its unit,
// so the block scheduler's dynamic balance is kept without paying a CTA
// launch, barrier initialisation and pipeline ramp per unit.  The producer
// tells the consumers which tile a stage holds through a per-stage slot
// (written before the stage's mbarrier arrive, read after its wait); -1 ends.
#ifndef LMBP_EW_UNIT
#define LMBP_EW_UNIT 1
#endif

// Optional per-CTA lookup table in shared memory: an Op with
// `static constexpr int kLut` and `static float lut_entry(const Params &, int)`
// gets the filled table as a trailing `const float *` argument of apply().
template <class Op, class = void> struct LutOf { static constexpr int value = 0; };
template <class Op> struct LutOf<Op, std::void_t<decltype(Op::kLut)>> { static constexpr int value = Op::kLut; };

template <class Op, class P, int NIN>
__device__ __forceinline__ uint32_t apply_op(const uint4 (&v)[NIN], uint32_t c, int64_t i, const P &p,
                                             const float *lut, Tabs tab) {
  if constexpr (LutOf<Op>::value > 0) return Op::apply(v, c, i, p, lut);
  else if constexpr (Tab16Of<Op>::value || CtabOf<Op>::value) return Op::apply(v, c, i, p, tab);
  else return Op::apply(v, c, i, p);
}

#ifdef LMBP_TRACE
// Diagnostic build only (tools/trace_ew.py): one record per running CTA --
// smid, entry time, first tile's data arrival, last tile done, tiles -- in
// globaltimer nanoseconds.  Each translation unit has its own buffer.
static __device__ unsigned long long lmbp_trace_buf[8192 * 5];
static __device__ unsigned int lmbp_trace_n;
static __device__ unsigned long long lmbp_trace_units[65536 * 2];  // (unit claimed via CLC, time)
static __device__ unsigned int lmbp_trace_un;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

// One 16-bit table entry from shared memory (tab = shared-window address).
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
  uint32_t r;
  asm volatile("ld.shared.u16 %0, [%1];" : "=r"(r) : "r"(addr));
  return r;
}
// Two packed 16-bit inputs -> two packed 16-bit table outputs.
// The halves are extracted with PRMT so each address is PRMT + LEA (2 issue
// slots; written as shifts and masks ptxas emits IADD + LOP3 + IADD).
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
  uint32_t r;
  asm volatile("ld.shared.u8 %0, [%1];" : "=r"(r) : "r"(addr));
  return r;
}
__device__ __forceinline__ uint32_t tab16_pair(uint32_t tab, uint32_t w) {
  const uint32_t lo = lds_u16(tab + 2u * __byte_perm(w, 0u, 0x4410));
  const uint32_t hi = lds_u16(tab + 2u * __byte_perm(w, 0u, 0x4432));
  return __byte_perm(lo, hi, 0x5410);
}

template <class Op>
__global__ void __launch_bounds__(EwShape<Op>::kThreads, MinBlocksOf<Op>::value) ew_tma(const typename ParamsOf<Op>::type p) {
  extern __shared__ __align__(128) uint8_t smem_all[];
  using Sh = EwShape<Op>;
  constexpr int W = Op::W, U = Op::U, S = Op::S, NIN = Op::kIn, TILE = Sh::kTile;
  constexpr size_t kYTab = Tab16Of<Op>::value ? kTab16Bytes : 0;
  const Tabs tab{smem_u32(smem_all), smem_u32(smem_all + kYTab)};  // [y table][code table]
  uint8_t *smem = smem_all + Sh::kTabBytes;                 // stages
  uint8_t *cstage = smem + (size_t)S * Sh::kStageBytes;  // codes staging, one slice per warp
  uint64_t *full = reinterpret_cast<uint64_t *>(cstage + Sh::kCodeStage);
  uint64_t *empty = full + S;
  uint64_t *clc_bar = empty + S;
  uint64_t *tab_bar = clc_bar + 1;
  int64_t *slot = reinterpret_cast<int64_t *>(clc_bar + 2);   // tile index held by each stage
  uint4 *clc_resp = reinterpret_cast<uint4 *>(reinterpret_cast<uint8_t *>(slot) + Sh::kSlotBytes);  // 16 B aligned
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef LMBP_TRACE
  const unsigned long long tr_entry = gtimer();
  unsigned long long tr_first = 0;
  unsigned int tr_tiles = 0;
#endif
  const int64_t ntiles = p.nvec / TILE;
  const int64_t nitems = ntiles + 1;                           // + the leftover pseudo-tile

  constexpr int kLut = LutOf<Op>::value;
  const float *lut = nullptr;
  if constexpr (kLut > 0) {
    __shared__ float lut_s[kLut];
    if (threadIdx.x < kLut) lut_s[threadIdx.x] = Op::lut_entry(p, threadIdx.x);
    lut = lut_s;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], W);
    }
    mbar_init(clc_bar, 1);
    mbar_init(tab_bar, 1);
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == W) {  // producer
    if (lane == 0) {
      if constexpr (Tab16Of<Op>::value) {
        mbar_arrive_expect_tx(tab_bar, kTab16Bytes);
        const uint8_t *src = reinterpret_cast<const uint8_t *>(Op::tab16());
#pragma unroll
        for (int q = 0; q < 4; ++q)
          bulk_g2s(smem_all + q * (kTab16Bytes / 4), src + q * (kTab16Bytes / 4), kTab16Bytes / 4, tab_bar);
      }
      // The table is module data; everything below reads inputs (PDL: wait
      // for the previous grid here, common.cuh).
      pdl_wait();
      pdl_trigger();
      int k = 0;
      int64_t unit = blockIdx.x;
      uint32_t clc_phase = 0;
      bool more = true;
      while (more) {
        // request the next unit now; the answer arrives while this unit streams
        mbar_arrive_expect_tx(clc_bar, 16);
        clc_try_cancel(clc_resp, clc_bar);
        const int64_t t_end = min(nitems, (unit + 1) * LMBP_EW_UNIT);
        for (int64_t t = unit * LMBP_EW_UNIT; t < t_end; ++t, ++k) {
          const int s = k % S;
          mbar_wait(&empty[s], ((uint32_t)(k / S) & 1u) ^ 1u);
          slot[s] = t;
          if (t == ntiles) {             // leftover pseudo-tile: nothing to load
            mbar_arrive(&full[s]);
            continue;
          }
          mbar_arrive_expect_tx(&full[s], (uint32_t)Sh::kStageBytes);
          uint8_t *st = smem + (size_t)s * Sh::kStageBytes;
#pragma unroll
          for (int m = 0; m < NIN; ++m) bulk_g2s(st + (size_t)m * TILE * 16, p.in[m] + t * TILE, TILE * 16, &full[s]);
          if constexpr (Op::kCodeIn > 0)
            bulk_g2s(st + (size_t)NIN * TILE * 16, p.codes_in + t * TILE * Op::kCodeIn, TILE * Op::kCodeIn,
                     &full[s]);
        }
        mbar_wait(clc_bar, clc_phase);
        clc_phase ^= 1u;
        const int next = clc_query(clc_resp);
#ifdef LMBP_TRACE
        if (next >= 0) {
          const unsigned int q = atomicAdd(&lmbp_trace_un, 1u);
          if (q < 65536) {
            lmbp_trace_units[2 * q] = (unsigned long long)next;
            lmbp_trace_units[2 * q + 1] = gtimer();
          }
        }
#endif
        more = next >= 0;
        unit = next;
      }
      const int s = k % S;                 // end of stream
      mbar_wait(&empty[s], ((uint32_t)(k / S) & 1u) ^ 1u);
      slot[s] = -1;
      mbar_arrive(&full[s]);
    }
    return;
  }

  if constexpr (CtabOf<Op>::value) {
    Op::fill_ctab(smem_all + kYTab, p, threadIdx.x, W * 32);
    asm volatile("bar.sync 1, %0;" ::"r"(W * 32) : "memory");  // consumers only
  }
  if constexpr (Tab16Of<Op>::value) mbar_wait(tab_bar, 0);
  pdl_wait();  // consumers store outputs (and the leftover path loads inputs) only after it
  for (int k = 0;; ++k) {
    const int s = k % S;
    mbar_wait(&full[s], (uint32_t)(k / S) & 1u);
    const int64_t t = slot[s];
#ifdef LMBP_TRACE
    if (k == 0) tr_first = gtimer();
    ++tr_tiles;
#endif
    if (t < 0) break;
    if (t == ntiles) {
      // Leftover vectors (< one tile) with direct loads, then the ragged tail.
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      for (int64_t i = ntiles * TILE + threadIdx.x; i < p.nvec; i += W * 32) {
        uint4 v[NIN];
#pragma unroll
        for (int m = 0; m < NIN; ++m) v[m] = ld_stream(p.in[m] + i);
        const uint32_t co = apply_op<Op>(v, code_word<Op::kCodeIn>(p.codes_in, i), i, p, lut, tab);
        put_code<Op::kCodeOut>(p.codes_out, i, co);
      }
      if (threadIdx.x == 0) {
        if constexpr (Tab16Of<Op>::value || CtabOf<Op>::value) Op::tail(p, tab);
        else Op::tail(p);
      }
      continue;
    }
    const uint8_t *st = smem + (size_t)s * Sh::kStageBytes;
    // Warp w owns the contiguous vectors [w 32 U, (w + 1) 32 U) of the tile;
    // each warp instruction still touches 512 contiguous bytes.
    uint4 v[U][NIN];
    uint32_t c[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const int vi = warp * (32 * U) + j * 32 + lane;
#pragma unroll
      for (int m = 0; m < NIN; ++m) v[j][m] = lds128(st + ((size_t)m * TILE + vi) * 16);
      c[j] = code_word<Op::kCodeIn>(st + (size_t)NIN * TILE * 16, vi);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // the stage may be refilled while we compute
    const int64_t wbase = t * TILE + warp * (32 * U);
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const uint32_t co = apply_op<Op>(v[j], c[j], wbase + j * 32 + lane, p, lut, tab);
      if constexpr (Op::kCodeOut > 0) put_code<Op::kCodeOut>(cstage + warp * Sh::kWarpCodeBytes, j * 32 + lane, co);
    }
    if constexpr (Op::kCodeOut > 0) {
      // The warp's codes are one contiguous run of 32 U words: write them as
      // full 16-byte vectors (whole 128-byte lines for 16-bit types) instead
      // of 2-byte stores from every lane.
      __syncwarp();
      constexpr int kChunks = (int)(Sh::kWarpCodeBytes / 16);
      if (lane < kChunks) {
        const uint4 w = lds128(cstage + warp * Sh::kWarpCodeBytes + lane * 16);
        st_stream(reinterpret_cast<uint4 *>(p.codes_out + wbase * Op::kCodeOut) + lane, w);
      }
      __syncwarp();
    }
  }
#ifdef LMBP_TRACE
  if (threadIdx.x == 0) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    const unsigned int r = atomicAdd(&lmbp_trace_n, 1u);
    if (r < 8192) {
      unsigned long long *b = lmbp_trace_buf + 5 * r;
      b[0] = smid;
      b[1] = tr_entry;
      b[2] = tr_first;
      b[3] = gtimer();
      b[4] = tr_tiles - 1;
    }
  }
#endif
}

// Launch one CTA per work unit; resident CTAs steal the rest through CLC.
template <class Op>
cudaError_t launch_ew(const typename ParamsOf<Op>::type &p_in, cudaStream_t stream) {
  using Sh = EwShape<Op>;
  auto kern = ew_tma<Op>;
  static std::atomic<unsigned long long> smem_set{0};
  const cudaError_t e = ensure_dyn_smem(kern, Sh::kSmem, smem_set);
  if (e != cudaSuccess) return e;
  typename ParamsOf<Op>::type p = p_in;
  const int64_t items = p.nvec / Sh::kTile + 1;
  const int64_t units = (items + LMBP_EW_UNIT - 1) / LMBP_EW_UNIT;
  if (units > 0x7fffffff) return cudaErrorInvalidValue;
  const int grid = (int)units;  // CTAs beyond the resident ones are taken over via CLC
  launch_k(kern, grid, Sh::kThreads, Sh::kSmem, stream, p);
  return cudaGetLastError();
}

}  // namespace lmbp
