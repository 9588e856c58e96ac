// mas_fwd4.cu -- K1: the forward DP of the maximum-path call, four text rows
// per lane (128 rows per warp).
//
// Restates the parallel engine's relax_column (src/parallel.cpp:25-31) and
// the reference engine's forward_reference (src/reference.cpp:9-36) with one
// direction bit per cell, bit(i, c) = Q[i-1][c] > Q[i][c] (strict, as
// backtrack.hpp:26):
//   * lane k of warp g owns rows 128 g + 4k .. 128 g + 4k + 3.  Per column
//     only the first of the four needs the row above from another lane (one
//     SHFL + one FSEL per four cells), and the four rows are four
//     independent FMNMX/FADD chains;
//   * q is staged per warp in 32-column stages by ONE TMA box
//     {32 columns, 32 lane groups, 4 row residues} of a 3-D view of the
//     input (rows split by i mod 4), 128-byte swizzle: every LDS.128 of a
//     residue tile is conflict-free;
//   * direction bits: FSET (0.0 / 1.0) + FFMA into a float accumulator per
//     row and 16-column half-word (no predicates, see bits4); four rows x
//     one word per 32-column stage, stored as one 16-byte STG per lane (L2
//     evict_last) -- or into shared memory for the one-launch tail (OUT 2);
//   * the compute warps wait and probe with warp-uniform votes, so a warp
//     never enters a stage's shuffles partly diverged;
//   * boundary row between warps: 32-column FIFO hand-offs (st.async into
//     the consumer's shared memory, DSMEM across the CTAs of a cluster) with
//     look-ahead mbarrier probes;
//   * NonFinite (types.cpp:107-115) folded as max.NaN over |q| (one
//     3-input FMNMX per two values); the output's zero fill rides along as
//     linear bulk stores of a zero tile.
// Variants: SRC 1 computes q in the CTA from the Gaussian prior on the
// tensor cores (K1g); OUT 1 writes the score table back (K1s); OUT 2 walks
// small items in the same launch (K1t).  DESIGN.md 3.
//
// (DESIGN.md 3 quotes per-warp clock64 breakdowns and ablations measured with
// instrumented builds of earlier revisions; the product source carries none.)
#include <algorithm>
#include <cstdio>
#include <mutex>

#include "mas_kernels.h"
#include "mas_ptx.cuh"
#include "mas_umma.cuh"

namespace mas {

namespace {

// R = text rows per lane (4): a warp owns 32 R rows; a stage is one
// [R residues][32 groups][32 cols] fp32 box (R * 4 KiB).
constexpr int kCols4 = 32;  // columns per TMA box / direction word ("chunk")
constexpr int kSC = 32;     // columns per stage (32 or 64)
constexpr int kChunks = kSC / kCols4;   // chunks (direction words per row) per stage
// The output's fused zero fill: linear bulk stores of a {32 R rows x kZCols}
// zero tile's bytes (LinearZero below).
constexpr int kZCols = kZeroCols;
constexpr int kBandPub = 4;  // quads per band-progress publication
__host__ __device__ constexpr int rows_of(int R) { return 32 * R; }
__host__ __device__ constexpr int chunk_bytes(int R) { return rows_of(R) * kCols4 * 4; }
__host__ __device__ constexpr int stage_bytes(int R) { return chunk_bytes(R) * kChunks; }
constexpr int kQuad = 32;           // columns per FIFO hand-off (16 or 32)
constexpr int kSlot4 = kQuad * 4;           // FIFO slot bytes
constexpr int kQuadsPerStage = kSC / kQuad;
constexpr int kFifoIt4 = kFifoSlots / kQuadsPerStage;  // FIFO depth in stages

struct Smem4 {
  uint32_t ring, bars, ebars, full, empty, sink, fifo, zero, ticket, tbl, total;
  // Gaussian source (SRC 1): B operand stages, their barriers, TMEM slot
  uint32_t zst, zbars, tslot;
};

// Gaussian source: at most this many B stages / TMEM accumulator buffers in
// flight (the launch picks a.gstages / a.gacc within smem and TMEM).
constexpr int kGStages = 4;
constexpr int kGAcc = 4;

__host__ __device__ inline Smem4 smem4_layout(int R, int W, int N, int Kp = 0, int gstages = 0,
                                              int gN = 0, int tail_bytes = 0) {
  Smem4 L;
  L.ring = 0;
  L.bars = static_cast<uint32_t>(W * N * stage_bytes(R));
  L.ebars = L.bars + static_cast<uint32_t>(W * N * 8);
  L.full = L.ebars + static_cast<uint32_t>(W * N * 8);
  // W + 1 FIFOs: index W is the band drain's staging FIFO (the band's last
  // warp hands its bottom row to the producer warp, which publishes it)
  L.empty = L.full + static_cast<uint32_t>((W + 1) * kFifoSlots * 8);
  // one extra "empty" set and sink (index W): the band feeder's, when the
  // first warp of a band gets its row above from global memory
  L.sink = L.empty + static_cast<uint32_t>((W + 1) * kFifoIt4 * 8);
  L.fifo = (L.sink + static_cast<uint32_t>((W + 1) * 16) + 127u) & ~127u;
  L.zero = L.fifo + static_cast<uint32_t>((W + 1) * kFifoSlots * kSlot4);
  L.ticket = L.zero + static_cast<uint32_t>(rows_of(R) * kZCols);  // after the uint8 zero tile
  // one-launch tail (OUT 2): the item's direction words, tail_bytes (see
  // tail_bytes() below), 16-byte aligned
  L.tbl = (L.ticket + 16u + 15u) & ~15u;
  L.total = L.tbl + static_cast<uint32_t>(tail_bytes);
  L.zst = L.zbars = L.tslot = L.total;
  if (Kp > 0) {
    // zfull[kGStages] zfree[kGStages] dfull[kGAcc] dempty[kGAcc] aready, then the slot
    L.zst = (L.total + 1023u) & ~1023u;
    L.zbars = L.zst + static_cast<uint32_t>(gstages * (Kp / umma::kAtomK) * gN * 128);
    L.tslot = (L.zbars + static_cast<uint32_t>((2 * kGStages + 2 * kGAcc + 1) * 8) + 15u) & ~15u;
    L.total = L.tslot + 16u;
  }
  return L;
}

template <int R>
struct Lane4 {
  float o[R];   // Q of the lane's rows at the previous column
  float acc[R / 2];  // max.NaN of |q| (independent chains, one per row pair):
                     // NaN / +inf iff a non-finite q was seen
  float vlast;  // producer's bottom row at the previous column
};

struct Fifo4 {
  uint32_t full, empty;            // my FIFO's "full" barriers, my "empty" barriers
  uint32_t next_fifo, next_full;   // consumer's slots and "full" barriers
  uint32_t prev_empty, prev_sink;  // producer's "empty" barriers and release sink
  const uint8_t* buf;              // my FIFO's slots
  bool has_in, has_out;
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void mbar_arrive_local(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// The four direction bits of one column.  Each bit is a 0.0 / 1.0 compare
// (FSET, ALU pipe) folded into a float accumulator with one FFMA (FMA
// pipe): wf[r] += (row above beats row r) * 2^BIT.  The accumulators start
// at 2^23, so the 16 bits of a quad sit in the low mantissa bits
// (__float_as_uint(wf) & 0xffff).  No predicate registers are involved: a
// predicated form (FSETP -> @P IMAD) lets ptxas funnel the four compares
// through a single predicate whenever other predicates are live, which
// serialises the column behind FSETP->IMAD latencies.
template <int BIT>
__device__ __forceinline__ void bit1(float& wf, float a, float b) {
  constexpr float kBit = static_cast<float>(1u << BIT);
  asm("{\n\t.reg .f32 t;\n\tset.gt.f32.f32 t, %1, %2;\n\tfma.rn.f32 %0, t, %3, %0;\n\t}"
      : "+f"(wf)
      : "f"(a), "f"(b), "f"(kBit));
}
template <int R, int BIT>
__device__ __forceinline__ void bits4(float (&wf)[R], float up, const float (&o)[R]) {
  // the bits that do not need `up` (the shuffled row above) first
#pragma unroll
  for (int r = 1; r < R; ++r) bit1<BIT>(wf[r], o[r - 1], o[r]);
  bit1<BIT>(wf[0], up, o[0]);
}
constexpr float kBitsBase = 8388608.0f;  // 2^23

// Four columns (one LDS.128 per row residue, one of the FIFO slot) of the
// DP for one warp.  U0 = index of the first column within the stage.
// std::max(a, b) as the reference evaluates it: (a < b) ? b : a (the first
// argument on ties, signed zeros and NaNs included) -- the score export's
// arithmetic, where the table itself is the output.
__device__ __forceinline__ float ref_max(float a, float b) { return a < b ? b : a; }

// OUT 1 (score export): the same columns computed with ref_max and written
// back over q in the stage (rows below the item's text length keep q), no
// direction bits, no NonFinite fold.
template <int R, int MODE, bool GENERIC, int U0, int OUT>
__device__ __forceinline__ bool fwd4_group(const uint8_t* __restrict__ tile, uint32_t coff,
                                          const float4* __restrict__ slot, float (&ex)[kQuad],
                                          Lane4<R>& L, float (&wf)[R], bool is31, int srclane,
                                          int c_base, int nvalid, int row0, float mnv,
                                          bool row0_is_zero, uint32_t live) {
  if (GENERIC && U0 >= nvalid) return false;
  float4 qv[R];
#pragma unroll
  for (int r = 0; r < R; ++r)
    qv[r] = *reinterpret_cast<const float4*>(tile + r * 4096 + coff);
  const float4 vv = slot[(U0 % kQuad) / 4];  // producer's bottom row
  const float bnds[4] = {L.vlast, vv.x, vv.y, vv.z};
  float4 res[R];
  if constexpr (OUT) {
#pragma unroll
    for (int r = 0; r < R; ++r) res[r] = qv[r];
  }
  auto put_back = [&]() {
    if constexpr (OUT) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (live & (1u << r))
          *reinterpret_cast<float4*>(const_cast<uint8_t*>(tile) + r * 4096 + coff) = res[r];
    }
  };
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if (GENERIC && U0 + e >= nvalid) {
      put_back();
      return false;
    }
    float q[R];
#pragma unroll
    for (int r = 0; r < R; ++r) q[r] = e == 0 ? qv[r].x : e == 1 ? qv[r].y : e == 2 ? qv[r].z : qv[r].w;
    const float send = is31 ? bnds[e] : L.o[R - 1];
    float up = __shfl_sync(0xffffffffu, send, srclane);
    float n[R];
    if constexpr (OUT) {
      // reference.cpp:20-24: row 0 is a running sum (prev + q, not a max)
      if (MODE == 1 && row0_is_zero) up = L.o[0];
      n[0] = q[0] + ref_max(up, L.o[0]);
#pragma unroll
      for (int r = 1; r < R; ++r) n[r] = q[r] + ref_max(L.o[r - 1], L.o[r]);
    } else {
      switch ((U0 + e) % 16) {  // compile-time bit 15 - column-in-half-word
#define MAS_B4(U)                   \
  case U:                           \
    bits4<R, 15 - U>(wf, up, L.o);  \
    break;
        MAS_B4(0) MAS_B4(1) MAS_B4(2) MAS_B4(3) MAS_B4(4) MAS_B4(5) MAS_B4(6) MAS_B4(7)
        MAS_B4(8) MAS_B4(9) MAS_B4(10) MAS_B4(11) MAS_B4(12) MAS_B4(13) MAS_B4(14) MAS_B4(15)
#undef MAS_B4
      }
      n[0] = q[0] + fmaxf(up, L.o[0]);
#pragma unroll
      for (int r = 1; r < R; ++r) n[r] = q[r] + fmaxf(L.o[r - 1], L.o[r]);
    }
    if (GENERIC) {
      const int c = c_base + U0 + e;
      if (MODE == 1) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (c < row0 + r) n[r] = mnv;
      }
      if (c == 0) {  // first column: parallel.cpp:73-75 / reference.cpp:16-24
        // (the reference engine's running sum starts at 0.f + q[0][0])
        n[0] = row0_is_zero ? (OUT && MODE == 1 ? 0.f + q[0] : q[0]) : mnv;
#pragma unroll
        for (int r = 1; r < R; ++r) n[r] = mnv;
      }
    }
    if constexpr (!OUT) {
#pragma unroll
      for (int r = 0; r + 1 < R; r += 2) fold_abs_max_nan(L.acc[r / 2], q[r], q[r + 1]);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (e == 0) res[r].x = n[r];
        if (e == 1) res[r].y = n[r];
        if (e == 2) res[r].z = n[r];
        if (e == 3) res[r].w = n[r];
      }
    }
    ex[(U0 % kQuad) + e] = n[R - 1];
#pragma unroll
    for (int r = 0; r < R; ++r) L.o[r] = n[r];
  }
  put_back();
  L.vlast = vv.w;
  return true;
}

// One FIFO quad (32 columns) with the hand-off around it.
// Look-ahead probes of the next stage's load and of the next iteration's
// FIFO "empty" slot, made inside the first quad's straight-line block so
// their results are consumed only after it (see fwd4_quad).
template <bool V>
struct BoolTag {
  static constexpr bool value = V;
};

struct Probes {
  uint32_t stage_bar, stage_par;  // next stage's "loaded" barrier
  uint32_t empty_bar, empty_par;  // next iteration's consumer-slot barrier
  bool arm_empty;                 // arm empty_bar (expect_tx, lane 31) first
  bool stage_ok, empty_ok;        // results
};

template <int R, int MODE, bool GENERIC, int K, int OUT>
__device__ __forceinline__ bool fwd4_quad(const uint8_t* stage, const uint32_t (&coff)[8],
                                         const Fifo4& F, float (&ex)[kQuad], Lane4<R>& L,
                                         uint32_t (&w)[kChunks][R], bool& ready, bool more, bool is31,
                                         int lane, int srclane, int q, int c_base, int nvalid,
                                         int row0, float mnv, bool row0_is_zero,
                                         Probes& P, uint32_t live) {
  if (GENERIC && K * kQuad >= nvalid) return false;
  const int fs = q & (kFifoSlots - 1);
  mbar_wait_all_unless(!F.has_in || ready, F.full + 8u * fs,
                       static_cast<uint32_t>(q / kFifoSlots) & 1u);
  const bool next = K + 1 < kQuadsPerStage ? (!GENERIC || (K + 1) * kQuad < nvalid) : more;
  const int q1 = q + 1;
  const uint32_t bar1 = F.full + 8u * (q1 & (kFifoSlots - 1));
  mbar_arrive_expect_tx_if(lane == 0 && next && F.has_in, bar1, kSlot4);
  const bool probe = mbar_test_wait_all(bar1, static_cast<uint32_t>(q1 / kFifoSlots) & 1u);
  bool p_stage = false, p_empty = false;
  if (K == 0) {
    mbar_arrive_expect_tx_if(P.arm_empty && is31, P.empty_bar, 4u);
    p_stage = mbar_test_wait_all(P.stage_bar, P.stage_par);
    p_empty = mbar_test_wait_all(P.empty_bar, P.empty_par);
  }
  const float4* slot = reinterpret_cast<const float4*>(F.buf + fs * kSlot4);
  bool ok = true;
  float wf[R];
  // Groups of four columns; the bits of each 16-column half-word collect in
  // wf (columns 0..15 of the stage -> word bits 31..16, 16..31 -> 15..0).
#define MAS_G4(A)                                                                               \
  if constexpr (4 * (A) < kQuad) {                                                              \
    constexpr int U0 = K * kQuad + 4 * (A);                                                     \
    if constexpr (U0 % 16 == 0) {                                                               \
      _Pragma("unroll") for (int r = 0; r < R; ++r) wf[r] = kBitsBase;                          \
    }                                                                                           \
    if (ok)                                                                                     \
      ok = fwd4_group<R, MODE, GENERIC, U0, OUT>(stage + (U0 / kCols4) * chunk_bytes(R),       \
                                                 coff[(U0 / 4) & 7], slot, ex, L, wf, is31,     \
                                                 srclane, c_base, nvalid, row0, mnv,            \
                                                 row0_is_zero, live);                           \
    if constexpr (U0 % 16 == 12 && !OUT) {                                                      \
      _Pragma("unroll") for (int r = 0; r < R; ++r) {                                           \
        const uint32_t v = __float_as_uint(wf[r]) & 0xffffu;                                    \
        w[U0 / kCols4][r] |= U0 % kCols4 < 16 ? v << 16 : v;                                    \
      }                                                                                         \
    }                                                                                           \
  }
  MAS_G4(0) MAS_G4(1) MAS_G4(2) MAS_G4(3) MAS_G4(4) MAS_G4(5) MAS_G4(6) MAS_G4(7)
  MAS_G4(8) MAS_G4(9) MAS_G4(10) MAS_G4(11) MAS_G4(12) MAS_G4(13) MAS_G4(14) MAS_G4(15)
#undef MAS_G4
  ready = probe;
  if (K == 0) {
    P.stage_ok = p_stage;
    P.empty_ok = p_empty;
  }
  if (F.has_out && is31) {
    const uint32_t dst = F.next_fifo + static_cast<uint32_t>(fs * kSlot4);
    const uint32_t fbar = F.next_full + 8u * fs;
#pragma unroll
    for (int q4 = 0; q4 < kQuad / 4; ++q4)
      st_async_v4(dst + 16u * q4, ex[4 * q4], ex[4 * q4 + 1], ex[4 * q4 + 2], ex[4 * q4 + 3], fbar);
  }
  return ok;
}

template <int R, int MODE, bool GENERIC, int OUT>
__device__ __forceinline__ void fwd4_stage(const uint8_t* stage, const uint32_t (&coff)[8],
                                          const Fifo4& F, float (&ex)[kQuad], Lane4<R>& L,
                                          uint32_t (&w)[kChunks][R], bool& ready, bool more, bool is31,
                                          int lane, int srclane, int q0, int c_base, int nvalid,
                                          int row0, float mnv, bool row0_is_zero,
                                          Probes& P, uint32_t live) {
  if (!fwd4_quad<R, MODE, GENERIC, 0, OUT>(stage, coff, F, ex, L, w, ready, more, is31, lane,
                                           srclane, q0, c_base, nvalid, row0, mnv, row0_is_zero,
                                           P, live))
    return;
  if constexpr (kQuadsPerStage > 1)
    fwd4_quad<R, MODE, GENERIC, 1, OUT>(stage, coff, F, ex, L, w, ready, more, is31, lane, srclane,
                                        q0 + 1, c_base, nvalid, row0, mnv, row0_is_zero, P, live);
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

// The output's fused zero fill as linear bulk stores: a warp's rows
// [i0, i0 + rows) of item b are one contiguous range of the
// [B][T_cap][S_cap] output, written in zero-tile-sized (8 KB) chunks spread
// evenly over the item's nit stages.  Rows past T_cap belong to the next
// item and are never written.  (The same DRAM time as {256 x 128} TMA boxes
// of 256-byte row segments, r13, and no spill into the next item.)
struct LinearZero {
  uint8_t* dst = nullptr;
  int64_t len = 0;
  int nchunks = 0, next = 0, nit = 1;
  static constexpr int kBytes = 128 * kZCols;  // the zero tile
  __device__ LinearZero(const FwdArgs& a, int b, int i0, int rows_max, int nit_) : nit(nit_) {
    if (!a.zero_fill || !a.out) return;
    const int rows = min(rows_max, a.T_cap - i0);
    if (rows <= 0) return;
    dst = a.out + (static_cast<int64_t>(b) * a.T_cap + i0) * a.S_cap;
    len = static_cast<int64_t>(rows) * a.S_cap;
    nchunks = static_cast<int>((len + kBytes - 1) / kBytes);
  }
  // chunks due once stage m is issued (all of them by the last stage)
  __device__ bool due(int m) const {
    return next < nchunks && static_cast<int64_t>(next) * nit < static_cast<int64_t>(m + 1) * nchunks;
  }
  __device__ void issue_upto(int m, uint32_t zero_tile) {
    while (due(m)) {
      const int64_t off = static_cast<int64_t>(next) * kBytes;
      const uint32_t bytes = static_cast<uint32_t>(len - off < kBytes ? len - off : kBytes);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off),
                   "r"(zero_tile), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      ++next;
    }
  }
};

// ---- one-launch tail (OUT 2, small batches) --------------------------------
// Items that fit one single-CTA cluster (K = 1, one band) keep their
// direction words in shared memory instead of global memory: word k of row i
// at tbl[kTailGuard + k * rows + i] (rows = the CTA's W * 32R rows), then the
// CTA walks and expands its own item after the forward pass, so the batch is
// ONE launch (no backtrack kernel, no global round trip of the words).
// Layout of the region: a guard of kTailGuard words (the walk's look-ahead
// reads up to 4 rows below row 0 of word 0), the table, then the per-word
// walk records rec_y[M], rec_ex[M].
constexpr int kTailGuard = 16;
__host__ __device__ inline int tail_bytes(int M, int rows) {
  return (kTailGuard + M * rows + 2 * M) * 4;
}

// The backtrack (backtrack.hpp:21-32) over the shared-memory table, one
// thread: the K2 walker's row-to-row steps (mas_bt.cu) without windows --
// per 64-column word pair, exits are the lowest set bits of the bit-reversed
// words, four branch-free steps per block; records each word's entry row and
// exit mask.
__device__ __noinline__ void tail_walk(const uint32_t* tbl, int rows, int t, int s, int* rec_y,
                                       uint32_t* rec_ex) {
  int y = t - 1;
  int ml = (s - 1) >> 5;
  // positions of the item's last word up to s - 1 (column s - 2)
  uint32_t lim = 0xffffffffu << (31 - ((s - 1) & 31));
  auto ld64 = [&](int k, int row, bool pair) -> uint64_t {
    const uint64_t lo = tbl[k * rows + row];
    return pair ? lo | (static_cast<uint64_t>(tbl[(k - 1) * rows + row]) << 32) : lo;
  };
  while (ml >= 0) {
    if (y <= 0) {  // the walk reached row 0: the rest stays there
      rec_y[ml] = 0;
      rec_ex[ml] = 0u;
      --ml;
      continue;
    }
    const bool pair = ml > 0;
    rec_y[ml] = y;
    uint64_t x = ld64(ml, y, pair) & (static_cast<uint64_t>(0xffffffffu) << 32 | lim);
    lim = 0xffffffffu;
    uint64_t exw = 0;
    int yy = y;
    while (true) {
#pragma unroll
      for (int k = 1; k <= 4; ++k) {
        const uint64_t d = x - 1u;
        exw |= x & ~d;
        x = ld64(ml, yy - k, pair) & ~(x ^ d);
      }
      yy -= 4;
      if ((x & 0x7fffffffffffffffull) == 0u) break;
    }
    exw |= x;  // a pending exit at the pair's position 0
    const int ex_lo = __popc(static_cast<uint32_t>(exw));
    const int ex = ex_lo + __popc(static_cast<uint32_t>(exw >> 32));
    rec_ex[ml] = static_cast<uint32_t>(exw);
    if (pair) {
      rec_ex[ml - 1] = static_cast<uint32_t>(exw >> 32);
      rec_y[ml - 1] = y - ex_lo;
    }
    y -= ex;
    ml -= pair ? 2 : 1;
  }
}

// SRC 0: q streamed from HBM by TMA.  SRC 1: q computed in the CTA from the
// Gaussian prior (mas_gauss.cu operands): tmq is then the map of the B
// operand; the producer warp's lane 0 loads B stages, warp W+1 issues the
// tcgen05 MMAs (A resident in TMEM; the whole warp waits, one lane issues),
// and four epilogue warps (warps W+2..W+5, one per TMEM sub-partition) add
// the row bias and write each 32-column tile into the compute warps' ring in
// the layout TMA would have used.  The compute warps run unchanged.
//
// OUT 1 (SRC 0 only): score export, parallel::forward_parallel /
// reference::forward_reference (parallel.cpp:95-108, reference.cpp:9-36):
// the compute warps write each stage's Q values back over q in the ring and
// the producer lane TMA-stores the stage to tm_out (q's own storage, a 4-D
// {columns, row groups, residues, items} map, so stores clip at the item's
// last row) before refilling the slot.  No direction words, flags or zero
// fill.
//
// OUT 2 (SRC 0 only): the one-launch tail for items of one single-CTA
// cluster: direction words to shared memory, then the CTA walks and expands
// its own item (tail_walk), no backtrack kernel.
template <int R, int MODE, int SRC, int OUT>
__global__ void __launch_bounds__(SRC ? 12 * 32 : (kMaxWarpsPerCta + 1) * 32, 1)
    mas_fwd4_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tm_out,
                    const FwdArgs a) {
  constexpr int kExport = OUT == 1 ? 1 : 0;  // score export
  constexpr bool kTail = OUT == 2;           // one-launch tail
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_addr(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* const sbase = smem_raw + (base - raw);
  const int W = a.W;  // compute warps; warp W is the CTA's TMA producer
  const int N = a.N;
  constexpr int kRows4 = rows_of(R);
  constexpr int kStage4 = stage_bytes(R);
  const Smem4 SL = smem4_layout(R, W, N, SRC ? a.Kp : 0, SRC ? a.gstages : 0, SRC ? a.gN : 0,
                                kTail ? tail_bytes(a.M, W * rows_of(R)) : 0);
  const int NB = a.gstages, NA = a.gacc;  // Gaussian source pipeline depths
  const int GN = a.gN;                    // frames per MMA (64 or 128)
  const int kGS = GN / umma::kStageN;     // K1 stages per MMA group
  const uint32_t atom_bytes = static_cast<uint32_t>(GN * 128);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int crank = static_cast<int>(cluster_ctarank());
  // (item, band) of this cluster: the cluster index, or with bands a ticket
  // drawn by rank 0 in launch order (band-major) and shared over DSMEM.
  int cl = static_cast<int>(blockIdx.x) / a.K;
  if (a.bands > 1) {
    cluster_sync_all();  // every peer CTA has started before its shared memory is written
    if (crank == 0 && threadIdx.x == 0) {
      const int t = atomicAdd(a.ticket, 1);
      for (int r = 0; r < a.K; ++r)
        asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(mapa(base + SL.ticket, r)), "r"(t)
                     : "memory");
    }
    cluster_sync_all();
    cl = *reinterpret_cast<volatile int*>(sbase + SL.ticket);
  }
  const int band_idx = cl / a.nb;
  const int b = a.b0 + cl % a.nb;
  const int t_b = static_cast<int>(a.lengths[2 * b]);
  const int s_b = static_cast<int>(a.lengths[2 * b + 1]);
  const int nit = (s_b + kSC - 1) / kSC;

  const int band = band_idx * a.band_rows;  // first text row of this cluster
  const bool fed = band_idx > 0;              // band's first warp fed from the band above
  // this band's bottom row continues in the band below (drained to global)
  const bool drains = band_idx + 1 < a.bands && band + a.band_rows < t_b && s_b > 0;
  if (warp < W) {
    const int g = crank * W + warp;
    const bool has_in = g > 0 || fed;
    const uint32_t bar0 = base + SL.bars + static_cast<uint32_t>(warp * N * 8);
    const uint32_t ebar0 = base + SL.ebars + static_cast<uint32_t>(warp * N * 8);
    const uint32_t my_full = base + SL.full + static_cast<uint32_t>(warp * kFifoSlots * 8);
    const uint32_t my_empty = base + SL.empty + static_cast<uint32_t>(warp * kFifoIt4 * 8);
    uint8_t* const my_fifo = sbase + SL.fifo + warp * kFifoSlots * kSlot4;
    if (lane == 0) {
      for (int s = 0; s < N; ++s) {
        // stage loaded: the producer's expect_tx + TMA bytes, or the four
        // epilogue warps of the Gaussian source
        mbar_init(bar0 + 8u * s, SRC ? 4u : 1u);
        mbar_init(ebar0 + 8u * s, 1u);  // stage consumed (this warp's lane 0)
      }
      for (int s = 0; s < kFifoSlots; ++s) mbar_init(my_full + 8u * s, 1u);
      for (int s = 0; s < kFifoIt4; ++s) mbar_init(my_empty + 8u * s, 1u);
    }
    if (!has_in) {
      // The first warp of an item has no producer: its FIFO permanently
      // holds the value above row 0 (max_neg_val, or -inf for
      // reference.cpp:20-24).
      for (int k = lane; k < kFifoSlots * kQuad; k += 32)
        reinterpret_cast<float*>(my_fifo)[k] = a.row0_up;
    }
  } else if (warp == W) {
    for (int k = lane; k < kRows4 * kZCols / 16; k += 32)
      reinterpret_cast<uint4*>(sbase + SL.zero)[k] = make_uint4(0u, 0u, 0u, 0u);
    if (lane == 0) {
      for (int s = 0; s < kFifoIt4; ++s)
        mbar_init(base + SL.empty + static_cast<uint32_t>((W * kFifoIt4 + s) * 8), 1u);
      for (int s = 0; s < kFifoSlots; ++s)
        mbar_init(base + SL.full + static_cast<uint32_t>((W * kFifoSlots + s) * 8), 1u);
    }
  }
  uint32_t tmem = 0, tmem_cols = 0;
  if constexpr (SRC == 1) {
    tmem_cols = umma::tmem_cols_pow2(static_cast<uint32_t>(W * a.Kp / 2 + NA * W * GN));
    if (warp == W + 2) {
      if (lane == 0) {
        // zfull / zfree: TMA + commit; dfull: commit; dempty, aready: every
        // epilogue warp (4 per compute warp)
        for (int k = 0; k < 2 * kGStages + 2 * kGAcc + 1; ++k)
          mbar_init(base + SL.zbars + 8u * k,
                    k >= 2 * kGStages + kGAcc ? static_cast<uint32_t>(4 * W) : 1u);
      }
      umma::tmem_alloc(base + SL.tslot, tmem_cols);
    }
    umma::fence_before_sync();
  }
  // Pipelined plans: this launch may run alongside the previous batch's
  // backtrack; the one two batches back read the same direction-word buffer
  // and must have finished with it (one poll in practice).
  if (a.bt_done && threadIdx.x == 0) {
    unsigned v;
    while (true) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bt_done) : "memory");
      if (v >= a.bt_need) break;
      __nanosleep(256);
    }
  }
  // the item's NonFinite flag starts at 0 (set by atomicOr only after the
  // cluster barrier below, and in the bands below after this band's
  // progress releases)
  if (!kExport && band_idx == 0 && crank == 0 && threadIdx.x == 0) a.flags[b] = 0;
  fence_proxy_async_smem();
  fence_mbar_init();
  cluster_sync_all();  // every CTA's FIFO / stage barriers exist before any use
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if constexpr (SRC == 1) {
    umma::fence_after_sync();
    tmem = *reinterpret_cast<volatile uint32_t*>(sbase + SL.tslot);
  }

  if (SRC == 1 && warp == W + 1) {
    // ---- Gaussian source, MMA warp: waits converged, lane 0 issues --------
    const uint32_t zb = base + SL.zbars;
    const uint32_t zfull = zb, zfree = zb + 8u * kGStages;
    const uint32_t dfull = zb + 8u * (2 * kGStages), dempty = dfull + 8u * kGAcc;
    const uint32_t aready = dempty + 8u * kGAcc;
    const uint32_t stage_bytes = static_cast<uint32_t>(a.Kp / umma::kAtomK) * atom_bytes;
    int wl = 0;
    for (int v = 0; v < W; ++v)
      if (s_b > 0 && band + (crank * W + v) * kRows4 < t_b) wl = v + 1;
    if (wl > 0) {
      const uint32_t idesc = umma::idesc_bf16_f32(umma::kM, GN);
      mbar_wait(aready, 0u);
      umma::fence_after_sync();
      const int ngr = (nit + kGS - 1) / kGS;  // MMA groups of kGS stages
      for (int m = 0; m < ngr; ++m) {
        const int zs = m % NB, d = m % NA;
        mbar_wait(zfull + 8u * zs, static_cast<uint32_t>(m / NB) & 1u);
        if (m >= NA) mbar_wait(dempty + 8u * d, (static_cast<uint32_t>(m / NA) & 1u) ^ 1u);
        umma::fence_after_sync();
        __syncwarp();
        if (lane == 0) {
          umma::mma_tiles(tmem + static_cast<uint32_t>(W * a.Kp / 2 + d * W * GN),
                          static_cast<uint32_t>(GN), tmem, static_cast<uint32_t>(a.Kp / 2), wl,
                          base + SL.zst + zs * stage_bytes, a.Kp, idesc, atom_bytes);
          umma::mma_commit(zfree + 8u * zs);
          umma::mma_commit(dfull + 8u * d);
        }
        __syncwarp();
      }
    }
    __syncwarp();
    cluster_sync_all();
    return;
  }

  if (SRC == 1 && warp > W + 1) {
    // ---- Gaussian source, epilogue warp (TMEM sub-partition qd, tile w) ---
    // Warps W+2 .. W+1+4W: tile w = (warp - W - 2) / 4, so each compute
    // warp's tiles are written by its own four warps and the two compute
    // warps' rings fill independently.
    const int qd = warp & 3;
    const int w = (warp - W - 2) >> 2;
    const uint32_t zb = base + SL.zbars;
    const uint32_t dfull = zb + 8u * (2 * kGStages), dempty = dfull + 8u * kGAcc;
    const uint32_t aready = dempty + 8u * kGAcc;
    const uint32_t lane_base = static_cast<uint32_t>(32 * qd) << 16;
    // TMEM lane 32 qd + lane holds tile row 32 qd + 4 (lane & 7) + (lane >> 3):
    // each 8-lane phase of a ring store then covers eight row groups (eight
    // distinct swizzled 16-byte chunks): STS.128 without bank conflicts
    // (the natural order put four residues of one group in a phase: 16
    // wavefronts per store instead of 4, r12 ncu).
    const int grp = 32 * qd + 4 * (lane & 7) + (lane >> 3);  // row within the warp's 128-row tile
    const int row = band + (crank * W + w) * kRows4 + grp;
    const bool live_w = s_b > 0 && band + (crank * W + w) * kRows4 < t_b;
    float bias = 0.f;
    if (live_w) {
      // rows i0w + 32 qd + lane: their A rows into TMEM, their bias into a register
      const uint32_t* src = reinterpret_cast<const uint32_t*>(a.gA) +
                            (static_cast<int64_t>(b) * a.Tp + row) * (a.Kp / 2);
      for (int c = 0; c < a.Kp / 2; c += 8) {
        uint32_t v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = __ldg(src + c + e);
        umma::tmem_st8(tmem + lane_base + static_cast<uint32_t>(w * a.Kp / 2 + c), v);
      }
      bias = __ldg(a.gbias + static_cast<int64_t>(b) * a.Tp + row);
      umma::tmem_wait_st();
    }
    umma::fence_before_sync();
    __syncwarp();
    if (lane == 0) mbar_arrive_local(aready);
    const uint32_t rbase = static_cast<uint32_t>((grp & 3) * 4096 + (grp >> 2) * 128);
    const uint32_t sw = static_cast<uint32_t>((grp >> 2) & 7);
    uint8_t* const ring_w = sbase + SL.ring + w * N * kStage4 + rbase;
    int wl = 0;
    for (int v = 0; v < W; ++v)
      if (s_b > 0 && band + (crank * W + v) * kRows4 < t_b) wl = v + 1;
    const int ngr = wl > 0 ? (nit + kGS - 1) / kGS : 0;
    for (int gi = 0; gi < ngr; ++gi) {
      const int d = gi % NA;
      mbar_wait(dfull + 8u * d, static_cast<uint32_t>(gi / NA) & 1u);
      umma::fence_after_sync();
      // 32-frame chunks: TMEM -> registers; the accumulator is released
      // after the last chunk is read, each chunk written to its ring stage
      for (int h = 0; h < kGS; ++h) {
        const int m = gi * kGS + h;
        float v[32];
        if (live_w) {
          umma::tmem_ld32(tmem + lane_base +
                              static_cast<uint32_t>(W * a.Kp / 2 + (d * W + w) * GN + h * umma::kStageN),
                          v);
          umma::tmem_wait_ld();
        }
        if (h == kGS - 1) {
          umma::fence_before_sync();
          __syncwarp();
          if (lane == 0) mbar_arrive_local(dempty + 8u * d);
        }
        if (!live_w || m >= nit) continue;
        const int st = m % N;
        if (m >= N)  // ring slot st of warp w consumed in iteration m - N
          mbar_wait(base + SL.ebars + static_cast<uint32_t>((w * N + st) * 8),
                         (static_cast<uint32_t>(m / N) & 1u) ^ 1u);
        uint8_t* dst = ring_w + st * kStage4;
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4)
          *reinterpret_cast<float4*>(dst + ((c4 ^ sw) << 4)) =
              make_float4(v[4 * c4] + bias, v[4 * c4 + 1] + bias, v[4 * c4 + 2] + bias,
                          v[4 * c4 + 3] + bias);
        __syncwarp();
        if (lane == 0) mbar_arrive_local(base + SL.bars + static_cast<uint32_t>((w * N + st) * 8));
      }
    }
    umma::fence_before_sync();
    __syncwarp();
    cluster_sync_all();
    if (warp == W + 2) umma::tmem_dealloc(tmem, tmem_cols);
    return;
  }

  if (warp == W) {
    // ---- TMA producer warp: loads every compute warp's stages and issues
    // the output's zero fill, so the compute warps only wait and compute.
    // Lane w serves compute warp w on its own (independent thread
    // scheduling lets each lane block on its warp's "stage consumed"
    // barrier without holding up the others).  Stages further ahead than
    // the shared-memory ring are prefetched into L2 (kL2Ahead4 stages), so
    // a ring refill finds its data in L2 when DRAM latency exceeds the
    // ring's lead.
    const int w = lane;
    const int i0w = band + (crank * W + w) * kRows4;
    if (w == W && fed && crank == 0 && s_b > 0 && band < t_b) {
      // Band feeder: the band's first warp (warp 0 of rank 0) gets the row
      // above the band, written by the previous band's last warp, through
      // its ordinary FIFO: 64-byte bulk copies completing its "full"
      // barriers; slots are released to this lane's "empty" set (index W).
      const size_t link = static_cast<size_t>(b) * (a.bands - 1) + (band_idx - 1);
      const float* src = a.bnd + link * a.bnd_pitch;
      const int* prog = a.progress + link;
      int avail = 0;  // quads the band above has published
      const uint32_t fempty = base + SL.empty + static_cast<uint32_t>(W * kFifoIt4 * 8);
      for (int m = 0; m < nit; ++m) {
        if (m >= kFifoIt4) {
          const uint32_t eb = fempty + 8u * static_cast<uint32_t>(m % kFifoIt4);
          mbar_arrive_expect_tx(eb, 4u);
          mbar_wait(eb, (static_cast<uint32_t>(m / kFifoIt4) & 1u) ^ 1u);
        }
        const int nvalid = s_b - m * kSC < kSC ? s_b - m * kSC : kSC;
        for (int k = 0; k < kQuadsPerStage && k * kQuad < nvalid; ++k) {
          const int qq = kQuadsPerStage * m + k;
          const int fs = qq & (kFifoSlots - 1);
          while (avail <= qq) {
            avail = ld_acquire_gpu(prog);
            if (avail <= qq) __nanosleep(128);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  base + SL.fifo + static_cast<uint32_t>(fs * kSlot4)),
              "l"(src + qq * kQuad), "r"(kSlot4),
              "r"(base + SL.full + static_cast<uint32_t>(fs * 8))
              : "memory");
        }
      }
    }
    if (w == W + 1 && drains && crank == a.K - 1) {
      // Band drain: the band's last warp (warp W-1 of the last rank) sends
      // its bottom row into staging FIFO W like into a consumer's FIFO; this
      // lane publishes each quad to global memory (release) for the band
      // below and releases the slots as that warp's consumer would.
      const size_t link = static_cast<size_t>(b) * (a.bands - 1) + band_idx;
      float* dst = a.bnd + link * a.bnd_pitch;
      int* prog = a.progress + link;
      const uint32_t dfull = base + SL.full + static_cast<uint32_t>(W * kFifoSlots * 8);
      const uint8_t* dfifo = sbase + SL.fifo + W * kFifoSlots * kSlot4;
      const uint32_t lempty =
          mapa(base + SL.empty + static_cast<uint32_t>((W - 1) * kFifoIt4 * 8), crank);
      const uint32_t lsink = mapa(base + SL.sink + static_cast<uint32_t>((W - 1) * 16), crank);
      const int nq = (s_b + kQuad - 1) / kQuad;
      mbar_arrive_expect_tx(dfull, kSlot4);
      for (int q = 0; q < nq; ++q) {
        const int fs = q & (kFifoSlots - 1);
        if (q + 1 < nq)
          mbar_arrive_expect_tx(dfull + 8u * static_cast<uint32_t>((q + 1) & (kFifoSlots - 1)),
                                kSlot4);
        mbar_wait(dfull + 8u * static_cast<uint32_t>(fs), static_cast<uint32_t>(q / kFifoSlots) & 1u);
        const float4* sp = reinterpret_cast<const float4*>(dfifo + fs * kSlot4);
        float4* gp = reinterpret_cast<float4*>(dst + q * kQuad);
#pragma unroll
        for (int q4 = 0; q4 < kQuad / 4; ++q4) gp[q4] = sp[q4];
        // publish every kBandPub quads: a release at GPU scope waits for the
        // stores to be performed (~1 us), longer than a quad takes to compute
        if ((q + 1) % kBandPub == 0 || q + 1 == nq) st_release_gpu(prog, q + 1);
        if ((q + 1) % kQuadsPerStage == 0 || q + 1 == nq) {
          const int m = q / kQuadsPerStage;
          st_async_b32(lsink, static_cast<uint32_t>(m),
                       lempty + 8u * static_cast<uint32_t>(m % kFifoIt4));
        }
      }
    }
    if (SRC == 1 && s_b > 0) {
      const uint32_t zb = base + SL.zbars;
      const uint32_t zfull = zb, zfree = zb + 8u * kGStages;
      const uint32_t stage_bytes = static_cast<uint32_t>(a.Kp / umma::kAtomK) * atom_bytes;
      int wl = 0;
      for (int v = 0; v < W; ++v)
        if (band + (crank * W + v) * kRows4 < t_b) wl = v + 1;
      if (lane == 0 && wl > 0) {  // B stages of this item's frames
        prefetch_tensormap(&tmq);
        const uint64_t pol_b = policy_evict_last();  // the cluster's CTAs share them
        const int ngr = (nit + kGS - 1) / kGS;
        for (int m = 0; m < ngr; ++m) {
          const int zs = m % NB;
          if (m >= NB) mbar_wait(zfree + 8u * zs, (static_cast<uint32_t>(m / NB) & 1u) ^ 1u);
          mbar_arrive_expect_tx(zfull + 8u * zs, stage_bytes);
          for (int at = 0; at < a.Kp / umma::kAtomK; ++at)
            tma_load_2d(base + SL.zst + zs * stage_bytes + at * atom_bytes, &tmq,
                        at * umma::kAtomK, b * a.Sp + m * GN, zfull + 8u * zs, pol_b);
        }
      } else if (lane >= 2 && lane < 2 + W && a.zero_fill != 0) {  // zero fill of warp lane-2's rows
        const int v = lane - 2;
        const int i0v = band + (crank * W + v) * kRows4;
        if (i0v < t_b) {
          LinearZero lz(a, b, i0v, kRows4, nit);
          for (int m = 0; m < nit; ++m) {
            if (!lz.due(m)) continue;
            if (m >= N) {  // paced by the compute warp's ring
              const int st = m % N;
              mbar_wait(base + SL.ebars + static_cast<uint32_t>((v * N + st) * 8),
                        (static_cast<uint32_t>(m / N) & 1u) ^ 1u);
            }
            lz.issue_upto(m, base + SL.zero);
          }
          bulk_store_drain();
        }
      }
    }
    // one-launch tail (one CTA per item): the last warp's zero fill also
    // covers the item's rows past the CTA's W * 128 (a ragged batch whose
    // longest text is shorter than text_cap)
    const int zrows = kTail && w == W - 1 ? a.T_cap : kRows4;
    if (kTail && w < W && a.zero_fill && !(s_b > 0 && i0w < t_b)) {
      // one-launch tail, a warp with no rows to compute (past a short item's
      // text, or an empty item): its rows of the output are zeroed at once
      LinearZero lz(a, b, i0w, zrows, 1);
      lz.issue_upto(0, base + SL.zero);
      bulk_store_complete();
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    if (SRC == 0 && w < W && s_b > 0 && i0w < t_b) {
      LinearZero lz(a, b, i0w, zrows, nit);
      prefetch_tensormap(&tmq);
      // evict_unchanged: evict_first re-read 8 % of q (r12, profiles/r12_l2_policy.md)
      const uint64_t pol_q = policy_evict_unchanged();
      const bool zero_fill = a.zero_fill != 0;
      const uint32_t zero_tile = base + SL.zero;
      const int group = (b * a.T_pad + i0w) / R;
      const int l2a = a.l2_ahead;
      for (int m = 0; m < l2a && m < nit; ++m) tma_prefetch_3d(&tmq, m * kSC, group, 0);
      // OUT: the stage's Q values go back to q's storage (this item's row
      // groups i0w / R ..) before the slot is refilled
      const int ogroup = i0w / R;
      auto store_stage = [&](int mm) {
        tma_store_4d(&tm_out,
                     base + SL.ring + static_cast<uint32_t>((w * N + mm % N) * kStage4),
                     mm * kSC, ogroup, 0, b);
      };
      for (int m = 0; m < nit; ++m) {
        const int st = m % N;
        const uint32_t bar = base + SL.bars + static_cast<uint32_t>((w * N + st) * 8);
        if (m >= N) {
          // stage st of warp w was consumed in iteration m - N
          const uint32_t eb = base + SL.ebars + static_cast<uint32_t>((w * N + st) * 8);
          mbar_wait(eb, (static_cast<uint32_t>(m / N) & 1u) ^ 1u);
          if constexpr (kExport) {
            store_stage(m - N);
            bulk_store_drain();  // the store has read the slot
          }
        }
        if (l2a > 0 && m + l2a < nit) tma_prefetch_3d(&tmq, (m + l2a) * kSC, group, 0);
        mbar_arrive_expect_tx(bar, kStage4);
#pragma unroll
        for (int c = 0; c < kChunks; ++c)
          tma_load_3d(base + SL.ring +
                          static_cast<uint32_t>((w * N + st) * kStage4 + c * chunk_bytes(R)),
                      &tmq, m * kSC + c * kCols4, group, 0, bar, pol_q);
        if (zero_fill) lz.issue_upto(m, zero_tile);
      }
      if (zero_fill) {
        if constexpr (kTail) {
          // the tail writes the ones into these rows: the zeros must be in
          // memory (not only read out of shared memory) and visible to the
          // generic proxy first
          bulk_store_complete();
          asm volatile("fence.proxy.async.global;" ::: "memory");
        } else {
          bulk_store_drain();
        }
      }
      if constexpr (kExport) {
        for (int m = nit > N ? nit - N : 0; m < nit; ++m) {
          mbar_wait(base + SL.ebars + static_cast<uint32_t>((w * N + m % N) * 8),
                    static_cast<uint32_t>(m / N) & 1u);
          store_stage(m);
        }
        bulk_store_complete();
      }
    }
    __syncwarp();
    // one-launch tail: the compute warps expand only after this warp's zero
    // fill is complete (named barrier 2: W compute warps + this warp)
    if constexpr (kTail) asm volatile("bar.arrive 2, %0;" ::"r"((W + 1) * 32) : "memory");
    cluster_sync_all();
    return;
  }

  // one-launch tail: the direction-word table (generic pointer into shared memory)
  uint32_t* const tail_tbl = reinterpret_cast<uint32_t*>(sbase + SL.tbl) + kTailGuard;
  const int tail_rows = W * kRows4;
  (void)tail_tbl;
  (void)tail_rows;
  const int g = crank * W + warp;
  const int i0 = band + g * kRows4;
  const bool has_in = g > 0 || fed;
  const bool last_in_band = g == a.K * W - 1;  // its consumer is the band drain
  const bool live = i0 < t_b && s_b > 0;
  if (live) {
    const uint32_t bar0 = base + SL.bars + static_cast<uint32_t>(warp * N * 8);
    const uint32_t ebar0 = base + SL.ebars + static_cast<uint32_t>(warp * N * 8);
    const uint32_t my_full = base + SL.full + static_cast<uint32_t>(warp * kFifoSlots * 8);
    const uint32_t my_empty = base + SL.empty + static_cast<uint32_t>(warp * kFifoIt4 * 8);
    uint8_t* const my_fifo = sbase + SL.fifo + warp * kFifoSlots * kSlot4;
    const bool has_out = i0 + kRows4 < t_b && (!last_in_band || drains);
    int nw = warp + 1, nr = crank;
    if (last_in_band) {
      nw = W;  // staging FIFO W of this CTA
    } else if (nw == W) {
      nw = 0;
      nr = crank + 1;
    }
    int pw = warp - 1, pr = crank;
    if (g == 0) {  // fed by the band feeder (producer warp lane W)
      pw = W;
      pr = crank;
    } else if (pw < 0) {
      pw = W - 1;
      pr = crank - 1;
    }
    Fifo4 F;
    F.full = my_full;
    F.empty = my_empty;
    F.next_fifo =
        has_out ? mapa(base + SL.fifo + static_cast<uint32_t>(nw * kFifoSlots * kSlot4), nr) : 0u;
    F.next_full =
        has_out ? mapa(base + SL.full + static_cast<uint32_t>(nw * kFifoSlots * 8), nr) : 0u;
    F.prev_empty =
        has_in ? mapa(base + SL.empty + static_cast<uint32_t>(pw * kFifoIt4 * 8), pr) : 0u;
    F.prev_sink = has_in ? mapa(base + SL.sink + static_cast<uint32_t>(pw * 16), pr) : 0u;
    F.buf = my_fifo;
    F.has_in = has_in;
    F.has_out = has_out;

    const uint8_t* ring_ptr = sbase + SL.ring + warp * N * kStage4;
    uint32_t coff[8];
#pragma unroll
    for (int a4 = 0; a4 < 8; ++a4) coff[a4] = lane * 128u + ((a4 ^ (lane & 7)) << 4);
    const uint64_t pol_dir = policy_evict_last();

    const bool is31 = lane == 31;
    const int srclane = (lane + 31) & 31;
    const int row0 = i0 + R * lane;
    const bool row0_is_zero = row0 == 0;
    const uint32_t row0_mask = row0_is_zero ? 0u : 0xffffffffu;
    uint32_t live_rows = 0;  // OUT: this lane's rows inside the item's text
#pragma unroll
    for (int r = 0; r < R; ++r) live_rows |= row0 + r < t_b ? 1u << r : 0u;
    const float mnv = a.mnv;
    Lane4<R> L;
#pragma unroll
    for (int r = 0; r < R; ++r) L.o[r] = 0.0f;
#pragma unroll
    for (int r = 0; r < R / 2; ++r) L.acc[r] = 0.0f;
    L.vlast = a.row0_up;
    float ex[kQuad];
#pragma unroll
    for (int u = 0; u < kQuad; ++u) ex[u] = 0.0f;
    uint32_t* dirs_ptr = a.dirs + static_cast<size_t>(b) * a.M * a.T_alloc + i0 + R * lane;

    bool ready = false;  // FIFO quad look-ahead
    if (has_in && lane == 0) mbar_arrive_expect_tx(my_full, kSlot4);
    // Look-ahead results of the previous iteration's probes (see Probes).
    bool stage_ready = false;
    bool empty_ready = true;

    auto store_words = [&](uint32_t* p, const uint32_t (&v)[R]) {
      if constexpr (R == 4)
        asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p),
                     "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "l"(pol_dir));
      else
        asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(v[0]),
                     "r"(v[1]), "l"(pol_dir));
    };
    int slot = 0;
    uint32_t par = 0;
    // One 32-column stage.  GEN: the first stage, the reference engine's
    // pinned prefix and a partial last stage take the generic code; every
    // other stage runs the straight-line one in its own loop below, so the
    // per-stage bookkeeping between fast stages is only the waits, the
    // release (predicated, no branch) and the word store.
    auto stage_body = [&](int m, auto gen_tag) {
      constexpr bool GEN = decltype(gen_tag)::value;
      mbar_wait_all_unless(stage_ready, bar0 + 8u * slot, par);
      const uint8_t* stage = ring_ptr + slot * kStage4;
      const int c_base = m * kSC;
      const int nvalid = GEN ? (s_b - c_base < kSC ? s_b - c_base : kSC) : kSC;
      uint32_t w[kChunks][R];
#pragma unroll
      for (int c = 0; c < kChunks; ++c)
#pragma unroll
        for (int r = 0; r < R; ++r) w[c][r] = 0u;
      // This iteration's slots in the consumer are free once it released
      // iteration m - kFifoIt4 (4-byte st.async on empty[m % kFifoIt4]).
      mbar_wait_all_unless(!has_out || m < kFifoIt4 || empty_ready,
                           my_empty + 8u * static_cast<uint32_t>(m % kFifoIt4),
                           (static_cast<uint32_t>(m / kFifoIt4) & 1u) ^ 1u);
      const bool more = m + 1 < nit;
      Probes P;
      {
        const int ns = slot + 1 == N ? 0 : slot + 1;
        P.stage_bar = bar0 + 8u * ns;
        P.stage_par = ns == 0 ? par ^ 1u : par;
        const int m1 = m + 1;
        P.empty_bar = my_empty + 8u * static_cast<uint32_t>(m1 % kFifoIt4);
        P.empty_par = (static_cast<uint32_t>(m1 / kFifoIt4) & 1u) ^ 1u;
        P.arm_empty = has_out && m1 >= kFifoIt4 && more;  // lane 31 arms
        P.stage_ok = false;
        P.empty_ok = false;
      }
      fwd4_stage<R, MODE, GEN, kExport>(stage, coff, F, ex, L, w, ready, more, is31, lane, srclane,
                                    kQuadsPerStage * m, c_base, nvalid, row0, mnv, row0_is_zero,
                                    P, live_rows);
      // OUT: the Q values written into the stage are read by the producer's
      // TMA store (async proxy)
      if constexpr (kExport) fence_proxy_async_smem();
      stage_ready = P.stage_ok;
      empty_ready = P.empty_ok || !P.arm_empty;
      // Every value of this stage and of this iteration's FIFO slots has been
      // consumed: hand the stage back to the producer warp and release the
      // slots to the warp above (lane 0; predicated, no branch).
      __syncwarp();
      mbar_arrive_local_if(lane == 0, ebar0 + 8u * slot);
      st_async_b32_if(lane == 0 && has_in, F.prev_sink, static_cast<uint32_t>(m),
                      F.prev_empty + 8u * static_cast<uint32_t>(m % kFifoIt4));
      if constexpr (!kExport) {
        // Row 0 and column -1 are stored as zero bits (the backtrack never
        // steps above row 0 or left of column 0).
        if (GEN && m == 0) {
#pragma unroll
          for (int r = 0; r < R; ++r) w[0][r] &= 0x7fffffffu;
        }
#pragma unroll
        for (int c = 0; c < kChunks; ++c) {
          w[c][0] &= row0_mask;
          if constexpr (kTail) {
            static_assert(R == 4, "the tail table stores four rows per lane");
            const int k = m * kChunks + c;
            *reinterpret_cast<uint4*>(tail_tbl + k * tail_rows + i0 + R * lane) =
                make_uint4(w[c][0], w[c][1], w[c][2], w[c][3]);
          } else {
            if (c == 0 || m * kChunks + c < a.M) store_words(dirs_ptr + c * a.T_alloc, w[c]);
          }
        }
        if constexpr (!kTail) dirs_ptr += kChunks * a.T_alloc;
      }
      slot = slot + 1 == N ? 0 : slot + 1;
      par ^= slot == 0 ? 1u : 0u;
    };
    // stages [mf0, mf1) take the fast code: after the first, past the
    // reference engine's pinned cells (c_base >= i0 + kRows4 - 1), before a
    // partial last stage
    int mf0 = 1;
    if (MODE == 1) mf0 = max(mf0, (i0 + kRows4 - 1 + kSC - 1) / kSC);
    const int mf1 = s_b % kSC == 0 ? nit : nit - 1;
    int m = 0;
    while (m < nit) {
      if (m >= mf0 && m < mf1) {
        // two stages per iteration: half the loop-back branch resolutions
        // (interleaved A/B: pipelined 0.2304 -> 0.2264 ms, plain 0.2711 ->
        // 0.2701); not for the Gaussian source or the score export, whose
        // larger stage bodies then spill (K1g 331 -> 377 us, K1s 400 -> 417 us)
        constexpr int kUnroll = SRC == 0 && OUT == 0 ? 2 : 1;
#pragma unroll kUnroll
        for (; m < mf1; ++m) stage_body(m, BoolTag<false>{});
      } else {
        stage_body(m, BoolTag<true>{});
        ++m;
      }
    }
    __syncwarp();
    bool bad = false;
#pragma unroll
    for (int r = 0; r < R; ++r) bad |= row0 + r < t_b;
    bool nonfinite = false;
#pragma unroll
    for (int r = 0; r < R / 2; ++r) nonfinite |= !(L.acc[r] < INFINITY);
    bad = bad && nonfinite;
    if (!kExport && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flags + b, 1);
  }
  __syncwarp();
  if constexpr (kTail) {
    // ---- one-launch tail: walk and expand this CTA's item ----------------
    // (every compute warp, live or not, takes part in the barriers)
    const int nthr = W * 32;
    const int tid = threadIdx.x;
    int* const rec_y = reinterpret_cast<int*>(tail_tbl + a.M * tail_rows);
    uint32_t* const rec_ex = reinterpret_cast<uint32_t*>(rec_y + a.M);
    int32_t* const path = a.path ? a.path + static_cast<size_t>(b) * a.S_cap : nullptr;
    int32_t* const dur = a.dur ? a.dur + static_cast<size_t>(b) * a.T_cap : nullptr;
    uint8_t* const out = a.out ? a.out + static_cast<size_t>(b) * a.T_cap * a.S_cap : nullptr;
    const bool any = t_b > 0 && s_b > 0;
    // durations buffer first holds each row's last column (-1 before column 0)
    if (dur)
      for (int i = tid; i < a.T_cap; i += nthr) dur[i] = any ? -1 : 0;
    if (path)
      for (int j = (any ? s_b : 0) + tid; j < a.S_cap; j += nthr) path[j] = -1;
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");  // the table is complete
    if (any && tid == 0 && s_b > 1) tail_walk(tail_tbl, tail_rows, t_b, s_b, rec_y, rec_ex);
    // the zeros are in memory (producer warp, barrier 2) and the walk is done
    asm volatile("bar.sync 2, %0;" ::"r"((W + 1) * 32) : "memory");
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
    if (any) {
      if (tid == 0) {  // backtrack.hpp:23-24: the last column is on the last row
        if (path) path[s_b - 1] = t_b - 1;
        if (out) out[static_cast<size_t>(t_b - 1) * a.S_cap + s_b - 1] = 1;
        if (dur) dur[t_b - 1] = s_b - 1;
      }
      // word k covers columns 32k - 1 .. 32k + 30 (position p = column + 1 - 32k)
      const int ktop = (s_b - 1) >> 5;
      for (int k = warp; k <= ktop && s_b > 1; k += W) {
        const int j = 32 * k + lane - 1;
        const bool valid = j >= 0 && j <= s_b - 2;
        const uint32_t rx = rec_ex[k];
        const int row = rec_y[k] - __popc(rx << lane);
        if (valid) {
          if (path) path[j] = row;
          if (out) out[static_cast<size_t>(row) * a.S_cap + j] = 1;
          // an exit here: the row's last column
          if (dur && ((rx >> (31 - lane)) & 1u)) dur[row] = j;
        }
      }
    }
    if (dur) {
      asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
      if (warp == 0) {  // last columns -> durations: dur[r] = last[r] - last[r - 1], 0 past t
        int carry = -1;
        for (int r0 = 0; r0 < a.T_cap; r0 += 32) {
          const int r = r0 + lane;
          const int v = r < t_b ? dur[r] : 0;
          const int up = __shfl_up_sync(0xffffffffu, v, 1);
          const int prev = lane == 0 ? carry : up;
          carry = __shfl_sync(0xffffffffu, v, 31);
          if (r < a.T_cap) dur[r] = r < t_b ? v - prev : 0;
        }
      }
    }
  }
  cluster_sync_all();  // no CTA leaves while a peer may still write its FIFO
}

}  // namespace

// Gaussian source pipeline for W tiles of Kp: 128-frame MMAs (half the MMA
// issues of 64-frame ones; r12) when A, one 128-column accumulator per tile
// and one B stage fit TMEM / shared memory, else 64-frame MMAs with more
// buffers.
GaussCfg gauss_cfg(int W, int Kp) {
  GaussCfg c{0, 0, 0};
  if (Kp <= 0 || W < 1) return c;
  const int a_cols = W * Kp / 2;
  if (a_cols + W * 128 <= 512 && Kp <= 192) {
    c.gN = 128;
    c.gacc = std::min(2, (512 - a_cols) / (W * 128));
    c.gstages = 1;
  } else {
    c.gN = 64;
    c.gacc = std::min(kGAcc, (512 - a_cols) / (W * 64));
    c.gstages = Kp <= 192 ? 2 : 1;
  }
  return c;
}
size_t fwd4_tail_bytes(int R, int W, int M) { return static_cast<size_t>(tail_bytes(M, W * rows_of(R))); }
size_t fwd4_smem_bytes(int R, int W, int N, int Kp) {
  const GaussCfg c = gauss_cfg(W, Kp);
  return smem4_layout(R, W, N, Kp, c.gstages, c.gN).total + 1024u;
}

namespace {
template <int R, int MODE, int SRC, int OUT>
const void* fwd4_fn() {
  return reinterpret_cast<const void*>(&mas_fwd4_kernel<R, MODE, SRC, OUT>);
}
// src 0: q from HBM, 1: Gaussian source, 2: q from HBM with score export
const void* fwd4_fn(int R, int mode, int src = 0) {
  (void)R;  // four rows per lane
  if (src == 1) return mode == 0 ? fwd4_fn<4, 0, 1, 0>() : fwd4_fn<4, 1, 1, 0>();
  if (src == 2) return mode == 0 ? fwd4_fn<4, 0, 0, 1>() : fwd4_fn<4, 1, 0, 1>();
  if (src == 3) return mode == 0 ? fwd4_fn<4, 0, 0, 2>() : fwd4_fn<4, 1, 0, 2>();
  return mode == 0 ? fwd4_fn<4, 0, 0, 0>() : fwd4_fn<4, 1, 0, 0>();
}
}  // namespace

cudaError_t fwd4_configure() {
  constexpr int kMaxDevices = 64;
  static std::once_flag once[kMaxDevices];
  static cudaError_t status[kMaxDevices];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  std::call_once(once[dev], [dev] {
    int smem_max = 0;
    cudaError_t r = cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    for (int v = 0; v < 8 && r == cudaSuccess; ++v) {
      const void* fn = fwd4_fn(4, v & 1, v >> 1);
      r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
      if (r == cudaSuccess)
        r = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    status[dev] = r;
  });
  return status[dev];
}

int fwd4_max_active_clusters(int R, int W, int N, int K, int Kp) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(K), 1, 1);
  cfg.blockDim = dim3(static_cast<unsigned>((W + 1 + (Kp > 0 ? 1 + 4 * W : 0)) * 32), 1, 1);
  cfg.dynamicSmemBytes = fwd4_smem_bytes(R, W, N, Kp);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(K);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, fwd4_fn(R, 0, Kp > 0 ? 1 : 0), &cfg) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return n;
}

cudaError_t launch_fwd4(int R, int mode, const CUtensorMap& tmq, const CUtensorMap& tm_out,
                        const FwdArgs& a, int B, cudaStream_t stream) {
  const bool gauss = a.Kp > 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(B * a.K), 1, 1);
  // + the producer warp (+ the MMA warp and four epilogue warps for the Gaussian source)
  cfg.blockDim = dim3(static_cast<unsigned>((a.W + 1 + (gauss ? 1 + 4 * a.W : 0)) * 32), 1, 1);
  cfg.dynamicSmemBytes = fwd4_smem_bytes(R, a.W, a.N, a.Kp) +
                         (a.tail ? static_cast<size_t>(tail_bytes(a.M, a.W * rows_of(R))) : 0);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(a.K);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cudaLaunchAttribute attrs2[2] = {attr[0], {}};
  if (a.pdl) {
    // may start while the previous kernel in the stream (a backtrack that
    // triggered early) still runs; it shares no buffer with it
    attrs2[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs2[1].val.programmaticStreamSerializationAllowed = 1;
  }
  cfg.attrs = attrs2;
  cfg.numAttrs = a.pdl ? 2 : 1;
  if (R != 4) return cudaErrorInvalidValue;
  if (gauss)
    return mode == 0 ? cudaLaunchKernelEx(&cfg, mas_fwd4_kernel<4, 0, 1, 0>, tmq, tm_out, a)
                     : cudaLaunchKernelEx(&cfg, mas_fwd4_kernel<4, 1, 1, 0>, tmq, tm_out, a);
  if (a.scores)
    return mode == 0 ? cudaLaunchKernelEx(&cfg, mas_fwd4_kernel<4, 0, 0, 1>, tmq, tm_out, a)
                     : cudaLaunchKernelEx(&cfg, mas_fwd4_kernel<4, 1, 0, 1>, tmq, tm_out, a);
  if (a.tail)
    return mode == 0 ? cudaLaunchKernelEx(&cfg, mas_fwd4_kernel<4, 0, 0, 2>, tmq, tm_out, a)
                     : cudaLaunchKernelEx(&cfg, mas_fwd4_kernel<4, 1, 0, 2>, tmq, tm_out, a);
  return mode == 0 ? cudaLaunchKernelEx(&cfg, mas_fwd4_kernel<4, 0, 0, 0>, tmq, tm_out, a)
                   : cudaLaunchKernelEx(&cfg, mas_fwd4_kernel<4, 1, 0, 0>, tmq, tm_out, a);
}

}  // namespace mas
