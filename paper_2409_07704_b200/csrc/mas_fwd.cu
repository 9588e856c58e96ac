// mas_fwd.cu -- K1: the forward maximum-path DP on sm_100a.
//
// Restates, bit for bit on the alignment, the reference's forward passes:
//   parallel engine  relax_column      src/parallel.cpp:25-31 (driven :73-80)
//   reference engine forward_reference src/reference.cpp:9-36
// and stores only what the backtrack (src/backtrack.hpp:21-32) reads: one
// direction bit per cell,
//   bit(i, c) = Q[i-1][c] > Q[i][c]          (strict: ties stay, :26)
// which is exactly the comparison the next column's max performs, so it is
// produced for free while computing column c+1.
//
// Work decomposition:
//   * one thread-block cluster of K CTAs per item; CTA rank c, warp w owns
//     the 64 text rows [64 g, 64 g + 64), g = c * W + w; lane k owns rows
//     64 g + 2k and 64 g + 2k + 1 in registers (the running column);
//   * speech columns are walked in order, 64 per iteration; the row above a
//     lane's first row arrives by __shfl_sync from lane k-1, and for lane 0
//     from the previous warp through a FIFO of 64-column slots in shared
//     memory, filled by the producer with st.async (DSMEM when the producer
//     lives in another CTA of the cluster) and tracked by mbarriers;
//   * q is streamed per warp with TMA into an N-stage ring of 64-row x
//     64-column fp32 tiles (128-byte swizzle, rows de-interleaved by parity
//     so every LDS.128 is conflict-free), L2 evict_first; nothing else is
//     read;
//   * direction words (one u32 per row per 32 columns, bit-reversed: the
//     bit of column 32m + p - 1 is bit 31 - p of word m) are written with
//     L2 evict_last so the backtrack finds them in L2; the output's zero
//     fill is issued alongside as asynchronous TMA stores of a zero tile;
//   * NonFinite validation (types.cpp:107-115) is fused: an FFMA per cell
//     folds q * 0 into a per-lane accumulator (NaN iff some q is inf/NaN);
//     a flagged item is re-scanned exactly by the locator kernel on the
//     error path only;
//   * per step the ALU pipe (the bottleneck, 2 cycles per warp instruction
//     per SM sub-partition) carries only FMNMX x2, FSETP x2 and the shuffle
//     select; bit packing (predicated IMAD) and the NonFinite fold (FFMA) run
//     on the FMA pipe next to the FADDs.
#include <mutex>

#include "mas_kernels.h"
#include "mas_ptx.cuh"

namespace mas {

namespace {

constexpr int kSubCols = 32;                            // columns per TMA box / dirs word
constexpr int kSubBytes = kRowsPerWarp * kSubCols * 4;  // 8 KiB: [parity][32 rows][32 cols]
constexpr int kSlotBytes = kQuadCols * 4;               // one FIFO slot (16 floats)
constexpr int kFifoIters = kFifoSlots / (kStageCols / kQuadCols);  // FIFO depth in iterations
#ifndef MAS_L2_AHEAD
#define MAS_L2_AHEAD 0
#endif
constexpr int kL2Ahead = MAS_L2_AHEAD;  // iterations of L2 prefetch beyond the smem ring

struct SmemLayout {
  uint32_t ring, bars, full, empty, sink, fifo, zero, total;
};

// Per CTA: W rings of N TMA stages, the TMA mbarriers, and per warp a
// kFifoSlots-deep boundary-row FIFO with its "full" barriers (completed by
// the producer's st.async bytes) and the "empty" barriers of the FIFO this
// warp feeds (arrived remotely by its consumer); plus one zero tile.
__host__ __device__ inline SmemLayout smem_layout(int W, int N) {
  SmemLayout L;
  L.ring = 0;
  L.bars = static_cast<uint32_t>(W * N * kStageBytes);
  L.full = L.bars + static_cast<uint32_t>(W * N * 8);
  L.empty = L.full + static_cast<uint32_t>(W * kFifoSlots * 8);
  L.sink = L.empty + static_cast<uint32_t>(W * kFifoSlots * 8);  // st.async target of releases
  L.fifo = (L.sink + static_cast<uint32_t>(W * 16) + 127u) & ~127u;
  L.zero = L.fifo + static_cast<uint32_t>(W * kFifoSlots * kSlotBytes);
  L.total = L.zero + static_cast<uint32_t>(kRowsPerWarp * kStageCols);
  return L;
}

// Per-warp state of the running column.
struct Lane {
  float o0, o1;  // Q of the lane's two rows at the previous column
  float acc;     // sum of q * 0: NaN iff a non-finite q was seen
  float vlast;   // producer's bottom row at the previous column
};

// Four steps (one LDS.128 per row parity) of the DP for one warp.
template <int MODE, bool GENERIC, int SUB, int A4>
__device__ __forceinline__ bool fwd_group(const uint8_t* __restrict__ tile, const uint32_t (&coff)[8],
                                         const float4* __restrict__ slot, float (&ex)[kQuadCols],
                                         Lane& L, uint32_t& w0, uint32_t& w1, bool is31,
                                         int srclane, int c_base, int nvalid, int row0, float mnv,
                                         bool row0_is_zero, uint32_t one, float zero) {
  constexpr int ug = SUB * 32 + A4 * 4;  // step index within the iteration
  if (GENERIC && ug >= nvalid) return false;
  const float4 qa = *reinterpret_cast<const float4*>(tile + coff[A4]);
  const float4 qb = *reinterpret_cast<const float4*>(tile + 4096 + coff[A4]);
  const float4 vv = slot[A4 & 3];  // producer's bottom row, columns c-1 .. c+2
  const float qs0[4] = {qa.x, qa.y, qa.z, qa.w};
  const float qs1[4] = {qb.x, qb.y, qb.z, qb.w};
  const float bnds[4] = {L.vlast, vv.x, vv.y, vv.z};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    if (GENERIC && ug + e >= nvalid) return false;
    const float q0 = qs0[e];
    const float q1 = qs1[e];
    // Lane 31 forwards the previous warp's bottom row (column c-1) to lane
    // 0; every other lane forwards its own bottom row to lane k+1.
    const float send = is31 ? bnds[e] : L.o1;
    const float up = __shfl_sync(0xffffffffu, send, srclane);
    switch (A4 * 4 + e) {  // compile-time bit position
#define MAS_BITS(U)                          \
  case U:                                    \
    set_bit_if_gt<31 - U>(w0, up, L.o0, one); \
    set_bit_if_gt<31 - U>(w1, L.o0, L.o1, one); \
    break;
      MAS_BITS(0) MAS_BITS(1) MAS_BITS(2) MAS_BITS(3) MAS_BITS(4) MAS_BITS(5) MAS_BITS(6)
      MAS_BITS(7) MAS_BITS(8) MAS_BITS(9) MAS_BITS(10) MAS_BITS(11) MAS_BITS(12) MAS_BITS(13)
      MAS_BITS(14) MAS_BITS(15) MAS_BITS(16) MAS_BITS(17) MAS_BITS(18) MAS_BITS(19)
      MAS_BITS(20) MAS_BITS(21) MAS_BITS(22) MAS_BITS(23) MAS_BITS(24) MAS_BITS(25)
      MAS_BITS(26) MAS_BITS(27) MAS_BITS(28) MAS_BITS(29) MAS_BITS(30) MAS_BITS(31)
#undef MAS_BITS
    }
    float n0 = q0 + fmaxf(up, L.o0);  // bit(row0, c-1) = up > o0 above
    float n1 = q1 + fmaxf(L.o0, L.o1);
    if (GENERIC) {
      const int c = c_base + ug + e;
      if (MODE == 1) {
        if (c < row0) n0 = mnv;
        if (c < row0 + 1) n1 = mnv;
      }
      if (c == 0) {  // first column: parallel.cpp:73-75 / reference.cpp:16-24
        n0 = row0_is_zero ? q0 : mnv;
        n1 = mnv;
      }
    }
    fold_nonfinite(L.acc, q0, zero);
    fold_nonfinite(L.acc, q1, zero);
    ex[(A4 & 3) * 4 + e] = n1;
    L.o0 = n0;
    L.o1 = n1;
  }
  L.vlast = vv.w;
  return true;
}

// Endpoints of a warp's boundary-row FIFOs: the one it consumes (its
// producer is the warp above) and the one it feeds (in the warp below,
// possibly in another CTA of the cluster: cluster shared-window addresses).
struct Fifo {
  uint32_t full, empty;            // my FIFO's "full" barriers, my "empty" barriers
  uint32_t next_fifo, next_full;   // consumer's slots and "full" barriers
  uint32_t prev_empty, prev_sink;  // producer's "empty" barriers and release sink
  const uint8_t* buf;              // my FIFO's slots (generic pointer)
  bool has_in, has_out;
};

// One quad = 16 columns = 4 groups, with the FIFO hand-off around it: wait
// for the producer's 16 bottom-row values, compute, release the slot, and
// (lane 31) pass this warp's own 16 bottom-row values on.  Handing off per
// 16 columns keeps each warp only ~16 columns behind the warp above, so the
// wavefront across an item's warps fills and drains 4x faster than with
// whole-iteration hand-offs.  GENERIC handles column 0, reference-engine
// masking (cells with c < i stay exactly max_neg_val, reference.cpp:12-17,
// :30) and a partial last iteration; the steady-state instantiation has
// none of those checks.  Per step the ALU pipe carries FMNMX x2, FSETP x2
// and the shuffle select, the FMA pipe FADD x2, the bit IMADs and the
// NonFinite FFMAs.
template <int MODE, bool GENERIC, int K>
__device__ __forceinline__ bool fwd_quad(const uint8_t* stage, const uint32_t (&coff)[8],
                                        const Fifo& F, float (&ex)[kQuadCols], Lane& L,
                                        uint32_t (&w)[4], bool& ready, bool more, bool is31,
                                        int lane, int srclane, int q, int c_base, int nvalid,
                                        int row0, float mnv, bool row0_is_zero, uint32_t one,
                                        float zero) {
  constexpr int SUB = K / 2;
  if (GENERIC && K * kQuadCols >= nvalid) return false;
  const int fs = q & (kFifoSlots - 1);
  // The producer's 16 values arrive as 64 bytes of st.async on full[fs]
  // (armed with expect_tx one quad earlier).  Usually the look-ahead probe
  // made during the previous quad already saw them land; otherwise block.
  if (F.has_in && !ready) mbar_wait(F.full + 8u * fs, static_cast<uint32_t>(q / kFifoSlots) & 1u);
  // Arm and probe the next quad's slot now, in straight-line code so the
  // probe's result is only consumed after this quad's 16 columns.  (A warp
  // without a producer probes its own never-armed barrier: harmless.)
  const bool next = K < 3 ? (!GENERIC || (K + 1) * kQuadCols < nvalid) : more;
  const int q1 = q + 1;
  const uint32_t bar1 = F.full + 8u * (q1 & (kFifoSlots - 1));
  if (lane == 0 && next && F.has_in) mbar_arrive_expect_tx(bar1, kSlotBytes);
  const bool probe = mbar_test_wait(bar1, static_cast<uint32_t>(q1 / kFifoSlots) & 1u);
  const uint8_t* tile = stage + SUB * kSubBytes;
  const float4* slot = reinterpret_cast<const float4*>(F.buf + fs * kSlotBytes);
  bool ok = true;
#define MAS_GROUP(A)                                                                             \
  if (ok)                                                                                        \
    ok = fwd_group<MODE, GENERIC, SUB, A>(tile, coff, slot, ex, L, w[2 * SUB], w[2 * SUB + 1], \
                                          is31, srclane, c_base, nvalid, row0, mnv,            \
                                          row0_is_zero, one, zero);
  MAS_GROUP((K & 1) * 4 + 0) MAS_GROUP((K & 1) * 4 + 1) MAS_GROUP((K & 1) * 4 + 2)
  MAS_GROUP((K & 1) * 4 + 3)
#undef MAS_GROUP
  ready = probe;
  if (F.has_out && is31) {
    // The consumer's slot is free: checked once per iteration (fwd loop).
    const uint32_t dst = F.next_fifo + static_cast<uint32_t>(fs * kSlotBytes);
    const uint32_t fbar = F.next_full + 8u * fs;
#pragma unroll
    for (int q4 = 0; q4 < kQuadCols / 4; ++q4)
      st_async_v4(dst + 16u * q4, ex[4 * q4], ex[4 * q4 + 1], ex[4 * q4 + 2], ex[4 * q4 + 3], fbar);
  }
  return ok;
}

// One iteration: 64 columns = one TMA stage = two direction words per row.
template <int MODE, bool GENERIC>
__device__ __forceinline__ void fwd_iter(const uint8_t* stage, const uint32_t (&coff)[8],
                                         const Fifo& F, float (&ex)[kQuadCols], Lane& L,
                                         uint32_t (&w)[4], bool& ready, bool more, bool is31,
                                         int lane, int srclane, int q0, int c_base, int nvalid,
                                         int row0, float mnv, bool row0_is_zero, uint32_t one,
                                         float zero) {
#define MAS_QUAD(K)                                                                              \
  if (!fwd_quad<MODE, GENERIC, K>(stage, coff, F, ex, L, w, ready, more, is31, lane, srclane,   \
                                  q0 + K, c_base, nvalid, row0, mnv, row0_is_zero, one, zero)) \
    return;
  MAS_QUAD(0) MAS_QUAD(1) MAS_QUAD(2) MAS_QUAD(3)
#undef MAS_QUAD
}

// L2 prefetch of a whole stage (no shared memory, no completion): issued
// kL2Ahead iterations before the stage's TMA load so DRAM latency jitter is
// absorbed by L2 instead of stalling the warp chain.
__device__ __forceinline__ void prefetch_stage(const CUtensorMap* tm0, const CUtensorMap* tm1,
                                               int col, int row_pair) {
  tma_prefetch_2d(tm0, col, row_pair);
  tma_prefetch_2d(tm1, col, row_pair);
  tma_prefetch_2d(tm0, col + kSubCols, row_pair);
  tma_prefetch_2d(tm1, col + kSubCols, row_pair);
}

__device__ __forceinline__ void issue_stage(uint32_t dst, uint32_t bar, const CUtensorMap* tm0,
                                            const CUtensorMap* tm1, int col, int row_pair,
                                            uint64_t pol) {
  mbar_arrive_expect_tx(bar, kStageBytes);
  tma_load_2d(dst, tm0, col, row_pair, bar, pol);
  tma_load_2d(dst + 4096u, tm1, col, row_pair, bar, pol);
  tma_load_2d(dst + kSubBytes, tm0, col + kSubCols, row_pair, bar, pol);
  tma_load_2d(dst + kSubBytes + 4096u, tm1, col + kSubCols, row_pair, bar, pol);
}

template <int MODE>
__global__ void __launch_bounds__(kMaxWarpsPerCta * 32, 1)
    mas_fwd_kernel(const __grid_constant__ CUtensorMap tm0, const __grid_constant__ CUtensorMap tm1,
                   const __grid_constant__ CUtensorMap tm_out, const FwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_addr(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* const sbase = smem_raw + (base - raw);
  const int W = a.W;
  const int N = a.N;
  const SmemLayout SL = smem_layout(W, N);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int crank = static_cast<int>(cluster_ctarank());
  const int b = a.b0 + static_cast<int>(blockIdx.x) / a.K;
  const int g = crank * W + warp;
  const int i0 = g * kRowsPerWarp;
  const int t_b = static_cast<int>(a.lengths[2 * b]);
  const int s_b = static_cast<int>(a.lengths[2 * b + 1]);
  const bool has_in = g > 0;

  const uint32_t bar0 = base + SL.bars + static_cast<uint32_t>(warp * N * 8);
  const uint32_t my_full = base + SL.full + static_cast<uint32_t>(warp * kFifoSlots * 8);
  const uint32_t my_empty = base + SL.empty + static_cast<uint32_t>(warp * kFifoSlots * 8);
  uint8_t* const my_fifo = sbase + SL.fifo + warp * kFifoSlots * kSlotBytes;
  if (lane == 0) {
    for (int s = 0; s < N; ++s) mbar_init(bar0 + 8u * s, 1u);
    for (int s = 0; s < kFifoSlots; ++s) {
      mbar_init(my_full + 8u * s, 1u);
      mbar_init(my_empty + 8u * s, 1u);
    }
  }
  if (!has_in) {
    // The first warp of an item has no producer: its FIFO permanently holds
    // the value above row 0 (max_neg_val, or -inf for reference.cpp:20-24).
    for (int k = lane; k < kFifoSlots * kQuadCols; k += 32)
      reinterpret_cast<float*>(my_fifo)[k] = a.row0_up;
  }
  // A zeroed 64 x 64-byte tile, the TMA-store source of the fused output fill.
  for (int k = threadIdx.x; k < kRowsPerWarp * kStageCols / 16; k += blockDim.x)
    reinterpret_cast<uint4*>(sbase + SL.zero)[k] = make_uint4(0u, 0u, 0u, 0u);
  fence_proxy_async_smem();
  fence_mbar_init();
  cluster_sync_all();  // every CTA's FIFO state exists before any remote access
  // Let the backtrack grid (programmatic dependent launch) get resident on
  // the SMs this grid leaves idle; it waits for our completion before it
  // touches any data (griddepcontrol.wait).
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  const bool live = i0 < t_b && s_b > 0;
  if (live) {
    const bool has_out = i0 + kRowsPerWarp < t_b;
    int nw = warp + 1, nr = crank;
    if (nw == W) {
      nw = 0;
      nr = crank + 1;
    }
    int pw = warp - 1, pr = crank;
    if (pw < 0) {
      pw = W - 1;
      pr = crank - 1;
    }
    // FIFO endpoints: my consumer's slots + "full" barriers, my producer's
    // "empty" barriers (addresses in the cluster shared window).
    const uint32_t next_fifo =
        has_out ? mapa(base + SL.fifo + static_cast<uint32_t>(nw * kFifoSlots * kSlotBytes), nr)
                : 0u;
    const uint32_t next_full =
        has_out ? mapa(base + SL.full + static_cast<uint32_t>(nw * kFifoSlots * 8), nr) : 0u;
    const uint32_t prev_empty =
        has_in ? mapa(base + SL.empty + static_cast<uint32_t>(pw * kFifoSlots * 8), pr) : 0u;
    const uint32_t prev_sink = has_in ? mapa(base + SL.sink + static_cast<uint32_t>(pw * 16), pr) : 0u;

    const uint32_t ring = base + SL.ring + static_cast<uint32_t>(warp * N * kStageBytes);
    const uint8_t* ring_ptr = sbase + SL.ring + warp * N * kStageBytes;
    uint32_t coff[8];
#pragma unroll
    for (int a4 = 0; a4 < 8; ++a4) coff[a4] = lane * 128u + ((a4 ^ (lane & 7)) << 4);

    const int nit = (s_b + kStageCols - 1) / kStageCols;
    const int row_pair = (b * a.T_pad + i0) / 2;
    const int out_row = b * a.T_cap + i0;
    const uint32_t zero_tile = base + SL.zero;
    const bool zero_fill = a.zero_fill != 0;
    uint64_t pol_q = 0;
    const uint64_t pol_dir = policy_evict_last();
    if (lane == 0) {
      prefetch_tensormap(&tm0);
      prefetch_tensormap(&tm1);
      pol_q = policy_evict_first();
      const int pro = nit < N - 1 ? nit : N - 1;
      for (int it = 0; it < pro; ++it)
        issue_stage(ring + static_cast<uint32_t>(it * kStageBytes), bar0 + 8u * it, &tm0, &tm1,
                    it * kStageCols, row_pair, pol_q);
      const int pre = nit < N - 1 + kL2Ahead ? nit : N - 1 + kL2Ahead;
      for (int it = pro; it < pre; ++it) prefetch_stage(&tm0, &tm1, it * kStageCols, row_pair);
    }

    const bool is31 = lane == 31;
    const int srclane = (lane + 31) & 31;
    const int row0 = i0 + 2 * lane;
    const bool row0_is_zero = row0 == 0;
    const float mnv = a.mnv;
    const uint32_t one = a.one;  // opaque constants (see set_bit_if_gt / fold_nonfinite)
    const float zero = a.zero;
    Lane L;
    L.o0 = 0.0f;
    L.o1 = 0.0f;
    L.acc = 0.0f;
    L.vlast = a.row0_up;
    float ex[kQuadCols];
#pragma unroll
    for (int u = 0; u < kQuadCols; ++u) ex[u] = 0.0f;
    uint32_t* dirs_ptr = a.dirs + static_cast<size_t>(b) * a.M * a.T_alloc + i0 + 2 * lane;
    Fifo F;
    F.full = my_full;
    F.empty = my_empty;
    F.next_fifo = next_fifo;
    F.next_full = next_full;
    F.prev_empty = prev_empty;
    F.prev_sink = prev_sink;
    F.buf = my_fifo;
    F.has_in = has_in;
    F.has_out = has_out;

    // Quad 0's slot is armed here; every later one by the quad before it.
    bool ready = false;
    if (has_in && lane == 0) mbar_arrive_expect_tx(my_full, kSlotBytes);

    // Ring position of iteration m (slot, parity) and the slot refilled at
    // its start (iteration m + N - 1 goes where iteration m - 1 was).
    int slot = 0;
    uint32_t par = 0;
    int free_slot = N - 1;
    for (int m = 0; m < nit; ++m) {
      if (m + N - 1 < nit) {
        __syncwarp();
        if (lane == 0) {
          // The slot being refilled was last read in iteration m-1 by every
          // lane (generic proxy); order those reads before the async write.
          fence_proxy_async_smem();
          issue_stage(ring + static_cast<uint32_t>(free_slot * kStageBytes), bar0 + 8u * free_slot,
                      &tm0, &tm1, (m + N - 1) * kStageCols, row_pair, pol_q);
          if (m + N - 1 + kL2Ahead < nit)
            prefetch_stage(&tm0, &tm1, (m + N - 1 + kL2Ahead) * kStageCols, row_pair);
        }
      }
      mbar_wait(bar0 + 8u * slot, par);

      const uint8_t* stage = ring_ptr + slot * kStageBytes;
      const int c_base = m * kStageCols;
      const int nvalid = s_b - c_base < kStageCols ? s_b - c_base : kStageCols;
      uint32_t w[4] = {0u, 0u, 0u, 0u};
      const bool generic =
          m == 0 || nvalid < kStageCols || (MODE == 1 && c_base < i0 + kRowsPerWarp - 1);
      if (has_out && is31 && m >= kFifoIters) {
        // This iteration's slots are free once the consumer released
        // iteration m - kFifoIters (4-byte st.async on empty[m % kFifoIters]).
        const uint32_t eb = my_empty + 8u * static_cast<uint32_t>(m % kFifoIters);
        mbar_arrive_expect_tx(eb, 4u);
        mbar_wait(eb, (static_cast<uint32_t>(m / kFifoIters) & 1u) ^ 1u);
      }
      const bool more = m + 1 < nit;
      if (generic) {
        fwd_iter<MODE, true>(stage, coff, F, ex, L, w, ready, more, is31, lane, srclane, 4 * m,
                             c_base, nvalid, row0, mnv, row0_is_zero, one, zero);
      } else {
        fwd_iter<MODE, false>(stage, coff, F, ex, L, w, ready, more, is31, lane, srclane, 4 * m,
                              c_base, kStageCols, row0, mnv, row0_is_zero, one, zero);
      }
      if (has_in) {
        // Every value of this iteration's slots has been consumed above:
        // release them with a 4-byte st.async completing the producer's
        // "empty" transaction (prompt, fence-free signalling).
        __syncwarp();
        if (lane == 0)
          st_async_b32(prev_sink, static_cast<uint32_t>(m),
                       prev_empty + 8u * static_cast<uint32_t>(m % kFifoIters));
      }

      // The backtrack never needs (and must never take) a step above row 0
      // or at column -1: store those bits as 0.
      if (m == 0) {
        w[0] &= 0x7fffffffu;
        w[1] &= 0x7fffffffu;
      }
      if (row0_is_zero) {
        w[0] = 0u;
        w[2] = 0u;
      }
      st_global_v2_evict_last(dirs_ptr, w[0], w[1], pol_dir);
      if (2 * m + 1 < a.M) st_global_v2_evict_last(dirs_ptr + a.T_alloc, w[2], w[3], pol_dir);
      dirs_ptr += 2 * static_cast<size_t>(a.T_alloc);

      if (zero_fill && lane == 0) {
        // Fused zero fill of the output tile this warp covers (the backtrack
        // scatters the ones later): one asynchronous TMA store of the zero
        // tile, rows [i0, i0+64) x columns [64m, 64m+64), clipped by TMA.
        tma_store_2d(&tm_out, zero_tile, c_base, out_row);
      }

      slot = slot + 1 == N ? 0 : slot + 1;
      par ^= slot == 0 ? 1u : 0u;
      free_slot = free_slot + 1 == N ? 0 : free_slot + 1;
    }
    if (zero_fill && lane == 0) bulk_store_drain();
    __syncwarp();

    const bool bad = row0 < t_b && !(L.acc < INFINITY);
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flags + b, 1);
  }
  __syncwarp();
  cluster_sync_all();  // no CTA leaves while a peer may still write its FIFO
}

}  // namespace

size_t fwd_smem_bytes(int W, int N) { return smem_layout(W, N).total + 1024u; }

// Kernel attributes are per function, not per launch, so concurrent plans
// with different geometries must not race on them: once per device, allow
// the largest dynamic shared memory the device offers and non-portable
// cluster sizes (each launch still requests only what it needs).
cudaError_t fwd_configure(int W, int N, int K) {
  (void)K;
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
    for (int mode = 0; mode < 2 && r == cudaSuccess; ++mode) {
      const void* fn = mode == 0 ? reinterpret_cast<const void*>(&mas_fwd_kernel<0>)
                                 : reinterpret_cast<const void*>(&mas_fwd_kernel<1>);
      r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
      if (r == cudaSuccess)
        r = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    status[dev] = r;
  });
  if (status[dev] != cudaSuccess) return status[dev];
  int smem_max = 0;
  e = cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  return static_cast<int>(fwd_smem_bytes(W, N)) <= smem_max ? cudaSuccess
                                                            : cudaErrorInvalidConfiguration;
}

static cudaLaunchConfig_t fwd_launch_config(int B, int K, int W, int N, cudaStream_t stream,
                                            cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(B * K), 1, 1);
  cfg.blockDim = dim3(static_cast<unsigned>(W * 32), 1, 1);
  cfg.dynamicSmemBytes = fwd_smem_bytes(W, N);
  cfg.stream = stream;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(K);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

int fwd_max_active_clusters(int W, int N, int K, int mode) {
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = fwd_launch_config(K, K, W, N, nullptr, attr);
  int n = 0;
  const void* fn = mode == 0 ? reinterpret_cast<const void*>(&mas_fwd_kernel<0>)
                             : reinterpret_cast<const void*>(&mas_fwd_kernel<1>);
  if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return n;
}

cudaError_t launch_fwd(int mode, const CUtensorMap& tm0, const CUtensorMap& tm1,
                       const CUtensorMap& tm_out, const FwdArgs& a, int B, cudaStream_t stream) {
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = fwd_launch_config(B, a.K, a.W, a.N, stream, attr);
  if (mode == 0) return cudaLaunchKernelEx(&cfg, mas_fwd_kernel<0>, tm0, tm1, tm_out, a);
  return cudaLaunchKernelEx(&cfg, mas_fwd_kernel<1>, tm0, tm1, tm_out, a);
}

}  // namespace mas
