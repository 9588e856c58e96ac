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
//   * speech columns are walked in order; the row above a lane's first row
//     arrives by __shfl_sync from lane k-1, and for lane 0 from the previous
//     warp through a 32-column-block FIFO in shared memory (DSMEM when the
//     previous warp lives in another CTA of the cluster);
//   * q is streamed per warp with TMA into an N-stage ring of 64 x 32 fp32
//     tiles (128-byte swizzle, rows de-interleaved by parity so every
//     LDS.128 is conflict-free), L2 evict_first; nothing else is read;
//   * direction words (one u32 per row per 32 columns) are written with
//     L2 evict_last so the backtrack finds them in L2;
//   * NonFinite validation (types.cpp:107-115) is fused: max.NaN over |q|
//     per lane, one FMNMX3 per two cells; a flagged item is re-scanned
//     exactly by the locator kernel on the error path only.
#include "mas_kernels.h"
#include "mas_ptx.cuh"

namespace mas {

namespace {

struct SmemLayout {
  uint32_t ring, bars, full, empty, fifo, zero, total;
};

// Per CTA: W rings of N TMA stages, the TMA mbarriers, and per warp a
// kFifoSlots-deep boundary-row FIFO with its "full" barriers (completed by
// the producer's st.async bytes) and the "empty" barriers of the FIFO this
// warp feeds (arrived remotely by its consumer).
__host__ __device__ inline SmemLayout smem_layout(int W, int N) {
  SmemLayout L;
  L.ring = 0;
  L.bars = static_cast<uint32_t>(W * N * kStageBytes);
  L.full = L.bars + static_cast<uint32_t>(W * N * 8);
  L.empty = L.full + static_cast<uint32_t>(W * kFifoSlots * 8);
  L.fifo = (L.empty + static_cast<uint32_t>(W * kFifoSlots * 8) + 127u) & ~127u;
  L.zero = L.fifo + static_cast<uint32_t>(W * kFifoSlots * 32 * 4);
  L.total = L.zero + static_cast<uint32_t>(kRowsPerWarp * 32);
  return L;
}

// One 32-column block of the DP for one warp.  GENERIC handles column 0,
// reference-engine masking (cells with c < i stay exactly max_neg_val,
// reference.cpp:12-17, :30) and a partial last block; the steady-state
// instantiation has none of those checks.
template <int MODE, bool GENERIC>
__device__ __forceinline__ void fwd_block(const uint8_t* __restrict__ stage,
                                          const uint32_t (&coff)[8], const float (&v)[32],
                                          float vprev, float (&ex)[32], float& o0, float& o1,
                                          uint32_t& w0, uint32_t& w1, float& acc, bool is31,
                                          int srclane, int c_base, int nvalid, int row0,
                                          float mnv, bool row0_is_zero) {
  w0 = 0u;
  w1 = 0u;
#pragma unroll
  for (int a4 = 0; a4 < 8; ++a4) {
    if (GENERIC && a4 * 4 >= nvalid) return;
    const float4 qa = *reinterpret_cast<const float4*>(stage + coff[a4]);
    const float4 qb = *reinterpret_cast<const float4*>(stage + 4096 + coff[a4]);
    const float qs0[4] = {qa.x, qa.y, qa.z, qa.w};
    const float qs1[4] = {qb.x, qb.y, qb.z, qb.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int u = a4 * 4 + e;
      if (GENERIC && u >= nvalid) return;
      const float q0 = qs0[e];
      const float q1 = qs1[e];
      // Lane 31 forwards the previous warp's bottom row (column c-1) to lane
      // 0; every other lane forwards its own bottom row to lane k+1.
      const float bnd = (u == 0) ? vprev : v[u - 1];
      const float send = is31 ? bnd : o1;
      const float up = __shfl_sync(0xffffffffu, send, srclane);
      const uint32_t p0 = gt_mask(up, o0);  // bit(row0, c-1)
      const uint32_t p1 = gt_mask(o0, o1);  // bit(row1, c-1)
      float n0 = q0 + fmaxf(up, o0);
      float n1 = q1 + fmaxf(o0, o1);
      if (GENERIC) {
        const int c = c_base + u;
        if (MODE == 1) {
          if (c < row0) n0 = mnv;
          if (c < row0 + 1) n1 = mnv;
        }
        if (c == 0) {  // first column: parallel.cpp:73-75 / reference.cpp:16-24
          n0 = row0_is_zero ? q0 : mnv;
          n1 = mnv;
        }
      }
      w0 |= p0 & (1u << u);
      w1 |= p1 & (1u << u);
      fold_abs_max_nan(acc, q0, q1);
      ex[u] = n1;
      o0 = n0;
      o1 = n1;
    }
  }
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
  const SmemLayout L = smem_layout(W, N);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int crank = static_cast<int>(cluster_ctarank());
  const int b = blockIdx.x / a.K;
  const int g = crank * W + warp;
  const int i0 = g * kRowsPerWarp;
  const int t_b = static_cast<int>(a.lengths[2 * b]);
  const int s_b = static_cast<int>(a.lengths[2 * b + 1]);

  const uint32_t bar0 = base + L.bars + static_cast<uint32_t>(warp * N * 8);
  const uint32_t my_full = base + L.full + static_cast<uint32_t>(warp * kFifoSlots * 8);
  const uint32_t my_empty = base + L.empty + static_cast<uint32_t>(warp * kFifoSlots * 8);
  if (lane == 0) {
    for (int s = 0; s < N; ++s) mbar_init(bar0 + 8u * s, 1u);
    for (int s = 0; s < kFifoSlots; ++s) {
      mbar_init(my_full + 8u * s, 1u);
      mbar_init(my_empty + 8u * s, 1u);
    }
  }
  // A zeroed 64 x 32-byte tile, the TMA-store source of the fused output fill.
  for (int k = threadIdx.x; k < kRowsPerWarp * 32 / 16; k += blockDim.x)
    reinterpret_cast<uint4*>(sbase + L.zero)[k] = make_uint4(0u, 0u, 0u, 0u);
  fence_proxy_async_smem();
  fence_mbar_init();
  cluster_sync_all();  // every CTA's FIFO state exists before any remote access

  const bool live = i0 < t_b && s_b > 0;
  if (live) {
    const bool has_in = g > 0;
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
        has_out ? mapa(base + L.fifo + static_cast<uint32_t>(nw * kFifoSlots * 128), nr) : 0u;
    const uint32_t next_full =
        has_out ? mapa(base + L.full + static_cast<uint32_t>(nw * kFifoSlots * 8), nr) : 0u;
    const uint32_t prev_empty =
        has_in ? mapa(base + L.empty + static_cast<uint32_t>(pw * kFifoSlots * 8), pr) : 0u;
    const uint8_t* my_fifo = sbase + L.fifo + warp * kFifoSlots * 128;

    const uint32_t ring = base + L.ring + static_cast<uint32_t>(warp * N * kStageBytes);
    const uint8_t* ring_ptr = sbase + L.ring + warp * N * kStageBytes;
    uint32_t coff[8];
#pragma unroll
    for (int a4 = 0; a4 < 8; ++a4) coff[a4] = lane * 128u + ((a4 ^ (lane & 7)) << 4);

    const int nblk = (s_b + kStageCols - 1) / kStageCols;
    const int row_pair = (b * a.T_pad + i0) / 2;
    const int out_row = b * a.T_cap + i0;
    const uint32_t zero_tile = base + L.zero;
    const bool zero_fill = a.zero_fill != 0;
    uint64_t pol_q = 0;
    const uint64_t pol_dir = policy_evict_last();
    if (lane == 0) {
      prefetch_tensormap(&tm0);
      prefetch_tensormap(&tm1);
      pol_q = policy_evict_first();
      const int pro = nblk < N - 1 ? nblk : N - 1;
      for (int blk = 0; blk < pro; ++blk) {
        const uint32_t bar = bar0 + 8u * blk;
        const uint32_t dst = ring + static_cast<uint32_t>(blk * kStageBytes);
        mbar_arrive_expect_tx(bar, kStageBytes);
        tma_load_2d(dst, &tm0, blk * kStageCols, row_pair, bar, pol_q);
        tma_load_2d(dst + 4096u, &tm1, blk * kStageCols, row_pair, bar, pol_q);
      }
    }

    const bool is31 = lane == 31;
    const int srclane = (lane + 31) & 31;
    const int row0 = i0 + 2 * lane;
    const bool row0_is_zero = row0 == 0;
    const float mnv = a.mnv;
    float o0 = 0.0f, o1 = 0.0f, acc = 0.0f;
    float vprev = a.row0_up;
    float v[32];
    float ex[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      v[u] = a.row0_up;
      ex[u] = 0.0f;
    }
    uint32_t* dirs_ptr = a.dirs + static_cast<size_t>(b) * a.M * a.T_alloc + i0 + 2 * lane;

    // Ring position of block m (slot, parity) and of the block refilled at
    // its start (m + N - 1 goes into the slot block m - 1 used).
    int slot = 0;
    uint32_t par = 0;
    int free_slot = N - 1;
    for (int m = 0; m < nblk; ++m) {
      const int fs = m & (kFifoSlots - 1);
      const uint32_t fpar = static_cast<uint32_t>(m >> 3) & 1u;
      if (m + N - 1 < nblk) {
        __syncwarp();
        if (lane == 0) {
          // The slot being refilled was last read in block m-1 by every lane
          // (generic proxy); order those reads before the async-proxy write.
          fence_proxy_async_smem();
          const int blk = m + N - 1;
          const uint32_t bar = bar0 + 8u * free_slot;
          const uint32_t dst = ring + static_cast<uint32_t>(free_slot * kStageBytes);
          mbar_arrive_expect_tx(bar, kStageBytes);
          tma_load_2d(dst, &tm0, blk * kStageCols, row_pair, bar, pol_q);
          tma_load_2d(dst + 4096u, &tm1, blk * kStageCols, row_pair, bar, pol_q);
        }
      }
      mbar_wait(bar0 + 8u * slot, par);

      if (has_in) {
        // Producer's block m arrives as 128 bytes of st.async on full[fs].
        if (lane == 0) mbar_arrive_expect_tx(my_full + 8u * fs, 128u);
        mbar_wait(my_full + 8u * fs, fpar);
        const float4* f = reinterpret_cast<const float4*>(my_fifo + fs * 128);
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4) {
          const float4 x = f[q4];
          v[4 * q4 + 0] = x.x;
          v[4 * q4 + 1] = x.y;
          v[4 * q4 + 2] = x.z;
          v[4 * q4 + 3] = x.w;
        }
      }

      const uint8_t* stage = ring_ptr + slot * kStageBytes;
      const int c_base = m * kStageCols;
      const int nvalid = s_b - c_base < kStageCols ? s_b - c_base : kStageCols;
      uint32_t w0, w1;
      const bool generic =
          m == 0 || nvalid < kStageCols || (MODE == 1 && c_base < i0 + kRowsPerWarp - 1);
      if (generic) {
        fwd_block<MODE, true>(stage, coff, v, vprev, ex, o0, o1, w0, w1, acc, is31, srclane,
                              c_base, nvalid, row0, mnv, row0_is_zero);
      } else {
        fwd_block<MODE, false>(stage, coff, v, vprev, ex, o0, o1, w0, w1, acc, is31, srclane,
                               c_base, kStageCols, row0, mnv, row0_is_zero);
      }
      vprev = v[31];
      if (has_in) {
        // Every value read from slot fs has been consumed by the block above.
        __syncwarp();
        if (lane == 0) mbar_arrive_remote_relaxed(prev_empty + 8u * fs);
      }

      st_global_v2_evict_last(dirs_ptr, w0, w1, pol_dir);
      dirs_ptr += a.T_alloc;

      if (has_out && is31) {
        // Slot fs of the consumer is free once it released block m - F.
        if (m >= kFifoSlots) mbar_wait(my_empty + 8u * fs, fpar ^ 1u);
        const uint32_t dst = next_fifo + static_cast<uint32_t>(fs * 128);
        const uint32_t fbar = next_full + 8u * fs;
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4)
          st_async_v4(dst + 16u * q4, ex[4 * q4], ex[4 * q4 + 1], ex[4 * q4 + 2], ex[4 * q4 + 3],
                      fbar);
      }
      if (zero_fill && lane == 0) {
        // Fused zero fill of the output tile this warp covers (the backtrack
        // scatters the ones later): one asynchronous TMA store of a zero
        // tile, rows [i0, i0+64) x columns [32m, 32m+32), clipped by TMA.
        tma_store_2d(&tm_out, zero_tile, c_base, out_row);
      }

      slot = slot + 1 == N ? 0 : slot + 1;
      par ^= slot == 0 ? 1u : 0u;
      free_slot = free_slot + 1 == N ? 0 : free_slot + 1;
    }
    if (zero_fill && lane == 0) bulk_store_drain();
    __syncwarp();

    const bool bad = row0 < t_b && !(acc < INFINITY);
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.flags + b, 1);
  }
  __syncwarp();
  cluster_sync_all();  // no CTA leaves while a peer may still write its FIFO
}

}  // namespace

size_t fwd_smem_bytes(int W, int N) { return smem_layout(W, N).total + 1024u; }

cudaError_t fwd_configure(int W, int N, int K) {
  const int smem = static_cast<int>(fwd_smem_bytes(W, N));
  cudaError_t e;
  for (int mode = 0; mode < 2; ++mode) {
    const void* fn = mode == 0 ? reinterpret_cast<const void*>(&mas_fwd_kernel<0>)
                               : reinterpret_cast<const void*>(&mas_fwd_kernel<1>);
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (K > 8) {
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
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
