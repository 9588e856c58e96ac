// mas_scores.cu -- score-table export: the entry
// points, and the general kernel for layouts the forward kernel's export
// (mas_fwd4.cu OUT 1, forward_scores_fwd4 in mas_abi.cu; tried first)
// cannot map.  The parallel engine's forward pass written back in place, as
// the reference's parallel::forward_parallel does on a MutableLikelihoodView
// (include/monoalign/parallel.hpp:17, src/parallel.cpp:95-108):
//
//   Q[i][0] = mnv                            i >= 1   (Q[0][0] = q[0][0])
//   Q[0][j] = q[0][j] + max(mnv, Q[0][j-1])           j >= 1
//   Q[i][j] = q[i][j] + max(Q[i-1][j-1], Q[i][j-1])   i, j >= 1
//
// with max(a, b) = (a < b) ? b : a (std::max, first argument on ties), so the
// table is bit-identical to the reference's, signed zeros included.  This is
// the call tests use to check scores cell by cell (test_parallel.cpp:91-103);
// it is not on the maximum-path call, which never materialises Q (K1 keeps it
// in registers and emits direction bits).  Costs 8 B/cell (read q, write Q).
//
// Layout: CTAs of 8/R warps; a warp owns 32R rows (lane l: rows l, l+32, ...;
// R = 2 for grids that fit the GPU once, else 1) and walks the item in 32-column tiles.  Within a warp the value of
// the row above comes from a shuffle (tiles are read and written coalesced,
// lane = column, and transposed through shared memory; reads are cp.async
// prefetches two tiles ahead into a 3-buffer ring per warp); across warps, the last row of warp w-1
// is handed to warp w through a 4-tile shared-memory ring with per-warp
// progress counters, so the warps run as a skewed wavefront.  Texts longer
// than 256 rows are split into 256-row strips, one CTA each, running
// concurrently: the first warp of a strip reads the last row of the strip
// above back from the table (L2) as soon as that strip's progress counter
// (release/acquire, global) says the tile is stored.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <algorithm>
#include <mutex>
#include <vector>

#include <cuda_runtime.h>

#include "monoalign_b200.h"
#include "mas_kernels.h"

namespace {

// R rows per lane: lane l owns rows l, l + 32, ... of its warp's 32R-row
// block; CTAs of 8/R warps, so a strip is 256 rows either way.
constexpr int kStripRows = 256;
#define MAS_SCORES_R 2  // rows per lane of the spread launch (R = 4 measured 1.6x slower at c3)
constexpr int kSpreadSmem = 160 * 1024;  // one CTA per SM for the spread launch
constexpr int kStripPub = 8;  // tiles per cross-strip progress release
constexpr int kTile = 32;
constexpr int kRing = 4;
template <int R>
struct Geo {
  static constexpr int kWarps = 8 / R;
  static constexpr int kWarpRows = 32 * R;
  static constexpr int kBufs = R == 1 ? 3 : 2;  // per-warp tile buffers (prefetch distance kBufs-1)
  static constexpr int kTileFloats = kWarpRows * (kTile + 1);
  static constexpr int kTileSmem = kWarps * kBufs * kTileFloats * sizeof(float);
};
static_assert(Geo<1>::kWarps * Geo<1>::kWarpRows == kStripRows, "strip");
static_assert(Geo<2>::kWarps * Geo<2>::kWarpRows == kStripRows, "strip");
static_assert(Geo<4>::kWarps * Geo<4>::kWarpRows == kStripRows, "strip");

__device__ __forceinline__ float ref_max(float a, float b) { return a < b ? b : a; }

__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// 4-byte cp.async; src_bytes = 0 zero-fills without reading.
__device__ __forceinline__ void cp_async4(float* dst, const float* src, int src_bytes) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Rows r0..r0+63, columns j0..j0+31 of the item into buf[row][col]: lane =
// column, so each warp-wide copy reads one contiguous 128-byte segment.
template <int ROWS>
__device__ __forceinline__ void prefetch_tile(float (*buf)[kTile + 1], const float* item,
                                              int64_t pitch, int r0, int j0, int t, int s,
                                              int lane) {
  const bool col_ok = j0 + lane < s;
#pragma unroll 8
  for (int i = 0; i < ROWS; ++i) {
    const bool ok = col_ok && r0 + i < t;
    const float* src = ok ? item + static_cast<int64_t>(r0 + i) * pitch + j0 + lane : item;
    cp_async4(&buf[i][lane], src, ok ? 4 : 0);
  }
}

// MODE 0: parallel::forward_parallel (parallel.cpp:95-108).  MODE 1: the
// reference engine's cache (reference.cpp:9-36): row 0 the running sum
// 0 + q[0][0] + q[0][1] + ..., cells with i > j stay exactly mnv, every
// other cell max(Q[i-1][j-1], Q[i][j-1]) + q[i][j].
template <int R, int MODE>
__global__ void __launch_bounds__(Geo<R>::kWarps * 32, 1)
forward_scores_kernel(float* __restrict__ q, int64_t pitch, int T_cap, int S_cap,
                      const uint32_t* __restrict__ lengths, float mnv, int nstrips,
                      int strips_per_cta, int* __restrict__ ticket, int* __restrict__ progress) {
  constexpr int kWarps = Geo<R>::kWarps, kWarpRows = Geo<R>::kWarpRows, kBufs = Geo<R>::kBufs;
  constexpr int kTileFloats = Geo<R>::kTileFloats;
  extern __shared__ float tiles_raw[];  // [kWarps][kBufs][kWarpRows][kTile + 1]
  __shared__ float ring[kWarps][kRing][kTile];
  __shared__ volatile int published[kWarps];  // tiles warp w has put in its ring
  __shared__ volatile int consumed[kWarps];   // tiles warp w has read from warp w-1's ring
  __shared__ int vblock;
  // Strips are taken in ticket order, so the strip above is always running or
  // done before a strip waits on it (no reliance on block dispatch order).
  if (threadIdx.x == 0) vblock = atomicAdd(ticket, 1);
  __syncthreads();
  const int ngroups = (nstrips + strips_per_cta - 1) / strips_per_cta;
  const int b = vblock / ngroups, first_strip = vblock % ngroups * strips_per_cta;
  const int t = lengths ? static_cast<int>(lengths[2 * b]) : T_cap;
  const int s = lengths ? static_cast<int>(lengths[2 * b + 1]) : S_cap;
  if (t < 1 || s < 1) return;  // uniform per CTA
  float* item = q + static_cast<int64_t>(b) * T_cap * pitch;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = (s + kTile - 1) / kTile;
  auto buf = [&](int c) {
    return reinterpret_cast<float(*)[kTile + 1]>(tiles_raw + (warp * kBufs + c % kBufs) * kTileFloats);
  };

  const int last_strip = min(nstrips, first_strip + strips_per_cta);
  for (int strip = first_strip; strip < last_strip; ++strip) {
    const int base = strip * kStripRows;
    if (base >= t) break;  // uniform per CTA
    int* const my_progress = progress + static_cast<int64_t>(b) * nstrips + strip;
    if (threadIdx.x < kWarps) {
      published[threadIdx.x] = 0;
      consumed[threadIdx.x] = 0;
    }
    __syncthreads();
    const int r0 = base + warp * kWarpRows;
    if (r0 < t) {
      const int r = r0 + lane;
      const bool has_next = warp + 1 < kWarps && r0 + kWarpRows < t;
      const float* above =
          warp == 0 && base > 0 ? item + static_cast<int64_t>(base - 1) * pitch : nullptr;
      const bool publish_down = warp == kWarps - 1 && base + kStripRows < t;
      float prev[R];  // Q[r + 32m][j-1]
#pragma unroll
      for (int m = 0; m < R; ++m) prev[m] = 0.f;
      float prev_above = mnv;          // lane 0: Q[r0-1][j-1]
#pragma unroll 1
      for (int c = 0; c < kBufs - 1; ++c) {
        if (c < ntiles) prefetch_tile<kWarpRows>(buf(c), item, pitch, r0, c * kTile, t, s, lane);
        cp_async_commit();
      }
      for (int c = 0; c < ntiles; ++c) {
        const int j0 = c * kTile;
        // the buffer of tile c+2 was drained by tile c-1's stores (synced below)
        if (c + kBufs - 1 < ntiles)
          prefetch_tile<kWarpRows>(buf(c + kBufs - 1), item, pitch, r0, j0 + (kBufs - 1) * kTile, t, s, lane);
        cp_async_commit();
        // lane k: Q[r0-1][j0+k] (row 0 has the sentinel above it)
        float bnd = mnv;
        if (warp > 0) {
          if (lane == 0)
            while (published[warp - 1] <= c) __nanosleep(32);
          __syncwarp();
          __threadfence_block();
          bnd = ring[warp - 1][c % kRing][lane];
          __syncwarp();
          if (lane == 0) consumed[warp] = c + 1;
        } else if (above) {
          // the strip above publishes tile c after its last row is stored
          // relaxed polling (an acquire load per poll invalidates L1), one
          // acquire fence once the count is seen
          if (lane == 0) {
            if (ld_relaxed(my_progress - 1) <= c) {
              while (ld_relaxed(my_progress - 1) <= c) __nanosleep(64);
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
          }
          __syncwarp();
          bnd = j0 + lane < s ? __ldcg(above + j0 + lane) : 0.f;
        }
        cp_async_wait<kBufs - 1>();
        __syncwarp();
        float(*tile)[kTile + 1] = buf(c);
        float v[R][kTile];
#pragma unroll
        for (int m = 0; m < R; ++m)
#pragma unroll
          for (int k = 0; k < kTile; ++k) v[m][k] = tile[lane + 32 * m][k];
#pragma unroll
        for (int k = 0; k < kTile; ++k) {
          const int j = j0 + k;
          // row r + 32m's upper neighbour is lane l-1's row m, except lane
          // 0's, which is lane 31's row m-1 (or the row above the block)
          float up[R];
          up[0] = __shfl_up_sync(0xffffffffu, prev[0], 1);
#pragma unroll
          for (int m = 1; m < R; ++m)
            up[m] = __shfl_sync(0xffffffffu, lane == 31 ? prev[m - 1] : prev[m], (lane + 31) & 31);
          const float b_prev = __shfl_sync(0xffffffffu, bnd, (k + 31) & 31);
          if (lane == 0) up[0] = k == 0 ? prev_above : b_prev;
#pragma unroll
          for (int m = 0; m < R; ++m) {
            float n;
            const int row = r + 32 * m;
            if (MODE == 0) {
              if (j == 0)
                n = row == 0 ? v[m][k] : mnv;
              else
                n = v[m][k] + ref_max(up[m], prev[m]);
            } else {
              if (row == 0)
                n = (j == 0 ? 0.f : prev[m]) + v[m][k];  // run += q[0][j]
              else if (j < row)
                n = mnv;
              else
                n = ref_max(up[m], prev[m]) + v[m][k];
            }
            v[m][k] = n;
            prev[m] = n;
          }
        }
        prev_above = __shfl_sync(0xffffffffu, bnd, 31);
        // hand the last row to the next warp before writing the tile back
        if (has_next && lane == 31) {
          while (consumed[warp + 1] + kRing <= c) __nanosleep(32);
          float* slot = ring[warp][c % kRing];
#pragma unroll
          for (int k = 0; k < kTile; ++k) slot[k] = v[R - 1][k];
          __threadfence_block();
          published[warp] = c + 1;
        }
#pragma unroll
        for (int m = 0; m < R; ++m)
#pragma unroll
          for (int k = 0; k < kTile; ++k) tile[lane + 32 * m][k] = v[m][k];
        __syncwarp();
        const bool col_ok = j0 + lane < s;
#pragma unroll 16
        for (int i = 0; i < kWarpRows; ++i)
          if (col_ok && r0 + i < t) item[static_cast<int64_t>(r0 + i) * pitch + j0 + lane] = tile[i][lane];
        __syncwarp();  // the buffer is refilled by the prefetch two tiles on
        if (publish_down && lane == 0 && ((c + 1) % kStripPub == 0 || c + 1 == ntiles)) {
          __threadfence();
          st_release(my_progress, c + 1);
        }
      }
      cp_async_wait<0>();
    }
    __syncthreads();
  }
}

int fail(mas_error_t* err, int status, int errc, const std::string& msg) {
  if (err) {
    std::memset(err, 0, sizeof(*err));
    err->status = status;
    err->errc = errc;
    err->item = -1;
    err->i = err->j = -1;
    std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
  }
  return status;
}

// Kernel attributes are per device: set them once on each device before its
// first launch.
cudaError_t scores_configure() {
  constexpr int kMaxDevices = 64;
  static std::once_flag once[kMaxDevices];
  static cudaError_t status[kMaxDevices];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  std::call_once(once[dev], [dev] {
    cudaError_t r = cudaSuccess;
    const void* spread[2] = {reinterpret_cast<const void*>(forward_scores_kernel<MAS_SCORES_R, 0>),
                             reinterpret_cast<const void*>(forward_scores_kernel<MAS_SCORES_R, 1>)};
    const void* dense[2] = {reinterpret_cast<const void*>(forward_scores_kernel<1, 0>),
                            reinterpret_cast<const void*>(forward_scores_kernel<1, 1>)};
    for (int m = 0; m < 2 && r == cudaSuccess; ++m) {
      r = cudaFuncSetAttribute(dense[m], cudaFuncAttributeMaxDynamicSharedMemorySize,
                               Geo<1>::kTileSmem);
      if (r == cudaSuccess)
        r = cudaFuncSetAttribute(spread[m], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kSpreadSmem);
    }
    status[dev] = r;
  });
  return status[dev];
}

int sm_count() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

void clear(mas_error_t* err) {
  if (err) {
    std::memset(err, 0, sizeof(*err));
    err->item = -1;
    err->i = err->j = -1;
  }
}

// Shape checks shared by the score-table entry points.
int check_table(int64_t row_pitch, int32_t batch, int32_t text_cap, int32_t speech_cap,
                const uint32_t* lengths, mas_error_t* err) {
  if (batch < 1 || text_cap < 1 || speech_cap < 1)
    return fail(err, MAS_E_VALIDATION, MAS_ERRC_ZERO_DIM, "batch and capacities must be at least 1");
  if (row_pitch < speech_cap)
    return fail(err, MAS_E_VALIDATION, MAS_ERRC_SHAPE_MISMATCH,
                "row pitch is smaller than the speech capacity");
  if (lengths)
    for (int32_t b = 0; b < batch; ++b)
      if (lengths[2 * b] > static_cast<uint32_t>(text_cap) ||
          lengths[2 * b + 1] > static_cast<uint32_t>(speech_cap)) {
        const int rc = fail(err, MAS_E_VALIDATION, MAS_ERRC_LENGTHS_OUT_OF_RANGE,
                            "item " + std::to_string(b) + ": lengths exceed the capacities");
        if (err) err->item = b;
        return rc;
      }
  return MAS_OK;
}

// Direction words of a score table in the backtrack kernel's layout
// (DESIGN.md 2): word m of row i holds the decisions of columns
// 32m-1 ... 32m+30, column 32m+p-1 at bit 31-p, bit(i, c) = Q[i-1][c] > Q[i][c]
// (the strict compare of backtrack.hpp:26); row 0, column -1 and cells past
// the item's lengths are 0.  One warp per (item, row, word): lane p reads
// column 32m+p-1 of rows i-1 and i (coalesced), the ballot is the word.
__global__ void scores_to_dirs_kernel(const float* __restrict__ q, int64_t pitch, int T_cap,
                                      int S_cap, const uint32_t* __restrict__ lengths, int M,
                                      int T_alloc, int B, uint32_t* __restrict__ dirs) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t total = static_cast<int64_t>(B) * M * T_alloc;
  for (int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < total;
       w += nwarps) {
    const int i = static_cast<int>(w % T_alloc);
    const int64_t bm = w / T_alloc;
    const int m = static_cast<int>(bm % M);
    const int b = static_cast<int>(bm / M);
    const int t = lengths ? static_cast<int>(lengths[2 * b]) : T_cap;
    const int s = lengths ? static_cast<int>(lengths[2 * b + 1]) : S_cap;
    const int c = 32 * m + lane - 1;
    bool bit = false;
    if (i >= 1 && i < t && c >= 0 && c < s) {
      const float* row = q + (static_cast<int64_t>(b) * T_cap + i) * pitch;
      bit = row[c - pitch] > row[c];
    }
    const uint32_t word = __brev(__ballot_sync(0xffffffffu, bit));
    if (lane == 0) dirs[w] = word;  // w = (b * M + m) * T_alloc + i
  }
}

// parallel::detail::relax_column (parallel.cpp:25-31): one thread per text lane.
__global__ void relax_column_kernel(const float* __restrict__ prev, float* __restrict__ cur,
                                    int lanes, float sentinel) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < lanes; i += gridDim.x * blockDim.x)
    cur[i] += ref_max(i == 0 ? sentinel : prev[i - 1], prev[i]);
}

// NonFinite flags of a batch (types.cpp:107-115 scan, flag only; the exact
// location comes from the locator on the error path).
__global__ void flag_nonfinite_kernel(const float* __restrict__ q, int64_t pitch, int rows_per_item,
                                      int S_cap, const uint32_t* __restrict__ lengths, int B,
                                      int* __restrict__ flags) {
  const int64_t per_item = static_cast<int64_t>(rows_per_item) * S_cap;
  const int64_t total = per_item * B;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int b = static_cast<int>(k / per_item);
    const int64_t r = k - b * per_item;
    const int i = static_cast<int>(r / S_cap), j = static_cast<int>(r % S_cap);
    if (i < static_cast<int>(lengths[2 * b]) && j < static_cast<int>(lengths[2 * b + 1]) &&
        !isfinite(q[(static_cast<int64_t>(b) * rows_per_item + i) * pitch + j]))
      flags[b] = 1;
  }
}

int forward_scores(float* d_values, int64_t row_pitch, int32_t batch, int32_t text_cap,
                   int32_t speech_cap, const uint32_t* lengths, int mode, float max_neg_val,
                   void* stream_v, mas_error_t* err) {
  clear(err);
  int rc = check_table(row_pitch, batch, text_cap, speech_cap, lengths, err);
  if (rc != MAS_OK) return rc;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  // K1 with the score export (mas_fwd4.cu OUT 1) when q's layout suits TMA
  rc = mas::forward_scores_fwd4(d_values, row_pitch, batch, text_cap, speech_cap, lengths, mode,
                                max_neg_val, stream, err);
  if (rc != MAS_E_UNSUPPORTED) return rc;
  clear(err);
  const int nstrips = (text_cap + kStripRows - 1) / kStripRows;
  // Strips run concurrently (one CTA each, handing rows down through L2)
  // while the batch alone would not fill the GPU; otherwise each CTA walks
  // its item's strips in order and the hand-downs are all local.
  const int sms = sm_count();
  const int strips_per_cta = batch >= sms ? nstrips : 1;
  const int64_t blocks = static_cast<int64_t>(batch) * ((nstrips + strips_per_cta - 1) / strips_per_cta);
  const int64_t nprogress = static_cast<int64_t>(batch) * nstrips;
  if (blocks > 0x7fffffff)
    return fail(err, MAS_E_UNSUPPORTED, -1, "forward_scores: batch x strips exceeds the grid");
  cudaError_t e = scores_configure();
  if (e != cudaSuccess)
    return fail(err, MAS_E_CUDA, -1, std::string("forward_scores: ") + cudaGetErrorString(e));
  // workspace: [B][2] uint32 lengths | ticket | progress[B * nstrips]
  const size_t len_bytes = lengths ? static_cast<size_t>(batch) * 2 * sizeof(uint32_t) : 0;
  const size_t sync_bytes = (1 + static_cast<size_t>(nprogress)) * sizeof(int);
  char* ws = nullptr;
  e = mas::pool_alloc(reinterpret_cast<void**>(&ws), len_bytes + sync_bytes, stream);
  uint32_t* d_len = lengths ? reinterpret_cast<uint32_t*>(ws) : nullptr;
  int* sync = reinterpret_cast<int*>(ws + len_bytes);
  if (e == cudaSuccess && lengths)
    e = cudaMemcpyAsync(d_len, lengths, len_bytes, cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(sync, 0, sync_bytes, stream);
  // A grid that fits the GPU once over runs R = 2 rows per lane spread one
  // CTA per SM (the shared-memory request alone keeps a second CTA off: the
  // strips are latency-bound chains, co-residency only slows them); larger
  // grids run R = 1 with three 8-warp CTAs per SM.
  if (e == cudaSuccess) {
    const unsigned g = static_cast<unsigned>(blocks);
    if (blocks <= sms) {
      auto k = mode ? forward_scores_kernel<MAS_SCORES_R, 1> : forward_scores_kernel<MAS_SCORES_R, 0>;
      k<<<g, Geo<MAS_SCORES_R>::kWarps * 32, kSpreadSmem, stream>>>(
          d_values, row_pitch, text_cap, speech_cap, d_len, max_neg_val, nstrips, strips_per_cta,
          sync, sync + 1);
    } else {
      auto k = mode ? forward_scores_kernel<1, 1> : forward_scores_kernel<1, 0>;
      k<<<g, Geo<1>::kWarps * 32, Geo<1>::kTileSmem, stream>>>(
          d_values, row_pitch, text_cap, speech_cap, d_len, max_neg_val, nstrips, strips_per_cta,
          sync, sync + 1);
    }
    e = cudaGetLastError();
  }
  if (ws) {
    const cudaError_t f = cudaFreeAsync(ws, stream);
    if (e == cudaSuccess) e = f;
  }
  if (e != cudaSuccess)
    return fail(err, MAS_E_CUDA, -1, std::string("forward_scores: ") + cudaGetErrorString(e));
  return MAS_OK;
}

}  // namespace

namespace mas {

cudaError_t launch_scores_to_dirs(const float* q, int64_t pitch, int rows_per_item, int S_cap,
                                  const uint32_t* d_lengths, int M, int T_alloc, int B,
                                  uint32_t* dirs, cudaStream_t stream) {
  const int64_t warps = static_cast<int64_t>(B) * M * T_alloc;
  const int64_t blocks = std::min<int64_t>((warps + 7) / 8, static_cast<int64_t>(sm_count()) * 16);
  scores_to_dirs_kernel<<<static_cast<unsigned>(std::max<int64_t>(blocks, 1)), 256, 0, stream>>>(
      q, pitch, rows_per_item, S_cap, d_lengths, M, T_alloc, B, dirs);
  return cudaGetLastError();
}

cudaError_t launch_flag_nonfinite(const float* q, int64_t pitch, int rows_per_item, int S_cap,
                                  const uint32_t* d_lengths, int B, int* flags,
                                  cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(flags, 0, sizeof(int) * B, stream);
  if (e != cudaSuccess) return e;
  const int64_t total = static_cast<int64_t>(B) * rows_per_item * S_cap;
  const int64_t blocks = std::min<int64_t>((total + 255) / 256, static_cast<int64_t>(sm_count()) * 16);
  flag_nonfinite_kernel<<<static_cast<unsigned>(std::max<int64_t>(blocks, 1)), 256, 0, stream>>>(
      q, pitch, rows_per_item, S_cap, d_lengths, B, flags);
  return cudaGetLastError();
}

int forward_scores_host_lengths(float* d_values, int64_t row_pitch, int32_t batch,
                                int32_t rows_per_item, int32_t speech_cap, const uint32_t* lengths,
                                float max_neg_val, cudaStream_t stream, mas_error_t* err) {
  return forward_scores(d_values, row_pitch, batch, rows_per_item, speech_cap, lengths, 0,
                        max_neg_val, stream, err);
}

}  // namespace mas

extern "C" {

int mas_forward_scores(float* d_values, int64_t row_pitch, int32_t batch, int32_t text_cap,
                       int32_t speech_cap, const uint32_t* lengths, float max_neg_val,
                       void* stream, mas_error_t* err) {
  return forward_scores(d_values, row_pitch, batch, text_cap, speech_cap, lengths, 0, max_neg_val,
                        stream, err);
}

int mas_forward_scores_ex(float* d_values, int64_t row_pitch, int32_t batch, int32_t text_cap,
                          int32_t speech_cap, const uint32_t* lengths, int32_t engine,
                          float max_neg_val, void* stream, mas_error_t* err) {
  if (engine != MAS_ENGINE_REFERENCE && engine != MAS_ENGINE_PARALLEL) {
    clear(err);
    return fail(err, MAS_E_VALIDATION, MAS_ERRC_INVALID_CONFIG, "unknown engine");
  }
  return forward_scores(d_values, row_pitch, batch, text_cap, speech_cap, lengths,
                        engine == MAS_ENGINE_REFERENCE ? 1 : 0, max_neg_val, stream, err);
}

int mas_backtrack_scores(const float* d_scores, int64_t row_pitch, int32_t batch, int32_t text_cap,
                         int32_t speech_cap, const uint32_t* lengths, int32_t* d_paths,
                         void* stream_v, mas_error_t* err) {
  clear(err);
  int rc = check_table(row_pitch, batch, text_cap, speech_cap, lengths, err);
  if (rc != MAS_OK) return rc;
  if (!d_paths) return MAS_OK;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  // The backtrack kernel's window copies need 16-byte row groups: rows per
  // item padded to a multiple of 16, windows of up to 256 rows.
  const int T_alloc = (text_cap + 15) & ~15;
  const int M = (speech_cap + 31) / 32;
  const size_t len_bytes = static_cast<size_t>(batch) * 2 * sizeof(uint32_t);
  const size_t dir_bytes = static_cast<size_t>(batch) * M * T_alloc * sizeof(uint32_t);
  std::vector<uint32_t> full;
  if (!lengths) {
    full.resize(static_cast<size_t>(batch) * 2);
    for (int32_t b = 0; b < batch; ++b) {
      full[2 * b] = static_cast<uint32_t>(text_cap);
      full[2 * b + 1] = static_cast<uint32_t>(speech_cap);
    }
    lengths = full.data();
  }
  char* ws = nullptr;
  cudaError_t e = mas::pool_alloc(reinterpret_cast<void**>(&ws), dir_bytes + len_bytes, stream);
  uint32_t* d_dirs = reinterpret_cast<uint32_t*>(ws);
  uint32_t* d_len = reinterpret_cast<uint32_t*>(ws + dir_bytes);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_len, lengths, len_bytes, cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess)
    e = mas::launch_scores_to_dirs(d_scores, row_pitch, text_cap, speech_cap, d_len, M, T_alloc,
                                   batch, d_dirs, stream);
  if (e == cudaSuccess) {
    mas::BtArgs ba = {};
    ba.b0 = 0;
    ba.lengths = d_len;
    ba.dirs = d_dirs;
    ba.path = d_paths;
    ba.B = batch;
    ba.T_cap = text_cap;
    ba.S_cap = speech_cap;
    ba.M = M;
    ba.T_alloc = T_alloc;
    ba.R = std::min(256, T_alloc);
    e = mas::launch_backtrack(ba, stream, nullptr);
  }
  if (ws) {
    const cudaError_t f = cudaFreeAsync(ws, stream);
    if (e == cudaSuccess) e = f;
  }
  if (e != cudaSuccess)
    return fail(err, MAS_E_CUDA, -1, std::string("backtrack_scores: ") + cudaGetErrorString(e));
  return MAS_OK;
}

int mas_relax_column(const float* d_prev, float* d_cur, int32_t lanes, float sentinel,
                     void* stream_v, mas_error_t* err) {
  clear(err);
  if (lanes < 1) return MAS_OK;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  const int blocks = std::min((lanes + 255) / 256, sm_count() * 8);
  relax_column_kernel<<<blocks, 256, 0, stream>>>(d_prev, d_cur, lanes, sentinel);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return fail(err, MAS_E_CUDA, -1, std::string("relax_column: ") + cudaGetErrorString(e));
  return MAS_OK;
}

}  // extern "C"
