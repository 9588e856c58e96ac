// mas_bt.cu -- K2: the backtrack, plus the generator (K3) and the NonFinite
// locator.
//
// The reference walk (src/backtrack.hpp:21-32) is one serial pass per item:
//   cur = t-1; path[s-1] = cur;
//   for j = s-2..0: if (cur > 0 && Q[cur-1][j] > Q[cur][j]) --cur; path[j] = cur;
// followed by write_path (src/types.cpp:181-185) into a zeroed [T][S] byte
// matrix (types.cpp:40-47).  Here the walk reads the forward kernel's
// direction bits, bit(i, j) == (Q[i-1][j] > Q[i][j]), stored as one u32 per
// row per 32 columns (word m of row i holds columns 32m-1 .. 32m+30).  The
// zero fill of the output happens in the forward kernel (or a memset for
// ragged shapes), so this kernel only walks and scatters the ones:
//
//   one warp per item walks row to row rather than column to column --
//   inside a 32-column word the next step down is a find-last-set-bit, so
//   an item costs ~(t + s/32) dependent steps instead of s.  The window of
//   direction words the walk can reach in a block (at most 32 rows per
//   block) is prefetched kWinStages blocks ahead with cp.async; lane 0 walks
//   with a one-row load lookahead; each finished 32-column block is expanded
//   by the whole warp (popc of the exit mask) into path[] and the ones of
//   the alignment matrix.
#include <cstdio>
#include <cstdlib>

#include "mas_kernels.h"

namespace mas {

namespace {

constexpr int kWinStages = 8;                      // blocks prefetched ahead
constexpr int kWinWords = 9;                       // words per lane per stage
constexpr int kWinRows = 32 * kWinWords;           // >= 32 * kWinStages + 1 rows

__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Prefetch block m's direction words for rows [base - kWinRows + 1, base]
// into stage `st`: lane l copies rows base - l - 32 i.
__device__ __forceinline__ void prefetch_window(uint32_t win_smem, int st, const uint32_t* src,
                                                int T_alloc, int m, int base, int lane) {
  if (m >= 0) {
    const uint32_t* col = src + static_cast<size_t>(m) * T_alloc;
#pragma unroll
    for (int i = 0; i < kWinWords; ++i) {
      const int idx = lane + 32 * i;
      const int row = base - idx;
      cp_async4(win_smem + static_cast<uint32_t>((st * kWinRows + idx) * 4),
                col + (row >= 0 ? row : 0), row >= 0);
    }
  }
  cp_async_commit();
}

__global__ void __launch_bounds__(32) bt_walk_kernel(const BtArgs a) {
  __shared__ uint32_t win[kWinStages * kWinRows];
  const int b = blockIdx.x;
  const int lane = threadIdx.x;
  const int t = static_cast<int>(a.lengths[2 * b]);
  const int s = static_cast<int>(a.lengths[2 * b + 1]);
  int32_t* path = a.path ? a.path + static_cast<size_t>(b) * a.S_cap : nullptr;
  uint8_t* out = a.out ? a.out + static_cast<size_t>(b) * a.T_cap * a.S_cap : nullptr;
  if (path)
    for (int j = (s > 0 ? s : 0) + lane; j < a.S_cap; j += 32) path[j] = -1;
  if (t <= 0 || s <= 0) return;
  const uint32_t* src = a.dirs + static_cast<size_t>(b) * a.M * a.T_alloc;
  const uint32_t win_smem = static_cast<uint32_t>(__cvta_generic_to_shared(win));

  int cur = t - 1;
  if (lane == 0) {  // backtrack.hpp:23-24
    if (path) path[s - 1] = cur;
    if (out) out[static_cast<size_t>(cur) * a.S_cap + s - 1] = 1;
  }
  // Column j's bit sits at position p = j + 1; the walk covers p = s-1 .. 1.
  const int mtop = (s - 1) >> 5;
  int base[kWinStages];
#pragma unroll
  for (int i = 0; i < kWinStages; ++i) {
    base[i] = cur;
    prefetch_window(win_smem, (mtop - i) & (kWinStages - 1), src, a.T_alloc, mtop - i, cur, lane);
  }
  for (int m = mtop; m >= 0; --m) {
    const int st = m & (kWinStages - 1);
    cp_async_wait<kWinStages - 1>();
    __syncwarp();
    const int wb = base[0];
    const int p_top = (m == mtop) ? ((s - 1) & 31) : 31;
    const int p_min = (m == 0) ? 1 : 0;
    uint32_t ex = 0;
    int y = cur;
    if (lane == 0 && y > 0 && p_top >= p_min) {
      const uint32_t* w_st = win + st * kWinRows + wb;  // row y at w_st[-y]
      const uint32_t lo_mask = (m == 0) ? ~1u : ~0u;
      int p = p_top;
      uint32_t w = w_st[-y];
      while (true) {
        const uint32_t w_next = w_st[-(y - 1)];  // lookahead: the next row is always y-1
        const uint32_t hit = w & lo_mask & (0xffffffffu >> (31 - p));
        if (hit == 0u) break;
        const int e = 31 - __clz(hit);
        ex |= 1u << e;
        --y;
        p = e - 1;
        if (y == 0 || p < p_min) break;
        w = w_next;
      }
    }
    ex = __shfl_sync(0xffffffffu, ex, 0);
    const int cur_top = cur;
    cur = __shfl_sync(0xffffffffu, y, 0);
#pragma unroll
    for (int i = 0; i < kWinStages - 1; ++i) base[i] = base[i + 1];
    base[kWinStages - 1] = cur;
    __syncwarp();
    prefetch_window(win_smem, st, src, a.T_alloc, m - kWinStages, cur, lane);
    // Expand the block: column 32m + u - 1 (position u) sits at row
    // cur_top - #exits at positions >= u.
    const int u = lane;
    if (u >= p_min && u <= p_top) {
      const int col = 32 * m + u - 1;
      const int row = cur_top - __popc(ex >> u);
      if (path) path[col] = row;
      if (out) out[static_cast<size_t>(row) * a.S_cap + col] = 1;
    }
  }
}

// Reference-order serial walk, one thread per item -- kept as a
// cross-check (MAS_BT_SERIAL=1) for the segmented kernels.
__global__ void bt_serial_kernel(const BtArgs a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.B) return;
  const int t = static_cast<int>(a.lengths[2 * b]);
  const int s = static_cast<int>(a.lengths[2 * b + 1]);
  if (t <= 0 || s <= 0) return;
  const uint32_t* src = a.dirs + static_cast<size_t>(b) * a.M * a.T_alloc;
  uint8_t* out = a.out ? a.out + static_cast<size_t>(b) * a.T_cap * a.S_cap : nullptr;
  int32_t* prow = a.path ? a.path + static_cast<size_t>(b) * a.S_cap : nullptr;
  int cur = t - 1;
  if (out) out[static_cast<size_t>(cur) * a.S_cap + s - 1] = 1;
  if (prow) prow[s - 1] = cur;
  for (int j = s - 2; j >= 0; --j) {
    if (cur > 0) {
      const int p = j + 1;
      const uint32_t w = src[static_cast<size_t>(p >> 5) * a.T_alloc + cur];
      if ((w >> (p & 31)) & 1u) --cur;
    }
    if (out) out[static_cast<size_t>(cur) * a.S_cap + j] = 1;
    if (prow) prow[j] = cur;
  }
}

__global__ void fill_paths_kernel(int32_t* paths, size_t n) {
  if (!paths) return;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    paths[i] = -1;
}

// Exact NonFinite locator (error path only): lowest row-major (i, j) in the
// valid region of item b (types.cpp:107-115), as i * s + j via atomicMin.
__global__ void locate_nonfinite_kernel(const float* q, int64_t row_pitch, int T_pad, int b, int t,
                                        int s, unsigned long long* result) {
  const size_t total = static_cast<size_t>(t) * s;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t i = idx / s;
    const size_t j = idx - i * s;
    const float v = q[(static_cast<size_t>(b) * T_pad + i) * row_pitch + j];
    if (!isfinite(v)) atomicMin(result, static_cast<unsigned long long>(idx));
  }
}

// K3: bench::generate_random_batch (bench.cpp:164-180), counter-addressed:
// element n of the stream is fin(s0 + (n+1) * phi) (bench.hpp:79-91).  The
// affine map uses explicit round-to-nearest double ops (the CPU build has
// no FMA contraction).
__global__ void generate_kernel(uint64_t s0, int64_t first_elem, int B, int T, int S, int64_t pitch,
                                float* out) {
  const size_t total = static_cast<size_t>(B) * T * S;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const uint64_t n = static_cast<uint64_t>(first_elem) + idx;
    uint64_t z = s0 + (n + 1ull) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z = z ^ (z >> 31);
    const double u = __dmul_rn(static_cast<double>(z >> 11), 0x1.0p-53);
    const float v = __double2float_rn(__dadd_rn(-5.0, __dmul_rn(10.0, u)));
    const size_t ts = static_cast<size_t>(T) * S;
    const size_t bb = idx / ts;
    const size_t r = idx - bb * ts;
    const size_t i = r / S;
    const size_t j = r - i * S;
    out[(bb * T + i) * pitch + j] = v;
  }
}

int grid_for(size_t n, int threads) {
  size_t g = (n + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

}  // namespace

cudaError_t launch_backtrack(const BtArgs& a, cudaStream_t stream, int* launches) {
  static const bool serial = [] {
    const char* e = std::getenv("MAS_BT_SERIAL");
    return e && e[0] == '1';
  }();
  if (serial) {
    fill_paths_kernel<<<grid_for(static_cast<size_t>(a.B) * a.S_cap, 256), 256, 0, stream>>>(
        a.path, static_cast<size_t>(a.B) * a.S_cap);
    bt_serial_kernel<<<(a.B + 63) / 64, 64, 0, stream>>>(a);
    if (launches) *launches = 2;
    return cudaGetLastError();
  }
  bt_walk_kernel<<<a.B, 32, 0, stream>>>(a);
  if (launches) *launches = 1;
  return cudaGetLastError();
}

cudaError_t bt_configure(int /*T_alloc*/, int /*L*/) { return cudaSuccess; }

cudaError_t launch_locate_nonfinite(const float* q, int64_t row_pitch, int T_pad, int b, int t,
                                    int s, unsigned long long* d_result, cudaStream_t stream) {
  const size_t total = static_cast<size_t>(t) * s;
  locate_nonfinite_kernel<<<grid_for(total, 256), 256, 0, stream>>>(q, row_pitch, T_pad, b, t, s,
                                                                   d_result);
  return cudaGetLastError();
}

cudaError_t launch_generate(uint64_t s0, int64_t first_elem, int B, int T, int S, int64_t pitch,
                            float* out, cudaStream_t stream) {
  const size_t total = static_cast<size_t>(B) * T * S;
  generate_kernel<<<grid_for(total, 256), 256, 0, stream>>>(s0, first_elem, B, T, S, pitch, out);
  return cudaGetLastError();
}

}  // namespace mas
