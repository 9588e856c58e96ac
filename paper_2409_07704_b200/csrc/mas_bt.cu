// mas_bt.cu -- K2: the backtrack and output writer, plus the generator (K3)
// and the NonFinite locator.
//
// The reference walk (src/backtrack.hpp:21-32) is one serial pass per item:
//   cur = t-1; path[s-1] = cur;
//   for j = s-2..0: if (cur > 0 && Q[cur-1][j] > Q[cur][j]) --cur; path[j] = cur;
// followed by write_path (src/types.cpp:181-185) into a zeroed [T][S] byte
// matrix (types.cpp:40-47).  Here the walk reads the forward kernel's
// direction bits, bit(i, j) == (Q[i-1][j] > Q[i][j]), and is split over
// speech segments of L columns so it runs on the whole GPU:
//
//   pass 1 (bt_segmap):  for every segment k and EVERY possible entry row x,
//       G_k(x) = row of the walk at column kL when it is at row x at column
//       (k+1)L -- independent walks, one thread each, over the segment's
//       direction words staged in shared memory.  The walk jumps row to row
//       with a find-last-set-bit per 32-column word (one step per text row,
//       not per speech column).  The CTA of the item's last segment walks
//       from (t-1, s-1) instead; the last CTA of the item to finish then
//       chains P_k = G_k(P_{k+1}) down to column 0.
//   pass 2 (bt_write):  each segment re-walks from its known entry row,
//       producing path[j], and writes its [T_cap x L] slice of the output
//       with 16-byte stores (zeros everywhere but the path) plus the int32
//       path row -- so the dense output is written exactly once.
#include <cstdio>
#include <cstdlib>

#include "mas_kernels.h"

namespace mas {

namespace {

constexpr int kBtThreads = 256;

// Highest set-bit position <= p (and >= lo) in row y of the staged words,
// or -1.  Word wi of the tile holds positions (m0 + wi) * 32 + [0, 32);
// position p == column p-1 (direction words are offset by one column).
__device__ __forceinline__ int find_exit(const uint32_t* __restrict__ words, int nrows_stride, int y,
                                         int p, int lo, int m0) {
  int wi = (p >> 5) - m0;
  uint32_t w = words[wi * nrows_stride + y] & (0xffffffffu >> (31 - (p & 31)));
  const int lo_wi = (lo >> 5) - m0;
  const uint32_t lo_mask = 0xffffffffu << (lo & 31);
  if (wi == lo_wi) w &= lo_mask;
  while (w == 0u) {
    --wi;
    if (wi < lo_wi) return -1;
    w = words[wi * nrows_stride + y];
    if (wi == lo_wi) w &= lo_mask;
  }
  return (m0 + wi) * 32 + 31 - __clz(w);
}

// Walk from row y entering at position p (testing column p-1 first) down to
// position lo; returns the row at column lo-1.  Optionally records
// path[j - col0] for every column j visited.
__device__ __forceinline__ int walk(const uint32_t* __restrict__ words, int stride, int y, int p,
                                   int lo, int m0, int32_t* path, int col0) {
  while (y > 0 && p >= lo) {
    const int pe = find_exit(words, stride, y, p, lo, m0);
    if (pe < 0) break;
    if (path) {
      for (int j = p - 1; j >= pe; --j) path[j - col0] = y;  // columns pe..p-1 stay in row y
      path[pe - 1 - col0] = y - 1;
    }
    --y;
    p = pe - 1;
  }
  if (path) {
    for (int j = p - 1; j >= lo - 1; --j) path[j - col0] = y;
  }
  return y;
}

__global__ void __launch_bounds__(kBtThreads) bt_segmap_kernel(const BtArgs a, int* counters) {
  extern __shared__ uint32_t words[];  // [NW][t_b]
  __shared__ int s_last;
  const int k = blockIdx.x;
  const int b = blockIdx.y;
  const int t_b = static_cast<int>(a.lengths[2 * b]);
  const int s_b = static_cast<int>(a.lengths[2 * b + 1]);
  if (t_b <= 0 || s_b <= 0) return;
  const int Kb = (s_b + a.L - 1) / a.L;
  if (k >= Kb) return;
  const int NW = a.L / 32 + 1;
  const int m0 = (k * a.L) >> 5;

  // Stage the segment's direction words for rows [0, t_b).
  const uint32_t* src = a.dirs + static_cast<size_t>(b) * a.M * a.T_alloc;
  const int nw_avail = (a.M - m0) < NW ? (a.M - m0) : NW;
  for (int idx = threadIdx.x; idx < NW * t_b; idx += blockDim.x) {
    const int wi = idx / t_b;
    const int y = idx - wi * t_b;
    words[idx] = wi < nw_avail ? __ldcg(src + static_cast<size_t>(m0 + wi) * a.T_alloc + y) : 0u;
  }
  __syncthreads();

  const int lo = k * a.L + 1;  // column kL
  int32_t* segrow = a.seg_row + static_cast<size_t>(b) * (a.Kseg + 1);
  if (k < Kb - 1) {
    int32_t* map = a.seg_map + (static_cast<size_t>(b) * a.Kseg + k) * a.T_alloc;
    const int p_in = (k + 1) * a.L;  // column (k+1)L - 1
    for (int x = threadIdx.x; x < t_b; x += blockDim.x) {
      map[x] = walk(words, t_b, x, p_in, lo, m0, nullptr, 0);
    }
  } else if (threadIdx.x == 0) {
    // Last segment: path[s-1] = t-1 (backtrack.hpp:23-24).
    segrow[Kb] = t_b - 1;
    segrow[Kb - 1] = s_b >= 2 ? walk(words, t_b, t_b - 1, s_b - 1, lo, m0, nullptr, 0) : t_b - 1;
  }

  // The last CTA of this item to finish chains the maps down to column 0.
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const int old = atomicAdd(counters + b, 1);
    s_last = old == Kb - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    int P = __ldcg(segrow + (Kb - 1));
    for (int kk = Kb - 2; kk >= 0; --kk) {
      P = __ldcg(a.seg_map + (static_cast<size_t>(b) * a.Kseg + kk) * a.T_alloc + P);
      segrow[kk] = P;
    }
    counters[b] = 0;  // ready for the next call (stream-ordered)
  }
}

template <int VEC>
__device__ __forceinline__ void store_chunk(uint8_t* dst, const uint8_t* v);

template <>
__device__ __forceinline__ void store_chunk<16>(uint8_t* dst, const uint8_t* v) {
  *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(v);
}
template <>
__device__ __forceinline__ void store_chunk<4>(uint8_t* dst, const uint8_t* v) {
  *reinterpret_cast<uint32_t*>(dst) = *reinterpret_cast<const uint32_t*>(v);
}
template <>
__device__ __forceinline__ void store_chunk<1>(uint8_t* dst, const uint8_t* v) {
  *dst = *v;
}

template <int VEC>
__global__ void __launch_bounds__(kBtThreads) bt_write_kernel(const BtArgs a) {
  extern __shared__ uint32_t dyn[];
  __shared__ int s_rlo, s_rhi;
  const int k = blockIdx.x;
  const int b = blockIdx.y;
  const int t_b = static_cast<int>(a.lengths[2 * b]);
  const int s_b = static_cast<int>(a.lengths[2 * b + 1]);
  const int c0 = k * a.L;
  const int ncols = (a.S_cap - c0) < a.L ? (a.S_cap - c0) : a.L;
  int32_t* path = reinterpret_cast<int32_t*>(dyn);  // [L]
  uint32_t* words = dyn + a.L;                      // [NW][rows]
  const bool active = t_b > 0 && s_b > 0 && c0 < s_b;

  if (threadIdx.x == 0) {
    s_rlo = 1;
    s_rhi = 0;
  }
  for (int j = threadIdx.x; j < a.L; j += blockDim.x) path[j] = -1;
  __syncthreads();

  if (active) {
    const int Kb = (s_b + a.L - 1) / a.L;
    const int32_t* segrow = a.seg_row + static_cast<size_t>(b) * (a.Kseg + 1);
    const int r_hi = __ldcg(segrow + k + 1);  // row at column (k+1)L, or t-1 at s-1
    const int r_lo = __ldcg(segrow + k);      // row at column kL
    const int nrows = r_hi - r_lo + 1;
    const int NW = a.L / 32 + 1;
    const int m0 = c0 >> 5;
    const int nw_avail = (a.M - m0) < NW ? (a.M - m0) : NW;
    const uint32_t* src = a.dirs + static_cast<size_t>(b) * a.M * a.T_alloc;
    for (int idx = threadIdx.x; idx < NW * nrows; idx += blockDim.x) {
      const int wi = idx / nrows;
      const int y = idx - wi * nrows;
      words[idx] =
          wi < nw_avail ? __ldcg(src + static_cast<size_t>(m0 + wi) * a.T_alloc + r_lo + y) : 0u;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // Walk in tile-local row coordinates (row r_lo maps to 0).  The walk
      // never leaves [r_lo, r_hi]: the pass-1 maps said it ends at r_lo.
      const bool last = k == Kb - 1;
      const int p_in = last ? s_b - 1 : (k + 1) * a.L;
      const int lo = c0 + 1;
      if (last) path[s_b - 1 - c0] = r_hi - r_lo;
      walk(words, nrows, r_hi - r_lo, p_in, lo, m0, path, c0);
      // Shift back to absolute rows (walk leaves row 0 == r_lo untouched: y > 0 check
      // is relative; rows below r_lo are never needed since the walk ends at r_lo).
      s_rlo = r_lo;
      s_rhi = r_hi;
    }
    __syncthreads();
    const int last_col = (s_b - c0) < a.L ? (s_b - c0) : a.L;
    for (int j = threadIdx.x; j < last_col; j += blockDim.x) path[j] += s_rlo;
    __syncthreads();
  }

  // paths row
  if (a.paths) {
    int32_t* prow = a.paths + static_cast<size_t>(b) * a.S_cap + c0;
    for (int j = threadIdx.x; j < ncols; j += blockDim.x) prow[j] = path[j];
  }
  // dense output slice [T_cap][ncols]
  if (a.out) {
    const int rlo = s_rlo, rhi = s_rhi;
    const int nchunk = (ncols + VEC - 1) / VEC;
    uint8_t* base = a.out + static_cast<size_t>(b) * a.T_cap * a.S_cap + c0;
    for (int idx = threadIdx.x; idx < a.T_cap * nchunk; idx += blockDim.x) {
      const int i = idx / nchunk;
      const int ch = idx - i * nchunk;
      alignas(16) uint8_t v[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) v[e] = 0;
      if (i >= rlo && i <= rhi) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
          const int j = ch * VEC + e;
          v[e] = (j < ncols && path[j] == i) ? 1 : 0;
        }
      }
      store_chunk<VEC>(base + static_cast<size_t>(i) * a.S_cap + ch * VEC, v);
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
  int32_t* prow = a.paths ? a.paths + static_cast<size_t>(b) * a.S_cap : nullptr;
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
  int n = 0;
  if (serial) {
    if (a.out) {
      cudaError_t e = cudaMemsetAsync(a.out, 0, static_cast<size_t>(a.B) * a.T_cap * a.S_cap, stream);
      if (e != cudaSuccess) return e;
    }
    if (a.paths) {
      fill_paths_kernel<<<grid_for(static_cast<size_t>(a.B) * a.S_cap, 256), 256, 0, stream>>>(
          a.paths, static_cast<size_t>(a.B) * a.S_cap);
      ++n;
    }
    bt_serial_kernel<<<(a.B + 63) / 64, 64, 0, stream>>>(a);
    ++n;
    if (launches) *launches = n;
    return cudaGetLastError();
  }
  const int NW = a.L / 32 + 1;
  // counters live right after seg_row's [B][Kseg+1] block (see mas_abi.cu).
  int* counters = reinterpret_cast<int*>(a.seg_row + static_cast<size_t>(a.B) * (a.Kseg + 1));
  const size_t smem1 = static_cast<size_t>(NW) * a.T_alloc * 4;
  bt_segmap_kernel<<<dim3(a.Kseg, a.B), kBtThreads, smem1, stream>>>(a, counters);
  ++n;
  const size_t smem2 = static_cast<size_t>(a.L) * 4 + static_cast<size_t>(NW) * (a.L + 1) * 4;
  const dim3 grid2(a.Kseg, a.B);
  if (a.S_cap % 16 == 0)
    bt_write_kernel<16><<<grid2, kBtThreads, smem2, stream>>>(a);
  else if (a.S_cap % 4 == 0)
    bt_write_kernel<4><<<grid2, kBtThreads, smem2, stream>>>(a);
  else
    bt_write_kernel<1><<<grid2, kBtThreads, smem2, stream>>>(a);
  ++n;
  if (launches) *launches = n;
  return cudaGetLastError();
}

cudaError_t bt_configure(int T_alloc, int L) {
  const int NW = L / 32 + 1;
  const int smem1 = NW * T_alloc * 4;
  cudaError_t e = cudaFuncSetAttribute(bt_segmap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem1 > 48 * 1024 ? smem1 : 48 * 1024);
  if (e != cudaSuccess) return e;
  const int smem2 = L * 4 + NW * (L + 1) * 4;
  const int s2 = smem2 > 48 * 1024 ? smem2 : 48 * 1024;
  e = cudaFuncSetAttribute(bt_write_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(bt_write_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(bt_write_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, s2);
}

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
