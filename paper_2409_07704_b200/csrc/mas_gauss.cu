// mas_gauss.cu -- the log-likelihood q of the Glow-TTS / VITS prior
// (SURVEY.md 8(f) rank 2), on the tensor cores:
//
//   q[b][i][j] = sum_c log N(z[b][c][j]; mean[b][c][i], exp(logstd[b][c][i]))
//              = sum_k A[b][i][k] * B[b][k][j] + bias[b][i]
//
//   A[i][c]     = -0.5 exp(-2 logstd[c][i])           B[c][j]     = z[c][j]^2
//   A[i][C + c] = mean[c][i] exp(-2 logstd[c][i])     B[C + c][j] = z[c][j]
//   bias[i]     = sum_c (-0.5 log(2 pi) - logstd[c][i] - 0.5 mean[c][i]^2 exp(-2 logstd[c][i]))
//
// (the expanded form Glow-TTS computes with two matmuls), A and B in bf16,
// accumulated in fp32 by tcgen05.mma: D[128 rows x 32 frames] per MMA group,
// A resident in TMEM, B streamed through shared memory by TMA.
//
//   K4a gauss_prep_kernel  A, B (bf16, K padded to Kp = 64 * ceil(2C / 64))
//                          and bias (fp32) from z, mean, logstd
//   K4b gauss_q_kernel     q itself, written to HBM (the unfused path, and
//                          the reference the fused K1 is checked against)
//   K1g (mas_fwd4.cu)      the same MMAs feeding the DP's shared-memory
//                          ring directly: q never reaches HBM
//
// K4b and K1g issue the same MMA sequence (M = 128, N = 32, K in steps of 16,
// same descriptors) and the same bias addition, so their q values are
// identical bit for bit.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "mas_kernels.h"
#include "mas_ptx.cuh"
#include "mas_umma.cuh"
#include "monoalign_b200.h"

namespace mas {

namespace {

// ---- K4a: operands -----------------------------------------------------------
// A block stages 32 text rows (or frames) of every channel in shared memory
// (reads coalesced along the row / frame index of mean, logstd, z) and then
// writes the 32 K-major rows of Kp bf16 as consecutive 32-bit pairs
// (coalesced: the 32 rows are one contiguous 32 x Kp block).
constexpr int kPrepRows = 32;

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&p);
}

__global__ void __launch_bounds__(256) gauss_prep_rows_kernel(
    const float* __restrict__ mean, const float* __restrict__ logstd, int B, int C, int T, int Tp,
    int Kp, __nv_bfloat16* __restrict__ A, float* __restrict__ bias) {
  extern __shared__ float sm[];  // [kPrepRows][2C + 1]: -0.5 e^{-2ls}, m e^{-2ls}
  __shared__ float sbias[8][kPrepRows];
  const int ld = 2 * C + 1;  // odd row stride: conflict-free in both phases
  const int blocks_per_item = Tp / kPrepRows;
  const int b = blockIdx.x / blocks_per_item, i0 = blockIdx.x % blocks_per_item * kPrepRows;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float acc = 0.f;
  for (int c = wid; c < C; c += 8) {
    const int i = i0 + lane;
    float lo = 0.f, hi = 0.f;
    if (i < T) {
      const int64_t x = (static_cast<int64_t>(b) * C + c) * T + i;
      const float ls = logstd[x], m = mean[x];
      const float inv_var = expf(-2.f * ls);
      lo = -0.5f * inv_var;
      hi = m * inv_var;
      acc += -0.91893853320467274f - ls - 0.5f * m * m * inv_var;  // -0.5 log(2 pi)
    }
    sm[lane * ld + c] = lo;
    sm[lane * ld + C + c] = hi;
  }
  sbias[wid][lane] = acc;
  __syncthreads();
  if (threadIdx.x < kPrepRows) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += sbias[w][threadIdx.x];
    bias[static_cast<int64_t>(b) * Tp + i0 + threadIdx.x] = t;
  }
  // warp wid writes rows wid, wid + 8, ...: lanes cover a row's Kp/2 words
  uint32_t* out = reinterpret_cast<uint32_t*>(A + (static_cast<int64_t>(b) * Tp + i0) * Kp);
  for (int r = wid; r < kPrepRows; r += 8)
    for (int kw = lane; kw < Kp / 2; kw += 32) {
      const int k = 2 * kw;
      const float v0 = k < 2 * C ? sm[r * ld + k] : 0.f;
      const float v1 = k + 1 < 2 * C ? sm[r * ld + k + 1] : 0.f;
      out[r * (Kp / 2) + kw] = pack_bf16x2(v0, v1);
    }
}

// 64 frames per block: each warp loads its channels' 64 frames as float2
// per lane (256-byte segments, every load of the thread issued before the
// first shared store), the block transposes through shared memory (row
// stride C + 1), and writes its 64 K-major rows as 16-byte vectors of eight
// bf16 (the 64 x Kp block is contiguous).
constexpr int kPrepFrames = 64;
constexpr int kPrepPer = (kGaussMaxChannels + 7) / 8;  // channels per warp, at most
__global__ void __launch_bounds__(256) gauss_prep_frames_kernel(const float* __restrict__ z, int B,
                                                                 int C, int S, int Sp, int Kp,
                                                                 __nv_bfloat16* __restrict__ Bm) {
  extern __shared__ float sm[];  // [kPrepFrames][C + 1] z
  const int ld = C + 1;
  const int blocks_per_item = Sp / kPrepFrames;
  const int b = blockIdx.x / blocks_per_item, j0 = blockIdx.x % blocks_per_item * kPrepFrames;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int j = j0 + 2 * lane;  // this lane's two frames
  float2 zv[kPrepPer];
#pragma unroll
  for (int u = 0; u < kPrepPer; ++u) {
    const int c = wid + 8 * u;
    zv[u] = make_float2(0.f, 0.f);
    if (c < C) {
      const float* row = z + (static_cast<int64_t>(b) * C + c) * S;
      if (j + 1 < S && (S & 1) == 0)
        zv[u] = __ldg(reinterpret_cast<const float2*>(row + j));
      else
        zv[u] = make_float2(j < S ? __ldg(row + j) : 0.f, j + 1 < S ? __ldg(row + j + 1) : 0.f);
    }
  }
#pragma unroll
  for (int u = 0; u < kPrepPer; ++u) {
    const int c = wid + 8 * u;
    if (c < C) {
      sm[(2 * lane) * ld + c] = zv[u].x;
      sm[(2 * lane + 1) * ld + c] = zv[u].y;
    }
  }
  __syncthreads();
  // row r (frame j0 + r), 16-byte vector v: K indices 8v .. 8v + 7 (z^2 rows
  // first, then z, zero past 2C)
  uint4* out = reinterpret_cast<uint4*>(Bm + (static_cast<int64_t>(b) * Sp + j0) * Kp);
  const int vec_per_row = Kp / 8;
  for (int e = threadIdx.x; e < kPrepFrames * vec_per_row; e += blockDim.x) {
    const int r = e / vec_per_row, v = e - r * vec_per_row;
    uint32_t w[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      float x[2];
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int kk = 8 * v + 2 * h + q;
        const float zz = kk < 2 * C ? sm[r * ld + (kk < C ? kk : kk - C)] : 0.f;
        x[q] = kk < C ? zz * zz : zz;
      }
      w[h] = pack_bf16x2(x[0], x[1]);
    }
    out[e] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// ---- K4b: q to HBM -----------------------------------------------------------
constexpr int kQStages = 4;       // B stages in flight
constexpr int kQColsPerCta = 1024;
constexpr int kQThreads = 6 * 32;  // TMA warp, MMA warp, 4 epilogue warps

struct QArgs {
  const __nv_bfloat16* A;  // [B][Tp][Kp]
  const float* bias;       // [B][Tp]
  float* q;                // [B][T][pitch]
  int64_t pitch;
  int B, T, S, Tp, Sp, Kp;
  int tmem_cols;
};

// Epilogue staging per warp: two [32 rows][32 frames] fp32 tiles (128-byte
// swizzle), each written out by one TMA store {32, 32, 1} of the 3-D q map
// {S, T, B} (clipped per item at T and S).
constexpr uint32_t kQStage = 32 * 32 * 4;

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int c0, int c1,
                                             int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(src), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(kQThreads, 1)
    gauss_q_kernel(const __grid_constant__ CUtensorMap tmb, const __grid_constant__ CUtensorMap tmq,
                   const QArgs a) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment for the swizzled B atoms
  const uint32_t raw = smem_addr(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* const sbase = smem_raw + (base - raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int Kp = a.Kp;
  const uint32_t stage_bytes = static_cast<uint32_t>((Kp / umma::kAtomK) * umma::kAtomBytes);
  const uint32_t bars = base + kQStages * stage_bytes;  // zfull[S] zfree[S] dfull[2] dempty[2]
  const uint32_t zfull = bars, zfree = bars + 8u * kQStages;
  const uint32_t dfull = zfree + 8u * kQStages, dempty = dfull + 16u;
  volatile uint32_t* tmem_slot = reinterpret_cast<volatile uint32_t*>(sbase + kQStages * stage_bytes + 8 * (2 * kQStages + 4));
  const uint32_t qstage = base + kQStages * stage_bytes + 1024;  // [4 warps][2][kQStage]

  const int tiles_t = a.Tp / umma::kM;
  const int cblocks = (a.Sp + kQColsPerCta - 1) / kQColsPerCta;
  const int b = blockIdx.x / (tiles_t * cblocks);
  const int tr = (blockIdx.x / cblocks) % tiles_t;
  const int cb = blockIdx.x % cblocks;
  const int c0 = cb * kQColsPerCta;
  const int nst = min(kQColsPerCta, a.Sp - c0) / umma::kN;
  const uint32_t colA = 0, colD = static_cast<uint32_t>(Kp / 2);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kQStages; ++s) {
      mbar_init(zfull + 8u * s, 1u);
      mbar_init(zfree + 8u * s, 1u);
    }
    for (int d = 0; d < 2; ++d) {
      mbar_init(dfull + 8u * d, 1u);
      mbar_init(dempty + 8u * d, 4u);
    }
    fence_mbar_init();
  }
  if (warp == 2) umma::tmem_alloc(smem_addr(const_cast<uint32_t*>(tmem_slot)), a.tmem_cols);
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 2) {
    // A rows of this tile into TMEM: the warp of sub-partition qd owns TMEM
    // lanes 32 qd .. 32 qd + 31 = rows 32 qd + lane.
    const int qd = warp & 3;
    const int row = tr * umma::kM + 32 * qd + lane;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.A + (static_cast<int64_t>(b) * a.Tp + row) * Kp);
    for (int c = 0; c < Kp / 2; c += 8) {
      uint32_t v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = src[c + e];
      umma::tmem_st8(tmem + (static_cast<uint32_t>(32 * qd) << 16) + colA + static_cast<uint32_t>(c), v);
    }
    umma::tmem_wait_st();
  }
  umma::fence_before_sync();
  __syncthreads();
  umma::fence_after_sync();

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA: B stages
      prefetch_tensormap(&tmb);
      for (int m = 0; m < nst; ++m) {
        const int s = m % kQStages;
        if (m >= kQStages) mbar_wait(zfree + 8u * s, ((m / kQStages) & 1u) ^ 1u);
        mbar_arrive_expect_tx(zfull + 8u * s, stage_bytes);
        for (int at = 0; at < Kp / umma::kAtomK; ++at)
          tma_load_2d(base + s * stage_bytes + at * umma::kAtomBytes, &tmb, at * umma::kAtomK,
                      b * a.Sp + c0 + m * umma::kN, zfull + 8u * s, policy_evict_first());
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issue
      const uint32_t idesc = umma::idesc_bf16_f32(umma::kM, umma::kN);
      for (int m = 0; m < nst; ++m) {
        const int s = m % kQStages, d = m & 1;
        mbar_wait(zfull + 8u * s, (m / kQStages) & 1u);
        if (m >= 2) mbar_wait(dempty + 8u * d, ((m / 2) & 1u) ^ 1u);
        umma::fence_after_sync();
        umma::mma_tile(tmem + colD + static_cast<uint32_t>(d * umma::kN), tmem + colA,
                       base + s * stage_bytes, Kp, idesc);
        umma::mma_commit(zfree + 8u * s);
        umma::mma_commit(dfull + 8u * d);
      }
    }
  } else {  // ---- epilogue: TMEM -> +bias -> swizzled smem tile -> TMA store
    const int qd = warp & 3;
    const int i = tr * umma::kM + 32 * qd + lane;
    const float bi = a.bias[static_cast<int64_t>(b) * a.Tp + i];
    const uint32_t my_stage = qstage + static_cast<uint32_t>(qd) * 2 * kQStage;
    uint8_t* const my_stage_p = sbase + (my_stage - base);
    int buf = 0;
    if (lane == 0) prefetch_tensormap(&tmq);
    for (int m = 0; m < nst; ++m) {
      const int d = m & 1;
      mbar_wait(dfull + 8u * d, (m / 2) & 1u);
      umma::fence_after_sync();
      float v[2][32];
#pragma unroll
      for (int h = 0; h < 2; ++h)
        umma::tmem_ld32(tmem + (static_cast<uint32_t>(32 * qd) << 16) + colD +
                            static_cast<uint32_t>(d * umma::kN + h * umma::kStageN),
                        v[h]);
      umma::tmem_wait_ld();
      umma::fence_before_sync();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(dempty + 8u * d) : "memory");
      const int j0 = c0 + m * umma::kN;
#pragma unroll
      for (int h = 0; h < 2; ++h, buf ^= 1) {
        // the buffer's previous store (two tiles ago) has been read
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        __syncwarp();
        uint8_t* t = my_stage_p + buf * kQStage + lane * 128;
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4)
          *reinterpret_cast<float4*>(t + ((c4 ^ (lane & 7)) << 4)) =
              make_float4(v[h][4 * c4] + bi, v[h][4 * c4 + 1] + bi, v[h][4 * c4 + 2] + bi,
                          v[h][4 * c4 + 3] + bi);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0)
          tma_store_3d(&tmq, my_stage + buf * kQStage, j0 + 32 * h, tr * umma::kM + 32 * qd, b);
      }
    }
    if (lane == 0) bulk_store_drain();
    __syncwarp();
  }
  umma::fence_before_sync();
  __syncthreads();
  if (warp == 2) umma::tmem_dealloc(tmem, a.tmem_cols);
}

size_t q_smem_bytes(int Kp) {
  return 1024 + static_cast<size_t>(kQStages) * (Kp / umma::kAtomK) * umma::kAtomBytes + 1024 +
         4 * 2 * kQStage;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

}  // namespace

cudaError_t gauss_alloc(int B, int C, int T, int S, cudaStream_t stream, GaussOperands* g,
                        void** ws) {
  g->Kp = gauss_kp(C);
  g->Tp = (T + umma::kM - 1) / umma::kM * umma::kM;
  g->Sp = (S + 127) / 128 * 128;  // whole 64- and 128-frame MMA groups
  const size_t a_bytes = static_cast<size_t>(B) * g->Tp * g->Kp * 2;
  const size_t b_bytes = static_cast<size_t>(B) * g->Sp * g->Kp * 2;
  const size_t bias_bytes = static_cast<size_t>(B) * g->Tp * 4;
  char* p = nullptr;
  const cudaError_t e = pool_alloc(reinterpret_cast<void**>(&p), a_bytes + b_bytes + bias_bytes, stream);
  if (e != cudaSuccess) return e;
  *ws = p;
  g->A = reinterpret_cast<__nv_bfloat16*>(p);
  g->B = reinterpret_cast<__nv_bfloat16*>(p + a_bytes);
  g->bias = reinterpret_cast<float*>(p + a_bytes + b_bytes);
  return cudaSuccess;
}

int gauss_kp(int C) { return ((2 * C + umma::kAtomK - 1) / umma::kAtomK) * umma::kAtomK; }

bool encode_gauss_b_map(const void* Bm, int64_t rows, int Kp, CUtensorMap* m, int box_rows) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(Kp), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(Kp) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(umma::kAtomK), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(Bm), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t gauss_prep(const float* z, const float* mean, const float* logstd, int B, int C, int T,
                       int S, const GaussOperands& g, cudaStream_t stream) {
  constexpr int kMaxDevices = 64;
  static std::once_flag once[kMaxDevices];
  static cudaError_t status[kMaxDevices];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || dev >= kMaxDevices) return e != cudaSuccess ? e : cudaErrorInvalidDevice;
  std::call_once(once[dev], [dev] {
    const int max_bytes = std::max((2 * kGaussMaxChannels + 1) * kPrepRows,
                                   (kGaussMaxChannels + 1) * kPrepFrames) * 4;
    cudaError_t r = cudaFuncSetAttribute(gauss_prep_rows_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(gauss_prep_frames_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, max_bytes);
    status[dev] = r;
  });
  if (status[dev] != cudaSuccess) return status[dev];
  gauss_prep_rows_kernel<<<static_cast<unsigned>(B * (g.Tp / kPrepRows)), 256,
                           static_cast<size_t>(2 * C + 1) * kPrepRows * 4, stream>>>(
      mean, logstd, B, C, T, g.Tp, g.Kp, g.A, g.bias);
  gauss_prep_frames_kernel<<<static_cast<unsigned>(B * (g.Sp / kPrepFrames)), 256,
                             static_cast<size_t>(C + 1) * kPrepFrames * 4, stream>>>(z, B, C, S, g.Sp,
                                                                                   g.Kp, g.B);
  return cudaGetLastError();
}

cudaError_t gauss_q(const GaussOperands& g, int B, int T, int S, float* q, int64_t pitch,
                    cudaStream_t stream) {
  if ((pitch % 4) != 0 || (reinterpret_cast<uintptr_t>(q) & 15u) != 0) {
    // the TMA store needs 16-byte rows: compute into an aligned scratch copy
    const int64_t p4 = (static_cast<int64_t>(S) + 3) & ~int64_t(3);
    float* tmp = nullptr;
    cudaError_t e = pool_alloc(reinterpret_cast<void**>(&tmp),
                               static_cast<size_t>(B) * T * p4 * sizeof(float), stream);
    if (e == cudaSuccess) e = gauss_q(g, B, T, S, tmp, p4, stream);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(q, pitch * sizeof(float), tmp, p4 * sizeof(float), S * sizeof(float),
                            static_cast<size_t>(B) * T, cudaMemcpyDeviceToDevice, stream);
    if (tmp) cudaFreeAsync(tmp, stream);
    return e;
  }
  CUtensorMap tmb, tmq;
  if (!encode_gauss_b_map(g.B, static_cast<int64_t>(B) * g.Sp, g.Kp, &tmb)) return cudaErrorInvalidValue;
  {
    EncodeTiledFn enc = encode_fn();
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(S), static_cast<cuuint64_t>(T),
                                static_cast<cuuint64_t>(B)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(pitch) * 4,
                                   static_cast<cuuint64_t>(pitch) * 4 * T};
    const cuuint32_t box[3] = {32, 32, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    if (!enc || (pitch * 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(q) & 15u) != 0 ||
        enc(&tmq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, q, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const size_t smem = q_smem_bytes(g.Kp);
  constexpr int kMaxDevices = 64;
  static std::once_flag once[kMaxDevices];
  static cudaError_t status[kMaxDevices];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess || dev >= kMaxDevices) return e != cudaSuccess ? e : cudaErrorInvalidDevice;
  std::call_once(once[dev], [dev] {
    status[dev] = cudaFuncSetAttribute(gauss_q_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       q_smem_bytes(gauss_kp(kGaussMaxChannels)));
  });
  if (status[dev] != cudaSuccess) return status[dev];
  QArgs qa;
  qa.A = g.A;
  qa.bias = g.bias;
  qa.q = q;
  qa.pitch = pitch;
  qa.B = B;
  qa.T = T;
  qa.S = S;
  qa.Tp = g.Tp;
  qa.Sp = g.Sp;
  qa.Kp = g.Kp;
  qa.tmem_cols = static_cast<int>(umma::tmem_cols_pow2(static_cast<uint32_t>(g.Kp / 2 + 2 * umma::kN)));
  const int tiles = g.Tp / umma::kM, cblocks = (g.Sp + kQColsPerCta - 1) / kQColsPerCta;
  gauss_q_kernel<<<static_cast<unsigned>(B * tiles * cblocks), kQThreads, smem, stream>>>(tmb, tmq, qa);
  return cudaGetLastError();
}

}  // namespace mas

extern "C" {

int mas_gaussian_loglik_device(const float* d_z, const float* d_mean, const float* d_logstd,
                               int32_t batch, int32_t channels, int32_t text_cap,
                               int32_t speech_cap, float* d_q, int64_t q_pitch, void* stream_v,
                               mas_error_t* err) {
  if (err) {
    std::memset(err, 0, sizeof(*err));
    err->item = -1;
    err->i = err->j = -1;
  }
  auto fail = [&](int status, int errc, const std::string& msg) {
    if (err) {
      err->status = status;
      err->errc = errc;
      std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
    }
    return status;
  };
  if (batch < 1 || channels < 1 || text_cap < 1 || speech_cap < 1)
    return fail(MAS_E_VALIDATION, MAS_ERRC_ZERO_DIM, "every dimension must be at least 1");
  if (channels > mas::kGaussMaxChannels)
    return fail(MAS_E_UNSUPPORTED, -1,
                "gaussian log-likelihood: at most " + std::to_string(mas::kGaussMaxChannels) +
                    " channels");
  if (q_pitch < speech_cap)
    return fail(MAS_E_VALIDATION, MAS_ERRC_SHAPE_MISMATCH, "row pitch is smaller than the speech capacity");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  mas::GaussOperands g;
  void* ws = nullptr;
  cudaError_t e = mas::gauss_alloc(batch, channels, text_cap, speech_cap, stream, &g, &ws);
  if (e == cudaSuccess)
    e = mas::gauss_prep(d_z, d_mean, d_logstd, batch, channels, text_cap, speech_cap, g, stream);
  if (e == cudaSuccess) e = mas::gauss_q(g, batch, text_cap, speech_cap, d_q, q_pitch, stream);
  if (ws) {
    const cudaError_t f = cudaFreeAsync(ws, stream);
    if (e == cudaSuccess) e = f;
  }
  if (e != cudaSuccess)
    return fail(MAS_E_CUDA, -1, std::string("gaussian log-likelihood: ") + cudaGetErrorString(e));
  return MAS_OK;
}

}  // extern "C"
