// mas_kernels.h -- launch parameters shared by the host ABI (mas_abi.cu) and
// the device kernels.  See DESIGN.md for the data layout in HBM.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "monoalign_b200.h"

namespace mas {

constexpr int kFifoSlots = 32;  // boundary-row FIFO depth, in quads
constexpr int kMaxWarpsPerCta = 8;
constexpr int kZeroCols = 64;  // mas_fwd4: zero tile {32 R rows x kZeroCols} (8 KB bulk stores)
constexpr int kMaxClusterCtas = 16;

// Stream-ordered device allocation from the library's own pool on the
// current device (mas_abi.cu); free with cudaFreeAsync.
cudaError_t pool_alloc(void** ptr, size_t bytes, cudaStream_t stream);

// mas_gauss.cu: the Gaussian log-likelihood operands (bf16, K-major, K
// padded to Kp = 64 * ceil(2C / 64); rows padded to Tp = 128 * ceil(T / 128),
// frames to Sp = 32 * ceil(S / 32)).
constexpr int kGaussMaxChannels = 192;  // Kp <= 384: A (Kp/2) + D fit TMEM's 512 columns at W = 2
struct GaussOperands {
  __nv_bfloat16* A;  // [B][Tp][Kp]  row coefficients
  __nv_bfloat16* B;  // [B][Sp][Kp]  z^2, z per frame
  float* bias;       // [B][Tp]
  int Tp, Sp, Kp;
};
int gauss_kp(int C);
cudaError_t gauss_alloc(int B, int C, int T, int S, cudaStream_t stream, GaussOperands* g, void** ws);
cudaError_t gauss_prep(const float* z, const float* mean, const float* logstd, int B, int C, int T,
                       int S, const GaussOperands& g, cudaStream_t stream);
cudaError_t gauss_q(const GaussOperands& g, int B, int T, int S, float* q, int64_t pitch,
                    cudaStream_t stream);
bool encode_gauss_b_map(const void* Bm, int64_t rows, int Kp, CUtensorMap* m, int box_rows = 64);

struct FwdArgs {
  int b0;                   // first item of this launch (items b0 .. b0 + grid/K - 1)
  const uint32_t* lengths;  // [B][2] (t, s); t == 0 marks an item not to run
  uint32_t* dirs;           // [B][M][T_alloc] direction words, see DESIGN.md
  int* flags;               // [B] NonFinite candidate flags
  int T_pad;                // rows between items in the (pitched) input
  int M;                    // direction words per row = ceil(S_cap / 32)
  int T_alloc;              // rows per item in `dirs` = K * W * 64
  int K;                    // CTAs per item (cluster size)
  int W;                    // warps per CTA
  int N;                    // TMA stages per warp
  float mnv;                // max_neg_val
  float row0_up;            // value above row 0: mnv (parallel) / -inf (reference)
  int zero_fill;            // 1: zero the warps' rows of `out` as we go (linear bulk stores)
  uint8_t* out;             // the output [B][T_cap][S_cap] (zero_fill)
  int T_cap, S_cap;         // output shape
  int l2_ahead;             // mas_fwd4: stages prefetched into L2 beyond the smem ring
  // mas_fwd4 bands (texts taller than one cluster): an item is `bands`
  // clusters of band_rows rows each, all in ONE launch.  Clusters take
  // (band, item) from a ticket counter in band-major order, so a cluster
  // waiting for the band above only waits for clusters already running.
  // The bottom row of band k goes through bnd [B][bands-1][bnd_pitch]
  // floats, its progress (32-column quads published) through
  // progress [B][bands-1]; ticket and progress are zeroed before the launch.
  int bands, band_rows, nb;
  float* bnd;
  int* progress;
  int* ticket;
  int bnd_pitch;
  // Gaussian source (Kp > 0): q computed in-kernel from mas_gauss.cu's operands
  int Kp;                   // padded K (0: q read from HBM)
  int gstages, gacc, gN;    // B stages / TMEM accumulators in flight, frames per MMA (gauss_cfg)
  int Tp, Sp;               // padded rows / frames per item of the operands
  const __nv_bfloat16* gA;  // [B][Tp][Kp]
  const float* gbias;       // [B][Tp]
  // pipelined plans: before writing `dirs`, wait until *bt_done >= bt_need
  // (the backtrack that last read this buffer has finished with it)
  const unsigned* bt_done;
  unsigned bt_need;
  int pdl;                  // launched with programmatic stream serialization
  int scores;               // 1: score export (Q written over q through tm_out; no dirs/flags)
  int tail;                 // 1: one-launch tail (K = 1, one band): words in shared memory,
                            //    the CTA walks and expands its item (no backtrack kernel)
  int32_t* path;            // tail outputs: [B][S_cap] path rows, [B][T_cap] durations (or null)
  int32_t* dur;
  uint32_t one;             // 1 and 0.0f passed at run time so ptxas keeps the
  float zero;               //   bit IMADs / NonFinite FFMAs on the FMA pipe
};

struct BtArgs {
  int b0;                   // first item of this launch; B items from there
  const uint32_t* lengths;  // [B][2]
  const uint32_t* dirs;     // [B][M][T_alloc]
  int32_t* path;            // [B][S_cap] int32 path rows, -1 past s_b, or null
  uint8_t* out;             // [B][T_cap][S_cap] (already zero-filled) or null
  int32_t* dur;             // [B][T_cap] int32 durations (row sums of the alignment) or null
  int B, T_cap, S_cap, M, T_alloc;
  int R;                    // rows per backtrack window (<= 256, <= T_alloc)
  unsigned* done;           // pipelined plans: +1 per CTA once its direction words are read
};

cudaError_t launch_backtrack(const BtArgs& a, cudaStream_t stream, int* launches);
cudaError_t launch_locate_nonfinite(const float* q, int64_t row_pitch, int T_pad, int b, int t,
                                    int s, unsigned long long* d_result, cudaStream_t stream);
cudaError_t launch_generate(uint64_t s0, int64_t first_elem, int B, int T, int S, int64_t pitch,
                            float* out, cudaStream_t stream);
// mas_fwd4.cu: R = 4 rows per lane, 32 R rows per warp, 32-column stages.
// mas_scores.cu: score tables (std::max arithmetic, bit-exact with the
// reference's forward_parallel) and their direction words in the backtrack
// kernel's [B][M][T_alloc] layout; used for NaN sentinels (mas_abi.cu).
cudaError_t launch_scores_to_dirs(const float* q, int64_t pitch, int rows_per_item, int S_cap,
                                  const uint32_t* d_lengths, int M, int T_alloc, int B,
                                  uint32_t* dirs, cudaStream_t stream);
cudaError_t launch_flag_nonfinite(const float* q, int64_t pitch, int rows_per_item, int S_cap,
                                  const uint32_t* d_lengths, int B, int* flags,
                                  cudaStream_t stream);
// mas_forward_scores over items `rows_per_item` rows apart, host lengths.
int forward_scores_host_lengths(float* d_values, int64_t row_pitch, int32_t batch,
                                int32_t rows_per_item, int32_t speech_cap, const uint32_t* lengths,
                                float max_neg_val, cudaStream_t stream, mas_error_t* err);
// mas_abi.cu: the score export through mas_fwd4 (OUT 1) when q's layout
// suits its TMA maps; MAS_E_UNSUPPORTED (nothing launched) otherwise.
int forward_scores_fwd4(float* d_values, int64_t pitch, int B, int T_cap, int S_cap,
                        const uint32_t* lengths, int mode, float mnv, cudaStream_t stream,
                        mas_error_t* err);
size_t fwd4_smem_bytes(int R, int W, int N, int Kp = 0);
size_t fwd4_tail_bytes(int R, int W, int M);  // shared memory of the one-launch tail
struct GaussCfg {
  int gN, gstages, gacc;
};
GaussCfg gauss_cfg(int W, int Kp);
cudaError_t fwd4_configure();
int fwd4_max_active_clusters(int R, int W, int N, int K, int Kp = 0);
cudaError_t launch_fwd4(int R, int mode, const CUtensorMap& tmq, const CUtensorMap& tm_out,
                        const FwdArgs& a, int B, cudaStream_t stream);

}  // namespace mas
