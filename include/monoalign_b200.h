/*
 * monoalign_b200.h -- the C-ABI drop-in boundary of the B200-native
 * maximum-path (Monotonic Alignment Search) call.
 *
 * Plain pointers and sizes only; no torch / CUDA-runtime types in the
 * signatures (streams are passed as `void*` = cudaStream_t).  Implemented in
 * paper_2409_07704_b200/csrc/ and built into
 * paper_2409_07704_b200/_lib/libmonoalign_b200.so.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj):
 *
 *   mas_align_host    monoalign::align(const LikelihoodBatch&, const MasConfig&)
 *                       include/monoalign/align.hpp:9-12, i.e. what the pybind
 *                       binding's align_arrays / align_paths call
 *                       (bindings/module.cpp:120-154) after copying numpy data
 *                       into a LikelihoodBatch (module.cpp:88-99).
 *   mas_align_device  same call on caller-owned device buffers (no host copy;
 *                       the reference has no equivalent -- SURVEY.md 8(b)).
 *   MAS_FLAG_UNCHECKED  parallel::detail::align_unchecked / reference::detail::
 *                       align_unchecked (parallel.hpp:29-31, reference.hpp:42-44):
 *                       skips validate_config so -inf / -1e9 sentinels run.
 *   mas_plan_*        the same call split into enqueue-only + check, so the
 *                       kernels can be captured in a CUDA graph / timed alone.
 *   mas_generate_device  bench::generate_random_batch (bench.hpp:58,
 *                       bench.cpp:164-180), bit-identical, for any item shard.
 *   mas_errc_name     errc_name (types.cpp:8-29).
 *   mas_validate_config / mas_validate_host
 *                     validate_config / validate_batch / validate_item
 *                       (types.cpp:59-130), for the C++ mirror in
 *                       include/monoalign/.
 *
 * Error convention: every entry returns a mas_status; on MAS_E_VALIDATION
 * `err->errc` holds the reference Errc (errors.hpp:8-30 order) and
 * `err->message` the exact text the reference's ValidationError carries
 * (types.cpp:59-130), so a binding can raise ValueError with identical text
 * (module.cpp:210-220).  MAS_E_CUDA means the device path failed (no CPU
 * fallback exists).
 */
#ifndef MONOALIGN_B200_H
#define MONOALIGN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MAS_ABI_VERSION 3

#if defined(__GNUC__)
#define MAS_API __attribute__((visibility("default")))
#else
#define MAS_API
#endif

/* include/monoalign/errors.hpp:8-30, declaration order. */
enum mas_errc {
  MAS_ERRC_ZERO_DIM = 0,
  MAS_ERRC_INFEASIBLE_LENGTHS = 1,
  MAS_ERRC_LENGTHS_OUT_OF_RANGE = 2,
  MAS_ERRC_NON_FINITE = 3,
  MAS_ERRC_SPEECH_TOO_LONG = 4,
  MAS_ERRC_SHAPE_MISMATCH = 5,
  MAS_ERRC_INVALID_PATH = 6,
  MAS_ERRC_INVALID_MATRIX = 7,
  MAS_ERRC_INVALID_CONFIG = 8,
  MAS_ERRC_TOO_LARGE = 9,
  MAS_ERRC_EMPTY_REPORT = 10,
  MAS_ERRC_INSUFFICIENT_POINTS = 11,
  MAS_ERRC_IO_FAILURE = 12,
  MAS_ERRC_BAD_MAGIC = 13,
  MAS_ERRC_UNSUPPORTED_VERSION = 14,
  MAS_ERRC_TRUNCATED_FILE = 15,
  MAS_ERRC_DIMENSION_OVERFLOW = 16
};

enum mas_status {
  MAS_OK = 0,
  MAS_E_VALIDATION = 1, /* reference ValidationError -> ValueError / exit 2 */
  MAS_E_IO = 2,         /* reference IoError -> OSError / exit 1 */
  MAS_E_CUDA = 3,       /* CUDA runtime / launch failure */
  MAS_E_UNSUPPORTED = 4 /* shape outside what the device path supports */
};

/* EngineKind, types.hpp:28 (declaration order). */
enum mas_engine { MAS_ENGINE_REFERENCE = 0, MAS_ENGINE_PARALLEL = 1 };

#define MAS_FLAG_UNCHECKED 0x1u /* skip validate_config (detail::align_unchecked) */
/* ABI 3, mas_align_device[_ex] only: do not read the NonFinite flags back
 * (no host synchronisation; the call is enqueue-only).  Host-detectable
 * errors (config, lengths) are still returned; a non-finite likelihood is
 * then NOT reported and its item's alignment is undefined. */
#define MAS_FLAG_NO_CHECK 0x2u
/* ABI 3, mas_plan_create only: consecutive enqueues of the plan may overlap
 * -- batch i's backtrack kernel runs concurrently with batch i+1's forward
 * kernel (programmatic dependent launch; two direction-word buffers, the
 * forward waits on a device counter before reusing the one a backtrack two
 * batches back read).  The caller must give consecutive enqueues distinct
 * output buffers.  Not for CUDA-graph capture. */
#define MAS_FLAG_PIPELINED 0x4u

typedef struct mas_error {
  int32_t status;     /* enum mas_status */
  int32_t errc;       /* enum mas_errc when status == MAS_E_VALIDATION, else -1 */
  int32_t item;       /* failing item index, -1 if not item-specific */
  int32_t reserved;
  int64_t i, j;       /* NonFinite location (row, column), else -1 */
  char message[512];  /* exact reference what() text */
} mas_error_t;

/* MasConfig, types.hpp:32-39. */
typedef struct mas_config {
  int32_t engine;       /* enum mas_engine, default MAS_ENGINE_PARALLEL */
  float max_neg_val;    /* default -1e32f (kDefaultMaxNegVal, types.hpp:19) */
  int32_t lane_padding; /* LanePadding; accepted and unobservable (parallel.hpp:12-15) */
  int32_t threads;      /* validated >= 0 (types.cpp:66-68), otherwise ignored */
  uint32_t flags;       /* MAS_FLAG_* */
} mas_config_t;

/* Fills the MasConfig defaults. */
MAS_API void mas_config_default(mas_config_t* cfg);

/*
 * Host buffers in, host buffers out (pageable or pinned).
 *   values   [batch][text_cap][speech_cap] float32 row-major (LikelihoodBatch::values)
 *   lengths  [batch][2] uint32 (text, speech) (LikelihoodBatch::lengths) or NULL = full
 *   out      [batch][text_cap][speech_cap] uint8 (AlignmentMatrix::values) or NULL
 *   paths    [batch][speech_cap] int32, -1 past each item's speech length, or NULL
 * Uses the calling thread's current CUDA device.  Synchronous.
 */
MAS_API int mas_align_host(const float* values, int32_t batch, int32_t text_cap, int32_t speech_cap,
                   const uint32_t* lengths, const mas_config_t* cfg, uint8_t* out,
                   int32_t* paths, mas_error_t* err);
/* The same plus per-token durations (ABI 2):
 *   durations [batch][text_cap] int32, the row sums of the alignment
 *   (columns spent on each text row; 0 past the item's text length), or NULL.
 * With out == NULL the dense [B][T][S] output is neither zeroed nor written. */
MAS_API int mas_align_host_ex(const float* values, int32_t batch, int32_t text_cap,
                      int32_t speech_cap, const uint32_t* lengths, const mas_config_t* cfg,
                      uint8_t* out, int32_t* paths, int32_t* durations, mas_error_t* err);

/*
 * Device buffers (caller-owned, current device).  `row_pitch` = elements
 * between consecutive text rows (>= speech_cap); items are text_cap rows
 * apart.  `lengths` is a HOST array as above.  Enqueues on `stream` and
 * synchronises it before returning (the NonFinite check needs the result),
 * unless cfg->flags has MAS_FLAG_NO_CHECK.  Plans (validation, geometry,
 * workspace, tensor maps) are cached across calls of the same shape, lengths,
 * config and stream (ABI 3).
 */
MAS_API int mas_align_device(const float* d_values, int64_t row_pitch, int32_t batch, int32_t text_cap,
                     int32_t speech_cap, const uint32_t* lengths, const mas_config_t* cfg,
                     uint8_t* d_out, int32_t* d_paths, void* stream, mas_error_t* err);
/* ... plus device durations [batch][text_cap] int32 (see mas_align_host_ex). */
MAS_API int mas_align_device_ex(const float* d_values, int64_t row_pitch, int32_t batch,
                        int32_t text_cap, int32_t speech_cap, const uint32_t* lengths,
                        const mas_config_t* cfg, uint8_t* d_out, int32_t* d_paths,
                        int32_t* d_durations, void* stream, mas_error_t* err);

/* ---- plan API: validation + workspace once, enqueue-only execution ------ */
typedef struct mas_plan mas_plan_t;

/* Validates config and lengths (host side) and allocates the workspace.
 * Host-detectable item errors are recorded and reported by mas_plan_finish
 * (lowest failing item wins, parallel.cpp:160-165). */
MAS_API int mas_plan_create(int32_t batch, int32_t text_cap, int32_t speech_cap, int64_t row_pitch,
                    const uint32_t* lengths, const mas_config_t* cfg, mas_plan_t** plan,
                    mas_error_t* err);
/* Enqueues the kernels on `stream`; no host synchronisation. */
MAS_API int mas_plan_enqueue(mas_plan_t* plan, const float* d_values, uint8_t* d_out, int32_t* d_paths,
                     void* stream, mas_error_t* err);
/* The same, restricted to a subset of the kernels (MAS_PART_* bits), so a
 * caller can bracket each kernel with its own events.  The forward part
 * (direction bits, NonFinite flags, output zero fill) must precede the
 * backtrack part (paths / ones of the alignment) on `stream`. */
#define MAS_PART_FORWARD 0x1u
#define MAS_PART_BACKTRACK 0x2u
#define MAS_PART_ALL 0x3u
MAS_API int mas_plan_enqueue_part(mas_plan_t* plan, uint32_t parts, const float* d_values,
                          uint8_t* d_out, int32_t* d_paths, void* stream, mas_error_t* err);
/* mas_plan_enqueue_part plus device durations [batch][text_cap] int32. */
MAS_API int mas_plan_enqueue_ex(mas_plan_t* plan, uint32_t parts, const float* d_values,
                        uint8_t* d_out, int32_t* d_paths, int32_t* d_durations, void* stream,
                        mas_error_t* err);
/* Synchronises `stream` and turns device-side NonFinite flags and recorded
 * host-side item errors into the reference's error (or MAS_OK). */
MAS_API int mas_plan_finish(mas_plan_t* plan, const float* d_values, void* stream, mas_error_t* err);
/* Number of kernel launches one mas_plan_enqueue issues. */
MAS_API int mas_plan_launches(const mas_plan_t* plan);
/* Launch geometry chosen by the plan: {rows_per_warp, warps_per_cta,
 * ctas_per_item (cluster size), stages, segment_columns, max co-resident
 * clusters of the forward kernel}. */
MAS_API void mas_plan_geometry(const mas_plan_t* plan, int32_t geom[6]);
MAS_API void mas_plan_destroy(mas_plan_t* plan);

/* validate_config (types.cpp:59-69): MAS_OK or MAS_E_VALIDATION with the
 * reference's InvalidConfig text. */
MAS_API int mas_validate_config(const mas_config_t* cfg, mas_error_t* err);

/* validate_batch / validate_item (types.cpp:81-130) of host data: the
 * length checks on the host, the NonFinite scan on the device (the forward
 * kernel runs without outputs).  `item_base` is added to the item index in
 * messages, so validate_item(batch, b) can pass item b alone. */
MAS_API int mas_validate_host(const float* values, int32_t batch, int32_t text_cap,
                      int32_t speech_cap, const uint32_t* lengths, int32_t item_base,
                      mas_error_t* err);

/* bench::generate_random_batch(batch, text_cap, speech_cap, seed), items
 * [first_item, first_item + batch) of that stream, written pitched into
 * d_out[(b * text_cap + i) * row_pitch + j].  Bit-identical to the CPU. */
MAS_API int mas_generate_device(uint64_t seed, int32_t batch, int32_t text_cap, int32_t speech_cap,
                        int64_t first_item, int64_t row_pitch, float* d_out, void* stream);

/* parallel::forward_parallel (parallel.hpp:17, parallel.cpp:95-108) over a
 * device batch, in place: every item's [t][s] region of d_values becomes the
 * parallel engine's score table Q, bit-identical to the reference (std::max
 * tie rule, signed zeros).  lengths [B][2] host (t, s) or NULL = full; items
 * with t or s = 0 are left untouched.  Stream-ordered; nothing is validated
 * beyond shapes (forward_parallel validates nothing). */
MAS_API int mas_forward_scores(float* d_values, int64_t row_pitch, int32_t batch, int32_t text_cap,
                               int32_t speech_cap, const uint32_t* lengths, float max_neg_val,
                               void* stream, mas_error_t* err);

/* ABI 3.  The same table in either engine's arithmetic: engine
 * MAS_ENGINE_PARALLEL is mas_forward_scores; MAS_ENGINE_REFERENCE is
 * reference::forward_reference (reference.hpp:33, reference.cpp:9-36): row 0
 * the running sum 0 + q[0][0] + ... + q[0][j], cells with i > j exactly
 * max_neg_val, every other cell max(Q[i-1][j-1], Q[i][j-1]) + q[i][j]. */
MAS_API int mas_forward_scores_ex(float* d_values, int64_t row_pitch, int32_t batch,
                                  int32_t text_cap, int32_t speech_cap, const uint32_t* lengths,
                                  int32_t engine, float max_neg_val, void* stream,
                                  mas_error_t* err);

/* ABI 3.  parallel::backward_parallel / reference::backward_reference
 * (parallel.hpp:21, reference.hpp:37; the shared walk of backtrack.hpp:21-32):
 * the argmax walk from (t-1, s-1) to column 0 over a device score table
 * (either engine's), strict > (ties keep the current row).  d_paths
 * [batch][speech_cap] int32, -1 past each item's speech length.  The
 * decisions Q[i-1][j] > Q[i][j] are packed into direction words on the device
 * and walked by the same backtrack kernel as the maximum-path call.
 * Stream-ordered. */
MAS_API int mas_backtrack_scores(const float* d_scores, int64_t row_pitch, int32_t batch,
                                 int32_t text_cap, int32_t speech_cap, const uint32_t* lengths,
                                 int32_t* d_paths, void* stream, mas_error_t* err);

/* ABI 3.  parallel::detail::relax_column (parallel.hpp:39, parallel.cpp:25-31)
 * on device columns: cur[0] += max(sentinel, prev[0]);
 * cur[i] += max(prev[i-1], prev[i]), max(a, b) = (a < b) ? b : a.
 * Stream-ordered. */
MAS_API int mas_relax_column(const float* d_prev, float* d_cur, int32_t lanes, float sentinel,
                             void* stream, mas_error_t* err);

/* ---- fused log-likelihood -----
 * The Glow-TTS / VITS prior's log-likelihood matrix
 *   q[b][i][j] = sum_c log N(z[b][c][j]; mean[b][c][i], exp(logstd[b][c][i]))
 * computed on the tensor cores (bf16 operands of the expanded form, fp32
 * accumulation).  z [batch][channels][speech_cap], mean / logstd
 * [batch][channels][text_cap], fp32, device.  channels <= 192.  (ABI 3)
 * mas_gaussian_loglik_device writes q [batch][text_cap][q_pitch] fp32. */
MAS_API int mas_gaussian_loglik_device(const float* d_z, const float* d_mean,
                                       const float* d_logstd, int32_t batch, int32_t channels,
                                       int32_t text_cap, int32_t speech_cap, float* d_q,
                                       int64_t q_pitch, void* stream, mas_error_t* err);
/* The maximum-path call on that q without materialising it: the forward
 * kernel computes each 32-frame tile of q on the tensor cores (A in TMEM, B
 * by TMA) and feeds it straight to the DP, so q never reaches HBM.  Same
 * outputs, validation, errors and engines as mas_align_device_ex (lengths a
 * HOST [batch][2] array or NULL; a non-finite q is reported at its exact
 * (i, j)); the alignment equals mas_align_device_ex on the q
 * mas_gaussian_loglik_device writes, bit for bit.  The fused kernel handles
 * texts up to one cluster of rows (4096); taller texts, and NaN sentinels of
 * the parallel engine, materialise q on the device and take the ordinary
 * path.  Synchronises `stream`.  (ABI 3) */
MAS_API int mas_align_gaussian_device(const float* d_z, const float* d_mean,
                                      const float* d_logstd, int32_t batch, int32_t channels,
                                      int32_t text_cap, int32_t speech_cap,
                                      const uint32_t* lengths, const mas_config_t* cfg,
                                      uint8_t* d_out, int32_t* d_paths, int32_t* d_durations,
                                      void* stream, mas_error_t* err);
/* Enqueue-only form for training loops (a plan, like mas_plan_create): the
 * operand workspace and validation once, then per batch the operand prep and
 * the fused kernels only, no host synchronisation (CUDA-graph capturable).
 * mas_plan_finish(plan, NULL, ...) reports validation / NonFinite errors of
 * the last enqueue (a flagged item materialises q to locate the cell).
 * MAS_E_UNSUPPORTED where mas_align_gaussian_device would materialise q
 * (texts taller than 4096 rows, NaN sentinels of the parallel engine).
 * Destroy with mas_plan_destroy.  (ABI 3) */
MAS_API int mas_plan_create_gaussian(int32_t batch, int32_t channels, int32_t text_cap,
                                     int32_t speech_cap, const uint32_t* lengths,
                                     const mas_config_t* cfg, mas_plan_t** plan,
                                     mas_error_t* err);
MAS_API int mas_plan_enqueue_gaussian(mas_plan_t* plan, const float* d_z, const float* d_mean,
                                      const float* d_logstd, uint8_t* d_out, int32_t* d_paths,
                                      int32_t* d_durations, void* stream, mas_error_t* err);

/* ---- MASTENS v1 tensor files (tensor_io.hpp:11-23, tensor_io.cpp) --------
 * Host-only.  Errors are MAS_E_IO with the reference's IoError code and text
 * (IoFailure, BadMagic, UnsupportedVersion, TruncatedFile, DimensionOverflow).
 * dtype: 0 = float32 (LikelihoodBatch), 1 = uint8 (AlignmentMatrix).
 * The header is validated -- including the byte budget (read_tensor's
 * byte_budget, default 1 GiB) -- before any payload is read. */
#define MAS_IO_DEFAULT_BYTE_BUDGET (1ull << 30)
MAS_API int mas_io_read_header(const char* path, uint64_t byte_budget, int32_t* dtype,
                               int64_t dims[3], int32_t* lengths_present, mas_error_t* err);
/* Payload into `values` (dims product x dtype size bytes) and the lengths
 * table into `lengths` [B][2] (full lengths when the file has none).
 * `dtype` / `dims` are what mas_io_read_header returned and what the buffers
 * were sized for; a file whose header no longer matches them (replaced
 * between the two calls) is rejected with IoFailure before anything is
 * written (ABI 3). */
MAS_API int mas_io_read(const char* path, uint64_t byte_budget, int32_t dtype, const int64_t dims[3],
                        void* values, uint32_t* lengths, mas_error_t* err);
/* write_tensor: header, payload, lengths table ([B][2] or NULL = full). */
MAS_API int mas_io_write(const char* path, int32_t dtype, int64_t batch, int64_t text_cap,
                         int64_t speech_cap, const void* values, const uint32_t* lengths,
                         mas_error_t* err);

MAS_API const char* mas_errc_name(int32_t errc);
MAS_API int mas_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* MONOALIGN_B200_H */
