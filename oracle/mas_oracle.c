/*
 * mas_oracle.c -- CPU restatement of the monoalign maximum-path call.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * path; it is never linked into, loaded by, or called from the product
 * library (paper_2409_07704_b200/).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Parity is pinned two ways (see tests/test_oracle.py):
 *   1. the reference's own known-answer tests (test_reference.cpp,
 *      test_parallel.cpp, test_smoke.py, acceptance.cpp KATs), and
 *   2. byte-for-byte comparison with the reference itself, compiled from
 *      /root/reference/proj/src by oracle/Makefile into oracle/_ref/, on
 *      seeded random batches, and the golden fixtures in tests/golden/.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/proj).  Plain C99, single-threaded, no allocation of
 * more than one item's score table.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Errc numbering mirrors include/monoalign/errors.hpp:8-30 (declaration
 * order). */
enum {
  OR_ZERO_DIM = 0,
  OR_INFEASIBLE_LENGTHS = 1,
  OR_LENGTHS_OUT_OF_RANGE = 2,
  OR_NON_FINITE = 3,
  OR_SPEECH_TOO_LONG = 4,
  OR_SHAPE_MISMATCH = 5,
  OR_INVALID_CONFIG = 8,
};

/* types.hpp:26 */
#define OR_MAX_SPEECH_LEN 100000
/* types.hpp:22 */
#define OR_MAX_NEG_VAL_CEILING (-1e30f)

typedef struct {
  int32_t errc;  /* -1 = ok */
  int32_t item;  /* failing item, -1 for config / batch-level errors */
  int64_t i, j;  /* NonFinite location */
} oracle_error_t;

/* std::max(a, b) == (a < b) ? b : a  (the reference's relax_column,
 * parallel.cpp:27-30, and forward_reference, reference.cpp:32). */
static inline float or_max(float a, float b) { return (a < b) ? b : a; }

/* ---- RNG: bench.hpp:79-91 and bench.cpp:164-180 ------------------------- */

uint64_t oracle_splitmix64(uint64_t* state) {
  uint64_t z;
  *state += 0x9e3779b97f4a7c15ULL;
  z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

uint64_t oracle_mix_seed(uint64_t seed, uint64_t index) {
  uint64_t state = seed ^ (0xd1342543de82ef95ULL * (index + 1));
  return oracle_splitmix64(&state);
}

/* generate_random_batch (bench.cpp:164-180): uniform [-5, 5] float32 from
 * one splitmix64 stream seeded by mix_seed(seed, 0).  `first` skips that
 * many elements of the stream so a shard [first, first + n) can be produced
 * on its own (the stream is counter-addressable: state_n = s0 + (n+1)*phi). */
void oracle_generate(uint64_t seed, int64_t first, int64_t n, float* out) {
  const uint64_t s0 = oracle_mix_seed(seed, 0);
  uint64_t state = s0 + (uint64_t)first * 0x9e3779b97f4a7c15ULL;
  for (int64_t k = 0; k < n; ++k) {
    const double u = (double)(oracle_splitmix64(&state) >> 11) * 0x1.0p-53;
    volatile double prod = 10.0 * u; /* no FMA contraction, as the -O3 x86-64 build */
    out[k] = (float)(-5.0 + prod);
  }
}

/* ---- validation: types.cpp:59-69, :81-116 -------------------------------- */

int oracle_validate_config(float max_neg_val, int threads) {
  if (!isfinite(max_neg_val) || max_neg_val > OR_MAX_NEG_VAL_CEILING) return OR_INVALID_CONFIG;
  if (threads < 0) return OR_INVALID_CONFIG;
  return -1;
}

/* validate_item (types.cpp:81-116): order ZeroDim, LengthsOutOfRange,
 * SpeechTooLong, InfeasibleLengths, then a row-major NonFinite scan of the
 * valid region. */
static int validate_item(const float* item, int T, int S, uint32_t t, uint32_t s,
                         int64_t* bi, int64_t* bj) {
  if (t < 1 || s < 1) return OR_ZERO_DIM;
  if (t > (uint32_t)T || s > (uint32_t)S) return OR_LENGTHS_OUT_OF_RANGE;
  if (s > OR_MAX_SPEECH_LEN) return OR_SPEECH_TOO_LONG;
  if (t > s) return OR_INFEASIBLE_LENGTHS;
  for (uint32_t i = 0; i < t; ++i) {
    for (uint32_t j = 0; j < s; ++j) {
      if (!isfinite(item[(size_t)i * S + j])) {
        *bi = i;
        *bj = j;
        return OR_NON_FINITE;
      }
    }
  }
  return -1;
}

/* ---- backtrack: src/backtrack.hpp:21-32 ---------------------------------- */
/* Generic strided score access so both engines share one walk, exactly as
 * the reference's ScoreView (backtrack.hpp:9-15). Tie rule: stay unless the
 * upper-left score is strictly greater. */
static void backtrack(const float* Q, ptrdiff_t row_stride, ptrdiff_t col_stride, int t, int s,
                      int32_t* path) {
  int cur = t - 1;
  path[s - 1] = cur;
  for (int j = s - 2; j >= 0; --j) {
    if (cur > 0 && Q[(cur - 1) * row_stride + j * col_stride] > Q[cur * row_stride + j * col_stride]) {
      --cur;
    }
    path[j] = cur;
  }
}

/* ---- parallel engine item: parallel.cpp:57-84 ---------------------------- */
/* Speech-major scratch (transpose_into, :38-52), first column rows 1..t-1 =
 * sentinel (:73-75), then relax_column (:25-31) for j = 1..s-1 (:77-80):
 *   cur[0] += max(sentinel, prev[0]); cur[i] += max(prev[i-1], prev[i]). */
static void align_one_parallel(const float* item, int S, int t, int s, float mnv, float* scratch,
                               int32_t* path) {
  for (int i = 0; i < t; ++i)
    for (int j = 0; j < s; ++j) scratch[(size_t)j * t + i] = item[(size_t)i * S + j];
  for (int i = 1; i < t; ++i) scratch[i] = mnv;
  for (int j = 1; j < s; ++j) {
    const float* prev = scratch + (size_t)(j - 1) * t;
    float* cur = scratch + (size_t)j * t;
    cur[0] += or_max(mnv, prev[0]);
    for (int i = 1; i < t; ++i) cur[i] += or_max(prev[i - 1], prev[i]);
  }
  backtrack(scratch, 1, t, t, s, path);
}

/* ---- reference engine item: reference.cpp:9-36 -------------------------- */
/* Q initialised to the sentinel (:12-17), row 0 the running sum (:20-24),
 * rows i >= 1 only for j >= i (:30-34); cells with i > j stay exactly mnv. */
static void align_one_reference(const float* item, int S, int t, int s, float mnv, float* Q,
                                int32_t* path) {
  for (size_t k = 0; k < (size_t)t * s; ++k) Q[k] = mnv;
  float run = 0.0f;
  for (int j = 0; j < s; ++j) {
    run += item[j];
    Q[j] = run;
  }
  for (int i = 1; i < t; ++i)
    for (int j = i; j < s; ++j)
      Q[(size_t)i * s + j] =
          or_max(Q[(size_t)(i - 1) * s + j - 1], Q[(size_t)i * s + j - 1]) + item[(size_t)i * S + j];
  backtrack(Q, s, 1, t, s, path);
}

/*
 * oracle_align: the whole maximum-path call, detail::align_unchecked of
 * either engine (parallel.cpp:117-167, reference.cpp:45-54) -- i.e. WITHOUT
 * validate_config; callers that want the public behaviour call
 * oracle_validate_config first (parallel.cpp:171-174, reference.cpp:58-61).
 *
 *   q        [B][T][S] float32, row-major
 *   lengths  [B][2] (text, speech) or NULL for full lengths
 *   engine   0 = parallel, 1 = reference
 *   out      [B][T][S] uint8 or NULL  (zeros + one 1 per valid column)
 *   paths    [B][S] int32 or NULL     (-1 past each item's speech length)
 *
 * Returns -1 on success, else the Errc of the lowest failing item
 * (parallel.cpp:160-165; validate_batch stops at the first, types.cpp:127).
 */
int oracle_align(const float* q, int B, int T, int S, const uint32_t* lengths, float mnv,
                 int engine, uint8_t* out, int32_t* paths, oracle_error_t* err) {
  err->errc = -1;
  err->item = -1;
  err->i = err->j = -1;
  if (B < 1 || T < 1 || S < 1) {
    err->errc = OR_ZERO_DIM;
    return OR_ZERO_DIM;
  }
  if (out) memset(out, 0, (size_t)B * T * S);
  if (paths)
    for (size_t k = 0; k < (size_t)B * S; ++k) paths[k] = -1;
  float* scratch = (float*)malloc(sizeof(float) * (size_t)T * S);
  int32_t* path = (int32_t*)malloc(sizeof(int32_t) * (size_t)S);
  if (!scratch || !path) {
    free(scratch);
    free(path);
    return -2;
  }
  for (int b = 0; b < B; ++b) {
    const float* item = q + (size_t)b * T * S;
    const uint32_t t = lengths ? lengths[2 * b] : (uint32_t)T;
    const uint32_t s = lengths ? lengths[2 * b + 1] : (uint32_t)S;
    int64_t bi = -1, bj = -1;
    const int code = validate_item(item, T, S, t, s, &bi, &bj);
    if (code >= 0) {
      err->errc = code;
      err->item = b;
      err->i = bi;
      err->j = bj;
      break;
    }
    if (engine == 1)
      align_one_reference(item, S, (int)t, (int)s, mnv, scratch, path);
    else
      align_one_parallel(item, S, (int)t, (int)s, mnv, scratch, path);
    /* write_path (types.cpp:181-185) */
    for (uint32_t j = 0; j < s; ++j) {
      if (out) out[(size_t)b * T * S + (size_t)path[j] * S + j] = 1;
      if (paths) paths[(size_t)b * S + j] = path[j];
    }
  }
  free(scratch);
  free(path);
  return err->errc;
}

/* Score table of the parallel engine for one item (forward_parallel,
 * parallel.cpp:95-108), exposed so tests can check direction bits. */
void oracle_forward_parallel(float* q, int t, int s, ptrdiff_t row_stride, float mnv) {
  for (int i = 1; i < t; ++i) q[i * row_stride] = mnv;
  for (int j = 1; j < s; ++j) {
    q[j] += or_max(mnv, q[j - 1]);
    for (int i = 1; i < t; ++i)
      q[i * row_stride + j] += or_max(q[(i - 1) * row_stride + j - 1], q[i * row_stride + j - 1]);
  }
}
