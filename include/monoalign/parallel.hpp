// monoalign/parallel.hpp -- "parallel" engine entry points (reference
// include/monoalign/parallel.hpp:10-39).  Arithmetic: the column recurrence
// of src/parallel.cpp:25-31 (row above row 0 = max_neg_val, every lane
// relaxed), executed by mas_fwd_kernel<0>.
#pragma once

#include "monoalign/types.hpp"

namespace monoalign::parallel {

/// Lane count the reference would use (parallel.cpp:14-19); informational.
MONOALIGN_API int pad_lanes(int t, LanePadding policy);

/// In-place score table of the parallel engine (reference parallel.hpp:17,
/// parallel.cpp:95-108), bit-identical; computed on the GPU
/// (mas_forward_scores: the forward kernel's score export), the item
/// round-tripping through device memory.
MONOALIGN_API void forward_parallel(MutableLikelihoodView q, const MasConfig& cfg = {});

/// Argmax walk over scores produced by forward_parallel (reference
/// parallel.hpp:21, backtrack.hpp:21-32; ties keep the current row).  The
/// table is copied to the device, its decisions packed into direction words
/// and walked by the backtrack kernel (mas_backtrack_scores).
MONOALIGN_API PathVector backward_parallel(const LikelihoodView& scores);

MONOALIGN_API AlignmentMatrix align_parallel(const LikelihoodBatch& batch,
                                             const MasConfig& cfg = {});

namespace detail {
/// align_parallel without validate_config: -inf / -1e9 sentinels run.
MONOALIGN_API AlignmentMatrix align_unchecked(const LikelihoodBatch& batch, const MasConfig& cfg);

/// The per-column recurrence (reference parallel.hpp:39, parallel.cpp:25-31):
/// cur[i] = max(prev[i-1], prev[i]) + cur[i], prev[-1] read as `sentinel`.
/// Host columns in and out; computed by relax_column_kernel (mas_relax_column).
MONOALIGN_API void relax_column(const float* prev, float* cur, int lanes, float sentinel);
}  // namespace detail

}  // namespace monoalign::parallel
