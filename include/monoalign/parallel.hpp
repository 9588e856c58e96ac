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
/// (forward_scores_kernel via mas_forward_scores), the item round-tripping
/// through device memory.
MONOALIGN_API void forward_parallel(MutableLikelihoodView q, const MasConfig& cfg = {});

MONOALIGN_API AlignmentMatrix align_parallel(const LikelihoodBatch& batch,
                                             const MasConfig& cfg = {});

namespace detail {
/// align_parallel without validate_config: -inf / -1e9 sentinels run.
MONOALIGN_API AlignmentMatrix align_unchecked(const LikelihoodBatch& batch, const MasConfig& cfg);
}  // namespace detail

}  // namespace monoalign::parallel
