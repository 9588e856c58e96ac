// monoalign/align.hpp -- the maximum-path call (reference
// include/monoalign/align.hpp:9-12), served by the sm_100a kernels through
// the C-ABI of include/monoalign_b200.h.
#pragma once

#include "monoalign/parallel.hpp"
#include "monoalign/reference.hpp"

namespace monoalign {

/// Engine dispatch on cfg.engine; both engines run on the current CUDA
/// device and produce the reference engines' alignments bit for bit.
inline AlignmentMatrix align(const LikelihoodBatch& batch, const MasConfig& cfg = {}) {
  return cfg.engine == EngineKind::Reference ? reference::align_reference(batch, cfg)
                                             : parallel::align_parallel(batch, cfg);
}

/// align() returning one path per item (what the Python align_paths
/// returns), computed on the device without the dense matrix.
MONOALIGN_API std::vector<PathVector> align_paths(const LikelihoodBatch& batch,
                                                  const MasConfig& cfg = {});

}  // namespace monoalign
