// monoalign/tensor_io.hpp -- MASTENS v1 tensor files of the drop-in C++ API.
//
// Same names and behaviour as the reference's include/monoalign/tensor_io.hpp
// (layout :11-23, kHeaderSize, kDefaultByteBudget, Tensor, write_tensor,
// read_tensor): the header is fully validated, including the byte budget,
// before the payload is allocated; failures throw IoError with the
// reference's code and text.  Implemented over mas_io_* (include/monoalign_b200.h).
#pragma once

#include <cstddef>
#include <filesystem>
#include <variant>

#include "monoalign/types.hpp"

namespace monoalign::io {

inline constexpr std::size_t kHeaderSize = 39;
inline constexpr std::size_t kDefaultByteBudget = std::size_t{1} << 30;

using Tensor = std::variant<LikelihoodBatch, AlignmentMatrix>;

MONOALIGN_API void write_tensor(const std::filesystem::path& path, const LikelihoodBatch& batch);
MONOALIGN_API void write_tensor(const std::filesystem::path& path, const AlignmentMatrix& m);

MONOALIGN_API Tensor read_tensor(const std::filesystem::path& path,
                                 std::size_t byte_budget = kDefaultByteBudget);

}  // namespace monoalign::io
