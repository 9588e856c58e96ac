// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference
// library (/root/reference/proj/src/*.cpp compiled in place by
// oracle/Makefile into oracle/_ref/libmonoalign_ref.so).
//
// TEST INFRASTRUCTURE ONLY: used by tests/ to pin the oracle restatement and
// the CUDA path against the reference itself, and by bench.py's
// `--impl reference` / cpu_baseline legs to time the reference CPU engines.
// Never loaded by the product library.
//
// Calls go through the reference's own public C++ API:
//   monoalign::align                     include/monoalign/align.hpp:9-12
//   parallel::detail::align_unchecked    include/monoalign/parallel.hpp:29-31
//   reference::detail::align_unchecked   include/monoalign/reference.hpp:42-44
//   path_from_matrix                     include/monoalign/types.hpp:155-158
//   bench::generate_random_batch         include/monoalign/bench.hpp:58
//   oracle::best_paths                   include/monoalign/oracle.hpp:33
//   io::write_tensor / io::read_tensor   include/monoalign/tensor_io.hpp:29-36
//   parallel::forward_parallel           include/monoalign/parallel.hpp:17
//   reference::forward_reference         include/monoalign/reference.hpp:33
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>

#include "monoalign/align.hpp"
#include "monoalign/bench.hpp"
#include "monoalign/oracle.hpp"
#include "monoalign/parallel.hpp"
#include "monoalign/reference.hpp"
#include "monoalign/tensor_io.hpp"

namespace {

void put_msg(const std::string& s, char* buf, int cap) {
  if (!buf || cap <= 0) return;
  std::size_t n = s.size() < static_cast<std::size_t>(cap - 1) ? s.size() : cap - 1;
  std::memcpy(buf, s.data(), n);
  buf[n] = '\0';
}

}  // namespace

extern "C" {

/// Returns -1 on success, else the Errc value (errors.hpp:8-30 order) with
/// the exception text copied to msg.  unchecked=1 routes through
/// detail::align_unchecked (no validate_config), the only way to run -inf /
/// -1e9 sentinels.
int ref_align(const float* q, int B, int T, int S, const std::int64_t* lengths, int engine,
              float max_neg_val, int threads, int unchecked, std::uint8_t* out,
              std::int32_t* paths, char* msg, int msg_cap) {
  try {
    monoalign::LikelihoodBatch batch(B, T, S);
    std::memcpy(batch.values.data(), q, batch.values.size() * sizeof(float));
    if (lengths) {
      for (int b = 0; b < B; ++b) {
        batch.lengths[b] = {static_cast<std::uint32_t>(lengths[2 * b]),
                            static_cast<std::uint32_t>(lengths[2 * b + 1])};
      }
    }
    monoalign::MasConfig cfg;
    cfg.engine = engine == 1 ? monoalign::EngineKind::Reference : monoalign::EngineKind::Parallel;
    cfg.max_neg_val = max_neg_val;
    cfg.threads = threads;
    monoalign::AlignmentMatrix m;
    if (unchecked) {
      m = engine == 1 ? monoalign::reference::detail::align_unchecked(batch, cfg)
                      : monoalign::parallel::detail::align_unchecked(batch, cfg);
    } else {
      m = monoalign::align(batch, cfg);
    }
    if (out) std::memcpy(out, m.values.data(), m.values.size());
    if (paths) {
      for (int b = 0; b < B; ++b) {
        const monoalign::PathVector p = monoalign::path_from_matrix(m, b);
        for (int j = 0; j < S; ++j) {
          paths[static_cast<std::size_t>(b) * S + j] =
              j < static_cast<int>(p.size()) ? p[static_cast<std::size_t>(j)] : -1;
        }
      }
    }
    return -1;
  } catch (const monoalign::Error& e) {
    put_msg(e.what(), msg, msg_cap);
    return static_cast<int>(e.code());
  } catch (const std::exception& e) {
    put_msg(e.what(), msg, msg_cap);
    return 1000;
  }
}

/// bench::generate_random_batch(b, t, s, seed) into out[b*t*s].
int ref_generate(int b, int t, int s, std::uint64_t seed, float* out) {
  try {
    const monoalign::LikelihoodBatch batch = monoalign::bench::generate_random_batch(b, t, s, seed);
    std::memcpy(out, batch.values.data(), batch.values.size() * sizeof(float));
    return -1;
  } catch (const monoalign::Error& e) {
    return static_cast<int>(e.code());
  }
}

std::uint64_t ref_mix_seed(std::uint64_t seed, std::uint64_t index) {
  return monoalign::bench::detail::mix_seed(seed, index);
}

std::uint64_t ref_splitmix64(std::uint64_t* state) {
  return monoalign::bench::detail::splitmix64(*state);
}

/// Exhaustive oracle (oracle.cpp): number of optimal paths (<= cap copied
/// into paths[cap][s]) and the fp64 maximum score.  Returns -1 or Errc.
int ref_best_paths(const float* q, int t, int s, double* max_score, int* n_paths,
                   std::int32_t* paths, int cap) {
  try {
    const monoalign::LikelihoodView view{q, t, s, s};
    const monoalign::oracle::BestPaths best = monoalign::oracle::best_paths(view);
    *max_score = best.max_score;
    *n_paths = static_cast<int>(best.paths.size());
    for (int k = 0; k < cap && k < *n_paths; ++k) {
      std::memcpy(paths + static_cast<std::size_t>(k) * s, best.paths[k].data(),
                  sizeof(std::int32_t) * s);
    }
    return -1;
  } catch (const monoalign::Error& e) {
    return static_cast<int>(e.code());
  }
}

/// parallel::forward_parallel on one [t][s] item (row stride `stride`), in
/// place: the parallel engine's score table.
void ref_forward_parallel(float* q, int t, int s, std::int64_t stride, float max_neg_val) {
  monoalign::MasConfig cfg;
  cfg.max_neg_val = max_neg_val;
  monoalign::parallel::forward_parallel(monoalign::MutableLikelihoodView{q, t, s, stride}, cfg);
}

/// reference::forward_reference on one [t][s] item (row stride `stride`):
/// the reference engine's QCache, copied to `out` [t][s] (reference.hpp:33).
void ref_forward_reference(const float* q, int t, int s, std::int64_t stride, float max_neg_val,
                           float* out) {
  monoalign::MasConfig cfg;
  cfg.max_neg_val = max_neg_val;
  const monoalign::reference::QCache c =
      monoalign::reference::forward_reference(monoalign::LikelihoodView{q, t, s, stride}, cfg);
  for (int i = 0; i < t; ++i)
    for (int j = 0; j < s; ++j) out[static_cast<std::size_t>(i) * s + j] = c.at(i, j);
}

unsigned ref_hardware_threads() { return std::thread::hardware_concurrency(); }

/// Timing harness for bench.py's reference arm / cpu_baseline: a pre-built
/// LikelihoodBatch (bench::generate_random_batch) and monoalign::align timed
/// alone with steady_clock, as the reference's own bench does
/// (bench.cpp:275-303, timing :293-296).
void* ref_batch_create(int b, int t, int s, std::uint64_t seed) {
  try {
    return new monoalign::LikelihoodBatch(monoalign::bench::generate_random_batch(b, t, s, seed));
  } catch (...) {
    return nullptr;
  }
}

void ref_batch_destroy(void* batch) { delete static_cast<monoalign::LikelihoodBatch*>(batch); }

/// One monoalign::align call on the batch; returns milliseconds, < 0 on error.
/// `checksum` (optional) receives the sum of path rows, so the work is used.
double ref_batch_time_align(void* batch, int engine, int threads, std::int64_t* checksum) {
  const auto& bt = *static_cast<monoalign::LikelihoodBatch*>(batch);
  monoalign::MasConfig cfg;
  cfg.engine = engine == 1 ? monoalign::EngineKind::Reference : monoalign::EngineKind::Parallel;
  cfg.threads = threads;
  try {
    const auto t0 = std::chrono::steady_clock::now();
    const monoalign::AlignmentMatrix m = monoalign::align(bt, cfg);
    const auto t1 = std::chrono::steady_clock::now();
    if (checksum) {
      std::int64_t acc = 0;
      for (std::size_t k = 0; k < m.values.size(); k += 4099) acc += m.values[k];
      *checksum = acc;
    }
    return std::chrono::duration<double, std::milli>(t1 - t0).count();
  } catch (...) {
    return -1.0;
  }
}

/// io::write_tensor of a LikelihoodBatch (dtype 0) or AlignmentMatrix
/// (dtype 1) built from values / lengths ([B][2] u32 or null = full).
int ref_tensor_write(const char* path, int dtype, int B, int T, int S, const void* values,
                     const std::uint32_t* lengths, char* msg, int msg_cap) {
  try {
    auto fill = [&](auto& c) {
      std::memcpy(c.values.data(), values, c.values.size() * sizeof(c.values[0]));
      if (lengths)
        for (int b = 0; b < B; ++b) c.lengths[b] = {lengths[2 * b], lengths[2 * b + 1]};
    };
    if (dtype == 0) {
      monoalign::LikelihoodBatch batch(B, T, S);
      fill(batch);
      monoalign::io::write_tensor(path, batch);
    } else {
      monoalign::AlignmentMatrix m(B, T, S);
      fill(m);
      monoalign::io::write_tensor(path, m);
    }
    return -1;
  } catch (const monoalign::Error& e) {
    put_msg(e.what(), msg, msg_cap);
    return static_cast<int>(e.code());
  } catch (const std::exception& e) {
    put_msg(e.what(), msg, msg_cap);
    return 1000;
  }
}

/// io::read_tensor(path, budget): dtype, dims and (if non-null) the payload
/// and lengths table copied out.
int ref_tensor_read(const char* path, std::uint64_t budget, int* dtype, std::int64_t* dims,
                    void* values, std::uint32_t* lengths, char* msg, int msg_cap) {
  try {
    const monoalign::io::Tensor t = monoalign::io::read_tensor(path, budget);
    auto out = [&](const auto& c, int code) {
      *dtype = code;
      dims[0] = c.batch;
      dims[1] = c.text_cap;
      dims[2] = c.speech_cap;
      if (values) std::memcpy(values, c.values.data(), c.values.size() * sizeof(c.values[0]));
      if (lengths)
        for (int b = 0; b < c.batch; ++b) {
          lengths[2 * b] = c.lengths[b].text;
          lengths[2 * b + 1] = c.lengths[b].speech;
        }
    };
    if (const auto* batch = std::get_if<monoalign::LikelihoodBatch>(&t))
      out(*batch, 0);
    else
      out(std::get<monoalign::AlignmentMatrix>(t), 1);
    return -1;
  } catch (const monoalign::Error& e) {
    put_msg(e.what(), msg, msg_cap);
    return static_cast<int>(e.code());
  } catch (const std::exception& e) {
    put_msg(e.what(), msg, msg_cap);
    return 1000;
  }
}

}  // extern "C"
