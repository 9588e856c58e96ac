// C++ drop-in check: code written against the reference's public headers
// (include/monoalign/*.hpp of /root/reference/proj) compiles against this
// repo's include/monoalign/ and links libmonoalign_b200.so; the cases are
// the reference tests' known answers (test_reference.cpp, test_parallel.cpp,
// test_types.cpp, acceptance.cpp criterion 4).  Needs a GPU; run by
// tests/test_cpp_api.py.  Prints "ALL OK" and exits 0 on success.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <limits>
#include <random>
#include <string>

#include "monoalign/align.hpp"
#include "monoalign/bench.hpp"
#include "monoalign/parallel.hpp"
#include "monoalign/tensor_io.hpp"

#include <filesystem>
#include <variant>

namespace ma = monoalign;

static int g_fail = 0;
#define EXPECT(cond)                                                          \
  do {                                                                        \
    if (!(cond)) {                                                            \
      ++g_fail;                                                               \
      std::fprintf(stderr, "%s:%d: expectation failed: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                         \
  } while (0)

static bool throws_with(const std::function<void()>& f, ma::Errc code, const std::string& msg) {
  try {
    f();
  } catch (const ma::ValidationError& e) {
    const bool ok = e.code() == code && (msg.empty() || msg == e.what());
    if (!ok) std::fprintf(stderr, "  got %s: %s\n", ma::errc_name(e.code()), e.what());
    return ok;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "  unexpected exception: %s\n", e.what());
    return false;
  }
  return false;
}

static ma::LikelihoodBatch item(int t, int s, std::vector<float> v) {
  ma::LikelihoodBatch b(1, t, s);
  b.values = std::move(v);
  return b;
}

int main() {
  // 2x3 known answer: path [0, 1, 1] (test_reference.cpp:25-35).
  for (auto eng : {ma::EngineKind::Parallel, ma::EngineKind::Reference}) {
    ma::MasConfig cfg;
    cfg.engine = eng;
    const auto m = ma::align(item(2, 3, {1, 2, 3, 4, 5, 6}), cfg);
    EXPECT((m.values == std::vector<std::uint8_t>{1, 0, 0, 0, 1, 1}));
    EXPECT((ma::path_from_matrix(m, 0) == ma::PathVector{0, 1, 1}));
    EXPECT((ma::align_paths(item(2, 3, {1, 2, 3, 4, 5, 6}), cfg)[0] == ma::PathVector{0, 1, 1}));
  }
  // Tie rule on all zeros (test_parallel.cpp:78-83).
  EXPECT((ma::path_from_matrix(ma::align(item(3, 5, std::vector<float>(15, 0.f)))) ==
          ma::PathVector{0, 1, 2, 2, 2}));
  // t = 1 and t = s (test_reference.cpp:70-81).
  EXPECT((ma::path_from_matrix(ma::align(item(1, 4, {3, -1, 2, 0}))) == ma::PathVector{0, 0, 0, 0}));
  {
    std::vector<float> v(16);
    for (int k = 0; k < 16; ++k) v[k] = static_cast<float>((k * 7) % 5) - 2.f;
    EXPECT((ma::path_from_matrix(ma::align(item(4, 4, v))) == ma::PathVector{0, 1, 2, 3}));
  }
  // Engines agree; ragged items keep zeros outside their valid region.
  {
    std::mt19937 rng(99);
    std::uniform_real_distribution<float> u(-5.f, 5.f);
    ma::LikelihoodBatch b(8, 32, 64);
    for (auto& x : b.values) x = u(rng);
    b.lengths[3] = {10, 20};
    b.lengths[5] = {1, 64};
    ma::MasConfig ref;
    ref.engine = ma::EngineKind::Reference;
    const auto a = ma::parallel::align_parallel(b);
    const auto r = ma::reference::align_reference(b, ref);
    EXPECT(a == r);
    EXPECT(a.lengths == b.lengths);
    int outside = 0;
    for (int i = 0; i < 32; ++i)
      for (int j = 0; j < 64; ++j)
        if (i >= 10 || j >= 20) outside += a.at(3, i, j);
    EXPECT(outside == 0);
    const auto paths = ma::align_paths(b);
    EXPECT(paths[3].size() == 20u);
    EXPECT(paths[3] == ma::path_from_matrix(a, 3));
  }
  // Validation codes and messages (types.cpp:59-130).
  {
    ma::MasConfig bad;
    bad.max_neg_val = -1e9f;
    EXPECT(throws_with([&] { ma::align(item(2, 3, {1, 2, 3, 4, 5, 6}), bad); },
                       ma::Errc::InvalidConfig,
                       "max_neg_val must be finite and at most -1e+30, got -1e+09"));
    ma::MasConfig thr;
    thr.threads = -1;
    EXPECT(throws_with([&] { ma::validate_config(thr); }, ma::Errc::InvalidConfig,
                       "threads must be >= 0"));
    EXPECT(throws_with([&] { ma::align(item(3, 2, std::vector<float>(6, 0.f))); },
                       ma::Errc::InfeasibleLengths,
                       "item 0: text length 3 exceeds speech length 2; every text unit needs at "
                       "least one frame"));
    ma::LikelihoodBatch nan(3, 4, 9);
    nan.at(1, 2, 5) = std::numeric_limits<float>::quiet_NaN();
    nan.at(2, 0, 0) = std::numeric_limits<float>::infinity();
    EXPECT(throws_with([&] { ma::align(nan); }, ma::Errc::NonFinite,
                       "item 1: non-finite likelihood at (2, 5)"));
    EXPECT(throws_with([&] { ma::validate_item(nan, 2); }, ma::Errc::NonFinite,
                       "item 2: non-finite likelihood at (0, 0)"));
    EXPECT(throws_with([&] { ma::validate_batch(nan); }, ma::Errc::NonFinite,
                       "item 1: non-finite likelihood at (2, 5)"));
    ma::LikelihoodBatch z(2, 4, 9);
    z.lengths[1] = {0, 3};
    EXPECT(throws_with([&] { ma::align(z); }, ma::Errc::ZeroDim,
                       "item 1: valid lengths must be at least 1, got (0, 3)"));
    ma::LikelihoodBatch shp(2, 4, 9);
    shp.values.pop_back();
    EXPECT(throws_with([&] { ma::align(shp); }, ma::Errc::ShapeMismatch,
                       "container sizes do not match the declared dimensions"));
    EXPECT(throws_with([&] { ma::validate_path({0, 2, 2}, 3, 3); }, ma::Errc::InvalidPath,
                       "step of 2 at frame 1; only 0 and 1 are allowed"));
  }
  // Sentinel adversarial (acceptance.cpp:208-244): -1e32 never selects an
  // infeasible cell; the unchecked -1e9 reference engine does.
  {
    ma::LikelihoodBatch b(1, 32, 2048);
    for (int i = 0; i < 32; ++i)
      for (int j = 0; j < 2048; ++j) b.at(0, i, j) = i > j ? 1e8f : -1e8f;
    auto infeasible = [](const ma::AlignmentMatrix& m) {
      long n = 0;
      for (int i = 0; i < m.text_cap; ++i)
        for (int j = 0; j < m.speech_cap; ++j) n += m.at(0, i, j) != 0 && i > j;
      return n;
    };
    ma::MasConfig ref;
    ref.engine = ma::EngineKind::Reference;
    EXPECT(infeasible(ma::align(b)) == 0);
    EXPECT(infeasible(ma::align(b, ref)) == 0);
    ma::MasConfig weak = ref;
    weak.max_neg_val = -1e9f;
    EXPECT(infeasible(ma::reference::detail::align_unchecked(b, weak)) > 0);
  }
  // matrix_from_path / path_from_matrix round trip.
  {
    const ma::PathVector p{0, 0, 1, 2, 2, 3};
    EXPECT(ma::path_from_matrix(ma::matrix_from_path(p, 4, 6), 0) == p);
  }
  // bench::generate_random_batch: the counter-addressed splitmix64 stream.
  {
    const auto g = ma::bench::generate_random_batch(2, 3, 5, 7);
    std::uint64_t st = ma::bench::detail::mix_seed(7, 0);
    bool same = true;
    for (float v : g.values) {
      const double u = static_cast<double>(ma::bench::detail::splitmix64(st) >> 11) * 0x1.0p-53;
      same = same && v == static_cast<float>(-5.0 + 10.0 * u);
    }
    EXPECT(same);
    EXPECT(throws_with([] { ma::bench::generate_random_batch(1, 6, 5, 0); },
                       ma::Errc::InfeasibleLengths, "text length t exceeds speech length s"));
  }
  // io::write_tensor / read_tensor round trip and a budget rejection
  // (test_io.cpp cases), through include/monoalign/tensor_io.hpp.
  {
    const auto path = std::filesystem::temp_directory_path() / "mas_b200_cpp_io.bin";
    auto batch = ma::bench::generate_random_batch(2, 3, 4, 1);
    batch.lengths[1] = {2, 3};
    ma::io::write_tensor(path, batch);
    const ma::io::Tensor t = ma::io::read_tensor(path);
    const auto* back = std::get_if<ma::LikelihoodBatch>(&t);
    EXPECT(back && back->values == batch.values && back->lengths[1].text == 2 &&
           back->lengths[1].speech == 3);
    bool rejected = false;
    try {
      ma::io::read_tensor(path, 8);
    } catch (const ma::IoError& e) {
      rejected = e.code() == ma::Errc::DimensionOverflow;
    }
    EXPECT(rejected);
    const auto m = ma::align(batch);
    ma::io::write_tensor(path, m);
    const ma::io::Tensor t2 = ma::io::read_tensor(path);
    const auto* m2 = std::get_if<ma::AlignmentMatrix>(&t2);
    EXPECT(m2 && m2->values == m.values);
    std::filesystem::remove(path);
  }
  // forward_parallel score table, in place (test_parallel.cpp:44-68).
  {
    auto b = item(2, 3, {1, 2, 3, 4, 5, 6});
    ma::parallel::forward_parallel(ma::item_view(b, 0));
    EXPECT(b.values[0] == 1.0f && b.values[1] == 3.0f && b.values[2] == 6.0f);
    EXPECT(b.values[3] <= -1e30f && b.values[4] == 6.0f && b.values[5] == 12.0f);
    auto z = item(3, 5, std::vector<float>(15, 0.0f));
    ma::parallel::forward_parallel(ma::item_view(z, 0));
    for (int i = 0; i < 3; ++i)
      for (int j = i; j < 5; ++j) EXPECT(z.values[i * 5 + j] == 0.0f);
    auto one = item(1, 1, {7.0f});
    ma::parallel::forward_parallel(ma::item_view(one, 0));
    EXPECT(one.values[0] == 7.0f);
  }
  if (g_fail) {
    std::fprintf(stderr, "%d expectation(s) failed\n", g_fail);
    return 1;
  }
  std::printf("ALL OK\n");
  return 0;
}
