// mas_cli.cpp -- the `monoalign` command line (the reference's tools/main.cpp
// surface: subcommands align / verify / bench, the same options, defaults,
// checks and stable exit codes 0 ok, 1 IO/engine failure, 2 usage or
// validation error, 3 verification mismatch), over the B200 library.
//
//   align   MASTENS file -> monoalign::align on the GPU -> MASTENS file
//   verify  both device engines against an exhaustive enumeration of every
//           monotonic path (double accumulation; the checker of
//           tools/main.cpp:84-132 / src/oracle.cpp), on random small items
//   bench   monoalign::bench::run_bench (csrc/mas_bench.cpp), CSV or Markdown
//
// The reference parses with CLI11 (not vendored in /root/reference); this is a
// small parser of its own with the same observable behaviour for the options
// above (`--opt value` and `--opt=value`, comma-delimited lists, --help).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <variant>
#include <vector>

#include "monoalign/align.hpp"
#include "monoalign/bench.hpp"
#include "monoalign/tensor_io.hpp"

namespace {

constexpr int kExitOk = 0;
constexpr int kExitIo = 1;
constexpr int kExitUsage = 2;
constexpr int kExitMismatch = 3;

struct Usage {
  std::string what;
};

// ---- option table -----------------------------------------------------------

struct Option {
  std::string name;  // "--input"
  std::string help;
  bool flag = false;
  bool required = false;
  std::function<void(const std::string&)> set;  // throws Usage on a bad value
  bool seen = false;
};

struct Command {
  std::string name;
  std::string help;
  std::vector<Option> options;

  void print_help(std::ostream& os) const {
    os << "monoalign " << name << ": " << help << "\nOptions:\n  -h,--help\n";
    for (const Option& o : options)
      os << "  " << o.name << (o.flag ? "" : " VALUE") << (o.required ? " (required)" : "")
         << "\n      " << o.help << "\n";
  }

  // Returns false when --help was given.
  bool parse(const std::vector<std::string>& args) {
    for (std::size_t k = 0; k < args.size(); ++k) {
      std::string a = args[k];
      if (a == "-h" || a == "--help") return false;
      std::optional<std::string> inline_value;
      if (const auto eq = a.find('='); a.rfind("--", 0) == 0 && eq != std::string::npos) {
        inline_value = a.substr(eq + 1);
        a = a.substr(0, eq);
      }
      auto it = std::find_if(options.begin(), options.end(), [&](const Option& o) { return o.name == a; });
      if (it == options.end()) throw Usage{"the following argument was not expected: " + args[k]};
      it->seen = true;
      if (it->flag) {
        it->set("1");
        continue;
      }
      if (!inline_value) {
        if (k + 1 >= args.size()) throw Usage{a + " requires a value"};
        inline_value = args[++k];
      }
      it->set(*inline_value);
    }
    for (const Option& o : options)
      if (o.required && !o.seen) throw Usage{o.name + " is required"};
    return true;
  }
};

long long to_int(const std::string& name, const std::string& v) {
  char* end = nullptr;
  errno = 0;
  const long long x = std::strtoll(v.c_str(), &end, 10);
  if (v.empty() || *end != '\0' || errno) throw Usage{name + ": value " + v + " is not an integer"};
  return x;
}

std::uint64_t to_u64(const std::string& name, const std::string& v) {
  char* end = nullptr;
  errno = 0;
  const unsigned long long x = std::strtoull(v.c_str(), &end, 10);
  if (v.empty() || v[0] == '-' || *end != '\0' || errno)
    throw Usage{name + ": value " + v + " is not an unsigned integer"};
  return x;
}

double to_double(const std::string& name, const std::string& v) {
  char* end = nullptr;
  const double x = std::strtod(v.c_str(), &end);
  if (v.empty() || *end != '\0') throw Usage{name + ": value " + v + " is not a number"};
  return x;
}

int checked_int(const std::string& name, const std::string& v, long long lo, long long hi) {
  const long long x = to_int(name, v);
  if (x < lo || x > hi)
    throw Usage{name + ": value " + v + " not in range [" + std::to_string(lo) + " - " +
                std::to_string(hi) + "]"};
  return static_cast<int>(x);
}

std::vector<std::string> split_commas(const std::string& v) {
  std::vector<std::string> parts;
  std::stringstream ss(v);
  for (std::string p; std::getline(ss, p, ',');) parts.push_back(p);
  return parts;
}

std::string engine_member(const std::string& name, const std::string& v) {
  if (v != "reference" && v != "parallel")
    throw Usage{name + ": " + v + " not in {reference,parallel}"};
  return v;
}

monoalign::EngineKind engine_of(const std::string& v) {
  return v == "reference" ? monoalign::EngineKind::Reference : monoalign::EngineKind::Parallel;
}

constexpr int kIntMax = 0x7fffffff;

// ---- align ------------------------------------------------------------------

struct AlignArgs {
  std::string input, output, engine = "parallel";
  double neg_val = static_cast<double>(monoalign::kDefaultMaxNegVal);
  int threads = 0;
};

int run_align(const AlignArgs& a) {
  monoalign::io::Tensor tensor = monoalign::io::read_tensor(a.input);
  const auto* batch = std::get_if<monoalign::LikelihoodBatch>(&tensor);
  if (!batch)
    throw monoalign::ValidationError(
        monoalign::Errc::ShapeMismatch,
        a.input + " holds a uint8 alignment tensor; align needs float32 likelihoods");
  monoalign::MasConfig cfg;
  cfg.engine = engine_of(a.engine);
  cfg.max_neg_val = static_cast<float>(a.neg_val);
  cfg.threads = a.threads;
  monoalign::io::write_tensor(a.output, monoalign::align(*batch, cfg));
  return kExitOk;
}

// ---- verify -----------------------------------------------------------------

struct VerifyArgs {
  int trials = 1000, t_max = 6, s_max = 10;
  std::uint64_t seed = 0;
  bool inject_fault = false;
};

// Every monotonic path of a t x s item (path[0] = 0, path[s-1] = t-1, each
// step stays or climbs one row), scored in double; returns the maximum and
// every path within 1e-9 of it (the reference oracle's contract,
// include/monoalign/oracle.hpp:12-36).
struct Optima {
  double best = -INFINITY;
  std::vector<monoalign::PathVector> paths;
};

void enumerate(const monoalign::LikelihoodView& q, monoalign::PathVector& path, int j, double sum,
               std::vector<std::pair<double, monoalign::PathVector>>& all) {
  const int t = q.text, s = q.speech;
  const int i = path[j];
  sum += static_cast<double>(q.at(i, j));
  if (j == s - 1) {
    if (i == t - 1) all.emplace_back(sum, path);
    return;
  }
  for (int next = i; next <= std::min(i + 1, t - 1); ++next) {
    if (t - 1 - next > s - 2 - j) continue;  // cannot reach the last row any more
    path[j + 1] = next;
    enumerate(q, path, j + 1, sum, all);
  }
}

Optima exhaustive(const monoalign::LikelihoodView& q) {
  std::vector<std::pair<double, monoalign::PathVector>> all;
  monoalign::PathVector path(static_cast<std::size_t>(q.speech), 0);
  enumerate(q, path, 0, 0.0, all);
  Optima o;
  for (const auto& [score, p] : all) o.best = std::max(o.best, score);
  for (const auto& [score, p] : all)
    if (std::abs(score - o.best) <= 1e-9) o.paths.push_back(p);
  return o;
}

int run_verify(const VerifyArgs& a) {
  using monoalign::bench::detail::mix_seed;
  using monoalign::bench::detail::splitmix64;
  int pass = 0, fail = 0;
  for (int k = 0; k < a.trials; ++k) {
    // instance dimensions drawn as tools/main.cpp:89-95 draws them
    const std::uint64_t seed = mix_seed(a.seed, static_cast<std::uint64_t>(k));
    std::uint64_t st = seed;
    const int t = std::min(1 + static_cast<int>(splitmix64(st) % static_cast<std::uint64_t>(a.t_max)),
                           a.s_max);
    const int s = t + static_cast<int>(splitmix64(st) % static_cast<std::uint64_t>(a.s_max - t + 1));
    const monoalign::LikelihoodBatch batch = monoalign::bench::generate_random_batch(1, t, s, seed);
    const monoalign::LikelihoodView q = monoalign::item_view(batch, 0);
    const monoalign::PathVector ref =
        monoalign::path_from_matrix(monoalign::reference::align_reference(batch));
    monoalign::PathVector par =
        monoalign::path_from_matrix(monoalign::parallel::align_parallel(batch));
    if (a.inject_fault && !par.empty()) par.back() += par.back() > 0 ? -1 : 1;
    const Optima best = exhaustive(q);
    double score = 0.0;
    for (int j = 0; j < s; ++j) score += static_cast<double>(q.at(ref[j], j));
    bool ok = std::abs(score - best.best) <= 1e-5 * std::max(1.0, std::abs(best.best)) && par == ref;
    if (ok && best.paths.size() == 1) ok = ref == best.paths.front();
    if (ok) {
      ++pass;
    } else {
      ++fail;
      std::cerr << "mismatch: seed=" << seed << " t=" << t << " s=" << s
                << " engine_score=" << score << " oracle_score=" << best.best << "\n";
    }
  }
  std::cout << "trials " << a.trials << " pass " << pass << " fail " << fail << "\n";
  return fail == 0 ? kExitOk : kExitMismatch;
}

// ---- bench ------------------------------------------------------------------

struct BenchArgs {
  monoalign::bench::BenchPlan plan;
  std::string format = "csv", out = "-";
};

int run_bench(const BenchArgs& a) {
  const auto report = monoalign::bench::run_bench(a.plan);
  const std::string text = monoalign::bench::emit_report(
      report, a.format == "markdown" ? monoalign::bench::ReportFormat::Markdown
                                     : monoalign::bench::ReportFormat::Csv);
  if (a.out == "-") {
    std::cout << text;
    return kExitOk;
  }
  std::ofstream f(a.out);
  f << text;
  f.flush();
  if (!f) throw monoalign::IoError(monoalign::Errc::IoFailure, "cannot write report: " + a.out);
  return kExitOk;
}

void print_top_help(std::ostream& os) {
  os << "monotonic alignment toolkit (B200 engines)\n"
        "Usage: monoalign SUBCOMMAND [OPTIONS]\n"
        "Subcommands:\n"
        "  align    align a likelihood tensor file\n"
        "  verify   check both engines against the exhaustive oracle\n"
        "  bench    timing sweep over instance sizes\n";
}

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> args(argv + 1, argv + argc);
  AlignArgs al;
  VerifyArgs ve;
  BenchArgs be;
  std::map<std::string, Command> cmds;
  cmds["align"] = {"align", "align a likelihood tensor file",
                   {{"--input", "input tensor file", false, true, [&](const std::string& v) { al.input = v; }},
                    {"--output", "output tensor file", false, true, [&](const std::string& v) { al.output = v; }},
                    {"--engine", "engine to run (reference|parallel, default parallel)", false, false,
                     [&](const std::string& v) { al.engine = engine_member("--engine", v); }},
                    {"--neg-val", "sentinel for infeasible cells (default -1e32)", false, false,
                     [&](const std::string& v) { al.neg_val = to_double("--neg-val", v); }},
                    {"--threads", "accepted for compatibility (the GPU sets its parallelism)", false, false,
                     [&](const std::string& v) { al.threads = checked_int("--threads", v, -kIntMax, kIntMax); }}}};
  cmds["verify"] = {"verify", "check both engines against the exhaustive oracle",
                    {{"--trials", "random instances to run (default 1000)", false, false,
                      [&](const std::string& v) { ve.trials = checked_int("--trials", v, 1, kIntMax); }},
                     {"--t-max", "max text length, 1..6 (default 6)", false, false,
                      [&](const std::string& v) { ve.t_max = checked_int("--t-max", v, 1, 6); }},
                     {"--s-max", "max speech length, 1..10 (default 10)", false, false,
                      [&](const std::string& v) { ve.s_max = checked_int("--s-max", v, 1, 10); }},
                     {"--seed", "base seed (default 0)", false, false,
                      [&](const std::string& v) { ve.seed = to_u64("--seed", v); }},
                     {"--inject-fault", "perturb the parallel path (self-test)", true, false,
                      [&](const std::string&) { ve.inject_fault = true; }}}};
  cmds["bench"] = {"bench", "timing sweep over instance sizes",
                   {{"--t-values", "text lengths to sweep, comma separated", false, false,
                     [&](const std::string& v) {
                       be.plan.t_values.clear();
                       for (const auto& p : split_commas(v))
                         be.plan.t_values.push_back(checked_int("--t-values", p, 1, kIntMax));
                     }},
                    {"--batch-size", "items per batch (default 32)", false, false,
                     [&](const std::string& v) { be.plan.batch_size = checked_int("--batch-size", v, 1, kIntMax); }},
                    {"--s-ratio", "speech length as multiple of T (default 4)", false, false,
                     [&](const std::string& v) { be.plan.s_ratio = checked_int("--s-ratio", v, 1, kIntMax); }},
                    {"--repeats", "timed runs per configuration (default 20)", false, false,
                     [&](const std::string& v) { be.plan.repeats = checked_int("--repeats", v, 1, kIntMax); }},
                    {"--warmup", "discarded runs per configuration (default 3)", false, false,
                     [&](const std::string& v) { be.plan.warmup = checked_int("--warmup", v, 0, kIntMax); }},
                    {"--engines", "engines to time, comma separated (default reference,parallel)", false, false,
                     [&](const std::string& v) {
                       be.plan.engines.clear();
                       for (const auto& p : split_commas(v))
                         be.plan.engines.push_back(engine_of(engine_member("--engines", p)));
                     }},
                    {"--seed", "base seed (default 0)", false, false,
                     [&](const std::string& v) { be.plan.seed = to_u64("--seed", v); }},
                    {"--threads", "accepted for compatibility", false, false,
                     [&](const std::string& v) { be.plan.threads = checked_int("--threads", v, -kIntMax, kIntMax); }},
                    {"--format", "report format (csv|markdown, default csv)", false, false,
                     [&](const std::string& v) {
                       if (v != "csv" && v != "markdown") throw Usage{"--format: " + v + " not in {csv,markdown}"};
                       be.format = v;
                     }},
                    {"--out", "report destination (- = stdout)", false, false,
                     [&](const std::string& v) { be.out = v; }}}};

  std::string sub;
  try {
    if (!args.empty() && (args[0] == "-h" || args[0] == "--help")) {
      print_top_help(std::cout);
      return kExitOk;
    }
    if (args.empty()) throw Usage{"A subcommand is required"};
    sub = args[0];
    const auto it = cmds.find(sub);
    if (it == cmds.end()) throw Usage{"the following argument was not expected: " + sub};
    if (!it->second.parse({args.begin() + 1, args.end()})) {
      it->second.print_help(std::cout);
      return kExitOk;
    }
  } catch (const Usage& u) {
    std::cerr << u.what << "\nRun with --help for more information.\n";
    return kExitUsage;
  }

  try {
    if (sub == "align") return run_align(al);
    if (sub == "verify") return run_verify(ve);
    return run_bench(be);
  } catch (const monoalign::ValidationError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const monoalign::IoError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitIo;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitIo;
  }
}
