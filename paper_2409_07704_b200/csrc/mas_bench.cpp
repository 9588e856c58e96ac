// mas_bench.cpp -- the timing harness of the reference's bench.hpp:12-77
// (src/bench.cpp:17-307 defines the protocol and the report formats) over the
// device engines.  Host-side bookkeeping only: every timed call is
// monoalign::align, i.e. the sm_100a kernels behind mas_align_host with the
// host containers copied in and out, timed by wall clock around that call
// alone (the reference's protocol, bench.cpp:283-290), so rows are directly
// comparable with the reference CLI's CSV.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <fstream>
#include <iomanip>
#include <numeric>
#include <sstream>
#include <thread>

#include <cuda_runtime.h>

#include "monoalign/align.hpp"
#include "monoalign/bench.hpp"

namespace monoalign::bench {

namespace {

// bench.cpp:19-38: the checks and their order.
void check_plan(const BenchPlan& plan) {
  const char* problem = nullptr;
  if (std::any_of(plan.t_values.begin(), plan.t_values.end(), [](int t) { return t < 1; }))
    problem = "t values must be at least 1";
  else if (plan.batch_size < 1)
    problem = "batch size must be at least 1";
  else if (plan.s_ratio < 1)
    problem = "s ratio must be at least 1";
  else if (plan.repeats < 1)
    problem = "repeats must be at least 1";
  else if (plan.warmup < 0)
    problem = "warmup cannot be negative";
  if (problem) throw ValidationError(Errc::InvalidConfig, std::string("bench plan: ") + problem);
}

// Quantile q in [0, 1] of an ascending sample, interpolating linearly
// between the two nearest ranks (rank = q * (n - 1)).
double quantile(const std::vector<double>& asc, double q) {
  const double pos = q * static_cast<double>(asc.size() - 1);
  const std::size_t k = static_cast<std::size_t>(pos);
  if (k + 1 >= asc.size()) return asc.back();
  return asc[k] + (pos - static_cast<double>(k)) * (asc[k + 1] - asc[k]);
}

std::string ms4(double v) {
  std::ostringstream o;
  o << std::fixed << std::setprecision(4) << v;
  return o.str();
}

std::string device_name() {
  int dev = 0;
  cudaDeviceProp prop;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&prop, dev) != cudaSuccess) {
    cudaGetLastError();
    return "no CUDA device";
  }
  std::ostringstream o;
  o << prop.name << ", sm_" << prop.major << prop.minor;
  return o.str();
}

}  // namespace

std::vector<int> default_t_values() {
  std::vector<int> ts(16);
  for (int k = 0; k < 16; ++k) ts[k] = 128 * (k + 1);
  return ts;
}

BenchReport run_bench(const BenchPlan& plan) {
  return detail::run_bench_with(
      plan, [](const LikelihoodBatch& batch, const MasConfig& cfg) { return align(batch, cfg); });
}

namespace detail {

BenchReport run_bench_with(const BenchPlan& plan, const AlignFn& align_fn) {
  check_plan(plan);
  BenchReport report;
  report.env = collect_env_info();
  using clock = std::chrono::steady_clock;
  for (const int t : plan.t_values) {
    const int s = t * plan.s_ratio;
    const LikelihoodBatch batch =
        generate_random_batch(plan.batch_size, t, s, mix_seed(plan.seed, static_cast<std::uint64_t>(t)));
    for (const EngineKind engine : plan.engines) {
      MasConfig cfg;
      cfg.engine = engine;
      cfg.threads = plan.threads;
      for (int w = 0; w < plan.warmup; ++w) (void)align_fn(batch, cfg);
      std::vector<double> ms(static_cast<std::size_t>(plan.repeats));
      for (double& m : ms) {
        const clock::time_point t0 = clock::now();
        const AlignmentMatrix out = align_fn(batch, cfg);
        m = std::chrono::duration<double, std::milli>(clock::now() - t0).count();
        (void)out;
      }
      std::sort(ms.begin(), ms.end());
      BenchRow row;
      row.engine = engine;
      row.t = t;
      row.s = s;
      row.b = plan.batch_size;
      row.mean_ms = std::accumulate(ms.begin(), ms.end(), 0.0) / static_cast<double>(ms.size());
      row.p20_ms = quantile(ms, 0.2);
      row.median_ms = quantile(ms, 0.5);
      row.p80_ms = quantile(ms, 0.8);
      report.rows.push_back(row);
    }
  }
  return report;
}

}  // namespace detail

std::string emit_report(const BenchReport& report, ReportFormat format) {
  if (report.rows.empty()) throw ValidationError(Errc::EmptyReport, "report has no rows");
  const EnvInfo& env = report.env;
  std::ostringstream o;
  if (format == ReportFormat::Csv) {
    o << "# cpu: " << env.cpu_model << "\n# hardware_threads: " << env.hardware_threads
      << "\n# compiler: " << env.compiler << "\n# build: " << env.build << "\n";
    o << "engine,T,S,B,mean_ms,median_ms,p20_ms,p80_ms\n";
    for (const BenchRow& r : report.rows)
      o << engine_name(r.engine) << ',' << r.t << ',' << r.s << ',' << r.b << ',' << ms4(r.mean_ms)
        << ',' << ms4(r.median_ms) << ',' << ms4(r.p20_ms) << ',' << ms4(r.p80_ms) << '\n';
    return o.str();
  }
  // Markdown: engines in order of first appearance as columns, T ascending as rows.
  std::vector<EngineKind> engines;
  std::vector<int> ts;
  for (const BenchRow& r : report.rows) {
    if (std::find(engines.begin(), engines.end(), r.engine) == engines.end())
      engines.push_back(r.engine);
    if (std::find(ts.begin(), ts.end(), r.t) == ts.end()) ts.push_back(r.t);
  }
  std::sort(ts.begin(), ts.end());
  auto lookup = [&](EngineKind e, int t) -> const BenchRow* {
    for (const BenchRow& r : report.rows)
      if (r.engine == e && r.t == t) return &r;
    return nullptr;
  };
  o << "CPU: " << env.cpu_model << " (" << env.hardware_threads << " hardware threads)\n";
  o << "Compiler: " << env.compiler << ", " << env.build << " build\n\n";
  o << "| T | S | B |";
  for (EngineKind e : engines) o << ' ' << engine_name(e) << " median (ms) |";
  o << "\n|---|---|---|";
  for (std::size_t k = 0; k < engines.size(); ++k) o << "---|";
  o << '\n';
  for (const int t : ts) {
    const BenchRow* first = nullptr;
    for (EngineKind e : engines)
      if (!first) first = lookup(e, t);
    o << "| " << t << " | " << first->s << " | " << first->b << " |";
    for (EngineKind e : engines) {
      const BenchRow* r = lookup(e, t);
      o << ' ' << (r ? ms4(r->median_ms) : std::string("-")) << " |";
    }
    o << '\n';
  }
  return o.str();
}

ScalingFit fit_scaling(const BenchReport& report, EngineKind engine) {
  std::vector<std::pair<double, double>> pts;  // (T*S cells, median ms)
  for (const BenchRow& r : report.rows)
    if (r.engine == engine) pts.emplace_back(static_cast<double>(r.t) * r.s, r.median_ms);
  std::vector<double> sizes;
  for (const auto& p : pts) sizes.push_back(p.first);
  std::sort(sizes.begin(), sizes.end());
  const auto distinct = std::unique(sizes.begin(), sizes.end()) - sizes.begin();
  if (distinct < 4)
    throw ValidationError(Errc::InsufficientPoints, "scaling fit needs at least 4 distinct sizes, got " +
                                                        std::to_string(distinct));
  const double n = static_cast<double>(pts.size());
  double mx = 0, my = 0;
  for (const auto& [x, y] : pts) {
    mx += x / n;
    my += y / n;
  }
  double sxx = 0, sxy = 0;
  for (const auto& [x, y] : pts) {
    sxx += (x - mx) * (x - mx);
    sxy += (x - mx) * (y - my);
  }
  ScalingFit fit;
  fit.slope_ms_per_cell = sxy / sxx;
  double res = 0, tot = 0;
  for (const auto& [x, y] : pts) {
    const double e = y - (my + fit.slope_ms_per_cell * (x - mx));
    res += e * e;
    tot += (y - my) * (y - my);
  }
  fit.r_squared = tot > 0 ? 1.0 - res / tot : 0.0;
  return fit;
}

EnvInfo collect_env_info() {
  EnvInfo env;
  env.cpu_model = "unknown";
  std::ifstream cpuinfo("/proc/cpuinfo");
  for (std::string line; std::getline(cpuinfo, line);) {
    if (line.compare(0, 10, "model name") != 0) continue;
    const auto colon = line.find(':');
    const auto start = colon == std::string::npos ? colon : line.find_first_not_of(" \t", colon + 1);
    if (start != std::string::npos) env.cpu_model = line.substr(start);
    break;
  }
  env.hardware_threads = std::thread::hardware_concurrency();
#if defined(__clang__)
  env.compiler = "clang " __clang_version__;
#elif defined(__GNUC__)
  env.compiler = "gcc " __VERSION__;
#else
  env.compiler = "unknown";
#endif
  // The engines run on the device; name it next to the build kind.
  env.build = "release (" + device_name() + ")";
  return env;
}

}  // namespace monoalign::bench
