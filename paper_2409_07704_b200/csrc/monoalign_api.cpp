// monoalign_api.cpp -- the reference's C++ API (include/monoalign/*.hpp of
// /root/reference/proj) over the C-ABI of include/monoalign_b200.h.
//
// Host-side only: container construction, the ShapeMismatch container check
// (parallel.cpp:118-125), exception mapping (errors.hpp:32-53), and the
// path/matrix helpers of types.cpp:132-185.  Every alignment and the
// NonFinite validation are computed by the sm_100a kernels behind
// mas_align_host / mas_validate_host; there is no CPU fallback -- a device
// failure throws DeviceError.
#include <cstdint>
#include <sstream>
#include <string>
#include <vector>

#include <sys/mman.h>

#include "monoalign/align.hpp"
#include "monoalign/bench.hpp"
#include "monoalign/tensor_io.hpp"

#include <cuda_runtime.h>
#include "../../include/monoalign_b200.h"
#include "mas_kernels.h"

namespace monoalign {

namespace {

[[noreturn]] void throw_for(int rc, const mas_error_t& err) {
  const std::string msg(err.message);
  if (rc == MAS_E_VALIDATION) throw ValidationError(static_cast<Errc>(err.errc), msg);
  if (rc == MAS_E_IO) throw IoError(static_cast<Errc>(err.errc), msg);
  throw DeviceError("monoalign device path failed: " + msg);
}

mas_config_t to_c(const MasConfig& cfg, bool unchecked) {
  mas_config_t c;
  mas_config_default(&c);
  c.engine = cfg.engine == EngineKind::Reference ? MAS_ENGINE_REFERENCE : MAS_ENGINE_PARALLEL;
  c.max_neg_val = cfg.max_neg_val;
  c.lane_padding = cfg.lane_padding == LanePadding::NextPowerOfTwo ? 1 : 0;
  c.threads = cfg.threads;
  c.flags = unchecked ? MAS_FLAG_UNCHECKED : 0u;
  return c;
}

// parallel.cpp:118-125 / types.cpp:119-126
void check_containers(const LikelihoodBatch& batch) {
  if (batch.batch < 1 || batch.text_cap < 1 || batch.speech_cap < 1)
    throw ValidationError(Errc::ZeroDim, "batch and capacities must be at least 1");
  if (batch.lengths.size() != static_cast<std::size_t>(batch.batch) ||
      batch.values.size() != static_cast<std::size_t>(batch.batch) * batch.item_stride())
    throw ValidationError(Errc::ShapeMismatch,
                          "container sizes do not match the declared dimensions");
}

std::vector<uint32_t> flat_lengths(const LikelihoodBatch& batch) {
  std::vector<uint32_t> l(static_cast<std::size_t>(batch.batch) * 2);
  for (int b = 0; b < batch.batch; ++b) {
    l[2 * b] = batch.lengths[b].text;
    l[2 * b + 1] = batch.lengths[b].speech;
  }
  return l;
}

AlignmentMatrix run(const LikelihoodBatch& batch, const MasConfig& cfg, bool unchecked) {
  const mas_config_t c = to_c(cfg, unchecked);
  mas_error_t err;
  if (!unchecked) {
    const int rc = mas_validate_config(&c, &err);
    if (rc != MAS_OK) throw_for(rc, err);
  }
  check_containers(batch);
  AlignmentMatrix out(batch.batch, batch.text_cap, batch.speech_cap);
  out.lengths = batch.lengths;
  const std::vector<uint32_t> l = flat_lengths(batch);
  const int rc = mas_align_host(batch.values.data(), batch.batch, batch.text_cap, batch.speech_cap,
                                l.data(), &c, out.values.data(), nullptr, &err);
  if (rc != MAS_OK) throw_for(rc, err);
  return out;
}


// Device scratch for the table round trips below (forward_parallel,
// forward_reference, backward_*, relax_column): stream-ordered on the calling
// thread's per-thread stream, freed on scope exit.
class DeviceScratch {
 public:
  explicit DeviceScratch(std::size_t bytes) : stream_(cudaStreamPerThread) {
    if (bytes) check(mas::pool_alloc(&p_, bytes, stream_));
  }
  ~DeviceScratch() {
    if (p_) cudaFreeAsync(p_, stream_);
    cudaStreamSynchronize(stream_);
  }
  DeviceScratch(const DeviceScratch&) = delete;
  DeviceScratch& operator=(const DeviceScratch&) = delete;
  template <typename T>
  T* as(std::size_t byte_offset = 0) const {
    return reinterpret_cast<T*>(static_cast<char*>(p_) + byte_offset);
  }
  cudaStream_t stream() const { return stream_; }
  static void check(cudaError_t e) {
    if (e != cudaSuccess)
      throw DeviceError(std::string("monoalign device path failed: ") + cudaGetErrorString(e));
  }
  void sync() const { check(cudaStreamSynchronize(stream_)); }

 private:
  void* p_ = nullptr;
  cudaStream_t stream_;
};

// Host -> device copy of a [t][s] table with row stride `src_stride` into a
// dense [t][dst_pitch] device table.
void put_table(float* d, std::ptrdiff_t dst_pitch, const float* h, std::ptrdiff_t src_stride,
               int t, int s, cudaStream_t st) {
  DeviceScratch::check(cudaMemcpy2DAsync(d, dst_pitch * sizeof(float), h,
                                         src_stride * sizeof(float), s * sizeof(float), t,
                                         cudaMemcpyHostToDevice, st));
}

void get_table(float* h, std::ptrdiff_t dst_stride, const float* d, std::ptrdiff_t src_pitch,
               int t, int s, cudaStream_t st) {
  DeviceScratch::check(cudaMemcpy2DAsync(h, dst_stride * sizeof(float), d,
                                         src_pitch * sizeof(float), s * sizeof(float), t,
                                         cudaMemcpyDeviceToHost, st));
}

// The shared backtrack walk (backtrack.hpp:21-32) over a host score table:
// the table goes to the device, the walk runs there (mas_backtrack_scores).
PathVector walk_scores(const float* scores, std::ptrdiff_t row_stride, int t, int s) {
  if (t < 1 || s < 1) return PathVector(static_cast<std::size_t>(s > 0 ? s : 0), 0);
  const std::size_t table = static_cast<std::size_t>(t) * s * sizeof(float);
  DeviceScratch d(table + static_cast<std::size_t>(s) * sizeof(int32_t));
  float* dq = d.as<float>();
  int32_t* dpath = d.as<int32_t>(table);
  put_table(dq, s, scores, row_stride, t, s, d.stream());
  mas_error_t err;
  const int rc = mas_backtrack_scores(dq, s, 1, t, s, nullptr, dpath, d.stream(), &err);
  if (rc != MAS_OK) throw_for(rc, err);
  PathVector path(static_cast<std::size_t>(s));
  DeviceScratch::check(cudaMemcpyAsync(path.data(), dpath, s * sizeof(int32_t),
                                       cudaMemcpyDeviceToHost, d.stream()));
  d.sync();
  return path;
}

}  // namespace

const char* errc_name(Errc code) { return mas_errc_name(static_cast<int32_t>(code)); }

void validate_config(const MasConfig& cfg) {
  const mas_config_t c = to_c(cfg, false);
  mas_error_t err;
  const int rc = mas_validate_config(&c, &err);
  if (rc != MAS_OK) throw_for(rc, err);
}

namespace {
// A zero-filled container of n elements whose large buffers are backed by
// transparent huge pages where the kernel allows it (madvise mode): glibc
// serves allocations above 32 MB with fresh mmap pages on every call, and
// first-touching them 4 KB at a time cost ~12 ms for a 33.5 MB alignment
// matrix on the B200 hosts (the acceptance suite's B8 T1024 S4096 point),
// against ~1.6 ms for 25.7 MB still recycled by malloc.  Same contents and
// semantics as vector(n, 0).
template <typename T>
void zeroed(std::vector<T>& v, std::size_t n) {
  v.reserve(n);
  const std::size_t bytes = n * sizeof(T);
  constexpr std::size_t kHuge = std::size_t(2) << 20;
  if (bytes >= 4 * kHuge) {
    const auto lo = (reinterpret_cast<std::uintptr_t>(v.data()) + 4095) & ~std::uintptr_t(4095);
    const auto hi = (reinterpret_cast<std::uintptr_t>(v.data()) + bytes) & ~std::uintptr_t(4095);
    if (hi > lo) madvise(reinterpret_cast<void*>(lo), hi - lo, MADV_HUGEPAGE);  // advisory
  }
  v.resize(n);
}
}  // namespace

LikelihoodBatch::LikelihoodBatch(int batch_size, int text_capacity, int speech_capacity)
    : batch(batch_size),
      text_cap(text_capacity),
      speech_cap(speech_capacity),
      lengths(static_cast<std::size_t>(batch_size),
              ValidLengths{static_cast<std::uint32_t>(text_capacity),
                           static_cast<std::uint32_t>(speech_capacity)}) {
  zeroed(values, static_cast<std::size_t>(batch_size) * text_capacity * speech_capacity);
}

AlignmentMatrix::AlignmentMatrix(int batch_size, int text_capacity, int speech_capacity)
    : batch(batch_size),
      text_cap(text_capacity),
      speech_cap(speech_capacity),
      lengths(static_cast<std::size_t>(batch_size),
              ValidLengths{static_cast<std::uint32_t>(text_capacity),
                           static_cast<std::uint32_t>(speech_capacity)}) {
  zeroed(values, static_cast<std::size_t>(batch_size) * text_capacity * speech_capacity);
}

LikelihoodView item_view(const LikelihoodBatch& batch, int b) {
  return {batch.item(b).data(), static_cast<int>(batch.lengths[b].text),
          static_cast<int>(batch.lengths[b].speech), batch.speech_cap};
}

MutableLikelihoodView item_view(LikelihoodBatch& batch, int b) {
  return {batch.item(b).data(), static_cast<int>(batch.lengths[b].text),
          static_cast<int>(batch.lengths[b].speech), batch.speech_cap};
}

void validate_batch(const LikelihoodBatch& batch) {
  check_containers(batch);
  const std::vector<uint32_t> l = flat_lengths(batch);
  mas_error_t err;
  const int rc = mas_validate_host(batch.values.data(), batch.batch, batch.text_cap,
                                   batch.speech_cap, l.data(), 0, &err);
  if (rc != MAS_OK) throw_for(rc, err);
}

void validate_item(const LikelihoodBatch& batch, int b) {
  check_containers(batch);
  const uint32_t l[2] = {batch.lengths[b].text, batch.lengths[b].speech};
  mas_error_t err;
  const int rc = mas_validate_host(batch.item(b).data(), 1, batch.text_cap, batch.speech_cap, l, b,
                                   &err);
  if (rc != MAS_OK) throw_for(rc, err);
}

void validate_path(const PathVector& path, int t, int s) {
  if (t < 1 || s < 1 || t > s)
    throw ValidationError(Errc::InvalidPath, "dimensions do not admit a monotonic path");
  if (path.size() != static_cast<std::size_t>(s))
    throw ValidationError(Errc::InvalidPath, "path length does not equal the speech length");
  if (path.front() != 0 || path.back() != t - 1)
    throw ValidationError(Errc::InvalidPath, "path must start at 0 and end at t-1");
  for (int j = 1; j < s; ++j) {
    const std::int32_t d = path[j] - path[j - 1];
    if (d == 0 || d == 1) continue;
    std::ostringstream m;
    m << "step of " << d << " at frame " << j << "; only 0 and 1 are allowed";
    throw ValidationError(Errc::InvalidPath, m.str());
  }
}

AlignmentMatrix matrix_from_path(const PathVector& path, int t, int s) {
  validate_path(path, t, s);
  AlignmentMatrix m(1, t, s);
  write_path(m, 0, path);
  return m;
}

PathVector path_from_matrix(const AlignmentMatrix& m, int b) {
  const ValidLengths v = m.lengths[b];
  PathVector path(v.speech, -1);
  for (std::uint32_t j = 0; j < v.speech; ++j) {
    int ones = 0;
    for (std::uint32_t i = 0; i < v.text; ++i)
      if (m.at(b, static_cast<int>(i), static_cast<int>(j))) {
        ++ones;
        path[j] = static_cast<std::int32_t>(i);
      }
    if (ones == 1) continue;
    std::ostringstream msg;
    msg << "item " << b << ": column " << j << " carries " << ones << " ones, expected 1";
    throw ValidationError(Errc::InvalidMatrix, msg.str());
  }
  return path;
}

void write_path(AlignmentMatrix& out, int b, const PathVector& path) {
  for (std::size_t j = 0; j < path.size(); ++j) out.at(b, path[j], static_cast<int>(j)) = 1;
}

std::vector<PathVector> align_paths(const LikelihoodBatch& batch, const MasConfig& cfg) {
  const mas_config_t c = to_c(cfg, false);
  mas_error_t err;
  int rc = mas_validate_config(&c, &err);
  if (rc != MAS_OK) throw_for(rc, err);
  check_containers(batch);
  const std::vector<uint32_t> l = flat_lengths(batch);
  std::vector<int32_t> flat(static_cast<std::size_t>(batch.batch) * batch.speech_cap);
  rc = mas_align_host(batch.values.data(), batch.batch, batch.text_cap, batch.speech_cap, l.data(),
                      &c, nullptr, flat.data(), &err);
  if (rc != MAS_OK) throw_for(rc, err);
  std::vector<PathVector> out(batch.batch);
  for (int b = 0; b < batch.batch; ++b) {
    const auto* row = flat.data() + static_cast<std::size_t>(b) * batch.speech_cap;
    out[b].assign(row, row + batch.lengths[b].speech);
  }
  return out;
}

namespace parallel {

int pad_lanes(int t, LanePadding policy) {
  if (policy == LanePadding::None || t <= 1) return t;
  unsigned v = 1;
  while (v < static_cast<unsigned>(t)) v <<= 1;
  return static_cast<int>(v);
}

void forward_parallel(MutableLikelihoodView q, const MasConfig& cfg) {
  // The item round-trips through device memory; mas_forward_scores
  // computes the table on the GPU, nothing is computed here.
  if (q.text < 1 || q.speech < 1) return;
  DeviceScratch d(static_cast<std::size_t>(q.text) * q.speech * sizeof(float));
  float* dq = d.as<float>();
  put_table(dq, q.speech, q.data, q.row_stride, q.text, q.speech, d.stream());
  mas_error_t err;
  const int rc = mas_forward_scores(dq, q.speech, 1, q.text, q.speech, nullptr, cfg.max_neg_val,
                                    d.stream(), &err);
  if (rc != MAS_OK) throw_for(rc, err);
  get_table(q.data, q.row_stride, dq, q.speech, q.text, q.speech, d.stream());
  d.sync();
}

PathVector backward_parallel(const LikelihoodView& scores) {
  return walk_scores(scores.data, scores.row_stride, scores.text, scores.speech);
}

void detail::relax_column(const float* prev, float* cur, int lanes, float sentinel) {
  if (lanes < 1) return;
  const std::size_t col = static_cast<std::size_t>(lanes) * sizeof(float);
  DeviceScratch d(2 * col);
  float* dprev = d.as<float>();
  float* dcur = d.as<float>(col);
  DeviceScratch::check(cudaMemcpyAsync(dprev, prev, col, cudaMemcpyHostToDevice, d.stream()));
  DeviceScratch::check(cudaMemcpyAsync(dcur, cur, col, cudaMemcpyHostToDevice, d.stream()));
  mas_error_t err;
  const int rc = mas_relax_column(dprev, dcur, lanes, sentinel, d.stream(), &err);
  if (rc != MAS_OK) throw_for(rc, err);
  DeviceScratch::check(cudaMemcpyAsync(cur, dcur, col, cudaMemcpyDeviceToHost, d.stream()));
  d.sync();
}

AlignmentMatrix align_parallel(const LikelihoodBatch& batch, const MasConfig& cfg) {
  MasConfig c = cfg;
  c.engine = EngineKind::Parallel;
  return run(batch, c, false);
}

AlignmentMatrix detail::align_unchecked(const LikelihoodBatch& batch, const MasConfig& cfg) {
  MasConfig c = cfg;
  c.engine = EngineKind::Parallel;
  return run(batch, c, true);
}

}  // namespace parallel

namespace reference {

QCache forward_reference(const LikelihoodView& q, const MasConfig& cfg) {
  const int t = q.text;
  const int s = q.speech;
  // reference.cpp:12-15: an odd multiple of 16 floats
  int stride = (s + 15) & ~15;
  if ((stride / 16) % 2 == 0) stride += 16;
  QCache cache{t, s, stride,
               std::vector<float>(static_cast<std::size_t>(t > 0 ? t : 0) * stride,
                                  cfg.max_neg_val)};
  if (t < 1 || s < 1) return cache;
  DeviceScratch d(static_cast<std::size_t>(t) * stride * sizeof(float));
  float* dq = d.as<float>();
  put_table(dq, stride, q.data, q.row_stride, t, s, d.stream());
  mas_error_t err;
  const int rc = mas_forward_scores_ex(dq, stride, 1, t, s, nullptr, MAS_ENGINE_REFERENCE,
                                       cfg.max_neg_val, d.stream(), &err);
  if (rc != MAS_OK) throw_for(rc, err);
  get_table(cache.values.data(), stride, dq, stride, t, s, d.stream());
  d.sync();
  return cache;
}

PathVector backward_reference(const QCache& cache) {
  return walk_scores(cache.values.data(), cache.stride, cache.text, cache.speech);
}

AlignmentMatrix align_reference(const LikelihoodBatch& batch, const MasConfig& cfg) {
  MasConfig c = cfg;
  c.engine = EngineKind::Reference;
  return run(batch, c, false);
}

AlignmentMatrix detail::align_unchecked(const LikelihoodBatch& batch, const MasConfig& cfg) {
  MasConfig c = cfg;
  c.engine = EngineKind::Reference;
  return run(batch, c, true);
}

}  // namespace reference

namespace bench {

LikelihoodBatch generate_random_batch(int b, int t, int s, std::uint64_t seed) {
  if (b < 1 || t < 1 || s < 1)
    throw ValidationError(Errc::ZeroDim, "batch dimensions must be at least 1");
  if (t > s) throw ValidationError(Errc::InfeasibleLengths, "text length t exceeds speech length s");
  LikelihoodBatch batch(b, t, s);
  const size_t bytes = batch.values.size() * sizeof(float);
  float* d = nullptr;
  cudaStream_t st = cudaStreamPerThread;
  cudaError_t e = mas::pool_alloc(reinterpret_cast<void**>(&d), bytes, st);
  if (e == cudaSuccess &&
      mas_generate_device(seed, b, t, s, 0, s, d, st) != MAS_OK)
    e = cudaErrorLaunchFailure;
  if (e == cudaSuccess) e = cudaMemcpyAsync(batch.values.data(), d, bytes, cudaMemcpyDeviceToHost, st);
  if (d) cudaFreeAsync(d, st);
  const cudaError_t e2 = cudaStreamSynchronize(st);
  if (e != cudaSuccess || e2 != cudaSuccess)
    throw DeviceError(std::string("generate_random_batch: ") +
                      cudaGetErrorString(e != cudaSuccess ? e : e2));
  return batch;
}

const char* engine_name(EngineKind engine) {
  return engine == EngineKind::Reference ? "reference" : "parallel";
}

}  // namespace bench

namespace io {

namespace {
std::vector<std::uint32_t> flat(const std::vector<ValidLengths>& lengths) {
  std::vector<std::uint32_t> v(2 * lengths.size());
  for (std::size_t b = 0; b < lengths.size(); ++b) {
    v[2 * b] = lengths[b].text;
    v[2 * b + 1] = lengths[b].speech;
  }
  return v;
}
}  // namespace

void write_tensor(const std::filesystem::path& path, const LikelihoodBatch& batch) {
  const std::vector<std::uint32_t> lens = flat(batch.lengths);
  mas_error_t err;
  const int rc = mas_io_write(path.string().c_str(), 0, batch.batch, batch.text_cap,
                              batch.speech_cap, batch.values.data(), lens.data(), &err);
  if (rc != MAS_OK) throw_for(rc, err);
}

void write_tensor(const std::filesystem::path& path, const AlignmentMatrix& m) {
  const std::vector<std::uint32_t> lens = flat(m.lengths);
  mas_error_t err;
  const int rc = mas_io_write(path.string().c_str(), 1, m.batch, m.text_cap, m.speech_cap,
                              m.values.data(), lens.data(), &err);
  if (rc != MAS_OK) throw_for(rc, err);
}

Tensor read_tensor(const std::filesystem::path& path, std::size_t byte_budget) {
  const std::string p = path.string();
  mas_error_t err;
  std::int32_t dtype = 0, has_lengths = 0;
  std::int64_t dims[3] = {0, 0, 0};
  int rc = mas_io_read_header(p.c_str(), byte_budget, &dtype, dims, &has_lengths, &err);
  if (rc != MAS_OK) throw_for(rc, err);
  const int b = static_cast<int>(dims[0]), t = static_cast<int>(dims[1]),
            s = static_cast<int>(dims[2]);
  std::vector<std::uint32_t> lens(2 * static_cast<std::size_t>(b));
  auto unflat = [&](std::vector<ValidLengths>& out) {
    for (int i = 0; i < b; ++i) out[static_cast<std::size_t>(i)] = {lens[2 * i], lens[2 * i + 1]};
  };
  if (dtype == 0) {
    LikelihoodBatch batch(b, t, s);
    rc = mas_io_read(p.c_str(), byte_budget, dtype, dims, batch.values.data(), lens.data(), &err);
    if (rc != MAS_OK) throw_for(rc, err);
    unflat(batch.lengths);
    return batch;
  }
  AlignmentMatrix m(b, t, s);
  rc = mas_io_read(p.c_str(), byte_budget, dtype, dims, m.values.data(), lens.data(), &err);
  if (rc != MAS_OK) throw_for(rc, err);
  unflat(m.lengths);
  return m;
}

}  // namespace io

}  // namespace monoalign
