// mas_io.cpp -- MASTENS v1 tensor files: the
// reference's on-disk format for likelihood batches and alignments,
// include/monoalign/tensor_io.hpp:11-23 (layout), src/tensor_io.cpp
// (behaviour: header validated before any payload allocation, the reader's
// byte budget, the IoError codes and texts), restated as C-ABI entry points.
//
//   offset  size  field
//        0     8  magic "MASTENS\0"
//        8     4  version (u32 LE) = 1
//       12     1  dtype: 0 = float32, 1 = uint8
//       13     1  ndims = 3
//       14    24  dims: B, T, S (u64 LE)
//       38     1  lengths_present (0 / 1)
//       39     .  payload, row-major
//        .     .  if lengths_present: B x (t_b, s_b) u32 LE
//
// Host-only code; the bytes are produced and checked without the GPU.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "monoalign_b200.h"

namespace {

constexpr char kMagic[8] = {'M', 'A', 'S', 'T', 'E', 'N', 'S', '\0'};
constexpr uint32_t kVersion = 1;
constexpr size_t kHeader = 39;

int io_error(mas_error_t* err, int errc, const std::string& msg) {
  if (err) {
    std::memset(err, 0, sizeof(*err));
    err->status = MAS_E_IO;
    err->errc = errc;
    err->item = -1;
    err->i = err->j = -1;
    std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
  }
  return MAS_E_IO;
}

void clear(mas_error_t* err) {
  if (err) {
    std::memset(err, 0, sizeof(*err));
    err->item = -1;
    err->i = err->j = -1;
  }
}

void put_le(uint8_t* p, uint64_t v, int bytes) {
  for (int k = 0; k < bytes; ++k) p[k] = static_cast<uint8_t>(v >> (8 * k));
}
uint64_t get_le(const uint8_t* p, int bytes) {
  uint64_t v = 0;
  for (int k = 0; k < bytes; ++k) v |= static_cast<uint64_t>(p[k]) << (8 * k);
  return v;
}

struct FileCloser {
  void operator()(FILE* f) const {
    if (f) std::fclose(f);
  }
};
using File = std::unique_ptr<FILE, FileCloser>;

struct Header {
  int dtype = 0;
  uint64_t dims[3] = {0, 0, 0};
  bool lengths_present = false;
  size_t count = 0;  // payload elements
};

// Reads exactly `bytes` or reports a truncation of `what`.
int read_exact(FILE* f, void* dst, size_t bytes, const std::string& path, const char* what,
               mas_error_t* err) {
  const size_t got = bytes ? std::fread(dst, 1, bytes, f) : 0;
  if (got != bytes) {
    std::ostringstream m;
    m << path << ": truncated " << what << " (expected " << bytes << " bytes, got " << got << ")";
    return io_error(err, MAS_ERRC_TRUNCATED_FILE, m.str());
  }
  return MAS_OK;
}

// Opens `path` and validates the header in the reference's order: magic,
// version, dtype, rank, lengths flag, then zero / out-of-range dims and the
// byte budget -- all before the payload is touched.
int open_and_check(const char* path_c, uint64_t byte_budget, File* file, Header* h,
                   mas_error_t* err) {
  const std::string path = path_c ? path_c : "";
  File f(std::fopen(path.c_str(), "rb"));
  if (!f) return io_error(err, MAS_ERRC_IO_FAILURE, "cannot open: " + path);
  uint8_t buf[kHeader];
  int rc = read_exact(f.get(), buf, kHeader, path, "header", err);
  if (rc) return rc;
  if (std::memcmp(buf, kMagic, sizeof(kMagic)) != 0)
    return io_error(err, MAS_ERRC_BAD_MAGIC, "not a tensor file: " + path);
  const uint32_t version = static_cast<uint32_t>(get_le(buf + 8, 4));
  std::ostringstream m;
  if (version != kVersion) {
    m << path << ": unsupported format version " << version;
    return io_error(err, MAS_ERRC_UNSUPPORTED_VERSION, m.str());
  }
  if (buf[12] > 1) {
    m << path << ": unsupported dtype code " << int{buf[12]};
    return io_error(err, MAS_ERRC_UNSUPPORTED_VERSION, m.str());
  }
  if (buf[13] != 3) {
    m << path << ": unsupported rank " << int{buf[13]};
    return io_error(err, MAS_ERRC_UNSUPPORTED_VERSION, m.str());
  }
  h->dtype = buf[12];
  for (int d = 0; d < 3; ++d) h->dims[d] = get_le(buf + 14 + 8 * d, 8);
  if (buf[38] > 1) {
    m << path << ": unsupported lengths flag " << int{buf[38]};
    return io_error(err, MAS_ERRC_UNSUPPORTED_VERSION, m.str());
  }
  h->lengths_present = buf[38] == 1;
  for (uint64_t d : h->dims) {
    if (d == 0)
      return io_error(err, MAS_ERRC_DIMENSION_OVERFLOW, path + ": header declares a zero dimension");
    if (d > static_cast<uint64_t>(std::numeric_limits<int>::max())) {
      m << path << ": dimension " << d << " out of range";
      return io_error(err, MAS_ERRC_DIMENSION_OVERFLOW, m.str());
    }
  }
  const uint64_t elem = h->dtype == 0 ? 4 : 1;
  const uint64_t budget_elems = byte_budget / elem;
  uint64_t count = 1;
  for (uint64_t d : h->dims) {
    if (count > budget_elems / d) {
      m << path << ": payload of " << h->dims[0] << "x" << h->dims[1] << "x" << h->dims[2]
        << " elements exceeds the " << byte_budget << "-byte budget";
      return io_error(err, MAS_ERRC_DIMENSION_OVERFLOW, m.str());
    }
    count *= d;
  }
  h->count = static_cast<size_t>(count);
  *file = std::move(f);
  return MAS_OK;
}

}  // namespace

extern "C" {

int mas_io_read_header(const char* path, uint64_t byte_budget, int32_t* dtype, int64_t dims[3],
                       int32_t* lengths_present, mas_error_t* err) {
  clear(err);
  File f;
  Header h;
  const int rc = open_and_check(path, byte_budget, &f, &h, err);
  if (rc) return rc;
  if (dtype) *dtype = h.dtype;
  if (dims)
    for (int d = 0; d < 3; ++d) dims[d] = static_cast<int64_t>(h.dims[d]);
  if (lengths_present) *lengths_present = h.lengths_present ? 1 : 0;
  return MAS_OK;
}

int mas_io_read(const char* path, uint64_t byte_budget, int32_t dtype, const int64_t dims[3],
                void* values, uint32_t* lengths, mas_error_t* err) {
  clear(err);
  File f;
  Header h;
  int rc = open_and_check(path, byte_budget, &f, &h, err);
  if (rc) return rc;
  const std::string p = path;
  // The caller sized `values` / `lengths` from an earlier header read; the
  // file must still describe exactly that tensor.
  if (!dims || h.dtype != dtype || static_cast<int64_t>(h.dims[0]) != dims[0] ||
      static_cast<int64_t>(h.dims[1]) != dims[1] || static_cast<int64_t>(h.dims[2]) != dims[2])
    return io_error(err, MAS_ERRC_IO_FAILURE,
                    "tensor header differs from the expected dtype and dimensions: " + p);
  const size_t bytes = h.count * (h.dtype == 0 ? 4 : 1);
  rc = read_exact(f.get(), values, bytes, p, "payload", err);
  if (rc) return rc;
  const size_t B = static_cast<size_t>(h.dims[0]);
  if (h.lengths_present) {
    std::vector<uint8_t> raw(B * 8);
    rc = read_exact(f.get(), raw.data(), raw.size(), p, "lengths table", err);
    if (rc) return rc;
    if (lengths)
      for (size_t b = 0; b < B; ++b) {
        lengths[2 * b] = static_cast<uint32_t>(get_le(raw.data() + 8 * b, 4));
        lengths[2 * b + 1] = static_cast<uint32_t>(get_le(raw.data() + 8 * b + 4, 4));
      }
  } else if (lengths) {  // full lengths, as the LikelihoodBatch / AlignmentMatrix ctors set
    for (size_t b = 0; b < B; ++b) {
      lengths[2 * b] = static_cast<uint32_t>(h.dims[1]);
      lengths[2 * b + 1] = static_cast<uint32_t>(h.dims[2]);
    }
  }
  return MAS_OK;
}

int mas_io_write(const char* path_c, int32_t dtype, int64_t batch, int64_t text_cap,
                 int64_t speech_cap, const void* values, const uint32_t* lengths,
                 mas_error_t* err) {
  clear(err);
  const std::string path = path_c ? path_c : "";
  uint8_t hdr[kHeader];
  std::memcpy(hdr, kMagic, sizeof(kMagic));
  put_le(hdr + 8, kVersion, 4);
  hdr[12] = static_cast<uint8_t>(dtype == 0 ? 0 : 1);
  hdr[13] = 3;
  put_le(hdr + 14, static_cast<uint64_t>(batch), 8);
  put_le(hdr + 22, static_cast<uint64_t>(text_cap), 8);
  put_le(hdr + 30, static_cast<uint64_t>(speech_cap), 8);
  hdr[38] = 1;  // writers always store the lengths table
  std::vector<uint8_t> tail(static_cast<size_t>(batch) * 8);
  for (int64_t b = 0; b < batch; ++b) {
    const uint32_t t = lengths ? lengths[2 * b] : static_cast<uint32_t>(text_cap);
    const uint32_t s = lengths ? lengths[2 * b + 1] : static_cast<uint32_t>(speech_cap);
    put_le(tail.data() + 8 * b, t, 4);
    put_le(tail.data() + 8 * b + 4, s, 4);
  }
  File f(std::fopen(path.c_str(), "wb"));
  if (!f) return io_error(err, MAS_ERRC_IO_FAILURE, "cannot open for writing: " + path);
  const size_t payload = static_cast<size_t>(batch * text_cap * speech_cap) * (dtype == 0 ? 4 : 1);
  bool ok = std::fwrite(hdr, 1, kHeader, f.get()) == kHeader;
  ok = ok && (payload == 0 || std::fwrite(values, 1, payload, f.get()) == payload);
  ok = ok && (tail.empty() || std::fwrite(tail.data(), 1, tail.size(), f.get()) == tail.size());
  ok = ok && std::fflush(f.get()) == 0;
  if (!ok) return io_error(err, MAS_ERRC_IO_FAILURE, "write failed: " + path);
  return MAS_OK;
}

}  // extern "C"
