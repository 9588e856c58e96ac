// mas_abi.cu -- the extern "C" boundary (include/monoalign_b200.h):
// host-side validation with the reference's exact error text, workspace and
// launch-geometry planning, TMA descriptor encoding, and the host / device
// entry points.  There is no CPU compute path: every alignment is produced
// by the kernels in mas_fwd4.cu / mas_bt.cu.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>

#include <unistd.h>
#include <new>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/monoalign_b200.h"
#include "mas_kernels.h"

namespace mas {
cudaError_t bt_configure(int T_alloc, int L);
}

namespace {

// ---- reference constants (include/monoalign/types.hpp:19-26) --------------
constexpr float kDefaultMaxNegVal = -1e32f;
constexpr float kMaxNegValCeiling = -1e30f;
constexpr int64_t kMaxSpeechLen = 100000;

const char* const kErrcNames[] = {
    "ZeroDim",     "InfeasibleLengths", "LengthsOutOfRange",  "NonFinite", "SpeechTooLong",
    "ShapeMismatch", "InvalidPath",     "InvalidMatrix",      "InvalidConfig", "TooLarge",
    "EmptyReport", "InsufficientPoints", "IoFailure",         "BadMagic",  "UnsupportedVersion",
    "TruncatedFile", "DimensionOverflow"};

void clear_error(mas_error_t* err) {
  if (!err) return;
  err->status = MAS_OK;
  err->errc = -1;
  err->item = -1;
  err->reserved = 0;
  err->i = err->j = -1;
  err->message[0] = '\0';
}

int set_error(mas_error_t* err, int status, int errc, int item, const std::string& msg) {
  if (err) {
    err->status = status;
    err->errc = errc;
    err->item = item;
    std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
  }
  return status;
}

int cuda_error(mas_error_t* err, cudaError_t e, const char* what) {
  std::string msg = std::string(what) + ": " + cudaGetErrorString(e);
  return set_error(err, MAS_E_CUDA, -1, -1, msg);
}

#define MAS_CUDA(call, what)                               \
  do {                                                     \
    cudaError_t e_ = (call);                               \
    if (e_ != cudaSuccess) return cuda_error(err, e_, what); \
  } while (0)

// validate_config, types.cpp:59-69 (same ostream formatting of the floats).
int validate_config(const mas_config_t& cfg, mas_error_t* err) {
  if (cfg.flags & MAS_FLAG_UNCHECKED) return MAS_OK;
  if (!std::isfinite(cfg.max_neg_val) || cfg.max_neg_val > kMaxNegValCeiling) {
    std::ostringstream msg;
    msg << "max_neg_val must be finite and at most " << kMaxNegValCeiling << ", got "
        << cfg.max_neg_val;
    return set_error(err, MAS_E_VALIDATION, MAS_ERRC_INVALID_CONFIG, -1, msg.str());
  }
  if (cfg.threads < 0)
    return set_error(err, MAS_E_VALIDATION, MAS_ERRC_INVALID_CONFIG, -1, "threads must be >= 0");
  if (cfg.engine != MAS_ENGINE_REFERENCE && cfg.engine != MAS_ENGINE_PARALLEL)
    return set_error(err, MAS_E_VALIDATION, MAS_ERRC_INVALID_CONFIG, -1, "unknown engine");
  return MAS_OK;
}

// Batch-level checks (types.cpp:119-126 / parallel.cpp:118-125).
int validate_dims(int32_t B, int32_t T, int32_t S, mas_error_t* err) {
  if (B < 1 || T < 1 || S < 1)
    return set_error(err, MAS_E_VALIDATION, MAS_ERRC_ZERO_DIM, -1,
                     "batch and capacities must be at least 1");
  return MAS_OK;
}

struct ItemError {
  int item = -1;
  int errc = -1;
  std::string message;
};

// validate_item's length checks, types.cpp:81-106, in the reference order;
// the NonFinite scan (:107-115) runs on the device.
bool length_error(int b, uint32_t t, uint32_t s, int32_t T, int32_t S, ItemError* out) {
  std::ostringstream d;
  int code = -1;
  if (t < 1 || s < 1) {
    d << "valid lengths must be at least 1, got (" << t << ", " << s << ")";
    code = MAS_ERRC_ZERO_DIM;
  } else if (t > static_cast<uint32_t>(T) || s > static_cast<uint32_t>(S)) {
    d << "valid lengths (" << t << ", " << s << ") exceed capacities (" << T << ", " << S << ")";
    code = MAS_ERRC_LENGTHS_OUT_OF_RANGE;
  } else if (s > kMaxSpeechLen) {
    d << "speech length " << s << " exceeds the supported maximum " << kMaxSpeechLen;
    code = MAS_ERRC_SPEECH_TOO_LONG;
  } else if (t > s) {
    d << "text length " << t << " exceeds speech length " << s
      << "; every text unit needs at least one frame";
    code = MAS_ERRC_INFEASIBLE_LENGTHS;
  }
  if (code < 0) return false;
  std::ostringstream msg;
  msg << "item " << b << ": " << d.str();  // fail_item, types.cpp:73-77
  out->item = b;
  out->errc = code;
  out->message = msg.str();
  return true;
}

std::string nonfinite_message(int b, int64_t i, int64_t j) {
  std::ostringstream msg;
  msg << "item " << b << ": non-finite likelihood at (" << i << ", " << j << ")";
  return msg.str();
}

// ---- TMA descriptor encoding through the runtime's driver entry point ----
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}


struct Geometry {
  int R = 4;            // text rows per lane of mas_fwd4.cu
  int W = 1, K = 1, N = 2, L = 256, Kseg = 1, T_alloc = 128, M = 1;
  int bands = 1;       // mas_fwd4: launches of K*W*128 rows each (text longer than a cluster)
  int band_rows = 128;
};

bool choose_geometry(int B, int t_max, int S_cap, Geometry* g, int kp) {
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t budget = 220 * 1024;
  g->R = 4;
  g->M = (S_cap + 31) / 32;
  g->L = 256;
  g->Kseg = (S_cap + g->L - 1) / g->L;
  {
    // 32 R rows per warp; an item's warps form `bands` clusters of K CTAs of
    // W compute warps, all in one launch (mas_fwd4.cu, bands).  Candidates
    // (W, stages) in order of preference (few warps per CTA spread an item
    // over more SMs; more stages give the TMA ring more lead); for each, the
    // fewest bands whose clusters all run in one wave of co-resident
    // clusters (cudaOccupancyMaxActiveClusters accounts for shared memory
    // and the GPC placement of clusters).  The first candidate reaching one
    // wave wins, otherwise the fewest waves, then the fewest bands.
    static const int band_warps_cap = [] {
      const char* e = std::getenv("MAS_BAND_WARPS");  // test hook: force short bands
      return e ? std::max(1, std::min(4 * mas::kMaxClusterCtas, std::atoi(e)))
               : 4 * mas::kMaxClusterCtas;
    }();
    const int rows = 32 * g->R;
    const int warps_total = std::max(1, (t_max + rows - 1) / rows);
    static const int cand4[][2] = {{2, 4}, {4, 3}, {2, 3}, {1, 4}, {2, 2}, {4, 2}, {1, 2}};
    const int(*cand)[2] = cand4;
    const int ncand = 7;
    int best = -1;
    int64_t best_waves = 0;
    int best_bands = 0;
    for (int c = 0; c < ncand && !(best >= 0 && best_waves == 1); ++c) {
      const int W = std::min(cand[c][0], warps_total), N = cand[c][1];
      if (mas::fwd4_smem_bytes(g->R, W, N, kp) > budget) continue;
      // Gaussian source: A (Kp/2 columns per warp) and two 32-column
      // accumulators per warp in TMEM's 512 columns; one band only
      if (kp > 0 && (W > 2 || W * kp / 2 + W * 64 > 512)) continue;
      int last_K = -1;
      for (int nb = 1; nb <= (kp > 0 ? 1 : warps_total); ++nb) {
        const int per_band = (warps_total + nb - 1) / nb;
        if (per_band > band_warps_cap && kp == 0) continue;
        const int K = (per_band + W - 1) / W;
        if (K > mas::kMaxClusterCtas || K == last_K) continue;
        last_K = K;
        const int bands = (warps_total + K * W - 1) / (K * W);
        const int act = mas::fwd4_max_active_clusters(g->R, W, N, K, kp);
        if (act <= 0) continue;
        const int64_t waves = (static_cast<int64_t>(B) * bands + act - 1) / act;
        if (best < 0 || waves < best_waves || (waves == best_waves && bands < best_bands)) {
          best = c;
          best_waves = waves;
          best_bands = bands;
          g->W = W;
          g->N = N;
          g->K = K;
        }
        if (waves == 1) break;
      }
    }
    if (best < 0) return false;
    g->band_rows = g->K * g->W * rows;
    g->bands = (std::max(t_max, 1) + g->band_rows - 1) / g->band_rows;
    g->T_alloc = g->bands * g->band_rows;
    return true;
  }
}

// choose_geometry queries the occupancy API for every candidate (tens of
// microseconds per call); plans of the same shape on the same device reuse
// the answer.
bool cached_geometry(int B, int t_max, int S_cap, Geometry* g, int kp = 0) {
  struct Entry {
    int dev, B, t, S, kp;
    Geometry g;
    bool ok;
  };
  static std::mutex mu;
  static std::vector<Entry> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(mu);
    for (const Entry& e : cache)
      if (e.dev == dev && e.B == B && e.t == t_max && e.S == S_cap && e.kp == kp) {
        *g = e.g;
        return e.ok;
      }
  }
  // the occupancy queries need the kernels' shared-memory attributes set;
  // a failed query must not be cached as "no geometry"
  if (mas::fwd4_configure() != cudaSuccess) return false;
  const bool ok = choose_geometry(B, t_max, S_cap, g, kp);
  std::lock_guard<std::mutex> lk(mu);
  if (cache.size() >= 256) cache.erase(cache.begin());
  cache.push_back({dev, B, t_max, S_cap, kp, *g, ok});
  return ok;
}

// The input [B*T_pad][pitch] as a 3-D tensor {columns, row groups of R,
// row residue mod R}: one {32, 32, R} box is a 32R-row x 32-column stage of
// mas_fwd4.cu laid out [residue][group][column] (128-byte swizzle).
// 256-byte promotion: each 128-byte row segment also brings the row's next
// stage into L2 (K1 15 us faster than without; r12, profiles/r12_l2_policy.md)
constexpr CUtensorMapL2promotion kQPromotion = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;

bool encode_map4(const float* q, int64_t pitch, int64_t rows_total, int64_t S, int R,
                 CUtensorMap* m) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(S), static_cast<cuuint64_t>(rows_total / R),
                              static_cast<cuuint64_t>(R)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(R * pitch * 4),
                                 static_cast<cuuint64_t>(pitch * 4)};
  const cuuint32_t box[3] = {32, 32, static_cast<cuuint32_t>(R)};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(q), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, kQPromotion,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}


}  // namespace

// Device memory comes from a stream-ordered pool owned by this library (one
// per device) whose release threshold is raised, so repeated calls reuse it
// instead of re-mapping pages (and cudaFree's device-wide synchronisation is
// avoided).  A private pool leaves the device's default pool -- which torch
// (cudaMallocAsync backend), CuPy or the caller may use -- untouched.
namespace {
cudaError_t device_pool(int dev, cudaMemPool_t* out) {
  constexpr int kMaxDevices = 64;
  static std::once_flag once[kMaxDevices];
  static cudaError_t status[kMaxDevices];
  static cudaMemPool_t pools[kMaxDevices];
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  std::call_once(once[dev], [dev] {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaError_t r = cudaMemPoolCreate(&pools[dev], &props);
    uint64_t keep = ~0ull;
    if (r == cudaSuccess)
      r = cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    status[dev] = r;
  });
  *out = pools[dev];
  return status[dev];
}
}  // namespace

namespace mas {
cudaError_t pool_alloc(void** ptr, size_t bytes, cudaStream_t stream) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  cudaMemPool_t pool;
  if (e == cudaSuccess) e = device_pool(dev, &pool);
  if (e == cudaSuccess) e = cudaMallocFromPoolAsync(ptr, bytes, pool, stream);
  return e;
}
}  // namespace mas

struct mas_plan {
  int32_t B = 0, T = 0, S = 0;
  int64_t pitch = 0;
  int T_pad = 0;
  int mode = 0;  // 0 parallel, 1 reference
  float mnv = kDefaultMaxNegVal;
  Geometry geo;
  std::vector<uint32_t> lengths;  // [B][2], zeroed for items with host errors
  ItemError first_host_error;
  // device workspace
  uint32_t* d_lengths = nullptr;
  uint32_t* d_dirs = nullptr;       // the buffer of the current batch
  uint32_t* d_dirs_buf[2] = {nullptr, nullptr};  // pipelined: two, alternating
  bool pipelined = false;
  int dirs_par = 0;
  unsigned* d_bt_done = nullptr;     // pipelined: finished backtrack CTAs per buffer
  unsigned bt_issued[2] = {0u, 0u};  // backtrack CTAs launched per buffer
  bool all_full = true;  // every item spans the full [T_cap x S_cap]
  int* d_flags = nullptr;  // the current batch's NonFinite flags
  int* d_flags_buf[2] = {nullptr, nullptr};
  unsigned long long* d_locate = nullptr;
  int launches = 0;
  int device = 0;
  int bt_rows = 64;       // backtrack window rows
  float* d_bnd = nullptr; // bands: [B][bands-1][bnd_pitch] boundary rows
  cudaEvent_t ws_ready = nullptr;  // deferred plans: workspace set-up recorded here
  // tensor maps of the last input / output buffers enqueued (reused)
  CUtensorMap tm_in;
  const float* tm_in_ptr = nullptr;
  int64_t tm_in_pitch = 0;
  int tm_in_tpad = 0;
  int* d_sync = nullptr;  // bands: tickets [B] (one per launch, at its first item) +
                          //        progress [B][bands-1]
  int bnd_pitch = 0;
  bool internal = false;  // created by mas_align_host / _device, which order the frees
  int item_base = 0;      // added to item indices in messages (validate_item of one item)
  // caller-held plans: per stream, an event recorded after the last enqueue
  std::vector<std::pair<cudaStream_t, cudaEvent_t>> done;
  bool captured = false;  // enqueued while a stream was capturing
  bool nan_parallel = false;  // parallel engine, NaN sentinel (unchecked): score-table forward
  // Gaussian source (mas_align_gaussian_device): K1 computes q from these
  int gauss_kp = 0;
  const mas::GaussOperands* gauss = nullptr;
  const CUtensorMap* gauss_map = nullptr;
  // Gaussian plans (mas_plan_create_gaussian): the operands they own
  int channels = 0;
  void* gauss_ws = nullptr;
  mas::GaussOperands gauss_own = {};
  CUtensorMap gauss_tmb;
};

extern "C" {

void mas_config_default(mas_config_t* cfg) {
  cfg->engine = MAS_ENGINE_PARALLEL;
  cfg->max_neg_val = kDefaultMaxNegVal;
  cfg->lane_padding = 0;
  cfg->threads = 0;
  cfg->flags = 0;
}

const char* mas_errc_name(int32_t errc) {
  if (errc < 0 || errc >= static_cast<int32_t>(sizeof(kErrcNames) / sizeof(kErrcNames[0])))
    return "Unknown";
  return kErrcNames[errc];
}

int mas_abi_version(void) { return MAS_ABI_VERSION; }

void mas_plan_destroy(mas_plan_t* p) {
  if (!p) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  // A caller-held plan may still have kernels in flight on the caller's
  // streams: wait for the last enqueue on each before the workspace goes back
  // to the pool (enqueues made under stream capture are only known to the
  // graph, so then the whole device is synchronised).
  if (!p->internal) {
    if (p->captured) cudaDeviceSynchronize();
    for (auto& se : p->done) cudaEventSynchronize(se.second);
  }
  for (auto& se : p->done) cudaEventDestroy(se.second);
  cudaStream_t st = cudaStreamPerThread;
  cudaFreeAsync(p->d_lengths, st);
  cudaFreeAsync(p->d_dirs_buf[0], st);
  if (p->d_dirs_buf[1]) cudaFreeAsync(p->d_dirs_buf[1], st);
  if (p->d_bt_done) cudaFreeAsync(p->d_bt_done, st);
  cudaFreeAsync(p->d_flags_buf[0], st);
  cudaFreeAsync(p->d_locate, st);
  if (p->d_bnd) cudaFreeAsync(p->d_bnd, st);
  if (p->d_sync) cudaFreeAsync(p->d_sync, st);
  if (p->gauss_ws) cudaFreeAsync(p->gauss_ws, st);
  if (p->ws_ready) cudaEventDestroy(p->ws_ready);
  cudaSetDevice(prev);
  delete p;
}

}  // extern "C"

namespace {
int plan_create(int32_t batch, int32_t text_cap, int32_t speech_cap, int64_t row_pitch,
                const uint32_t* lengths, const mas_config_t* cfg_in, int item_base,
                mas_plan_t** plan_out, mas_error_t* err, bool deferred = false, int gauss_kp = 0);
}  // namespace

extern "C" {

int mas_plan_create(int32_t batch, int32_t text_cap, int32_t speech_cap, int64_t row_pitch,
                    const uint32_t* lengths, const mas_config_t* cfg_in, mas_plan_t** plan_out,
                    mas_error_t* err) {
  return plan_create(batch, text_cap, speech_cap, row_pitch, lengths, cfg_in, 0, plan_out, err);
}

}  // extern "C"

namespace {

// deferred: the workspace set-up is ordered before the plan's first
// enqueue by an event instead of a host synchronisation (internal plans of
// mas_align_host / _device, whose enqueues are never captured).
int plan_create(int32_t batch, int32_t text_cap, int32_t speech_cap, int64_t row_pitch,
                const uint32_t* lengths, const mas_config_t* cfg_in, int item_base,
                mas_plan_t** plan_out, mas_error_t* err, bool deferred, int gauss_kp) {
  clear_error(err);
  *plan_out = nullptr;
  mas_config_t cfg;
  if (cfg_in)
    cfg = *cfg_in;
  else
    mas_config_default(&cfg);
  int rc = validate_config(cfg, err);  // align_parallel / align_reference first step
  if (rc) return rc;
  rc = validate_dims(batch, text_cap, speech_cap, err);
  if (rc) return rc;
  if (row_pitch < speech_cap)
    return set_error(err, MAS_E_UNSUPPORTED, -1, -1, "row_pitch must be >= speech_cap");

  auto* p = new (std::nothrow) mas_plan();
  if (!p) return set_error(err, MAS_E_UNSUPPORTED, -1, -1, "out of host memory");
  cudaGetDevice(&p->device);
  p->item_base = item_base;
  p->B = batch;
  p->T = text_cap;
  p->S = speech_cap;
  p->pitch = row_pitch;
  p->T_pad = text_cap;
  p->mode = cfg.engine == MAS_ENGINE_REFERENCE ? 1 : 0;
  p->mnv = cfg.max_neg_val;
  p->nan_parallel = p->mode == 0 && std::isnan(cfg.max_neg_val) && gauss_kp == 0;
  p->gauss_kp = gauss_kp;
  p->lengths.resize(static_cast<size_t>(batch) * 2);
  int t_max = 0;
  for (int b = 0; b < batch; ++b) {
    const uint32_t t = lengths ? lengths[2 * b] : static_cast<uint32_t>(text_cap);
    const uint32_t s = lengths ? lengths[2 * b + 1] : static_cast<uint32_t>(speech_cap);
    ItemError ie;
    if (length_error(b + item_base, t, s, text_cap, speech_cap, &ie)) {
      if (p->first_host_error.item < 0) p->first_host_error = ie;
      p->lengths[2 * b] = 0;
      p->lengths[2 * b + 1] = 0;
      p->all_full = false;
    } else {
      p->lengths[2 * b] = t;
      p->lengths[2 * b + 1] = s;
      if (t != static_cast<uint32_t>(text_cap) || s != static_cast<uint32_t>(speech_cap))
        p->all_full = false;
      t_max = std::max<int>(t_max, static_cast<int>(t));
    }
  }
  if (mas::fwd4_configure() != cudaSuccess) {
    delete p;
    return set_error(err, MAS_E_CUDA, -1, -1, "forward kernel configuration failed");
  }
  if (!cached_geometry(batch, std::max(t_max, 1), speech_cap, &p->geo, gauss_kp)) {
    delete p;
    return set_error(err, MAS_E_UNSUPPORTED, -1, -1,
                     "no launch geometry fits this shape on the device");
  }
  const Geometry& g = p->geo;
  auto fail = [&](cudaError_t e, const char* what) {
    mas_plan_destroy(p);
    return cuda_error(err, e, what);
  };
  cudaError_t e;
  if ((e = mas::fwd4_configure()) != cudaSuccess)
    return fail(e, "fwd_configure");
  if ((e = mas::bt_configure(g.T_alloc, g.L)) != cudaSuccess) return fail(e, "bt_configure");
  // Workspace from the stream-ordered pool on this thread's default stream;
  // synchronised below, so it is valid on any stream afterwards.
  cudaStream_t st = cudaStreamPerThread;
  const size_t nB = static_cast<size_t>(batch);
  if ((e = mas::pool_alloc(reinterpret_cast<void**>(&p->d_lengths), nB * 2 * sizeof(uint32_t),
                           st)) != cudaSuccess)
    return fail(e, "mas::pool_alloc(lengths)");
  if ((e = cudaMemcpyAsync(p->d_lengths, p->lengths.data(), nB * 2 * sizeof(uint32_t),
                           cudaMemcpyHostToDevice, st)) != cudaSuccess)
    return fail(e, "cudaMemcpyAsync(lengths)");
  p->pipelined = (cfg.flags & MAS_FLAG_PIPELINED) != 0u && !deferred;
  for (int k = 0; k < (p->pipelined ? 2 : 1); ++k)
    if ((e = mas::pool_alloc(reinterpret_cast<void**>(&p->d_dirs_buf[k]),
                             nB * g.M * g.T_alloc * sizeof(uint32_t), st)) != cudaSuccess)
      return fail(e, "mas::pool_alloc(dirs)");
  p->d_dirs = p->d_dirs_buf[0];
  if (p->pipelined) {
    if ((e = mas::pool_alloc(reinterpret_cast<void**>(&p->d_bt_done), 2 * sizeof(unsigned), st)) !=
            cudaSuccess ||
        (e = cudaMemsetAsync(p->d_bt_done, 0, 2 * sizeof(unsigned), st)) != cudaSuccess)
      return fail(e, "backtrack counters");
  }
  p->bt_rows = std::min(256, g.T_alloc);  // backtrack window rows
  if (g.bands > 1) {
    p->bnd_pitch = (speech_cap + 31) & ~31;
    if ((e = mas::pool_alloc(reinterpret_cast<void**>(&p->d_bnd),
                             nB * (g.bands - 1) * p->bnd_pitch * sizeof(float), st)) !=
        cudaSuccess)
      return fail(e, "mas::pool_alloc(boundary rows)");
    if ((e = mas::pool_alloc(reinterpret_cast<void**>(&p->d_sync),
                             nB * g.bands * sizeof(int), st)) != cudaSuccess)
      return fail(e, "mas::pool_alloc(band progress)");
  }
  // pipelined plans: consecutive forward kernels may overlap, so each
  // direction-word buffer has its own NonFinite flags
  if ((e = mas::pool_alloc(reinterpret_cast<void**>(&p->d_flags_buf[0]),
                           (p->pipelined ? 2 : 1) * nB * sizeof(int), st)) != cudaSuccess)
    return fail(e, "mas::pool_alloc(flags)");
  p->d_flags_buf[1] = p->pipelined ? p->d_flags_buf[0] + nB : nullptr;
  p->d_flags = p->d_flags_buf[0];
  if ((e = mas::pool_alloc(reinterpret_cast<void**>(&p->d_locate), sizeof(unsigned long long),
                           st)) != cudaSuccess)
    return fail(e, "mas::pool_alloc(locate)");
  if (deferred) {
    if ((e = cudaEventCreateWithFlags(&p->ws_ready, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventRecord(p->ws_ready, st)) != cudaSuccess)
      return fail(e, "plan workspace");
  } else if ((e = cudaStreamSynchronize(st)) != cudaSuccess) {
    return fail(e, "plan workspace");
  }
  *plan_out = p;
  return MAS_OK;
}

}  // namespace

extern "C" {

int mas_plan_launches(const mas_plan_t* p) { return p ? p->launches : 0; }

void mas_plan_geometry(const mas_plan_t* p, int32_t geom[6]) {
  geom[5] = mas::fwd4_max_active_clusters(p->geo.R, p->geo.W, p->geo.N, p->geo.K, p->gauss_kp);
  geom[0] = 32 * p->geo.R;
  geom[1] = p->geo.W;
  geom[2] = p->geo.K;
  geom[3] = p->geo.N;
  geom[4] = p->geo.L;
}

}  // extern "C"

namespace {

// Enqueues the kernels (MAS_PART_* bits) for items [b0, b0 + nb) of the
// plan's batch.  d_values / d_out / d_paths are the whole batch's buffers.
// The one-launch tail (mas_fwd4.cu OUT 2) applies to a whole-batch enqueue of
// a plain (not pipelined, not Gaussian, not NaN-sentinel) plan whose items
// each fit one single-CTA cluster, when the direction words fit shared memory.
bool tail_ok(const mas_plan_t* p, uint32_t parts, const uint8_t* d_out, const int32_t* d_paths,
             const int32_t* d_dur) {
  const Geometry& g = p->geo;
  if (p->pipelined || p->gauss || p->nan_parallel || g.K != 1 || g.bands != 1) return false;
  if ((parts & MAS_PART_ALL) != MAS_PART_ALL || !(d_out || d_paths || d_dur)) return false;
  constexpr size_t kSmemMax = 227 * 1024;
  return mas::fwd4_smem_bytes(g.R, g.W, g.N) + mas::fwd4_tail_bytes(g.R, g.W, g.M) <= kSmemMax;
}

int enqueue_items(mas_plan_t* p, uint32_t parts, int b0, int nb, const float* d_values,
                  uint8_t* d_out, int32_t* d_paths, int32_t* d_dur, cudaStream_t stream,
                  mas_error_t* err) {
  if (!p->gauss &&
      ((reinterpret_cast<uintptr_t>(d_values) & 15u) != 0 || (p->pitch & 3) != 0 || (p->T_pad & 3)))
    return set_error(err, MAS_E_UNSUPPORTED, -1, -1,
                     "device layout needs a 16-byte base, pitch % 4 == 0 and text_cap % 4 == 0");
  const Geometry& g = p->geo;
  if (p->ws_ready) MAS_CUDA(cudaStreamWaitEvent(stream, p->ws_ready, 0), "workspace wait");
  int nfwd = 0, nbt = 0;
  if (p->pipelined && (parts & MAS_PART_FORWARD)) {  // next direction-word / flags buffers
    p->dirs_par ^= 1;
    p->d_dirs = p->d_dirs_buf[p->dirs_par];
    p->d_flags = p->d_flags_buf[p->dirs_par];
  }
  if ((parts & MAS_PART_FORWARD) && p->nan_parallel) {
    // parallel::detail::align_unchecked with a NaN sentinel: std::max's rule
    // ((a < b) ? b : a, a NaN first operand wins) shapes the score table,
    // which K1's FMNMX does not follow.  The table is computed with that rule
    // (forward_scores_kernel, bit-exact with forward_parallel) in a scratch
    // copy and its decisions are packed into the plan's direction words, so
    // K2 runs unchanged.  Unchecked (test-only) sentinels only.
    const size_t item_floats = static_cast<size_t>(p->T_pad) * p->pitch;
    float* scratch = nullptr;
    MAS_CUDA(mas::pool_alloc(reinterpret_cast<void**>(&scratch), nb * item_floats * 4, stream),
             "pool_alloc(nan scratch)");
    const float* src = d_values + b0 * item_floats;
    cudaError_t e = cudaMemcpyAsync(scratch, src, nb * item_floats * 4, cudaMemcpyDeviceToDevice, stream);
    mas_error_t sub;
    int rc = MAS_OK;
    if (e == cudaSuccess)
      rc = mas::forward_scores_host_lengths(scratch, p->pitch, nb, p->T_pad, p->S,
                                            p->lengths.data() + 2 * static_cast<size_t>(b0), p->mnv,
                                            stream, &sub);
    if (e == cudaSuccess && rc == MAS_OK)
      e = mas::launch_scores_to_dirs(scratch, p->pitch, p->T_pad, p->S, p->d_lengths + 2 * b0, g.M,
                                     g.T_alloc, nb, p->d_dirs + static_cast<size_t>(b0) * g.M * g.T_alloc,
                                     stream);
    if (e == cudaSuccess && rc == MAS_OK)
      e = mas::launch_flag_nonfinite(src, p->pitch, p->T_pad, p->S, p->d_lengths + 2 * b0, nb,
                                     p->d_flags + b0, stream);
    if (e == cudaSuccess && rc == MAS_OK && d_out)
      e = cudaMemsetAsync(d_out + b0 * static_cast<size_t>(p->T) * p->S, 0,
                          nb * static_cast<size_t>(p->T) * p->S, stream);
    cudaFreeAsync(scratch, stream);
    if (rc != MAS_OK) return set_error(err, rc, -1, -1, sub.message);
    MAS_CUDA(e, "NaN-sentinel forward");
    nfwd = 4;
  } else if (parts & MAS_PART_FORWARD) {
    CUtensorMap tm0;
    // Tensor maps depend only on the buffers and the plan's layout: encoded
    // once per input pointer and reused by later enqueues (host cost).
    const bool reuse_in = p->tm_in_ptr == d_values && p->tm_in_pitch == p->pitch &&
                          p->tm_in_tpad == p->T_pad;
    if (p->gauss) {
      tm0 = *p->gauss_map;
    } else if (reuse_in) {
      tm0 = p->tm_in;
    } else if (!encode_map4(d_values, p->pitch, static_cast<int64_t>(p->B) * p->T_pad, p->S, g.R,
                            &tm0)) {
      return set_error(err, MAS_E_CUDA, -1, -1, "cuTensorMapEncodeTiled failed");
    } else {
      p->tm_in = tm0;
      p->tm_in_ptr = d_values;
      p->tm_in_pitch = p->pitch;
      p->tm_in_tpad = p->T_pad;
    }
    mas::FwdArgs fa = {};
    fa.b0 = b0;
    fa.lengths = p->d_lengths;
    fa.dirs = p->d_dirs;
    fa.flags = p->d_flags;
    fa.T_pad = p->T_pad;
    fa.M = g.M;
    fa.T_alloc = g.T_alloc;
    fa.K = g.K;
    fa.W = g.W;
    fa.N = g.N;
    fa.mnv = p->mnv;
    fa.row0_up = p->mode == 1 ? -std::numeric_limits<float>::infinity() : p->mnv;
    // The output's zero fill rides along with the forward pass when every
    // item is full length (its warps then cover every row and column) and
    // K1 is bound by its column chains: the stores are then nearly free.
    // When K1 is HBM-bound, interleaving 1 B/cell of writes with the
    // 4 B/cell read stream costs more than a separate memset (measured at
    // B256 T512 S4096: 527 us fused vs 380 + ~80 us).  Estimate: the chains
    // take S x ~50 cycles per warp (x warps per SM sub-partition beyond
    // one), the stream cells x 4.125 B at ~5.9 TB/s.  Ragged batches always
    // take the memset.
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
    const double warps = static_cast<double>(nb) * g.bands * g.K * g.W;
    const double chain_s = p->S * 50.0 / 1.9e9 * std::max(1.0, warps / (4.0 * sms));
    const double stream_s = static_cast<double>(nb) * p->T * p->S * 4.125 / 5.9e12;
    const bool chain_bound = stream_s <= 1.1 * chain_s;
    // (each warp zeroes its own rows, so every row is covered only when every
    // item is full length -- or in the one-launch tail, whose producer lanes
    // also zero the rows of warps past a short item; the bulk stores need
    // 16-byte rows)
    const bool tail = tail_ok(p, parts, d_out, d_paths, d_dur);
    const bool fused_zero = d_out && (tail || (chain_bound && p->all_full)) && (p->S % 16) == 0 &&
                            (reinterpret_cast<uintptr_t>(d_out) & 15u) == 0;
    const size_t item_bytes = static_cast<size_t>(p->T) * p->S;
    if (d_out && !fused_zero) {
      MAS_CUDA(cudaMemsetAsync(d_out + b0 * item_bytes, 0, nb * item_bytes, stream),
               "cudaMemsetAsync(out)");
    }
    CUtensorMap tm_out;  // (the score export's store map; unused here)
    std::memset(&tm_out, 0, sizeof(tm_out));
    fa.zero_fill = fused_zero ? 1 : 0;
    fa.out = d_out;
    fa.l2_ahead = 0;  // measured: an L2 prefetch lead beyond the ring only hurts
    fa.one = 1u;
    fa.zero = 0.0f;
    fa.T_cap = p->T;
    fa.S_cap = p->S;
    fa.bands = g.bands;
    fa.band_rows = g.band_rows;
    fa.nb = nb;
    fa.bnd = p->d_bnd;
    fa.bnd_pitch = p->bnd_pitch;
    if (p->gauss) {
      fa.Kp = p->gauss->Kp;
      const mas::GaussCfg gc = mas::gauss_cfg(g.W, fa.Kp);
      fa.gstages = gc.gstages;
      fa.gacc = gc.gacc;
      fa.gN = gc.gN;
      fa.Tp = p->gauss->Tp;
      fa.Sp = p->gauss->Sp;
      fa.gA = p->gauss->A;
      fa.gbias = p->gauss->bias;
    }
    if (p->pipelined) {
      fa.bt_done = p->d_bt_done + p->dirs_par;
      fa.bt_need = p->bt_issued[p->dirs_par];
      fa.pdl = 1;
    }
    // One launch for small batches: every item one single-CTA cluster (K = 1,
    // one band) whose direction words fit shared memory beside the ring; the
    // CTA then walks and expands its own item, and no backtrack kernel runs.
    if (tail) {
      fa.tail = 1;
      fa.path = d_paths;
      fa.dur = d_dur;
    }
    fa.ticket = p->d_sync ? p->d_sync + b0 : nullptr;
    fa.progress = p->d_sync ? p->d_sync + p->B : nullptr;
    // All bands of all items in one launch (clusters ordered by ticket).
    if (g.bands > 1) {
      MAS_CUDA(cudaMemsetAsync(fa.ticket, 0, sizeof(int), stream), "cudaMemsetAsync(ticket)");
      MAS_CUDA(cudaMemsetAsync(fa.progress + static_cast<size_t>(b0) * (g.bands - 1), 0,
                               sizeof(int) * nb * (g.bands - 1), stream),
               "cudaMemsetAsync(progress)");
    }
    MAS_CUDA(mas::launch_fwd4(g.R, p->mode, tm0, tm_out, fa, nb * g.bands, stream),
             "launch mas_fwd4");
    nfwd = 1;
  }
  if ((parts & MAS_PART_BACKTRACK) && (d_out || d_paths || d_dur) &&
      !tail_ok(p, parts, d_out, d_paths, d_dur)) {
    mas::BtArgs ba = {};
    ba.b0 = b0;
    ba.lengths = p->d_lengths;
    ba.dirs = p->d_dirs;
    ba.path = d_paths;
    ba.out = d_out;
    ba.dur = d_dur;
    ba.B = nb;
    ba.T_cap = p->T;
    ba.S_cap = p->S;
    ba.M = g.M;
    ba.T_alloc = g.T_alloc;
    ba.R = p->bt_rows;
    ba.done = p->pipelined ? p->d_bt_done + p->dirs_par : nullptr;
    MAS_CUDA(mas::launch_backtrack(ba, stream, &nbt), "launch backtrack");
    if (p->pipelined) p->bt_issued[p->dirs_par] += static_cast<unsigned>(nb);
  }
  p->launches = nfwd + nbt;
  return MAS_OK;
}

// q's storage as the score export's store target: {columns, row groups of R
// within an item, residue, item}, so a warp's {32, 32, R, 1} box clips at its
// item's last row (a flat row map would spill into the next item, whose own
// CTAs may already have written it).
bool encode_scores_map4(float* q, int64_t pitch, int T_cap, int64_t S, int B, int R,
                        CUtensorMap* m) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[4] = {static_cast<cuuint64_t>(S), static_cast<cuuint64_t>(T_cap / R),
                              static_cast<cuuint64_t>(R), static_cast<cuuint64_t>(B)};
  const cuuint64_t strides[3] = {static_cast<cuuint64_t>(R * pitch * 4),
                                 static_cast<cuuint64_t>(pitch * 4),
                                 static_cast<cuuint64_t>(T_cap * pitch * 4)};
  const cuuint32_t box[4] = {32, 32, static_cast<cuuint32_t>(R), 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, q, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

namespace mas {

// Score export (parallel::forward_parallel / reference::forward_reference)
// through K1 with OUT = 1: the forward pass of the maximum-path call with
// its Q values written back over q by TMA stores (8 B/cell, HBM-bound),
// instead of mas_scores.cu's general kernel.  Needs the TMA layout K1 reads
// (16-byte base, pitch % 4 == 0, text_cap % 4 == 0); returns
// MAS_E_UNSUPPORTED without launching anything otherwise.
int forward_scores_fwd4(float* d_values, int64_t pitch, int B, int T_cap, int S_cap,
                        const uint32_t* lengths, int mode, float mnv, cudaStream_t stream,
                        mas_error_t* err) {
  if ((reinterpret_cast<uintptr_t>(d_values) & 15u) != 0 || (pitch & 3) != 0 || (T_cap & 3) != 0 ||
      (pitch * 4) % 16 != 0)
    return MAS_E_UNSUPPORTED;
  std::vector<uint32_t> lens(static_cast<size_t>(B) * 2);
  int t_max = 0;
  for (int b = 0; b < B; ++b) {
    lens[2 * b] = lengths ? lengths[2 * b] : static_cast<uint32_t>(T_cap);
    lens[2 * b + 1] = lengths ? lengths[2 * b + 1] : static_cast<uint32_t>(S_cap);
    if (lens[2 * b + 1] > 0) t_max = std::max<int>(t_max, static_cast<int>(lens[2 * b]));
  }
  if (fwd4_configure() != cudaSuccess) return MAS_E_UNSUPPORTED;
  Geometry g;
  if (!cached_geometry(B, std::max(t_max, 1), S_cap, &g)) return MAS_E_UNSUPPORTED;
  CUtensorMap tm_in, tm_st;
  if (!encode_map4(d_values, pitch, static_cast<int64_t>(B) * T_cap, S_cap, g.R, &tm_in) ||
      !encode_scores_map4(d_values, pitch, T_cap, S_cap, B, g.R, &tm_st))
    return MAS_E_UNSUPPORTED;
  // workspace: lengths [B][2] | band links [B][bands-1][bnd_pitch] | ticket + progress
  const int bnd_pitch = (S_cap + 31) & ~31;
  // (sub-buffers 256-byte aligned: the band links are copied in 16-byte vectors and bulk copies)
  const size_t len_bytes = (static_cast<size_t>(B) * 2 * sizeof(uint32_t) + 255) & ~size_t{255};
  const size_t bnd_bytes =
      g.bands > 1 ? static_cast<size_t>(B) * (g.bands - 1) * bnd_pitch * sizeof(float) : 0;
  const size_t sync_bytes = g.bands > 1 ? (1 + static_cast<size_t>(B) * (g.bands - 1)) * sizeof(int) : 0;
  char* ws = nullptr;
  MAS_CUDA(pool_alloc(reinterpret_cast<void**>(&ws), len_bytes + bnd_bytes + sync_bytes, stream),
           "forward_scores: workspace");
  FwdArgs fa = {};
  fa.lengths = reinterpret_cast<uint32_t*>(ws);
  fa.bnd = g.bands > 1 ? reinterpret_cast<float*>(ws + len_bytes) : nullptr;
  fa.ticket = g.bands > 1 ? reinterpret_cast<int*>(ws + len_bytes + bnd_bytes) : nullptr;
  fa.progress = g.bands > 1 ? fa.ticket + 1 : nullptr;
  fa.bnd_pitch = bnd_pitch;
  fa.b0 = 0;
  fa.T_pad = T_cap;
  fa.M = g.M;
  fa.T_alloc = g.T_alloc;
  fa.K = g.K;
  fa.W = g.W;
  fa.N = g.N;
  fa.mnv = mnv;
  fa.row0_up = mode == 1 ? -std::numeric_limits<float>::infinity() : mnv;
  fa.T_cap = T_cap;
  fa.S_cap = S_cap;
  fa.bands = g.bands;
  fa.band_rows = g.band_rows;
  fa.nb = B;
  fa.one = 1u;
  fa.scores = 1;
  cudaError_t e = cudaMemcpyAsync(ws, lens.data(), lens.size() * sizeof(uint32_t),
                                  cudaMemcpyHostToDevice, stream);
  if (e == cudaSuccess && sync_bytes)
    e = cudaMemsetAsync(fa.ticket, 0, sync_bytes, stream);
  if (e == cudaSuccess) e = launch_fwd4(g.R, mode, tm_in, tm_st, fa, B * g.bands, stream);
  const cudaError_t f = cudaFreeAsync(ws, stream);
  if (e == cudaSuccess) e = f;
  MAS_CUDA(e, "forward_scores");
  return MAS_OK;
}

}  // namespace mas

extern "C" {

int mas_plan_enqueue(mas_plan_t* p, const float* d_values, uint8_t* d_out, int32_t* d_paths,
                     void* stream_v, mas_error_t* err) {
  return mas_plan_enqueue_ex(p, MAS_PART_ALL, d_values, d_out, d_paths, nullptr, stream_v, err);
}

int mas_plan_enqueue_part(mas_plan_t* p, uint32_t parts, const float* d_values, uint8_t* d_out,
                          int32_t* d_paths, void* stream_v, mas_error_t* err) {
  return mas_plan_enqueue_ex(p, parts, d_values, d_out, d_paths, nullptr, stream_v, err);
}

int mas_plan_enqueue_ex(mas_plan_t* p, uint32_t parts, const float* d_values, uint8_t* d_out,
                        int32_t* d_paths, int32_t* d_durations, void* stream_v,
                        mas_error_t* err) {
  clear_error(err);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (!p->internal) MAS_CUDA(cudaStreamIsCapturing(stream, &cap), "cudaStreamIsCapturing");
  if (p->pipelined && cap != cudaStreamCaptureStatusNone)
    return set_error(err, MAS_E_UNSUPPORTED, -1, -1,
                     "pipelined plans cannot be captured in a CUDA graph");
  const int rc = enqueue_items(p, parts, 0, p->B, d_values, d_out, d_paths, d_durations, stream, err);
  if (rc != MAS_OK || p->internal) return rc;
  // remember the enqueue so mas_plan_destroy can wait for it
  if (cap != cudaStreamCaptureStatusNone) {
    p->captured = true;
    return MAS_OK;
  }
  cudaEvent_t ev = nullptr;
  for (auto& se : p->done)
    if (se.first == stream) ev = se.second;
  if (!ev) {
    MAS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
    p->done.emplace_back(stream, ev);
  }
  MAS_CUDA(cudaEventRecord(ev, stream), "cudaEventRecord");
  return MAS_OK;
}

int mas_plan_finish(mas_plan_t* p, const float* d_values, void* stream_v, mas_error_t* err) {
  clear_error(err);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  // (a device-to-pageable copy returns once the stream's earlier work and
  // the copy are done: one host round trip)
  std::vector<int> flags(p->B);
  MAS_CUDA(cudaMemcpyAsync(flags.data(), p->d_flags, sizeof(int) * p->B, cudaMemcpyDeviceToHost,
                           stream),
           "cudaMemcpyAsync(flags)");
  MAS_CUDA(cudaStreamSynchronize(stream), "flags readback");
  // first_host_error.item carries item_base (message numbering); flags are
  // indexed from 0 within this plan.
  const int limit = p->first_host_error.item >= 0
                        ? std::max(0, std::min(p->B, p->first_host_error.item - p->item_base))
                        : p->B;
  // Gaussian plans: q exists only as tiles inside the forward kernel; a
  // flagged item materialises it (error path only) from the operands of the
  // last enqueue for the exact row-major location.
  float* q_tmp = nullptr;
  struct QTmp {
    float*& q;
    cudaStream_t s;
    ~QTmp() {
      if (q) cudaFreeAsync(q, s);
    }
  } q_guard{q_tmp, stream};
  if (p->gauss_ws && !d_values) {
    bool any = false;
    for (int b = 0; b < limit; ++b) any = any || flags[b] != 0;
    if (any) {
      MAS_CUDA(mas::pool_alloc(reinterpret_cast<void**>(&q_tmp),
                               static_cast<size_t>(p->B) * p->T_pad * p->pitch * sizeof(float),
                               stream),
               "pool_alloc(q)");
      MAS_CUDA(mas::gauss_q(p->gauss_own, p->B, p->T, p->S, q_tmp, p->pitch, stream),
               "gaussian q");
      d_values = q_tmp;
    }
  }
  for (int b = 0; b < limit; ++b) {
    if (!flags[b]) continue;
    // Conservative device flag: confirm and locate exactly (row-major first).
    const unsigned long long none = ~0ull;
    MAS_CUDA(cudaMemcpyAsync(p->d_locate, &none, sizeof(none), cudaMemcpyHostToDevice, stream),
             "locate init");
    MAS_CUDA(mas::launch_locate_nonfinite(d_values, p->pitch, p->T_pad, b,
                                          static_cast<int>(p->lengths[2 * b]),
                                          static_cast<int>(p->lengths[2 * b + 1]), p->d_locate,
                                          stream),
             "locate");
    unsigned long long hit = none;
    MAS_CUDA(cudaMemcpyAsync(&hit, p->d_locate, sizeof(hit), cudaMemcpyDeviceToHost, stream),
             "locate read");
    MAS_CUDA(cudaStreamSynchronize(stream), "locate sync");
    if (hit != none) {
      const int64_t s = p->lengths[2 * b + 1];
      const int64_t i = static_cast<int64_t>(hit / s), j = static_cast<int64_t>(hit % s);
      set_error(err, MAS_E_VALIDATION, MAS_ERRC_NON_FINITE, b + p->item_base,
                nonfinite_message(b + p->item_base, i, j));
      if (err) {
        err->i = i;
        err->j = j;
      }
      return MAS_E_VALIDATION;
    }
  }
  if (p->first_host_error.item >= 0)
    return set_error(err, MAS_E_VALIDATION, p->first_host_error.errc, p->first_host_error.item,
                     p->first_host_error.message);
  return MAS_OK;
}

int mas_align_device(const float* d_values, int64_t row_pitch, int32_t batch, int32_t text_cap,
                     int32_t speech_cap, const uint32_t* lengths, const mas_config_t* cfg,
                     uint8_t* d_out, int32_t* d_paths, void* stream_v, mas_error_t* err) {
  return mas_align_device_ex(d_values, row_pitch, batch, text_cap, speech_cap, lengths, cfg, d_out,
                             d_paths, nullptr, stream_v, err);
}

}  // extern "C"

namespace {

// Plans of mas_align_device_ex kept across calls (a training loop calls with
// the same shape every step): validation, geometry, workspace and tensor maps
// once, then each call is the kernels and (unless MAS_FLAG_NO_CHECK) one
// flags readback.  Keyed by everything the plan depends on, including the
// stream (its workspace is stream-ordered); a plan is checked out while in
// use, so concurrent callers never share one.
struct PlanKey {
  int dev;
  cudaStream_t stream;
  int32_t B, T, S;
  int64_t pitch;
  int32_t engine, threads;
  uint32_t flags;
  uint32_t mnv_bits;
  std::vector<uint32_t> lengths;
  bool operator==(const PlanKey& o) const {
    return dev == o.dev && stream == o.stream && B == o.B && T == o.T && S == o.S &&
           pitch == o.pitch && engine == o.engine && threads == o.threads && flags == o.flags &&
           mnv_bits == o.mnv_bits && lengths == o.lengths;
  }
};

class PlanCache {
 public:
  static PlanCache& get() {
    static PlanCache* c = new PlanCache();  // never destroyed: plans outlive static teardown
    return *c;
  }
  mas_plan_t* take(const PlanKey& k) {
    std::lock_guard<std::mutex> lk(mu_);
    for (size_t i = 0; i < idle_.size(); ++i)
      if (idle_[i].first == k) {
        mas_plan_t* p = idle_[i].second;
        idle_.erase(idle_.begin() + static_cast<long>(i));
        return p;
      }
    return nullptr;
  }
  void give(PlanKey k, mas_plan_t* p) {
    mas_plan_t* evict = nullptr;
    {
      std::lock_guard<std::mutex> lk(mu_);
      idle_.emplace_back(std::move(k), p);
      if (idle_.size() > kMax) {
        evict = idle_.front().second;
        idle_.erase(idle_.begin());
      }
    }
    if (evict) mas_plan_destroy(evict);
  }

 private:
  static constexpr size_t kMax = 16;
  std::mutex mu_;
  std::vector<std::pair<PlanKey, mas_plan_t*>> idle_;
};

PlanKey plan_key(cudaStream_t stream, int32_t B, int32_t T, int32_t S, int64_t pitch,
                 const uint32_t* lengths, const mas_config_t& c) {
  PlanKey k;
  cudaGetDevice(&k.dev);
  k.stream = stream;
  k.B = B;
  k.T = T;
  k.S = S;
  k.pitch = pitch;
  k.engine = c.engine;
  k.threads = c.threads;
  k.flags = c.flags & MAS_FLAG_UNCHECKED;
  std::memcpy(&k.mnv_bits, &c.max_neg_val, 4);
  if (lengths) k.lengths.assign(lengths, lengths + 2 * static_cast<size_t>(B));
  return k;
}

}  // namespace

extern "C" {

int mas_align_device_ex(const float* d_values, int64_t row_pitch, int32_t batch,
                        int32_t text_cap, int32_t speech_cap, const uint32_t* lengths,
                        const mas_config_t* cfg, uint8_t* d_out, int32_t* d_paths,
                        int32_t* d_durations, void* stream_v, mas_error_t* err) {
  clear_error(err);
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  mas_config_t c;
  if (cfg)
    c = *cfg;
  else
    mas_config_default(&c);
  const bool check = (c.flags & MAS_FLAG_NO_CHECK) == 0u;
  const bool repitch = (reinterpret_cast<uintptr_t>(d_values) & 15u) != 0 || (row_pitch & 3) != 0 ||
                       (text_cap & 3) != 0;
  if (repitch) {
    mas_plan_t* plan = nullptr;
    int rc = plan_create(batch, text_cap, speech_cap, row_pitch, lengths, &c, 0, &plan, err, true);
    if (rc) return rc;
    plan->internal = true;
    // Re-pitch into an aligned [B][T_pad][pitch'] copy the TMA path accepts.
    const int T_pad = (text_cap + 3) & ~3;
    const int64_t pitch2 = (static_cast<int64_t>(speech_cap) + 3) & ~int64_t(3);
    float* scratch = nullptr;
    cudaError_t e = mas::pool_alloc(reinterpret_cast<void**>(&scratch),
                                    static_cast<size_t>(batch) * T_pad * pitch2 * 4, stream);
    if (e != cudaSuccess) {
      mas_plan_destroy(plan);
      return cuda_error(err, e, "mas::pool_alloc(repitch)");
    }
    for (int b = 0; b < batch && e == cudaSuccess; ++b) {
      e = cudaMemcpy2DAsync(scratch + static_cast<size_t>(b) * T_pad * pitch2, pitch2 * 4,
                            d_values + static_cast<size_t>(b) * text_cap * row_pitch,
                            row_pitch * 4, static_cast<size_t>(speech_cap) * 4, text_cap,
                            cudaMemcpyDeviceToDevice, stream);
    }
    if (e != cudaSuccess) {
      cudaFreeAsync(scratch, stream);
      mas_plan_destroy(plan);
      return cuda_error(err, e, "repitch copy");
    }
    plan->pitch = pitch2;
    plan->T_pad = T_pad;
    rc = mas_plan_enqueue_ex(plan, MAS_PART_ALL, scratch, d_out, d_paths, d_durations, stream, err);
    if (rc == MAS_OK) rc = mas_plan_finish(plan, scratch, stream, err);
    cudaFreeAsync(scratch, stream);
    cudaStreamSynchronize(stream);
    mas_plan_destroy(plan);
    return rc;
  }
  PlanKey key = plan_key(stream, batch, text_cap, speech_cap, row_pitch, lengths, c);
  mas_plan_t* plan = PlanCache::get().take(key);
  if (!plan) {
    const int rc = plan_create(batch, text_cap, speech_cap, row_pitch, lengths, &c, 0, &plan, err,
                               true);
    if (rc) return rc;
    plan->internal = true;
  }
  int rc = mas_plan_enqueue_ex(plan, MAS_PART_ALL, d_values, d_out, d_paths, d_durations, stream,
                               err);
  if (rc == MAS_OK) {
    if (check) {
      rc = mas_plan_finish(plan, d_values, stream, err);
    } else if (plan->first_host_error.item >= 0) {
      // no device readback: host-detected item errors are still reported
      rc = set_error(err, MAS_E_VALIDATION, plan->first_host_error.errc,
                     plan->first_host_error.item, plan->first_host_error.message);
    }
  }
  if (rc == MAS_OK || rc == MAS_E_VALIDATION) {
    PlanCache::get().give(std::move(key), plan);
  } else {
    cudaStreamSynchronize(stream);
    mas_plan_destroy(plan);
  }
  return rc;
}

}  // extern "C"

namespace {

// ---- pageable host buffers --------------------------------------------
// A numpy array (the reference binding's input) is pageable memory, which
// the copy engines only reach through the driver's small bounce buffers.
// Such calls stage every chunk through pinned buffers instead: host threads
// copy the chunk into a pinned slot while the copy engine moves the previous
// one, and the alignment comes back the same way.

bool is_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Fixed pool of host copy threads; copy() splits one memcpy over them.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  void copy(void* dst, const void* src, size_t bytes) {
    // (a forked child inherits this object but not its threads)
    if (bytes < (4u << 20) || workers_.empty() || getpid() != owner_) {
      std::memcpy(dst, src, bytes);
      return;
    }
    std::lock_guard<std::mutex> one_job(job_mu_);  // one parallel copy at a time
    const size_t parts = workers_.size() + 1;
    const size_t chunk = ((bytes + parts - 1) / parts + 63) & ~size_t(63);
    {
      std::lock_guard<std::mutex> lk(mu_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      bytes_ = bytes;
      chunk_ = chunk;
      next_.store(0);
      pending_ = parts;
      ++gen_;
    }
    cv_.notify_all();
    run_parts();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  CopyPool() : owner_(getpid()) {
    const unsigned hw = std::thread::hardware_concurrency();
    const unsigned n = std::min(15u, hw > 1 ? hw - 1 : 0u);
    for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void run_parts() {
    while (true) {
      const size_t i = next_.fetch_add(1);
      const size_t off = i * chunk_;
      if (off < bytes_) std::memcpy(dst_ + off, src_ + off, std::min(chunk_, bytes_ - off));
      if (off >= bytes_) break;
    }
    std::lock_guard<std::mutex> lk(mu_);
    if (--pending_ == 0) done_cv_.notify_all();
  }
  void loop() {
    uint64_t seen = 0;
    while (true) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      run_parts();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex job_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0, chunk_ = 0, pending_ = 0;
  std::atomic<size_t> next_{0};
  uint64_t gen_ = 0;
  bool stop_ = false;
  pid_t owner_;
};

// Pinned buffers kept for reuse across calls (pinning costs milliseconds),
// bounded: at most kKeepBytes stay page-locked while idle; beyond that idle
// buffers are released (largest first) before new ones are pinned, and
// returned buffers are released instead of kept.
class PinnedPool {
 public:
  static constexpr size_t kKeepBytes = size_t(2) << 30;
  static PinnedPool& get() {
    static PinnedPool pool;
    return pool;
  }
  void* take(size_t bytes) {
    std::lock_guard<std::mutex> lk(mu_);
    size_t best = free_.size();
    for (size_t i = 0; i < free_.size(); ++i)
      if (free_[i].second >= bytes && (best == free_.size() || free_[i].second < free_[best].second))
        best = i;
    if (best < free_.size()) {
      void* p = free_[best].first;
      free_.erase(free_.begin() + static_cast<long>(best));
      return p;
    }
    while (!free_.empty() && pinned_ + bytes > kKeepBytes) {
      auto largest = std::max_element(free_.begin(), free_.end(),
                                      [](const auto& a, const auto& b) { return a.second < b.second; });
      release(*largest);
      free_.erase(largest);
    }
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    pinned_ += bytes;
    sizes_.push_back({p, bytes});
    return p;
  }
  void give(void* p) {
    if (!p) return;
    std::lock_guard<std::mutex> lk(mu_);
    for (const auto& e : sizes_)
      if (e.first == p) {
        if (pinned_ > kKeepBytes)
          release(e);
        else
          free_.push_back(e);
        return;
      }
  }

 private:
  // caller holds mu_
  void release(std::pair<void*, size_t> e) {
    cudaFreeHost(e.first);
    pinned_ -= e.second;
    for (size_t i = 0; i < sizes_.size(); ++i)
      if (sizes_[i].first == e.first) {
        sizes_.erase(sizes_.begin() + static_cast<long>(i));
        break;
      }
  }
  std::mutex mu_;
  std::vector<std::pair<void*, size_t>> free_, sizes_;
  size_t pinned_ = 0;
};

// Two non-blocking streams and a join event per (host thread, device),
// created once: stream creation and destruction are a visible part of a
// small call's latency.
struct HostStreams {
  cudaStream_t st[2] = {nullptr, nullptr};
  cudaEvent_t ready = nullptr;
};
cudaError_t host_streams(int dev, HostStreams** out) {
  constexpr int kMaxDevices = 64;
  thread_local HostStreams cache[kMaxDevices];
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  HostStreams& h = cache[dev];
  cudaError_t e = cudaSuccess;
  for (int k = 0; k < 2 && e == cudaSuccess; ++k)
    if (!h.st[k]) e = cudaStreamCreateWithFlags(&h.st[k], cudaStreamNonBlocking);
  if (e == cudaSuccess && !h.ready) e = cudaEventCreateWithFlags(&h.ready, cudaEventDisableTiming);
  *out = &h;
  return e;
}

int align_host_impl(const float* values, int32_t batch, int32_t text_cap, int32_t speech_cap,
                    const uint32_t* lengths, const mas_config_t* cfg, uint8_t* out,
                    int32_t* paths, int32_t* durations, int item_base, mas_error_t* err) {
  clear_error(err);
  {
    mas_config_t c;
    if (cfg)
      c = *cfg;
    else
      mas_config_default(&c);
    int rc = validate_config(c, err);
    if (rc) return rc;
    rc = validate_dims(batch, text_cap, speech_cap, err);
    if (rc) return rc;
  }
  const int T_pad = (text_cap + 3) & ~3;
  const int64_t pitch = (static_cast<int64_t>(speech_cap) + 3) & ~int64_t(3);
  const size_t q_item = static_cast<size_t>(T_pad) * pitch;  // floats per item on the device
  const size_t o_item = static_cast<size_t>(text_cap) * speech_cap;
  mas_plan_t* plan = nullptr;
  int rc = plan_create(batch, text_cap, speech_cap, pitch, lengths, cfg, item_base, &plan, err,
                       true);
  if (rc) return rc;
  plan->internal = true;
  plan->T_pad = T_pad;

  // Items are processed in chunks on two streams, so the host->device copy
  // of chunk c+1 runs while chunk c computes and copies its alignment back
  // (PCIe is full duplex): the call costs about one pass over the input on
  // the bus instead of input + output + compute in sequence.
  // Chunks of at least ~8 MB of input (launch costs stay small), up to one
  // item each: the finer the chunks, the shorter the un-overlapped head
  // (first H2D) and tail (last compute + D2H).  B32 T1024 S8192: 32 chunks,
  // 13.1 Gcells/s vs 12.2 with 4 (PCIe-bound either way).
  const int64_t in_bytes = static_cast<int64_t>(batch) * text_cap * speech_cap * 4;
  const int by_size = static_cast<int>(std::max<int64_t>(1, in_bytes / (8ll << 20)));
  const int nchunk = std::min(batch, std::min(by_size, 64));
  const int per = (batch + nchunk - 1) / nchunk;
  // Pageable input / output: stage through pinned slots (two each).
  const size_t in_chunk = static_cast<size_t>(per) * o_item * sizeof(float);
  const size_t out_chunk = static_cast<size_t>(per) * o_item;
  // (below ~64 MB the driver's own staging of a pageable copy is quicker
  // than waking the copy threads: B32 T200 S800 1.7 ms direct vs 3.2 staged)
  const bool big = in_bytes >= (64ll << 20);
  const bool stage_in = big && nchunk > 1 && !is_pinned(values);
  const bool stage_out = big && nchunk > 1 && out && !is_pinned(out);
  void* pin_in[2] = {nullptr, nullptr};
  void* pin_out[2] = {nullptr, nullptr};
  cudaEvent_t in_done[2] = {nullptr, nullptr}, out_done[2] = {nullptr, nullptr};
  bool staged = true;
  for (int k = 0; k < 2 && staged; ++k) {
    if (stage_in) staged = (pin_in[k] = PinnedPool::get().take(in_chunk)) != nullptr &&
                           cudaEventCreateWithFlags(&in_done[k], cudaEventDisableTiming) ==
                               cudaSuccess;
    if (stage_out && staged)
      staged = (pin_out[k] = PinnedPool::get().take(out_chunk)) != nullptr &&
               cudaEventCreateWithFlags(&out_done[k], cudaEventDisableTiming) == cudaSuccess;
  }
  const bool use_in = stage_in && staged, use_out = stage_out && staged;
  cudaStream_t st[2] = {nullptr, nullptr};
  float* d_q = nullptr;
  uint8_t* d_out = nullptr;
  int32_t* d_paths = nullptr;
  int32_t* d_dur = nullptr;
  cudaError_t e = cudaSuccess;
  HostStreams* hs = nullptr;
  e = host_streams(plan->device, &hs);
  if (e == cudaSuccess) {
    st[0] = hs->st[0];
    st[1] = hs->st[1];
  }
  if (e == cudaSuccess)
    e = mas::pool_alloc(reinterpret_cast<void**>(&d_q), batch * q_item * sizeof(float), st[0]);
  if (e == cudaSuccess && out)
    e = mas::pool_alloc(reinterpret_cast<void**>(&d_out), batch * o_item, st[0]);
  if (e == cudaSuccess && paths)
    e = mas::pool_alloc(reinterpret_cast<void**>(&d_paths),
                        static_cast<size_t>(batch) * speech_cap * sizeof(int32_t), st[0]);
  if (e == cudaSuccess && durations)
    e = mas::pool_alloc(reinterpret_cast<void**>(&d_dur),
                        static_cast<size_t>(batch) * text_cap * sizeof(int32_t), st[0]);
  cudaEvent_t ready = hs ? hs->ready : nullptr;
  if (e == cudaSuccess) e = cudaEventRecord(ready, st[0]);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st[1], ready, 0);
  if (e != cudaSuccess) rc = cuda_error(err, e, "host path setup");
  for (int c = 0; c < nchunk && rc == MAS_OK; ++c) {
    const int b0 = c * per;
    const int nb = std::min(per, batch - b0);
    if (nb <= 0) break;
    cudaStream_t s = st[c & 1];
    const float* src = values + b0 * o_item;
    if (use_in) {
      // the slot's previous chunk (c - 2) must have left it
      if (c >= 2 && (e = cudaEventSynchronize(in_done[c & 1])) != cudaSuccess) {
        rc = cuda_error(err, e, "host staging");
        break;
      }
      CopyPool::get().copy(pin_in[c & 1], src, static_cast<size_t>(nb) * o_item * sizeof(float));
      src = static_cast<const float*>(pin_in[c & 1]);
    }
    for (int b = 0; b < nb && e == cudaSuccess; ++b)
      e = cudaMemcpy2DAsync(d_q + (b0 + b) * q_item, pitch * 4, src + b * o_item,
                            static_cast<size_t>(speech_cap) * 4,
                            static_cast<size_t>(speech_cap) * 4, text_cap, cudaMemcpyHostToDevice,
                            s);
    if (use_in && e == cudaSuccess) e = cudaEventRecord(in_done[c & 1], s);
    if (e != cudaSuccess) {
      rc = cuda_error(err, e, "host->device staging");
      break;
    }
    rc = enqueue_items(plan, MAS_PART_ALL, b0, nb, d_q, d_out, d_paths, d_dur, s, err);
    if (rc != MAS_OK) break;
    if (out && use_out) {
      // slot c & 1 held chunk c - 2, copied out at iteration c - 1
      if ((e = cudaMemcpyAsync(pin_out[c & 1], d_out + b0 * o_item, nb * o_item,
                               cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
          (e = cudaEventRecord(out_done[c & 1], s)) != cudaSuccess)
        rc = cuda_error(err, e, "device->host out");
    } else if (out &&
               (e = cudaMemcpyAsync(out + b0 * o_item, d_out + b0 * o_item, nb * o_item,
                                    cudaMemcpyDeviceToHost, s)) != cudaSuccess) {
      rc = cuda_error(err, e, "device->host out");
    }
    // the previous chunk's alignment: from its pinned slot to the caller
    if (rc == MAS_OK && use_out && c >= 1) {
      const int pb0 = (c - 1) * per, pnb = std::min(per, batch - pb0);
      if ((e = cudaEventSynchronize(out_done[(c - 1) & 1])) != cudaSuccess)
        rc = cuda_error(err, e, "device->host out");
      else
        CopyPool::get().copy(out + pb0 * o_item, pin_out[(c - 1) & 1], pnb * o_item);
    }

  }
  if (rc == MAS_OK && use_out) {  // the last chunk's alignment
    const int c = (batch + per - 1) / per - 1;
    const int pb0 = c * per, pnb = std::min(per, batch - pb0);
    if ((e = cudaEventSynchronize(out_done[c & 1])) != cudaSuccess)
      rc = cuda_error(err, e, "device->host out");
    else
      CopyPool::get().copy(out + pb0 * o_item, pin_out[c & 1], pnb * o_item);
  }
  // Join the second stream into the first; the NonFinite check and the
  // frees follow on st[0].
  if (st[1] && ready) {
    cudaEventRecord(ready, st[1]);
    cudaStreamWaitEvent(st[0], ready, 0);
  }
  // paths and durations are small: one copy each after the last chunk (a
  // per-chunk copy into pageable memory would serialise the pipeline)
  if (rc == MAS_OK && paths &&
      (e = cudaMemcpyAsync(paths, d_paths, static_cast<size_t>(batch) * speech_cap * sizeof(int32_t),
                           cudaMemcpyDeviceToHost, st[0])) != cudaSuccess)
    rc = cuda_error(err, e, "device->host paths");
  if (rc == MAS_OK && durations &&
      (e = cudaMemcpyAsync(durations, d_dur, static_cast<size_t>(batch) * text_cap * sizeof(int32_t),
                           cudaMemcpyDeviceToHost, st[0])) != cudaSuccess)
    rc = cuda_error(err, e, "device->host durations");
  if (rc == MAS_OK) rc = mas_plan_finish(plan, d_q, st[0], err);
  if (d_q) cudaFreeAsync(d_q, st[0]);
  if (d_out) cudaFreeAsync(d_out, st[0]);
  if (d_paths) cudaFreeAsync(d_paths, st[0]);
  if (d_dur) cudaFreeAsync(d_dur, st[0]);
  if (st[0]) cudaStreamSynchronize(st[0]);
  for (int k = 0; k < 2; ++k) {
    if (in_done[k]) cudaEventDestroy(in_done[k]);
    if (out_done[k]) cudaEventDestroy(out_done[k]);
    PinnedPool::get().give(pin_in[k]);
    PinnedPool::get().give(pin_out[k]);
  }
  mas_plan_destroy(plan);
  return rc;
}

}  // namespace

extern "C" {

int mas_align_host(const float* values, int32_t batch, int32_t text_cap, int32_t speech_cap,
                   const uint32_t* lengths, const mas_config_t* cfg, uint8_t* out, int32_t* paths,
                   mas_error_t* err) {
  return align_host_impl(values, batch, text_cap, speech_cap, lengths, cfg, out, paths, nullptr, 0,
                         err);
}

int mas_align_host_ex(const float* values, int32_t batch, int32_t text_cap, int32_t speech_cap,
                      const uint32_t* lengths, const mas_config_t* cfg, uint8_t* out,
                      int32_t* paths, int32_t* durations, mas_error_t* err) {
  return align_host_impl(values, batch, text_cap, speech_cap, lengths, cfg, out, paths, durations,
                         0, err);
}

int mas_validate_config(const mas_config_t* cfg, mas_error_t* err) {
  clear_error(err);
  mas_config_t c;
  if (cfg)
    c = *cfg;
  else
    mas_config_default(&c);
  c.flags &= ~MAS_FLAG_UNCHECKED;
  return validate_config(c, err);
}

int mas_validate_host(const float* values, int32_t batch, int32_t text_cap, int32_t speech_cap,
                      const uint32_t* lengths, int32_t item_base, mas_error_t* err) {
  mas_config_t c;
  mas_config_default(&c);
  c.flags = MAS_FLAG_UNCHECKED;
  return align_host_impl(values, batch, text_cap, speech_cap, lengths, &c, nullptr, nullptr,
                         nullptr, item_base, err);
}

int mas_generate_device(uint64_t seed, int32_t batch, int32_t text_cap, int32_t speech_cap,
                        int64_t first_item, int64_t row_pitch, float* d_out, void* stream) {
  // s0 = mix_seed(seed, 0) (bench.hpp:87-91, bench.cpp:172)
  uint64_t st = seed ^ (0xd1342543de82ef95ULL * 1ull);
  st += 0x9e3779b97f4a7c15ULL;
  uint64_t z = st;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  const uint64_t s0 = z ^ (z >> 31);
  const int64_t first_elem = first_item * static_cast<int64_t>(text_cap) * speech_cap;
  const cudaError_t e = mas::launch_generate(s0, first_elem, batch, text_cap, speech_cap, row_pitch,
                                             d_out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? MAS_OK : MAS_E_CUDA;
}

}  // extern "C"

extern "C" {

int mas_plan_create_gaussian(int32_t batch, int32_t channels, int32_t text_cap,
                             int32_t speech_cap, const uint32_t* lengths, const mas_config_t* cfg,
                             mas_plan_t** plan_out, mas_error_t* err) {
  clear_error(err);
  if (plan_out) *plan_out = nullptr;
  if (!plan_out) return set_error(err, MAS_E_VALIDATION, -1, -1, "plan_out is null");
  if (channels < 1 || batch < 1 || text_cap < 1 || speech_cap < 1)
    return set_error(err, MAS_E_VALIDATION, MAS_ERRC_ZERO_DIM, -1,
                     "every dimension must be at least 1");
  if (channels > mas::kGaussMaxChannels)
    return set_error(err, MAS_E_UNSUPPORTED, -1, -1,
                     "gaussian log-likelihood: at most " + std::to_string(mas::kGaussMaxChannels) +
                         " channels");
  mas_config_t c;
  if (cfg)
    c = *cfg;
  else
    mas_config_default(&c);
  if ((c.flags & MAS_FLAG_UNCHECKED) && std::isnan(c.max_neg_val) && c.engine == MAS_ENGINE_PARALLEL)
    return set_error(err, MAS_E_UNSUPPORTED, -1, -1,
                     "gaussian plans: NaN sentinels of the parallel engine need the score table "
                     "(use mas_align_gaussian_device)");
  const int kp = mas::gauss_kp(channels);
  uint32_t t_max = 0;
  for (int32_t b = 0; lengths && b < batch; ++b)
    if (lengths[2 * b] <= static_cast<uint32_t>(text_cap)) t_max = std::max(t_max, lengths[2 * b]);
  if (!lengths) t_max = static_cast<uint32_t>(text_cap);
  Geometry probe;
  if (!cached_geometry(batch, std::max<int>(static_cast<int>(t_max), 1), speech_cap, &probe, kp))
    return set_error(err, MAS_E_UNSUPPORTED, -1, -1,
                     "gaussian plans: the text does not fit one cluster of the fused kernel "
                     "(use mas_align_gaussian_device)");
  c.flags &= ~MAS_FLAG_PIPELINED;
  mas_plan_t* p = nullptr;
  int rc = plan_create(batch, text_cap, speech_cap, speech_cap, lengths, &c, 0, &p, err, false, kp);
  if (rc) return rc;
  cudaStream_t st = cudaStreamPerThread;
  cudaError_t e = mas::gauss_alloc(batch, channels, text_cap, speech_cap, st, &p->gauss_own,
                                   &p->gauss_ws);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess &&
      !mas::encode_gauss_b_map(p->gauss_own.B, static_cast<int64_t>(batch) * p->gauss_own.Sp,
                               p->gauss_own.Kp, &p->gauss_tmb,
                               mas::gauss_cfg(p->geo.W, p->gauss_own.Kp).gN))
    e = cudaErrorInvalidValue;
  if (e != cudaSuccess) {
    mas_plan_destroy(p);
    return cuda_error(err, e, "gaussian plan workspace");
  }
  p->channels = channels;
  p->gauss = &p->gauss_own;
  p->gauss_map = &p->gauss_tmb;
  *plan_out = p;
  return MAS_OK;
}

int mas_plan_enqueue_gaussian(mas_plan_t* p, const float* d_z, const float* d_mean,
                              const float* d_logstd, uint8_t* d_out, int32_t* d_paths,
                              int32_t* d_durations, void* stream_v, mas_error_t* err) {
  clear_error(err);
  if (!p || !p->gauss_ws)
    return set_error(err, MAS_E_VALIDATION, -1, -1, "not a gaussian plan (mas_plan_create_gaussian)");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  MAS_CUDA(mas::gauss_prep(d_z, d_mean, d_logstd, p->B, p->channels, p->T, p->S, p->gauss_own,
                           stream),
           "gaussian operands");
  return mas_plan_enqueue_ex(p, MAS_PART_ALL, nullptr, d_out, d_paths, d_durations, stream_v, err);
}

int mas_align_gaussian_device(const float* d_z, const float* d_mean, const float* d_logstd,
                              int32_t batch, int32_t channels, int32_t text_cap,
                              int32_t speech_cap, const uint32_t* lengths, const mas_config_t* cfg,
                              uint8_t* d_out, int32_t* d_paths, int32_t* d_durations,
                              void* stream_v, mas_error_t* err) {
  clear_error(err);
  if (channels < 1)
    return set_error(err, MAS_E_VALIDATION, MAS_ERRC_ZERO_DIM, -1,
                     "every dimension must be at least 1");
  if (channels > mas::kGaussMaxChannels)
    return set_error(err, MAS_E_UNSUPPORTED, -1, -1,
                     "gaussian log-likelihood: at most " + std::to_string(mas::kGaussMaxChannels) +
                         " channels");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  mas_config_t c;
  if (cfg)
    c = *cfg;
  else
    mas_config_default(&c);
  // Texts taller than one cluster of rows (the fused kernel runs one band)
  // and NaN sentinels of the parallel engine (std::max's NaN rule needs the
  // score table, see nan_parallel): q is materialised, still on the device,
  // and aligned by the ordinary path.
  bool fused_ok = true;
  {
    uint32_t t_max = 0;
    for (int32_t b = 0; lengths && b < batch; ++b) t_max = std::max(t_max, lengths[2 * b]);
    if (!lengths) t_max = static_cast<uint32_t>(text_cap);
    Geometry probe;
    fused_ok = batch >= 1 && text_cap >= 1 && speech_cap >= 1 &&
               cached_geometry(batch, std::max<int>(static_cast<int>(t_max), 1), speech_cap, &probe,
                               mas::gauss_kp(channels));
  }
  if (!fused_ok || ((c.flags & MAS_FLAG_UNCHECKED) && std::isnan(c.max_neg_val) &&
                    c.engine == MAS_ENGINE_PARALLEL)) {
    float* q = nullptr;
    if (batch < 1 || text_cap < 1 || speech_cap < 1)
      return set_error(err, MAS_E_VALIDATION, MAS_ERRC_ZERO_DIM, -1,
                       "every dimension must be at least 1");
    const int64_t pitch = (static_cast<int64_t>(speech_cap) + 3) & ~int64_t(3);
    cudaError_t e = mas::pool_alloc(reinterpret_cast<void**>(&q),
                                    static_cast<size_t>(batch) * text_cap * pitch * sizeof(float),
                                    stream);
    int rc = MAS_OK;
    if (e == cudaSuccess)
      rc = mas_gaussian_loglik_device(d_z, d_mean, d_logstd, batch, channels, text_cap,
                                      speech_cap, q, pitch, stream_v, err);
    if (e == cudaSuccess && rc == MAS_OK)
      rc = mas_align_device_ex(q, pitch, batch, text_cap, speech_cap, lengths, &c, d_out, d_paths,
                               d_durations, stream_v, err);
    if (q) cudaFreeAsync(q, stream);
    cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return cuda_error(err, e, "gaussian alignment");
    return rc;
  }
  mas_plan_t* plan = nullptr;
  int rc = mas_plan_create_gaussian(batch, channels, text_cap, speech_cap, lengths, &c, &plan, err);
  if (rc) return rc;
  plan->internal = true;
  rc = mas_plan_enqueue_gaussian(plan, d_z, d_mean, d_logstd, d_out, d_paths, d_durations, stream_v,
                                 err);
  // NonFinite: the compute warps flag items whose q is not finite; only then
  // is q materialised (error path) for the exact row-major location.
  if (rc == MAS_OK) rc = mas_plan_finish(plan, nullptr, stream_v, err);
  cudaStreamSynchronize(stream);
  mas_plan_destroy(plan);
  return rc;
}

}  // extern "C"
