// libfllf C ABI: plan creation, workspace layout, fp64 coefficient math and
// launch sequencing (DESIGN.md "Boundary" and "Data layout in HBM").
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: no-ops unless a tool (nsys) is attached

#include "fllf.h"
#include "fllf_internal.h"

namespace {

thread_local std::string g_last_error;

fllf_status fail(fllf_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

fllf_status cuda_fail(cudaError_t e, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return FLLF_ERR_CUDA;
}

constexpr double kPi = 3.14159265358979323846;

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Scoped switch to the plan's device.
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) {
      ok = false;
      return;
    }
    if (dev >= 0 && dev != prev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

bool is_finite(double v) { return std::isfinite(v); }

}  // namespace

struct fllf_plan_s {
  fllf_plan_desc d{};
  int KL = 0;          // local orders
  int kb = 1;          // first global order
  int device = 0;
  int nlev = 0;
  int Hs[FLLF_MAX_LEVELS]{}, Ws[FLLF_MAX_LEVELS]{};
  // row band (NEXT-1): own rows [bb[l], be[l]) and allocated rows [al[l], ah[l]]
  // (own rows + up to 2 halo rows per side) of every level, global indices
  bool band = false;
  int bb[FLLF_MAX_LEVELS]{}, be[FLLF_MAX_LEVELS]{}, al[FLLF_MAX_LEVELS]{}, ah[FLLF_MAX_LEVELS]{};
  fllf::DevLevel lv[FLLF_MAX_LEVELS]{};
  void* ws = nullptr;
  size_t ws_bytes = 0;
  void* maps_ws = nullptr;
  size_t maps_ws_bytes = 0;
  int maps_slots = 0;                           // map-pyramid slots (fllf_apply_maps: one per map pair)
  long long maps_slot_stride[FLLF_MAX_LEVELS] = {};  // floats between slots, per level
  // fllf_apply_maps, map-batched applies: one D plane per pair and level
  // (mbD_slots planes, fstride_r apart) with their tensor maps; mb_active
  // while its launches are issued (apply_level_impl / apply_impl read it)
  void* mbD_ws = nullptr;
  int mbD_slots = 0;
  float* mbD[FLLF_MAX_LEVELS] = {};
  CUtensorMap tmD_mb[FLLF_MAX_LEVELS];
  bool tmD_mb_ok = false;
  bool mb_active = false;
  int mb_n = 0;  // map pairs of the active batched call
  long long mb_map_fstride = 0;  // floats between the level-0 maps of consecutive pairs
  const char* dbg_out_lo = nullptr;  // debug-bounds builds: the current apply's output range
  const char* dbg_out_hi = nullptr;
  bool built = false;
  const float* img = nullptr;  // the image of the most recent build
  long long img_pitch = 0;     // floats
  float* stage_in = nullptr;
  float* stage_out = nullptr;
  // fllf_enhance_rgb workspace: Y, U, V, Y', sigma map, m map (H x W each, pitch W)
  float* color_ws = nullptr;
  float color_sigma = -1.f;  // sigma value the sigma map currently holds
  int last_launches = 0;
  // profiling: one (start, stop) event pair per launch record
  bool profiling = false;
  bool last_was_apply = false;
  std::vector<cudaEvent_t> ev_start, ev_stop;
  std::vector<int> rec_kind, rec_level;
  int nrec = 0;
  // CUDA graph of the whole filter sequence (build + apply), replayed on the
  // caller's stream; re-captured when the buffers or the profiling flag change
  bool use_graph = true;
  bool use_pdl = true;  // programmatic dependent launch between the kernels of a sequence
  int design = FLLF_DESIGN_AUTO;  // fllf_plan_set_design
  int fused_levels = 0;           // fllf_plan_set_fused_levels (0: by design)
  bool capturing = false;
  cudaStream_t cap_stream = nullptr;
  struct GraphEntry {
    cudaGraphExec_t exec = nullptr;
    const void* in = nullptr;
    const void* out = nullptr;
    size_t in_pitch = 0, out_pitch = 0;
    bool prof = false;
    int launches = 0;
    int nrec = 0;
    unsigned long long used = 0;  // LRU stamp
  };
  static constexpr int kGraphCache = 4;  // buffer pairs (fllf_filter_host_frames alternates two)
  GraphEntry graphs[kGraphCache];
  unsigned long long graph_clock = 0;
  // fllf_filter_host_frames: double-buffered device staging and the copy streams
  static constexpr int kPipe = 2;  // staging slots (double-buffered; 3 measured no faster)
  bool pipe_ready = false;  // every staging buffer, stream and event below exists
  float* pipe_in[kPipe] = {};
  float* pipe_out[kPipe] = {};
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  cudaEvent_t ev_pstart = nullptr, ev_pend = nullptr;
  cudaEvent_t ev_in[kPipe] = {}, ev_done[kPipe] = {}, ev_out[kPipe] = {};
  void* flush_buf = nullptr;  // bench tooling: L2 flush between pipelined frames
  size_t flush_bytes = 0;
  // TMA descriptors of each level's Z planes (k_apply_cl): as the coarse
  // level (box 128 floats x 6 rows) and as the fine level (box 256 x 8)
  bool tm_ok = false;
  CUtensorMap tmc[FLLF_MAX_LEVELS];
  CUtensorMap tmf[FLLF_MAX_LEVELS];
  CUtensorMap tmG[FLLF_MAX_LEVELS];  // G_l planes, box 120 x 8 (tile header g rows)
  CUtensorMap tmD[FLLF_MAX_LEVELS];  // D_l planes, box 68 x 6 (tile header D rows)
  CUtensorMap tmI;                   // the image of the last build (level-0 g rows)
  bool tmI_ok = false;
  const float* tmI_ptr = nullptr;
  long long tmI_pitch = 0;
};

namespace {
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    cudaGetLastError();
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// Z planes of one level as a 3-D fp32 tensor: (2 * zpitch floats) x the
// stored rows lo .. lo + rows - 1 x (batch * KL) planes; box (bx floats, by
// rows, 1 plane).  Row coordinates are relative to row lo.
bool encode_z_map(CUtensorMap* m, const fllf::DevLevel& L, int lo, int rows, int planes, unsigned bx, unsigned by) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  void* base = const_cast<float2*>(L.Z - fllf::ZHALO + (long long)lo * L.zpitch);
  const cuuint64_t dims[3] = {(cuuint64_t)(2 * L.zpitch), (cuuint64_t)rows, (cuuint64_t)planes};
  const cuuint64_t strides[2] = {(cuuint64_t)L.zpitch * 8, (cuuint64_t)L.kstride_z * 8};
  const cuuint32_t box[3] = {bx, by, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// A real fp32 plane stack as a 3-D tensor: W floats x H rows x planes, row
// stride pitch floats, plane stride fstride floats; box (bx, by, 1).
bool encode_real_map(CUtensorMap* m, const float* base, int W, int H, int planes, long long pitch,
                     long long fstride, unsigned bx, unsigned by) {
  auto enc = tensor_map_encoder();
  if (!enc) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((pitch * 4) & 15) || ((fstride * 4) & 15)) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)planes};
  const cuuint64_t strides[2] = {(cuuint64_t)pitch * 4, (cuuint64_t)fstride * 4};
  const cuuint32_t box[3] = {bx, by, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// NVTX range around each kernel launch ("fllf <kind>", payload = level), so
// an nsys trace shows every libfllf launch beside the NCCL / copy activity.
struct NvtxRange {
  NvtxRange(const char* name, int level) {
    nvtxEventAttributes_t a = {};
    a.version = NVTX_VERSION;
    a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    a.messageType = NVTX_MESSAGE_TYPE_ASCII;
    a.message.ascii = name;
    a.payloadType = NVTX_PAYLOAD_TYPE_INT32;
    a.payload.iValue = level;
    nvtxRangePushEx(&a);
  }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

const char* kind_name(int kind) {
  switch (kind) {
    case FLLF_K_BUILD0: return "fllf build0";
    case FLLF_K_BUILD: return "fllf build";
    case FLLF_K_MAPBUILD: return "fllf mapbuild";
    case FLLF_K_APPLY: return "fllf apply";
    case FLLF_K_APPLY0: return "fllf apply0";
    case FLLF_K_FUSE: return "fllf fuse";
    case FLLF_K_COLLAPSE: return "fllf collapse";
  }
  return "fllf";
}

// Bracket one launch with profiling events (no-op when profiling is off) and
// an NVTX range.
struct ProfScope {
  fllf_plan p;
  cudaStream_t s;
  int idx = -1;
  NvtxRange range;
  ProfScope(fllf_plan p_, cudaStream_t s_, int kind, int level) : p(p_), s(s_), range(kind_name(kind), level) {
    if (!p->profiling) return;
    idx = p->nrec++;
    if ((int)p->ev_start.size() <= idx) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      p->ev_start.push_back(a);
      p->ev_stop.push_back(b);
      p->rec_kind.push_back(0);
      p->rec_level.push_back(0);
    }
    p->rec_kind[idx] = kind;
    p->rec_level[idx] = level;
    cudaEventRecordWithFlags(p->ev_start[idx], s, p->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
  }
  ~ProfScope() {
    if (idx >= 0)
      cudaEventRecordWithFlags(p->ev_stop[idx], s, p->capturing ? cudaEventRecordExternal : cudaEventRecordDefault);
  }
};
}  // namespace

extern "C" {

const char* fllf_status_string(fllf_status st) {
  switch (st) {
    case FLLF_OK: return "FLLF_OK";
    case FLLF_ERR_INVALID_ARGUMENT: return "FLLF_ERR_INVALID_ARGUMENT";
    case FLLF_ERR_TOO_MANY_LEVELS: return "FLLF_ERR_TOO_MANY_LEVELS";
    case FLLF_ERR_OUT_OF_MEMORY: return "FLLF_ERR_OUT_OF_MEMORY";
    case FLLF_ERR_CUDA: return "FLLF_ERR_CUDA";
    case FLLF_ERR_NOT_BUILT: return "FLLF_ERR_NOT_BUILT";
    case FLLF_ERR_BAD_POINTER: return "FLLF_ERR_BAD_POINTER";
  }
  return "FLLF_ERR_UNKNOWN";
}

const char* fllf_last_error_message(void) { return g_last_error.c_str(); }

// Eq. 9-11: omega_k = 2 pi k/T, alpha_k = sigma sqrt(2 pi)/T
// exp(-(omega_k sigma)^2/2), a_k = m * 2 sigma^2 alpha_k omega_k.
fllf_status fllf_coefficients(int K, double T, double sigma_r, double m, double* omega_out,
                              double* a_out) {
  if (K < 1 || !(T > 0) || !(sigma_r > 0) || !is_finite(T) || !is_finite(sigma_r) || !is_finite(m))
    return fail(FLLF_ERR_INVALID_ARGUMENT, "fllf_coefficients: need K>=1, T>0, sigma_r>0, finite m");
  if (!omega_out && !a_out) return fail(FLLF_ERR_BAD_POINTER, "fllf_coefficients: no output array");
  for (int k = 1; k <= K; ++k) {
    const double w = 2.0 * kPi * k / T;
    const double alpha = sigma_r * std::sqrt(2.0 * kPi) / T * std::exp(-0.5 * (w * sigma_r) * (w * sigma_r));
    if (omega_out) omega_out[k - 1] = w;
    if (a_out) a_out[k - 1] = m * 2.0 * sigma_r * sigma_r * alpha * w;
  }
  return FLLF_OK;
}

static double period_error(double T, int K, double sigma, double R) {
  return std::erfc(kPi * sigma * (2.0 * K + 1.0) / T) + std::erfc((T - R) / sigma);
}

fllf_status fllf_optimal_period(int K, double sigma_r, double R, double* T_out) {
  if (!T_out) return fail(FLLF_ERR_BAD_POINTER, "fllf_optimal_period: NULL output");
  if (K < 1 || !(sigma_r > 0) || !is_finite(sigma_r) || !(R > 0) || !is_finite(R))
    return fail(FLLF_ERR_INVALID_ARGUMENT, "fllf_optimal_period: need K>=1, sigma_r>0, R>0");
  const double lo = R, hi = R + 12.0 * sigma_r;
  const int n = 4000;
  int best = 0;
  double bv = period_error(lo, K, sigma_r, R);
  for (int i = 1; i <= n; ++i) {
    const double v = period_error(lo + (hi - lo) * i / n, K, sigma_r, R);
    if (v < bv) {
      bv = v;
      best = i;
    }
  }
  double a = lo + (hi - lo) * std::max(best - 1, 0) / n, b = lo + (hi - lo) * std::min(best + 1, n) / n;
  const double phi = (std::sqrt(5.0) - 1.0) / 2.0;
  double c = b - phi * (b - a), d = a + phi * (b - a);
  while (b - a > 1e-6) {
    if (period_error(c, K, sigma_r, R) < period_error(d, K, sigma_r, R)) {
      b = d;
      d = c;
      c = b - phi * (b - a);
    } else {
      a = c;
      c = d;
      d = a + phi * (b - a);
    }
  }
  *T_out = 0.5 * (a + b);
  return FLLF_OK;
}

fllf_status fllf_plan_create(int H, int W, int levels, int K, double T, double sigma_r, double m,
                             fllf_plan* out) {
  fllf_plan_desc d{};
  d.H = H; d.W = W; d.levels = levels; d.K = K; d.T = T; d.sigma_r = sigma_r; d.m = m;
  d.batch = 1; d.k_begin = 0; d.k_end = 0; d.include_base = 1; d.device = -1; d.row_begin = 0; d.row_end = 0;
  return fllf_plan_create_ex(&d, out);
}

fllf_status fllf_plan_create_ex(const fllf_plan_desc* din, fllf_plan* out) {
  if (!din || !out) return fail(FLLF_ERR_BAD_POINTER, "fllf_plan_create: NULL argument");
  *out = nullptr;
  fllf_plan_desc d = *din;
  if (d.H < 1 || d.W < 1) return fail(FLLF_ERR_INVALID_ARGUMENT, "H and W must be >= 1");
  if (d.levels < 2) return fail(FLLF_ERR_INVALID_ARGUMENT, "levels must be >= 2");
  if (d.K < 1 || d.K > FLLF_MAX_K) return fail(FLLF_ERR_INVALID_ARGUMENT, "K must be in 1..32");
  if (!is_finite(d.T) || !(d.T > 0)) return fail(FLLF_ERR_INVALID_ARGUMENT, "T must be finite and > 0");
  if (!is_finite(d.sigma_r) || !(d.sigma_r > 0))
    return fail(FLLF_ERR_INVALID_ARGUMENT, "sigma_r must be finite and > 0");
  if (!is_finite(d.m)) return fail(FLLF_ERR_INVALID_ARGUMENT, "m must be finite");
  if (d.batch < 1) return fail(FLLF_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (d.k_begin == 0 && d.k_end == 0) {
    d.k_begin = 1;
    d.k_end = d.K + 1;
  }
  if (d.k_begin < 1 || d.k_end <= d.k_begin || d.k_end > d.K + 1)
    return fail(FLLF_ERR_INVALID_ARGUMENT, "order range must satisfy 1 <= k_begin < k_end <= K+1");
  if (d.levels > FLLF_MAX_LEVELS) return fail(FLLF_ERR_TOO_MANY_LEVELS, "levels > FLLF_MAX_LEVELS");
  if (d.row_begin == 0 && d.row_end == 0) d.row_end = d.H;
  {
    const int align = 1 << (d.levels - 1);
    if (d.row_begin < 0 || d.row_end <= d.row_begin || d.row_end > d.H)
      return fail(FLLF_ERR_INVALID_ARGUMENT, "row band must satisfy 0 <= row_begin < row_end <= H");
    if (d.row_begin % align || (d.row_end != d.H && d.row_end % align))
      return fail(FLLF_ERR_INVALID_ARGUMENT, "row band boundaries must be multiples of 2^(levels-1) (or H)");
    if ((d.row_begin != 0 || d.row_end != d.H) && d.batch != 1)
      return fail(FLLF_ERR_INVALID_ARGUMENT, "row bands need batch 1");
  }
  int h = d.H, w = d.W;
  for (int l = 1; l < d.levels; ++l) {
    h = (h + 1) / 2;
    w = (w + 1) / 2;
  }
  if (h < 3 || w < 3)
    return fail(FLLF_ERR_TOO_MANY_LEVELS, "coarsest level would be smaller than 3x3 (" + std::to_string(h) +
                                              "x" + std::to_string(w) + ")");

  fllf_plan p = new (std::nothrow) fllf_plan_s();
  if (!p) return fail(FLLF_ERR_OUT_OF_MEMORY, "host allocation failed");
  p->d = d;
  p->KL = d.k_end - d.k_begin;
  p->kb = d.k_begin;
  p->nlev = d.levels;
  {
    const char* ng = std::getenv("FLLF_NO_GRAPH");
    p->use_graph = !(ng && ng[0] == '1');
    const char* np = std::getenv("FLLF_NO_PDL");
    p->use_pdl = !(np && np[0] == '1');
  }
  int dev = d.device;
  if (dev < 0) {
    if (cudaGetDevice(&dev) != cudaSuccess) {
      delete p;
      cudaGetLastError();
      return fail(FLLF_ERR_CUDA, "no CUDA device available (libfllf has no CPU fallback)");
    }
  }
  p->device = dev;
  DeviceGuard guard(dev);
  if (!guard.ok) {
    delete p;
    cudaGetLastError();
    return fail(FLLF_ERR_CUDA, "cannot select CUDA device " + std::to_string(dev));
  }

  p->Hs[0] = d.H;
  p->Ws[0] = d.W;
  for (int l = 1; l < d.levels; ++l) {
    p->Hs[l] = (p->Hs[l - 1] + 1) / 2;
    p->Ws[l] = (p->Ws[l - 1] + 1) / 2;
  }
  p->band = d.row_begin != 0 || d.row_end != d.H;
  for (int l = 0; l < d.levels; ++l) {
    p->bb[l] = d.row_begin >> l;
    p->be[l] = d.row_end == d.H ? p->Hs[l] : d.row_end >> l;
    p->al[l] = std::max(0, p->bb[l] - 2);
    p->ah[l] = std::min(p->Hs[l], p->be[l] + 2) - 1;
  }
  // workspace layout: per level l >= 1: G | D | Z  (each 256-byte aligned)
  const size_t B = (size_t)d.batch;
  size_t off = 0;
  std::vector<size_t> offG(d.levels), offD(d.levels), offZ(d.levels);
  for (int l = 1; l < d.levels; ++l) {
    const size_t pitch = align_up((size_t)p->Ws[l], 32);                              // floats (128 B)
    const size_t zpitch = align_up((size_t)p->Ws[l] + fllf::ZHALO + fllf::ZPAD, 16);  // float2 (128 B)
    fllf::DevLevel& L = p->lv[l];
    L.H = p->Hs[l];
    L.W = p->Ws[l];
    L.pitch = (int)pitch;
    L.zpitch = (int)zpitch;
    const int rows = p->ah[l] - p->al[l] + 1;  // allocated rows (all of them without a band)
    L.fstride_r = (long long)rows * pitch;
    L.kstride_z = (long long)rows * zpitch;
    L.fstride_z = (long long)p->KL * L.kstride_z;
    offG[l] = off;
    off = align_up(off + B * L.fstride_r * sizeof(float), 256);
    offD[l] = off;
    off = align_up(off + B * L.fstride_r * sizeof(float), 256);
    offZ[l] = off;
    off = align_up(off + B * (size_t)L.fstride_z * sizeof(float2), 256);
  }
  p->ws_bytes = off;
  cudaError_t e = cudaMalloc(&p->ws, off);
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete p;
    return e == cudaErrorMemoryAllocation
               ? fail(FLLF_ERR_OUT_OF_MEMORY, "workspace cudaMalloc of " + std::to_string(off) + " bytes failed")
               : cuda_fail(e, "cudaMalloc");
  }
  char* base = static_cast<char*>(p->ws);
  for (int l = 1; l < d.levels; ++l) {
    // plane pointers address GLOBAL row indices: row al[l] is the first allocated row
    fllf::DevLevel& L = p->lv[l];
    L.G = reinterpret_cast<float*>(base + offG[l]) - (long long)p->al[l] * L.pitch;
    L.D = reinterpret_cast<float*>(base + offD[l]) - (long long)p->al[l] * L.pitch;
    L.Z = reinterpret_cast<float2*>(base + offZ[l]) + fllf::ZHALO - (long long)p->al[l] * L.zpitch;
  }
  {
    bool ok = true;
    for (int l = 1; l < d.levels && ok; ++l) {
      const fllf::DevLevel& L = p->lv[l];
      // maps over the stored rows al .. ah only (kernels subtract cr_lo / fr_lo)
      const int lo = p->al[l], rows = p->ah[l] - p->al[l] + 1;
      ok = encode_z_map(&p->tmc[l], L, lo, rows, (int)B * p->KL, 128, 6) &&
           encode_z_map(&p->tmf[l], L, lo, rows, (int)B * p->KL, 256, 8) &&
           encode_real_map(&p->tmG[l], L.G + (long long)lo * L.pitch, L.W, rows, (int)B, L.pitch, L.fstride_r, 120, 8) &&
           encode_real_map(&p->tmD[l], L.D + (long long)lo * L.pitch, L.W, rows, (int)B, L.pitch, L.fstride_r, 68, 6);
    }
    const char* nt = std::getenv("FLLF_NO_TENSOR_TMA");
    p->tm_ok = ok && !(nt && nt[0] == '1');
  }
  // halo / padding cells that no kernel writes must hold finite values
  e = cudaMemset(p->ws, 0, off);
  if (e != cudaSuccess) {
    cudaFree(p->ws);
    delete p;
    return cuda_fail(e, "workspace memset");
  }
  *out = p;
  return FLLF_OK;
}

static void pipe_release(fllf_plan p);

fllf_status fllf_destroy(fllf_plan p) {
  if (!p) return FLLF_OK;
  {
    DeviceGuard guard(p->device);
    cudaDeviceSynchronize();
    if (p->ws) cudaFree(p->ws);
    if (p->maps_ws) cudaFree(p->maps_ws);
    if (p->mbD_ws) cudaFree(p->mbD_ws);
    if (p->stage_in) cudaFree(p->stage_in);
    if (p->color_ws) cudaFree(p->color_ws);
    if (p->stage_out) cudaFree(p->stage_out);
    for (cudaEvent_t e : p->ev_start) cudaEventDestroy(e);
    for (cudaEvent_t e : p->ev_stop) cudaEventDestroy(e);
    for (auto& g : p->graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    pipe_release(p);
    if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
    cudaGetLastError();
  }
  delete p;
  return FLLF_OK;
}

static fllf_status check_image(const void* ptr, size_t pitch_bytes, int W, const char* what,
                               long long* pitch_floats) {
  if (!ptr) return fail(FLLF_ERR_BAD_POINTER, std::string(what) + ": NULL pointer");
  if (pitch_bytes == 0) pitch_bytes = (size_t)W * 4;
  if (pitch_bytes < (size_t)W * 4 || (pitch_bytes & 3))
    return fail(FLLF_ERR_BAD_POINTER, std::string(what) + ": pitch must be >= W*4 and a multiple of 4");
  if (reinterpret_cast<uintptr_t>(ptr) & 3)
    return fail(FLLF_ERR_BAD_POINTER, std::string(what) + ": pointer not 4-byte aligned");
  *pitch_floats = (long long)(pitch_bytes / 4);
  return FLLF_OK;
}

// One build step, level l -> l+1 (l = 0 from the image).  `img` is the
// row-0 (virtual for bands) image pointer, pitch in floats.
static fllf_status build_level_impl(fllf_plan p, const float* img, long long pitch, int l, cudaStream_t stream,
                                    bool pdl) {
  fllf::BuildParams bp{};
  bp.img.p = img;
  bp.img.H = p->d.H;
  bp.img.W = p->d.W;
  bp.img.pitch = pitch;
  bp.img.fstride = pitch * p->d.H;
  if (l > 0) bp.src = p->lv[l];
  bp.dst = p->lv[l + 1];
  bp.Hf = p->Hs[l];
  bp.Wf = p->Ws[l];
  bp.Hc = p->Hs[l + 1];
  bp.Wc = p->Ws[l + 1];
  bp.KL = p->KL;
  bp.kbase = p->kb;
  bp.maps = 0;
  bp.invT = (float)(1.0 / p->d.T);
  bp.o_begin = p->bb[l + 1];
  bp.o_end = p->be[l + 1];
  bp.fr_lo = p->al[l];
  bp.fr_hi = p->ah[l];
  bp.dbg_lo = static_cast<const char*>(p->ws);
  bp.dbg_hi = bp.dbg_lo + p->ws_bytes;
  cudaError_t e;
  {
    ProfScope ps(p, stream, l == 0 ? FLLF_K_BUILD0 : FLLF_K_BUILD, l);
    e = fllf::launch_build(bp, l, p->d.batch, stream, pdl);
  }
  return e == cudaSuccess ? FLLF_OK : cuda_fail(e, "build kernel launch");
}

fllf_status fllf_build_fourier_pyramids(fllf_plan p, const float* d_img, size_t pitch_bytes, void* s) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  if (p->band)
    return fail(FLLF_ERR_INVALID_ARGUMENT,
                "build_fourier_pyramids: row-band plans need the per-level calls (halo exchange between levels)");
  long long pitch;
  fllf_status st = check_image(d_img, pitch_bytes, p->d.W, "build: d_img", &pitch);
  if (st != FLLF_OK) return st;
  DeviceGuard guard(p->device);
  cudaStream_t stream = static_cast<cudaStream_t>(s);
  const float* img = d_img - (long long)p->d.row_begin * pitch;  // global row 0 (bands: virtual)
  int launches = 0;
  p->nrec = 0;
  p->last_was_apply = false;
  for (int l = 0; l + 1 < p->nlev; ++l) {
    st = build_level_impl(p, img, pitch, l, stream, p->use_pdl && l > 0 && !p->band);
    if (st != FLLF_OK) return st;
    ++launches;
  }
  p->built = true;
  p->img = img;
  p->img_pitch = pitch;
  p->last_launches = launches;
  return FLLF_OK;
}

fllf_status fllf_build_level(fllf_plan p, const float* d_img, size_t pitch_bytes, int level, void* s) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  if (level < 0 || level + 1 >= p->nlev) return fail(FLLF_ERR_INVALID_ARGUMENT, "build_level: level out of range");
  long long pitch;
  fllf_status st = check_image(d_img, pitch_bytes, p->d.W, "build_level: d_img", &pitch);
  if (st != FLLF_OK) return st;
  DeviceGuard guard(p->device);
  const float* img = d_img - (long long)p->d.row_begin * pitch;
  if (level == 0) p->nrec = 0;
  p->last_was_apply = false;
  st = build_level_impl(p, img, pitch, level, static_cast<cudaStream_t>(s), false);
  if (st != FLLF_OK) return st;
  p->img = img;
  p->img_pitch = pitch;
  p->last_launches = 1;
  if (level + 2 == p->nlev) p->built = true;
  return FLLF_OK;
}

// Map-pyramid workspace with `slots` slots per level (slot j: G_l[sigma_j],
// then G_l[m_j]); lv[l].MS / MM point at slot 0.
static fllf_status ensure_maps_ws(fllf_plan p, int slots = 1) {
  if (p->maps_ws && p->maps_slots >= slots) return FLLF_OK;
  if (p->maps_ws) {
    cudaError_t e = cudaFree(p->maps_ws);  // (callers are stream-ordered before the next kernels)
    if (e != cudaSuccess) return cuda_fail(e, "map pyramid cudaFree");
    p->maps_ws = nullptr;
    p->maps_slots = 0;
  }
  size_t off = 0;
  std::vector<size_t> offs(p->nlev);
  for (int l = 1; l < p->nlev; ++l) {
    offs[l] = off;
    p->maps_slot_stride[l] = 2 * p->lv[l].fstride_r;
    off = align_up(off + (size_t)slots * 2 * (size_t)p->lv[l].fstride_r * sizeof(float), 256);
  }
  cudaError_t e = cudaMalloc(&p->maps_ws, off);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(FLLF_ERR_OUT_OF_MEMORY, "map pyramid cudaMalloc failed");
  }
  p->maps_ws_bytes = off;
  p->maps_slots = slots;
  char* base = static_cast<char*>(p->maps_ws);
  for (int l = 1; l < p->nlev; ++l) {
    p->lv[l].MS = reinterpret_cast<float*>(base + offs[l]);
    p->lv[l].MM = p->lv[l].MS + p->lv[l].fstride_r;
  }
  return FLLF_OK;
}

// Clenshaw coefficient pairs of one order with coefficient a: the polyphase
// up-sampling scales 1/64 (even row, even col), 1/16 (mixed), 1/4 (odd, odd)
// and the same-level term, with the sign pattern of
// Im(e^{-i k theta} V) = cos(k theta) V_im - sin(k theta) V_re folded in
// (fllf::ApplyParams::cw).
static void clenshaw_pairs(float a, float2 (&cw)[4]) {
  cw[0] = make_float2(-a / 64.f, a / 64.f);
  cw[1] = make_float2(-a / 16.f, a / 16.f);
  cw[2] = make_float2(-a / 4.f, a / 4.f);
  cw[3] = make_float2(a, -a);
}

// One apply level (coarse to fine; l = lmax-1 .. 0) with the prepared parameters.
static fllf_status apply_level_impl(fllf_plan p, fllf::ApplyParams& ap, int l, bool maps, cudaStream_t stream,
                                    bool pdl) {
  const int lmax = p->nlev - 1;
  if (l > 0) ap.fine = p->lv[l];
  ap.coarse = p->lv[l + 1];
  ap.use_tm = p->tm_ok ? 1 : 0;
  ap.use_tm_g = ap.use_tm_d = 0;
  ap.ms_fstride = p->mb_active && l > 0 ? p->maps_slot_stride[l] : 0;
  if (p->tm_ok) {
    ap.tm_coarse = p->tmc[l + 1];
    ap.tm_d = p->mb_active ? p->tmD_mb[l + 1] : p->tmD[l + 1];
    ap.use_tm_d = (!p->mb_active || p->tmD_mb_ok) ? 1 : 0;
    if (l > 0) {
      ap.tm_fine = p->tmf[l];
      ap.tm_g = p->tmG[l];
      ap.use_tm_g = 1;
    } else {
      if (p->tmI_ptr != p->img || p->tmI_pitch != p->img_pitch) {
        // the rows the plan reads (al[0] .. ah[0]; a band's caller may hold only those)
        p->tmI_ok = encode_real_map(&p->tmI, p->img + (long long)p->al[0] * p->img_pitch, p->d.W,
                                    p->ah[0] - p->al[0] + 1, p->d.batch, p->img_pitch, p->img_pitch * p->d.H, 120, 8);
        p->tmI_ptr = p->img;
        p->tmI_pitch = p->img_pitch;
      }
      if (p->tmI_ok) {
        ap.tm_g = p->tmI;
        ap.use_tm_g = 1;
      }
    }
  }
  ap.Hf = p->Hs[l];
  ap.Wf = p->Ws[l];
  ap.Hc = p->Hs[l + 1];
  ap.Wc = p->Ws[l + 1];
  ap.r_begin = p->bb[l + 1];
  ap.r_end = p->be[l + 1];
  ap.cr_lo = p->al[l + 1];
  ap.cr_hi = p->ah[l + 1];
  ap.fr_lo = p->al[l];
  ap.fr_hi = p->ah[l];
  const bool has_d = (l + 1) < lmax;  // D_lmax = 0
  ap.wait_first = (l == lmax - 1 || !pdl) ? 1 : 0;
  if (l == 0) {
    ap.dbg_lo = p->dbg_out_lo;
    ap.dbg_hi = p->dbg_out_hi;
  } else {
    ap.dbg_lo = static_cast<const char*>(p->ws);
    ap.dbg_hi = ap.dbg_lo + p->ws_bytes;
  }
  static const bool dbg_selftest = [] {  // debug-bounds builds: an empty range must trap
    const char* e = std::getenv("FLLF_DEBUG_BOUNDS_SELFTEST");
    return e && e[0] == '1';
  }();
  if (dbg_selftest) ap.dbg_hi = ap.dbg_lo;
  cudaError_t e;
  {
    ProfScope ps(p, stream, l == 0 ? FLLF_K_APPLY0 : FLLF_K_APPLY, l);
    e = fllf::launch_apply(ap, l, has_d, maps, p->mb_active ? p->mb_n : p->d.batch, stream, pdl);
  }
  return e == cudaSuccess ? FLLF_OK : cuda_fail(e, "apply kernel launch");
}

// Apply levels hi down to lo (coarse to fine): fllf_apply (lo = 0, hi = l_max-1),
// fllf_apply_level (lo = hi = level) and design F's AB levels / level 0
// (chain_pdl: PDL-linked to the launches before it).
// maps_prebuilt: MAPS with the map pyramids already in lv[l].MS / MM
// (fllf_apply_maps builds those of all its map pairs in one launch per level).
static fllf_status apply_impl(fllf_plan p, const fllf_apply_args* a, float* d_out, size_t out_pitch_bytes, void* s,
                              int lo, int hi, bool accumulate = false, bool chain_pdl = false,
                              bool maps_prebuilt = false) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  if (!p->built) return fail(FLLF_ERR_NOT_BUILT, "fllf_apply before fllf_build_fourier_pyramids");
  long long opitch;
  fllf_status st = check_image(d_out, out_pitch_bytes, p->d.W, "apply: d_out", &opitch);
  if (st != FLLF_OK) return st;
  const int mode = a ? a->mode : FLLF_SCALAR;
  if (mode != FLLF_SCALAR && mode != FLLF_COEFFS && mode != FLLF_MAPS)
    return fail(FLLF_ERR_INVALID_ARGUMENT, "apply: unknown mode");
  if (mode == FLLF_MAPS && p->band) return fail(FLLF_ERR_INVALID_ARGUMENT, "apply(MAPS) is not supported on row bands");
  const bool partial = !(lo == 0 && hi == p->nlev - 2);
  if (partial && mode == FLLF_MAPS) return fail(FLLF_ERR_INVALID_ARGUMENT, "apply_level: MAPS not supported");
  if (lo < 0 || hi >= p->nlev - 1 || lo > hi) return fail(FLLF_ERR_INVALID_ARGUMENT, "apply_level: level out of range");
  DeviceGuard guard(p->device);
  cudaStream_t stream = static_cast<cudaStream_t>(s);
  const double T = p->d.T;
  const double w1 = 2.0 * kPi / T;

  fllf::ApplyParams ap{};
  ap.gz = ap.zz = p->mb_active ? 0 : 1;  // map-batched: tiles of pair j share G, I and Z
  ap.img.p = p->img;
  ap.img.H = p->d.H;
  ap.img.W = p->d.W;
  ap.img.pitch = p->img_pitch;
  ap.img.fstride = p->img_pitch * p->d.H;
  ap.out = d_out - (long long)p->d.row_begin * opitch;  // global row 0 (bands: virtual)
  ap.accumulate = accumulate ? 1 : 0;
  // debug-bounds builds: level 0 writes the caller's rows, levels >= 1 the workspace
  p->dbg_out_lo = reinterpret_cast<const char*>(d_out);
  p->dbg_out_hi = p->dbg_out_lo + ((size_t)((p->mb_active ? p->mb_n : p->d.batch) - 1) * p->d.H +
                                     (p->d.row_end - p->d.row_begin)) * (size_t)opitch * sizeof(float);
  ap.out_pitch = opitch;
  ap.out_fstride = opitch * p->d.H;
  ap.KL = p->KL;
  ap.kbase = p->kb;
  ap.include_base = p->d.include_base;
  ap.invT = (float)(1.0 / T);
  ap.c0 = (float)(2.0 * w1 * std::sqrt(2.0 * kPi) / T);
  ap.hq = (float)(0.5 * w1 * w1);

  if (mode == FLLF_SCALAR || mode == FLLF_COEFFS) {
    std::vector<double> om(p->d.K), ak(p->d.K);
    if (mode == FLLF_SCALAR) {
      fllf_coefficients(p->d.K, T, p->d.sigma_r, p->d.m, om.data(), ak.data());
      for (int i = 0; i < p->KL; ++i) ap.a[i] = (float)ak[p->kb - 1 + i];
    } else {
      if (!a->a_k) return fail(FLLF_ERR_BAD_POINTER, "apply(COEFFS): a_k is NULL");
      for (int i = 0; i < p->KL; ++i) {
        if (!is_finite(a->a_k[i])) return fail(FLLF_ERR_INVALID_ARGUMENT, "apply(COEFFS): non-finite a_k");
        ap.a[i] = (float)a->a_k[i];
      }
    }
  }
  for (int i = 0; i < p->KL; ++i) {
    // MAPS (Clenshaw kernel): the per-pixel a_k(q) = [m sigma^3 c0 exp(...)](q) * k, the k here
    const float a = mode == FLLF_MAPS ? (float)(p->kb + i) : ap.a[i];
    ap.wk[i][0] = make_float2(ap.a[i], ap.a[i]);
    ap.wk[i][1] = make_float2(-ap.a[i] / 64.f, -ap.a[i] / 64.f);
    ap.wk[i][2] = make_float2(-ap.a[i] / 16.f, -ap.a[i] / 16.f);
    ap.wk[i][3] = make_float2(-ap.a[i] / 4.f, -ap.a[i] / 4.f);
    clenshaw_pairs(a, ap.cw[i]);
    // MAPS (k_apply_cl): (k^2, log2 k) of the global order k
    if (mode == FLLF_MAPS) ap.cw[i][0] = make_float2(a * a, (float)std::log2((double)(p->kb + i)));
  }
  int launches = 0;
  if (p->last_was_apply) p->nrec = 0;
  p->last_was_apply = true;
  const bool maps = mode == FLLF_MAPS;
  if (maps) {
    long long mp1, mp2;
    st = check_image(a->d_sigma_r, a->map_pitch_bytes, p->d.W, "apply(MAPS): d_sigma_r", &mp1);
    if (st != FLLF_OK) return st;
    st = check_image(a->d_m, a->map_pitch_bytes, p->d.W, "apply(MAPS): d_m", &mp2);
    if (st != FLLF_OK) return st;
    if (!maps_prebuilt) st = ensure_maps_ws(p);
    if (st != FLLF_OK) return st;
    ap.smap.p = a->d_sigma_r;
    ap.smap.pitch = mp1;
    ap.mmap.p = a->d_m;
    ap.mmap.pitch = mp2;
    ap.smap.fstride = ap.mmap.fstride = p->mb_active ? p->mb_map_fstride : 0;
    // Gaussian pyramids of the two maps, levels 1 .. l_max-1 (reading R7)
    for (int l = 0; l + 2 < p->nlev && !maps_prebuilt; ++l) {
      fllf::BuildParams bp{};
      bp.img.p = a->d_sigma_r;
      bp.img.pitch = mp1;
      bp.img.fstride = 0;
      bp.img2.p = a->d_m;
      bp.img2.pitch = mp2;
      bp.img2.fstride = 0;
      if (l > 0) bp.src = p->lv[l];
      bp.dst = p->lv[l + 1];
      bp.Hf = p->Hs[l];
      bp.Wf = p->Ws[l];
      bp.Hc = p->Hs[l + 1];
      bp.Wc = p->Ws[l + 1];
      bp.KL = 0;
      bp.kbase = p->kb;
      bp.maps = 1;
      bp.o_begin = 0;
      bp.o_end = p->Hs[l + 1];
      bp.fr_lo = 0;
      bp.fr_hi = p->Hs[l] - 1;
      bp.invT = (float)(1.0 / T);
      bp.dbg_lo = static_cast<const char*>(p->maps_ws);  // the map pyramids
      bp.dbg_hi = bp.dbg_lo + p->maps_ws_bytes;
      cudaError_t e;
      {
        ProfScope ps(p, stream, FLLF_K_MAPBUILD, l);
        e = fllf::launch_build(bp, l, 1, stream, false);
      }
      if (e != cudaSuccess) return cuda_fail(e, "map pyramid kernel launch");
      ++launches;
    }
  }
  const int lmax = p->nlev - 1;
  for (int l = hi; l >= lo; --l) {
    st = apply_level_impl(p, ap, l, maps, stream, p->use_pdl && !p->band && (!partial || chain_pdl));
    if (st != FLLF_OK) return st;
    ++launches;
  }
  p->last_launches = launches;
  return FLLF_OK;
}

fllf_status fllf_apply(fllf_plan p, const fllf_apply_args* a, float* d_out, size_t out_pitch_bytes, void* s) {
  if (p && p->band)
    return fail(FLLF_ERR_INVALID_ARGUMENT,
                "apply: row-band plans need the per-level calls (halo exchange between levels)");
  return apply_impl(p, a, d_out, out_pitch_bytes, s, 0, p ? p->nlev - 2 : 0);
}

fllf_status fllf_apply_maps(fllf_plan p, int n, const float* d_sigma_r, const float* d_m, size_t map_pitch_bytes,
                            size_t map_stride_bytes, float* d_out, size_t out_pitch_bytes, size_t out_stride_bytes,
                            void* s) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  if (p->band) return fail(FLLF_ERR_INVALID_ARGUMENT, "apply_maps: not for row-band plans");
  if (!p->built) return fail(FLLF_ERR_NOT_BUILT, "apply_maps before fllf_build_fourier_pyramids");
  if (n < 1) return fail(FLLF_ERR_INVALID_ARGUMENT, "apply_maps: n >= 1");
  if (!d_sigma_r || !d_m || !d_out) return fail(FLLF_ERR_BAD_POINTER, "apply_maps: NULL pointer");
  const size_t mpitch = map_pitch_bytes ? map_pitch_bytes : (size_t)p->d.W * sizeof(float);
  const size_t opitch = out_pitch_bytes ? out_pitch_bytes : (size_t)p->d.W * sizeof(float);
  const size_t mstride = map_stride_bytes ? map_stride_bytes : mpitch * p->d.H;
  const size_t ostride = out_stride_bytes ? out_stride_bytes : opitch * p->d.H * p->d.batch;
  if ((mstride & 15) || mstride < mpitch * p->d.H)
    return fail(FLLF_ERR_INVALID_ARGUMENT, "apply_maps: map stride not a multiple of 16 bytes or below one map");
  if ((ostride & 3) || ostride < opitch * p->d.H * p->d.batch)
    return fail(FLLF_ERR_INVALID_ARGUMENT, "apply_maps: output stride below one output");
  long long mp1, mp2;
  fllf_status st = check_image(d_sigma_r, mpitch, p->d.W, "apply_maps: d_sigma_r", &mp1);
  if (st != FLLF_OK) return st;
  st = check_image(d_m, mpitch, p->d.W, "apply_maps: d_m", &mp2);
  if (st != FLLF_OK) return st;
  DeviceGuard guard(p->device);
  cudaStream_t stream = static_cast<cudaStream_t>(s);
  st = ensure_maps_ws(p, n);
  if (st != FLLF_OK) return st;
  p->nrec = 0;  // profiling records of this call: the map builds, then every pair's applies
  // the map pyramids of all n pairs, one launch per level (blockIdx.z = pair)
  int launches = 0;
  for (int l = 0; l + 2 < p->nlev; ++l) {
    fllf::BuildParams bp{};
    bp.img.p = d_sigma_r;
    bp.img.pitch = mp1;
    bp.img.fstride = (long long)(mstride / sizeof(float));
    bp.img2.p = d_m;
    bp.img2.pitch = mp2;
    bp.img2.fstride = (long long)(mstride / sizeof(float));
    if (l > 0) bp.src = p->lv[l];
    bp.dst = p->lv[l + 1];
    bp.ms_stride_src = l > 0 ? p->maps_slot_stride[l] : 0;
    bp.ms_stride_dst = p->maps_slot_stride[l + 1];
    bp.Hf = p->Hs[l];
    bp.Wf = p->Ws[l];
    bp.Hc = p->Hs[l + 1];
    bp.Wc = p->Ws[l + 1];
    bp.KL = 0;
    bp.kbase = p->kb;
    bp.maps = 1;
    bp.o_begin = 0;
    bp.o_end = p->Hs[l + 1];
    bp.fr_lo = 0;
    bp.fr_hi = p->Hs[l] - 1;
    bp.invT = (float)(1.0 / p->d.T);
    bp.dbg_lo = static_cast<const char*>(p->maps_ws);
    bp.dbg_hi = bp.dbg_lo + p->maps_ws_bytes;
    cudaError_t e;
    {
      ProfScope ps(p, stream, FLLF_K_MAPBUILD, l);
      e = fllf::launch_build(bp, l, n, stream, false);
    }
    if (e != cudaSuccess) return cuda_fail(e, "map pyramid kernel launch");
    ++launches;
  }
  // map-batched applies: one launch per level for all n pairs (tile frame
  // index = pair; G, I and Z shared, D / map planes / output per pair) --
  // single-frame plans, 16-byte aligned map rows (the TMA-staged MAPS path)
  const bool aligned = ((reinterpret_cast<uintptr_t>(d_sigma_r) | reinterpret_cast<uintptr_t>(d_m)) & 15) == 0 &&
                       (mp1 & 3) == 0 && mp1 == mp2 && (p->d.W & 3) == 0 && ((mstride / 4) & 3) == 0;
  static const bool mb_off = [] {  // FLLF_APPLY_MAPS_PER_PAIR=1: applies pair by pair (A/B)
    const char* e = std::getenv("FLLF_APPLY_MAPS_PER_PAIR");
    return e && e[0] == '1';
  }();
  if (!mb_off && p->d.batch == 1 && aligned && ostride == opitch * p->d.H) {
    if (p->mbD_slots < n) {  // per-pair D planes of every level >= 1
      if (p->mbD_ws) cudaFree(p->mbD_ws);
      p->mbD_ws = nullptr;
      p->mbD_slots = 0;
      // guard bands: the tile-header copies of D rows start 4 columns left of
      // a row and may run past its end (as inside the plan's workspace)
      size_t off = 256;
      std::vector<size_t> offs(p->nlev);
      for (int l = 1; l < p->nlev; ++l) {
        offs[l] = off;
        off = align_up(off + (size_t)n * p->lv[l].fstride_r * sizeof(float) + 256, 256);
      }
      off += 4096;
      cudaError_t e = cudaMalloc(&p->mbD_ws, off);
      if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(FLLF_ERR_OUT_OF_MEMORY, "apply_maps: D planes cudaMalloc failed");
      }
      e = cudaMemset(p->mbD_ws, 0, off);
      if (e != cudaSuccess) return cuda_fail(e, "apply_maps: D planes memset");
      p->mbD_slots = n;
      bool ok = p->tm_ok;
      for (int l = 1; l < p->nlev; ++l) {
        p->mbD[l] = reinterpret_cast<float*>(static_cast<char*>(p->mbD_ws) + offs[l]);
        if (ok)
          ok = encode_real_map(&p->tmD_mb[l], p->mbD[l], p->lv[l].W, p->lv[l].H, n, p->lv[l].pitch,
                               p->lv[l].fstride_r, 68, 6);
      }
      p->tmD_mb_ok = ok;
    }
    fllf::DevLevel saved[FLLF_MAX_LEVELS];
    for (int l = 1; l < p->nlev; ++l) {
      saved[l] = p->lv[l];
      p->lv[l].D = p->mbD[l];
    }
    p->mb_active = true;
    p->mb_n = n;
    p->mb_map_fstride = (long long)(mstride / sizeof(float));
    fllf_apply_args a{};
    a.mode = FLLF_MAPS;
    a.d_sigma_r = d_sigma_r;
    a.d_m = d_m;
    a.map_pitch_bytes = mpitch;
    p->last_was_apply = false;
    st = apply_impl(p, &a, d_out, opitch, s, 0, p->nlev - 2, false, false, true);
    launches += p->last_launches;
    p->mb_active = false;
    p->mb_n = 0;
    p->mb_map_fstride = 0;
    for (int l = 1; l < p->nlev; ++l) p->lv[l] = saved[l];
    p->last_launches = launches;
    return st;
  }
  // the applies, pair by pair, each reading its slot of the map pyramids
  fllf::DevLevel saved[FLLF_MAX_LEVELS];
  for (int l = 1; l < p->nlev; ++l) saved[l] = p->lv[l];
  for (int j = 0; j < n && st == FLLF_OK; ++j) {
    for (int l = 1; l < p->nlev; ++l) {
      p->lv[l].MS = saved[l].MS + j * p->maps_slot_stride[l];
      p->lv[l].MM = saved[l].MM + j * p->maps_slot_stride[l];
    }
    fllf_apply_args a{};
    a.mode = FLLF_MAPS;
    a.d_sigma_r = reinterpret_cast<const float*>(reinterpret_cast<const char*>(d_sigma_r) + j * mstride);
    a.d_m = reinterpret_cast<const float*>(reinterpret_cast<const char*>(d_m) + j * mstride);
    a.map_pitch_bytes = mpitch;
    float* out = reinterpret_cast<float*>(reinterpret_cast<char*>(d_out) + j * ostride);
    p->last_was_apply = false;  // keep the records of the launches before
    st = apply_impl(p, &a, out, opitch, s, 0, p->nlev - 2, false, false, true);
    launches += p->last_launches;
  }
  for (int l = 1; l < p->nlev; ++l) p->lv[l] = saved[l];
  p->last_launches = launches;
  return st;
}

fllf_status fllf_apply_accumulate(fllf_plan p, const fllf_apply_args* a, float* d_out, size_t out_pitch_bytes,
                                  void* s) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  if (a && a->mode == FLLF_MAPS) return fail(FLLF_ERR_INVALID_ARGUMENT, "apply_accumulate: SCALAR / COEFFS only");
  if (p->band) return fail(FLLF_ERR_INVALID_ARGUMENT, "apply_accumulate: not for row-band plans");
  return apply_impl(p, a, d_out, out_pitch_bytes, s, 0, p->nlev - 2, true);
}

fllf_status fllf_ipc_alloc(size_t bytes, void** d_ptr, void* handle_out) {
  if (!d_ptr || !handle_out || bytes == 0) return fail(FLLF_ERR_BAD_POINTER, "ipc_alloc: NULL argument or 0 bytes");
  *d_ptr = nullptr;
  cudaError_t e = cudaMalloc(d_ptr, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(FLLF_ERR_OUT_OF_MEMORY, "ipc_alloc: cudaMalloc failed");
  }
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, *d_ptr);
  if (e != cudaSuccess) {
    cudaFree(*d_ptr);
    *d_ptr = nullptr;
    return cuda_fail(e, "cudaIpcGetMemHandle");
  }
  std::memcpy(handle_out, &h, sizeof(h));
  return FLLF_OK;
}

fllf_status fllf_ipc_free(void* d_ptr) {
  if (!d_ptr) return FLLF_OK;
  cudaError_t e = cudaFree(d_ptr);
  return e == cudaSuccess ? FLLF_OK : cuda_fail(e, "ipc_free: cudaFree");
}

fllf_status fllf_ipc_open(const void* handle, void** d_ptr) {
  if (!handle || !d_ptr) return fail(FLLF_ERR_BAD_POINTER, "ipc_open: NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  *d_ptr = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? FLLF_OK : cuda_fail(e, "cudaIpcOpenMemHandle");
}

fllf_status fllf_ipc_close(void* d_ptr) {
  if (!d_ptr) return FLLF_OK;
  cudaError_t e = cudaIpcCloseMemHandle(d_ptr);
  return e == cudaSuccess ? FLLF_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

fllf_status fllf_apply_level(fllf_plan p, const fllf_apply_args* a, float* d_out, size_t out_pitch_bytes, int level,
                             void* s) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  if (level < 0 || level >= p->nlev - 1) return fail(FLLF_ERR_INVALID_ARGUMENT, "apply_level: level out of range");
  return apply_impl(p, a, d_out, out_pitch_bytes, s, level, level);
}

fllf_status fllf_plan_band_plane(fllf_plan p, int level, int kind, void** d_ptr, size_t* pitch_bytes, int* first_row,
                                 int* rows, int* planes, size_t* plane_stride_bytes) {
  if (!p || !d_ptr || !pitch_bytes || !first_row || !rows || !planes || !plane_stride_bytes)
    return fail(FLLF_ERR_BAD_POINTER, "band_plane: NULL argument");
  if (level < 1 || level >= p->nlev || kind < 0 || kind > 2)
    return fail(FLLF_ERR_INVALID_ARGUMENT, "band_plane: level 1..levels-1, kind 0 (G), 1 (Z), 2 (D)");
  const fllf::DevLevel& L = p->lv[level];
  const int lo = p->al[level];
  *first_row = lo;
  *rows = p->ah[level] - lo + 1;
  if (kind == 1) {
    *d_ptr = const_cast<float2*>(L.Z - fllf::ZHALO + (long long)lo * L.zpitch);
    *pitch_bytes = (size_t)L.zpitch * sizeof(float2);
    *planes = p->KL * p->d.batch;
    *plane_stride_bytes = (size_t)L.kstride_z * sizeof(float2);
  } else {
    const float* b = kind == 0 ? L.G : L.D;
    *d_ptr = const_cast<float*>(b + (long long)lo * L.pitch);
    *pitch_bytes = (size_t)L.pitch * sizeof(float);
    *planes = p->d.batch;
    *plane_stride_bytes = (size_t)L.fstride_r * sizeof(float);
  }
  return FLLF_OK;
}

// Design F is used for the levels l >= 1 whose pixel count over the batch is
// at least FLLF_FUSE_MIN_MP megapixels (default 4): from the finest level up to
// the first smaller one ("fused levels" 1 .. LF-1); the coarser levels, where
// a fused launch is latency-bound, keep design AB (build + apply).  Full-frame
// plans with levels >= 3 whose order count has a supported per-warp split;
// FLLF_NO_FUSE=1 disables it.  Returns LF (1 = design AB everywhere).
static int fuse_levels(fllf_plan p) {
  static const bool off = [] {
    const char* e = std::getenv("FLLF_NO_FUSE");
    return e && e[0] == '1';
  }();
  static const double min_mp = [] {
    const char* e = std::getenv("FLLF_FUSE_MIN_MP");
    return e ? std::atof(e) : 4.0;
  }();
  if (off || p->design == FLLF_DESIGN_AB || p->band || p->nlev < 3 || fllf::fuse_orders_per_warp(p->KL) <= 0)
    return 1;
  const int lmax = p->nlev - 1;
  if (p->fused_levels > 0) return std::min(p->fused_levels + 1, lmax);
  if (p->design == FLLF_DESIGN_F) return lmax;
  int lf = 1;
  while (lf < lmax && (double)p->d.batch * p->Hs[lf] * p->Ws[lf] >= min_mp * 1e6) ++lf;
  return lf;
}

// Design F, fused levels 1 .. LF-1: build0; for
// l = 1 .. LF-1 the fused build step l -> l+1 + level-l order sum S_l (into
// D_l); design AB for the coarser levels (build steps LF .. l_max-1, applies
// l_max-1 .. LF, which leave the final D_LF); the collapse D_l += up(D_{l+1})
// for l = min(LF, l_max-1)-1 .. 1 (D_{l_max-1} = S_{l_max-1} needs none); the
// level-0 apply (reads D_1).  All launches after the first are PDL-chained;
// each kernel waits for its predecessor before it triggers the next one, so
// when a kernel starts every kernel two or more places earlier has completed
// (the level-0 apply may stage Z_1 before its own wait).
static fllf_status filter_fused(fllf_plan p, const float* d_img, size_t in_pitch_bytes, float* d_out,
                                size_t out_pitch_bytes, void* s, int LF) {
  long long pitch;
  fllf_status st = check_image(d_img, in_pitch_bytes, p->d.W, "filter: d_img", &pitch);
  if (st != FLLF_OK) return st;
  long long opitch;
  st = check_image(d_out, out_pitch_bytes, p->d.W, "filter: d_out", &opitch);
  if (st != FLLF_OK) return st;
  DeviceGuard guard(p->device);
  cudaStream_t stream = static_cast<cudaStream_t>(s);
  const int lmax = p->nlev - 1;
  const bool pdl = p->use_pdl;
  p->nrec = 0;
  p->last_was_apply = false;
  int launches = 0;
  st = build_level_impl(p, d_img, pitch, 0, stream, false);
  if (st != FLLF_OK) return st;
  ++launches;
  fllf::FuseParams fp{};
  {
    std::vector<double> om(p->d.K), ak(p->d.K);
    fllf_coefficients(p->d.K, p->d.T, p->d.sigma_r, p->d.m, om.data(), ak.data());
    for (int i = 0; i < p->KL; ++i) clenshaw_pairs((float)ak[p->kb - 1 + i], fp.cw[i]);
  }
  fp.KL = p->KL;
  fp.kbase = p->kb;
  fp.invT = (float)(1.0 / p->d.T);
  fp.dbg_lo = static_cast<const char*>(p->ws);
  fp.dbg_hi = fp.dbg_lo + p->ws_bytes;
  for (int l = 1; l < LF; ++l) {
    fp.src = p->lv[l];
    fp.dst = p->lv[l + 1];
    fp.Hf = p->Hs[l];
    fp.Wf = p->Ws[l];
    fp.Hc = p->Hs[l + 1];
    fp.Wc = p->Ws[l + 1];
    cudaError_t e;
    {
      ProfScope ps(p, stream, FLLF_K_FUSE, l);
      e = fllf::launch_fuse(fp, p->d.batch, stream, pdl);
    }
    if (e != cudaSuccess) return cuda_fail(e, "fuse kernel launch");
    ++launches;
  }
  for (int l = LF; l < lmax; ++l) {  // design AB above the fused levels: build steps
    st = build_level_impl(p, d_img, pitch, l, stream, pdl);
    if (st != FLLF_OK) return st;
    ++launches;
  }
  p->built = true;
  p->img = d_img;
  p->img_pitch = pitch;
  if (LF < lmax) {  // ... and applies l_max-1 .. LF
    st = apply_impl(p, nullptr, d_out, out_pitch_bytes, s, LF, lmax - 1, false, true);
    if (st != FLLF_OK) return st;
    launches += p->last_launches;
    p->last_was_apply = false;
  }
  for (int l = std::min(LF, lmax - 1) - 1; l >= 1; --l) {
    fllf::CollapseParams cp{};
    const fllf::DevLevel& F = p->lv[l];
    const fllf::DevLevel& C = p->lv[l + 1];
    cp.coarse = C.D;
    cp.cpitch = C.pitch;
    cp.cfstride = C.fstride_r;
    cp.fine = F.D;
    cp.fpitch = F.pitch;
    cp.ffstride = F.fstride_r;
    cp.Hf = F.H;
    cp.Wf = F.W;
    cp.Hc = C.H;
    cp.Wc = C.W;
    cp.dbg_lo = static_cast<const char*>(p->ws);
    cp.dbg_hi = cp.dbg_lo + p->ws_bytes;
    cudaError_t e;
    {
      ProfScope ps(p, stream, FLLF_K_COLLAPSE, l);
      e = fllf::launch_collapse(cp, p->d.batch, stream, pdl);
    }
    if (e != cudaSuccess) return cuda_fail(e, "collapse kernel launch");
    ++launches;
  }
  st = apply_impl(p, nullptr, d_out, out_pitch_bytes, s, 0, 0, false, true);
  if (st != FLLF_OK) return st;
  p->last_launches = launches + 1;
  return FLLF_OK;
}

static fllf_status filter_eager(fllf_plan p, const float* d_img, size_t in_pitch_bytes, float* d_out,
                                size_t out_pitch_bytes, void* s) {
  const int lf = fuse_levels(p);
  if (lf > 1) return filter_fused(p, d_img, in_pitch_bytes, d_out, out_pitch_bytes, s, lf);
  fllf_status st = fllf_build_fourier_pyramids(p, d_img, in_pitch_bytes, s);
  if (st != FLLF_OK) return st;
  const int nb = p->last_launches;
  st = fllf_apply(p, nullptr, d_out, out_pitch_bytes, s);
  if (st == FLLF_OK) p->last_launches += nb;
  return st;
}

fllf_status fllf_filter(fllf_plan p, const float* d_img, size_t in_pitch_bytes, float* d_out,
                        size_t out_pitch_bytes, void* s) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  if (p->band)
    return fail(FLLF_ERR_INVALID_ARGUMENT, "filter: row-band plans need the per-level calls (halo exchange)");
  if (!p->use_graph) return filter_eager(p, d_img, in_pitch_bytes, d_out, out_pitch_bytes, s);
  DeviceGuard guard(p->device);
  fllf_plan_s::GraphEntry* g = nullptr;
  for (auto& c : p->graphs)
    if (c.exec && c.in == d_img && c.out == d_out && c.in_pitch == in_pitch_bytes && c.out_pitch == out_pitch_bytes &&
        c.prof == p->profiling)
      g = &c;
  if (!g) {
    g = &p->graphs[0];  // an empty slot, else the least recently used one
    for (auto& c : p->graphs) {
      if (!c.exec) {
        g = &c;
        break;
      }
      if (c.used < g->used) g = &c;
    }
    if (g->exec) {
      cudaGraphExecDestroy(g->exec);
      g->exec = nullptr;
    }
    if (!p->cap_stream) {
      cudaError_t e = cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking);
      if (e != cudaSuccess) return cuda_fail(e, "capture stream");
    }
    cudaError_t e = cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamBeginCapture");
    p->capturing = true;
    fllf_status st = filter_eager(p, d_img, in_pitch_bytes, d_out, out_pitch_bytes, p->cap_stream);
    p->capturing = false;
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(p->cap_stream, &graph);
    if (st != FLLF_OK) {
      if (graph) cudaGraphDestroy(graph);
      return st;
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&g->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      g->exec = nullptr;
      return cuda_fail(e, "cudaGraphInstantiate");
    }
    g->in = d_img;
    g->out = d_out;
    g->in_pitch = in_pitch_bytes;
    g->out_pitch = out_pitch_bytes;
    g->prof = p->profiling;
    g->launches = p->last_launches;
    g->nrec = p->nrec;
  }
  g->used = ++p->graph_clock;
  cudaError_t e = cudaGraphLaunch(g->exec, static_cast<cudaStream_t>(s));
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphLaunch");
  // the replay leaves the plan in the state of a fresh build + apply
  p->built = true;
  p->img = d_img;
  p->img_pitch = (long long)((in_pitch_bytes ? in_pitch_bytes : (size_t)p->d.W * 4) / 4);
  p->last_was_apply = true;
  p->last_launches = g->launches;
  p->nrec = g->nrec;
  return FLLF_OK;
}

fllf_status fllf_filter_host(fllf_plan p, const float* h_img, float* h_out, void* s) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  if (!h_img || !h_out) return fail(FLLF_ERR_BAD_POINTER, "filter_host: NULL host pointer");
  DeviceGuard guard(p->device);
  const size_t bytes = (size_t)p->d.batch * p->d.H * p->d.W * sizeof(float);
  if (!p->stage_in || !p->stage_out) {
    if (cudaMalloc(&p->stage_in, bytes) != cudaSuccess || cudaMalloc(&p->stage_out, bytes) != cudaSuccess) {
      if (p->stage_in) cudaFree(p->stage_in);
      if (p->stage_out) cudaFree(p->stage_out);
      p->stage_in = p->stage_out = nullptr;
      cudaGetLastError();
      return fail(FLLF_ERR_OUT_OF_MEMORY, "staging cudaMalloc failed");
    }
  }
  cudaStream_t stream = static_cast<cudaStream_t>(s);
  cudaError_t e = cudaMemcpyAsync(p->stage_in, h_img, bytes, cudaMemcpyHostToDevice, stream);
  if (e != cudaSuccess) return cuda_fail(e, "H2D copy");
  fllf_status st = fllf_filter(p, p->stage_in, 0, p->stage_out, 0, s);
  if (st != FLLF_OK) return st;
  e = cudaMemcpyAsync(h_out, p->stage_out, bytes, cudaMemcpyDeviceToHost, stream);
  if (e != cudaSuccess) return cuda_fail(e, "D2H copy");
  return FLLF_OK;
}

// Release everything pipe_setup created (any subset); leaves the plan as before setup.
static void pipe_release(fllf_plan p) {
  for (int i = 0; i < fllf_plan_s::kPipe; ++i) {
    if (p->pipe_in[i]) cudaFree(p->pipe_in[i]);
    if (p->pipe_out[i]) cudaFree(p->pipe_out[i]);
    p->pipe_in[i] = p->pipe_out[i] = nullptr;
    for (cudaEvent_t* ev : {&p->ev_in[i], &p->ev_done[i], &p->ev_out[i]}) {
      if (*ev) cudaEventDestroy(*ev);
      *ev = nullptr;
    }
  }
  for (cudaEvent_t* ev : {&p->ev_pstart, &p->ev_pend}) {
    if (*ev) cudaEventDestroy(*ev);
    *ev = nullptr;
  }
  for (cudaStream_t* st : {&p->s_h2d, &p->s_d2h}) {
    if (*st) cudaStreamDestroy(*st);
    *st = nullptr;
  }
  cudaGetLastError();
}

// Staging buffers, copy streams and events of fllf_filter_host_frames, created
// once; all or nothing (a failure releases what was created, so the next call
// retries from scratch instead of running with missing pieces).
static fllf_status pipe_setup(fllf_plan p, size_t bytes) {
  if (p->pipe_ready) return FLLF_OK;
  for (int i = 0; i < fllf_plan_s::kPipe; ++i) {
    if (cudaMalloc(&p->pipe_in[i], bytes) != cudaSuccess || cudaMalloc(&p->pipe_out[i], bytes) != cudaSuccess) {
      pipe_release(p);
      return fail(FLLF_ERR_OUT_OF_MEMORY, "filter_host_frames: staging cudaMalloc failed");
    }
  }
  cudaError_t e = cudaStreamCreateWithFlags(&p->s_h2d, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->s_d2h, cudaStreamNonBlocking);
  for (cudaEvent_t* ev : {&p->ev_pstart, &p->ev_pend})
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
  for (int i = 0; i < fllf_plan_s::kPipe; ++i)
    for (cudaEvent_t* ev : {&p->ev_in[i], &p->ev_done[i], &p->ev_out[i]})
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    pipe_release(p);
    return cuda_fail(e, "filter_host_frames: stream / event creation");
  }
  p->pipe_ready = true;
  return FLLF_OK;
}

fllf_status fllf_filter_host_frames(fllf_plan p, const float* h_in, size_t in_stride_bytes, float* h_out,
                                    size_t out_stride_bytes, int nframes, void* s) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  if (!h_in || !h_out) return fail(FLLF_ERR_BAD_POINTER, "filter_host_frames: NULL host pointer");
  if (nframes < 0) return fail(FLLF_ERR_INVALID_ARGUMENT, "filter_host_frames: nframes < 0");
  if (p->band) return fail(FLLF_ERR_INVALID_ARGUMENT, "filter_host_frames: not for row-band plans");
  if (p->capturing) return fail(FLLF_ERR_INVALID_ARGUMENT, "filter_host_frames: not inside a stream capture");
  if (nframes == 0) return FLLF_OK;
  DeviceGuard guard(p->device);
  const size_t bytes = (size_t)p->d.batch * p->d.H * p->d.W * sizeof(float);
  fllf_status st = pipe_setup(p, bytes);
  if (st != FLLF_OK) return st;
  cudaStream_t cs = static_cast<cudaStream_t>(s);
  const char* hi = reinterpret_cast<const char*>(h_in);
  char* ho = reinterpret_cast<char*>(h_out);
  // the copies start after the work already queued on s
  cudaError_t e = cudaEventRecord(p->ev_pstart, cs);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_h2d, p->ev_pstart, 0);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_d2h, p->ev_pstart, 0);
  if (e != cudaSuccess) return cuda_fail(e, "filter_host_frames: fork");
  int launches = 0;
  for (int i = 0; i < nframes; ++i) {
    const int b = i % fllf_plan_s::kPipe;
    const bool reuse = i >= fllf_plan_s::kPipe;  // slot b held batch i - kPipe
    // H2D of batch i into slot b once batch i-kPipe's build has read it
    if (reuse) e = cudaStreamWaitEvent(p->s_h2d, p->ev_done[b], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(p->pipe_in[b], hi + (size_t)i * in_stride_bytes, bytes, cudaMemcpyHostToDevice, p->s_h2d);
    if (e == cudaSuccess) e = cudaEventRecord(p->ev_in[b], p->s_h2d);
    // filter on s once the input has landed and batch i-kPipe's result has left slot b
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, p->ev_in[b], 0);
    if (e == cudaSuccess && reuse) e = cudaStreamWaitEvent(cs, p->ev_out[b], 0);
    if (e == cudaSuccess && p->flush_buf) e = cudaMemsetAsync(p->flush_buf, i & 0xff, p->flush_bytes, cs);
    if (e != cudaSuccess) return cuda_fail(e, "filter_host_frames: H2D stage");
    st = fllf_filter(p, p->pipe_in[b], 0, p->pipe_out[b], 0, s);
    if (st != FLLF_OK) return st;
    launches += p->last_launches;
    e = cudaEventRecord(p->ev_done[b], cs);
    // D2H of frame i's result
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_d2h, p->ev_done[b], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(ho + (size_t)i * out_stride_bytes, p->pipe_out[b], bytes, cudaMemcpyDeviceToHost, p->s_d2h);
    if (e == cudaSuccess) e = cudaEventRecord(p->ev_out[b], p->s_d2h);
    if (e != cudaSuccess) return cuda_fail(e, "filter_host_frames: D2H stage");
  }
  // join: s completes after the last result has reached the host
  e = cudaEventRecord(p->ev_pend, p->s_d2h);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, p->ev_pend, 0);
  if (e != cudaSuccess) return cuda_fail(e, "filter_host_frames: join");
  p->last_launches = launches;
  return FLLF_OK;
}

fllf_status fllf_plan_set_l2_flush(fllf_plan p, void* d_buf, size_t bytes) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  if (!d_buf && bytes) return fail(FLLF_ERR_BAD_POINTER, "set_l2_flush: NULL buffer");
  p->flush_buf = bytes ? d_buf : nullptr;
  p->flush_bytes = bytes;
  return FLLF_OK;
}

// ---------------------------------------------------------------- NEXT-3
static fllf_status color_common(const float* a, const float* b, int H, int W, size_t pitch_bytes,
                                long long* pitch) {
  if (H < 1 || W < 1) return fail(FLLF_ERR_INVALID_ARGUMENT, "colour: H and W must be >= 1");
  fllf_status st = check_image(a, pitch_bytes, W, "colour: input", pitch);
  if (st != FLLF_OK) return st;
  st = check_image(b, pitch_bytes, W, "colour: output", pitch);
  if (st != FLLF_OK) return st;
  if (a == b) return fail(FLLF_ERR_BAD_POINTER, "colour: input and output may not alias");
  return FLLF_OK;
}

static fllf::ColorParams color_params(const float* src, float* dst, int H, int W, long long pitch) {
  fllf::ColorParams c{};
  for (int i = 0; i < 3; ++i) {
    c.src[i] = src + (long long)i * H * pitch;
    c.dst[i] = dst + (long long)i * H * pitch;
  }
  c.H = H;
  c.W = W;
  c.pitch = pitch;
  return c;
}

fllf_status fllf_rgb_to_yuv(const float* d_rgb, float* d_yuv, int H, int W, size_t pitch_bytes, void* s) {
  long long pitch;
  fllf_status st = color_common(d_rgb, d_yuv, H, W, pitch_bytes, &pitch);
  if (st != FLLF_OK) return st;
  NvtxRange r("fllf rgb_to_yuv", 0);
  cudaError_t e = fllf::launch_rgb_to_yuv(color_params(d_rgb, d_yuv, H, W, pitch), static_cast<cudaStream_t>(s));
  return e == cudaSuccess ? FLLF_OK : cuda_fail(e, "rgb_to_yuv launch");
}

fllf_status fllf_yuv_to_rgb(const float* d_yuv, float* d_rgb, int H, int W, size_t pitch_bytes, void* s) {
  long long pitch;
  fllf_status st = color_common(d_yuv, d_rgb, H, W, pitch_bytes, &pitch);
  if (st != FLLF_OK) return st;
  NvtxRange r("fllf yuv_to_rgb", 0);
  cudaError_t e = fllf::launch_yuv_to_rgb(color_params(d_yuv, d_rgb, H, W, pitch), static_cast<cudaStream_t>(s));
  return e == cudaSuccess ? FLLF_OK : cuda_fail(e, "yuv_to_rgb launch");
}

static fllf_status check_gain(const fllf_gain_desc* g) {
  if (!g) return fail(FLLF_ERR_BAD_POINTER, "gain: NULL description");
  if (g->radius < 0 || g->radius > FLLF_MAX_GAIN_RADIUS)
    return fail(FLLF_ERR_INVALID_ARGUMENT, "gain: radius must be in 0..FLLF_MAX_GAIN_RADIUS");
  if (!is_finite(g->m_lo) || !is_finite(g->m_hi) || !is_finite(g->v_ref) || !(g->v_ref > 0))
    return fail(FLLF_ERR_INVALID_ARGUMENT, "gain: m_lo, m_hi finite and v_ref > 0 required");
  return FLLF_OK;
}

fllf_status fllf_gain_map(const float* d_y, size_t y_pitch_bytes, int H, int W, const fllf_gain_desc* g,
                          float* d_m, size_t m_pitch_bytes, void* s) {
  if (H < 1 || W < 1) return fail(FLLF_ERR_INVALID_ARGUMENT, "gain: H and W must be >= 1");
  fllf_status st = check_gain(g);
  if (st != FLLF_OK) return st;
  long long yp, mp;
  st = check_image(d_y, y_pitch_bytes, W, "gain: d_y", &yp);
  if (st != FLLF_OK) return st;
  st = check_image(d_m, m_pitch_bytes, W, "gain: d_m", &mp);
  if (st != FLLF_OK) return st;
  fllf::GainParams gp{};
  gp.y = d_y;
  gp.y_pitch = yp;
  gp.m = d_m;
  gp.m_pitch = mp;
  gp.H = H;
  gp.W = W;
  gp.radius = g->radius;
  gp.m_lo = g->m_lo;
  gp.m_hi = g->m_hi;
  gp.inv_vref = 1.0 / g->v_ref;
  NvtxRange r("fllf gain_map", 0);
  cudaError_t e = fllf::launch_gain_map(gp, static_cast<cudaStream_t>(s));
  return e == cudaSuccess ? FLLF_OK : cuda_fail(e, "gain_map launch");
}

fllf_status fllf_enhance_rgb(fllf_plan p, const float* d_rgb, float* d_rgb_out, size_t pitch_bytes,
                             const fllf_gain_desc* g, void* s) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  if (p->d.batch != 1 || p->band) return fail(FLLF_ERR_INVALID_ARGUMENT, "enhance_rgb: plan batch must be 1, full frame");
  fllf_status st = check_gain(g);
  if (st != FLLF_OK) return st;
  const int H = p->d.H, W = p->d.W;
  long long pitch;
  st = color_common(d_rgb, d_rgb_out, H, W, pitch_bytes, &pitch);
  if (st != FLLF_OK) return st;
  if (pitch != W) return fail(FLLF_ERR_BAD_POINTER, "enhance_rgb: planes must be dense (pitch_bytes 0 or W*4)");
  DeviceGuard guard(p->device);
  cudaStream_t stream = static_cast<cudaStream_t>(s);
  const size_t plane = (size_t)H * W;
  if (!p->color_ws) {
    if (cudaMalloc(&p->color_ws, 6 * plane * sizeof(float)) != cudaSuccess) {
      cudaGetLastError();
      p->color_ws = nullptr;
      return fail(FLLF_ERR_OUT_OF_MEMORY, "enhance_rgb workspace cudaMalloc failed");
    }
    p->color_sigma = -1.f;
  }
  float* yuv = p->color_ws;             // Y, U, V
  float* yo = p->color_ws + 3 * plane;  // Y' (the LLF output)
  float* smap = p->color_ws + 4 * plane;
  float* mmap = p->color_ws + 5 * plane;
  cudaError_t e = fllf::launch_rgb_to_yuv(color_params(d_rgb, yuv, H, W, pitch), stream);
  if (e != cudaSuccess) return cuda_fail(e, "rgb_to_yuv launch");
  st = fllf_build_fourier_pyramids(p, yuv, 0, s);
  if (st != FLLF_OK) return st;
  st = fllf_gain_map(yuv, 0, H, W, g, mmap, 0, s);
  if (st != FLLF_OK) return st;
  const float sig = (float)p->d.sigma_r;
  if (p->color_sigma != sig) {  // the uniform sigma_r map (R16), filled once per plan
    e = fllf::launch_fill(smap, W, H, W, sig, stream);
    if (e != cudaSuccess) return cuda_fail(e, "sigma map fill");
    p->color_sigma = sig;
  }
  fllf_apply_args a{};
  a.mode = FLLF_MAPS;
  a.d_sigma_r = smap;
  a.d_m = mmap;
  a.map_pitch_bytes = 0;
  st = fllf_apply(p, &a, yo, 0, s);
  if (st != FLLF_OK) return st;
  fllf::ColorParams c{};
  c.src[0] = yo;
  c.src[1] = yuv + plane;
  c.src[2] = yuv + 2 * plane;
  for (int i = 0; i < 3; ++i) c.dst[i] = d_rgb_out + (long long)i * H * pitch;
  c.H = H;
  c.W = W;
  c.pitch = pitch;
  e = fllf::launch_yuv_to_rgb(c, stream);
  if (e != cudaSuccess) return cuda_fail(e, "yuv_to_rgb launch");
  return FLLF_OK;
}

// ---------------------------------------------------------------- NEXT-2
fllf_status fllf_naive_llf(fllf_plan p, const float* d_img, size_t pitch_bytes, int remap_mode, float* d_out,
                           size_t out_pitch_bytes, void* s) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  if (p->d.batch != 1 || p->kb != 1 || p->KL != p->d.K || !p->d.include_base || p->band)
    return fail(FLLF_ERR_INVALID_ARGUMENT, "naive_llf: needs batch 1, all orders, include_base, full frame");
  if (remap_mode != 0 && remap_mode != 1) return fail(FLLF_ERR_INVALID_ARGUMENT, "naive_llf: remap_mode 0 or 1");
  if (p->nlev > FLLF_NAIVE_MAX_LEVELS) return fail(FLLF_ERR_TOO_MANY_LEVELS, "naive_llf: levels > FLLF_NAIVE_MAX_LEVELS");
  long long ipitch, opitch;
  fllf_status st = check_image(d_img, pitch_bytes, p->d.W, "naive: d_img", &ipitch);
  if (st != FLLF_OK) return st;
  st = check_image(d_out, out_pitch_bytes, p->d.W, "naive: d_out", &opitch);
  if (st != FLLF_OK) return st;
  st = fllf_build_fourier_pyramids(p, d_img, pitch_bytes, s);
  if (st != FLLF_OK) return st;
  DeviceGuard guard(p->device);
  cudaStream_t stream = static_cast<cudaStream_t>(s);
  fllf::NaiveParams np{};
  np.img = d_img;
  np.img_pitch = ipitch;
  for (int l = 0; l < p->nlev; ++l) {
    np.Hs[l] = p->Hs[l];
    np.Ws[l] = p->Ws[l];
    if (l >= 1) {
      np.G[l] = p->lv[l].G;
      np.gpitch[l] = p->lv[l].pitch;
      np.L[l] = p->lv[l].D;
      np.lpitch[l] = p->lv[l].pitch;
    }
  }
  np.L[0] = d_out;
  np.lpitch[0] = opitch;
  np.mode = remap_mode;
  np.K = p->d.K;
  np.m = p->d.m;
  np.inv2s2 = 1.0 / (2.0 * p->d.sigma_r * p->d.sigma_r);
  {
    std::vector<double> om(p->d.K), ak(p->d.K);
    fllf_coefficients(p->d.K, p->d.T, p->d.sigma_r, p->d.m, om.data(), ak.data());
    for (int k = 0; k < p->d.K; ++k) {
      np.omega[k] = om[k];
      np.a[k] = ak[k];
    }
  }
  const int lmax = p->nlev - 1;
  for (int l = 0; l < lmax; ++l) {
    np.level = l;
    NvtxRange r("fllf naive_level", l);
    cudaError_t e = fllf::launch_naive_level(np, stream);
    if (e != cudaSuccess) return cuda_fail(e, "naive level launch");
  }
  // collapse (Eq. 4): O_l = L_l + up(O_{l+1}), O_lmax = G_lmax
  for (int l = lmax - 1; l >= 0; --l) {
    float* fine = l == 0 ? d_out : p->lv[l].D;
    const long long fp = l == 0 ? opitch : p->lv[l].pitch;
    const float* coarse = (l + 1 == lmax) ? p->lv[l + 1].G : p->lv[l + 1].D;
    cudaError_t e = fllf::launch_collapse_up(fine, fp, coarse, p->lv[l + 1].pitch, p->Hs[l], p->Ws[l], p->Hs[l + 1],
                                             p->Ws[l + 1], stream);
    if (e != cudaSuccess) return cuda_fail(e, "collapse launch");
  }
  p->last_launches += 2 * lmax;
  return FLLF_OK;
}

fllf_status fllf_plan_get_desc(fllf_plan p, fllf_plan_desc* out) {
  if (!p || !out) return fail(FLLF_ERR_BAD_POINTER, "plan_get_desc: NULL argument");
  *out = p->d;
  out->device = p->device;
  return FLLF_OK;
}

fllf_status fllf_plan_level_dims(fllf_plan p, int level, int* H, int* W) {
  if (!p || !H || !W) return fail(FLLF_ERR_BAD_POINTER, "NULL argument");
  if (level < 0 || level >= p->nlev) return fail(FLLF_ERR_INVALID_ARGUMENT, "level out of range");
  *H = p->Hs[level];
  *W = p->Ws[level];
  return FLLF_OK;
}

fllf_status fllf_workspace_bytes(fllf_plan p, size_t* bytes) {
  if (!p || !bytes) return fail(FLLF_ERR_BAD_POINTER, "NULL argument");
  *bytes = p->ws_bytes;
  return FLLF_OK;
}

fllf_status fllf_read_pyramid(fllf_plan p, int frame, int level, int channel, float* d_dst,
                              size_t dst_pitch_bytes, void* s) {
  if (!p || !d_dst) return fail(FLLF_ERR_BAD_POINTER, "NULL argument");
  if (!p->built) return fail(FLLF_ERR_NOT_BUILT, "read_pyramid before build");
  if (p->band) return fail(FLLF_ERR_INVALID_ARGUMENT, "read_pyramid: use fllf_plan_band_plane on row bands");
  if (level < 1 || level >= p->nlev || frame < 0 || frame >= p->d.batch || channel < 0 || channel > p->KL)
    return fail(FLLF_ERR_INVALID_ARGUMENT, "read_pyramid: frame/level/channel out of range");
  DeviceGuard guard(p->device);
  const fllf::DevLevel& L = p->lv[level];
  const void* src;
  size_t spitch, wbytes;
  if (channel == 0) {
    src = L.G + (long long)frame * L.fstride_r;
    spitch = (size_t)L.pitch * sizeof(float);
    wbytes = (size_t)L.W * sizeof(float);
  } else {
    src = L.Z + (long long)frame * L.fstride_z + (long long)(channel - 1) * L.kstride_z;
    spitch = (size_t)L.zpitch * sizeof(float2);
    wbytes = (size_t)L.W * sizeof(float2);
  }
  if (dst_pitch_bytes == 0) dst_pitch_bytes = wbytes;
  if (dst_pitch_bytes < wbytes) return fail(FLLF_ERR_BAD_POINTER, "read_pyramid: destination pitch too small");
  cudaError_t e = cudaMemcpy2DAsync(d_dst, dst_pitch_bytes, src, spitch, wbytes, (size_t)L.H,
                                    cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(s));
  if (e != cudaSuccess) return cuda_fail(e, "read_pyramid copy");
  return FLLF_OK;
}

int fllf_plan_last_launch_count(fllf_plan p) { return p ? p->last_launches : 0; }

fllf_status fllf_plan_set_profiling(fllf_plan p, int enable) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  p->profiling = enable != 0;
  p->nrec = 0;
  return FLLF_OK;
}

static void drop_graphs(fllf_plan p) {  // cached graphs hold the previous launch sequence
  DeviceGuard guard(p->device);
  for (auto& g : p->graphs)
    if (g.exec) {
      cudaGraphExecDestroy(g.exec);
      g.exec = nullptr;
    }
}

fllf_status fllf_plan_set_design(fllf_plan p, int design) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  if (design != FLLF_DESIGN_AUTO && design != FLLF_DESIGN_AB && design != FLLF_DESIGN_F)
    return fail(FLLF_ERR_INVALID_ARGUMENT, "set_design: FLLF_DESIGN_AUTO, _AB or _F");
  drop_graphs(p);
  p->design = design;
  p->fused_levels = 0;
  return FLLF_OK;
}

fllf_status fllf_plan_set_fused_levels(fllf_plan p, int n) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  if (n < 0) return fail(FLLF_ERR_INVALID_ARGUMENT, "set_fused_levels: n >= 0");
  drop_graphs(p);
  p->fused_levels = n;
  if (n == 0) p->design = FLLF_DESIGN_AUTO;
  return FLLF_OK;
}

fllf_status fllf_plan_set_graphs(fllf_plan p, int enable) {
  if (!p) return fail(FLLF_ERR_BAD_POINTER, "NULL plan");
  p->use_graph = enable != 0;
  return FLLF_OK;
}

fllf_status fllf_plan_kernel_times(fllf_plan p, int capacity, int* kind, int* level, float* ms, int* count) {
  if (!p || !count) return fail(FLLF_ERR_BAD_POINTER, "NULL argument");
  DeviceGuard guard(p->device);
  const int n = std::min(capacity, p->nrec);
  for (int i = 0; i < n; ++i) {
    cudaError_t e = cudaEventSynchronize(p->ev_stop[i]);
    if (e != cudaSuccess) return cuda_fail(e, "kernel_times: event sync");
    float t = 0.f;
    e = cudaEventElapsedTime(&t, p->ev_start[i], p->ev_stop[i]);
    if (e != cudaSuccess) return cuda_fail(e, "kernel_times: elapsed");
    if (kind) kind[i] = p->rec_kind[i];
    if (level) level[i] = p->rec_level[i];
    if (ms) ms[i] = t;
  }
  *count = n;
  return FLLF_OK;
}

}  // extern "C"
