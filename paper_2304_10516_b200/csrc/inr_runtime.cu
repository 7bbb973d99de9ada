// inr_runtime.cu — host runtime behind the C ABI of include/inr.h.
//
// Owns model memory (parameters, gradients, Adam state, counters: one device
// allocation per model), builds the per-group kernel parameter blocks, runs the
// fit loop (optionally as a replayed CUDA graph per step), dispatches decode,
// and implements the FIFO timestep window.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <deque>
#include <list>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/inr.h"
#include "launch.h"

using namespace inr;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};

namespace inr {
void count_launch(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}

static inr_status fail(inr_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

static inr_status cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation) return fail(INR_ERR_OOM, "%s: %s", what, cudaGetErrorString(e));
  return fail(INR_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CK(call)                                        \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

#define CK_LAUNCH(what)                                  \
  do {                                                   \
    cudaError_t e_ = cudaGetLastError();                 \
    if (e_ != cudaSuccess) return cuda_fail(e_, what);   \
  } while (0)

extern "C" const char* inr_last_error(void) { return g_err.c_str(); }

// ------------------------------------------------------------------ profiling
enum ProfKind { PK_STEP_BEGIN, PK_FIT_FP32, PK_SAMPLE, PK_ENCODE_FWD, PK_PREP, PK_MLP_TC, PK_ENCODE_BWD, PK_ADAM,
                PK_DECODE_GRID, PK_DECODE_QUERY, PK_PROBE, PK_RANGE, PK_PATHLINE, PK_COUNT };
static const char* kProfNames[PK_COUNT] = {"step_begin", "fit_fp32", "sample", "encode_fwd", "prep_image", "mlp_tc",
                                           "encode_bwd", "adam", "decode_grid", "decode_query", "probe", "range",
                                           "pathline"};
struct ProfRec { int kind; cudaEvent_t a, b; };
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_event_pool;
static bool g_prof_on = false;

static cudaEvent_t prof_event() {
  cudaEvent_t e;
  if (!g_event_pool.empty()) { e = g_event_pool.back(); g_event_pool.pop_back(); return e; }
  cudaEventCreate(&e);
  return e;
}

// Brackets one kernel launch with events on its stream when profiling is on.
// (inside a stream capture the records must be "external" to become event nodes)
static void prof_record(cudaEvent_t e, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
  else cudaEventRecord(e, st);
}

// INR_DEBUG_SYNC=1: synchronize after every library kernel and report the first
// failing one by name on stderr (debugging aid; no effect otherwise).
static const bool g_debug_sync = getenv("INR_DEBUG_SYNC") != nullptr;

struct ProfScope {
  int kind;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(int k, cudaStream_t s) : kind(k), st(s) {
    if (g_prof_on) { a = prof_event(); prof_record(a, st); }
  }
  ~ProfScope() {
    if (g_debug_sync) {
      cudaError_t e = cudaStreamSynchronize(st);
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e != cudaSuccess) fprintf(stderr, "[libinr] kernel %s failed: %s\n", kProfNames[kind], cudaGetErrorString(e));
    }
    if (a) {
      cudaEvent_t b = prof_event();
      prof_record(b, st);
      g_prof.push_back({kind, a, b});
    }
  }
};

static void prof_clear() {
  for (auto& r : g_prof) { g_event_pool.push_back(r.a); g_event_pool.push_back(r.b); }
  g_prof.clear();
}

extern "C" inr_status inr_profile_enable(int32_t on) {
  g_prof_on = on != 0;
  if (g_prof_on) prof_clear();
  return INR_OK;
}

extern "C" inr_status inr_profile_span(double* span_ms) {
  if (!span_ms) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  *span_ms = 0;
  if (g_prof.empty()) return INR_OK;
  CK(cudaEventSynchronize(g_prof.back().b));
  float t = 0;
  CK(cudaEventElapsedTime(&t, g_prof.front().a, g_prof.back().b));
  *span_ms = t;
  return INR_OK;
}

extern "C" inr_status inr_profile_read(const char* kernel, double* total_ms, int64_t* launches) {
  if (!kernel || !total_ms || !launches) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  int kind = -1;
  for (int k = 0; k < PK_COUNT; ++k)
    if (!strcmp(kernel, kProfNames[k])) kind = k;
  if (kind < 0) return fail(INR_ERR_INVALID_ARG, "unknown kernel class '%s'", kernel);
  double ms = 0;
  int64_t n = 0;
  for (auto& r : g_prof) {
    if (r.kind != kind) continue;
    CK(cudaEventSynchronize(r.b));
    float t = 0;
    CK(cudaEventElapsedTime(&t, r.a, r.b));
    ms += t;
    ++n;
  }
  *total_ms = ms;
  *launches = n;
  return INR_OK;
}
extern "C" int64_t inr_kernel_launches(void) { return g_launches.load(); }

// ------------------------------------------------------------------ model
struct inr_model {
  inr_config cfg;
  inr_block blk;
  int device;
  NetDesc net;
  int64_t P;            // declared parameters (API)
  int64_t P_pad;        // internal (aligned, padded) length of each array
  void* mem = nullptr;
  float* params = nullptr;
  float* grads = nullptr;
  float* adam_m = nullptr;
  float* adam_v = nullptr;
  unsigned long long* gfx = nullptr;
  long long* step_total = nullptr;
  long long* step_cur = nullptr;
  double* acc = nullptr;
  int* flag = nullptr;
  int64_t steps = 0;
  uint32_t block_id = 0;
  int nfaces = 0;
  int faces[6] = {0, 0, 0, 0, 0, 0};
  float vmin[kMaxD] = {0.f, 0.f, 0.f}, vmax[kMaxD] = {1.f, 1.f, 1.f};   // per-channel range of the last fit
  double last_inv_u = 0.0, last_inv_b = 0.0;   // 1/(B_u D), 1/(B_b D) of the last fit step (report)
  double* mesh = nullptr;                      // rectilinear (R36): device node coordinates, 3 slices
  int mesh_n[3] = {0, 0, 0};
  double plo[3] = {0, 0, 0}, pspan[3] = {0, 0, 0};
  bool frozen = false;       // cache snapshot: parameters only
  bool host_resident = false;
  float* host_params = nullptr;  // pinned copy (host-resident snapshot)
  bool staged = false;           // params (device) holds the host / fp16 copy
  __half* h16 = nullptr;         // fp16-stored snapshot (device, or pinned host if host_resident)
};

static inr_status validate_config(const inr_config* c) {
  if (!c) return fail(INR_ERR_INVALID_ARG, "config is NULL");
  if (c->levels < 1) return fail(INR_ERR_INVALID_ARG, "levels must be >= 1");
  if (c->features < 1) return fail(INR_ERR_INVALID_ARG, "features must be >= 1");
  if (c->log2_table_size < 1 || c->log2_table_size > 30)
    return fail(INR_ERR_INVALID_ARG, "log2_table_size must be in 1..30 (T a power of two)");
  if (c->base_resolution < 1) return fail(INR_ERR_INVALID_ARG, "base_resolution must be >= 1");
  if (!(c->per_level_scale > 1.f)) return fail(INR_ERR_INVALID_ARG, "per_level_scale must be > 1");
  if (c->levels >= 1 &&
      std::floor((double)c->base_resolution * std::pow((double)c->per_level_scale, (double)(c->levels - 1))) >
          (double)(1 << 30))
    return fail(INR_ERR_INVALID_ARG, "finest level resolution N_{L-1} exceeds 2^30 (int32 cell index) [R3]");
  if (c->mlp_hidden_layers < 1) return fail(INR_ERR_INVALID_ARG, "mlp_hidden_layers must be >= 1");
  if (c->mlp_width < 1) return fail(INR_ERR_INVALID_ARG, "mlp_width must be >= 1");
  if (c->out_dim < 1) return fail(INR_ERR_INVALID_ARG, "out_dim must be >= 1");
  if (c->precision != INR_PREC_FP32 && c->precision != INR_PREC_FP16_MLP)
    return fail(INR_ERR_INVALID_ARG, "unknown precision");
  if (c->reduction != INR_REDUCE_ATOMIC && c->reduction != INR_REDUCE_DETERMINISTIC)
    return fail(INR_ERR_INVALID_ARG, "unknown reduction");
  if (c->features != 1 && c->features != 2 && c->features != 4 && c->features != 8)
    return fail(INR_ERR_UNSUPPORTED, "features must be 1, 2, 4 or 8 in this build");
  if (c->levels > kMaxLevels) return fail(INR_ERR_UNSUPPORTED, "at most %d levels", kMaxLevels);
  if (c->levels * c->features > 64) return fail(INR_ERR_UNSUPPORTED, "levels*features must be <= 64");
  if (c->log2_table_size > 24) return fail(INR_ERR_UNSUPPORTED, "log2_table_size must be <= 24 in this build");
  if (c->mlp_width != kWidth) return fail(INR_ERR_UNSUPPORTED, "mlp_width must be 64 in this build");
  if (c->mlp_hidden_layers > kMaxLayers - 1) return fail(INR_ERR_UNSUPPORTED, "at most 8 hidden layers");
  if (c->out_dim != 1 && c->out_dim != 3) return fail(INR_ERR_UNSUPPORTED, "out_dim must be 1 or 3 in this build");
  if (c->precision == INR_PREC_FP16_MLP && (c->levels * c->features) % 16 != 0)
    return fail(INR_ERR_UNSUPPORTED, "fp16 MLP needs levels*features to be a multiple of 16");
  return INR_OK;
}

static inr_status validate_block(const inr_block* b) {
  if (!b) return fail(INR_ERR_INVALID_ARG, "block is NULL");
  for (int d = 0; d < 3; ++d) {
    if (b->n[d] < 1 || b->global_dims[d] < 1 || b->origin[d] < 0)
      return fail(INR_ERR_INVALID_ARG, "block extents must be positive");
    if (b->origin[d] % b->n[d] != 0) return fail(INR_ERR_INVALID_ARG, "block origin must be a multiple of n");
    if (b->origin[d] >= b->global_dims[d]) return fail(INR_ERR_INVALID_ARG, "block origin outside the volume");
    if (b->global_dims[d] >= (1ll << 24)) return fail(INR_ERR_UNSUPPORTED, "global dims must be < 2^24");
  }
  return INR_OK;
}

// N_l = floor(N_min * b^l) in double (R3); S_l = min(T, (N_l+1)^3) (R2).
static void build_net(const inr_config& c, NetDesc& net) {
  memset(&net, 0, sizeof net);
  net.L = c.levels;
  net.F = c.features;
  net.H = c.mlp_hidden_layers;
  net.LF = c.levels * c.features;
  net.D = c.out_dim;
  net.bias = c.mlp_bias ? 1 : 0;
  uint64_t T = 1ull << c.log2_table_size;
  net.table_mask = (uint32_t)(T - 1);
  int64_t off = 0, decl = 0;
  auto add_tensor = [&](int64_t len, int fan_in) {
    off = (off + kTensorAlign - 1) / kTensorAlign * kTensorAlign;
    int t = net.ntensors++;
    net.t_off[t] = off;
    net.t_decl[t] = decl;
    net.t_len[t] = len;
    net.t_fan_in[t] = fan_in;
    off += len;
    decl += len;
    return net.t_off[t];
  };
  for (int l = 0; l < c.levels; ++l) {
    double r = std::floor((double)c.base_resolution * std::pow((double)c.per_level_scale, (double)l));
    uint64_t res = (uint64_t)r;
    double dense = std::pow((double)res + 1.0, 3.0);
    LevelInfo& lv = net.lv[l];
    lv.res = (uint32_t)res;
    if (dense <= (double)T) { lv.size = (uint32_t)((res + 1) * (res + 1) * (res + 1)); lv.dense = 1; }
    else { lv.size = (uint32_t)T; lv.dense = 0; }
    lv.offset = add_tensor((int64_t)lv.size * c.features, 0);
  }
  for (int k = 0; k <= net.H; ++k) {
    net.in_dim[k] = k == 0 ? net.LF : kWidth;
    net.out_dim[k] = k == net.H ? net.D : kWidth;
    net.w_off[k] = add_tensor((int64_t)net.in_dim[k] * net.out_dim[k], net.in_dim[k]);
    net.b_off[k] = net.bias ? add_tensor(net.out_dim[k], -1) : -1;
  }
  net.nparams = (off + kTensorAlign - 1) / kTensorAlign * kTensorAlign;
  net.ndecl = decl;
}

static void philox_key(uint64_t seed, uint32_t stream, uint32_t& k0, uint32_t& k1) {
  k0 = (uint32_t)(seed & 0xffffffffu);
  k1 = (uint32_t)(seed >> 32) ^ stream;
}

static void block_geometry(inr_model* m) {
  const inr_block& b = m->blk;
  int64_t B[3], c[3];
  for (int d = 0; d < 3; ++d) { B[d] = (b.global_dims[d] + b.n[d] - 1) / b.n[d]; c[d] = b.origin[d] / b.n[d]; }
  m->block_id = (uint32_t)((c[2] * B[1] + c[1]) * B[0] + c[0]);
  m->nfaces = 0;
  for (int d = 0; d < 3; ++d) {
    if (b.origin[d] > 0) m->faces[m->nfaces++] = 2 * d;
    if (b.origin[d] + b.n[d] < b.global_dims[d]) m->faces[m->nfaces++] = 2 * d + 1;
  }
}

// frozen: parameters only; host_only: no device parameter buffer (staged lazily on decode).
static inr_status alloc_model(inr_model* m, bool frozen, bool host_only = false) {
  m->P = m->net.ndecl;
  m->P_pad = m->net.nparams;
  size_t bytes = (size_t)m->P_pad * sizeof(float) * (host_only ? 0 : (frozen ? 1 : 4)) + 256;
  if (!frozen && m->cfg.reduction == INR_REDUCE_DETERMINISTIC) bytes += (size_t)m->P_pad * 8;
  CK(cudaMalloc(&m->mem, bytes));
  char* p = (char*)m->mem;
  if (!host_only) { m->params = (float*)p; p += m->P_pad * 4; }
  if (!frozen) {
    m->grads = (float*)p; p += m->P_pad * 4;
    m->adam_m = (float*)p; p += m->P_pad * 4;
    m->adam_v = (float*)p; p += m->P_pad * 4;
    if (m->cfg.reduction == INR_REDUCE_DETERMINISTIC) { m->gfx = (unsigned long long*)p; p += m->P_pad * 8; }
  }
  m->step_total = (long long*)p;
  m->step_cur = (long long*)(p + 8);
  m->acc = (double*)(p + 16);
  m->flag = (int*)(p + 48);
  CK(cudaMemset(p, 0, 256));
  return INR_OK;
}

static inr_status init_state(inr_model* m, uint64_t seed, cudaStream_t st, bool keep_params = false) {
  if (!keep_params) {
    uint32_t k0, k1;
    philox_key(seed, 0, k0, k1);
    launch_init_params(m->net, m->params, k0, k1, m->block_id, st);
    CK_LAUNCH("init_params");
  }
  size_t n = (size_t)m->P_pad * 4;
  CK(cudaMemsetAsync(m->grads, 0, n * 3, st));  // grads, m, v are contiguous
  if (m->gfx) CK(cudaMemsetAsync(m->gfx, 0, (size_t)m->P_pad * 8, st));
  char* tail = (char*)m->step_total;
  CK(cudaMemsetAsync(tail, 0, 256, st));
  m->steps = 0;
  return INR_OK;
}

extern "C" inr_status inr_create(const inr_config* cfg, const inr_block* block, int device, inr_model** out) {
  if (!out) return fail(INR_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  inr_status s = validate_config(cfg);
  if (s) return s;
  if ((s = validate_block(block))) return s;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(INR_ERR_INVALID_ARG, "device %d out of range", device);
  CK(cudaSetDevice(device));
  inr_model* m = new inr_model();
  m->cfg = *cfg;
  m->blk = *block;
  m->device = device;
  build_net(*cfg, m->net);
  block_geometry(m);
  if ((s = alloc_model(m, false)) || (s = init_state(m, cfg->seed, 0))) {
    if (m->mem) cudaFree(m->mem);
    delete m;
    return s;
  }
  CK(cudaStreamSynchronize(0));
  *out = m;
  return INR_OK;
}

extern "C" inr_status inr_reset(inr_model* m, uint64_t seed) {
  if (!m) return fail(INR_ERR_INVALID_ARG, "model is NULL");
  if (m->frozen) return fail(INR_ERR_STATE, "model is a frozen cache snapshot");
  CK(cudaSetDevice(m->device));
  CK(cudaDeviceSynchronize());   // work queued on any stream may still use the parameters
  m->cfg.seed = seed;
  inr_status s = init_state(m, seed, 0);
  if (s) return s;
  CK(cudaStreamSynchronize(0));
  return INR_OK;
}

// Rectilinear mesh (NEXT-4; R36): keep the block's slice of the global
// node coordinates on the device; the fit samples and the decodes go through it.
static inr_status set_mesh_slices(inr_model* m, const double* const* slices, const int n[3], bool device_src) {
  const size_t tot = (size_t)n[0] + n[1] + n[2];
  double* dm = nullptr;
  CK(cudaSetDevice(m->device));
  CK(cudaMalloc((void**)&dm, tot * sizeof(double)));
  size_t off = 0;
  for (int d = 0; d < 3; ++d) {
    cudaError_t e = cudaMemcpy(dm + off, slices[d], (size_t)n[d] * sizeof(double),
                               device_src ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice);
    if (e != cudaSuccess) { cudaFree(dm); return cuda_fail(e, "mesh copy"); }
    off += n[d];
  }
  if (m->mesh) cudaFree(m->mesh);
  m->mesh = dm;
  for (int d = 0; d < 3; ++d) m->mesh_n[d] = n[d];
  return INR_OK;
}

extern "C" inr_status inr_set_mesh(inr_model* m, const double* const coords[3]) {
  if (!m) return fail(INR_ERR_INVALID_ARG, "model is NULL");
  if (m->frozen) return fail(INR_ERR_STATE, "model is a frozen cache snapshot");
  if (!coords) {   // back to the uniform mesh
    if (m->mesh) { cudaSetDevice(m->device); cudaFree(m->mesh); }
    m->mesh = nullptr;
    return INR_OK;
  }
  const double* slices[3];
  int n[3];
  double lo[3], hi[3];
  for (int d = 0; d < 3; ++d) {
    if (!coords[d]) return fail(INR_ERR_INVALID_ARG, "coords[%d] is NULL", d);
    const int64_t N = m->blk.global_dims[d], o = m->blk.origin[d];
    for (int64_t i = 0; i + 1 < N; ++i)
      if (!(coords[d][i + 1] > coords[d][i]))
        return fail(INR_ERR_INVALID_ARG, "mesh coordinates must be strictly increasing (axis %d)", d);
    const int64_t last = std::min<int64_t>(o + m->blk.n[d], N - 1);
    slices[d] = coords[d] + o;
    n[d] = (int)(last - o + 1);
    lo[d] = coords[d][o];
    hi[d] = coords[d][last];
  }
  inr_status s = set_mesh_slices(m, slices, n, false);
  if (s) return s;
  for (int d = 0; d < 3; ++d) { m->plo[d] = lo[d]; m->pspan[d] = hi[d] - lo[d]; }
  return INR_OK;
}

// ---- model state transfer (NEXT-4 block stealing): [host meta 256 B][device tail 256 B][params][m][v]
struct StateMeta {
  int64_t steps;
  float vmin[kMaxD], vmax[kMaxD];
  double last_inv_u, last_inv_b;
  int64_t P_pad;
  uint32_t block_id, magic;
};
static const uint32_t kStateMagic = 0x494e5253u;

extern "C" inr_status inr_state_bytes(const inr_model* m, int64_t* bytes) {
  if (!m || !bytes) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  *bytes = 512 + 3 * (int64_t)m->P_pad * 4;
  return INR_OK;
}

extern "C" inr_status inr_export_state(const inr_model* m, void* dst, cudaStream_t st) {
  if (!m || !dst) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  if (m->frozen) return fail(INR_ERR_STATE, "a frozen cache snapshot has no optimizer state");
  static thread_local StateMeta meta;   // pinned-free host source: the copy completes before return (sync)
  memset(&meta, 0, sizeof meta);
  meta.steps = m->steps;
  memcpy(meta.vmin, m->vmin, sizeof meta.vmin);
  memcpy(meta.vmax, m->vmax, sizeof meta.vmax);
  meta.last_inv_u = m->last_inv_u;
  meta.last_inv_b = m->last_inv_b;
  meta.P_pad = m->P_pad;
  meta.block_id = m->block_id;
  meta.magic = kStateMagic;
  char* d = (char*)dst;
  const size_t n = (size_t)m->P_pad * 4;
  CK(cudaSetDevice(m->device));
  CK(cudaMemcpyAsync(d, &meta, sizeof meta, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d + 256, m->step_total, 256, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(d + 512, m->params, n, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(d + 512 + n, m->adam_m, 2 * n, cudaMemcpyDeviceToDevice, st));   // m, v contiguous
  CK(cudaStreamSynchronize(st));
  return INR_OK;
}

extern "C" inr_status inr_import_state(inr_model* m, const void* src, cudaStream_t st) {
  if (!m || !src) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  if (m->frozen) return fail(INR_ERR_STATE, "model is a frozen cache snapshot");
  StateMeta meta;
  const char* s = (const char*)src;
  CK(cudaSetDevice(m->device));
  CK(cudaMemcpyAsync(&meta, s, sizeof meta, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (meta.magic != kStateMagic || meta.P_pad != m->P_pad || meta.block_id != m->block_id)
    return fail(INR_ERR_INVALID_ARG, "state was exported by a model of another configuration or block");
  const size_t n = (size_t)m->P_pad * 4;
  CK(cudaMemcpyAsync(m->step_total, s + 256, 256, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(m->params, s + 512, n, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(m->adam_m, s + 512 + n, 2 * n, cudaMemcpyDeviceToDevice, st));
  CK(cudaStreamSynchronize(st));
  m->steps = meta.steps;
  memcpy(m->vmin, meta.vmin, sizeof meta.vmin);
  memcpy(m->vmax, meta.vmax, sizeof meta.vmax);
  m->last_inv_u = meta.last_inv_u;
  m->last_inv_b = meta.last_inv_b;
  return INR_OK;
}

extern "C" inr_status inr_reset_optimizer(inr_model* m) {
  if (!m) return fail(INR_ERR_INVALID_ARG, "model is NULL");
  if (m->frozen) return fail(INR_ERR_STATE, "model is a frozen cache snapshot");
  CK(cudaSetDevice(m->device));
  CK(cudaDeviceSynchronize());
  inr_status s = init_state(m, m->cfg.seed, 0, true);
  if (s) return s;
  CK(cudaStreamSynchronize(0));
  return INR_OK;
}

static void purge_graphs(const inr_model* m);

extern "C" inr_status inr_destroy(inr_model* m) {
  if (!m) return INR_OK;
  purge_graphs(m);   // cached fit graphs holding this model's pointers
  cudaSetDevice(m->device);
  if ((m->host_resident || m->h16) && m->params) cudaFree(m->params);
  if (m->mesh) cudaFree(m->mesh);
  if (m->mem) cudaFree(m->mem);
  if (m->host_params) cudaFreeHost(m->host_params);
  if (m->h16) { if (m->host_resident) cudaFreeHost(m->h16); else cudaFree(m->h16); }
  delete m;
  return INR_OK;
}

extern "C" inr_status inr_param_count(const inr_model* m, int64_t* count) {
  if (!m || !count) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  *count = m->P;
  return INR_OK;
}

extern "C" inr_status inr_param_bytes(const inr_model* m, int64_t* bytes) {
  if (!m || !bytes) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  *bytes = m->P * (int64_t)sizeof(float);
  return INR_OK;
}

extern "C" inr_status inr_steps(const inr_model* m, int64_t* steps) {
  if (!m || !steps) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  *steps = m->steps;
  return INR_OK;
}

extern "C" void inr_fit_opts_default(inr_fit_opts* o) {
  if (!o) return;
  o->lambda = 0.5;
  o->boundary_batch = 0;
  o->lr0 = 1e-2;
  o->lr_decay = 0.8;
  o->lr_step = 500;
  o->beta1 = 0.9;
  o->beta2 = 0.999;
  o->eps = 1e-8;
  o->vmin = 0.0;
  o->vmax = 1.0;
  for (int c = 0; c < INR_MAX_CHANNELS; ++c) { o->vmin_c[c] = 0.0; o->vmax_c[c] = 1.0; }
  o->target_psnr = 0.0;
  o->check_interval = 0;
  o->sparse_adam = 0;
  o->split_step = 1;
}

// Make sure device-resident parameters exist for a (possibly host-resident) model.
// Staging is done once, under a lock, and completes before `staged` is set (the
// stream is synchronized), so a later decode of the same snapshot on another
// stream never reads a half-written staging buffer.
static inr_status ensure_device_params(const inr_model* cm, cudaStream_t st) {
  inr_model* m = const_cast<inr_model*>(cm);
  if (!m->host_resident && !m->h16) return INR_OK;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (m->staged) return INR_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(st, &cs));
  if (cs != cudaStreamCaptureStatusNone)
    return fail(INR_ERR_STATE, "a host-resident or fp16 cache snapshot is first decoded inside a stream capture");
  if (!m->params) CK(cudaMalloc((void**)&m->params, (size_t)m->P_pad * 4));
  if (m->h16) {   // fp16-stored snapshot: widen into the fp32 staging buffer
    const __half* src = m->h16;
    void* tmp = nullptr;
    if (m->host_resident) {
      CK(cudaMallocAsync(&tmp, (size_t)m->P_pad * 2, st));
      CK(cudaMemcpyAsync(tmp, m->h16, (size_t)m->P_pad * 2, cudaMemcpyHostToDevice, st));
      src = (const __half*)tmp;
    }
    launch_convert_f16_f32(src, m->params, m->P_pad, st);
    CK_LAUNCH("convert_f16_f32");
    if (tmp) CK(cudaFreeAsync(tmp, st));
  } else {
    CK(cudaMemcpyAsync(m->params, m->host_params, (size_t)m->P_pad * 4, cudaMemcpyHostToDevice, st));
  }
  CK(cudaStreamSynchronize(st));
  m->staged = true;
  return INR_OK;
}

static ModelDev model_dev(const inr_model* m) {
  ModelDev d;
  memset(&d, 0, sizeof d);
  d.params = m->params;
  d.grads = m->grads;
  d.adam_m = m->adam_m;
  d.adam_v = m->adam_v;
  d.grads_fx = m->gfx;
  d.step_total = m->step_total;
  d.step_cur = m->step_cur;
  d.acc = m->acc;
  d.flag = m->flag;
  for (int k = 0; k < 3; ++k) {
    d.o[k] = (int)m->blk.origin[k];
    d.n[k] = m->blk.n[k];
    d.N[k] = (int)m->blk.global_dims[k];
  }
  d.block_id = m->block_id;
  d.nfaces = m->nfaces;
  for (int k = 0; k < 6; ++k) d.faces[k] = m->faces[k];
  if (m->mesh) {
    size_t off = 0;
    for (int k = 0; k < 3; ++k) {
      d.mesh[k] = m->mesh + off;
      off += (size_t)m->mesh_n[k];
      d.mesh_n[k] = m->mesh_n[k];
      d.plo[k] = m->plo[k];
      d.pspan[k] = m->pspan[k];
    }
  }
  for (int c = 0; c < kMaxD; ++c) {
    d.vmin[c] = m->vmin[c];
    d.vrange[c] = m->vmax[c] - m->vmin[c];
    d.inv_range[c] = m->vmax[c] > m->vmin[c] ? (float)(1.0 / ((double)m->vmax[c] - (double)m->vmin[c])) : 0.f;
  }
  return d;
}

static bool same_shape(const inr_config& a, const inr_config& b) {
  // (the seed may differ: each model draws its own Philox streams)
  return a.levels == b.levels && a.features == b.features && a.log2_table_size == b.log2_table_size &&
         a.base_resolution == b.base_resolution && a.per_level_scale == b.per_level_scale &&
         a.mlp_width == b.mlp_width && a.mlp_hidden_layers == b.mlp_hidden_layers && a.out_dim == b.out_dim &&
         a.mlp_bias == b.mlp_bias && a.precision == b.precision && a.reduction == b.reduction;
}

static inr_status validate_view(const inr_model* m, const inr_view* v) {
  if (!v || !v->base) return fail(INR_ERR_INVALID_ARG, "view is NULL");
  for (int d = 0; d < 3; ++d) {
    int64_t need_lo = m->blk.origin[d];
    int64_t need_hi = std::min<int64_t>(m->blk.origin[d] + m->blk.n[d], m->blk.global_dims[d] - 1);
    if (v->lo[d] > need_lo || v->lo[d] + v->dims[d] - 1 < need_hi)
      return fail(INR_ERR_INVALID_ARG, "view does not cover nodes [o, min(o+n, N-1)] on axis %d", d);
  }
  return INR_OK;
}

// Keep stream-ordered workspace allocations in the device's pool between calls
// (the default release threshold of 0 unmaps them at every synchronization).
static void keep_pool(int device) {
  static bool done[64] = {false};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[device] = true;
}

// One-step CUDA graphs of recent fit calls.  A graph's kernels read everything by
// value from their launch parameters (GroupArgs, FitScalars, AdamScalars, the
// workspace pointers), so a later call whose parameter bytes are identical replays
// the cached graph instead of capturing and instantiating a new one (the host
// cost of a capture is ~1 ms, a step ~1.3 ms).  Each entry owns its workspace.
// Entries are dropped by inr_destroy (a model's memory may be reused).
struct FitGraph {
  std::vector<unsigned char> key;
  cudaGraphExec_t exec = nullptr;
  cudaGraphExec_t exec_first = nullptr;   // split step: the first step of a call (no deferred Adam)
  void* ws = nullptr;
  int device = -1;
  unsigned long long last_use = 0;
  int users = 0;                  // fit calls replaying it right now (never evicted then)
};
static std::mutex g_graph_mu;
static std::list<FitGraph> g_graphs;
static unsigned long long g_graph_clock = 0;
constexpr size_t kGraphCache = 4;

// ---- split fit step (one launch group of >= 2 models): the group's two halves A and B
// run the pipeline in turn, and each half's Adam (HBM-bound) runs on a second stream
// beside the other half's tensor-core MLP (latency-bound), on the SMs' spare registers
// and warps, its tail beside the start of that half's scatter:
//   fwd_A {mlp_A bwd_A | adam_B(s-1)} fwd_B {mlp_B bwd_B | adam_A(s)}   (prep_X beside fwd_X)
// Half B's Adam of the last step is flushed at the end of the call.  Per model the
// order of operations is the unsplit step's (blocks are independent).
static GroupArgs sub_group(const GroupArgs& g, int j0, int n) {
  GroupArgs s;
  memset(&s, 0, sizeof s);
  s.net = g.net;
  s.nmodels = n;
  for (int j = 0; j < n; ++j) s.md[j] = g.md[j0 + j];
  return s;
}

static LmWorkspace sub_workspace(const LmWorkspace& w, const NetDesc& net, int j0) {
  LmWorkspace s = w;
  s.samples += (size_t)j0 * w.Bs;
  s.featimg += (size_t)j0 * (w.Bs / 128) * w.geom.tile_bytes;
  s.dfeat += (size_t)j0 * w.Bs * net.LF;
  s.wimg += (size_t)j0 * w.img_bytes;
  if (s.targets) s.targets += (size_t)j0 * w.Bs;
  return s;
}

// the side stream and fork / join events of the split step (for a capture, or for one
// call's live steps)
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t ev[8] = {};
  SideStream() {
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  }
  ~SideStream() {
    for (auto& e : ev) cudaEventDestroy(e);
    cudaStreamDestroy(s);
  }
};

static void free_graph(FitGraph& f) {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(f.device);
  if (f.exec) cudaGraphExecDestroy(f.exec);
  if (f.exec_first) cudaGraphExecDestroy(f.exec_first);
  if (f.ws) cudaFree(f.ws);
  cudaSetDevice(cur);
  f.exec = nullptr;
  f.exec_first = nullptr;
  f.ws = nullptr;
}

// Drop the cached graphs whose launch parameters hold this model's parameter pointer.
static void purge_graphs(const inr_model* m) {
  std::lock_guard<std::mutex> lock(g_graph_mu);
  const void* p = m->params;
  for (auto it = g_graphs.begin(); it != g_graphs.end();) {
    bool hit = false;
    for (size_t i = 0; !hit && i + sizeof p <= it->key.size(); ++i) hit = !memcmp(&it->key[i], &p, sizeof p);
    if (hit && it->users == 0) {
      free_graph(*it);
      it = g_graphs.erase(it);
    } else {
      ++it;
    }
  }
}

static inr_status fit_impl(inr_model* const* models, const inr_view* views, int32_t nmodels, int32_t steps,
                           int32_t batch, const inr_fit_opts* opts, inr_fit_report* out, cudaStream_t st) {
  if (!models || !views || nmodels < 1) return fail(INR_ERR_INVALID_ARG, "models/views missing");
  if (!opts) return fail(INR_ERR_INVALID_ARG, "opts is NULL");
  if (steps < 1) return fail(INR_ERR_INVALID_ARG, "steps must be >= 1");
  if (batch < 1) return fail(INR_ERR_INVALID_ARG, "batch must be >= 1");
  if (!(opts->lambda >= 0.0 && opts->lambda <= 1.0)) return fail(INR_ERR_INVALID_ARG, "lambda must be in [0,1]");
  if (opts->boundary_batch < 0) return fail(INR_ERR_INVALID_ARG, "boundary_batch must be >= 0");
  if (opts->lr_step < 1) return fail(INR_ERR_INVALID_ARG, "lr_step must be >= 1");
  if (!models || !models[0]) return fail(INR_ERR_INVALID_ARG, "model 0 is NULL");
  const int D = models[0]->net.D;
  // the per-channel ranges of this call: vmin/vmax for scalar fields, vmin_c/vmax_c for vector fields
  double lo[kMaxD], hi[kMaxD];
  for (int c = 0; c < D; ++c) {
    lo[c] = D == 1 ? opts->vmin : opts->vmin_c[c];
    hi[c] = D == 1 ? opts->vmax : opts->vmax_c[c];
    if (!(hi[c] >= lo[c])) return fail(INR_ERR_INVALID_ARG, "vmax < vmin (channel %d)", c);
  }
  bool all_constant = true;
  for (int c = 0; c < D; ++c) all_constant &= hi[c] == lo[c];
  for (int i = 0; i < nmodels; ++i) {
    if (!models[i]) return fail(INR_ERR_INVALID_ARG, "model %d is NULL", i);
    if (models[i]->frozen) return fail(INR_ERR_STATE, "model %d is a frozen cache snapshot", i);
    if (models[i]->device != models[0]->device || !same_shape(models[i]->cfg, models[0]->cfg))
      return fail(INR_ERR_INVALID_ARG, "all models of a group must share device and config");
    inr_status s = validate_view(models[i], &views[i]);
    if (s) return s;
    if (std::max(1, views[i].channels) != D)
      return fail(INR_ERR_INVALID_ARG, "view %d has %d channels, the model outputs %d", i, views[i].channels, D);
  }
  const inr_model* m0 = models[0];
  CK(cudaSetDevice(m0->device));
  keep_pool(m0->device);
  const bool tc = m0->cfg.precision == INR_PREC_FP16_MLP;
  if (tc && !tc_supported(m0->net)) return fail(INR_ERR_UNSUPPORTED, "configuration not supported by the tcgen05 MLP");

  FitScalars fs;
  memset(&fs, 0, sizeof fs);   // (the parameter bytes key the graph cache)
  fs.B_u = batch;
  fs.B_b = opts->boundary_batch;
  fs.lambda = (float)opts->lambda;
  fs.det = m0->cfg.reduction == INR_REDUCE_DETERMINISTIC;
  AdamScalars as;
  memset(&as, 0, sizeof as);
  as.lr0 = opts->lr0;
  as.lr_decay = opts->lr_decay;
  as.lr_step = opts->lr_step;
  as.beta1 = opts->beta1;
  as.beta2 = opts->beta2;
  as.b1 = (float)opts->beta1;
  as.b2 = (float)opts->beta2;
  as.ob1 = (float)(1.0 - opts->beta1);
  as.ob2 = (float)(1.0 - opts->beta2);
  as.eps = (float)opts->eps;
  as.sparse = opts->sparse_adam != 0;
  as.table_end = m0->net.w_off[0];   // tables: internal parameters [0, w_off[0])

  for (int i = 0; i < nmodels; ++i) {
    for (int c = 0; c < D; ++c) {
      models[i]->vmin[c] = (float)lo[c];
      models[i]->vmax[c] = (float)hi[c];
    }
    const int bb = models[i]->nfaces > 0 ? opts->boundary_batch : 0;
    models[i]->last_inv_u = 1.0 / ((double)batch * D);
    models[i]->last_inv_b = bb > 0 ? 1.0 / ((double)bb * D) : 0.0;
  }
  // the models still training, in chunks of <= 64 per fused launch; with PSNR-target
  // stopping a model leaves the group at the first check where it reaches the target
  // (each model stops exactly as if fitted alone; blocks are independent)
  std::vector<int> active(nmodels);
  for (int i = 0; i < nmodels; ++i) active[i] = i;
  std::vector<GroupArgs> groups;
  int nchunks = 0;
  auto build_groups = [&]() {
    nchunks = ((int)active.size() + kMaxGroup - 1) / kMaxGroup;
    groups.assign(nchunks, GroupArgs());
    for (int c = 0; c < nchunks; ++c) {
      GroupArgs& g = groups[c];
      memset(&g, 0, sizeof g);
      g.net = m0->net;
      g.nmodels = std::min(kMaxGroup, (int)active.size() - c * kMaxGroup);
      for (int j = 0; j < g.nmodels; ++j) {
        const int i = active[c * kMaxGroup + j];
        const inr_model* m = models[i];
        const inr_view& v = views[i];
        ModelDev& d = g.md[j];
        d = model_dev(m);
        d.vbase = v.base;
        uint32_t k0;
        philox_key(m->cfg.seed, 1, d.k0, d.k1u);
        philox_key(m->cfg.seed, 2, k0, d.k1b);
        for (int k = 0; k < 3; ++k) { d.vlo[k] = v.lo[k]; d.vstride[k] = v.stride[k]; }
      }
    }
  };
  build_groups();
  const bool probing = out && opts->target_psnr > 0.0 && opts->check_interval > 0;
  const int launches_per_step = (tc ? 5 : 3) * nchunks;   // (graphs only without probing: fixed groups)
  // CUDA graphs (launch-gap free): without probing, one step is captured once and
  // replayed per step, and the instantiated graph is cached across calls (above);
  // while profiling, the whole loop (with its event records) is captured once, so
  // per-kernel timings come from the same graph execution.
  const bool graphs = st != nullptr && !probing;
  const bool whole = graphs && g_prof_on && steps >= 2;
  const bool cached = graphs && !whole;
  // The split step pays where a half's Adam and the other half's MLP take comparable times
  // (measured: Adam ~6 GB/ms, the MLP ~55 ns per 128-sample tile at one CTA per SM); when
  // either dominates, the halves' extra kernel tails cost more than the overlap saves and
  // the one-pipeline step is faster (cfg5's T = 2^22: 45.2 vs 41.8 ms per step; cfg2 at
  // T = 2^15: 0.80 vs 0.70 ms).
  auto split_ok = [&](int nm) {
    const double adam_ms = 28.0 * (double)m0->net.nparams * (nm / 2) / 6.0e9;
    const double mlp_ms = 55e-6 * ((batch + opts->boundary_batch + 127) / 128) * (nm / 2);
    return tc && nchunks == 1 && nm >= 2 && opts->split_step != 0 && adam_ms <= 4.0 * mlp_ms &&
           mlp_ms <= 4.0 * adam_ms;
  };
  const bool split = graphs && split_ok(nmodels);
  // without graphs (PSNR-target stopping, the legacy stream) the same split step is enqueued
  // live; half B's deferred Adam is flushed before every probe (which reads the parameters)
  bool live = !graphs && split_ok(nmodels);
  const int Bs = (batch + opts->boundary_batch + 127) / 128 * 128;
  const int per = std::min(nmodels, kMaxGroup);
  const size_t ws_bytes = tc ? lm_workspace_bytes(m0->net, per, Bs) : 0;
  std::vector<unsigned char> key;
  if (cached) {
    auto put = [&](const void* p, size_t n) {
      const unsigned char* b = (const unsigned char*)p;
      key.insert(key.end(), b, b + n);
    };
    int hdr[6] = {m0->device, (int)tc, Bs, nchunks, (int)ws_bytes, (int)split};
    put(hdr, sizeof hdr);
    put(&fs, sizeof fs);
    put(&as, sizeof as);
    for (int c = 0; c < nchunks; ++c) put(&groups[c], sizeof(GroupArgs));
  }
  // fp16 path: level-major pipeline with a workspace (per call, stream-ordered; or the
  // cached graph's own)
  void* ws_mem = nullptr;        // per-call workspace (freed at the end of the call)
  void* ws_base = nullptr;
  LmWorkspace ws{};
  cudaGraphExec_t exec = nullptr;
  FitGraph* entry = nullptr;
  std::unique_lock<std::mutex> glock(g_graph_mu, std::defer_lock);
  if (cached) {
    glock.lock();
    for (auto& f : g_graphs)
      if (f.device == m0->device && f.key == key) { entry = &f; break; }
    if (entry) {
      exec = entry->exec;
      ws_base = entry->ws;
      entry->last_use = ++g_graph_clock;
      ++entry->users;
    }
  }
  if (tc && !ws_base) {
    if (cached) CK(cudaMalloc(&ws_base, ws_bytes));
    else { CK(cudaMallocAsync(&ws_mem, ws_bytes, st)); ws_base = ws_mem; }
  }
  if (tc) ws = lm_workspace(ws_base, m0->net, per, Bs);
  GroupArgs gh[2];
  LmWorkspace wh[2];
  auto set_halves = [&]() {
    const int h = groups[0].nmodels / 2;
    gh[0] = sub_group(groups[0], 0, h);
    gh[1] = sub_group(groups[0], h, groups[0].nmodels - h);
    wh[0] = sub_workspace(ws, m0->net, 0);
    wh[1] = sub_workspace(ws, m0->net, h);
  };
  if (split || live) set_halves();
  std::unique_ptr<SideStream> live_side(live ? new SideStream() : nullptr);
  bool live_first = true;   // no deferred Adam pending
  // beside each other: one MLP CTA (256 threads, half the registers) and one TMA-fed Adam
  // CTA (512 threads, 96 KB of operands in flight) per SM
  // (the device's SM count: 148 on B200)
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, m0->device);
  const int kSplitMlpCtas = nsm, kSplitAdamCtas = nsm;
  // fork / join between the launching stream and the side stream (inside a capture)
  auto fork = [](cudaStream_t from, cudaStream_t to, cudaEvent_t e) {
    cudaEventRecord(e, from);
    cudaStreamWaitEvent(to, e, 0);
  };
  auto enqueue_split = [&](cudaStream_t s, const SideStream& side, bool first) {
    for (int hf = 0; hf < 2; ++hf) {
      const GroupArgs& g = gh[hf];
      const LmWorkspace& w = wh[hf];
      const GroupArgs& o = gh[hf ^ 1];
      // this half's weight image on the side stream beside its encode: it needs this half's
      // Adam of the previous step, which the side stream ran before it
      fork(s, side.s, side.ev[4 * hf]);
      { ProfScope p(PK_PREP, side.s); launch_prep_image(g, g.nmodels, w.wimg, side.s); }
      cudaEventRecord(side.ev[4 * hf + 1], side.s);
      { ProfScope p(PK_ENCODE_FWD, s); launch_encode_fwd(g, g.nmodels, fs, w, s); }
      cudaStreamWaitEvent(s, side.ev[4 * hf + 1], 0);
      const bool side_adam = hf == 1 || !first;   // the other half's Adam (of the previous step for B)
      if (side_adam) {
        fork(s, side.s, side.ev[4 * hf + 2]);
        { ProfScope p(PK_ADAM, side.s); launch_adam(o, o.nmodels, as, side.s, kSplitAdamCtas); }
      }
      { ProfScope p(PK_MLP_TC, s);
        launch_mlp_tc(g, g.nmodels, fs, w.featimg, w.wimg, w.samples, w.targets, w.dfeat, w.Bs, s,
                      side_adam ? kSplitMlpCtas : 0); }
      { ProfScope p(PK_ENCODE_BWD, s); launch_encode_bwd(g, g.nmodels, fs, w, s); }
      // (joined after the scatter: the Adam's tail may also run beside this half's scatter)
      if (side_adam) fork(side.s, s, side.ev[4 * hf + 3]);
    }
  };
  auto flush_split = [&](cudaStream_t s) {   // half B's Adam of the last step
    ProfScope p(PK_ADAM, s);
    launch_adam(gh[1], gh[1].nmodels, as, s);
  };
  auto enqueue_step = [&](cudaStream_t s, const SideStream* side) {
    for (int c = 0; c < nchunks; ++c) {
      const GroupArgs& g = groups[c];
      if (tc) {
        // (encode_fwd zeroes the gradient and the loss sums and draws the step's samples with
        // step_total, encode_bwd advances the step counters for Adam: no step_begin launch;
        // captured, the weight image is prepared on the side stream beside encode_fwd)
        if (side) {
          fork(s, side->s, side->ev[0]);
          { ProfScope p(PK_PREP, side->s); launch_prep_image(g, g.nmodels, ws.wimg, side->s); }
          cudaEventRecord(side->ev[1], side->s);
        }
        { ProfScope p(PK_ENCODE_FWD, s); launch_encode_fwd(g, g.nmodels, fs, ws, s); }
        if (side) cudaStreamWaitEvent(s, side->ev[1], 0);
        else { ProfScope p(PK_PREP, s); launch_prep_image(g, g.nmodels, ws.wimg, s); }
        { ProfScope p(PK_MLP_TC, s); launch_mlp_tc(g, g.nmodels, fs, ws.featimg, ws.wimg, ws.samples, ws.targets, ws.dfeat, ws.Bs, s); }
        { ProfScope p(PK_ENCODE_BWD, s); launch_encode_bwd(g, g.nmodels, fs, ws, s); }
        { ProfScope p(PK_ADAM, s); launch_adam(g, g.nmodels, as, s); }
      } else {
        { ProfScope p(PK_STEP_BEGIN, s); launch_step_begin(g, g.nmodels, 0, s); }
        { ProfScope p(PK_FIT_FP32, s); launch_fit_simt(g, g.nmodels, fs, s); }
        { ProfScope p(PK_ADAM, s); launch_adam(g, g.nmodels, as, s); }
      }
    }
  };
  struct WsFree {
    void*& p; cudaStream_t s;
    ~WsFree() { if (p) cudaFreeAsync(p, s); }
  } ws_free{ws_mem, st};
  cudaGraphExec_t exec_first = entry ? entry->exec_first : nullptr;
  if (graphs && !exec) {
    // variant 0: the step (steady split step); variant 1: the split step of a call's first step
    std::unique_ptr<SideStream> side(tc ? new SideStream() : nullptr);
    for (int variant = 0; variant < (split && !whole ? 2 : 1); ++variant) {
      cudaGraph_t graph;
      {
        cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) { if (cached) cudaFree(ws_base); return cuda_fail(e, "cudaStreamBeginCapture"); }
      }
      long long before = g_launches.load();
      for (int s = 0; s < (whole ? steps : 1); ++s) {
        if (split) enqueue_split(st, *side, whole ? s == 0 : variant == 1);
        else enqueue_step(st, side.get());
      }
      if (split && whole) flush_split(st);
      g_launches.store(before);  // captured launches are counted per replay below
      cudaError_t e = cudaStreamEndCapture(st, &graph);
      if (e != cudaSuccess) { if (cached) cudaFree(ws_base); return cuda_fail(e, "cudaStreamEndCapture"); }
      cudaGraphExec_t x = nullptr;
      e = cudaGraphInstantiate(&x, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) { if (cached) cudaFree(ws_base); return cuda_fail(e, "cudaGraphInstantiate"); }
      (variant == 0 ? exec : exec_first) = x;
    }
    if (cached) {   // insert, evicting the least recently used idle entry beyond kGraphCache
      if (g_graphs.size() >= kGraphCache) {
        auto lru = g_graphs.end();
        for (auto it = g_graphs.begin(); it != g_graphs.end(); ++it)
          if (it->users == 0 && (lru == g_graphs.end() || it->last_use < lru->last_use)) lru = it;
        if (lru != g_graphs.end()) {
          free_graph(*lru);
          g_graphs.erase(lru);
        }
      }
      FitGraph f;
      f.key = key;
      f.exec = exec;
      f.exec_first = exec_first;
      f.ws = ws_base;
      f.device = m0->device;
      f.last_use = ++g_graph_clock;
      f.users = 1;
      g_graphs.push_back(std::move(f));
      entry = &g_graphs.back();
    }
  }
  if (glock.owns_lock()) glock.unlock();
  struct Release {   // the entry may be evicted again once this call is done with it
    FitGraph*& e;
    ~Release() {
      if (!e) return;
      std::lock_guard<std::mutex> lock(g_graph_mu);
      --e->users;
    }
  } release{entry};
  int taken = 0;
  std::vector<double> psnr(nmodels, 0.0);
  std::vector<int> reached(nmodels, 0), steps_of(nmodels, -1);
  for (int s = 0; s < steps; ++s) {
    if (exec) {
      if (whole && s > 0) { taken = s + 1; continue; }
      cudaError_t e = cudaGraphLaunch(s == 0 && exec_first ? exec_first : exec, st);
      if (e != cudaSuccess) {
        if (!cached) cudaGraphExecDestroy(exec);
        return cuda_fail(e, "cudaGraphLaunch");
      }
      // (split: 10 launches per step, 9 in a call's first, + the final Adam flush)
      count_launch(split ? (whole ? 10ll * steps : (s == 0 ? 9 : 10)) : (long long)launches_per_step * (whole ? steps : 1));
    } else if (live) {
      enqueue_split(st, *live_side, live_first);
      live_first = false;
      CK_LAUNCH("fit step");
    } else {
      enqueue_step(st, nullptr);
      CK_LAUNCH("fit step");
    }
    taken = s + 1;
    if (probing && taken % opts->check_interval == 0) {
      if (live && !live_first) {
        flush_split(st);
        live_first = true;
      }
      for (int c = 0; c < nchunks; ++c)
        for (int j = 0; j < groups[c].nmodels; ++j)
          CK(cudaMemsetAsync(groups[c].md[j].acc + 2, 0, sizeof(double), st));
      for (int c = 0; c < nchunks; ++c) { ProfScope p(PK_PROBE, st); launch_probe(groups[c], groups[c].nmodels, st); }
      CK_LAUNCH("probe");
      CK(cudaStreamSynchronize(st));
      std::vector<int> still;
      for (int i : active) {
        double sse = 0;
        CK(cudaMemcpy(&sse, models[i]->acc + 2, sizeof sse, cudaMemcpyDeviceToHost));
        double mse = sse / (32768.0 * D);
        psnr[i] = mse <= 0 ? 200.0 : std::min(200.0, -10.0 * std::log10(mse));
        reached[i] = psnr[i] >= opts->target_psnr;
        if (reached[i]) steps_of[i] = taken;
        else still.push_back(i);
      }
      if (still.empty()) break;
      if (still.size() != active.size()) {   // the converged models leave the group
        active.swap(still);
        build_groups();
        live = live && split_ok((int)active.size());
        if (live) set_halves();
      }
    }
  }
  if (split && !whole) flush_split(st);   // (counts its own launch)
  if (live && !live_first) flush_split(st);
  if (exec && !cached) cudaGraphExecDestroy(exec);
  if (exec_first && !cached) cudaGraphExecDestroy(exec_first);
  for (int i = 0; i < nmodels; ++i) {
    if (steps_of[i] < 0) steps_of[i] = taken;
    models[i]->steps += steps_of[i];
  }
  if (!out) return INR_OK;
  CK(cudaStreamSynchronize(st));
  bool nonfinite = false;
  for (int i = 0; i < nmodels; ++i) {
    const inr_model* m = models[i];
    // one copy per model: acc[0..2] (doubles at +16) and the flag (int at +48) are adjacent
    unsigned char tail[40];
    CK(cudaMemcpy(tail, m->acc, sizeof tail, cudaMemcpyDeviceToHost));
    double acc[2];
    int flag = 0;
    memcpy(acc, tail, sizeof acc);
    memcpy(&flag, tail + 32, sizeof flag);
    inr_fit_report& r = out[i];
    r.steps_taken = steps_of[i];
    r.reached_target = reached[i];
    r.constant_field = all_constant;
    int bb = m->nfaces > 0 ? opts->boundary_batch : 0;
    r.loss_uniform = acc[0] / ((double)batch * D);
    r.loss_boundary = bb > 0 ? acc[1] / ((double)bb * D) : 0.0;
    r.probe_psnr = psnr[i];
    if (flag || !std::isfinite(r.loss_uniform) || !std::isfinite(r.loss_boundary)) nonfinite = true;
  }
  if (nonfinite) return fail(INR_ERR_NONFINITE, "non-finite loss or parameter after %d steps", taken);
  if (all_constant) g_err = "warning: constant field (vmax == vmin), targets are 0";
  return INR_OK;
}

extern "C" inr_status inr_fit_losses(inr_model* const* models, int32_t nmodels, double* out, cudaStream_t st) {
  if (!models || !out || nmodels < 1) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  for (int c0 = 0; c0 < nmodels; c0 += kMaxGroup) {
    LossReportArgs a;
    memset(&a, 0, sizeof a);
    a.n = std::min(kMaxGroup, nmodels - c0);
    for (int j = 0; j < a.n; ++j) {
      const inr_model* m = models[c0 + j];
      if (!m || m->frozen) return fail(INR_ERR_INVALID_ARG, "model %d is NULL or frozen", c0 + j);
      a.acc[j] = m->acc;
      a.flag[j] = m->flag;
      a.inv_u[j] = m->last_inv_u;
      a.inv_b[j] = m->last_inv_b;
    }
    CK(cudaSetDevice(models[c0]->device));
    launch_loss_report(a, out + 3 * (size_t)c0, st);
  }
  CK_LAUNCH("loss report");
  return INR_OK;
}

extern "C" inr_status inr_fit(inr_model* m, const inr_view* v, int32_t steps, int32_t batch,
                              const inr_fit_opts* opts, inr_fit_report* out, cudaStream_t st) {
  if (!m) return fail(INR_ERR_INVALID_ARG, "model is NULL");
  return fit_impl(&m, v, 1, steps, batch, opts, out, st);
}

extern "C" inr_status inr_fit_group(inr_model* const* models, const inr_view* views, int32_t nmodels,
                                    int32_t steps, int32_t batch, const inr_fit_opts* opts, inr_fit_report* out,
                                    cudaStream_t st) {
  return fit_impl(models, views, nmodels, steps, batch, opts, out, st);
}

// ------------------------------------------------------------------ decode
extern "C" inr_status inr_decode_grid_part(const inr_model* m, const int32_t res[3], const int32_t count[3],
                                           float* out, const int64_t* out_stride, const float* ref, double* sse_dev,
                                           cudaStream_t st) {
  if (!m || !res || !out) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  for (int d = 0; d < 3; ++d) {
    if (res[d] < 1 || res[d] > (1 << 20)) return fail(INR_ERR_INVALID_ARG, "res must be in 1..2^20");
    if (count && (count[d] < 1 || count[d] > res[d])) return fail(INR_ERR_INVALID_ARG, "count must be in 1..res");
  }
  if (ref && !sse_dev) return fail(INR_ERR_INVALID_ARG, "ref given without sse_dev");
  CK(cudaSetDevice(m->device));
  inr_status s = ensure_device_params(m, st);
  if (s) return s;
  long long os[3];
  if (out_stride) { for (int d = 0; d < 3; ++d) os[d] = out_stride[d]; }
  else {
    const long long D = m->net.D;
    os[0] = D; os[1] = D * res[0]; os[2] = D * res[0] * res[1];
  }
  int r[3] = {res[0], res[1], res[2]};
  int c[3] = {count ? count[0] : res[0], count ? count[1] : res[1], count ? count[2] : res[2]};
  if (m->mesh)
    for (int d = 0; d < 3; ++d)
      if (r[d] != m->blk.n[d] || c[d] > m->mesh_n[d])
        return fail(INR_ERR_INVALID_ARG, "a rectilinear model decodes its nodes: res = n, count <= its node count");
  ModelDev md = model_dev(m);
  {
    ProfScope p(PK_DECODE_GRID, st);
    if (m->cfg.precision == INR_PREC_FP16_MLP)
      launch_decode_grid_tc(m->net, md, r, c, out, os, ref, ref ? sse_dev : nullptr, st);
    else
      launch_decode_grid_simt(m->net, md, r, c, out, os, ref, ref ? sse_dev : nullptr, st);
  }
  CK_LAUNCH("decode_grid");
  return INR_OK;
}

extern "C" inr_status inr_decode_grid(const inr_model* m, const int32_t res[3], float* out,
                                      const int64_t* out_stride, const float* ref, double* sse_dev,
                                      cudaStream_t st) {
  return inr_decode_grid_part(m, res, nullptr, out, out_stride, ref, sse_dev, st);
}

// One chunk of <= kMaxGroup models of a decode group: queries routed to blocks of
// the chunk are decoded, those of the group's other chunks (slot -2) are left
// untouched, those of blocks no model holds get NaN.
static inr_status decode_chunk(const inr_model* const* models, int32_t nmodels, int32_t c0, int32_t c1,
                               const float* xyz, int64_t q, float* out, int* dflag, cudaStream_t st) {
  const inr_model* m0 = models[0];
  QueryArgs* qa = new QueryArgs();
  memset(qa, 0, sizeof *qa);
  qa->net = m0->net;
  long long nb = 1;
  for (int d = 0; d < 3; ++d) {
    qa->n[d] = m0->blk.n[d];
    qa->N[d] = (int)m0->blk.global_dims[d];
    qa->B[d] = (int)((m0->blk.global_dims[d] + m0->blk.n[d] - 1) / m0->blk.n[d]);
    nb *= qa->B[d];
  }
  if (nb > kMaxRouteBlocks) { delete qa; return fail(INR_ERR_UNSUPPORTED, "at most %d blocks in a volume", kMaxRouteBlocks); }
  qa->nblocks = (int)nb;
  for (long long b = 0; b < nb; ++b) qa->slot_of_block[b] = -1;
  for (int i = 0; i < nmodels; ++i) {
    const inr_model* m = models[i];
    if (!m || !same_shape(m->cfg, m0->cfg) || m->device != m0->device) {
      delete qa;
      return fail(INR_ERR_INVALID_ARG, "decode group models must share config and device");
    }
    for (int d = 0; d < 3; ++d)
      if (m->blk.n[d] != m0->blk.n[d] || m->blk.global_dims[d] != m0->blk.global_dims[d]) {
        delete qa;
        return fail(INR_ERR_INVALID_ARG, "decode group models must tile one volume");
      }
    if (m->block_id >= (uint32_t)nb) { delete qa; return fail(INR_ERR_INVALID_ARG, "block id outside the volume"); }
    if (i < c0 || i >= c1) {
      qa->slot_of_block[m->block_id] = -2;
      continue;
    }
    inr_status s = ensure_device_params(m, st);
    if (s) { delete qa; return s; }
    qa->md[i - c0] = model_dev(m);
    qa->slot_of_block[m->block_id] = (int16_t)(i - c0);
  }
  const int nm = c1 - c0;
  qa->nmodels = nm;
  if (q > 0 && m0->cfg.precision == INR_PREC_FP16_MLP) {
    // tensor-core path: bucket the queries by block, then 128-query tiles of one block each
    void* ws = nullptr;
    cudaError_t e = cudaMallocAsync(&ws, query_workspace_bytes(q, nm), st);
    if (e != cudaSuccess) { delete qa; return cuda_fail(e, "query workspace"); }
    QueryBuckets qb;
    launch_query_buckets(*qa, xyz, q, out, dflag, ws, qb, st);
    GroupArgs* g = new GroupArgs();
    g->net = qa->net;
    g->nmodels = nm;
    for (int i = 0; i < nm; ++i) g->md[i] = qa->md[i];
    { ProfScope p(PK_DECODE_QUERY, st); launch_decode_query_tc(*g, xyz, q, out, qb, st); }
    delete g;
    cudaFreeAsync(ws, st);
  } else if (q > 0) {
    ProfScope p(PK_DECODE_QUERY, st);
    launch_decode_query_simt(*qa, xyz, q, out, dflag, st);
  }
  delete qa;
  return INR_OK;
}

static inr_status decode_group_impl(const inr_model* const* models, int32_t nmodels, const float* xyz, int64_t q,
                                    float* out, int32_t strict, cudaStream_t st) {
  if (!models || nmodels < 1 || (q > 0 && (!xyz || !out))) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  if (q < 0) return fail(INR_ERR_INVALID_ARG, "q must be >= 0");
  const inr_model* m0 = models[0];
  if (!m0) return fail(INR_ERR_INVALID_ARG, "model 0 is NULL");
  CK(cudaSetDevice(m0->device));
  keep_pool(m0->device);
  int* dflag = nullptr;
  if (strict) {
    cudaError_t e = cudaMallocAsync((void**)&dflag, sizeof(int), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(dflag, 0, sizeof(int), st);
    if (e != cudaSuccess) return cuda_fail(e, "strict flag");
  }
  // groups of more than kMaxGroup models: one routed pass per chunk of models
  for (int c0 = 0; c0 < nmodels; c0 += kMaxGroup) {
    inr_status s = decode_chunk(models, nmodels, c0, std::min(nmodels, c0 + kMaxGroup), xyz, q, out, dflag, st);
    if (s) { if (dflag) cudaFreeAsync(dflag, st); return s; }
  }
  CK_LAUNCH("decode_query");
  if (strict) {
    int h = 0;
    CK(cudaMemcpyAsync(&h, dflag, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    cudaFreeAsync(dflag, st);
    if (h) return fail(INR_ERR_DOMAIN, "a query coordinate lies outside the global domain");
  }
  return INR_OK;
}

extern "C" inr_status inr_decode(const inr_model* m, const float* xyz, int64_t q, float* out, int32_t strict,
                                 cudaStream_t st) {
  if (!m) return fail(INR_ERR_INVALID_ARG, "model is NULL");
  return decode_group_impl(&m, 1, xyz, q, out, strict, st);
}

extern "C" inr_status inr_decode_group(const inr_model* const* models, int32_t nmodels, const float* xyz, int64_t q,
                                       float* out, int32_t strict, cudaStream_t st) {
  return decode_group_impl(models, nmodels, xyz, q, out, strict, st);
}

extern "C" inr_status inr_value_range(const inr_view* v, float* minmax, cudaStream_t st) {
  if (!v || !v->base || !minmax) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  for (int d = 0; d < 3; ++d)
    if (v->dims[d] < 1) return fail(INR_ERR_INVALID_ARG, "view dims must be >= 1");
  int dims[3] = {v->dims[0], v->dims[1], v->dims[2]};
  long long s[3] = {v->stride[0], v->stride[1], v->stride[2]};
  const int ch = std::max(1, v->channels);
  if (ch != 1 && ch != 3) return fail(INR_ERR_INVALID_ARG, "view channels must be 1 or 3");
  { ProfScope p(PK_RANGE, st); launch_range(v->base, dims, s, ch, minmax, st); }
  CK_LAUNCH("value_range");
  return INR_OK;
}

// ------------------------------------------------------------ parity surface
// internal (aligned) device layout <-> declared (contiguous) host layout
static inr_status copy_tensors(const NetDesc& net, float* dst, const float* src, cudaMemcpyKind kind) {
  for (int t = 0; t < net.ntensors; ++t) {
    if (kind == cudaMemcpyDeviceToHost)
      CK(cudaMemcpy(dst + net.t_decl[t], src + net.t_off[t], (size_t)net.t_len[t] * 4, kind));
    else if (kind == cudaMemcpyHostToDevice)
      CK(cudaMemcpy(dst + net.t_off[t], src + net.t_decl[t], (size_t)net.t_len[t] * 4, kind));
    else  // host internal -> host declared
      memcpy(dst + net.t_decl[t], src + net.t_off[t], (size_t)net.t_len[t] * 4);
  }
  return INR_OK;
}

static inr_status copy_out(const inr_model* m, const float* src, float* host, int64_t n) {
  if (!m || !host) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  if (n != m->P) return fail(INR_ERR_INVALID_ARG, "n must equal inr_param_count (%lld)", (long long)m->P);
  if (!src) return fail(INR_ERR_STATE, "this state does not exist on a frozen snapshot");
  CK(cudaSetDevice(m->device));
  CK(cudaDeviceSynchronize());
  return copy_tensors(m->net, host, src, cudaMemcpyDeviceToHost);
}

extern "C" inr_status inr_get_params(const inr_model* m, float* host, int64_t n) {
  if (m && m->h16 && !m->staged) {
    CK(cudaSetDevice(m->device));
    inr_status s = ensure_device_params(m, 0);
    if (s) return s;
  }
  if (m && m->host_resident && !m->staged) {
    if (!host || n != m->P) return fail(INR_ERR_INVALID_ARG, "bad arguments");
    return copy_tensors(m->net, host, m->host_params, cudaMemcpyHostToHost);
  }
  return copy_out(m, m ? m->params : nullptr, host, n);
}
extern "C" inr_status inr_get_grads(const inr_model* m, float* host, int64_t n) {
  return copy_out(m, m ? m->grads : nullptr, host, n);
}
extern "C" inr_status inr_get_adam_state(const inr_model* m, float* mh, float* vh, int64_t n) {
  inr_status s = copy_out(m, m ? m->adam_m : nullptr, mh, n);
  if (s) return s;
  return copy_out(m, m->adam_v, vh, n);
}
extern "C" inr_status inr_set_params(inr_model* m, const float* host, int64_t n) {
  if (!m || !host) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  if (m->frozen) return fail(INR_ERR_STATE, "model is a frozen cache snapshot");
  if (n != m->P) return fail(INR_ERR_INVALID_ARG, "n must equal inr_param_count (%lld)", (long long)m->P);
  CK(cudaSetDevice(m->device));
  CK(cudaDeviceSynchronize());
  return copy_tensors(m->net, m->params, host, cudaMemcpyHostToDevice);
}

extern "C" inr_status inr_debug_encode(const inr_model* m, const float* x01, int64_t q, uint32_t* idx, float* feat,
                                       cudaStream_t st) {
  if (!m || (q > 0 && !x01)) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  if (q <= 0) return INR_OK;
  CK(cudaSetDevice(m->device));
  inr_status s = ensure_device_params(m, st);
  if (s) return s;
  launch_debug_encode(m->net, m->params, x01, q, idx, feat, st);
  CK_LAUNCH("debug_encode");
  return INR_OK;
}

extern "C" inr_status inr_debug_forward(const inr_model* m, const float* x01, int64_t q, float* y, cudaStream_t st) {
  if (!m || (q > 0 && (!x01 || !y))) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  if (q <= 0) return INR_OK;
  CK(cudaSetDevice(m->device));
  inr_status s = ensure_device_params(m, st);
  if (s) return s;
  if (m->cfg.precision == INR_PREC_FP16_MLP) launch_debug_forward_tc(m->net, m->params, x01, q, y, st);
  else launch_debug_forward_simt(m->net, m->params, x01, q, y, st);
  CK_LAUNCH("debug_forward");
  return INR_OK;
}

// ------------------------------------------------------------------ cache
struct CacheSlot {
  int64_t timestep;
  std::vector<inr_model*> models;
  std::vector<const inr_model*> cmodels;
};

struct inr_cache {
  int capacity;
  bool host_resident;
  bool fp16;
  int device;
  std::deque<CacheSlot> slots;
  int64_t bytes = 0;
};

static void free_slot(inr_cache* c, CacheSlot& s) {
  for (inr_model* m : s.models) {
    c->bytes -= m->P * (c->fp16 ? 2 : 4);
    inr_destroy(m);
  }
  s.models.clear();
}

extern "C" inr_status cache_create(int32_t capacity, int32_t flags, int device, inr_cache** out) {
  if (!out) return fail(INR_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (capacity < 1) return fail(INR_ERR_INVALID_ARG, "capacity must be >= 1");
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(INR_ERR_INVALID_ARG, "device %d out of range", device);
  inr_cache* c = new inr_cache();
  c->capacity = capacity;
  if (flags & ~(CACHE_HOST_RESIDENT | CACHE_FP16)) { delete c; return fail(INR_ERR_INVALID_ARG, "unknown cache flags"); }
  c->host_resident = (flags & CACHE_HOST_RESIDENT) != 0;
  c->fp16 = (flags & CACHE_FP16) != 0;
  c->device = device;
  *out = c;
  return INR_OK;
}

extern "C" inr_status cache_destroy(inr_cache* c) {
  if (!c) return INR_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (auto& s : c->slots) free_slot(c, s);
  delete c;
  return INR_OK;
}

extern "C" inr_status cache_evict(inr_cache* c, int64_t* evicted) {
  if (!c) return fail(INR_ERR_INVALID_ARG, "cache is NULL");
  if (c->slots.empty()) return fail(INR_ERR_STATE, "evict on an empty cache");
  CK(cudaSetDevice(c->device));
  CK(cudaDeviceSynchronize());  // snapshots may still be read by queued decodes
  if (evicted) *evicted = c->slots.front().timestep;
  free_slot(c, c->slots.front());
  c->slots.pop_front();
  return INR_OK;
}

extern "C" inr_status cache_insert(inr_cache* c, int64_t timestep, inr_model* const* blocks, int32_t nblocks,
                                   int64_t* evicted, cudaStream_t st) {
  if (!c || !blocks || nblocks < 1) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  if (!c->slots.empty() && timestep <= c->slots.back().timestep)
    return fail(INR_ERR_INVALID_ARG, "timesteps must be strictly increasing (last %lld)",
                (long long)c->slots.back().timestep);
  for (int i = 0; i < nblocks; ++i)
    if (!blocks[i] || blocks[i]->device != c->device) return fail(INR_ERR_INVALID_ARG, "block %d invalid", i);
  if (evicted) *evicted = -1;
  CK(cudaSetDevice(c->device));
  if ((int)c->slots.size() == c->capacity) {
    inr_status s = cache_evict(c, evicted);
    if (s) return s;
  }
  CacheSlot slot;
  slot.timestep = timestep;
  for (int i = 0; i < nblocks; ++i) {
    const inr_model* src = blocks[i];
    inr_model* m = new inr_model();
    m->cfg = src->cfg;
    m->blk = src->blk;
    m->device = src->device;
    m->net = src->net;
    m->block_id = src->block_id;
    m->nfaces = src->nfaces;
    memcpy(m->faces, src->faces, sizeof m->faces);
    memcpy(m->vmin, src->vmin, sizeof m->vmin);
    memcpy(m->vmax, src->vmax, sizeof m->vmax);
    if (src->mesh) {
      const double* sl[3] = {src->mesh, src->mesh + src->mesh_n[0], src->mesh + src->mesh_n[0] + src->mesh_n[1]};
      inr_status ms = set_mesh_slices(m, sl, src->mesh_n, true);
      if (ms) { delete m; for (auto* x : slot.models) inr_destroy(x); return ms; }
      memcpy(m->plo, src->plo, sizeof m->plo);
      memcpy(m->pspan, src->pspan, sizeof m->pspan);
    }
    m->steps = src->steps;
    m->frozen = true;
    inr_status s = alloc_model(m, true, c->host_resident || c->fp16);
    if (s) { inr_destroy(m); for (auto* x : slot.models) inr_destroy(x); return s; }
    m->host_resident = c->host_resident;
    m->staged = false;
    cudaError_t e = cudaSuccess;
    if (c->fp16) {
      // fp16 storage (2x compression ratio, NEXT-4): narrow on the device, then keep it there or in RAM
      void* dst = nullptr;
      if (c->host_resident) {
        e = cudaMallocHost(&dst, (size_t)m->P_pad * 2);
        m->h16 = (__half*)dst;
        void* tmp = nullptr;
        if (e == cudaSuccess) e = cudaMallocAsync(&tmp, (size_t)m->P_pad * 2, st);
        if (e == cudaSuccess) {
          launch_convert_f32_f16(src->params, (__half*)tmp, m->P_pad, st);
          e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(m->h16, tmp, (size_t)m->P_pad * 2, cudaMemcpyDeviceToHost, st);
        if (tmp) cudaFreeAsync(tmp, st);
      } else {
        e = cudaMalloc(&dst, (size_t)m->P_pad * 2);
        m->h16 = (__half*)dst;
        if (e == cudaSuccess) {
          launch_convert_f32_f16(src->params, m->h16, m->P_pad, st);
          e = cudaGetLastError();
        }
      }
    } else if (c->host_resident) {
      // "the learned neural network parameters are cached in system RAM"
      e = cudaMallocHost((void**)&m->host_params, (size_t)m->P_pad * 4);
      if (e == cudaSuccess) e = cudaMemcpyAsync(m->host_params, src->params, (size_t)m->P_pad * 4, cudaMemcpyDeviceToHost, st);
    } else {
      e = cudaMemcpyAsync(m->params, src->params, (size_t)m->P_pad * 4, cudaMemcpyDeviceToDevice, st);
    }
    if (e != cudaSuccess) { inr_destroy(m); for (auto* x : slot.models) inr_destroy(x); return cuda_fail(e, "cache copy"); }
    c->bytes += m->P * (c->fp16 ? 2 : 4);  // stored parameter bytes (declared count)
    slot.models.push_back(m);
    slot.cmodels.push_back(m);
  }
  if (c->host_resident) CK(cudaStreamSynchronize(st));
  c->slots.push_back(std::move(slot));
  return INR_OK;
}

extern "C" inr_status cache_size(const inr_cache* c, int32_t* n) {
  if (!c || !n) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  *n = (int32_t)c->slots.size();
  return INR_OK;
}

extern "C" inr_status cache_bytes(const inr_cache* c, int64_t* bytes) {
  if (!c || !bytes) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  *bytes = c->bytes;
  return INR_OK;
}

extern "C" inr_status cache_get(const inr_cache* c, int32_t i, int64_t* timestep, const inr_model* const** blocks,
                                int32_t* nblocks) {
  if (!c) return fail(INR_ERR_INVALID_ARG, "cache is NULL");
  if (i < 0 || i >= (int)c->slots.size()) return fail(INR_ERR_INVALID_ARG, "slot %d out of range", i);
  const CacheSlot& s = c->slots[i];
  if (timestep) *timestep = s.timestep;
  if (blocks) *blocks = s.cmodels.data();
  if (nblocks) *nblocks = (int32_t)s.cmodels.size();
  return INR_OK;
}

// ------------------------------------------------------------------ pathlines
// NEXT-2: RK4 over a window of decoded
// velocity grids, at most two resident, one launch per interval.
static inr_status check_path_args(const void* seeds, int32_t nseeds, double dt, int32_t max_steps, const void* vert,
                                  const void* counts, const void* reasons) {
  if (nseeds < 0) return fail(INR_ERR_INVALID_ARG, "nseeds must be >= 0");
  if (nseeds > 0 && (!seeds || !vert || !counts || !reasons)) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  if (!(dt > 0.0)) return fail(INR_ERR_INVALID_ARG, "dt must be > 0");
  if (max_steps < 0) return fail(INR_ERR_INVALID_ARG, "max_steps must be >= 0");
  return INR_OK;
}

extern "C" inr_status inr_trace_grids(const float* const* grids, const double* times, int32_t ngrids,
                                      const int64_t dims[3], double sign, const double* seeds, int32_t nseeds,
                                      double dt, int32_t max_steps, double* vertices, int32_t* counts,
                                      int32_t* reasons, cudaStream_t st) {
  if (!grids || !times || !dims) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  if (ngrids < 2) return fail(INR_ERR_INVALID_ARG, "a pathline window needs at least two grids");
  inr_status s = check_path_args(seeds, nseeds, dt, max_steps, vertices, counts, reasons);
  if (s) return s;
  for (int i = 0; i + 1 < ngrids; ++i)
    if (!(times[i + 1] > times[i])) return fail(INR_ERR_INVALID_ARG, "times must be strictly increasing");
  long long n[3] = {dims[0], dims[1], dims[2]};
  for (int d = 0; d < 3; ++d)
    if (n[d] < 1) return fail(INR_ERR_INVALID_ARG, "dims must be >= 1");
  if (nseeds == 0) return INR_OK;
  ProfScope p(PK_PATHLINE, st);
  launch_path_init(grids[0], grids[1], n, times[0], sign, seeds, nseeds, max_steps, vertices, counts, reasons, st);
  for (int i = 0; i + 1 < ngrids; ++i)
    launch_path_interval(grids[i], grids[i + 1], n, times[i], times[i + 1], dt, sign, max_steps, nseeds, vertices,
                         counts, reasons, st);
  launch_path_finish(nseeds, reasons, st);
  CK_LAUNCH("pathlines");
  return INR_OK;
}

// Decode every block of one window element into the global velocity grid.
static inr_status decode_element(const CacheSlot& slot, float* grid, const int64_t N[3], cudaStream_t st) {
  const inr_model* m0 = slot.cmodels[0];
  const int64_t B[3] = {(N[0] + m0->blk.n[0] - 1) / m0->blk.n[0], (N[1] + m0->blk.n[1] - 1) / m0->blk.n[1],
                        (N[2] + m0->blk.n[2] - 1) / m0->blk.n[2]};
  if ((int64_t)slot.cmodels.size() != B[0] * B[1] * B[2])
    return fail(INR_ERR_INVALID_ARG, "a window element must hold every block of the volume");
  const int64_t os[3] = {3, 3 * N[0], 3 * N[0] * N[1]};
  for (const inr_model* m : slot.cmodels) {
    if (m->net.D != 3) return fail(INR_ERR_INVALID_ARG, "pathlines need vector-field (out_dim 3) models");
    int32_t res[3], cnt[3];
    int64_t off = 0;
    for (int d = 0; d < 3; ++d) {
      if (m->blk.global_dims[d] != N[d] || m->blk.n[d] != m0->blk.n[d])
        return fail(INR_ERR_INVALID_ARG, "window element models must tile one volume");
      res[d] = m->blk.n[d];
      cnt[d] = (int32_t)std::min<int64_t>(m->blk.n[d], N[d] - m->blk.origin[d]);
      off += m->blk.origin[d] * os[d];
    }
    inr_status s = inr_decode_grid_part(m, res, cnt, grid + off, os, nullptr, nullptr, st);
    if (s) return s;
  }
  return INR_OK;
}

extern "C" inr_status inr_pathlines(const inr_cache* c, int32_t window_ops, const double* seeds, int32_t nseeds,
                                    double dt, int32_t max_steps, double* vertices, int32_t* counts,
                                    int32_t* reasons, cudaStream_t st) {
  if (!c) return fail(INR_ERR_INVALID_ARG, "cache is NULL");
  if (c->slots.size() < 2) return fail(INR_ERR_INVALID_ARG, "a pathline window needs at least two timesteps");
  inr_status s = check_path_args(seeds, nseeds, dt, max_steps, vertices, counts, reasons);
  if (s) return s;
  if (nseeds == 0) return INR_OK;
  const int W = (int)c->slots.size();
  const inr_model* m0 = c->slots[0].cmodels[0];
  const int64_t N[3] = {m0->blk.global_dims[0], m0->blk.global_dims[1], m0->blk.global_dims[2]};
  const long long n[3] = {N[0], N[1], N[2]};
  const bool rev = window_ops & INR_WINDOW_REVERSE;
  const double sign = (window_ops & INR_WINDOW_NEGATE) ? -1.0 : 1.0;
  // element i of the (reversed) window and its time (tau_i = t_last - t_{W-1-i} when reversed)
  auto elem = [&](int i) -> const CacheSlot& { return c->slots[rev ? W - 1 - i : i]; };
  auto time = [&](int i) -> double {
    return rev ? (double)c->slots[W - 1].timestep - (double)c->slots[W - 1 - i].timestep
               : (double)c->slots[i].timestep;
  };
  CK(cudaSetDevice(c->device));
  keep_pool(c->device);
  float* buf[2] = {nullptr, nullptr};
  const size_t bytes = (size_t)N[0] * N[1] * N[2] * 3 * sizeof(float);
  CK(cudaMallocAsync((void**)&buf[0], bytes, st));
  CK(cudaMallocAsync((void**)&buf[1], bytes, st));
  struct Free {
    float** b; cudaStream_t s;
    ~Free() { cudaFreeAsync(b[0], s); cudaFreeAsync(b[1], s); }
  } release{buf, st};
  // two grids resident: element i + 1 is decoded into the buffer element i - 1 held
  s = decode_element(elem(0), buf[0], N, st);
  if (s) return s;
  s = decode_element(elem(1), buf[1], N, st);
  if (s) return s;
  {
    ProfScope p(PK_PATHLINE, st);
    launch_path_init(buf[0], buf[1], n, time(0), sign, seeds, nseeds, max_steps, vertices, counts, reasons, st);
  }
  for (int i = 0; i + 1 < W; ++i) {
    if (i > 0) {
      s = decode_element(elem(i + 1), buf[(i + 1) & 1], N, st);
      if (s) return s;
    }
    ProfScope p(PK_PATHLINE, st);
    launch_path_interval(buf[i & 1], buf[(i + 1) & 1], n, time(i), time(i + 1), dt, sign, max_steps, nseeds,
                         vertices, counts, reasons, st);
  }
  {
    ProfScope p(PK_PATHLINE, st);
    launch_path_finish(nseeds, reasons, st);
  }
  CK_LAUNCH("pathlines");
  return INR_OK;
}


// ------------------------------------------------------------------ rendering
// NEXT-3: direct-query DVR of one rank's
// blocks by sample streaming, macro-cell skipping, sort-last compositing.
struct inr_renderer {
  int device = 0;
  std::vector<const inr_model*> models;
  int cells = 16;
  int n[3], B[3];
  int* slot_of_block = nullptr;   // device [nblocks]
  float2* range = nullptr;        // device [nmodels][cells^3] (data units, padded)
  uint8_t* empty = nullptr;       // device [nmodels][cells^3]
  int64_t evaluated = 0, skipped = 0;
  int waves = 0;
};

extern "C" inr_status inr_renderer_destroy(inr_renderer* r) {
  if (!r) return INR_OK;
  cudaSetDevice(r->device);
  cudaFree(r->slot_of_block);
  cudaFree(r->range);
  cudaFree(r->empty);
  delete r;
  return INR_OK;
}

extern "C" inr_status inr_renderer_create(const inr_model* const* models, int32_t nmodels, int32_t cells, double pad,
                                          cudaStream_t st, inr_renderer** out) {
  if (!out) return fail(INR_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (!models || nmodels < 1) return fail(INR_ERR_INVALID_ARG, "models missing");
  if (nmodels > kMaxGroup) return fail(INR_ERR_UNSUPPORTED, "at most %d models per renderer", kMaxGroup);
  if (cells < 1 || cells > 64) return fail(INR_ERR_INVALID_ARG, "cells must be in 1..64");
  if (!(pad >= 0.0)) return fail(INR_ERR_INVALID_ARG, "pad must be >= 0");
  const inr_model* m0 = models[0];
  if (!m0) return fail(INR_ERR_INVALID_ARG, "model 0 is NULL");
  if (m0->net.D != 1) return fail(INR_ERR_UNSUPPORTED, "volume rendering needs scalar-field (out_dim 1) models");
  long long nb = 1;
  int n[3], B[3];
  for (int d = 0; d < 3; ++d) {
    n[d] = m0->blk.n[d];
    B[d] = (int)((m0->blk.global_dims[d] + n[d] - 1) / n[d]);
    nb *= B[d];
  }
  if (nb > kMaxRouteBlocks) return fail(INR_ERR_UNSUPPORTED, "at most %d blocks in a volume", kMaxRouteBlocks);
  std::vector<int> sob((size_t)nb, -1);
  for (int i = 0; i < nmodels; ++i) {
    const inr_model* m = models[i];
    if (!m || !same_shape(m->cfg, m0->cfg) || m->device != m0->device)
      return fail(INR_ERR_INVALID_ARG, "renderer models must share config and device");
    for (int d = 0; d < 3; ++d)
      if (m->blk.n[d] != n[d] || m->blk.global_dims[d] != m0->blk.global_dims[d])
        return fail(INR_ERR_INVALID_ARG, "renderer models must tile one volume");
    sob[m->block_id] = i;
  }
  CK(cudaSetDevice(m0->device));
  keep_pool(m0->device);
  inr_renderer* r = new inr_renderer();
  r->device = m0->device;
  r->models.assign(models, models + nmodels);
  r->cells = cells;
  for (int d = 0; d < 3; ++d) { r->n[d] = n[d]; r->B[d] = B[d]; }
  const long long nc = (long long)nmodels * cells * cells * cells;
  if (cudaMalloc((void**)&r->slot_of_block, sizeof(int) * nb) != cudaSuccess ||
      cudaMalloc((void**)&r->range, sizeof(float2) * nc) != cudaSuccess ||
      cudaMalloc((void**)&r->empty, nc) != cudaSuccess) {
    inr_renderer_destroy(r);
    return fail(INR_ERR_OOM, "renderer allocation");
  }
  CK(cudaMemcpyAsync(r->slot_of_block, sob.data(), sizeof(int) * nb, cudaMemcpyHostToDevice, st));
  // probe lattice per block: R = 4 cells per axis, decoded on the library's grid path
  const int P = 4, R = cells * P;
  float* probes = nullptr;
  CK(cudaMallocAsync((void**)&probes, sizeof(float) * (size_t)nmodels * R * R * R, st));
  const int32_t res[3] = {R, R, R};
  for (int i = 0; i < nmodels; ++i) {
    inr_status s = inr_decode_grid(models[i], res, probes + (size_t)i * R * R * R, nullptr, nullptr, nullptr, st);
    if (s) { cudaFreeAsync(probes, st); inr_renderer_destroy(r); return s; }
  }
  launch_mc_reduce(probes, nmodels, cells, P, (float)pad, r->range, st);
  CK_LAUNCH("macro-cells");
  CK(cudaFreeAsync(probes, st));
  *out = r;
  return INR_OK;
}

static inr_status render_tf(const inr_transfer_fn* tf, RenderTF& t) {
  if (!tf) return fail(INR_ERR_INVALID_ARG, "transfer function is NULL");
  if (tf->npoints < 2 || tf->npoints > kTfMaxPoints)
    return fail(INR_ERR_INVALID_ARG, "transfer function needs 2..%d points", kTfMaxPoints);
  if (!(tf->vmax > tf->vmin)) return fail(INR_ERR_INVALID_ARG, "transfer function vmax must exceed vmin");
  if (!(tf->base_step > 0.0)) return fail(INR_ERR_INVALID_ARG, "base_step must be > 0");
  memset(&t, 0, sizeof t);
  t.n = tf->npoints;
  for (int i = 0; i < tf->npoints; ++i) {
    if (i > 0 && !(tf->s[i] > tf->s[i - 1])) return fail(INR_ERR_INVALID_ARG, "transfer function s must increase");
    t.s[i] = tf->s[i];
    for (int c = 0; c < 4; ++c) {
      if (!(tf->rgba[i][c] >= 0.f && tf->rgba[i][c] <= 1.f)) return fail(INR_ERR_INVALID_ARG, "rgba outside [0, 1]");
      t.rgba[i][c] = tf->rgba[i][c];
    }
  }
  t.vmin = (float)tf->vmin;
  t.inv_range = (float)(1.0 / (tf->vmax - tf->vmin));
  return INR_OK;
}

extern "C" inr_status inr_render(inr_renderer* r, const inr_camera* cam, const inr_transfer_fn* tf,
                                 const double lo[3], const double hi[3], double step, double stop_alpha,
                                 int32_t use_mc, float* frag, cudaStream_t st) {
  if (!r || !cam || !lo || !hi || !frag) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  if (cam->width < 1 || cam->height < 1 || (long long)cam->width * cam->height > (1ll << 28))
    return fail(INR_ERR_INVALID_ARG, "image size");
  if (!(cam->fovy_deg > 0.0 && cam->fovy_deg < 180.0)) return fail(INR_ERR_INVALID_ARG, "fovy must be in (0, 180)");
  if (!(step > 0.0)) return fail(INR_ERR_INVALID_ARG, "step must be > 0");
  RenderArgs a;
  memset(&a, 0, sizeof a);
  inr_status s = render_tf(tf, a.tf);
  if (s) return s;
  // camera basis (R33): f = normalize(look - eye), r = normalize(f x up), u = r x f
  double f[3], rr[3], u[3];
  for (int c = 0; c < 3; ++c) f[c] = cam->look[c] - cam->eye[c];
  double nf = std::sqrt(f[0] * f[0] + f[1] * f[1] + f[2] * f[2]);
  if (!(nf > 0.0)) return fail(INR_ERR_INVALID_ARG, "eye == look");
  for (int c = 0; c < 3; ++c) f[c] /= nf;
  rr[0] = f[1] * cam->up[2] - f[2] * cam->up[1];
  rr[1] = f[2] * cam->up[0] - f[0] * cam->up[2];
  rr[2] = f[0] * cam->up[1] - f[1] * cam->up[0];
  double nr = std::sqrt(rr[0] * rr[0] + rr[1] * rr[1] + rr[2] * rr[2]);
  if (!(nr > 0.0)) return fail(INR_ERR_INVALID_ARG, "up is parallel to the view direction");
  for (int c = 0; c < 3; ++c) rr[c] /= nr;
  u[0] = rr[1] * f[2] - rr[2] * f[1];
  u[1] = rr[2] * f[0] - rr[0] * f[2];
  u[2] = rr[0] * f[1] - rr[1] * f[0];
  for (int c = 0; c < 3; ++c) {
    a.eye[c] = cam->eye[c]; a.f[c] = f[c]; a.r[c] = rr[c]; a.u[c] = u[c];
    a.lo[c] = lo[c]; a.hi[c] = hi[c];
    a.n[c] = r->n[c]; a.B[c] = r->B[c];
  }
  a.th = std::tan(cam->fovy_deg * M_PI / 180.0 / 2.0);
  a.width = cam->width;
  a.height = cam->height;
  a.npix = cam->width * cam->height;
  a.step = step;
  a.exponent = (float)(step / tf->base_step);
  a.stop_alpha = (float)stop_alpha;
  a.cells = r->cells;
  a.slot_of_block = r->slot_of_block;
  CK(cudaSetDevice(r->device));
  const int nm = (int)r->models.size();
  const long long nc = (long long)nm * r->cells * r->cells * r->cells;
  if (use_mc) {
    launch_mc_mark(r->range, nc, a.tf, r->empty, st);
    a.empty = r->empty;
  }
  const long long npix = a.npix;
  const int S = (int)std::max<long long>(4, std::min<long long>(64, (1ll << 26) / npix));
  // per-call workspace (stream-ordered): ray state, wave queries and values
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) / 256 * 256; return o; };
  const size_t o_dir = take(24 * npix), o_t0 = take(8 * npix), o_t1 = take(8 * npix), o_k = take(8 * npix),
               o_live = take(4 * npix), o_C = take(16 * npix), o_base = take(4 * npix), o_nq = take(4 * npix),
               o_q = take(12 * npix * S), o_v = take(4 * npix * S), o_cnt = take(16);
  char* ws = nullptr;
  CK(cudaMallocAsync((void**)&ws, off, st));
  struct Free { char* p; cudaStream_t s; ~Free() { cudaFreeAsync(p, s); } } release{ws, st};
  RayState rs;
  rs.dir = (double*)(ws + o_dir);
  rs.t_enter = (double*)(ws + o_t0);
  rs.t_exit = (double*)(ws + o_t1);
  rs.k = (long long*)(ws + o_k);
  rs.live = (int*)(ws + o_live);
  rs.C = (float*)(ws + o_C);
  int* base = (int*)(ws + o_base);
  int* nq = (int*)(ws + o_nq);
  float* qxyz = (float*)(ws + o_q);
  float* vals = (float*)(ws + o_v);
  int* qcount = (int*)(ws + o_cnt);
  unsigned long long* skipped = (unsigned long long*)(ws + o_cnt + 8);
  CK(cudaMemsetAsync(ws + o_cnt, 0, 16, st));
  r->evaluated = 0;
  r->waves = 0;
  launch_ray_init(a, rs, st);
  for (;;) {
    CK(cudaMemsetAsync(qcount, 0, sizeof(int), st));
    launch_gen(a, rs, S, qxyz, qcount, base, nq, skipped, st);
    CK_LAUNCH("render gen");
    int q = 0;
    CK(cudaMemcpyAsync(&q, qcount, sizeof q, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (q == 0) break;
    s = decode_group_impl(r->models.data(), nm, qxyz, q, vals, 0, st);
    if (s) return s;
    launch_composite(a, rs, vals, base, nq, st);
    CK_LAUNCH("render composite");
    r->evaluated += q;
    ++r->waves;
  }
  launch_fragments(a, rs, frag, st);
  CK_LAUNCH("render fragments");
  unsigned long long sk = 0;
  CK(cudaMemcpyAsync(&sk, skipped, sizeof sk, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  r->skipped = (int64_t)sk;
  return INR_OK;
}

extern "C" inr_status inr_render_stats(const inr_renderer* r, int64_t* evaluated, int64_t* skipped, int32_t* waves) {
  if (!r) return fail(INR_ERR_INVALID_ARG, "renderer is NULL");
  if (evaluated) *evaluated = r->evaluated;
  if (skipped) *skipped = r->skipped;
  if (waves) *waves = r->waves;
  return INR_OK;
}

extern "C" inr_status inr_composite(const float* frags, int32_t nfrag, int64_t npix, const float bg[3], float* img,
                                    cudaStream_t st) {
  if (!frags || !img || !bg) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  if (nfrag < 1 || nfrag > kMaxFragments) return fail(INR_ERR_INVALID_ARG, "nfrag must be in 1..%d", kMaxFragments);
  if (npix < 0) return fail(INR_ERR_INVALID_ARG, "npixels must be >= 0");
  if (npix == 0) return INR_OK;
  launch_blend(frags, nfrag, npix, bg, img, st);
  CK_LAUNCH("composite");
  return INR_OK;
}

// ------------------------------------------------------------ peer memory
// Fused decode + gather over NVLink (a18): a rank exports the allocation behind a
// device pointer as a CUDA IPC handle, the other ranks open it and the decode
// kernels store their slabs straight into the destination through peer memory.
extern "C" inr_status inr_ipc_handle(const void* ptr, unsigned char handle[64], int64_t* offset) {
  if (!ptr || !handle || !offset) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  // the allocation's base: a driver-API query, resolved at run time (no link-time libcuda)
  typedef CUresult (*GetRange)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(INR_ERR_CUDA, "cuMemGetAddressRange unavailable");
    get_range = (GetRange)fn;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS)
    return fail(INR_ERR_CUDA, "cuMemGetAddressRange failed (not a device allocation?)");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, (void*)base));
  static_assert(sizeof h == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle, &h, 64);
  *offset = (int64_t)((CUdeviceptr)ptr - base);
  return INR_OK;
}

extern "C" inr_status inr_ipc_open(const unsigned char handle[64], int64_t offset, int device, void** ptr,
                                   void** base) {
  if (!handle || !ptr || !base) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  CK(cudaSetDevice(device));
  void* b = nullptr;
  CK(cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess));
  *base = b;
  *ptr = (char*)b + offset;
  return INR_OK;
}

extern "C" inr_status inr_ipc_close(void* base) {
  if (!base) return fail(INR_ERR_INVALID_ARG, "NULL argument");
  CK(cudaIpcCloseMemHandle(base));
  return INR_OK;
}

