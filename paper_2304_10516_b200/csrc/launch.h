// launch.h — internal interface between the C-ABI runtime (inr_runtime.cu)
// and the kernel translation units.  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace inr {

// Kernel-parameter block for a group of models (<= kMaxGroup) sharing one config.
struct GroupArgs {
  NetDesc net;
  int nmodels;
  ModelDev md[kMaxGroup];
};

struct FitScalars {
  int B_u, B_b;       // uniform / boundary samples per model per step
  float lambda;
  int det;            // deterministic reduction
};

struct AdamScalars {
  double lr0, lr_decay, beta1, beta2;
  long long lr_step;
  float b1, b2, ob1, ob2, eps;   // fp32 beta, 1 - beta (formed in fp64), eps
  int sparse;                    // R37: touched-only table updates
  long long table_end;           // internal offset where the MLP parameters start
};

constexpr int kMaxRouteBlocks = 4096;
struct QueryArgs {
  NetDesc net;
  int n[3], N[3], B[3];
  int nblocks;
  int nmodels;
  ModelDev md[kMaxGroup];
  int16_t slot_of_block[kMaxRouteBlocks];
};
inline int qa_nmodels(const QueryArgs& qa) { return qa.nmodels; }

void count_launch(long long n = 1);

// stream-ordered loss report (kernels_simt.cu)
struct LossReportArgs {
  int n;
  const double* acc[kMaxGroup];
  const int* flag[kMaxGroup];
  double inv_u[kMaxGroup], inv_b[kMaxGroup];
};
void launch_loss_report(const LossReportArgs& a, double* out, cudaStream_t st);

// volume rendering (kernels_render.cu, NEXT-3)
constexpr int kTfMaxPoints = 16;
constexpr int kMaxFragments = 64;
struct RenderTF {
  int n;
  float s[kTfMaxPoints];
  float rgba[kTfMaxPoints][4];
  float vmin, inv_range;
};
struct RenderArgs {
  double eye[3], f[3], r[3], u[3], th;   // camera: forward, right, up, tan(fovy / 2)
  int width, height, npix;
  double lo[3], hi[3];                   // the brick (global node coordinates)
  double step;
  float exponent, stop_alpha;            // step / base_step; early-termination opacity
  RenderTF tf;
  int n[3], B[3], cells;                 // block geometry (R5 routing) and macro-cells per block axis
  const int* slot_of_block;              // [nblocks] slot or -1
  const uint8_t* empty;                  // [slot][cells^3] 1 = no opacity for tf, or null (no skipping)
};
struct RayState {
  double* dir;       // [npix][3]
  double* t_enter;   // [npix]
  double* t_exit;
  long long* k;      // next sample index
  int* live;
  float* C;          // [npix][4] premultiplied RGB, A
};
void launch_mc_reduce(const float* probes, int nslots, int cells, int P, float pad, float2* range, cudaStream_t st);
void launch_mc_mark(const float2* range, long long n, const RenderTF& tf, uint8_t* empty, cudaStream_t st);
void launch_ray_init(const RenderArgs& a, const RayState& rs, cudaStream_t st);
void launch_gen(const RenderArgs& a, const RayState& rs, int S, float* qxyz, int* qcount, int* base, int* nq,
                unsigned long long* skipped, cudaStream_t st);
void launch_composite(const RenderArgs& a, const RayState& rs, const float* vals, const int* base, const int* nq,
                      cudaStream_t st);
void launch_fragments(const RenderArgs& a, const RayState& rs, float* frag, cudaStream_t st);
void launch_blend(const float* frags, int nfrag, long long npix, const float bg[3], float* img, cudaStream_t st);

// pathlines (kernels_path.cu)
void launch_path_init(const float* g0, const float* g1, const long long n[3], double t0, double sign,
                      const double* seeds, int M, int max_steps, double* vert, int* count, int* reason,
                      cudaStream_t st);
void launch_path_interval(const float* g0, const float* g1, const long long n[3], double ta, double tb, double dt,
                          double sign, int max_steps, int M, double* vert, int* count, int* reason, cudaStream_t st);
void launch_path_finish(int M, int* reason, cudaStream_t st);

void launch_init_params(const NetDesc& net, float* params, uint32_t k0, uint32_t k1, uint32_t block_id,
                        cudaStream_t st);
void launch_step_begin(const GroupArgs& g, int nmodels, long long zero_from, cudaStream_t st);
void launch_fit_simt(const GroupArgs& g, int nmodels, const FitScalars& fs, cudaStream_t st);
// ctas > 0: total CTAs of the launch (the split fit step runs it beside an MLP launch)
void launch_adam(const GroupArgs& g, int nmodels, const AdamScalars& as, cudaStream_t st, int ctas = 0);
void launch_probe(const GroupArgs& g, int nmodels, cudaStream_t st);
void launch_decode_grid_simt(const NetDesc& net, const ModelDev& md, const int res[3], const int cnt[3], float* out,
                             const long long os[3], const float* ref, double* sse, cudaStream_t st);
void launch_decode_query_simt(const QueryArgs& qa, const float* xyz, long long q, float* out, int* dflag,
                              cudaStream_t st);
void launch_convert_f32_f16(const float* src, __half* dst, long long n, cudaStream_t st);
void launch_convert_f16_f32(const __half* src, float* dst, long long n, cudaStream_t st);
void launch_range(const float* base, const int dims[3], const long long s[3], int channels, float* minmax,
                  cudaStream_t st);
void launch_debug_encode(const NetDesc& net, const float* P, const float* x01, long long q, uint32_t* idx,
                         float* feat, cudaStream_t st);
void launch_debug_forward_simt(const NetDesc& net, const float* P, const float* x01, long long q, float* y,
                               cudaStream_t st);

// level-major fp16 fit pipeline — kernels_lm.cu (CUDA cores) + kernels_tc.cu (tcgen05)
// Geometry of the fp16 feature tile images the encode writes and the tensor-core
// MLP bulk-copies: 128 samples x (LF + ones) columns in the canonical layout.
struct FeatGeom {
  uint32_t sbo;         // row-group stride (bytes)
  uint32_t tile_bytes;  // bytes per 128-sample tile
  int ones;             // width of the constant-ones column group (0 or 8)
};
bool tc_fit_geometry(const NetDesc& net, FeatGeom* geom, uint32_t* img_bytes);

struct LmWorkspace {
  float4* samples;   // [model][Bs] (x, y, z, target)
  uint8_t* featimg;  // [model][Bs/128] fp16 h_0 tile images
  float* dfeat;      // [model][level][Bs][F] fp32
  uint8_t* wimg;     // [model] fp16 weight images (tiles, biases, output layer)
  float4* targets;   // [model][Bs] (t_0, t_1, t_2, 0) for vector fields, else null
  FeatGeom geom;
  uint32_t img_bytes;
  int Bs;            // per-model sample stride (multiple of 128)
};
size_t lm_workspace_bytes(const NetDesc& net, int nmodels, int Bs);
LmWorkspace lm_workspace(void* base, const NetDesc& net, int nmodels, int Bs);
void launch_prep_image(const GroupArgs& g, int nmodels, uint8_t* wimg, cudaStream_t st);

void launch_encode_fwd(const GroupArgs& g, int nmodels, const FitScalars& fs, const LmWorkspace& w, cudaStream_t st);
void launch_encode_bwd(const GroupArgs& g, int nmodels, const FitScalars& fs, const LmWorkspace& w, cudaStream_t st);
bool tc_supported(const NetDesc& net);
void launch_mlp_tc(const GroupArgs& g, int nmodels, const FitScalars& fs, const uint8_t* featimg, const uint8_t* wimg,
                   const float4* samples, const float4* targets, float* dfeat, int Bs, cudaStream_t st,
                   int ctas = 0);   // ctas > 0: at most this many CTAs in all (deterministic mode: ignored)
void launch_debug_forward_tc(const NetDesc& net, const float* P, const float* x01, long long q, float* y,
                             cudaStream_t st);
void launch_decode_grid_tc(const NetDesc& net, const ModelDev& md, const int res[3], const int cnt[3], float* out,
                           const long long os[3], const float* ref, double* sse, cudaStream_t st);
struct QueryBuckets {
  int* perm;       // [q + 128 nmodels] query index or -1, bucket-sorted, each bucket padded to 128
  int* tile_slot;  // model slot of each 128-query tile
  int* ntiles;     // device scalar
};
void launch_decode_query_tc(const GroupArgs& g, const float* xyz, long long q, float* out, const QueryBuckets& b,
                            cudaStream_t st);
size_t query_workspace_bytes(long long q, int nmodels);
void launch_query_prep(const GroupArgs& g, const float* xyz, const QueryBuckets& b, long long j0, long long n,
                       float4* qx, cudaStream_t st);
void launch_encode_query(const GroupArgs& g, const float4* qx, long long n, uint8_t* featimg, const FeatGeom& geom,
                         cudaStream_t st);
void launch_query_buckets(const QueryArgs& qa, const float* xyz, long long q, float* out, int* dflag, void* ws,
                          QueryBuckets& b, cudaStream_t st);

}  // namespace inr
