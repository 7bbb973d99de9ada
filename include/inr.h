/*
 * inr.h — C ABI of the B200 (sm_100a) hash-grid INR library `libinr.so`.
 *
 * The operation is the hot path of arXiv 2304.10516 ("distributed neural
 * representation", DNR): one implicit neural representation per spatial block
 * of a scalar (or vector, D = 3) volume,
 *     Phi : R^3 -> R^D, (x,y,z) -> v                    (Eq. 1)
 * built from a multiresolution hash-grid encoding and a small ReLU MLP
 * (PAPER.md L157-158, L217-218), fitted to uniformly sampled, interpolated and
 * normalized targets (L172-173, L204-205) with the boundary-weighted L1 loss
 *     L = (1 - lambda) L1(X_Uniform, Y_Uniform) + lambda L1(X_Bound, Y_Bound)
 * (Eq. 2) and Adam with a step learning-rate schedule (L220), then
 * decoded by coordinate query or to a grid (L175-176, L268), and cached in a
 * FIFO window of timesteps (L238, L271-274, L290); plus the paper's consumers
 * of that window — backward pathlines (L411-424) and direct-query volume
 * rendering (L268, L293-300) — and the multi-GPU plumbing around them.  Where
 * the paper is silent the readings R1..R36 of DESIGN.md apply; they are cited
 * below as [Rn].
 *
 * Conventions
 *  - Every function returns an inr_status and never aborts or throws.  On a
 *    non-OK status, inr_last_error() returns thread-local text describing it.
 *  - All pointers marked (dev) are device pointers on the model's device; the
 *    caller owns them and keeps them valid until the stream has executed the
 *    call's work.  The library never retains caller buffers.  (host) pointers
 *    are ordinary host memory.
 *  - The library owns everything behind handles: tables, MLP weights, grads,
 *    Adam state, workspaces.
 *  - Coordinates are (x, y, z); volumes are x-fastest, then y, then z.
 *  - A block with core origin o and n cells per axis maps node position p to
 *    the block-normalized x = (p - o)/n in [0,1]^3 (cell-span convention, so
 *    neighbouring blocks share the face plane o + n) [R5]; on a rectilinear
 *    mesh (inr_set_mesh) through the node coordinates instead [R36].
 *  - Sticky CUDA errors surface as INR_ERR_CUDA at the next call.
 *  - There is no CPU fallback: without a usable sm_100 device every call that
 *    needs one fails with INR_ERR_CUDA.
 */
#ifndef INR_H
#define INR_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define INR_API __attribute__((visibility("default")))
#else
#define INR_API
#endif

typedef struct CUstream_st* cudaStream_t;  /* identical to the CUDA runtime typedef */

typedef enum {
  INR_OK = 0,
  INR_ERR_INVALID_ARG = 1,   /* null handle, bad config or option, steps < 1, ... */
  INR_ERR_DOMAIN = 2,        /* strict decode: a coordinate outside [0, N-1]^3 */
  INR_ERR_NONFINITE = 3,     /* non-finite loss or parameter detected after a step */
  INR_ERR_OOM = 4,
  INR_ERR_CUDA = 5,
  INR_ERR_STATE = 6,         /* evict on empty cache; fit on a frozen (cached) model */
  INR_ERR_UNSUPPORTED = 7    /* a valid configuration outside this build's kernels */
} inr_status;

/* Thread-local text of the last non-OK status of this thread ("" if none). */
INR_API const char* inr_last_error(void);

#define INR_MAX_CHANNELS 3

enum { INR_PREC_FP32 = 0,      /* MLP on CUDA cores in fp32 (parity mode) */
       INR_PREC_FP16_MLP = 1   /* MLP on tcgen05 tensor cores: fp16 operands, fp32
                                  accumulate in TMEM, fp32 master weights [R17] */ };
enum { INR_REDUCE_ATOMIC = 0,          /* fp32 atomics: fastest, run-to-run rounding noise */
       INR_REDUCE_DETERMINISTIC = 1 }; /* exact int64 fixed-point sums: bitwise reproducible [R21] */

/* Network configuration.
 *   levels L >= 1, features F in {1,2,4,8}, table size T = 2^log2_table_size
 *   (1..24 in this build), base resolution N_min >= 1, per_level_scale b > 1; level l has
 *   resolution N_l = floor(N_min * b^l) [R3], at most 2^30 (the cell index is an
 *   int32: INR_ERR_INVALID_ARG beyond), and min(T, (N_l+1)^3) entries
 *   (dense x-fastest index when (N_l+1)^3 <= T, else the spatial hash of S:L236) [R1, R2].
 *   mlp_width W = 64 (this build), mlp_hidden_layers H in 1..8 (H hidden layers
 *   => H+1 weight matrices [R16]), out_dim D in {1, 3} (scalar or vector field,
 *   P:L156), mlp_bias in {0,1} [R15].
 *   L*F <= 64 and, for INR_PREC_FP16_MLP, a multiple of 16; fitting in
 *   INR_PREC_FP16_MLP also needs the tensor-memory weight-gradient accumulators
 *   to fit, 64 + sum_k (in_k + 8) <= 512 columns (H <= 6 at L*F = 32, H <= 5 at
 *   64), else inr_fit returns INR_ERR_UNSUPPORTED (decode has no such limit).
 *   seed selects the Philox4x32-10 streams for init (0), uniform samples (1),
 *   boundary samples (2) [R8, R14]. */
typedef struct {
  int32_t levels, features, log2_table_size, base_resolution;
  float per_level_scale;
  int32_t mlp_width, mlp_hidden_layers, out_dim, mlp_bias;
  int32_t precision, reduction;
  uint64_t seed;
} inr_config;

/* A block (partition core) of a volume, in node units.
 * origin[d] is a multiple of n[d]; the volume has global_dims[d] nodes; blocks
 * tile it with ceil(N/n) blocks per axis; block id = (bz*By + by)*Bx + bx. */
typedef struct {
  int64_t origin[3];
  int32_t n[3];
  int64_t global_dims[3];
} inr_block;

typedef struct inr_model inr_model;  /* opaque; lives on one CUDA device */

/* Allocate a model on `device` and initialise it from cfg->seed [R14]
 * (tables U[-1e-4,1e-4], weights He-uniform, biases 0; Philox stream 0,
 * counter (param index j, block id, 0, 0)).  Errors: INVALID_ARG, UNSUPPORTED,
 * OOM, CUDA. */
INR_API inr_status inr_create(const inr_config* cfg, const inr_block* block, int device, inr_model** out);
/* Re-initialise parameters from `seed`, zero Adam state and grads, step = 0
 * (fresh init per timestep, [R22]).  INR_ERR_STATE on a frozen model. */
INR_API inr_status inr_reset(inr_model* m, uint64_t seed);
/* Warm start (a semantics change versus R22's fresh init):
 * keep the parameters, zero the Adam moments, gradients and step counter (the
 * learning-rate schedule restarts), so the next inr_fit continues from the
 * previous timestep's network.  INR_ERR_STATE on a frozen model. */
INR_API inr_status inr_reset_optimizer(inr_model* m);
/* Rectilinear mesh (NEXT-4; "for uniform and rectilinear meshes, we
 * provide a native data sampler") [R36]: coords[d] (host) holds the
 * N_d strictly increasing physical node coordinates of axis d of the global
 * volume; the model keeps its block's slice.  From then on the block's network
 * takes the block-normalized PHYSICAL coordinate x = (P - P_lo)/(P_hi - P_lo),
 * P_lo/P_hi the coordinates of nodes o and min(o + n, N - 1); fit samples are
 * uniform in that physical box and their targets trilinear in the physical
 * cell; inr_decode_grid decodes the block's nodes (res must equal n) and queries
 * (still global node-index coordinates, routed by R5) are mapped through the
 * mesh's piecewise-linear node -> coordinate map.  coords NULL restores the
 * uniform mesh.  Synchronous. */
INR_API inr_status inr_set_mesh(inr_model* m, const double* const coords[3]);
/* Model state transfer (NEXT-4 cross-GPU block stealing): the trainable state —
 * parameters, Adam moments, step counters, value range — as one opaque device
 * buffer of inr_state_bytes bytes, e.g. to continue a block's fit on another GPU
 * (the buffer travels by NCCL / peer copy).  Importing into a model of the same
 * configuration and block makes its next fit steps bitwise those the exporter
 * would have taken.  Both calls synchronize `stream`. */
INR_API inr_status inr_state_bytes(const inr_model* m, int64_t* bytes);
INR_API inr_status inr_export_state(const inr_model* m, void* dst, cudaStream_t stream);
INR_API inr_status inr_import_state(inr_model* m, const void* src, cudaStream_t stream);
/* Free a model (NULL is a no-op).  Models borrowed from a cache must not be destroyed. */
INR_API inr_status inr_destroy(inr_model* m);
/* Number of fp32 parameters in the declared order (tables by level, then
 * W_0, b_0, ..., W_H, b_H) and the stored bytes (4 per parameter) [R24]. */
INR_API inr_status inr_param_count(const inr_model* m, int64_t* count);
INR_API inr_status inr_param_bytes(const inr_model* m, int64_t* bytes);
/* Adam steps taken so far. */
INR_API inr_status inr_steps(const inr_model* m, int64_t* steps);

/* Fit options.  Defaults in
 * inr_fit_opts_default(): lambda 0.5, boundary_batch 0, lr0 1e-2, lr_decay 0.8,
 * lr_step 500, beta1 0.9, beta2 0.999, eps 1e-8, vmin 0, vmax 1,
 * target_psnr 0, check_interval 0.
 *   lambda in [0,1]; boundary_batch B_b >= 0 boundary samples per step (lambda'
 *   = 0 when B_b = 0 or the block has no interior face [R11]); lr at 0-based
 *   step s is lr0 * lr_decay^floor(s / lr_step) [R13]; Adam is PyTorch's dense
 *   form [R12]; [vmin, vmax] is the global value range shared by all blocks
 *    — vmax == vmin is legal (targets 0, report.constant_field = 1);
 *   target_psnr > 0 with check_interval > 0 stops once the PSNR on a 32^3
 *   cell-centred probe lattice reaches the target.
 *   Vector fields (out_dim 3) take per-channel ranges [vmin_c[c], vmax_c[c]]
 *   instead (vmin/vmax are then ignored); the L1 terms and the probe
 *   MSE pool over samples and channels [R28].
 *   sparse_adam != 0 (default 0; NEXT-4, a flagged semantics change versus
 *   R12, DESIGN R37): a hash-table parameter is updated only if its aligned
 *   group of 8 table floats (one 32-B sector) received a non-zero gradient this
 *   step; untouched groups keep p, m and v.  MLP parameters stay dense.
 *   split_step != 0 (default 1): a call that fits one launch group of >= 2 fp16
 *   models whose Adam does not dominate its MLP (not for cfg5's T = 2^22
 *   tables) runs each step as two halves of the group, and each half's Adam
 *   runs beside the other half's tensor-core MLP ("split fit
 *   step"); with PSNR-target stopping the deferred Adam is completed before
 *   every probe.  Every model takes the same
 *   operations in the same order as with split_step = 0, so the deterministic
 *   reduction mode gives bitwise the same parameters either way. */
typedef struct {
  double lambda;
  int32_t boundary_batch;
  double lr0, lr_decay;
  int32_t lr_step;
  double beta1, beta2, eps;   /* double so that 1 - beta is exact as in PyTorch's Adam */
  double vmin, vmax;
  double target_psnr;
  int32_t check_interval;
  double vmin_c[INR_MAX_CHANNELS], vmax_c[INR_MAX_CHANNELS];
  int32_t sparse_adam;        /* R37: touched-only table updates (0 = dense PyTorch Adam) */
  int32_t split_step;         /* 1 (default): split fit step, see below; 0: one pipeline */
} inr_fit_opts;
INR_API void inr_fit_opts_default(inr_fit_opts* o);

typedef struct {
  int32_t steps_taken, reached_target, constant_field;
  double loss_uniform, loss_boundary;  /* Eq. 2 terms of the last step taken */
  double probe_psnr;                   /* last probe PSNR (dB), 0 if never probed */
} inr_fit_report;

/* Strided device view of fp32 node values: node (i,j,k) of the volume (global
 * indices, lo[d] <= i < lo[d] + dims[d]) is base[(i-lo0)*stride0 + (j-lo1)*stride1
 * + (k-lo2)*stride2] (strides in elements).  For a block it must cover nodes
 * [o_d, min(o_d + n_d, N_d - 1)] per axis (the core plus the 1-node high-side
 * ghost layer [R6]); many blocks may share one allocation (zero-copy).
 * channels: 0 or 1 for a scalar field; 3 for a vector field whose channel c of
 * a node sits at +c (interleaved); it must equal the model's out_dim. */
typedef struct {
  const float* base;
  int64_t lo[3];
  int32_t dims[3];
  int64_t stride[3];
  int32_t channels;
} inr_view;

/* Train one model for `steps` >= 1 steps of `batch` >= 1 uniform samples plus
 * opts->boundary_batch boundary samples: Philox samples,
 * trilinear targets from the view, encode, MLP forward, Eq. 2, MLP backward,
 * table scatter-add, Adam.  Parameters continue from the model's current
 * step.  If `out` is non-NULL the call synchronizes `stream` and fills the
 * report (INR_ERR_NONFINITE if a non-finite loss/parameter appeared); if `out`
 * is NULL the call is stream-ordered and asynchronous (no probe stopping).
 * The gradients of the last step stay readable through inr_get_grads. */
INR_API inr_status inr_fit(inr_model* m, const inr_view* block_values, int32_t steps, int32_t batch,
                   const inr_fit_opts* opts, inr_fit_report* out, cudaStream_t stream);
/* Same semantics for `nmodels` independent models (one block each, all with the
 * same inr_config and device) in one fused launch per kernel per step
 * (decentralized DNR: no communication between models).  `out`,
 * if non-NULL, is an array of nmodels reports.  With PSNR-target stopping each
 * model leaves the group at the first check where it reaches the target, so it
 * ends exactly as if fitted alone (report.steps_taken per model) while the
 * others continue.
 * Execution (both calls): on a non-NULL stream and without PSNR-target stopping
 * one step is captured as a CUDA graph and replayed per step; the instantiated
 * graph and its workspace are cached (the last 4 distinct argument sets, keyed by
 * every value the step's kernels read) so later calls with the same models,
 * views and options replay it without a new capture; inr_destroy of any of the
 * models releases the entry. */
INR_API inr_status inr_fit_group(inr_model* const* models, const inr_view* views, int32_t nmodels,
                         int32_t steps, int32_t batch, const inr_fit_opts* opts,
                         inr_fit_report* out, cudaStream_t stream);

/* Stream-ordered report of the models' last fit step, for pipelined loops that
 * must not synchronize per step: enqueues one kernel writing, per model i,
 * out[3i..3i+2] = (L1_uniform, L1_boundary, 1.0 if a non-finite loss or
 * parameter appeared else 0.0) as inr_fit_report would.  out: device memory or
 * pinned host memory (mapped under unified addressing); read it after the
 * stream reaches this point (e.g. an event).  Asynchronous. */
INR_API inr_status inr_fit_losses(inr_model* const* models, int32_t nmodels, double* out, cudaStream_t stream);

/* Direct queries: xyz (dev) holds q global node
 * coordinates (x,y,z interleaved); out (dev) receives q x D values in data units
 * v = Phi(x) (vmax - vmin) + vmin (per channel, channels interleaved).  A query p goes to the block
 * min(max(floor(p/n), 0), B-1) per axis and x = fl32(fl32(p - o)/n) [R5];
 * inr_decode uses the one model, inr_decode_group routes among `nmodels`
 * models (a point whose block is not among them gets NaN; any number of models,
 * decoded in routed passes of <= 64 models; at most 4096 blocks in the volume,
 * else INR_ERR_UNSUPPORTED).  strict != 0
 * reports INR_ERR_DOMAIN after the fact if any coordinate lies outside
 * [0, N-1]^3 (values are still written, clamped); strict synchronizes. */
INR_API inr_status inr_decode(const inr_model* m, const float* xyz, int64_t q, float* out, int32_t strict,
                      cudaStream_t stream);
INR_API inr_status inr_decode_group(const inr_model* const* models, int32_t nmodels, const float* xyz,
                            int64_t q, float* out, int32_t strict, cudaStream_t stream);

/* Decode to grid: res[d] >= 1 samples per axis at
 * x_j = fl32(j / res_d), j < res_d (half-open, so blocks tile without
 * duplicates [R19]); value written to out[jx*os0 + jy*os1 + jz*os2 (+ c for
 * channel c of a vector field)] where os = out_stride (elements) or, if
 * out_stride is NULL, the dense x-fastest strides (D, D res0, D res0 res1).
 * If ref (dev, same layout) is non-NULL, the sum over the lattice (and
 * channels) of ((pred - ref)/(vmax - vmin))^2 is atomically added
 * to *sse_dev (dev double; caller zeroes it; many blocks may accumulate into
 * one scalar) (S:L75-83 PSNR in normalized units [R18]).  Asynchronous. */
INR_API inr_status inr_decode_grid(const inr_model* m, const int32_t res[3], float* out,
                           const int64_t* out_stride, const float* ref, double* sse_dev,
                           cudaStream_t stream);
/* The same for only the first count[d] <= res[d] lattice points per axis
 * (j_d < count_d, still at x_j = fl32(j / res_d)): a block at the upper domain
 * face whose remaining nodes N - o are fewer than n decodes res = n,
 * count = N - o, i.e. exactly its nodes (count NULL = res). */
INR_API inr_status inr_decode_grid_part(const inr_model* m, const int32_t res[3], const int32_t count[3],
                                float* out, const int64_t* out_stride, const float* ref, double* sse_dev,
                                cudaStream_t stream);

/* Min/max over the nodes of a view: atomically
 * folds into minmax_dev[2c] (min) and minmax_dev[2c+1] (max) of every channel c
 * of the view (dev floats, caller initialises to +inf/-inf).  The cross-GPU
 * all-reduce is the caller's. */
INR_API inr_status inr_value_range(const inr_view* view, float* minmax_dev, cudaStream_t stream);

/* ---- the temporal window ---- */
typedef struct inr_cache inr_cache;
/* capacity >= 1 timesteps; flags (bitmask): CACHE_HOST_RESIDENT keeps snapshots in
 * pinned host memory ("cached in system RAM") and stages them to the device
 * on decode; CACHE_FP16 stores the parameters as fp16 (half the bytes, 2x the
 * compression ratio; decode widens them back to fp32 — SURVEY §8(f) NEXT-4).
 * Otherwise snapshots stay fp32 in device memory.  Staged copies live until the
 * slot is evicted. */
enum { CACHE_HOST_RESIDENT = 1, CACHE_FP16 = 2 };
INR_API inr_status cache_create(int32_t capacity, int32_t flags, int device, inr_cache** out);
INR_API inr_status cache_destroy(inr_cache* c);
/* Copy a frozen parameter snapshot (no optimizer state) of `nblocks`
 * models as timestep `timestep` (> every cached timestep); when full,
 * the oldest timestep is evicted first and reported in *evicted_timestep
 * (-1 if none).  The source models stay usable.  Stream-ordered. */
INR_API inr_status cache_insert(inr_cache* c, int64_t timestep, inr_model* const* blocks, int32_t nblocks,
                        int64_t* evicted_timestep, cudaStream_t stream);
/* Evict the oldest timestep (INR_ERR_STATE if empty). */
INR_API inr_status cache_evict(inr_cache* c, int64_t* evicted_timestep);
INR_API inr_status cache_size(const inr_cache* c, int32_t* n);
/* Snapshot bytes currently held (device or host). */
INR_API inr_status cache_bytes(const inr_cache* c, int64_t* bytes);
/* Borrow slot i (0 = oldest): its timestep and frozen models (decode only;
 * valid until that slot is evicted; inr_fit/inr_reset on them -> INR_ERR_STATE). */
INR_API inr_status cache_get(const inr_cache* c, int32_t i, int64_t* timestep, const inr_model* const** blocks,
                     int32_t* nblocks);

/* ---- pathlines over the window (NEXT-2) ----
 * Positions are global node coordinates (float64), velocities node units per
 * unit time.  Classical RK4 with a fixed step: each window interval
 * [t_i, t_{i+1}] is split into k_i = max(1, ceil((t_{i+1} - t_i)/dt - 1e-12))
 * equal substeps; the velocity is trilinear in space (clamped indices, per
 * channel) and linear in time between the two bounding elements [R29-R31].
 * A seed ends when a substep would put its result or any RK stage position
 * outside [0, N-1]^3 (OUT_OF_DOMAIN; a seed outside at t_0 gets no vertex),
 * after max_steps substeps (MAX_STEPS), or at the window's end.
 * Outputs (device): vertices[M][max_steps + 1][5] rows (x, y, z, t, |V|) —
 * only the first counts[s] rows of seed s are written — counts[M], reasons[M].
 * Stream-ordered and asynchronous. */
enum { INR_PATH_WINDOW_EXHAUSTED = 0, INR_PATH_OUT_OF_DOMAIN = 1, INR_PATH_MAX_STEPS = 2 };
/* Trace on explicit velocity grids: grids (host array of ngrids >= 2 device
 * pointers) each [dims2][dims1][dims0][3] fp32, channels interleaved, at
 * strictly increasing times (host); every value is multiplied by sign. */
INR_API inr_status inr_trace_grids(const float* const* grids, const double* times, int32_t ngrids,
                           const int64_t dims[3], double sign, const double* seeds, int32_t nseeds, double dt,
                           int32_t max_steps, double* vertices, int32_t* counts, int32_t* reasons,
                           cudaStream_t stream);
/* Trace over a cached window of vector-field (out_dim 3) models, each element
 * holding every block of the volume, at times = the cached timesteps.
 * window_ops: INR_WINDOW_REVERSE (element i -> W-1-i, time tau_i = t_{W-1} -
 * t_{W-1-i}) and/or INR_WINDOW_NEGATE (every value times -1) — so
 * INR_WINDOW_REVERSE | INR_WINDOW_NEGATE is the paper's backward tracing
 * pathline(negate(reverse(W))).  Elements are decoded to the
 * global grid on demand, at most two resident (2 x 12 N^3 bytes of
 * stream-ordered scratch). */
enum { INR_WINDOW_REVERSE = 1, INR_WINDOW_NEGATE = 2 };
INR_API inr_status inr_pathlines(const inr_cache* c, int32_t window_ops, const double* seeds, int32_t nseeds,
                         double dt, int32_t max_steps, double* vertices, int32_t* counts, int32_t* reasons,
                         cudaStream_t stream);

/* ---- direct-query volume rendering (NEXT-3) ----
 * Scalar-field (out_dim 1) models only.  World coordinates = global node
 * coordinates.  The optical model and sampling are DESIGN.md R32-R35:
 *   pixel (px, py), py = 0 the top row, ray eye + t d with d = normalize(f +
 *   a r + b u), a = (2 (px + .5)/W - 1) tan(fovy/2) W/H, b = (1 - 2 (py + .5)/H)
 *   tan(fovy/2), f = normalize(look - eye), r = normalize(f x up), u = r x f;
 *   samples at t_k = (k + 0.5) step (global along the ray), a brick [lo, hi]
 *   takes t_enter <= t_k < t_exit; value v = the DNR query at the fp32-rounded
 *   position (routed as inr_decode_group); s = clamp((v - vmin)/(vmax - vmin));
 *   RGBA = piecewise-linear transfer function; a = 1 - (1 - a_tf)^(step/base_step);
 *   C += (1 - A) a c, A += (1 - A) a, stop when A >= stop_alpha. */
#define INR_TF_MAX_POINTS 16
typedef struct {
  double eye[3], look[3], up[3];
  double fovy_deg;
  int32_t width, height;
} inr_camera;
typedef struct {
  int32_t npoints;                       /* 2..INR_TF_MAX_POINTS, s strictly increasing in [0, 1] */
  float s[INR_TF_MAX_POINTS];
  float rgba[INR_TF_MAX_POINTS][4];      /* colour and opacity in [0, 1] */
  double vmin, vmax;                     /* data values mapped to s = 0 and 1 */
  double base_step;                      /* the step the opacities are defined for */
} inr_transfer_fn;
typedef struct inr_renderer inr_renderer;
/* Bind nmodels (<= 64) models of one volume (one rank's blocks) and build the
 * macro-cell grid: cells^3 cells per block, each cell's value range from a
 * (4 cells)^3 probe lattice decoded per block (cells of an axis take their own
 * probes and the neighbouring probe across each face), padded by pad (data
 * units) ("macro-cell acceleration structure").  The models
 * must outlive the renderer and stay frozen while it is used. */
INR_API inr_status inr_renderer_create(const inr_model* const* models, int32_t nmodels, int32_t cells, double pad,
                               cudaStream_t stream, inr_renderer** out);
INR_API inr_status inr_renderer_destroy(inr_renderer* r);
/* Ray-march the brick [brick_lo, brick_hi] (normally this rank's core box)
 * by sample streaming: waves of up to 64 samples per live ray are generated
 * (samples in macro-cells whose transfer-function opacity is 0 over their
 * range are skipped when use_macrocells != 0), decoded with the tensor-core
 * query path, and composited.  fragments (dev) [H*W][5] = (C_r, C_g, C_b, A,
 * t_enter), t_enter = +inf for rays that miss the brick.  Synchronizes stream
 * once per wave. */
INR_API inr_status inr_render(inr_renderer* r, const inr_camera* cam, const inr_transfer_fn* tf,
                      const double brick_lo[3], const double brick_hi[3], double step, double stop_alpha,
                      int32_t use_macrocells, float* fragments, cudaStream_t stream);
/* Samples evaluated / skipped and waves of the last inr_render. */
INR_API inr_status inr_render_stats(const inr_renderer* r, int64_t* evaluated, int64_t* skipped, int32_t* waves);
/* Sort-last compositing: fragments (dev) [nfrag][npixels][5] from
 * nfrag <= 64 bricks, front to back by t_enter per pixel, then the background
 * bg (host RGB): image (dev) [npixels][4] RGBA. */
INR_API inr_status inr_composite(const float* fragments, int32_t nfrag, int64_t npixels, const float bg[3],
                         float* image, cudaStream_t stream);

/* ---- peer memory (a18 fused with the decode over NVLink) ----
 * inr_ipc_handle: the CUDA IPC handle (64 bytes) of the allocation holding the
 * device pointer ptr and ptr's offset in it; inr_ipc_open (in another process):
 * maps it on `device` with peer access (*ptr = mapping + offset; *base for
 * inr_ipc_close).  With it every rank decodes its blocks straight into rank 0's
 * global volume (inr_decode_grid with out = the peer pointer): the decode
 * kernels' stores are the gather. */
INR_API inr_status inr_ipc_handle(const void* ptr, unsigned char handle[64], int64_t* offset);
INR_API inr_status inr_ipc_open(const unsigned char handle[64], int64_t offset, int device, void** ptr, void** base);
INR_API inr_status inr_ipc_close(void* base);

/* ---- parity / test surface ---- */
/* Copy n = inr_param_count floats of parameters / last-step gradients / Adam m /
 * Adam v in the declared order (synchronous). */
INR_API inr_status inr_get_params(const inr_model* m, float* host, int64_t n);
INR_API inr_status inr_set_params(inr_model* m, const float* host, int64_t n);
INR_API inr_status inr_get_grads(const inr_model* m, float* host, int64_t n);
INR_API inr_status inr_get_adam_state(const inr_model* m, float* m_host, float* v_host, int64_t n);
/* Encode q block-normalized coordinates x01 (dev, q x 3): corner indices
 * idx (dev, q x L x 8 uint32, level-local table index) and/or features
 * feat (dev, q x L*F fp32); either may be NULL.  Asynchronous. */
INR_API inr_status inr_debug_encode(const inr_model* m, const float* x01, int64_t q, uint32_t* idx, float* feat,
                            cudaStream_t stream);
/* Network output Phi(x) in normalized units for q block-normalized coordinates
 * (dev q x 3 -> dev q x D), in the model's configured precision.  Asynchronous. */
INR_API inr_status inr_debug_forward(const inr_model* m, const float* x01, int64_t q, float* y, cudaStream_t stream);
/* Kernel timing for benchmarks: while enabled, every kernel the library
 * launches is bracketed by CUDA events recorded on its launching stream.  A
 * multi-step fit without probing is then captured as ONE CUDA graph of all its
 * steps (event records included as graph nodes), instead of the one-step graph
 * replayed per step when profiling is off; the kernels and their order are the
 * same.  inr_profile_read synchronizes and returns the summed device time (ms)
 * and launch count of one kernel class: "step_begin", "fit_fp32", "encode_fwd",
 * "prep_image", "mlp_tc", "encode_bwd", "adam", "decode_grid", "decode_query",
 * "probe", "range", "pathline".  inr_profile_enable(1) also clears previous
 * records. */
INR_API inr_status inr_profile_enable(int32_t on);
INR_API inr_status inr_profile_read(const char* kernel, double* total_ms, int64_t* launches);
/* Device time (ms) from the first recorded kernel start to the last recorded
 * kernel end since inr_profile_enable(1), i.e. the span of the timed work
 * without host-side launch or graph-capture time. */
INR_API inr_status inr_profile_span(double* span_ms);
/* Number of kernels this library has launched since load (bench evidence). */
INR_API int64_t inr_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* INR_H */
