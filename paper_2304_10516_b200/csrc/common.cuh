// common.cuh — device-side building blocks of libinr (sm_100a).
//
// Shared by the fit, decode, Adam and debug kernels of THIS library only (the
// oracle in /oracle is an independent implementation and shares nothing).
//   * Philox4x32-10 (Salmon et al. SC'11) for init / sample streams [R8, R14]
//   * hash-grid level lookup, corner indices and trilinear weights
//      with the pinned fp32 index
//     arithmetic of DESIGN.md R4/R20 (__fmul_rn, floorf, no contraction)
//   * the block sampler: uniform / boundary samples, trilinear targets with
//     clamp-to-edge, value normalization (R5-R9)
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace inr {

constexpr int kWidth = 64;        // MLP width of this build
constexpr int kMaxLevels = 32;
constexpr int kMaxLayers = 9;     // H <= 8 hidden layers => <= 9 weight matrices
constexpr int kMaxGroup = 64;     // models per fused launch
constexpr int kMaxD = 3;          // output channels: scalar (1) or vector (3) fields
constexpr uint32_t kPrimeY = 2654435761u;
constexpr uint32_t kPrimeZ = 805459861u;
constexpr int kFixedShift = 40;   // deterministic mode: int64 fixed point with 2^-40 resolution [R21]

struct LevelInfo {
  uint32_t res;     // N_l
  uint32_t size;    // S_l entries
  uint32_t dense;   // 1 if (N_l+1)^3 <= T
  uint32_t pad;
  int64_t offset;   // float offset of the level table in the parameter vector
};

constexpr int kMaxTensors = kMaxLevels + 2 * kMaxLayers;
constexpr int kTensorAlign = 64;  // internal tensor offsets are multiples of 64 floats (256 B)

// Per-configuration constants (same for every model of a group); passed by value.
// Parameters are stored in the declared order (tables by level, then W_0, b_0,
// ..., W_H, b_H) but every tensor starts at a 256-B aligned internal offset, so
// an F = 2 entry pair {2k, 2k+1} is one 16-B aligned vector (paired corners).
struct NetDesc {
  int L, F, H, LF, D, bias;
  uint32_t table_mask;              // T - 1
  int64_t nparams;                  // internal (padded) parameter count
  int64_t ndecl;                    // declared parameter count
  int ntensors;
  int64_t t_off[kMaxTensors];       // internal offset of tensor t
  int64_t t_decl[kMaxTensors];      // declared offset of tensor t
  int64_t t_len[kMaxTensors];
  int t_fan_in[kMaxTensors];        // 0: table, > 0: weight matrix (He-uniform), -1: bias
  int64_t w_off[kMaxLayers];        // float offset of W_k (row-major [out][in])
  int64_t b_off[kMaxLayers];        // float offset of b_k (or -1)
  int in_dim[kMaxLayers], out_dim[kMaxLayers];
  LevelInfo lv[kMaxLevels];
};

// Per-model device state (passed by value in kernel parameters).
struct ModelDev {
  float* params;
  float* grads;
  float* adam_m;
  float* adam_v;
  unsigned long long* grads_fx;     // deterministic mode accumulators (or null)
  long long* step_total;            // Adam steps taken (device copy)
  long long* step_cur;              // the step being executed
  double* acc;                      // [0] sum|y-t| uniform, [1] boundary, [2] probe SSE
  int* flag;                        // non-finite flag
  const float* vbase;               // training view
  long long vlo[3], vstride[3];
  int o[3], n[3], N[3];
  uint32_t block_id;
  int nfaces;
  int faces[6];
  float vmin[kMaxD], vrange[kMaxD], inv_range[kMaxD];   // per-channel normalization (inv_range 0: constant)
  uint32_t k0, k1u, k1b;            // Philox keys (seed_lo, seed_hi ^ 1), (seed_lo, seed_hi ^ 2) [R8]
  // rectilinear mesh (R36): the block's node coordinates X[o .. o + mesh_n - 1] per axis
  // (device) and its physical box [plo, plo + pspan]; mesh[0] == null: uniform mesh
  const double* mesh[3];
  int mesh_n[3];
  double plo[3], pspan[3];
};

// Rectilinear (R36): local cell i (clamped to the block's cells) and fraction of the
// physical coordinate P on axis d, by binary search over the block's nodes.
__device__ __forceinline__ int mesh_cell(const ModelDev& md, int d, double P, double& frac) {
  const double* X = md.mesh[d];
  const int m = md.mesh_n[d];
  if (m < 2) { frac = 0.0; return 0; }
  int lo = 0, hi = m - 1;               // invariant X[lo] <= P < X[hi] (when inside)
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (X[mid] <= P) lo = mid; else hi = mid;
  }
  frac = __ddiv_rn(__dsub_rn(P, X[lo]), __dsub_rn(X[lo + 1], X[lo]));
  return lo;
}

// Rectilinear: block-normalized coordinate of a physical coordinate.
__device__ __forceinline__ float mesh_x(const ModelDev& md, int d, double P) {
  return md.pspan[d] > 0.0 ? (float)__ddiv_rn(__dsub_rn(P, md.plo[d]), md.pspan[d]) : 0.f;
}

// Rectilinear: the physical coordinate of continuous global node index p (float)
// routed to this block: the mesh's piecewise-linear map on the block's nodes.
__device__ __forceinline__ double mesh_physical(const ModelDev& md, int d, float p) {
  const int m = md.mesh_n[d];
  const double* X = md.mesh[d];
  if (m < 2) return X[0];
  const double r = fmin(fmax((double)p - (double)md.o[d], 0.0), (double)(m - 1));
  const int i = min((int)floor(r), m - 2);
  return __dadd_rn(X[i], __dmul_rn(__dsub_rn(r, (double)i), __dsub_rn(X[i + 1], X[i])));
}

// --------------------------------------------------------------- Philox4x32-10
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                     uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  return {c0, c1, c2, c3};
}

__device__ __forceinline__ float u01(uint32_t u) { return (float)(u >> 8) * 5.9604644775390625e-08f; }

// Uniform sample i of (block, step) on stream 1; boundary sample j on stream 2 (R8, R9).
__device__ __forceinline__ void draw_sample(const ModelDev& md, int i, int B_u, uint32_t step, float x[3]) {
  const uint32_t k0 = md.k0, k1u = md.k1u, k1b = md.k1b;
  if (i < B_u) {
    U4 u = philox((uint32_t)i, step, md.block_id, 0u, k0, k1u);
    x[0] = u01(u.x); x[1] = u01(u.y); x[2] = u01(u.z);
  } else {
    U4 u = philox((uint32_t)(i - B_u), step, md.block_id, 0u, k0, k1b);
    uint32_t sel = (uint32_t)(((unsigned long long)(u.x >> 8) * (unsigned long long)md.nfaces) >> 24);
    int face = md.faces[sel];
    int d = face >> 1;
    float a = u01(u.y), b = u01(u.z);
    int e0 = d == 0 ? 1 : 0, e1 = d == 2 ? 1 : 2;
    x[d] = (float)(face & 1);
    x[e0] = a;
    x[e1] = b;
  }
}

// Trilinear interpolation of the view at r = o + x n (node units), clamp-to-edge,
// then normalization with the global range, per channel for
// vector fields (channel c of a node at +c).
template <int D>
__device__ __forceinline__ void sample_target(const ModelDev& md, const float x[3], float t[D]) {
  int i0[3], i1[3];
  float f[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    if (md.mesh[0]) {   // rectilinear (R36): P = P_lo + x (P_hi - P_lo), located in the block's cells
      double fr;
      const int c = mesh_cell(md, d, __dadd_rn(md.plo[d], __dmul_rn((double)x[d], md.pspan[d])), fr);
      i0[d] = md.o[d] + c;
      f[d] = fminf(fmaxf((float)fr, 0.f), 1.f);
      i1[d] = f[d] > 0.f ? i0[d] + 1 : i0[d];
      continue;
    }
    float r = __fadd_rn((float)md.o[d], __fmul_rn(x[d], (float)md.n[d]));
    r = fminf(fmaxf(r, 0.f), (float)(md.N[d] - 1));
    float fl = floorf(r);
    i0[d] = (int)fl;
    f[d] = __fsub_rn(r, fl);
    // the upper node only when it has weight: on the block's far face (r = o + n)
    // the view may end at node o + n (its contract), so node o + n + 1 must not be read
    i1[d] = f[d] > 0.f ? min(i0[d] + 1, md.N[d] - 1) : i0[d];
  }
  float acc[D];
#pragma unroll
  for (int c = 0; c < D; ++c) acc[c] = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    int ix = (k & 1) ? i1[0] : i0[0];
    int iy = (k & 2) ? i1[1] : i0[1];
    int iz = (k & 4) ? i1[2] : i0[2];
    float w = ((k & 1) ? f[0] : 1.f - f[0]) * ((k & 2) ? f[1] : 1.f - f[1]) * ((k & 4) ? f[2] : 1.f - f[2]);
    long long off = (ix - md.vlo[0]) * md.vstride[0] + (iy - md.vlo[1]) * md.vstride[1] +
                    (iz - md.vlo[2]) * md.vstride[2];
#pragma unroll
    for (int c = 0; c < D; ++c) acc[c] = fmaf(w, __ldg(md.vbase + off + c), acc[c]);
  }
#pragma unroll
  for (int c = 0; c < D; ++c) t[c] = (acc[c] - md.vmin[c]) * md.inv_range[c];
}

// ------------------------------------------------------------- level lookup
// pos_d = fl32(x_d * N_l); i_d = min(floor(pos_d), N_l - 1); w_d = pos_d - i_d (R4, R20).
struct Cell {
  uint32_t i[3];
  float w[3];
};

__device__ __forceinline__ Cell level_cell(const float x[3], uint32_t res) {
  Cell c;
  float N = (float)res;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    float xc = fminf(fmaxf(x[d], 0.f), 1.f);
    float p = __fmul_rn(xc, N);
    int i = min((int)floorf(p), (int)res - 1);
    c.i[d] = (uint32_t)i;
    c.w[d] = __fsub_rn(p, (float)i);
  }
  return c;
}

// Table index of corner c (bit0 -> x, bit1 -> y, bit2 -> z) (R1, R2).
__device__ __forceinline__ uint32_t corner_index(const Cell& cell, int c, const LevelInfo& lv, uint32_t mask) {
  uint32_t vx = cell.i[0] + (c & 1), vy = cell.i[1] + ((c >> 1) & 1), vz = cell.i[2] + ((c >> 2) & 1);
  if (lv.dense) {
    uint32_t s = lv.res + 1;
    return vx + s * (vy + s * vz);
  }
  return (vx ^ (vy * kPrimeY) ^ (vz * kPrimeZ)) & mask;
}

__device__ __forceinline__ float corner_weight(const Cell& cell, int c) {
  float wx = (c & 1) ? cell.w[0] : 1.f - cell.w[0];
  float wy = (c & 2) ? cell.w[1] : 1.f - cell.w[1];
  float wz = (c & 4) ? cell.w[2] : 1.f - cell.w[2];
  return wx * wy * wz;
}

// F-wide vector gather / accumulate helpers.
template <int F> struct FVec { float v[F]; };

template <int F>
__device__ __forceinline__ FVec<F> load_entry(const float* __restrict__ p) {
  FVec<F> r;
  if constexpr (F == 1) { r.v[0] = __ldg(p); }
  else if constexpr (F == 2) { float2 a = __ldg(reinterpret_cast<const float2*>(p)); r.v[0] = a.x; r.v[1] = a.y; }
  else if constexpr (F == 4) { float4 a = __ldg(reinterpret_cast<const float4*>(p)); r.v[0] = a.x; r.v[1] = a.y; r.v[2] = a.z; r.v[3] = a.w; }
  else {
#pragma unroll
    for (int h = 0; h < F / 4; ++h) {
      float4 a = __ldg(reinterpret_cast<const float4*>(p) + h);
      r.v[4 * h] = a.x; r.v[4 * h + 1] = a.y; r.v[4 * h + 2] = a.z; r.v[4 * h + 3] = a.w;
    }
  }
  return r;
}

// Encode one level: feat[f] = sum_c w_c theta[idx_c][f] (summed in corner order).
// The two x-neighbour corners (c, c+1) of a cell land in one aligned entry pair
// {2k, 2k+1} whenever idx_c ^ idx_{c+1} == 1 (always for even x on hashed
// levels, since h(x+1) = h(x) ^ 1 there; for even idx on dense levels): then one
// 16-B (F = 2) or 8-B (F = 1) load fetches both.
template <int F>
__device__ __forceinline__ void encode_level(const float* __restrict__ params, const LevelInfo& lv, uint32_t mask,
                                             const float x[3], float feat[F]) {
  Cell cell = level_cell(x, lv.res);
  const float* tab = params + lv.offset;
#pragma unroll
  for (int f = 0; f < F; ++f) feat[f] = 0.f;
#pragma unroll
  for (int c = 0; c < 8; c += 2) {
    const uint32_t i0 = corner_index(cell, c, lv, mask), i1 = corner_index(cell, c + 1, lv, mask);
    const float w0 = corner_weight(cell, c), w1 = corner_weight(cell, c + 1);
    FVec<F> e0, e1;
    if constexpr (F <= 2) {
      if ((i0 ^ i1) == 1u) {
        const uint32_t lo = min(i0, i1);
        FVec<2 * F> pr = load_entry<2 * F>(tab + (size_t)lo * F);
        const bool swap = i0 > i1;
#pragma unroll
        for (int f = 0; f < F; ++f) {
          e0.v[f] = swap ? pr.v[F + f] : pr.v[f];
          e1.v[f] = swap ? pr.v[f] : pr.v[F + f];
        }
      } else {
        e0 = load_entry<F>(tab + (size_t)i0 * F);
        e1 = load_entry<F>(tab + (size_t)i1 * F);
      }
    } else {
      e0 = load_entry<F>(tab + (size_t)i0 * F);
      e1 = load_entry<F>(tab + (size_t)i1 * F);
    }
#pragma unroll
    for (int f = 0; f < F; ++f) feat[f] = fmaf(w0, e0.v[f], feat[f]);
#pragma unroll
    for (int f = 0; f < F; ++f) feat[f] = fmaf(w1, e1.v[f], feat[f]);
  }
}

// Inference variant (decode): when the position is a lattice vertex of this level
// (all three fractional weights are 0, e.g. x = j/R with N_l >= R, DESIGN R19)
// only corner 0 has a non-zero weight, and it is 1: fetch that one entry.  The
// skipped corners have weight exactly 0, so for finite tables the result is
// bitwise the 8-corner sum (fma(0, v, acc) == acc).
template <int F>
__device__ __forceinline__ void encode_level_infer(const float* __restrict__ params, const LevelInfo& lv,
                                                   uint32_t mask, const float x[3], float feat[F]) {
  Cell cell = level_cell(x, lv.res);
  if (cell.w[0] == 0.f && cell.w[1] == 0.f && cell.w[2] == 0.f) {
    FVec<F> e = load_entry<F>(params + lv.offset + (size_t)corner_index(cell, 0, lv, mask) * F);
#pragma unroll
    for (int f = 0; f < F; ++f) feat[f] = fmaf(1.f, e.v[f], 0.f);
    return;
  }
  encode_level<F>(params, lv, mask, x, feat);
}

// Scatter-add of one level's gradient: dtheta[idx_c][f] += w_c dfeat[f].
__device__ __forceinline__ void red_add(float* p, float v) { atomicAdd(p, v); }

__device__ __forceinline__ void red_add_fx(unsigned long long* p, float v) {
  long long q = __double2ll_rn((double)v * (double)(1ll << kFixedShift));
  atomicAdd(p, (unsigned long long)q);
}

template <int F>
__device__ __forceinline__ void scatter_level(float* __restrict__ grads, unsigned long long* __restrict__ gfx,
                                              const LevelInfo& lv, uint32_t mask, const float x[3],
                                              const float dfeat[F]) {
  Cell cell = level_cell(x, lv.res);
#pragma unroll
  for (int c = 0; c < 8; c += 2) {
    const uint32_t i0 = corner_index(cell, c, lv, mask), i1 = corner_index(cell, c + 1, lv, mask);
    const float w0 = corner_weight(cell, c), w1 = corner_weight(cell, c + 1);
    if (gfx) {
#pragma unroll
      for (int f = 0; f < F; ++f) {
        red_add_fx(gfx + (size_t)lv.offset + (size_t)i0 * F + f, w0 * dfeat[f]);
        red_add_fx(gfx + (size_t)lv.offset + (size_t)i1 * F + f, w1 * dfeat[f]);
      }
      continue;
    }
    float* base = grads + lv.offset;
    if constexpr (F == 2) {
      if ((i0 ^ i1) == 1u) {  // both corners in one aligned 16-B entry pair: one vector red
        const bool swap = i0 > i1;
        const float wl = swap ? w1 : w0, wh = swap ? w0 : w1;
        atomicAdd(reinterpret_cast<float4*>(base + (size_t)min(i0, i1) * 2),
                  make_float4(wl * dfeat[0], wl * dfeat[1], wh * dfeat[0], wh * dfeat[1]));
      } else {
        atomicAdd(reinterpret_cast<float2*>(base + (size_t)i0 * 2), make_float2(w0 * dfeat[0], w0 * dfeat[1]));
        atomicAdd(reinterpret_cast<float2*>(base + (size_t)i1 * 2), make_float2(w1 * dfeat[0], w1 * dfeat[1]));
      }
    } else if constexpr (F == 1) {
      if ((i0 ^ i1) == 1u) {
        const bool swap = i0 > i1;
        atomicAdd(reinterpret_cast<float2*>(base + min(i0, i1)),
                  swap ? make_float2(w1 * dfeat[0], w0 * dfeat[0]) : make_float2(w0 * dfeat[0], w1 * dfeat[0]));
      } else {
        atomicAdd(base + i0, w0 * dfeat[0]);
        atomicAdd(base + i1, w1 * dfeat[0]);
      }
    } else if constexpr (F == 4) {
      atomicAdd(reinterpret_cast<float4*>(base + (size_t)i0 * 4), make_float4(w0 * dfeat[0], w0 * dfeat[1], w0 * dfeat[2], w0 * dfeat[3]));
      atomicAdd(reinterpret_cast<float4*>(base + (size_t)i1 * 4), make_float4(w1 * dfeat[0], w1 * dfeat[1], w1 * dfeat[2], w1 * dfeat[3]));
    } else {
#pragma unroll
      for (int q = 0; q < F; q += 4) {
        atomicAdd(reinterpret_cast<float4*>(base + (size_t)i0 * F + q),
                  make_float4(w0 * dfeat[q], w0 * dfeat[q + 1], w0 * dfeat[q + 2], w0 * dfeat[q + 3]));
        atomicAdd(reinterpret_cast<float4*>(base + (size_t)i1 * F + q),
                  make_float4(w1 * dfeat[q], w1 * dfeat[q + 1], w1 * dfeat[q + 2], w1 * dfeat[q + 3]));
      }
    }
  }
}

__device__ __forceinline__ void grad_add(float* grads, unsigned long long* gfx, size_t off, float v) {
  if (gfx) red_add_fx(gfx + off, v);
  else atomicAdd(grads + off, v);
}

}  // namespace inr
