// kernels_render.cu — sort-last direct-query volume rendering of a DNR (NEXT-3):
//   P:L268, "sample-streaming algorithm and the macro-cell
//   acceleration structure ... sort-last parallel rendering system ... does not
//   require decoding the neural representation back to a grid".
//
// Sample streaming (host loop in inr_runtime.cu, one sync per wave):
//   gen_kernel        every live ray emits its next <= S non-empty samples
//                     (macro-cells whose transfer-function opacity is 0 over their
//                     value range are skipped without a query), compacted into
//                     one dense query list (warp-aggregated atomics)
//   [decode]          the library's bucketed tensor-core query decode
//   composite_kernel  front-to-back emission-absorption of each ray's samples,
//                     early termination
// Macro-cells: mc_reduce_kernel folds a probe lattice (decoded on tensor cores)
// into per-cell value ranges, mc_mark_kernel marks cells empty for a TF.
// sort-last: blend_kernel sorts each pixel's fragments by entry depth.
// Arithmetic of the ray setup and t is float64 (R32-R35); sample
// positions are rounded to fp32 as every query is; colours are fp32.
#include <algorithm>

#include "launch.h"
#include "render.cuh"

namespace inr {

// ---------------------------------------------------------------- macro-cells
// probes: per slot a dense [R][R][R] lattice at x_j = j / R, R = cells * P.
// Cell c of an axis takes probes [cP - 1, (c + 1) P] (clamped): its own and
// the neighbours across both faces.
__global__ void mc_reduce_kernel(const float* __restrict__ probes, int nslots, int cells, int P, float pad,
                                 float2* __restrict__ range) {
  const long long ncell = (long long)cells * cells * cells;
  const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (id >= ncell * nslots) return;
  const int slot = (int)(id / ncell);
  const long long c = id - slot * ncell;
  const int cx = (int)(c % cells), cy = (int)((c / cells) % cells), cz = (int)(c / ((long long)cells * cells));
  const int R = cells * P;
  const float* pr = probes + (size_t)slot * R * R * R;
  float lo = __int_as_float(0x7f800000), hi = -lo;
  const int x0 = max(cx * P - 1, 0), x1 = min((cx + 1) * P, R - 1);
  const int y0 = max(cy * P - 1, 0), y1 = min((cy + 1) * P, R - 1);
  const int z0 = max(cz * P - 1, 0), z1 = min((cz + 1) * P, R - 1);
  for (int z = z0; z <= z1; ++z)
    for (int y = y0; y <= y1; ++y)
      for (int x = x0; x <= x1; ++x) {
        const float v = __ldg(pr + ((size_t)z * R + y) * R + x);
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
      }
  range[id] = make_float2(lo - pad, hi + pad);
}

__device__ __forceinline__ float tf_alpha_max(const RenderTF& tf, float s0, float s1) {
  // piecewise linear: the maximum over [s0, s1] is at an end or a control point inside
  float m = fmaxf(tf_eval(tf, s0).w, tf_eval(tf, s1).w);
  for (int i = 0; i < tf.n; ++i)
    if (tf.s[i] > s0 && tf.s[i] < s1) m = fmaxf(m, tf.rgba[i][3]);
  return m;
}

__global__ void mc_mark_kernel(const float2* __restrict__ range, long long n, RenderTF tf,
                               uint8_t* __restrict__ empty) {
  const long long id = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (id >= n) return;
  const float2 r = range[id];
  const float s0 = tf_norm(tf, r.x), s1 = tf_norm(tf, r.y);
  empty[id] = tf_alpha_max(tf, s0, s1) == 0.f;
}

// ------------------------------------------------------------------ rays
__global__ void ray_init_kernel(RenderArgs a, RayState rs) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.npix) return;
  const int px = i % a.width, py = i / a.width;
  // the oracle's operation order, no contraction (R33)
  const double ax = __dmul_rn(__dmul_rn(__dsub_rn(__ddiv_rn(__dmul_rn(2.0, px + 0.5), (double)a.width), 1.0), a.th),
                              __ddiv_rn((double)a.width, (double)a.height));
  const double by = __dmul_rn(__dsub_rn(1.0, __ddiv_rn(__dmul_rn(2.0, py + 0.5), (double)a.height)), a.th);
  double d[3];
  for (int c = 0; c < 3; ++c) d[c] = __dadd_rn(__dadd_rn(a.f[c], __dmul_rn(ax, a.r[c])), __dmul_rn(by, a.u[c]));
  const double nd = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(d[0], d[0]), __dmul_rn(d[1], d[1])), __dmul_rn(d[2], d[2])));
  for (int c = 0; c < 3; ++c) d[c] = __ddiv_rn(d[c], nd);
  double t0 = 0.0, t1 = 1e300;
  bool hit = true;
  for (int c = 0; c < 3; ++c) {
    if (d[c] != 0.0) {
      const double ta = (a.lo[c] - a.eye[c]) / d[c], tb = (a.hi[c] - a.eye[c]) / d[c];
      t0 = fmax(t0, fmin(ta, tb));
      t1 = fmin(t1, fmax(ta, tb));
    } else if (!(a.lo[c] <= a.eye[c] && a.eye[c] <= a.hi[c])) {
      hit = false;
    }
  }
  hit &= t1 > t0;
  for (int c = 0; c < 3; ++c) rs.dir[3 * (size_t)i + c] = d[c];
  rs.t_exit[i] = t1;
  rs.t_enter[i] = t0;
  // first sample: one index early, the t >= t_enter test decides (as the oracle)
  rs.k[i] = hit ? (long long)fmax(0.0, ceil(t0 / a.step - 0.5) - 1.0) : 0;
  rs.live[i] = hit;
  rs.C[4 * (size_t)i] = rs.C[4 * (size_t)i + 1] = rs.C[4 * (size_t)i + 2] = rs.C[4 * (size_t)i + 3] = 0.f;
}

// Owner block of p (R5) and its macro-cell; true if the sample must be evaluated.
__device__ __forceinline__ bool sample_needed(const RenderArgs& a, const float p[3]) {
  if (!a.empty) return true;
  int bc[3], cell[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int b = (int)floorf(__fdiv_rn(p[d], (float)a.n[d]));
    bc[d] = min(max(b, 0), a.B[d] - 1);
    const float x = __fdiv_rn(__fsub_rn(p[d], (float)(bc[d] * a.n[d])), (float)a.n[d]);
    cell[d] = min(max((int)floorf(x * a.cells), 0), a.cells - 1);
  }
  const int bid = (bc[2] * a.B[1] + bc[1]) * a.B[0] + bc[0];
  const int slot = a.slot_of_block[bid];
  if (slot < 0) return true;
  const long long cid = ((long long)slot * a.cells + cell[2]) * a.cells * a.cells + (long long)cell[1] * a.cells + cell[0];
  return !a.empty[cid];
}

// Walk ray i from sample k: the next <= S needed samples (skipped cells cost no
// query).  write = false only counts; returns the index after the last visited.
__device__ __forceinline__ long long walk(const RenderArgs& a, const RayState& rs, int i, long long k, int S,
                                          int& cnt, unsigned long long& nskip, float* __restrict__ out) {
  const double t0 = rs.t_enter[i], t1 = rs.t_exit[i];
  const double d[3] = {rs.dir[3 * (size_t)i], rs.dir[3 * (size_t)i + 1], rs.dir[3 * (size_t)i + 2]};
  cnt = 0;
  nskip = 0;
  while (cnt < S) {
    const double t = (k + 0.5) * a.step;
    if (t >= t1) break;
    if (t >= t0) {
      float p[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) p[c] = (float)__dadd_rn(a.eye[c], __dmul_rn(t, d[c]));
      if (sample_needed(a, p)) {
        if (out) {
#pragma unroll
          for (int c = 0; c < 3; ++c) out[3 * (size_t)cnt + c] = p[c];
        }
        ++cnt;
      } else {
        ++nskip;
      }
    }
    ++k;
  }
  return k;
}

__global__ void gen_kernel(RenderArgs a, RayState rs, int S, float* __restrict__ qxyz, int* __restrict__ qcount,
                           int* __restrict__ base, int* __restrict__ nq, unsigned long long* __restrict__ skipped) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const bool mine = i < a.npix && rs.live[i];
  int cnt = 0;
  unsigned long long nskip = 0;
  long long k0 = 0, k1 = 0;
  if (mine) {
    k0 = rs.k[i];
    k1 = walk(a, rs, i, k0, S, cnt, nskip, nullptr);       // pass 1: count
  }
  // dense compaction: warp inclusive scan, one atomic per warp
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(full, incl, o);
    if (lane >= o) incl += v;
  }
  int wbase = 0;
  if (lane == 31 && incl > 0) wbase = atomicAdd(qcount, incl);
  wbase = __shfl_sync(full, wbase, 31);
  unsigned long long ws = nskip;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ws += __shfl_xor_sync(full, ws, o);
  if (lane == 0 && ws) atomicAdd(skipped, ws);
  if (i >= a.npix) return;
  const int b = wbase + incl - cnt;
  base[i] = b;
  nq[i] = cnt;
  if (!mine) return;
  if (cnt > 0) {
    int c2;
    unsigned long long s2;
    walk(a, rs, i, k0, S, c2, s2, qxyz + 3 * (size_t)b);  // pass 2: write the positions
  }
  rs.k[i] = k1;
  if (cnt == 0) rs.live[i] = 0;       // no samples left in the brick
}

__global__ void composite_kernel(RenderArgs a, RayState rs, const float* __restrict__ vals,
                                 const int* __restrict__ base, const int* __restrict__ nq) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.npix || !rs.live[i]) return;
  float* Cp = rs.C + 4 * (size_t)i;
  float C0 = Cp[0], C1 = Cp[1], C2 = Cp[2], A = Cp[3];
  const int b = base[i], n = nq[i];
  for (int j = 0; j < n; ++j) {
    const float4 c = tf_eval(a.tf, tf_norm(a.tf, __ldg(vals + b + j)));
    const float al = 1.f - powf(1.f - c.w, a.exponent);   // opacity correction (R32)
    const float w = (1.f - A) * al;
    C0 += w * c.x;
    C1 += w * c.y;
    C2 += w * c.z;
    A += w;
    if (A >= a.stop_alpha) { rs.live[i] = 0; break; }
  }
  Cp[0] = C0; Cp[1] = C1; Cp[2] = C2; Cp[3] = A;
}

__global__ void fragment_kernel(RenderArgs a, RayState rs, float* __restrict__ frag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.npix) return;
  const bool hit = rs.t_exit[i] > rs.t_enter[i];
  float* f = frag + 5 * (size_t)i;
  f[0] = rs.C[4 * (size_t)i];
  f[1] = rs.C[4 * (size_t)i + 1];
  f[2] = rs.C[4 * (size_t)i + 2];
  f[3] = rs.C[4 * (size_t)i + 3];
  f[4] = hit ? (float)rs.t_enter[i] : __int_as_float(0x7f800000);
}

// sort-last: per pixel, fragments front to back by entry depth, then the background
__global__ void blend_kernel(const float* __restrict__ frags, int nfrag, long long npix, float bg0, float bg1,
                             float bg2, float* __restrict__ img) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= npix) return;
  int order[kMaxFragments];
  float depth[kMaxFragments];
  int m = 0;
  for (int j = 0; j < nfrag; ++j) {
    const float t = frags[((size_t)j * npix + i) * 5 + 4];
    int p = m++;
    while (p > 0 && depth[p - 1] > t) { depth[p] = depth[p - 1]; order[p] = order[p - 1]; --p; }   // stable
    depth[p] = t;
    order[p] = j;
  }
  float C0 = 0.f, C1 = 0.f, C2 = 0.f, A = 0.f;
  for (int q = 0; q < m; ++q) {
    if (!(depth[q] < __int_as_float(0x7f800000))) continue;   // missed brick
    const float* f = frags + ((size_t)order[q] * npix + i) * 5;
    const float w = 1.f - A;
    C0 += w * f[0];
    C1 += w * f[1];
    C2 += w * f[2];
    A += w * f[3];
  }
  const float w = 1.f - A;
  img[4 * i] = C0 + w * bg0;
  img[4 * i + 1] = C1 + w * bg1;
  img[4 * i + 2] = C2 + w * bg2;
  img[4 * i + 3] = A;
}

// ============================================================ host launchers
void launch_mc_reduce(const float* probes, int nslots, int cells, int P, float pad, float2* range, cudaStream_t st) {
  const long long n = (long long)nslots * cells * cells * cells;
  mc_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(probes, nslots, cells, P, pad, range);
  count_launch();
}

void launch_mc_mark(const float2* range, long long n, const RenderTF& tf, uint8_t* empty, cudaStream_t st) {
  mc_mark_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(range, n, tf, empty);
  count_launch();
}

void launch_ray_init(const RenderArgs& a, const RayState& rs, cudaStream_t st) {
  ray_init_kernel<<<(a.npix + 255) / 256, 256, 0, st>>>(a, rs);
  count_launch();
}

void launch_gen(const RenderArgs& a, const RayState& rs, int S, float* qxyz, int* qcount, int* base, int* nq,
                unsigned long long* skipped, cudaStream_t st) {
  gen_kernel<<<(a.npix + 127) / 128, 128, 0, st>>>(a, rs, S, qxyz, qcount, base, nq, skipped);
  count_launch();
}

void launch_composite(const RenderArgs& a, const RayState& rs, const float* vals, const int* base, const int* nq,
                      cudaStream_t st) {
  composite_kernel<<<(a.npix + 255) / 256, 256, 0, st>>>(a, rs, vals, base, nq);
  count_launch();
}

void launch_fragments(const RenderArgs& a, const RayState& rs, float* frag, cudaStream_t st) {
  fragment_kernel<<<(a.npix + 255) / 256, 256, 0, st>>>(a, rs, frag);
  count_launch();
}

void launch_blend(const float* frags, int nfrag, long long npix, const float bg[3], float* img, cudaStream_t st) {
  blend_kernel<<<(unsigned)((npix + 255) / 256), 256, 0, st>>>(frags, nfrag, npix, bg[0], bg[1], bg[2], img);
  count_launch();
}

}  // namespace inr
