// kernels_path.cu — windowed RK4 pathlines over decoded velocity grids (NEXT-2):
//   P:L411 "integral curves of a time-varying vector field ... Euler or
//   Runge-Kutta methods"; P:L422 the field "decoded back to the original mesh
//   grid ... on an on-demand basis, allowing for the retention of only two
//   additional copies of the mesh grid"; S:L495-512 (rk4_step, trace_pathlines).
//
// One thread per seed.  The host walks the window one interval [t_a, t_b] at a
// time with the two bounding grids resident; a launch advances every live seed
// through the interval's k equal substeps (no RK stage straddles a window
// element, R30).  The seed's state is its last vertex, so successive
// launches need no other carry.  Arithmetic is float64 with explicit _rn
// intrinsics (no FMA contraction) in the order DESIGN.md R31 fixes: trilinear
// per channel in corner order with weights ((1 * w_x) * w_y) * w_z, linear in
// time, classical RK4; the grids hold fp32 values in node units per time unit.
// The velocity gathers are random per seed (8 corners x 3 channels x 2 grids
// per stage) and the grids are 2 x 12 N^3 bytes, so the kernel is bound by
// gather latency from L2/HBM; seeds are few (thousands) in the paper's use.
#include <algorithm>
#include <cmath>

#include "launch.h"

namespace inr {

constexpr int kPathThreads = 128;

struct PathGrid {
  const float* g0;
  const float* g1;
  long long n[3];   // nodes per axis (x, y, z); grid[((z ny + y) nx + x) 3 + c]
};

__device__ __forceinline__ void trilinear3(const float* __restrict__ g, const long long n[3], const double p[3],
                                           double out[3]) {
  long long i0[3], i1[3];
  double f[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double r = fmin(fmax(p[d], 0.0), (double)(n[d] - 1));   // clamp to the domain
    i0[d] = (long long)floor(r);
    f[d] = __dsub_rn(r, (double)i0[d]);
    i1[d] = min(i0[d] + 1, n[d] - 1);
  }
  out[0] = out[1] = out[2] = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const long long ix = (c & 1) ? i1[0] : i0[0];
    const long long iy = (c & 2) ? i1[1] : i0[1];
    const long long iz = (c & 4) ? i1[2] : i0[2];
    double w = 1.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) w = __dmul_rn(w, ((c >> d) & 1) ? f[d] : __dsub_rn(1.0, f[d]));
    const float* v = g + ((iz * n[1] + iy) * n[0] + ix) * 3;
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) out[ch] = __dadd_rn(out[ch], __dmul_rn(w, (double)__ldg(v + ch)));
  }
}

// sign * ((1 - alpha) V_a(p) + alpha V_b(p))
__device__ __forceinline__ void velocity(const PathGrid& G, double alpha, double sign, const double p[3],
                                         double v[3]) {
  double v0[3], v1[3];
  trilinear3(G.g0, G.n, p, v0);
  trilinear3(G.g1, G.n, p, v1);
  const double oa = __dsub_rn(1.0, alpha);
#pragma unroll
  for (int c = 0; c < 3; ++c) v[c] = __dmul_rn(sign, __dadd_rn(__dmul_rn(oa, v0[c]), __dmul_rn(alpha, v1[c])));
}

__device__ __forceinline__ bool in_domain(const PathGrid& G, const double q[3]) {
  bool ok = true;
#pragma unroll
  for (int d = 0; d < 3; ++d) ok &= q[d] >= 0.0 && q[d] <= (double)(G.n[d] - 1);
  return ok;
}

__device__ __forceinline__ double speed(const double v[3]) {
  return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(v[0], v[0]), __dmul_rn(v[1], v[1])), __dmul_rn(v[2], v[2])));
}

__device__ __forceinline__ void put_vertex(double* __restrict__ vert, const double p[3], double t, double s) {
  vert[0] = p[0]; vert[1] = p[1]; vert[2] = p[2]; vert[3] = t; vert[4] = s;
}

// First vertex of every seed (or OUT_OF_DOMAIN with no vertex).
__global__ void __launch_bounds__(kPathThreads) path_init_kernel(PathGrid G, double t0, double sign,
                                                                 const double* __restrict__ seeds, int M, int stride,
                                                                 double* __restrict__ vert, int* __restrict__ count,
                                                                 int* __restrict__ reason) {
  const int s = blockIdx.x * kPathThreads + threadIdx.x;
  if (s >= M) return;
  const double p[3] = {seeds[3 * (size_t)s], seeds[3 * (size_t)s + 1], seeds[3 * (size_t)s + 2]};
  if (!in_domain(G, p)) {
    count[s] = 0;
    reason[s] = 1;   // out of domain
    return;
  }
  double v[3];
  velocity(G, 0.0, sign, p, v);
  put_vertex(vert + (size_t)s * stride * 5, p, t0, speed(v));
  count[s] = 1;
  reason[s] = -1;   // running
}

// Advance every live seed across [ta, tb] in k substeps of h.
__global__ void __launch_bounds__(kPathThreads) path_interval_kernel(PathGrid G, double ta, double tb, double h, int k,
                                                                     double sign, int max_steps, int M, int stride,
                                                                     double* __restrict__ vert, int* __restrict__ count,
                                                                     int* __restrict__ reason) {
  const int s = blockIdx.x * kPathThreads + threadIdx.x;
  if (s >= M || reason[s] != -1) return;
  double* vs = vert + (size_t)s * stride * 5;
  int cnt = count[s];
  double p[3] = {vs[(cnt - 1) * 5], vs[(cnt - 1) * 5 + 1], vs[(cnt - 1) * 5 + 2]};
  const double span = __dsub_rn(tb, ta);
  int why = -1;
  for (int j = 0; j < k; ++j) {
    if (cnt - 1 >= max_steps) { why = 2; break; }
    const double t = __dadd_rn(ta, __dmul_rn((double)j, h));
    const double hh = __dmul_rn(0.5, h);
    const double tm = __dadd_rn(t, hh), te = __dadd_rn(t, h);
    double k1[3], k2[3], k3[3], k4[3], p2[3], p3[3], p4[3], pn[3];
    velocity(G, __ddiv_rn(__dsub_rn(t, ta), span), sign, p, k1);
#pragma unroll
    for (int d = 0; d < 3; ++d) p2[d] = __dadd_rn(p[d], __dmul_rn(hh, k1[d]));
    velocity(G, __ddiv_rn(__dsub_rn(tm, ta), span), sign, p2, k2);
#pragma unroll
    for (int d = 0; d < 3; ++d) p3[d] = __dadd_rn(p[d], __dmul_rn(hh, k2[d]));
    velocity(G, __ddiv_rn(__dsub_rn(tm, ta), span), sign, p3, k3);
#pragma unroll
    for (int d = 0; d < 3; ++d) p4[d] = __dadd_rn(p[d], __dmul_rn(h, k3[d]));
    velocity(G, __ddiv_rn(__dsub_rn(te, ta), span), sign, p4, k4);
    const double h6 = __ddiv_rn(h, 6.0);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double sum = __dadd_rn(__dadd_rn(__dadd_rn(k1[d], __dmul_rn(2.0, k2[d])), __dmul_rn(2.0, k3[d])), k4[d]);
      pn[d] = __dadd_rn(p[d], __dmul_rn(h6, sum));
    }
    if (!(in_domain(G, pn) && in_domain(G, p2) && in_domain(G, p3) && in_domain(G, p4))) { why = 1; break; }
#pragma unroll
    for (int d = 0; d < 3; ++d) p[d] = pn[d];
    const double tn = __dadd_rn(ta, __dmul_rn((double)(j + 1), h));
    double v[3];
    velocity(G, __ddiv_rn(__dsub_rn(tn, ta), span), sign, p, v);
    put_vertex(vs + (size_t)cnt * 5, p, tn, speed(v));
    ++cnt;
  }
  count[s] = cnt;
  reason[s] = why;
}

__global__ void path_finish_kernel(int M, int* __restrict__ reason) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < M && reason[s] == -1) reason[s] = 0;   // window exhausted
}

static PathGrid path_grid(const float* g0, const float* g1, const long long n[3]) {
  PathGrid G;
  G.g0 = g0;
  G.g1 = g1;
  for (int d = 0; d < 3; ++d) G.n[d] = n[d];
  return G;
}

void launch_path_init(const float* g0, const float* g1, const long long n[3], double t0, double sign,
                      const double* seeds, int M, int max_steps, double* vert, int* count, int* reason,
                      cudaStream_t st) {
  path_init_kernel<<<(M + kPathThreads - 1) / kPathThreads, kPathThreads, 0, st>>>(
      path_grid(g0, g1, n), t0, sign, seeds, M, max_steps + 1, vert, count, reason);
  count_launch();
}

void launch_path_interval(const float* g0, const float* g1, const long long n[3], double ta, double tb, double dt,
                          double sign, int max_steps, int M, double* vert, int* count, int* reason, cudaStream_t st) {
  const int k = std::max(1, (int)std::ceil((tb - ta) / dt - 1e-12));
  const double h = (tb - ta) / k;
  path_interval_kernel<<<(M + kPathThreads - 1) / kPathThreads, kPathThreads, 0, st>>>(
      path_grid(g0, g1, n), ta, tb, h, k, sign, max_steps, M, max_steps + 1, vert, count, reason);
  count_launch();
}

void launch_path_finish(int M, int* reason, cudaStream_t st) {
  path_finish_kernel<<<(M + 255) / 256, 256, 0, st>>>(M, reason);
  count_launch();
}

}  // namespace inr
