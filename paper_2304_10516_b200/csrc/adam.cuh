// adam.cuh — the PyTorch-form Adam update (DESIGN R12, R13) over a
// range of one model's parameters, shared by the stand-alone Adam kernel and
// the fused backward + Adam kernel.
#pragma once
#include "common.cuh"

namespace inr {

struct AdamStep {   // per-model scalars of the current step
  float step_size, inv_sqrt_bc2, b1, b2, ob1, ob2, eps;
};

// lr_s = lr0 decay^floor(s/lr_step); bias corrections in fp64 (t = s + 1).
__device__ __forceinline__ AdamStep adam_step_scalars(long long s, double lr0, double lr_decay, long long lr_step,
                                                      double beta1, double beta2, float b1, float b2, float ob1,
                                                      float ob2, float eps) {
  const double lr = lr0 * pow(lr_decay, (double)(s / lr_step));
  const double bc1 = 1.0 - pow(beta1, (double)(s + 1));
  const double bc2 = 1.0 - pow(beta2, (double)(s + 1));
  AdamStep a;
  a.step_size = (float)(lr / bc1);
  a.inv_sqrt_bc2 = (float)(1.0 / sqrt(bc2));
  a.b1 = b1; a.b2 = b2; a.ob1 = ob1; a.ob2 = ob2; a.eps = eps;
  return a;
}

// m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2; p -= step_size m / (sqrt(v)/sqrt(bc2) + eps)
// over [i0, i1) (multiples of 4), threads t = tid, tid + nth, ...  Deterministic
// mode converts the exact int64 sums first (and stores the fp32 gradient).
// Gradients are read with .cg (L2) loads: they may have just been produced by
// other CTAs' atomics.  Returns true if a non-finite parameter appeared.
__device__ __forceinline__ float4 adam_grad4(const ModelDev& md, long long i) {
  if (md.grads_fx) {
    const float sc = 1.f / (float)(1ll << kFixedShift);
    const unsigned long long* X = md.grads_fx + 4 * i;
    const float4 gg = make_float4((float)((double)(long long)__ldcg(X) * (double)sc),
                                  (float)((double)(long long)__ldcg(X + 1) * (double)sc),
                                  (float)((double)(long long)__ldcg(X + 2) * (double)sc),
                                  (float)((double)(long long)__ldcg(X + 3) * (double)sc));
    reinterpret_cast<float4*>(md.grads)[i] = gg;
    return gg;
  }
  return __ldcg(reinterpret_cast<const float4*>(md.grads) + i);
}

__device__ __forceinline__ bool adam4(const ModelDev& md, const AdamStep& a, long long i, float4 gg) {
  float4* __restrict__ P = reinterpret_cast<float4*>(md.params);
  float4* __restrict__ M = reinterpret_cast<float4*>(md.adam_m);
  float4* __restrict__ V = reinterpret_cast<float4*>(md.adam_v);
  float4 mm = M[i];
  float4 vv = V[i];
  float4 pp = P[i];
  bool bad = false;
#define ADAM1(c)                                                                  \
  mm.c = fmaf(a.b1, mm.c, a.ob1 * gg.c);                                          \
  vv.c = fmaf(a.b2, vv.c, a.ob2 * gg.c * gg.c);                                   \
  pp.c = pp.c - a.step_size * mm.c / (sqrtf(vv.c) * a.inv_sqrt_bc2 + a.eps);      \
  bad |= !isfinite(pp.c);
  ADAM1(x) ADAM1(y) ADAM1(z) ADAM1(w)
#undef ADAM1
  M[i] = mm;
  V[i] = vv;
  P[i] = pp;
  return bad;
}

__device__ __forceinline__ bool adam_range(const ModelDev& md, const AdamStep& a, long long i0, long long i1,
                                           int tid, int nth) {
  bool bad = false;
  for (long long i = i0 / 4 + tid; i < i1 / 4; i += nth) bad |= adam4(md, a, i, adam_grad4(md, i));
  return bad;
}

// R37 touched-only variant over the tables [i0, i1) (multiples of 8): one thread
// per aligned 8-float group; a group whose 8 gradients are all zero is skipped
// (p, m, v keep their values), any other group takes the dense update.
__device__ __forceinline__ bool adam_range_sparse(const ModelDev& md, const AdamStep& a, long long i0, long long i1,
                                                  int tid, int nth) {
  bool bad = false;
  for (long long j = i0 / 8 + tid; j < i1 / 8; j += nth) {
    const float4 g0 = adam_grad4(md, 2 * j), g1 = adam_grad4(md, 2 * j + 1);
    if (g0.x == 0.f && g0.y == 0.f && g0.z == 0.f && g0.w == 0.f && g1.x == 0.f && g1.y == 0.f && g1.z == 0.f &&
        g1.w == 0.f)
      continue;
    bad |= adam4(md, a, 2 * j, g0);
    bad |= adam4(md, a, 2 * j + 1, g1);
  }
  return bad;
}

}  // namespace inr
