// render.cuh — transfer-function evaluation for the renderer kernels (NEXT-3, R32).
#pragma once
#include "launch.h"

namespace inr {

// s = clamp((v - vmin) / (vmax - vmin), 0, 1)
__device__ __forceinline__ float tf_norm(const RenderTF& tf, float v) {
  return fminf(fmaxf((v - tf.vmin) * tf.inv_range, 0.f), 1.f);
}

// piecewise-linear RGBA over sorted control points, constant beyond the ends (np.interp)
__device__ __forceinline__ float4 tf_eval(const RenderTF& tf, float s) {
  if (s <= tf.s[0]) return make_float4(tf.rgba[0][0], tf.rgba[0][1], tf.rgba[0][2], tf.rgba[0][3]);
  const int n = tf.n;
  if (s >= tf.s[n - 1])
    return make_float4(tf.rgba[n - 1][0], tf.rgba[n - 1][1], tf.rgba[n - 1][2], tf.rgba[n - 1][3]);
  int i = 0;
  while (i + 2 < n && s >= tf.s[i + 1]) ++i;
  const float w = (s - tf.s[i]) / (tf.s[i + 1] - tf.s[i]);
  float o[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) o[c] = tf.rgba[i][c] + w * (tf.rgba[i + 1][c] - tf.rgba[i][c]);
  return make_float4(o[0], o[1], o[2], o[3]);
}

}  // namespace inr
