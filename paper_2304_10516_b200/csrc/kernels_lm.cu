// kernels_lm.cu — the CUDA-core stages of the level-major fp16 fit pipeline:
//
//   sample_kernel      x ~ Philox (uniform / boundary), trilinear target      (a2-a4)
//   encode_fwd_kernel  per (level, sample): 8 corner gathers, blend -> fp16   (a5-a7)
//   [mlp_fit_kernel, kernels_tc.cu: tensor-core MLP fwd, Eq. 2, bwd]          (a8-a10)
//   encode_bwd_kernel  per (level, sample): scatter-add w_c * dfeat           (a11)
//
// The encode kernels run level-major (grid = samples x levels x models, x
// fastest), so at any time the CTAs in flight touch one or two levels of one
// block: that level's table (<= T F 4 B, 4 MB at T = 2^19, F = 2) and gradient
// stay L2-resident instead of the whole block (48.7 MB) or group (390 MB).
// Small dense levels accumulate gradients in shared memory first (their few
// entries receive every sample: global atomics would serialize on them).
#include <algorithm>

#include "common.cuh"
#include "launch.h"

namespace inr {

constexpr int kLmThreads = 256;
constexpr int kSmemAccFloats = 12288;   // levels with S_l * F <= this accumulate in smem (48 KB)
constexpr int kBwdChunk = 2048;         // samples per CTA in the backward scatter

__global__ void __launch_bounds__(kLmThreads) sample_kernel(GroupArgs g, FitScalars fs, float4* __restrict__ samples,
                                                             int Bs) {
  const int m = blockIdx.y;
  const ModelDev& md = g.md[m];
  const int total = fs.B_u + (md.nfaces > 0 ? fs.B_b : 0);
  const int i = blockIdx.x * kLmThreads + threadIdx.x;
  if (i >= total) return;
  const uint32_t step = (uint32_t)*md.step_cur;
  float x[3];
  draw_sample(md, i, fs.B_u, step, x);
  samples[(size_t)m * Bs + i] = make_float4(x[0], x[1], x[2], sample_target(md, x));
}

template <int F>
__global__ void __launch_bounds__(kLmThreads) encode_fwd_kernel(GroupArgs g, FitScalars fs,
                                                                 const float4* __restrict__ samples,
                                                                 __half* __restrict__ feat, int Bs) {
  const int m = blockIdx.z, l = blockIdx.y;
  const ModelDev& md = g.md[m];
  const int total = fs.B_u + (md.nfaces > 0 ? fs.B_b : 0);
  const int i = blockIdx.x * kLmThreads + threadIdx.x;
  if (i >= total) return;
  const float4 s = __ldg(samples + (size_t)m * Bs + i);
  const float x[3] = {s.x, s.y, s.z};
  float f[F];
  encode_level<F>(md.params, g.net.lv[l], g.net.table_mask, x, f);
  __half* o = feat + (((size_t)m * g.net.L + l) * Bs + i) * F;
  if constexpr (F == 1) {
    o[0] = __float2half_rn(f[0]);
  } else {
#pragma unroll
    for (int j = 0; j < F; j += 2) *reinterpret_cast<__half2*>(o + j) = __floats2half2_rn(f[j], f[j + 1]);
  }
}

template <int F>
__global__ void __launch_bounds__(kLmThreads) encode_bwd_kernel(GroupArgs g, FitScalars fs,
                                                                 const float4* __restrict__ samples,
                                                                 const float* __restrict__ dfeat, int Bs) {
  extern __shared__ __align__(16) unsigned char acc_raw[];
  const int m = blockIdx.z, l = blockIdx.y;
  const ModelDev& md = g.md[m];
  const LevelInfo& lv = g.net.lv[l];
  const int total = fs.B_u + (md.nfaces > 0 ? fs.B_b : 0);
  const int i0 = blockIdx.x * kBwdChunk;
  if (i0 >= total) return;
  const int i1 = min(i0 + kBwdChunk, total);
  const int nfl = (int)lv.size * F;
  const bool small = nfl <= kSmemAccFloats;
  float* G = md.grads;
  unsigned long long* GX = md.grads_fx;
  float* accf = reinterpret_cast<float*>(acc_raw);
  unsigned long long* accx = reinterpret_cast<unsigned long long*>(acc_raw);
  if (small) {
    for (int e = threadIdx.x; e < nfl; e += kLmThreads) {
      if (GX) accx[e] = 0ull; else accf[e] = 0.f;
    }
    __syncthreads();
  }
  const float* dfl = dfeat + ((size_t)m * g.net.L + l) * Bs * F;
  for (int i = i0 + threadIdx.x; i < i1; i += kLmThreads) {
    const float4 s = __ldg(samples + (size_t)m * Bs + i);
    const float x[3] = {s.x, s.y, s.z};
    float d[F];
    if constexpr (F == 1) { d[0] = __ldg(dfl + i); }
    else if constexpr (F == 2) { float2 v = __ldg(reinterpret_cast<const float2*>(dfl) + i); d[0] = v.x; d[1] = v.y; }
    else {
#pragma unroll
      for (int q = 0; q < F; q += 4) {
        float4 v = __ldg(reinterpret_cast<const float4*>(dfl + (size_t)i * F + q));
        d[q] = v.x; d[q + 1] = v.y; d[q + 2] = v.z; d[q + 3] = v.w;
      }
    }
    if (small) {
      Cell cell = level_cell(x, lv.res);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint32_t idx = corner_index(cell, c, lv, g.net.table_mask);
        float w = corner_weight(cell, c);
#pragma unroll
        for (int f = 0; f < F; ++f) {
          if (GX) {
            long long q = __double2ll_rn((double)(w * d[f]) * (double)(1ll << kFixedShift));
            atomicAdd(accx + idx * F + f, (unsigned long long)q);
          } else {
            atomicAdd(accf + idx * F + f, w * d[f]);
          }
        }
      }
    } else {
      scatter_level<F>(G, GX, lv, g.net.table_mask, x, d);
    }
  }
  if (small) {
    __syncthreads();
    for (int e = threadIdx.x; e < nfl; e += kLmThreads) {
      if (GX) {
        unsigned long long v = accx[e];
        if (v) atomicAdd(GX + lv.offset + e, v);
      } else {
        float v = accf[e];
        if (v != 0.f) atomicAdd(G + lv.offset + e, v);
      }
    }
  }
}

// ============================================================ host launchers
#define LM_DISPATCH_F(F_, ...)                           \
  switch (F_) {                                          \
    case 1: { constexpr int FF = 1; __VA_ARGS__; } break; \
    case 2: { constexpr int FF = 2; __VA_ARGS__; } break; \
    case 4: { constexpr int FF = 4; __VA_ARGS__; } break; \
    case 8: { constexpr int FF = 8; __VA_ARGS__; } break; \
    default: break;                                      \
  }

size_t lm_workspace_bytes(const NetDesc& net, int nmodels, int Bs) {
  size_t s = (size_t)nmodels * Bs;
  return s * sizeof(float4) + s * net.LF * sizeof(__half) + s * net.LF * sizeof(float) + 3 * 256;
}

LmWorkspace lm_workspace(void* base, const NetDesc& net, int nmodels, int Bs) {
  LmWorkspace w;
  size_t s = (size_t)nmodels * Bs;
  char* p = (char*)base;
  auto align = [](size_t v) { return (v + 255) / 256 * 256; };
  w.samples = reinterpret_cast<float4*>(p);
  p += align(s * sizeof(float4));
  w.feat = reinterpret_cast<__half*>(p);
  p += align(s * net.LF * sizeof(__half));
  w.dfeat = reinterpret_cast<float*>(p);
  w.Bs = Bs;
  return w;
}

void launch_sample(const GroupArgs& g, int nmodels, const FitScalars& fs, const LmWorkspace& w, cudaStream_t st) {
  dim3 grid((fs.B_u + fs.B_b + kLmThreads - 1) / kLmThreads, nmodels);
  sample_kernel<<<grid, kLmThreads, 0, st>>>(g, fs, w.samples, w.Bs);
  count_launch();
}

void launch_encode_fwd(const GroupArgs& g, int nmodels, const FitScalars& fs, const LmWorkspace& w,
                       cudaStream_t st) {
  dim3 grid((fs.B_u + fs.B_b + kLmThreads - 1) / kLmThreads, g.net.L, nmodels);
  LM_DISPATCH_F(g.net.F, encode_fwd_kernel<FF><<<grid, kLmThreads, 0, st>>>(g, fs, w.samples, w.feat, w.Bs));
  count_launch();
}

void launch_encode_bwd(const GroupArgs& g, int nmodels, const FitScalars& fs, const LmWorkspace& w,
                       cudaStream_t st) {
  dim3 grid((fs.B_u + fs.B_b + kBwdChunk - 1) / kBwdChunk, g.net.L, nmodels);
  size_t sm = (size_t)kSmemAccFloats * (fs.det ? 8 : 4);
  LM_DISPATCH_F(g.net.F,
                cudaFuncSetAttribute(encode_bwd_kernel<FF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
                encode_bwd_kernel<FF><<<grid, kLmThreads, sm, st>>>(g, fs, w.samples, w.dfeat, w.Bs));
  count_launch();
}

}  // namespace inr
