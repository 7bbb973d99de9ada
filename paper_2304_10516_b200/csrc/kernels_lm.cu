// kernels_lm.cu — the CUDA-core stages of the level-major fp16 fit pipeline:
//
//   encode_fwd_kernel  per (level, sample): x ~ Philox (uniform / boundary),   (a2-a7)
//                      8 corner gathers, blend -> fp16; level 0 also stores the
//                      sample and its trilinear target(s)
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
constexpr int kBwdChunk = 768;          // samples per CTA in the backward scatter (tuned: 512..2048 measured)

// Writes straight into the tensor-core MLP's h_0 tile images (canonical layout,
// see tc_common.cuh): sample i -> tile i/128, row i%128, columns [l F, l F + F).
// Padding samples (total <= i < Bs) write zeros; level 0 also writes the
// constant-ones group (column LF).
template <int F>
__global__ void __launch_bounds__(kLmThreads) encode_fwd_kernel(GroupArgs g, FitScalars fs,
                                                                 float4* __restrict__ samples,
                                                                 float4* __restrict__ targets,
                                                                 uint8_t* __restrict__ featimg, int Bs,
                                                                 FeatGeom geom) {
  const int m = blockIdx.z, l = blockIdx.y;
  const ModelDev& md = g.md[m];
  const int total = fs.B_u + (md.nfaces > 0 ? fs.B_b : 0);
  {
    // this step's gradient zeroing rides along (this kernel is L1-gather bound):
    // CTA (x, l) of model m clears one contiguous slice of the model's gradient
    const long long n4 = g.net.nparams / 4;   // nparams is a multiple of 64
    const long long ctas = (long long)gridDim.x * gridDim.y;
    const long long per = (n4 + ctas - 1) / ctas;
    const long long c = (long long)blockIdx.y * gridDim.x + blockIdx.x;
    const long long a = c * per, b = min(a + per, n4);
    if (md.grads_fx) {
      for (long long q = 4 * a + threadIdx.x; q < 4 * b; q += blockDim.x) md.grads_fx[q] = 0ull;
    } else {
      float4* g4 = reinterpret_cast<float4*>(md.grads);
      for (long long q = a + threadIdx.x; q < b; q += blockDim.x) g4[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  if (blockIdx.x == 0 && l == 0 && threadIdx.x == 0) {   // this step's loss sums (the MLP adds to them)
    md.acc[0] = 0.0;
    md.acc[1] = 0.0;
  }
  const int i = blockIdx.x * kLmThreads + threadIdx.x;
  if (i >= Bs) return;
  float f[F];
#pragma unroll
  for (int j = 0; j < F; ++j) f[j] = 0.f;
  if (i < total) {
    // the sample is drawn here (Philox, R8) for every level; level 0's CTAs also
    // store it with its trilinear target(s) for the MLP and the scatter kernels
    float x[3];
    // the step being executed: step_total, which encode_bwd_kernel advances
    draw_sample(md, i, fs.B_u, (uint32_t)*md.step_total, x);
    if (l == 0) {
      if (g.net.D == 1) {
        float t[1];
        sample_target<1>(md, x, t);
        samples[(size_t)m * Bs + i] = make_float4(x[0], x[1], x[2], t[0]);
      } else {
        float t[3];
        sample_target<3>(md, x, t);
        samples[(size_t)m * Bs + i] = make_float4(x[0], x[1], x[2], t[0]);
        targets[(size_t)m * Bs + i] = make_float4(t[0], t[1], t[2], 0.f);
      }
    }
    encode_level<F>(md.params, g.net.lv[l], g.net.table_mask, x, f);
  }
  const int r = i & 127;
  uint8_t* tile = featimg + ((size_t)m * (Bs >> 7) + (i >> 7)) * geom.tile_bytes;
  uint8_t* row = tile + (r & 7) * 16 + (r >> 3) * geom.sbo;
  const int c = l * F;
  if constexpr (F == 1) {
    *reinterpret_cast<__half*>(row + (c >> 3) * 128 + (c & 7) * 2) = __float2half_rn(f[0]);
  } else {
#pragma unroll
    for (int j = 0; j < F; j += 2)
      *reinterpret_cast<__half2*>(row + ((c + j) >> 3) * 128 + ((c + j) & 7) * 2) = __floats2half2_rn(f[j], f[j + 1]);
  }
  if (l == 0 && geom.ones)
    *reinterpret_cast<uint4*>(row + (g.net.LF >> 3) * 128) = make_uint4(0x3C00u, 0u, 0u, 0u);
}

// Scatter-add of samples [i0, i1) of model m at level l.  Small dense
// levels accumulate in shared memory first and flush once.
template <int F>
__device__ __forceinline__ void scatter_chunk(const GroupArgs& g, const ModelDev& md, int m, int l,
                                              const float4* __restrict__ samples, const float* __restrict__ dfeat,
                                              int Bs, int i0, int i1, unsigned char* acc_raw) {
  const LevelInfo& lv = g.net.lv[l];
  const int nfl = (int)lv.size * F;
  const bool small = nfl <= kSmemAccFloats;
  float* G = md.grads;
  unsigned long long* GX = md.grads_fx;
  float* accf = reinterpret_cast<float*>(acc_raw);
  unsigned long long* accx = reinterpret_cast<unsigned long long*>(acc_raw);
  if (small) {
    for (int e = threadIdx.x; e < nfl; e += blockDim.x) {
      if (GX) accx[e] = 0ull; else accf[e] = 0.f;
    }
    __syncthreads();
  }
  const float* dfl = dfeat + ((size_t)m * g.net.L + l) * Bs * F;
  for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
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
    for (int e = threadIdx.x; e < nfl; e += blockDim.x) {
      if (GX) {
        unsigned long long v = accx[e];
        if (v) atomicAdd(GX + lv.offset + e, v);
      } else {
        float v = accf[e];
        if (v != 0.f) atomicAdd(G + lv.offset + e, v);
      }
    }
    __syncthreads();
  }
}

template <int F>
__global__ void __launch_bounds__(kLmThreads) encode_bwd_kernel(GroupArgs g, FitScalars fs,
                                                                 const float4* __restrict__ samples,
                                                                 const float* __restrict__ dfeat, int Bs) {
  extern __shared__ __align__(16) unsigned char acc_raw[];
  const int m = blockIdx.z, l = blockIdx.y;
  const ModelDev& md = g.md[m];
  const int total = fs.B_u + (md.nfaces > 0 ? fs.B_b : 0);
  if (blockIdx.x == 0 && l == 0 && threadIdx.x == 0) {
    // open the step for Adam: step_cur = the step executed (step_total, with which
    // encode_fwd drew the samples), step_total += 1 (nothing else in the step reads them)
    const long long s = *md.step_total;
    *md.step_cur = s;
    *md.step_total = s + 1;
  }
  const int i0 = blockIdx.x * kBwdChunk;
  if (i0 >= total) return;
  scatter_chunk<F>(g, md, m, l, samples, dfeat, Bs, i0, min(i0 + kBwdChunk, total), acc_raw);
}

// ---------------------------------------------- level-major query encode
// Bucketed queries [c0*128, c0*128 + n) -> qx[j] = (x, y, z, slot bits): the
// block-normalized coordinate x = fl32(fl32(p - o) / n) (R5); slot -1 = padding.
__global__ void query_prep_kernel(GroupArgs g, const float* __restrict__ xyz, const int* __restrict__ perm,
                                  const int* __restrict__ tile_slot, const int* __restrict__ ntiles, long long j0,
                                  long long n, float4* __restrict__ qx) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= n) return;
  const long long jj = j0 + j;
  const int qi = jj < (long long)*ntiles * 128 ? perm[jj] : -1;
  if (qi < 0) { qx[j] = make_float4(0.f, 0.f, 0.f, __int_as_float(-1)); return; }
  const int slot = tile_slot[jj >> 7];
  const ModelDev& md = g.md[slot];
  float x[3];
#pragma unroll
  for (int d = 0; d < 3; ++d)
    x[d] = md.mesh[0] ? mesh_x(md, d, mesh_physical(md, d, __ldg(xyz + 3 * (long long)qi + d)))   // R36
                      : __fdiv_rn(__fsub_rn(__ldg(xyz + 3 * (long long)qi + d), (float)md.o[d]), (float)md.n[d]);
  qx[j] = make_float4(x[0], x[1], x[2], __int_as_float(slot));
}

// Level-major (grid.y = level): the CTAs in flight gather from one level of every
// block (<= 8 x 4 MB at cfg2) instead of all levels of one or two blocks, so the
// tables stay L2-resident as in the fit's encode_fwd_kernel.  Writes the fp16 h_0
// tile images of the tensor-core forward (forward layout: no ones group).
template <int F>
__global__ void __launch_bounds__(kLmThreads) encode_query_kernel(GroupArgs g, const float4* __restrict__ qx,
                                                                   long long n, uint8_t* __restrict__ featimg,
                                                                   FeatGeom geom) {
  const int l = blockIdx.y;
  const long long j = blockIdx.x * (long long)kLmThreads + threadIdx.x;
  if (j >= n) return;
  const float4 s = __ldg(qx + j);
  const int slot = __float_as_int(s.w);
  float f[F];
#pragma unroll
  for (int k = 0; k < F; ++k) f[k] = 0.f;
  if (slot >= 0) {
    const float x[3] = {s.x, s.y, s.z};
    encode_level<F>(g.md[slot].params, g.net.lv[l], g.net.table_mask, x, f);
  }
  const int r = (int)(j & 127);
  uint8_t* row = featimg + (size_t)(j >> 7) * geom.tile_bytes + (r & 7) * 16 + (r >> 3) * geom.sbo;
  const int c = l * F;
  if constexpr (F == 1) {
    *reinterpret_cast<__half*>(row + (c >> 3) * 128 + (c & 7) * 2) = __float2half_rn(f[0]);
  } else {
#pragma unroll
    for (int k = 0; k < F; k += 2)
      *reinterpret_cast<__half2*>(row + ((c + k) >> 3) * 128 + ((c + k) & 7) * 2) = __floats2half2_rn(f[k], f[k + 1]);
  }
}

// ------------------------------------------------------- query bucketing
// Decode queries on tensor cores need every 128-query tile to come from one
// block: route each query to its block (R5), count per block, lay the blocks'
// buckets out padded to 128, scatter query indices into them.  Bucket order is
// not deterministic, but each query's value does not depend on its tile slot.
__global__ void route_kernel(QueryArgs qa, const float* __restrict__ xyz, long long q, int* __restrict__ slot_of,
                             int* __restrict__ counts, int* __restrict__ dflag, float* __restrict__ out) {
  // per-CTA histogram in shared memory, one global atomic per (CTA, block): the
  // few per-block counters would otherwise serialize every warp's atomics
  __shared__ int cnt[kMaxGroup];
  for (int s = threadIdx.x; s < qa.nmodels; s += blockDim.x) cnt[s] = 0;
  __syncthreads();
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j < q) {
    int bc[3];
    bool outside = false;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const float p = __ldg(xyz + 3 * j + d);
      outside |= !(p >= 0.f && p <= (float)(qa.N[d] - 1));
      const int b = (int)floorf(__fdiv_rn(p, (float)qa.n[d]));
      bc[d] = min(max(b, 0), qa.B[d] - 1);
    }
    const int bid = (bc[2] * qa.B[1] + bc[1]) * qa.B[0] + bc[0];
    const int slot = bid < qa.nblocks ? qa.slot_of_block[bid] : -1;
    slot_of[j] = slot;
    // slot -1: no model has this block (NaN); -2: another chunk of the group decodes it
    if (slot >= 0) atomicAdd(cnt + slot, 1);
    else if (slot == -1)
      for (int c = 0; c < qa.net.D; ++c) out[j * qa.net.D + c] = __int_as_float(0x7fc00000);
    if (outside && dflag) atomicOr(dflag, 1);
  }
  __syncthreads();
  for (int s = threadIdx.x; s < qa.nmodels; s += blockDim.x)
    if (cnt[s]) atomicAdd(counts + s, cnt[s]);
}

__global__ void bucket_offsets_kernel(const int* __restrict__ counts, int nmodels, int* __restrict__ offsets,
                                      int* __restrict__ tile_slot, int* __restrict__ ntiles) {
  __shared__ int off[kMaxGroup + 1];
  if (threadIdx.x == 0) {
    int o = 0;
    for (int s = 0; s < nmodels; ++s) { off[s] = o; o += (counts[s] + 127) / 128 * 128; }
    off[nmodels] = o;
    *ntiles = o / 128;
  }
  __syncthreads();
  for (int s = threadIdx.x; s < nmodels; s += blockDim.x) offsets[s] = off[s];
  for (int s = 0; s < nmodels; ++s)
    for (int tt = off[s] / 128 + threadIdx.x; tt < off[s + 1] / 128; tt += blockDim.x) tile_slot[tt] = s;
}

__global__ void bucket_scatter_kernel(const int* __restrict__ slot_of, long long q, int nmodels,
                                      const int* __restrict__ offsets, int* __restrict__ cursor,
                                      int* __restrict__ perm) {
  // rank within the CTA's share of each bucket (shared atomics), then one global
  // reservation per (CTA, block)
  __shared__ int cnt[kMaxGroup], base[kMaxGroup];
  for (int s = threadIdx.x; s < nmodels; s += blockDim.x) cnt[s] = 0;
  __syncthreads();
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int s = j < q ? slot_of[j] : -1;
  const int local = s >= 0 ? atomicAdd(cnt + s, 1) : 0;
  __syncthreads();
  for (int t = threadIdx.x; t < nmodels; t += blockDim.x)
    if (cnt[t]) base[t] = atomicAdd(cursor + t, cnt[t]);
  __syncthreads();
  if (s >= 0) perm[offsets[s] + base[s] + local] = (int)j;
}

size_t query_workspace_bytes(long long q, int nmodels) {
  return (size_t)q * 4 + (size_t)(q + 128ll * nmodels) * 4 + 3 * 4 * kMaxGroup + (size_t)(q / 128 + nmodels + 2) * 4 +
         6 * 256;
}

void launch_query_buckets(const QueryArgs& qa, const float* xyz, long long q, float* out, int* dflag, void* ws,
                          QueryBuckets& b, cudaStream_t st) {
  char* p = (char*)ws;
  auto take = [&](size_t bytes) { char* r = p; p += (bytes + 255) / 256 * 256; return r; };
  int* slot_of = (int*)take((size_t)q * 4);
  b.perm = (int*)take((size_t)(q + 128ll * qa_nmodels(qa)) * 4);
  int* counts = (int*)take(4 * kMaxGroup);
  int* offsets = (int*)take(4 * kMaxGroup);
  int* cursor = (int*)take(4 * kMaxGroup);
  b.tile_slot = (int*)take((size_t)(q / 128 + qa_nmodels(qa) + 2) * 4);
  b.ntiles = (int*)take(4);
  cudaMemsetAsync(counts, 0, 4 * kMaxGroup, st);
  cudaMemsetAsync(cursor, 0, 4 * kMaxGroup, st);
  cudaMemsetAsync(b.perm, 0xff, (size_t)(q + 128ll * qa_nmodels(qa)) * 4, st);
  const unsigned grid = (unsigned)((q + 255) / 256);
  route_kernel<<<grid, 256, 0, st>>>(qa, xyz, q, slot_of, counts, dflag, out);
  bucket_offsets_kernel<<<1, 128, 0, st>>>(counts, qa_nmodels(qa), offsets, b.tile_slot, b.ntiles);
  bucket_scatter_kernel<<<grid, 256, 0, st>>>(slot_of, q, qa_nmodels(qa), offsets, cursor, b.perm);
  count_launch(3);
}

void launch_query_prep(const GroupArgs& g, const float* xyz, const QueryBuckets& b, long long j0, long long n,
                       float4* qx, cudaStream_t st) {
  query_prep_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g, xyz, b.perm, b.tile_slot, b.ntiles, j0, n, qx);
  count_launch();
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
  FeatGeom geom;
  uint32_t img = 0;
  tc_fit_geometry(net, &geom, &img);
  size_t s = (size_t)nmodels * Bs;
  return s * sizeof(float4) * (net.D > 1 ? 2 : 1) + (size_t)nmodels * (Bs / 128) * geom.tile_bytes +
         s * net.LF * sizeof(float) + (size_t)nmodels * img + 5 * 256;
}

LmWorkspace lm_workspace(void* base, const NetDesc& net, int nmodels, int Bs) {
  LmWorkspace w;
  tc_fit_geometry(net, &w.geom, &w.img_bytes);
  size_t s = (size_t)nmodels * Bs;
  char* p = (char*)base;
  auto align = [](size_t v) { return (v + 255) / 256 * 256; };
  w.samples = reinterpret_cast<float4*>(p);
  p += align(s * sizeof(float4));
  w.featimg = reinterpret_cast<uint8_t*>(p);
  p += align((size_t)nmodels * (Bs / 128) * w.geom.tile_bytes);
  w.dfeat = reinterpret_cast<float*>(p);
  p += align(s * net.LF * sizeof(float));
  w.wimg = reinterpret_cast<uint8_t*>(p);
  p += align((size_t)nmodels * w.img_bytes);
  w.targets = net.D > 1 ? reinterpret_cast<float4*>(p) : nullptr;
  w.Bs = Bs;
  return w;
}

void launch_encode_query(const GroupArgs& g, const float4* qx, long long n, uint8_t* featimg, const FeatGeom& geom,
                         cudaStream_t st) {
  dim3 grid((unsigned)((n + kLmThreads - 1) / kLmThreads), g.net.L);
  LM_DISPATCH_F(g.net.F, encode_query_kernel<FF><<<grid, kLmThreads, 0, st>>>(g, qx, n, featimg, geom));
  count_launch();
}

void launch_encode_fwd(const GroupArgs& g, int nmodels, const FitScalars& fs, const LmWorkspace& w,
                       cudaStream_t st) {
  dim3 grid((w.Bs + kLmThreads - 1) / kLmThreads, g.net.L, nmodels);
  LM_DISPATCH_F(g.net.F,
                encode_fwd_kernel<FF><<<grid, kLmThreads, 0, st>>>(g, fs, w.samples, w.targets, w.featimg, w.Bs,
                                                                    w.geom));
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
