// kernels_tc.cu — the fused fit step with the MLP on 5th-generation tensor
// cores (tcgen05.mma, kind::f16: fp16 operands in shared memory, fp32
// accumulators in TMEM), INR_PREC_FP16_MLP (R17).
//
// One CTA = 4 warps = 128 threads; a tile is 128 samples, sample t <-> thread t
// <-> TMEM lane t.  Per tile:
//   sampler + encode (CUDA cores, common.cuh) -> fp16 feature tile h_0 in smem
//   forward  z_k = h_k W_k^T   : M=128, N=64,   K=in_k   (A K-major, B K-major)
//   epilogue (TMEM -> regs): + b_k, ReLU, fp16 -> h_{k+1} tile; last hidden
//            layer feeds the 64->1 output layer on CUDA cores (fp32), Eq. 2
//   backward dW_k += dz_k^T h_k : M=64,  N=in_k+8, K=128 (A MN-major, B MN-major;
//            the +8 columns hold a constant 1 so column in_k accumulates db_k)
//            dh_k = dz_k W_k     : M=128, N=in_k,   K=64  (A K-major, B MN-major)
//   table scatter-add of dfeat (CUDA cores, common.cuh)
// dW_k stays in TMEM across all tiles a CTA processes and is flushed once.
// dz is scaled by 2^s (loss scaling, exact) so fp16 keeps its precision.
//
// Shared-memory operand tiles use the canonical SWIZZLE_NONE ("interleaved")
// layout: 8 rows x 16 B core matrices; element (row r, col c) of a tile with
// C columns sits at byte  (r%8)*16 + (r/8)*SBO + (c/8)*128 + (c%8)*2,
// SBO = (C/8)*128.  Read with (row = M/N dim, col = K dim) it is the K-major
// layout (LBO = 128, SBO); read with (row = K dim, col = M/N dim) it is the
// MN-major layout (SBO' = 128, LBO' = SBO).  So every tile serves both GEMMs
// that need it without a transposed copy.
#include <algorithm>

#include "launch.h"
#include "tc_common.cuh"

namespace inr {



using namespace tc;

// Fit-kernel setup: TMEM allocation, barriers, the constant ones groups of
// h_1..h_{H-1}, and one TMA bulk copy of the step's prepared weight image.
__device__ __forceinline__ uint32_t mlp_setup_fit(const NetDesc& net, const uint8_t* wimg, uint8_t* smem,
                                                  const Layout& lay) {
  const int t = threadIdx.x, warp = t >> 5;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + lay.tslot);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "r"(lay.ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (t == 0) {
    mbar_init(smem_u32(smem + lay.mbar), 1);
    mbar_init(smem_u32(smem + lay.mbar_img), 1);
    mbar_init(smem_u32(smem + lay.mbar_feat[0]), 1);
    mbar_init(smem_u32(smem + lay.mbar_feat[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (lay.ones && t < kTileM) {
    for (int k = 1; k < net.H; ++k) {
      uint4 u = make_uint4(0x3C00u, 0u, 0u, 0u);   // half(1.0), then zeros
      *reinterpret_cast<uint4*>(smem + lay.h[k] + (t & 7) * 16 + (t >> 3) * lay.h_sbo[k] +
                                (net.in_dim[k] >> 3) * 128) = u;
    }
  }
  __syncthreads();
  if (t == 0) {
    mbar_expect_tx(smem_u32(smem + lay.mbar_img), lay.img_bytes);
    bulk_g2s(smem_u32(smem), wimg, lay.img_bytes, smem_u32(smem + lay.mbar_img));
  }
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  mbar_wait(smem_u32(smem + lay.mbar_img), 0);
  return *tslot;
}

// Per step (fit) or call (decode): each model's fp32 MLP weights -> the fp16 weight
// image (canonical tiles + fp32 biases and output layer) that every CTA bulk-copies.
// It reads only the parameters, so the fit runs it beside encode_fwd.
__global__ void __launch_bounds__(256) prep_image_kernel(GroupArgs g, Layout lay, uint8_t* __restrict__ wimg) {
  const NetDesc& net = g.net;
  const float* __restrict__ P = g.md[blockIdx.x].params;
  uint8_t* dst = wimg + (size_t)blockIdx.x * lay.img_bytes;
  // CTA (model, y) converts rows y, y + gridDim.y, ... of every weight tile
  for (int k = 0; k < net.H; ++k) {
    const int in = net.in_dim[k];
    for (int n = blockIdx.y * blockDim.y + threadIdx.y; n < 64; n += gridDim.y * blockDim.y) {
      for (int i = threadIdx.x; i < in; i += blockDim.x)
        *reinterpret_cast<__half*>(dst + lay.w[k] + tile_off(lay.w_sbo[k], n, i)) =
            __float2half_rn(P[net.w_off[k] + n * in + i]);
    }
  }
  if (blockIdx.y != 0) return;
  const int t = threadIdx.y * blockDim.x + threadIdx.x;
  float* bias = reinterpret_cast<float*>(dst + lay.bias);
  float* wout = reinterpret_cast<float*>(dst + lay.wout);
  for (int e = t; e < net.H * 64; e += 256) bias[e] = net.bias ? P[net.b_off[e / 64] + (e % 64)] : 0.f;
  // output layer W_H [D][64] row-major, then b_H [D]
  for (int i = t; i < net.D * 64; i += 256) wout[i] = P[net.w_off[net.H] + i];
  if (t < net.D) wout[net.D * 64 + t] = net.bias ? P[net.b_off[net.H] + t] : 0.f;
}

__device__ __forceinline__ void mlp_teardown(uint32_t tmem, const Layout& lay) {
  fence_before();
  __syncthreads();
  fence_after();
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(lay.ncols));
}

// ---------------------------------------------------------------------------
// MLP forward + Eq. 2 + backward on tensor cores for level-major features
// (the middle kernel of the fp16 fit pipeline).  256 threads: thread t owns
// row r = t % 128 of the tile (TMEM lane r) and column half t / 128 (32 of the
// 64 columns), so every epilogue is split across two threads and twice as many
// warps hide the MMA and TMEM latencies.  featimg: fp16 h_0 tile images,
// samples: float4 (x, y, z, target); writes dfeat fp32 [model][level][Bs][F];
// adds dW, db into the model's gradient.
constexpr int kFitQ = 2;                      // threads per tile row (column groups of 64 / kFitQ)
constexpr int kFitCW = 64 / kFitQ;              // columns per thread
constexpr int kFitThreads = kTileM * kFitQ;
constexpr int kDetCtasPerModel = 32;   // deterministic mode: MLP CTAs per model, independent of the group

// Sum 16 per-lane values over the warp; lanes l and l + 16 end with the sum of column l.
__device__ __forceinline__ float warp_transpose_reduce16(float* v, int lane) {
#pragma unroll
  for (int half = 8, off = 8; off >= 1; half >>= 1, off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int j = 0; j < half; ++j) {
      float keep = up ? v[j + half] : v[j];
      float send = up ? v[j] : v[j + half];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

// Sum 32 per-lane values over the warp; lane l ends with the sum of column l.
__device__ __forceinline__ float warp_transpose_reduce32(float* v, int lane) {
#pragma unroll
  for (int half = 16, off = 16; off >= 1; half >>= 1, off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int j = 0; j < half; ++j) {
      float keep = up ? v[j + half] : v[j];
      float send = up ? v[j] : v[j + half];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

__device__ __forceinline__ void red_smem(float* red, unsigned long long* redx, bool det, int i, float v) {
  if (det) atomicAdd(redx + i, (unsigned long long)__double2ll_rn((double)v * (double)(1ll << kFixedShift)));
  else atomicAdd(red + i, v);
}

template <int F, int D>
__global__ void __launch_bounds__(kFitThreads, 2) mlp_fit_kernel(GroupArgs g, FitScalars fs, Layout lay,
                                                                float loss_scale, const uint8_t* __restrict__ featimg,
                                                                const uint8_t* __restrict__ wimg,
                                                                const float4* __restrict__ samples,
                                                                const float4* __restrict__ targets,
                                                                float* __restrict__ dfeat, int Bs) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const NetDesc& net = g.net;
  const int m = blockIdx.y;
  const ModelDev& md = g.md[m];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int r = t & (kTileM - 1), q = t >> 7, cb = q * kFitCW;   // row, column group
  const int H = net.H, L = net.L, ones = lay.ones;
  const int B_b = md.nfaces > 0 ? fs.B_b : 0;
  const int total = fs.B_u + B_b;
  const int ntiles = (total + kTileM - 1) / kTileM;
  float* __restrict__ G = md.grads;
  unsigned long long* __restrict__ GX = md.grads_fx;
  const bool det = GX != nullptr;
  const float inv_scale = 1.f / loss_scale;
  const uint8_t* featm = featimg + (size_t)m * (Bs / kTileM) * lay.feat_tile_bytes;
  float* dfeatm = dfeat + (size_t)m * L * Bs * F;

  float* bias = reinterpret_cast<float*>(smem + lay.bias);
  float* wout = reinterpret_cast<float*>(smem + lay.wout);
  // dW_H [D][64] / db_H [D] partial sums of this CTA: fp32, or exact int64 fixed
  // point in the deterministic mode (the warps add in a run-dependent order)
  float* red = reinterpret_cast<float*>(smem + lay.red);
  unsigned long long* redx = reinterpret_cast<unsigned long long*>(smem + lay.red);
  float* ypart = reinterpret_cast<float*>(smem + lay.ypart);   // [D][kFitQ][128] output-layer partial sums
  const uint32_t mbar = smem_u32(smem + lay.mbar);
  for (int i = t; i < D * 65; i += kFitThreads) redx[i] = 0ull;
  const uint32_t tmem = mlp_setup_fit(net, wimg + (size_t)m * lay.img_bytes, smem, lay);
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  uint32_t phase = 0;
  bool first = true;
  const float lam = B_b > 0 ? fs.lambda : 0.f;
  const uint32_t hbuf[2] = {smem_u32(smem + lay.h[0]), smem_u32(smem + lay.h0b)};
  const uint32_t fbar[2] = {smem_u32(smem + lay.mbar_feat[0]), smem_u32(smem + lay.mbar_feat[1])};
  if (t == 0 && (int)blockIdx.x < ntiles) {   // prefetch the first feature tile
    mbar_expect_tx(fbar[0], lay.feat_tile_bytes);
    bulk_g2s(hbuf[0], featm + (size_t)blockIdx.x * lay.feat_tile_bytes, lay.feat_tile_bytes, fbar[0]);
  }

  int it = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int i = tile * kTileM + r;
    const bool valid = i < total;
    const bool is_b = i >= fs.B_u;
    float target[D];
    if constexpr (D == 1) {
      target[0] = valid ? samples[(size_t)m * Bs + i].w : 0.f;
    } else {
      const float4 tg = valid ? targets[(size_t)m * Bs + i] : make_float4(0.f, 0.f, 0.f, 0.f);
      target[0] = tg.x; target[1] = tg.y; target[2] = tg.z;
    }
    const int b = it & 1;
    const uint32_t h0 = hbuf[b];
    if (t == 0 && tile + (int)gridDim.x < ntiles) {   // prefetch the next tile into the other buffer
      mbar_expect_tx(fbar[b ^ 1], lay.feat_tile_bytes);
      bulk_g2s(hbuf[b ^ 1], featm + (size_t)(tile + gridDim.x) * lay.feat_tile_bytes, lay.feat_tile_bytes,
               fbar[b ^ 1]);
    }
    mbar_wait(fbar[b], (uint32_t)(it >> 1) & 1u);
    // ---- forward through the hidden layers (this thread: columns [cb, cb + kFitCW)).  The
    // ReLU masks of the backward pass are read back from the stored activations:
    // 1[z_{k-1} > 0] = 1[h_k > 0] (h_k = ReLU(z_{k-1}) rounded to fp16; only 0 < z < 2^-25
    // rounds to h = 0, below the fp16 MLP's own rounding of z), and from hH for the last layer
    float hH[kFitCW];
    for (int k = 0; k < H; ++k) {
      const int in = net.in_dim[k];
      if (t == 0) {
        fence_after();
        gemm(tmem, k == 0 ? h0 : smem_u32(smem + lay.h[k]), 128, lay.h_sbo[k], 256, smem_u32(smem + lay.w[k]), 128,
             lay.w_sbo[k], 256, in / 16, make_idesc(128, 64, 0, 0), false);
        mma_commit(mbar);
      }
      mbar_wait(mbar, phase);
      phase ^= 1;
      fence_after();
      float z[kFitCW];
#pragma unroll
      for (int c = 0; c < kFitCW; c += 16) tmem_ld16(tmem + lane_base + cb + c, z + c);
      tmem_wait_ld();
      // padding rows (i >= total) need no clamp: their h_0 rows are zeros and the ones
      // group (encode_fwd), so every activation stays finite, and their dy = 0 makes
      // every dz row 0, so they add nothing to dW, db or dfeat
#pragma unroll
      for (int n = 0; n < kFitCW; n += 4) {
        const float4 b4 = *reinterpret_cast<const float4*>(bias + k * 64 + cb + n);
        z[n] = fmaxf(z[n] + b4.x, 0.f);
        z[n + 1] = fmaxf(z[n + 1] + b4.y, 0.f);
        z[n + 2] = fmaxf(z[n + 2] + b4.z, 0.f);
        z[n + 3] = fmaxf(z[n + 3] + b4.w, 0.f);
      }
      if (k + 1 < H) {
#pragma unroll
        for (int j = 0; j < kFitCW / 8; ++j)
          st_row8(smem + lay.h[k + 1], lay.h_sbo[k + 1], r, q * (kFitCW / 8) + j, z + 8 * j);
      } else {
        float yp[D];
#pragma unroll
        for (int c = 0; c < D; ++c) yp[c] = 0.f;
#pragma unroll
        for (int n = 0; n < kFitCW; ++n) {
          hH[n] = z[n];
#pragma unroll
          for (int c = 0; c < D; ++c) yp[c] = fmaf(wout[c * 64 + cb + n], z[n], yp[c]);
        }
#pragma unroll
        for (int c = 0; c < D; ++c) ypart[(kFitQ * c + q) * kTileM + r] = yp[c];
      }
      fence_async_smem();
      fence_before();
      __syncthreads();
    }
    // ---- output layer (fp32, CUDA cores) and Eq. 2, L1 pooled over the D channels [R28]
    float dy[D];
    double ad = 0.0;
#pragma unroll
    for (int c = 0; c < D; ++c) {
      float y = wout[D * 64 + c];
#pragma unroll
      for (int p = 0; p < kFitQ; ++p) y += ypart[(kFitQ * c + p) * kTileM + r];
      const float d = y - target[c];
      const float sg = valid ? (d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f)) : 0.f;
      dy[c] = is_b ? lam * sg / (float)(max(B_b, 1) * D) : (1.f - lam) * sg / (float)(fs.B_u * D);
      ad += fabs((double)d);
    }
    if (q == 0) {
      double au = (valid && !is_b) ? ad : 0.0;
      double ab = (valid && is_b) ? ad : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        au += __shfl_xor_sync(0xffffffffu, au, o);
        ab += __shfl_xor_sync(0xffffffffu, ab, o);
      }
      if (lane == 0) {
        if (au != 0.0) atomicAdd(md.acc + 0, au);
        if (ab != 0.0) atomicAdd(md.acc + 1, ab);
      }
#pragma unroll
      for (int c = 0; c < D; ++c) {
        float s = dy[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red_smem(red, redx, det, D * 64 + c, s);   // db_H[c]
      }
    }
#pragma unroll
    for (int c = 0; c < D; ++c) {   // dW_H[c][n] = sum_s dy_c,s h_H[s][n] for this thread's columns
      float v[kFitCW];
#pragma unroll
      for (int n = 0; n < kFitCW; ++n) v[n] = dy[c] * hH[n];
      if constexpr (kFitCW == 32) {
        red_smem(red, redx, det, c * 64 + cb + lane, warp_transpose_reduce32(v, lane));
      } else {
        const float sv = warp_transpose_reduce16(v, lane);
        if (lane < 16) red_smem(red, redx, det, c * 64 + cb + lane, sv);
      }
    }
    {   // dz_{H-1} = (sum_c dy_c W_H[c]) * 1[z_{H-1} > 0], scaled by 2^s
      float dz[kFitCW];
#pragma unroll
      for (int n = 0; n < kFitCW; ++n) {
        float a = 0.f;
#pragma unroll
        for (int c = 0; c < D; ++c) a = fmaf(dy[c] * loss_scale, wout[c * 64 + cb + n], a);
        dz[n] = hH[n] > 0.f ? a : 0.f;
      }
#pragma unroll
      for (int j = 0; j < kFitCW / 8; ++j) st_row8(smem + lay.dz, lay.dz_sbo, r, q * (kFitCW / 8) + j, dz + 8 * j);
    }
    fence_async_smem();
    fence_before();
    __syncthreads();

    // ---- backward through the hidden layers
    for (int k = H - 1; k >= 0; --k) {
      const int in = net.in_dim[k];
      // dz_k lives in dz / dz2 alternately, so dW_k may still read its tile while the
      // epilogue writes dz_{k-1} into the other one
      const uint32_t dzk = smem_u32(smem + (((H - 1 - k) & 1) ? lay.dz2 : lay.dz));
      if (t == 0) {
        fence_after();
        auto dW = [&] {   // dW_k (+ db_k in column in_k): A = dz^T (MN-major), B = h_k (MN-major), K = 128 samples
          gemm(tmem + lay.col_dw[k], dzk, lay.dz_sbo, 128, 2 * lay.dz_sbo,
               k == 0 ? h0 : smem_u32(smem + lay.h[k]), lay.h_sbo[k], 128, 2 * lay.h_sbo[k], kTileM / 16,
               make_idesc(64, in + ones, 1, 1), !first);
        };
        auto dH = [&] {   // dh_k = dz_k W_k: A = dz (K-major, K = 64 outputs), B = W_k (MN-major, N = in_k)
          gemm(tmem, dzk, 128, lay.dz_sbo, 256, smem_u32(smem + lay.w[k]), lay.w_sbo[k], 128,
               2 * lay.w_sbo[k], 64 / 16, make_idesc(128, in, 0, 1), false);
        };
        if (k > 0) {
          // the epilogue waits for dh_k only; dW_k runs under it (the next commit, which
          // every later wait follows, covers it: MMAs of one thread complete in order)
          dH();
          mma_commit(mbar);
          dW();
        } else {
          // the last layer of the tile commits both: the next tile's TMA prefetch
          // overwrites the h_0 buffer dW_0 reads
          dW();
          dH();
          mma_commit(mbar);
        }
      }
      mbar_wait(mbar, phase);
      phase ^= 1;
      fence_after();
      if (cb < in) {   // warp-uniform: this group has columns of dh
        float dh[kFitCW];
#pragma unroll
        for (int c = 0; c < kFitCW; c += 16) tmem_ld16(tmem + lane_base + cb + c, dh + c);
        tmem_wait_ld();
        if (k > 0) {
          // dz_{k-1} = dh_k * 1[h_k > 0] on packed fp16 pairs (the mask multiplies by 1 or 0)
          const uint8_t* hrow = smem + lay.h[k] + (r & 7) * 16 + (r >> 3) * lay.h_sbo[k];
          uint8_t* drow = smem + (((H - k) & 1) ? lay.dz2 : lay.dz) + (r & 7) * 16 + (r >> 3) * lay.dz_sbo;
          const __half2 zero2 = __float2half2_rn(0.f);
#pragma unroll
          for (int j = 0; j < kFitCW / 8; ++j) {
            uint4 hv = *reinterpret_cast<const uint4*>(hrow + (q * (kFitCW / 8) + j) * 128);
            const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
            uint32_t o[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) {
              const __half2 h2 = *reinterpret_cast<const __half2*>(&hw[p]);
              __half2 d2 = __hmul2(__floats2half2_rn(dh[8 * j + 2 * p], dh[8 * j + 2 * p + 1]), __hgt2(h2, zero2));
              o[p] = *reinterpret_cast<uint32_t*>(&d2);
            }
            *reinterpret_cast<uint4*>(drow + (q * (kFitCW / 8) + j) * 128) = make_uint4(o[0], o[1], o[2], o[3]);
          }
        } else if (valid) {
          // dfeat, unscaled, level-major (coalesced across the tile)
          float* const o0 = dfeatm + ((size_t)(q * (kFitCW / F)) * Bs + i) * F;
          const size_t lstride = (size_t)Bs * F;
#pragma unroll
          for (int c = 0; c < kFitCW; c += F) {
            if (cb + c < net.LF) {
              float* o = o0 + (size_t)(c / F) * lstride;
              if constexpr (F == 1) { o[0] = dh[c] * inv_scale; }
              else if constexpr (F == 2) { *reinterpret_cast<float2*>(o) = make_float2(dh[c] * inv_scale, dh[c + 1] * inv_scale); }
              else {
#pragma unroll
                for (int u = 0; u < F; u += 4)
                  *reinterpret_cast<float4*>(o + u) = make_float4(dh[c + u] * inv_scale, dh[c + u + 1] * inv_scale,
                                                                  dh[c + u + 2] * inv_scale, dh[c + u + 3] * inv_scale);
              }
            }
          }
        }
      }
      fence_async_smem();
      fence_before();
      __syncthreads();
    }
    first = false;
  }

  // ---- flush the CTA's weight gradients (TMEM dW_k, smem dW_H) once
  if (!first) {
    fence_after();
    for (int k = 0; k < H; ++k) {
      const int in = net.in_dim[k];
      const int ncol = in + ones;
      // M = 64 accumulator: row 16w + l lives in lane 32w + l (l < 16); groups take alternate 16-column chunks
      for (int c = q * 16; c < ncol; c += 16 * kFitQ) {
        float v[16];
        tmem_ld16(tmem + lane_base + lay.col_dw[k] + c, v);
        tmem_wait_ld();
        if (lane < 16) {
          const int n = (warp & 3) * 16 + lane;
          if (!det && c + 16 <= in) {
            // 16 weights of row n: four 16-B vector reductions (in and the tensor offset are
            // multiples of 4 floats)
            float4* dst = reinterpret_cast<float4*>(G + net.w_off[k] + (size_t)n * in + c);
#pragma unroll
            for (int j = 0; j < 16; j += 4)
              atomicAdd(dst + j / 4, make_float4(v[j] * inv_scale, v[j + 1] * inv_scale, v[j + 2] * inv_scale,
                                                 v[j + 3] * inv_scale));
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              int col = c + j;
              float gval = v[j] * inv_scale;
              if (col < in) grad_add(G, GX, net.w_off[k] + (size_t)n * in + col, gval);
              else if (col == in && ones) grad_add(G, GX, net.b_off[k] + n, gval);
            }
          }
        }
      }
    }
  }
  __syncthreads();
  if (!first) {
    if (det) {
      for (int n = t; n < D * 64; n += kFitThreads) atomicAdd(GX + net.w_off[H] + n, redx[n]);
      if (t < D && net.bias) atomicAdd(GX + net.b_off[H] + t, redx[D * 64 + t]);
    } else {
      for (int n = t; n < D * 64; n += kFitThreads) atomicAdd(G + net.w_off[H] + n, red[n]);
      if (t < D && net.bias) atomicAdd(G + net.b_off[H] + t, red[D * 64 + t]);
    }
  }
  mlp_teardown(tmem, lay);
}

// ============================================================ host side
// train: the fit layout (ones groups, dz tile, dW accumulators in TMEM);
// otherwise the forward-only layout (64 TMEM columns).
static bool build_layout(const NetDesc& net, Layout& L, bool train = true) {
  memset(&L, 0, sizeof L);
  if (net.LF % 16 != 0 || net.LF > 64 || net.H < 1 || net.H > kMaxLayers - 1 || (net.D != 1 && net.D != 3))
    return false;
  L.ones = (net.bias && train) ? 8 : 0;
  uint32_t off = 0;
  auto take = [&](uint32_t bytes, uint32_t align) {
    off = (off + align - 1) / align * align;
    uint32_t o = off;
    off += bytes;
    return o;
  };
  // the weight image (copied as one block in the fit kernel): weight tiles, biases, output layer
  for (int k = 0; k < net.H; ++k) {
    L.w_sbo[k] = (uint32_t)(net.in_dim[k] / 8) * 128;
    L.w[k] = take(64 * net.in_dim[k] * 2, 1024);
  }
  L.bias = take(net.H * 64 * 4, 16);
  L.wout = take((net.D * 64 + 4) * 4, 16);
  L.img_bytes = (off + 15) / 16 * 16;
  off = L.img_bytes;
  if (train) {   // every activation tile is kept for the backward pass
    for (int k = 0; k < net.H; ++k) {
      int in = net.in_dim[k];
      L.h_sbo[k] = (uint32_t)((in + L.ones) / 8) * 128;
      L.h[k] = take(kTileM * (in + L.ones) * 2, 1024);
    }
  } else {       // forward only: one activation buffer.  Layer k's epilogue overwrites its own
                 // input h_k with h_{k+1}: it runs after the MMA reading h_k has completed
                 // (mbarrier), and the smaller footprint lets 5 CTAs share an SM
    const uint32_t hb = take(kTileM * 64 * 2, 1024);
    for (int k = 0; k < net.H; ++k) {
      L.h_sbo[k] = (uint32_t)(net.in_dim[k] / 8) * 128;
      L.h[k] = hb;
    }
  }
  L.feat_tile_bytes = kTileM * (net.LF + L.ones) * 2;
  if (train) L.h0b = take(L.feat_tile_bytes, 1024);
  L.dz_sbo = 8 * 128;
  if (train) L.dz = take(kTileM * 64 * 2, 1024);
  if (train) L.dz2 = take(kTileM * 64 * 2, 1024);
  L.red = take((net.D * 65 + 1) * 8, 16);
  L.ypart = take(net.D * 4 * kTileM * 4, 16);   // [D][<= 4 column groups][128]
  L.mbar = take(8, 8);
  L.mbar_img = take(8, 8);
  L.mbar_feat[0] = take(8, 8);
  L.mbar_feat[1] = take(8, 8);
  L.tslot = take(4, 4);
  if (!train) L.stage = take(kStageFloats * 4, 16);
  if (!train) L.stbox = take(kMaxLevels * 8 * 4, 16);
  // TMEM: [0, 64) layer accumulator; then dW_k (M = 64 rows, in_k + ones columns)
  // (8-column granularity; the last region is padded so 16-column loads stay inside)
  uint32_t col = 64;
  if (train) {
    for (int k = 0; k < net.H; ++k) {
      L.col_dw[k] = col;
      col += (uint32_t)(net.in_dim[k] + L.ones);
    }
    col = std::max(col, L.col_dw[net.H - 1] + (uint32_t)((net.in_dim[net.H - 1] + L.ones + 15) / 16 * 16));
  }
  if (col > 512) return false;
  L.ncols = 32;
  while (L.ncols < col) L.ncols <<= 1;
  L.ctas_per_sm = (int)(512 / L.ncols);
  // request enough shared memory that no more CTAs than TMEM allows share an SM
  uint32_t need = off + 128;
  uint32_t floor_bytes = 232448u / (uint32_t)(L.ctas_per_sm + 1) + 1024;
  L.bytes = std::max(need, std::min<uint32_t>(floor_bytes, 232448u));
  if (need > 232448u) return false;
  // actual residency is then limited by both shared memory and TMEM
  L.ctas_per_sm = std::min<int>(L.ctas_per_sm, (int)(232448u / L.bytes));
  if (!train) L.ctas_per_sm = std::min(L.ctas_per_sm, 4);   // forward_tc_kernel: 256 threads x <= 64 registers
  return L.ctas_per_sm >= 1;
}

bool tc_supported(const NetDesc& net) {
  Layout L;
  return build_layout(net, L);
}

static float loss_scale_for(int B_u) {
  int e = 0;
  while ((1 << (e + 1)) <= B_u && e < 24) ++e;
  return (float)(1 << e);
}

bool tc_fit_geometry(const NetDesc& net, FeatGeom* geom, uint32_t* img_bytes) {
  Layout L;
  if (!build_layout(net, L)) return false;
  if (geom) { geom->sbo = L.h_sbo[0]; geom->tile_bytes = L.feat_tile_bytes; geom->ones = L.ones; }
  if (img_bytes) *img_bytes = L.img_bytes;
  return true;
}

void launch_prep_image(const GroupArgs& g, int nmodels, uint8_t* wimg, cudaStream_t st) {
  Layout L;
  if (!build_layout(g.net, L)) return;
  prep_image_kernel<<<dim3(nmodels, 16), dim3(64, 4), 0, st>>>(g, L, wimg);
  count_launch();
}

void launch_mlp_tc(const GroupArgs& g, int nmodels, const FitScalars& fs, const uint8_t* featimg, const uint8_t* wimg,
                   const float4* samples, const float4* targets, float* dfeat, int Bs, cudaStream_t st, int ctas) {
  Layout L;
  if (!build_layout(g.net, L)) return;
  const int total = fs.B_u + fs.B_b;
  const int ntiles = (total + kTileM - 1) / kTileM;
  const int slots = ctas > 0 ? ctas : 148 * L.ctas_per_sm;
  // CTAs per model: fill the machine; in the deterministic mode a fixed count, so
  // that the tiles each CTA accumulates in fp32 TMEM (and hence the exact result)
  // do not depend on how many models share the launch
  // (ctas > 0: at most ctas in all, so that every CTA has its SM slot beside the side Adam)
  int per_model = fs.det ? std::min(ntiles, kDetCtasPerModel)
                         : std::max(1, std::min(ntiles, ctas > 0 ? slots / nmodels : (slots + nmodels - 1) / nmodels));
  dim3 grid(per_model, nmodels);
  float ls = loss_scale_for(fs.B_u);
  switch (g.net.F * 10 + g.net.D) {
#define CASE_FD(FF, DD)                                                                                   \
  case FF * 10 + DD:                                                                                      \
    cudaFuncSetAttribute(mlp_fit_kernel<FF, DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, L.bytes);   \
    mlp_fit_kernel<FF, DD><<<grid, kFitThreads, L.bytes, st>>>(g, fs, L, ls, featimg, wimg, samples, targets, \
                                                                dfeat, Bs);                                \
    break;
    CASE_FD(1, 1) CASE_FD(2, 1) CASE_FD(4, 1) CASE_FD(8, 1) CASE_FD(1, 3) CASE_FD(2, 3) CASE_FD(4, 3) CASE_FD(8, 3)
#undef CASE_FD
    default: break;
  }
  count_launch();
}

// ------------------------------------------------------------ forward only
// Network inference on tensor cores for 128-point tiles (same forward as the fit):
//   MODE 0  debug: block-normalized x01[q] -> y[q] (normalized units)
//   MODE 1  decode grid: x_j = fl32(j / R) lattice of one block, denormalized
//           strided stores, optional fused SSE against ref (R18, R19)
//   MODE 3  decode query: tiles of bucket-sorted queries, every tile from one
//           block, whose fp16 h_0 tile images were encoded level-major
//           (encode_query_kernel, kernels_lm.cu) and arrive by TMA bulk copy
struct FwdArgs {
  const float* x01;
  float* y;
  long long q;
  int res[3], cnt[3];   // decode grid: lattice resolution, points decoded per axis (cnt <= res)
  float* out;
  long long os[3];
  const float* ref;
  double* sse;
  const float* xyz;
  const int* perm;
  const int* tile_slot;
  const int* ntiles_dev;
  const uint8_t* wimg;   // prepared weight images, one per model slot (prep_image_kernel)
  const uint8_t* featimg;   // MODE 3: h_0 tile images of tiles [tile0, tile1)
  long long tile0, tile1;
  int nst;                            // MODE 1: levels [0, nst) are staged per brick in shared memory
  int st_off[kMaxLevels + 1];         //   float offset of level l's vertex box in the stage area
  int na;                             // MODE 1: levels [na, L) are vertex-aligned (one entry per point, R19)
  float rinv[3];                      //   1 / R_d when R_d is a power of two (x_j = j / R_d exactly), else 0
};

// MODE 1 brick staging (grid decode): the levels coarser than the
// lattice (N_l < R) have fractional weights at most lattice points, and the
// 128 points of an 8 x 4 x 4 brick touch only a small box of their vertices
// (cfg2, R = 128: 27-45 vertices per level instead of 8 corner reads per point).
// The box is computed from the brick's first and last lattice point per axis
// with the same pinned index arithmetic as level_cell (R4, R20).
__device__ __forceinline__ int cell_of(float x, uint32_t res) {
  const float p = __fmul_rn(fminf(fmaxf(x, 0.f), 1.f), (float)res);
  return min((int)floorf(p), (int)res - 1);
}

__device__ __forceinline__ uint32_t vertex_index(uint32_t vx, uint32_t vy, uint32_t vz, const LevelInfo& lv,
                                                 uint32_t mask) {
  if (lv.dense) {
    const uint32_t s = lv.res + 1;
    return vx + s * (vy + s * vz);
  }
  return (vx ^ (vy * kPrimeY) ^ (vz * kPrimeZ)) & mask;
}

// feat = sum_c w_c theta[idx_c] from the staged box (lo, n): the same weights
// (corner_weight) and the same corner-ordered fma chain as encode_level, so the
// result is bitwise the global-memory encode (grid == query decode stays exact).
template <int F>
__device__ __forceinline__ void blend_staged(const float* __restrict__ box, const int lo[3], const int n[3],
                                             uint32_t res, const float x[3], float feat[F]) {
  Cell cell = level_cell(x, res);
  const float ox = 1.f - cell.w[0], oy = 1.f - cell.w[1];
  const float wxy[4] = {ox * oy, cell.w[0] * oy, ox * cell.w[1], cell.w[0] * cell.w[1]};
  const float wz[2] = {1.f - cell.w[2], cell.w[2]};
  const int n0 = n[0], n01 = n[0] * n[1];
  const float* e0 = box + ((int)cell.i[0] - lo[0] + n0 * ((int)cell.i[1] - lo[1] + n[1] * ((int)cell.i[2] - lo[2]))) * F;
#pragma unroll
  for (int f = 0; f < F; ++f) feat[f] = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float* e = e0 + ((c & 1) + ((c >> 1) & 1) * n0 + (c >> 2) * n01) * F;
    const float w = wxy[c & 3] * wz[c >> 2];
#pragma unroll
    for (int f = 0; f < F; ++f) feat[f] = fmaf(w, e[f], feat[f]);
  }
}

// fp16 feature columns [c, c + F) of this thread's h_0 row (canonical layout)
template <int F>
__device__ __forceinline__ void put_feat(uint8_t* row, int c, const float fl[F]) {
  if constexpr (F == 1) {
    *reinterpret_cast<__half*>(row + (c >> 3) * 128 + (c & 7) * 2) = __float2half_rn(fl[0]);
  } else {
#pragma unroll
    for (int jj = 0; jj < F; jj += 2)
      *reinterpret_cast<__half2*>(row + ((c + jj) >> 3) * 128 + ((c + jj) & 7) * 2) = __floats2half2_rn(fl[jj], fl[jj + 1]);
  }
}

// 256 threads per 128-point tile: thread t owns row r = t % 128 (TMEM lane r) and
// half hf = t / 128, which encodes every other level (l % 2 == hf) and, in the
// epilogues, columns [32 hf, 32 hf + 32): half the serial work per thread of a
// one-thread-per-row tile, at ~64 registers, so 4 CTAs (32 warps) share an SM.
template <int F, int MODE, int D>
__global__ void __launch_bounds__(kFwdThreads, 4) forward_tc_kernel(GroupArgs g, FwdArgs a, Layout lay) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const NetDesc& net = g.net;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int r = t & (kTileM - 1), hf = t >> 7, cb = hf * 32;
  const int H = net.H;
  const float* bias = reinterpret_cast<const float*>(smem + lay.bias);
  float* wout = reinterpret_cast<float*>(smem + lay.wout);
  float* ypart = reinterpret_cast<float*>(smem + lay.ypart);   // [D][2][128] output-layer half sums
  const uint32_t mbar = smem_u32(smem + lay.mbar);
  const uint32_t mbar_img = smem_u32(smem + lay.mbar_img);
  const uint32_t mbar_feat = smem_u32(smem + lay.mbar_feat[0]);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + lay.tslot);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)),
                 "r"(lay.ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (t == 0) {
    mbar_init(mbar, 1);
    mbar_init(mbar_img, 1);
    mbar_init(mbar_feat, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  uint32_t phase = 0, img_phase = 0, feat_phase = 0;
  int cur = -1;  // model whose weight image is in smem
  // tiles are visited grid-stride: the CTAs in flight work on consecutive tiles
  // (MODE 3: tiles grouped by block, so one or two blocks' weights at a time); a
  // CTA reloads the weight image only when its next tile belongs to another block
  long long t0 = blockIdx.x, t1;
  // MODE 1: tile = 8 super-brick + sub-brick; a CTA takes the 8 bricks of one 2 x 2 x 2
  // super-brick in a row (their coarse levels staged once), then jumps gridDim.x on
  const int nbx = (a.cnt[0] + kBrickX - 1) / kBrickX, nby = (a.cnt[1] + kBrickY - 1) / kBrickY,
            nbz = (a.cnt[2] + kBrickZ - 1) / kBrickZ;
  const int nsx = (nbx + kSupX - 1) / kSupX, nsy = (nby + kSupY - 1) / kSupY, nsz = (nbz + kSupZ - 1) / kSupZ;
  if constexpr (MODE == 0) t1 = (a.q + kTileM - 1) / kTileM;
  else if constexpr (MODE == 1) { t0 *= kSubs; t1 = (long long)kSubs * nsx * nsy * nsz; }
  else { t0 += a.tile0; t1 = min(a.tile1, (long long)*a.ntiles_dev); }
  const long long tstep = gridDim.x;
  for (long long tile = t0; tile < t1;
       tile = MODE == 1 ? (tile % kSubs == kSubs - 1 ? tile + kSubs * (tstep - 1) + 1 : tile + 1) : tile + tstep) {
    const int slot = MODE == 3 ? a.tile_slot[tile] : 0;
    if (slot != cur) {   // one TMA bulk copy of this block's prepared weight image
      __syncthreads();
      if (t == 0) {
        mbar_expect_tx(mbar_img, lay.img_bytes);
        bulk_g2s(smem_u32(smem), a.wimg + (size_t)slot * lay.img_bytes, lay.img_bytes, mbar_img);
      }
      mbar_wait(mbar_img, img_phase);
      img_phase ^= 1;
      cur = slot;
    }
    const ModelDev& md = g.md[slot];
    const float* P = md.params;
    const long long j = tile * kTileM + r;
    bool valid;
    float x[3] = {0.f, 0.f, 0.f};
    long long dst = 0;
    if constexpr (MODE == 0) {
      valid = j < a.q;
      if (valid) { x[0] = __ldg(a.x01 + 3 * j); x[1] = __ldg(a.x01 + 3 * j + 1); x[2] = __ldg(a.x01 + 3 * j + 2); }
    } else if constexpr (MODE == 1) {
      // brick (bx, by, bz) of 8 x 4 x 4 lattice points, sub-brick (tile & 7) of super-brick
      // tile >> 3; points past cnt are computed at the clamped (last) lattice point and not
      // stored (32-bit: a grid whose output fits in device memory has < 2^31 bricks)
      const unsigned su = (unsigned)(tile / kSubs), sr = su / (unsigned)nsx;
      const int sx = (int)(su - sr * nsx), sy = (int)(sr % (unsigned)nsy), sz = (int)(sr / (unsigned)nsy);
      const int sub = (int)(tile % kSubs);
      const int bx = kSupX * sx + sub % kSupX, by = kSupY * sy + (sub / kSupX) % kSupY, bz = kSupZ * sz + sub / (kSupX * kSupY);
      if (bx >= nbx || by >= nby || bz >= nbz) continue;   // (uniform over the CTA)
      const int jx = bx * kBrickX + (r & 7), jy = by * kBrickY + ((r >> 3) & 3), jz = bz * kBrickZ + (r >> 5);
      valid = jx < a.cnt[0] && jy < a.cnt[1] && jz < a.cnt[2];
      const int jj[3] = {min(jx, a.cnt[0] - 1), min(jy, a.cnt[1] - 1), min(jz, a.cnt[2] - 1)};
#pragma unroll
      for (int d = 0; d < 3; ++d)
        x[d] = a.rinv[d] != 0.f ? (float)jj[d] * a.rinv[d] : __fdiv_rn((float)jj[d], (float)a.res[d]);
      if (md.mesh[0]) {   // rectilinear (R36): the block's nodes (no staging: nst = 0)
#pragma unroll
        for (int d = 0; d < 3; ++d) x[d] = mesh_x(md, d, md.mesh[d][min(jj[d], md.mesh_n[d] - 1)]);
      }
      dst = jx * a.os[0] + jy * a.os[1] + jz * a.os[2];
      if (sub == 0 && a.nst > 0 && t < 32) {
        // the super-brick's vertex box per staged level (lane l: level l): lo / n per axis from
        // its first and last lattice point, with level_cell's pinned arithmetic
        int* box = reinterpret_cast<int*>(smem + lay.stbox);
        if (t < a.nst) {
          const int b0[3] = {sx * kSupX * kBrickX, sy * kSupY * kBrickY, sz * kSupZ * kBrickZ};
          const int b1[3] = {min(b0[0] + kSupX * kBrickX, a.cnt[0]) - 1, min(b0[1] + kSupY * kBrickY, a.cnt[1]) - 1,
                             min(b0[2] + kSupZ * kBrickZ, a.cnt[2]) - 1};
          const uint32_t res = net.lv[t].res;
          int lo[3], n[3];
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            lo[d] = cell_of(__fdiv_rn((float)b0[d], (float)a.res[d]), res);
            n[d] = cell_of(__fdiv_rn((float)b1[d], (float)a.res[d]), res) + 2 - lo[d];
          }
          *reinterpret_cast<int4*>(box + 8 * t) = make_int4(lo[0], lo[1], lo[2], n[0]);
          *reinterpret_cast<int4*>(box + 8 * t + 4) = make_int4(n[1], n[2], n[0] * n[1] * n[2], 0);
        }
      }
    } else {
      const int qi = a.perm[j];
      valid = qi >= 0;
      dst = qi;
    }
    if constexpr (MODE == 3) {   // the level-major encoded h_0 tile, one bulk copy
      if (t == 0) {
        mbar_expect_tx(mbar_feat, lay.feat_tile_bytes);
        bulk_g2s(smem_u32(smem + lay.h[0]), a.featimg + (size_t)(tile - a.tile0) * lay.feat_tile_bytes,
                 lay.feat_tile_bytes, mbar_feat);
      }
      mbar_wait(mbar_feat, feat_phase);
      feat_phase ^= 1;
    } else {
      // features straight into row r of the h_0 tile; this thread: levels l = hf, hf + 2, ...
      uint8_t* row = smem + lay.h[0] + (r & 7) * 16 + (r >> 3) * lay.h_sbo[0];
      if constexpr (MODE == 0) {
#pragma unroll 2
        for (int l = hf; l < net.L; l += 2) {
          float fl[F];
          encode_level<F>(P, net.lv[l], net.table_mask, x, fl);
          put_feat<F>(row, l * F, fl);
        }
      } else {
        // this half's vertex-aligned fine levels (R19: one entry each) are gathered in
        // batches whose loads are all in flight before any is used; the first batch
        // flies while this half's staged coarse levels blend from shared memory
        constexpr int NB = F == 1 ? 8 : F == 2 ? 6 : 16 / F;   // batch: <= 16 fp32 registers of gathered entries
        FVec<F> e[NB];
        const int lf0 = a.na + ((a.na & 1) != hf);   // this half's first aligned level
        auto issue = [&](int l0) {
#pragma unroll
          for (int u = 0; u < NB; ++u)
            if (l0 + 2 * u < net.L) {
              const LevelInfo& lv = net.lv[l0 + 2 * u];
              const float N = (float)lv.res;
              const uint32_t v0 = (uint32_t)__fmul_rn(x[0], N), v1 = (uint32_t)__fmul_rn(x[1], N),
                             v2 = (uint32_t)__fmul_rn(x[2], N);
              e[u] = load_entry<F>(P + lv.offset + (size_t)vertex_index(v0, v1, v2, lv, net.table_mask) * F);
            }
        };
        auto consume = [&](int l0) {
#pragma unroll
          for (int u = 0; u < NB; ++u)
            if (l0 + 2 * u < net.L) {
              float fl[F];
#pragma unroll
              for (int f = 0; f < F; ++f) fl[f] = fmaf(1.f, e[u].v[f], 0.f);   // == the 8-corner sum (R19)
              put_feat<F>(row, (l0 + 2 * u) * F, fl);
            }
        };
        issue(lf0);
        if (a.nst > 0 && (MODE != 1 || tile % kSubs == 0)) {   // (MODE 1: once per super-brick)
          // stage the staged levels' vertex boxes: one entry per thread over the
          // concatenated boxes (every load in flight at once, with the fine gathers above)
          __syncthreads();   // the box table
          const int* box = reinterpret_cast<const int*>(smem + lay.stbox);
          float* stage = reinterpret_cast<float*>(smem + lay.stage);
          int l = 0, base = 0;
          for (int v = t;; v += kFwdThreads) {
            while (l < a.nst && v >= base + box[8 * l + 6]) base += box[8 * l + 6], ++l;
            if (l >= a.nst) break;
            const int4 b4 = *reinterpret_cast<const int4*>(box + 8 * l);
            const int n1 = box[8 * l + 4];
            const int w = v - base;
            const int vx = w % b4.w, vy = (w / b4.w) % n1, vz = w / (b4.w * n1);
            const LevelInfo& lv = net.lv[l];
            const uint32_t idx = vertex_index(b4.x + vx, b4.y + vy, b4.z + vz, lv, net.table_mask);
            const FVec<F> ev = load_entry<F>(P + lv.offset + (size_t)idx * F);
#pragma unroll
            for (int f = 0; f < F; ++f) stage[a.st_off[l] + w * F + f] = ev.v[f];
          }
          __syncthreads();   // the staged entries
        }
        for (int l = hf; l < a.na; l += 2) {
          float fl[F];
          if (l < a.nst) {
            const int* box = reinterpret_cast<const int*>(smem + lay.stbox) + 8 * l;
            const int4 b4 = *reinterpret_cast<const int4*>(box);
            const int4 b5 = *reinterpret_cast<const int4*>(box + 4);
            const int lo[3] = {b4.x, b4.y, b4.z}, n[3] = {b4.w, b5.x, b5.y};
            blend_staged<F>(reinterpret_cast<const float*>(smem + lay.stage) + a.st_off[l], lo, n, net.lv[l].res, x,
                            fl);
          } else {
            encode_level_infer<F>(P, net.lv[l], net.table_mask, x, fl);
          }
          put_feat<F>(row, l * F, fl);
        }
        consume(lf0);
        for (int l0 = lf0 + 2 * NB; l0 < net.L; l0 += 2 * NB) {
          issue(l0);
          consume(l0);
        }
      }
    }
    fence_async_smem();
    fence_before();
    __syncthreads();
    for (int k = 0; k < H; ++k) {
      if (t == 0) {
        fence_after();
        gemm(tmem, smem_u32(smem + lay.h[k]), 128, lay.h_sbo[k], 256, smem_u32(smem + lay.w[k]), 128,
             lay.w_sbo[k], 256, net.in_dim[k] / 16, make_idesc(128, 64, 0, 0), false);
        mma_commit(mbar);
      }
      mbar_wait(mbar, phase);
      phase ^= 1;
      fence_after();
      float z[32];
      tmem_ld16(tmem + lane_base + cb, z);
      tmem_ld16(tmem + lane_base + cb + 16, z + 16);
      tmem_wait_ld();
#pragma unroll
      for (int n = 0; n < 32; n += 4) {
        const float4 b4 = *reinterpret_cast<const float4*>(bias + k * 64 + cb + n);
        z[n] += b4.x;
        z[n + 1] += b4.y;
        z[n + 2] += b4.z;
        z[n + 3] += b4.w;
      }
      if (k + 1 < H) {
        // ReLU on packed fp16 pairs: max(round(z + b), 0) == round(max(z + b, 0))
        uint8_t* tile = smem + lay.h[k + 1] + (r & 7) * 16 + (r >> 3) * lay.h_sbo[k + 1] + hf * 4 * 128;
        const __half2 zero2 = __float2half2_rn(0.f);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u;
          __half2 h0 = __hmax2(__floats2half2_rn(z[8 * q], z[8 * q + 1]), zero2);
          __half2 h1 = __hmax2(__floats2half2_rn(z[8 * q + 2], z[8 * q + 3]), zero2);
          __half2 h2 = __hmax2(__floats2half2_rn(z[8 * q + 4], z[8 * q + 5]), zero2);
          __half2 h3 = __hmax2(__floats2half2_rn(z[8 * q + 6], z[8 * q + 7]), zero2);
          u.x = *reinterpret_cast<uint32_t*>(&h0);
          u.y = *reinterpret_cast<uint32_t*>(&h1);
          u.z = *reinterpret_cast<uint32_t*>(&h2);
          u.w = *reinterpret_cast<uint32_t*>(&h3);
          *reinterpret_cast<uint4*>(tile + q * 128) = u;
        }
      } else {   // the 64 -> D output layer, fp32 on CUDA cores: this half's 32 columns
#pragma unroll
        for (int c = 0; c < D; ++c) {
          float yp = 0.f;
#pragma unroll
          for (int n = 0; n < 32; ++n) yp = fmaf(wout[c * 64 + cb + n], fmaxf(z[n], 0.f), yp);
          ypart[(2 * c + hf) * kTileM + r] = yp;
        }
      }
      fence_async_smem();
      fence_before();
      __syncthreads();
    }
    if (hf == 0) {
      float y[D];
#pragma unroll
      for (int c = 0; c < D; ++c) y[c] = wout[D * 64 + c] + ypart[(2 * c) * kTileM + r] + ypart[(2 * c + 1) * kTileM + r];
      if constexpr (MODE == 0) {
        if (valid) {
#pragma unroll
          for (int c = 0; c < D; ++c) a.y[j * D + c] = y[c];
        }
      } else {
        double e = 0.0;
        if (valid) {
          if constexpr (MODE == 3) dst *= D;   // query outputs: q x D, channels interleaved
#pragma unroll
          for (int c = 0; c < D; ++c) {
            const float v = fmaf(y[c], md.vrange[c], md.vmin[c]);
            a.out[dst + c] = v;
            if (MODE == 1 && a.ref) {
              // a constant channel (vrange 0) is 0 in normalized units on both sides
              const double dd =
                  md.vrange[c] > 0.f ? ((double)v - (double)__ldg(a.ref + dst + c)) / (double)md.vrange[c] : 0.0;
              e += dd * dd;
            }
          }
        }
        if (MODE == 1 && a.sse) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
          if (lane == 0 && e != 0.0) atomicAdd(a.sse, e);
        }
      }
    }
  }
  mlp_teardown(tmem, lay);
}

template <int MODE>
static void launch_forward(const GroupArgs& g, const FwdArgs& a0, long long ntiles_hint, cudaStream_t st) {
  Layout L;
  if (!build_layout(g.net, L, false)) return;
  FwdArgs a = a0;
  uint8_t* wimg = nullptr;   // the models' fp16 weight images (stream-ordered scratch)
  if (cudaMallocAsync((void**)&wimg, (size_t)g.nmodels * L.img_bytes, st) != cudaSuccess) return;
  a.wimg = wimg;
  prep_image_kernel<<<dim3(g.nmodels, 16), dim3(64, 4), 0, st>>>(g, L, wimg);
  count_launch();
  unsigned grid = (unsigned)std::max<long long>(1, std::min<long long>(ntiles_hint, 148ll * L.ctas_per_sm));
  switch (g.net.F * 10 + g.net.D) {
#define CASE_FD(FF, DD)                                                                                             \
  case FF * 10 + DD:                                                                                                \
    cudaFuncSetAttribute(forward_tc_kernel<FF, MODE, DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, L.bytes);   \
    forward_tc_kernel<FF, MODE, DD><<<grid, kFwdThreads, L.bytes, st>>>(g, a, L);                                     \
    break;
    CASE_FD(1, 1) CASE_FD(2, 1) CASE_FD(4, 1) CASE_FD(8, 1) CASE_FD(1, 3) CASE_FD(2, 3) CASE_FD(4, 3) CASE_FD(8, 3)
#undef CASE_FD
    default: break;
  }
  count_launch();
  cudaFreeAsync(wimg, st);
}

static GroupArgs* single_group(const NetDesc& net, const ModelDev& md) {
  static thread_local GroupArgs g;
  g.net = net;
  g.nmodels = 1;
  g.md[0] = md;
  return &g;
}

void launch_debug_forward_tc(const NetDesc& net, const float* P, const float* x01, long long q, float* y,
                             cudaStream_t st) {
  ModelDev md;
  memset(&md, 0, sizeof md);
  md.params = const_cast<float*>(P);
  FwdArgs a;
  memset(&a, 0, sizeof a);
  a.x01 = x01;
  a.y = y;
  a.q = q;
  launch_forward<0>(*single_group(net, md), a, (q + kTileM - 1) / kTileM, st);
}

void launch_decode_grid_tc(const NetDesc& net, const ModelDev& md, const int res[3], const int cnt[3], float* out,
                           const long long os[3], const float* ref, double* sse, cudaStream_t st) {
  FwdArgs a;
  memset(&a, 0, sizeof a);
  for (int d = 0; d < 3; ++d) { a.res[d] = res[d]; a.cnt[d] = cnt[d]; a.os[d] = os[d]; }
  a.out = out;
  a.ref = ref;
  a.sse = sse;
  // staged levels: the coarse levels (N_l < R on every axis) whose worst-case vertex
  // box per brick, (ceil((B_d - 1) N_l / R_d) + 2) per axis, fits the stage area
  const int B[3] = {kSupX * kBrickX, kSupY * kBrickY, kSupZ * kBrickZ};   // the staged super-brick
  int off = 0;
  a.nst = 0;
  a.st_off[0] = 0;
  for (int l = 0; l < net.L && !md.mesh[0]; ++l) {
    const long long N = net.lv[l].res;
    long long cap = 1;
    bool coarse = true;
    for (int d = 0; d < 3; ++d) {
      coarse &= N < res[d];
      cap *= ((long long)(B[d] - 1) * N + res[d] - 1) / res[d] + 2;
    }
    if (!coarse || off + cap * net.F > kStageFloats) break;
    off += (int)cap * net.F;
    a.nst = l + 1;
    a.st_off[l + 1] = off;
  }
  // vertex-aligned levels: x_j = j / R_d is exact (R_d a power of two) and N_l a
  // multiple of R_d, so x_j N_l is an integer vertex for every lattice point (R19)
  a.na = net.L;
  for (int l = net.L - 1; l >= a.nst && !md.mesh[0]; --l) {
    bool al = true;
    for (int d = 0; d < 3; ++d)
      al &= (res[d] & (res[d] - 1)) == 0 && net.lv[l].res % (uint32_t)res[d] == 0;
    if (!al) break;
    a.na = l;
  }
  for (int d = 0; d < 3; ++d) a.rinv[d] = (res[d] & (res[d] - 1)) == 0 ? 1.f / (float)res[d] : 0.f;
  const long long nbx = (cnt[0] + kBrickX - 1) / kBrickX, nby = (cnt[1] + kBrickY - 1) / kBrickY,
                  nbz = (cnt[2] + kBrickZ - 1) / kBrickZ;
  const long long nsb = ((nbx + kSupX - 1) / kSupX) * ((nby + kSupY - 1) / kSupY) * ((nbz + kSupZ - 1) / kSupZ);
  launch_forward<1>(*single_group(net, md), a, nsb, st);
}

// Queries: per chunk of <= 2^15 bucketed tiles, x per query (query_prep_kernel),
// level-major fp16 encode into tile images (encode_query_kernel), then the
// tensor-core MLP over the tiles (MODE 3).  Stream-ordered chunk workspace.
void launch_decode_query_tc(const GroupArgs& g, const float* xyz, long long q, float* out, const QueryBuckets& b,
                            cudaStream_t st) {
  Layout L;
  if (!build_layout(g.net, L, false)) return;
  const long long ub = q / kTileM + g.nmodels + 1;        // upper bound of the device tile count
  const long long nchunks = (ub + (1ll << 15) - 1) >> 15;   // balanced chunks of <= ~2^15 tiles
  const long long chunk = (ub + nchunks - 1) / nchunks;
  FeatGeom geom;
  geom.sbo = L.h_sbo[0];
  geom.tile_bytes = L.feat_tile_bytes;
  geom.ones = 0;
  uint8_t* ws = nullptr;
  const size_t qx_bytes = (size_t)chunk * kTileM * sizeof(float4);
  if (cudaMallocAsync((void**)&ws, qx_bytes + (size_t)chunk * L.feat_tile_bytes, st) != cudaSuccess) return;
  float4* qx = reinterpret_cast<float4*>(ws);
  uint8_t* featimg = ws + qx_bytes;
  for (long long c0 = 0; c0 < ub; c0 += chunk) {
    const long long nt = std::min(chunk, ub - c0);
    launch_query_prep(g, xyz, b, c0 * kTileM, nt * kTileM, qx, st);
    launch_encode_query(g, qx, nt * kTileM, featimg, geom, st);
    FwdArgs a;
    memset(&a, 0, sizeof a);
    a.out = out;
    a.perm = b.perm;
    a.tile_slot = b.tile_slot;
    a.ntiles_dev = b.ntiles;
    a.featimg = featimg;
    a.tile0 = c0;
    a.tile1 = c0 + nt;
    launch_forward<3>(g, a, nt, st);
  }
  cudaFreeAsync(ws, st);
}

}  // namespace inr
