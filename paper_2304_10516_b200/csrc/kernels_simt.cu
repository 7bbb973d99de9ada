// kernels_simt.cu — fp32 CUDA-core kernels of libinr (sm_100a):
//   * parameter init (R14), step bookkeeping, the fused fp32 fit step
//     (sample -> target -> encode -> MLP fwd -> Eq. 2 -> MLP bwd -> scatter),
//     the PyTorch-form Adam (R12), decode (grid / query), probe PSNR,
//     value range, debug encode/forward.
// The fp32 fit kernel is the parity mode (INR_PREC_FP32); the tensor-core fit
// kernel for INR_PREC_FP16_MLP lives in kernels_tc.cu and shares the sampler,
// encode and scatter code of common.cuh.
#include <algorithm>

#include "adam.cuh"
#include "common.cuh"
#include "launch.h"
#include "tc_common.cuh"

namespace inr {

constexpr int kTile = 64;        // samples per CTA (one per thread) in the SIMT kernels
constexpr int kLd = kTile + 1;   // smem row stride (bank-conflict-free column access)

// ----------------------------------------------------------------- init
// value_j = fl32(lo + (hi - lo) * U_j) in fp64 with each op rounded, U_j =
// u01(Philox(key(seed, 0), (j, block_id, 0, 0)).x) (R14).
__global__ void init_params_kernel(NetDesc net, float* __restrict__ params, uint32_t k0, uint32_t k1,
                                   uint32_t block_id) {
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < net.nparams;
       p += (long long)gridDim.x * blockDim.x) {
    float v = 0.f;  // padding and biases
    for (int t = 0; t < net.ntensors; ++t) {
      if (p < net.t_off[t] || p >= net.t_off[t] + net.t_len[t]) continue;
      const int fan = net.t_fan_in[t];
      if (fan < 0) break;
      const long long j = net.t_decl[t] + (p - net.t_off[t]);   // declared index: the Philox counter
      const double a = fan == 0 ? 1e-4 : sqrt(6.0 / (double)fan);
      U4 u = philox((uint32_t)j, block_id, 0u, 0u, k0, k1);
      double U = (double)(u.x >> 8) * 5.9604644775390625e-08;
      double lo = -a, hi = a;
      v = __double2float_rn(__dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), U)));
      break;
    }
    params[p] = v;
  }
}

// --------------------------------------------------------- step bookkeeping
// Zero this step's gradient accumulators and loss sums; step_cur <- step_total++.
__global__ void step_begin_kernel(GroupArgs g, long long zero_from) {
  const ModelDev& md = g.md[blockIdx.y];
  long long n = g.net.nparams;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    long long s = *md.step_total;
    *md.step_cur = s;
    *md.step_total = s + 1;
    md.acc[0] = 0.0;
    md.acc[1] = 0.0;
  }
  long long stride = (long long)gridDim.x * blockDim.x;
  long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (md.grads_fx) {
    for (long long i = zero_from + i0; i < n; i += stride) md.grads_fx[i] = 0ull;
  } else {   // zero_from and n are multiples of 64
    float4* g4 = reinterpret_cast<float4*>(md.grads);
    for (long long i = zero_from / 4 + i0; i < n / 4; i += stride) g4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
}

// ------------------------------------------------------------ SIMT MLP fwd
// act: smem rows of kLd floats; rows [0, LF) hold the features of the tile;
// rows LF + 64 k + n hold the pre-activation z_k[n] of hidden layer k.
// Writes y[0..D).  h_{k+1} = max(z_k, 0).
__device__ void mlp_forward_simt(const NetDesc& net, const float* __restrict__ P, float* act, int t,
                                 float y[kMaxD]) {
  const float* hin = act;
  int in = net.LF;
  bool relu = false;
  for (int k = 0; k < net.H; ++k) {
    const float* W = P + net.w_off[k];
    float* z = act + (size_t)(net.LF + kWidth * k) * kLd;
    for (int n = 0; n < kWidth; ++n) {
      float acc = net.bias ? __ldg(P + net.b_off[k] + n) : 0.f;
      const float* Wr = W + (size_t)n * in;
      for (int i = 0; i < in; ++i) {
        float h = hin[i * kLd + t];
        if (relu) h = fmaxf(h, 0.f);
        acc = fmaf(__ldg(Wr + i), h, acc);
      }
      z[n * kLd + t] = acc;
    }
    hin = z;
    in = kWidth;
    relu = true;
  }
  for (int c = 0; c < net.D; ++c) {
    const float* W = P + net.w_off[net.H] + (size_t)c * in;
    float acc = net.bias ? __ldg(P + net.b_off[net.H] + c) : 0.f;
    for (int i = 0; i < in; ++i) {
      float h = hin[i * kLd + t];
      if (relu) h = fmaxf(h, 0.f);
      acc = fmaf(__ldg(W + i), h, acc);
    }
    y[c] = acc;
  }
}

__device__ __forceinline__ void sample_target_rt(const ModelDev& md, int D, const float x[3], float t[kMaxD]) {
  if (D == 1) sample_target<1>(md, x, t);
  else sample_target<3>(md, x, t);
}

template <int F>
__device__ __forceinline__ void encode_to_smem(const NetDesc& net, const float* __restrict__ P, const float x[3],
                                               float* act, int t) {
  for (int l = 0; l < net.L; ++l) {
    float f[F];
    encode_level<F>(P, net.lv[l], net.table_mask, x, f);
#pragma unroll
    for (int j = 0; j < F; ++j) act[(l * F + j) * kLd + t] = f[j];
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// --------------------------------------------------------- fused fit (fp32)
// One CTA = kTile samples of one model; blockIdx.y = model.  Sample i < B_u is
// uniform, B_u <= i < B_u + B_b boundary (B_b = 0 for blocks without interior
// faces, lambda' = 0 then [R11]).  The per-tile MLP weight gradient is summed in
// sample order inside the CTA and added once per tile (atomic or exact int64).
template <int F>
__global__ void __launch_bounds__(kTile) fit_simt_kernel(GroupArgs g, FitScalars fs) {
  extern __shared__ float smem[];
  const NetDesc& net = g.net;
  const ModelDev& md = g.md[blockIdx.y];
  const int t = threadIdx.x;
  const int B_b = md.nfaces > 0 ? fs.B_b : 0;
  const int total = fs.B_u + B_b;
  const int i = blockIdx.x * kTile + t;
  if (blockIdx.x * kTile >= total) return;
  const bool valid = i < total;
  const float* __restrict__ P = md.params;
  float* __restrict__ G = md.grads;
  unsigned long long* __restrict__ GX = md.grads_fx;

  float* act = smem;                                   // (LF + 64 H) rows
  float* dzA = act + (size_t)(net.LF + kWidth * net.H) * kLd;
  float* dzB = dzA + (size_t)kWidth * kLd;
  __shared__ double red[2][kTile / 32];

  const uint32_t step = (uint32_t)*md.step_cur;
  const int D = net.D;
  float x[3] = {0.f, 0.f, 0.f};
  float target[kMaxD] = {0.f, 0.f, 0.f};
  if (valid) {
    draw_sample(md, i, fs.B_u, step, x);
    sample_target_rt(md, D, x, target);
  }
  encode_to_smem<F>(net, P, x, act, t);
  // No barrier needed: every thread only touches its own smem column until the
  // per-tile weight-gradient reduction below.
  float y[kMaxD];
  mlp_forward_simt(net, P, act, t, y);

  // Eq. 2 (L1 pooled over the D channels, R28): dL/dy_c = (1 - lambda') sgn(y_c - t_c) / (B_u D)
  // (uniform) or lambda' sgn / (B_b D).
  float lam = B_b > 0 ? fs.lambda : 0.f;
  bool is_b = i >= fs.B_u;
  float dy[kMaxD];
  double ad = 0.0;
  for (int c = 0; c < D; ++c) {
    float d = y[c] - target[c];
    float sg = valid ? (d > 0.f ? 1.f : (d < 0.f ? -1.f : 0.f)) : 0.f;
    dy[c] = is_b ? lam * sg / (float)(max(B_b, 1) * D) : (1.f - lam) * sg / (float)(fs.B_u * D);
    ad += fabs((double)d);
  }
  {
    double au = (valid && !is_b) ? ad : 0.0;
    double ab = (valid && is_b) ? ad : 0.0;
    au = warp_sum(au);
    ab = warp_sum(ab);
    if ((t & 31) == 0) { red[0][t >> 5] = au; red[1][t >> 5] = ab; }
  }

  // ---- backward through the output layer
  const int H = net.H;
  const float* hH = act + (size_t)(net.LF + kWidth * (H - 1)) * kLd;   // z_{H-1}
  {
    const float* Wo = P + net.w_off[H];
    for (int n = 0; n < kWidth; ++n) {
      float z = hH[n * kLd + t];
      float acc = 0.f;
      for (int c = 0; c < D; ++c) acc = fmaf(__ldg(Wo + (size_t)c * kWidth + n), dy[c], acc);
      dzA[n * kLd + t] = z > 0.f ? acc : 0.f;                            // dz_{H-1}
    }
  }
  __shared__ float dys[kMaxD][kTile];
  for (int c = 0; c < D; ++c) dys[c][t] = dy[c];
  __syncthreads();
  if (t == 0) {
    double su = 0, sb = 0;
    for (int w = 0; w < kTile / 32; ++w) { su += red[0][w]; sb += red[1][w]; }
    if (su != 0.0) atomicAdd(md.acc + 0, su);
    if (sb != 0.0) atomicAdd(md.acc + 1, sb);
  }
  // dW_H[c][n] = sum_s dy_c,s relu(z_{H-1}[n][s]); db_H[c] = sum_s dy_c,s  (thread n owns column n)
  for (int c = 0; c < D; ++c) {
    float acc = 0.f;
    for (int s = 0; s < kTile; ++s) acc = fmaf(dys[c][s], fmaxf(hH[t * kLd + s], 0.f), acc);
    if (acc != 0.f) grad_add(G, GX, net.w_off[H] + (size_t)c * kWidth + t, acc);
    if (net.bias && t == 0) {
      float b = 0.f;
      for (int s = 0; s < kTile; ++s) b += dys[c][s];
      if (b != 0.f) grad_add(G, GX, net.b_off[H] + c, b);
    }
  }
  // ---- hidden layers k = H-1 .. 0:  z_k = W_k h_k + b_k
  float* dz = dzA;
  float* dzn = dzB;
  float dfeat[64];
  for (int k = H - 1; k >= 0; --k) {
    const int in = net.in_dim[k];
    const float* hk = k == 0 ? act : act + (size_t)(net.LF + kWidth * (k - 1)) * kLd;
    const bool relu = k > 0;
    // weight gradient of layer k: entry e = n*in + ii, summed over the tile in sample order
    for (int e = t; e < kWidth * in; e += kTile) {
      int n = e / in, ii = e - n * in;
      float acc = 0.f;
      for (int s = 0; s < kTile; ++s) {
        float h = hk[ii * kLd + s];
        if (relu) h = fmaxf(h, 0.f);
        acc = fmaf(dz[n * kLd + s], h, acc);
      }
      if (acc != 0.f) grad_add(G, GX, net.w_off[k] + e, acc);
    }
    if (net.bias) {
      float acc = 0.f;
      for (int s = 0; s < kTile; ++s) acc += dz[t * kLd + s];
      if (acc != 0.f) grad_add(G, GX, net.b_off[k] + t, acc);
    }
    // dh_k = W_k^T dz_k for this thread's sample; dz_{k-1} = dh_k * 1[z_{k-1} > 0]
    const float* W = P + net.w_off[k];
    if (k > 0) {
      const float* zprev = act + (size_t)(net.LF + kWidth * (k - 1)) * kLd;
      for (int ii = 0; ii < in; ++ii) {
        float acc = 0.f;
        for (int n = 0; n < kWidth; ++n) acc = fmaf(__ldg(W + (size_t)n * in + ii), dz[n * kLd + t], acc);
        dzn[ii * kLd + t] = zprev[ii * kLd + t] > 0.f ? acc : 0.f;
      }
      __syncthreads();
      float* tmp = dz; dz = dzn; dzn = tmp;
    } else {
      for (int ii = 0; ii < in; ++ii) {
        float acc = 0.f;
        for (int n = 0; n < kWidth; ++n) acc = fmaf(__ldg(W + (size_t)n * in + ii), dz[n * kLd + t], acc);
        dfeat[ii] = acc;
      }
    }
  }
  // ---- table scatter-add
  if (valid) {
    for (int l = 0; l < net.L; ++l) {
      float df[F];
#pragma unroll
      for (int j = 0; j < F; ++j) df[j] = dfeat[l * F + j];
      scatter_level<F>(G, GX, net.lv[l], net.table_mask, x, df);
    }
  }
}

// ------------------------------------------------------------------- Adam
// PyTorch torch.optim.Adam (R12): m = b1 m + (1-b1) g; v = b2 v + (1-b2) g^2;
// p -= (lr/bc1) m / (sqrt(v)/sqrt(bc2) + eps); lr = lr0 decay^floor(s/lr_step) (R13).
// Deterministic mode converts the exact int64 sums to fp32 first.
template <int SIDE>   // SIDE: launched beside the MLP (its own carveout attribute)
__global__ void adam_kernel(GroupArgs g, AdamScalars as) {
  const ModelDev& md = g.md[blockIdx.y];
  const AdamStep a = adam_step_scalars(*md.step_cur, as.lr0, as.lr_decay, as.lr_step, as.beta1, as.beta2, as.b1,
                                       as.b2, as.ob1, as.ob2, as.eps);
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  const bool bad = as.sparse ? adam_range_sparse(md, a, 0, as.table_end, tid, nth) |
                                   adam_range(md, a, as.table_end, g.net.nparams, tid, nth)
                             : adam_range(md, a, 0, g.net.nparams, tid, nth);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(md.flag, 1);
}

// Adam with its operands streamed by TMA bulk copies (same arithmetic as adam4): each
// CTA owns a contiguous run of chunks of one model's p, g, m, v, kept STAGES deep in
// flight in shared memory instead of in registers, so a few warps per SM keep HBM
// busy -- the split fit step runs it on the SMs' spare warps beside the tensor-core
// MLP (whose CTAs hold half the register file).  Per stage a "full" mbarrier (the
// bulk copies' bytes) and an "empty" one (one arrival per warp done with it): the
// warps run ahead independently; only the issuing thread waits for a stage to drain.
// Plain fp32 gradients only (the deterministic mode and R37 use adam_kernel).
constexpr size_t adam_tma_smem(int chunk, int stages) { return (size_t)stages * 4 * chunk * 4 + stages * 16; }

template <int THREADS, int CHUNK, int STAGES>
__global__ void __launch_bounds__(THREADS) adam_tma_kernel(GroupArgs g, AdamScalars as) {
  extern __shared__ __align__(128) uint8_t adam_smem[];
  constexpr int kWarps = THREADS / 32, C4 = CHUNK / 4;
  const ModelDev& md = g.md[blockIdx.y];
  const AdamStep a = adam_step_scalars(*md.step_cur, as.lr0, as.lr_decay, as.lr_step, as.beta1, as.beta2, as.b1,
                                       as.b2, as.ob1, as.ob2, as.eps);
  const int t = threadIdx.x;
  float* stage = reinterpret_cast<float*>(adam_smem);   // [stage][p, g, m, v][CHUNK]
  const uint32_t full0 = tc::smem_u32(adam_smem + (size_t)STAGES * 4 * CHUNK * 4);
  const uint32_t empty0 = full0 + 8 * STAGES;
  const long long n = g.net.nparams;
  const long long nch = (n + CHUNK - 1) / CHUNK;
  const long long per = (nch + gridDim.x - 1) / gridDim.x;
  const long long c0 = (long long)blockIdx.x * per, c1 = min(nch, c0 + per);
  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(full0 + 8 * s, 1);
      tc::mbar_init(empty0 + 8 * s, kWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const float* src[4] = {md.params, md.grads, md.adam_m, md.adam_v};
  auto issue = [&](long long c) {
    const int s = (int)((c - c0) % STAGES);
    const long long off = c * CHUNK;
    const uint32_t bytes = (uint32_t)(min((long long)CHUNK, n - off) * 4);
    tc::fence_async_smem();   // the stage's previous contents were read by the generic proxy
    tc::mbar_expect_tx(full0 + 8 * s, 4 * bytes);
    for (int q = 0; q < 4; ++q)
      tc::bulk_g2s(tc::smem_u32(stage + ((size_t)s * 4 + q) * CHUNK), src[q] + off, bytes, full0 + 8 * s);
  };
  if (t == 0)
    for (long long c = c0; c < min(c1, c0 + STAGES - 1); ++c) issue(c);
  float4* __restrict__ P = reinterpret_cast<float4*>(md.params);
  float4* __restrict__ M = reinterpret_cast<float4*>(md.adam_m);
  float4* __restrict__ V = reinterpret_cast<float4*>(md.adam_v);
  bool bad = false;
  for (long long c = c0; c < c1; ++c) {
    const long long u = c - c0;
    const int s = (int)(u % STAGES);
    if (t == 0 && c + STAGES - 1 < c1) {
      // chunk c + S - 1 goes where chunk c - 1 was: wait until every warp is done with it
      if (u > 0) tc::mbar_wait(empty0 + 8 * (int)((u - 1) % STAGES), (uint32_t)(((u - 1) / STAGES) & 1));
      issue(c + STAGES - 1);
    }
    tc::mbar_wait(full0 + 8 * s, (uint32_t)((u / STAGES) & 1));
    const float4* sp = reinterpret_cast<const float4*>(stage + (size_t)s * 4 * CHUNK);
    const long long base = c * C4;
    const int cnt4 = (int)(min((long long)CHUNK, n - c * CHUNK) / 4);
#pragma unroll
    for (int k = 0; k < (C4 + THREADS - 1) / THREADS; ++k) {
      const int e = t + k * THREADS;
      if (e < cnt4) {
        float4 pp = sp[e], gg = sp[C4 + e], mm = sp[2 * C4 + e], vv = sp[3 * C4 + e];
#define ADAM1(c)                                                                  \
  mm.c = fmaf(a.b1, mm.c, a.ob1 * gg.c);                                          \
  vv.c = fmaf(a.b2, vv.c, a.ob2 * gg.c * gg.c);                                   \
  pp.c = pp.c - a.step_size * mm.c / (sqrtf(vv.c) * a.inv_sqrt_bc2 + a.eps);      \
  bad |= !isfinite(pp.c);
        ADAM1(x) ADAM1(y) ADAM1(z) ADAM1(w)
#undef ADAM1
        M[base + e] = mm;
        V[base + e] = vv;
        P[base + e] = pp;
      }
    }
    __syncwarp();
    if ((t & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(empty0 + 8 * s) : "memory");
  }
  if (__any_sync(0xffffffffu, bad) && (t & 31) == 0) atomicOr(md.flag, 1);
}

// ------------------------------------------------------------- decode grid
// x_j = fl32(j / R) per axis (R19); v = y (vmax - vmin) + vmin; optional SSE
// in normalized units against ref (R18).
template <int F>
__global__ void __launch_bounds__(kTile) decode_grid_simt_kernel(NetDesc net, ModelDev md, int rx, int ry, int rz,
                                                                 int cx, int cy, int cz,
                                                                 float* __restrict__ out, long long os0,
                                                                 long long os1, long long os2,
                                                                 const float* __restrict__ ref,
                                                                 double* __restrict__ sse) {
  extern __shared__ float smem[];
  const int t = threadIdx.x;
  const long long total = (long long)cx * cy * cz;   // the first c_d of the R_d lattice points per axis
  const long long j = blockIdx.x * (long long)kTile + t;
  const bool valid = j < total;
  int jx = 0, jy = 0, jz = 0;
  if (valid) {
    jx = (int)(j % cx);
    long long r = j / cx;
    jy = (int)(r % cy);
    jz = (int)(r / cy);
  }
  float x[3] = {__fdiv_rn((float)jx, (float)rx), __fdiv_rn((float)jy, (float)ry), __fdiv_rn((float)jz, (float)rz)};
  if (md.mesh[0]) {   // rectilinear (R36): the block's nodes, x_j = fl32((X_{o+j} - P_lo) / (P_hi - P_lo))
    const int jj[3] = {jx, jy, jz};
    for (int d = 0; d < 3; ++d) x[d] = mesh_x(md, d, md.mesh[d][min(jj[d], md.mesh_n[d] - 1)]);
  }
  encode_to_smem<F>(net, md.params, x, smem, t);
  float y[kMaxD];
  mlp_forward_simt(net, md.params, smem, t, y);
  double e = 0.0;
  if (valid) {
    long long off = jx * os0 + jy * os1 + jz * os2;
    for (int c = 0; c < net.D; ++c) {
      float v = fmaf(y[c], md.vrange[c], md.vmin[c]);
      out[off + c] = v;
      if (ref) {
        // a constant channel (vrange 0) is 0 in normalized units on both sides
        double dd = md.vrange[c] > 0.f ? ((double)v - (double)__ldg(ref + off + c)) / (double)md.vrange[c] : 0.0;
        e += dd * dd;
      }
    }
  }
  if (sse) {
    e = warp_sum(e);
    if ((t & 31) == 0 && e != 0.0) atomicAdd(sse, e);
  }
}

// ------------------------------------------------------------ decode query
// Route p to block min(max(floor(p/n),0),B-1) (R5); x = fl32(fl32(p - o) / n).
template <int F>
__global__ void __launch_bounds__(kTile) decode_query_simt_kernel(QueryArgs qa, const float* __restrict__ xyz,
                                                                  long long q, float* __restrict__ out,
                                                                  int* __restrict__ domain_flag) {
  extern __shared__ float smem[];
  const int t = threadIdx.x;
  const long long j = blockIdx.x * (long long)kTile + t;
  const bool valid = j < q;
  float p[3] = {0.f, 0.f, 0.f};
  if (valid) {
    p[0] = __ldg(xyz + 3 * j); p[1] = __ldg(xyz + 3 * j + 1); p[2] = __ldg(xyz + 3 * j + 2);
  }
  int bc[3];
  bool outside = false;
  for (int d = 0; d < 3; ++d) {
    outside |= !(p[d] >= 0.f && p[d] <= (float)(qa.N[d] - 1));
    int b = (int)floorf(__fdiv_rn(p[d], (float)qa.n[d]));
    bc[d] = min(max(b, 0), qa.B[d] - 1);
  }
  int bid = (bc[2] * qa.B[1] + bc[1]) * qa.B[0] + bc[0];
  int slot = bid < qa.nblocks ? qa.slot_of_block[bid] : -1;
  const ModelDev& md = qa.md[slot < 0 ? 0 : slot];
  float x[3];
  for (int d = 0; d < 3; ++d)
    x[d] = md.mesh[0] ? mesh_x(md, d, mesh_physical(md, d, p[d]))          // rectilinear (R36)
                      : __fdiv_rn(__fsub_rn(p[d], (float)md.o[d]), (float)md.n[d]);
  encode_to_smem<F>(qa.net, md.params, x, smem, t);
  float y[kMaxD];
  mlp_forward_simt(qa.net, md.params, smem, t, y);
  if (valid) {   // (slot -2: another chunk of the group decodes this query)
    const int D = qa.net.D;
    if (slot != -2)
      for (int c = 0; c < D; ++c)
        out[j * D + c] = slot < 0 ? __int_as_float(0x7fc00000) : fmaf(y[c], md.vrange[c], md.vmin[c]);
    if (outside && domain_flag) atomicOr(domain_flag, 1);
  }
}

// -------------------------------------------------------------- probe PSNR
// SSE of Phi against sampler targets on the 32^3 cell-centred probe lattice
// x = (j + 0.5)/32, accumulated into md.acc[2].
template <int F>
__global__ void __launch_bounds__(kTile) probe_simt_kernel(GroupArgs g) {
  extern __shared__ float smem[];
  const ModelDev& md = g.md[blockIdx.y];
  const int t = threadIdx.x;
  const int j = blockIdx.x * kTile + t;  // < 32768
  float x[3] = {((j & 31) + 0.5f) / 32.f, (((j >> 5) & 31) + 0.5f) / 32.f, ((j >> 10) + 0.5f) / 32.f};
  float tgt[kMaxD], y[kMaxD];
  sample_target_rt(md, g.net.D, x, tgt);
  encode_to_smem<F>(g.net, md.params, x, smem, t);
  mlp_forward_simt(g.net, md.params, smem, t, y);
  double e = 0.0;
  for (int c = 0; c < g.net.D; ++c) e += (double)(y[c] - tgt[c]) * (double)(y[c] - tgt[c]);
  e = warp_sum(e);
  if ((t & 31) == 0) atomicAdd(md.acc + 2, e);
}

// ------------------------------------------------------ stream-ordered report
// out[3 i .. 3 i + 2] = (L1_uniform, L1_boundary, non-finite flag) of model i's last step
__global__ void loss_report_kernel(LossReportArgs a, double* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const double u = a.acc[i][0], b = a.acc[i][1];
  const int bad = *a.flag[i];
  out[3 * i] = u * a.inv_u[i];
  out[3 * i + 1] = b * a.inv_b[i];
  out[3 * i + 2] = (bad || !isfinite(u) || !isfinite(b)) ? 1.0 : 0.0;
}

void launch_loss_report(const LossReportArgs& a, double* out, cudaStream_t st) {
  loss_report_kernel<<<1, 64, 0, st>>>(a, out);
  count_launch();
}

// ------------------------------------------------------- fp16 cache storage
__global__ void convert_f32_f16_kernel(const float* __restrict__ s, __half* __restrict__ d, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    d[i] = __float2half_rn(s[i]);
}
__global__ void convert_f16_f32_kernel(const __half* __restrict__ s, float* __restrict__ d, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    d[i] = __half2float(s[i]);
}

// ------------------------------------------------------------ value range
__device__ __forceinline__ void atomic_min_f(float* a, float v) {
  if (v >= 0.f) atomicMin(reinterpret_cast<int*>(a), __float_as_int(v));
  else atomicMax(reinterpret_cast<unsigned int*>(a), __float_as_uint(v));
}
__device__ __forceinline__ void atomic_max_f(float* a, float v) {
  if (v >= 0.f) atomicMax(reinterpret_cast<int*>(a), __float_as_int(v));
  else atomicMin(reinterpret_cast<unsigned int*>(a), __float_as_uint(v));
}

// blockIdx.y = channel c (at +c of every node), folded into minmax[2c], [2c+1]
__global__ void range_kernel(const float* __restrict__ base, int dx, int dy, int dz, long long s0, long long s1,
                             long long s2, float* __restrict__ minmax) {
  base += blockIdx.y;
  minmax += 2 * blockIdx.y;
  float lo = __int_as_float(0x7f800000), hi = -lo;
  const long long total = (long long)dx * dy * dz;
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < total;
       j += (long long)gridDim.x * blockDim.x) {
    int ix = (int)(j % dx);
    long long r = j / dx;
    int iy = (int)(r % dy), iz = (int)(r / dy);
    float v = __ldg(base + ix * s0 + iy * s1 + iz * s2);
    lo = fminf(lo, v);
    hi = fmaxf(hi, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomic_min_f(minmax, lo);
    atomic_max_f(minmax + 1, hi);
  }
}

// ----------------------------------------------------------- debug encode
template <int F>
__global__ void debug_encode_kernel(NetDesc net, const float* __restrict__ P, const float* __restrict__ x01,
                                    long long q, uint32_t* __restrict__ idx, float* __restrict__ feat) {
  long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= q) return;
  float x[3] = {__ldg(x01 + 3 * j), __ldg(x01 + 3 * j + 1), __ldg(x01 + 3 * j + 2)};
  for (int l = 0; l < net.L; ++l) {
    if (idx) {
      Cell c = level_cell(x, net.lv[l].res);
      for (int k = 0; k < 8; ++k) idx[(j * net.L + l) * 8 + k] = corner_index(c, k, net.lv[l], net.table_mask);
    }
    if (feat) {
      float f[F];
      encode_level<F>(P, net.lv[l], net.table_mask, x, f);
      for (int k = 0; k < F; ++k) feat[j * net.LF + l * F + k] = f[k];
    }
  }
}

template <int F>
__global__ void __launch_bounds__(kTile) debug_forward_simt_kernel(NetDesc net, const float* __restrict__ P,
                                                                   const float* __restrict__ x01, long long q,
                                                                   float* __restrict__ y) {
  extern __shared__ float smem[];
  const int t = threadIdx.x;
  long long j = blockIdx.x * (long long)kTile + t;
  float x[3] = {0.f, 0.f, 0.f};
  if (j < q) { x[0] = __ldg(x01 + 3 * j); x[1] = __ldg(x01 + 3 * j + 1); x[2] = __ldg(x01 + 3 * j + 2); }
  encode_to_smem<F>(net, P, x, smem, t);
  float v[kMaxD];
  mlp_forward_simt(net, P, smem, t, v);
  if (j < q)
    for (int c = 0; c < net.D; ++c) y[j * net.D + c] = v[c];
}

// ============================================================ host launchers
static size_t simt_fwd_smem(const NetDesc& net) { return (size_t)(net.LF + kWidth * net.H) * kLd * sizeof(float); }
static size_t simt_fit_smem(const NetDesc& net) { return simt_fwd_smem(net) + 2 * (size_t)kWidth * kLd * sizeof(float); }

#define DISPATCH_F(F_, ...)                              \
  switch (F_) {                                          \
    case 1: { constexpr int FF = 1; __VA_ARGS__; } break; \
    case 2: { constexpr int FF = 2; __VA_ARGS__; } break; \
    case 4: { constexpr int FF = 4; __VA_ARGS__; } break; \
    case 8: { constexpr int FF = 8; __VA_ARGS__; } break; \
    default: break;                                      \
  }

template <typename K>
static void set_smem(K kernel, size_t bytes) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

void launch_init_params(const NetDesc& net, float* params, uint32_t k0, uint32_t k1, uint32_t block_id,
                        cudaStream_t st) {
  int blocks = (int)std::min<long long>((net.nparams + 255) / 256, 148 * 16);
  init_params_kernel<<<blocks, 256, 0, st>>>(net, params, k0, k1, block_id);
  count_launch();
}

void launch_step_begin(const GroupArgs& g, int nmodels, long long zero_from, cudaStream_t st) {
  int bx = (int)std::min<long long>(((g.net.nparams - zero_from) / 4 + 255) / 256, 148 * 4 / max(1, nmodels) + 1);
  step_begin_kernel<<<dim3(max(bx, 1), nmodels), 256, 0, st>>>(g, zero_from);
  count_launch();
}

void launch_fit_simt(const GroupArgs& g, int nmodels, const FitScalars& fs, cudaStream_t st) {
  int total = fs.B_u + fs.B_b;
  dim3 grid((total + kTile - 1) / kTile, nmodels);
  size_t sm = simt_fit_smem(g.net);
  DISPATCH_F(g.net.F, set_smem(fit_simt_kernel<FF>, sm); fit_simt_kernel<FF><<<grid, kTile, sm, st>>>(g, fs));
  count_launch();
}

void launch_adam(const GroupArgs& g, int nmodels, const AdamScalars& as, cudaStream_t st, int ctas) {
  if (ctas > 0) {
    // beside the MLP (split fit step): the MLP's shared-memory carveout, so that an SM
    // running the MLP CTA also takes these (a carveout change waits for the SM to drain)
    const int bx = std::max(1, ctas / nmodels);   // at most ctas in all: one per SM beside the MLP
    if (!as.sparse && !g.md[0].grads_fx) {
      constexpr int kT = 512, kC = 2048, kS = 3;   // 96 KB of operands in flight per CTA
      cudaFuncSetAttribute(adam_tma_kernel<kT, kC, kS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)adam_tma_smem(kC, kS));
      cudaFuncSetAttribute(adam_tma_kernel<kT, kC, kS>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      adam_tma_kernel<kT, kC, kS><<<dim3(bx, nmodels), kT, adam_tma_smem(kC, kS), st>>>(g, as);
    } else {
      cudaFuncSetAttribute(adam_kernel<1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      adam_kernel<1><<<dim3(bx, nmodels), 256, 0, st>>>(g, as);
    }
    count_launch();
    return;
  }
  long long per = (g.net.nparams / 4 + 255) / 256;
  int bx = (int)std::max<long long>(1, std::min<long long>(per, (148 * 8 + nmodels - 1) / nmodels));
  adam_kernel<0><<<dim3(bx, nmodels), 256, 0, st>>>(g, as);
  count_launch();
}

void launch_probe(const GroupArgs& g, int nmodels, cudaStream_t st) {
  size_t sm = simt_fwd_smem(g.net);
  DISPATCH_F(g.net.F, set_smem(probe_simt_kernel<FF>, sm);
             probe_simt_kernel<FF><<<dim3(32768 / kTile, nmodels), kTile, sm, st>>>(g));
  count_launch();
}

void launch_decode_grid_simt(const NetDesc& net, const ModelDev& md, const int res[3], const int cnt[3], float* out,
                             const long long os[3], const float* ref, double* sse, cudaStream_t st) {
  long long total = (long long)cnt[0] * cnt[1] * cnt[2];
  size_t sm = simt_fwd_smem(net);
  unsigned grid = (unsigned)((total + kTile - 1) / kTile);
  DISPATCH_F(net.F, set_smem(decode_grid_simt_kernel<FF>, sm);
             decode_grid_simt_kernel<FF><<<grid, kTile, sm, st>>>(net, md, res[0], res[1], res[2], cnt[0], cnt[1],
                                                                  cnt[2], out, os[0], os[1], os[2], ref, sse));
  count_launch();
}

void launch_decode_query_simt(const QueryArgs& qa, const float* xyz, long long q, float* out, int* dflag,
                              cudaStream_t st) {
  size_t sm = simt_fwd_smem(qa.net);
  unsigned grid = (unsigned)((q + kTile - 1) / kTile);
  DISPATCH_F(qa.net.F, set_smem(decode_query_simt_kernel<FF>, sm);
             decode_query_simt_kernel<FF><<<grid, kTile, sm, st>>>(qa, xyz, q, out, dflag));
  count_launch();
}

void launch_convert_f32_f16(const float* src, __half* dst, long long n, cudaStream_t st) {
  convert_f32_f16_kernel<<<148 * 8, 256, 0, st>>>(src, dst, n);
  count_launch();
}
void launch_convert_f16_f32(const __half* src, float* dst, long long n, cudaStream_t st) {
  convert_f16_f32_kernel<<<148 * 8, 256, 0, st>>>(src, dst, n);
  count_launch();
}

void launch_range(const float* base, const int dims[3], const long long s[3], int channels, float* minmax,
                  cudaStream_t st) {
  long long total = (long long)dims[0] * dims[1] * dims[2];
  int blocks = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, 148 * 8));
  range_kernel<<<dim3(blocks, channels), 256, 0, st>>>(base, dims[0], dims[1], dims[2], s[0], s[1], s[2], minmax);
  count_launch();
}

void launch_debug_encode(const NetDesc& net, const float* P, const float* x01, long long q, uint32_t* idx,
                         float* feat, cudaStream_t st) {
  unsigned grid = (unsigned)((q + 127) / 128);
  DISPATCH_F(net.F, debug_encode_kernel<FF><<<grid, 128, 0, st>>>(net, P, x01, q, idx, feat));
  count_launch();
}

void launch_debug_forward_simt(const NetDesc& net, const float* P, const float* x01, long long q, float* y,
                               cudaStream_t st) {
  size_t sm = simt_fwd_smem(net);
  unsigned grid = (unsigned)((q + kTile - 1) / kTile);
  DISPATCH_F(net.F, set_smem(debug_forward_simt_kernel<FF>, sm);
             debug_forward_simt_kernel<FF><<<grid, kTile, sm, st>>>(net, P, x01, q, y));
  count_launch();
}

}  // namespace inr
