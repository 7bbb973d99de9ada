// tc_common.cuh — tcgen05 / TMEM / mbarrier helpers and the canonical
// SWIZZLE_NONE shared-memory operand layout used by the tensor-core kernels.
//
// Canonical layout: 8 rows x 16 B core matrices; element (row r, col c) of a
// tile with C columns sits at byte (r%8)*16 + (r/8)*SBO + (c/8)*128 + (c%8)*2,
// SBO = (C/8)*128.  Read with (row = M/N dim, col = K dim) it is the K-major
// layout (LBO = 128, SBO); read with (row = K dim, col = M/N dim) it is the
// MN-major layout (SBO' = 128, LBO' = SBO) — so one tile serves every GEMM
// that needs it, without a transposed copy.
#pragma once
#include "common.cuh"

namespace inr {
namespace tc {

constexpr int kThreads = 128;
constexpr int kTileM = 128;
// grid decode tiles are 8 x 4 x 4 bricks of lattice points (thread t <-> (t & 7, (t >> 3) & 3, t >> 5))
constexpr int kBrickX = 8, kBrickY = 4, kBrickZ = 4;
constexpr int kStageFloats = 1536;   // smem floats for the staged coarse-level vertices of one super-brick
// grid decode: a CTA stages the coarse levels once per super-brick of kSupX x kSupY x kSupZ bricks
// (measured: 2 x 2 x 2 beats 1 x 2 x 2, 2 x 2 x 1, 4 x 2 x 2 and 4 x 4 x 2)
constexpr int kSupX = 2, kSupY = 2, kSupZ = 2, kSubs = kSupX * kSupY * kSupZ;
constexpr int kFwdThreads = 256;     // forward-only kernel: thread t <-> row t % 128, column / level half t / 128

struct Layout {
  uint32_t w[kMaxLayers];        // fp16 W_k tile [64 x in_k] (k < H)
  uint32_t w_sbo[kMaxLayers];
  uint32_t h[kMaxLayers];        // fp16 h_k tile [128 x (in_k + ones)] (k < H), h_0 = features
  uint32_t h_sbo[kMaxLayers];
  uint32_t dz, dz_sbo;           // fp16 dz tile [128 x 64]
  uint32_t dz2;                  // second dz tile (backward layers alternate)
  uint32_t bias;                 // fp32 [H][64]
  uint32_t wout;                 // fp32 W_H[D][64], then b_H[D]
  uint32_t red;                  // dW_H[D][64], db_H[D] partials (fp32 or int64 fixed point)
  uint32_t ypart;                // fp32 [D][2][128] output-layer partial sums (fit)
  uint32_t mbar;                 // 8 B: MMA completion
  uint32_t mbar_img;             // 8 B: weight-image bulk copy (fit)
  uint32_t mbar_feat[2];         // 8 B each: feature-tile bulk copies (fit, double buffered)
  uint32_t h0b;                  // second h_0 buffer (fit)
  uint32_t img_bytes;            // [0, img_bytes): weight tiles + biases + output layer (the weight image)
  uint32_t feat_tile_bytes;      // one 128-sample h_0 tile image
  uint32_t tslot;                // 4 B: TMEM base address
  uint32_t stage;                // forward only: per-brick staging of coarse-level vertices (kStageFloats fp32)
  uint32_t bytes;                // dynamic smem requested
  uint32_t col_dw[kMaxLayers];   // TMEM column of the dW_k accumulator
  uint32_t ncols;                // TMEM columns allocated (power of 2)
  int ones;                      // 8 if biases (ones group appended), else 0
  uint32_t stbox;                // forward only: per staged level int[8] = lo[3], n[3] of the brick's vertex box
  int ctas_per_sm;
};

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version 1 (sm_100); base offset 0; SWIZZLE_NONE
  return d;
}

// kind::f16 instruction descriptor: fp16 A/B, fp32 D.
__host__ __device__ constexpr uint32_t make_idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(mbar)
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(mbar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(mbar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// TMA bulk copy global -> shared, completion (bytes) reported on an mbarrier.
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst_smem, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   dst_smem),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

// 16 consecutive fp32 columns of this thread's TMEM lane.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Row r of a canonical tile: write 8 consecutive columns [8j, 8j+8) as fp16.
__device__ __forceinline__ void st_row8(uint8_t* tile, uint32_t sbo, int r, int j, const float* v) {
  __half2 h0 = __floats2half2_rn(v[0], v[1]), h1 = __floats2half2_rn(v[2], v[3]);
  __half2 h2 = __floats2half2_rn(v[4], v[5]), h3 = __floats2half2_rn(v[6], v[7]);
  uint4 u;
  u.x = *reinterpret_cast<uint32_t*>(&h0);
  u.y = *reinterpret_cast<uint32_t*>(&h1);
  u.z = *reinterpret_cast<uint32_t*>(&h2);
  u.w = *reinterpret_cast<uint32_t*>(&h3);
  *reinterpret_cast<uint4*>(tile + (r & 7) * 16 + (r >> 3) * sbo + j * 128) = u;
}

__device__ __forceinline__ uint32_t tile_off(uint32_t sbo, int r, int c) {
  return (r & 7) * 16 + (r >> 3) * sbo + (c >> 3) * 128 + (c & 7) * 2;
}

// Sum 64 per-lane values over the warp; lane l ends with the column sums of
// columns c0 = 32 b4 + 16 b3 + 8 b2 + 4 b1 + 2 b0 and c0 + 1 (b = lane bits).
__device__ __forceinline__ void warp_transpose_reduce64(float* v, int lane) {
#pragma unroll
  for (int half = 32, off = 16; off >= 1; half >>= 1, off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int j = 0; j < half; ++j) {
      float keep = up ? v[j + half] : v[j];
      float send = up ? v[j] : v[j + half];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
}

}  // namespace tc

// Issue the K loop of one GEMM (single thread).  a/b: start addresses; the
// per-K-step (16 elements) advance of each operand is given explicitly.
__device__ __forceinline__ void gemm(uint32_t tmem_d, uint32_t a, uint32_t a_lbo, uint32_t a_sbo, uint32_t a_step,
                                     uint32_t b, uint32_t b_lbo, uint32_t b_sbo, uint32_t b_step, int ksteps,
                                     uint32_t idesc, bool accum_first) {
  for (int k = 0; k < ksteps; ++k) {
    uint64_t ad = tc::make_desc(a + k * a_step, a_lbo, a_sbo);
    uint64_t bd = tc::make_desc(b + k * b_step, b_lbo, b_sbo);
    tc::mma_f16(tmem_d, ad, bd, idesc, (k > 0 || accum_first) ? 1u : 0u);
  }
}

}  // namespace inr
