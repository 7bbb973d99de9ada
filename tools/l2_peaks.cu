// l2_peaks.cu — microbenchmarks for the rooflines of the gather / scatter
// kernels (MEASURED_PEAKS.json has HBM copy and GEMM peaks only): random 8-B
// and 16-B loads and random red.global.add.v2/.v4.f32 over a buffer of a given
// size, one uniformly random index per access (a hash of the thread's counter),
// 8 independent accesses per thread per iteration like the encode kernels.
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int VEC>   // VEC floats per access (2 or 4)
__global__ void gather_kernel(const float* __restrict__ buf, uint32_t mask, long long n_iters, float* out) {
  float acc = 0.f;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  for (long long it = 0; it < n_iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint32_t e = mix(t * 8u + c + (uint32_t)it * 0x9E3779B9u) & mask;   // entry index
      if constexpr (VEC == 2) { float2 v = __ldg(reinterpret_cast<const float2*>(buf) + e); acc += v.x + v.y; }
      else { float4 v = __ldg(reinterpret_cast<const float4*>(buf) + e); acc += v.x + v.y + v.z + v.w; }
    }
  }
  if (acc == 12345.f) out[t] = acc;
}

template <int VEC>
__global__ void red_kernel(float* __restrict__ buf, uint32_t mask, long long n_iters) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  for (long long it = 0; it < n_iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      uint32_t e = mix(t * 8u + c + (uint32_t)it * 0x9E3779B9u) & mask;
      if constexpr (VEC == 2) atomicAdd(reinterpret_cast<float2*>(buf) + e, make_float2(1e-9f, 1e-9f));
      else atomicAdd(reinterpret_cast<float4*>(buf) + e, make_float4(1e-9f, 1e-9f, 1e-9f, 1e-9f));
    }
  }
}

// kind: 0 gather 8 B, 1 gather 16 B, 2 red 8 B, 3 red 16 B.  Returns accesses per second.
extern "C" __attribute__((visibility("default"))) double l2_peak(int kind, long long buffer_bytes, long long accesses) {
  const int vec = (kind == 0 || kind == 2) ? 2 : 4;
  const long long entries = buffer_bytes / (4 * vec);
  uint32_t mask = 1;
  while ((long long)mask * 2 <= entries) mask *= 2;
  mask -= 1;
  float* buf;
  cudaMalloc(&buf, buffer_bytes);
  cudaMemset(buf, 0, buffer_bytes);
  float* out;
  cudaMalloc(&out, 4 << 20);
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, blocks = nsm * 8;
  const long long per_iter = (long long)threads * blocks * 8;
  const long long iters = (accesses + per_iter - 1) / per_iter;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {   // first pass warms
    cudaEventRecord(a);
    switch (kind) {
      case 0: gather_kernel<2><<<blocks, threads>>>(buf, mask, iters, out); break;
      case 1: gather_kernel<4><<<blocks, threads>>>(buf, mask, iters, out); break;
      case 2: red_kernel<2><<<blocks, threads>>>(buf, mask, iters); break;
      default: red_kernel<4><<<blocks, threads>>>(buf, mask, iters); break;
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(buf);
  cudaFree(out);
  return (double)(iters * per_iter) / (ms / 1e3);
}
