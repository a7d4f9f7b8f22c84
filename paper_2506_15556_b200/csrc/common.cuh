// Shared device helpers for the predict-and-verify decoder runtime (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace ps {

constexpr int kPage = 64;          // KV page size in tokens (= attention split)
constexpr int kMaxWindow = 256;    // rows per device pass (longer passes are chunked)
constexpr int kEos = 0;

// Per-pass parameters that kernels read from device memory, so a captured
// decode step (CUDA graph) can be replayed back to back while the position
// advances on the device.
struct PassCtx {
  int n0;       // absolute position of the first row of this pass
  int rows;     // rows in this pass
  int stop;     // decode loop: set once EOS was produced; later steps no-op
  int stop_on_eos;
  int step;     // decode steps executed since the last reset
  int pad[3];
};

__device__ __forceinline__ float bf2f(__nv_bfloat16 v) { return __bfloat162float(v); }

// Programmatic dependent launch (fp32 path): every kernel launched with
// launch_pdl waits for its predecessor's completion (and memory flush) before
// touching any data, then lets its own successor start launching, so the
// launch latency of each step of the chain overlaps the previous kernel.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

template <typename T> __device__ __forceinline__ float ld_as_f32(const T* p);
template <> __device__ __forceinline__ float ld_as_f32<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float ld_as_f32<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// warp_sum of V values at once, transposed: at each xor level a lane keeps
// half of its values and trades the other half with its partner, so the V
// sums cost V - 2 shuffles instead of 5V. Every sum is formed by exactly
// warp_sum's adds (own + partner at offsets 16, 8, 4, 2, 1), hence bitwise
// equal to it. On return lane l holds the sums of values V/32*l .. +V/32-1
// in a[0 .. V/32-1].
template <int V>
__device__ __forceinline__ void warp_sum_transposed(float (&a)[V], int lane) {
  static_assert(V % 32 == 0, "V must be a multiple of 32");
#pragma unroll
  for (int o = 16, m = V; o > 0; o >>= 1, m >>= 1) {
    const bool hi = lane & o;  // keeps the upper half
#pragma unroll
    for (int j = 0; j < m / 2; ++j) {
      const float keep = hi ? a[j + m / 2] : a[j];
      const float send = hi ? a[j] : a[j + m / 2];
      a[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
}

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// (value, index) argmax with ties to the lowest index — `np.argmax`
// semantics, /root/reference/pkg/src/specstream/lm.py:134-136.
__device__ __forceinline__ void argmax_merge(float& v, int& i, float v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

__device__ __forceinline__ void warp_argmax(float& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    float v2 = __shfl_xor_sync(0xffffffffu, v, o);
    int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    argmax_merge(v, i, v2, i2);
  }
}

// Deterministic block sum (fixed tree: warp butterflies then warp 0).
template <int kThreads>
__device__ __forceinline__ float block_sum(float v, float* scratch) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) scratch[w] = v;
  __syncthreads();
  float r = 0.f;
  if (w == 0) {
    r = (l < kThreads / 32) ? scratch[l] : 0.f;
    r = warp_sum(r);
    if (l == 0) scratch[0] = r;
  }
  __syncthreads();
  r = scratch[0];
  __syncthreads();
  return r;
}

}  // namespace ps
