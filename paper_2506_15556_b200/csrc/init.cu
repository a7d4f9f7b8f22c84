// Counter-based weight generator: every element is a pure function of
// (seed, tensor id, index), so 16 GB of random-init weights appear in HBM in
// milliseconds and oracle/weights.py reproduces the identical bits on the CPU.
//
//   h = mix(key(seed, tid) + (i+1)*G);  u = h >> 41;  w = fp32(u - 2^22) * scale
#include "common.cuh"
#include "kernels.h"

namespace ps {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t weight_key(uint64_t seed, uint32_t tid) {
  return mix64(seed * 0x9E3779B97F4A7C15ull + uint64_t(tid) * 0xD1B54A32D192ED03ull +
               0x632BE59BD9B4E019ull);
}

float weight_scale(double stddev) {
  return float(stddev * 1.7320508075688772 / double(1 << 22));
}

template <typename T>
__global__ void init_uniform_kernel(T* __restrict__ out, uint64_t count, uint64_t first, uint64_t key,
                                    float scale) {
  uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (; i < count; i += stride) {
    uint64_t h = mix64(key + (first + i + 1) * 0x9E3779B97F4A7C15ull);
    int32_t u = int32_t(h >> 41) - (1 << 22);
    out[i] = from_f32<T>(__fmul_rn(float(u), scale));
  }
}

template <typename T>
void launch_init_uniform(T* out, uint64_t count, uint64_t first, uint64_t seed, uint32_t tid, double stddev,
                         cudaStream_t st) {
  if (count == 0) return;
  const int threads = 256;
  uint64_t blocks = (count + threads - 1) / threads;
  if (blocks > 148ull * 64) blocks = 148ull * 64;
  init_uniform_kernel<T><<<unsigned(blocks), threads, 0, st>>>(out, count, first, weight_key(seed, tid),
                                                               weight_scale(stddev));
}

// Same values, written to permuted destination rows (row r of the tensor ->
// perm_row(r)); the fused bf16 matrices store partner rows next to each other
// so the GEMM epilogue exchanges them with one shuffle (see kernels.h).
template <typename T>
__global__ void init_rows_permuted_kernel(T* __restrict__ out, uint64_t rows, uint64_t cols, uint64_t key,
                                          float scale, RowPerm perm) {
  const uint64_t count = rows * cols;
  uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (; i < count; i += stride) {
    const uint64_t r = i / cols, c = i % cols;
    uint64_t h = mix64(key + (i + 1) * 0x9E3779B97F4A7C15ull);
    int32_t u = int32_t(h >> 41) - (1 << 22);
    out[uint64_t(perm.dst(int(r))) * cols + c] = from_f32<T>(__fmul_rn(float(u), scale));
  }
}

template <typename T>
void launch_init_rows_permuted(T* out, uint64_t rows, uint64_t cols, RowPerm perm, uint64_t seed, uint32_t tid,
                               double stddev, cudaStream_t st) {
  const uint64_t count = rows * cols;
  if (count == 0) return;
  uint64_t blocks = (count + 255) / 256;
  if (blocks > 148ull * 64) blocks = 148ull * 64;
  init_rows_permuted_kernel<T><<<unsigned(blocks), 256, 0, st>>>(out, rows, cols, weight_key(seed, tid),
                                                                weight_scale(stddev), perm);
}

template void launch_init_rows_permuted<__nv_bfloat16>(__nv_bfloat16*, uint64_t, uint64_t, RowPerm, uint64_t,
                                                       uint32_t, double, cudaStream_t);
template void launch_init_rows_permuted<float>(float*, uint64_t, uint64_t, RowPerm, uint64_t, uint32_t, double,
                                               cudaStream_t);

template void launch_init_uniform<float>(float*, uint64_t, uint64_t, uint64_t, uint32_t, double, cudaStream_t);
template void launch_init_uniform<__nv_bfloat16>(__nv_bfloat16*, uint64_t, uint64_t, uint64_t, uint32_t, double,
                                                 cudaStream_t);

}  // namespace ps
