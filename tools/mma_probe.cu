// Legacy tensor-core path on the B200: latency and throughput of
// mma.sync.m16n8k16 (bf16 in, fp32 accumulate) — the instruction the
// megakernel's attention units run on. One CTA, `warps` warps; each warp runs
// `chains` independent accumulator chains for `iters` steps.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_probe_bin tools/mma_probe.cu
//   tools/mma_probe_bin
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int CH>
__global__ void probe(int iters, long long* cycles, float* sink) {
  float d[CH][4];
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = 0.f;
  uint32_t a0 = threadIdx.x * 0x00010001u, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 ^ 5, b1 = a0 ^ 7;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int CH>
void run(int warps, int iters) {
  long long* dc;
  float* ds;
  cudaMalloc(&dc, sizeof(long long));
  cudaMalloc(&ds, 1024 * sizeof(float));
  probe<CH><<<1, 32 * warps>>>(iters, dc, ds);  // warm
  probe<CH><<<1, 32 * warps>>>(iters, dc, ds);
  long long c = 0;
  cudaMemcpy(&c, dc, sizeof(c), cudaMemcpyDeviceToHost);
  const double per_warp = double(c) / (double(iters) * CH);
  std::printf("warps %2d chains %d: %.2f cycles per mma per warp, SM issue %.2f cycles per mma\n", warps, CH, per_warp,
              per_warp / warps);
  cudaFree(dc);
  cudaFree(ds);
}

int main() {
  const int iters = 4096;
  run<1>(1, iters);   // latency of a dependent chain
  run<8>(1, iters);   // one warp, 8 independent chains
  run<8>(4, iters);   // one warp per SMSP
  run<8>(8, iters);
  run<8>(16, iters);
  return 0;
}
