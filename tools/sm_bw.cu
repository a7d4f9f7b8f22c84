// Streaming bandwidth from HBM into shared memory when only k SMs pull
// (1D cp.async.bulk, 16 KB chunks, a ring of `stages` buffers per CTA).
// Answers: how many SMs does a weight-streaming phase need to saturate HBM?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sm_bw tools/sm_bw.cu && /tmp/sm_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void stream_kernel(const char* src, size_t bytes_per_cta, int stages, int chunk, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar[16];
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const char* base = src + size_t(blockIdx.x) * bytes_per_cta;
  const int n = int(bytes_per_cta / chunk);
  auto issue = [&](int i) {
    const int s = i % stages;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[s])), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     s32(sm + size_t(s) * chunk)),
                 "l"(base + size_t(i) * chunk), "r"(chunk), "r"(s32(&bar[s]))
                 : "memory");
  };
  for (int i = 0; i < stages && i < n; ++i) issue(i);
  unsigned acc = 0;
  for (int i = 0; i < n; ++i) {
    const int s = i % stages;
    const uint32_t ph = (i / stages) & 1;
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok)
                   : "r"(s32(&bar[s])), "r"(ph)
                   : "memory");
    acc += sm[size_t(s) * chunk];
    if (i + stages < n) issue(i + stages);
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

int main() {
  const size_t total = size_t(4) << 30;  // 4 GB source, larger than L2
  char* src;
  unsigned long long* sink;
  cudaMalloc(&src, total);
  cudaMalloc(&sink, 8);
  cudaMemset(src, 1, total);
  const int chunk = 16384, stages = 12;
  const int smem = stages * chunk;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int ks[] = {1, 2, 4, 8, 16, 24, 32, 48, 64, 74, 96, 128, 148};
  for (int k : ks) {
    // each CTA streams 2048 chunks (32 MB) or the source split k ways, whichever is smaller
    size_t per = total / k;
    if (per > size_t(2048) * chunk) per = size_t(2048) * chunk;
    per -= per % chunk;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      stream_kernel<<<k, 32, smem>>>(src, per, stages, chunk, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const double gbs = double(per) * k / (best * 1e-3) / 1e9;
    std::printf("sms=%3d  total %8.1f GB/s  per-SM %7.1f GB/s\n", k, gbs, gbs / k);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
