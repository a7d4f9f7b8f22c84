// Grid-barrier latency on one B200: 148 co-resident CTAs (cooperative launch),
// back-to-back barriers, optionally after each CTA stores `wbytes` to global
// (the partials a GEMM phase publishes before its barrier).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/barrier_probe_bin tools/barrier_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel(unsigned* p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void red_rlx(unsigned* p) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void fence_ar() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int V>
__global__ void __launch_bounds__(192) probe(unsigned* bar, unsigned* flags, float* scratch, int iters, int wfloats) {
  __shared__ volatile int seen;
  const int G = gridDim.x, c = blockIdx.x;
  float* mine = scratch + size_t(c) * wfloats;
  for (int it = 1; it <= iters; ++it) {
    for (int i = threadIdx.x; i < wfloats / 4; i += blockDim.x)
      reinterpret_cast<float4*>(mine)[i] = make_float4(it, i, c, 0);
    __syncthreads();
    if (V == 0) {  // red.release + ld.acquire polling (the megakernel's)
      if (threadIdx.x == 0) {
        red_rel(bar);
        while (ld_acq(bar) < unsigned(G) * it) {
        }
      }
    } else if (V == 1) {  // fence + relaxed red + relaxed polling + fence
      if (threadIdx.x == 0) {
        fence_ar();
        red_rlx(bar);
        while (ld_rlx(bar) < unsigned(G) * it) {
        }
        fence_ar();
      }
    } else if (V == 2) {  // red.release + relaxed polling + one fence
      if (threadIdx.x == 0) {
        red_rel(bar);
        while (ld_rlx(bar) < unsigned(G) * it) {
        }
        fence_ar();
      }
    } else if (V == 3) {  // per-CTA flags, warp 0 polls all of them
      if (threadIdx.x == 0) st_rel(flags + c * 32, it);
      if (threadIdx.x < 32) {
        for (;;) {
          bool ok = true;
          for (int j = threadIdx.x; j < G; j += 32) ok &= ld_acq(flags + j * 32) >= unsigned(it);
          if (__all_sync(0xffffffffu, ok)) break;
        }
      }
    } else if (V == 4) {  // red.release, two pollers in different warps, first one tells the CTA
      if (threadIdx.x == 0) {
        seen = 0;
        red_rel(bar);
      }
      if (threadIdx.x == 0 || threadIdx.x == 64 || threadIdx.x == 128) {
        while (!seen && ld_acq(bar) < unsigned(G) * it) {
        }
        seen = 1;
      }
    } else if (V == 6) {  // arrival counter + generation flag in another line (pollers never touch the counter)
      if (threadIdx.x == 0) {
        unsigned old;
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
        if (old == unsigned(G) * it - 1) st_rel(flags, it);
        else
          while (ld_acq(flags) < unsigned(it)) {
          }
      }
    } else if (V == 5) {  // two loads in flight per poll round
      if (threadIdx.x == 0) {
        red_rel(bar);
        const unsigned t = unsigned(G) * it;
        for (;;) {
          unsigned a = ld_rlx(bar);
          __nanosleep(100);
          unsigned b = ld_rlx(bar);
          if (a >= t || b >= t) break;
        }
        fence_ar();
      }
    }
    __syncthreads();
  }
}

template <int V>
float run(unsigned* bar, unsigned* flags, float* scratch, int iters, int wfloats) {
  cudaMemset(bar, 0, 4);
  cudaMemset(flags, 0, 148 * 128);
  void* args[] = {&bar, &flags, &scratch, &iters, &wfloats};
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchCooperativeKernel((void*)probe<V>, 148, 192, args, 0, 0);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms * 1e3f / iters;
}

int main() {
  unsigned *bar, *flags;
  float* scratch;
  cudaMalloc(&bar, 256);
  cudaMalloc(&flags, 148 * 128);
  cudaMalloc(&scratch, size_t(148) * 16384 * 4);
  const char* names[] = {"red.release + ld.acquire poll", "fence + red.relaxed + relaxed poll + fence",
                         "red.release + relaxed poll + fence", "per-CTA flags, warp polls all",
                         "red.release, 3 pollers", "2 relaxed loads in flight + fence",
                         "atom.acq_rel + generation flag"};
  for (int wf : {0, 1024, 4096, 16384}) {
    for (int rep = 0; rep < 2; ++rep) {
      float t[7];
      t[0] = run<0>(bar, flags, scratch, 4000, wf);
      t[1] = run<1>(bar, flags, scratch, 4000, wf);
      t[2] = run<2>(bar, flags, scratch, 4000, wf);
      t[3] = run<3>(bar, flags, scratch, 4000, wf);
      t[4] = run<4>(bar, flags, scratch, 4000, wf);
      t[5] = run<5>(bar, flags, scratch, 4000, wf);
      t[6] = run<6>(bar, flags, scratch, 4000, wf);
      if (rep)
        for (int v = 0; v < 7; ++v) printf("stores %6d B/CTA  %-45s %.3f us/barrier\n", wf * 4, names[v], t[v]);
    }
  }
  return 0;
}
