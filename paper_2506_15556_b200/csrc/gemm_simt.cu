// fp32 SIMT GEMV/GEMM for the bit-exact fp32 mode (configs c1/c2).
//
// One warp owns 2 output rows; lane l streams the float4 chunks c ≡ l (mod
// 32) of its K-split in order (coalesced 128-bit weight loads), then an xor
// butterfly sums the lanes. The arithmetic for an output (t, n) is therefore
// fixed by (n, K-split) alone: a row scored in a 72-row verify pass is
// bit-identical to the same row scored by a 1-row decode pass.
#include "common.cuh"
#include "f32_math.cuh"
#include "kernels.h"

namespace ps {

template <int TT>
__global__ void __launch_bounds__(256) gemm_f32_kernel(const PassCtx* __restrict__ ctx, const float* __restrict__ X,
                                                       int ldx, const float* __restrict__ W, float* __restrict__ part,
                                                       int N, int K, int ksplit) {
  pdl_enter();
  extern __shared__ float4 xs4[];
  if (ctx->stop) return;
  const int rows = ctx->rows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * 16 + warp * 2;
  const int s = blockIdx.y;
  const int kbeg = s * ksplit;
  const int nvec = ksplit >> 2;
  const float4* w0 = reinterpret_cast<const float4*>(W + size_t(n0) * K + kbeg);
  const float4* w1 = reinterpret_cast<const float4*>(W + size_t(n0 + 1) * K + kbeg);
  // blockIdx.z takes every gridDim.z-th chunk of TT tokens (more CTAs for
  // narrow N; the per-output arithmetic does not depend on the chunking)
  for (int tt = blockIdx.z * TT; tt < rows; tt += TT * gridDim.z) {
    const int nt = min(TT, rows - tt);
    __syncthreads();
    for (int e = threadIdx.x; e < TT * nvec; e += 256) {
      const int t = e / nvec, c = e % nvec;
      xs4[e] = t < nt ? reinterpret_cast<const float4*>(X + size_t(tt + t) * ldx + kbeg)[c]
                      : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    float a0[TT], a1[TT];
#pragma unroll
    for (int t = 0; t < TT; ++t) a0[t] = a1[t] = 0.f;
    for (int c = lane; c < nvec; c += 32) {
      const float4 u = __ldg(w0 + c), v = __ldg(w1 + c);
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        const float4 x = xs4[t * nvec + c];
        a0[t] = fmaf(x.x, u.x, a0[t]); a0[t] = fmaf(x.y, u.y, a0[t]);
        a0[t] = fmaf(x.z, u.z, a0[t]); a0[t] = fmaf(x.w, u.w, a0[t]);
        a1[t] = fmaf(x.x, v.x, a1[t]); a1[t] = fmaf(x.y, v.y, a1[t]);
        a1[t] = fmaf(x.z, v.z, a1[t]); a1[t] = fmaf(x.w, v.w, a1[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < TT; ++t) {
      a0[t] = warp_sum(a0[t]);
      a1[t] = warp_sum(a1[t]);
    }
#pragma unroll
    for (int t = 0; t < TT; ++t) {
      if (lane == t && t < nt) {
        float* o = part + (size_t(s) * kMaxWindow + tt + t) * N + n0;
        o[0] = a0[t];
        o[1] = a1[t];
      }
    }
  }
}

void launch_gemm_f32(const PassCtx* ctx, int max_rows, const float* X, int ldx, const float* W,
                     float* part, int N, int K, int splits, cudaStream_t st) {
  const int ksplit = K / splits;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_f32_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(gemm_f32_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  dim3 grid(N / 16, splits, max_rows <= 1 ? 1 : (max_rows + 15) / 16);
  if (max_rows <= 1)
    launch_pdl(gemm_f32_kernel<1>, dim3(grid), dim3(256), size_t(ksplit) * 4, st, ctx, X, ldx, W, part, N, K, ksplit);
  else
    launch_pdl(gemm_f32_kernel<16>, dim3(grid), dim3(256), size_t(ksplit) * 16 * 4, st, ctx, X, ldx, W, part, N, K, ksplit);
}

// LM head: 64 vocab ids per CTA (8 warps x 2 rows x 4 passes), fused
// bias + argmax; logits are written only when logits_out != nullptr (parity).
template <int TT>
__global__ void __launch_bounds__(256) lmhead_f32_kernel(PassCtx* ctx, const float* __restrict__ hn_cache,
                                                         const float* __restrict__ W, const float* __restrict__ bias,
                                                         int v_begin, int v_count, int H, float* __restrict__ am_val,
                                                         int* __restrict__ am_idx, float* __restrict__ logits_out,
                                                         int ld_logits) {
  pdl_enter();
  extern __shared__ float4 xs4[];
  __shared__ float bv[8][TT];
  __shared__ int bi[8][TT];
  if (ctx->stop) return;
  const int rows = ctx->rows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nvec = H >> 2;
  // blockIdx.x = tile * Z + z: the Z token chunks of a vocab tile are
  // neighbouring CTAs, so the tile's weights are read from DRAM once and
  // from L2 by the others
  const int ntiles = (v_count + kLmTileF32 - 1) / kLmTileF32;
  const int Z = int(gridDim.x) / ntiles, tile = blockIdx.x / Z, z = blockIdx.x % Z;
  const float* X = hn_cache + size_t(ctx->n0) * H;
  for (int tt = z * TT; tt < rows; tt += TT * Z) {
    const int nt = min(TT, rows - tt);
    __syncthreads();
    for (int e = threadIdx.x; e < TT * nvec; e += 256) {
      const int t = e / nvec, c = e % nvec;
      xs4[e] = t < nt ? reinterpret_cast<const float4*>(X + size_t(tt + t) * H)[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    float best = -INFINITY;
    int besti = 0x7fffffff;
    for (int it = 0; it < kLmTileF32 / 16; ++it) {
      const int r0 = tile * kLmTileF32 + it * 16 + warp * 2;  // local vocab row
      if (r0 >= v_count) break;
      const bool has1 = r0 + 1 < v_count;
      const float4* w0 = reinterpret_cast<const float4*>(W + size_t(r0) * H);  // shard-local rows
      const float4* w1 = reinterpret_cast<const float4*>(W + size_t(has1 ? r0 + 1 : r0) * H);
      float a0[TT], a1[TT];
#pragma unroll
      for (int t = 0; t < TT; ++t) a0[t] = a1[t] = 0.f;
      for (int c = lane; c < nvec; c += 32) {
        const float4 u = __ldg(w0 + c), v = __ldg(w1 + c);
#pragma unroll
        for (int t = 0; t < TT; ++t) {
          const float4 x = xs4[t * nvec + c];
          a0[t] = fmaf(x.x, u.x, a0[t]); a0[t] = fmaf(x.y, u.y, a0[t]);
          a0[t] = fmaf(x.z, u.z, a0[t]); a0[t] = fmaf(x.w, u.w, a0[t]);
          a1[t] = fmaf(x.x, v.x, a1[t]); a1[t] = fmaf(x.y, v.y, a1[t]);
          a1[t] = fmaf(x.z, v.z, a1[t]); a1[t] = fmaf(x.w, v.w, a1[t]);
        }
      }
      const float b0 = bias[v_begin + r0], b1 = has1 ? bias[v_begin + r0 + 1] : 0.f;
#pragma unroll
      for (int t = 0; t < TT; ++t) {
        const float l0 = warp_sum(a0[t]) + b0;
        const float l1 = warp_sum(a1[t]) + b1;
        if (lane == t && t < nt) {
          argmax_merge(best, besti, l0, v_begin + r0);
          if (has1) argmax_merge(best, besti, l1, v_begin + r0 + 1);
          if (logits_out) {
            float* lo = logits_out + size_t(tt + t) * ld_logits + r0;
            lo[0] = l0;
            if (has1) lo[1] = l1;
          }
        }
      }
    }
    if (lane < TT) { bv[warp][lane] = best; bi[warp][lane] = besti; }
    __syncthreads();
    if (threadIdx.x < nt) {
      float v = bv[0][threadIdx.x];
      int i = bi[0][threadIdx.x];
      for (int w = 1; w < 8; ++w) argmax_merge(v, i, bv[w][threadIdx.x], bi[w][threadIdx.x]);
      am_val[size_t(tile) * kMaxWindow + tt + threadIdx.x] = v;
      am_idx[size_t(tile) * kMaxWindow + tt + threadIdx.x] = i;
    }
  }
}

void launch_lmhead_f32(const PassCtx* ctx, int max_rows, const float* hn_cache, int pos_offset,
                       const float* W, const float* bias, int v_begin, int v_count, int hidden,
                       float* am_val, int* am_idx, float* logits_out, int ld_logits, cudaStream_t st) {
  (void)pos_offset;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(lmhead_f32_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(lmhead_f32_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const int tiles = (v_count + kLmTileF32 - 1) / kLmTileF32;
  PassCtx* c = const_cast<PassCtx*>(ctx);
  if (max_rows <= 1)
    launch_pdl(lmhead_f32_kernel<1>, dim3(tiles), dim3(256), size_t(hidden) * 4, st, c, hn_cache, W, bias, v_begin, v_count, hidden,
                                                                 am_val, am_idx, logits_out, ld_logits);
  else {
    const int Z = (max_rows + 15) / 16;  // token chunks per vocab tile (gridDim.x = tiles * Z)
    launch_pdl(lmhead_f32_kernel<16>, dim3(tiles * Z), dim3(256), size_t(hidden) * 16 * 4, st, 
        c, hn_cache, W, bias, v_begin, v_count, hidden, am_val, am_idx, logits_out, ld_logits);
  }
}

}  // namespace ps
