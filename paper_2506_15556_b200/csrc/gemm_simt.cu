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

// L2 prefetch of `nrows` weight rows (`floats` each, `ld` apart) by one warp,
// one request per 128-byte line. Issued BEFORE the programmatic-dependency
// wait: weights never depend on the previous kernel of the chain, so their
// DRAM latency overlaps its tail. (Register loads cannot be placed there —
// ptxas hoists griddepcontrol.wait above every LDG — but prefetches and
// cp.async stay where they are written.)
__device__ __forceinline__ void prefetch_rows_l2(const float* base, size_t ld, int nrows, int floats, int lane) {
  for (int r = 0; r < nrows; ++r)
    for (int off = lane * 32; off < floats; off += 32 * 32)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(base + r * ld + off));
}

// x rows [tt, tt + TT) of this K-split -> shared memory, every 16-byte copy in
// flight at once (cp.async; rows past nt are zero-filled). One round trip
// instead of one per loop iteration.
__device__ __forceinline__ void stage_x_async(float4* xs4, const float* X, size_t ldx, int kbeg, int tt, int nt, int TT,
                                              int nvec) {
  for (int e = threadIdx.x; e < TT * nvec; e += blockDim.x) {
    const int t = e / nvec, c = e % nvec;
    const float* src = X + size_t(tt + min(t, nt - 1)) * ldx + kbeg + 4 * c;
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(xs4 + e));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(t < nt ? 16 : 0) : "memory");
  }
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// Decode GEMV (1 row). The warp's two weight rows are prefetched into L2
// before the programmatic-dependency wait; after it, each lane requests all of
// its chunks (up to kPre per row) at once, together with the staged x. The
// FMA order (chunks c = lane, lane + 32, ... ascending, then warp_sum) is the
// wide kernels' (batch invariance).
constexpr int kGemvPre = 8;
__global__ void __launch_bounds__(256) gemm_f32_gemv_kernel(const PassCtx* __restrict__ ctx, const float* __restrict__ X,
                                                            int ldx, const float* __restrict__ W,
                                                            float* __restrict__ part, int N, int K, int ksplit) {
  extern __shared__ float4 xs4[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * 16 + warp * 2;
  const int s = blockIdx.y;
  const int kbeg = s * ksplit;
  const int nvec = ksplit >> 2;
  const float4* w0 = reinterpret_cast<const float4*>(W + size_t(n0) * K + kbeg);
  const float4* w1 = reinterpret_cast<const float4*>(W + size_t(n0 + 1) * K + kbeg);
  prefetch_rows_l2(W + size_t(n0) * K + kbeg, K, 2, ksplit, lane);
  pdl_enter();
  if (ctx->stop || ctx->rows < 1) return;
  float4 u[kGemvPre], v[kGemvPre];
#pragma unroll
  for (int i = 0; i < kGemvPre; ++i) {
    const int c = lane + 32 * i;
    if (c < nvec) {
      u[i] = __ldg(w0 + c);
      v[i] = __ldg(w1 + c);
    }
  }
  for (int e = threadIdx.x; e < nvec; e += 256) xs4[e] = reinterpret_cast<const float4*>(X + kbeg)[e];
  __syncthreads();
  float a0 = 0.f, a1 = 0.f;
#pragma unroll
  for (int i = 0; i < kGemvPre; ++i) {
    const int c = lane + 32 * i;
    if (c < nvec) {
      const float4 x = xs4[c];
      a0 = fmaf(x.x, u[i].x, a0); a0 = fmaf(x.y, u[i].y, a0);
      a0 = fmaf(x.z, u[i].z, a0); a0 = fmaf(x.w, u[i].w, a0);
      a1 = fmaf(x.x, v[i].x, a1); a1 = fmaf(x.y, v[i].y, a1);
      a1 = fmaf(x.z, v[i].z, a1); a1 = fmaf(x.w, v[i].w, a1);
    }
  }
  for (int c = lane + 32 * kGemvPre; c < nvec; c += 32) {  // K-splits longer than 32 * kPre chunks
    const float4 uu = __ldg(w0 + c), vv = __ldg(w1 + c), x = xs4[c];
    a0 = fmaf(x.x, uu.x, a0); a0 = fmaf(x.y, uu.y, a0);
    a0 = fmaf(x.z, uu.z, a0); a0 = fmaf(x.w, uu.w, a0);
    a1 = fmaf(x.x, vv.x, a1); a1 = fmaf(x.y, vv.y, a1);
    a1 = fmaf(x.z, vv.z, a1); a1 = fmaf(x.w, vv.w, a1);
  }
  a0 = warp_sum(a0);
  a1 = warp_sum(a1);
  if (lane == 0) {
    float* o = part + size_t(s) * kMaxWindow * N + n0;
    o[0] = a0;
    o[1] = a1;
  }
}

// Lane-slice partials of R weight rows x TT staged tokens over one K-split:
// lane l accumulates the float4 chunks c ≡ l (mod 32) in order (the decode
// GEMV's order), with the next chunk's weights in flight.
template <int TT, int R>
__device__ __forceinline__ void rows_x_tokens(float (&a)[R * TT], const float4* const (&w)[R], const float4* xs4,
                                              int nvec, int lane, const float4 (&w_first)[R]) {
#pragma unroll
  for (int v = 0; v < R * TT; ++v) a[v] = 0.f;
  float4 wc[R];
#pragma unroll
  for (int i = 0; i < R; ++i) wc[i] = w_first[i];
  for (int c = lane; c < nvec; c += 32) {
    float4 wn[R];
    if (c + 32 < nvec) {
#pragma unroll
      for (int i = 0; i < R; ++i) wn[i] = __ldg(w[i] + c + 32);
    }
#pragma unroll
    for (int t = 0; t < TT; ++t) {
      const float4 x = xs4[t * nvec + c];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        float& d = a[i * TT + t];
        d = fmaf(x.x, wc[i].x, d); d = fmaf(x.y, wc[i].y, d);
        d = fmaf(x.z, wc[i].z, d); d = fmaf(x.w, wc[i].w, d);
      }
    }
#pragma unroll
    for (int i = 0; i < R; ++i) wc[i] = wn[i];
  }
}

// Wide passes: a warp owns R output rows x TT tokens (R*TT = 64 lane-slice
// partials per lane), so each staged x float4 feeds 4R FMAs and each weight
// float4 4*TT; the next chunk's weights are in flight while the current one
// is consumed. Lane l still accumulates exactly the chunks c ≡ l (mod 32) of
// the K-split in order, and the 32 lane partials of every output are summed
// by a transposed butterfly whose adds are warp_sum's (same pairs, same
// order), so every output is bitwise the decode GEMV's.
template <int TT, int R>
__global__ void __launch_bounds__(256, 2) gemm_f32_wide_kernel(const PassCtx* __restrict__ ctx,
                                                               const float* __restrict__ X, int ldx,
                                                               const float* __restrict__ W, float* __restrict__ part,
                                                               int N, int K, int ksplit) {
  static_assert(R * TT == 64, "the transposed butterfly leaves 2 of the 64 sums per lane");
  extern __shared__ float4 xs4[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = blockIdx.x * (8 * R) + warp * R;
  const int s = blockIdx.y;
  const int kbeg = s * ksplit;
  const int nvec = ksplit >> 2;
  const float4* w[R];
#pragma unroll
  for (int i = 0; i < R; ++i) w[i] = reinterpret_cast<const float4*>(W + size_t(min(nb + i, N - 1)) * K + kbeg);
  // the warp's weight rows do not depend on the previous kernel: into L2
  // before the programmatic-dependency wait
  prefetch_rows_l2(W + size_t(min(nb, N - 1)) * K + kbeg, K, min(R, N - nb), ksplit, lane);
  pdl_enter();
  if (ctx->stop) return;
  float4 wf[R];
  if (lane < nvec) {
#pragma unroll
    for (int i = 0; i < R; ++i) wf[i] = __ldg(w[i] + lane);
  }
  const int rows = ctx->rows;
  for (int tt = blockIdx.z * TT; tt < rows; tt += TT * gridDim.z) {
    const int nt = min(TT, rows - tt);
    __syncthreads();
    stage_x_async(xs4, X, ldx, kbeg, tt, nt, TT, nvec);
    __syncthreads();
    float a[R * TT];
    rows_x_tokens<TT, R>(a, w, xs4, nvec, lane, wf);
    warp_sum_transposed<R * TT>(a, lane);
    // lane l now holds the sums of values 2l and 2l + 1 (value = i * TT + t)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int v = 2 * lane + j, i = v / TT, t = v % TT;
      if (t < nt && nb + i < N) part[(size_t(s) * kMaxWindow + tt + t) * N + nb + i] = a[j];
    }
  }
}

void launch_gemm_f32(const PassCtx* ctx, int max_rows, const float* X, int ldx, const float* W,
                     float* part, int N, int K, int splits, cudaStream_t st) {
  const int ksplit = K / splits;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_f32_wide_kernel<16, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(gemm_f32_gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  if (max_rows <= 1) {
    launch_pdl(gemm_f32_gemv_kernel, dim3(N / 16, splits, 1), dim3(256), size_t(ksplit) * 4, st, ctx, X, ldx, W, part,
               N, K, ksplit);
  } else {
    const dim3 grid((N + 31) / 32, splits, (max_rows + 15) / 16);
    launch_pdl(gemm_f32_wide_kernel<16, 4>, grid, dim3(256), size_t(ksplit) * 16 * 4, st, ctx, X, ldx, W, part, N, K,
               ksplit);
  }
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

// Wide passes: 64 vocab ids per CTA as 2 passes of 8 warps x 4 rows, each
// warp's 4 rows x 16 tokens summed with the transposed butterfly (bitwise the
// decode kernel's warp_sum), then bias and the (max, lowest id) merge.
template <int TT, int R>
__global__ void __launch_bounds__(256, 2) lmhead_f32_wide_kernel(PassCtx* ctx, const float* __restrict__ hn_cache,
                                                                 const float* __restrict__ W,
                                                                 const float* __restrict__ bias, int v_begin,
                                                                 int v_count, int H, float* __restrict__ am_val,
                                                                 int* __restrict__ am_idx,
                                                                 float* __restrict__ logits_out, int ld_logits) {
  static_assert(R * TT == 64 && TT == 16, "lane l ends with tokens 2(l & 7), +1 of row l >> 3");
  extern __shared__ float4 xs4[];
  __shared__ float bv[8][TT];
  __shared__ int bi[8][TT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nvec = H >> 2;
  const int ntiles = (v_count + kLmTileF32 - 1) / kLmTileF32;
  const int Z = int(gridDim.x) / ntiles, tile = blockIdx.x / Z, z = blockIdx.x % Z;
  pdl_enter();
  if (ctx->stop) return;
  const int rows = ctx->rows;
  const float* X = hn_cache + size_t(ctx->n0) * H;
  const int i_mine = lane >> 3, t_mine = 2 * (lane & 7);
  for (int tt = z * TT; tt < rows; tt += TT * Z) {
    const int nt = min(TT, rows - tt);
    __syncthreads();
    stage_x_async(xs4, X, H, 0, tt, nt, TT, nvec);
    __syncthreads();
    float best[2] = {-INFINITY, -INFINITY};
    int besti[2] = {0x7fffffff, 0x7fffffff};
    for (int it = 0; it < kLmTileF32 / (8 * R); ++it) {
      const int r0 = tile * kLmTileF32 + it * 8 * R + warp * R;  // local vocab row
      if (r0 >= v_count) break;
      const float4* w[R];
#pragma unroll
      for (int i = 0; i < R; ++i) w[i] = reinterpret_cast<const float4*>(W + size_t(min(r0 + i, v_count - 1)) * H);
      float4 wf[R];
      if (lane < nvec) {
#pragma unroll
        for (int i = 0; i < R; ++i) wf[i] = __ldg(w[i] + lane);
      }
      float a[R * TT];
      rows_x_tokens<TT, R>(a, w, xs4, nvec, lane, wf);
      warp_sum_transposed<R * TT>(a, lane);
      const int r = r0 + i_mine;
      if (r < v_count) {
        const float b = bias[v_begin + r];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int t = t_mine + j;
          const float l = a[j] + b;
          if (t < nt) {
            argmax_merge(best[j], besti[j], l, v_begin + r);
            if (logits_out) logits_out[size_t(tt + t) * ld_logits + r] = l;
          }
        }
      }
    }
    // the 4 lanes holding the same tokens (lane & 7 equal) merge; lanes 0-7 publish
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
      for (int o = 8; o <= 16; o <<= 1) {
        const float v2 = __shfl_xor_sync(0xffffffffu, best[j], o);
        const int i2 = __shfl_xor_sync(0xffffffffu, besti[j], o);
        argmax_merge(best[j], besti[j], v2, i2);
      }
      if (lane < 8) {
        bv[warp][t_mine + j] = best[j];
        bi[warp][t_mine + j] = besti[j];
      }
    }
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
    cudaFuncSetAttribute(lmhead_f32_wide_kernel<16, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
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
    launch_pdl(lmhead_f32_wide_kernel<16, 4>, dim3(tiles * Z), dim3(256), size_t(hidden) * 16 * 4, st, 
        c, hn_cache, W, bias, v_begin, v_count, hidden, am_val, am_idx, logits_out, ld_logits);
  }
}

}  // namespace ps
