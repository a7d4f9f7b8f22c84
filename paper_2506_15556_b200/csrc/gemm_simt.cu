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
// partials per lane), so each staged x float4 feeds 4R FMAs. Lane l still
// accumulates exactly the chunks c ≡ l (mod 32) of the K-split in order, and
// the 32 lane partials of every output are summed by a transposed butterfly
// whose adds are warp_sum's (same pairs, same order), so every output is
// bitwise the decode GEMV's.
// A CTA stages its TT-token chunk of x once and then walks its units j =
// blockIdx.x, + gridDim.x, ...; a unit is U consecutive 8R-row sub-tiles.
// Weight chunks stream through a per-warp kWideStages-stage shared-memory ring
// with cp.async, kWideStages - 1 chunks ahead and across sub-tile boundaries
// (3, 4 and 5 stages measured the same: c2 verify 4.44-4.46 ms): each lane copies
// and later reads only its own chunks, so a per-thread wait_group is the only
// synchronisation. (Register prefetch of the next chunk was sunk by the
// compiler to the end of the current one, and every chunk then waited a full
// L2/DRAM round trip.) epi(sums, first row of the warp, tt, nt) gets the two
// sums lane l holds after the butterfly (values 2l, 2l + 1; value = i*TT + t);
// unit_done(j) runs after each unit.
#ifndef PS_WIDE_STAGES
#define PS_WIDE_STAGES 3
#endif
constexpr int kWideStages = PS_WIDE_STAGES;  // weight chunks in flight: kWideStages - 1 ahead
// weight rows per warp in the wide GEMM (x 16 tokens): 8 rows halve the staged-x
// shared-memory reads per FMA against 4 (one 256-thread CTA per SM)
#ifndef PS_WIDE_R
#define PS_WIDE_R 8
#endif
constexpr int kWideR = PS_WIDE_R;
template <int TT, int R, int U, class Epi, class UnitDone>
__device__ __forceinline__ void wide_walk(const float* __restrict__ W, int N, int K, int kbeg, int nvec, int units,
                                          const float* __restrict__ X, int ldx, int rows, float4* xs4, Epi&& epi,
                                          UnitDone&& unit_done) {
  static_assert(R * TT % 64 == 0, "the transposed butterfly leaves R * TT / 32 sums per lane");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kmax = (nvec + 31) / 32;  // chunk steps per sub-tile (lanes past nvec%32 skip the last)
  const int my_units = int(blockIdx.x) < units ? (units - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;
  const int total = my_units * U * kmax;
  float4* ring = xs4 + TT * nvec + warp * (kWideStages * R * 32);  // [stage][R][lane]
  auto first_row = [&](int q) {  // first weight row of this warp in chunk step q's sub-tile
    const int st = q / kmax;
    return ((int(blockIdx.x) + (st / U) * int(gridDim.x)) * U + st % U) * (8 * R) + warp * R;
  };
  auto issue = [&](int q) {
    if (q < total) {
      const int c = lane + 32 * (q % kmax);
      if (c < nvec) {
        const int nb = first_row(q);
        float4* dst = ring + (q % kWideStages) * (R * 32) + lane;
#pragma unroll
        for (int i = 0; i < R; ++i) {
          const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst + i * 32));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d),
                       "l"(W + size_t(min(nb + i, N - 1)) * K + kbeg + 4 * c)
                       : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int tt = blockIdx.z * TT; tt < rows; tt += TT * gridDim.z) {
    const int nt = min(TT, rows - tt);
    __syncthreads();
#pragma unroll
    for (int q0 = 0; q0 < kWideStages - 1; ++q0) issue(q0);
    stage_x_async(xs4, X, ldx, kbeg, tt, nt, TT, nvec);  // (waits for every group: chunks 0, 1 too)
    __syncthreads();
    int q = 0;
    for (int j = blockIdx.x; j < units; j += gridDim.x) {
      for (int u = 0; u < U; ++u) {
        const int nb = first_row(q);
        float a[R * TT];
#pragma unroll
        for (int v = 0; v < R * TT; ++v) a[v] = 0.f;
        for (int k = 0; k < kmax; ++k, ++q) {
          issue(q + kWideStages - 1);
          asm volatile("cp.async.wait_group %0;" ::"n"(kWideStages - 1) : "memory");
          const int c = lane + 32 * k;
          if (c < nvec) {
            const float4* wr = ring + (q % kWideStages) * (R * 32) + lane;
            float4 wc[R];
#pragma unroll
            for (int i = 0; i < R; ++i) wc[i] = wr[i * 32];
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
          }
        }
        warp_sum_transposed<R * TT>(a, lane);
        epi(a, nb, tt, nt);
      }
      unit_done(j, tt, nt);
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");  // no copy into the ring outlives this chunk of x
  }
}

// this warp's weight rows of every unit the CTA will walk do not depend on the
// previous kernel: into L2 before the programmatic-dependency wait
template <int R, int U>
__device__ __forceinline__ void wide_prefetch(const float* W, int N, int K, int kbeg, int ksplit, int units) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int j = blockIdx.x; j < units; j += gridDim.x)
    for (int u = 0; u < U; ++u) {
      const int nb = (j * U + u) * (8 * R) + warp * R;
      if (nb < N) prefetch_rows_l2(W + size_t(nb) * K + kbeg, K, min(R, N - nb), ksplit, lane);
    }
}

template <int TT, int R>
__global__ void __launch_bounds__(256, R * TT > 64 ? 1 : 2) gemm_f32_wide_kernel(const PassCtx* __restrict__ ctx,
                                                               const float* __restrict__ X, int ldx,
                                                               const float* __restrict__ W, float* __restrict__ part,
                                                               int N, int K, int ksplit) {
  extern __shared__ float4 xs4[];
  const int lane = threadIdx.x & 31;
  const int ntiles = (N + 8 * R - 1) / (8 * R);
  const int s = blockIdx.y, kbeg = s * ksplit;
  wide_prefetch<R, 1>(W, N, K, kbeg, ksplit, ntiles);
  pdl_enter();
  if (ctx->stop) return;
  wide_walk<TT, R, 1>(
      W, N, K, kbeg, ksplit >> 2, ntiles, X, ldx, ctx->rows, xs4,
      [&](const float (&a)[R * TT], int nb, int tt, int nt) {
        constexpr int per = R * TT / 32;  // sums lane l holds: values per*l .. per*l + per - 1
#pragma unroll
        for (int jj = 0; jj < per; ++jj) {
          const int v = per * lane + jj, i = v / TT, t = v % TT;
          if (t < nt && nb + i < N) part[(size_t(s) * kMaxWindow + tt + t) * N + nb + i] = a[jj];
        }
      },
      [](int, int, int) {});
}

// CTAs per (K-split, token chunk) of a wide GEMM: about two resident CTAs per
// SM in total, never more than the tiles
static int wide_gx(int ntiles, int splits, int z, int per_sm = 2) {
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  const int per = (ntiles + max(1, per_sm * sms / (splits * z)) - 1) / max(1, per_sm * sms / (splits * z));  // tiles per CTA
  return (ntiles + per - 1) / per;
}

void launch_gemm_f32(const PassCtx* ctx, int max_rows, const float* X, int ldx, const float* W,
                     float* part, int N, int K, int splits, cudaStream_t st) {
  const int ksplit = K / splits;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_f32_wide_kernel<16, kWideR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(gemm_f32_gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  if (max_rows <= 1) {
    launch_pdl(gemm_f32_gemv_kernel, dim3(N / 16, splits, 1), dim3(256), size_t(ksplit) * 4, st, ctx, X, ldx, W, part,
               N, K, ksplit);
  } else {
    const int z = (max_rows + 15) / 16;
    const dim3 grid(wide_gx((N + 8 * kWideR - 1) / (8 * kWideR), splits, z, kWideR > 4 ? 1 : 2), splits, z);
    const size_t smem = size_t(ksplit) * 16 * 4 + size_t(8) * kWideStages * kWideR * 32 * 16;  // x chunk + weight rings
    launch_pdl(gemm_f32_wide_kernel<16, kWideR>, grid, dim3(256), smem, st, ctx, X, ldx, W, part, N, K, ksplit);
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
    launch_pdl(lmhead_f32_wide_kernel<16, 4>, dim3(tiles * Z), dim3(256), size_t(hidden) * 16 * 4, st, c, hn_cache, W,
               bias, v_begin, v_count, hidden, am_val, am_idx, logits_out, ld_logits);
  }
}

}  // namespace ps
