// Per-element arithmetic of the fp32 (bit-exact parity) path (layers.cu).
// Every product that feeds an add is spelled with an explicit-rounding
// intrinsic, so the value of an element cannot depend on how the compiler
// contracts the surrounding code; the same kernels score 1-row decode steps
// and wide passes, so a row is bitwise the same in both (batch invariance,
// SPEC.md:452), which the reference's lossless greedy property relies on.
#pragma once

#include "common.cuh"

namespace ps {

// RMSNorm scale of a row from its sum of squares
__device__ __forceinline__ float f32_rstd(float ss, int H, float eps) {
  return __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, float(H)), eps)));
}

// RoPE on a rotate-half pair (dims i, i + hd/2) with (cos, sin) = cs
__device__ __forceinline__ void f32_rope(float a, float b, float2 cs, float& ra, float& rb) {
  ra = __fsub_rn(__fmul_rn(a, cs.x), __fmul_rn(b, cs.y));
  rb = __fadd_rn(__fmul_rn(b, cs.x), __fmul_rn(a, cs.y));
}

// SwiGLU: silu(gate) * up
__device__ __forceinline__ float f32_swiglu(float g, float u) {
  return __fmul_rn(__fdiv_rn(g, __fadd_rn(1.0f, expf(-g))), u);
}

// Attention of one query head over one 64-token page, staged in shared memory
// (Ks [64][hd+1], Vs [64][hd]); one warp: lane j scores keys j and j + 32,
// then lanes own head dims lane, lane + 32, ... of P.V. Writes the page-local
// (O, m, l) at slot.
__device__ __forceinline__ void f32_attn_page_head(const float* qs, const float* Ks, const float* Vs, int hd,
                                                   int nkeys, float scale, int lane, float* __restrict__ o_slot,
                                                   float* __restrict__ ml_slot) {
  float sc[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int j = lane + 32 * r;
    float acc = 0.f;
    if (j < nkeys) {
      const float* kr = Ks + j * (hd + 1);
      for (int d = 0; d < hd; ++d) acc = fmaf(qs[d], kr[d], acc);
      sc[r] = __fmul_rn(acc, scale);
    } else {
      sc[r] = -INFINITY;
    }
  }
  const float m = warp_max(fmaxf(sc[0], sc[1]));
  const float p0 = (lane < nkeys) ? expf(__fsub_rn(sc[0], m)) : 0.f;
  const float p1 = (lane + 32 < nkeys) ? expf(__fsub_rn(sc[1], m)) : 0.f;
  const float l = warp_sum(__fadd_rn(p0, p1));
  for (int d = lane; d < hd; d += 32) {
    float acc = 0.f;
    for (int j = 0; j < nkeys; ++j) {
      const float pj = __shfl_sync(0xffffffffu, j < 32 ? p0 : p1, j & 31);
      acc = fmaf(pj, Vs[j * hd + d], acc);
    }
    o_slot[d] = acc;
  }
  if (lane == 0) {
    ml_slot[0] = m;
    ml_slot[1] = l;
  }
}

// p[0][c] + p[1][c] + ... + p[splits-1][c] in split order (rows `stride` apart),
// every load issued before the first add (up to 8 splits in flight).
__device__ __forceinline__ float f32_sum_splits(const float* __restrict__ p, int splits, size_t stride) {
  float v[8];
#pragma unroll
  for (int s = 0; s < 8; ++s)
    if (s < splits) v[s] = __ldcg(p + s * stride);
  float d = v[0];
#pragma unroll
  for (int s = 1; s < 8; ++s)
    if (s < splits) d += v[s];
  for (int s = 8; s < splits; ++s) d += __ldcg(p + s * stride);
  return d;
}

// Combine of one (row, head, dim) over its pages in page order.
__device__ __forceinline__ float f32_attn_combine(const float* __restrict__ o_part, const float* __restrict__ ml_part,
                                                  size_t base, int nsplit, int hd, int d) {
  float M = -INFINITY;
  for (int s = 0; s < nsplit; ++s) M = fmaxf(M, __ldcg(ml_part + (base + s) * 2));
  float L = 0.f, acc = 0.f;
  for (int s = 0; s < nsplit; ++s) {
    const float f = expf(__fsub_rn(__ldcg(ml_part + (base + s) * 2), M));
    L = fmaf(__ldcg(ml_part + (base + s) * 2 + 1), f, L);
    acc = fmaf(__ldcg(o_part + (base + s) * hd + d), f, acc);
  }
  return __fdiv_rn(acc, L);
}

}  // namespace ps
