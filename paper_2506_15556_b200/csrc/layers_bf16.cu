// Row kernels of the bf16 decode chain, launched with programmatic dependent
// launch (PDL) so their launch latency hides under the previous kernel.
//
//   embed_bf16      x = E[tok] (fp32 master), xb = bf16 copy (the next GEMM's
//                   B operand), rstd = 1/sqrt(mean(x^2)+eps) (applied by the
//                   GEMM epilogue: W.(x*rstd) == rstd*(W.x), gamma = 1)
//   attention_bf16  causal GQA attention over 64-token KV pages; CTA =
//                   (row, kv head, page); the last page CTA of a (row, kv
//                   head) merges the page partials in page order and writes
//                   the bf16 output — no separate combine launch.
#include "common.cuh"
#include "kernels.h"

namespace ps {

namespace {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
void launch_maybe_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
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
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, args...);
}

}  // namespace

__global__ void __launch_bounds__(256) embed_bf16_kernel(PassCtx* ctx, const int* __restrict__ tok_in,
                                                         int* __restrict__ tokens_dev, const int* __restrict__ argmax_pos,
                                                         const __nv_bfloat16* __restrict__ embed, float* __restrict__ x,
                                                         __nv_bfloat16* __restrict__ xb, float* __restrict__ rstd,
                                                         int H, float eps) {
  __shared__ float red[32];
  __shared__ int s_tok;
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x;
  if (ctx->stop || t >= ctx->rows) return;
  const int pos = ctx->n0 + t;
  if (threadIdx.x == 0) {
    int tok;
    if (tok_in) {
      tok = tok_in[t];
    } else {
      tok = argmax_pos[pos - 1];
      if (ctx->stop_on_eos && tok == kEos) ctx->stop = 1;
    }
    tokens_dev[pos] = tok;
    s_tok = tok;
  }
  __syncthreads();
  if (ctx->stop) return;
  const uint4* e = reinterpret_cast<const uint4*>(embed + size_t(s_tok) * H);
  uint4* ob = reinterpret_cast<uint4*>(xb + size_t(t) * H);
  float* xr = x + size_t(t) * H;
  float ss = 0.f;
  for (int c = threadIdx.x; c < H / 8; c += 256) {
    const uint4 raw = e[c];
    ob[c] = raw;
    const __nv_bfloat16* v = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float f = __bfloat162float(v[i]);
      xr[c * 8 + i] = f;
      ss = fmaf(f, f, ss);
    }
  }
  ss = block_sum<256>(ss, red);
  if (threadIdx.x == 0) rstd[t] = 1.0f / sqrtf(ss / float(H) + eps);
}

void launch_embed_bf16(PassCtx* ctx, int max_rows, const int* tok_in, int* tokens_dev, const int* argmax_pos,
                       const __nv_bfloat16* embed, float* x, __nv_bfloat16* xb, float* rstd, int hidden, float eps,
                       cudaStream_t st, bool pdl) {
  launch_maybe_pdl(embed_bf16_kernel, dim3(max_rows), dim3(256), 0, st, pdl, ctx, tok_in, tokens_dev, argmax_pos,
                   embed, x, xb, rstd, hidden, eps);
}

__global__ void attention_bf16_kernel(PassCtx* ctx, const __nv_bfloat16* __restrict__ q,
                                      const __nv_bfloat16* __restrict__ kpool, const __nv_bfloat16* __restrict__ vpool,
                                      const int* __restrict__ page_table, KvGeom g, int layer, int heads,
                                      int max_splits, float scale, float* __restrict__ o_part,
                                      float* __restrict__ ml_part, unsigned* __restrict__ cnt,
                                      __nv_bfloat16* __restrict__ out) {
  extern __shared__ float sm[];
  __shared__ int s_last;
  pdl_trigger();
  pdl_wait();
  const int t = blockIdx.x, kvh = blockIdx.y, s = blockIdx.z;
  if (ctx->stop || t >= ctx->rows) return;
  const int pos = ctx->n0 + t;
  const int nsplit = pos / kPage + 1;
  if (s >= nsplit) return;
  const int hd = g.head_dim, grp = heads / g.kv_heads;
  const int nkeys = min(kPage, pos + 1 - s * kPage);
  float* Ks = sm;                     // [64][hd+1]
  float* Vs = Ks + kPage * (hd + 1);  // [64][hd]
  float* Qs = Vs + kPage * hd;        // [grp][hd]
  const size_t page = size_t(page_table[s]);
  const size_t off = size_t(layer) * g.layer_stride() + (page * g.kv_heads + kvh) * kPage * hd;
  const int vec_per_row = hd / 8;
  for (int e = threadIdx.x; e < nkeys * vec_per_row; e += blockDim.x) {
    const int j = e / vec_per_row, d0 = (e % vec_per_row) * 8;
    const uint4 kr = *reinterpret_cast<const uint4*>(kpool + off + size_t(j) * hd + d0);
    const uint4 vr = *reinterpret_cast<const uint4*>(vpool + off + size_t(j) * hd + d0);
    const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(&kr);
    const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(&vr);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      Ks[j * (hd + 1) + d0 + i] = __bfloat162float(kb[i]);
      Vs[j * hd + d0 + i] = __bfloat162float(vb[i]);
    }
  }
  const __nv_bfloat16* qrow = q + size_t(t) * heads * hd + size_t(kvh) * grp * hd;
  for (int e = threadIdx.x; e < grp * hd; e += blockDim.x) Qs[e] = __bfloat162float(qrow[e]);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int h = kvh * grp + w;
  if (w < grp) {
    const float* qs = Qs + w * hd;
    float sc[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int j = lane + 32 * r;
      float acc = 0.f;
      if (j < nkeys) {
        const float* kr = Ks + j * (hd + 1);
        for (int d = 0; d < hd; ++d) acc = fmaf(qs[d], kr[d], acc);
        sc[r] = acc * scale;
      } else {
        sc[r] = -INFINITY;
      }
    }
    const float m = warp_max(fmaxf(sc[0], sc[1]));
    const float p0 = (lane < nkeys) ? expf(sc[0] - m) : 0.f;
    const float p1 = (lane + 32 < nkeys) ? expf(sc[1] - m) : 0.f;
    const float l = warp_sum(p0 + p1);
    const size_t slot = (size_t(t) * heads + h) * max_splits + s;
    for (int d = lane; d < hd; d += 32) {
      float acc = 0.f;
      for (int j = 0; j < nkeys; ++j) {
        const float pj = __shfl_sync(0xffffffffu, j < 32 ? p0 : p1, j & 31);
        acc = fmaf(pj, Vs[j * hd + d], acc);
      }
      o_part[slot * hd + d] = acc;
    }
    if (lane == 0) {
      ml_part[slot * 2] = m;
      ml_part[slot * 2 + 1] = l;
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* c = cnt + size_t(t) * g.kv_heads + kvh;
    const unsigned old = atomicAdd(c, 1u);
    s_last = old == unsigned(nsplit - 1);
    if (s_last) *c = 0u;
  }
  __syncthreads();
  if (!s_last || w >= grp) return;
  __threadfence();
  // merge the page partials in page order (same arithmetic for any pass width)
  const size_t base = (size_t(t) * heads + h) * max_splits;
  float M = -INFINITY;
  for (int sp = 0; sp < nsplit; ++sp) M = fmaxf(M, __ldcg(ml_part + (base + sp) * 2));
  for (int d = lane; d < hd; d += 32) {
    float L = 0.f, acc = 0.f;
    for (int sp = 0; sp < nsplit; ++sp) {
      const float f = expf(__ldcg(ml_part + (base + sp) * 2) - M);
      L = fmaf(__ldcg(ml_part + (base + sp) * 2 + 1), f, L);
      acc = fmaf(__ldcg(o_part + (base + sp) * hd + d), f, acc);
    }
    out[size_t(t) * heads * hd + size_t(h) * hd + d] = __float2bfloat16_rn(acc / L);
  }
}

void launch_attention_bf16(PassCtx* ctx, int max_rows, int max_pos, const __nv_bfloat16* q,
                           const __nv_bfloat16* kpool, const __nv_bfloat16* vpool, const int* page_table, KvGeom g,
                           int layer, int heads, float* o_part, float* ml_part, unsigned* cnt,
                           __nv_bfloat16* attn_out, cudaStream_t st, bool pdl) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attention_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr = true;
  }
  const int max_splits = max_pos / kPage + 1;
  const int grp = heads / g.kv_heads, hd = g.head_dim;
  const size_t smem = (size_t(kPage) * (hd + 1) + size_t(kPage) * hd + size_t(grp) * hd) * sizeof(float);
  const float scale = float(1.0 / sqrt(double(hd)));
  launch_maybe_pdl(attention_bf16_kernel, dim3(max_rows, g.kv_heads, max_splits), dim3(grp * 32), smem, st, pdl,
                   ctx, q, kpool, vpool, page_table, g, layer, heads, max_splits, scale, o_part, ml_part, cnt,
                   attn_out);
}

}  // namespace ps
