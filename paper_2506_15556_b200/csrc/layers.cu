// Row-parallel kernels around the GEMMs: embedding + RMSNorm, split-K
// reduction fused with bias/RoPE/KV-append, paged causal attention,
// residual + RMSNorm, SwiGLU, argmax reduction and the greedy-verify compare.
//
// Batch invariance (what keeps greedy speculation lossless):
// every output element is produced by an arithmetic sequence that depends
// only on its own row and absolute position — never on how many rows share
// the pass. Split-K boundaries depend on (N, K) only and partials are summed
// in split order; attention splits at absolute 64-token page boundaries and
// combines them in order. A row computed inside a 72-row verify pass is
// therefore bit-identical to the same row computed by a 1-row decode step.
#include "common.cuh"
#include "f32_math.cuh"
#include "kernels.h"

namespace ps {

// ---------------------------------------------------------------------------
// embedding gather + first RMSNorm (one CTA per row)
// decode mode (tok_in == nullptr): the row's token is the argmax of the
// previous position, so consecutive graph replays chain on the device.
template <typename T>
__global__ void __launch_bounds__(256) embed_norm_kernel(PassCtx* ctx, const int* __restrict__ tok_in,
                                                         int* __restrict__ tokens_dev,
                                                         const int* __restrict__ argmax_pos,
                                                         const T* __restrict__ embed, float* __restrict__ x,
                                                         T* __restrict__ xn, int H, float eps) {
  pdl_enter();
  __shared__ float red[32];
  __shared__ int s_tok;
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
  const T* e = embed + size_t(s_tok) * H;
  float* xr = x + size_t(t) * H;
  float ss = 0.f;
  for (int c = threadIdx.x; c < H; c += 256) {
    float v = ld_as_f32(e + c);
    xr[c] = v;
    ss = fmaf(v, v, ss);
  }
  ss = block_sum<256>(ss, red);
  const float rstd = f32_rstd(ss, H, eps);
  T* o = xn + size_t(t) * H;
  for (int c = threadIdx.x; c < H; c += 256) o[c] = from_f32<T>(__fmul_rn(xr[c], rstd));
}

template <typename T>
void launch_embed_norm(const PassCtx* ctx, int max_rows, const int* tok_in, int* tokens_dev,
                       const int* argmax_pos, const T* embed, float* x, T* xn, int hidden, float eps,
                       cudaStream_t st) {
  launch_pdl(embed_norm_kernel<T>, dim3(max_rows), dim3(256), 0, st, const_cast<PassCtx*>(ctx), tok_in, tokens_dev,
                                                  argmax_pos, embed, x, xn, hidden, eps);
}

// ---------------------------------------------------------------------------
// split-K sum + bias + RoPE (rotate-half) + q store + paged K/V append
template <typename T>
__global__ void __launch_bounds__(128) qkv_finalize_kernel(const PassCtx* __restrict__ ctx,
                                                           const float* __restrict__ part, int splits,
                                                           int N, const T* __restrict__ bias,
                                                           const float2* __restrict__ rope, T* __restrict__ q,
                                                           T* __restrict__ kpool, T* __restrict__ vpool,
                                                           const int* __restrict__ page_table, KvGeom g,
                                                           int layer, int heads) {
  pdl_enter();
  const int t = blockIdx.x;
  if (ctx->stop || t >= ctx->rows) return;
  const int pos = ctx->n0 + t;
  const int hd = g.head_dim, half = hd >> 1;
  const int nq = heads * half, nk = g.kv_heads * half;
  // one (pair) item per thread: blockIdx.y spreads the row's items over CTAs,
  // so a 1-row decode pass has all its loads in flight at once
  const size_t sstride = size_t(kMaxWindow) * N;
  const float* pr = part + size_t(t) * N;
  auto sum_col = [&](int c) {
    float v = f32_sum_splits(pr + c, splits, sstride);  // split order, loads in flight together
    if (bias) v += ld_as_f32(bias + c);
    return v;
  };
  const size_t page = size_t(page_table[pos / kPage]);
  const int slot = pos % kPage;
  const size_t lbase = size_t(layer) * g.layer_stride();
  for (int p = blockIdx.y * blockDim.x + threadIdx.x; p < nq + 2 * nk; p += blockDim.x * gridDim.y) {
    if (p < nq + nk) {
      const bool is_q = p < nq;
      const int pp = is_q ? p : p - nq;
      const int h = pp / half, i = pp % half;
      const int col = (is_q ? 0 : heads * hd) + h * hd + i;
      const float a = sum_col(col), b = sum_col(col + half);
      float ra, rb;
      f32_rope(a, b, rope[size_t(pos) * half + i], ra, rb);
      if (is_q) {
        T* qr = q + size_t(t) * heads * hd + h * hd;
        qr[i] = from_f32<T>(ra);
        qr[i + half] = from_f32<T>(rb);
      } else {
        T* kr = kpool + lbase + ((page * g.kv_heads + h) * kPage + slot) * hd;
        kr[i] = from_f32<T>(ra);
        kr[i + half] = from_f32<T>(rb);
      }
    } else {
      const int pp = p - nq - nk;  // v pairs: write two plain elements
      const int h = pp / half, i = pp % half;
      const int col = (heads + g.kv_heads) * hd + h * hd + i;
      T* vr = vpool + lbase + ((page * g.kv_heads + h) * kPage + slot) * hd;
      vr[i] = from_f32<T>(sum_col(col));
      vr[i + half] = from_f32<T>(sum_col(col + half));
    }
  }
}

template <typename T>
void launch_qkv_finalize(const PassCtx* ctx, int max_rows, const float* part, int splits, int ldp,
                         const T* bias, const float2* rope, T* q, T* kpool, T* vpool,
                         const int* page_table, KvGeom g, int layer, int heads, cudaStream_t st) {
  const int items = (heads + 2 * g.kv_heads) * g.head_dim / 2;
  launch_pdl(qkv_finalize_kernel<T>, dim3(max_rows, (items + 127) / 128), dim3(128), 0, st, ctx, part, splits, ldp, bias,
             rope, q, kpool, vpool, page_table, g, layer, heads);
}

// ---------------------------------------------------------------------------
// causal attention over the paged prefix. CTA = (query row, kv head, page);
// one warp per query head of the GQA group. Scores: lane j owns keys j and
// j+32 of the page; values: lane owns head dims lane, lane+32, ...
template <typename T>
__global__ void attention_page_kernel(const PassCtx* __restrict__ ctx, const T* __restrict__ q,
                                      const T* __restrict__ kpool, const T* __restrict__ vpool,
                                      const int* __restrict__ page_table, KvGeom g, int layer, int heads,
                                      int max_splits, float scale, float* __restrict__ o_part,
                                      float* __restrict__ ml_part) {
  pdl_enter();
  extern __shared__ float sm[];
  const int t = blockIdx.x, kvh = blockIdx.y, s = blockIdx.z;
  if (ctx->stop || t >= ctx->rows) return;
  const int pos = ctx->n0 + t;
  if (s > pos / kPage) return;
  const int hd = g.head_dim, grp = heads / g.kv_heads;
  const int nkeys = min(kPage, pos + 1 - s * kPage);
  float* Ks = sm;                       // [64][hd+1]
  float* Vs = Ks + kPage * (hd + 1);    // [64][hd]
  float* Qs = Vs + kPage * hd;          // [grp][hd]
  const size_t page = size_t(page_table[s]);
  const size_t off = size_t(layer) * g.layer_stride() + (page * g.kv_heads + kvh) * kPage * hd;
  if constexpr (sizeof(T) == 4) {
    // float4 loads, four in flight per thread for K and for V (hd is a multiple of 4)
    const int n4 = nkeys * hd / 4;
    for (int e0 = threadIdx.x; e0 < n4; e0 += blockDim.x * 4) {
      float4 kv[4], vv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + int(blockDim.x) * u;
        if (e < n4) {
          kv[u] = __ldg(reinterpret_cast<const float4*>(kpool + off) + e);
          vv[u] = __ldg(reinterpret_cast<const float4*>(vpool + off) + e);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + int(blockDim.x) * u;
        if (e < n4) {
          const int j = (4 * e) / hd, d = (4 * e) % hd;
          float* kr = Ks + j * (hd + 1) + d;
          kr[0] = kv[u].x; kr[1] = kv[u].y; kr[2] = kv[u].z; kr[3] = kv[u].w;
          *reinterpret_cast<float4*>(Vs + j * hd + d) = vv[u];
        }
      }
    }
  } else {
    for (int e = threadIdx.x; e < nkeys * hd; e += blockDim.x) {
      const int j = e / hd, d = e % hd;
      Ks[j * (hd + 1) + d] = ld_as_f32(kpool + off + e);
      Vs[j * hd + d] = ld_as_f32(vpool + off + e);
    }
  }
  const T* qrow = q + size_t(t) * heads * hd + size_t(kvh) * grp * hd;
  for (int e = threadIdx.x; e < grp * hd; e += blockDim.x) Qs[e] = ld_as_f32(qrow + e);
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w >= grp) return;
  const size_t slot = (size_t(t) * heads + kvh * grp + w) * max_splits + s;
  f32_attn_page_head(Qs + w * hd, Ks, Vs, hd, nkeys, scale, lane, o_part + slot * hd, ml_part + slot * 2);
}

template <typename T>
__global__ void attention_combine_kernel(const PassCtx* __restrict__ ctx, int heads, int hd, int max_splits,
                                         const float* __restrict__ o_part, const float* __restrict__ ml_part,
                                         T* __restrict__ out) {
  pdl_enter();
  const int t = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
  if (ctx->stop || t >= ctx->rows) return;
  const int nsplit = (ctx->n0 + t) / kPage + 1;
  const size_t base = (size_t(t) * heads + h) * max_splits;
  out[size_t(t) * heads * hd + size_t(h) * hd + d] = from_f32<T>(f32_attn_combine(o_part, ml_part, base, nsplit, hd, d));
}

// Decode steps (1 row): qkv_finalize and attention_page in one launch. CTA =
// (kv head, page) as attention_page_kernel's; every CTA finalises the q of
// its GQA group itself (split-K sum + bias + RoPE: qkv_finalize's arithmetic,
// so q is bitwise the same), and the CTA of the row's last page also
// finalises the step's k / v and appends them to the paged cache before
// staging that page (no other CTA reads them). One kernel and one global
// round trip less per layer than the separate pair.
__global__ void __launch_bounds__(512) qkv_attention_decode_kernel(
    const PassCtx* __restrict__ ctx, const float* __restrict__ part, int splits, int N, const float* __restrict__ bias,
    const float2* __restrict__ rope, float* __restrict__ kpool, float* __restrict__ vpool,
    const int* __restrict__ page_table, KvGeom g, int layer, int heads, int max_splits, float scale,
    float* __restrict__ o_part, float* __restrict__ ml_part) {
  pdl_enter();
  extern __shared__ float sm[];
  const int kvh = blockIdx.x, s = blockIdx.y;
  if (ctx->stop || ctx->rows < 1) return;
  const int pos = ctx->n0;  // row t = 0
  if (s > pos / kPage) return;
  const int hd = g.head_dim, half = hd >> 1, grp = heads / g.kv_heads;
  const int nkeys = min(kPage, pos + 1 - s * kPage);
  float* Ks = sm;                     // [64][hd+1]
  float* Vs = Ks + kPage * (hd + 1);  // [64][hd]
  float* Qs = Vs + kPage * hd;        // [grp][hd]
  const size_t sstride = size_t(kMaxWindow) * N;
  auto sum_col = [&](int c) {
    float v = f32_sum_splits(part + c, splits, sstride);
    if (bias) v += bias[c];
    return v;
  };
  const size_t page = size_t(page_table[s]);
  const size_t off = size_t(layer) * g.layer_stride() + (page * g.kv_heads + kvh) * kPage * hd;
  const bool last = s == pos / kPage;
  // q of the group's heads (pairs), and on the last page the step's k / v
  const int nqp = grp * half, nkp = last ? half : 0, nv = last ? half : 0;
  for (int p = threadIdx.x; p < nqp + nkp + nv; p += blockDim.x) {
    if (p < nqp + nkp) {
      const bool is_q = p < nqp;
      const int pp = is_q ? p : p - nqp;
      const int h = pp / half, i = pp % half;  // (local head for q)
      const int col = is_q ? (kvh * grp + h) * hd + i : heads * hd + kvh * hd + i;
      float ra, rb;
      f32_rope(sum_col(col), sum_col(col + half), rope[size_t(pos) * half + i], ra, rb);
      if (is_q) {
        Qs[h * hd + i] = ra;
        Qs[h * hd + i + half] = rb;
      } else {
        float* kr = kpool + off + size_t(pos % kPage) * hd;
        kr[i] = ra;
        kr[i + half] = rb;
      }
    } else {
      const int i = p - nqp - nkp;
      const int col = (heads + g.kv_heads) * hd + kvh * hd + i;
      float* vr = vpool + off + size_t(pos % kPage) * hd;
      vr[i] = sum_col(col);
      vr[i + half] = sum_col(col + half);
    }
  }
  __syncthreads();  // the appended k / v row is read back below (L2 loads, same CTA)
  const int n4 = nkeys * hd / 4;
  for (int e0 = threadIdx.x; e0 < n4; e0 += blockDim.x * 4) {
    float4 kv[4], vv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + int(blockDim.x) * u;
      if (e < n4) {
        kv[u] = __ldcg(reinterpret_cast<const float4*>(kpool + off) + e);
        vv[u] = __ldcg(reinterpret_cast<const float4*>(vpool + off) + e);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + int(blockDim.x) * u;
      if (e < n4) {
        const int j = (4 * e) / hd, d = (4 * e) % hd;
        float* kr = Ks + j * (hd + 1) + d;
        kr[0] = kv[u].x; kr[1] = kv[u].y; kr[2] = kv[u].z; kr[3] = kv[u].w;
        *reinterpret_cast<float4*>(Vs + j * hd + d) = vv[u];
      }
    }
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (w >= grp) return;
  const size_t slot = (size_t(kvh * grp + w)) * max_splits + s;  // row t = 0
  f32_attn_page_head(Qs + w * hd, Ks, Vs, hd, nkeys, scale, lane, o_part + slot * hd, ml_part + slot * 2);
}

void launch_qkv_attention_decode(const PassCtx* ctx, int max_pos, const float* part, int splits, int N,
                                 const float* bias, const float2* rope, float* kpool, float* vpool,
                                 const int* page_table, KvGeom g, int layer, int heads, float* o_part,
                                 float* ml_part, float* attn_out, cudaStream_t st) {
  const int max_splits = max_pos / kPage + 1;
  const int grp = heads / g.kv_heads, hd = g.head_dim;
  const size_t smem = (size_t(kPage) * (hd + 1) + size_t(kPage) * hd + size_t(grp) * hd) * sizeof(float);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(qkv_attention_decode_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr = true;
  }
  const float scale = float(1.0 / sqrt(double(hd)));
  launch_pdl(qkv_attention_decode_kernel, dim3(g.kv_heads, max_splits), dim3(max(grp, 4) * 32), smem, st, ctx, part,
             splits, N, bias, rope, kpool, vpool, page_table, g, layer, heads, max_splits, scale, o_part, ml_part);
  launch_pdl(attention_combine_kernel<float>, dim3(1, heads), dim3(hd), 0, st, ctx, heads, hd, max_splits, o_part,
             ml_part, attn_out);
}

template <typename T>
void launch_attention(const PassCtx* ctx, int max_rows, int max_pos, const T* q, const T* kpool,
                      const T* vpool, const int* page_table, KvGeom g, int layer, int heads,
                      float* o_part, float* ml_part, T* attn_out, cudaStream_t st) {
  const int max_splits = max_pos / kPage + 1;
  const int grp = heads / g.kv_heads;
  const int hd = g.head_dim;
  const size_t smem = (size_t(kPage) * (hd + 1) + size_t(kPage) * hd + size_t(grp) * hd) * sizeof(float);
  static bool attr_set[2] = {false, false};
  const int key = sizeof(T) == 4 ? 0 : 1;
  if (!attr_set[key]) {
    cudaFuncSetAttribute(attention_page_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr_set[key] = true;
  }
  const float scale = float(1.0 / sqrt(double(hd)));
  dim3 grid(max_rows, g.kv_heads, max_splits);
  launch_pdl(attention_page_kernel<T>, dim3(grid), dim3(grp * 32), smem, st, ctx, q, kpool, vpool, page_table, g, layer, heads,
                                                         max_splits, scale, o_part, ml_part);
  launch_pdl(attention_combine_kernel<T>, dim3(dim3(max_rows, heads)), dim3(hd), 0, st, ctx, heads, hd, max_splits, o_part,
                                                                     ml_part, attn_out);
}

// ---------------------------------------------------------------------------
// x += sum_s part[s]; then RMSNorm -> xn (next GEMM input) or, after the last
// layer, -> hn_cache[pos] (LM-head input, kept per position for lazy rows).
template <typename T>
__global__ void __launch_bounds__(256) residual_norm_kernel(const PassCtx* __restrict__ ctx, float* __restrict__ x,
                                                            const float* __restrict__ part, int splits,
                                                            T* __restrict__ xn, T* __restrict__ hn_cache, int H,
                                                            float eps) {
  pdl_enter();
  __shared__ float red[32];
  const int t = blockIdx.x;
  if (ctx->stop || t >= ctx->rows) return;
  const size_t sstride = size_t(kMaxWindow) * H;
  float* xr = x + size_t(t) * H;
  const float* pr = part + size_t(t) * H;
  float ss = 0.f;
  // elements c = tid, tid + 256, ... in order; kBatch of them with every load
  // (residual and split partials) in flight before the first add
  constexpr int kBatch = 4;
  for (int c0 = threadIdx.x; c0 < H; c0 += 256 * kBatch) {
    float xv[kBatch], dv[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int c = c0 + 256 * j;
      if (c < H) {
        xv[j] = xr[c];
        dv[j] = f32_sum_splits(pr + c, splits, sstride);
      }
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int c = c0 + 256 * j;
      if (c < H) {
        const float v = __fadd_rn(xv[j], dv[j]);
        xr[c] = v;
        ss = fmaf(v, v, ss);
      }
    }
  }
  ss = block_sum<256>(ss, red);
  const float rstd = f32_rstd(ss, H, eps);
  T* o = hn_cache ? hn_cache + size_t(ctx->n0 + t) * H : xn + size_t(t) * H;
  for (int c = threadIdx.x; c < H; c += 256) o[c] = from_f32<T>(__fmul_rn(xr[c], rstd));
}

template <typename T>
void launch_residual_norm(const PassCtx* ctx, int max_rows, float* x, const float* part, int splits,
                          int ldp, T* xn, T* hn_cache, int hidden, float eps, cudaStream_t st) {
  (void)ldp;
  launch_pdl(residual_norm_kernel<T>, dim3(max_rows), dim3(256), 0, st, ctx, x, part, splits, xn, hn_cache, hidden, eps);
}

// ---------------------------------------------------------------------------
template <typename T>
__global__ void swiglu_kernel(const PassCtx* __restrict__ ctx, const float* __restrict__ part, int splits,
                              T* __restrict__ act, int I) {
  pdl_enter();
  const int t = blockIdx.y;
  if (ctx->stop || t >= ctx->rows) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= I) return;
  const int N = 2 * I;
  const size_t sstride = size_t(kMaxWindow) * N;
  const float* pr = part + size_t(t) * N;
  const float gsum = f32_sum_splits(pr + i, splits, sstride), usum = f32_sum_splits(pr + I + i, splits, sstride);
  act[size_t(t) * I + i] = from_f32<T>(f32_swiglu(gsum, usum));
}

template <typename T>
void launch_swiglu(const PassCtx* ctx, int max_rows, const float* part, int splits, int ldp, T* act,
                   int inter, cudaStream_t st) {
  (void)ldp;
  launch_pdl(swiglu_kernel<T>, dim3(dim3((inter + 255) / 256, max_rows)), dim3(256), 0, st, ctx, part, splits, act, inter);
}

// ---------------------------------------------------------------------------
// argmax over vocab-tile partials; ties -> lowest id (merge is a total order,
// so the result does not depend on reduction order).
__global__ void __launch_bounds__(256) argmax_reduce_kernel(PassCtx* ctx, const float* __restrict__ am_val,
                                                            const int* __restrict__ am_idx, int tiles,
                                                            int* __restrict__ argmax_pos,
                                                            unsigned long long* __restrict__ packed_out) {
  pdl_enter();
  __shared__ float sv[8];
  __shared__ int si[8];
  const int t = blockIdx.x;
  if (ctx->stop || t >= ctx->rows) return;
  float v = -INFINITY;
  int i = 0x7fffffff;
  for (int k = threadIdx.x; k < tiles; k += 256)
    argmax_merge(v, i, am_val[size_t(k) * kMaxWindow + t], am_idx[size_t(k) * kMaxWindow + t]);
  warp_argmax(v, i);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sv[w] = v; si[w] = i; }
  __syncthreads();
  if (w == 0) {
    v = l < 8 ? sv[l] : -INFINITY;
    i = l < 8 ? si[l] : 0x7fffffff;
    warp_argmax(v, i);
    if (l == 0) {
      argmax_pos[ctx->n0 + t] = i;
      if (packed_out) {
        // orderable float key in the high word, (0xFFFFFFFF - id) low: a
        // uint64 MAX across vocab shards yields (max value, lowest id).
        unsigned u = __float_as_uint(v);
        u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
        packed_out[t] = (static_cast<unsigned long long>(u) << 32) | (0xFFFFFFFFull - unsigned(i));
      }
    }
  }
}

void launch_argmax_reduce(const PassCtx* ctx, int max_rows, const float* am_val, const int* am_idx,
                          int tiles, int* argmax_pos, unsigned long long* packed_out, cudaStream_t st) {
  launch_pdl(argmax_reduce_kernel, dim3(max_rows), dim3(256), 0, st, const_cast<PassCtx*>(ctx), am_val, am_idx, tiles, argmax_pos,
                                                 packed_out);
}

// ---------------------------------------------------------------------------
// greedy verify epilogue (one warp): accept length + first terminator of R.
__global__ void verify_compare_kernel(const int* __restrict__ argmax_pos, int p0, const int* __restrict__ cand,
                                      int n_cand, const unsigned char* __restrict__ term_mask,
                                      int* __restrict__ res) {
  const int lane = threadIdx.x;
  int k = n_cand, first_term = -1;
  for (int base = 0; base < n_cand; base += 32) {
    const int i = base + lane;
    bool miss = false, term = false;
    if (i < n_cand) {
      const int tok = cand[i];
      miss = argmax_pos[p0 - 1 + i] != tok;
      term = term_mask[tok] != 0;
    }
    const unsigned mb = __ballot_sync(0xffffffffu, miss);
    const unsigned tb = __ballot_sync(0xffffffffu, term);
    if (first_term < 0 && tb) first_term = base + __ffs(tb) - 1;
    if (mb) { k = base + __ffs(mb) - 1; break; }
  }
  // keep scanning for the terminator past the mismatch
  if (first_term < 0) {
    for (int base = (k / 32) * 32; base < n_cand; base += 32) {
      const int i = base + lane;
      const bool term = i < n_cand && term_mask[cand[i]] != 0;
      const unsigned tb = __ballot_sync(0xffffffffu, term);
      if (tb) { first_term = base + __ffs(tb) - 1; break; }
    }
  }
  if (lane == 0) { res[0] = k; res[1] = first_term; }
}

void launch_verify_compare(const int* argmax_pos, int p0, const int* cand, int n_cand,
                           const unsigned char* term_mask, int* res, cudaStream_t st) {
  verify_compare_kernel<<<1, 32, 0, st>>>(argmax_pos, p0, cand, n_cand, term_mask, res);
}

// Top-k verification rule (verify_topk, verify.py:100-113; topk_tokens,
// lm.py:139-145): candidate token t of row i is inside the top k iff its rank
// #{j : s_j > s_t  or  (s_j == s_t and j < t)} is below k. No sort: every
// block counts a slice of the vocabulary for one row and adds its integer
// count (order-free, so exact). logits: [n][ld] fp32, the LM phase's values.
__global__ void topk_rank_kernel(const float* __restrict__ logits, int ld, int V, const int* __restrict__ cand, int n,
                                 int* __restrict__ rank) {
  const int i = blockIdx.y;
  if (i >= n) return;
  const int t = cand[i];
  const float* row = logits + size_t(i) * ld;
  const float st = row[t];
  int cnt = 0;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < V; j += gridDim.x * blockDim.x) {
    const float sj = row[j];
    cnt += (sj > st || (sj == st && j < t)) ? 1 : 0;
  }
  cnt = warp_sum_int(cnt);
  __shared__ int part[8];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) tot += part[w];
    if (tot) atomicAdd(rank + i, tot);
  }
}

void launch_topk_rank(const float* logits, int ld, int V, const int* cand, int n, int* rank, cudaStream_t st) {
  cudaMemsetAsync(rank, 0, sizeof(int) * n, st);
  const dim3 grid((V + 256 * 16 - 1) / (256 * 16), n);
  topk_rank_kernel<<<grid, 256, 0, st>>>(logits, ld, V, cand, n, rank);
}

// Vocab-sharded LM head: after the packed (value, id) keys of this pass were
// MAX-all-reduced across shards (or not, when merge == 0), store them per
// position and decode the global argmax; in decode mode also advance n0.
__global__ void shard_unpack_kernel(PassCtx* ctx, const unsigned long long* __restrict__ keys,
                                    unsigned long long* __restrict__ keys_pos, int* __restrict__ argmax_pos, int merge,
                                    int advance) {
  if (ctx->stop) return;
  const int rows = ctx->rows, n0 = ctx->n0;
  for (int t = threadIdx.x; t < rows; t += blockDim.x) {
    const unsigned long long k = keys[t];
    keys_pos[n0 + t] = k;
    if (merge) argmax_pos[n0 + t] = int(0xFFFFFFFFu - unsigned(k & 0xFFFFFFFFull));
  }
  __syncthreads();
  if (advance && threadIdx.x == 0) {
    ctx->n0 = n0 + 1;
    ctx->step += 1;
  }
}

void launch_shard_unpack(PassCtx* ctx, const unsigned long long* keys, unsigned long long* keys_pos, int* argmax_pos,
                         int merge, int advance, cudaStream_t st) {
  shard_unpack_kernel<<<1, 256, 0, st>>>(ctx, keys, keys_pos, argmax_pos, merge, advance);
}

__global__ void advance_kernel(PassCtx* ctx) {
  pdl_enter();
  if (!ctx->stop) { ctx->n0 += 1; ctx->step += 1; }
}

void launch_advance(PassCtx* ctx, cudaStream_t st) { launch_pdl(advance_kernel, dim3(1), dim3(1), 0, st, ctx); }

#define PS_INST(T)                                                                                       \
  template void launch_embed_norm<T>(const PassCtx*, int, const int*, int*, const int*, const T*, float*, \
                                     T*, int, float, cudaStream_t);                                     \
  template void launch_qkv_finalize<T>(const PassCtx*, int, const float*, int, int, const T*,           \
                                       const float2*, T*, T*, T*, const int*, KvGeom, int, int,          \
                                       cudaStream_t);                                                    \
  template void launch_attention<T>(const PassCtx*, int, int, const T*, const T*, const T*, const int*,  \
                                    KvGeom, int, int, float*, float*, T*, cudaStream_t);                 \
  template void launch_residual_norm<T>(const PassCtx*, int, float*, const float*, int, int, T*, T*, int, \
                                        float, cudaStream_t);                                            \
  template void launch_swiglu<T>(const PassCtx*, int, const float*, int, int, T*, int, cudaStream_t);
PS_INST(float)
PS_INST(__nv_bfloat16)

}  // namespace ps
