// Kernel launchers of the predict-and-verify runtime. Every kernel that sits
// on a decode step reads its position/row count from a device PassCtx so the
// step can be captured once in a CUDA graph and replayed.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "common.cuh"

namespace ps {

uint64_t weight_key(uint64_t seed, uint32_t tid);
float weight_scale(double stddev);
template <typename T>
void launch_init_uniform(T* out, uint64_t count, uint64_t first, uint64_t seed, uint32_t tid, double stddev,
                         cudaStream_t st);

// Geometry of the paged KV pool: [layer][page][kv_head][kPage][head_dim] for K and for V.
struct KvGeom {
  int layers, kv_heads, head_dim, pages;
  __host__ __device__ size_t layer_stride() const { return size_t(pages) * kv_heads * kPage * head_dim; }
};

struct LayerDims {
  int hidden, heads, kv_heads, head_dim, inter;
  float eps;
};

template <typename T>
void launch_embed_norm(const PassCtx* ctx, int max_rows, const int* tok_in, int* tokens_dev,
                       const int* argmax_pos, const T* embed, float* x, T* xn, int hidden, float eps,
                       cudaStream_t st);

template <typename T>
void launch_qkv_finalize(const PassCtx* ctx, int max_rows, const float* part, int splits, int ldp,
                         const T* bias, const float2* rope, T* q, T* kpool, T* vpool,
                         const int* page_table, KvGeom g, int layer, int heads, cudaStream_t st);

template <typename T>
void launch_attention(const PassCtx* ctx, int max_rows, int max_pos, const T* q, const T* kpool,
                      const T* vpool, const int* page_table, KvGeom g, int layer, int heads,
                      float* o_part, float* ml_part, T* attn_out, cudaStream_t st);

template <typename T>
void launch_residual_norm(const PassCtx* ctx, int max_rows, float* x, const float* part, int splits,
                          int ldp, T* xn, T* hn_cache, int hidden, float eps, cudaStream_t st);

template <typename T>
void launch_swiglu(const PassCtx* ctx, int max_rows, const float* part, int splits, int ldp, T* act,
                   int inter, cudaStream_t st);

// fp32 SIMT split-K GEMM: part[s][t][n] = sum_{k in split s} X[t][k] * W[n][k]
void launch_gemm_f32(const PassCtx* ctx, int max_rows, const float* X, int ldx, const float* W,
                     float* part, int N, int K, int splits, cudaStream_t st);

// fp32 SIMT LM head with fused argmax partials over vocab tiles of 64 ids.
// hn rows start at absolute position ctx->n0 (+ pos_offset) of hn_cache.
void launch_lmhead_f32(const PassCtx* ctx, int max_rows, const float* hn_cache, int pos_offset,
                       const float* W, const float* bias, int v_begin, int v_count, int hidden,
                       float* am_val, int* am_idx, float* logits_out, int ld_logits, cudaStream_t st);
constexpr int kLmTileF32 = 64;

// Reduce per-tile argmax partials into argmax_pos[n0 + t] (+ optional packed key out).
void launch_argmax_reduce(const PassCtx* ctx, int max_rows, const float* am_val, const int* am_idx,
                          int tiles, int* argmax_pos, unsigned long long* packed_out,
                          cudaStream_t st);

// Greedy verify epilogue: k = first i with argmax_pos[p0-1+i] != cand[i];
// first terminator index in cand; writes {k, first_term} to res.
void launch_verify_compare(const int* argmax_pos, int p0, const int* cand, int n_cand,
                           const unsigned char* term_mask, int* res, cudaStream_t st);

// decode-step bookkeeping: advance n0 unless stopped.
void launch_advance(PassCtx* ctx, cudaStream_t st);

// ---- bf16 tcgen05 path (gemm_tc.cu) ----
struct TmaDesc {
  alignas(64) unsigned char bytes[128];
};
bool encode_tma_2d_bf16(TmaDesc* out, const void* base, uint64_t inner, uint64_t outer,
                        uint32_t box_inner, uint32_t box_outer);
// part[s][t][n] = sum X[t][k] W[n][k] over split s, tensor cores (tcgen05, TMEM accumulators)
void launch_gemm_tc(const PassCtx* ctx, const TmaDesc* tmW, const TmaDesc* tmX, float* part, int N,
                    int K, int splits, int ntok, int x_row_offset_from_ctx, cudaStream_t st);
void launch_lmhead_tc(const PassCtx* ctx, const TmaDesc* tmW, const TmaDesc* tmX, const float* bias,
                      int v_begin, int v_count, int hidden, int ntok, int pos_offset, float* am_val,
                      int* am_idx, float* logits_out, int ld_logits, cudaStream_t st);
constexpr int kTileTc = 128;
int tc_gemm_smem_bytes(int ntok);

}  // namespace ps
