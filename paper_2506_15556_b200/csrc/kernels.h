// Kernel launchers of the predict-and-verify runtime. Every kernel that sits
// on a decode step reads its position/row count from a device PassCtx so the
// step can be captured once in a CUDA graph and replayed.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <cuda.h>

#include "common.cuh"

namespace ps {

uint64_t weight_key(uint64_t seed, uint32_t tid);
float weight_scale(double stddev);
template <typename T>
void launch_init_uniform(T* out, uint64_t count, uint64_t first, uint64_t seed, uint32_t tid, double stddev,
                         cudaStream_t st);

// Row permutations of the fused bf16 weight matrices.
//   kHeadPairs: within each head of `hd` rows, dims i and i+hd/2 (a RoPE
//               rotate-half pair) sit at rows 2i and 2i+1;
//   kGateUp:    gate feature j -> row 2j, up feature j -> row 2j+1
//               (`off` = 0 for gate, 1 for up), so a 128-row tile holds 64
//               complete SwiGLU pairs.
struct RowPerm {
  enum Kind : int { kIdentity = 0, kHeadPairs = 1, kGateUp = 2 };
  int kind = kIdentity;
  int hd = 0;       // kHeadPairs
  int off = 0;      // kGateUp
  int base = 0;     // destination row offset inside the fused matrix
  __host__ __device__ int dst(int r) const {
    if (kind == kHeadPairs) {
      const int h = r / hd, i = r % hd, half = hd / 2;
      return base + h * hd + (i < half ? 2 * i : 2 * (i - half) + 1);
    }
    if (kind == kGateUp) return base + 2 * r + off;
    return base + r;
  }
};
template <typename T>
void launch_init_rows_permuted(T* out, uint64_t rows, uint64_t cols, RowPerm perm, uint64_t seed, uint32_t tid,
                               double stddev, cudaStream_t st);

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

// 1-row passes: qkv_finalize + attention_page fused (CTA = kv head x page), then the combine
void launch_qkv_attention_decode(const PassCtx* ctx, int max_pos, const float* part, int splits, int N,
                                 const float* bias, const float2* rope, float* kpool, float* vpool,
                                 const int* page_table, KvGeom g, int layer, int heads, float* o_part,
                                 float* ml_part, float* attn_out, cudaStream_t st);

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
// rank of each candidate token in its row's logits (ties -> lower id first)
void launch_topk_rank(const float* logits, int ld, int V, const int* cand, int n, int* rank, cudaStream_t st);
void launch_verify_compare(const int* argmax_pos, int p0, const int* cand, int n_cand,
                           const unsigned char* term_mask, int* res, cudaStream_t st);

void launch_shard_unpack(PassCtx* ctx, const unsigned long long* keys, unsigned long long* keys_pos, int* argmax_pos,
                         int merge, int advance, cudaStream_t st);

// decode-step bookkeeping: advance n0 unless stopped.
void launch_advance(PassCtx* ctx, cudaStream_t st);

// ---- bf16 tensor maps (tma.cu) ----
struct TmaDesc {
  alignas(64) unsigned char bytes[128];
};
bool encode_tma_2d_bf16(TmaDesc* out, const void* base, uint64_t inner, uint64_t outer,
                        uint32_t box_inner, uint32_t box_outer);
bool encode_tma_2d_f32(TmaDesc* out, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                       uint32_t box_outer);
constexpr int kXBoxRows = 8;  // rows per residual-row box of the wide finalisation

constexpr int kTileTc = 128;

// ---- persistent megakernel (megakernel.cu): one cooperative launch per pass ----
struct MegaParams {
  PassCtx* ctx;
  int decode;               // 1: 1-row step, token = previous argmax
  int advance;              // decode: last LM CTA advances ctx->n0
  const int* tok_in;        // extend passes
  int L, H, qd, kvd, I, hd, heads, kv_heads, vocab_local, v_begin;
  int hd_shift;             // log2(hd): hd is 64 or 128 on the bf16 path
  int ntok, stages, acc_cols, max_splits_attn;
  float eps, attn_scale;
  const CUtensorMap* wmaps; // [4L + 1] device-resident tensor maps
  const CUtensorMap* xmaps; // [4] activation maps for this ntok: xb, attn, act, hn
  const CUtensorMap* xrows; // fp32 residual x [kMaxWindow][H], boxes of 128 features x kXBoxRows rows
  int* tokens_dev;
  int* argmax_pos;
  const __nv_bfloat16* embed;
  const __nv_bfloat16* qkv_bias;  // [L][qd+2kvd] or null
  const float2* rope;
  const float* lm_bias;
  float* x;
  __nv_bfloat16* xb;
  float* rstd0;
  float* ssq_part;
  __nv_bfloat16* q;
  __nv_bfloat16* kpool;
  __nv_bfloat16* vpool;
  const int* page_table;
  KvGeom g;
  __nv_bfloat16* attn;
  __nv_bfloat16* act;
  __nv_bfloat16* hn_cache;
  float* rstd_cache;
  float* o_part;
  float* ml_part;
  unsigned* acnt;
  float* part;              // [G][2][kMaxWindow][128] stream-K piece partials (wide passes)
  unsigned long long* tags; // [G][2][128] (tag, fp32) piece partials of 1-row passes
  unsigned* epoch;          // pass counter (partial tags), advanced by CTA 0 at the end of each pass
  unsigned* tile_cnt;       // [phase][max_tiles], zeroed before the pass
  int max_tiles;
  unsigned* lm_cnt;
  float* am_val;
  int* am_idx;
  unsigned long long* keys;
  unsigned* bar;            // grid barrier counter, zeroed before launch
  unsigned* bar2;           // wide passes: attention-merge sync counter (one arrival per CTA per layer)
  int lm_only;              // 1: LM head + argmax over resident rows [n0, n0+rows) only (hn / rstd caches)
  float* logits_out;        // optional fp32 logits [rows][ld_logits] from the LM epilogue
  // fused top-k verification (wide passes of <= kTopkRows rows): the LM epilogue
  // writes each (tile, row)'s best L = topk_list (value, id) in the (-score, id)
  // order of topk_tokens (lm.py:139-145); FINAL merges them per row and writes
  // rank_pos[n0 + t] = rank of tokens_dev[n0 + t + 1] in row t, or L when it
  // is not among the best L (the verifier's k: rank < k is all it asks)
  int topk_list;            // 0: off; else L (1..kTopkList)
  float* tk_val;            // [LM tiles][kTopkRows][kTopkList]
  int* tk_idx;
  int* rank_pos;            // [max_seq + kMaxWindow]
  int ld_logits;
  unsigned long long* trace;  // optional [nphases][G][12] globaltimer stamps
  int pre_max;              // weight stages issued ahead of a phase barrier (<= stages)
  int pf[8];                // per phase kind: weight boxes L2-prefetched ahead of the phase barrier
  int gcap[8];              // per phase kind: cap on the stream-K CTA count (0 = none; PS_SK_G)
};
// attention staging of the megakernel (see AttnSmem in megakernel.cu): decode
// passes one unit buffer of bf16 K, V [64][hd+8] and q [4 * grp][hd+8]
// wide passes: K and V only (q fragments are read from global memory); a
// buffer also holds the staged RMSNorm partials of up to kRstdStageRows rows
constexpr int kTopkList = 8;    // fused top-k: list length per (LM tile, row); k <= kTopkList
constexpr int kTopkRows = 160;  // fused top-k: pass widths whose LM tiles all use the vectorised epilogue
constexpr int kRstdStageRows = 80;
__host__ __device__ inline int mega_attn_buf_wide(int hd, int H) {
  const int kv = 2 * kPage * (hd + 8) * 2, rs = 4 * (H / 128) * kRstdStageRows * 4;
  return kv > rs ? kv : rs;
}
inline int mega_attn_bytes(int hd, int grp, bool wide, int H) {
  return wide ? 2 * mega_attn_buf_wide(hd, H) : (2 * kPage * (hd + 8) * 2 + 4 * grp * (hd + 8) * 2);
}
int mega_stages(int ntok, int attn_floats, bool wide);
int mega_smem_bytes(int ntok, int stages, int attn_floats);
// wide: the pass may have more than one row (max_rows > 1)
cudaError_t launch_mega(const MegaParams& P, bool wide, int grid, int smem, cudaStream_t st);
int mega_max_blocks_per_sm(int smem, bool wide);

}  // namespace ps
