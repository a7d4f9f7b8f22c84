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

void launch_shard_unpack(PassCtx* ctx, const unsigned long long* keys, unsigned long long* keys_pos, int* argmax_pos,
                         int merge, int advance, cudaStream_t st);

// decode-step bookkeeping: advance n0 unless stopped.
void launch_advance(PassCtx* ctx, cudaStream_t st);

// ---- bf16 tcgen05 path (gemm_tc.cu) ----
struct TmaDesc {
  alignas(64) unsigned char bytes[128];
};
bool encode_tma_2d_bf16(TmaDesc* out, const void* base, uint64_t inner, uint64_t outer,
                        uint32_t box_inner, uint32_t box_outer);
// Fused epilogues of the tcgen05 weight-streaming GEMM. Split-K partials
// are summed (in split order) by the last-arriving CTA of each 128-row tile,
// which then applies the epilogue for its rows:
//   QKV    * rstd + bias, RoPE, q -> q buffer, k/v -> paged KV
//   SWIGLU * rstd, act = silu(gate) * up   (gate/up rows interleaved per tile)
//   RESID  x += y; xb = bf16(x); per-tile sum of squares -> the grid's last
//          tile writes rstd per row (the next GEMM applies it: y = rstd*W.xb)
//   ARGMAX logits = rstd * (E.xb) + bias; per-tile (max, lowest id); the
//          grid's last tile reduces over tiles -> argmax_pos[n0+t]
enum TcMode : int { TC_EPI_QKV = 0, TC_EPI_SWIGLU = 1, TC_EPI_RESID = 2, TC_EPI_ARGMAX = 3 };
struct TcEpilogue {
  int mode = 0;
  float* part = nullptr;             // split-K partials [split][kMaxWindow][N]
  unsigned* tile_cnt = nullptr;      // per-tile arrival counters (self-resetting)
  unsigned* grid_cnt = nullptr;      // grid-wide arrival counter (RESID / ARGMAX)
  const float* rstd_in = nullptr;    // per-row rstd (QKV/SWIGLU: [t]; ARGMAX: [n0+t])
  // QKV
  const __nv_bfloat16* bias = nullptr;
  const float2* rope = nullptr;
  __nv_bfloat16* q = nullptr;
  __nv_bfloat16* kpool = nullptr;
  __nv_bfloat16* vpool = nullptr;
  const int* page_table = nullptr;
  KvGeom g{};
  int layer = 0, q_dim = 0, kv_dim = 0;
  // SWIGLU
  __nv_bfloat16* act = nullptr;
  int inter = 0;
  // RESID
  float* x = nullptr;
  __nv_bfloat16* xb_out = nullptr;
  int xb_out_pos = 0;                // 1: row index n0+t (hn_cache) instead of t
  float* ssq_part = nullptr;         // [tile][kMaxWindow]
  float* rstd_out = nullptr;
  int rstd_out_pos = 0;
  int hidden = 0;
  float eps = 0.f;
  // ARGMAX
  const float* lbias = nullptr;
  int v_begin = 0;
  float* am_val = nullptr;
  int* am_idx = nullptr;
  float* logits_out = nullptr;
  int ld_logits = 0;
  int* argmax_pos = nullptr;
  unsigned long long* packed_out = nullptr;
  int advance = 0;                   // decode step: last CTA advances ctx->n0
};
void launch_tc(PassCtx* ctx, const TmaDesc* tmW, const TmaDesc* tmX, int N, int K, int splits, int ntok,
               int x_row_from_ctx, const TcEpilogue& e, cudaStream_t st, bool pdl);

constexpr int kTileTc = 128;
int tc_gemm_smem_bytes(int ntok);

// ---- persistent megakernel (megakernel.cu): one cooperative launch per pass ----
struct MegaParams {
  PassCtx* ctx;
  int decode;               // 1: 1-row step, token = previous argmax
  int advance;              // decode: last LM CTA advances ctx->n0
  const int* tok_in;        // extend passes
  int L, H, qd, kvd, I, hd, heads, kv_heads, vocab_local, v_begin;
  int ntok, stages, acc_cols, max_splits_attn;
  float eps, attn_scale;
  const CUtensorMap* wmaps; // [4L + 1] device-resident tensor maps
  const CUtensorMap* xmaps; // [4] activation maps for this ntok: xb, attn, act, hn
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
  float* part;              // [G][2][kMaxWindow][128] stream-K piece partials (u64 tagged for <= 8 rows)
  unsigned* epoch;          // pass counter (partial tags), advanced by CTA 0 at the end of each pass
  unsigned* tile_cnt;       // [phase][max_tiles], zeroed before the pass
  int max_tiles;
  unsigned* lm_cnt;
  float* am_val;
  int* am_idx;
  unsigned long long* keys;
  unsigned* bar;            // grid barrier counter, zeroed before launch
  unsigned long long* trace;  // optional [nphases][G][12] globaltimer stamps
};
// attention staging of the megakernel (see AttnSmem in megakernel.cu): two
// unit buffers of bf16 K, V [64][hd+8] and q [4 * grp][hd+8]
inline int mega_attn_bytes(int hd, int grp) { return 2 * (2 * kPage * (hd + 8) * 2 + 4 * grp * (hd + 8) * 2); }
int mega_stages(int ntok, int attn_floats);
int mega_smem_bytes(int ntok, int stages, int attn_floats);
cudaError_t launch_mega(const MegaParams& P, int grid, int smem, cudaStream_t st);
int mega_max_blocks_per_sm(int smem);

}  // namespace ps
