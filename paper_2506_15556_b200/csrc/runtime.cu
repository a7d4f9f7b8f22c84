// C-ABI runtime (include/predgen_b200.h): weights, paged KV, passes, decode graph.
//
// Host control flow per call is deliberately thin: token ids in, argmax ids /
// accept length out, one stream, one synchronisation at the end of each call.
#include <cuda_runtime.h>

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "kernels.h"
#include "predgen_b200.h"

using namespace ps;

namespace {

// ---- NCCL, loaded at run time (no link dependency; the process's own
// libnccl — e.g. the one torch loaded — is preferred via PS_NCCL_LIB) ----
struct NcclApi {
  void* lib = nullptr;
  int (*get_unique_id)(void*) = nullptr;
  int (*comm_init_rank)(void**, int, const void* /*ncclUniqueId by value, 128 B*/, int) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  const char* (*error_string)(int) = nullptr;
};
struct NcclUniqueId {
  char internal[128];
};

NcclApi* nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api.lib ? &api : nullptr;
  tried = true;
  const char* cands[] = {std::getenv("PS_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
  for (const char* c : cands) {
    if (!c) continue;
    api.lib = dlopen(c, RTLD_NOW | RTLD_GLOBAL);
    if (api.lib) break;
  }
  if (!api.lib) return nullptr;
  api.get_unique_id = reinterpret_cast<int (*)(void*)>(dlsym(api.lib, "ncclGetUniqueId"));
  api.all_reduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(
      dlsym(api.lib, "ncclAllReduce"));
  api.comm_destroy = reinterpret_cast<int (*)(void*)>(dlsym(api.lib, "ncclCommDestroy"));
  api.error_string = reinterpret_cast<const char* (*)(int)>(dlsym(api.lib, "ncclGetErrorString"));
  if (!api.get_unique_id || !api.all_reduce || !api.comm_destroy || !dlsym(api.lib, "ncclCommInitRank")) {
    api.lib = nullptr;
    return nullptr;
  }
  return &api;
}

// ncclCommInitRank takes ncclUniqueId by value: call through a typed pointer
int nccl_comm_init(NcclApi* api, void** comm, int world, const NcclUniqueId& id, int rank) {
  auto fn = reinterpret_cast<int (*)(void**, int, NcclUniqueId, int)>(dlsym(api->lib, "ncclCommInitRank"));
  return fn(comm, world, id, rank);
}
constexpr int kNcclUint64 = 5, kNcclMax = 2;

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(expr)                                                                               \
  do {                                                                                         \
    cudaError_t e_ = (expr);                                                                   \
    if (e_ != cudaSuccess) return fail(PS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// weight tensor ids (oracle/weights.py)
constexpr int TID_EMBED = 1, TID_HEAD = 2;
constexpr int WQ = 0, WK = 1, WV = 2, WO = 3, WGATE = 4, WUP = 5, WDOWN = 6, BQ = 7, BK = 8, BV = 9;
int layer_tid(int l, int w) { return 64 + 16 * l + w; }

struct Gemm {
  void* w = nullptr;
  int N = 0, K = 0, splits = 1;
  TmaDesc tm;
};

struct Layer {
  Gemm qkv, o, gu, d;
  void* bqkv = nullptr;
};

struct ActDescs {
  TmaDesc xn, attn, act, hn;
};

struct WEntry {
  int tid;
  void* ptr;
  int64_t count;
  int64_t cols = 0;
  RowPerm perm{};           // storage row of source row r = perm.dst(r) (bf16 fused matrices)
};

constexpr int kCtxSlots = 64;
constexpr int kMaxSteps = 256;
constexpr int kProfClasses = 8;

int round_up(int a, int b) { return (a + b - 1) / b * b; }

int choose_splits(int N, int K, int tile_n, int kgran, int max_ksplit) {
  const int tiles = N / tile_n;
  int s = 1;
  while (tiles * s < 2 * 148 && K % (2 * s * kgran) == 0 && K / (2 * s) >= 512) s *= 2;
  while (max_ksplit > 0 && K / s > max_ksplit && K % (2 * s * kgran) == 0) s *= 2;
  return s;
}

// tcgen05 path: split-K so the grid fills the 148 SMs (2 CTAs each) in one
// balanced wave; splits need not divide K (uneven k-block ranges are fixed by
// (N, K) alone, so results stay independent of the pass width).
int choose_splits_tc(int N, int K) {
  // measured on B200 (tools/sweep_splits.py): one wave of <= 2 CTAs per SM;
  // wide GEMMs (>= 148 tiles) run unsplit — their partial reduction costs more
  // than the imbalance it removes.
  const int tiles = (N + kTileTc - 1) / kTileTc, kb = K / 64;
  if (tiles >= 148) return 1;
  int s = std::min(16, (2 * 148) / tiles);
  while (s > 1 && kb / s < 4) --s;
  return std::max(1, s);
}

}  // namespace

struct Prof {
  cudaEvent_t ev[2 * 40 * 12 + 8];
  int n = 0;
  int cls[2 * 40 * 12 + 8];
};

struct ps_handle {
  ps_config cfg{};
  bool bf16 = false;
  size_t esz = 4;
  cudaStream_t st = nullptr;
  std::vector<void*> allocs;
  std::vector<void*> host_allocs;

  int H = 0, V = 0, L = 0, nh = 0, nkv = 0, hd = 0, I = 0, qd = 0, kvd = 0;
  int v_begin = 0, v_count = 0;

  void* embed = nullptr;
  void* head = nullptr;
  float* lm_bias = nullptr;
  std::vector<Layer> layers;
  TmaDesc tm_head;
  std::vector<WEntry> wreg;
  double weight_bytes = 0;

  void* kpool = nullptr;
  void* vpool = nullptr;
  KvGeom g{};
  int* d_page_table = nullptr;
  int* h_page_table = nullptr;  // pinned
  std::vector<int> free_pages;
  int pages_mapped = 0;

  float* x = nullptr;
  void* xn = nullptr;
  void* q = nullptr;
  void* attn = nullptr;
  void* act = nullptr;
  float* part = nullptr;
  float* o_part = nullptr;
  float* ml_part = nullptr;
  void* hn_cache = nullptr;
  float* am_val = nullptr;
  int* am_idx = nullptr;
  int am_tiles = 0;
  int* argmax_pos = nullptr;
  int* tokens_dev = nullptr;
  unsigned char* term_mask = nullptr;
  float2* rope = nullptr;
  int* d_tok = nullptr;
  int* d_cand = nullptr;
  int* d_res = nullptr;
  PassCtx* d_ctx = nullptr;
  PassCtx* d_ctx_aux = nullptr;
  float* logits_buf = nullptr;  // [kMaxWindow][v_count] fp32 logits (parity rows, top-k ranks)
  // top-k verify: the pass itself writes its rows' logits into logits_buf (no
  // LM-head re-run); cap_n0 / cap_rows = the positions the last chunk covered
  bool capture_logits = false;
  int cap_n0 = -1, cap_rows = 0;
  // fused top-k (bf16): wide passes of 2..tk_rows_max rows keep per-(LM tile,
  // row) best-kTopkList lists instead of logits; tk_n0 / tk_rows = the positions
  // whose ranks the last such pass wrote into rank_pos
  bool topk_fused = false;
  int topk_k = 0;  // list length of fused top-k passes (the verifier's k <= kTopkList)
  int tk_rows_max = 0, tk_n0 = -1, tk_rows = 0;
  float* tk_val = nullptr;
  int* tk_idx = nullptr;
  int* rank_pos = nullptr;
  // bf16 chain state
  float* rstd = nullptr;        // [kMaxWindow] rstd of the current residual rows
  float* rstd_cache = nullptr;  // [seq_rows] rstd of the final hidden per position
  float* ssq_part = nullptr;    // [H/128][kMaxWindow]
  unsigned* counters = nullptr; // self-resetting arrival counters
  unsigned* acnt = nullptr;     // attention page-merge counters [kMaxWindow][kv_heads]
  // megakernel
  bool mega = true;
  int sms = 148;
  CUtensorMap* d_wmaps = nullptr;           // [4L+1]
  CUtensorMap* d_xmaps = nullptr;           // [ntok/16][4]
  std::vector<int> xmaps_ready;             // per ntok/16
  __nv_bfloat16* qkv_bias_all = nullptr;
  float* mega_part = nullptr;
  unsigned long long* mega_tags = nullptr;  // [sms][2][128] tagged decode partials
  unsigned* mega_cnt = nullptr;             // [0]=bar, [1]=lm_cnt, [2]=bar2, [64..] per-phase tile counters
  int mega_max_tiles = 0;
  size_t mega_cnt_words = 0;
  unsigned* mega_epoch = nullptr;
  unsigned long long* mega_trace = nullptr;  // PS_TRACE=1: per-phase globaltimer stamps
  // vocab sharding (c4)
  unsigned long long* keys = nullptr;      // [kMaxWindow] packed (value, id) of this pass
  unsigned long long* keys_pos = nullptr;  // [seq_rows] per position
  void* nccl_comm = nullptr;

  PassCtx* h_ctx = nullptr;   // pinned ring [kCtxSlots]
  int* h_tok = nullptr;       // pinned ring [kCtxSlots][kMaxWindow]
  int* h_res = nullptr;       // pinned [4 + kMaxWindow]
  int* h_argmax = nullptr;    // pinned [max_seq + kMaxWindow]
  int* h_steps_tok = nullptr; // pinned [kMaxSteps]
  int ring = 0;

  std::vector<int> resident;
  std::vector<int> argmax_host;

  std::map<int, ActDescs> act_tm;
  cudaGraphExec_t graph = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<cudaEvent_t> step_ev;
  ps_stats stats{};
  Prof* prof = nullptr;
  bool prof_on = false;

  template <typename T>
  T* dalloc(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, n * sizeof(T) + 256) != cudaSuccess) return nullptr;
    // stream-ordered with the init kernels (a legacy-stream memset would race
    // them: the runtime stream is non-blocking)
    cudaMemsetAsync(p, 0, n * sizeof(T) + 256, st);
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
  template <typename T>
  T* halloc(size_t n) {
    void* p = nullptr;
    if (cudaMallocHost(&p, n * sizeof(T)) != cudaSuccess) return nullptr;
    std::memset(p, 0, n * sizeof(T));
    host_allocs.push_back(p);
    return static_cast<T*>(p);
  }
};

namespace {

void* alloc_weights(ps_handle* h, size_t count) {
  return h->bf16 ? static_cast<void*>(h->dalloc<__nv_bfloat16>(count)) : static_cast<void*>(h->dalloc<float>(count));
}

void init_tensor(ps_handle* h, void* dst, uint64_t count, uint64_t first, int tid, bool registry = true) {
  if (h->bf16)
    launch_init_uniform(static_cast<__nv_bfloat16*>(dst), count, first, h->cfg.seed, tid, 0.02, h->st);
  else
    launch_init_uniform(static_cast<float*>(dst), count, first, h->cfg.seed, tid, 0.02, h->st);
  if (registry) h->wreg.push_back({tid, dst, int64_t(count)});
}

void* offset_ptr(ps_handle* h, void* base, size_t elems) {
  return static_cast<unsigned char*>(base) + elems * h->esz;
}

// A blocking copy ordered with the runtime stream. (A plain cudaMemcpy runs on
// the legacy stream, which does not order with the non-blocking runtime
// stream: e.g. the LM-bias upload in ps_create could land BEFORE the
// stream-ordered zero-fill of its allocation, which then wiped it.)
cudaError_t copy_sync(ps_handle* h, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, h->st);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(h->st);
}

cudaError_t copy_async(ps_handle* h, void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
  if (kind == cudaMemcpyHostToDevice) h->stats.h2d_bytes += int64_t(bytes);
  if (kind == cudaMemcpyDeviceToHost) h->stats.d2h_bytes += int64_t(bytes);
  return cudaMemcpyAsync(dst, src, bytes, kind, h->st);
}

int map_pages(ps_handle* h, int n_tokens) {
  const int need = (n_tokens + kPage - 1) / kPage;
  if (need > h->g.pages) return fail(PS_ERR_CAPACITY, "context exceeds KV capacity (max_seq)");
  const int first_new = h->pages_mapped;
  while (h->pages_mapped < need) {
    const int phys = h->free_pages.back();
    h->free_pages.pop_back();
    h->h_page_table[h->pages_mapped++] = phys;
  }
  if (need > first_new) {
    CK(copy_async(h, h->d_page_table + first_new, h->h_page_table + first_new, sizeof(int) * (need - first_new),
                  cudaMemcpyHostToDevice));
  }
  h->stats.kv_pages_used = h->pages_mapped;
  return PS_OK;
}

void truncate_to(ps_handle* h, int n) {
  if (n >= int(h->resident.size())) return;
  h->stats.rollbacks += 1;
  h->resident.resize(n);
  h->argmax_host.resize(n);
  const int keep = (n + kPage - 1) / kPage;
  while (h->pages_mapped > keep) h->free_pages.push_back(h->h_page_table[--h->pages_mapped]);
  h->stats.kv_tokens = n;
  h->stats.kv_pages_used = h->pages_mapped;
}

const ActDescs* act_descs(ps_handle* h, int ntok) {
  auto it = h->act_tm.find(ntok);
  if (it != h->act_tm.end()) return &it->second;
  ActDescs d;
  bool ok = encode_tma_2d_bf16(&d.xn, h->xn, h->H, kMaxWindow, 64, ntok);
  ok = ok && encode_tma_2d_bf16(&d.attn, h->attn, h->qd, kMaxWindow, 64, ntok);
  ok = ok && encode_tma_2d_bf16(&d.act, h->act, h->I, kMaxWindow, 64, ntok);
  ok = ok && encode_tma_2d_bf16(&d.hn, h->hn_cache, h->H, h->cfg.max_seq + kMaxWindow, 64, ntok);
  if (!ok) return nullptr;
  return &h->act_tm.emplace(ntok, d).first->second;
}

void prof_mark(ps_handle* h, int cls) {
  Prof* p = h->prof;
  if (!p || !h->prof_on) return;
  cudaEventRecord(p->ev[p->n], h->st);
  p->cls[p->n] = cls;
  p->n++;
}

void enqueue_shard_merge(ps_handle* h, PassCtx* ctx, int max_rows, bool decode);

// Passes produce packed (max, lowest id) keys and join them across shards when
// the LM head is vocab-sharded, or when a communicator is attached to a
// one-shard instance (a 1-rank NCCL world: the whole join path on one GPU).
bool keyed(const ps_handle* h) { return h->cfg.vocab_shards > 1 || h->nccl_comm != nullptr; }

// One forward pass of the decoder body + LM head + argmax over `max_rows`
// rows at ctx->n0 (device-side). tok_in == nullptr selects decode mode.
template <typename T>
void enqueue_pass_simt(ps_handle* h, PassCtx* ctx, int max_rows, const int* tok_in, int max_pos) {
  cudaStream_t st = h->st;
  const int ntok = round_up(std::max(max_rows, 1), 16);
  const ActDescs* ad = nullptr;
  T* xn = static_cast<T*>(h->xn);
  T* qb = static_cast<T*>(h->q);
  T* attn = static_cast<T*>(h->attn);
  T* act = static_cast<T*>(h->act);
  T* hn = static_cast<T*>(h->hn_cache);
  (void)ntok;
  auto gemm = [&](const Gemm& gm, const void* X, const TmaDesc* tmx) {
    (void)tmx;
    launch_gemm_f32(ctx, max_rows, static_cast<const float*>(X), gm.K, static_cast<const float*>(gm.w), h->part,
                    gm.N, gm.K, gm.splits, st);
  };
  prof_mark(h, 0);
  launch_embed_norm<T>(ctx, max_rows, tok_in, h->tokens_dev, h->argmax_pos, static_cast<const T*>(h->embed), h->x, xn,
                       h->H, h->cfg.rms_eps, st);
  for (int l = 0; l < h->L; ++l) {
    const Layer& ly = h->layers[l];
    prof_mark(h, 1);
    gemm(ly.qkv, xn, ad ? &ad->xn : nullptr);
    prof_mark(h, 7);
    if (max_rows <= 1) {  // decode step: finalize + page attention in one kernel
      launch_qkv_attention_decode(ctx, max_pos, h->part, ly.qkv.splits, ly.qkv.N, static_cast<const float*>(ly.bqkv),
                                  h->rope, static_cast<float*>(h->kpool), static_cast<float*>(h->vpool),
                                  h->d_page_table, h->g, l, h->nh, h->o_part, h->ml_part,
                                  reinterpret_cast<float*>(attn), st);
    } else {
      launch_qkv_finalize<T>(ctx, max_rows, h->part, ly.qkv.splits, ly.qkv.N, static_cast<const T*>(ly.bqkv), h->rope,
                             qb, static_cast<T*>(h->kpool), static_cast<T*>(h->vpool), h->d_page_table, h->g, l,
                             h->nh, st);
      prof_mark(h, 2);
      launch_attention<T>(ctx, max_rows, max_pos, qb, static_cast<const T*>(h->kpool),
                          static_cast<const T*>(h->vpool), h->d_page_table, h->g, l, h->nh, h->o_part, h->ml_part,
                          attn, st);
    }
    prof_mark(h, 3);
    gemm(ly.o, attn, ad ? &ad->attn : nullptr);
    prof_mark(h, 0);
    launch_residual_norm<T>(ctx, max_rows, h->x, h->part, ly.o.splits, h->H, xn, nullptr, h->H, h->cfg.rms_eps, st);
    prof_mark(h, 4);
    gemm(ly.gu, xn, ad ? &ad->xn : nullptr);
    // (measured slower and not kept: the SwiGLU fused into the decode down
    // GEMV's staging, recomputed by each of its 448 CTAs, 0.99 -> 1.10 ms per
    // c2 decode step; the attention page combine fused into the page kernel as
    // a last-arrival merge, 1.007 -> 1.041 ms)
    prof_mark(h, 7);
    launch_swiglu<T>(ctx, max_rows, h->part, ly.gu.splits, ly.gu.N, act, h->I, st);
    prof_mark(h, 5);
    gemm(ly.d, act, ad ? &ad->act : nullptr);
    prof_mark(h, 0);
    launch_residual_norm<T>(ctx, max_rows, h->x, h->part, ly.d.splits, h->H, xn, l == h->L - 1 ? hn : nullptr, h->H,
                            h->cfg.rms_eps, st);
  }
  prof_mark(h, 6);
  launch_lmhead_f32(ctx, max_rows, static_cast<const float*>(h->hn_cache), 0, static_cast<const float*>(h->head),
                      h->lm_bias, h->v_begin, h->v_count, h->H, h->am_val, h->am_idx,
                      h->capture_logits ? h->logits_buf : nullptr, h->capture_logits ? h->v_count : 0, st);
  const bool sharded = keyed(h);
  launch_argmax_reduce(ctx, max_rows, h->am_val, h->am_idx, h->am_tiles, h->argmax_pos, sharded ? h->keys : nullptr,
                       st);
  if (sharded) enqueue_shard_merge(h, ctx, max_rows, false);
  prof_mark(h, 7);
}

int launches_per_pass(const ps_handle* h, int max_rows) {
  if (h->mega) return 1 + (keyed(h) ? 1 : 0);
  // embed; per layer QKV, finalize, attention, combine, O, norm, GU, SwiGLU, D, norm; LM head, argmax
  // (1-row passes: finalize + attention are one kernel)
  return 1 + (max_rows <= 1 ? 9 : 10) * h->L + 2;
}


// (max, lowest id) across vocab shards: uint64 MAX all-reduce of the packed
// keys over NCCL (one message of 8 B per row), then decode the global id.
void enqueue_shard_merge(ps_handle* h, PassCtx* ctx, int max_rows, bool decode) {
  if (h->nccl_comm) {
    NcclApi* api = nccl_api();
    api->all_reduce(h->keys, h->keys, size_t(max_rows), kNcclUint64, kNcclMax, h->nccl_comm, h->st);
  }
  launch_shard_unpack(ctx, h->keys, h->keys_pos, h->argmax_pos, h->nccl_comm ? 1 : 0, decode ? 1 : 0, h->st);
}

// bf16 pass as ONE persistent cooperative kernel (megakernel.cu). lm_only:
// LM head + argmax over resident rows [ctx->n0, +rows) from the per-position
// hn / rstd caches (logits_out, if given, receives the fp32 logits).
void enqueue_mega(ps_handle* h, PassCtx* ctx, int max_rows, const int* tok_in, bool decode, bool lm_only = false,
                  float* logits_out = nullptr) {
  using bf = __nv_bfloat16;
  const int ntok = round_up(std::max(max_rows, 1), 16);
  const int grp = h->nh / h->nkv;
  const int attn_floats = mega_attn_bytes(h->hd, grp, max_rows > 1, h->H) / 4;
  MegaParams P{};
  P.ctx = ctx;
  P.decode = decode ? 1 : 0;
  const bool sharded = keyed(h);
  P.advance = (decode && !sharded) ? 1 : 0;
  P.tok_in = tok_in;
  P.L = h->L; P.H = h->H; P.qd = h->qd; P.kvd = h->kvd; P.I = h->I; P.hd = h->hd;
  P.heads = h->nh; P.kv_heads = h->nkv; P.vocab_local = h->v_count; P.v_begin = h->v_begin;
  P.hd_shift = h->hd == 128 ? 7 : 6;
  P.ntok = ntok;
  P.stages = mega_stages(ntok, attn_floats, max_rows > 1);
  {
    // ring depth caps, PS_MAX_STAGES="decode:wide" overrides. Decode measured
    // 7/8/9/10 stages = 2.813/2.803/2.794/2.804 ms (same box); wide takes all
    // the smem allows (5 at 72 rows)
    static int cap_dec = -1, cap_wide = -1;
    if (cap_dec < 0) {
      cap_dec = 9;
      cap_wide = 64;
      if (const char* e = std::getenv("PS_MAX_STAGES")) std::sscanf(e, "%d:%d", &cap_dec, &cap_wide);
    }
    P.stages = std::min(P.stages, max_rows > 1 ? cap_wide : cap_dec);
  }
  int cols = 32;
  while (cols < ntok) cols <<= 1;
  P.acc_cols = cols;
  P.max_splits_attn = h->cfg.max_seq / kPage + 1;
  P.eps = h->cfg.rms_eps;
  P.attn_scale = float(1.0 / std::sqrt(double(h->hd)));
  P.wmaps = h->d_wmaps;
  P.xmaps = h->d_xmaps + size_t(ntok / 16 - 1) * 4;
  P.xrows = h->d_xmaps + size_t(kMaxWindow / 16) * 4;
  P.tokens_dev = h->tokens_dev;
  P.argmax_pos = h->argmax_pos;
  P.embed = static_cast<const bf*>(h->embed);
  P.qkv_bias = h->qkv_bias_all;
  P.rope = h->rope;
  P.lm_bias = h->lm_bias;
  P.x = h->x;
  P.xb = static_cast<bf*>(h->xn);
  P.rstd0 = h->rstd;
  P.ssq_part = h->ssq_part;
  P.q = static_cast<bf*>(h->q);
  P.kpool = static_cast<bf*>(h->kpool);
  P.vpool = static_cast<bf*>(h->vpool);
  P.page_table = h->d_page_table;
  P.g = h->g;
  P.attn = static_cast<bf*>(h->attn);
  P.act = static_cast<bf*>(h->act);
  P.hn_cache = static_cast<bf*>(h->hn_cache);
  P.rstd_cache = h->rstd_cache;
  P.o_part = h->o_part;
  P.ml_part = h->ml_part;
  P.acnt = h->acnt;
  P.part = h->mega_part;
  P.tags = h->mega_tags;
  P.epoch = h->mega_epoch;
  P.tile_cnt = h->mega_cnt + 64;
  P.max_tiles = h->mega_max_tiles;
  P.lm_cnt = h->mega_cnt + 1;
  P.am_val = h->am_val;
  P.am_idx = h->am_idx;
  P.keys = (sharded && !lm_only) ? h->keys : nullptr;
  P.bar = h->mega_cnt;
  P.bar2 = h->mega_cnt + 2;
  P.lm_only = lm_only ? 1 : 0;
  const bool tk = h->topk_fused && max_rows >= 2 && max_rows <= h->tk_rows_max && h->cfg.vocab_shards == 1;
  P.logits_out = (logits_out == nullptr && h->capture_logits && !lm_only && !tk) ? h->logits_buf : logits_out;
  P.ld_logits = h->v_count;
  P.topk_list = tk ? h->topk_k : 0;
  P.tk_val = h->tk_val;
  P.tk_idx = h->tk_idx;
  P.rank_pos = h->rank_pos;
  if (tk) {
    h->tk_n0 = -2;  // set by the caller (the pass's first position is device-side)
    h->tk_rows = max_rows;
  }
  P.trace = h->mega_trace;
  {
    // L2 prefetch depth (weight boxes per CTA beyond the smem ring) for the
    // phases QKV, O, GU, D, LM; PS_PF_DECODE / PS_PF_WIDE="q:o:gu:d:lm" override
    static int pf_dec[5] = {0, 0, 0, 0, 0}, pf_wide[5] = {0, 0, 0, 0, 0};
    static bool pf_init = false;
    if (!pf_init) {
      if (const char* e = std::getenv("PS_PF_DECODE"))
        std::sscanf(e, "%d:%d:%d:%d:%d", &pf_dec[0], &pf_dec[1], &pf_dec[2], &pf_dec[3], &pf_dec[4]);
      if (const char* e = std::getenv("PS_PF_WIDE"))
        std::sscanf(e, "%d:%d:%d:%d:%d", &pf_wide[0], &pf_wide[1], &pf_wide[2], &pf_wide[3], &pf_wide[4]);
      pf_init = true;
    }
    const int* pf = max_rows > 1 ? pf_wide : pf_dec;
    static int pre_dec = 8, pre_wide = 8;
    static bool pre_init = false;
    if (!pre_init) {
      if (const char* e = std::getenv("PS_PRE")) std::sscanf(e, "%d:%d", &pre_dec, &pre_wide);
      pre_init = true;
    }
    P.pre_max = max_rows > 1 ? pre_wide : pre_dec;
    // stream-K CTA caps "q:o:gu:d:lm" (identical for decode and wide passes, so
    // the per-row arithmetic stays pass-width independent)
    static int gcap[5] = {0, 0, 0, 0, 0};
    static bool gcap_init = false;
    if (!gcap_init) {
      if (const char* e = std::getenv("PS_SK_G"))
        std::sscanf(e, "%d:%d:%d:%d:%d", &gcap[0], &gcap[1], &gcap[2], &gcap[3], &gcap[4]);
      gcap_init = true;
    }
    for (int k = 0; k < 5; ++k) P.gcap[1 + (k == 0 ? 0 : k + 1)] = gcap[k];
    for (int k = 0; k < 5; ++k) P.pf[1 + (k == 0 ? 0 : k + 1)] = pf[k];  // kinds QKV=1, O=3, GU=4, D=5, LM=6
  }
  // 1-row passes use only the barrier words (the per-phase tile counters
  // serve the wide finalisation)
  cudaMemsetAsync(h->mega_cnt, 0, sizeof(unsigned) * (max_rows > 1 ? h->mega_cnt_words : 64), h->st);
  prof_mark(h, 7);
  const cudaError_t e = launch_mega(P, max_rows > 1, h->sms, mega_smem_bytes(ntok, P.stages, attn_floats), h->st);
  if (e != cudaSuccess) std::fprintf(stderr, "predgen_b200: megakernel launch failed: %s\n", cudaGetErrorString(e));
  if (sharded && !lm_only) enqueue_shard_merge(h, ctx, max_rows, decode);
  prof_mark(h, 6);
}

void enqueue_pass_bf16(ps_handle* h, PassCtx* ctx, int max_rows, const int* tok_in, int max_pos, bool decode) {
  (void)max_pos;
  enqueue_mega(h, ctx, max_rows, tok_in, decode);
}

// decode == true: 1-row step whose token is the previous row's argmax; the
// step advances ctx->n0 on the device (bf16: inside the LM-head kernel).
void enqueue_pass_any(ps_handle* h, PassCtx* ctx, int max_rows, const int* tok_in, int max_pos, bool decode = false) {
  h->stats.launches += launches_per_pass(h, max_rows) + (decode && !h->bf16 ? 1 : 0);
  if (h->bf16) {
    enqueue_pass_bf16(h, ctx, max_rows, tok_in, max_pos, decode);
  } else {
    enqueue_pass_simt<float>(h, ctx, max_rows, tok_in, max_pos);
    if (decode) launch_advance(ctx, h->st);
  }
}

PassCtx* next_ctx_slot(ps_handle* h, int* slot) {
  *slot = h->ring;
  h->ring = (h->ring + 1) % kCtxSlots;
  return h->h_ctx + *slot;
}

// Append tokens[0..n) to the resident sequence: chunks of <= kMaxWindow rows.
// Enqueue only; the caller synchronises and then calls finish_extend.
int enqueue_extend(ps_handle* h, const int* tokens, int n, int* base_out) {
  const int base = int(h->resident.size());
  *base_out = base;
  if (base + n > h->cfg.max_seq) return fail(PS_ERR_CAPACITY, "context exceeds KV capacity (max_seq)");
  if (int rc = map_pages(h, base + n)) return rc;
  for (int done = 0; done < n;) {
    const int rows = std::min(kMaxWindow, n - done);
    int slot;
    PassCtx* hc = next_ctx_slot(h, &slot);
    *hc = PassCtx{base + done, rows, 0, 0, 0, {0, 0, 0}};
    int* ht = h->h_tok + size_t(slot) * kMaxWindow;
    std::memcpy(ht, tokens + done, sizeof(int) * rows);
    CK(copy_async(h, h->d_ctx, hc, sizeof(PassCtx), cudaMemcpyHostToDevice));
    CK(copy_async(h, h->d_tok, ht, sizeof(int) * rows, cudaMemcpyHostToDevice));
    enqueue_pass_any(h, h->d_ctx, rows, h->d_tok, base + done + rows - 1);
    CK(cudaGetLastError());
    if (h->capture_logits) {
      h->cap_n0 = base + done;
      h->cap_rows = rows;
    }
    if (h->tk_n0 == -2) h->tk_n0 = base + done;  // this pass wrote fused top-k ranks
    h->stats.passes += 1;
    h->stats.rows += rows;
    done += rows;
  }
  CK(copy_async(h, h->h_argmax + base, h->argmax_pos + base, sizeof(int) * n, cudaMemcpyDeviceToHost));
  return PS_OK;
}

void finish_extend(ps_handle* h, const int* tokens, int n, int base) {
  h->resident.insert(h->resident.end(), tokens, tokens + n);
  h->argmax_host.insert(h->argmax_host.end(), h->h_argmax + base, h->h_argmax + base + n);
  h->stats.kv_tokens = int64_t(h->resident.size());
}

int lcp_with(const ps_handle* h, const int* tokens, int n) {
  const int m = std::min(n, int(h->resident.size()));
  int i = 0;
  while (i < m && h->resident[i] == tokens[i]) ++i;
  return i;
}

// Bring the resident sequence to exactly tokens[0..n) (rollback + extend).
// Leaves the stream unsynchronised when *enqueued is set.
// A context that is a prefix of the resident sequence costs nothing; the
// longer resident tail is kept unless `exact` (decode must append at n).
int sync_to(ps_handle* h, const int* tokens, int n, int* computed, int* base, bool* enqueued, bool exact) {
  const int lcp = lcp_with(h, tokens, n);
  *enqueued = false;
  *computed = 0;
  if (lcp == n) {
    if (exact) truncate_to(h, n);
    h->stats.prefix_hits += 1;
    return PS_OK;
  }
  truncate_to(h, lcp);
  if (int rc = enqueue_extend(h, tokens + lcp, n - lcp, base)) return rc;
  *computed = n - lcp;
  *enqueued = true;
  return PS_OK;
}

int capture_decode_graph(ps_handle* h) {
  if (h->graph) return PS_OK;
  CK(cudaStreamBeginCapture(h->st, cudaStreamCaptureModeThreadLocal));
  enqueue_pass_any(h, h->d_ctx, 1, nullptr, h->cfg.max_seq - 1, true);
  h->stats.launches -= launches_per_pass(h, 1) + (h->bf16 ? 0 : 1);  // capture is not a launch (fp32: + advance); replays are counted
  cudaGraph_t graph = nullptr;
  cudaError_t e = cudaStreamEndCapture(h->st, &graph);
  if (e != cudaSuccess) return fail(PS_ERR_CUDA, std::string("decode graph capture: ") + cudaGetErrorString(e));
  e = cudaGraphInstantiate(&h->graph, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return fail(PS_ERR_CUDA, std::string("decode graph instantiate: ") + cudaGetErrorString(e));
  return PS_OK;
}

// `steps` 1-row decode steps starting at position n0 (device-chained).
int run_decode_steps(ps_handle* h, int n0, int steps, int stop_at_eos, int* executed, float* step_ms) {
  if (n0 + steps > h->cfg.max_seq) return fail(PS_ERR_CAPACITY, "decode exceeds KV capacity (max_seq)");
  if (int rc = map_pages(h, n0 + steps)) return rc;
  int slot;
  PassCtx* hc = next_ctx_slot(h, &slot);
  *hc = PassCtx{n0, 1, 0, stop_at_eos, 0, {0, 0, 0}};
  CK(copy_async(h, h->d_ctx, hc, sizeof(PassCtx), cudaMemcpyHostToDevice));
  if (h->cfg.use_graphs) {
    if (int rc = capture_decode_graph(h)) return rc;
  }
  while (int(h->step_ev.size()) < steps + 1) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    h->step_ev.push_back(e);
  }
  CK(cudaEventRecord(h->step_ev[0], h->st));
  for (int i = 0; i < steps; ++i) {
    if (h->graph) {
      CK(cudaGraphLaunch(h->graph, h->st));
      h->stats.launches += launches_per_pass(h, 1) + (h->bf16 ? 0 : 1);
    } else {
      enqueue_pass_any(h, h->d_ctx, 1, nullptr, n0 + steps - 1, true);
    }
    CK(cudaEventRecord(h->step_ev[i + 1], h->st));
  }
  int s2;
  PassCtx* back = next_ctx_slot(h, &s2);
  CK(copy_async(h, back, h->d_ctx, sizeof(PassCtx), cudaMemcpyDeviceToHost));
  CK(copy_async(h, h->h_argmax + n0, h->argmax_pos + n0, sizeof(int) * steps, cudaMemcpyDeviceToHost));
  CK(copy_async(h, h->h_steps_tok, h->tokens_dev + n0, sizeof(int) * steps, cudaMemcpyDeviceToHost));
  CK(cudaStreamSynchronize(h->st));
  CK(cudaGetLastError());
  *executed = back->step;
  for (int i = 0; i < steps; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->step_ev[i], h->step_ev[i + 1]);
    if (step_ms) step_ms[i] = ms;
    h->stats.gpu_ms += ms;
  }
  h->stats.decode_steps += *executed;
  h->stats.passes += *executed;
  h->stats.rows += *executed;
  return PS_OK;
}

}  // namespace

extern "C" {

const char* ps_last_error(void) { return g_err.c_str(); }

int ps_create(const ps_config* cfg, ps_handle** out) {
  if (!cfg || !out) return fail(PS_ERR_INVALID, "null argument");
  *out = nullptr;
  const ps_config& c = *cfg;
  if (c.vocab <= 4 || c.hidden % 128 || c.head_dim % 64 || c.heads % c.kv_heads || c.intermediate % 128 ||
      c.layers <= 0 || (c.mode != PS_MODE_F32 && c.mode != PS_MODE_BF16) || c.max_seq % kPage || c.max_seq <= 0)
    return fail(PS_ERR_INVALID, "unsupported decoder shape");
  const int shards = std::max(1, c.vocab_shards);
  if (c.shard_rank < 0 || c.shard_rank >= shards) return fail(PS_ERR_INVALID, "bad shard rank");
  // one extend call cycles through the pinned PassCtx/token ring without waiting
  // (kMaxWindow rows per slot, two slots kept for the verify compare and the read-back)
  if (c.max_seq > (kCtxSlots - 2) * kMaxWindow)
    return fail(PS_ERR_INVALID, "max_seq exceeds what one extend call can stage (62 x 256 tokens)");
  CK(cudaSetDevice(c.device));
  ps_handle* h = new ps_handle();
  h->cfg = c;
  h->bf16 = c.mode == PS_MODE_BF16;
  h->esz = h->bf16 ? 2 : 4;
  h->H = c.hidden;
  h->V = c.vocab;
  h->L = c.layers;
  h->nh = c.heads;
  h->nkv = c.kv_heads;
  h->hd = c.head_dim;
  h->I = c.intermediate;
  h->qd = c.heads * c.head_dim;
  h->kvd = c.kv_heads * c.head_dim;
  // vocab shard: contiguous block, multiple of 128 ids except the last
  const int per = round_up((c.vocab + shards - 1) / shards, 128);
  h->v_begin = std::min(c.vocab, per * c.shard_rank);
  h->v_count = std::min(c.vocab, h->v_begin + per) - h->v_begin;
  if (h->bf16 && (h->qd % 128 || (2 * h->I) % 128))
    return (delete h, fail(PS_ERR_INVALID, "bf16 mode needs 128-multiple projections"));
  auto bad = [&](const char* what) {
    ps_destroy(h);
    return fail(PS_ERR_CUDA, std::string("allocation failed: ") + what);
  };
  if (cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking) != cudaSuccess) return bad("stream");
  cudaEventCreate(&h->ev0);
  cudaEventCreate(&h->ev1);

  const int H = h->H, V = h->V, I = h->I, qd = h->qd, kvd = h->kvd;
  // ---- weights (generated on device) ----
  h->embed = alloc_weights(h, size_t(V) * H);
  if (!h->embed) return bad("embedding");
  init_tensor(h, h->embed, size_t(V) * H, 0, TID_EMBED);
  if (c.tied_embeddings) {
    h->head = offset_ptr(h, h->embed, size_t(h->v_begin) * H);
  } else {
    h->head = alloc_weights(h, size_t(h->v_count) * H);
    if (!h->head) return bad("lm head");
    init_tensor(h, h->head, size_t(h->v_count) * H, size_t(h->v_begin) * H, TID_HEAD, false);
    h->wreg.push_back({TID_HEAD, h->head, int64_t(h->v_count) * H});
  }
  h->lm_bias = h->dalloc<float>(V);
  {
    std::vector<float> b(V, 0.f);
    b[0] = c.eos_bias;
    for (int i = 1; i < 4; ++i) b[i] = c.term_bias;
    if (copy_sync(h, h->lm_bias, b.data(), sizeof(float) * V, cudaMemcpyHostToDevice) != cudaSuccess) return (ps_destroy(h), fail(PS_ERR_CUDA, "initial upload failed"));
  }
  h->layers.resize(h->L);
  if (h->bf16 && c.qkv_bias) {
    h->qkv_bias_all = h->dalloc<__nv_bfloat16>(size_t(h->L) * (qd + 2 * kvd));
    if (!h->qkv_bias_all) return bad("qkv bias");
  }
  // experiment hook: PS_TC_SPLITS="qkv,o,gu,d" overrides the split-K choice
  int force_splits[4] = {0, 0, 0, 0};
  if (const char* env = std::getenv("PS_TC_SPLITS")) std::sscanf(env, "%d,%d,%d,%d", &force_splits[0], &force_splits[1],
                                                                 &force_splits[2], &force_splits[3]);
  int gemm_idx = 0;
  const int tile_n = h->bf16 ? kTileTc : 16, kgran = h->bf16 ? 64 : 32, maxk = h->bf16 ? 0 : 2048;
  size_t part_elems = 0;
  for (int l = 0; l < h->L; ++l) {
    Layer& ly = h->layers[l];
    auto setup = [&](Gemm& gm, int N, int K) {
      gm.N = N;
      gm.K = K;
      gm.splits = h->bf16 ? choose_splits_tc(N, K) : choose_splits(N, K, tile_n, kgran, maxk);
      if (h->bf16 && force_splits[gemm_idx % 4] > 0) gm.splits = force_splits[gemm_idx % 4];
      ++gemm_idx;
      gm.w = alloc_weights(h, size_t(N) * K);
      part_elems = std::max(part_elems, size_t(gm.splits) * kMaxWindow * N);
      return gm.w != nullptr;
    };
    if (!setup(ly.qkv, qd + 2 * kvd, H) || !setup(ly.o, H, qd) || !setup(ly.gu, 2 * I, H) || !setup(ly.d, H, I))
      return bad("layer weights");
    if (h->bf16) {
      // q/k/v rows stored with RoPE pairs adjacent (kHeadPairs), see kernels.h
      auto* w = static_cast<__nv_bfloat16*>(ly.qkv.w);
      const int bases[3] = {0, qd, qd + kvd}, nrows[3] = {qd, kvd, kvd}, ids[3] = {WQ, WK, WV};
      for (int k = 0; k < 3; ++k) {
        RowPerm pm{RowPerm::kHeadPairs, h->hd, 0, bases[k]};
        launch_init_rows_permuted(w, nrows[k], H, pm, c.seed, layer_tid(l, ids[k]), 0.02, h->st);
        WEntry we{layer_tid(l, ids[k]), w, int64_t(nrows[k]) * H, H, pm};
        h->wreg.push_back(we);
      }
    } else {
      init_tensor(h, ly.qkv.w, size_t(qd) * H, 0, layer_tid(l, WQ));
      init_tensor(h, offset_ptr(h, ly.qkv.w, size_t(qd) * H), size_t(kvd) * H, 0, layer_tid(l, WK));
      init_tensor(h, offset_ptr(h, ly.qkv.w, size_t(qd + kvd) * H), size_t(kvd) * H, 0, layer_tid(l, WV));
    }
    init_tensor(h, ly.o.w, size_t(H) * qd, 0, layer_tid(l, WO));
    if (h->bf16) {
      // gate/up rows interleaved in 64-row blocks so one 128-row GEMM tile
      // holds matching gate and up features (SwiGLU in the GEMM epilogue)
      auto* gu = static_cast<__nv_bfloat16*>(ly.gu.w);
      const RowPerm pg{RowPerm::kGateUp, 0, 0, 0}, pu{RowPerm::kGateUp, 0, 1, 0};
      launch_init_rows_permuted(gu, I, H, pg, c.seed, layer_tid(l, WGATE), 0.02, h->st);
      launch_init_rows_permuted(gu, I, H, pu, c.seed, layer_tid(l, WUP), 0.02, h->st);
      h->wreg.push_back({layer_tid(l, WGATE), gu, int64_t(I) * H, H, pg});
      h->wreg.push_back({layer_tid(l, WUP), gu, int64_t(I) * H, H, pu});
    } else {
      init_tensor(h, ly.gu.w, size_t(I) * H, 0, layer_tid(l, WGATE));
      init_tensor(h, offset_ptr(h, ly.gu.w, size_t(I) * H), size_t(I) * H, 0, layer_tid(l, WUP));
    }
    init_tensor(h, ly.d.w, size_t(H) * I, 0, layer_tid(l, WDOWN));
    if (c.qkv_bias) {
      ly.bqkv = h->qkv_bias_all ? static_cast<void*>(h->qkv_bias_all + size_t(l) * (qd + 2 * kvd))
                                : alloc_weights(h, size_t(qd + 2 * kvd));
      if (!ly.bqkv) return bad("bias");
      if (h->bf16) {
        auto* b = static_cast<__nv_bfloat16*>(ly.bqkv);
        const int bases[3] = {0, qd, qd + kvd}, nrows[3] = {qd, kvd, kvd}, ids[3] = {BQ, BK, BV};
        for (int k = 0; k < 3; ++k) {
          RowPerm pm{RowPerm::kHeadPairs, h->hd, 0, bases[k]};
          launch_init_rows_permuted(b, nrows[k], 1, pm, c.seed, layer_tid(l, ids[k]), 0.02, h->st);
          WEntry we{layer_tid(l, ids[k]), b, int64_t(nrows[k]), 1, pm};
          h->wreg.push_back(we);
        }
      } else {
        init_tensor(h, ly.bqkv, qd, 0, layer_tid(l, BQ));
        init_tensor(h, offset_ptr(h, ly.bqkv, qd), kvd, 0, layer_tid(l, BK));
        init_tensor(h, offset_ptr(h, ly.bqkv, qd + kvd), kvd, 0, layer_tid(l, BV));
      }
    }
    if (h->bf16) {
      bool ok = encode_tma_2d_bf16(&ly.qkv.tm, ly.qkv.w, H, ly.qkv.N, 64, kTileTc);
      ok = ok && encode_tma_2d_bf16(&ly.o.tm, ly.o.w, qd, H, 64, kTileTc);
      ok = ok && encode_tma_2d_bf16(&ly.gu.tm, ly.gu.w, H, 2 * I, 64, kTileTc);
      ok = ok && encode_tma_2d_bf16(&ly.d.tm, ly.d.w, I, H, 64, kTileTc);
      if (!ok) return (ps_destroy(h), fail(PS_ERR_CUDA, "TMA descriptor encode failed"));
    }
  }
  if (h->bf16 && ((qd % kTileTc) || (kvd % kTileTc) || (I % 64) || (h->hd != 64 && h->hd != 128)))
    return (ps_destroy(h), fail(PS_ERR_INVALID, "bf16 path needs q/kv dims multiple of 128, I multiple of 64"));
  h->weight_bytes = double(h->esz) * (double(h->L) * (double(qd + 2 * kvd) * H + double(H) * qd + 3.0 * H * I) +
                                      double(h->v_count) * H);
  h->stats.weight_bytes = h->weight_bytes;
  if (h->bf16 && !encode_tma_2d_bf16(&h->tm_head, h->head, H, h->v_count, 64, kTileTc))
    return (ps_destroy(h), fail(PS_ERR_CUDA, "TMA descriptor encode failed"));

  // ---- paged KV pool ----
  h->g = KvGeom{h->L, h->nkv, h->hd, c.max_seq / kPage};
  const size_t kv_elems = size_t(h->L) * h->g.layer_stride();
  h->kpool = alloc_weights(h, kv_elems);
  h->vpool = alloc_weights(h, kv_elems);
  h->d_page_table = h->dalloc<int>(h->g.pages);
  h->h_page_table = h->halloc<int>(h->g.pages);
  if (!h->kpool || !h->vpool || !h->d_page_table || !h->h_page_table) return bad("kv pool");
  for (int p = h->g.pages - 1; p >= 0; --p) h->free_pages.push_back(p);

  // ---- workspaces ----
  const int max_splits_attn = c.max_seq / kPage + 1;
  const size_t seq_rows = size_t(c.max_seq) + kMaxWindow;
  h->x = h->dalloc<float>(size_t(kMaxWindow) * H);
  h->xn = alloc_weights(h, size_t(kMaxWindow) * H);
  h->q = alloc_weights(h, size_t(kMaxWindow) * qd);
  h->attn = alloc_weights(h, size_t(kMaxWindow) * qd);
  h->act = alloc_weights(h, size_t(kMaxWindow) * I);
  h->part = h->dalloc<float>(part_elems);
  h->o_part = h->dalloc<float>(size_t(kMaxWindow) * h->nh * max_splits_attn * h->hd);
  h->ml_part = h->dalloc<float>(size_t(kMaxWindow) * h->nh * max_splits_attn * 2);
  h->hn_cache = alloc_weights(h, seq_rows * H);
  h->am_tiles = h->bf16 ? (h->v_count + kTileTc - 1) / kTileTc : (h->v_count + kLmTileF32 - 1) / kLmTileF32;
  // bf16: one partial per 32-row warp quadrant of each 128-row vocab tile
  // bf16: one partial per CTA of the megakernel (<= 4 per vocab tile covers both uses)
  h->am_val = h->dalloc<float>(size_t(std::max(h->am_tiles * (h->bf16 ? 4 : 1), 1024)) * kMaxWindow);
  h->am_idx = h->dalloc<int>(size_t(std::max(h->am_tiles * (h->bf16 ? 4 : 1), 1024)) * kMaxWindow);
  h->argmax_pos = h->dalloc<int>(seq_rows);
  h->tokens_dev = h->dalloc<int>(seq_rows);
  h->term_mask = h->dalloc<unsigned char>(V);
  h->rope = h->dalloc<float2>(seq_rows * (h->hd / 2));
  h->d_tok = h->dalloc<int>(kMaxWindow);
  h->d_cand = h->dalloc<int>(c.max_seq);
  h->d_res = h->dalloc<int>(4 + kMaxWindow);  // [k, first_term, -, -, top-k ranks...]
  h->rstd = h->dalloc<float>(kMaxWindow);
  h->rstd_cache = h->dalloc<float>(seq_rows);
  h->ssq_part = h->dalloc<float>(size_t(4) * (H / kTileTc + 1) * kMaxWindow);
  h->counters = h->dalloc<unsigned>(4096 + 64);
  h->acnt = h->dalloc<unsigned>(size_t(kMaxWindow) * h->nkv);
  if (!h->rstd || !h->rstd_cache || !h->ssq_part || !h->counters || !h->acnt) return bad("bf16 chain buffers");
  h->keys = h->dalloc<unsigned long long>(kMaxWindow);
  h->keys_pos = h->dalloc<unsigned long long>(seq_rows);
  if (!h->keys || !h->keys_pos) return bad("shard keys");
  h->d_ctx = h->dalloc<PassCtx>(1);
  h->d_ctx_aux = h->dalloc<PassCtx>(1);
  h->h_ctx = h->halloc<PassCtx>(kCtxSlots);
  h->h_tok = h->halloc<int>(size_t(kCtxSlots) * kMaxWindow);
  h->h_res = h->halloc<int>(4 + kMaxWindow);
  h->h_argmax = h->halloc<int>(seq_rows);
  h->h_steps_tok = h->halloc<int>(std::max(kMaxSteps, c.max_seq));
  if (!h->x || !h->xn || !h->q || !h->attn || !h->act || !h->part || !h->o_part || !h->ml_part || !h->hn_cache ||
      !h->am_val || !h->am_idx || !h->argmax_pos || !h->tokens_dev || !h->term_mask || !h->rope || !h->d_tok ||
      !h->d_cand || !h->d_res || !h->d_ctx || !h->d_ctx_aux || !h->h_ctx || !h->h_tok || !h->h_res ||
      !h->h_argmax || !h->h_steps_tok)
    return bad("workspace");
  h->mega = h->bf16;
  // the megakernel's attention fragments: head_dim a multiple of 32, at most 128
  if (h->mega && (h->hd % 32 != 0 || h->hd > 128))
    return (ps_destroy(h), fail(PS_ERR_UNSUPPORTED, "bf16 path needs head_dim in {32, 64, 96, 128}"));
  if (h->mega) {
    int dev_sms = 0;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, c.device);
    h->sms = dev_sms > 0 ? dev_sms : 148;
    h->mega_part = h->dalloc<float>(size_t(h->sms) * 2 * kMaxWindow * 128);
    // 1-row passes publish (tag, value) words in a buffer of their own, so a
    // wide pass's fp32 partials can never be read as a tagged word
    h->mega_tags = h->dalloc<unsigned long long>(size_t(h->sms) * 2 * 128);
    h->mega_epoch = h->dalloc<unsigned>(1);
    // per-phase counter block: one counter per tile plus the all-split
    // phases' grid-sync counter at index `tiles` (megakernel.cu)
    h->mega_max_tiles = (std::max(std::max(h->qd + 2 * h->kvd, 2 * h->I), std::max(h->H, h->v_count)) + 127) / 128 + 1;
    // fused top-k needs every LM tile on the vectorised epilogue (rows * 512 <= 2 * attention buffer)
    h->tk_rows_max = std::min(kTopkRows, mega_attn_buf_wide(h->hd, h->H) / 256);
    h->mega_cnt_words = 64 + size_t(3 + 5 * h->L) * h->mega_max_tiles;
    h->mega_cnt = h->dalloc<unsigned>(h->mega_cnt_words);
    h->d_wmaps = h->dalloc<CUtensorMap>(size_t(4) * h->L + 1);
    h->d_xmaps = h->dalloc<CUtensorMap>(size_t(kMaxWindow / 16) * 4 + 1);  // + the fp32 residual-row map
    if (!h->mega_part || !h->mega_tags || !h->mega_epoch || !h->mega_cnt || !h->d_wmaps || !h->d_xmaps) return bad("megakernel buffers");
    if (const char* tr = std::getenv("PS_TRACE"); tr && tr[0] == '1')
      h->mega_trace = h->dalloc<unsigned long long>(size_t(3 + 5 * h->L) * h->sms * 16);
    std::vector<CUtensorMap> wm(size_t(4) * h->L + 1);
    for (int l = 0; l < h->L; ++l) {
      std::memcpy(&wm[4 * l + 0], h->layers[l].qkv.tm.bytes, sizeof(CUtensorMap));
      std::memcpy(&wm[4 * l + 1], h->layers[l].o.tm.bytes, sizeof(CUtensorMap));
      std::memcpy(&wm[4 * l + 2], h->layers[l].gu.tm.bytes, sizeof(CUtensorMap));
      std::memcpy(&wm[4 * l + 3], h->layers[l].d.tm.bytes, sizeof(CUtensorMap));
    }
    std::memcpy(&wm[4 * h->L], h->tm_head.bytes, sizeof(CUtensorMap));
    if (copy_sync(h, h->d_wmaps, wm.data(), sizeof(CUtensorMap) * wm.size(), cudaMemcpyHostToDevice) != cudaSuccess) return (ps_destroy(h), fail(PS_ERR_CUDA, "initial upload failed"));
    std::vector<CUtensorMap> xm(size_t(kMaxWindow / 16) * 4 + 1);
    {
      TmaDesc xr;
      if (!encode_tma_2d_f32(&xr, h->x, h->H, kMaxWindow, 128, kXBoxRows))
        return (ps_destroy(h), fail(PS_ERR_CUDA, "TMA descriptor encode failed"));
      std::memcpy(&xm[size_t(kMaxWindow / 16) * 4], xr.bytes, sizeof(CUtensorMap));
    }
    for (int k = 0; k < kMaxWindow / 16; ++k) {
      const ActDescs* ad = act_descs(h, 16 * (k + 1));
      if (!ad) return (ps_destroy(h), fail(PS_ERR_CUDA, "TMA descriptor encode failed"));
      std::memcpy(&xm[4 * k + 0], ad->xn.bytes, sizeof(CUtensorMap));
      std::memcpy(&xm[4 * k + 1], ad->attn.bytes, sizeof(CUtensorMap));
      std::memcpy(&xm[4 * k + 2], ad->act.bytes, sizeof(CUtensorMap));
      std::memcpy(&xm[4 * k + 3], ad->hn.bytes, sizeof(CUtensorMap));
    }
    if (copy_sync(h, h->d_xmaps, xm.data(), sizeof(CUtensorMap) * xm.size(), cudaMemcpyHostToDevice) != cudaSuccess) return (ps_destroy(h), fail(PS_ERR_CUDA, "initial upload failed"));
    // every pass width must fit one CTA per SM (co-residency of the grid)
    const int grp = h->nh / h->nkv;
    for (int ntok = 16; ntok <= kMaxWindow; ntok += 16)
      for (int wide = 0; wide < 2; ++wide) {
        const int attn_floats = mega_attn_bytes(h->hd, grp, wide != 0, h->H) / 4;
        const int st = mega_stages(ntok, attn_floats, wide != 0);
        if (st < 2 || mega_max_blocks_per_sm(mega_smem_bytes(ntok, st, attn_floats), wide != 0) < 1)
          return (ps_destroy(h), fail(PS_ERR_CUDA, "megakernel does not fit one CTA per SM"));
      }
  }
  {
    // RoPE table (rotate-half pairs): angle = pos * theta^(-2i/hd), in fp64.
    const int half = h->hd / 2;
    std::vector<float2> tab(seq_rows * half);
    for (size_t p = 0; p < seq_rows; ++p)
      for (int i = 0; i < half; ++i) {
        const double inv = std::pow(double(c.rope_theta), -(2.0 * i) / double(h->hd));
        const double a = double(p) * inv;
        tab[p * half + i] = make_float2(float(std::cos(a)), float(std::sin(a)));
      }
    if (copy_sync(h, h->rope, tab.data(), sizeof(float2) * tab.size(), cudaMemcpyHostToDevice) != cudaSuccess) return (ps_destroy(h), fail(PS_ERR_CUDA, "initial upload failed"));
    std::vector<unsigned char> tm(V, 0);
    tm[1] = tm[2] = tm[3] = 1;
    if (copy_sync(h, h->term_mask, tm.data(), V, cudaMemcpyHostToDevice) != cudaSuccess) return (ps_destroy(h), fail(PS_ERR_CUDA, "initial upload failed"));
  }
  if (cudaDeviceSynchronize() != cudaSuccess || cudaGetLastError() != cudaSuccess)
    return (ps_destroy(h), fail(PS_ERR_CUDA, "device initialisation failed"));
  *out = h;
  return PS_OK;
}

void ps_destroy(ps_handle* h) {
  if (!h) return;
  cudaSetDevice(h->cfg.device);
  if (h->st) cudaStreamSynchronize(h->st);
  if (h->graph) cudaGraphExecDestroy(h->graph);
  for (auto e : h->step_ev) cudaEventDestroy(e);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  for (void* p : h->allocs) cudaFree(p);
  for (void* p : h->host_allocs) cudaFreeHost(p);
  if (h->logits_buf) cudaFree(h->logits_buf);
  if (h->tk_val) cudaFree(h->tk_val);
  if (h->tk_idx) cudaFree(h->tk_idx);
  if (h->rank_pos) cudaFree(h->rank_pos);
  if (h->nccl_comm) nccl_api()->comm_destroy(h->nccl_comm);
  if (h->st) cudaStreamDestroy(h->st);
  delete h->prof;
  delete h;
}

int ps_forward(ps_handle* h, const int32_t* tokens, int32_t n, int32_t row_from, int32_t* argmax_out,
               int32_t* computed_out, float* gpu_ms) {
  if (!h || !tokens || n <= 0 || row_from < 0 || row_from > n) return fail(PS_ERR_INVALID, "bad forward arguments");
  CK(cudaSetDevice(h->cfg.device));
  int computed = 0, base = 0;
  bool enq = false;
  CK(cudaEventRecord(h->ev0, h->st));
  if (int rc = sync_to(h, tokens, n, &computed, &base, &enq, false)) return rc;
  CK(cudaEventRecord(h->ev1, h->st));
  CK(cudaStreamSynchronize(h->st));
  CK(cudaGetLastError());
  if (enq) finish_extend(h, tokens + (n - computed), computed, base);
  float ms = 0.f;
  if (computed) cudaEventElapsedTime(&ms, h->ev0, h->ev1);
  h->stats.gpu_ms += ms;
  if (gpu_ms) *gpu_ms = ms;
  if (computed_out) *computed_out = computed;
  if (argmax_out) std::memcpy(argmax_out, h->argmax_host.data() + row_from, sizeof(int) * (n - row_from));
  return PS_OK;
}

namespace {

// fp32 logits of resident rows [first, first + rows) into h->logits_buf, by the
// same LM-head arithmetic the passes used (bf16: the megakernel's LM phase in
// LM-only mode; fp32: lmhead_f32_kernel), so every value is the one the device
// argmax saw. rows <= kMaxWindow. Enqueued on h->st.
int enqueue_logits_rows(ps_handle* h, int first, int rows, bool write_logits = true) {
  if (write_logits && !h->logits_buf) CK(cudaMalloc(&h->logits_buf, sizeof(float) * size_t(kMaxWindow) * h->v_count));
  int slot;
  PassCtx* hc = next_ctx_slot(h, &slot);
  *hc = PassCtx{first, rows, 0, 0, 0, {0, 0, 0}};
  CK(copy_async(h, h->d_ctx_aux, hc, sizeof(PassCtx), cudaMemcpyHostToDevice));
  if (h->bf16) {
    enqueue_mega(h, h->d_ctx_aux, rows, nullptr, false, true, write_logits ? h->logits_buf : nullptr);
  } else {
    launch_lmhead_f32(h->d_ctx_aux, rows, static_cast<const float*>(h->hn_cache), 0,
                      static_cast<const float*>(h->head), h->lm_bias, h->v_begin, h->v_count, h->H, h->am_val,
                      h->am_idx, h->logits_buf, h->v_count, h->st);
  }
  h->stats.launches += 1;
  return PS_OK;
}

// Shared by ps_verify_greedy (topk == 0) and ps_verify_topk: one pass over the
// non-resident tail of P ++ R, the compare / first-terminator kernel, and for
// top-k the rank of every candidate token in its row; KV rolled back to |P| + k.
int verify_impl(ps_handle* h, const int32_t* prompt, int32_t n_prompt, const int32_t* cand, int32_t n_cand,
                int32_t topk, int32_t* k_out, int32_t* first_term_out, int32_t* argmax_out, int32_t* rank_out,
                float* gpu_ms) {
  if (!h || !prompt || n_prompt <= 0 || n_cand < 0 || (n_cand > 0 && !cand))
    return fail(PS_ERR_INVALID, "verification requires a nonempty prompt context");
  if (topk > 0 && n_cand > kMaxWindow) return fail(PS_ERR_INVALID, "top-k verification: candidate longer than 256");
  if (topk > 0 && h->cfg.vocab_shards > 1)
    return fail(PS_ERR_UNSUPPORTED, "top-k verification over a vocab-sharded LM head is not implemented");
  for (int i = 0; i < n_cand; ++i)
    if (cand[i] < 0 || cand[i] >= h->cfg.vocab) return fail(PS_ERR_INVALID, "candidate token id out of range");
  CK(cudaSetDevice(h->cfg.device));
  std::vector<int> seq(prompt, prompt + n_prompt);
  if (n_cand) seq.insert(seq.end(), cand, cand + n_cand);
  const int n = int(seq.size());
  int computed = 0, base = 0;
  bool enq = false;
  // bf16, k <= kTopkList: ranks from the fused per-tile lists (no logits rows)
  const bool fused_topk = topk > 0 && topk <= kTopkList && h->bf16 && h->tk_rows_max >= 2;
  if (fused_topk && !h->tk_val) {
    const size_t n_tk = size_t(h->am_tiles) * kTopkRows * kTopkList;
    CK(cudaMalloc(&h->tk_val, sizeof(float) * n_tk));
    CK(cudaMalloc(&h->tk_idx, sizeof(int) * n_tk));
    CK(cudaMalloc(&h->rank_pos, sizeof(int) * (size_t(h->cfg.max_seq) + kMaxWindow)));
  }
  if (topk > 0 && !h->logits_buf) CK(cudaMalloc(&h->logits_buf, sizeof(float) * size_t(kMaxWindow) * h->v_count));
  CK(cudaEventRecord(h->ev0, h->st));
  h->capture_logits = topk > 0;
  h->topk_fused = fused_topk;
  h->topk_k = topk;
  h->cap_n0 = -1;
  h->tk_n0 = -1;
  const int sync_rc = sync_to(h, seq.data(), n, &computed, &base, &enq, false);
  h->capture_logits = false;
  h->topk_fused = false;
  if (sync_rc) return sync_rc;
  if (n_cand) {
    int slot;
    next_ctx_slot(h, &slot);
    int* ht = h->h_tok + size_t(slot) * kMaxWindow;
    // a candidate that fits one ring slot is staged in pinned memory; a longer one
    // (top-k rejects those, greedy allows up to max_seq) is copied from the
    // caller's pageable buffer (cudaMemcpyAsync stages it synchronously)
    const int* src = cand;
    if (n_cand <= kMaxWindow) {
      std::memcpy(ht, cand, sizeof(int) * n_cand);
      src = ht;
    }
    CK(copy_async(h, h->d_cand, src, sizeof(int) * n_cand, cudaMemcpyHostToDevice));
    launch_verify_compare(h->argmax_pos, n_prompt, h->d_cand, n_cand, h->term_mask, h->d_res, h->st);
    h->stats.launches += 1;
    if (topk > 0) {  // rows n_prompt-1 .. n_prompt+n_cand-2 score the candidate tokens
      const int first = n_prompt - 1;
      const bool pass_ranked = enq && h->tk_n0 >= 0 && h->tk_n0 <= first && first + n_cand <= h->tk_n0 + h->tk_rows;
      if (fused_topk && (pass_ranked || (n_cand >= 2 && n_cand <= h->tk_rows_max))) {
        if (!pass_ranked) {  // rows resident from an earlier pass: LM head over them, lists only
          h->topk_fused = true;
          const int rc = enqueue_logits_rows(h, first, n_cand, false);
          h->topk_fused = false;
          if (rc) return rc;
        }
        CK(cudaMemcpyAsync(h->d_res + 4, h->rank_pos + first, sizeof(int) * n_cand, cudaMemcpyDeviceToDevice, h->st));
      } else {
        const float* rows = h->logits_buf;
        if (enq && h->cap_n0 >= 0 && h->cap_n0 <= first && first + n_cand <= h->cap_n0 + h->cap_rows) {
          rows = h->logits_buf + size_t(first - h->cap_n0) * h->v_count;  // written by this very pass
        } else {  // rows resident from an earlier pass (or a chunked extend): LM head over them
          if (int rc = enqueue_logits_rows(h, first, n_cand)) return rc;
        }
        launch_topk_rank(rows, h->v_count, h->v_count, h->d_cand, n_cand, h->d_res + 4, h->st);
        h->stats.launches += 1;
      }
    }
    CK(copy_async(h, h->h_res, h->d_res, sizeof(int) * (topk > 0 ? 4 + n_cand : 2), cudaMemcpyDeviceToHost));
  }
  CK(cudaEventRecord(h->ev1, h->st));
  CK(cudaStreamSynchronize(h->st));
  CK(cudaGetLastError());
  if (enq) finish_extend(h, seq.data() + (n - computed), computed, base);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, h->ev0, h->ev1);
  h->stats.gpu_ms += ms;
  int k = n_cand ? h->h_res[0] : 0;
  if (topk > 0) {  // maximal prefix whose tokens rank inside the top k
    k = n_cand;
    for (int i = 0; i < n_cand; ++i)
      if (h->h_res[4 + i] >= topk) {
        k = i;
        break;
      }
    if (rank_out) std::memcpy(rank_out, h->h_res + 4, sizeof(int) * n_cand);
  }
  const int first_term = n_cand ? h->h_res[1] : -1;
  if (argmax_out) std::memcpy(argmax_out, h->argmax_host.data() + (n_prompt - 1), sizeof(int) * (n_cand + 1));
  truncate_to(h, n_prompt + k);  // KV rollback to the accepted prefix
  if (k_out) *k_out = k;
  if (first_term_out) *first_term_out = first_term;
  if (gpu_ms) *gpu_ms = ms;
  return PS_OK;
}

}  // namespace

int ps_logits_rows(ps_handle* h, int32_t first, int32_t n, float* out) {
  if (!h || !out || first < 0 || n <= 0 || first + n > int(h->resident.size()))
    return fail(PS_ERR_INVALID, "logits rows outside the resident sequence");
  CK(cudaSetDevice(h->cfg.device));
  for (int done = 0; done < n;) {
    const int rows = std::min(kMaxWindow, n - done);
    if (int rc = enqueue_logits_rows(h, first + done, rows)) return rc;
    CK(copy_async(h, out + size_t(done) * h->v_count, h->logits_buf, sizeof(float) * size_t(rows) * h->v_count,
                  cudaMemcpyDeviceToHost));
    CK(cudaStreamSynchronize(h->st));
    done += rows;
  }
  CK(cudaGetLastError());
  return PS_OK;
}

int ps_verify_greedy(ps_handle* h, const int32_t* prompt, int32_t n_prompt, const int32_t* cand, int32_t n_cand,
                     int32_t* k_out, int32_t* first_term_out, int32_t* argmax_out, float* gpu_ms) {
  return verify_impl(h, prompt, n_prompt, cand, n_cand, 0, k_out, first_term_out, argmax_out, nullptr, gpu_ms);
}

int ps_verify_topk(ps_handle* h, const int32_t* prompt, int32_t n_prompt, const int32_t* cand, int32_t n_cand,
                   int32_t topk, int32_t* k_out, int32_t* first_term_out, int32_t* argmax_out, int32_t* rank_out,
                   float* gpu_ms) {
  if (topk < 1) return fail(PS_ERR_INVALID, "top-k verification requires k >= 1");
  return verify_impl(h, prompt, n_prompt, cand, n_cand, topk, k_out, first_term_out, argmax_out, rank_out, gpu_ms);
}

int ps_decode_greedy(ps_handle* h, const int32_t* seq, int32_t n_seq, int32_t max_tokens, int32_t stop_at_eos,
                     int32_t* tokens_out, int32_t* n_out, float* token_ms) {
  if (!h || !seq || n_seq <= 0 || max_tokens <= 0 || !tokens_out || !n_out)
    return fail(PS_ERR_INVALID, "bad decode arguments");
  CK(cudaSetDevice(h->cfg.device));
  int computed = 0, base = 0;
  bool enq = false;
  CK(cudaEventRecord(h->ev0, h->st));
  if (int rc = sync_to(h, seq, n_seq, &computed, &base, &enq, true)) return rc;
  CK(cudaEventRecord(h->ev1, h->st));
  CK(cudaStreamSynchronize(h->st));
  CK(cudaGetLastError());
  float first_ms = 0.f;
  if (enq) {
    finish_extend(h, seq + (n_seq - computed), computed, base);
    cudaEventElapsedTime(&first_ms, h->ev0, h->ev1);
    h->stats.gpu_ms += first_ms;
  }
  int produced = 0;
  tokens_out[produced] = h->argmax_host[n_seq - 1];
  if (token_ms) token_ms[produced] = first_ms;
  produced = 1;
  bool stopped = stop_at_eos && tokens_out[0] == kEos;
  std::vector<float> ms(kMaxSteps);
  while (!stopped && produced < max_tokens) {
    const int n0 = int(h->resident.size());
    // never ask for steps past the KV capacity (a request that EOS ends early
    // must not fail): the loop stops at the capacity with the tokens produced
    // so far; the next call that needs another position gets PS_ERR_CAPACITY
    const int room = h->cfg.max_seq - n0;
    if (room <= 0) break;
    const int steps = std::min(std::min(kMaxSteps, max_tokens - produced), room);
    int executed = 0;
    if (int rc = run_decode_steps(h, n0, steps, stop_at_eos, &executed, ms.data())) return rc;
    // step i processed token (previous argmax) at position n0+i and produced argmax_pos[n0+i]
    for (int i = 0; i < executed; ++i) {
      h->resident.push_back(h->h_steps_tok[i]);
      h->argmax_host.push_back(h->h_argmax[n0 + i]);
      tokens_out[produced] = h->h_argmax[n0 + i];
      if (token_ms) token_ms[produced] = ms[i];
      ++produced;
      if (stop_at_eos && tokens_out[produced - 1] == kEos) {
        stopped = true;
        break;
      }
    }
    h->stats.kv_tokens = int64_t(h->resident.size());
    if (executed < steps) stopped = true;
  }
  // pages mapped for steps that never ran are released
  {
    const int keep = (int(h->resident.size()) + kPage - 1) / kPage;
    while (h->pages_mapped > keep) h->free_pages.push_back(h->h_page_table[--h->pages_mapped]);
  }
  *n_out = produced;
  return PS_OK;
}

int ps_truncate(ps_handle* h, int32_t n) {
  if (!h || n < 0) return fail(PS_ERR_INVALID, "bad truncate length");
  truncate_to(h, n);
  return PS_OK;
}

int ps_resident(ps_handle* h, int32_t* out, int32_t cap, int32_t* n) {
  if (!h || !n) return fail(PS_ERR_INVALID, "null argument");
  *n = int(h->resident.size());
  if (out) std::memcpy(out, h->resident.data(), sizeof(int) * std::min<size_t>(cap, h->resident.size()));
  return PS_OK;
}

int ps_argmax_rows(ps_handle* h, int32_t first, int32_t n, int32_t* out) {
  if (!h || !out || first < 0 || n < 0 || first + n > int(h->argmax_host.size()))
    return fail(PS_ERR_INVALID, "rows outside the resident sequence");
  std::memcpy(out, h->argmax_host.data() + first, sizeof(int) * n);
  return PS_OK;
}

int ps_set_terminators(ps_handle* h, const uint8_t* mask, int32_t vocab) {
  if (!h || !mask || vocab != h->V) return fail(PS_ERR_INVALID, "terminator mask must cover the vocabulary");
  CK(cudaSetDevice(h->cfg.device));
  CK(copy_sync(h, h->term_mask, mask, vocab, cudaMemcpyHostToDevice));
  return PS_OK;
}

int ps_read_weights(ps_handle* h, int32_t tid, int64_t offset, int64_t count, float* out) {
  if (!h || !out || offset < 0 || count < 0) return fail(PS_ERR_INVALID, "bad arguments");
  CK(cudaSetDevice(h->cfg.device));
  for (const WEntry& e : h->wreg) {
    if (e.tid != tid) continue;
    if (offset + count > e.count) return fail(PS_ERR_INVALID, "range outside tensor");
    if (e.perm.kind != RowPerm::kIdentity) {
      std::vector<uint16_t> row(e.cols);
      for (int64_t i = 0; i < count;) {
        const int64_t src = offset + i, r = src / e.cols, c = src % e.cols;
        const int64_t dr = e.perm.dst(int(r));
        const int64_t take = std::min<int64_t>(count - i, e.cols - c);
        CK(copy_sync(h, row.data(), static_cast<uint16_t*>(e.ptr) + dr * e.cols + c, 2 * take, cudaMemcpyDeviceToHost));
        for (int64_t k = 0; k < take; ++k) {
          uint32_t b = uint32_t(row[k]) << 16;
          std::memcpy(out + i + k, &b, 4);
        }
        i += take;
      }
      return PS_OK;
    }
    if (h->bf16) {
      std::vector<uint16_t> tmp(count);
      CK(copy_sync(h, tmp.data(), static_cast<uint16_t*>(e.ptr) + offset, 2 * count, cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < count; ++i) {
        uint32_t b = uint32_t(tmp[i]) << 16;
        std::memcpy(out + i, &b, 4);
      }
    } else {
      CK(copy_sync(h, out, static_cast<float*>(e.ptr) + offset, 4 * count, cudaMemcpyDeviceToHost));
    }
    return PS_OK;
  }
  return fail(PS_ERR_INVALID, "unknown tensor id");
}

int ps_get_stats(ps_handle* h, ps_stats* out) {
  if (!h || !out) return fail(PS_ERR_INVALID, "null argument");
  *out = h->stats;
  out->kv_tokens = int64_t(h->resident.size());
  return PS_OK;
}

int ps_profile_decode(ps_handle* h, int32_t steps, double* ms_out, double* bytes_out) {
  if (!h || steps <= 0 || !ms_out) return fail(PS_ERR_INVALID, "bad arguments");
  if (h->resident.empty()) return fail(PS_ERR_INVALID, "profile needs a resident context");
  CK(cudaSetDevice(h->cfg.device));
  const int n0 = int(h->resident.size());
  if (n0 + steps > h->cfg.max_seq) return fail(PS_ERR_CAPACITY, "profile exceeds KV capacity");
  if (int rc = map_pages(h, n0 + steps)) return rc;
  if (!h->prof) {
    h->prof = new Prof();
    for (auto& e : h->prof->ev) cudaEventCreate(&e);
  }
  for (int c = 0; c < kProfClasses; ++c) ms_out[c] = 0.0;
  int slot;
  PassCtx* hc = next_ctx_slot(h, &slot);
  *hc = PassCtx{n0, 1, 0, 0, 0, {0, 0, 0}};
  CK(copy_async(h, h->d_ctx, hc, sizeof(PassCtx), cudaMemcpyHostToDevice));
  h->prof_on = true;
  for (int s = 0; s < steps; ++s) {
    h->prof->n = 0;
    enqueue_pass_any(h, h->d_ctx, 1, nullptr, n0 + steps - 1, true);
    cudaError_t e = cudaStreamSynchronize(h->st);
    if (e != cudaSuccess) {
      h->prof_on = false;
      return fail(PS_ERR_CUDA, std::string("profile step: ") + cudaGetErrorString(e));
    }
    for (int i = 0; i + 1 < h->prof->n; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, h->prof->ev[i], h->prof->ev[i + 1]);
      ms_out[h->prof->cls[i]] += ms;
    }
  }
  h->prof_on = false;
  // the profiled steps only wrote positions >= n0: release their pages
  {
    const int keepp = (n0 + kPage - 1) / kPage;
    while (h->pages_mapped > keepp) h->free_pages.push_back(h->h_page_table[--h->pages_mapped]);
  }
  for (int c = 0; c < kProfClasses; ++c) ms_out[c] /= steps;
  if (bytes_out) {
    const double e = double(h->esz), H = h->H, qd = h->qd, kvd = h->kvd, I = h->I, Ld = h->L;
    const double ctx = n0 + steps / 2.0;
    bytes_out[0] = Ld * 2 * H * 4 * 3;                     // residual streams (approx.)
    bytes_out[1] = Ld * (qd + 2 * kvd) * H * e;            // qkv weights
    bytes_out[2] = Ld * 2 * kvd * ctx * e;                 // KV read
    bytes_out[3] = Ld * H * qd * e;                        // o weights
    bytes_out[4] = Ld * 2 * I * H * e;                     // gate/up weights
    bytes_out[5] = Ld * H * I * e;                         // down weights
    bytes_out[6] = double(h->v_count) * H * e;             // LM head weights
    bytes_out[7] = 0;
    if (h->mega) {  // one kernel per pass: report the whole pass under "other"
      double all = 0;
      for (int i = 0; i < 7; ++i) all += bytes_out[i];
      for (int i = 0; i < 7; ++i) bytes_out[i] = 0;
      bytes_out[7] = all - Ld * 2 * H * 4 * 3 + Ld * 2 * kvd * e;  // weights + KV read + KV append
    }
  }
  CK(cudaGetLastError());
  return PS_OK;
}

int ps_trace(ps_handle* h, uint64_t* out, int64_t cap, int32_t* nphases, int32_t* ctas) {
  if (!h || !nphases || !ctas) return fail(PS_ERR_INVALID, "null argument");
  if (!h->mega_trace) return fail(PS_ERR_INVALID, "tracing is off (set PS_TRACE=1 before ps_create)");
  *nphases = 3 + 5 * h->L;
  *ctas = h->sms;
  const int64_t n = int64_t(*nphases) * h->sms * 16;
  if (out) CK(copy_sync(h, out, h->mega_trace, sizeof(uint64_t) * std::min<int64_t>(cap, n), cudaMemcpyDeviceToHost));
  return PS_OK;
}

int ps_nccl_unique_id(void* out128) {
  NcclApi* api = nccl_api();
  if (!api) return fail(PS_ERR_UNSUPPORTED, "libnccl not found (set PS_NCCL_LIB)");
  if (!out128) return fail(PS_ERR_INVALID, "null argument");
  const int rc = api->get_unique_id(out128);
  return rc ? fail(PS_ERR_CUDA, std::string("ncclGetUniqueId: ") + api->error_string(rc)) : PS_OK;
}

int ps_shard_init(ps_handle* h, const void* id, int32_t rank, int32_t world) {
  if (!h || !id) return fail(PS_ERR_INVALID, "null argument");
  if (world != std::max(1, h->cfg.vocab_shards) || rank != h->cfg.shard_rank)
    return fail(PS_ERR_INVALID, "communicator does not match the configured vocab shards");
  NcclApi* api = nccl_api();
  if (!api) return fail(PS_ERR_UNSUPPORTED, "libnccl not found (set PS_NCCL_LIB)");
  CK(cudaSetDevice(h->cfg.device));
  NcclUniqueId uid;
  std::memcpy(uid.internal, id, sizeof(uid.internal));
  void* comm = nullptr;
  const int rc = nccl_comm_init(api, &comm, world, uid, rank);
  if (rc) return fail(PS_ERR_CUDA, std::string("ncclCommInitRank: ") + api->error_string(rc));
  if (h->graph) {  // the captured decode step must now include the all-reduce
    cudaGraphExecDestroy(h->graph);
    h->graph = nullptr;
  }
  h->nccl_comm = comm;
  return PS_OK;
}

int ps_shard_keys(ps_handle* h, int32_t first, int32_t n, uint64_t* out) {
  if (!h || !out || first < 0 || n < 0 || first + n > int(h->resident.size()))
    return fail(PS_ERR_INVALID, "rows outside the resident sequence");
  if (!keyed(h)) return fail(PS_ERR_INVALID, "not a vocab-sharded instance (and no communicator attached)");
  CK(cudaSetDevice(h->cfg.device));
  CK(copy_sync(h, out, h->keys_pos + first, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost));
  return PS_OK;
}

}  // extern "C"
