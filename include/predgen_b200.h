/*
 * predgen_b200 — C ABI of the B200 predict-and-verify decoder runtime.
 *
 * Drop-in boundary for PredGen's input-time predict-and-verify loop
 * (arXiv 2506.15556). The reference package `specstream` reaches all model
 * arithmetic through ONE Python surface, `LanguageModel`
 * (/root/reference/pkg/src/specstream/lm.py:157-213); it has no native FFI.
 * These entry points are what a native backend behind that surface binds
 * (INTEGRATION.md shows the ctypes stub). Each function names the reference
 * interface it replaces.
 *
 * Conventions: plain pointers and sizes, no framework types. Every function
 * returns PS_OK (0) or a negative status; ps_last_error() gives the message.
 * Buffers are caller-owned host memory. One handle = one decoder instance
 * with one resident token sequence (bs = 1), driven by one thread at a time
 * (SPEC.md:168-169); distinct handles may live on distinct GPUs/threads.
 */
#ifndef PREDGEN_B200_H_
#define PREDGEN_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; Python maps them onto the reference's exception types */
#define PS_OK 0
#define PS_ERR_INVALID (-1)   /* ValueError (lm.py:52-54, verify.py:70-71)        */
#define PS_ERR_PREFIX (-2)    /* PrefixViolationError (lm.py:32-33, 192-199)      */
#define PS_ERR_CUDA (-3)      /* device / driver failure                          */
#define PS_ERR_CAPACITY (-4)  /* context longer than the KV capacity (max_seq)   */
#define PS_ERR_UNSUPPORTED (-5)

#define PS_MODE_F32 0   /* fp32 storage, fp32 SIMT math: bit-exact parity mode  */
#define PS_MODE_BF16 1  /* bf16 storage, fp32 accumulate, tcgen05 tensor cores  */

typedef struct ps_config {
  int32_t vocab, hidden, layers, heads, kv_heads, head_dim, intermediate;
  int32_t tied_embeddings, qkv_bias, mode;
  float rope_theta, rms_eps;
  float term_bias, eos_bias; /* logit bias on ids 1..3 ('.','?','!') and on EOS id 0 */
  uint64_t seed;             /* weight generator seed (oracle/weights.py spec)     */
  int32_t max_seq;           /* KV capacity in tokens (multiple of 64)             */
  int32_t device;            /* CUDA device ordinal                                */
  int32_t vocab_shards;      /* >1: this instance holds LM-head rows of one shard  */
  int32_t shard_rank;
  int32_t use_graphs;        /* capture the 1-row decode step in a CUDA graph       */
  int32_t reserved[7];
} ps_config;

typedef struct ps_handle ps_handle;

typedef struct ps_stats {
  int64_t passes;          /* device passes launched (extend or decode step)       */
  int64_t rows;            /* rows (positions) computed                            */
  int64_t decode_steps;    /* graph-replayed 1-row steps                           */
  int64_t prefix_hits;     /* forward/verify calls answered from resident KV      */
  int64_t kv_tokens;       /* resident tokens                                      */
  int64_t kv_pages_used;
  int64_t rollbacks;       /* truncations of the resident sequence (KV rollback)  */
  int64_t launches;        /* kernels launched by this handle (graph nodes counted per replay) */
  int64_t h2d_bytes;       /* host->device bytes copied by API calls               */
  int64_t d2h_bytes;       /* device->host bytes copied by API calls               */
  double weight_bytes;     /* weights streamed by one full pass                    */
  double gpu_ms;           /* accumulated measured device time                     */
} ps_stats;

const char* ps_last_error(void);

/* Allocate weights (generated on the device from cfg->seed), the paged KV
 * pool and workspaces. Replaces `LanguageModel.__init__` (lm.py:166-169). */
int ps_create(const ps_config* cfg, ps_handle** out);
void ps_destroy(ps_handle* h);

/* Make the resident sequence equal to tokens[0..n): reuse the longest common
 * prefix, roll back the rest (free its pages) and run one pass over the new
 * tail. argmax_out (nullable) receives the argmax id of rows [row_from, n).
 * *computed_out = rows actually computed, *gpu_ms = device time of the pass.
 * Replaces `LanguageModel.forward` (lm.py:182-203) minus the logits rows. */
int ps_forward(ps_handle* h, const int32_t* tokens, int32_t n, int32_t row_from, int32_t* argmax_out,
               int32_t* computed_out, float* gpu_ms);

/* Materialise fp32 logits rows for resident positions [first, first+n) into
 * out[n][vocab_local] (parity / slow path: `LogitsBlock.rows`, lm.py:84-104). */
int ps_logits_rows(ps_handle* h, int32_t first, int32_t n, float* out);

/* Fused greedy verify: pass over prompt ++ cand (resident prefix reused),
 * per-row argmax, compare to cand, first mismatch = accept length k, first
 * terminator of cand; KV rolled back to len(prompt)+k. argmax_out (nullable)
 * gets the n_cand+1 argmax ids of rows len(prompt)-1 .. len(prompt)+n_cand-1
 * (the last one is the correction / bonus token).
 * Replaces `verify_greedy` -> `_verify_by_rule` -> `_accepted_prefix` /
 * `_sentence_covered` (verify.py:43-97). */
int ps_verify_greedy(ps_handle* h, const int32_t* prompt, int32_t n_prompt, const int32_t* cand,
                     int32_t n_cand, int32_t* k_out, int32_t* first_term_out, int32_t* argmax_out,
                     float* gpu_ms);

/* Fused top-k verify: the greedy pass, then the rank of every candidate token
 * in its row, rank = #{j : s_j > s_t or (s_j == s_t and j < t)} in the fp32
 * logits the pass's LM head produced (no sort, no host rows); k = the longest
 * prefix of cand whose ranks are < topk. KV rolled back to len(prompt)+k.
 * bf16 with topk <= 8 and a pass of 2..160 rows: the LM epilogue keeps each
 * (vocab tile, row)'s best topk (value, id) and the pass merges them — no
 * logits rows exist — so a rank >= topk reads topk (the verifier only asks
 * rank < topk). Otherwise ranks are counted exactly over materialised rows.
 * rank_out (nullable) gets the n_cand ranks; the other outputs are as in
 * ps_verify_greedy. topk == 1 accepts exactly what ps_verify_greedy accepts.
 * Unsupported (PS_ERR_UNSUPPORTED) on a vocab-sharded LM head.
 * Replaces `verify_topk` -> `_verify_by_rule` with `topk_tokens`
 * (verify.py:100-113, lm.py:139-145). */
int ps_verify_topk(ps_handle* h, const int32_t* prompt, int32_t n_prompt, const int32_t* cand,
                   int32_t n_cand, int32_t topk, int32_t* k_out, int32_t* first_term_out,
                   int32_t* argmax_out, int32_t* rank_out, float* gpu_ms);

/* Greedy continuation of seq[0..n_seq): up to max_tokens argmax tokens, the
 * first from row n_seq-1 (free when already resident), the rest from
 * back-to-back 1-row decode steps replayed from a CUDA graph without host
 * round trips; stops after EOS when stop_at_eos, and at the KV capacity
 * (max_seq positions: *n_out < max_tokens without an error). token_ms (nullable) gets the
 * measured device ms attributable to each produced token. The last produced
 * token is not resident. Replaces the decode loop of `ar_generate`
 * (generate.py:163-176) / `greedy_decode` (lm.py:373-381). */
int ps_decode_greedy(ps_handle* h, const int32_t* seq, int32_t n_seq, int32_t max_tokens,
                     int32_t stop_at_eos, int32_t* tokens_out, int32_t* n_out, float* token_ms);

/* Roll the resident sequence back to its first n tokens (CacheHandle.truncated, lm.py:76-81). */
int ps_truncate(ps_handle* h, int32_t n);
/* Resident token count (and tokens when out != NULL, capacity cap). */
int ps_resident(ps_handle* h, int32_t* out, int32_t cap, int32_t* n);
/* Cached argmax ids of resident rows [first, first+n). */
int ps_argmax_rows(ps_handle* h, int32_t first, int32_t n, int32_t* out);

/* One byte per vocab id, nonzero for sentence terminators (text.py:28). */
int ps_set_terminators(ps_handle* h, const uint8_t* mask, int32_t vocab);

/* Read back `count` stored weights of tensor `tid` starting at element
 * `offset`, as fp32 (test hook: parity of the device generator). */
int ps_read_weights(ps_handle* h, int32_t tid, int64_t offset, int64_t count, float* out);

int ps_get_stats(ps_handle* h, ps_stats* out);

/* Per-kernel-class device time of eager (non-graph) 1-row decode steps:
 * runs `steps` steps from the resident state with CUDA events around every
 * launch, then rolls back. ms_out[0..7] = {embed+norms, qkv gemm, attention,
 * o gemm, gate/up gemm, down gemm, lm head, other}; bytes_out[0..7] = the
 * algorithmic bytes of each class per step. */
int ps_profile_decode(ps_handle* h, int32_t steps, double* ms_out, double* bytes_out);

/* Megakernel timeline of the last pass (only when PS_TRACE=1 at ps_create):
 * out[(phase * ctas + cta) * 8 + slot] in ns (globaltimer); slots: 0 producer
 * passed the barrier, 1 workers passed it, 2 workers finished the phase, 3 MMA
 * issue finished, 4 workers saw the last accumulator, 5 partials published,
 * 6 deferred finalisation done. */
int ps_trace(ps_handle* h, uint64_t* out, int64_t cap, int32_t* nphases, int32_t* ctas);

/* Vocab-sharded LM head (config c4). Each instance holds LM-head rows
 * [v_begin, v_begin + V/G) (cfg->vocab_shards = G, cfg->shard_rank). The
 * per-row (max logit, lowest id) is packed as orderable_f32 << 32 |
 * (0xFFFFFFFF - id); after ps_shard_init the keys of every pass are
 * all-reduced with a uint64 MAX over NCCL (NVLink), which yields the global
 * argmax with the lowest-id tie-break of lm.py:134-136. Without a
 * communicator argmax ids stay shard-local and ps_shard_keys exposes the keys
 * (tests merge them on the host). libnccl is dlopen'ed (PS_NCCL_LIB). */
int ps_nccl_unique_id(void* out_128b);
int ps_shard_init(ps_handle* h, const void* nccl_unique_id_128b, int32_t rank, int32_t world);
int ps_shard_keys(ps_handle* h, int32_t first, int32_t n, uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* PREDGEN_B200_H_ */
