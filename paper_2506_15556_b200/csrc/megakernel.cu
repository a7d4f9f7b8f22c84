// Persistent decode/verify kernel for the bf16 path: ONE launch per pass.
//
// Grid = one CTA per SM (cooperative launch, all CTAs co-resident). The pass is
// a fixed sequence of phases — EMBED, then per layer QKV, ATTN, O, GU, DOWN,
// then LM — separated by grid barriers (a monotonic arrival counter). Warp
// roles per CTA (192 threads):
//   warp 0     TMA producer. Weight tiles of the NEXT GEMM phase are issued
//              before waiting for the barrier that guards its activations, so
//              HBM keeps streaming across phase boundaries (the ring holds
//              up to 8 x 16 KB weight stages per SM).
//   warp 1     TMEM owner + tcgen05.mma issuer (M=128 weights x N=rows tokens,
//              fp32 accumulators in TMEM, double-buffered across pieces).
//   warps 2-5  epilogue (TMEM lane quadrant = warp % 4), attention and embed.
//
// GEMM work is split stream-K style: the k-blocks of all 128-row tiles of a
// phase are laid end to end and CTA c takes blocks [c*T/G, (c+1)*T/G). A tile
// cut by a CTA boundary has 2-3 pieces; each piece's partial goes to a slot
// of its CTA and the last arriving piece sums them in CTA order. The
// decomposition depends only on (N, K, #SMs), never on the pass width, so a
// row's arithmetic is identical in a 72-row verify pass and a 1-row decode
// step (batch invariance, see layers.cu).
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace ps {

namespace {

enum Phase : int { PH_EMBED = 0, PH_QKV, PH_ATTN, PH_O, PH_GU, PH_D, PH_LM, PH_FINAL };
// Worker threads: warps 2.. of the CTA (4 warps in the decode kernel, 6 in the
// wide kernel). TMEM-lane work (one warp per lane quadrant) stays on the first
// four; row-parallel work (vectorised finalisation, merges, RMSNorm
// reductions) spreads over all of them.
#define kWorkers (int(blockDim.x) - 64)
#define kWorkerWarps ((int(blockDim.x) - 64) >> 5)

__device__ __forceinline__ void wk_bar() { asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x - 64) : "memory"); }

struct Gemm {
  int N, KB, T;  // rows, k-blocks per tile, total k-blocks
  int tiles;
  int G;         // CTAs sharing this phase (<= grid): at most 8 pieces per tile
};

__device__ __forceinline__ Gemm gemm_of(const MegaParams& P, int kind) {
  Gemm g;
  switch (kind) {
    case PH_QKV: g.N = P.qd + 2 * P.kvd; g.KB = P.H / kBK; break;
    case PH_O: g.N = P.H; g.KB = P.qd / kBK; break;
    case PH_GU: g.N = 2 * P.I; g.KB = P.H / kBK; break;
    case PH_D: g.N = P.H; g.KB = P.I / kBK; break;
    default: g.N = P.vocab_local; g.KB = P.H / kBK; break;
  }
  g.tiles = (g.N + 127) / 128;
  g.T = g.tiles * g.KB;
  // pieces per tile <= ceil(KB / (T/G)) + 1 <= 8  <=>  G <= 7 * tiles
  g.G = min(min(int(gridDim.x), 7 * g.tiles), g.T);  // and T >= G: no empty CTA ranges
  if (P.gcap[kind] > 0) g.G = min(g.G, P.gcap[kind]);  // tuning hook (same for every pass width)
  return g;
}

// (c * T fits in 32 bits: T <= 1002 tiles x 64 k-blocks, c <= 148)
__device__ __forceinline__ int sk_start(int c, int G, int T) { return (c * T) / G; }
// CTA whose k-block range contains global block x
__device__ __forceinline__ int sk_owner(int x, int G, int T) { return ((x + 1) * G + T - 1) / T - 1; }

// A CTA's k-blocks, one piece per tile touched, in natural order (keeps
// DRAM access sequential). Processing the split pieces first, so their
// finalisation could overlap whole tiles' mainloop, was measured slower
// (verify +1%: the delayed whole-tile epilogues land on the phase tail).
struct PieceOrder {
  int lo, hi, KB, t_first, np;
  __device__ __forceinline__ PieceOrder(int lo_, int hi_, int KB_) : lo(lo_), hi(hi_), KB(KB_), t_first(lo_ / KB_) {
    np = hi > lo ? (hi - 1) / KB - t_first + 1 : 0;
  }
  __device__ __forceinline__ int npieces() const { return np; }
  __device__ __forceinline__ void piece(int j, int& plo, int& phi) const {
    plo = max(lo, (t_first + j) * KB);
    phi = min(hi, (t_first + j + 1) * KB);
  }
};

// atomic add with acquire+release at GPU scope: orders this CTA's prior
// writes (made visible to thread 0 by the preceding bar.sync) before the
// counter update, and the finalizer's later reads after it.
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

__device__ __forceinline__ void grid_arrive(unsigned* bar) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
}

// Acquire-load polling. (Relaxed polling plus one fence after the target is
// seen measured slower: +1.2% decode, +3% verify — DESIGN.md.)
__device__ __forceinline__ void grid_wait(const unsigned* bar, unsigned target) {
  PS_SPIN_START;
  while (ld_acquire_gpu(bar) < target) {
    PS_SPIN_CHECK;  // debug builds: bounded (tc_common.cuh)
  }
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// PS_TRACE slots per (phase, CTA), read by tools/trace_mega.py: 0 producer
// passed the barrier, 1 workers passed it, 2 workers finished the phase,
// 4 workers saw the last accumulator, 5 workers published all partials,
// 6 finalisation done, 7/8 split-tile counters (or the grid sync) passed,
// 9 shares finalised, 7-11 attention milestones in ATTN phases, 12 producer
// issued its last load, 13 MMA issued its last block, 14/15 attention S and
// softmax of the first unit
constexpr int kTraceSlots = 16;
__device__ __forceinline__ void stamp(const MegaParams& P, int p, int c, int G, int slot) {
  if (P.trace) P.trace[(size_t(p) * G + c) * kTraceSlots + slot] = gtime();
}

__device__ __forceinline__ int phase_kind(int p, int L) {
  if (p == 0) return PH_EMBED;
  if (p == 1 + 5 * L) return PH_LM;
  if (p == 2 + 5 * L) return PH_FINAL;
  return PH_QKV + (p - 1) % 5;
}

__device__ __forceinline__ const CUtensorMap* wmap_of(const MegaParams& P, int p, int kind) {
  if (kind == PH_LM) return P.wmaps + 4 * P.L;
  const int l = (p - 1) / 5;
  const int which = kind == PH_QKV ? 0 : kind == PH_O ? 1 : kind == PH_GU ? 2 : 3;
  return P.wmaps + 4 * l + which;
}

__device__ __forceinline__ const CUtensorMap* xmap_of(const MegaParams& P, int kind) {
  return P.xmaps + (kind == PH_O ? 1 : kind == PH_D ? 2 : kind == PH_LM ? 3 : 0);
}

// 2^x on the SFU (ex2.approx.ftz: one MUFU op; 2^-inf = 0, results below
// 2^-126 flush to 0 — negligible softmax weights)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// The finishing arithmetic of every GEMM epilogue, spelled with explicit
// rounding so that the TMEM-lane epilogues (finish_chunk) and the vectorised
// wide-pass finalisation (finish_share_vec) compute bitwise the same values.
__device__ __forceinline__ float epi_scale_bias(float acc, float rstd, float bias) { return fmaf(acc, rstd, bias); }
// RoPE on a rotate-half pair: the even row holds dim i, the odd row dim i+hd/2
__device__ __forceinline__ float rope_even(float val, float other, float c, float s) {
  return fmaf(val, c, -__fmul_rn(other, s));
}
__device__ __forceinline__ float rope_odd(float val, float other, float c, float s) {
  return fmaf(val, c, __fmul_rn(other, s));
}
__device__ __forceinline__ float swiglu(float gate, float up) {
  return __fmul_rn(__fdividef(gate, __fadd_rn(1.0f, ex2(__fmul_rn(gate, -1.4426950408889634f)))), up);
}

// ---------------------------------------------------------------------------
// epilogue math for one finished 8-column chunk of tile rows [128*tile, +128)
// RW: rows a pass of this instantiation can have (decode: 1, sized 16)
template <int RW>
struct EpiSmemT {
  static constexpr int kRows = RW;
  float am_v[6][RW];  // LM head: running (max, id) per worker warp (or quadrant) and row
  int am_i[6][RW];
  float red_v[4][8];
  int red_i[4][8];
  float rstd[RW];
  int flag;
  int rflag[32 * 4];  // [unit][row] of the ATT phase's deferred unit list
  int ulist[32][4];   // (t0, t1, kv head, page) of units computed, not yet counted
  int pg[8];          // wide passes: physical KV pages of logical pages n0/64 .. (n0+rows-1)/64
};

// Barrier-free: every warp finishes its own 32 rows. RoPE / SwiGLU partners
// are adjacent rows (RowPerm kHeadPairs / kGateUp) -> one shuffle; row sums
// (sum of squares, argmax) stay per warp quadrant and are combined by their
// consumer in a fixed order.
// NR: rows the call site can have in this chunk (8, or 1 for the decode finaliser).
// Per-row inputs of a chunk's finishing math that do not depend on the
// accumulator (RoPE cos/sin and KV page for QKV, the residual for O/D): the
// call sites issue them together with the partial loads / ahead of the TMEM
// read, so a chunk costs one memory round trip.
struct EpiPre {
  float a[8], b[8];
  int c[8];
};

template <int NR = 8>
__device__ __forceinline__ void epi_load(const MegaParams& P, int kind, int rows, int n0, int tile, int m, int c0,
                                         EpiPre& e) {
  const int n = tile * 128 + m;
  if (kind == PH_QKV) {
    const int half = P.hd >> 1, pi = (n & (P.hd - 1)) >> 1;
    const bool is_q = n < P.qd, is_k = !is_q && n < P.qd + P.kvd;
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const int t = c0 + j, pos = n0 + t;
      const float2 cs = (t < rows && (is_q || is_k)) ? __ldg(P.rope + size_t(pos) * half + pi) : make_float2(1.f, 0.f);
      e.a[j] = cs.x;
      e.b[j] = cs.y;
      e.c[j] = (t < rows && !is_q) ? __ldg(P.page_table + pos / kPage) : 0;
    }
  } else if (kind == PH_O || kind == PH_D) {
#pragma unroll
    for (int j = 0; j < NR; ++j) e.a[j] = (c0 + j < rows) ? __ldcg(P.x + size_t(c0 + j) * P.H + n) : 0.f;
  }
}

template <int NR = 8, class ES>
__device__ __forceinline__ void finish_chunk(const MegaParams& P, int kind, int layer, int rows, int n0, int tile, int m, int q,
                             int lane, int c0, const float (&v)[8], ES& es, const EpiPre& pre) {
  const int n = tile * 128 + m;
  if (kind == PH_QKV) {
    const int hd = P.hd, half = hd >> 1;
    const int r = n & (hd - 1), pi = r >> 1;  // hd is 64 or 128 (ps_create)
    const bool even = (r & 1) == 0;
    const int dim = even ? pi : pi + half;  // dimension within the head
    const bool is_q = n < P.qd, is_k = !is_q && n < P.qd + P.kvd;
    const float bias = P.qkv_bias ? __bfloat162float(P.qkv_bias[size_t(layer) * (P.qd + 2 * P.kvd) + n]) : 0.f;
    float2 cs[NR];
    int page[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      cs[j] = make_float2(pre.a[j], pre.b[j]);
      page[j] = pre.c[j];
    }
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const int t = c0 + j;
      const bool valid = t < rows;
      const float val = valid ? epi_scale_bias(v[j], es.rstd[t], bias) : 0.f;
      const float other = __shfl_xor_sync(0xffffffffu, val, 1);
      if (!valid) continue;
      const int pos = n0 + t;
      float out = val;
      if (is_q || is_k) out = even ? rope_even(val, other, cs[j].x, cs[j].y) : rope_odd(val, other, cs[j].x, cs[j].y);
      const __nv_bfloat16 ob = __float2bfloat16_rn(out);
      const int col = n - r + dim;  // original (unpermuted) output column
      if (is_q) {
        P.q[size_t(t) * P.qd + col] = ob;
      } else {
        const int cc = col - P.qd - (is_k ? 0 : P.kvd);
        const int h = cc >> P.hd_shift;
        const size_t off = size_t(layer) * P.g.layer_stride() +
                           ((size_t(page[j]) * P.g.kv_heads + h) * kPage + pos % kPage) * hd + (cc & (hd - 1));
        (is_k ? P.kpool : P.vpool)[off] = ob;
      }
    }
  } else if (kind == PH_GU) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const int t = c0 + j;
      const float val = t < rows ? __fmul_rn(v[j], es.rstd[t]) : 0.f;
      const float up = __shfl_xor_sync(0xffffffffu, val, 1);
      if (t < rows && (m & 1) == 0) P.act[size_t(t) * P.I + tile * 64 + (m >> 1)] = __float2bfloat16_rn(swiglu(val, up));
    }
  } else if (kind == PH_O || kind == PH_D) {
    const bool to_hn = kind == PH_D && layer == P.L - 1;
    const float* xo = pre.a;
    float sq[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const int t = c0 + j;
      sq[j] = 0.f;
      if (t < rows) {
        float* xp = P.x + size_t(t) * P.H + n;
        const float xi = __fadd_rn(xo[j], v[j]);
        *xp = xi;
        __nv_bfloat16* dst = to_hn ? P.hn_cache + size_t(n0 + t) * P.H : P.xb + size_t(t) * P.H;
        dst[n] = __float2bfloat16_rn(xi);
        sq[j] = __fmul_rn(xi, xi);
      }
    }
    if constexpr (NR == 8) {
      // transposed butterfly over the 8 rows: lane l pairs with l^16, l^8, l^4,
      // l^2, l^1 exactly as warp_sum does (and a + b == b + a), so each row's
      // sum is bitwise the decode step's; lane 4r ends with row r
#pragma unroll
      for (int step = 0; step < 3; ++step) {
        const int half = 4 >> step;
        const bool hi = (lane >> (4 - step)) & 1;
#pragma unroll
        for (int k = 0; k < half; ++k) {
          const float send = hi ? sq[k] : sq[half + k];
          const float recv = __shfl_xor_sync(0xffffffffu, send, 16 >> step);
          if (hi) sq[k] = sq[half + k];
          sq[k] += recv;
        }
      }
      sq[0] += __shfl_xor_sync(0xffffffffu, sq[0], 2);
      sq[0] += __shfl_xor_sync(0xffffffffu, sq[0], 1);
      const int t = c0 + (lane >> 2);
      if ((lane & 3) == 0 && t < rows) P.ssq_part[size_t(tile * 4 + q) * kMaxWindow + t] = sq[0];
    } else {
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const int t = c0 + j;
        const float r = warp_sum(sq[j]);
        if (lane == 0 && t < rows) P.ssq_part[size_t(tile * 4 + q) * kMaxWindow + t] = r;
      }
    }
  } else {  // PH_LM: logits = rstd * acc + bias; per-quadrant (max, lowest id)
    const bool valid = n < P.vocab_local;
    const int vid = P.v_begin + n;
    const float b = valid ? P.lm_bias[vid] : 0.f;
    float lv[NR];
    int li[NR];
#pragma unroll
    for (int j = 0; j < NR; ++j) {
      const int t = c0 + j;
      lv[j] = -INFINITY;
      li[j] = 0x7fffffff;
      if (valid && t < rows) {
        lv[j] = epi_scale_bias(v[j], es.rstd[t], b);
        li[j] = vid;
        if (P.logits_out) P.logits_out[size_t(t) * P.ld_logits + n] = lv[j];  // exactly the values the argmax sees
      }
    }
    if constexpr (NR == 8) {
      // transposed butterfly: each step halves the rows a lane carries (xor 16,
      // 8, 4), then xor 2, 1 finish; lane 4r ends with row r. (max, lowest id)
      // is a total order, so the tree does not change the result.
#pragma unroll
      for (int step = 0; step < 3; ++step) {
        const int half = 4 >> step;  // rows kept after this step
        const bool hi = (lane >> (4 - step)) & 1;
#pragma unroll
        for (int k = 0; k < half; ++k) {
          const float sv = hi ? lv[k] : lv[half + k];
          const int si = hi ? li[k] : li[half + k];
          const float rv = __shfl_xor_sync(0xffffffffu, sv, 16 >> step);
          const int ri = __shfl_xor_sync(0xffffffffu, si, 16 >> step);
          if (hi) { lv[k] = lv[half + k]; li[k] = li[half + k]; }
          argmax_merge(lv[k], li[k], rv, ri);
        }
      }
#pragma unroll
      for (int o = 2; o > 0; o >>= 1) {
        const float rv = __shfl_xor_sync(0xffffffffu, lv[0], o);
        const int ri = __shfl_xor_sync(0xffffffffu, li[0], o);
        argmax_merge(lv[0], li[0], rv, ri);
      }
      const int t = c0 + (lane >> 2);
      if ((lane & 3) == 0 && t < rows) argmax_merge(es.am_v[q][t], es.am_i[q][t], lv[0], li[0]);
    } else {
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        const int t = c0 + j;
        warp_argmax(lv[j], li[j]);
        if (lane == 0 && t < rows) argmax_merge(es.am_v[q][t], es.am_i[q][t], lv[j], li[j]);
      }
    }
  }
}

// rstd of every row of the pass from the per-tile sums of squares of the
// previous RESID phase (or the embed rstd), one warp per row, fixed tree.
// Rows are processed kRstdBatch at a time with every load in flight. Wide
// passes of up to kRstdStageRows rows stage the partials in shared memory
// instead (rstd_stage_issue / rstd_stage_reduce, same tree).
constexpr int kRstdBatch = 4;
template <class ES>
__device__ __forceinline__ void load_rstd(const MegaParams& P, bool from_embed, int rows, int w, int lane, ES& es) {
  if (from_embed) {
    for (int t = w * 32 + lane; t < rows; t += kWorkers) es.rstd[t] = __ldcg(P.rstd0 + t);
    return;
  }
  // 4 quadrant partials per tile; lane sums entries lane, lane+32, ... in order
  const int nparts = 4 * (P.H / 128);  // <= 4 * 64
  const int nw = kWorkerWarps;
  for (int t0 = w; t0 < rows; t0 += nw * kRstdBatch) {
    float vals[kRstdBatch][8];
#pragma unroll
    for (int r = 0; r < kRstdBatch; ++r) {
      const int t = t0 + nw * r;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = lane + 32 * u;
        vals[r][u] = (t < rows && e < nparts) ? __ldcg(P.ssq_part + size_t(e) * kMaxWindow + t) : 0.f;
      }
    }
#pragma unroll
    for (int r = 0; r < kRstdBatch; ++r) {
      const int t = t0 + nw * r;
      float a = 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) a += vals[r][u];
      const float ssq = warp_sum(a);
      if (lane == 0 && t < rows) es.rstd[t] = 1.0f / sqrtf(ssq / float(P.H) + P.eps);
    }
  }
}

// ---------------------------------------------------------------------------
// Attention over the paged KV cache (SIMT, fp32 math on bf16 operands).
//
// One unit = (kv head, 64-token page s, block of up to kAttnRows query rows).
// Per (row, q head): scores for the page's keys, page-local softmax stats and
// P.V; the last page to finish for a (row, kv head) merges all pages in page
// order. The per-(row, head) arithmetic does not depend on the block, the
// pass width or how heads are spread over warps (batch invariance).
//
// Operands are staged raw (bf16) in shared memory with cp.async, two unit
// buffers: the keys cached by earlier passes are requested while the CTA is
// still in the layer's QKV phase, only this pass's rows (and q) after the
// barrier, and unit i+1's loads overlap unit i's math.
constexpr int kAttnRows = 4;  // query rows per attention unit (share one KV page load)
// wide passes: query rows per unit (one 4-row M-tile per worker warp): 16 when
// the pass's units fit one round over the grid, else 24 (all 6 worker warps),
// so long contexts take fewer rounds (attention_rows_wide)
constexpr int kAttnRowsW = 16;
constexpr int kAttnRowsW2 = 24;
__device__ __forceinline__ int attention_rows_wide(const MegaParams& P, int rows, int n0, int G) {
  const int npages = (n0 + rows - 1) / kPage + 1;
  return ((rows + kAttnRowsW - 1) / kAttnRowsW) * P.kv_heads * npages <= G ? kAttnRowsW : kAttnRowsW2;
}

struct AttnSmem {  // two unit buffers [K | V | Q] at base + b * buf
  unsigned char* base;
  int buf, koff_v, koff_q;  // bytes: buffer stride, V and Q offsets within a buffer
  // rows padded to hd + 8 elements (272 B for hd = 128): the 8 rows touched by
  // one fragment load / ldmatrix phase fall in distinct banks
  // K: [64 keys][hd + 8], V: [64 keys][hd + 8], Q: [kAttnRows * grp pairs][hd + 8]
  __device__ __forceinline__ __nv_bfloat16* K(int b) const { return reinterpret_cast<__nv_bfloat16*>(base + b * buf); }
  __device__ __forceinline__ __nv_bfloat16* V(int b) const {
    return reinterpret_cast<__nv_bfloat16*>(base + b * buf + koff_v);
  }
  __device__ __forceinline__ __nv_bfloat16* Q(int b) const {
    return reinterpret_cast<__nv_bfloat16*>(base + b * buf + koff_q);
  }
};

// wide passes stage no q (fragments come from global memory) but reuse a
// buffer for the RMSNorm partials of up to kRstdStageRows rows
__device__ __forceinline__ AttnSmem attn_smem(void* base, int hd, int grp, bool wide, int H) {
  AttnSmem a;
  a.base = static_cast<unsigned char*>(base);
  a.koff_v = kPage * (hd + 8) * 2;
  a.koff_q = 2 * a.koff_v;
  a.buf = wide ? mega_attn_buf_wide(hd, H) : a.koff_q + kAttnRows * grp * (hd + 8) * 2;
  return a;
}

__device__ __forceinline__ void cp_async16(const void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Wide passes: the sum-of-squares partials of every row (4 per 128-column
// tile of the previous RESID phase) are staged into attention buffer 1 —
// idle during GEMM phases — with cp.async as the phase starts, and reduced
// with load_rstd's per-row tree (lane-strided sums, then the xor butterfly,
// here transposed over 8 rows) when the first epilogue needs them.
__device__ __forceinline__ int rstd_stage_ld(int rows) { return (rows + 3) & ~3; }
__device__ __forceinline__ bool rstd_stage_fits(const MegaParams& P, const AttnSmem& A, int rows) {
  return 4 * (P.H / 128) * rstd_stage_ld(rows) * 4 <= A.buf;
}
__device__ __forceinline__ void rstd_stage_issue(const MegaParams& P, const AttnSmem& A, int rows, int w, int lane) {
  float* S = reinterpret_cast<float*>(A.K(1));
  const int nparts = 4 * (P.H / 128), ld = rstd_stage_ld(rows);
  for (int e = w; e < nparts; e += kWorkerWarps)
    for (int v = 4 * lane; v < ld; v += 128) cp_async16(S + e * ld + v, P.ssq_part + size_t(e) * kMaxWindow + v);
}
template <class ES>
__device__ __forceinline__ void rstd_stage_reduce(const MegaParams& P, const AttnSmem& A, int rows, int w, int lane,
                                                  ES& es) {
  const float* S = reinterpret_cast<const float*>(A.K(1));
  const int nparts = 4 * (P.H / 128), ld = rstd_stage_ld(rows);
  for (int g0 = w * 8; g0 < rows; g0 += 8 * kWorkerWarps) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int t = g0 + j;
      a[j] = 0.f;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = lane + 32 * u;
        a[j] += (e < nparts && t < rows) ? S[e * ld + t] : 0.f;
      }
    }
#pragma unroll
    for (int step = 0; step < 3; ++step) {
      const int half = 4 >> step;
      const bool hi = (lane >> (4 - step)) & 1;
#pragma unroll
      for (int k = 0; k < half; ++k) {
        const float send = hi ? a[k] : a[half + k];
        const float recv = __shfl_xor_sync(0xffffffffu, send, 16 >> step);
        if (hi) a[k] = a[half + k];
        a[k] += recv;
      }
    }
    a[0] += __shfl_xor_sync(0xffffffffu, a[0], 2);
    a[0] += __shfl_xor_sync(0xffffffffu, a[0], 1);
    const int t = g0 + (lane >> 2);
    if ((lane & 3) == 0 && t < rows) es.rstd[t] = 1.0f / sqrtf(a[0] / float(P.H) + P.eps);
  }
}

struct AttnUnit {
  int t0, t1, kvh, s;
  bool valid;
};

// The i-th unit (i >= 0 counts only units with work) of CTA c: units are
// dealt round-robin (u = c, c + G, ...), page fastest.
__device__ __forceinline__ AttnUnit attn_unit_from(const MegaParams& P, int R, int rows, int n0, int u_start, int G,
                                                   int& u_next) {
  const int npages = (n0 + rows - 1) / kPage + 1;
  const int nblocks = (rows + R - 1) / R;
  const int units = nblocks * P.kv_heads * npages;
  AttnUnit U{0, 0, 0, 0, false};
  for (int u = u_start; u < units; u += G) {
    const int s = u % npages, r = u / npages;
    const int t0 = (r / P.kv_heads) * R, t1 = min(rows, t0 + R);
    if (s > (n0 + t1 - 1) / kPage) continue;  // no row of the block reaches this page
    U = AttnUnit{t0, t1, r % P.kv_heads, s, true};
    u_next = u + G;
    return U;
  }
  u_next = units;
  return U;
}

// Request a unit's operands into buffer b: part 0 = keys written by earlier
// passes (positions < n0), part 1 = this pass's keys and the q rows.
template <bool kWide>
__device__ __forceinline__ void attn_issue(const MegaParams& P, int layer, const AttnUnit& U, int n0, const AttnSmem& A,
                                           int b, int part, int tid) {
  const int hd = P.hd, grp = P.heads / P.kv_heads, vpr = hd / 8;
  const int kmax = min(kPage, n0 + U.t1 - U.s * kPage);  // keys needed by the block's last row
  const int kc = max(0, min(kmax, n0 - U.s * kPage));    // of which cached before this pass
  const int jlo = part == 0 ? 0 : kc, jhi = part == 0 ? kc : kmax;
  const size_t page = size_t(P.page_table[U.s]);
  const size_t off = size_t(layer) * P.g.layer_stride() + (page * P.kv_heads + U.kvh) * kPage * hd;
  for (int e = tid; e < (jhi - jlo) * vpr; e += kWorkers) {
    const int j = jlo + e / vpr, d0 = (e % vpr) * 8;
    cp_async16(A.K(b) + j * (hd + 8) + d0, P.kpool + off + size_t(j) * hd + d0);
    cp_async16(A.V(b) + j * (hd + 8) + d0, P.vpool + off + size_t(j) * hd + d0);
  }
  if (part == 1) {
    // V rows past the last needed key meet p = 0 in the tensor-core P.V: they
    // must be finite, so zero them (stale shared memory may hold NaN bits)
    for (int e = tid; e < (kPage - kmax) * vpr; e += kWorkers) {
      const int j = kmax + e / vpr, d0 = (e % vpr) * 8;
      *reinterpret_cast<uint4*>(A.V(b) + j * (hd + 8) + d0) = make_uint4(0u, 0u, 0u, 0u);
    }
    const int qvec_row = grp * hd / 8;
    for (int e = tid; !kWide && e < (U.t1 - U.t0) * qvec_row; e += kWorkers) {
      const int r = e / qvec_row, rem = (e % qvec_row) * 8;
      // pair (r, head) -> Q row r * grp + head
      cp_async16(A.Q(b) + (r * grp + rem / hd) * (hd + 8) + rem % hd,
                 P.q + size_t(U.t0 + r) * P.qd + size_t(U.kvh) * grp * hd + rem);
    }
  }
}

__device__ __forceinline__ void mma_bf16(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// Math of a unit whose operands are resident in buffer b, on the tensor cores
// (mma.sync m16n8k16, bf16 in / fp32 accumulate): M = the unit's (row, head)
// pairs in tiles of 16, N = keys (S) or head dims (O), K = head dims (S) or
// keys (O). Every warp computes S for the whole page (64 keys) and the
// page-local softmax in registers, then P.V for its quarter of the head dims;
// P enters the second product as a bf16 hi + lo pair (~16-bit mantissa). An
// output row depends only on its own (row, head) pair, never on where the
// pair sits in the tile, so 1-row decode and wide verify agree bitwise.
// Then the page arrival count and, for rows whose last page this was, the merge.
__device__ __forceinline__ void attention_unit(const MegaParams& P, const AttnUnit& U, int n0, const AttnSmem& A, int b,
                                               int w, int lane, int trace_p = -1) {
  const bool tr = trace_p >= 0 && threadIdx.x == 64;
  const int hd = P.hd, grp = P.heads / P.kv_heads;
  const int t0 = U.t0, t1 = U.t1, kvh = U.kvh, s = U.s;
  const int nrows = t1 - t0;
  const int npairs = nrows * grp;
  const uint32_t qbase = smem_u32(A.Q(b)), kbase = smem_u32(A.K(b));
  const uint32_t vbase = smem_u32(A.V(b));
  const uint32_t rs = uint32_t(hd + 8) * 2;  // staged row stride in bytes (conflict-free ldmatrix phases)
  // log2-domain softmax: v = s * scale * log2(e), p = 2^(v - max)
  const float sl2 = P.attn_scale * 1.4426950408889634f;
  if (tr) stamp(P, trace_p, blockIdx.x, gridDim.x, 8);
  const int g8 = lane >> 2, q4 = lane & 3;
  const int mi = lane >> 3, mr = lane & 7;  // ldmatrix: this lane addresses row mr of matrix mi
  for (int mt = 0; mt * 16 < npairs; ++mt) {
    const int p0 = mt * 16 + g8, p1 = p0 + 8;
    // ---- S = Q K^T for 16 pairs x 64 keys. Fragments by ldmatrix; rows of
    // the tile past npairs hold stale data, which only reaches their own
    // (masked, never stored) rows.
    float S[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) S[nt][0] = S[nt][1] = S[nt][2] = S[nt][3] = 0.f;
    const uint32_t qa = qbase + uint32_t(mt * 16 + (mi & 1) * 8 + mr) * rs + uint32_t(mi >> 1) * 16;
    const uint32_t ka = kbase + uint32_t((mi >> 1) * 8 + mr) * rs + uint32_t(mi & 1) * 16;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {  // hd / 16 <= 8 k-steps, unrolled so fragment loads run ahead
      if (ks < hd / 16) {
        uint32_t a0, a1, a2, a3;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                     : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                     : "r"(qa + ks * 32));
#pragma unroll
        for (int nt = 0; nt < 8; nt += 2) {
          uint32_t b0, b1, b2, b3;
          asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                       : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                       : "r"(ka + uint32_t(nt * 8) * rs + ks * 32));
          mma_bf16(S[nt], a0, a1, a2, a3, b0, b1);
          mma_bf16(S[nt + 1], a0, a1, a2, a3, b2, b3);
        }
      }
    }
    if (tr && mt == 0) { float z = S[0][0] + S[7][3]; if (z == 12345.f) stamp(P, trace_p, blockIdx.x, gridDim.x, 15); stamp(P, trace_p, blockIdx.x, gridDim.x, 14); }
    // ---- causal mask + page-local softmax; rows p0 (S[.][0..1]) and p1 (S[.][2..3])
    int nk[2];
    float mx[2], l[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int pp = h ? p1 : p0;
      const int pos = n0 + t0 + pp / grp;
      nk[h] = (pp < npairs) ? min(kPage, pos + 1 - s * kPage) : 0;  // <= 0: the row does not reach this page
      float m = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int key = nt * 8 + q4 * 2 + e;
          const float v = key < nk[h] ? S[nt][2 * h + e] * sl2 : -INFINITY;
          S[nt][2 * h + e] = v;
          m = fmaxf(m, v);
        }
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
      if (nk[h] <= 0) m = 0.f;
      float sum = 0.f;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const float pv = nk[h] > 0 ? ex2(S[nt][2 * h + e] - m) : 0.f;  // 2^(-inf) = 0 past the mask
          S[nt][2 * h + e] = pv;
          sum += pv;
        }
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      mx[h] = m;
      l[h] = sum;
    }
    if (tr && mt == 0) { float z = l[0] + l[1]; if (z == 12345.f) stamp(P, trace_p, blockIdx.x, gridDim.x, 14); stamp(P, trace_p, blockIdx.x, gridDim.x, 15); }
    // ---- O = P V for this warp's quarter of the head dims (n-tiles of 8)
    const int ndt = hd / 32;  // dim tiles per warp
    float O[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) O[i][0] = O[i][1] = O[i][2] = O[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {  // 16 keys per step: S n-tiles 2kk, 2kk+1
      uint32_t ah[4], al[4];
      const float* x0 = S[2 * kk];
      const float* x1 = S[2 * kk + 1];
      const float src[4][2] = {{x0[0], x0[1]}, {x0[2], x0[3]}, {x1[0], x1[1]}, {x1[2], x1[3]}};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const __nv_bfloat162 hi = __floats2bfloat162_rn(src[i][0], src[i][1]);
        const float2 hf = __bfloat1622float2(hi);
        ah[i] = *reinterpret_cast<const uint32_t*>(&hi);
        al[i] = pack_bf16(src[i][0] - hf.x, src[i][1] - hf.y);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (i < ndt) {
          const int dt = w * ndt + i;
          // V[keys kk*16 .. +16][dims dt*8 .. +8], transposed into the B fragment
          const uint32_t addr = vbase + uint32_t(((kk * 16 + (lane & 15)) * (hd + 8) + dt * 8) * 2);
          uint32_t b0, b1;
          asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];"
                       : "=r"(b0), "=r"(b1)
                       : "r"(addr));
          mma_bf16(O[i], ah[0], ah[1], ah[2], ah[3], b0, b1);
          mma_bf16(O[i], al[0], al[1], al[2], al[3], b0, b1);
        }
      }
    }
    // ---- page-local outputs of the pairs whose row reaches this page
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (nk[h] <= 0) continue;
      const int pp = h ? p1 : p0;
      const int t = t0 + pp / grp, head = kvh * grp + pp % grp;
      const size_t slot = (size_t(t) * P.heads + head) * P.max_splits_attn + s;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < ndt) {
          const int dim = (w * ndt + i) * 8 + q4 * 2;
          *reinterpret_cast<float2*>(P.o_part + slot * hd + dim) = make_float2(O[i][2 * h], O[i][2 * h + 1]);
        }
      if (w == 0 && q4 == 0) {
        P.ml_part[slot * 2] = mx[h];
        P.ml_part[slot * 2 + 1] = l[h];
      }
    }
  }
  wk_bar();
  if (tr) stamp(P, trace_p, blockIdx.x, gridDim.x, 9);
}

// Wide passes: unit = (kv head, page, block of kAttnRowsW rows); worker warp
// w owns the M-tile of rows t0+4w .. +3 (x grp heads) and computes its S,
// page-local softmax and P.V over all head dims. q fragments come straight
// from global memory (L2); K and V are staged in buffer b. The per-pair
// operation sequence (fragment values, MMA order over k-steps and key steps,
// softmax, hi/lo P) is attention_unit's, so results are bitwise the decode
// step's. Page-local (O, m, l) go to o_part / ml_part; the merge runs after
// a grid-wide sync (attn_merge_items).
// q fragments of this warp's M-tile of unit U (pairs p0 = lane / 4, p1 = p0 + 8;
// zero past the tile's pairs), all k-steps: requested before the unit's K / V
// wait so the two round trips overlap
__device__ __forceinline__ void attn_q_frags_wide(const MegaParams& P, const AttnUnit& U, int w, int lane,
                                                  uint32_t (&qf)[8][4]) {
  const int hd = P.hd, grp = P.heads / P.kv_heads;
  const int r0 = U.t0 + 4 * w;
  const int npairs = max(0, min(4, U.t1 - r0)) * grp;
  const int g8 = lane >> 2, q4 = lane & 3;
  const int p0 = g8, p1 = g8 + 8;
  const bool va = U.valid && p0 < npairs, vb = U.valid && p1 < npairs;
  const uint32_t* qa = reinterpret_cast<const uint32_t*>(P.q + size_t(r0 + p0 / grp) * P.qd +
                                                         size_t(U.kvh * grp + p0 % grp) * hd) + q4;
  const uint32_t* qb = reinterpret_cast<const uint32_t*>(P.q + size_t(r0 + p1 / grp) * P.qd +
                                                         size_t(U.kvh * grp + p1 % grp) * hd) + q4;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    const bool k_ok = ks < hd / 16;
    qf[ks][0] = (va && k_ok) ? __ldcg(qa + ks * 8) : 0u;
    qf[ks][1] = (vb && k_ok) ? __ldcg(qb + ks * 8) : 0u;
    qf[ks][2] = (va && k_ok) ? __ldcg(qa + ks * 8 + 4) : 0u;
    qf[ks][3] = (vb && k_ok) ? __ldcg(qb + ks * 8 + 4) : 0u;
  }
}

__device__ __forceinline__ void attention_unit_wide(const MegaParams& P, const AttnUnit& U, int n0, const AttnSmem& A,
                                                    int b, int w, int lane, const uint32_t (&qf)[8][4]) {
  const int hd = P.hd, grp = P.heads / P.kv_heads;
  const int r0 = U.t0 + 4 * w;
  const int nr = min(4, U.t1 - r0);
  if (nr <= 0) return;
  const int npairs = nr * grp;
  const int s = U.s, kvh = U.kvh;
  const uint32_t kbase = smem_u32(A.K(b)), vbase = smem_u32(A.V(b));
  const uint32_t rs = uint32_t(hd + 8) * 2;
  const float sl2 = P.attn_scale * 1.4426950408889634f;
  const int g8 = lane >> 2, q4 = lane & 3;
  const int mi = lane >> 3, mr = lane & 7;
  const int p0 = g8, p1 = g8 + 8;
  float S[8][4];
#pragma unroll
  for (int nt = 0; nt < 8; ++nt) S[nt][0] = S[nt][1] = S[nt][2] = S[nt][3] = 0.f;
  const uint32_t ka = kbase + uint32_t((mi >> 1) * 8 + mr) * rs + uint32_t(mi & 1) * 16;
#pragma unroll
  for (int ks = 0; ks < 8; ++ks) {
    if (ks < hd / 16) {
#pragma unroll
      for (int nt = 0; nt < 8; nt += 2) {
        uint32_t b0, b1, b2, b3;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                     : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                     : "r"(ka + uint32_t(nt * 8) * rs + ks * 32));
        mma_bf16(S[nt], qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3], b0, b1);
        mma_bf16(S[nt + 1], qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3], b2, b3);
      }
    }
  }
  int nk[2];
  float mx[2], l[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int pp = h ? p1 : p0;
    const int pos = n0 + r0 + pp / grp;
    nk[h] = (pp < npairs) ? min(kPage, pos + 1 - s * kPage) : 0;
    float m = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int key = nt * 8 + q4 * 2 + e;
        const float v = key < nk[h] ? S[nt][2 * h + e] * sl2 : -INFINITY;
        S[nt][2 * h + e] = v;
        m = fmaxf(m, v);
      }
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
    if (nk[h] <= 0) m = 0.f;
    float sum = 0.f;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const float pv = nk[h] > 0 ? ex2(S[nt][2 * h + e] - m) : 0.f;
        S[nt][2 * h + e] = pv;
        sum += pv;
      }
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    mx[h] = m;
    l[h] = sum;
  }
  // P as bf16 hi + lo fragments, per 16-key step
  uint32_t ah[4][4], al[4][4];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const float* x0 = S[2 * kk];
    const float* x1 = S[2 * kk + 1];
    const float src[4][2] = {{x0[0], x0[1]}, {x0[2], x0[3]}, {x1[0], x1[1]}, {x1[2], x1[3]}};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 hi = __floats2bfloat162_rn(src[i][0], src[i][1]);
      const float2 hf = __bfloat1622float2(hi);
      ah[kk][i] = *reinterpret_cast<const uint32_t*>(&hi);
      al[kk][i] = pack_bf16(src[i][0] - hf.x, src[i][1] - hf.y);
    }
  }
  size_t slot[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int pp = h ? p1 : p0;
    slot[h] = (size_t(r0 + pp / grp) * P.heads + kvh * grp + pp % grp) * P.max_splits_attn + s;
  }
  // O = P V over the head dims, 8 dim tiles (64 dims) at a time
  for (int d0 = 0; d0 < hd / 8; d0 += 8) {
    float O[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) O[i][0] = O[i][1] = O[i][2] = O[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t addr = vbase + uint32_t(((kk * 16 + (lane & 15)) * (hd + 8) + (d0 + i) * 8) * 2);
        uint32_t b0, b1;
        asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0, %1}, [%2];" : "=r"(b0), "=r"(b1) : "r"(addr));
        mma_bf16(O[i], ah[kk][0], ah[kk][1], ah[kk][2], ah[kk][3], b0, b1);
        mma_bf16(O[i], al[kk][0], al[kk][1], al[kk][2], al[kk][3], b0, b1);
      }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (nk[h] <= 0) continue;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        *reinterpret_cast<float2*>(P.o_part + slot[h] * hd + (d0 + i) * 8 + q4 * 2) =
            make_float2(O[i][2 * h], O[i][2 * h + 1]);
    }
  }
#pragma unroll
  for (int h = 0; h < 2; ++h)
    if (nk[h] > 0 && q4 == 0) {
      P.ml_part[slot[h] * 2] = mx[h];
      P.ml_part[slot[h] * 2 + 1] = l[h];
    }
}

// One (row, head) merge by a whole warp. Lane sp owns page sp's (m, l): M is
// the warp max, L the butterfly sum of l * 2^(m - M); the output sums run over
// pages in order, lane d owning dims 4d..4d+3. The first 8 pages' operands
// are requested up front (MergeLoad), so a merge over up to 512 tokens costs
// one memory round trip; two items per warp overlap theirs.
struct MergeLoad {
  float2 ml;     // (m, l) of page `lane` (lane < nsplit)
  float4 o[8];   // dims 4*lane.. of pages 0..7
  int t, h, nsplit;
  size_t base;
};

__device__ __forceinline__ void attn_merge_load(const MegaParams& P, int n0, int t, int h, int lane, MergeLoad& L) {
  const int hd = P.hd;
  L.t = t;
  L.h = h;
  L.nsplit = (n0 + t) / kPage + 1;
  L.base = (size_t(t) * P.heads + h) * P.max_splits_attn;
  L.ml = lane < L.nsplit ? __ldcg(reinterpret_cast<const float2*>(P.ml_part) + L.base + lane)
                         : make_float2(-INFINITY, 0.f);
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (u < L.nsplit && lane * 4 < hd)
      L.o[u] = __ldcg(reinterpret_cast<const float4*>(P.o_part + (L.base + u) * hd + lane * 4));
}

// More than 8 pages: pages beyond the first 8 are streamed in batches of 8.
__device__ __forceinline__ void attn_merge_general(const MegaParams& P, int lane, const MergeLoad& L) {
  const int hd = P.hd, nsplit = L.nsplit;
  const size_t base = L.base;
  float M = L.ml.x;
  for (int sp = lane + 32; sp < nsplit; sp += 32) M = fmaxf(M, __ldcg(P.ml_part + (base + sp) * 2));
  M = warp_max(M);
  float Lp = 0.f;
  if (lane < nsplit) Lp += L.ml.y * ex2(L.ml.x - M);
  for (int sp = lane + 32; sp < nsplit; sp += 32)
    Lp += __ldcg(P.ml_part + (base + sp) * 2 + 1) * ex2(__ldcg(P.ml_part + (base + sp) * 2) - M);
  const float Ls = warp_sum(Lp);
  // hd <= 128 (ps_create): lane owns dims 4 * lane .. +3. Pages 0-7 come from
  // the operands attn_merge_load already holds, later pages in batches of 8
  // with every load of a batch in flight; f of page u is ex2(m_u - M) either way
  const int d4 = lane * 4;
  const bool has = d4 < hd;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int u = 0; u < 8; ++u) {  // nsplit > 8 here
    const float f = ex2(__shfl_sync(0xffffffffu, L.ml.x, u) - M);
    if (has) {
      acc.x = fmaf(L.o[u].x, f, acc.x);
      acc.y = fmaf(L.o[u].y, f, acc.y);
      acc.z = fmaf(L.o[u].z, f, acc.z);
      acc.w = fmaf(L.o[u].w, f, acc.w);
    }
  }
  for (int sp0 = 8; has && sp0 < nsplit; sp0 += 8) {
    float f[8];
    float4 o[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (sp0 + u < nsplit) {
        f[u] = ex2(__ldcg(P.ml_part + (base + sp0 + u) * 2) - M);
        o[u] = __ldcg(reinterpret_cast<const float4*>(P.o_part + (base + sp0 + u) * hd + d4));
      }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (sp0 + u < nsplit) {
        acc.x = fmaf(o[u].x, f[u], acc.x);
        acc.y = fmaf(o[u].y, f[u], acc.y);
        acc.z = fmaf(o[u].z, f[u], acc.z);
        acc.w = fmaf(o[u].w, f[u], acc.w);
      }
  }
  if (has) {
    __nv_bfloat16* dst = P.attn + size_t(L.t) * P.qd + size_t(L.h) * hd + d4;
    dst[0] = __float2bfloat16_rn(acc.x / Ls);
    dst[1] = __float2bfloat16_rn(acc.y / Ls);
    dst[2] = __float2bfloat16_rn(acc.z / Ls);
    dst[3] = __float2bfloat16_rn(acc.w / Ls);
  }
}

// The same arithmetic from the preloaded operands when nsplit <= 8, hd <= 128.
__device__ __forceinline__ void attn_merge_finish(const MegaParams& P, int lane, const MergeLoad& L) {
  const int hd = P.hd, nsplit = L.nsplit;
  if (nsplit > 8) {
    attn_merge_general(P, lane, L);
    return;
  }
  const float M = warp_max(L.ml.x);
  float Lp = 0.f;
  if (lane < nsplit) Lp += L.ml.y * ex2(L.ml.x - M);
  const float Ls = warp_sum(Lp);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const float f = ex2(__shfl_sync(0xffffffffu, L.ml.x, u) - M);
    if (u < nsplit) {
      acc.x = fmaf(L.o[u].x, f, acc.x);
      acc.y = fmaf(L.o[u].y, f, acc.y);
      acc.z = fmaf(L.o[u].z, f, acc.z);
      acc.w = fmaf(L.o[u].w, f, acc.w);
    }
  }
  if (lane * 4 < hd) {
    __nv_bfloat16* dst = P.attn + size_t(L.t) * P.qd + size_t(L.h) * hd + lane * 4;
    dst[0] = __float2bfloat16_rn(acc.x / Ls);
    dst[1] = __float2bfloat16_rn(acc.y / Ls);
    dst[2] = __float2bfloat16_rn(acc.z / Ls);
    dst[3] = __float2bfloat16_rn(acc.w / Ls);
  }
}

__device__ __forceinline__ void attn_merge_one(const MegaParams& P, int n0, int t, int h, int lane) {
  MergeLoad L;
  attn_merge_load(P, n0, t, h, lane, L);
  attn_merge_finish(P, lane, L);
}

// Page arrival counts, then merges, for the units this CTA computed (deferred
// so the unit loop runs math back to back). Thread (unit k, row r) counts;
// the last page of a (row, kv head) merges its grp heads, one warp per (row,
// head): lane sp owns page sp for the scalars (fixed butterfly); the output
// sums run over pages in order, loads batched.
template <class ES>
__device__ __forceinline__ void attn_count_merge(const MegaParams& P, int n0, int nunits, int w, int lane, ES& es) {
  const int tid = threadIdx.x - 64;
  const int grp = P.heads / P.kv_heads;
  if (tid < nunits * kAttnRows) {
    const int k = tid / kAttnRows, r = tid % kAttnRows;
    const int t0 = es.ulist[k][0], t1 = es.ulist[k][1], kvh = es.ulist[k][2], s = es.ulist[k][3];
    int f = 0;
    if (t0 + r < t1) {
      const int t = t0 + r, pos = n0 + t;
      if (s <= pos / kPage) {
        unsigned* cnt = P.acnt + size_t(t) * P.kv_heads + kvh;
        const unsigned old = atom_add_acq_rel(cnt, 1u);
        if (old == unsigned(pos / kPage)) {
          f = 1;
          *cnt = 0u;
        }
      }
    }
    es.rflag[tid] = f;
  }
  wk_bar();
  for (int it = w; it < nunits * kAttnRows * grp; it += 4) {
    const int kr = it / grp, hh = it % grp;
    if (!es.rflag[kr]) continue;
    const int k = kr / kAttnRows;
    const int t = es.ulist[k][0] + kr % kAttnRows, kvh = es.ulist[k][2];
    attn_merge_one(P, n0, t, kvh * grp + hh, lane);
  }
  wk_bar();
}


// Partial slot of a piece: slot 0 holds a CTA's first tile, slot 1 its last
// (a CTA's middle tiles are whole and never stored). For the pieces of a
// tile, every CTA after c_first starts its range inside the tile (slot 0);
// c_first's piece is its first tile only when its range starts on the tile.
__device__ __forceinline__ int piece_off_slot(int cc, int slot, int m) { return (cc * 2 + slot) * kMaxWindow * 128 + m; }
__device__ __forceinline__ int tag_off_slot(int cc, int slot, int m) { return (cc * 2 + slot) * 128 + m; }
__device__ __forceinline__ int first_piece_slot(int c_first, int tile, const Gemm& g) {
  return sk_start(c_first, g.G, g.T) == tile * g.KB ? 0 : 1;
}

// Few-row passes (decode): a piece's partial is published as one 64-bit
// relaxed store of (tag, fp32 bits) — single-copy atomic, so a reader that sees
// the pass/phase tag sees the value, with no fence or arrival counter on the
// writer's side. The tile's finaliser is fixed: the CTA holding the tile's
// first k-block (for it that piece is the last of its range, so it finishes
// last) — it adds its own accumulator from registers and polls the others.
__device__ __forceinline__ void st_tagged(unsigned long long* p, unsigned tag, float v) {
  const unsigned long long w = (static_cast<unsigned long long>(tag) << 32) | __float_as_uint(v);
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long ld_tagged(const unsigned long long* p) {
  unsigned long long w;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  return w;
}

// Finaliser of a split tile in a 1-row pass (decode): own partial (CTA
// c_first) plus the tagged partials of CTAs c_first+1 .. c_first+npieces-1,
// summed in CTA order (the order of the wide finalisation), then the phase's
// finishing math. The O/D residual load is issued with the partial loads.
template <class ES>
__device__ __forceinline__ void finish_tagged(const MegaParams& P, int kind, int layer, int n0, int tile, int m, int q,
                                              int lane, int c_first, int npieces, const Gemm& g, unsigned tag, float own,
                                              ES& es) {
  const unsigned long long* part = P.tags;
  EpiPre pre;
  epi_load<1>(P, kind, 1, n0, tile, m, 0, pre);
  unsigned long long w[7];
#pragma unroll
  for (int pc = 1; pc < 8; ++pc)
    if (pc < npieces) w[pc - 1] = ld_tagged(part + tag_off_slot(c_first + pc, 0, m));
  bool again = true;
  PS_SPIN_START;
  while (again) {
    PS_SPIN_CHECK;
    again = false;
#pragma unroll
    for (int pc = 1; pc < 8; ++pc)
      if (pc < npieces && unsigned(w[pc - 1] >> 32) != tag) {
        w[pc - 1] = ld_tagged(part + tag_off_slot(c_first + pc, 0, m));
        again = true;
      }
  }
  float v[8];
  v[0] = own;
#pragma unroll
  for (int pc = 1; pc < 8; ++pc)
    if (pc < npieces) v[0] += __uint_as_float(unsigned(w[pc - 1]));
  finish_chunk<1>(P, kind, layer, 1, n0, tile, m, q, lane, 0, v, es, pre);
}


// A split tile this CTA finalises a row share of (wide passes).
struct DefTile {
  int tile, c_first, npieces, r_lo, r_hi, slot0;
};

// (v, id) ahead of (v2, id2) in the (-score, id) order of topk_tokens (lm.py:139-145)
__device__ __forceinline__ bool tk_before(float v, int i, float v2, int i2) { return v > v2 || (v == v2 && i < i2); }
__device__ __forceinline__ void tk_cswap(float& va, int& ia, float& vb, int& ib) {
  if (tk_before(vb, ib, va, ia)) {
    const float tv = va;
    const int ti = ia;
    va = vb;
    ia = ib;
    vb = tv;
    ib = ti;
  }
}

// Fused top-k (wide LM epilogue): the best L = P.topk_list (value, id) of one row's
// 128 logits of one LM tile (4 per lane), best first, into tk_val / tk_idx.
// Each lane sorts its 4; every round the warp's (max, lowest id) head is
// selected (a total order: ties cannot split) and popped by its owner.
__device__ __forceinline__ void warp_topl(const MegaParams& P, int tile, int t, float (&v)[4], int (&id)[4], int lane) {
  tk_cswap(v[0], id[0], v[1], id[1]);
  tk_cswap(v[2], id[2], v[3], id[3]);
  tk_cswap(v[0], id[0], v[2], id[2]);
  tk_cswap(v[1], id[1], v[3], id[3]);
  tk_cswap(v[1], id[1], v[2], id[2]);
  float mv = -INFINITY;
  int mi = 0x7fffffff;
  const int L = P.topk_list;
#pragma unroll
  for (int r = 0; r < kTopkList; ++r) {
    if (r >= L) break;
    float hv = v[0];
    int hi = id[0];
    warp_argmax(hv, hi);
    if (id[0] == hi) {  // owner pops its head
      v[0] = v[1]; id[0] = id[1];
      v[1] = v[2]; id[1] = id[2];
      v[2] = v[3]; id[2] = id[3];
      v[3] = -INFINITY; id[3] = 0x7fffffff;
    }
    if (lane == r) {
      mv = hv;
      mi = hi;
    }
  }
  if (lane < L) {
    const size_t o = (size_t(tile) * kTopkRows + t) * kTopkList + lane;
    P.tk_val[o] = mv;
    P.tk_idx[o] = mi;
  }
}

// One row t of the vectorised finishing math: features 4*lane .. +3 of
// `tile` (acc = their fp32 sums, X = the row's residual / RoPE inputs).
template <class ES>
__device__ __forceinline__ void vec_finish_row(const MegaParams& P, int kind, int layer, int n0, int w, int lane,
                                               int tile, int t, float4 acc, const float* X, ES& es) {
  const int hd = P.hd, half = hd >> 1;
  const int f0 = 4 * lane;
  const int n = tile * 128 + f0;
  if (kind == PH_QKV) {
    const int rr = n & (hd - 1), pi0 = rr >> 1;  // features f0, f0+1 = dims pi0, pi0+half; f0+2, f0+3 = pi0+1, ..
    const bool is_q = n < P.qd, is_k = !is_q && n < P.qd + P.kvd;
    float bias[4] = {0.f, 0.f, 0.f, 0.f};
    if (P.qkv_bias) {
      const __nv_bfloat16* bp = P.qkv_bias + size_t(layer) * (P.qd + 2 * P.kvd) + n;
#pragma unroll
      for (int e = 0; e < 4; ++e) bias[e] = __bfloat162float(bp[e]);
    }
    const float rs = es.rstd[t];
    const float v0 = epi_scale_bias(acc.x, rs, bias[0]), v1 = epi_scale_bias(acc.y, rs, bias[1]);
    const float v2 = epi_scale_bias(acc.z, rs, bias[2]), v3 = epi_scale_bias(acc.w, rs, bias[3]);
    float o0 = v0, o1 = v1, o2 = v2, o3 = v3;
    if (is_q || is_k) {
      const float4 cs = *reinterpret_cast<const float4*>(X + 2 * pi0);  // (c, s) of pi0, pi0+1 (X: this row's RoPE)
      o0 = rope_even(v0, v1, cs.x, cs.y);
      o1 = rope_odd(v1, v0, cs.x, cs.y);
      o2 = rope_even(v2, v3, cs.z, cs.w);
      o3 = rope_odd(v3, v2, cs.z, cs.w);
    }
    const __nv_bfloat162 lo = __floats2bfloat162_rn(o0, o2), hi = __floats2bfloat162_rn(o1, o3);
    const int col = n - rr + pi0;  // original column of dim pi0 (the odd rows are dims + half)
    __nv_bfloat16* d;
    if (is_q) {
      d = P.q + size_t(t) * P.qd + col;
    } else {
      const int pos = n0 + t;
      const int cc = col - P.qd - (is_k ? 0 : P.kvd);
      const int h = cc >> P.hd_shift;
      const int page = es.pg[(pos >> 6) - (n0 >> 6)];
      d = (is_k ? P.kpool : P.vpool) + size_t(layer) * P.g.layer_stride() +
          ((size_t(page) * P.g.kv_heads + h) * kPage + (pos & (kPage - 1))) * hd + (cc & (hd - 1));
    }
    *reinterpret_cast<__nv_bfloat162*>(d) = lo;
    *reinterpret_cast<__nv_bfloat162*>(d + half) = hi;
  } else if (kind == PH_GU) {
    const float rs = es.rstd[t];
    const float g0 = __fmul_rn(acc.x, rs), u0 = __fmul_rn(acc.y, rs);
    const float g1 = __fmul_rn(acc.z, rs), u1 = __fmul_rn(acc.w, rs);
    *reinterpret_cast<__nv_bfloat162*>(P.act + size_t(t) * P.I + tile * 64 + 2 * lane) =
        __floats2bfloat162_rn(swiglu(g0, u0), swiglu(g1, u1));
  } else if (kind == PH_O || kind == PH_D) {
    const float4 xo = *reinterpret_cast<const float4*>(X + f0);  // (X: this row's residual)
    const float4 xi = make_float4(__fadd_rn(xo.x, acc.x), __fadd_rn(xo.y, acc.y), __fadd_rn(xo.z, acc.z),
                                  __fadd_rn(xo.w, acc.w));
    *reinterpret_cast<float4*>(P.x + size_t(t) * P.H + n) = xi;
    const bool to_hn = kind == PH_D && layer == P.L - 1;
    __nv_bfloat16* dst = (to_hn ? P.hn_cache + size_t(n0 + t) * P.H : P.xb + size_t(t) * P.H) + n;
    const __nv_bfloat162 b01 = __floats2bfloat162_rn(xi.x, xi.y), b23 = __floats2bfloat162_rn(xi.z, xi.w);
    uint2 pk;
    pk.x = *reinterpret_cast<const uint32_t*>(&b01);
    pk.y = *reinterpret_cast<const uint32_t*>(&b23);
    *reinterpret_cast<uint2*>(dst) = pk;
    float s0 = __fmul_rn(xi.x, xi.x), s1 = __fmul_rn(xi.y, xi.y), s2 = __fmul_rn(xi.z, xi.z), s3 = __fmul_rn(xi.w, xi.w);
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      s3 += __shfl_xor_sync(0xffffffffu, s3, o);
    }
    const float tot = (s0 + s2) + (s1 + s3);
    if ((lane & 7) == 0) P.ssq_part[size_t(tile * 4 + (lane >> 3)) * kMaxWindow + t] = tot;
  } else {  // PH_LM
    const float rs = es.rstd[t];
    const float a4[4] = {acc.x, acc.y, acc.z, acc.w};
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    float tv[4];
    int ti[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      tv[e] = -INFINITY;
      ti[e] = 0x7fffffff;
      if (n + e < P.vocab_local) {
        const float lv = epi_scale_bias(a4[e], rs, P.lm_bias[P.v_begin + n + e]);
        if (P.logits_out) P.logits_out[size_t(t) * P.ld_logits + n + e] = lv;
        argmax_merge(bv, bi, lv, P.v_begin + n + e);
        tv[e] = lv;
        ti[e] = P.v_begin + n + e;
      }
    }
    if (P.topk_list) warp_topl(P, tile, t, tv, ti, lane);
    warp_argmax(bv, bi);
    if (lane == 0) argmax_merge(es.am_v[w][t], es.am_i[w][t], bv, bi);
  }
}

// Wide passes: a split tile's row share, finalised from shared memory with a
// vectorised thread map. The pieces' partial rows (contiguous per piece slot)
// and the per-row inputs (residual rows for O/D, RoPE rows for QKV) are
// fetched with 1D bulk copies by one thread onto an mbarrier; then thread
// (fg, w) handles features 4fg..4fg+3 of rows r_lo+w, r_lo+w+4, ... RoPE and
// SwiGLU partners are in-thread; the O/D row sums of squares follow warp_sum's
// pairing (feature bits 4,3,2 across lanes, then 1,0 in-thread), so every value
// is bitwise the TMEM-lane epilogue's (finish_chunk / finish_tagged).
template <class ES>
__device__ __forceinline__ void finish_share_vec(const MegaParams& P, int kind, int layer, int n0, int w, int lane,
                                                 const DefTile& T, float* S, int cap_floats, uint32_t wbar,
                                                 uint32_t& wphase, ES& es, int trace_p = -1) {
  const int tid = threadIdx.x - 64;
  const int np = T.npieces;
  const bool has_x = kind == PH_O || kind == PH_D;
  const int hd = P.hd, half = hd >> 1;
  const int rope_row = half * 2;  // floats per RoPE row (cos, sin pairs)
  // staged per row: the pieces' partials, and for O/D the residual row (its
  // boxes are kXBoxRows rows, so the residual area is padded to a multiple);
  // QKV's RoPE (cos, sin) is read straight from the (L1-cached) table
  const int per_row = np * 128 + (has_x ? 128 : 0);
  const int batch = has_x ? (cap_floats - kXBoxRows * 128) / per_row / kXBoxRows * kXBoxRows  // >= 8 rows
                          : cap_floats / per_row;
  const int f0 = 4 * lane;               // this thread's first feature within the tile
  for (int b0 = T.r_lo; b0 < T.r_hi; b0 += batch) {
    const int nb = min(batch, T.r_hi - b0);
    float* X = S + np * nb * 128;
    if (tid == 0) {
      fence_proxy_async_global();  // generic writes of other CTAs (acquired) -> async-proxy reads
      if (trace_p >= 0 && b0 == T.r_lo) stamp(P, trace_p, blockIdx.x, gridDim.x, 10);
      const int xboxes = has_x ? (nb + kXBoxRows - 1) / kXBoxRows : 0;
      const uint32_t bytes = uint32_t(np * nb * 512 + xboxes * kXBoxRows * 512);
      mbar_expect_tx(wbar, bytes);
      for (int pc = 0; pc < np; ++pc)
        bulk_g2s(smem_u32(S + pc * nb * 128),
                 P.part + piece_off_slot(T.c_first + pc, pc == 0 ? T.slot0 : 0, 0) + size_t(b0) * 128, nb * 512, wbar);
      for (int j = 0; j < xboxes; ++j)  // residual rows b0 + 8j .., 128 features of the tile
        tma_load_2d(smem_u32(X + j * kXBoxRows * 128), P.xrows, wbar, T.tile * 128, b0 + j * kXBoxRows);
      if (trace_p >= 0 && b0 == T.r_lo) stamp(P, trace_p, blockIdx.x, gridDim.x, 3);
    }
    mbar_wait(wbar, wphase);
    wphase ^= 1u;
    if (trace_p >= 0 && tid == 0 && b0 == T.r_lo) stamp(P, trace_p, blockIdx.x, gridDim.x, 14);
    for (int r = w; r < nb; r += kWorkerWarps) {
      const int t = b0 + r;
      float4 acc = *reinterpret_cast<const float4*>(S + r * 128 + f0);
      for (int pc = 1; pc < np; ++pc) {
        const float4 o = *reinterpret_cast<const float4*>(S + (pc * nb + r) * 128 + f0);
        acc.x += o.x;
        acc.y += o.y;
        acc.z += o.z;
        acc.w += o.w;
      }
      const float* xin = has_x ? X + r * 128 : reinterpret_cast<const float*>(P.rope) + size_t(n0 + t) * rope_row;
      vec_finish_row(P, kind, layer, n0, w, lane, T.tile, t, acc, xin, es);
    }
    if (trace_p >= 0 && tid == 0 && b0 == T.r_lo) stamp(P, trace_p, blockIdx.x, gridDim.x, 15);
    wk_bar();  // the staging area is reused by the next batch / tile
  }
}

}  // namespace

// kWide: passes of more than one row (verify / prefill chunks / Jacobi
// windows) — split tiles are finalised by all their pieces' CTAs (row shares
// of fp32 partials). !kWide: 1-row decode steps — tagged single-word partials
// and a fixed finaliser. Two instantiations keep each one's code and register
// allocation free of the other's paths; the per-row arithmetic is the same
// source, so a row is bitwise identical in both (tests/test_gpu_parity.py).
template <bool kWide>
__global__ void __launch_bounds__(kWide ? 256 : 192, 1) mega_kernel(const __grid_constant__ MegaParams P) {
  // the launch shape is fixed per instantiation: lets the inlined helpers fold
  // the worker count (kWorkers, kWorkerWarps, wk_bar) to a constant
  __builtin_assume(blockDim.x == (kWide ? 256u : 192u));
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // [full x kMaxStages][empty x kMaxStages][acc_full x 2][acc_empty x 2][workers' staging]
  __shared__ uint64_t bars[2 * kMaxStages + 4 + 1];
  __shared__ uint32_t tmem_holder;
  __shared__ EpiSmemT<kWide ? kMaxWindow : 16> es;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x, G = gridDim.x;
  const int ST = P.stages;
  // partial tags of this pass: epoch * nphases + phase (the epoch advances once per pass)
  const unsigned epoch = *P.epoch;
  const unsigned tag0 = epoch * unsigned(3 + 5 * P.L);
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int b_bytes = P.ntok * 128;
  auto a_tile = [&](int s) { return base + size_t(s) * (kTileABytes + b_bytes); };
  auto b_tile = [&](int s) { return a_tile(s) + kTileABytes; };
  const AttnSmem A = attn_smem(base + size_t(ST) * (kTileABytes + b_bytes), P.hd, P.heads / P.kv_heads, kWide, P.H);
  const uint32_t full0 = smem_u32(&bars[0]), empty0 = smem_u32(&bars[kMaxStages]);
  const uint32_t acc_full0 = smem_u32(&bars[2 * kMaxStages]), acc_empty0 = smem_u32(&bars[2 * kMaxStages + 2]);
  const uint32_t wbar = smem_u32(&bars[2 * kMaxStages + 4]);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full0 + 8 * b, 1);
      mbar_init(acc_empty0 + 8 * b, 1);
    }
    mbar_init(wbar, 1);  // workers' bulk staging (wide finalisation)
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_holder)),
                 "r"(2 * P.acc_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const int n0 = P.ctx->n0;
  const int rows = P.ctx->rows;
  const int nphases = 3 + 5 * P.L;
  // LM-only passes (logits of resident rows) start at the LM phase; barrier
  // generation g counts the phases completed so far (the embed is generation 1)
  const int p_first = P.lm_only ? 1 + 5 * P.L : 1;

  if (warp == 0) {
    // ======================= TMA producer =======================
    // Weight tiles of a phase are issued into the ring before waiting for the
    // barrier that guards its activations; weights stream with an L2
    // evict-first policy (read once per pass) so activations, KV pages and
    // split-K partials stay L2-resident. (A TMA L2-prefetch cursor running
    // further ahead was measured slower: prefetched lines were evicted before
    // use and DRAM traffic grew 1.8x — see DESIGN.md.)
    if (lane == 0) {
      grid_wait(P.bar, unsigned(G));  // embed done (and the stop flag settled)
      if (!P.ctx->stop) {
        const int xrow_lm = n0;
        const uint64_t pol_stream = l2_policy_evict_first();
        uint32_t it = 0;
        for (int p = p_first; p < nphases; ++p) {
          const int kind = phase_kind(p, P.L);
          if (kind == PH_ATTN || kind == PH_FINAL) continue;
          const Gemm g = gemm_of(P, kind);
          const int kb_lo = c < g.G ? sk_start(c, g.G, g.T) : 0, kb_hi = c < g.G ? sk_start(c + 1, g.G, g.T) : 0;
          const int nk = kb_hi - kb_lo;
          const PieceOrder po(kb_lo, kb_hi, g.KB);
          const CUtensorMap* wm = wmap_of(P, p, kind);
          const CUtensorMap* xm = xmap_of(P, kind);
          const int xrow = kind == PH_LM ? xrow_lm : 0;
          const uint32_t tx = kTileABytes + b_bytes;
          const int pre = min(min(nk, ST), P.pre_max);
          // Block cursor over the pieces in processing order, and the ring
          // slot/parity, advanced incrementally: this single thread issues
          // every load of the CTA, so no per-block divisions.
          struct Cursor {
            const PieceOrder& po;
            int KB, j, x, hi, tile, kb;
            __device__ __forceinline__ void start(int jj) {
              j = jj;
              po.piece(j, x, hi);
              tile = x / KB;
              kb = x - tile * KB;
            }
            __device__ __forceinline__ void next() {
              ++x;
              if (++kb == KB) {
                kb = 0;
                ++tile;
              }
              if (x == hi && j + 1 < po.npieces()) start(j + 1);
            }
          };
          Cursor cur{po, g.KB, 0, 0, 0, 0, 0}, bcur{po, g.KB, 0, 0, 0, 0, 0};
          if (nk > 0) {
            cur.start(0);
            bcur.start(0);
          }
          uint32_t s0 = it % ST, ph0 = (it / ST) & 1;  // slot and parity of this phase's first block
          uint32_t s = s0, ph = ph0;
          auto bump = [&](uint32_t& ss, uint32_t& pp) {
            if (++ss == uint32_t(ST)) {
              ss = 0;
              pp ^= 1u;
            }
          };
          for (int i = 0; i < pre; ++i, cur.next(), bump(s, ph)) {
            mbar_wait(empty0 + 8 * s, ph ^ 1);
            mbar_expect_tx(full0 + 8 * s, tx);
            tma_load_2d_hint(smem_u32(a_tile(s)), wm, full0 + 8 * s, cur.kb * kBK, cur.tile * 128, pol_stream);
          }
          // HBM is idle while the grid finishes the previous phase (its tail,
          // and all of ATTN): the next P.pf[kind] boxes of this CTA's range
          // beyond the ring go to L2 now, and the ring reads them from there
          for (int i = pre; i < nk && i < pre + P.pf[kind]; ++i) {
            const int x = kb_lo + i;
            tma_prefetch_2d(wm, (x % g.KB) * kBK, (x / g.KB) * 128);
          }
          grid_wait(P.bar, unsigned(G) * unsigned(p - p_first + 1));  // activations of this phase are complete
          stamp(P, p, c, G, 0);
          fence_proxy_async_global();
          {
            uint32_t sb = s0, pb = ph0;
            for (int i = 0; i < pre; ++i, bcur.next(), bump(sb, pb))
              tma_load_2d(smem_u32(b_tile(sb)), xm, full0 + 8 * sb, bcur.kb * kBK, xrow);
          }
          for (int i = pre; i < nk; ++i, cur.next(), bump(s, ph)) {
            mbar_wait(empty0 + 8 * s, ph ^ 1);
            mbar_expect_tx(full0 + 8 * s, tx);
            tma_load_2d_hint(smem_u32(a_tile(s)), wm, full0 + 8 * s, cur.kb * kBK, cur.tile * 128, pol_stream);
            tma_load_2d(smem_u32(b_tile(s)), xm, full0 + 8 * s, cur.kb * kBK, xrow);
          }
          stamp(P, p, c, G, 12);
          it += nk;
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer =======================
    if (lane == 0) {
      grid_wait(P.bar, unsigned(G));
      if (!P.ctx->stop) {
        const uint32_t idesc = idesc_bf16(P.ntok);
        uint32_t it = 0, acc_it = 0;
        uint32_t ms = 0, mph = 0;  // ring slot / parity of block `it`, advanced incrementally
        for (int p = p_first; p < nphases; ++p) {
          const int kind = phase_kind(p, P.L);
          if (kind == PH_ATTN || kind == PH_FINAL) continue;
          const Gemm g = gemm_of(P, kind);
          const int kb_lo = c < g.G ? sk_start(c, g.G, g.T) : 0, kb_hi = c < g.G ? sk_start(c + 1, g.G, g.T) : 0;
          const PieceOrder po(kb_lo, kb_hi, g.KB);
          for (int j = 0; j < po.npieces(); ++j) {  // one piece per tile touched by this CTA
            int x, piece_hi;
            po.piece(j, x, piece_hi);
            const uint32_t b = acc_it & 1, aph = (acc_it >> 1) & 1;
            mbar_wait(acc_empty0 + 8 * b, aph ^ 1);
            tc_fence_after();
            const uint32_t dcol = tmem + b * uint32_t(P.acc_cols);
            for (int y = x; y < piece_hi; ++y, ++it) {
              const uint32_t s = ms, ph = mph;
              if (++ms == uint32_t(ST)) {
                ms = 0;
                mph ^= 1u;
              }
              mbar_wait(full0 + 8 * s, ph);
              tc_fence_after();
              const uint32_t sa = smem_u32(a_tile(s)), sb = smem_u32(b_tile(s));
#pragma unroll
              for (int k = 0; k < kBK / 16; ++k)
                umma_bf16(dcol, umma_desc_sw128(sa + k * 32), umma_desc_sw128(sb + k * 32), idesc,
                          (y > x || k > 0) ? 1u : 0u);
              umma_commit(empty0 + 8 * s);
            }
            umma_commit(acc_full0 + 8 * b);
            ++acc_it;
          }
          stamp(P, p, c, G, 13);
        }
      }
    }
  } else {
    // ======================= workers: epilogue / attention / embed =======================
    const int w = warp - 2;       // 0..3
    const int q = warp & 3;       // TMEM lane quadrant
    const int m = q * 32 + lane;  // row within a 128-row tile
    const int tid = threadIdx.x - 64;
    uint32_t acc_it = 0;
    uint32_t wphase = 0;  // parity of the workers' staging mbarrier
    if (kWide && tid < 8) {
      const int lp = (n0 >> 6) + tid;
      es.pg[tid] = lp <= ((n0 + rows - 1) >> 6) ? P.page_table[lp] : 0;
    }
    // ---- phase 0: embedding rows (t ≡ c mod G) ----
    for (int t = c; t < (P.lm_only ? 0 : rows); t += G) {
      const int pos = n0 + t;
      if (tid == 0) {
        int tok;
        if (P.decode) {
          tok = P.argmax_pos[pos - 1];
          if (P.ctx->stop_on_eos && tok == kEos) P.ctx->stop = 1;
        } else {
          tok = P.tok_in[t];
        }
        P.tokens_dev[pos] = tok;
        es.flag = tok;
      }
      wk_bar();
      const int tok = es.flag;
      const uint4* e = reinterpret_cast<const uint4*>(P.embed + size_t(tok) * P.H);
      uint4* ob = reinterpret_cast<uint4*>(P.xb + size_t(t) * P.H);
      float* xr = P.x + size_t(t) * P.H;
      float ss = 0.f;
      // the first 4 worker warps only, stride 128: rstd0's sum tree is the same
      // in both instantiations
      for (int cc = tid; w < 4 && cc < P.H / 8; cc += 128) {
        const uint4 raw = e[cc];
        ob[cc] = raw;
        const __nv_bfloat16* vv = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float f = __bfloat162float(vv[i]);
          xr[cc * 8 + i] = f;
          ss = fmaf(f, f, ss);
        }
      }
      ss = warp_sum(ss);
      if (lane == 0 && w < 4) es.red_v[w][0] = ss;
      wk_bar();
      if (tid == 0) P.rstd0[t] = 1.0f / sqrtf((((es.red_v[0][0] + es.red_v[1][0]) + es.red_v[2][0]) + es.red_v[3][0]) / float(P.H) + P.eps);
      wk_bar();
    }
    wk_bar();
    if (tid == 0) {
      stamp(P, 0, c, G, 2);
      grid_arrive(P.bar);
    }
    const int rw = kWide ? attention_rows_wide(P, rows, n0, G) : kAttnRows;  // attention unit rows
    for (int p = p_first; p < nphases; ++p) {
      const int kind = phase_kind(p, P.L);
      const int layer = kind == PH_LM ? P.L - 1 : (p - 1) / 5;
      if (tid == 0) {
        grid_wait(P.bar, unsigned(G) * unsigned(p - p_first + 1));
        stamp(P, p, c, G, 1);
      }
      wk_bar();
      if (P.ctx->stop) break;
      // wide passes: stage the RMSNorm partials now, reduce them at first use
      bool rstd_pending = false;
      if (kWide && !P.lm_only && (kind == PH_GU || kind == PH_LM || (kind == PH_QKV && layer > 0)) &&
          rstd_stage_fits(P, A, rows)) {
        rstd_stage_issue(P, A, rows, w, lane);
        cp_async_commit();
        rstd_pending = true;
      }
      if (kind == PH_QKV) {
        // keys cached by earlier passes for this CTA's first attention unit of
        // the layer: requested now, consumed after the next barrier
        int un = 0;
        const AttnUnit U0 = attn_unit_from(P, kWide ? rw : kAttnRows, rows, n0, c, G, un);
        if (U0.valid) attn_issue<kWide>(P, layer, U0, n0, A, 0, 0, tid);
        if (U0.valid || rstd_pending) cp_async_commit();  // (the staged partials are the group before)
      }
      auto ensure_rstd = [&]() {
        if (!rstd_pending) return;
        if (kind == PH_QKV) cp_async_wait<1>(); else cp_async_wait<0>();
        wk_bar();
        rstd_stage_reduce(P, A, rows, w, lane, es);
        wk_bar();
        if (kind == PH_LM && c == 0)
          for (int t = tid; t < rows; t += kWorkers) P.rstd_cache[n0 + t] = es.rstd[t];
        rstd_pending = false;
      };
      if (kind == PH_FINAL) {
        // argmax of every row over the per-CTA partials of the LM phase;
        // rows are spread over CTAs (t = c, c+G, ...), one warp per row
        for (int t = c * kWorkerWarps + w; t < rows; t += kWorkerWarps * G) {
          float bv = -INFINITY;
          int bi = 0x7fffffff;
          float vv[8];
          int ii[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {  // G <= 256
            const int cc = lane + 32 * u;
            vv[u] = cc < G ? __ldcg(P.am_val + size_t(cc) * kMaxWindow + t) : -INFINITY;
            ii[u] = cc < G ? __ldcg(P.am_idx + size_t(cc) * kMaxWindow + t) : 0x7fffffff;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) argmax_merge(bv, bi, vv[u], ii[u]);
          warp_argmax(bv, bi);
          if (kWide && P.topk_list) {
            // best L of the row over every LM tile's list: lane takes tiles
            // lane, lane + 32, ... (heads of four requested at once) into a
            // sorted local list, then the warp selects heads as in warp_topl;
            // the rank of the row's next token is its position there (L: not
            // among them)
            const int L = P.topk_list;
            const int ntl = (P.vocab_local + 127) / 128;
            float lv[kTopkList];
            int li[kTopkList];
#pragma unroll
            for (int k = 0; k < kTopkList; ++k) {
              lv[k] = -INFINITY;
              li[k] = 0x7fffffff;
            }
            auto worst = [&](float& v, int& i) {  // lv[L - 1], li[L - 1]
              v = lv[0];
              i = li[0];
#pragma unroll
              for (int k = 1; k < kTopkList; ++k)
                if (k < L) {
                  v = lv[k];
                  i = li[k];
                }
            };
            for (int tl0 = lane; tl0 < ntl; tl0 += 32 * 4) {
              float hv[4];
              int hi[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int tl = tl0 + 32 * u;
                const size_t o = (size_t(tl) * kTopkRows + t) * kTopkList;
                hv[u] = tl < ntl ? __ldcg(P.tk_val + o) : -INFINITY;
                hi[u] = tl < ntl ? __ldcg(P.tk_idx + o) : 0x7fffffff;
              }
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const size_t o = (size_t(tl0 + 32 * u) * kTopkRows + t) * kTopkList;
                float v = hv[u];
                int i = hi[u];
                for (int k = 0; k < L; ++k) {  // tile lists are sorted: stop at the first that misses
                  if (k > 0) {
                    v = __ldcg(P.tk_val + o + k);
                    i = __ldcg(P.tk_idx + o + k);
                  }
                  float wv;
                  int wi;
                  worst(wv, wi);
                  if (!tk_before(v, i, wv, wi)) break;
#pragma unroll
                  for (int q = 0; q < kTopkList; ++q) tk_cswap(lv[q], li[q], v, i);  // insert, shifting down
                }
              }
            }
            const int tok = __ldcg(P.tokens_dev + n0 + t + 1);
            int rank = L;
#pragma unroll
            for (int r = 0; r < kTopkList; ++r) {
              if (r >= L) break;
              float hv = lv[0];
              int hi = li[0];
              warp_argmax(hv, hi);
              if (li[0] == hi) {
#pragma unroll
                for (int q = 0; q + 1 < kTopkList; ++q) {
                  lv[q] = lv[q + 1];
                  li[q] = li[q + 1];
                }
                lv[kTopkList - 1] = -INFINITY;
                li[kTopkList - 1] = 0x7fffffff;
              }
              if (hi == tok && rank == L) rank = r;
            }
            if (lane == 0) P.rank_pos[n0 + t] = rank;
          }
          if (lane == 0) {
            P.argmax_pos[n0 + t] = bi;
            if (P.keys) {
              unsigned uu = __float_as_uint(bv);
              uu = (uu & 0x80000000u) ? ~uu : (uu | 0x80000000u);
              P.keys[t] = (static_cast<unsigned long long>(uu) << 32) | (0xFFFFFFFFull - unsigned(bi));
            }
            if (t == 0 && P.advance) {  // decode: one row, handled by CTA 0 warp 0
              P.ctx->n0 = n0 + 1;
              P.ctx->step += 1;
            }
          }
        }
      } else if (kind == PH_ATTN && kWide) {
        // units (kv head, page, 16-row block), double-buffered K/V; the first
        // unit's cached keys were requested in the QKV phase
        int un = 0, un2 = 0;
        AttnUnit cur = attn_unit_from(P, rw, rows, n0, c, G, un);
        AttnUnit nxt{0, 0, 0, 0, false};
        if (cur.valid) {
          attn_issue<kWide>(P, layer, cur, n0, A, 0, 1, tid);
          cp_async_commit();
          nxt = attn_unit_from(P, rw, rows, n0, un, G, un2);
          if (nxt.valid) {
            attn_issue<kWide>(P, layer, nxt, n0, A, 1, 0, tid);
            attn_issue<kWide>(P, layer, nxt, n0, A, 1, 1, tid);
          }
          cp_async_commit();
        }
        for (int i = 0; cur.valid; ++i) {
          uint32_t qf[8][4];
          attn_q_frags_wide(P, cur, w, lane, qf);
          cp_async_wait<1>();
          wk_bar();
          if (tid == 0 && i == 0) stamp(P, p, c, G, 7);
          attention_unit_wide(P, cur, n0, A, i & 1, w, lane, qf);
          wk_bar();  // buffer i&1 is free again
          if (tid == 0 && i == 0) stamp(P, p, c, G, 9);
          AttnUnit nn{0, 0, 0, 0, false};
          int un3 = un2;
          if (nxt.valid) nn = attn_unit_from(P, rw, rows, n0, un2, G, un3);
          if (nn.valid) {
            attn_issue<kWide>(P, layer, nn, n0, A, i & 1, 0, tid);
            attn_issue<kWide>(P, layer, nn, n0, A, i & 1, 1, tid);
          }
          cp_async_commit();
          cur = nxt;
          nxt = nn;
          un2 = un3;
        }
        // every page of every (row, head) is written: grid-wide sync on a
        // second counter, then the merges spread over all warps of the grid
        if (tid == 0) {
          stamp(P, p, c, G, 10);
          grid_arrive(P.bar2);
          grid_wait(P.bar2, unsigned(G) * unsigned(layer + 1));
        }
        wk_bar();
        const int items = rows * P.heads;
        for (int it = c * kWorkerWarps + w; it < items; it += kWorkerWarps * G)
          attn_merge_one(P, n0, it / P.heads, it % P.heads, lane);
        if (tid == 0) stamp(P, p, c, G, 11);
      } else if (kind == PH_ATTN) {
        // decode: about one unit per CTA, so one operand buffer (the smem it
        // frees deepens the weight ring); the first unit's cached keys were
        // requested in the QKV phase
        int un = 0;
        AttnUnit cur = attn_unit_from(P, kAttnRows, rows, n0, c, G, un);
        for (int i = 0; cur.valid; ++i) {
          if (i > 0) attn_issue<kWide>(P, layer, cur, n0, A, 0, 0, tid);
          attn_issue<kWide>(P, layer, cur, n0, A, 0, 1, tid);
          cp_async_commit();
          cp_async_wait<0>();
          wk_bar();
          if (tid == 0 && i == 0) stamp(P, p, c, G, 7);
          attention_unit(P, cur, n0, A, 0, w, lane, i == 0 ? p : -1);  // ends with wk_bar
          if (tid == 0) {
            es.ulist[0][0] = cur.t0;
            es.ulist[0][1] = cur.t1;
            es.ulist[0][2] = cur.kvh;
            es.ulist[0][3] = cur.s;
          }
          wk_bar();
          attn_count_merge(P, n0, 1, w, lane, es);  // ends with wk_bar
          int un2 = un;
          cur = attn_unit_from(P, kAttnRows, rows, n0, un, G, un2);
          un = un2;
        }
      } else {
        if (P.lm_only) {  // LM head over resident rows: the final rstd of each position is cached
          for (int t = tid; t < rows; t += kWorkers) es.rstd[t] = P.rstd_cache[n0 + t];
          wk_bar();
        } else if ((kind == PH_QKV || kind == PH_GU || kind == PH_LM) && !rstd_pending) {
          load_rstd(P, kind == PH_QKV && layer == 0, rows, w, lane, es);
          wk_bar();
          if (kind == PH_LM && c == 0)
            for (int t = tid; t < rows; t += kWorkers) P.rstd_cache[n0 + t] = es.rstd[t];
        }
        const Gemm g = gemm_of(P, kind);
        const int kb_lo = c < g.G ? sk_start(c, g.G, g.T) : 0, kb_hi = c < g.G ? sk_start(c + 1, g.G, g.T) : 0;
        // per-phase arrival counters (zeroed before the pass): no resets, no reuse races
        unsigned* cnt = P.tile_cnt + size_t(p) * P.max_tiles;
        // 1-row pass (decode): pieces publish tagged partials and the tile's
        // first-block CTA finalizes (finish_tagged). Wider passes (verify /
        // prefill): every piece publishes without blocking and counts in,
        // then each piece's CTA finalizes its own share of the rows.
        constexpr bool spread = kWide;
        // wide phases where no CTA range holds a whole tile (QKV, O, D at the
        // 8B shape): every tile is split, so the finalisation is spread evenly
        // over the grid after one grid-wide sync instead of per-tile counters
        const bool all_split = kWide && (g.T + g.G - 1) / g.G < g.KB;
        int dtile0 = -1, dtile1 = -1;  // split tiles whose finalisation is deferred (<= 2 per CTA)
        if (kind == PH_LM) {
          constexpr int RW = decltype(es)::kRows;
          for (int e = tid; e < 6 * RW; e += kWorkers) {
            es.am_v[e / RW][e % RW] = -INFINITY;
            es.am_i[e / RW][e % RW] = 0x7fffffff;
          }
          wk_bar();
        }
        // wide, not all-split: finalise this CTA's row shares of its split tiles
        bool finalized = false;
        auto finalize_split_tiles = [&]() {
          // second pass: wait for the split tiles' pieces, then finalise this
          // CTA's row share of each (every piece's CTA takes a share)
          // Row shares are weighted so that every CTA finalises about the same
          // number of rows in total: a CTA with two split tiles (its first and
          // last piece) takes half-weight shares of each.
          auto split_pieces = [&](int cc) {
            const int lo = sk_start(cc, g.G, g.T), hi = sk_start(cc + 1, g.G, g.T);
            const int t0 = lo / g.KB, t1 = (hi - 1) / g.KB;
            const int first = (lo != t0 * g.KB || hi < (t0 + 1) * g.KB) ? 1 : 0;
            const int last = (t1 != t0 && hi != (t1 + 1) * g.KB) ? 1 : 0;
            return first + last;
          };
          auto def_of = [&](int tile) {
            const int c_first = sk_owner(tile * g.KB, g.G, g.T), c_last = sk_owner((tile + 1) * g.KB - 1, g.G, g.T);
            const int npieces = c_last - c_first + 1;
            int wsum = 0, wbefore = 0, wmine = 0;
            for (int pc = 0; pc < npieces; ++pc) {
              const int wt = split_pieces(c_first + pc) > 1 ? 1 : 2;
              if (c_first + pc < c) wbefore += wt;
              if (c_first + pc == c) wmine = wt;
              wsum += wt;
            }
            return DefTile{tile, c_first, npieces, wbefore * rows / wsum, (wbefore + wmine) * rows / wsum,
                           first_piece_slot(c_first, tile, g)};
          };
          // dtile1 is only set once dtile0 is
          const int nd = (dtile0 >= 0) + (dtile1 >= 0);
          DefTile D[2] = {dtile0 >= 0 ? def_of(dtile0) : DefTile{0, 0, 1, 0, 0, 0},
                          dtile1 >= 0 ? def_of(dtile1) : DefTile{0, 0, 1, 0, 0, 0}};
          if (tid == 0) {
            if (nd > 0) grid_wait(cnt + D[0].tile, unsigned(D[0].npieces));
            if (nd > 1) grid_wait(cnt + D[1].tile, unsigned(D[1].npieces));
            stamp(P, p, c, G, 7);
          }
          wk_bar();
          if (tid == 0) stamp(P, p, c, G, 8);
          // staging area: both attention buffers, except in QKV where buffer 0
          // holds the next ATTN phase's prefetched keys
          float* stage = reinterpret_cast<float*>(kind == PH_QKV ? A.K(1) : A.K(0));
          const int cap = (kind == PH_QKV ? A.buf : 2 * A.buf) / 4;
#pragma unroll
          for (int d = 0; d < 2; ++d)
            if (d < nd && D[d].r_lo < D[d].r_hi)
              finish_share_vec(P, kind, layer, n0, w, lane, D[d], stage, cap, wbar, wphase, es, d == 0 ? p : -1);
          if (tid == 0) stamp(P, p, c, G, 9);
          finalized = true;
        };
        const PieceOrder po(kb_lo, kb_hi, g.KB);
        // the workers are idle until the first accumulator: reduce the staged
        // RMSNorm partials now rather than on the tail's critical path
        if (kWide) ensure_rstd();
        for (int pj = 0; pj < po.npieces(); ++pj) {
          int x, piece_hi;
          po.piece(pj, x, piece_hi);
          const int tile = x / g.KB;
          const int c_first = sk_owner(tile * g.KB, g.G, g.T), c_last = sk_owner((tile + 1) * g.KB - 1, g.G, g.T);
          const int npieces = c_last - c_first + 1;  // <= 8 by the choice of g.G
          {
            const int n = tile * 128 + m;
            if (kind == PH_O || kind == PH_D) prefetch_l1(P.x + n);
            if (kind == PH_QKV) prefetch_l1(P.rope + size_t(n0) * (P.hd >> 1) + ((n % P.hd) >> 1));
            if (kind == PH_LM && n < P.vocab_local) prefetch_l1(P.lm_bias + P.v_begin + n);
          }
          // Wide GU / LM phases, a tile of exactly two pieces: the CTA holding the
          // tile's first k-blocks (c_first; for it the piece is the last of its
          // range) finalises the whole tile from its own accumulator plus the
          // partner's partial, which the partner (c_first + 1, its first piece)
          // published early in the phase — so neither waits for the other at
          // the tail. The sum own + partner is the CTA-order sum of the
          // row-share finalisation and of the decode finaliser (finish_tagged).
          const bool pair_tile = kWide && !all_split && npieces == 2 && (kind == PH_GU || kind == PH_LM) &&
                                 rows * 512 <= A.buf;
          float* const own_s = reinterpret_cast<float*>(A.K(0));
          float* const mate_s = reinterpret_cast<float*>(A.K(1));
          if (pair_tile && c == c_first && tid == 0) {
            // the partner's piece: acquire its arrival, then stage its rows
            // (bulk copy, overlapping this CTA's last k-blocks)
            grid_wait(cnt + tile, 1u);
            fence_proxy_async_global();
            mbar_expect_tx(wbar, uint32_t(rows) * 512u);
            bulk_g2s(smem_u32(mate_s), P.part + piece_off_slot(c + 1, 0, 0), uint32_t(rows) * 512u, wbar);
          }
          const uint32_t b = acc_it & 1, aph = (acc_it >> 1) & 1;
          mbar_wait(acc_full0 + 8 * b, aph);
          tc_fence_after();
          if (tid == 0) stamp(P, p, c, G, 4);
          const uint32_t trow = tmem + b * uint32_t(P.acc_cols) + (uint32_t(q * 32) << 16);
          if (pair_tile && c == c_first) {
            ensure_rstd();
            for (int c0 = 0; w < 4 && c0 < rows; c0 += 32) {  // TMEM lane quadrants: first 4 warps
              float v[32];
              tmem_ld32(trow + c0, v);
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (c0 + j < rows) own_s[(c0 + j) * 128 + m] = v[j];
            }
            tc_fence_before();
            wk_bar();
            if (tid == 0) mbar_arrive(acc_empty0 + 8 * b);
            mbar_wait(wbar, wphase);
            wphase ^= 1u;
            for (int t = w; t < rows; t += kWorkerWarps) {
              float4 acc = *reinterpret_cast<const float4*>(own_s + t * 128 + 4 * lane);
              const float4 o = *reinterpret_cast<const float4*>(mate_s + t * 128 + 4 * lane);
              acc.x += o.x;
              acc.y += o.y;
              acc.z += o.z;
              acc.w += o.w;
              vec_finish_row(P, kind, layer, n0, w, lane, tile, t, acc, own_s, es);
            }
            wk_bar();  // the staging areas are reused by the next tile
          } else if (kWide && npieces == 1 && (kind == PH_GU || kind == PH_LM) && rows * 512 <= 2 * A.buf) {
            // whole tile of a wide pass: accumulators -> smem [row][128] (a
            // transpose through the idle attention buffers), TMEM released, then
            // the vectorised row math (4 features per thread, as finish_share_vec)
            ensure_rstd();
            float* S = reinterpret_cast<float*>(A.K(0));
            for (int c0 = 0; w < 4 && c0 < rows; c0 += 32) {  // TMEM lane quadrants: first 4 warps
              float v[32];
              tmem_ld32(trow + c0, v);
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (c0 + j < rows) S[(c0 + j) * 128 + m] = v[j];
            }
            tc_fence_before();
            wk_bar();
            if (tid == 0) mbar_arrive(acc_empty0 + 8 * b);
            for (int t = w; t < rows; t += kWorkerWarps)
              vec_finish_row(P, kind, layer, n0, w, lane, tile, t, *reinterpret_cast<const float4*>(S + t * 128 + 4 * lane),
                             S, es);
            wk_bar();  // S is reused by the next tile
          } else if (npieces == 1) {
            ensure_rstd();
            // the next chunk's per-row inputs are in flight while this one finishes
            EpiPre cur, nxt;
            if (w < 4) epi_load(P, kind, rows, n0, tile, m, 0, cur);
            for (int c0 = 0; w < 4 && c0 < rows; c0 += 8) {  // TMEM lane quadrants: first 4 warps
              if (c0 + 8 < rows) epi_load(P, kind, rows, n0, tile, m, c0 + 8, nxt);
              float v[8];
              tmem_ld8(trow + c0, v);
              finish_chunk(P, kind, layer, rows, n0, tile, m, q, lane, c0, v, es, cur);
              cur = nxt;
            }
            tc_fence_before();
            wk_bar();
            if (tid == 0) mbar_arrive(acc_empty0 + 8 * b);
          } else if (!spread && c == c_first) {
            // fixed finaliser (few rows): own accumulator + the other pieces' tagged partials
            float v[8];
            tmem_ld8(trow, v);
            tc_fence_before();
            wk_bar();
            if (tid == 0) mbar_arrive(acc_empty0 + 8 * b);
            finish_tagged(P, kind, layer, n0, tile, m, q, lane, c_first, npieces, g, tag0 + unsigned(p), v[0], es);
          } else if (!spread) {
            unsigned long long* mine = P.tags + tag_off_slot(c, pj == 0 ? 0 : 1, m);
            float v[8];
            tmem_ld8(trow, v);
            st_tagged(mine, tag0 + unsigned(p), v[0]);
            tc_fence_before();
            wk_bar();
            if (tid == 0) mbar_arrive(acc_empty0 + 8 * b);
          } else {
            float* mine = P.part + piece_off_slot(c, pj == 0 ? 0 : 1, m);
            for (int c0 = 0; w < 4 && c0 < rows; c0 += 32) {  // TMEM lane quadrants: first 4 warps
              float v[32];
              tmem_ld32(trow + c0, v);
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (c0 + j < rows) mine[size_t(c0 + j) * 128] = v[j];
            }
            tc_fence_before();
            wk_bar();
            if (tid == 0) {
              mbar_arrive(acc_empty0 + 8 * b);
              // (all-split phases sync once per CTA after the piece loop instead)
              if (!all_split) {
                const unsigned old = atom_add_acq_rel(cnt + tile, 1u);
                es.flag = old == unsigned(npieces - 1);
              }
            }
            if (!all_split) wk_bar();
            // finalisation is deferred until all of this CTA's pieces are
            // published, so a tile's finaliser never delays the next tile's piece
            // (a two-piece GU / LM tile is finalised by its c_first instead)
            if (!pair_tile && (spread || es.flag)) {
              if (dtile0 < 0) dtile0 = tile; else dtile1 = tile;
            }
          }
          ++acc_it;
          (void)piece_hi;
        }
        if (tid == 0) stamp(P, p, c, G, 5);
        ensure_rstd();  // (also completes the staging copies before the buffer is reused)
        if (kWide && all_split) {
          // every CTA's pieces are out: one grid-wide sync on a per-phase
          // counter, then CTA c finalises rows [c*I/G, (c+1)*I/G) of the
          // I = tiles x rows (tile, row) items — at most two tile segments
          wk_bar();  // every worker's partial stores precede the release below
          if (tid == 0) {
            if (c < g.G) grid_arrive(cnt + g.tiles);
            grid_wait(cnt + g.tiles, unsigned(g.G));
            stamp(P, p, c, G, 7);
          }
          wk_bar();
          if (tid == 0) stamp(P, p, c, G, 8);
          const int items = g.tiles * rows;
          const int a = int((long long)c * items / G), e = int((long long)(c + 1) * items / G);
          float* stage = reinterpret_cast<float*>(kind == PH_QKV ? A.K(1) : A.K(0));
          const int cap = (kind == PH_QKV ? A.buf : 2 * A.buf) / 4;
          for (int i0 = a; i0 < e;) {
            const int tile = i0 / rows, r0 = i0 - tile * rows, r1 = min(rows, e - tile * rows);
            const int c_first = sk_owner(tile * g.KB, g.G, g.T), c_last = sk_owner((tile + 1) * g.KB - 1, g.G, g.T);
            const DefTile T{tile, c_first, c_last - c_first + 1, r0, r1, first_piece_slot(c_first, tile, g)};
            finish_share_vec(P, kind, layer, n0, w, lane, T, stage, cap, wbar, wphase, es, i0 == a ? p : -1);
            i0 = tile * rows + r1;
          }
          if (tid == 0) stamp(P, p, c, G, 9);
        } else if (kWide && !finalized) {
          finalize_split_tiles();
        }
        if (tid == 0) stamp(P, p, c, G, 6);
        if (kind == PH_LM) {
          // this CTA's (max, lowest id) per row: its 4 warp slots merged in order
          wk_bar();
          for (int t = tid; t < rows; t += kWorkers) {
            float bv = es.am_v[0][t];
            int bi = es.am_i[0][t];
            for (int qq = 1; qq < 6; ++qq) argmax_merge(bv, bi, es.am_v[qq][t], es.am_i[qq][t]);
            P.am_val[size_t(c) * kMaxWindow + t] = bv;
            P.am_idx[size_t(c) * kMaxWindow + t] = bi;
          }
        }
      }
      wk_bar();
      if (tid == 0) {
        stamp(P, p, c, G, 2);
        grid_arrive(P.bar);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  // every CTA read the epoch before the embed barrier, which CTA 0 passed
  if (c == 0 && threadIdx.x == 0) *P.epoch = epoch + 1;
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * P.acc_cols) : "memory");
  }
}

// static shared memory of one instantiation (the decode kernel's EpiSmem is small)
int mega_static_smem(bool wide) {
  static int st[2] = {-1, -1};
  if (st[wide] < 0) {
    cudaFuncAttributes fa{};
    const cudaError_t e = wide ? cudaFuncGetAttributes(&fa, mega_kernel<true>) : cudaFuncGetAttributes(&fa, mega_kernel<false>);
    st[wide] = e == cudaSuccess ? int(fa.sharedSizeBytes) : 16 * 1024;
  }
  return st[wide];
}

// One fixed attribute per instantiation (the most any pass width may use),
// set once, so handles created later never shrink it under a running one.
cudaError_t mega_set_smem_attr() {
  static cudaError_t done = cudaErrorNotReady;
  if (done == cudaErrorNotReady) {
    done = cudaFuncSetAttribute(mega_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                227 * 1024 - mega_static_smem(false));
    if (done == cudaSuccess)
      done = cudaFuncSetAttribute(mega_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  227 * 1024 - mega_static_smem(true));
  }
  return done;
}

int mega_stages(int ntok, int attn_floats, bool wide) {
  const int static_smem = mega_static_smem(wide);
  const int stage = kTileABytes + ntok * 128;
  // 227 KB per CTA minus static shared memory, attention staging and the
  // 1 KB alignment slack
  const int avail = 227 * 1024 - static_smem - attn_floats * 4 - 1024;
  int s = avail / stage;
  return s > kMaxStages ? kMaxStages : s;
}

int mega_smem_bytes(int ntok, int stages, int attn_floats) {
  return stages * (kTileABytes + ntok * 128) + attn_floats * 4 + 1024;
}

cudaError_t launch_mega(const MegaParams& P, bool wide, int grid, int smem, cudaStream_t st) {
  if (const cudaError_t e = mega_set_smem_attr(); e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(wide ? 256 : 192);  // wide: 6 worker warps (the register budget stays 255)
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr1[1];
  attr1[0].id = cudaLaunchAttributeCooperative;
  attr1[0].val.cooperative = 1;
  cfg.attrs = attr1;
  cfg.numAttrs = 1;
  return wide ? cudaLaunchKernelEx(&cfg, mega_kernel<true>, P) : cudaLaunchKernelEx(&cfg, mega_kernel<false>, P);
}

int mega_max_blocks_per_sm(int smem, bool wide) {
  if (mega_set_smem_attr() != cudaSuccess) return 0;
  int n = 0;
  const cudaError_t e = wide ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, mega_kernel<true>, 256, smem)
                             : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, mega_kernel<false>, 192, smem);
  return e == cudaSuccess ? n : 0;
}

}  // namespace ps
