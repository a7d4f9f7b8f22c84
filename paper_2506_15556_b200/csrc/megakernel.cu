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

enum Phase : int { PH_EMBED = 0, PH_QKV, PH_ATTN, PH_O, PH_GU, PH_D, PH_LM };
constexpr int kWorkers = 128;  // warps 2..5

__device__ __forceinline__ void wk_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

struct Gemm {
  int N, KB, T;  // rows, k-blocks per tile, total k-blocks
  int tiles;
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
  return g;
}

__device__ __forceinline__ int sk_start(int c, int G, int T) { return int((long long)c * T / G); }
// CTA whose k-block range contains global block x
__device__ __forceinline__ int sk_owner(int x, int G, int T) {
  return int(((long long)(x + 1) * G + T - 1) / T) - 1;
}

__device__ __forceinline__ void grid_arrive(unsigned* bar) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
}

__device__ __forceinline__ void grid_wait(const unsigned* bar, unsigned target) {
  while (ld_acquire_gpu(bar) < target) __nanosleep(40);
}

__device__ __forceinline__ int phase_kind(int p, int L) {
  if (p == 0) return PH_EMBED;
  if (p == 1 + 5 * L) return PH_LM;
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

// ---------------------------------------------------------------------------
// epilogue math for one finished 8-column chunk of tile rows [128*tile, +128)
struct EpiSmem {
  float xch[8][128];
  float red_v[4][8];
  int red_i[4][8];
  float rstd[kMaxWindow];
  int flag;
};

__device__ void finish_chunk(const MegaParams& P, int kind, int layer, int rows, int n0, int tile, int m, int q,
                             int lane, int c0, const float (&v)[8], EpiSmem& es) {
  const int n = tile * 128 + m;
  if (kind == PH_QKV || kind == PH_GU) {
    float val[8];
    const __nv_bfloat16* bias = (kind == PH_QKV && P.qkv_bias) ? P.qkv_bias + size_t(layer) * (P.qd + 2 * P.kvd) : nullptr;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int t = c0 + j;
      val[j] = 0.f;
      if (t < rows) {
        val[j] = v[j] * es.rstd[t];
        if (bias) val[j] += __bfloat162float(bias[n]);
      }
      es.xch[j][m] = val[j];
    }
    wk_bar();
    if (kind == PH_QKV) {
      const int hd = P.hd, half = hd >> 1;
      const int i = m % hd;
      const int partner = i < half ? m + half : m - half;
      const bool is_q = n < P.qd, is_k = !is_q && n < P.qd + P.kvd;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int t = c0 + j;
        if (t >= rows) continue;
        const int pos = n0 + t;
        float out = val[j];
        if (is_q || is_k) {
          const float other = es.xch[j][partner];
          const float a = i < half ? val[j] : other, b = i < half ? other : val[j];
          const float2 cs = P.rope[size_t(pos) * half + (i % half)];
          out = i < half ? a * cs.x - b * cs.y : b * cs.x + a * cs.y;
        }
        const __nv_bfloat16 ob = __float2bfloat16_rn(out);
        if (is_q) {
          P.q[size_t(t) * P.qd + n] = ob;
        } else {
          const int cc = n - P.qd - (is_k ? 0 : P.kvd);
          const int h = cc / hd;
          const size_t page = size_t(P.page_table[pos / kPage]);
          const size_t off = size_t(layer) * P.g.layer_stride() +
                             ((page * P.g.kv_heads + h) * kPage + pos % kPage) * hd + (cc % hd);
          (is_k ? P.kpool : P.vpool)[off] = ob;
        }
      }
    } else if (m < 64) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int t = c0 + j;
        if (t >= rows) continue;
        const float g = val[j], u = es.xch[j][m + 64];
        P.act[size_t(t) * P.I + tile * 64 + m] = __float2bfloat16_rn(g / (1.0f + expf(-g)) * u);
      }
    }
    wk_bar();
  } else if (kind == PH_O || kind == PH_D) {
    const bool to_hn = kind == PH_D && layer == P.L - 1;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int t = c0 + j;
      float sq = 0.f;
      if (t < rows) {
        float* xp = P.x + size_t(t) * P.H + n;
        const float xi = *xp + v[j];
        *xp = xi;
        __nv_bfloat16* dst = to_hn ? P.hn_cache + size_t(n0 + t) * P.H : P.xb + size_t(t) * P.H;
        dst[n] = __float2bfloat16_rn(xi);
        sq = xi * xi;
      }
      sq = warp_sum(sq);
      if (lane == 0) es.red_v[q][j] = sq;
    }
    wk_bar();
    if (m < 8 && c0 + m < rows)
      P.ssq_part[size_t(tile) * kMaxWindow + c0 + m] =
          ((es.red_v[0][m] + es.red_v[1][m]) + es.red_v[2][m]) + es.red_v[3][m];
    wk_bar();
  } else {  // PH_LM: logits = rstd * acc + bias; per-tile (max, lowest id)
    const bool valid = n < P.vocab_local;
    const int vid = P.v_begin + n;
    const float b = valid ? P.lm_bias[vid] : 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int t = c0 + j;
      float lv = -INFINITY;
      int li = 0x7fffffff;
      if (valid && t < rows) {
        lv = v[j] * es.rstd[t] + b;
        li = vid;
      }
      warp_argmax(lv, li);
      if (lane == 0) {
        es.red_v[q][j] = lv;
        es.red_i[q][j] = li;
      }
    }
    wk_bar();
    if (m < 8 && c0 + m < rows) {
      float bv = es.red_v[0][m];
      int bi = es.red_i[0][m];
      for (int qq = 1; qq < 4; ++qq) argmax_merge(bv, bi, es.red_v[qq][m], es.red_i[qq][m]);
      P.am_val[size_t(tile) * kMaxWindow + c0 + m] = bv;
      P.am_idx[size_t(tile) * kMaxWindow + c0 + m] = bi;
    }
    wk_bar();
  }
}

// rstd of every row of the pass from the per-tile sums of squares of the
// previous RESID phase (or the embed rstd), one warp per row, fixed tree.
__device__ void load_rstd(const MegaParams& P, bool from_embed, int rows, int w, int lane, EpiSmem& es) {
  const int ntiles = P.H / 128;
  for (int t = w; t < rows; t += 4) {
    if (from_embed) {
      if (lane == 0) es.rstd[t] = __ldcg(P.rstd0 + t);
    } else {
      float a0 = lane < ntiles ? __ldcg(P.ssq_part + size_t(lane) * kMaxWindow + t) : 0.f;
      float a1 = lane + 32 < ntiles ? __ldcg(P.ssq_part + size_t(lane + 32) * kMaxWindow + t) : 0.f;
      const float ssq = warp_sum(a0 + a1);
      if (lane == 0) es.rstd[t] = 1.0f / sqrtf(ssq / float(P.H) + P.eps);
    }
  }
}

// ---------------------------------------------------------------------------
__device__ void attention_unit(const MegaParams& P, int layer, int t, int kvh, int s, int n0, float* sm,
                               int w, int lane, int* s_flag) {
  const int pos = n0 + t;
  const int nsplit = pos / kPage + 1;
  const int hd = P.hd, grp = P.heads / P.kv_heads;
  const int nkeys = min(kPage, pos + 1 - s * kPage);
  float* Ks = sm;
  float* Vs = Ks + kPage * (hd + 1);
  float* Qs = Vs + kPage * hd;
  const int tid = threadIdx.x - 64;
  const size_t page = size_t(P.page_table[s]);
  const size_t off = size_t(layer) * P.g.layer_stride() + (page * P.kv_heads + kvh) * kPage * hd;
  const int vpr = hd / 8;
  for (int e = tid; e < nkeys * vpr; e += kWorkers) {
    const int j = e / vpr, d0 = (e % vpr) * 8;
    const uint4 kr = __ldcg(reinterpret_cast<const uint4*>(P.kpool + off + size_t(j) * hd + d0));
    const uint4 vr = __ldcg(reinterpret_cast<const uint4*>(P.vpool + off + size_t(j) * hd + d0));
    const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(&kr);
    const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(&vr);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      Ks[j * (hd + 1) + d0 + i] = __bfloat162float(kb[i]);
      Vs[j * hd + d0 + i] = __bfloat162float(vb[i]);
    }
  }
  const __nv_bfloat16* qrow = P.q + size_t(t) * P.qd + size_t(kvh) * grp * hd;
  for (int e = tid; e < grp * hd; e += kWorkers) Qs[e] = __bfloat162float(__ldcg(qrow + e));
  wk_bar();
  for (int hh = w; hh < grp; hh += 4) {
    const int h = kvh * grp + hh;
    const float* qs = Qs + hh * hd;
    float sc[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int j = lane + 32 * r;
      float acc = 0.f;
      if (j < nkeys) {
        const float* kr = Ks + j * (hd + 1);
        for (int d = 0; d < hd; ++d) acc = fmaf(qs[d], kr[d], acc);
        sc[r] = acc * P.attn_scale;
      } else {
        sc[r] = -INFINITY;
      }
    }
    const float m = warp_max(fmaxf(sc[0], sc[1]));
    const float p0 = (lane < nkeys) ? expf(sc[0] - m) : 0.f;
    const float p1 = (lane + 32 < nkeys) ? expf(sc[1] - m) : 0.f;
    const float l = warp_sum(p0 + p1);
    const size_t slot = (size_t(t) * P.heads + h) * P.max_splits_attn + s;
    for (int d = lane; d < hd; d += 32) {
      float acc = 0.f;
      for (int j = 0; j < nkeys; ++j) {
        const float pj = __shfl_sync(0xffffffffu, j < 32 ? p0 : p1, j & 31);
        acc = fmaf(pj, Vs[j * hd + d], acc);
      }
      P.o_part[slot * hd + d] = acc;
    }
    if (lane == 0) {
      P.ml_part[slot * 2] = m;
      P.ml_part[slot * 2 + 1] = l;
    }
  }
  __threadfence();
  wk_bar();
  if (tid == 0) {
    unsigned* c = P.acnt + size_t(t) * P.kv_heads + kvh;
    const unsigned old = atomicAdd(c, 1u);
    *s_flag = old == unsigned(nsplit - 1);
    if (*s_flag) *c = 0u;
  }
  wk_bar();
  if (*s_flag) {
    __threadfence();
    for (int hh = w; hh < grp; hh += 4) {
      const int h = kvh * grp + hh;
      const size_t base = (size_t(t) * P.heads + h) * P.max_splits_attn;
      float M = -INFINITY;
      for (int sp = 0; sp < nsplit; ++sp) M = fmaxf(M, __ldcg(P.ml_part + (base + sp) * 2));
      for (int d = lane; d < hd; d += 32) {
        float L = 0.f, acc = 0.f;
        for (int sp = 0; sp < nsplit; ++sp) {
          const float f = expf(__ldcg(P.ml_part + (base + sp) * 2) - M);
          L = fmaf(__ldcg(P.ml_part + (base + sp) * 2 + 1), f, L);
          acc = fmaf(__ldcg(P.o_part + (base + sp) * hd + d), f, acc);
        }
        P.attn[size_t(t) * P.qd + size_t(h) * hd + d] = __float2bfloat16_rn(acc / L);
      }
    }
  }
  wk_bar();
}

}  // namespace

__global__ void __launch_bounds__(192, 1) mega_kernel(const __grid_constant__ MegaParams P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint64_t bars[2 * 8 + 4];
  __shared__ uint32_t tmem_holder;
  __shared__ EpiSmem es;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x, G = gridDim.x;
  const int ST = P.stages;
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int b_bytes = P.ntok * 128;
  auto a_tile = [&](int s) { return base + size_t(s) * (kTileABytes + b_bytes); };
  auto b_tile = [&](int s) { return a_tile(s) + kTileABytes; };
  float* attn_sm = reinterpret_cast<float*>(base + size_t(ST) * (kTileABytes + b_bytes));
  const uint32_t full0 = smem_u32(&bars[0]), empty0 = smem_u32(&bars[8]);
  const uint32_t acc_full0 = smem_u32(&bars[16]), acc_empty0 = smem_u32(&bars[18]);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(acc_full0 + 8 * b, 1);
      mbar_init(acc_empty0 + 8 * b, 1);
    }
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
  const int nphases = 2 + 5 * P.L;

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      grid_wait(P.bar, unsigned(G));  // embed done (and the stop flag settled)
      if (!P.ctx->stop) {
        const int xrow_lm = n0;
        uint32_t it = 0;
        for (int p = 1; p < nphases; ++p) {
          const int kind = phase_kind(p, P.L);
          if (kind == PH_ATTN) continue;
          const Gemm g = gemm_of(P, kind);
          const int kb_lo = sk_start(c, G, g.T), kb_hi = sk_start(c + 1, G, g.T);
          const int nk = kb_hi - kb_lo;
          const CUtensorMap* wm = wmap_of(P, p, kind);
          const CUtensorMap* xm = xmap_of(P, kind);
          const int xrow = kind == PH_LM ? xrow_lm : 0;
          const uint32_t tx = kTileABytes + b_bytes;
          const int pre = nk < ST ? nk : ST;
          for (int i = 0; i < pre; ++i) {
            const uint32_t s = (it + i) % ST, ph = ((it + i) / ST) & 1;
            mbar_wait(empty0 + 8 * s, ph ^ 1);
            mbar_expect_tx(full0 + 8 * s, tx);
            const int x = kb_lo + i, tile = x / g.KB, kb = x % g.KB;
            tma_load_2d(smem_u32(a_tile(s)), wm, full0 + 8 * s, kb * kBK, tile * 128);
          }
          grid_wait(P.bar, unsigned(G) * unsigned(p));  // activations of this phase are complete
          fence_proxy_async_global();
          for (int i = 0; i < pre; ++i) {
            const uint32_t s = (it + i) % ST;
            const int x = kb_lo + i, kb = x % g.KB;
            tma_load_2d(smem_u32(b_tile(s)), xm, full0 + 8 * s, kb * kBK, xrow);
          }
          for (int i = pre; i < nk; ++i) {
            const uint32_t s = (it + i) % ST, ph = ((it + i) / ST) & 1;
            mbar_wait(empty0 + 8 * s, ph ^ 1);
            mbar_expect_tx(full0 + 8 * s, tx);
            const int x = kb_lo + i, tile = x / g.KB, kb = x % g.KB;
            tma_load_2d(smem_u32(a_tile(s)), wm, full0 + 8 * s, kb * kBK, tile * 128);
            tma_load_2d(smem_u32(b_tile(s)), xm, full0 + 8 * s, kb * kBK, xrow);
          }
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
        for (int p = 1; p < nphases; ++p) {
          const int kind = phase_kind(p, P.L);
          if (kind == PH_ATTN) continue;
          const Gemm g = gemm_of(P, kind);
          const int kb_lo = sk_start(c, G, g.T), kb_hi = sk_start(c + 1, G, g.T);
          int x = kb_lo;
          while (x < kb_hi) {  // one piece per tile touched by this CTA
            const int tile = x / g.KB;
            const int piece_hi = min(kb_hi, (tile + 1) * g.KB);
            const uint32_t b = acc_it & 1, aph = (acc_it >> 1) & 1;
            mbar_wait(acc_empty0 + 8 * b, aph ^ 1);
            tc_fence_after();
            const uint32_t dcol = tmem + b * uint32_t(P.acc_cols);
            for (int y = x; y < piece_hi; ++y, ++it) {
              const uint32_t s = it % ST, ph = (it / ST) & 1;
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
            x = piece_hi;
          }
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
    // ---- phase 0: embedding rows (t ≡ c mod G) ----
    for (int t = c; t < rows; t += G) {
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
      for (int cc = tid; cc < P.H / 8; cc += kWorkers) {
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
      if (lane == 0) es.red_v[w][0] = ss;
      wk_bar();
      if (tid == 0) P.rstd0[t] = 1.0f / sqrtf((((es.red_v[0][0] + es.red_v[1][0]) + es.red_v[2][0]) + es.red_v[3][0]) / float(P.H) + P.eps);
      wk_bar();
    }
    __threadfence();
    wk_bar();
    if (tid == 0) grid_arrive(P.bar);
    for (int p = 1; p < nphases; ++p) {
      const int kind = phase_kind(p, P.L);
      const int layer = kind == PH_LM ? P.L - 1 : (p - 1) / 5;
      if (tid == 0) grid_wait(P.bar, unsigned(G) * unsigned(p));
      wk_bar();
      if (P.ctx->stop) break;
      if (kind == PH_ATTN) {
        const int npages = (n0 + rows - 1) / kPage + 1;
        const int units = rows * P.kv_heads * npages;
        for (int u = c; u < units; u += G) {
          const int s = u % npages, r = u / npages;
          const int kvh = r % P.kv_heads, t = r / P.kv_heads;
          if (s > (n0 + t) / kPage) continue;
          attention_unit(P, layer, t, kvh, s, n0, attn_sm, w, lane, &es.flag);
        }
      } else {
        if (kind == PH_QKV || kind == PH_GU || kind == PH_LM) {
          load_rstd(P, kind == PH_QKV && layer == 0, rows, w, lane, es);
          wk_bar();
          if (kind == PH_LM && c == 0)
            for (int t = tid; t < rows; t += kWorkers) P.rstd_cache[n0 + t] = es.rstd[t];
        }
        const Gemm g = gemm_of(P, kind);
        const int kb_lo = sk_start(c, G, g.T), kb_hi = sk_start(c + 1, G, g.T);
        const int first_tile = kb_lo / g.KB;
        int x = kb_lo;
        while (x < kb_hi) {
          const int tile = x / g.KB;
          const int piece_hi = min(kb_hi, (tile + 1) * g.KB);
          const int c_first = sk_owner(tile * g.KB, G, g.T), c_last = sk_owner((tile + 1) * g.KB - 1, G, g.T);
          // CTAs between c_first and c_last with an empty range (T < G) hold no piece
          int npieces = 0;
          for (int cc = c_first; cc <= c_last; ++cc) npieces += sk_start(cc, G, g.T) < sk_start(cc + 1, G, g.T);
          const uint32_t b = acc_it & 1, aph = (acc_it >> 1) & 1;
          mbar_wait(acc_full0 + 8 * b, aph);
          tc_fence_after();
          const uint32_t trow = tmem + b * uint32_t(P.acc_cols) + (uint32_t(q * 32) << 16);
          if (npieces == 1) {
            for (int c0 = 0; c0 < rows; c0 += 8) {
              float v[8];
              tmem_ld8(trow + c0, v);
              finish_chunk(P, kind, layer, rows, n0, tile, m, q, lane, c0, v, es);
            }
            tc_fence_before();
            wk_bar();
            if (tid == 0) mbar_arrive(acc_empty0 + 8 * b);
          } else {
            const int slot = tile == first_tile ? 0 : 1;
            float* mine = P.part + (size_t(c * 2 + slot) * kMaxWindow) * 128 + m;
            for (int c0 = 0; c0 < rows; c0 += 8) {
              float v[8];
              tmem_ld8(trow + c0, v);
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (c0 + j < rows) mine[size_t(c0 + j) * 128] = v[j];
            }
            tc_fence_before();
            __threadfence();
            wk_bar();
            if (tid == 0) {
              mbar_arrive(acc_empty0 + 8 * b);
              const unsigned old = atomicAdd(P.tile_cnt + tile, 1u);
              es.flag = old == unsigned(npieces - 1);
              if (es.flag) P.tile_cnt[tile] = 0u;
            }
            wk_bar();
            if (es.flag) {
              __threadfence();
              for (int c0 = 0; c0 < rows; c0 += 8) {
                float v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = 0.f;
                bool first_piece = true;
                for (int cc = c_first; cc <= c_last; ++cc) {
                  if (sk_start(cc, G, g.T) == sk_start(cc + 1, G, g.T)) continue;
                  const int sl = (sk_start(cc, G, g.T) / g.KB == tile) ? 0 : 1;
                  const float* src = P.part + (size_t(cc * 2 + sl) * kMaxWindow) * 128 + m;
                  float tmp[8];
#pragma unroll
                  for (int j = 0; j < 8; ++j) tmp[j] = (c0 + j < rows) ? __ldcg(src + size_t(c0 + j) * 128) : 0.f;
#pragma unroll
                  for (int j = 0; j < 8; ++j) v[j] = first_piece ? tmp[j] : v[j] + tmp[j];
                  first_piece = false;
                }
                finish_chunk(P, kind, layer, rows, n0, tile, m, q, lane, c0, v, es);
              }
            }
          }
          ++acc_it;
          x = piece_hi;
        }
        if (kind == PH_LM) {
          // grid-wide argmax over vocab tiles: the last CTA to finish reduces
          __threadfence();
          wk_bar();
          if (tid == 0) {
            const unsigned old = atomicAdd(P.lm_cnt, 1u);
            es.flag = old == unsigned(G - 1);
            if (es.flag) *P.lm_cnt = 0u;
          }
          wk_bar();
          if (es.flag) {
            __threadfence();
            const int ntiles = g.tiles;
            for (int t = w; t < rows; t += 4) {
              float bv = -INFINITY;
              int bi = 0x7fffffff;
              for (int t0 = 0; t0 < ntiles; t0 += 32 * 8) {
                float vv[8];
                int ii[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                  const int tt = t0 + u * 32 + lane;
                  vv[u] = tt < ntiles ? __ldcg(P.am_val + size_t(tt) * kMaxWindow + t) : -INFINITY;
                  ii[u] = tt < ntiles ? __ldcg(P.am_idx + size_t(tt) * kMaxWindow + t) : 0x7fffffff;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) argmax_merge(bv, bi, vv[u], ii[u]);
              }
              warp_argmax(bv, bi);
              if (lane == 0) {
                P.argmax_pos[n0 + t] = bi;
                if (P.keys) {
                  unsigned uu = __float_as_uint(bv);
                  uu = (uu & 0x80000000u) ? ~uu : (uu | 0x80000000u);
                  P.keys[t] = (static_cast<unsigned long long>(uu) << 32) | (0xFFFFFFFFull - unsigned(bi));
                }
              }
            }
            wk_bar();
            if (tid == 0 && P.advance) {
              P.ctx->n0 = n0 + 1;
              P.ctx->step += 1;
            }
          }
        }
      }
      __threadfence();
      wk_bar();
      if (tid == 0) grid_arrive(P.bar);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * P.acc_cols) : "memory");
  }
}

int mega_stages(int ntok, int attn_floats) {
  const int stage = kTileABytes + ntok * 128;
  const int avail = 222 * 1024 - attn_floats * 4 - 2048;
  int s = avail / stage;
  return s > 8 ? 8 : s;
}

int mega_smem_bytes(int ntok, int stages, int attn_floats) {
  return stages * (kTileABytes + ntok * 128) + attn_floats * 4 + 1024;
}

cudaError_t launch_mega(const MegaParams& P, int grid, int smem, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(mega_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr1[1];
  attr1[0].id = cudaLaunchAttributeCooperative;
  attr1[0].val.cooperative = 1;
  cfg.attrs = attr1;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, mega_kernel, P);
}

}  // namespace ps
