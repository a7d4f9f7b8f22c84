// bf16 weight-streaming GEMM on the 5th-gen tensor cores (sm_100a).
//
// "Swap-AB" for bs=1 verify/decode: the weight tile is the MMA's M=128 side
// (A, K-major, TMA-staged with 128B swizzle) and the pass's tokens are the
// N side (B, N = rows rounded up to 16, <= 256). Accumulators live in TMEM
// (128 lanes x N fp32 columns). Warp roles per CTA (192 threads):
//   warp 0      one elected lane issues TMA loads into a `stages`-deep ring
//   warp 1      owns the TMEM allocation; one lane issues tcgen05.mma
//   warps 2..5  epilogue: tcgen05.ld -> registers -> fp32 split-K partials
//               (GEMM) or bias + vocab-tile argmax (LM head, logits never
//               written unless parity mode asks for them)
// Split-K boundaries depend on (N, K) only, so a token column's arithmetic is
// the same whatever the pass width (batch invariance, see layers.cu).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace ps {

namespace {

constexpr int kMaxSplits = 16;

int tmem_cols_for(int ntok) {
  int c = 32;
  while (c < ntok) c <<= 1;
  return c;
}

int tc_stages(int ntok) {
  int s = (96 * 1024) / (kTileABytes + ntok * 128);
  return s < 2 ? 2 : (s > 6 ? 6 : s);
}

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// named barrier over the 4 epilogue warps (128 threads)
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

struct TcParams {
  int N;            // output rows of this GEMM (vocab rows of the shard for the LM head)
  int kblocks;      // K/64 in total; split s covers k-blocks [s*KB/S, (s+1)*KB/S)
  int ntok;         // MMA N (multiple of 16)
  int stages;
  int tmem_cols;
  int x_row_from_ctx;
  TcEpilogue e;
};

// One 8-column chunk of the epilogue; v[j] is the finished fp32 sum for
// token column c0+j of output row n (= ntile*128 + m).
template <int kMode>
__device__ __forceinline__ void epilogue_chunk(const TcParams& p, const PassCtx* ctx, int rows, int ntile, int m,
                                               int q, int lane, int c0, const float (&v)[8],
                                               float (*xch)[kTileTc], float (*red_v)[8], int (*red_i)[8]) {
  const TcEpilogue& e = p.e;
  const int n = ntile * kTileTc + m;
  const int n0 = ctx->n0;
  if constexpr (kMode == TC_EPI_QKV || kMode == TC_EPI_SWIGLU) {
    float val[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int t = c0 + j;
      val[j] = 0.f;
      if (t < rows) {
        val[j] = v[j] * e.rstd_in[t];
        if (kMode == TC_EPI_QKV && e.bias) val[j] += __bfloat162float(e.bias[n]);
      }
      xch[j][m] = val[j];
    }
    epi_bar();
    if constexpr (kMode == TC_EPI_QKV) {
      const int hd = e.g.head_dim, half = hd >> 1;
      const int i = m % hd;
      const int partner = i < half ? m + half : m - half;
      const bool is_q = n < e.q_dim, is_k = !is_q && n < e.q_dim + e.kv_dim;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int t = c0 + j;
        if (t >= rows) continue;
        const int pos = n0 + t;
        float out = val[j];
        if (is_q || is_k) {
          const float other = xch[j][partner];
          const float a = i < half ? val[j] : other, b = i < half ? other : val[j];
          const float2 cs = e.rope[size_t(pos) * half + (i % half)];
          out = i < half ? a * cs.x - b * cs.y : b * cs.x + a * cs.y;
        }
        const __nv_bfloat16 ob = __float2bfloat16_rn(out);
        if (is_q) {
          e.q[size_t(t) * e.q_dim + n] = ob;
        } else {
          const int c = n - e.q_dim - (is_k ? 0 : e.kv_dim);
          const int h = c / hd;
          const size_t page = size_t(e.page_table[pos / kPage]);
          const size_t off = size_t(e.layer) * e.g.layer_stride() + ((page * e.g.kv_heads + h) * kPage + pos % kPage) * hd + (c % hd);
          (is_k ? e.kpool : e.vpool)[off] = ob;
        }
      }
    } else {
      if (m < kTileTc / 2) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int t = c0 + j;
          if (t >= rows) continue;
          const float g = val[j], u = xch[j][m + kTileTc / 2];
          e.act[size_t(t) * e.inter + ntile * (kTileTc / 2) + m] = __float2bfloat16_rn(g / (1.0f + expf(-g)) * u);
        }
      }
    }
    epi_bar();
  } else if constexpr (kMode == TC_EPI_RESID) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int t = c0 + j;
      float sq = 0.f;
      if (t < rows) {
        float* xp = e.x + size_t(t) * e.hidden + n;
        const float xi = *xp + v[j];
        *xp = xi;
        const size_t row = e.xb_out_pos ? size_t(n0 + t) : size_t(t);
        e.xb_out[row * e.hidden + n] = __float2bfloat16_rn(xi);
        sq = xi * xi;
      }
      sq = warp_sum(sq);
      if (lane == 0) red_v[q][j] = sq;
    }
    epi_bar();
    if (m < 8 && c0 + m < rows)
      e.ssq_part[size_t(ntile) * kMaxWindow + c0 + m] = ((red_v[0][m] + red_v[1][m]) + red_v[2][m]) + red_v[3][m];
    epi_bar();
  } else {  // TC_EPI_ARGMAX
    const bool valid = n < p.N;
    const int vid = e.v_begin + n;
    const float b = valid ? e.lbias[vid] : 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int t = c0 + j;
      float lv = -INFINITY;
      int li = 0x7fffffff;
      if (valid && t < rows) {
        lv = v[j] * e.rstd_in[n0 + t] + b;
        li = vid;
        if (e.logits_out) e.logits_out[size_t(t) * e.ld_logits + n] = lv;
      }
      warp_argmax(lv, li);
      if (lane == 0) {
        red_v[q][j] = lv;
        red_i[q][j] = li;
      }
    }
    epi_bar();
    if (m < 8 && c0 + m < rows) {
      float bv = red_v[0][m];
      int bi = red_i[0][m];
      for (int qq = 1; qq < 4; ++qq) argmax_merge(bv, bi, red_v[qq][m], red_i[qq][m]);
      e.am_val[size_t(ntile) * kMaxWindow + c0 + m] = bv;
      e.am_idx[size_t(ntile) * kMaxWindow + c0 + m] = bi;
    }
    epi_bar();
  }
}

template <int kMode>
__global__ void __launch_bounds__(192, 1) gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW,
                                                         const __grid_constant__ CUtensorMap tmX, PassCtx* ctx,
                                                         const __grid_constant__ TcParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint64_t bars[2 * 8 + 1];
  __shared__ uint32_t tmem_holder;
  __shared__ int s_flag[2];
  __shared__ float xch[8][kTileTc];
  __shared__ float red_v[4][8];
  __shared__ int red_i[4][8];

  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntile = blockIdx.x, split = blockIdx.y, S = gridDim.y;
  const int ST = p.stages;
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int b_bytes = p.ntok * 128;
  auto a_tile = [&](int s) { return base + size_t(s) * (kTileABytes + b_bytes); };
  auto b_tile = [&](int s) { return a_tile(s) + kTileABytes; };
  const uint32_t full0 = smem_u32(&bars[0]), empty0 = smem_u32(&bars[8]), accum = smem_u32(&bars[16]);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(accum, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_holder)),
                 "r"(p.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const int kb0 = split * p.kblocks / S;
  const int nkb = (split + 1) * p.kblocks / S - kb0;
  const int pre = nkb < ST ? nkb : ST;

  if (warp == 0 && lane == 0) {
    // ---- TMA producer: weights for the first stages stream before the
    // predecessor kernel has finished (PDL); activations after it has. ----
    const uint32_t tx = kTileABytes + b_bytes;
    for (int kb = 0; kb < pre; ++kb) {
      mbar_expect_tx(full0 + 8 * kb, tx);
      tma_load_2d(smem_u32(a_tile(kb)), &tmW, full0 + 8 * kb, (kb0 + kb) * kBK, ntile * kTileTc);
    }
    pdl_wait();
    const int stop = ctx->stop;
    const int xrow = p.x_row_from_ctx ? ctx->n0 : 0;
    for (int kb = 0; kb < pre; ++kb)
      tma_load_2d(smem_u32(b_tile(kb)), &tmX, full0 + 8 * kb, (kb0 + kb) * kBK, xrow);
    const int nk = stop ? pre : nkb;
    for (int kb = pre; kb < nk; ++kb) {
      const int s = kb % ST;
      const uint32_t ph = (kb / ST) & 1;
      mbar_wait(empty0 + 8 * s, ph ^ 1);
      mbar_expect_tx(full0 + 8 * s, tx);
      const int kc = (kb0 + kb) * kBK;
      tma_load_2d(smem_u32(a_tile(s)), &tmW, full0 + 8 * s, kc, ntile * kTileTc);
      tma_load_2d(smem_u32(b_tile(s)), &tmX, full0 + 8 * s, kc, xrow);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer ----
    const uint32_t idesc = idesc_bf16(p.ntok);
    pdl_wait();
    const int nk = ctx->stop ? pre : nkb;
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % ST;
      const uint32_t ph = (kb / ST) & 1;
      mbar_wait(full0 + 8 * s, ph);
      tc_fence_after();
      const uint32_t sa = smem_u32(a_tile(s)), sb = smem_u32(b_tile(s));
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k)
        umma_bf16(tmem, umma_desc_sw128(sa + k * 32), umma_desc_sw128(sb + k * 32), idesc, (kb > 0 || k > 0) ? 1u : 0u);
      umma_commit(empty0 + 8 * s);
    }
    umma_commit(accum);
  } else if (warp >= 2) {
    // ---- epilogue (warps 2..5; warp w reads TMEM lanes 32*(w%4)..) ----
    pdl_wait();
    const int q = warp & 3;
    const int m = q * 32 + lane;
    const int n = ntile * kTileTc + m;
    mbar_wait(accum, 0);
    tc_fence_after();
    const bool stopped = ctx->stop != 0;
    const int rows = ctx->rows;
    const uint32_t trow = tmem + (uint32_t(q * 32) << 16);
    const TcEpilogue& e = p.e;
    bool last = !stopped;
    if (!stopped && S > 1) {
      // split-K: publish this split's partial; the last CTA of the tile sums
      // all splits in split order (deterministic, independent of arrival).
      float* part = e.part + size_t(split) * kMaxWindow * p.N + n;
      for (int c0 = 0; c0 < rows; c0 += 8) {
        float v[8];
        tmem_ld8(trow + c0, v);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (c0 + j < rows) part[size_t(c0 + j) * p.N] = v[j];
      }
      __threadfence();
      epi_bar();
      if (m == 0) {
        const unsigned old = atomicAdd(&e.tile_cnt[ntile], 1u);
        s_flag[1] = old == unsigned(S - 1);
        if (old == unsigned(S - 1)) e.tile_cnt[ntile] = 0u;
      }
      epi_bar();
      last = s_flag[1] != 0;
      __threadfence();
    }
    if (last) {
      for (int c0 = 0; c0 < rows; c0 += 8) {
        float v[8];
        if (S > 1) {
          // all loads of the chunk in flight first, then the fixed-order sums
          const float* part = e.part + n;
          float buf[8][kMaxSplits];
#pragma unroll
          for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int s = 0; s < kMaxSplits; ++s)
              buf[j][s] = (s < S && c0 + j < rows) ? __ldcg(part + (size_t(s) * kMaxWindow + c0 + j) * p.N) : 0.f;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float acc = buf[j][0];
#pragma unroll
            for (int s = 1; s < kMaxSplits; ++s)
              if (s < S) acc += buf[j][s];
            v[j] = acc;
          }
        } else {
          tmem_ld8(trow + c0, v);
        }
        epilogue_chunk<kMode>(p, ctx, rows, ntile, m, q, lane, c0, v, xch, red_v, red_i);
      }
      if constexpr (kMode == TC_EPI_RESID || kMode == TC_EPI_ARGMAX) {
        // grid-wide finish: the last tile turns per-tile partials into
        // per-row results (rstd / argmax), in tile order.
        __threadfence();
        epi_bar();
        const int ntiles = gridDim.x;
        if (m == 0) {
          const unsigned old = atomicAdd(e.grid_cnt, 1u);
          s_flag[1] = old == unsigned(ntiles - 1);
          if (old == unsigned(ntiles - 1)) *e.grid_cnt = 0u;
        }
        epi_bar();
        if (s_flag[1]) {
          __threadfence();
          const int n0 = ctx->n0;
          const int w = warp - 2;
          if constexpr (kMode == TC_EPI_RESID) {
            // one warp per row: lane l sums tiles l, l+32 (in order), then a
            // fixed butterfly — the same tree for every pass width
            for (int t = w; t < rows; t += 4) {
              float a0 = lane < ntiles ? __ldcg(e.ssq_part + size_t(lane) * kMaxWindow + t) : 0.f;
              float a1 = lane + 32 < ntiles ? __ldcg(e.ssq_part + size_t(lane + 32) * kMaxWindow + t) : 0.f;
              const float ssq = warp_sum(a0 + a1);
              if (lane == 0) e.rstd_out[e.rstd_out_pos ? n0 + t : t] = 1.0f / sqrtf(ssq / float(e.hidden) + e.eps);
            }
          } else {
            for (int t = w; t < rows; t += 4) {
              float bv = -INFINITY;
              int bi = 0x7fffffff;
              for (int t0 = 0; t0 < ntiles; t0 += 32 * 8) {
                float vv[8];
                int ii[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                  const int tt = t0 + u * 32 + lane;
                  vv[u] = tt < ntiles ? __ldcg(e.am_val + size_t(tt) * kMaxWindow + t) : -INFINITY;
                  ii[u] = tt < ntiles ? __ldcg(e.am_idx + size_t(tt) * kMaxWindow + t) : 0x7fffffff;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) argmax_merge(bv, bi, vv[u], ii[u]);
              }
              warp_argmax(bv, bi);
              if (lane == 0) {
                e.argmax_pos[n0 + t] = bi;
                if (e.packed_out) {
                  unsigned u = __float_as_uint(bv);
                  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
                  e.packed_out[t] = (static_cast<unsigned long long>(u) << 32) | (0xFFFFFFFFull - unsigned(bi));
                }
              }
            }
            epi_bar();
            if (m == 0 && e.advance) {
              ctx->n0 = n0 + 1;
              ctx->step += 1;
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols) : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

template <int kMode>
void set_attr_once() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(gemm_tc_kernel<kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  done = true;
}

}  // namespace

int tc_gemm_smem_bytes(int ntok) { return tc_stages(ntok) * (kTileABytes + ntok * 128) + 1024; }

bool encode_tma_2d_bf16(TmaDesc* out, const void* base, uint64_t inner, uint64_t outer, uint32_t box_inner,
                        uint32_t box_outer) {
  static_assert(sizeof(CUtensorMap) <= sizeof(TmaDesc), "tensor map size");
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(reinterpret_cast<CUtensorMap*>(out->bytes), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

void launch_tc(PassCtx* ctx, const TmaDesc* tmW, const TmaDesc* tmX, int N, int K, int splits, int ntok,
               int x_row_from_ctx, const TcEpilogue& e, cudaStream_t st, bool pdl) {
  // Only the LM-head ARGMAX mode is live: the decode/verify passes run in the
  // persistent megakernel, whose weight layouts (kHeadPairs / kGateUp) the
  // QKV / SWIGLU modes below do not follow. ps_logits_rows uses ARGMAX with
  // logits_out for the parity path.
  if (e.mode != TC_EPI_ARGMAX) return;
  TcParams p{};
  p.N = N;
  p.kblocks = K / kBK;
  p.ntok = ntok;
  p.stages = tc_stages(ntok);
  p.tmem_cols = tmem_cols_for(ntok);
  p.x_row_from_ctx = x_row_from_ctx;
  p.e = e;
  const CUtensorMap* mw = reinterpret_cast<const CUtensorMap*>(tmW->bytes);
  const CUtensorMap* mx = reinterpret_cast<const CUtensorMap*>(tmX->bytes);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((N + kTileTc - 1) / kTileTc, splits);
  cfg.blockDim = dim3(192);
  cfg.dynamicSmemBytes = tc_gemm_smem_bytes(ntok);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  switch (e.mode) {
    case TC_EPI_QKV:
      set_attr_once<TC_EPI_QKV>();
      cudaLaunchKernelEx(&cfg, gemm_tc_kernel<TC_EPI_QKV>, *mw, *mx, ctx, p);
      break;
    case TC_EPI_SWIGLU:
      set_attr_once<TC_EPI_SWIGLU>();
      cudaLaunchKernelEx(&cfg, gemm_tc_kernel<TC_EPI_SWIGLU>, *mw, *mx, ctx, p);
      break;
    case TC_EPI_RESID:
      set_attr_once<TC_EPI_RESID>();
      cudaLaunchKernelEx(&cfg, gemm_tc_kernel<TC_EPI_RESID>, *mw, *mx, ctx, p);
      break;
    default:
      set_attr_once<TC_EPI_ARGMAX>();
      cudaLaunchKernelEx(&cfg, gemm_tc_kernel<TC_EPI_ARGMAX>, *mw, *mx, ctx, p);
      break;
  }
}

}  // namespace ps
