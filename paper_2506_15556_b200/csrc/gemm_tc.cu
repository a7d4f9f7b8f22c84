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

namespace ps {

namespace {

constexpr int kBK = 64;                        // K elements per stage (128 B rows)
constexpr int kTileABytes = kTileTc * kBK * 2;  // 16 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

// UMMA shared-memory descriptor: K-major operand, 128B swizzle, 8-row groups
// 1024 B apart (SBO), sm100 descriptor version 1.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr & 0x3FFFF) >> 4);
  d |= uint64_t(1) << 16;            // LBO (unused for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;    // SBO
  d |= uint64_t(1) << 46;            // version
  d |= uint64_t(2) << 61;            // SWIZZLE_128B
  return d;
}

// kind::f16 instruction descriptor: D=f32, A=B=bf16, both K-major, M=128.
__device__ __forceinline__ uint32_t idesc_bf16(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(n >> 3) << 17) | (uint32_t(kTileTc >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

int tmem_cols_for(int ntok) {
  int c = 32;
  while (c < ntok) c <<= 1;
  return c;
}

int tc_stages(int ntok) {
  int s = (96 * 1024) / (kTileABytes + ntok * 128);
  return s < 2 ? 2 : (s > 6 ? 6 : s);
}

struct TcArgs {
  float* part;           // GEMM: split-K partials [split][kMaxWindow][N]
  int N;                 // output features (GEMM) / vocab rows of this shard (LM head)
  int kblocks;           // K/64 per split
  int ntok;              // MMA N (multiple of 16)
  int stages;
  int tmem_cols;
  int x_row_from_ctx;    // LM head: B rows start at absolute position ctx->n0
  const float* bias;     // LM head only
  int v_begin;
  float* am_val;
  int* am_idx;
  float* logits_out;
  int ld_logits;
};

template <bool kArgmax>
__global__ void __launch_bounds__(192, 1) gemm_tc_kernel(const __grid_constant__ CUtensorMap tmW,
                                                         const __grid_constant__ CUtensorMap tmX,
                                                         const PassCtx* __restrict__ ctx, TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  __shared__ uint64_t bars[2 * 8 + 1];
  __shared__ uint32_t tmem_holder;
  __shared__ float red_v[4][256];
  __shared__ int red_i[4][256];

  if (ctx->stop) return;
  const int rows = ctx->rows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntile = blockIdx.x, split = blockIdx.y;
  const int S = a.stages;
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int b_bytes = a.ntok * 128;
  auto a_tile = [&](int s) { return base + size_t(s) * (kTileABytes + b_bytes); };
  auto b_tile = [&](int s) { return a_tile(s) + kTileABytes; };
  const uint32_t full0 = smem_u32(&bars[0]), empty0 = smem_u32(&bars[8]), accum = smem_u32(&bars[16]);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < S; ++s) {
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
                 "r"(a.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_holder;
  const int kb0 = split * a.kblocks;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    const int xrow = a.x_row_from_ctx ? ctx->n0 : 0;
    const uint32_t tx = kTileABytes + b_bytes;
    for (int kb = 0; kb < a.kblocks; ++kb) {
      const int s = kb % S;
      const uint32_t ph = (kb / S) & 1;
      mbar_wait(empty0 + 8 * s, ph ^ 1);
      mbar_expect_tx(full0 + 8 * s, tx);
      const int kc = (kb0 + kb) * kBK;
      tma_load_2d(smem_u32(a_tile(s)), &tmW, full0 + 8 * s, kc, ntile * kTileTc);
      tma_load_2d(smem_u32(b_tile(s)), &tmX, full0 + 8 * s, kc, xrow);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = idesc_bf16(a.ntok);
    for (int kb = 0; kb < a.kblocks; ++kb) {
      const int s = kb % S;
      const uint32_t ph = (kb / S) & 1;
      mbar_wait(full0 + 8 * s, ph);
      tc_fence_after();
      const uint32_t sa = smem_u32(a_tile(s)), sb = smem_u32(b_tile(s));
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k) {
        umma_bf16(tmem, umma_desc_sw128(sa + k * 32), umma_desc_sw128(sb + k * 32), idesc,
                  (kb > 0 || k > 0) ? 1u : 0u);
      }
      umma_commit(empty0 + 8 * s);
    }
    umma_commit(accum);
  } else if (warp >= 2) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const int m = q * 32 + lane;
    mbar_wait(accum, 0);
    tc_fence_after();
    const uint32_t trow = tmem + (uint32_t(q * 32) << 16);
    if (!kArgmax) {
      float* out = a.part + (size_t(split) * kMaxWindow) * a.N + size_t(ntile) * kTileTc + m;
      for (int c0 = 0; c0 < a.ntok; c0 += 8) {
        float v[8];
        tmem_ld8(trow + c0, v);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (c0 + j < rows) out[size_t(c0 + j) * a.N] = v[j];
      }
    } else {
      const int vloc = ntile * kTileTc + m;  // row within this shard
      const bool valid = vloc < a.N;
      const int vid = a.v_begin + vloc;
      const float b = valid ? a.bias[vid] : 0.f;
      for (int c0 = 0; c0 < a.ntok; c0 += 8) {
        float v[8];
        tmem_ld8(trow + c0, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int col = c0 + j;
          float lv = valid ? v[j] + b : -INFINITY;
          int li = valid ? vid : 0x7fffffff;
          if (a.logits_out && valid && col < rows) a.logits_out[size_t(col) * a.ld_logits + vloc] = lv;
          warp_argmax(lv, li);
          if (lane == 0) {
            red_v[q][col] = lv;
            red_i[q][col] = li;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (kArgmax) {
    for (int col = threadIdx.x; col < rows; col += blockDim.x) {
      float v = red_v[0][col];
      int i = red_i[0][col];
      for (int qq = 1; qq < 4; ++qq) argmax_merge(v, i, red_v[qq][col], red_i[qq][col]);
      a.am_val[size_t(ntile) * kMaxWindow + col] = v;
      a.am_idx[size_t(ntile) * kMaxWindow + col] = i;
    }
  }
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols) : "memory");
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

void set_attrs_once() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute(gemm_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(gemm_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
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

void launch_gemm_tc(const PassCtx* ctx, const TmaDesc* tmW, const TmaDesc* tmX, float* part, int N, int K,
                    int splits, int ntok, int x_row_offset_from_ctx, cudaStream_t st) {
  set_attrs_once();
  TcArgs a{};
  a.part = part;
  a.N = N;
  a.kblocks = K / kBK / splits;
  a.ntok = ntok;
  a.stages = tc_stages(ntok);
  a.tmem_cols = tmem_cols_for(ntok);
  a.x_row_from_ctx = x_row_offset_from_ctx;
  const CUtensorMap* mw = reinterpret_cast<const CUtensorMap*>(tmW->bytes);
  const CUtensorMap* mx = reinterpret_cast<const CUtensorMap*>(tmX->bytes);
  dim3 grid(N / kTileTc, splits);
  gemm_tc_kernel<false><<<grid, 192, tc_gemm_smem_bytes(ntok), st>>>(*mw, *mx, ctx, a);
}

void launch_lmhead_tc(const PassCtx* ctx, const TmaDesc* tmW, const TmaDesc* tmX, const float* bias, int v_begin,
                      int v_count, int hidden, int ntok, int pos_offset, float* am_val, int* am_idx,
                      float* logits_out, int ld_logits, cudaStream_t st) {
  (void)pos_offset;
  set_attrs_once();
  TcArgs a{};
  a.N = v_count;
  a.kblocks = hidden / kBK;
  a.ntok = ntok;
  a.stages = tc_stages(ntok);
  a.tmem_cols = tmem_cols_for(ntok);
  a.x_row_from_ctx = 1;
  a.bias = bias;
  a.v_begin = v_begin;
  a.am_val = am_val;
  a.am_idx = am_idx;
  a.logits_out = logits_out;
  a.ld_logits = ld_logits;
  const CUtensorMap* mw = reinterpret_cast<const CUtensorMap*>(tmW->bytes);
  const CUtensorMap* mx = reinterpret_cast<const CUtensorMap*>(tmX->bytes);
  dim3 grid((v_count + kTileTc - 1) / kTileTc, 1);
  gemm_tc_kernel<true><<<grid, 192, tc_gemm_smem_bytes(ntok), st>>>(*mw, *mx, ctx, a);
}

}  // namespace ps
