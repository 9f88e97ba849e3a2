// K1: persistent warp-specialised tcgen05 GEMM for sm_100a.
//
//   D[M,N] = epilogue(A[M,K] . B[K,N]),  bf16 operands, fp32 accumulation in TMEM.
//
// Replaces deskworld nn.linear (nn.py:43-47) and the matmul forward/backward of
// autodiff.Tensor.__matmul__ (autodiff.py:180-193): the forward (X.W), the input
// gradient (dY.W^T) and the weight gradient (X^T.dY) are the same kernel with the
// operand "major-ness" carried in the UMMA instruction descriptor, so no operand is
// ever transposed in HBM.
//
// Roles (320 threads, one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: A/B tiles -> smem ring (128B swizzle), mbarrier tx
//   warp 1      MMA issuer: one thread issues tcgen05.mma (M=128, N=BN, K=16)
//   warps 2..9  epilogue: tcgen05.ld TMEM -> registers -> fused epilogue -> HBM
//               (two warps per TMEM lane quarter, each owning half of the columns)
// TMEM holds two BN-column fp32 accumulators so the epilogue of tile i overlaps the
// main loop of tile i+1.
#include <stdlib.h>
#include <string.h>

#include <mutex>

#include "common.h"
#include "ptx.cuh"

#include <cuda_fp16.h>

#ifdef JZ_GEMM_PROF
__device__ unsigned long long g_gemm_prof[64 * 8];
__device__ int g_gemm_dbg;
__device__ long long g_gemm_ph[64 * 4];
#define PH_T(v) long long v = clock64()
#define PH_ADD(i, t0)                                                                     \
  do {                                                                                    \
    if (blockIdx.x == 0 && warp == 2 && lane == 0 && ti < 64) g_gemm_ph[ti * 4 + (i)] += clock64() - (t0); \
  } while (0)
#define GPROF(slot)                                                                     \
  do {                                                                                  \
    if (blockIdx.x == 0 && ti < 64) g_gemm_prof[ti * 8 + (slot)] = clock64();          \
  } while (0)
#define GDBG (dbg_)
#else
#define GDBG 0
#define PH_T(v) \
  do {          \
  } while (0)
#define PH_ADD(i, t0) \
  do {                \
  } while (0)
#define GPROF(slot) \
  do {              \
  } while (0)
#endif

namespace jz {

// epilogue warps: 2 per TMEM lane quarter (16 measured slower: register cap 96 + spills and one
// fewer pipeline stage)
#ifndef JZ_GEMM_EPI_WARPS
#define JZ_GEMM_EPI_WARPS 8
#endif
template <bool PAIR>
constexpr int epi_warps() { return PAIR ? JZ_GEMM_EPI_WARPS : 8; }
template <bool PAIR>
constexpr int gemm_threads() { return 64 + 32 * epi_warps<PAIR>(); }
constexpr int BM = 128;
constexpr int BK = 64;

struct GemmParams {
  int M, N, K;
  int m_tiles, n_tiles, splits, kb_total, kb_per_split;
  int epi;
  void* D;
  int64_t ldd;
  const float* bias;
  const void* aux;
  int64_t ldaux;
  void* D2;
  int64_t ldd2;
  float* colsum;  // optional per-32-row-block column sums of the bf16 output [ceil(M/32)][N]
  int tma_epi;    // 1: smem-staged epilogue, 0: direct per-thread stores (unaligned shapes)
  int store_tma;  // staged epilogue writes with TMA bulk stores (1) or coalesced st.global (0)
  // LayerNorm-fused epilogues (kernel template LNX != 0; N = 512 = two 256-column pair tiles of
  // the same rows, run back to back by one CTA pair so a row's statistics close in the pair):
  //   LNX = 1  D f32 = aux + acc + bias (the residual stream), ln_out16 = LN(D) bf16, mean/rstd out
  //   LNX = 2  LN backward of dy = acc: D f32 (the residual gradient) (+)= LN_bwd(dy; ln_x, mean,
  //            rstd, gamma); D2 bf16 copy of D; per-warp column partials of dgamma/dbeta/colsum(D)
  const float* ln_gamma;
  const float* ln_beta;
  float* ln_mean;
  float* ln_rstd;
  __nv_bfloat16* ln_out16;
  float* ln_part;        // LNX = 2: [3][nparts][N]
  int64_t ln_nparts;
  int64_t ln_skip;       // LNX = 1: rows r % ln_skip == 0 get no LN output; output rows compacted
  int ln_accumulate;     // LNX = 2: D += (1) or D = (0)
  float ln_eps;
};

struct EpiMaps {
  CUtensorMap d, d2, aux;
};

// Coalesced write-out of one warp's 32x128-byte staging tile (rows swizzled in 16-byte chunks):
// each instruction covers 4 rows x 128 contiguous bytes. The LSU path keeps the per-SM TMA unit
// free for operand loads (TMA stores measurably delayed them on epilogue-heavy shapes).
__device__ __forceinline__ void stg_write_rows(const uint8_t* stg, uint8_t* gbase, int64_t ld_bytes, int rows_ok,
                                               int cols_bytes, int lane) {
  const int c = lane & 7;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = 4 * i + (lane >> 3);
    if (r < rows_ok && c * 16 < cols_bytes)
      *reinterpret_cast<uint4*>(gbase + r * ld_bytes + c * 16) =
          *reinterpret_cast<const uint4*>(stg + r * 128 + ((c ^ (r & 7)) << 4));
  }
}

// PAIR: a cluster of two CTAs runs one cta_group::2 MMA of M = 256; each CTA stages its own 128
// rows of A and half of the BN columns of B, so operand bytes per MAC drop by a third.
// LNX (LayerNorm-fused epilogue): four 4 KB staging tiles per epilogue warp (prefetched fp32 input
// tiles + output tiles), paid for with three operand stages instead of six.
template <int BN, bool PAIR = false, int LNX = 0, bool DB = false>
struct GemmShape {
  static constexpr int B_ROWS = PAIR ? BN / 2 : BN;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // per epilogue warp: 32 rows x 128 B tiles, 128B-swizzled (LNX 1: two fp32 + two bf16 tiles,
  // LNX 2: four fp32 tiles)
  // DB: two 4 KB staging tiles per epilogue warp (aux prefetched one chunk ahead / two outputs in flight)
  static constexpr int STG_BYTES = LNX == 1 ? 12288 : (LNX == 2 ? 16384 : (DB ? 8192 : 4096));
  static constexpr int STAGES_RAW = ((PAIR ? 192 : 200) * 1024 - 8 * (STG_BYTES - 4096)) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int EW = epi_warps<PAIR>();
  static constexpr int BAR_BYTES = 512;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EW * STG_BYTES + 1024 + BAR_BYTES + BN * 4;
};

JZ_DEV float fast_tanh(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

JZ_DEV float gelu_fast(float x) {
  const float c = 0.7978845608028654f;
  float inner = (x + 0.044715f * (x * x * x)) * c;
  return 0.5f * (x * (1.0f + fast_tanh(inner)));
}

// gelu'(x) for two packed pre-activations in f16x2 arithmetic (one MUFU op per pair). Inputs are
// clamped to +-10 where gelu' is 0 / 1 to f16 precision; the error (~2^-11 absolute on tanh) matches
// the fp32 tanh.approx path it replaces, well inside the bf16 output rounding.
JZ_DEV float2 gelu_grad_pair(uint32_t pre_bf16x2) {
  const float2 f = unpack_bf16(pre_bf16x2);
  __half2 x = __floats2half2_rn(f.x, f.y);
  x = __hmax2(__hmin2(x, __float2half2_rn(10.0f)), __float2half2_rn(-10.0f));
  const __half2 one = __float2half2_rn(1.0f), half = __float2half2_rn(0.5f);
  const __half2 c = __float2half2_rn(0.7978845608028654f);
  const __half2 x2 = __hmul2(x, x);
  const __half2 inner = __hmul2(__hfma2(__hmul2(__float2half2_rn(0.044715f), x2), x, x), c);
  __half2 t;
  asm("tanh.approx.f16x2 %0, %1;" : "=r"(*reinterpret_cast<uint32_t*>(&t)) : "r"(*reinterpret_cast<const uint32_t*>(&inner)));
  const __half2 a = __hmul2(half, __hadd2(one, t));
  const __half2 b = __hmul2(__hmul2(__hmul2(half, x), __hfma2(__hneg2(t), t, one)),
                            __hmul2(c, __hfma2(__float2half2_rn(0.134145f), x2, one)));
  return __half22float2(__hadd2(a, b));
}

// gelu(x) (fp32, written as bf16) and gelu'(x) (f16x2, saved for the backward) of two packed
// values from one f16x2 tanh: the backward epilogue then only multiplies (JZ_EPI_MUL_F16).
// tanh.approx.f16x2 has ~2^-11 absolute error, the accuracy of the fp32 tanh.approx it shares.
JZ_DEV uint32_t gelu_and_grad_pair(float& x0, float& x1) {
  __half2 x = __floats2half2_rn(x0, x1);
  x = __hmax2(__hmin2(x, __float2half2_rn(10.0f)), __float2half2_rn(-10.0f));
  const float c = 0.7978845608028654f;
  const __half2 x2 = __hmul2(x, x);
  const __half2 inner = __hmul2(x, __hfma2(x2, __float2half2_rn(c * 0.044715f), __float2half2_rn(c)));
  __half2 t;
  asm("tanh.approx.f16x2 %0, %1;" : "=r"(*reinterpret_cast<uint32_t*>(&t)) : "r"(*reinterpret_cast<const uint32_t*>(&inner)));
  const __half2 half = __float2half2_rn(0.5f);
  const __half2 a = __hfma2(t, half, half);                                   // 0.5 (1 + t)
  const __half2 omt = __hfma2(__hneg2(t), t, __float2half2_rn(1.0f));         // 1 - t^2
  const __half2 poly = __hfma2(x2, __float2half2_rn(0.5f * c * 0.134145f), __float2half2_rn(0.5f * c));
  const __half2 g = __hfma2(__hmul2(x, poly), omt, a);                        // gelu'(x)
  const float2 af = __half22float2(a);
  x0 *= af.x;  // gelu = x * 0.5 (1 + t), on the unclamped fp32 value
  x1 *= af.y;
  return *reinterpret_cast<const uint32_t*>(&g);
}

JZ_DEV float2 unpack_f16(uint32_t w) { return __half22float2(*reinterpret_cast<const __half2*>(&w)); }

JZ_DEV float gelu_grad_fast(float x) {
  const float c = 0.7978845608028654f;
  float x2 = x * x;
  float t = fast_tanh((x + 0.044715f * x2 * x) * c);
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * (c * (1.0f + 0.134145f * x2));
}

// Epilogue for one thread: row m, 32 consecutive columns starting at n.
JZ_DEV void epilogue_chunk(const GemmParams& p, int m, int n, float (&v)[32], float* ws_out) {
  const int N = p.N;
  float gbuf_[32];
  const bool full = (n + 32 <= N);
  if (ws_out != nullptr) {  // split-K partial: plain fp32 [M][N]
    float* dst = ws_out + (int64_t)m * N + n;
    if (full && (N % 4 == 0)) {
#pragma unroll
      for (int j = 0; j < 32; j += 4)
        *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
      for (int j = 0; j < 32; ++j)
        if (n + j < N) dst[j] = v[j];
    }
    return;
  }
  const bool vec8 = full && (p.ldd % 8 == 0);
  switch (p.epi) {
    case JZ_EPI_F32:
    case JZ_EPI_F32_ACC:
    case JZ_EPI_RESID:
    case JZ_EPI_BF16_F32: {
      float* dst = reinterpret_cast<float*>(p.D) + (int64_t)m * p.ldd + n;
      if (p.epi == JZ_EPI_RESID) {
        const float* src = reinterpret_cast<const float*>(p.aux) + (int64_t)m * p.ldaux + n;
        if (full && (p.ldaux % 4 == 0)) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 r = *reinterpret_cast<const float4*>(src + j);
            v[j] += r.x; v[j + 1] += r.y; v[j + 2] += r.z; v[j + 3] += r.w;
          }
        } else {
          for (int j = 0; j < 32; ++j)
            if (n + j < N) v[j] += src[j];
        }
      } else if (p.epi == JZ_EPI_F32_ACC) {
        if (full && (p.ldd % 4 == 0)) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            float4 r = *reinterpret_cast<const float4*>(dst + j);
            v[j] += r.x; v[j + 1] += r.y; v[j + 2] += r.z; v[j + 3] += r.w;
          }
        } else {
          for (int j = 0; j < 32; ++j)
            if (n + j < N) v[j] += dst[j];
        }
      }
      if (full && (p.ldd % 4 == 0)) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
        for (int j = 0; j < 32; ++j)
          if (n + j < N) dst[j] = v[j];
      }
      if (p.epi == JZ_EPI_BF16_F32) {
        __nv_bfloat16* d2 = reinterpret_cast<__nv_bfloat16*>(p.D2) + (int64_t)m * p.ldd2 + n;
        if (full && (p.ldd2 % 8 == 0)) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            uint4 w = make_uint4(pack_bf16(v[j], v[j + 1]), pack_bf16(v[j + 2], v[j + 3]),
                                 pack_bf16(v[j + 4], v[j + 5]), pack_bf16(v[j + 6], v[j + 7]));
            *reinterpret_cast<uint4*>(d2 + j) = w;
          }
        } else {
          for (int j = 0; j < 32; ++j)
            if (n + j < N) d2[j] = __float2bfloat16_rn(v[j]);
        }
      }
      break;
    }
    case JZ_EPI_BF16:
    case JZ_EPI_GELU:
    case JZ_EPI_GELU_BWD:
    case JZ_EPI_GELU_DG:
    case JZ_EPI_MUL_F16: {
      if (p.epi == JZ_EPI_GELU_DG) {
        __half* d2 = reinterpret_cast<__half*>(p.D2) + (int64_t)m * p.ldd2 + n;
        for (int j = 0; j < 32; j += 2) {
          const uint32_t g = gelu_and_grad_pair(v[j], v[j + 1]);
          const float2 gf = unpack_f16(g);
          if (n + j < N) d2[j] = __float2half_rn(gf.x);
          if (n + j + 1 < N) d2[j + 1] = __float2half_rn(gf.y);
        }
      } else if (p.epi == JZ_EPI_MUL_F16) {
        const __half* g = reinterpret_cast<const __half*>(p.aux) + (int64_t)m * p.ldaux + n;
        for (int j = 0; j < 32; ++j)
          if (n + j < N) v[j] *= __half2float(g[j]);
      } else if (p.epi == JZ_EPI_GELU && p.D2 == nullptr) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = gelu_fast(v[j]);
      } else if (p.epi == JZ_EPI_GELU) {
        __nv_bfloat16* d2 = reinterpret_cast<__nv_bfloat16*>(p.D2) + (int64_t)m * p.ldd2 + n;
#pragma unroll
        for (int j = 0; j < 32; ++j) {  // D2 = pre-activation, v <- gelu(v)
          gbuf_[j] = v[j];
          v[j] = gelu_fast(v[j]);
        }
        if (full && (p.ldd2 % 8 == 0)) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            uint4 w = make_uint4(pack_bf16(gbuf_[j], gbuf_[j + 1]), pack_bf16(gbuf_[j + 2], gbuf_[j + 3]),
                                 pack_bf16(gbuf_[j + 4], gbuf_[j + 5]), pack_bf16(gbuf_[j + 6], gbuf_[j + 7]));
            *reinterpret_cast<uint4*>(d2 + j) = w;
          }
        } else {
          for (int j = 0; j < 32; ++j)
            if (n + j < N) d2[j] = __float2bfloat16_rn(gbuf_[j]);
        }
      } else if (p.epi == JZ_EPI_GELU_BWD) {
        const __nv_bfloat16* pre =
            reinterpret_cast<const __nv_bfloat16*>(p.aux) + (int64_t)m * p.ldaux + n;
        if (full && (p.ldaux % 8 == 0)) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) {
            uint4 w = *reinterpret_cast<const uint4*>(pre + j);
            float2 a = unpack_bf16(w.x), b = unpack_bf16(w.y), c = unpack_bf16(w.z),
                   d = unpack_bf16(w.w);
            v[j] *= gelu_grad_fast(a.x); v[j + 1] *= gelu_grad_fast(a.y);
            v[j + 2] *= gelu_grad_fast(b.x); v[j + 3] *= gelu_grad_fast(b.y);
            v[j + 4] *= gelu_grad_fast(c.x); v[j + 5] *= gelu_grad_fast(c.y);
            v[j + 6] *= gelu_grad_fast(d.x); v[j + 7] *= gelu_grad_fast(d.y);
          }
        } else {
          for (int j = 0; j < 32; ++j)
            if (n + j < N) v[j] *= gelu_grad_fast(__bfloat162float(pre[j]));
        }
      }
      __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(p.D) + (int64_t)m * p.ldd + n;
      if (vec8) {
#pragma unroll
        for (int j = 0; j < 32; j += 8) {
          uint4 w = make_uint4(pack_bf16(v[j], v[j + 1]), pack_bf16(v[j + 2], v[j + 3]),
                               pack_bf16(v[j + 4], v[j + 5]), pack_bf16(v[j + 6], v[j + 7]));
          *reinterpret_cast<uint4*>(dst + j) = w;
        }
      } else {
        for (int j = 0; j < 32; ++j)
          if (n + j < N) dst[j] = __float2bfloat16_rn(v[j]);
      }
      break;
    }
    default:
      break;
  }
}

// k-th output tile of a persistent CTA (pair).  LNX kernels run the two 256-column tiles of one
// 256-row block back to back (tile 2 mb + n in accumulator buffer n), so the epilogue owns whole
// 512-wide rows; everything else strides single tiles (split-K slabs innermost).
template <int LNX>
JZ_DEV bool tile_at(const GemmParams& p, int first, int stride, int it, int& tile, int& split) {
  if constexpr (LNX != 0) {
    const int mb = first + (it >> 1) * stride;
    if (mb >= p.m_tiles) return false;
    tile = 2 * mb + (it & 1);
    split = 0;
    return true;
  } else {
    const int u = first + it * stride;
    if (u >= p.m_tiles * p.n_tiles * p.splits) return false;
    tile = u / p.splits;
    split = u % p.splits;
    return true;
  }
}

// Row-statistics exchange between the two epilogue warps that share a TMEM lane quarter
// (column halves 0 and 1 of every 256-column tile): warp c1 posts its partial, warp c0 adds its
// own and posts the total, both use that one total (bitwise-identical statistics for the row).
JZ_DEV float2 ln_row_total(float* red, uint32_t quarter, int chalf, int lane, float a, float b) {
  float* slot = red + quarter * 64;
  const int bar = 2 + (int)quarter;
  if (chalf == 1) {
    slot[lane] = a;
    slot[32 + lane] = b;
  }
  asm volatile("bar.sync %0, 64;" ::"r"(bar) : "memory");
  if (chalf == 0) {
    a += slot[lane];
    b += slot[32 + lane];
    slot[lane] = a;
    slot[32 + lane] = b;
  }
  asm volatile("bar.sync %0, 64;" ::"r"(bar) : "memory");
  if (chalf == 1) {
    a = slot[lane];
    b = slot[32 + lane];
  }
  return make_float2(a, b);
}

// Column sums of a warp's 32 rows x 32 columns (lane = row) through its 4 KB staging tile
// (128B-swizzled rows: conflict-free row writes and column reads); returns column `lane`.
JZ_DEV float ln_colsum32(uint8_t* stg, const float (&v)[32], int lane) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    *reinterpret_cast<float4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) =
        make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
  __syncwarp();
  float s = 0.f;
  const int c = lane >> 2, w = (lane & 3) * 4;
#pragma unroll 8
  for (int r = 0; r < 32; ++r) s += *reinterpret_cast<const float*>(stg + r * 128 + ((c ^ (r & 7)) << 4) + w);
  __syncwarp();
  return s;
}

JZ_DEV void tmem_ld32f(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  tmem_ld_32x32b_x32(taddr, r);
  tmem_ld_wait();
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
}

// Staging-tile helpers (32 rows x 32 columns per warp; lane = row).  fp32 tiles: 128-byte rows,
// 128B swizzle (16-byte chunk c of row r at c ^ (r & 7)); bf16 tiles: 64-byte rows, 64B swizzle
// (chunk c at c ^ ((r >> 1) & 3)).  Row accesses by the 32 lanes are bank-conflict free.
JZ_DEV void stg_row_f32_ld(const uint8_t* t, int r, float (&v)[32]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const float4 w = *reinterpret_cast<const float4*>(t + r * 128 + ((c ^ (r & 7)) << 4));
    v[4 * c] = w.x; v[4 * c + 1] = w.y; v[4 * c + 2] = w.z; v[4 * c + 3] = w.w;
  }
}
JZ_DEV void stg_row_f32_st(uint8_t* t, int r, const float (&v)[32]) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    *reinterpret_cast<float4*>(t + r * 128 + ((c ^ (r & 7)) << 4)) = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
}
JZ_DEV void stg_row_bf16_st(uint8_t* t, int r, const float (&v)[32]) {
#pragma unroll
  for (int c = 0; c < 4; ++c)
    *reinterpret_cast<uint4*>(t + r * 64 + ((c ^ ((r >> 1) & 3)) << 4)) =
        make_uint4(pack_bf16(v[8 * c], v[8 * c + 1]), pack_bf16(v[8 * c + 2], v[8 * c + 3]),
                   pack_bf16(v[8 * c + 4], v[8 * c + 5]), pack_bf16(v[8 * c + 6], v[8 * c + 7]));
}

// acc[0] += v, then rotate left by one: after 8 calls every slot got its chunk's value in order
JZ_DEV void rot_add(float (&acc)[8], float v) {
  const float a0 = acc[0] + v;
#pragma unroll
  for (int i = 0; i < 7; ++i) acc[i] = acc[i + 1];
  acc[7] = a0;
}

// LNX epilogue of one CTA (8 warps; warp = lane quarter x column half), persistent over 256-row
// blocks.  Per block: accumulator buffer n holds columns [256 n, 256 n + 256) of the block's rows;
// a warp walks its 8 chunks of 32 columns (k = 4 n + cc).  Every global tile moves by TMA through
// the warp's 4 staging tiles T0..T3, the next chunk's input tiles prefetched while this one computes.
//  LNX = 1 (LayerNorm forward, nn.py:35-40, two-pass): pass A x = acc + bias + resid (T0/T1) -> D and
//          back into TMEM, row sums; pass B centred squares (TMEM only); pass C (x - mean) rstd gamma
//          + beta -> bf16 (two 2 KB tiles after T1) -> ln_out16.
//  LNX = 2 (LayerNorm backward): pass A x (T0/T1): row sums of dxn = dy gamma and dxn xhat, column
//          partials of dy xhat and dy (T2 scratch); pass B x, D (T0,T1 / T2,T3): dx = rstd (dxn -
//          mean(dxn) - xhat mean(dxn xhat)) added to D (in place in its tile) -> D, bf16 copy -> D2
//          (in the x tile), column partials of the new D.
template <int LNX, bool PAIR>
JZ_DEV void ln_epilogue(const GemmParams& p, const EpiMaps& em, uint32_t tmem_base, uint64_t* tfull_bar,
                        uint64_t* tempty_bar, uint64_t* bars, float* red, uint8_t* stg, int first_unit,
                        int unit_stride, uint32_t rank, int warp, int lane) {
  constexpr int TM = PAIR ? 2 * BM : BM;
  constexpr int TB = 4096;
  const uint32_t quarter = warp & 3;
  const int chalf = (warp - 2) >> 2;
  const int N = p.N;  // 512
  const float invN = 1.0f / (float)N;
  uint32_t acc_phase = 0;
  uint32_t bpar = 0;  // phase bit per staging barrier (bit = slot)
  float pdg[8], pdb[8], pdr[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) pdg[k] = pdb[k] = pdr[k] = 0.f;
  auto release = [&](int n) {
    tc_fence_before();
    __syncwarp();
    if (lane == 0) {
      if constexpr (PAIR) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&tempty_bar[n]), 0));
      else mbar_arrive_relaxed(&tempty_bar[n]);
    }
  };
  auto col_of = [&](int k) { return (k >> 2) * 256 + chalf * 128 + (k & 3) * 32; };
  auto tile = [&](int t) { return stg + t * TB; };
  // previous async (TMA) stores and generic reads of the tiles are done before they are refilled
  auto drain = [&]() {
    if (lane == 0) bulk_wait_read0();
    __syncwarp();
  };
  for (int mb = first_unit; mb < p.m_tiles; mb += unit_stride, acc_phase ^= 1) {
    const int row0 = mb * TM + (int)rank * BM + (int)quarter * 32;
    const int row = row0 + lane;
    const bool live = row < p.M;
    const uint32_t tq = tmem_base + ((quarter * 32) << 16) + chalf * 128;
    // loads one or two fp32 tiles of chunk k into T(2 slot), T(2 slot + 1) on bars[slot]
    auto load = [&](int k, int slot, const CUtensorMap* m0, uint8_t* d0, const CUtensorMap* m1, uint8_t* d1) {
      if (lane == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&bars[slot], m1 ? 2 * TB : TB);
        tma_load_2d(d0, m0, &bars[slot], col_of(k), row0);
        if (m1) tma_load_2d(d1, m1, &bars[slot], col_of(k), row0);
      }
    };
    auto wait_tiles = [&](int slot) {
      mbar_wait(&bars[slot], (bpar >> slot) & 1u);
      bpar ^= 1u << slot;
    };
    auto store = [&](const CUtensorMap* m, const uint8_t* src, int k) {
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) tma_store_2d(m, src, col_of(k), row0);
    };
    if constexpr (LNX == 1) {
      float s = 0.f;
      drain();
      load(0, 0, &em.aux, tile(0), nullptr, nullptr);
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        const int n = k >> 2, col = col_of(k);
        if ((k & 3) == 0) {
          mbar_wait(&tfull_bar[n], acc_phase);
          tc_fence_after();
        }
        if (k + 1 < 8) {
          drain();  // chunk k - 1's store out of this slot has read it
          load(k + 1, (k + 1) & 1, &em.aux, tile((k + 1) & 1), nullptr, nullptr);
        }
        float x[32], r[32];
        tmem_ld32f(tq + n * 256 + (k & 3) * 32, x);
        const float4* b4 = reinterpret_cast<const float4*>(p.bias + col);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 b = __ldg(b4 + j);
          x[4 * j] += b.x; x[4 * j + 1] += b.y; x[4 * j + 2] += b.z; x[4 * j + 3] += b.w;
        }
        wait_tiles(k & 1);
        uint8_t* t = tile(k & 1);
        stg_row_f32_ld(t, lane, r);
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j] += r[j];
        stg_row_f32_st(t, lane, x);
        store(&em.d, t, k);
        if (lane == 0) bulk_commit();
        if (live) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) s += (x[j] + x[j + 1]) + (x[j + 2] + x[j + 3]);
        }
        uint32_t* xu = reinterpret_cast<uint32_t*>(x);
        tmem_st_32x32b_x16(tq + n * 256 + (k & 3) * 32, *reinterpret_cast<const uint32_t(*)[16]>(xu));
        tmem_st_32x32b_x16(tq + n * 256 + (k & 3) * 32 + 16, *reinterpret_cast<const uint32_t(*)[16]>(xu + 16));
      }
      tmem_st_wait();
      const float mu = ln_row_total(red, quarter, chalf, lane, s, 0.f).x * invN;
      float q = 0.f;
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        float x[32];
        tmem_ld32f(tq + (k >> 2) * 256 + (k & 3) * 32, x);
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float a = x[j] - mu, b = x[j + 1] - mu;
          q += a * a + b * b;
        }
      }
      const float var = ln_row_total(red, quarter, chalf, lane, live ? q : 0.f, 0.f).x * invN;
      const float rs = 1.0f / sqrtf(var + p.ln_eps);
      const bool skip = p.ln_skip > 0;
      const bool out_ok = live && (!skip || (row % p.ln_skip) != 0);
      const int64_t orow = skip ? row - row / p.ln_skip - 1 : row;
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        const int n = k >> 2, col = col_of(k);
        float x[32];
        tmem_ld32f(tq + n * 256 + (k & 3) * 32, x);
        if ((k & 3) == 3) release(n);  // buffer n fully read: the next block's MMAs may overwrite it
        const float4* g4 = reinterpret_cast<const float4*>(p.ln_gamma + col);
        const float4* be4 = reinterpret_cast<const float4*>(p.ln_beta + col);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 g = __ldg(g4 + j), b = __ldg(be4 + j);
          x[4 * j] = (x[4 * j] - mu) * rs * g.x + b.x;
          x[4 * j + 1] = (x[4 * j + 1] - mu) * rs * g.y + b.y;
          x[4 * j + 2] = (x[4 * j + 2] - mu) * rs * g.z + b.z;
          x[4 * j + 3] = (x[4 * j + 3] - mu) * rs * g.w + b.w;
        }
        if (skip) {  // compacted rows (final LayerNorm dropping s = 0): per-row stores
          if (out_ok) {
            __nv_bfloat16* o16 = p.ln_out16 + orow * (int64_t)N + col;
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(o16 + 8 * j) =
                  make_uint4(pack_bf16(x[8 * j], x[8 * j + 1]), pack_bf16(x[8 * j + 2], x[8 * j + 3]),
                             pack_bf16(x[8 * j + 4], x[8 * j + 5]), pack_bf16(x[8 * j + 6], x[8 * j + 7]));
          }
        } else {
          if (lane == 0) bulk_wait_read1();  // chunk k - 2's store out of this tile has read it
          __syncwarp();
          uint8_t* t = stg + 2 * TB + (k & 1) * (TB / 2);  // 64-byte-row bf16 tiles
          stg_row_bf16_st(t, lane, x);
          store(&em.d2, t, k);
          if (lane == 0) bulk_commit();
        }
      }
      if (live && chalf == 0) {
        p.ln_mean[row] = mu;
        p.ln_rstd[row] = rs;
      }
    } else {
      const bool has16 = p.D2 != nullptr;
      const float mu = live ? p.ln_mean[row] : 0.f, rs = live ? p.ln_rstd[row] : 0.f;
      float s1 = 0.f, s2 = 0.f;
      drain();
      load(0, 0, &em.aux, tile(0), nullptr, nullptr);
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        const int n = k >> 2, col = col_of(k);
        if ((k & 3) == 0) {
          mbar_wait(&tfull_bar[n], acc_phase);
          tc_fence_after();
        }
        if (k + 1 < 8) load(k + 1, (k + 1) & 1, &em.aux, tile((k + 1) & 1), nullptr, nullptr);
        float g[32], x[32];
        tmem_ld32f(tq + n * 256 + (k & 3) * 32, g);
        wait_tiles(k & 1);
        stg_row_f32_ld(tile(k & 1), lane, x);
        if (!live) {
#pragma unroll
          for (int j = 0; j < 32; ++j) g[j] = x[j] = 0.f;
        }
        const float4* g4 = reinterpret_cast<const float4*>(p.ln_gamma + col);
        float gx[32];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 gm = __ldg(g4 + j);
          const float gmv[4] = {gm.x, gm.y, gm.z, gm.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = 4 * j + e;
            const float xh = (x[i] - mu) * rs;
            const float dn = g[i] * gmv[e];
            s1 += dn;
            s2 += dn * xh;
            gx[i] = g[i] * xh;
          }
        }
        __syncwarp();  // every lane has read its x row before the tile is refilled (next-next chunk)
        // k-th column partial: the accumulators rotate by one slot per chunk (register-resident; a
        // runtime index would put them in local memory), back in place after the 8 chunks
        rot_add(pdg, ln_colsum32(tile(2), gx, lane));
        rot_add(pdb, ln_colsum32(tile(2), g, lane));
      }
      const float2 tot = ln_row_total(red, quarter, chalf, lane, s1, s2);
      const float m1 = tot.x * invN, m2 = tot.y * invN;
      drain();
      load(0, 0, &em.aux, tile(0), &em.d, tile(1));
#pragma unroll 1
      for (int k = 0; k < 8; ++k) {
        const int n = k >> 2, col = col_of(k);
        if (k + 1 < 8) {
          drain();  // chunk k - 1's stores out of the other slot have read it
          const int sl = (k + 1) & 1;
          load(k + 1, sl, &em.aux, tile(2 * sl), &em.d, tile(2 * sl + 1));
        }
        float g[32], x[32], o[32];
        tmem_ld32f(tq + n * 256 + (k & 3) * 32, g);
        if ((k & 3) == 3) release(n);
        const int sl = k & 1;
        uint8_t* tx = tile(2 * sl);
        uint8_t* td = tile(2 * sl + 1);
        wait_tiles(sl);
        stg_row_f32_ld(tx, lane, x);
        if (p.ln_accumulate) stg_row_f32_ld(td, lane, o);
        else {
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = 0.f;
        }
        const float4* g4 = reinterpret_cast<const float4*>(p.ln_gamma + col);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float4 gm = __ldg(g4 + j);
          const float gmv[4] = {gm.x, gm.y, gm.z, gm.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = 4 * j + e;
            const float xh = (x[i] - mu) * rs;
            const float dn = g[i] * gmv[e];
            o[i] += rs * (dn - m1 - xh * m2);
          }
        }
        stg_row_f32_st(td, lane, o);
        store(&em.d, td, k);
        if (!live) {
#pragma unroll
          for (int j = 0; j < 32; ++j) o[j] = 0.f;
        }
        rot_add(pdr, ln_colsum32(tx, o, lane));  // x tile is free: column-sum scratch
        if (has16) {
          stg_row_bf16_st(tx, lane, o);
          store(&em.d2, tx, k);
        }
        if (lane == 0) bulk_commit();
      }
    }
  }
  if (lane == 0) bulk_wait0();
  if constexpr (LNX == 2) {
    // one partial row per (CTA, lane quarter); this warp owns columns chalf*128 + 256 n + 32 cc + lane
    const int64_t prow = (int64_t)blockIdx.x * 4 + quarter;
    const int64_t plane = p.ln_nparts * N;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int col = col_of(k) + lane;
      p.ln_part[prow * N + col] = pdg[k];
      p.ln_part[plane + prow * N + col] = pdb[k];
      p.ln_part[2 * plane + prow * N + col] = pdr[k];
    }
  }
}

template <int BN, bool A_MN, bool B_MN, bool PAIR, int LNX = 0, bool DB = false>
__global__ void __launch_bounds__(gemm_threads<PAIR>(), 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ EpiMaps em, GemmParams p, float* ws) {
  using S = GemmShape<BN, PAIR, LNX, DB>;
  constexpr int TM = PAIR ? 2 * BM : BM;  // rows per (pair) tile
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  const int first_unit = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int unit_stride = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int kEpiWarps = S::EW;
  uint8_t* stg_base = smem + S::STAGES * S::STAGE_BYTES;  // kEpiWarps x 4 KB (1024-aligned)
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stg_base + kEpiWarps * S::STG_BYTES);
  uint64_t* empty_bar = full_bar + S::STAGES;
  uint64_t* tfull_bar = empty_bar + S::STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint64_t* aux_bar = tempty_bar + 2;  // [kEpiWarps] ([2 kEpiWarps] for LNX / DB)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aux_bar + ((LNX || DB) ? 2 : 1) * kEpiWarps);
  float* sbias = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(full_bar) + S::BAR_BYTES);  // [BN]

  const uint32_t warp = __shfl_sync(0xffffffffu, warp_id(), 0);  // warp-uniform (uniform-datapath MMA operands)
  const uint32_t lane = lane_id();
#ifdef JZ_GEMM_PROF
  const int dbg_ = g_gemm_dbg;
#endif

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (p.tma_epi) {
      if (p.store_tma) tma_prefetch_desc(&em.d);
      if (p.store_tma && p.epi == JZ_EPI_GELU && p.D2 != nullptr) tma_prefetch_desc(&em.d2);
      if (p.epi == JZ_EPI_GELU_DG && p.store_tma) tma_prefetch_desc(&em.d2);
      if (p.epi == JZ_EPI_RESID || p.epi == JZ_EPI_F32_ACC || p.epi == JZ_EPI_GELU_BWD || p.epi == JZ_EPI_MUL_F16)
        tma_prefetch_desc(&em.aux);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < S::STAGES; ++i) {
      mbar_init(&full_bar[i], 1);
      mbar_init(&empty_bar[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull_bar[i], 1);
      mbar_init(&tempty_bar[i], (PAIR ? 2 : 1) * kEpiWarps);  // one arrival per epilogue warp of the pair
    }
    for (int i = 0; i < ((LNX || DB) ? 2 : 1) * kEpiWarps; ++i) mbar_init(&aux_bar[i], 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (PAIR) tmem_alloc_pair<S::TMEM_COLS>(tmem_slot);
    else tmem_alloc<S::TMEM_COLS>(tmem_slot);
  }
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // peer barriers initialised before any remote arrive
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  const int units = p.m_tiles * p.n_tiles * p.splits;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      // pair: every load signals the leader's full barrier, which expects both CTAs' bytes
      const uint32_t full0 = PAIR ? mapa_shared(smem_u32(&full_bar[0]), 0) : 0;
      int tile, split;
      for (int it = 0; tile_at<LNX>(p, first_unit, unit_stride, it, tile, split); ++it) {
        const int m0 = (tile / p.n_tiles) * TM + (int)rank * BM;
        const int nb0 = (tile % p.n_tiles) * BN + (int)rank * S::B_ROWS;
        const int kb0 = split * p.kb_per_split;
        const int kb1 = min(p.kb_total, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          if (rank == 0) mbar_arrive_expect_tx(&full_bar[stage], (PAIR ? 2 : 1) * S::STAGE_BYTES);
          uint8_t* a_dst = smem + stage * S::STAGE_BYTES;
          uint8_t* b_dst = a_dst + S::A_BYTES;
          const int k = kb * BK;
          auto load = [&](uint8_t* dst, const CUtensorMap* map, int c0, int c1) {
            if constexpr (PAIR) tma_load_2d_pair(dst, map, full0 + stage * 8, c0, c1);
            else tma_load_2d(dst, map, &full_bar[stage], c0, c1);
          };
          if (!A_MN) {
            load(a_dst, &tmA, k, m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) load(a_dst + j * (64 * BK * 2), &tmA, m0 + 64 * j, k);
          }
          if (!B_MN) {
            load(b_dst, &tmB, k, nb0);
          } else {
#pragma unroll
            for (int j = 0; j < S::B_ROWS / 64; ++j) load(b_dst + j * (64 * BK * 2), &tmB, nb0 + 64 * j, k);
          }
          if (++stage == S::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // the whole warp runs the issue loop (convergent: operands stay warp-uniform, no per-MMA
    // elect/R2UR waterfall); one elected lane issues each tcgen05 instruction
    if (rank == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(TM, BN, A_MN, B_MN);
      const uint32_t dhi = (uint32_t)(sdesc_sw128(0, 0, 1024) >> 32);
      const uint32_t smem_base4 = smem_u32(smem) >> 4;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int ti = 0;
      int tile_, split;
      for (int it = 0; tile_at<LNX>(p, first_unit, unit_stride, it, tile_, split); ++it, ++ti) {
        const int kb0 = split * p.kb_per_split;
        const int kb1 = min(p.kb_total, kb0 + p.kb_per_split);
        GPROF(0);
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        GPROF(1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
#ifdef JZ_GEMM_PROF
        long long fw = 0;
#endif
        for (int kb = kb0; kb < kb1; ++kb) {
#ifdef JZ_GEMM_PROF
          long long t0 = clock64();
#endif
          mbar_wait(&full_bar[stage], phase);
#ifdef JZ_GEMM_PROF
          fw += clock64() - t0;
#endif
          tc_fence_after();
          // SW128 descriptors: one shared high word, low word = (address >> 4) | (LBO >> 4) << 16
          const uint32_t a4 = (smem_base4 + stage * (S::STAGE_BYTES >> 4));
          const uint32_t b4 = a4 + (S::A_BYTES >> 4);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint32_t alo = A_MN ? a4 + kk * 128 + (((64 * BK * 2) >> 4) << 16) : a4 + kk * 2 + (1u << 16);
            const uint32_t blo = B_MN ? b4 + kk * 128 + (((64 * BK * 2) >> 4) << 16) : b4 + kk * 2 + (1u << 16);
            const uint64_t adesc = ((uint64_t)dhi << 32) | alo;
            const uint64_t bdesc = ((uint64_t)dhi << 32) | blo;
            if constexpr (PAIR) umma_bf16_ss_pair_w(d_tmem, adesc, bdesc, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
            else umma_bf16_ss_w(d_tmem, adesc, bdesc, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          if constexpr (PAIR) umma_commit_pair_w(&empty_bar[stage], 0x3);
          else umma_commit_w(&empty_bar[stage]);
          if (++stage == S::STAGES) { stage = 0; phase ^= 1; }
        }
        if constexpr (PAIR) umma_commit_pair_w(&tfull_bar[acc], 0x3);
        else umma_commit_w(&tfull_bar[acc]);
        GPROF(2);
#ifdef JZ_GEMM_PROF
        if (blockIdx.x == 0 && ti < 64) g_gemm_prof[ti * 8 + 6] = fw;
#endif
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if constexpr (LNX != 0) {
    ln_epilogue<LNX, PAIR>(p, em, tmem_base, tfull_bar, tempty_bar, aux_bar + 2 * (warp - 2), sbias,
                           stg_base + (warp - 2) * S::STG_BYTES, first_unit, unit_stride, rank, (int)warp, (int)lane);
  } else {
    // epilogue warps 2..9: TMEM lane quarter = warp % 4, column half = (warp - 2) / 4
    const uint32_t quarter = warp & 3;
    const int ew = warp - 2;
    const int chalf = ew >> 2;                 // column slot of this warp
    constexpr int HALF = BN / (kEpiWarps / 4);  // columns per warp
    const int etid = threadIdx.x - 64;  // 0 .. 32*kEpiWarps-1
    uint8_t* const stg_w = stg_base + ew * S::STG_BYTES;  // this warp's staging tile(s)
    uint8_t* stg = stg_w;
    uint32_t apar = 0;  // aux barrier phase bits (bit b: staging tile b under DB)
    int q = 0;          // staged chunks done by this warp (DB: the aux of chunk q sits in tile q & 1)
    int acc = 0;
    uint32_t acc_phase = 0;
    const bool has_bias = p.bias != nullptr && p.splits == 1;
    // DB with an aux operand: chunk q + 1's aux tile is loaded while chunk q computes.  The host
    // enables DB only with N % BN == 0, so every warp has columns in every tile and the next
    // processed chunk is always the next one in this sequence.
    const bool db_aux = DB && p.tma_epi && p.splits == 1 && (p.epi == JZ_EPI_GELU_BWD || p.epi == JZ_EPI_MUL_F16);
    constexpr int kChunks = HALF / 64;  // bf16-output chunks per tile per warp
    auto aux_prefetch = [&](int u_next, int cc_next, int slot) {  // chunk cc_next of unit u_next -> tile slot
      const int tile2 = u_next;  // splits == 1
      const int m0_2 = (tile2 / p.n_tiles) * TM + (int)rank * BM, n0_2 = (tile2 % p.n_tiles) * BN;
      if (lane == 0) {
        fence_proxy_async();
        mbar_arrive_expect_tx(&aux_bar[2 * ew + slot], 4096);
        tma_load_2d(stg_w + slot * 4096, &em.aux, &aux_bar[2 * ew + slot], n0_2 + chalf * HALF + cc_next * 64,
                    m0_2 + (int)quarter * 32);
      }
    };
    if (db_aux && first_unit < units) aux_prefetch(first_unit, 0, 0);
    // staged epilogue: bias comes straight from global (all lanes read the same address -> one
    // L1 broadcast per vector), so the epilogue warps never synchronise with each other
    const bool bias_vec = has_bias && (reinterpret_cast<uintptr_t>(p.bias) % 16 == 0) && (p.N % 4 == 0);
    int ti = 0;
    for (int u = first_unit; u < units; u += unit_stride, ++ti) {
      const int tile = u / p.splits, split = u % p.splits;
      const int m0 = (tile / p.n_tiles) * TM + (int)rank * BM, n0 = (tile % p.n_tiles) * BN;
      if (has_bias && !p.tma_epi) {  // direct path: stage this tile's bias in smem
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
        for (int c = etid; c < BN; c += 32 * kEpiWarps) sbias[c] = (n0 + c < p.N) ? p.bias[n0 + c] : 0.f;
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarps) : "memory");
      }
      if (warp == 2 && lane == 0) GPROF(3);
      mbar_wait(&tfull_bar[acc], acc_phase);
      if (warp == 2 && lane == 0) GPROF(4);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((quarter * 32) << 16) + acc * BN + chalf * HALF;
      const int row0 = m0 + quarter * 32;
      if (p.tma_epi) {
        // ---------- staged TMA epilogue ----------
        const bool f32out = p.splits > 1 || p.epi == JZ_EPI_F32 || p.epi == JZ_EPI_F32_ACC || p.epi == JZ_EPI_RESID;
        const bool need_aux = p.splits == 1 &&
                              (p.epi == JZ_EPI_RESID || p.epi == JZ_EPI_F32_ACC || p.epi == JZ_EPI_GELU_BWD ||
                               p.epi == JZ_EPI_MUL_F16);
        const int CW = f32out ? 32 : 64;
        const int esz = f32out ? 4 : 2;
        // split-K partials: slab `split` of the fp32 workspace, row pitch N
        uint8_t* dbase = p.splits > 1 ? reinterpret_cast<uint8_t*>(ws + (int64_t)split * p.M * p.N)
                                      : reinterpret_cast<uint8_t*>(p.D);
        const int64_t dld = (p.splits > 1 ? (int64_t)p.N : p.ldd) * esz;
        const int rows_ok = p.M - row0;
#pragma unroll 1
        for (int cc = 0; cc < HALF / CW; ++cc) {
          const int col = chalf * HALF + cc * CW;
          const int n = n0 + col;
          if (n >= p.N) break;  // warp-uniform
          const int cols_bytes = min(CW, p.N - n) * esz;
          PH_T(t_a);
          if (DB && db_aux) {
            // this chunk's aux is in tile q & 1; refill the other tile with the next chunk's once
            // the previous chunk's store has read it
            stg = stg_w + (q & 1) * 4096;
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
            if (cc + 1 < kChunks) aux_prefetch(u, cc + 1, (q + 1) & 1);
            else if (u + unit_stride < units) aux_prefetch(u + unit_stride, 0, (q + 1) & 1);
          } else if (DB && p.store_tma) {
            stg = stg_w;  // GELU_DG: gelu' goes through tile 0, gelu through tile 1
            if (lane == 0) bulk_wait_read1();  // the previous chunk's gelu' store has read tile 0
            __syncwarp();
          } else if (p.store_tma) {
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
          }
          PH_ADD(0, t_a);
          if (!DB && need_aux && lane == 0) {
            fence_proxy_async();  // generic reads of the previous chunk before the async-proxy write
            mbar_arrive_expect_tx(&aux_bar[ew], S::STG_BYTES);
            tma_load_2d(stg, &em.aux, &aux_bar[ew], n, row0);
          }
          float v[64];
          bool gelu_dg_staged = false;
          PH_T(t_b);
          {
            uint32_t* r = reinterpret_cast<uint32_t*>(v);
            tmem_ld_32x32b_x32(tbase + cc * CW, *reinterpret_cast<uint32_t(*)[32]>(r));
            if (!f32out) tmem_ld_32x32b_x32(tbase + cc * CW + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
            tmem_ld_wait();
          }
          PH_ADD(1, t_b);
          PH_T(t_c);
          if (bias_vec && n + CW <= p.N) {
            // full chunk: every bias vector load issued before the first add (no per-load predicate
            // chain; the loads are L1 broadcasts)
            const float4* b4p = reinterpret_cast<const float4*>(p.bias + n);
#pragma unroll
            for (int h = 0; h < 16; h += 8) {
              float4 b4[8];
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (4 * (h + j) < CW) b4[j] = __ldg(b4p + h + j);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                if (4 * (h + j) < CW) {
                  float* vv = v + 4 * (h + j);
                  vv[0] += b4[j].x; vv[1] += b4[j].y; vv[2] += b4[j].z; vv[3] += b4[j].w;
                }
              }
            }
          } else if (bias_vec) {
            const float4* b4p = reinterpret_cast<const float4*>(p.bias + n);
            const int nv = min(CW, p.N - n) >> 2;
#pragma unroll
            for (int j = 0; j < 64; j += 4) {
              if (j < CW && (j >> 2) < nv) {
                const float4 b4 = __ldg(b4p + (j >> 2));
                v[j] += b4.x; v[j + 1] += b4.y; v[j + 2] += b4.z; v[j + 3] += b4.w;
              }
            }
          } else if (has_bias) {
#pragma unroll
            for (int j = 0; j < 64; ++j)
              if (j < CW && n + j < p.N) v[j] += __ldg(p.bias + n + j);
          }
          if (need_aux) {
            if (DB && db_aux) {
              const int b = q & 1;
              mbar_wait(&aux_bar[2 * ew + b], (apar >> b) & 1u);
              apar ^= 1u << b;
            } else {
              mbar_wait(&aux_bar[ew], apar);
              apar ^= 1;
            }
            if (p.epi == JZ_EPI_MUL_F16) {
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                const uint4 w = *reinterpret_cast<const uint4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4));
                const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 gg = unpack_f16(ww[e]);  // gelu' saved by the forward (JZ_EPI_GELU_DG)
                  v[8 * c + 2 * e] *= gg.x;
                  v[8 * c + 2 * e + 1] *= gg.y;
                }
              }
            } else if (p.epi == JZ_EPI_GELU_BWD) {
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                const uint4 w = *reinterpret_cast<const uint4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4));
                const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 g = gelu_grad_pair(ww[e]);  // pre-activation stored by the forward
                  v[8 * c + 2 * e] *= g.x;
                  v[8 * c + 2 * e + 1] *= g.y;
                }
              }
            } else {
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                const float4 w = *reinterpret_cast<const float4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4));
                v[4 * c] += w.x; v[4 * c + 1] += w.y; v[4 * c + 2] += w.z; v[4 * c + 3] += w.w;
              }
            }
            __syncwarp();
          }
          if (f32out) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
              *reinterpret_cast<float4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) =
                  make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
          } else {
            if (p.epi == JZ_EPI_GELU && p.D2 == nullptr) {  // inference: gelu only
#pragma unroll
              for (int j = 0; j < 64; ++j) v[j] = gelu_fast(v[j]);
            } else if (p.epi == JZ_EPI_GELU_DG) {  // gelu' (f16) staged and stored first, gelu into D
#pragma unroll
              for (int c = 0; c < 8; ++c) {
                uint32_t gw[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) gw[e] = gelu_and_grad_pair(v[8 * c + 2 * e], v[8 * c + 2 * e + 1]);
                *reinterpret_cast<uint4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) = make_uint4(gw[0], gw[1], gw[2], gw[3]);
              }
              if (p.store_tma) {
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                  tma_store_2d(&em.d2, stg, n, row0);
                  bulk_commit();
                }
                // pack GELU while the bulk store reads the staging tile
                uint32_t pk[32];
#pragma unroll
                for (int c = 0; c < 32; ++c) pk[c] = pack_bf16(v[2 * c], v[2 * c + 1]);
                if (DB) {
                  stg = stg_w + 4096;  // tile 1: the previous chunk's gelu store has read it
                  if (lane == 0) bulk_wait_read1();
                } else if (lane == 0) {
                  bulk_wait_read0();
                }
                __syncwarp();
#pragma unroll
                for (int c = 0; c < 8; ++c)
                  *reinterpret_cast<uint4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) =
                      make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
                gelu_dg_staged = true;
              } else {
                __syncwarp();
                stg_write_rows(stg, reinterpret_cast<uint8_t*>(p.D2) + ((int64_t)row0 * p.ldd2 + n) * 2,
                               (int64_t)p.ldd2 * 2, rows_ok, cols_bytes, lane);
                __syncwarp();
              }
            } else if (p.epi == JZ_EPI_GELU) {  // pre-activation copy first (D2), then GELU into D
#pragma unroll
              for (int c = 0; c < 8; ++c)
                *reinterpret_cast<uint4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) =
                    make_uint4(pack_bf16(v[8 * c], v[8 * c + 1]), pack_bf16(v[8 * c + 2], v[8 * c + 3]),
                               pack_bf16(v[8 * c + 4], v[8 * c + 5]), pack_bf16(v[8 * c + 6], v[8 * c + 7]));
              if (p.store_tma) {
                fence_proxy_async();
                __syncwarp();
                if (lane == 0 && GDBG != 4) {
                  tma_store_2d(&em.d2, stg, n, row0);
                  bulk_commit();
                }
#pragma unroll
                for (int j = 0; j < 64; ++j) v[j] = gelu_fast(v[j]);  // overlaps the store's smem read
                if (lane == 0) bulk_wait_read0();
              } else {
                __syncwarp();
                stg_write_rows(stg, reinterpret_cast<uint8_t*>(p.D2) + ((int64_t)row0 * p.ldd2 + n) * 2,
                               (int64_t)p.ldd2 * 2, rows_ok, cols_bytes, lane);
#pragma unroll
                for (int j = 0; j < 64; ++j) v[j] = gelu_fast(v[j]);
              }
              __syncwarp();
            }
            if (gelu_dg_staged) {
              // already packed into the staging tile
            } else if (GDBG == 3) {
              uint32_t x = 0;
#pragma unroll
              for (int c = 0; c < 32; ++c) x ^= pack_bf16(v[2 * c], v[2 * c + 1]);
              if (x == 0x12345679u) *reinterpret_cast<uint32_t*>(stg) = x;
            } else if (GDBG != 2) {
#pragma unroll
            for (int c = 0; c < 8; ++c)
              *reinterpret_cast<uint4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) =
                  make_uint4(pack_bf16(v[8 * c], v[8 * c + 1]), pack_bf16(v[8 * c + 2], v[8 * c + 3]),
                             pack_bf16(v[8 * c + 4], v[8 * c + 5]), pack_bf16(v[8 * c + 6], v[8 * c + 7]));
            }
          }
          PH_ADD(2, t_c);
          PH_T(t_d);
          if (p.store_tma) {
            fence_proxy_async();
            __syncwarp();
            if (lane == 0 && GDBG != 1 && GDBG != 3) {
              tma_store_2d(&em.d, stg, n, row0);
              bulk_commit();
            }
          } else {
            __syncwarp();
            if (GDBG != 1 && GDBG != 3)
              stg_write_rows(stg, dbase + (int64_t)row0 * dld + (int64_t)n * esz, dld, rows_ok, cols_bytes, lane);
          }
          if (p.colsum != nullptr && !f32out) {
            // bias gradient of the next layer: column sums of this warp's 32 staged bf16 rows, one
            // fp32 partial row per 32-row block.  Lane reads 16-byte chunk (lane & 7) of rows
            // 4k + (lane >> 3); the four row groups are folded with two shuffles.
            const int cch = lane & 7;
            float cs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const int rr = 4 * k + (lane >> 3);
              if (rr < rows_ok) {
                const uint4 w = *reinterpret_cast<const uint4*>(stg + rr * 128 + ((cch ^ (rr & 7)) << 4));
                const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 f = unpack_bf16(ww[e]);
                  cs[2 * e] += f.x;
                  cs[2 * e + 1] += f.y;
                }
              }
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              cs[e] += __shfl_xor_sync(0xffffffffu, cs[e], 8);
              cs[e] += __shfl_xor_sync(0xffffffffu, cs[e], 16);
            }
            if (rows_ok > 0 && lane < 8 && 8 * cch < p.N - n) {
              float4* dst = reinterpret_cast<float4*>(p.colsum + (int64_t)(row0 >> 5) * p.N + n + 8 * cch);
              dst[0] = make_float4(cs[0], cs[1], cs[2], cs[3]);
              dst[1] = make_float4(cs[4], cs[5], cs[6], cs[7]);
            }
          }
          __syncwarp();
          PH_ADD(3, t_d);
          ++q;
        }
      } else {
        // ---------- direct epilogue (unaligned shapes) ----------
        const int m = row0 + lane;
        float* ws_out = (p.splits > 1) ? ws + (int64_t)split * p.M * p.N : nullptr;
#pragma unroll 1
        for (int c = 0; c < HALF / 32; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tbase + 32 * c, r);
          tmem_ld_wait();
          const int col = chalf * HALF + c * 32;
          const int n = n0 + col;
          if (m < p.M && n < p.N && p.epi != 7) {
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) + (has_bias ? sbias[col + j] : 0.f);
            epilogue_chunk(p, m, n, v, ws_out);
          }
        }
      }
      tc_fence_before();
      if (warp == 2 && lane == 0) GPROF(5);
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR) mbar_arrive_cluster_relaxed(mapa_shared(smem_u32(&tempty_bar[acc]), 0));
        else mbar_arrive_relaxed(&tempty_bar[acc]);
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) bulk_wait0();
  }
  __syncthreads();
  if constexpr (PAIR) cluster_sync_all();  // the peer's MMAs/arrivals target this CTA until here
  if (warp == 2) {
    tc_fence_after();
    if constexpr (PAIR) tmem_dealloc_pair<S::TMEM_COLS>(tmem_base);
    else tmem_dealloc<S::TMEM_COLS>(tmem_base);
  }
}

// Deterministic split-K reduction: fixed summation order over splits.
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int splits, int64_t MN, int N,
                                     float* __restrict__ D, int64_t ldd, const float* bias,
                                     int accumulate) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i < MN; i += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < splits; ++k) s += ws[(int64_t)k * MN + i];
    const int64_t m = i / N;
    const int n = (int)(i - m * N);
    if (bias) s += bias[n];
    float* dst = D + m * ldd + n;
    *dst = accumulate ? (*dst + s) : s;
  }
}

template <int BN, bool A_MN, bool B_MN, bool PAIR, int LNX = 0, bool DB = false>
static int launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const EpiMaps& em, const GemmParams& p,
                       float* ws, cudaStream_t stream) {
  using S = GemmShape<BN, PAIR, LNX, DB>;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(gemm_bf16_kernel<BN, A_MN, B_MN, PAIR, LNX, DB>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM_BYTES);
  });
  JZ_CUDA_TRY(attr_err);
  const int units = LNX ? p.m_tiles : p.m_tiles * p.n_tiles * p.splits;
  if constexpr (PAIR) {
    const int pairs = units < num_sms() / 2 ? units : num_sms() / 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs, 1, 1);
    cfg.blockDim = dim3(gemm_threads<PAIR>(), 1, 1);
    cfg.dynamicSmemBytes = S::SMEM_BYTES;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    JZ_CUDA_TRY(cudaLaunchKernelEx(&cfg, gemm_bf16_kernel<BN, A_MN, B_MN, PAIR, LNX, DB>, ta, tb, em, p, ws));
    count_launch();
  } else {
    const int grid = units < num_sms() ? units : num_sms();
    gemm_bf16_kernel<BN, A_MN, B_MN, PAIR, LNX, DB><<<grid, gemm_threads<PAIR>(), S::SMEM_BYTES, stream>>>(ta, tb, em, p, ws);
    JZ_LAUNCH_CHECK();
  }
  return JZ_OK;
}

template <int BN, bool PAIR = false>
static int dispatch_major(bool a_mn, bool b_mn, const CUtensorMap& ta, const CUtensorMap& tb, const EpiMaps& em,
                          const GemmParams& p, float* ws, cudaStream_t s) {
  if (!a_mn && !b_mn) return launch_gemm<BN, false, false, PAIR>(ta, tb, em, p, ws, s);
  if (!a_mn && b_mn) return launch_gemm<BN, false, true, PAIR>(ta, tb, em, p, ws, s);
  if (a_mn && !b_mn) return launch_gemm<BN, true, false, PAIR>(ta, tb, em, p, ws, s);
  return launch_gemm<BN, true, true, PAIR>(ta, tb, em, p, ws, s);
}

}  // namespace jz

using namespace jz;

// Tuning switches (read once): JZ_GEMM_PAIR=0 disables CTA pairs, JZ_GEMM_STORE=lsu replaces
// the staged epilogue's TMA bulk stores by coalesced st.global.
static bool pair_mode_enabled() {
  static const bool on = [] {
    const char* e = getenv("JZ_GEMM_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool db_enabled() {
  static const bool on = [] {
    const char* e = getenv("JZ_GEMM_DB");
    return !(e && e[0] == '0');
  }();
  return on;
}

static bool store_tma_enabled() {
  static const bool on = [] {
    const char* e = getenv("JZ_GEMM_STORE");
    return !(e && e[0] == 'l');
  }();
  return on;
}

extern "C" int64_t jz_gemm_workspace_bytes(int64_t M, int64_t N, int split_k) {
  return split_k <= 1 ? 0 : (int64_t)split_k * M * N * (int64_t)sizeof(float);
}

static int gemm_impl(const void* A, int64_t lda, int a_kmajor, const void* B, int64_t ldb, int b_kmajor, void* D,
                     int64_t ldd, int64_t M, int64_t N, int64_t K, int epilogue, const float* bias, const void* aux,
                     int64_t ldaux, void* D2, int64_t ldd2, int split_k, void* workspace, float* colsum,
                     jz_stream_t stream_);

extern "C" int jz_gemm_bf16(const void* A, int64_t lda, int a_kmajor, const void* B, int64_t ldb,
                            int b_kmajor, void* D, int64_t ldd, int64_t M, int64_t N, int64_t K,
                            int epilogue, const float* bias, const void* aux, int64_t ldaux,
                            void* D2, int64_t ldd2, int split_k, void* workspace,
                            jz_stream_t stream_) {
  return gemm_impl(A, lda, a_kmajor, B, ldb, b_kmajor, D, ldd, M, N, K, epilogue, bias, aux, ldaux, D2, ldd2,
                   split_k, workspace, nullptr, stream_);
}

extern "C" int64_t jz_gemm_colsum_parts(int64_t M) { return (M + 31) / 32; }

extern "C" int jz_gemm_bf16_colsum(const void* A, int64_t lda, int a_kmajor, const void* B, int64_t ldb,
                                   int b_kmajor, void* D, int64_t ldd, int64_t M, int64_t N, int64_t K,
                                   int epilogue, const float* bias, const void* aux, int64_t ldaux,
                                   void* D2, int64_t ldd2, float* colsum_part, jz_stream_t stream_) {
  JZ_CHECK_ARG(colsum_part != nullptr, "gemm colsum: null partial buffer");
  JZ_CHECK_ARG(epilogue == JZ_EPI_BF16 || epilogue == JZ_EPI_GELU || epilogue == JZ_EPI_GELU_BWD ||
                   epilogue == JZ_EPI_GELU_DG || epilogue == JZ_EPI_MUL_F16,
               "gemm colsum: bf16-output epilogues only (got %d)", epilogue);
  return gemm_impl(A, lda, a_kmajor, B, ldb, b_kmajor, D, ldd, M, N, K, epilogue, bias, aux, ldaux, D2, ldd2,
                   1, nullptr, colsum_part, stream_);
}

static int gemm_impl(const void* A, int64_t lda, int a_kmajor, const void* B, int64_t ldb, int b_kmajor, void* D,
                     int64_t ldd, int64_t M, int64_t N, int64_t K, int epilogue, const float* bias, const void* aux,
                     int64_t ldaux, void* D2, int64_t ldd2, int split_k, void* workspace, float* colsum,
                     jz_stream_t stream_) {
  cudaStream_t stream = reinterpret_cast<cudaStream_t>(stream_);
  JZ_CHECK_ARG(M > 0 && N > 0 && K > 0, "gemm: empty problem M=%lld N=%lld K=%lld", (long long)M,
               (long long)N, (long long)K);
  JZ_CHECK_ARG(M < (1ll << 31) && N < (1ll << 31) && K < (1ll << 31), "gemm: dims exceed int32");
  JZ_CHECK_ARG(lda % 8 == 0 && ldb % 8 == 0, "gemm: lda/ldb must be multiples of 8 (got %lld, %lld)",
               (long long)lda, (long long)ldb);
  JZ_CHECK_ARG(((uintptr_t)A % 16) == 0 && ((uintptr_t)B % 16) == 0, "gemm: A/B must be 16B aligned");
  JZ_CHECK_ARG(epilogue >= JZ_EPI_F32 && epilogue <= JZ_EPI_MUL_F16, "gemm: bad epilogue %d", epilogue);
  JZ_CHECK_ARG(D != nullptr, "gemm: null output");
  if (epilogue == JZ_EPI_GELU_DG) JZ_CHECK_ARG(D2 != nullptr, "gemm: epilogue %d needs D2", epilogue);
  if (epilogue == JZ_EPI_RESID || epilogue == JZ_EPI_GELU_BWD || epilogue == JZ_EPI_MUL_F16)
    JZ_CHECK_ARG(aux != nullptr, "gemm: epilogue %d needs aux", epilogue);
  if (epilogue == JZ_EPI_BF16_F32) JZ_CHECK_ARG(D2 != nullptr, "gemm: epilogue %d needs D2", epilogue);
  if (split_k < 1) split_k = 1;
  if (split_k > 1) {
    JZ_CHECK_ARG(epilogue == JZ_EPI_F32 || epilogue == JZ_EPI_F32_ACC,
                 "gemm: split-K only with fp32 epilogues");
    JZ_CHECK_ARG(workspace != nullptr, "gemm: split-K needs workspace");
  }

  const bool a_mn = !a_kmajor, b_mn = !b_kmajor;
  const int BN = N > 128 ? 256 : (N > 64 ? 128 : 64);
  // CTA pairs for the wide shapes: 256x256 tiles across two SMs (see GemmShape)
  const bool pair = BN == 256 && M > BM && pair_mode_enabled();
  const int TM = pair ? 2 * BM : BM;

  CUtensorMap ta, tb;
  int rc;
  if (!a_mn) rc = make_tmap_2d_bf16(&ta, A, K, M, lda, 64, 128);
  else rc = make_tmap_2d_bf16(&ta, A, M, K, lda, 64, 64);
  if (rc) return rc;
  if (!b_mn) rc = make_tmap_2d_bf16(&tb, B, K, N, ldb, 64, pair ? BN / 2 : BN);
  else rc = make_tmap_2d_bf16(&tb, B, N, K, ldb, 64, 64);
  if (rc) return rc;

  GemmParams p;
  p.M = (int)M; p.N = (int)N; p.K = (int)K;
  p.m_tiles = (int)((M + TM - 1) / TM);
  p.n_tiles = (int)((N + BN - 1) / BN);
  p.kb_total = (int)((K + BK - 1) / BK);
  if (split_k > p.kb_total) split_k = p.kb_total;
  p.kb_per_split = (p.kb_total + split_k - 1) / split_k;
  p.splits = (p.kb_total + p.kb_per_split - 1) / p.kb_per_split;
  p.epi = epilogue;
  p.D = D; p.ldd = ldd;
  p.bias = bias;
  p.aux = aux; p.ldaux = ldaux;
  p.D2 = D2; p.ldd2 = ldd2;
  p.colsum = colsum;

  float* ws = p.splits > 1 ? reinterpret_cast<float*>(workspace) : nullptr;
  // staged TMA epilogue when every global operand of the epilogue is TMA-legal
  EpiMaps em;
  memset(&em, 0, sizeof(em));
  p.tma_epi = 0;
  p.store_tma = 0;
  if (epilogue != 7) {
    const bool f32out = p.splits > 1 || epilogue == JZ_EPI_F32 || epilogue == JZ_EPI_F32_ACC || epilogue == JZ_EPI_RESID;
    const bool bf16out = epilogue == JZ_EPI_BF16 || epilogue == JZ_EPI_GELU || epilogue == JZ_EPI_GELU_BWD ||
                         epilogue == JZ_EPI_GELU_DG || epilogue == JZ_EPI_MUL_F16;
    // 32-column bf16 chunks (BN = 64) do not fill a 128-byte staging row.
    bool ok = (f32out || bf16out) && !(bf16out && BN == 64);
    auto al = [](const void* q) { return ((uintptr_t)q % 16) == 0; };
    if (ok && p.splits > 1) ok = al(ws) && N % 4 == 0;
    else if (ok && f32out) ok = al(D) && ldd % 4 == 0 && N % 4 == 0;
    else if (ok) ok = al(D) && ldd % 8 == 0 && N % 8 == 0;
    if (ok && p.splits == 1 && (epilogue == JZ_EPI_GELU || epilogue == JZ_EPI_GELU_DG) && D2 != nullptr)
      ok = al(D2) && ldd2 % 8 == 0;
    if (ok && p.splits == 1 && epilogue == JZ_EPI_RESID)
      ok = al(aux) && ldaux % 4 == 0 && make_tmap_2d(&em.aux, aux, 4, N, M, ldaux, 32, 32) == JZ_OK;
    if (ok && p.splits == 1 && epilogue == JZ_EPI_F32_ACC)
      ok = make_tmap_2d(&em.aux, D, 4, N, M, ldd, 32, 32) == JZ_OK;
    if (ok && p.splits == 1 && (epilogue == JZ_EPI_GELU_BWD || epilogue == JZ_EPI_MUL_F16))
      ok = al(aux) && ldaux % 8 == 0 && make_tmap_2d(&em.aux, aux, 2, N, M, ldaux, 64, 32) == JZ_OK;
    p.tma_epi = ok ? 1 : 0;
    // TMA bulk stores from the staging tiles (clip at M and N for free); split-K partial slabs
    // use st.global so a partial last tile cannot spill into the next slab
    if (ok && p.splits == 1 && store_tma_enabled()) {
      const bool ok2 = f32out ? make_tmap_2d(&em.d, D, 4, N, M, ldd, 32, 32) == JZ_OK
                              : make_tmap_2d(&em.d, D, 2, N, M, ldd, 64, 32) == JZ_OK;
      const bool ok3 = (epilogue != JZ_EPI_GELU && epilogue != JZ_EPI_GELU_DG) || D2 == nullptr ||
                       make_tmap_2d(&em.d2, D2, 2, N, M, ldd2, 64, 32) == JZ_OK;
      p.store_tma = ok2 && ok3 ? 1 : 0;
    }
  }
  if (colsum != nullptr)
    JZ_CHECK_ARG(p.tma_epi == 1 && (reinterpret_cast<uintptr_t>(colsum) % 16) == 0,
                 "gemm colsum: needs the staged epilogue (N %% 8 == 0, N > 64, aligned output) and a 16-byte aligned buffer");
  // double-buffered epilogue staging for the aux-reading GELU-backward epilogues: the next chunk's
  // aux tile loads while this one computes (MUL_F16 dX at M=148032, N=2048: 334.6 -> 326.7 us; the
  // two-stores-in-flight variant for GELU_DG measured 389.6 -> 393.5 us and is not used)
  const bool db = BN == 256 && pair && p.tma_epi && p.store_tma && p.splits == 1 && N % 256 == 0 && db_enabled() &&
                  (epilogue == JZ_EPI_MUL_F16 || epilogue == JZ_EPI_GELU_BWD);
  if (db && !a_mn && b_mn) rc = launch_gemm<256, false, true, true, 0, true>(ta, tb, em, p, ws, stream);
  else if (db && !a_mn && !b_mn) rc = launch_gemm<256, false, false, true, 0, true>(ta, tb, em, p, ws, stream);
  else if (BN == 256 && pair) rc = dispatch_major<256, true>(a_mn, b_mn, ta, tb, em, p, ws, stream);
  else if (BN == 256) rc = dispatch_major<256>(a_mn, b_mn, ta, tb, em, p, ws, stream);
  else if (BN == 128) rc = dispatch_major<128>(a_mn, b_mn, ta, tb, em, p, ws, stream);
  else rc = dispatch_major<64>(a_mn, b_mn, ta, tb, em, p, ws, stream);
  if (rc) return rc;
  if (p.splits > 1) {
    const int64_t MN = M * N;
    int blocks = (int)((MN + 255) / 256);
    if (blocks > num_sms() * 8) blocks = num_sms() * 8;
    splitk_reduce_kernel<<<blocks, 256, 0, stream>>>(ws, p.splits, MN, (int)N,
                                                     reinterpret_cast<float*>(D), ldd, bias,
                                                     epilogue == JZ_EPI_F32_ACC);
    JZ_LAUNCH_CHECK();
  }
  return JZ_OK;
}

// ---------------------------------------------------------------------------------------------
// LayerNorm-fused GEMMs (N = 512: one CTA pair owns whole rows, see ln_epilogue)
// ---------------------------------------------------------------------------------------------
static int ln_gemm_setup(const void* A, int64_t lda, int a_kmajor, const void* B, int64_t ldb, int b_kmajor,
                         int64_t M, int64_t N, int64_t K, CUtensorMap& ta, CUtensorMap& tb, GemmParams& p) {
  JZ_CHECK_ARG(N == 512, "LN-fused gemm: N must be 512 (got %lld)", (long long)N);
  JZ_CHECK_ARG(M > BM && M < (1ll << 31) && K > 0 && K < (1ll << 31), "LN-fused gemm: M=%lld K=%lld", (long long)M,
               (long long)K);
  JZ_CHECK_ARG(a_kmajor == 1, "LN-fused gemm: A must be K-major (activations)");
  JZ_CHECK_ARG(lda % 8 == 0 && ldb % 8 == 0 && ((uintptr_t)A % 16) == 0 && ((uintptr_t)B % 16) == 0,
               "LN-fused gemm: operand alignment");
  JZ_CHECK_ARG(pair_mode_enabled(), "LN-fused gemm needs CTA pairs (JZ_GEMM_PAIR=0 set)");
  int rc = make_tmap_2d_bf16(&ta, A, K, M, lda, 64, 128);
  if (rc) return rc;
  if (b_kmajor) rc = make_tmap_2d_bf16(&tb, B, K, N, ldb, 64, 128);
  else rc = make_tmap_2d_bf16(&tb, B, N, K, ldb, 64, 64);
  if (rc) return rc;
  memset(&p, 0, sizeof(p));
  p.M = (int)M; p.N = (int)N; p.K = (int)K;
  p.m_tiles = (int)((M + 2 * BM - 1) / (2 * BM));
  p.n_tiles = 2;
  p.kb_total = (int)((K + BK - 1) / BK);
  p.kb_per_split = p.kb_total;
  p.splits = 1;
  return JZ_OK;
}

extern "C" int jz_gemm_bf16_ln_fwd(const void* A, int64_t lda, int a_kmajor, const void* B, int64_t ldb, int b_kmajor,
                                   float* D, int64_t ldd, int64_t M, int64_t N, int64_t K, const float* bias,
                                   const float* resid, int64_t ld_resid, const float* gamma, const float* beta,
                                   float eps, void* xn_bf16, float* mean, float* rstd, int64_t skip_period,
                                   jz_stream_t s) {
  CUtensorMap ta, tb;
  GemmParams p;
  int rc = ln_gemm_setup(A, lda, a_kmajor, B, ldb, b_kmajor, M, N, K, ta, tb, p);
  if (rc) return rc;
  auto a16 = [](const void* q) { return ((uintptr_t)q % 16) == 0; };
  JZ_CHECK_ARG(D && resid && bias && gamma && beta && xn_bf16 && mean && rstd, "LN-fused gemm fwd: null pointer");
  JZ_CHECK_ARG(a16(D) && a16(resid) && a16(bias) && a16(gamma) && a16(beta) && a16(xn_bf16) && ldd % 4 == 0 &&
                   ld_resid % 4 == 0, "LN-fused gemm fwd: 16-byte alignment");
  p.epi = JZ_EPI_RESID;
  p.D = D; p.ldd = ldd;
  p.bias = bias;
  p.aux = resid; p.ldaux = ld_resid;
  p.ln_gamma = gamma; p.ln_beta = beta; p.ln_eps = eps;
  p.ln_out16 = reinterpret_cast<__nv_bfloat16*>(xn_bf16);
  p.ln_mean = mean; p.ln_rstd = rstd;
  p.ln_skip = skip_period;
  EpiMaps em;
  memset(&em, 0, sizeof(em));
  rc = make_tmap_2d(&em.aux, resid, 4, N, M, ld_resid, 32, 32);
  if (!rc) rc = make_tmap_2d(&em.d, D, 4, N, M, ldd, 32, 32);
  if (!rc && skip_period <= 0) rc = make_tmap_2d_sw(&em.d2, xn_bf16, 2, N, M, N, 32, 32, 64);
  if (rc) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
  return b_kmajor ? launch_gemm<256, false, false, true, 1>(ta, tb, em, p, nullptr, st)
                  : launch_gemm<256, false, true, true, 1>(ta, tb, em, p, nullptr, st);
}

extern "C" int64_t jz_gemm_ln_bwd_parts(int64_t M) {
  const int64_t mt = (M + 2 * BM - 1) / (2 * BM);
  const int64_t pairs = mt < num_sms() / 2 ? mt : num_sms() / 2;
  return 2 * pairs * 4;
}

extern "C" int jz_gemm_bf16_ln_bwd(const void* A, int64_t lda, int a_kmajor, const void* B, int64_t ldb, int b_kmajor,
                                   int64_t M, int64_t N, int64_t K, const float* x, const float* mean,
                                   const float* rstd, const float* gamma, float* dres, int accumulate,
                                   void* dres_bf16, float* part, int64_t nparts, float* dgamma, float* dbeta,
                                   float* dbias, jz_stream_t s) {
  CUtensorMap ta, tb;
  GemmParams p;
  int rc = ln_gemm_setup(A, lda, a_kmajor, B, ldb, b_kmajor, M, N, K, ta, tb, p);
  if (rc) return rc;
  auto a16 = [](const void* q) { return ((uintptr_t)q % 16) == 0; };
  JZ_CHECK_ARG(x && mean && rstd && gamma && dres && part, "LN-fused gemm bwd: null pointer");
  JZ_CHECK_ARG(a16(x) && a16(gamma) && a16(dres) && (dres_bf16 == nullptr || a16(dres_bf16)),
               "LN-fused gemm bwd: 16-byte alignment");
  JZ_CHECK_ARG(nparts == jz_gemm_ln_bwd_parts(M), "LN-fused gemm bwd: nparts %lld != %lld", (long long)nparts,
               (long long)jz_gemm_ln_bwd_parts(M));
  p.epi = JZ_EPI_F32;
  p.D = dres; p.ldd = N;
  p.aux = x; p.ldaux = N;
  p.D2 = dres_bf16; p.ldd2 = N;
  p.ln_gamma = gamma; p.ln_mean = const_cast<float*>(mean); p.ln_rstd = const_cast<float*>(rstd);
  p.ln_part = part; p.ln_nparts = nparts;
  p.ln_accumulate = accumulate;
  EpiMaps em;
  memset(&em, 0, sizeof(em));
  rc = make_tmap_2d(&em.aux, x, 4, N, M, N, 32, 32);
  if (!rc) rc = make_tmap_2d(&em.d, dres, 4, N, M, N, 32, 32);
  if (!rc && dres_bf16 != nullptr) rc = make_tmap_2d_sw(&em.d2, dres_bf16, 2, N, M, N, 32, 32, 64);
  if (rc) return rc;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
  rc = b_kmajor ? launch_gemm<256, false, false, true, 2>(ta, tb, em, p, nullptr, st)
                : launch_gemm<256, false, true, true, 2>(ta, tb, em, p, nullptr, st);
  if (rc) return rc;
  return jz_reduce_partials3(part, part + nparts * N, part + 2 * nparts * N, (int)nparts, N, dgamma, dbeta, dbias,
                             0, s);
}

#ifdef JZ_GEMM_PROF
extern "C" int jz_gemm_prof_ph(long long* host) {
  int rc = cudaMemcpyFromSymbol(host, g_gemm_ph, sizeof(long long) * 64 * 4) == cudaSuccess ? 0 : -3;
  static long long zeros[64 * 4];
  cudaMemcpyToSymbol(g_gemm_ph, zeros, sizeof(zeros));
  return rc;
}
extern "C" int jz_gemm_prof_dbg(int v) {
  return cudaMemcpyToSymbol(g_gemm_dbg, &v, sizeof(int)) == cudaSuccess ? 0 : -3;
}
extern "C" int jz_gemm_prof_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_gemm_prof, sizeof(unsigned long long) * 64 * 8) == cudaSuccess ? 0 : -3;
}
#endif
