// K3 backward (v3): spatial attention backward on tcgen05, per (frame, head) unit, S = 256 or 257.
//
// Replaces the backward of multi_head_attention(causal=False) (nn.py:80-110, autodiff through
// st.py:73) for the spatial sub-layer.  Same transposed formulation as v2 (csrc/attn_spatial.cu):
// blocks (key half j, 64-query block c) with S^T = K_j Q_c^T and dP^T = V_j dO_c^T in TMEM,
// P^T written back over S^T (bf16) for dV_j += P^T dO_c, dS^T staged in shared memory for
// dK_j += dS^T Q_c and dQ_t += dS K_j.  What changes (profiles/r02/spatial_bwd_v3.md):
//
//   * Staged input release.  The inputs are four groups: A = {K_0, V_0, token-256 rows},
//     B = {Q_0, dO_0}, C = {Q_1, dO_1}, D = {K_1, V_1}.  Each is released as soon as its last
//     reader is done (A after key half 0, B after block (1, 1), C/D at the unit end), so the next
//     unit's tiles stream in while this unit computes instead of after it.
//   * Token 256 on the tensor core.  Query 256 is a 16-column block (rows 256..271 of Q / dO,
//     only column 0 is read) in each key half: its S^T / dP^T give the query-256 row.  Key 256
//     against every query is an N = 16 MMA of each query tile with rows 256..271 of K / V.  The
//     CUDA cores only form the three row-256 gradients (ds / p weighted row sums, reduced with a
//     shuffle reduce-scatter) instead of 1024 dot products per unit.
//   * A ring of three 64-column S^T / dP^T slots (the dP^T slot is refilled as soon as the P/dS
//     warps have loaded it), which leaves 64 TMEM columns for the key-256 column MMAs.
//   * Epilogues stage each warp's 32 rows in shared memory and TMA-store them.
//
// Warps: 0 TMA, 1 MMA, 2 .. 2+kPds-1 P/dS (kPds/4 per TMEM lane quarter, 64/(kPds/4) query columns
// each), then 4 helper warps (key-256 column, epilogues, row-256 gradients).
#include <mutex>

#include "common.h"
#include "ptx.cuh"

#ifndef JZ_SPATIAL_PDS_WARPS
#define JZ_SPATIAL_PDS_WARPS 16
#endif

namespace jz {
namespace sb {

constexpr int TILE = 16384;                 // 128 rows x 64 bf16, 128B swizzle
constexpr int kPds = JZ_SPATIAL_PDS_WARPS;  // P/dS warps
static_assert(kPds == 8 || kPds == 16, "P/dS warps: 8 or 16");
constexpr int kCg = kPds / 4;   // column groups per TMEM lane quarter
constexpr int QW = 64 / kCg;    // query columns (and row-256 dims) per P/dS warp
constexpr int W_PDS = 2;
constexpr int W_HELP = 2 + kPds;
constexpr int kWarps = 2 + kPds + 4;
constexpr int kThreads = 32 * kWarps;

// shared memory map (bytes from a 1024-aligned base)
constexpr int S_Q = 0;                    // Q tiles: rows 0..127, 128..255
constexpr int S_DO = 2 * TILE;            // dO tiles
constexpr int S_K = 4 * TILE;             // K key halves
constexpr int S_V = 6 * TILE;             // V key halves
constexpr int S_TAIL = 8 * TILE;          // rows 256..271 of Q, dO, K, V (2 KB each)
constexpr int S_DS = S_TAIL + 4 * 2048;   // 4 dS^T slots [128 keys][64 queries]
constexpr int S_STG = S_DS + 4 * TILE;    // epilogue staging, 4 KB per helper warp
constexpr int S_END = S_STG + 4 * 4096;   // 221184
constexpr int T_Q = 0, T_DO = 1, T_K = 2, T_V = 3;  // tail row order (S_TAIL + 2048 * T_x)

// per-unit vector block (spatial_uvb_rows_kernel, layout sp::U_* in attn_spatial.cu)
constexpr int U_LSE2 = 0, U_DV = 260, U_PC = 520, U_DC = 521;
constexpr int kUvbHead = 524;    // floats loaded per unit
constexpr int kUvbStride = 780;  // floats per unit in the workspace

// TMEM columns
// S^T ring of three 64-column slots (block g uses slot g % 3), one dP^T slot; the gradient MMAs of
// block g are issued two blocks later, so S^T / dP^T of the next block are computed ahead of them
constexpr uint32_t C_RB = 64;  // dP^T slot
constexpr uint32_t C_DV = 256, C_DK = 320, C_DQ = 384;
JZ_DEV uint32_t sslot(uint32_t g) {
  const uint32_t m = g % 3;
  return m == 0 ? 0u : (m == 1 ? 128u : 192u);
}

struct Small {
  uint64_t full_a, full_b, full_c, full_d, free_a, free_b, free_cd;
  uint64_t sdp_full[2], dp_free[2], pds_full[3];
  uint64_t dkdv_full, dkdv_free, dq_full[2], dq_free[2], ds_free[2];
  uint64_t uvb_free[2], vec_ready, prow_full[2];
  uint32_t tmem_base;
  alignas(16) float uvb[2][kUvbHead];
  alignas(16) __nv_bfloat16 vec[4][64];  // row 0 of the tail tiles: q256, do256, k256, v256
  float p_row[256], ds_row[256];         // query 256 against every key (key-half epilogues)
  float part_dq[4][64];                  // dQ_256 partial sums per lane quarter
  float part_ct[4][128];                 // dK_256 | dV_256 partial sums per lane quarter
};
constexpr int SMEM = S_END + (int)sizeof(Small) + 1024;
static_assert(SMEM <= 232448, "spatial bwd v3 smem budget");

JZ_DEV void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

JZ_DEV float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

JZ_DEV uint32_t sw128(uint32_t r, uint32_t c) { return r * 128 + ((c ^ (r & 7)) << 4); }

#ifdef JZ_SPATIAL_BWD_PROF
// per-unit timeline of CTA 0 (clock64 marks), read back with jz_attn_bwd3_prof_read
__device__ unsigned long long g_tl[16][128];
__device__ unsigned long long g_tw[4][10][2][32];  // units 0..3: per-block, per-warp (loaded, done)
#define TW(x, k)                                                                                      \
  do {                                                                                                 \
    if (blockIdx.x == 0 && i < 4 && (threadIdx.x & 31) == 0) g_tw[i][x][k][threadIdx.x >> 5] = clock64(); \
  } while (0)
#define TL(slot)                                                             \
  do {                                                                       \
    if (blockIdx.x == 0 && i < 16 && (threadIdx.x & 31) == 0) g_tl[i][slot] = clock64(); \
  } while (0)
#else
#define TL(slot) do { } while (0)
#define TW(x, k) do { } while (0)
#endif

#ifdef JZ_SPATIAL_BWD_DEBUG
// bounded wait: report the stuck barrier (tag = source line) and trap
JZ_DEV void wait_dbg(uint64_t* bar, uint32_t parity, int tag) {
  const uint32_t addr = smem_u32(bar);
  for (long long n = 0;; ++n) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok) : "r"(addr), "r"(parity) : "memory");
    if (ok) return;
    if (n == 4000000 && blockIdx.x == 0 && (threadIdx.x & 31) == 0) {
      printf("spatial bwd3 stuck: block %d warp %d line %d parity %u\n", blockIdx.x, threadIdx.x / 32, tag, parity);
    }
    if (n == 40000000) asm volatile("trap;");
  }
}
#define MBAR_WAIT(bar, par) wait_dbg(bar, par, __LINE__)
#else
#define MBAR_WAIT(bar, par) mbar_wait(bar, par)
#endif

// Sum of v[0..N) over the 32 lanes of a warp, scattered: recursive halving with xor masks
// 16, 8, ... leaves each lane one element; for N = 32 lane l holds element l, for N = 16 lanes
// 2e and 2e+1 both hold element e.
template <int N>
JZ_DEV float warp_reduce_scatter(float (&v)[N], int lane) {
  static_assert(N == 16 || N == 32, "reduce-scatter width");
#pragma unroll
  for (int n = N, s = 16; n > 1; n >>= 1, s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int e = 0; e < n / 2; ++e) {
      const float send = up ? v[e] : v[e + n / 2];
      const float keep = up ? v[e + n / 2] : v[e];
      v[e] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  if (N == 16) v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  return v[0];
}

// the P/dS column loads / P^T stores of one warp (QW columns)
JZ_DEV void ld_cols(uint32_t taddr, uint32_t (&r)[32]) { tmem_ld_32x32b_x32(taddr, r); }
JZ_DEV void ld_cols(uint32_t taddr, uint32_t (&r)[16]) { tmem_ld_32x32b_x16(taddr, r); }
JZ_DEV void st_cols(uint32_t taddr, const uint32_t (&r)[16]) { tmem_st_32x32b_x16(taddr, r); }
JZ_DEV void st_cols(uint32_t taddr, const uint32_t (&r)[8]) { tmem_st_32x32b_x8(taddr, r); }

// Block order of a unit: key half 0 then 1; in each half the query-256 block (c = 4) first when
// S = 257, then the four 64-query blocks.
JZ_DEV void blk(int x, bool tail, int& j, int& c) {
  if (tail) {
    j = x >= 5;
    const int y = x - 5 * j;
    c = y == 0 ? 4 : y - 1;
  } else {
    j = x >> 2;
    c = x & 3;
  }
}

}  // namespace sb

using namespace sb;

__global__ void __launch_bounds__(sb::kThreads, 1)
    spatial_bwd3_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                        const __grid_constant__ CUtensorMap tm_qkv16, const __grid_constant__ CUtensorMap tm_do16,
                        const __grid_constant__ CUtensorMap tm_dq, const float* __restrict__ uvb,
                        __nv_bfloat16* __restrict__ dqkv, float* __restrict__ colsum, int frames, int S, int H) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  Small& sm = *reinterpret_cast<Small*>(smem + S_END);
  const int D = H * 64;
  const int warp = __shfl_sync(0xffffffffu, (int)warp_id(), 0), lane = lane_id();  // warp-uniform
  const int units = frames * H;
  const bool tail = S > 256;
  const int NB = tail ? 10 : 8;
  const float scale = 0.125f;
  const float c2 = 0.125f * 1.4426950408889634f;
  const int64_t ld3 = 3 * (int64_t)D;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_dq);
    if (tail) {
      tma_prefetch_desc(&tm_qkv16);
      tma_prefetch_desc(&tm_do16);
    }
  }
  if (warp == 1 && lane == 0) {
    mbar_init(&sm.full_a, 1); mbar_init(&sm.full_b, 1); mbar_init(&sm.full_c, 1); mbar_init(&sm.full_d, 1);
    mbar_init(&sm.free_a, 1 + 4); mbar_init(&sm.free_b, 1 + 4); mbar_init(&sm.free_cd, 1 + 4);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.sdp_full[b], 1);
      mbar_init(&sm.dp_free[b], kPds);
      mbar_init(&sm.dq_full[b], 1);
      mbar_init(&sm.dq_free[b], 4);
      mbar_init(&sm.ds_free[b], 1);
      mbar_init(&sm.uvb_free[b], 1);
    }
    mbar_init(&sm.dkdv_full, 1); mbar_init(&sm.dkdv_free, 4);
    for (int b = 0; b < 3; ++b) mbar_init(&sm.pds_full[b], kPds);
    mbar_init(&sm.vec_ready, 1);
    mbar_init(&sm.prow_full[0], 4); mbar_init(&sm.prow_full[1], 4);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem_base);
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, sm.tmem_base, 0);

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      int i = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
        const int f = u / H, h = u % H;
        const int row0 = f * S;
        if (i > 0) MBAR_WAIT(&sm.free_a, (i - 1) & 1);
        TL(0);
        if (i > 1) MBAR_WAIT(&sm.uvb_free[i & 1], ((i - 2) >> 1) & 1);
        mbar_arrive_expect_tx(&sm.full_a, 2 * TILE + (tail ? 4 * 2048 : 0) + kUvbHead * 4);
        bulk_load(sm.uvb[i & 1], uvb + (int64_t)u * kUvbStride, kUvbHead * 4, &sm.full_a);
        tma_load_2d(smem + S_K, &tm_qkv, &sm.full_a, D + h * 64, row0);
        tma_load_2d(smem + S_V, &tm_qkv, &sm.full_a, 2 * D + h * 64, row0);
        if (tail) {
          tma_load_2d(smem + S_TAIL + T_Q * 2048, &tm_qkv16, &sm.full_a, h * 64, row0 + 256);
          tma_load_2d(smem + S_TAIL + T_DO * 2048, &tm_do16, &sm.full_a, h * 64, row0 + 256);
          tma_load_2d(smem + S_TAIL + T_K * 2048, &tm_qkv16, &sm.full_a, D + h * 64, row0 + 256);
          tma_load_2d(smem + S_TAIL + T_V * 2048, &tm_qkv16, &sm.full_a, 2 * D + h * 64, row0 + 256);
        }
        // the rest of this unit's tiles are loaded once the previous unit releases them (late in that
        // unit): pull them into L2 now so those loads are L2 hits
        tma_prefetch_2d(&tm_qkv, h * 64, row0);
        tma_prefetch_2d(&tm_do, h * 64, row0);
        tma_prefetch_2d(&tm_qkv, h * 64, row0 + 128);
        tma_prefetch_2d(&tm_do, h * 64, row0 + 128);
        tma_prefetch_2d(&tm_qkv, D + h * 64, row0 + 128);
        tma_prefetch_2d(&tm_qkv, 2 * D + h * 64, row0 + 128);
        if (i > 0) MBAR_WAIT(&sm.free_b, (i - 1) & 1);
        TL(1);
        mbar_arrive_expect_tx(&sm.full_b, 2 * TILE);
        tma_load_2d(smem + S_Q, &tm_qkv, &sm.full_b, h * 64, row0);
        tma_load_2d(smem + S_DO, &tm_do, &sm.full_b, h * 64, row0);
        if (i > 0) MBAR_WAIT(&sm.free_cd, (i - 1) & 1);
        TL(2);
        mbar_arrive_expect_tx(&sm.full_c, 2 * TILE);
        tma_load_2d(smem + S_Q + TILE, &tm_qkv, &sm.full_c, h * 64, row0 + 128);
        tma_load_2d(smem + S_DO + TILE, &tm_do, &sm.full_c, h * 64, row0 + 128);
        mbar_arrive_expect_tx(&sm.full_d, 2 * TILE);
        tma_load_2d(smem + S_K + TILE, &tm_qkv, &sm.full_d, D + h * 64, row0 + 128);
        tma_load_2d(smem + S_V + TILE, &tm_qkv, &sm.full_d, 2 * D + h * 64, row0 + 128);
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer (whole warp, warp-uniform operands, one elected lane issues) ------------------------------
    constexpr uint32_t id_s = idesc_bf16_f32(128, 64, false, false);    // K_j Q_c^T, V_j dO_c^T
    constexpr uint32_t id_s16 = idesc_bf16_f32(128, 16, false, false);  // 16-row token-256 blocks
    constexpr uint32_t id_kv = idesc_bf16_f32(128, 64, false, true);    // P^T dO_c, dS^T Q_c
    constexpr uint32_t id_q = idesc_bf16_f32(128, 64, true, true);      // dS K_j
    const uint32_t dhi = (uint32_t)(sdesc_sw128(0, 0, 1024) >> 32);
    auto dsc = [dhi](uint32_t addr4, uint32_t off, uint32_t lbo) -> uint64_t {
      return ((uint64_t)dhi << 32) | (addr4 + (off >> 4) + ((lbo >> 4) << 16));
    };
    const uint32_t aq = smem_u32(smem + S_Q) >> 4, ado = smem_u32(smem + S_DO) >> 4, ak = smem_u32(smem + S_K) >> 4,
                   av = smem_u32(smem + S_V) >> 4, ads = smem_u32(smem + S_DS) >> 4,
                   at = smem_u32(smem + S_TAIL) >> 4;
    auto grad = [&](int i, int x) {
      int j, c;
      blk(x, tail, j, c);
      const uint32_t g = (uint32_t)(NB * i + x);
      MBAR_WAIT(&sm.pds_full[g % 3], (g / 3) & 1);
      tc_fence_after();
      TL(23 + x);
      if (c == 4) return;  // query-256 block: its row sums are CUDA-core work
      if (c == 0 && 2 * i + j > 0) {
        MBAR_WAIT(&sm.dkdv_free, (2 * i + j - 1) & 1);
        tc_fence_after();
      }
      if (j == 0 && (c & 1) && i > 0) {
        MBAR_WAIT(&sm.dq_free[c >> 1], (i - 1) & 1);
        tc_fence_after();
      }
      const uint32_t qoff = (c >> 1) * TILE + (c & 1) * 8192;  // rows 64c.. of Q / dO
      const uint32_t pcol = tmem + sslot(g);
      // P^T / dS^T of queries 16 ks .. 16 ks + 15: column group ks (QW = 16), packed bf16 pairs
      static_assert(QW == 16, "batched gradient MMAs assume 16 query columns per P/dS warp");
      umma4x2_bf16_ts_w(tmem + C_DV, pcol, dsc(ado, qoff, 8192), tmem + C_DK, pcol + QW / 2, dsc(aq, qoff, 8192), 16,
                        2048 >> 4, id_kv, c > 0);
      if (c & 1) {
        const int t = c >> 1;
        umma4_bf16_ss_w(tmem + C_DQ + 64 * t, dsc(ads, 2 * t * TILE, TILE), dsc(ak, j * TILE, 8192), 2048 >> 4,
                        2048 >> 4, id_q, j > 0);
        umma4_bf16_ss_w(tmem + C_DQ + 64 * t, dsc(ads, 2 * t * TILE + 4 * 2048, TILE),
                        dsc(ak, j * TILE + 4 * 2048, 8192), 2048 >> 4, 2048 >> 4, id_q, 1);
        umma_commit_w(&sm.ds_free[t]);
      }
      if (c == 3) umma_commit_w(&sm.dkdv_full);
      if (j == 0 && c == 3) umma_commit_w(&sm.free_a);
      if (j == 1 && c == 1) {
        umma_commit_w(&sm.free_b);
        umma_commit_w(&sm.dq_full[0]);
      }
      if (j == 1 && c == 3) {
        umma_commit_w(&sm.free_cd);
        umma_commit_w(&sm.dq_full[1]);
      }
    };
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      MBAR_WAIT(&sm.full_a, i & 1);
      MBAR_WAIT(&sm.full_b, i & 1);
      tc_fence_after();
      bool wc = false, wd = false;
      for (int x = 0; x < NB; ++x) {
        int j, c;
        blk(x, tail, j, c);
        const uint32_t g = (uint32_t)(NB * i + x), b = g & 1;
        if (!wc && (j == 1 || c == 2 || c == 3)) {
          MBAR_WAIT(&sm.full_c, i & 1);
          wc = true;
          tc_fence_after();
        }
        if (!wd && j == 1) {
          MBAR_WAIT(&sm.full_d, i & 1);
          wd = true;
          tc_fence_after();
        }
        const uint32_t dS = tmem + sslot(g), dP = tmem + C_RB;
        TL(3 + x);
        // S^T: the slot's previous P^T (block g - 3) was read by grad(g - 3), issued earlier by this
        // warp (in-order pipe)
        if (c == 4)
          umma4_bf16_ss_w(dS, dsc(ak, j * TILE, 16), dsc(at, T_Q * 2048, 16), 2, 2, id_s16, 0);
        else
          umma4_bf16_ss_w(dS, dsc(ak, j * TILE, 16), dsc(aq, (c >> 1) * TILE + (c & 1) * 8192, 16), 2, 2, id_s, 0);
        if (g > 0) {  // dP^T slot: the P/dS warps have loaded block g - 1
          MBAR_WAIT(&sm.dp_free[(g - 1) & 1], ((g - 1) >> 1) & 1);
          tc_fence_after();
        }
        TL(13 + x);
        if (c == 4)
          umma4_bf16_ss_w(dP, dsc(av, j * TILE, 16), dsc(at, T_DO * 2048, 16), 2, 2, id_s16, 0);
        else
          umma4_bf16_ss_w(dP, dsc(av, j * TILE, 16), dsc(ado, (c >> 1) * TILE + (c & 1) * 8192, 16), 2, 2, id_s, 0);
        umma_commit_w(&sm.sdp_full[b]);
        if (x >= 2) grad(i, x - 2);  // two blocks behind: S^T / dP^T of block x run ahead of them
      }
      // unit end: the last two blocks' gradients (their commits release the next unit's inputs)
      grad(i, NB - 2);
      grad(i, NB - 1);
    }
  } else if (warp < W_HELP) {
    // ------------------------------ P / dS warps ------------------------------
    const int quarter = warp & 3;
    const int cg = (warp - W_PDS) >> 2;  // column group within the quarter
    const int r = quarter * 32 + lane;   // key row within the key half (TMEM lane)
    const uint32_t lbase = tmem + ((quarter * 32) << 16);
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const float* uv = sm.uvb[i & 1];
      for (int x = 0; x < NB; ++x) {
        int j, c;
        blk(x, tail, j, c);
        const uint32_t g = (uint32_t)(NB * i + x), b = g & 1;
        const uint32_t tS = lbase + sslot(g), tP = lbase + C_RB;
        if (c < 4 && (c & 1) == 0 && 2 * i + j > 0) MBAR_WAIT(&sm.ds_free[c >> 1], (2 * i + j - 1) & 1);
        MBAR_WAIT(&sm.sdp_full[b], (g >> 1) & 1);
        tc_fence_after();
        if (warp == W_PDS) TL(33 + x);
        if (c == 4) {
          // query 256 against this key half: column 0 of the 16-column block
          const float s = __uint_as_float(tmem_ld_32x32b_x1(tS));
          const float dp = __uint_as_float(tmem_ld_32x32b_x1(tP));
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.dp_free[b]);
          const float p = ex2(s * c2 - uv[U_LSE2 + 256]);
          const float ds = p * (dp - uv[U_DV + 256]);
          if (cg == 0) {
            sm.p_row[128 * j + r] = p;
            sm.ds_row[128 * j + r] = ds;
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.prow_full[j]);  // one phase per unit and key half
          }
          // (the dQ_256 row, sum_k dS[256, k] K_k, is formed by the helper warps from ds_row)
          __syncwarp();
          if (warp == W_PDS) TL(43 + x);
          if (lane == 0) mbar_arrive(&sm.pds_full[g % 3]);
          continue;
        }
        uint32_t vs[QW], vd[QW];
        ld_cols(tS + QW * cg, vs);
        ld_cols(tP + QW * cg, vd);
        tmem_ld_wait();
        if (warp == W_PDS) TL(64 + x);
        TW(x, 0);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.dp_free[b]);
        const int q0 = 64 * c + QW * cg;
        const float* lse2 = uv + U_LSE2 + q0;
        const float* Dv = uv + U_DV + q0;
        uint32_t pp[QW / 2], pd[QW / 2];
#pragma unroll
        for (int e = 0; e < QW; e += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(lse2 + e);
          const float4 d4 = *reinterpret_cast<const float4*>(Dv + e);
          const float p0 = ex2(__uint_as_float(vs[e]) * c2 - l4.x);
          const float p1 = ex2(__uint_as_float(vs[e + 1]) * c2 - l4.y);
          const float p2 = ex2(__uint_as_float(vs[e + 2]) * c2 - l4.z);
          const float p3 = ex2(__uint_as_float(vs[e + 3]) * c2 - l4.w);
          pp[e / 2] = pack_bf16(p0, p1);
          pp[e / 2 + 1] = pack_bf16(p2, p3);
          pd[e / 2] = pack_bf16(p0 * (__uint_as_float(vd[e]) - d4.x), p1 * (__uint_as_float(vd[e + 1]) - d4.y));
          pd[e / 2 + 1] = pack_bf16(p2 * (__uint_as_float(vd[e + 2]) - d4.z), p3 * (__uint_as_float(vd[e + 3]) - d4.w));
        }
        // P^T (bf16 pairs) over the first half of this warp's own S^T columns; dS^T into smem slot c
        if (warp == W_PDS) TL(74 + x);
        st_cols(tS + QW * cg, pp);
        st_cols(tS + QW * cg + QW / 2, pd);  // dS^T for the dK MMA (A from TMEM); dQ reads the smem copy
        uint8_t* slot = smem + S_DS + c * TILE;
#pragma unroll
        for (int k = 0; k < QW / 8; ++k)
          *reinterpret_cast<uint4*>(slot + sw128(r, (QW / 8) * cg + k)) =
              make_uint4(pd[4 * k], pd[4 * k + 1], pd[4 * k + 2], pd[4 * k + 3]);
        tmem_st_wait();
        if (warp == W_PDS) TL(84 + x);
        fence_proxy_async();
        if (warp == W_PDS) TL(94 + x);
        tc_fence_before();
        __syncwarp();
        if (warp == W_PDS) TL(43 + x);
        TW(x, 1);
        if (lane == 0) mbar_arrive(&sm.pds_full[g % 3]);
      }
    }
  } else {
    // ------------------------------ helper warps ------------------------------
    const int quarter = warp & 3;
    const int hw = warp - W_HELP;
    const int ht = threadIdx.x - 32 * W_HELP;  // 0..127
    const int r = quarter * 32 + lane;         // TMEM lane
    const uint32_t lbase = tmem + ((quarter * 32) << 16);
    uint8_t* stg = smem + S_STG + hw * 4096;
    // TMEM row block (64 fp32 columns) -> sc * (acc + coef * vec) -> bf16 -> this warp's staging
    // rows (128B swizzle) -> TMA store; plus the column sums of the 32 rows (QKV bias gradient)
    // zero_sum: the columns sum to exactly 0 over the frame (dK: every dS row sums to 0), so the
    // partial row is written as 0 without reading the tile back
    auto epi = [&](uint32_t col, float coef, const __nv_bfloat16* vec, float sc, int gcol, int64_t grow, float* part,
                   bool zero_sum = false) {
      if (lane == 0) bulk_wait_read0();
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t vv[16];
        tmem_ld_32x32b_x16(lbase + col + 16 * q, vv);
        tmem_ld_wait();
        const uint4 v0 = *reinterpret_cast<const uint4*>(vec + 16 * q);
        const uint4 v1 = *reinterpret_cast<const uint4*>(vec + 16 * q + 8);
        const uint32_t vw[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
        uint32_t w[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float2 vf = unpack_bf16(vw[e]);
          w[e] = pack_bf16(sc * (__uint_as_float(vv[2 * e]) + coef * vf.x),
                           sc * (__uint_as_float(vv[2 * e + 1]) + coef * vf.y));
        }
        *reinterpret_cast<uint4*>(stg + sw128(lane, 2 * q)) = make_uint4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<uint4*>(stg + sw128(lane, 2 * q + 1)) = make_uint4(w[4], w[5], w[6], w[7]);
      }
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store_2d(&tm_dq, stg, gcol, (int)grow);
        bulk_commit();
      }
      if (part != nullptr && zero_sum) {
        if (lane < 8) {
          float4* dst = reinterpret_cast<float4*>(part + gcol + 8 * lane);
          dst[0] = make_float4(0.f, 0.f, 0.f, 0.f);
          dst[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      } else if (part != nullptr) {
        const int cch = lane & 7;
        float cs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int rr = 4 * k + (lane >> 3);
          const uint4 w = *reinterpret_cast<const uint4*>(stg + sw128(rr, cch));
          const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 fv = unpack_bf16(ww[e]);
            cs[2 * e] += fv.x;
            cs[2 * e + 1] += fv.y;
          }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          cs[e] += __shfl_xor_sync(0xffffffffu, cs[e], 8);
          cs[e] += __shfl_xor_sync(0xffffffffu, cs[e], 16);
        }
        if (lane < 8) {
          float4* dst = reinterpret_cast<float4*>(part + gcol + 8 * cch);
          dst[0] = make_float4(cs[0], cs[1], cs[2], cs[3]);
          dst[1] = make_float4(cs[4], cs[5], cs[6], cs[7]);
        }
      }
    };
    if (!tail && ht < 32) *reinterpret_cast<uint4*>(&sm.vec[ht >> 3][8 * (ht & 7)]) = make_uint4(0u, 0u, 0u, 0u);
    named_bar(2, 128);
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const int f = u / H, h = u % H;
      const int64_t row0 = (int64_t)f * S;
      const float* uv = sm.uvb[i & 1];
      // colsum partial rows: [frame][9][3D], row block = 4 * (row tile) + lane quarter, block 8 = token 256
      float* part0 = colsum ? colsum + ((int64_t)f * 9 + quarter) * ld3 : nullptr;
      float* part1 = colsum ? colsum + ((int64_t)f * 9 + 4 + quarter) * ld3 : nullptr;
      MBAR_WAIT(&sm.full_a, i & 1);
      float dsc0 = 0.f, dsc1 = 0.f;
      if (hw == 0) TL(53);
      if (tail) {
        if (hw == 0) {  // keep the token-256 rows: the tail tiles are released before the epilogues
          const int k = lane >> 3, ch = lane & 7;
          *reinterpret_cast<uint4*>(&sm.vec[k][8 * ch]) =
              *reinterpret_cast<const uint4*>(smem + S_TAIL + k * 2048 + 16 * ch);
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.vec_ready);
        }
        MBAR_WAIT(&sm.vec_ready, i & 1);
        // key 256 against the queries of both tiles (this thread: queries r and 128 + r): s = q . k256,
        // dp = dO . v256 from the staged Q / dO rows (these tiles are read below anyway)
        MBAR_WAIT(&sm.full_b, i & 1);
        MBAR_WAIT(&sm.full_c, i & 1);
        float s0 = 0.f, d0 = 0.f, s1 = 0.f, d1 = 0.f;
#pragma unroll 2
        for (int cc = 0; cc < 8; ++cc) {
          const uint4 kw = *reinterpret_cast<const uint4*>(&sm.vec[T_K][8 * cc]);
          const uint4 vw = *reinterpret_cast<const uint4*>(&sm.vec[T_V][8 * cc]);
          const uint4 q0 = *reinterpret_cast<const uint4*>(smem + S_Q + sw128(r, cc));
          const uint4 q1 = *reinterpret_cast<const uint4*>(smem + S_Q + TILE + sw128(r, cc));
          const uint4 g0 = *reinterpret_cast<const uint4*>(smem + S_DO + sw128(r, cc));
          const uint4 g1 = *reinterpret_cast<const uint4*>(smem + S_DO + TILE + sw128(r, cc));
          const uint32_t ka[4] = {kw.x, kw.y, kw.z, kw.w}, va[4] = {vw.x, vw.y, vw.z, vw.w};
          const uint32_t qa[4] = {q0.x, q0.y, q0.z, q0.w}, qb[4] = {q1.x, q1.y, q1.z, q1.w};
          const uint32_t ga[4] = {g0.x, g0.y, g0.z, g0.w}, gb[4] = {g1.x, g1.y, g1.z, g1.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 kf = unpack_bf16(ka[e]), vf = unpack_bf16(va[e]);
            const float2 x0 = unpack_bf16(qa[e]), x1 = unpack_bf16(qb[e]);
            const float2 y0 = unpack_bf16(ga[e]), y1 = unpack_bf16(gb[e]);
            s0 += x0.x * kf.x + x0.y * kf.y;
            s1 += x1.x * kf.x + x1.y * kf.y;
            d0 += y0.x * vf.x + y0.y * vf.y;
            d1 += y1.x * vf.x + y1.y * vf.y;
          }
        }
        const float p0 = ex2(s0 * c2 - uv[U_LSE2 + r]);
        const float p1 = ex2(s1 * c2 - uv[U_LSE2 + 128 + r]);
        dsc0 = p0 * (d0 - uv[U_DV + r]);
        dsc1 = p1 * (d1 - uv[U_DV + 128 + r]);
        // dK_256 += sum_q dS[q, 256] Q_q, dV_256 += sum_q P[q, 256] dO_q over this warp's 64 queries
#pragma unroll 1
        for (int pass = 0; pass < 4; ++pass) {
          const int half = pass & 1;
          const uint8_t* base = smem + (pass < 2 ? S_Q : S_DO);
          const float w0 = pass < 2 ? dsc0 : p0, w1 = pass < 2 ? dsc1 : p1;
          float v[32];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint4 a0 = *reinterpret_cast<const uint4*>(base + sw128(r, 4 * half + k));
            const uint4 a1 = *reinterpret_cast<const uint4*>(base + TILE + sw128(r, 4 * half + k));
            const uint32_t x0[4] = {a0.x, a0.y, a0.z, a0.w}, x1[4] = {a1.x, a1.y, a1.z, a1.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f0 = unpack_bf16(x0[e]), f1 = unpack_bf16(x1[e]);
              v[8 * k + 2 * e] = w0 * f0.x + w1 * f1.x;
              v[8 * k + 2 * e + 1] = w0 * f0.y + w1 * f1.y;
            }
          }
          const float a = warp_reduce_scatter<32>(v, lane);
          sm.part_ct[quarter][(pass >> 1) * 64 + 32 * half + lane] = a;
        }
      }
      if (tail) {
        // dQ_256 partials: sum_k dS[256, k] K_k over keys 64 hw .. 64 hw + 63 (lane: dims 2 lane,
        // 2 lane + 1), once the P/dS warps have written both key halves' ds_row; K is still staged
        MBAR_WAIT(&sm.prow_full[0], i & 1);
        MBAR_WAIT(&sm.prow_full[1], i & 1);
        const uint8_t* kt = smem + S_K + (hw >> 1) * TILE;
        const float* dsr = sm.ds_row + 64 * hw;
        float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll 8
        for (int kk = 0; kk < 64; kk += 2) {
          const int k = 64 * (hw & 1) + kk;
          const float2 ka = unpack_bf16(*reinterpret_cast<const uint32_t*>(kt + sw128(k, lane >> 2) + 4 * (lane & 3)));
          const float2 kb = unpack_bf16(*reinterpret_cast<const uint32_t*>(kt + sw128(k + 1, lane >> 2) + 4 * (lane & 3)));
          const float2 d = *reinterpret_cast<const float2*>(dsr + kk);
          a0 = fmaf(d.x, ka.x, a0);
          a1 = fmaf(d.x, ka.y, a1);
          b0 = fmaf(d.y, kb.x, b0);
          b1 = fmaf(d.y, kb.y, b1);
        }
        *reinterpret_cast<float2*>(&sm.part_dq[hw][2 * lane]) = make_float2(a0 + b0, a1 + b1);
      }
      __syncwarp();
      if (lane == 0) {  // done with the tail rows (A), Q_0 / dO_0 (B), Q_1 / dO_1 (C), K_1 (D)
        mbar_arrive(&sm.free_a);
        mbar_arrive(&sm.free_b);
        mbar_arrive(&sm.free_cd);
      }
      if (hw == 0) TL(54);
      const __nv_bfloat16* q256 = sm.vec[T_Q];  // zeros when S = 256 (the coefficients are 0 then too)
      const __nv_bfloat16* do256 = sm.vec[T_DO];
      const __nv_bfloat16* k256 = sm.vec[T_K];
      const int64_t rw = row0 + quarter * 32;
      // ---- dV_0 / dK_0 ----
      MBAR_WAIT(&sm.dkdv_full, (2 * i) & 1);
      if (tail) MBAR_WAIT(&sm.prow_full[0], i & 1);
      tc_fence_after();
      if (hw == 0) TL(55);
      epi(C_DV, tail ? sm.p_row[r] : 0.f, do256, 1.f, 2 * D + h * 64, rw, part0);
      epi(C_DK, tail ? sm.ds_row[r] : 0.f, q256, scale, D + h * 64, rw, part0, true);
      if (hw == 0) TL(56);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.dkdv_free);
      // ---- dQ_0 ----
      MBAR_WAIT(&sm.dq_full[0], i & 1);
      tc_fence_after();
      if (hw == 0) TL(57);
      epi(C_DQ, dsc0, k256, scale, h * 64, rw, part0);
      if (hw == 0) TL(58);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.dq_free[0]);
      // ---- dV_1 / dK_1 ----
      MBAR_WAIT(&sm.dkdv_full, (2 * i + 1) & 1);
      if (tail) MBAR_WAIT(&sm.prow_full[1], i & 1);
      tc_fence_after();
      if (hw == 0) TL(59);
      epi(C_DV, tail ? sm.p_row[128 + r] : 0.f, do256, 1.f, 2 * D + h * 64, rw + 128, part1);
      epi(C_DK, tail ? sm.ds_row[128 + r] : 0.f, q256, scale, D + h * 64, rw + 128, part1, true);
      if (hw == 0) TL(60);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.dkdv_free);
      // ---- dQ_1 ----
      MBAR_WAIT(&sm.dq_full[1], i & 1);
      tc_fence_after();
      if (hw == 0) TL(61);
      epi(C_DQ + 64, dsc1, k256, scale, h * 64, rw + 128, part1);
      if (hw == 0) TL(62);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.dq_free[1]);
      // ---- token 256: dQ_256, dK_256, dV_256 ----
      named_bar(2, 128);
      if (ht < 64) {
        const int d = ht;
        float* pr = colsum ? colsum + ((int64_t)f * 9 + 8) * ld3 + h * 64 + d : nullptr;
        if (tail) {
          // dQ_256 = scale (sum_k dS[256, k] K_k + dS[256, 256] k256)
          float aq = (sm.part_dq[0][d] + sm.part_dq[1][d]) + (sm.part_dq[2][d] + sm.part_dq[3][d]);
          aq = scale * (aq + uv[U_DC] * __bfloat162float(sm.vec[T_K][d]));
          const __nv_bfloat16 bq = __float2bfloat16_rn(aq);
          dqkv[(row0 + 256) * ld3 + h * 64 + d] = bq;
          if (pr) pr[0] = __bfloat162float(bq);
          float sk = uv[U_DC] * __bfloat162float(sm.vec[T_Q][d]);
          float sv = uv[U_PC] * __bfloat162float(sm.vec[T_DO][d]);
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) {
            sk += sm.part_ct[qq][d];
            sv += sm.part_ct[qq][64 + d];
          }
          const __nv_bfloat16 bk = __float2bfloat16_rn(scale * sk), bv = __float2bfloat16_rn(sv);
          dqkv[(row0 + 256) * ld3 + D + h * 64 + d] = bk;
          dqkv[(row0 + 256) * ld3 + 2 * D + h * 64 + d] = bv;
          if (pr) {
            pr[D] = 0.f;  // the k-bias gradient is exactly 0 (see epi's zero_sum)
            pr[2 * D] = __bfloat162float(bv);
          }
        } else if (pr) {  // S = 256: no token 256, its partial row is zero
          pr[0] = 0.f;
          pr[D] = 0.f;
          pr[2 * D] = 0.f;
        }
      }
      named_bar(2, 128);
      if (ht == 0) mbar_arrive(&sm.uvb_free[i & 1]);
      if (hw == 0) TL(63);
    }
    if (lane == 0) bulk_wait0();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int spatial_bwd3_launch(const void* qkv, const void* dout, const float* uvb, int64_t frames, int S, int H, void* dqkv,
                        float* colsum_part, cudaStream_t st) {
  const int D = H * 64;
  CUtensorMap tq, td, tq16, td16, tdq;
  int rc = make_tmap_2d_bf16(&tq, qkv, 3 * D, frames * S, 3 * D, 64, 128);
  if (!rc) rc = make_tmap_2d_bf16(&td, dout, D, frames * S, D, 64, 128);
  if (!rc) rc = make_tmap_2d_bf16(&tq16, qkv, 3 * D, frames * S, 3 * D, 64, 16);
  if (!rc) rc = make_tmap_2d_bf16(&td16, dout, D, frames * S, D, 64, 16);
  if (!rc) rc = make_tmap_2d_bf16(&tdq, dqkv, 3 * D, frames * S, 3 * D, 64, 32);
  if (rc) return rc;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(spatial_bwd3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sb::SMEM);
  });
  JZ_CUDA_TRY(attr_err);
  const int64_t units = frames * H;
  const int grid = (int)(units < num_sms() ? units : num_sms());
  spatial_bwd3_kernel<<<grid, sb::kThreads, sb::SMEM, st>>>(tq, td, tq16, td16, tdq, uvb,
                                                             reinterpret_cast<__nv_bfloat16*>(dqkv), colsum_part,
                                                             (int)frames, S, H);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

}  // namespace jz

#ifdef JZ_SPATIAL_BWD_PROF
extern "C" int jz_attn_bwd3_tw_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, jz::g_tw, sizeof(unsigned long long) * 4 * 10 * 2 * 32) == cudaSuccess ? 0 : -3;
}
extern "C" int jz_attn_bwd3_prof_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, jz::g_tl, sizeof(unsigned long long) * 16 * 128) == cudaSuccess ? 0 : -3;
}
#endif
