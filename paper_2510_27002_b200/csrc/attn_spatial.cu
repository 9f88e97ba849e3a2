// K3: spatial (intra-frame) attention on tcgen05 tensor cores, forward and backward.
//
// Replaces the spatial sub-layer's attention of st_block (st.py:73) =
// multi_head_attention(causal=False) (nn.py:80-110) with lead dims (B, T).
// One work unit = (frame, head): S = 256 (+1) tokens, hd = 64.
//
// S = 257 does not tile (256 patch tokens + the prepended action token,
// dynamics.py:118): tokens 0..255 run on the tensor cores as two 128-row query
// tiles against one 256-key tile; the 257th key's score is formed on CUDA cores
// and its value row rides on the PV MMA as a 17th K-step, and the 257th query row
// is computed by four "tail" warps on CUDA cores — exactly, no padding waste
// (SURVEY §7.4.1).
//
// qkv bf16 [M, 3D] (row = frame*S + s), out bf16 [M, D], lse f32 [frame][H][S].
#include <mutex>

#include "common.h"
#include "ptx.cuh"

namespace jz {

namespace sp {

constexpr int kFwdTailWarps = 4;  // query row 256 (S = 257) on CUDA cores
constexpr int kFwdTailThreads = 32 * kFwdTailWarps;
constexpr int W_TAIL = 18;  // w0 TMA, w1 MMA, w2-9 tile 0, w10-17 tile 1 (two warps per TMEM lane quarter), w18.. tail
constexpr int W_STORE = W_TAIL + kFwdTailWarps;  // the O / residual TMA store warp
constexpr int kFwdThreads = 32 * (W_STORE + 1);
constexpr int TILE = 16384;    // 128 rows x 128 B
// forward smem map (bytes, from a 1024-aligned base)
constexpr int F_Q = 0;                  // 2 tiles (query tiles 0 / 1)
constexpr int F_K = F_Q + 2 * TILE;     // 2 slots x 2 tiles (256 keys), slot = unit parity
constexpr int F_V = F_K + 4 * TILE;     // 2 slots x 2 tiles (256 values), slot = unit parity
constexpr int F_ST = F_V + 4 * TILE;    // O staging + residual staging, shared by the two query tiles
                                        // (their epilogues alternate with the exponential passes)
constexpr int F_VX = F_ST + 2 * TILE;   // 2 slots: value rows 256..271 for the PV MMA's 17th K-step, row 0 =
                                        // v_256 (TMA, with V), rows 1..15 stay zero
constexpr int F_ONES = F_VX + 2 * 2048;  // 16 rows x 128 B of bf16 1.0: the row-sum columns of the PV MMA
constexpr int F_END = F_ONES + 2048;     // 202752
constexpr int kFwdSmall = 8192;
constexpr int F_SMEM = F_END + kFwdSmall + 1024;

struct FwdSmallSmem {
  uint64_t q_full[2], q_free[2], k_full[2], k_free[2], v_full[2], v_free[2];
  uint64_t stg_full;     // a tile's O / residual rows are staged (one phase per tile epilogue)
  uint64_t stg_free;     // the staging tiles' previous TMA store has read them (one phase per tile epilogue)
  uint64_t s_full[2], p_full[2], o_full[2], tmem_free[2];
  uint64_t exp_turn[2];  // the two softmax warpgroups take turns on the exponentials
  uint32_t tmem_base;
  alignas(128) uint8_t krow[2][128];  // key 256 of the unit (TMA, arrives with K), slot = unit parity
  float tail_s[260];
  float tail_red[2 * kFwdTailWarps];
  float2 xch[2][2][128];  // [tile][column half][row]: half-row max and key-256 partial dot
};
static_assert(sizeof(FwdSmallSmem) <= kFwdSmall, "forward small smem budget");

#ifdef JZ_SPATIAL_FWD_PROF
// per-unit timeline of CTA 0 (clock64 marks), read back with jz_attn_fwd_prof_read
__device__ unsigned long long g_ftl[16][64];
#define FTL(slot)                                                                      \
  do {                                                                                 \
    if (blockIdx.x == 0 && i < 16 && (threadIdx.x & 31) == 0) g_ftl[i][slot] = clock64(); \
  } while (0)
#else
#define FTL(slot) do { } while (0)
#endif

JZ_DEV void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

JZ_DEV float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

JZ_DEV float fmax3(float a, float b, float c) {
  float y;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(y) : "f"(a), "f"(b), "f"(c));
  return y;
}

// byte offset of (row r, 16-byte chunk c in 0..7) inside a 128B-swizzled 128-row tile
JZ_DEV uint32_t sw128(uint32_t r, uint32_t c) { return r * 128 + ((c ^ (r & 7)) << 4); }

// dot product of a 64-wide bf16 row held as 8 16-byte chunks (row r of a swizzled tile) with an
// unswizzled 64-wide bf16 row; four partial sums
JZ_DEV float dot64_tile_row(const uint8_t* tile, uint32_t r, const uint8_t* row) {
  float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint4 w = *reinterpret_cast<const uint4*>(tile + sw128(r, c));
    const uint4 kw = *reinterpret_cast<const uint4*>(row + (c << 4));
    const uint32_t qa[4] = {w.x, w.y, w.z, w.w}, ka[4] = {kw.x, kw.y, kw.z, kw.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 x = unpack_bf16(qa[e]), y = unpack_bf16(ka[e]);
      a[e] = fmaf(x.x, y.x, a[e]);
      a[e] = fmaf(x.y, y.y, a[e]);
    }
  }
  return (a[0] + a[1]) + (a[2] + a[3]);
}

}  // namespace sp

using namespace sp;

// One CTA per SM walks (frame, head) units. Query tile t (rows 128t..128t+127) belongs to 8 softmax
// warps (two per TMEM lane quarter, one per 128-key half); S_t = Q_t K^T (128 x 256 fp32) sits in
// TMEM columns 256t..256t+255. P is written back as bf16 pairs (keys 0..127 at columns 0..63,
// keys 128..255 at 192..255, key 256 at 144) and O_t = P_t [V | 1] accumulates 64 dims + 16
// row-sum columns at 64..143. The two tiles take turns on the exponentials (exp_turn), so one
// tile's max pass, PV wait and epilogue overlap the other's MUFU-bound exponential pass. K and V
// are double-buffered by unit parity; a store warp issues the O / residual TMA stores.
// S = 257: the half-1 warps form the key-256 scores, the tail warps query row 256.
__global__ void __launch_bounds__(kFwdThreads, 1)
    spatial_fwd_kernel(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm_row,
                       const __grid_constant__ CUtensorMap tm_o, const __grid_constant__ CUtensorMap tm_olo,
                       const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ out,
                       __nv_bfloat16* __restrict__ out_lo, float* __restrict__ lse, int frames, int S, int H) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  FwdSmallSmem& sm = *reinterpret_cast<FwdSmallSmem*>(smem + F_END);
  const int D = H * 64;
  const int warp = __shfl_sync(0xffffffffu, (int)warp_id(), 0), lane = lane_id();  // warp-uniform
  const int units = frames * H;
  const bool has_tail = S > 256;
  const float c2 = 0.125f * 1.4426950408889634f;  // scale * log2(e)
  const int ntail = has_tail ? kFwdTailThreads : 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm);
    tma_prefetch_desc(&tm_row);
    tma_prefetch_desc(&tm_o);
    if (out_lo) tma_prefetch_desc(&tm_olo);
  }
  if (warp == 1 && lane == 0) {
    for (int t = 0; t < 2; ++t) {
      mbar_init(&sm.q_full[t], 1);
      mbar_init(&sm.q_free[t], 1 + (has_tail ? 256 : 0));  // S_t MMA commit (+ tile t's warps: key-256 column)
      mbar_init(&sm.k_full[t], 1);
      mbar_init(&sm.k_free[t], 1 + ntail + (has_tail ? 512 : 0));  // S_1 MMA commit + tail warps (+ softmax: key row 256)
      mbar_init(&sm.s_full[t], 1);
      mbar_init(&sm.p_full[t], 256);
      mbar_init(&sm.o_full[t], 1);
      mbar_init(&sm.tmem_free[t], 256);
      mbar_init(&sm.exp_turn[t], 8);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.v_full[b], 1);
      mbar_init(&sm.v_free[b], 1 + ntail);  // PV_1 MMA commit + tail warps
    }
    mbar_init(&sm.stg_full, 8);  // lane 0 of the tile's 8 warps
    mbar_init(&sm.stg_free, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem_base);
  for (int e = threadIdx.x; e < 2048 / 16; e += blockDim.x) {
    *reinterpret_cast<uint4*>(smem + F_ONES + 16 * e) = make_uint4(0x3f803f80u, 0x3f803f80u, 0x3f803f80u, 0x3f803f80u);
    *reinterpret_cast<uint4*>(smem + F_VX + 16 * e) = make_uint4(0u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(smem + F_VX + 2048 + 16 * e) = make_uint4(0u, 0u, 0u, 0u);
  }
  fence_proxy_async();  // generic writes of the ones tile before the tensor core reads it
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
        const int ks = i & 1;
        // in order of release: Q_0 (after S_0 of the previous unit), K slot (two units back), Q_1, V
        mbar_wait(&sm.q_free[0], (i & 1) ^ 1);
        FTL(30);
        mbar_arrive_expect_tx(&sm.q_full[0], TILE);
        tma_load_2d(smem + F_Q, &tm, &sm.q_full[0], h * 64, row0);
        mbar_wait(&sm.k_free[ks], ((i >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.k_full[ks], 2 * TILE + (has_tail ? 128 : 0));
        if (has_tail) tma_load_2d(sm.krow[ks], &tm_row, &sm.k_full[ks], D + h * 64, row0 + 256);
        tma_load_2d(smem + F_K + ks * 2 * TILE, &tm, &sm.k_full[ks], D + h * 64, row0);
        tma_load_2d(smem + F_K + ks * 2 * TILE + TILE, &tm, &sm.k_full[ks], D + h * 64, row0 + 128);
        mbar_wait(&sm.q_free[1], (i & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.q_full[1], TILE);
        tma_load_2d(smem + F_Q + TILE, &tm, &sm.q_full[1], h * 64, row0 + 128);
        mbar_wait(&sm.v_free[ks], ((i >> 1) & 1) ^ 1);
        FTL(31);
        mbar_arrive_expect_tx(&sm.v_full[ks], 2 * TILE + (has_tail ? 128 : 0));
        if (has_tail) tma_load_2d(smem + F_VX + ks * 2048, &tm_row, &sm.v_full[ks], 2 * D + h * 64, row0 + 256);
        tma_load_2d(smem + F_V + ks * 2 * TILE, &tm, &sm.v_full[ks], 2 * D + h * 64, row0);
        tma_load_2d(smem + F_V + ks * 2 * TILE + TILE, &tm, &sm.v_full[ks], 2 * D + h * 64, row0 + 128);
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer (whole warp, uniform operands) ------------------------------
    // Issue order follows the steady-state event order: S_0(i), PV_1(i-1), S_1(i), PV_0(i).
    constexpr uint32_t idesc_s = idesc_bf16_f32(128, 256, false, false);
    // PV with N = 80: dims 0..63 from V, dims 64..79 from the all-ones tile (every one of those
    // output columns is the row sum of the bf16 P the MMA multiplies)
    constexpr uint32_t idesc_o = idesc_bf16_f32(128, 80, false, true);
    const uint32_t dhi = (uint32_t)(sdesc_sw128(0, 0, 1024) >> 32);
    auto dsc = [dhi](uint32_t addr4, uint32_t off, uint32_t lbo) -> uint64_t {
      return ((uint64_t)dhi << 32) | (addr4 + (off >> 4) + ((lbo >> 4) << 16));
    };
    const uint32_t q4 = smem_u32(smem + F_Q) >> 4, k4 = smem_u32(smem + F_K) >> 4, v4 = smem_u32(smem + F_V) >> 4;

    auto issue_s = [&](int i, int t) {
      const int ks = i & 1;
      mbar_wait(&sm.q_full[t], i & 1);
      mbar_wait(&sm.tmem_free[t], (i & 1) ^ 1);
      tc_fence_after();
      FTL(1 + t);
      umma4_bf16_ss_w(tmem + 256 * t, dsc(q4, t * TILE, 16), dsc(k4, ks * 2 * TILE, 16), 2, 2, idesc_s, 0);
      umma_commit_w(&sm.s_full[t]);
      umma_commit_w(&sm.q_free[t]);
    };
    auto issue_pv = [&](int i, int t) {
      const int vs = i & 1;  // V slot
      mbar_wait(&sm.p_full[t], i & 1);
      tc_fence_after();
      FTL(4 + t);
      // O_t (cols 256t + 64 .. 143: 64 dims + 16 row-sum columns) = P_t V. P from TMEM as bf16 pairs:
      // keys 0..127 at columns 0..63, keys 128..255 at 192..255, key 256 at 144 (17th K-step).
      // The second 64-dim atom of B sits LBO bytes after the step's V rows: LBO points every step at
      // the ones tile (the step adds 2048 B to the address and removes it from LBO).
      const uint64_t bstep = (uint64_t)((int64_t)(2048 >> 4) - ((int64_t)(2048 >> 4) << 16));
#pragma unroll
      for (int g = 0; g < 4; ++g)
        umma4_bf16_ts_w(tmem + 256 * t + 64, tmem + 256 * t + (g < 2 ? 32 * g : 192 + 32 * (g - 2)),
                        dsc(v4, vs * 2 * TILE + g * 4 * 2048, F_ONES - F_V - vs * 2 * TILE - g * 4 * 2048), 8, bstep,
                        idesc_o, g > 0);
      if (has_tail)
        umma_bf16_ts_w(tmem + 256 * t + 64, tmem + 256 * t + 144,
                       dsc(v4, F_VX - F_V + vs * 2048, F_ONES - F_VX - vs * 2048), idesc_o, 1);
      umma_commit_w(&sm.o_full[t]);
    };
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      mbar_wait(&sm.k_full[i & 1], (i >> 1) & 1);
      FTL(0);
      issue_s(i, 0);
      if (i > 0) {
        issue_pv(i - 1, 1);
        umma_commit_w(&sm.v_free[(i - 1) & 1]);
      }
      issue_s(i, 1);
      umma_commit_w(&sm.k_free[i & 1]);
      mbar_wait(&sm.v_full[i & 1], (i >> 1) & 1);
      FTL(3);
      issue_pv(i, 0);
    }
    if (i > 0) {
      issue_pv(i - 1, 1);
      umma_commit_w(&sm.v_free[(i - 1) & 1]);
    }
  } else if (warp < W_TAIL) {
    // ------------------------------ softmax / epilogue warps ------------------------------
    // tile t = 8 warps: two per TMEM lane quarter, column half hc (keys 128 hc .. 128 hc + 127)
    const int sw = warp - 2;
    const int t = sw >> 3, hc = (sw >> 2) & 1, quarter = warp & 3;
    const int r = quarter * 32 + lane;             // query row within the tile
    const uint32_t lrow = tmem + ((quarter * 32) << 16) + 256 * t;
    const uint32_t scol = lrow + 128 * hc;         // this warp's S columns
    uint8_t* o16 = smem + F_ST;                    // [128 rows][64 bf16], 128B swizzle
    uint8_t* olo = o16 + TILE;                     // [128 rows][64 bf16] residual
    const int bar_pair = 4 + 4 * t + quarter;      // named barrier of the two warps of a lane quarter
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const uint32_t par = i & 1;
      const int f = u / H, h = u % H;
      // S = 257: q_r . k_256 on CUDA cores while S_t is computed, by the half-1 warp of the row (the
      // half-0 warp takes it through the exchange below). Splitting the dot product between the
      // two warps was measured to give wrong key-256 scores for some rows on a first launch.
      // Both warps wait for the tiles before arriving on their release barriers: an arrival for
      // unit i + 2 must not land in the K slot's phase of unit i (the tail warps may still be
      // reading that slot), and waiting for k_full of this unit guarantees that phase completed.
      float dpart = 0.f;
      if (has_tail) {
        mbar_wait(&sm.k_full[i & 1], (i >> 1) & 1);
        mbar_wait(&sm.q_full[t], par);
        if (hc == 1) dpart = dot64_tile_row(smem + F_Q + t * TILE, r, sm.krow[i & 1]);
        mbar_arrive(&sm.q_free[t]);      // done with the Q tile
        mbar_arrive(&sm.k_free[i & 1]);  // and with key row 256
      }
      if (quarter == 2 && hc == 0) FTL(8 + t);
      mbar_wait(&sm.s_full[t], par);
      if (quarter == 2 && hc == 0) FTL(10 + t);
      tc_fence_after();
      // max over this warp's 128 columns (64 per TMEM wait, three-input max), then the row's
      float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t v[64];
        tmem_ld_32x32b_x64_wait(scol + 64 * c, v);
#pragma unroll
        for (int j = 0; j < 64; j += 8) {
          m4[0] = fmax3(m4[0], __uint_as_float(v[j]), __uint_as_float(v[j + 1]));
          m4[1] = fmax3(m4[1], __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
          m4[2] = fmax3(m4[2], __uint_as_float(v[j + 4]), __uint_as_float(v[j + 5]));
          m4[3] = fmax3(m4[3], __uint_as_float(v[j + 6]), __uint_as_float(v[j + 7]));
        }
      }
      const float mh = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
      sm.xch[t][hc][r] = make_float2(mh, dpart);
      named_bar(bar_pair, 64);
      const float2 other = sm.xch[t][hc ^ 1][r];
      const float s_last = has_tail ? (hc ? dpart : other.y) : -INFINITY;
      const float mx = fmax3(mh, other.x, s_last);

      const float mb = mx * c2;
      if (quarter == 2 && hc == 0) FTL(14 + t);
      // take the turn on the exponentials: tile 1 after tile 0 of the same unit, tile 0 after
      // tile 1 of the previous unit
      if (t == 1) mbar_wait(&sm.exp_turn[0], par);
      else if (i > 0) mbar_wait(&sm.exp_turn[1], par ^ 1);
      if (quarter == 2 && hc == 0) FTL(12 + t);
      // exponentials, 32 keys per TMEM wait. P of keys 128 hc + 32 j .. + 31 goes to columns
      // 16 j .. (half 0) / 192 + 16 j .. (half 1, walked from its last 32 keys down) as bf16 pairs:
      // every column is read before this warp overwrites it.
      {
        // the next 32 columns load while these are exponentiated
        uint32_t va[32], vb[32];
        tmem_ld_32x32b_x32(scol + 32 * (hc ? 3 : 0), va);
#pragma unroll
        for (int jj = 0; jj < 4; jj += 2) {
          const int j0 = hc ? 3 - jj : jj, j1 = hc ? 2 - jj : jj + 1;
          uint32_t pk[16];
          tmem_ld_wait();
          tmem_ld_32x32b_x32(scol + 32 * j1, vb);
#pragma unroll
          for (int e = 0; e < 32; e += 2)
            pk[e / 2] = pack_bf16(ex2(fmaf(__uint_as_float(va[e]), c2, -mb)), ex2(fmaf(__uint_as_float(va[e + 1]), c2, -mb)));
          tmem_st_32x32b_x16(lrow + (hc ? 192 : 0) + 16 * j0, pk);
          tmem_ld_wait();
          if (jj + 2 < 4) tmem_ld_32x32b_x32(scol + 32 * (hc ? 1 - jj : jj + 2), va);
#pragma unroll
          for (int e = 0; e < 32; e += 2)
            pk[e / 2] = pack_bf16(ex2(fmaf(__uint_as_float(vb[e]), c2, -mb)), ex2(fmaf(__uint_as_float(vb[e + 1]), c2, -mb)));
          tmem_st_32x32b_x16(lrow + (hc ? 192 : 0) + 16 * j1, pk);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.exp_turn[t]);
      if (has_tail && hc == 1) {  // key 256: (p_256, 0) and zeros over the 17th K-step's columns 144..151
        const uint32_t px[8] = {pack_bf16(ex2(s_last * c2 - mb), 0.f), 0u, 0u, 0u, 0u, 0u, 0u, 0u};
        tmem_st_32x32b_x8(lrow + 144, px);
      }
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&sm.p_full[t]);
      if (quarter == 2 && hc == 0) FTL(16 + t);
      // O epilogue: dims 32 hc .. 32 hc + 31 of O (bf16) and, for the backward's Delta, its rounding
      // residual O - bf16(O) (bf16: O to ~16 bits), staged and TMA-stored per tile
      mbar_wait(&sm.o_full[t], par);
      if (quarter == 2 && hc == 0) FTL(18 + t);
      tc_fence_after();
      float sum;
      {
        uint32_t v[32];
        tmem_ld_32x32b_x32(lrow + 64 + 32 * hc, v);
        const uint32_t srow = tmem_ld_32x32b_x1(lrow + 128);  // sum of the bf16 P row (MMA, fp32)
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive_relaxed(&sm.tmem_free[t]);  // only TMEM reads precede (tcgen05.wait::ld done)
        sum = __uint_as_float(srow);
        const float inv = 1.0f / sum;
        if (quarter == 2 && hc == 0) FTL(22 + t);
        // the other tile's (or the previous unit's) store has read the staging tiles
        const int e = 2 * i + t;  // this CTA's tile epilogues alternate: e = 0, 1, 2, ...
        if (e > 0) mbar_wait(&sm.stg_free, (e - 1) & 1);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] = __uint_as_float(v[8 * q + e]) * inv;
          uint32_t hi[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) hi[e] = pack_bf16(o[2 * e], o[2 * e + 1]);
          *reinterpret_cast<uint4*>(o16 + sw128(r, 4 * hc + q)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
          if (out_lo) {
            uint32_t lo[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 hf = unpack_bf16(hi[e]);
              lo[e] = pack_bf16(o[2 * e] - hf.x, o[2 * e + 1] - hf.y);
            }
            *reinterpret_cast<uint4*>(olo + sw128(r, 4 * hc + q)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
          }
        }
      }
      if (quarter == 2 && hc == 0) FTL(24 + t);
      fence_proxy_async();  // generic staging writes before the store warp's bulk copy reads them
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.stg_full);
      if (quarter == 2 && hc == 0) FTL(26 + t);
      if (hc == 0) lse[((int64_t)f * H + h) * S + 128 * t + r] = mx * 0.125f + logf(sum);
      if (quarter == 2 && hc == 0) FTL(20 + t);
    }
  } else if (warp < W_STORE && has_tail) {
    // ------------------------------ tail warps (S = 257) ------------------------------
    // query row 256 against every key on CUDA cores (the key-256 column is formed by the softmax
    // warps, key 256's value row rides on the PV MMA)
    const int tid = threadIdx.x - 32 * W_TAIL;  // 0 .. kFwdTailThreads - 1
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const int ks = i & 1;
      const int f = u / H, h = u % H;
      const int64_t row0 = (int64_t)f * S;
      const __nv_bfloat16* q = qkv + (row0 + 256) * 3 * D + h * 64;
      uint4 qw[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) qw[c] = reinterpret_cast<const uint4*>(q)[c];
      const uint32_t qpair = *reinterpret_cast<const uint32_t*>(q + 2 * lane);  // dims 2 lane, 2 lane + 1
      if (tid == 0) FTL(40);
      mbar_wait(&sm.k_full[ks], (i >> 1) & 1);
      if (tid == 0) FTL(41);
      // scores against keys tid and 128 + tid (four partial sums each), key 256 by warp 10
      const uint8_t* kt = smem + F_K + ks * 2 * TILE;
      float a0[4] = {0.f, 0.f, 0.f, 0.f}, a1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 w0 = *reinterpret_cast<const uint4*>(kt + sw128(tid, c));
        const uint4 w1 = *reinterpret_cast<const uint4*>(kt + TILE + sw128(tid, c));
        const uint32_t qa[4] = {qw[c].x, qw[c].y, qw[c].z, qw[c].w};
        const uint32_t k0[4] = {w0.x, w0.y, w0.z, w0.w}, k1[4] = {w1.x, w1.y, w1.z, w1.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 x = unpack_bf16(qa[e]), y0 = unpack_bf16(k0[e]), y1 = unpack_bf16(k1[e]);
          a0[e] = fmaf(x.y, y0.y, fmaf(x.x, y0.x, a0[e]));
          a1[e] = fmaf(x.y, y1.y, fmaf(x.x, y1.x, a1[e]));
        }
      }
      const float s0 = (a0[0] + a0[1]) + (a0[2] + a0[3]);
      const float s1 = (a1[0] + a1[1]) + (a1[2] + a1[3]);
      float s256 = -INFINITY;
      if (warp == W_TAIL) {
        const float2 x = unpack_bf16(qpair), y = unpack_bf16(*reinterpret_cast<const uint32_t*>(sm.krow[ks] + 4 * lane));
        s256 = warp_sum(fmaf(x.y, y.y, x.x * y.x));
      }
      mbar_arrive(&sm.k_free[ks]);
      float mx = warp_max(fmax3(s0, s1, s256));
      if (lane == 0) sm.tail_red[warp - W_TAIL] = mx;
      named_bar(3, kFwdTailThreads);
      mx = fmaxf(fmaxf(sm.tail_red[0], sm.tail_red[1]), fmaxf(sm.tail_red[2], sm.tail_red[3]));
      const float mb = mx * c2;
      const float p0 = ex2(s0 * c2 - mb), p1 = ex2(s1 * c2 - mb);
      sm.tail_s[tid] = p0;
      sm.tail_s[128 + tid] = p1;
      float sum = p0 + p1;
      if (tid == 0) {
        const float p256 = ex2(s256 * c2 - mb);
        sm.tail_s[256] = p256;
        sum += p256;
      }
      sum = warp_sum(sum);
      if (lane == 0) sm.tail_red[kFwdTailWarps + warp - W_TAIL] = sum;
      named_bar(3, kFwdTailThreads);
      sum = (sm.tail_red[kFwdTailWarps] + sm.tail_red[kFwdTailWarps + 1]) +
            (sm.tail_red[kFwdTailWarps + 2] + sm.tail_red[kFwdTailWarps + 3]);
      // o[d] for d = 2 lane, 2 lane + 1; keys split into kFwdTailWarps parts by warp; even / odd keys
      // accumulate separately
      constexpr int KP = 256 / kFwdTailWarps;
      const int dpair = lane, part = tid >> 5;
      float oa0 = 0.f, oa1 = 0.f, ob0 = 0.f, ob1 = 0.f;
      if (tid == 0) FTL(44);
      mbar_wait(&sm.v_full[ks], (i >> 1) & 1);
      if (tid == 0) FTL(45);
      const uint32_t chunk = dpair >> 2, within = (dpair & 3) * 4;
      const uint8_t* vt = smem + F_V + ks * 2 * TILE + (part >> 1) * TILE;  // a part's 64 keys lie in one tile
#pragma unroll 8
      for (int k = (part * KP) & 127; k < ((part * KP) & 127) + KP; k += 2) {
        const float2 va = unpack_bf16(*reinterpret_cast<const uint32_t*>(vt + sw128(k, chunk) + within));
        const float2 vb = unpack_bf16(*reinterpret_cast<const uint32_t*>(vt + sw128(k + 1, chunk) + within));
        const float2 pp = *reinterpret_cast<const float2*>(sm.tail_s + (part >> 1) * 128 + k);
        oa0 = fmaf(pp.x, va.x, oa0);
        oa1 = fmaf(pp.x, va.y, oa1);
        ob0 = fmaf(pp.y, vb.x, ob0);
        ob1 = fmaf(pp.y, vb.y, ob1);
      }
      float o0 = oa0 + ob0, o1 = oa1 + ob1;
      if (part == kFwdTailWarps - 1) {  // value row 256 (row 0 of the PV MMA's 17th K-step tile)
        const float2 vl = unpack_bf16(*reinterpret_cast<const uint32_t*>(smem + F_VX + ks * 2048 + 4 * dpair));
        const float p256 = sm.tail_s[256];
        o0 = fmaf(p256, vl.x, o0);
        o1 = fmaf(p256, vl.y, o1);
      }
      mbar_arrive(&sm.v_free[ks]);
      if (tid == 0) FTL(46);
      named_bar(3, kFwdTailThreads);  // every part is done reading the probabilities in tail_s
      if (part > 0) {                 // partial outputs of parts 1.. into tail_s
        sm.tail_s[(part - 1) * 64 + 2 * dpair] = o0;
        sm.tail_s[(part - 1) * 64 + 2 * dpair + 1] = o1;
      }
      named_bar(3, kFwdTailThreads);
      if (part == 0) {
#pragma unroll
        for (int w = 0; w < kFwdTailWarps - 1; ++w) {
          o0 += sm.tail_s[w * 64 + 2 * dpair];
          o1 += sm.tail_s[w * 64 + 2 * dpair + 1];
        }
        o0 /= sum;
        o1 /= sum;
        *reinterpret_cast<uint32_t*>(out + (row0 + 256) * D + h * 64 + 2 * dpair) = pack_bf16(o0, o1);
        if (out_lo) {
          const float2 hi = unpack_bf16(pack_bf16(o0, o1));
          *reinterpret_cast<uint32_t*>(out_lo + (row0 + 256) * D + h * 64 + 2 * dpair) = pack_bf16(o0 - hi.x, o1 - hi.y);
        }
        if (tid == 0) lse[((int64_t)f * H + h) * S + 256] = mx * 0.125f + logf(sum);
      }
      named_bar(3, kFwdTailThreads);
    }
  } else if (warp == W_STORE && lane == 0) {
    // ------------------------------ store warp ------------------------------
    // the tile epilogues alternate (stg_free): store tile 0 then tile 1 of every unit, and release
    // the staging once the bulk copies have read it, so no softmax warp waits on a store
    int e = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int f = u / H, h = u % H;
      for (int t = 0; t < 2; ++t, ++e) {
        mbar_wait(&sm.stg_full, e & 1);
        const int row = f * S + 128 * t;
        tma_store_2d(&tm_o, smem + F_ST, h * 64, row);
        if (out_lo) tma_store_2d(&tm_olo, smem + F_ST + TILE, h * 64, row);
        bulk_commit();
        bulk_wait_read0();
        mbar_arrive(&sm.stg_free);
      }
    }
    bulk_wait0();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace jz

using namespace jz;

extern "C" int jz_attn_spatial_fwd(const void* qkv, int64_t frames, int S, int H, int head_dim, void* out,
                                   void* out_lo, float* lse, jz_stream_t s) {
  JZ_CHECK_ARG(head_dim == 64, "spatial attention: head_dim %d unsupported (64)", head_dim);
  JZ_CHECK_ARG(S == 256 || S == 257, "spatial attention: sequence length %d unsupported (256 or 257)", S);
  JZ_CHECK_ARG(frames >= 1 && frames * H < (1ll << 31), "spatial attention: frames");
  const int D = H * 64;
  CUtensorMap tm, tm_row, tm_o, tm_olo;
  int rc = make_tmap_2d_bf16(&tm, qkv, 3 * D, frames * S, 3 * D, 64, 128);
  if (!rc) rc = make_tmap_2d(&tm_row, qkv, 2, 3 * D, frames * S, 3 * D, 64, 1, /*swizzle128=*/false);
  if (!rc) rc = make_tmap_2d_bf16(&tm_o, out, D, frames * S, D, 64, 128);
  if (!rc && out_lo) rc = make_tmap_2d_bf16(&tm_olo, out_lo, D, frames * S, D, 64, 128);
  if (!out_lo) tm_olo = tm_o;
  if (rc) return rc;
  static bool attr_done = false;
  if (!attr_done) {
    JZ_CUDA_TRY(cudaFuncSetAttribute(spatial_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM));
    attr_done = true;
  }
  const int64_t units = frames * H;
  const int grid = (int)(units < num_sms() ? units : num_sms());
  spatial_fwd_kernel<<<grid, kFwdThreads, F_SMEM, reinterpret_cast<cudaStream_t>(s)>>>(
      tm, tm_row, tm_o, tm_olo, reinterpret_cast<const __nv_bfloat16*>(qkv), reinterpret_cast<__nv_bfloat16*>(out),
      reinterpret_cast<__nv_bfloat16*>(out_lo), lse, (int)frames, S, H);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

#ifdef JZ_SPATIAL_FWD_PROF
extern "C" int jz_attn_fwd_prof_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, jz::g_ftl, sizeof(jz::g_ftl)) == cudaSuccess ? 0 : -1;
}
#endif

// ============================================================================
// Backward: the tcgen05 kernel is csrc/attn_spatial_bwd.cu (v3); this file keeps the pass that
// forms its per-(frame, head) vectors.
// ============================================================================
namespace jz {
namespace sp {
// per-unit vector block written by spatial_uvb_rows_kernel, one per (frame, head), floats:
constexpr int U_LSE2 = 0;     // [0, 260)   lse * log2(e) per query row
constexpr int U_DV = 260;     // [260, 520) Delta = rowsum(dO o O) per query row
constexpr int U_PC = 520;     // p and dS of (query 256, key 256)
constexpr int U_DC = 521;
constexpr int U_Q = 524;      // q, k, v, dO of token 256 (fp32, 64 each)
constexpr int U_K = 588;
constexpr int U_V = 652;
constexpr int U_DO = 716;
constexpr int kUvbFloats = 780;  // 3120 bytes: 16-byte multiple for cp.async.bulk
}  // namespace sp
}  // namespace jz

// Per-unit vector blocks for the backward (layout sp::U_*): Delta_i = rowsum(dO_i o O_i) per head (dO
// the bf16 tensor the MMAs consume, O = the forward's bf16 output + its bf16 rounding residual), lse_i * log2(e) for every row, and for
// token 256 its q, k, v, dO vectors (fp32) and the (256, 256) entry p = exp(q.k / 8 - lse),
// dS = p (dO.v - Delta).  CTA (frame f, chunk c) owns rows [64 c, 64 c + 64) of the frame, so a
// launch has frames * ceil(S / 64) CTAs (one CTA per frame walking 257 rows was latency-bound at small
// batch: 90 -> 32 us at B = 8); each warp takes 8 rows, two at a time with both rows' loads in flight.
constexpr int kUvbMaxH = 16;
constexpr int kUvbRows = 64;
template <int NC>  // D / 128 column chunks per lane
__global__ void __launch_bounds__(256) spatial_uvb_rows_kernel(const __nv_bfloat16* __restrict__ out,
                                                               const __nv_bfloat16* __restrict__ out_lo,
                                                               const __nv_bfloat16* __restrict__ dout,
                                                               const __nv_bfloat16* __restrict__ qkv,
                                                               const float* __restrict__ lse, int64_t frames, int S,
                                                               int H, float* __restrict__ uvb) {
  using namespace jz::sp;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int D = H * 64;
  const float c2 = 0.125f * 1.4426950408889634f;
  const int chunks = (S + kUvbRows - 1) / kUvbRows;
  const int64_t f = blockIdx.x / chunks;
  const int c0 = (int)(blockIdx.x % chunks) * kUvbRows;
  // lse * log2(e) for this chunk's rows, every head
  for (int e = threadIdx.x; e < H * kUvbRows; e += blockDim.x) {
    const int h = e / kUvbRows, q = c0 + e % kUvbRows;
    if (q < S) uvb[(f * H + h) * kUvbFloats + U_LSE2 + q] = __ldg(lse + (f * H + h) * S + q) * 1.4426950408889634f;
  }
  // lane reads 8 consecutive columns (16-byte loads): column group g = lane + 32 j (D / 8 groups), head
  // g / 8, so the 8 lanes of a head fold with three shuffles
  constexpr int NG = 16 * NC, NJ = (NG + 31) / 32;
  for (int k0 = 0; k0 < kUvbRows / 8; k0 += 2) {
    float acc[2][NJ];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int sidx = c0 + warp * (kUvbRows / 8) + k0 + k;
#pragma unroll
      for (int jj = 0; jj < NJ; ++jj) {
        const int grp = lane + 32 * jj;
        float a = 0.f;
        if (sidx < S && grp < NG) {
          const int64_t row = f * S + sidx;
          const int col = 8 * grp;
          const uint4 hv = __ldg(reinterpret_cast<const uint4*>(out + row * D + col));
          const uint4 lv = __ldg(reinterpret_cast<const uint4*>(out_lo + row * D + col));
          const uint4 gv = __ldg(reinterpret_cast<const uint4*>(dout + row * D + col));
          const uint32_t hh[4] = {hv.x, hv.y, hv.z, hv.w}, ll[4] = {lv.x, lv.y, lv.z, lv.w}, gg[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 h2 = unpack_bf16(hh[e]), l2 = unpack_bf16(ll[e]), g2 = unpack_bf16(gg[e]);
            a += (h2.x + l2.x) * g2.x + (h2.y + l2.y) * g2.y;
          }
        }
        acc[k][jj] = a;
      }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int sidx = c0 + warp * (kUvbRows / 8) + k0 + k;
      if (sidx >= S) continue;
#pragma unroll
      for (int jj = 0; jj < NJ; ++jj) {
        float a = acc[k][jj];
#pragma unroll
        for (int m = 4; m >= 1; m >>= 1) a += __shfl_xor_sync(0xffffffffu, a, m);  // 8 lanes = one head
        const int grp = lane + 32 * jj;
        if ((lane & 7) == 0 && grp < NG) uvb[(f * H + grp / 8) * kUvbFloats + U_DV + sidx] = a;
      }
      if (sidx == 256) {  // token 256: its vectors and the (256, 256) entry, per head
        __syncwarp();  // Delta[256] of every head written above by this warp
        const int64_t row = f * S + sidx;
        const __nv_bfloat16* qr = qkv + row * 3 * (int64_t)D;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          {
            const int col = 128 * c + 4 * lane;
            const int h = col >> 6;
            float* ub = uvb + (f * H + h) * kUvbFloats;
            const uint2 gv = __ldg(reinterpret_cast<const uint2*>(dout + row * D + col));
            const uint2 qv = __ldg(reinterpret_cast<const uint2*>(qr + col));
            const uint2 kv = __ldg(reinterpret_cast<const uint2*>(qr + D + col));
            const uint2 vv = __ldg(reinterpret_cast<const uint2*>(qr + 2 * D + col));
            const float2 g0 = unpack_bf16(gv.x), g1 = unpack_bf16(gv.y);
            const float2 q0 = unpack_bf16(qv.x), q1 = unpack_bf16(qv.y), kk0 = unpack_bf16(kv.x),
                         kk1 = unpack_bf16(kv.y);
            const float2 v0 = unpack_bf16(vv.x), v1 = unpack_bf16(vv.y);
            const int d = col & 63;
            *reinterpret_cast<float4*>(ub + U_Q + d) = make_float4(q0.x, q0.y, q1.x, q1.y);
            *reinterpret_cast<float4*>(ub + U_K + d) = make_float4(kk0.x, kk0.y, kk1.x, kk1.y);
            *reinterpret_cast<float4*>(ub + U_V + d) = make_float4(v0.x, v0.y, v1.x, v1.y);
            *reinterpret_cast<float4*>(ub + U_DO + d) = make_float4(g0.x, g0.y, g1.x, g1.y);
            float sk = q0.x * kk0.x + q0.y * kk0.y + q1.x * kk1.x + q1.y * kk1.y;
            float dpv = g0.x * v0.x + g0.y * v0.y + g1.x * v1.x + g1.y * v1.y;
#pragma unroll
            for (int m = 8; m >= 1; m >>= 1) {
              sk += __shfl_xor_sync(0xffffffffu, sk, m);
              dpv += __shfl_xor_sync(0xffffffffu, dpv, m);
            }
            if ((lane & 15) == 0) {
              const float p = exp2f(sk * c2 - __ldg(lse + (f * H + h) * S + 256) * 1.4426950408889634f);
              ub[U_PC] = p;
              ub[U_DC] = p * (dpv - ub[U_DV + 256]);
            }
          }
        }
      }
    }
  }
}

namespace jz {
int spatial_bwd3_launch(const void* qkv, const void* dout, const float* uvb, int64_t frames, int S, int H, void* dqkv,
                        float* colsum_part, cudaStream_t st);
}

extern "C" int64_t jz_attn_spatial_bwd_workspace_bytes(int64_t frames, int S, int H) {
  (void)S;
  return frames * (int64_t)H * jz::sp::kUvbFloats * (int64_t)sizeof(float);
}

extern "C" int64_t jz_attn_spatial_colsum_parts(int64_t frames) { return frames * 9; }

extern "C" int jz_attn_spatial_bwd(const void* qkv, const void* out, const void* out_lo, const void* dout, const float* lse,
                                   int64_t frames, int S, int H, int head_dim, void* dqkv, void* workspace,
                                   float* colsum_part, jz_stream_t s) {
  using namespace jz;
  JZ_CHECK_ARG(head_dim == 64, "spatial attention bwd: head_dim %d unsupported (64)", head_dim);
  JZ_CHECK_ARG(S == 256 || S == 257, "spatial attention bwd: sequence length %d unsupported", S);
  const int D = H * 64;
  CUtensorMap tq, td;
  int rc = make_tmap_2d_bf16(&tq, qkv, 3 * D, frames * S, 3 * D, 64, 128);
  if (rc) return rc;
  rc = make_tmap_2d_bf16(&td, dout, D, frames * S, D, 64, 128);
  if (rc) return rc;
  JZ_CHECK_ARG(workspace != nullptr, "spatial attention bwd: workspace (jz_attn_spatial_bwd_workspace_bytes) required");
  JZ_CHECK_ARG(reinterpret_cast<uintptr_t>(workspace) % 16 == 0, "spatial attention bwd: workspace must be 16-byte aligned");
  float* uvb = reinterpret_cast<float*>(workspace);
  {
    JZ_CHECK_ARG(H <= kUvbMaxH, "spatial attention bwd: %d heads unsupported (<= 16)", H);
    const int64_t blocks = frames * ((S + kUvbRows - 1) / kUvbRows);
    JZ_CHECK_ARG(blocks < (1ll << 31), "spatial attention bwd: too many frames");
    JZ_CHECK_ARG(H % 2 == 0, "spatial attention bwd: an even head count is required (D multiple of 128)");
    JZ_CHECK_ARG(out != nullptr && out_lo != nullptr, "spatial attention bwd: the forward's output and its residual are required");
    auto oh = reinterpret_cast<const __nv_bfloat16*>(out);
    auto ol = reinterpret_cast<const __nv_bfloat16*>(out_lo);
    auto dd = reinterpret_cast<const __nv_bfloat16*>(dout);
    auto qq = reinterpret_cast<const __nv_bfloat16*>(qkv);
    auto st_ = reinterpret_cast<cudaStream_t>(s);
    switch (D / 128) {
      case 1: spatial_uvb_rows_kernel<1><<<(unsigned)blocks, 256, 0, st_>>>(oh, ol, dd, qq, lse, frames, S, H, uvb); break;
      case 2: spatial_uvb_rows_kernel<2><<<(unsigned)blocks, 256, 0, st_>>>(oh, ol, dd, qq, lse, frames, S, H, uvb); break;
      case 3: spatial_uvb_rows_kernel<3><<<(unsigned)blocks, 256, 0, st_>>>(oh, ol, dd, qq, lse, frames, S, H, uvb); break;
      case 4: spatial_uvb_rows_kernel<4><<<(unsigned)blocks, 256, 0, st_>>>(oh, ol, dd, qq, lse, frames, S, H, uvb); break;
      case 5: spatial_uvb_rows_kernel<5><<<(unsigned)blocks, 256, 0, st_>>>(oh, ol, dd, qq, lse, frames, S, H, uvb); break;
      case 6: spatial_uvb_rows_kernel<6><<<(unsigned)blocks, 256, 0, st_>>>(oh, ol, dd, qq, lse, frames, S, H, uvb); break;
      case 7: spatial_uvb_rows_kernel<7><<<(unsigned)blocks, 256, 0, st_>>>(oh, ol, dd, qq, lse, frames, S, H, uvb); break;
      default: spatial_uvb_rows_kernel<8><<<(unsigned)blocks, 256, 0, st_>>>(oh, ol, dd, qq, lse, frames, S, H, uvb); break;
    }
    JZ_LAUNCH_CHECK();
  }
  return spatial_bwd3_launch(qkv, dout, uvb, frames, S, H, dqkv, colsum_part, reinterpret_cast<cudaStream_t>(s));
}


