// K4: causal temporal (inter-frame) attention on tcgen05 tensor cores, forward and backward.
//
// Replaces the temporal sub-layer's attention of st_block (st.py:74-76) =
// multi_head_attention(causal=True) (nn.py:80-110) over the frame axis of each spatial slot,
// T <= 16 frames, head_dim 64.  The (B, T, S, D) -> (B, S, T, D) transpose of the reference
// never materialises: one work unit = (batch b, group of 8 spatial slots, head h) is a
// 128-row tile (8 slots x 16 frames) that TMA gathers from the (b, t, s)-ordered qkv rows with a
// 4-D box {64 columns, 16 frames, 8 slots, 1} over a (frame, slot)-permuted view of the tensor;
// tile row r = 16 slot + t.  Attention inside the tile is block-diagonal and causal: query (s, t)
// sees keys (s, t') with t' <= t, i.e. the row's own 16-column block.  The 128 x 128 score tile
// runs on the tensor core (dense: the work is HBM-bound, the masked MACs are free), the softmax
// reads one 32-column TMEM block per warp, and P / dS are block-diagonal bf16 tiles whose
// off-diagonal zeros are written once.
//
//   forward : S = Q K^T (TMEM), P = exp2(S c - m) masked, O = P V (TMEM), O / l -> TMA store, lse
//   backward: S = Q K^T, dP = dO V^T (TMEM); P = exp2(S c - lse), Delta = sum P dP (fp32, in the
//             row's registers), dS = P (dP - Delta); dV = P^T dO, dK = dS^T Q / 8, dQ = dS K / 8
//             (TMEM) -> TMA stores, + per-unit column sums of dqkv (the QKV bias gradient)
//
// Frames beyond T and slots beyond S are zero-filled by TMA on load and clipped on store; their
// rows contribute exactly zero to every gradient (their dO rows are zero).
#include <mutex>

#include "common.h"
#include "ptx.cuh"

namespace jz {
namespace ttc {

constexpr int TILE = 16384;     // 128 rows x 128 bytes (64 bf16), 128B-swizzled
constexpr int kThreads = 320;   // w0 TMA, w1 MMA, w2-5 softmax warpgroup, w6-9 epilogue warpgroup
constexpr int kSlots = 8;
constexpr int kFrames = 16;

// forward smem
constexpr int kFStages = 3;
constexpr int F_STAGE = 3 * TILE;             // q, k, v
constexpr int F_P = kFStages * F_STAGE;       // P: 2 atoms [128 query rows][64 keys] bf16
constexpr int F_O = F_P + 2 * TILE;           // 2 O staging tiles
constexpr int F_END = F_O + 2 * TILE;         // 212992
// backward smem
constexpr int kBStages = 2;
constexpr int B_STAGE = 4 * TILE;             // q, k, v, dO
constexpr int B_P = kBStages * B_STAGE;       // P (2 atoms)
constexpr int B_DS = B_P + 2 * TILE;          // dS (2 atoms)
constexpr int B_ST = B_DS + 2 * TILE;         // 2 output staging tiles
constexpr int B_END = B_ST + 2 * TILE;        // 229376

struct Bars {
  uint64_t full[3], empty[3];
  uint64_t a[2], b, c[2], d[2], e[2];  // per-kernel pipeline barriers (see the kernels)
  uint32_t tmem_base;
  float red[256];                      // fwd: row sums [2 buffers][128]; bwd: column partials [4 warps][64]
};
constexpr int F_SMEM = F_END + 1024 + (int)sizeof(Bars) + 16;
constexpr int B_SMEM = B_END + 1024 + (int)sizeof(Bars) + 16;
static_assert(B_SMEM <= 232448, "temporal tc bwd smem");

JZ_DEV uint32_t sw(uint32_t r, uint32_t c) { return r * 128 + ((c ^ (r & 7)) << 4); }
JZ_DEV void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
JZ_DEV float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

JZ_DEV uint32_t bf16_bits(float x) { return pack_bf16(x, 0.f) & 0xffffu; }

// the row's 16 block values (key frames t' = 0..15 of its slot): the warp's 32 rows are slots
// 2 quarter and 2 quarter + 1, whose keys are the 32 TMEM columns at 32 quarter; lanes 16..31 take
// the upper 16 (compile-time selects, no runtime register indexing)
JZ_DEV void gather_row(uint32_t taddr, int upper, float (&v)[16]) {
  uint32_t x[32];
  tmem_ld_32x32b_x32(taddr, x);
  tmem_ld_wait();
#pragma unroll
  for (int e = 0; e < 16; ++e) v[e] = __uint_as_float(upper ? x[16 + e] : x[e]);
}

// row r's 16 block values (keys 16 slot .. 16 slot + 15) as two 16-byte chunks of a block-diagonal
// K-major [128 rows][128 keys] bf16 tile (2 atoms of 64 keys)
JZ_DEV void put_block_row(uint8_t* tile, int r, const float (&v)[16]) {
  const int sl = r >> 4;
  uint8_t* atom = tile + (sl >> 2) * TILE;
#pragma unroll
  for (int h = 0; h < 2; ++h)
    *reinterpret_cast<uint4*>(atom + sw(r, 2 * (sl & 3) + h)) =
        make_uint4(pack_bf16(v[8 * h], v[8 * h + 1]), pack_bf16(v[8 * h + 2], v[8 * h + 3]),
                   pack_bf16(v[8 * h + 4], v[8 * h + 5]), pack_bf16(v[8 * h + 6], v[8 * h + 7]));
}

// Column sums over a warp's 32 rows of 32 values per lane (lane = row): returns the sum of column
// `lane` (fixed shuffle order: deterministic).
JZ_DEV float warp_colsum32(float (&v)[32], int lane) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const bool up = (lane & off) != 0;
#pragma unroll
    for (int k = 0; k < off; ++k) {
      const float send = up ? v[k] : v[k + off];
      const float keep = up ? v[k + off] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
    }
  }
  return v[0];
}

// 32 accumulator columns (TMEM) -> x sc -> bf16 into 16-byte chunks 4 half .. 4 half + 3 of row r
// of a 128B-swizzled tile; v gets the bf16-rounded values
JZ_DEV void stage_row32(uint32_t taddr, float sc, uint8_t* tile, int r, int half, float (&v)[32]) {
  uint32_t o[32];
  tmem_ld_32x32b_x32(taddr, o);
  tmem_ld_wait();
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      w[k] = pack_bf16(__uint_as_float(o[8 * c + 2 * k]) * sc, __uint_as_float(o[8 * c + 2 * k + 1]) * sc);
      const float2 f = unpack_bf16(w[k]);
      v[8 * c + 2 * k] = f.x;
      v[8 * c + 2 * k + 1] = f.y;
    }
    *reinterpret_cast<uint4*>(tile + sw(r, 4 * half + c)) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

}  // namespace ttc

using namespace ttc;

// Forward.  Barriers: a[buf] S ready (MMA -> softmax), b P staged (softmax -> MMA, 128 arrivals),
// c[buf] O ready (MMA -> epilogue), d[buf] S/O columns free (epilogue -> MMA, 128), e[buf] row sums
// of buffer buf written (softmax -> epilogue, 128).
__global__ void __launch_bounds__(ttc::kThreads, 1)
    temporal_tc_fwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_o,
                           float* __restrict__ lse, int B, int T, int S, int H, int NG) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  Bars& bar = *reinterpret_cast<Bars*>(smem + F_END);
  const int D = H * 64;
  const int warp = __shfl_sync(0xffffffffu, (int)warp_id(), 0), lane = lane_id();  // warp-uniform
  const int units = B * NG * H;
  const float c2 = 0.125f * 1.4426950408889634f;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_o);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < kFStages; ++i) {
      mbar_init(&bar.full[i], 1);
      mbar_init(&bar.empty[i], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar.a[b], 1);
      mbar_init(&bar.c[b], 1);
      mbar_init(&bar.d[b], 128);
      mbar_init(&bar.e[b], 128);
    }
    mbar_init(&bar.b, 128);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&bar.tmem_base);
  // P is block-sparse with a fixed zero pattern: zero it once, the rows rewrite only their window
  for (int i = threadIdx.x; i < 2 * TILE / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem + F_P)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, bar.tmem_base, 0);

  if (warp == 0) {
    if (lane == 0) {
      int i = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
        const int h = u % H, g = (u / H) % NG, b = u / (H * NG);
        const int st = i % kFStages;
        mbar_wait(&bar.empty[st], ((i / kFStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&bar.full[st], F_STAGE);
        uint8_t* dst = smem + st * F_STAGE;
        for (int w = 0; w < 3; ++w) tma_load_4d(dst + w * TILE, &tm_qkv, &bar.full[st], w * D + h * 64, 0, g * kSlots, b);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id_s = idesc_bf16_f32(128, 128, false, false);
    constexpr uint32_t id_o = idesc_bf16_f32(128, 64, false, true);
    const uint32_t dhi = (uint32_t)(sdesc_sw128(0, 0, 1024) >> 32);
    auto dsc = [dhi](uint32_t addr4, uint32_t off, uint32_t lbo) -> uint64_t {
      return ((uint64_t)dhi << 32) | (addr4 + (off >> 4) + ((lbo >> 4) << 16));
    };
    const uint32_t p4 = smem_u32(smem + F_P) >> 4;
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const int st = i % kFStages, buf = i & 1;
      const uint32_t q4 = smem_u32(smem + st * F_STAGE) >> 4;
      const uint32_t k4 = q4 + (TILE >> 4), v4 = q4 + (2 * TILE >> 4);
      mbar_wait(&bar.full[st], (i / kFStages) & 1);
      mbar_wait(&bar.d[buf], ((i >> 1) & 1) ^ 1);
      tc_fence_after();
      umma4_bf16_ss_w(tmem + 128 * buf, dsc(q4, 0, 16), dsc(k4, 0, 16), 2, 2, id_s, 0);
      umma_commit_w(&bar.a[buf]);
      mbar_wait(&bar.b, i & 1);
      tc_fence_after();
#pragma unroll
      for (int hk = 0; hk < 2; ++hk)
        umma4_bf16_ss_w(tmem + 256 + 64 * buf, dsc(p4, hk * TILE, 16), dsc(v4, hk * 4 * 2048, 8192), 2, 2048 >> 4, id_o,
                        hk);
      umma_commit_w(&bar.c[buf]);
      umma_commit_w(&bar.empty[st]);
    }
  } else if (warp < 6) {
    // ---- softmax warpgroup: row r = TMEM lane = query (slot r / 16, frame t = r % 16)
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int t = r & 15, sl = r >> 4;
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const int h = u % H, g = (u / H) % NG, b = u / (H * NG);
      const int buf = i & 1;
      mbar_wait(&bar.a[buf], (i >> 1) & 1);
      tc_fence_after();
      float s[16];
      gather_row(tmem + ((quarter * 32) << 16) + 128 * buf + 32 * quarter, lane >> 4, s);
      float mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < 16; ++e)
        if (e <= t) mx = fmaxf(mx, s[e]);
      const float mb = mx * c2;
      if (i > 0) mbar_wait(&bar.c[buf ^ 1], ((i - 1) >> 1) & 1);  // the previous unit's PV has read P
      float sum = 0.f, sum16 = 0.f;
      float p[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        p[e] = e <= t ? ex2(s[e] * c2 - mb) : 0.f;
        sum += p[e];
        sum16 += __uint_as_float(bf16_bits(p[e]) << 16);  // O is normalised with the probabilities the MMA sees
      }
      put_block_row(smem + F_P, r, p);
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&bar.b);
      bar.red[buf * 128 + r] = sum16;
      mbar_arrive(&bar.e[buf]);
      const int s_idx = g * kSlots + sl;
      if (t < T && s_idx < S) lse[(((int64_t)b * S + s_idx) * H + h) * T + t] = mx * 0.125f + logf(sum);
    }
  } else {
    // ---- epilogue warpgroup: O / l -> bf16 -> TMA store; each warp stores its own 32 rows
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    uint8_t* wst = smem + F_O + (warp - 6) * 2 * (TILE / 4);  // this warp's two 4 KB staging slices
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const int h = u % H, g = (u / H) % NG, b = u / (H * NG);
      const int buf = i & 1;
      mbar_wait(&bar.c[buf], (i >> 1) & 1);
      mbar_wait(&bar.e[buf], (i >> 1) & 1);
      tc_fence_after();
      const float inv = 1.0f / bar.red[buf * 128 + r];
      uint8_t* ot = wst + buf * (TILE / 4);
      if (lane == 0) bulk_wait_read1();  // this slice's store of two units ago has read it
      __syncwarp();
      float v[32];
      stage_row32(tmem + ((quarter * 32) << 16) + 256 + 64 * buf, inv, ot, lane, 0, v);
      stage_row32(tmem + ((quarter * 32) << 16) + 256 + 64 * buf + 32, inv, ot, lane, 1, v);
      tc_fence_before();
      mbar_arrive(&bar.d[buf]);
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) {
        tma_store_4d(&tm_o, ot, h * 64, 0, g * kSlots + 2 * quarter, b);
        bulk_commit();
      }
    }
    if (lane == 0) bulk_wait0();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// Backward.  Barriers: a[0] S and dP ready (MMA -> softmax), b P and dS staged (softmax -> MMA,
// 128), c[0] dV / dK / dQ ready (MMA -> epilogue; also: the gradient MMAs finished reading P / dS),
// d[0] gradient columns read (epilogue -> MMA, 128).
__global__ void __launch_bounds__(ttc::kThreads, 1)
    temporal_tc_bwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                           const __grid_constant__ CUtensorMap tm_dqkv, const float* __restrict__ lse,
                           float* __restrict__ colsum, int B, int T, int S, int H, int NG) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  Bars& bar = *reinterpret_cast<Bars*>(smem + B_END);
  const int D = H * 64;
  const int warp = __shfl_sync(0xffffffffu, (int)warp_id(), 0), lane = lane_id();  // warp-uniform
  const int units = B * NG * H;
  const float c2 = 0.125f * 1.4426950408889634f;
  constexpr uint32_t C_S = 0, C_DP = 128, C_DV = 256, C_DK = 320, C_DQ = 384;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
    tma_prefetch_desc(&tm_dqkv);
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < kBStages; ++i) {
      mbar_init(&bar.full[i], 1);
      mbar_init(&bar.empty[i], 1);
    }
    mbar_init(&bar.a[0], 1);
    mbar_init(&bar.b, 128);
    mbar_init(&bar.c[0], 1);
    mbar_init(&bar.d[0], 128);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&bar.tmem_base);
  for (int i = threadIdx.x; i < 4 * TILE / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem + B_P)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, bar.tmem_base, 0);

  if (warp == 0) {
    if (lane == 0) {
      int i = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
        const int h = u % H, g = (u / H) % NG, b = u / (H * NG);
        const int st = i % kBStages;
        mbar_wait(&bar.empty[st], ((i / kBStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&bar.full[st], B_STAGE);
        uint8_t* dst = smem + st * B_STAGE;
        for (int w = 0; w < 3; ++w) tma_load_4d(dst + w * TILE, &tm_qkv, &bar.full[st], w * D + h * 64, 0, g * kSlots, b);
        tma_load_4d(dst + 3 * TILE, &tm_do, &bar.full[st], h * 64, 0, g * kSlots, b);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id_s = idesc_bf16_f32(128, 128, false, false);  // S = Q K^T, dP = dO V^T
    constexpr uint32_t id_t = idesc_bf16_f32(128, 64, true, true);     // dV = P^T dO, dK = dS^T Q
    constexpr uint32_t id_q = idesc_bf16_f32(128, 64, false, true);    // dQ = dS K
    const uint32_t dhi = (uint32_t)(sdesc_sw128(0, 0, 1024) >> 32);
    auto dsc = [dhi](uint32_t addr4, uint32_t off, uint32_t lbo) -> uint64_t {
      return ((uint64_t)dhi << 32) | (addr4 + (off >> 4) + ((lbo >> 4) << 16));
    };
    const uint32_t p4 = smem_u32(smem + B_P) >> 4, ds4 = smem_u32(smem + B_DS) >> 4;
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const int st = i % kBStages;
      const uint32_t q4 = smem_u32(smem + st * B_STAGE) >> 4;
      const uint32_t k4 = q4 + (TILE >> 4), v4 = q4 + (2 * TILE >> 4), do4 = q4 + (3 * TILE >> 4);
      mbar_wait(&bar.full[st], (i / kBStages) & 1);
      tc_fence_after();
      // S / dP columns are free: this thread already waited on b for the previous unit
      umma4x2_bf16_ss_w(tmem + C_S, dsc(q4, 0, 16), dsc(k4, 0, 16), tmem + C_DP, dsc(do4, 0, 16), dsc(v4, 0, 16), 2, 2,
                        id_s, 0);
      umma_commit_w(&bar.a[0]);
      mbar_wait(&bar.b, i & 1);                // P / dS staged (S / dP read)
      mbar_wait(&bar.d[0], (i & 1) ^ 1);       // the previous unit's gradients left TMEM
      tc_fence_after();
#pragma unroll
      for (int hk = 0; hk < 2; ++hk) {
        // contraction over queries (16 rows = 2048 bytes per step); P^T / dS^T are MN-major reads
        umma4x2_bf16_ss_w(tmem + C_DV, dsc(p4, hk * 4 * 2048, TILE), dsc(do4, hk * 4 * 2048, 8192), tmem + C_DK,
                          dsc(ds4, hk * 4 * 2048, TILE), dsc(q4, hk * 4 * 2048, 8192), 2048 >> 4, 2048 >> 4, id_t, hk);
        // contraction over keys: dS K-major (atom hk), K rows MN-major
        umma4_bf16_ss_w(tmem + C_DQ, dsc(ds4, hk * TILE, 16), dsc(k4, hk * 4 * 2048, 8192), 2, 2048 >> 4, id_q, hk);
      }
      umma_commit_w(&bar.c[0]);
      umma_commit_w(&bar.empty[st]);
    }
  } else if (warp < 6) {
    // ---- softmax warpgroup: P, Delta, dS for query row r (slot r / 16, frame r % 16)
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int t = r & 15, sl = r >> 4;
    const uint32_t tl = tmem + ((quarter * 32) << 16);
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const int h = u % H, g = (u / H) % NG, b = u / (H * NG);
      const int s_idx = g * kSlots + sl;
      const bool live = t < T && s_idx < S;
      const float lse2 = live ? __ldg(lse + (((int64_t)b * S + s_idx) * H + h) * T + t) * 1.4426950408889634f : 0.f;
      mbar_wait(&bar.a[0], i & 1);
      tc_fence_after();
      float s[16], dp[16];
      gather_row(tl + C_S + 32 * quarter, lane >> 4, s);
      gather_row(tl + C_DP + 32 * quarter, lane >> 4, dp);
      // Delta_i = sum_j P_ij dP_ij from the row's own fp32 values (= dO_i . O_i in exact arithmetic)
      float p[16];
      float delta = 0.f;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        p[e] = (live && e <= t) ? ex2(s[e] * c2 - lse2) : 0.f;
        delta += p[e] * dp[e];
      }
      if (i > 0) mbar_wait(&bar.c[0], (i - 1) & 1);  // the previous unit's gradient MMAs read P / dS
      float ds[16];
#pragma unroll
      for (int e = 0; e < 16; ++e) ds[e] = p[e] * (dp[e] - delta);
      put_block_row(smem + B_P, r, p);
      put_block_row(smem + B_DS, r, ds);
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&bar.b);
    }
  } else {
    // ---- epilogue warpgroup: dQ (row = query, x 1/8), dK (row = key, x 1/8), dV (row = key).
    // Each warp stages and TMA-stores its own 32 rows (frames 4 quarter .. 4 quarter + 3 of the
    // tile): no cross-warp synchronisation per unit.  The grid is a multiple of H, so every unit of
    // this CTA has head blockIdx % H: the column sums (the QKV bias gradient) stay in registers
    // across all its units and are flushed once into the CTA's partial row.
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int etid = threadIdx.x - 192;
    const int wg_warp = warp - 6;
    const uint32_t tl = tmem + ((quarter * 32) << 16);
    uint8_t* wst = smem + B_ST + wg_warp * 2 * (TILE / 4);  // this warp's two 4 KB staging slices
    float acc[3][2] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};
    int cur_h = -1;
    float* part = colsum != nullptr ? colsum + (int64_t)blockIdx.x * 3 * D : nullptr;
    if (part != nullptr) {
      for (int c = etid; c < 3 * D; c += 128) part[c] = 0.f;
      named_bar(1, 128);
    }
    auto flush = [&](int h) {  // 4 warps' column sums of head h -> the CTA's partial row, fixed order
#pragma unroll 1
      for (int w = 0; w < 3; w += 2) {
        bar.red[wg_warp * 64 + lane] = acc[w][0];
        bar.red[wg_warp * 64 + 32 + lane] = acc[w][1];
        named_bar(1, 128);
        if (etid < 64)
          part[w * D + h * 64 + etid] =
              ((bar.red[etid] + bar.red[64 + etid]) + bar.red[128 + etid]) + bar.red[192 + etid];
        named_bar(1, 128);
        acc[w][0] = acc[w][1] = 0.f;
      }
    };
    int i = 0;
    int nst = 0;  // stores issued by this warp (staging slices alternate)
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const int h = u % H, g = (u / H) % NG, b = u / (H * NG);
      cur_h = h;
      mbar_wait(&bar.c[0], i & 1);
      tc_fence_after();
#pragma unroll 1
      for (int w = 0; w < 3; ++w, ++nst) {  // column block w of dqkv: 0 dQ, 1 dK, 2 dV
        const uint32_t c0 = w == 0 ? C_DQ : (w == 1 ? C_DK : C_DV);
        uint8_t* ot = wst + (nst & 1) * (TILE / 4);
        if (lane == 0) bulk_wait_read1();  // this slice's previous store (two ago) has read it
        __syncwarp();
        const float sc = w == 2 ? 1.0f : 0.125f;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {  // 32 columns at a time: staged, and their column sums
          float v[32];
          stage_row32(tl + c0 + 32 * hf, sc, ot, lane, hf, v);
          // the key-bias gradient is exactly zero (a bias on every key shifts a softmax row by a
          // constant): its partial columns stay zero
          if (part != nullptr && w != 1) acc[w][hf] += warp_colsum32(v, lane);
        }
        if (w == 2) {
          tc_fence_before();
          mbar_arrive(&bar.d[0]);  // gradient columns read: the next unit's gradient MMAs may start
        }
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          tma_store_4d(&tm_dqkv, ot, w * D + h * 64, 0, g * kSlots + 2 * quarter, b);
          bulk_commit();
        }
      }
    }
    if (part != nullptr && cur_h >= 0) flush(cur_h);
    if (lane == 0) bulk_wait0();
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// qkv-shaped [B, T, S, C] bf16 rows viewed with the frame and slot axes swapped, {C, T, S, B}
// (frame stride S C, slot stride C), as the 4-D box source {64 columns, 16 frames, slots, 1}
// (8 slots: a whole 128-row unit tile; 2 slots: one warp's 32-row slice of it)
static int make_unit_map(CUtensorMap* m, const void* base, int64_t B, int T, int S, int C, int slots = kSlots) {
  const uint64_t dims[4] = {(uint64_t)C, (uint64_t)T, (uint64_t)S, (uint64_t)B};
  const uint64_t strides[3] = {(uint64_t)S * C * 2, (uint64_t)C * 2, (uint64_t)T * S * C * 2};
  const uint32_t box[4] = {64, kFrames, (uint32_t)slots, 1};
  return make_tmap_4d_bf16(m, base, dims, strides, box);
}

int temporal_tc_fwd(const void* qkv, int64_t B, int T, int S, int H, void* out, float* lse, cudaStream_t st) {
  const int D = H * 64;
  const int NG = (S + kSlots - 1) / kSlots;
  CUtensorMap tq, to;
  int rc = make_unit_map(&tq, qkv, B, T, S, 3 * D);
  if (!rc) rc = make_unit_map(&to, out, B, T, S, D, 2);
  if (rc) return rc;
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(temporal_tc_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM);
  });
  JZ_CUDA_TRY(attr);
  const int64_t units = B * NG * H;
  const int grid = (int)(units < num_sms() ? units : num_sms());
  temporal_tc_fwd_kernel<<<grid, kThreads, F_SMEM, st>>>(tq, to, lse, (int)B, T, S, H, NG);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

// backward grid: a multiple of H (every CTA keeps one head), at most one CTA per SM
static int64_t bwd_grid(int64_t B, int S, int H) {
  const int64_t units = B * ((S + kSlots - 1) / kSlots) * H;
  int64_t grid = (num_sms() / H) * H;
  if (grid < H) grid = H;
  return units < grid ? units : grid;
}

int64_t temporal_tc_colsum_parts(int64_t B, int S, int H) { return bwd_grid(B, S, H); }  // one row per CTA

int temporal_tc_bwd(const void* qkv, const void* dout, const float* lse, int64_t B, int T, int S, int H, void* dqkv,
                    float* colsum, cudaStream_t st) {
  const int D = H * 64;
  const int NG = (S + kSlots - 1) / kSlots;
  CUtensorMap tq, td, tg;
  int rc = make_unit_map(&tq, qkv, B, T, S, 3 * D);
  if (!rc) rc = make_unit_map(&td, dout, B, T, S, D);
  if (!rc) rc = make_unit_map(&tg, dqkv, B, T, S, 3 * D, 2);
  if (rc) return rc;
  static std::once_flag once;
  static cudaError_t attr = cudaSuccess;
  std::call_once(once, [] {
    attr = cudaFuncSetAttribute(temporal_tc_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, B_SMEM);
  });
  JZ_CUDA_TRY(attr);
  const int grid = (int)bwd_grid(B, S, H);
  temporal_tc_bwd_kernel<<<grid, kThreads, B_SMEM, st>>>(tq, td, tg, lse, colsum, (int)B, T, S, H, NG);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

}  // namespace jz
