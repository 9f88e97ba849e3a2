// K3: spatial (intra-frame) attention on tcgen05 tensor cores, forward and backward.
//
// Replaces the spatial sub-layer's attention of st_block (st.py:73) =
// multi_head_attention(causal=False) (nn.py:80-110) with lead dims (B, T).
// One work unit = (frame, head): S = 256 (+1) tokens, hd = 64.
//
// S = 257 does not tile (256 patch tokens + the prepended action token,
// dynamics.py:118): tokens 0..255 run on the tensor cores as two 128-row query
// tiles against one 256-key tile; the 257th key is folded into each row's
// softmax on CUDA cores, and the 257th query row is computed by two "tail" warps
// on CUDA cores — exactly, no padding waste.
//
// qkv bf16 [M, 3D] (row = frame*S + s), out bf16 [M, D], lse f32 [frame][H][S].
#include <mutex>

#include "common.h"
#include "ptx.cuh"

namespace jz {

namespace sp {

constexpr int kFwdTailWarps = 4;  // query row 256 (S = 257) on CUDA cores, keys split 4 ways
constexpr int kFwdTailThreads = 32 * kFwdTailWarps;
constexpr int kFwdThreads = 320 + kFwdTailThreads;  // w0 TMA, w1 MMA, w2-5 tile 0, w6-9 tile 1, w10.. tail row
constexpr int TILE = 16384;    // 128 rows x 128 B
// forward smem map (bytes, from a 1024-aligned base)
constexpr int F_Q = 0;                 // 2 tiles
constexpr int F_K = F_Q + 2 * TILE;    // 2 tiles (256 keys)
constexpr int F_V = F_K + 2 * TILE;    // 2 tiles
constexpr int F_P0 = F_V + 2 * TILE;   // 4 atoms
constexpr int F_P1 = F_P0 + 4 * TILE;  // 4 atoms
constexpr int F_END = F_P1 + 4 * TILE; // 229376
constexpr int F_SMEM = F_END + 1024 + 2048;

struct FwdSmallSmem {
  uint64_t qk_full, v_full, qk_free, v_free;
  uint64_t s_full[2], p_full[2], o_full[2], tmem_free[2];
  uint32_t tmem_base;
  alignas(128) uint8_t krow[128];  // key 256 of the unit (TMA, arrives with Q/K)
  alignas(128) uint8_t vrow[128];  // value 256 of the unit (TMA, arrives with V)
  float tail_s[260];
  float tail_red[2 * kFwdTailWarps];
};
static_assert(sizeof(FwdSmallSmem) <= 2048, "forward small smem budget");

JZ_DEV void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

JZ_DEV float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// byte offset of (row r, 16-byte chunk c in 0..7) inside a 128B-swizzled 128-row tile
JZ_DEV uint32_t sw128(uint32_t r, uint32_t c) { return r * 128 + ((c ^ (r & 7)) << 4); }

}  // namespace sp

using namespace sp;

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

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm);
    tma_prefetch_desc(&tm_row);
    tma_prefetch_desc(&tm_o);
    if (out_lo) tma_prefetch_desc(&tm_olo);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(&sm.qk_full, 1); mbar_init(&sm.v_full, 1);
    // Q/K and V smem (+ rows 256) are released by the MMA commit, both softmax warpgroups and the tail
    mbar_init(&sm.qk_free, 1 + 256 + (has_tail ? kFwdTailThreads : 0));
    mbar_init(&sm.v_free, 1 + 256 + (has_tail ? kFwdTailThreads : 0));
    for (int t = 0; t < 2; ++t) {
      mbar_init(&sm.s_full[t], 1); mbar_init(&sm.p_full[t], 128);
      mbar_init(&sm.o_full[t], 1); mbar_init(&sm.tmem_free[t], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem_base);
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, sm.tmem_base, 0);

  if (warp == 0) {
    if (lane == 0) {
      int i = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
        const int f = u / H, h = u % H;
        const int row0 = f * S;
        mbar_wait(&sm.qk_free, (i & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.qk_full, 4 * TILE + (has_tail ? 128 : 0));
        if (has_tail) tma_load_2d(sm.krow, &tm_row, &sm.qk_full, D + h * 64, row0 + 256);
        tma_load_2d(smem + F_Q, &tm, &sm.qk_full, h * 64, row0);
        tma_load_2d(smem + F_Q + TILE, &tm, &sm.qk_full, h * 64, row0 + 128);
        tma_load_2d(smem + F_K, &tm, &sm.qk_full, D + h * 64, row0);
        tma_load_2d(smem + F_K + TILE, &tm, &sm.qk_full, D + h * 64, row0 + 128);
        mbar_wait(&sm.v_free, (i & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.v_full, 2 * TILE + (has_tail ? 128 : 0));
        if (has_tail) tma_load_2d(sm.vrow, &tm_row, &sm.v_full, 2 * D + h * 64, row0 + 256);
        tma_load_2d(smem + F_V, &tm, &sm.v_full, 2 * D + h * 64, row0);
        tma_load_2d(smem + F_V + TILE, &tm, &sm.v_full, 2 * D + h * 64, row0 + 128);
      }
    }
  } else if (warp == 1) {
    // the whole warp runs the loop (convergent: uniform operands); one elected lane issues
    {
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, 256, false, false);
      constexpr uint32_t idesc_o = idesc_bf16_f32(128, 64, false, true);
      // SW128 descriptors share one high word; low word = (address >> 4) | (LBO >> 4) << 16
      const uint32_t dhi = (uint32_t)(sdesc_sw128(0, 0, 1024) >> 32);
      auto dsc = [dhi](uint32_t addr4, uint32_t off, uint32_t lbo) -> uint64_t {
        return ((uint64_t)dhi << 32) | (addr4 + (off >> 4) + ((lbo >> 4) << 16));
      };
      const uint32_t q4 = smem_u32(smem + F_Q) >> 4, k4 = smem_u32(smem + F_K) >> 4, v4 = smem_u32(smem + F_V) >> 4;
      int i = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
        const uint32_t par = i & 1;
        mbar_wait(&sm.qk_full, par);
        for (int t = 0; t < 2; ++t) {
          mbar_wait(&sm.tmem_free[t], par ^ 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16_ss_w(tmem + 256 * t, dsc(q4, t * TILE + kk * 32, 16), dsc(k4, kk * 32, 16), idesc_s, kk > 0);
          umma_commit_w(&sm.s_full[t]);
        }
        umma_commit_w(&sm.qk_free);
        mbar_wait(&sm.v_full, par);
        for (int t = 0; t < 2; ++t) {
          mbar_wait(&sm.p_full[t], par);
          tc_fence_after();
          // O_t (cols 256t + 128 ..) += P_t V: P from TMEM (bf16 pairs over the first 128 S columns)
#pragma unroll
          for (int ks = 0; ks < 16; ++ks)
            umma_bf16_ts_w(tmem + 256 * t + 128, tmem + 256 * t + 8 * ks, dsc(v4, ks * 2048, 8192), idesc_o, ks > 0);
          umma_commit_w(&sm.o_full[t]);
        }
        umma_commit_w(&sm.v_free);
      }
    }
  } else if (warp < 10) {
    // softmax/epilogue warpgroup g owns query tile t = g; TMEM lane quarter = warp % 4
    const int t = (warp - 2) >> 2;
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;  // query row within the tile
    const int wtid = threadIdx.x - 64 - 128 * t;
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const uint32_t par = i & 1;
      const int f = u / H, h = u % H;
      const int64_t row0 = (int64_t)f * S;
      // previous unit's TMA stores must have finished reading this tile's P buffer
      if (wtid == 0) bulk_wait_read0();
      named_bar(1 + t, 128);
      mbar_wait(&sm.s_full[t], par);  // also implies Q/K (and key 256) landed in smem
      // score against the 257th key (CUDA cores): q row from the staged Q tile, k row 256 from smem
      float s_last = -INFINITY;
      if (has_tail) {
        const uint8_t* qt = smem + F_Q + t * TILE;
        const uint8_t* kr = sm.krow;
        float a = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 w = *reinterpret_cast<const uint4*>(qt + sw128(r, c));
          const uint4 kw = *reinterpret_cast<const uint4*>(kr + ((c ^ 0) << 4));
          const uint32_t qa[4] = {w.x, w.y, w.z, w.w}, ka[4] = {kw.x, kw.y, kw.z, kw.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 x = unpack_bf16(qa[e]), y = unpack_bf16(ka[e]);
            a += x.x * y.x + x.y * y.y;
          }
        }
        s_last = a;
      }
      mbar_arrive(&sm.qk_free);  // done with the Q tile and key row 256
      tc_fence_after();
      const uint32_t taddr = tmem + ((quarter * 32) << 16) + 256 * t;
      float mx = s_last;
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(taddr + 32 * c, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(v[j]));
      }
      const float mb = mx * c2;
      float sum = 0.f;
      uint8_t* pbuf = smem + (t ? F_P1 : F_P0);
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(taddr + 32 * c, v);
        tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float p0 = ex2(__uint_as_float(v[j]) * c2 - mb);
          const float p1 = ex2(__uint_as_float(v[j + 1]) * c2 - mb);
          pk[j / 2] = pack_bf16(p0, p1);
          const float2 pr = unpack_bf16(pk[j / 2]);  // normalise with the probabilities the MMA sees
          sum += pr.x + pr.y;
        }
        // keys 32c..32c+31 -> TMEM columns 16c..16c+15 as bf16 pairs (S columns already loaded)
        tmem_st_32x32b_x16(taddr + 16 * c, pk);
      }
      const float plast = has_tail ? ex2(s_last * c2 - mb) : 0.f;
      sum += plast;
      tmem_st_wait();
      tc_fence_before();
      mbar_arrive(&sm.p_full[t]);
      // O epilogue: stage O (bf16) and, for the backward's Delta, its rounding residual O - bf16(O)
      // (bf16: O to ~16 bits) in this tile's staging buffer, TMA-store both
      mbar_wait(&sm.o_full[t], par);
      tc_fence_after();
      const float inv = 1.0f / sum;
      const uint8_t* vrow = sm.vrow;
      uint8_t* o16 = pbuf;             // [128 rows][64 bf16], 128B swizzle
      uint8_t* olo = pbuf + TILE;      // [128 rows][64 bf16] residual
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(taddr + 128 + 32 * c, v);
        tmem_ld_wait();
        float o[32];
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
          const float2 vl = has_tail ? unpack_bf16(*reinterpret_cast<const uint32_t*>(vrow + 2 * (32 * c + j)))
                                     : make_float2(0.f, 0.f);
          o[j] = (__uint_as_float(v[j]) + plast * vl.x) * inv;
          o[j + 1] = (__uint_as_float(v[j + 1]) + plast * vl.y) * inv;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<uint4*>(o16 + sw128(r, 4 * c + q)) =
              make_uint4(pack_bf16(o[8 * q], o[8 * q + 1]), pack_bf16(o[8 * q + 2], o[8 * q + 3]),
                         pack_bf16(o[8 * q + 4], o[8 * q + 5]), pack_bf16(o[8 * q + 6], o[8 * q + 7]));
        if (out_lo) {
          uint32_t lo[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float2 hi = unpack_bf16(pack_bf16(o[2 * e], o[2 * e + 1]));
            lo[e] = pack_bf16(o[2 * e] - hi.x, o[2 * e + 1] - hi.y);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<uint4*>(olo + sw128(r, 4 * c + q)) = make_uint4(lo[4 * q], lo[4 * q + 1], lo[4 * q + 2], lo[4 * q + 3]);
        }
      }
      mbar_arrive(&sm.v_free);  // done with value row 256
      fence_proxy_async();
      named_bar(1 + t, 128);
      if (wtid == 0) {
        tma_store_2d(&tm_o, o16, h * 64, (int)(row0 + 128 * t));
        if (out_lo) tma_store_2d(&tm_olo, olo, h * 64, (int)(row0 + 128 * t));
        bulk_commit();
      }
      lse[((int64_t)f * H + h) * S + 128 * t + r] = mx * 0.125f + logf(sum);
      tc_fence_before();
      mbar_arrive_relaxed(&sm.tmem_free[t]);  // only TMEM reads precede (tcgen05.wait::ld done)
    }
  } else if (has_tail) {
    // tail warps: query row 256 on CUDA cores, reading K/V from the staged smem tiles
    const int tid = threadIdx.x - 320;  // 0 .. kFwdTailThreads - 1
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const uint32_t par = i & 1;
      const int f = u / H, h = u % H;
      const int64_t row0 = (int64_t)f * S;
      const __nv_bfloat16* q = qkv + (row0 + 256) * 3 * D + h * 64;
      float qf[64];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint4 w = reinterpret_cast<const uint4*>(q)[c];
        float2 a = unpack_bf16(w.x), b = unpack_bf16(w.y), cc = unpack_bf16(w.z), d = unpack_bf16(w.w);
        qf[8 * c] = a.x; qf[8 * c + 1] = a.y; qf[8 * c + 2] = b.x; qf[8 * c + 3] = b.y;
        qf[8 * c + 4] = cc.x; qf[8 * c + 5] = cc.y; qf[8 * c + 6] = d.x; qf[8 * c + 7] = d.y;
      }
      // key 256 from global, keys 0..255 from the swizzled K tile
      float mx = -INFINITY;
      mbar_wait(&sm.qk_full, par);
      if (tid == 0) {
        const uint4* kp = reinterpret_cast<const uint4*>(sm.krow);
        float a = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint4 w = kp[c];
          float2 x0 = unpack_bf16(w.x), x1 = unpack_bf16(w.y), x2 = unpack_bf16(w.z), x3 = unpack_bf16(w.w);
          a += qf[8 * c] * x0.x + qf[8 * c + 1] * x0.y + qf[8 * c + 2] * x1.x + qf[8 * c + 3] * x1.y +
               qf[8 * c + 4] * x2.x + qf[8 * c + 5] * x2.y + qf[8 * c + 6] * x3.x + qf[8 * c + 7] * x3.y;
        }
        sm.tail_s[256] = a;
        mx = a;
      }
      for (int k = tid; k < 256; k += kFwdTailThreads) {
        const uint8_t* kt = smem + F_K + (k >> 7) * TILE;
        float a = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint4 w = *reinterpret_cast<const uint4*>(kt + sw128(k & 127, c));
          float2 x0 = unpack_bf16(w.x), x1 = unpack_bf16(w.y), x2 = unpack_bf16(w.z), x3 = unpack_bf16(w.w);
          a += qf[8 * c] * x0.x + qf[8 * c + 1] * x0.y + qf[8 * c + 2] * x1.x + qf[8 * c + 3] * x1.y +
               qf[8 * c + 4] * x2.x + qf[8 * c + 5] * x2.y + qf[8 * c + 6] * x3.x + qf[8 * c + 7] * x3.y;
        }
        sm.tail_s[k] = a;
        mx = fmaxf(mx, a);
      }
      mbar_arrive(&sm.qk_free);
      mx = warp_max(mx);
      if (lane == 0) sm.tail_red[warp - 10] = mx;
      named_bar(3, kFwdTailThreads);
      mx = sm.tail_red[0];
#pragma unroll
      for (int w = 1; w < kFwdTailWarps; ++w) mx = fmaxf(mx, sm.tail_red[w]);
      const float mb = mx * c2;
      float sum = 0.f;
      for (int k = tid; k < S; k += kFwdTailThreads) {
        const float p = ex2(sm.tail_s[k] * c2 - mb);
        sm.tail_s[k] = p;
        sum += p;
      }
      sum = warp_sum(sum);
      if (lane == 0) sm.tail_red[kFwdTailWarps + warp - 10] = sum;
      named_bar(3, kFwdTailThreads);
      sum = 0.f;
#pragma unroll
      for (int w = 0; w < kFwdTailWarps; ++w) sum += sm.tail_red[kFwdTailWarps + w];
      // o[d] for d = 2*(tid&31) .. +1, keys split into kFwdTailWarps parts by warp
      constexpr int KP = 256 / kFwdTailWarps;
      const int dpair = tid & 31, part = tid >> 5;
      float o0 = 0.f, o1 = 0.f;
      mbar_wait(&sm.v_full, par);
      const uint32_t chunk = dpair >> 2, within = (dpair & 3) * 4;
#pragma unroll 8
      for (int k = part * KP; k < part * KP + KP; ++k) {
        const uint8_t* vt = smem + F_V + (k >> 7) * TILE;
        const float2 v = unpack_bf16(*reinterpret_cast<const uint32_t*>(vt + sw128(k & 127, chunk) + within));
        const float p = sm.tail_s[k];
        o0 += p * v.x;
        o1 += p * v.y;
      }
      if (part == kFwdTailWarps - 1) {  // value row 256, read before this thread releases V
        const float2 vl = unpack_bf16(*reinterpret_cast<const uint32_t*>(sm.vrow + 4 * dpair));
        const float p256 = sm.tail_s[256];
        o0 += p256 * vl.x;
        o1 += p256 * vl.y;
      }
      mbar_arrive(&sm.v_free);
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
  }
  if (warp >= 2 && warp < 10 && lane == 0) bulk_wait0();
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


