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
// Backward.  Per (frame, head) unit, in the transposed ("S^T") formulation, over
// 8 blocks x = (key half j in 0..1) x (64-query block c in 0..3):
//   S^T  = K_j Q_c^T,  dP^T = V_j dO_c^T          (TMEM, double-buffered 2 x 128 cols)
//   P^T  = exp2(S^T*c2 - lse2),  dS^T = P^T (dP^T - D)      (8 "P/dS" warps)
//        P^T goes back into TMEM over its own S^T columns (bf16 pairs), dS^T to smem slot c
//   dV_j += P^T dO_c  (A from TMEM),  dK_j += dS^T Q_c,   and per query tile t = c/2:
//   dQ_t += dS K_j    (A = slots 2t, 2t+1 read MN-major)    (TMEM accumulators, 256 cols)
// The MMA warp issues S/dP of block x+1 before the gradient MMAs of block x, so the
// tensor core overlaps the elementwise stage. Delta = rowsum(dO o O_f32) comes from a
// separate coalesced pass (spatial_delta_kernel). A 4-warp helper group forms the
// row-256 / key-256 dot products on CUDA cores as soon as the tiles land (off the P/dS
// critical path), reduces the row-256 gradients, runs the three epilogues (TMEM -> swizzled smem -> coalesced stores, TMEM
// released before the stores), and prefetches the next unit's lse / Delta / tail vectors.
// ============================================================================
#ifdef JZ_ATTN_PROF
__device__ unsigned long long g_attn_prof[64 * 32];
#define PROF_MARK(slot)                                                                   \
  do {                                                                                    \
    if (blockIdx.x == 0 && i < 32) g_attn_prof[i * 64 + (slot)] = clock64();             \
  } while (0)
#else
#define PROF_MARK(slot) \
  do {                  \
  } while (0)
#endif
namespace jz {
namespace sp {
constexpr int kBwdWarps = 14;  // w0 TMA, w1 MMA, w2-9 P/dS, w10-13 helper (tail + epilogues + prep)
constexpr int kBwdThreads2 = 32 * kBwdWarps;
constexpr int B_Q = 0;
constexpr int B_K = B_Q + 2 * TILE;
constexpr int B_V = B_K + 2 * TILE;
constexpr int B_DO = B_V + 2 * TILE;
constexpr int B_DS = B_DO + 2 * TILE;    // 4 slots [128 keys][64 queries] bf16, slot = query block
constexpr int B_ST = B_DS + 4 * TILE;    // epilogue staging tile [128 rows][64] bf16 (TMA store)
constexpr int B_END = B_ST + TILE;       // 212992
// per-unit vector block written by spatial_delta_kernel, one per (frame, head), floats:
constexpr int U_LSE2 = 0;     // [0, 260)   lse * log2(e) per query row
constexpr int U_DV = 260;     // [260, 520) Delta = rowsum(dO o O) per query row
constexpr int U_PC = 520;     // p and dS of (query 256, key 256)
constexpr int U_DC = 521;
constexpr int kUvbHead = 524;   // lse2, Delta, corner: the part the v3 backward loads (2096 bytes)
constexpr int U_Q = 524;      // q, k, v, dO of token 256 (fp32, 64 each)
constexpr int U_K = 588;
constexpr int U_V = 652;
constexpr int U_DO = 716;
constexpr int kUvbFloats = 780;  // 3120 bytes: 16-byte multiple for cp.async.bulk

struct BwdSmallSmem {
  uint64_t load_full, inputs_free, dkdv_full, dkdv_free, dq_full, dq_free;
  uint64_t sdp_full[2], pds_full[2], ds_free[2];

  uint32_t tmem_base;
  // per-unit vector block (UVB), double-buffered, bulk-loaded by the TMA warp with the tiles
  alignas(16) float uvb[2][kUvbFloats];
  float p_col[2][260], ds_col[2][260];  // key 256 column over queries 0..255 (helper, per unit)
  float p_row[260], ds_row[260];        // query 256 row over keys 0..256 (current unit)
  float tail_red[3][4][64];
};
constexpr int B_SMEM = B_END + 1024 + (int)sizeof(BwdSmallSmem) + 64;
static_assert(B_SMEM <= 232448, "spatial bwd smem budget");
}  // namespace sp

// One warp writes its 32 rows (64 bf16 each) coalesced: stage row-per-lane in its own 4 KB
// (128B-swizzled), then read back 4 rows x 128 B per instruction.
// TMEM row (64 fp32 columns at taddr) -> sc * (acc + coef * vec) -> bf16 straight into the staging row.
JZ_DEV void bwd_stage_acc(uint8_t* wstage, uint32_t taddr, float coef, const float* vec, float sc, int lane) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t vv[16];
    tmem_ld_32x32b_x16(taddr + 16 * q, vv);
    tmem_ld_wait();
    uint32_t w[8];
#pragma unroll
    for (int e = 0; e < 16; e += 2)
      w[e / 2] = pack_bf16(sc * (__uint_as_float(vv[e]) + coef * vec[16 * q + e]),
                           sc * (__uint_as_float(vv[e + 1]) + coef * vec[16 * q + e + 1]));
    *reinterpret_cast<uint4*>(wstage + lane * 128 + (((2 * q) ^ (lane & 7)) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
    *reinterpret_cast<uint4*>(wstage + lane * 128 + (((2 * q + 1) ^ (lane & 7)) << 4)) = make_uint4(w[4], w[5], w[6], w[7]);
  }
  __syncwarp();
}

// ... and, when `part` is set, the warp's column sums over its 32 rows (8 columns per lane of the
// first 8 lanes) into one partial row: part[col .. col + 63] (bias gradients of the QKV layer).
JZ_DEV void bwd_flush_rows(const uint8_t* wstage, __nv_bfloat16* dqkv, int64_t row_first, int64_t ld3, int64_t col,
                           int lane, float* part) {
  const int cch = lane & 7;
  float cs[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int rr = 4 * k + (lane >> 3);
    const uint4 w = *reinterpret_cast<const uint4*>(wstage + rr * 128 + ((cch ^ (rr & 7)) << 4));
    *reinterpret_cast<uint4*>(dqkv + (row_first + rr) * ld3 + col + 8 * cch) = w;
    if (part != nullptr) {
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = unpack_bf16(ww[e]);
        cs[2 * e] += f.x;
        cs[2 * e + 1] += f.y;
      }
    }
  }
  if (part != nullptr) {
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      cs[e] += __shfl_xor_sync(0xffffffffu, cs[e], 8);
      cs[e] += __shfl_xor_sync(0xffffffffu, cs[e], 16);
    }
    if (lane < 8) {
      float4* dst = reinterpret_cast<float4*>(part + col + 8 * cch);
      dst[0] = make_float4(cs[0], cs[1], cs[2], cs[3]);
      dst[1] = make_float4(cs[4], cs[5], cs[6], cs[7]);
    }
  }
  __syncwarp();
}

__global__ void __launch_bounds__(sp::kBwdThreads2, 1)
    spatial_bwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                       const float* __restrict__ uvb, __nv_bfloat16* __restrict__ dqkv, float* __restrict__ colsum,
                       int frames, int S, int H) {
  using namespace sp;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  BwdSmallSmem& sm = *reinterpret_cast<BwdSmallSmem*>(smem + B_END);
  const int D = H * 64;
  const int warp = __shfl_sync(0xffffffffu, (int)warp_id(), 0), lane = lane_id();  // warp-uniform
  const int units = frames * H;
  const bool has_tail = S > 256;
  const float scale = 0.125f;
  const float c2 = 0.125f * 1.4426950408889634f;
  const int64_t ld3 = 3 * (int64_t)D;
  constexpr uint32_t C_DV = 256, C_DK = 320, C_DQ = 384;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(&sm.load_full, 1);
    mbar_init(&sm.inputs_free, 1 + 4);  // MMA commit + 4 helper warps (row-256 reductions read the tiles)
    mbar_init(&sm.dkdv_full, 1);
    mbar_init(&sm.dkdv_free, 4);
    mbar_init(&sm.dq_full, 1);
    mbar_init(&sm.dq_free, 4);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.sdp_full[b], 1);
      mbar_init(&sm.pds_full[b], 8);
      mbar_init(&sm.ds_free[b], 1);
    }
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
        mbar_wait(&sm.inputs_free, (i & 1) ^ 1);
        PROF_MARK(53);
        mbar_arrive_expect_tx(&sm.load_full, 8 * TILE + kUvbFloats * 4);
        bulk_load(sm.uvb[i & 1], uvb + (int64_t)u * kUvbFloats, kUvbFloats * 4, &sm.load_full);
        for (int t = 0; t < 2; ++t) {
          tma_load_2d(smem + B_K + t * TILE, &tm_qkv, &sm.load_full, D + h * 64, row0 + 128 * t);
          tma_load_2d(smem + B_Q + t * TILE, &tm_qkv, &sm.load_full, h * 64, row0 + 128 * t);
          tma_load_2d(smem + B_V + t * TILE, &tm_qkv, &sm.load_full, 2 * D + h * 64, row0 + 128 * t);
          tma_load_2d(smem + B_DO + t * TILE, &tm_do, &sm.load_full, h * 64, row0 + 128 * t);
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ------------------------------
    // the whole warp runs the loop (convergent: uniform operands); one elected lane issues
    {
      constexpr uint32_t id_s = idesc_bf16_f32(128, 64, false, false);   // K_j Q_c^T, V_j dO_c^T
      constexpr uint32_t id_kv = idesc_bf16_f32(128, 64, false, true);   // P^T dO_c, dS^T Q_c
      constexpr uint32_t id_q = idesc_bf16_f32(128, 64, true, true);     // dS K_j
      // SW128 descriptors share one high word (SBO = 1024, version, swizzle); the low word is
      // (address >> 4) | (LBO >> 4) << 16, so each MMA's descriptor is one add on a shifted base
      const uint32_t dhi = (uint32_t)(sdesc_sw128(0, 0, 1024) >> 32);
      const uint32_t aq = smem_u32(smem + B_Q) >> 4, ak = smem_u32(smem + B_K) >> 4, av = smem_u32(smem + B_V) >> 4,
                     ado = smem_u32(smem + B_DO) >> 4, ads = smem_u32(smem + B_DS) >> 4;
      auto dsc = [dhi](uint32_t addr4, uint32_t off, uint32_t lbo) -> uint64_t {
        return ((uint64_t)dhi << 32) | (addr4 + (off >> 4) + ((lbo >> 4) << 16));
      };
      // gradient MMAs of block y of unit i (its P^T / dS^T are ready once pds_full fires)
      auto grad_mmas = [&](int i, int y) {
        const uint32_t gy = 8u * i + y, by = gy & 1;
        const int jy = y >> 2, cy = y & 3;
        mbar_wait(&sm.pds_full[by], (gy >> 1) & 1);
        PROF_MARK(10 + y);
        tc_fence_after();
        if (cy == 0 && 2 * i + jy > 0) {  // dV_j / dK_j are re-initialised: the epilogue must be done
          mbar_wait(&sm.dkdv_free, (2 * i + jy - 1) & 1);
          tc_fence_after();
        }
        if (cy == 1 && jy == 0 && i > 0) {  // dQ re-initialised: previous unit's dQ epilogue done
          mbar_wait(&sm.dq_free, (i - 1) & 1);
          tc_fence_after();
        }
        const uint32_t qoff = (cy >> 1) * TILE + (cy & 1) * 8192;  // rows 64c.. of Q / dO
        const uint32_t pcol = tmem + 128 * by;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint32_t pa = pcol + (ks < 2 ? 8 * ks : 32 + 8 * (ks - 2));
          umma_bf16_ts_w(tmem + C_DV, pa, dsc(ado, qoff + ks * 2048, 8192), id_kv, (cy > 0 || ks > 0));
          umma_bf16_ss_w(tmem + C_DK, dsc(ads, cy * TILE + ks * 32, 16),
                       dsc(aq, qoff + ks * 2048, 8192), id_kv, (cy > 0 || ks > 0));
        }
        if (cy & 1) {
          const int t = cy >> 1;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
            umma_bf16_ss_w(tmem + C_DQ + 64 * t, dsc(ads, 2 * t * TILE + ks * 2048, TILE),
                         dsc(ak, jy * TILE + ks * 2048, 8192), id_q, (jy > 0 || ks > 0));
          umma_commit_w(&sm.ds_free[t]);
        }
        if (cy == 3) umma_commit_w(&sm.dkdv_full);
        PROF_MARK(18 + y);
      };
      int i = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
        PROF_MARK(0);
        mbar_wait(&sm.load_full, i & 1);
        PROF_MARK(1);
        tc_fence_after();
        for (int x = 0; x < 8; ++x) {
          const uint32_t gx = 8u * i + x, b = gx & 1;
          const int j = x >> 2, c = x & 3;
          const uint32_t qoff = (c >> 1) * TILE + (c & 1) * 8192;
          // TMEM buffer b was last read by the dV MMA of block gx-2, issued earlier by this thread
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            umma_bf16_ss_w(tmem + 128 * b, dsc(ak, j * TILE + kk * 32, 16),
                         dsc(aq, qoff + kk * 32, 16), id_s, kk > 0);
            umma_bf16_ss_w(tmem + 128 * b + 64, dsc(av, j * TILE + kk * 32, 16),
                         dsc(ado, qoff + kk * 32, 16), id_s, kk > 0);
          }
          umma_commit_w(&sm.sdp_full[b]);
          PROF_MARK(2 + x);
          if (x > 0) grad_mmas(i, x - 1);
        }
        grad_mmas(i, 7);
        umma_commit_w(&sm.dq_full);
        umma_commit_w(&sm.inputs_free);
      }
    }
  } else if (warp < 10) {
    // ------------------------------ P / dS warps ------------------------------
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;      // query columns [32 half, 32 half + 32) of a block
    const int r = quarter * 32 + lane;     // key row within the key half (TMEM lane)
    const uint32_t base = tmem + ((quarter * 32) << 16);
    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const int pb = i & 1;
      mbar_wait(&sm.load_full, i & 1);  // tiles + this unit's vector block
      if (threadIdx.x == 64) PROF_MARK(26);
      const float* lse2 = sm.uvb[pb] + U_LSE2;
      const float* Dv = sm.uvb[pb] + U_DV;
      for (int x = 0; x < 8; ++x) {
        const uint32_t gx = 8u * i + x, b = gx & 1;
        const int j = x >> 2, c = x & 3;
        if ((c & 1) == 0 && 2 * i + j > 0) mbar_wait(&sm.ds_free[c >> 1], (2 * i + j - 1) & 1);
        mbar_wait(&sm.sdp_full[b], (gx >> 1) & 1);
        if (threadIdx.x == 64) PROF_MARK(27 + x);
        tc_fence_after();
        uint32_t vs[32], vd[32];
        tmem_ld_32x32b_x32(base + 128 * b + 32 * half, vs);
        tmem_ld_32x32b_x32(base + 128 * b + 64 + 32 * half, vd);
        tmem_ld_wait();
        const int q0 = 64 * c + 32 * half;
        uint32_t pp[16], pd[16];
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(lse2 + q0 + e);
          const float4 d4 = *reinterpret_cast<const float4*>(Dv + q0 + e);
          const float p0 = ex2(__uint_as_float(vs[e]) * c2 - l4.x);
          const float p1 = ex2(__uint_as_float(vs[e + 1]) * c2 - l4.y);
          const float p2 = ex2(__uint_as_float(vs[e + 2]) * c2 - l4.z);
          const float p3 = ex2(__uint_as_float(vs[e + 3]) * c2 - l4.w);
          pp[e / 2] = pack_bf16(p0, p1);
          pp[e / 2 + 1] = pack_bf16(p2, p3);
          pd[e / 2] = pack_bf16(p0 * (__uint_as_float(vd[e]) - d4.x), p1 * (__uint_as_float(vd[e + 1]) - d4.y));
          pd[e / 2 + 1] = pack_bf16(p2 * (__uint_as_float(vd[e + 2]) - d4.z), p3 * (__uint_as_float(vd[e + 3]) - d4.w));
        }
        // P^T (bf16 pairs) over this warp's own S^T columns; dS^T into smem slot c
        tmem_st_32x32b_x16(base + 128 * b + 32 * half, pp);
        uint8_t* slot = smem + B_DS + c * TILE;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          *reinterpret_cast<uint4*>(slot + sw128(r, 4 * half + k)) =
              make_uint4(pd[4 * k], pd[4 * k + 1], pd[4 * k + 2], pd[4 * k + 3]);
        tmem_st_wait();
        fence_proxy_async();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.pds_full[b]);
        if (threadIdx.x == 64) PROF_MARK(35 + x);
      }
    }
  } else {
    // ------------------------------ helper warpgroup ------------------------------
    const int quarter = warp & 3;
    const int ht = threadIdx.x - 320;     // 0..127
    const int hw = warp - 10;             // helper warp 0..3
    const int r = quarter * 32 + lane;    // TMEM lane for the epilogues
    const uint32_t base = tmem + ((quarter * 32) << 16);
    // one warp writes its 32 rows (64 bf16 each) coalesced: stage row-per-lane in its own 4 KB
    // of the staging tile (128B-swizzled), read back 4 rows x 128 B per instruction
    uint8_t* wstage = smem + B_ST + quarter * 4096;
#define stage_acc(col, coef, vec, sc) bwd_stage_acc(wstage, base + (col), (coef), (vec), (sc), lane)
// colsum partial rows: [frame][9][3D], row block = 4 * (row tile) + quarter, block 8 = token 256
#define flush_rows(row_first, col)                                                                        \
  bwd_flush_rows(wstage, dqkv, (row_first), ld3, (col), lane,                                             \
                 colsum ? colsum + ((int64_t)f * 9 + (((row_first) - row0) >> 5)) * ld3 : nullptr)

    int i = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const int f = u / H, h = u % H;
      const int64_t row0 = (int64_t)f * S;
      const int pb = i & 1;
      const float* uv = sm.uvb[pb];
      const float *q256 = uv + U_Q, *k256 = uv + U_K, *v256 = uv + U_V, *do256 = uv + U_DO;
      mbar_wait(&sm.load_full, i & 1);  // tiles + vector block (uvb[pb] is reloaded only after this
                                        // unit's inputs_free, which this group arrives on below)
      if (ht == 0) PROF_MARK(43);
      if (has_tail) {
        // CUDA-core tail terms (no tensor-core input needed, so they run while the helper would idle):
        //   query 256 against key idx  -> p_row, ds_row;   key 256 against query idx -> p_col, ds_col
        const float* lse2 = uv + U_LSE2;
        const float* Dv = uv + U_DV;
        named_bar(3, 128);  // p_row / ds_row are single-buffered: every helper warp is past unit i-1's (f)
#pragma unroll 1
        for (int jj = 0; jj < 2; ++jj) {
          const int idx = 128 * jj + ht;
          float a[2] = {0.f, 0.f}, dp[2] = {0.f, 0.f};
#pragma unroll 1
          for (int side = 0; side < 2; ++side) {  // 0: K.q256 / V.do256   1: Q.k256 / dO.v256
            const uint8_t* at = smem + (side == 0 ? B_K : B_Q) + jj * TILE;
            const uint8_t* bt = smem + (side == 0 ? B_V : B_DO) + jj * TILE;
            const float* va = side == 0 ? q256 : k256;
            const float* vb = side == 0 ? do256 : v256;
            float sa = 0.f, sb = 0.f;
#pragma unroll 4
            for (int cc = 0; cc < 8; ++cc) {
              const uint4 wa = *reinterpret_cast<const uint4*>(at + sw128(ht, cc));
              const uint4 wb = *reinterpret_cast<const uint4*>(bt + sw128(ht, cc));
              const float4 a0 = *reinterpret_cast<const float4*>(va + 8 * cc);
              const float4 a1 = *reinterpret_cast<const float4*>(va + 8 * cc + 4);
              const float4 b0 = *reinterpret_cast<const float4*>(vb + 8 * cc);
              const float4 b1 = *reinterpret_cast<const float4*>(vb + 8 * cc + 4);
              const float2 x0 = unpack_bf16(wa.x), x1 = unpack_bf16(wa.y), x2 = unpack_bf16(wa.z), x3 = unpack_bf16(wa.w);
              const float2 y0 = unpack_bf16(wb.x), y1 = unpack_bf16(wb.y), y2 = unpack_bf16(wb.z), y3 = unpack_bf16(wb.w);
              sa += x0.x * a0.x + x0.y * a0.y + x1.x * a0.z + x1.y * a0.w + x2.x * a1.x + x2.y * a1.y + x3.x * a1.z + x3.y * a1.w;
              sb += y0.x * b0.x + y0.y * b0.y + y1.x * b0.z + y1.y * b0.w + y2.x * b1.x + y2.y * b1.y + y3.x * b1.z + y3.y * b1.w;
            }
            if (side == 0) { a[0] = sa; dp[0] = sb; } else { a[1] = sa; dp[1] = sb; }
          }
          const float p = ex2(a[0] * c2 - lse2[256]);
          sm.p_row[idx] = p;
          sm.ds_row[idx] = p * (dp[0] - Dv[256]);
          const float pc = ex2(a[1] * c2 - lse2[idx]);
          sm.p_col[pb][idx] = pc;
          sm.ds_col[pb][idx] = pc * (dp[1] - Dv[idx]);
        }
        named_bar(3, 128);
      }
      const int64_t qrow0 = row0 + quarter * 32;  // first of this warp's 32 rows in a 128-row tile
      // ---- (e) dV_0 / dK_0 ----
      mbar_wait(&sm.dkdv_full, (2 * i) & 1);
      if (ht == 0) PROF_MARK(46);
      tc_fence_after();
      {
        const float cp = has_tail ? sm.p_row[r] : 0.f, cd = has_tail ? sm.ds_row[r] : 0.f;
        stage_acc(C_DV, cp, do256, 1.0f);
        flush_rows(qrow0, 2 * D + h * 64);
        stage_acc(C_DK, cd, q256, scale);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_relaxed(&sm.dkdv_free);
        flush_rows(qrow0, D + h * 64);
      }
      if (ht == 0) PROF_MARK(47);
      // ---- (b) row 256: dQ_256 = sum_k ds_row K_k, dK_256 = sum_q ds_col Q_q, dV_256 = sum_q p_col dO_q ----
      if (has_tail) {
        {
          const int dpair = ht & 31, part = ht >> 5;  // 2 dims, 64 rows per part
          const uint32_t chunk = dpair >> 2, within = (dpair & 3) * 4;
          float aq0 = 0.f, aq1 = 0.f, ak0 = 0.f, ak1 = 0.f, av0 = 0.f, av1 = 0.f;
          const uint8_t* kt = smem + B_K + (part >> 1) * TILE;
          const uint8_t* qt = smem + B_Q + (part >> 1) * TILE;
          const uint8_t* gt = smem + B_DO + (part >> 1) * TILE;
          const float* pc = sm.p_col[pb];
          const float* dc = sm.ds_col[pb];
#pragma unroll 4
          for (int k = 0; k < 64; ++k) {
            const int rr = (part & 1) * 64 + k;
            const uint32_t off = sw128(rr, chunk) + within;
            const int idx = (part >> 1) * 128 + rr;
            const float2 fk = unpack_bf16(*reinterpret_cast<const uint32_t*>(kt + off));
            const float2 fq = unpack_bf16(*reinterpret_cast<const uint32_t*>(qt + off));
            const float2 fg = unpack_bf16(*reinterpret_cast<const uint32_t*>(gt + off));
            const float dsr = sm.ds_row[idx], dsc = dc[idx], pcc = pc[idx];
            aq0 += dsr * fk.x; aq1 += dsr * fk.y;
            ak0 += dsc * fq.x; ak1 += dsc * fq.y;
            av0 += pcc * fg.x; av1 += pcc * fg.y;
          }
          sm.tail_red[0][part][2 * dpair] = aq0; sm.tail_red[0][part][2 * dpair + 1] = aq1;
          sm.tail_red[1][part][2 * dpair] = ak0; sm.tail_red[1][part][2 * dpair + 1] = ak1;
          sm.tail_red[2][part][2 * dpair] = av0; sm.tail_red[2][part][2 * dpair + 1] = av1;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.inputs_free);  // this warp is done with the staged tiles
        named_bar(3, 128);
        if (ht == 0) PROF_MARK(45);
        if (ht < 64) {
          const int d = ht;
          const int64_t rr = row0 + 256;
          float sq = uv[U_DC] * k256[d], skk = uv[U_DC] * q256[d], sv = uv[U_PC] * do256[d];
#pragma unroll
          for (int pt = 0; pt < 4; ++pt) {
            sq += sm.tail_red[0][pt][d];
            skk += sm.tail_red[1][pt][d];
            sv += sm.tail_red[2][pt][d];
          }
          const __nv_bfloat16 bq = __float2bfloat16_rn(scale * sq), bk = __float2bfloat16_rn(scale * skk),
                              bv = __float2bfloat16_rn(sv);
          dqkv[rr * ld3 + h * 64 + d] = bq;
          dqkv[rr * ld3 + D + h * 64 + d] = bk;
          dqkv[rr * ld3 + 2 * D + h * 64 + d] = bv;
          if (colsum) {
            float* pr = colsum + ((int64_t)f * 9 + 8) * ld3 + h * 64 + d;
            pr[0] = __bfloat162float(bq);
            pr[D] = __bfloat162float(bk);
            pr[2 * D] = __bfloat162float(bv);
          }
        }
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.inputs_free);
        if (colsum && ht < 64) {  // S = 256: no token 256, its partial row is zero
          float* pr = colsum + ((int64_t)f * 9 + 8) * ld3 + h * 64 + ht;
          pr[0] = 0.f;
          pr[D] = 0.f;
          pr[2 * D] = 0.f;
        }
      }
      if (ht == 0) PROF_MARK(48);
      // ---- (f) dV_1 / dK_1 ----
      mbar_wait(&sm.dkdv_full, (2 * i + 1) & 1);
      if (ht == 0) PROF_MARK(49);
      tc_fence_after();
      {
        const int key = 128 + r;
        const float cp = has_tail ? sm.p_row[key] : 0.f, cd = has_tail ? sm.ds_row[key] : 0.f;
        stage_acc(C_DV, cp, do256, 1.0f);
        flush_rows(qrow0 + 128, 2 * D + h * 64);
        stage_acc(C_DK, cd, q256, scale);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_relaxed(&sm.dkdv_free);
        flush_rows(qrow0 + 128, D + h * 64);
      }
      if (ht == 0) PROF_MARK(50);
      // ---- (g) dQ for query tiles 0, 1 (+ key-256 column term) ----
      mbar_wait(&sm.dq_full, i & 1);
      if (ht == 0) PROF_MARK(51);
      tc_fence_after();
      {
        stage_acc(C_DQ, has_tail ? sm.ds_col[pb][r] : 0.f, k256, scale);
        flush_rows(qrow0, h * 64);
        stage_acc(C_DQ + 64, has_tail ? sm.ds_col[pb][128 + r] : 0.f, k256, scale);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_relaxed(&sm.dq_free);
        flush_rows(qrow0 + 128, h * 64);
      }
      if (ht == 0) PROF_MARK(52);
      (void)hw;
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}
#undef stage_acc
#undef flush_rows

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
  constexpr int NC2 = NC / 2;  // 256-column chunks: lane reads 8 consecutive columns (16-byte loads)
  for (int k0 = 0; k0 < kUvbRows / 8; k0 += 2) {
    float acc[2][NC2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int sidx = c0 + warp * (kUvbRows / 8) + k0 + k;
      if (sidx >= S) continue;
      const int64_t row = f * S + sidx;
#pragma unroll
      for (int c = 0; c < NC2; ++c) {
        const int col = 256 * c + 8 * lane;
        const uint4 hv = __ldg(reinterpret_cast<const uint4*>(out + row * D + col));
        const uint4 lv = __ldg(reinterpret_cast<const uint4*>(out_lo + row * D + col));
        const uint4 gv = __ldg(reinterpret_cast<const uint4*>(dout + row * D + col));
        const uint32_t hh[4] = {hv.x, hv.y, hv.z, hv.w}, ll[4] = {lv.x, lv.y, lv.z, lv.w}, gg[4] = {gv.x, gv.y, gv.z, gv.w};
        float a = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 h2 = unpack_bf16(hh[e]), l2 = unpack_bf16(ll[e]), g2 = unpack_bf16(gg[e]);
          a += (h2.x + l2.x) * g2.x + (h2.y + l2.y) * g2.y;
        }
        acc[k][c] = a;
      }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int sidx = c0 + warp * (kUvbRows / 8) + k0 + k;
      if (sidx >= S) continue;
#pragma unroll
      for (int c = 0; c < NC2; ++c) {
        float a = acc[k][c];
#pragma unroll
        for (int m = 4; m >= 1; m >>= 1) a += __shfl_xor_sync(0xffffffffu, a, m);  // 8 lanes = one head
        const int h = (256 * c + 8 * lane) >> 6;
        if ((lane & 7) == 0) uvb[(f * H + h) * kUvbFloats + U_DV + sidx] = a;
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
  static const int version = [] {
    const char* e = getenv("JZ_SPATIAL_BWD");
    return e ? atoi(e) : 3;
  }();
  if (version != 2)
    return spatial_bwd3_launch(qkv, dout, uvb, frames, S, H, dqkv, colsum_part, reinterpret_cast<cudaStream_t>(s));
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(spatial_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sp::B_SMEM);
  });
  JZ_CUDA_TRY(attr_err);
  const int64_t units = frames * H;
  const int grid = (int)(units < num_sms() ? units : num_sms());
  spatial_bwd_kernel<<<grid, sp::kBwdThreads2, sp::B_SMEM, reinterpret_cast<cudaStream_t>(s)>>>(
      tq, td, uvb, reinterpret_cast<__nv_bfloat16*>(dqkv), colsum_part, (int)frames, S, H);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

#ifdef JZ_ATTN_PROF
extern "C" int jz_attn_prof_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_attn_prof, sizeof(unsigned long long) * 64 * 32) == cudaSuccess ? 0 : -3;
}
#endif
