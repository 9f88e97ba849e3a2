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
#include "common.h"
#include "ptx.cuh"

namespace jz {

namespace sp {

constexpr int kThreads = 256;   // backward: w0 TMA, w1 MMA, w2-5 P/dS + epilogues, w6-7 tail row
constexpr int kFwdThreads = 384;  // forward: w0 TMA, w1 MMA, w2-5 tile 0, w6-9 tile 1, w10-11 tail row
constexpr int kBwdThreads = 384;  // backward: w0 TMA, w1 MMA, w2-9 two P/dS warpgroups, w10-11 tail
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
  float tail_o[64];
  float tail_red[4];
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
                       const __grid_constant__ CUtensorMap tm_o, const __grid_constant__ CUtensorMap tm_o32,
                       const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ out,
                       float* __restrict__ out_f32, float* __restrict__ lse, int frames, int S, int H) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  FwdSmallSmem& sm = *reinterpret_cast<FwdSmallSmem*>(smem + F_END);
  const int D = H * 64;
  const int warp = warp_id(), lane = lane_id();
  const int units = frames * H;
  const bool has_tail = S > 256;
  const float c2 = 0.125f * 1.4426950408889634f;  // scale * log2(e)

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm);
    tma_prefetch_desc(&tm_row);
    tma_prefetch_desc(&tm_o);
    if (out_f32) tma_prefetch_desc(&tm_o32);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(&sm.qk_full, 1); mbar_init(&sm.v_full, 1);
    // Q/K and V smem (+ rows 256) are released by the MMA commit, both softmax warpgroups and the tail
    mbar_init(&sm.qk_free, 1 + 256 + (has_tail ? 64 : 0)); mbar_init(&sm.v_free, 1 + 256 + (has_tail ? 64 : 0));
    for (int t = 0; t < 2; ++t) {
      mbar_init(&sm.s_full[t], 1); mbar_init(&sm.p_full[t], 128);
      mbar_init(&sm.o_full[t], 1); mbar_init(&sm.tmem_free[t], 128);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem_base);
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

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
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, 256, false, false);
      constexpr uint32_t idesc_o = idesc_bf16_f32(128, 64, false, true);
      const uint32_t q_addr = smem_u32(smem + F_Q), k_addr = smem_u32(smem + F_K), v_addr = smem_u32(smem + F_V);
      int i = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
        const uint32_t par = i & 1;
        mbar_wait(&sm.qk_full, par);
        for (int t = 0; t < 2; ++t) {
          mbar_wait(&sm.tmem_free[t], par ^ 1);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16_ss(tmem + 256 * t, sdesc_sw128(q_addr + t * TILE + kk * 32, 16, 1024),
                         sdesc_sw128(k_addr + kk * 32, 16, 1024), idesc_s, kk > 0);
          umma_commit(&sm.s_full[t]);
        }
        umma_commit(&sm.qk_free);
        mbar_wait(&sm.v_full, par);
        for (int t = 0; t < 2; ++t) {
          mbar_wait(&sm.p_full[t], par);
          tc_fence_after();
          const uint32_t p_addr = smem_u32(smem + (t ? F_P1 : F_P0));
#pragma unroll
          for (int ks = 0; ks < 16; ++ks)
            umma_bf16_ss(tmem + 256 * t, sdesc_sw128(p_addr + (ks >> 2) * TILE + (ks & 3) * 32, 16, 1024),
                         sdesc_sw128(v_addr + ks * 2048, 8192, 1024), idesc_o, ks > 0);
          umma_commit(&sm.o_full[t]);
        }
        umma_commit(&sm.v_free);
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
      const int64_t grow = row0 + 128 * t + r;
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
        // keys 32c..32c+31 -> atom (c/2), 16B chunks (c%2)*4 .. +3
        uint8_t* atom = pbuf + (c >> 1) * TILE;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t chunk = (c & 1) * 4 + q;
          *reinterpret_cast<uint4*>(atom + sw128(r, chunk)) =
              make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
      }
      const float plast = has_tail ? ex2(s_last * c2 - mb) : 0.f;
      sum += plast;
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&sm.p_full[t]);
      // O epilogue: stage O (bf16 atom + two fp32 atoms) in this tile's P buffer, TMA-store it
      mbar_wait(&sm.o_full[t], par);
      tc_fence_after();
      const float inv = 1.0f / sum;
      const uint8_t* vrow = sm.vrow;
      uint8_t* o16 = pbuf;             // [128 rows][64 bf16], 128B swizzle
      uint8_t* o32 = pbuf + TILE;      // two [128 rows][32 f32] atoms
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(taddr + 32 * c, v);
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
        if (out_f32) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<float4*>(o32 + c * TILE + sw128(r, q)) =
                make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
        }
      }
      mbar_arrive(&sm.v_free);  // done with value row 256
      fence_proxy_async();
      named_bar(1 + t, 128);
      if (wtid == 0) {
        tma_store_2d(&tm_o, o16, h * 64, (int)(row0 + 128 * t));
        if (out_f32) {
          tma_store_2d(&tm_o32, o32, h * 64, (int)(row0 + 128 * t));
          tma_store_2d(&tm_o32, o32 + TILE, h * 64 + 32, (int)(row0 + 128 * t));
        }
        bulk_commit();
      }
      lse[((int64_t)f * H + h) * S + 128 * t + r] = mx * 0.125f + logf(sum);
      tc_fence_before();
      mbar_arrive(&sm.tmem_free[t]);
    }
  } else if (has_tail) {
    // tail warps: query row 256 on CUDA cores, reading K/V from the staged smem tiles
    const int tid = threadIdx.x - 320;  // 0..63
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
      for (int k = tid; k < 256; k += 64) {
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
      named_bar(3, 64);
      mx = fmaxf(sm.tail_red[0], sm.tail_red[1]);
      const float mb = mx * c2;
      float sum = 0.f;
      for (int k = tid; k < S; k += 64) {
        const float p = ex2(sm.tail_s[k] * c2 - mb);
        sm.tail_s[k] = p;
        sum += p;
      }
      sum = warp_sum(sum);
      if (lane == 0) sm.tail_red[2 + warp - 10] = sum;
      named_bar(3, 64);
      sum = sm.tail_red[2] + sm.tail_red[3];
      // o[d] for d = 2*(tid&31) .. +1, keys split in two halves by warp
      const int dpair = tid & 31, half = tid >> 5;
      float o0 = 0.f, o1 = 0.f;
      mbar_wait(&sm.v_full, par);
      const uint32_t chunk = dpair >> 2, within = (dpair & 3) * 4;
#pragma unroll 8
      for (int k = half * 128; k < half * 128 + 128; ++k) {
        const uint8_t* vt = smem + F_V + (k >> 7) * TILE;
        const float2 v = unpack_bf16(*reinterpret_cast<const uint32_t*>(vt + sw128(k & 127, chunk) + within));
        const float p = sm.tail_s[k];
        o0 += p * v.x;
        o1 += p * v.y;
      }
      mbar_arrive(&sm.v_free);
      if (half == 1) {
        const float2 vl = unpack_bf16(*reinterpret_cast<const uint32_t*>(sm.vrow + 4 * dpair));
        o0 += sm.tail_s[256] * vl.x;
        o1 += sm.tail_s[256] * vl.y;
        sm.tail_o[2 * dpair] = o0;
        sm.tail_o[2 * dpair + 1] = o1;
      }
      named_bar(3, 64);
      if (half == 0) {
        o0 = (o0 + sm.tail_o[2 * dpair]) / sum;
        o1 = (o1 + sm.tail_o[2 * dpair + 1]) / sum;
        *reinterpret_cast<uint32_t*>(out + (row0 + 256) * D + h * 64 + 2 * dpair) = pack_bf16(o0, o1);
        if (out_f32) *reinterpret_cast<float2*>(out_f32 + (row0 + 256) * D + h * 64 + 2 * dpair) = make_float2(o0, o1);
        if (tid == 0) lse[((int64_t)f * H + h) * S + 256] = mx * 0.125f + logf(sum);
      }
      named_bar(3, 64);
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
                                   float* out_f32, float* lse, jz_stream_t s) {
  JZ_CHECK_ARG(head_dim == 64, "spatial attention: head_dim %d unsupported (64)", head_dim);
  JZ_CHECK_ARG(S == 256 || S == 257, "spatial attention: sequence length %d unsupported (256 or 257)", S);
  JZ_CHECK_ARG(frames >= 1 && frames * H < (1ll << 31), "spatial attention: frames");
  const int D = H * 64;
  CUtensorMap tm, tm_row, tm_o, tm_o32;
  int rc = make_tmap_2d_bf16(&tm, qkv, 3 * D, frames * S, 3 * D, 64, 128);
  if (!rc) rc = make_tmap_2d(&tm_row, qkv, 2, 3 * D, frames * S, 3 * D, 64, 1, /*swizzle128=*/false);
  if (!rc) rc = make_tmap_2d_bf16(&tm_o, out, D, frames * S, D, 64, 128);
  if (!rc && out_f32) rc = make_tmap_2d(&tm_o32, out_f32, 4, D, frames * S, D, 32, 128);
  if (!out_f32) tm_o32 = tm_o;
  if (rc) return rc;
  static bool attr_done = false;
  if (!attr_done) {
    JZ_CUDA_TRY(cudaFuncSetAttribute(spatial_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM));
    attr_done = true;
  }
  const int64_t units = frames * H;
  const int grid = (int)(units < num_sms() ? units : num_sms());
  spatial_fwd_kernel<<<grid, kFwdThreads, F_SMEM, reinterpret_cast<cudaStream_t>(s)>>>(
      tm, tm_row, tm_o, tm_o32, reinterpret_cast<const __nv_bfloat16*>(qkv), reinterpret_cast<__nv_bfloat16*>(out),
      out_f32, lse, (int)frames, S, H);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

// ============================================================================
// Backward.  Per (frame, head), in the transposed ("S^T") formulation: for each
// key half j (128 keys) and query tile t (128 queries)
//   S^T  = K_j Q_t^T,  dP^T = V_j dO_t^T                         (TMEM, 2 x 128 cols)
//   P^T  = exp(S^T*scale - lse),  dS^T = P^T (dP^T - Dq)            (CUDA cores -> smem bf16)
//   dV_j += P^T dO_t,  dK_j += dS^T Q_t,  dQ_t += dS K_j           (TMEM accumulators)
// The dS tile written K-major over queries for dK is read MN-major as the A operand
// of dQ, so one smem copy serves both products.  Query/key 256 terms on CUDA cores.
// ============================================================================
#ifdef JZ_ATTN_PROF
__device__ unsigned long long g_attn_prof[64 * 32];
#define PROF_MARK(slot)                                                                   \
  do {                                                                                    \
    if (blockIdx.x == 0 && i < 32) g_attn_prof[i * 32 + (slot)] = clock64();             \
  } while (0)
#else
#define PROF_MARK(slot) \
  do {                  \
  } while (0)
#endif
namespace jz {
namespace sp {
constexpr int B_Q = 0;
constexpr int B_K = B_Q + 2 * TILE;
constexpr int B_V = B_K + 2 * TILE;
constexpr int B_DO = B_V + 2 * TILE;
constexpr int B_PT = B_DO + 2 * TILE;   // [2 query atoms][128 key rows][128 B]
constexpr int B_DST = B_PT + 2 * TILE;
constexpr int B_END = B_DST + 2 * TILE;  // 196608

struct BwdSmallSmem {
  uint64_t load_full, inputs_free, sdp_full, pds_full, pds_free, dkdv_full, dkdv_free, dq_full, dq_free,
      tail_ready;
  uint32_t tmem_base;
  float lse2[260];
  float Dv[260];
  float p_col[260], ds_col[260];  // key 256 column over queries 0..256
  float p_row[260], ds_row[260];  // query 256 row over keys 0..256
  float q256[64], do256[64], k256[64], v256[64];
  float tail_red[3][64][2];
};
constexpr int B_SMEM = B_END + 1024 + (int)sizeof(BwdSmallSmem) + 64;
}  // namespace sp

__global__ void __launch_bounds__(kBwdThreads, 1)
    spatial_bwd_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                       const __nv_bfloat16* __restrict__ qkv, const float* __restrict__ out,
                       const __nv_bfloat16* __restrict__ dout, const float* __restrict__ lse,
                       __nv_bfloat16* __restrict__ dqkv, int frames, int S, int H) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  BwdSmallSmem& sm = *reinterpret_cast<BwdSmallSmem*>(smem + B_END);
  const int D = H * 64;
  const int warp = warp_id(), lane = lane_id();
  const int units = frames * H;
  const bool has_tail = S > 256;
  const float scale = 0.125f;
  const float c2 = 0.125f * 1.4426950408889634f;
  constexpr uint32_t C_ST = 0, C_DPT = 128, C_DV = 256, C_DK = 320, C_DQ = 384;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tm_qkv);
    tma_prefetch_desc(&tm_do);
  }
  if (warp == 1 && lane == 0) {
    mbar_init(&sm.load_full, 1);
    mbar_init(&sm.inputs_free, has_tail ? 65 : 1);
    mbar_init(&sm.sdp_full, 1);
    mbar_init(&sm.pds_full, 256);
    mbar_init(&sm.pds_free, 1);
    mbar_init(&sm.dkdv_full, 1);
    mbar_init(&sm.dkdv_free, 256);
    mbar_init(&sm.dq_full, 1);
    mbar_init(&sm.dq_free, 256);
    mbar_init(&sm.tail_ready, 64);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&sm.tmem_base);
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;

  if (warp == 0) {
    if (lane == 0) {
      int i = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
        const int f = u / H, h = u % H;
        const int row0 = f * S;
        mbar_wait(&sm.inputs_free, (i & 1) ^ 1);
        mbar_arrive_expect_tx(&sm.load_full, 8 * TILE);
        for (int t = 0; t < 2; ++t) {
          tma_load_2d(smem + B_Q + t * TILE, &tm_qkv, &sm.load_full, h * 64, row0 + 128 * t);
          tma_load_2d(smem + B_K + t * TILE, &tm_qkv, &sm.load_full, D + h * 64, row0 + 128 * t);
          tma_load_2d(smem + B_V + t * TILE, &tm_qkv, &sm.load_full, 2 * D + h * 64, row0 + 128 * t);
          tma_load_2d(smem + B_DO + t * TILE, &tm_do, &sm.load_full, h * 64, row0 + 128 * t);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t id_s = idesc_bf16_f32(128, 128, false, false);
      constexpr uint32_t id_kv = idesc_bf16_f32(128, 64, false, true);
      constexpr uint32_t id_q = idesc_bf16_f32(128, 64, true, true);
      const uint32_t aq = smem_u32(smem + B_Q), ak = smem_u32(smem + B_K), av = smem_u32(smem + B_V),
                     ado = smem_u32(smem + B_DO), apt = smem_u32(smem + B_PT), adst = smem_u32(smem + B_DST);
      int i = 0;
      uint32_t g = 0;  // running (j,t) iteration counter
      for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
        mbar_wait(&sm.load_full, i & 1);
        for (int j = 0; j < 2; ++j) {
          for (int t = 0; t < 2; ++t, ++g) {
            if (t == 0) {
              // C_DV/C_DK (and at j == 0 also C_DQ) are overwritten: wait for their readers
              if (2 * i + j > 0) mbar_wait(&sm.dkdv_free, (2 * i + j - 1) & 1);
              if (j == 0 && i > 0) mbar_wait(&sm.dq_free, (i - 1) & 1);
              tc_fence_after();
            }
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              umma_bf16_ss(tmem + C_ST, sdesc_sw128(ak + j * TILE + kk * 32, 16, 1024),
                           sdesc_sw128(aq + t * TILE + kk * 32, 16, 1024), id_s, kk > 0);
              umma_bf16_ss(tmem + C_DPT, sdesc_sw128(av + j * TILE + kk * 32, 16, 1024),
                           sdesc_sw128(ado + t * TILE + kk * 32, 16, 1024), id_s, kk > 0);
            }
            umma_commit(&sm.sdp_full);
            mbar_wait(&sm.pds_full, g & 1);
            tc_fence_after();
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              const uint32_t aoff = (ks >> 2) * TILE + (ks & 3) * 32;
              umma_bf16_ss(tmem + C_DV, sdesc_sw128(apt + aoff, 16, 1024),
                           sdesc_sw128(ado + t * TILE + ks * 2048, 8192, 1024), id_kv, (t > 0 || ks > 0));
              umma_bf16_ss(tmem + C_DK, sdesc_sw128(adst + aoff, 16, 1024),
                           sdesc_sw128(aq + t * TILE + ks * 2048, 8192, 1024), id_kv, (t > 0 || ks > 0));
              umma_bf16_ss(tmem + C_DQ + 64 * t, sdesc_sw128(adst + ks * 2048, 16384, 1024),
                           sdesc_sw128(ak + j * TILE + ks * 2048, 8192, 1024), id_q, (j > 0 || ks > 0));
            }
            umma_commit(&sm.pds_free);
            if (t == 1) umma_commit(&sm.dkdv_full);
          }
        }
        umma_commit(&sm.dq_full);
        umma_commit(&sm.inputs_free);
      }
    }
  } else {
    const bool main_role = warp < 10;
    const int g = (warp - 2) >> 2;      // main: warpgroup 0/1
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;  // main: TMEM lane / row within a 128 tile
    const int wtid = threadIdx.x - 64;  // main: 0..255
    const int tid = threadIdx.x - 320;  // tail: 0..63
    int i = 0;
    uint32_t gi = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++i) {
      const int f = u / H, h = u % H;
      const int64_t row0 = (int64_t)f * S;
      const int64_t ld3 = 3 * (int64_t)D;
      // ---- prologue P1: vectors of row 256 + lse ----
      if (threadIdx.x == 64) PROF_MARK(0);
      named_bar(1, 320);
      if (threadIdx.x == 64) PROF_MARK(22);
      if (main_role) {
        if (wtid < 64) {
          const int d = wtid;
          const int64_t rr = row0 + 256;
          sm.q256[d] = has_tail ? __bfloat162float(qkv[rr * ld3 + h * 64 + d]) : 0.f;
          sm.k256[d] = has_tail ? __bfloat162float(qkv[rr * ld3 + D + h * 64 + d]) : 0.f;
          sm.v256[d] = has_tail ? __bfloat162float(qkv[rr * ld3 + 2 * D + h * 64 + d]) : 0.f;
          sm.do256[d] = has_tail ? __bfloat162float(dout[rr * D + h * 64 + d]) : 0.f;
        }
      } else {
        for (int q = tid; q < S; q += 64) sm.lse2[q] = lse[((int64_t)f * H + h) * S + q] * 1.4426950408889634f;
      }
      if (threadIdx.x == 64) PROF_MARK(23);
      named_bar(1, 320);
      if (threadIdx.x == 64) PROF_MARK(24);
      // ---- prologue P2: D_q = dO_q . O_q, key-256 column ----
      if (main_role) {
        const int q = 128 * g + r;
        const int64_t rr = row0 + q;
        // fp32 O row from HBM (all 16 loads in flight), dO and Q rows from the staged smem tiles
        const float4* op = reinterpret_cast<const float4*>(out + rr * D + h * 64);
        float4 ov[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) ov[c] = __ldg(op + c);
        mbar_wait(&sm.load_full, i & 1);
        const uint8_t* gt = smem + B_DO + g * TILE;
        const uint8_t* qt = smem + B_Q + g * TILE;
        float dd = 0.f, sk = 0.f, dpv = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 wg = *reinterpret_cast<const uint4*>(gt + sw128(r, c));
          const uint4 wq = *reinterpret_cast<const uint4*>(qt + sw128(r, c));
          const uint32_t ag[4] = {wg.x, wg.y, wg.z, wg.w}, aqv[4] = {wq.x, wq.y, wq.z, wq.w};
          const float of[8] = {ov[2 * c].x, ov[2 * c].y, ov[2 * c].z, ov[2 * c].w,
                               ov[2 * c + 1].x, ov[2 * c + 1].y, ov[2 * c + 1].z, ov[2 * c + 1].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 fg = unpack_bf16(ag[e]), fq = unpack_bf16(aqv[e]);
            const int d = 8 * c + 2 * e;
            dd += of[2 * e] * fg.x + of[2 * e + 1] * fg.y;
            sk += fq.x * sm.k256[d] + fq.y * sm.k256[d + 1];
            dpv += fg.x * sm.v256[d] + fg.y * sm.v256[d + 1];
          }
        }
        sm.Dv[q] = dd;
        if (threadIdx.x == 64) PROF_MARK(25);
        if (has_tail) {
          const float p = ex2(sk * c2 - sm.lse2[q]);
          sm.p_col[q] = p;
          sm.ds_col[q] = p * (dpv - dd);
        }
      } else if (has_tail) {
        // row 256: the 64 tail threads each take one head dim, reduce over both warps
        const int64_t rr = row0 + 256;
        const int d = tid;
        float dd = out[rr * D + h * 64 + d] * sm.do256[d];
        float sk = sm.q256[d] * sm.k256[d];
        float dpv = sm.do256[d] * sm.v256[d];
        dd = warp_sum(dd);
        sk = warp_sum(sk);
        dpv = warp_sum(dpv);
        if (lane == 0) {
          sm.tail_red[0][warp - 10][0] = dd;
          sm.tail_red[1][warp - 10][0] = sk;
          sm.tail_red[2][warp - 10][0] = dpv;
        }
        named_bar(2, 64);
        if (tid == 0) {
          const float ddt = sm.tail_red[0][0][0] + sm.tail_red[0][1][0];
          const float skt = sm.tail_red[1][0][0] + sm.tail_red[1][1][0];
          const float dpt = sm.tail_red[2][0][0] + sm.tail_red[2][1][0];
          sm.Dv[256] = ddt;
          const float p = ex2(skt * c2 - sm.lse2[256]);
          sm.p_col[256] = p;
          sm.ds_col[256] = p * (dpt - ddt);
        }
      }
      named_bar(1, 320);
      if (threadIdx.x == 64) PROF_MARK(1);

      if (main_role) {
        const uint32_t base = tmem + ((quarter * 32) << 16);
        for (int j = 0; j < 2; ++j) {
          for (int t = 0; t < 2; ++t, ++gi) {
            mbar_wait(&sm.sdp_full, gi & 1);
            if (threadIdx.x == 64) PROF_MARK(2 + 4 * (2 * j + t));
            tc_fence_after();
            if (gi > 0) mbar_wait(&sm.pds_free, (gi - 1) & 1);
            if (threadIdx.x == 64) PROF_MARK(3 + 4 * (2 * j + t));
            // warpgroup g computes query columns [64g, 64g + 64) of this (j, t) tile -> atom g
            uint8_t* at_p = smem + B_PT + g * TILE;
            uint8_t* at_d = smem + B_DST + g * TILE;
#pragma unroll 1
            for (int cc = 0; cc < 4; ++cc) {
              const int col = 64 * g + 16 * cc;
              uint32_t vs[16], vd[16];
              tmem_ld_32x32b_x16(base + C_ST + col, vs);
              tmem_ld_32x32b_x16(base + C_DPT + col, vd);
              tmem_ld_wait();
              uint32_t pp[8], pd[8];
#pragma unroll
              for (int e = 0; e < 16; e += 2) {
                const int q = 128 * t + col + e;
                const float p0 = ex2(__uint_as_float(vs[e]) * c2 - sm.lse2[q]);
                const float p1 = ex2(__uint_as_float(vs[e + 1]) * c2 - sm.lse2[q + 1]);
                pp[e / 2] = pack_bf16(p0, p1);
                pd[e / 2] = pack_bf16(p0 * (__uint_as_float(vd[e]) - sm.Dv[q]),
                                      p1 * (__uint_as_float(vd[e + 1]) - sm.Dv[q + 1]));
              }
#pragma unroll
              for (int qq = 0; qq < 2; ++qq) {
                const uint32_t off = sw128(r, 2 * cc + qq);
                *reinterpret_cast<uint4*>(at_p + off) = make_uint4(pp[4 * qq], pp[4 * qq + 1], pp[4 * qq + 2], pp[4 * qq + 3]);
                *reinterpret_cast<uint4*>(at_d + off) = make_uint4(pd[4 * qq], pd[4 * qq + 1], pd[4 * qq + 2], pd[4 * qq + 3]);
              }
            }
            fence_proxy_async();
            tc_fence_before();
            mbar_arrive(&sm.pds_full);
            if (threadIdx.x == 64) PROF_MARK(4 + 4 * (2 * j + t));
            if (t == 1) {
              if (j == 0 && has_tail) mbar_wait(&sm.tail_ready, i & 1);
              mbar_wait(&sm.dkdv_full, (2 * i + j) & 1);
              tc_fence_after();
              // warpgroup 0 writes dV, warpgroup 1 writes dK (key rows 128j + r)
              const int key = 128 * j + r;
              const int64_t rr = row0 + key;
              const float coef = has_tail ? (g == 0 ? sm.p_row[key] : sm.ds_row[key]) : 0.f;
              const float* vec = g == 0 ? sm.do256 : sm.q256;
              const float sc = g == 0 ? 1.0f : scale;
              uint4* dst = reinterpret_cast<uint4*>(dqkv + rr * ld3 + (g == 0 ? 2 * D : D) + h * 64);
#pragma unroll 1
              for (int c = 0; c < 2; ++c) {
                uint32_t vv[32];
                tmem_ld_32x32b_x32(base + (g == 0 ? C_DV : C_DK) + 32 * c, vv);
                tmem_ld_wait();
                float ov[32];
#pragma unroll
                for (int e = 0; e < 32; ++e) ov[e] = sc * (__uint_as_float(vv[e]) + coef * vec[32 * c + e]);
#pragma unroll
                for (int qq = 0; qq < 4; ++qq)
                  dst[4 * c + qq] = make_uint4(pack_bf16(ov[8 * qq], ov[8 * qq + 1]), pack_bf16(ov[8 * qq + 2], ov[8 * qq + 3]),
                                               pack_bf16(ov[8 * qq + 4], ov[8 * qq + 5]), pack_bf16(ov[8 * qq + 6], ov[8 * qq + 7]));
              }
              tc_fence_before();
              mbar_arrive(&sm.dkdv_free);
              if (threadIdx.x == 64) PROF_MARK(5 + 4 * (2 * j + t));
            }
          }
        }
        // dQ epilogue: warpgroup g -> query tile g
        mbar_wait(&sm.dq_full, i & 1);
        if (threadIdx.x == 64) PROF_MARK(18);
        tc_fence_after();
        {
          const int q = 128 * g + r;
          const int64_t rr = row0 + q;
          const float dsc = has_tail ? sm.ds_col[q] : 0.f;
          uint4* dq_dst = reinterpret_cast<uint4*>(dqkv + rr * ld3 + h * 64);
#pragma unroll 1
          for (int c = 0; c < 2; ++c) {
            uint32_t vq[32];
            tmem_ld_32x32b_x32(base + C_DQ + 64 * g + 32 * c, vq);
            tmem_ld_wait();
            float oq[32];
#pragma unroll
            for (int e = 0; e < 32; ++e) oq[e] = scale * (__uint_as_float(vq[e]) + dsc * sm.k256[32 * c + e]);
#pragma unroll
            for (int qq = 0; qq < 4; ++qq)
              dq_dst[4 * c + qq] = make_uint4(pack_bf16(oq[8 * qq], oq[8 * qq + 1]), pack_bf16(oq[8 * qq + 2], oq[8 * qq + 3]),
                                              pack_bf16(oq[8 * qq + 4], oq[8 * qq + 5]), pack_bf16(oq[8 * qq + 6], oq[8 * qq + 7]));
          }
        }
        tc_fence_before();
        mbar_arrive(&sm.dq_free);
        if (threadIdx.x == 64) PROF_MARK(19);
      } else if (has_tail) {
        // ---- tail: query 256 row and key 256 column ----
        mbar_wait(&sm.load_full, i & 1);
        for (int k = tid; k < 256; k += 64) {
          const uint8_t* kt = smem + B_K + (k >> 7) * TILE;
          const uint8_t* vt = smem + B_V + (k >> 7) * TILE;
          float a = 0.f, dp = 0.f;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint4 wk = *reinterpret_cast<const uint4*>(kt + sw128(k & 127, c));
            const uint4 wv = *reinterpret_cast<const uint4*>(vt + sw128(k & 127, c));
            const uint32_t ak[4] = {wk.x, wk.y, wk.z, wk.w}, av[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 fk = unpack_bf16(ak[e]), fv = unpack_bf16(av[e]);
              const int d = 8 * c + 2 * e;
              a += sm.q256[d] * fk.x + sm.q256[d + 1] * fk.y;
              dp += sm.do256[d] * fv.x + sm.do256[d + 1] * fv.y;
            }
          }
          const float p = ex2(a * c2 - sm.lse2[256]);
          sm.p_row[k] = p;
          sm.ds_row[k] = p * (dp - sm.Dv[256]);
        }
        if (tid == 0) {
          sm.p_row[256] = sm.p_col[256];
          sm.ds_row[256] = sm.ds_col[256];
        }
        mbar_arrive(&sm.tail_ready);
        if (tid == 0) PROF_MARK(20);
        named_bar(2, 64);
        const int dpair = tid & 31, half = tid >> 5;
        const uint32_t chunk = dpair >> 2, within = (dpair & 3) * 4;
        float aq0 = 0.f, aq1 = 0.f, ak0 = 0.f, ak1 = 0.f, av0 = 0.f, av1 = 0.f;
        const uint8_t* kt = smem + B_K + half * TILE;
        const uint8_t* qt = smem + B_Q + half * TILE;
        const uint8_t* gt = smem + B_DO + half * TILE;
#pragma unroll 4
        for (int rr = 0; rr < 128; ++rr) {
          const uint32_t off = sw128(rr, chunk) + within;
          const int idx = half * 128 + rr;
          const float2 fk = unpack_bf16(*reinterpret_cast<const uint32_t*>(kt + off));
          const float2 fq = unpack_bf16(*reinterpret_cast<const uint32_t*>(qt + off));
          const float2 fg = unpack_bf16(*reinterpret_cast<const uint32_t*>(gt + off));
          const float dsr = sm.ds_row[idx], dsc = sm.ds_col[idx], pc = sm.p_col[idx];
          aq0 += dsr * fk.x; aq1 += dsr * fk.y;   // dQ_256 over keys
          ak0 += dsc * fq.x; ak1 += dsc * fq.y;   // dK_256 over queries
          av0 += pc * fg.x; av1 += pc * fg.y;     // dV_256 over queries
        }
        mbar_arrive(&sm.inputs_free);
        if (tid == 0) PROF_MARK(21);
        if (half == 1) {
          const int d = 2 * dpair;
          aq0 += sm.ds_row[256] * sm.k256[d]; aq1 += sm.ds_row[256] * sm.k256[d + 1];
          ak0 += sm.ds_col[256] * sm.q256[d]; ak1 += sm.ds_col[256] * sm.q256[d + 1];
          av0 += sm.p_col[256] * sm.do256[d]; av1 += sm.p_col[256] * sm.do256[d + 1];
          sm.tail_red[0][dpair][0] = aq0; sm.tail_red[0][dpair][1] = aq1;
          sm.tail_red[1][dpair][0] = ak0; sm.tail_red[1][dpair][1] = ak1;
          sm.tail_red[2][dpair][0] = av0; sm.tail_red[2][dpair][1] = av1;
        }
        named_bar(2, 64);
        if (half == 0) {
          const int64_t rr = row0 + 256;
          const int d = 2 * dpair;
          aq0 += sm.tail_red[0][dpair][0]; aq1 += sm.tail_red[0][dpair][1];
          ak0 += sm.tail_red[1][dpair][0]; ak1 += sm.tail_red[1][dpair][1];
          av0 += sm.tail_red[2][dpair][0]; av1 += sm.tail_red[2][dpair][1];
          *reinterpret_cast<uint32_t*>(dqkv + rr * ld3 + h * 64 + d) = pack_bf16(scale * aq0, scale * aq1);
          *reinterpret_cast<uint32_t*>(dqkv + rr * ld3 + D + h * 64 + d) = pack_bf16(scale * ak0, scale * ak1);
          *reinterpret_cast<uint32_t*>(dqkv + rr * ld3 + 2 * D + h * 64 + d) = pack_bf16(av0, av1);
        }
        named_bar(2, 64);
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace jz

extern "C" int jz_attn_spatial_bwd(const void* qkv, const float* out_f32, const void* dout, const float* lse,
                                   int64_t frames, int S, int H, int head_dim, void* dqkv, jz_stream_t s) {
  using namespace jz;
  JZ_CHECK_ARG(head_dim == 64, "spatial attention bwd: head_dim %d unsupported (64)", head_dim);
  JZ_CHECK_ARG(S == 256 || S == 257, "spatial attention bwd: sequence length %d unsupported", S);
  const int D = H * 64;
  CUtensorMap tq, td;
  int rc = make_tmap_2d_bf16(&tq, qkv, 3 * D, frames * S, 3 * D, 64, 128);
  if (rc) return rc;
  rc = make_tmap_2d_bf16(&td, dout, D, frames * S, D, 64, 128);
  if (rc) return rc;
  static bool attr_done = false;
  if (!attr_done) {
    JZ_CUDA_TRY(cudaFuncSetAttribute(spatial_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sp::B_SMEM));
    attr_done = true;
  }
  const int64_t units = frames * H;
  const int grid = (int)(units < num_sms() ? units : num_sms());
  spatial_bwd_kernel<<<grid, sp::kBwdThreads, sp::B_SMEM, reinterpret_cast<cudaStream_t>(s)>>>(
      tq, td, reinterpret_cast<const __nv_bfloat16*>(qkv), out_f32,
      reinterpret_cast<const __nv_bfloat16*>(dout), lse, reinterpret_cast<__nv_bfloat16*>(dqkv), (int)frames, S, H);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

#ifdef JZ_ATTN_PROF
extern "C" int jz_attn_prof_read(unsigned long long* host) {
  return cudaMemcpyFromSymbol(host, g_attn_prof, sizeof(unsigned long long) * 64 * 32) == cudaSuccess ? 0 : -3;
}
#endif
