// K4: causal temporal (inter-frame) attention, forward and backward.
//
// Replaces the temporal sub-layer's attention of st_block (st.py:74-76) =
// multi_head_attention(causal=True) (nn.py:80-110, additive -1e9 mask) over the
// (B, S, T, D) transpose.  Nothing is transposed here: qkv stays in the (b, t, s)
// row order the GEMMs produce, and one CTA gathers the T <= 16 rows of one spatial
// slot (b, s) with cp.async into padded shared memory; warp h owns head h.
//
// Each (b, s, head) problem is a 16x16 causal attention with hd = 64: ~4 FLOP/B,
// HBM-bound and too small for tcgen05's M >= 64 tiles.  The
// per-warp math uses m16n8k16 register MMAs (S = QK^T, O = PV; backward dP, dV,
// dK, dQ) so the instruction count stays far below the memory time; the roofline
// that bounds this kernel is HBM bandwidth.
//
// qkv bf16 [M, 3D] (cols [q | k | v], head h = cols 64h..64h+63 of each),
// out bf16 [M, D], lse f32 [((b*S + s) * H + h) * T + t] (natural log).
#include <stdlib.h>

#include "common.h"
#include "ptx.cuh"

namespace jz {
namespace tp {

constexpr int HD = 64;
constexpr int LDP = 16;  // row pitch (elements) of the per-warp 16x16 P / dS tiles (unpadded: three backward CTAs per SM)

JZ_DEV void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
JZ_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

JZ_DEV void ldsm_x4(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
JZ_DEV void ldsm_x4_t(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}
JZ_DEV void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// A fragment (16 rows x 16 k) from row-major storage (row pitch ld) at column k0
JZ_DEV void load_a(uint32_t (&a)[4], const __nv_bfloat16* base, int ld, int k0) {
  const int L = lane_id();
  ldsm_x4(a, base + ((L & 7) + 8 * ((L >> 3) & 1)) * ld + k0 + 8 * (L >> 4));
}
// A = X^T with X stored [k rows][m cols]: A(m, k) = X[k][m]  (16 x 16)
JZ_DEV void load_a_trans(uint32_t (&a)[4], const __nv_bfloat16* base, int ld) {
  const int L = lane_id();
  ldsm_x4_t(a, base + ((L & 7) + 8 * (L >> 4)) * ld + 8 * ((L >> 3) & 1));
}
// B for n-tiles n0..n0+15 x k16, storage [n rows][k cols]
JZ_DEV void load_b_nk(uint32_t (&b)[4], const __nv_bfloat16* base, int ld, int n0, int k0) {
  const int L = lane_id();
  ldsm_x4(b, base + (n0 + (L & 7) + 8 * (L >> 4)) * ld + k0 + 8 * ((L >> 3) & 1));
}
// B for n-tiles n0..n0+15 x k16, storage [k rows][n cols]
JZ_DEV void load_b_kn(uint32_t (&b)[4], const __nv_bfloat16* base, int ld, int n0) {
  const int L = lane_id();
  ldsm_x4_t(b, base + ((L & 7) + 8 * ((L >> 3) & 1)) * ld + n0 + 8 * (L >> 4));
}

// stage rows t = 0..15 of `src` (row (b*T + t)*S + s) into smem [16][ld]; rows >= T are zeroed
JZ_DEV void stage_rows(__nv_bfloat16* dst, int ld, const __nv_bfloat16* src, int64_t src_ld, int cols, int64_t b,
                       int T, int S, int64_t s) {
  const int c16 = cols / 8;
  for (int i = threadIdx.x; i < 16 * c16; i += blockDim.x) {
    const int t = i / c16, c = i - t * c16;
    if (t < T)
      cp_async16(dst + t * ld + 8 * c, src + ((b * T + t) * S + s) * src_ld + 8 * c);
    else
      *reinterpret_cast<uint4*>(dst + t * ld + 8 * c) = make_uint4(0, 0, 0, 0);
  }
}

JZ_DEV float quad_max(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
JZ_DEV float quad_sum(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v + __shfl_xor_sync(0xffffffffu, v, 2);
}

// acc[n-tile][4] = X Y^T over hd (X rows pitch ldx, Y rows pitch ldy); C layout: rows L/4, L/4+8
JZ_DEV void xyT(float (&acc)[2][4], const __nv_bfloat16* x, int ldx, const __nv_bfloat16* y, int ldy) {
#pragma unroll
  for (int n = 0; n < 2; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[n][e] = 0.f;
#pragma unroll
  for (int kk = 0; kk < HD; kk += 16) {
    uint32_t a[4], b[4];
    load_a(a, x, ldx, kk);
    load_b_nk(b, y, ldy, 0, kk);
    mma16816(acc[0], a, b[0], b[1]);
    mma16816(acc[1], a, b[2], b[3]);
  }
}

// C-layout 16x16 (two n-tiles) -> A fragment
JZ_DEV void c_to_a(uint32_t (&a)[4], const float (&c)[2][4]) {
  a[0] = pack_bf16(c[0][0], c[0][1]);
  a[1] = pack_bf16(c[0][2], c[0][3]);
  a[2] = pack_bf16(c[1][0], c[1][1]);
  a[3] = pack_bf16(c[1][2], c[1][3]);
}

// C-layout 16x16 -> smem tile [16][LDP] (bf16)
JZ_DEV void c_to_smem(__nv_bfloat16* dst, const float (&c)[2][4]) {
  const int L = lane_id();
  const int r0 = L >> 2, cq = 2 * (L & 3);
#pragma unroll
  for (int n = 0; n < 2; ++n) {
    *reinterpret_cast<uint32_t*>(dst + r0 * LDP + 8 * n + cq) = pack_bf16(c[n][0], c[n][1]);
    *reinterpret_cast<uint32_t*>(dst + (r0 + 8) * LDP + 8 * n + cq) = pack_bf16(c[n][2], c[n][3]);
  }
}

// out[16 rows][64] = A(16x16) . B where B rows (k) are stored [k][n] pitch ld; writes rows < T of
// global `dst` (row index (b*T + r)*S + s, pitch dld, column offset col0) scaled by mul (per row)
// `part` (optional): column sums over the T stored rows of the bf16 values, one fp32 partial
// row for this (b, s) at columns col0 .. col0 + 63 (QKV bias gradients, no re-read of dqkv).
JZ_DEV void av_store(const uint32_t (&a)[4], const __nv_bfloat16* bsm, int ld, __nv_bfloat16* dst, int64_t dld,
                     int col0, int64_t b, int T, int S, int64_t s, float mul0, float mul1, float* part = nullptr) {
  const int L = lane_id();
  const int r0 = L >> 2, cq = 2 * (L & 3);
#pragma unroll
  for (int np = 0; np < HD / 16; ++np) {
    uint32_t bb[4];
    load_b_kn(bb, bsm, ld, 16 * np);
    float o0[4] = {0, 0, 0, 0}, o1[4] = {0, 0, 0, 0};
    mma16816(o0, a, bb[0], bb[1]);
    mma16816(o1, a, bb[2], bb[3]);
    const int dcol = col0 + 16 * np + cq;
    const uint32_t w00 = pack_bf16(o0[0] * mul0, o0[1] * mul0), w01 = pack_bf16(o1[0] * mul0, o1[1] * mul0);
    const uint32_t w10 = pack_bf16(o0[2] * mul1, o0[3] * mul1), w11 = pack_bf16(o1[2] * mul1, o1[3] * mul1);
    if (r0 < T) {
      __nv_bfloat16* row = dst + ((b * T + r0) * S + s) * dld + dcol;
      *reinterpret_cast<uint32_t*>(row) = w00;
      *reinterpret_cast<uint32_t*>(row + 8) = w01;
    }
    if (r0 + 8 < T) {
      __nv_bfloat16* row = dst + ((b * T + r0 + 8) * S + s) * dld + dcol;
      *reinterpret_cast<uint32_t*>(row) = w10;
      *reinterpret_cast<uint32_t*>(row + 8) = w11;
    }
    if (part != nullptr) {
      float2 c0 = r0 < T ? unpack_bf16(w00) : make_float2(0.f, 0.f);
      float2 c1 = r0 < T ? unpack_bf16(w01) : make_float2(0.f, 0.f);
      if (r0 + 8 < T) {
        const float2 e0 = unpack_bf16(w10), e1 = unpack_bf16(w11);
        c0.x += e0.x; c0.y += e0.y; c1.x += e1.x; c1.y += e1.y;
      }
#pragma unroll
      for (int m = 4; m <= 16; m <<= 1) {  // sum over the 8 row groups (lanes with equal L & 3)
        c0.x += __shfl_xor_sync(0xffffffffu, c0.x, m);
        c0.y += __shfl_xor_sync(0xffffffffu, c0.y, m);
        c1.x += __shfl_xor_sync(0xffffffffu, c1.x, m);
        c1.y += __shfl_xor_sync(0xffffffffu, c1.y, m);
      }
      if (r0 == 0) {
        *reinterpret_cast<float2*>(part + dcol) = c0;
        *reinterpret_cast<float2*>(part + dcol + 8) = c1;
      }
    }
  }
}

// out[16][64] = A . B (as av_store) kept in registers: o[np][0..3] = n-tile 2np, o[np][4..7] = 2np + 1
JZ_DEV void av_frag(const uint32_t (&a)[4], const __nv_bfloat16* bsm, int ld, float (&o)[HD / 16][8]) {
#pragma unroll
  for (int np = 0; np < HD / 16; ++np) {
    uint32_t bb[4];
    load_b_kn(bb, bsm, ld, 16 * np);
#pragma unroll
    for (int e = 0; e < 8; ++e) o[np][e] = 0.f;
    float o0[4] = {0, 0, 0, 0}, o1[4] = {0, 0, 0, 0};
    mma16816(o0, a, bb[0], bb[1]);
    mma16816(o1, a, bb[2], bb[3]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      o[np][e] = o0[e];
      o[np][4 + e] = o1[e];
    }
  }
}

// fragment -> bf16 smem tile [16][ld] at columns col0..col0+63 (rows r0: * mul0, r0 + 8: * mul1)
JZ_DEV void frag_to_smem(const float (&o)[HD / 16][8], __nv_bfloat16* dst, int ld, int col0, float mul0, float mul1) {
  const int L = lane_id();
  const int r0 = L >> 2, cq = 2 * (L & 3);
#pragma unroll
  for (int np = 0; np < HD / 16; ++np) {
    const int c = col0 + 16 * np + cq;
    *reinterpret_cast<uint32_t*>(dst + r0 * ld + c) = pack_bf16(o[np][0] * mul0, o[np][1] * mul0);
    *reinterpret_cast<uint32_t*>(dst + r0 * ld + c + 8) = pack_bf16(o[np][4] * mul0, o[np][5] * mul0);
    *reinterpret_cast<uint32_t*>(dst + (r0 + 8) * ld + c) = pack_bf16(o[np][2] * mul1, o[np][3] * mul1);
    *reinterpret_cast<uint32_t*>(dst + (r0 + 8) * ld + c + 8) = pack_bf16(o[np][6] * mul1, o[np][7] * mul1);
  }
}

}  // namespace tp

using namespace tp;

__global__ void __launch_bounds__(512) temporal_fwd_kernel(const __nv_bfloat16* __restrict__ qkv, int T, int S, int H,
                                                           __nv_bfloat16* __restrict__ out, float* __restrict__ lse,
                                                           float scale) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int D = H * HD;
  const int ld = 3 * D + 8;
  const int64_t bs = blockIdx.x;
  const int64_t b = bs / S, s = bs - b * S;
  __nv_bfloat16* sq = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  stage_rows(sq, ld, qkv, 3 * D, 3 * D, b, T, S, s);
  cp_async_wait_all();
  __syncthreads();
  const int h = warp_id(), L = lane_id();
  float sc[2][4];
  xyT(sc, sq + h * HD, ld, sq + D + h * HD, ld);
  const int r0 = L >> 2, cq = 2 * (L & 3);
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (int n = 0; n < 2; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int row = r0 + 8 * (e >> 1), col = 8 * n + cq + (e & 1);
      const float x = col <= row ? sc[n][e] * scale : -INFINITY;
      sc[n][e] = x;
      if (e < 2) m0 = fmaxf(m0, x); else m1 = fmaxf(m1, x);
    }
  m0 = quad_max(m0);
  m1 = quad_max(m1);
  float l0 = 0.f, l1 = 0.f;
#pragma unroll
  for (int n = 0; n < 2; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float p = __expf(sc[n][e] - (e < 2 ? m0 : m1));
      sc[n][e] = p;
      if (e < 2) l0 += p; else l1 += p;
    }
  l0 = quad_sum(l0);
  l1 = quad_sum(l1);
  uint32_t pa[4];
  c_to_a(pa, sc);
  float o[HD / 16][8];
  av_frag(pa, sq + 2 * D + h * HD, ld, o);
  __syncwarp();  // this head's q columns are consumed: O overwrites them in place
  frag_to_smem(o, sq, ld, h * HD, 1.0f / l0, 1.0f / l1);
  if ((L & 3) == 0) {
    float* lp = lse + (bs * H + h) * T;
    if (r0 < T) lp[r0] = m0 + logf(l0);
    if (r0 + 8 < T) lp[r0 + 8] = m1 + logf(l1);
  }
  __syncthreads();
  const int c16 = D / 8;  // coalesced write-out of the T token rows
  for (int i = threadIdx.x; i < T * c16; i += blockDim.x) {
    const int t = i / c16, c = i - t * c16;
    *reinterpret_cast<uint4*>(out + ((b * T + t) * S + s) * D + 8 * c) = *reinterpret_cast<const uint4*>(sq + t * ld + 8 * c);
  }
}

__global__ void __launch_bounds__(512) temporal_bwd_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                           const __nv_bfloat16* __restrict__ o,
                                                           const __nv_bfloat16* __restrict__ dout,
                                                           const float* __restrict__ lse, int T, int S, int H,
                                                           __nv_bfloat16* __restrict__ dqkv, float scale,
                                                           float* __restrict__ colsum) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int D = H * HD;
  const int ldq = 3 * D + 8, ldo = D + 8;
  const int64_t bs = blockIdx.x;
  const int64_t b = bs / S, s = bs - b * S;
  __nv_bfloat16* sq = reinterpret_cast<__nv_bfloat16*>(smem_raw);
  __nv_bfloat16* sdo = sq + 16 * ldq;
  __nv_bfloat16* sp_all = sdo + 16 * ldo;
  stage_rows(sq, ldq, qkv, 3 * D, 3 * D, b, T, S, s);
  stage_rows(sdo, ldo, dout, D, D, b, T, S, s);
  cp_async_wait_all();
  __syncthreads();
  const int h = warp_id(), L = lane_id();
  __nv_bfloat16* sP = sp_all + h * 2 * 16 * LDP;
  __nv_bfloat16* sdS = sP + 16 * LDP;
  const __nv_bfloat16* q = sq + h * HD;
  const __nv_bfloat16* k = sq + D + h * HD;
  const __nv_bfloat16* v = sq + 2 * D + h * HD;
  const __nv_bfloat16* dog = sdo + h * HD;
  const int r0 = L >> 2, cq = 2 * (L & 3);
  const float* lp = lse + (bs * H + h) * T;
  const float L0 = r0 < T ? lp[r0] : 0.f, L1 = r0 + 8 < T ? lp[r0 + 8] : 0.f;
  float P[2][4], dS[2][4];
  xyT(P, q, ldq, k, ldq);
  xyT(dS, dog, ldo, v, ldq);
  // Delta_t = sum_j P_tj dP_tj from the fp32 registers (= dO_t . O_t in exact arithmetic): no O
  // read, and dP - Delta does not cancel against the bf16 rounding of a stored O
  float D0 = 0.f, D1 = 0.f;
#pragma unroll
  for (int n = 0; n < 2; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int row = r0 + 8 * (e >> 1), col = 8 * n + cq + (e & 1);
      const float p = (col <= row && row < T) ? __expf(P[n][e] * scale - (e < 2 ? L0 : L1)) : 0.f;
      P[n][e] = p;
      if (e < 2) D0 += p * dS[n][e]; else D1 += p * dS[n][e];
    }
  D0 = quad_sum(D0);
  D1 = quad_sum(D1);
#pragma unroll
  for (int n = 0; n < 2; ++n)
#pragma unroll
    for (int e = 0; e < 4; ++e) dS[n][e] = P[n][e] * (dS[n][e] - (e < 2 ? D0 : D1));
  c_to_smem(sP, P);
  c_to_smem(sdS, dS);
  __syncwarp();
  // dQ = scale * dS K      (A = dS from registers, B = K stored [j][d])
  uint32_t a[4];
  float oq[HD / 16][8], ok[HD / 16][8], ov[HD / 16][8];
  c_to_a(a, dS);
  av_frag(a, k, ldq, oq);          // dQ = scale * dS K
  load_a_trans(a, sdS, LDP);
  av_frag(a, q, ldq, ok);          // dK = scale * dS^T Q
  load_a_trans(a, sP, LDP);
  av_frag(a, dog, ldo, ov);        // dV = P^T dO
  __syncwarp();  // this warp's q/k/v columns are consumed: its gradients overwrite them in place
  frag_to_smem(oq, sq, ldq, h * HD, scale, scale);
  frag_to_smem(ok, sq, ldq, D + h * HD, scale, scale);
  frag_to_smem(ov, sq, ldq, 2 * D + h * HD, 1.0f, 1.0f);
  __syncthreads();
  // coalesced write-out of the T token rows (3 KB contiguous each)
  const int c16 = 3 * D / 8;
  for (int i = threadIdx.x; i < T * c16; i += blockDim.x) {
    const int t = i / c16, c = i - t * c16;
    *reinterpret_cast<uint4*>(dqkv + ((b * T + t) * S + s) * (3 * D) + 8 * c) =
        *reinterpret_cast<const uint4*>(sq + t * ldq + 8 * c);
  }
  if (colsum) {  // QKV bias-gradient partial row of this (b, s): column sums over its T rows
    float* part = colsum + bs * (3 * D);
    for (int c2 = threadIdx.x; c2 < 3 * D / 2; c2 += blockDim.x) {
      float s0 = 0.f, s1 = 0.f;
      for (int t = 0; t < T; ++t) {
        const float2 f = unpack_bf16(*reinterpret_cast<const uint32_t*>(sq + t * ldq + 2 * c2));
        s0 += f.x;
        s1 += f.y;
      }
      *reinterpret_cast<float2*>(part + 2 * c2) = make_float2(s0, s1);
    }
  }
}

// ---------------------------------------------------------------------------
// Row-tile attention over L <= 16 * NT rows of one slot, causal or not (NT = 1, 2).
//
// The same (b, t, s) addressing serves two sub-layers:
//  - spatial attention of small frames (st.py:73, causal=False), S_sp <= 32: the reference's
//    patch-16 presets (S = 16 / 17), the MAE tokenizer (S = 16) and the ST-DiT (S = N + 2 = 18,
//    diffusion.py:164-180). Launched with B := frames, T := S_sp, S := 1, so a slot's rows are
//    the frame's contiguous tokens and lse lands as [frame][H][S_sp], the K3 layout;
//  - causal temporal attention with 16 < T <= 32 (st.py:74-76).
// One CTA per (slot, group of up to 4 heads); per warp (= head): query tile qt against all NT
// key tiles in registers (m16n8k16), P / dS
// tiles staged per warp in shared memory for the transposed dK / dV products. The backward
// forms Delta = sum_j P_ij dP_ij from its fp32 registers, as the T <= 16 kernel does (the forward
// output is not read). Tiles wholly above the causal
// diagonal are computed and masked (at most one per warp).
// ---------------------------------------------------------------------------
namespace tp {

// stage rows t = 0..R-1 (zero rows >= T), as stage_rows
JZ_DEV void stage_rows_n(__nv_bfloat16* dst, int ld, int R, const __nv_bfloat16* src, int64_t src_ld, int cols,
                         int64_t b, int T, int S, int64_t s) {
  const int c16 = cols / 8;
  for (int i = threadIdx.x; i < R * c16; i += blockDim.x) {
    const int t = i / c16, c = i - t * c16;
    if (t < T)
      cp_async16(dst + t * ld + 8 * c, src + ((b * T + t) * S + s) * src_ld + 8 * c);
    else
      *reinterpret_cast<uint4*>(dst + t * ld + 8 * c) = make_uint4(0, 0, 0, 0);
  }
}

// o += A . B (B stored [k][n] pitch ld), o as av_frag
JZ_DEV void av_acc(const uint32_t (&a)[4], const __nv_bfloat16* bsm, int ld, float (&o)[HD / 16][8]) {
#pragma unroll
  for (int np = 0; np < HD / 16; ++np) {
    uint32_t bb[4];
    load_b_kn(bb, bsm, ld, 16 * np);
    float o0[4] = {o[np][0], o[np][1], o[np][2], o[np][3]}, o1[4] = {o[np][4], o[np][5], o[np][6], o[np][7]};
    mma16816(o0, a, bb[0], bb[1]);
    mma16816(o1, a, bb[2], bb[3]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      o[np][e] = o0[e];
      o[np][4 + e] = o1[e];
    }
  }
}

JZ_DEV void zero_frag(float (&o)[HD / 16][8]) {
#pragma unroll
  for (int np = 0; np < HD / 16; ++np)
#pragma unroll
    for (int e = 0; e < 8; ++e) o[np][e] = 0.f;
}

// C-layout 16x16 -> bf16 smem tile (pitch ld)
JZ_DEV void c_to_smem_ld(__nv_bfloat16* dst, int ld, const float (&c)[2][4]) {
  const int L = lane_id();
  const int r0 = L >> 2, cq = 2 * (L & 3);
#pragma unroll
  for (int n = 0; n < 2; ++n) {
    *reinterpret_cast<uint32_t*>(dst + r0 * ld + 8 * n + cq) = pack_bf16(c[n][0], c[n][1]);
    *reinterpret_cast<uint32_t*>(dst + (r0 + 8) * ld + 8 * n + cq) = pack_bf16(c[n][2], c[n][3]);
  }
}

}  // namespace tp

template <int NT>
__global__ void __launch_bounds__(512) rowtile_fwd_kernel(const __nv_bfloat16* __restrict__ qkv, int T, int S, int H,
                                                          int causal, __nv_bfloat16* __restrict__ out,
                                                          float* __restrict__ lse, float scale) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  constexpr int R = 16 * NT;
  const int D = H * HD;
  const int hpc = blockDim.x / 32, h0 = blockIdx.y * hpc;  // this CTA's heads h0 .. h0 + hpc - 1
  const int Dl = hpc * HD, ld = 3 * Dl + 8;
  const int64_t bs = blockIdx.x;
  const int64_t b = bs / S, s = bs - b * S;
  __nv_bfloat16* sq = reinterpret_cast<__nv_bfloat16*>(smem_raw);  // [R][q | k | v of the CTA's heads]
#pragma unroll
  for (int part = 0; part < 3; ++part)
    stage_rows_n(sq + part * Dl, ld, R, qkv + part * D + h0 * HD, 3 * D, Dl, b, T, S, s);
  cp_async_wait_all();
  __syncthreads();
  const int w = warp_id(), h = h0 + w, L = lane_id();
  const int r0 = L >> 2, cq = 2 * (L & 3);
  float* lp = lse + (bs * H + h) * T;
#pragma unroll
  for (int qt = 0; qt < NT; ++qt) {
    float sc[NT][2][4];
#pragma unroll
    for (int kt = 0; kt < NT; ++kt) xyT(sc[kt], sq + 16 * qt * ld + w * HD, ld, sq + 16 * kt * ld + Dl + w * HD, ld);
    float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
    for (int kt = 0; kt < NT; ++kt)
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = 16 * qt + r0 + 8 * (e >> 1), col = 16 * kt + 8 * n + cq + (e & 1);
          const bool ok = col < T && (!causal || col <= row);
          const float x = ok ? sc[kt][n][e] * scale : -INFINITY;
          sc[kt][n][e] = x;
          if (e < 2) m0 = fmaxf(m0, x); else m1 = fmaxf(m1, x);
        }
    m0 = quad_max(m0);
    m1 = quad_max(m1);
    float l0 = 0.f, l1 = 0.f;
#pragma unroll
    for (int kt = 0; kt < NT; ++kt)
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p = __expf(sc[kt][n][e] - (e < 2 ? m0 : m1));
          sc[kt][n][e] = p;
          if (e < 2) l0 += p; else l1 += p;
        }
    l0 = quad_sum(l0);
    l1 = quad_sum(l1);
    float o[HD / 16][8];
    zero_frag(o);
#pragma unroll
    for (int kt = 0; kt < NT; ++kt) {
      uint32_t pa[4];
      c_to_a(pa, sc[kt]);
      av_acc(pa, sq + 16 * kt * ld + 2 * Dl + w * HD, ld, o);
    }
    __syncwarp();  // this head's q rows of tile qt are consumed: O overwrites them in place
    frag_to_smem(o, sq + 16 * qt * ld, ld, w * HD, 1.0f / l0, 1.0f / l1);
    if ((L & 3) == 0) {
      const int ra = 16 * qt + r0;
      if (ra < T) lp[ra] = m0 + logf(l0);
      if (ra + 8 < T) lp[ra + 8] = m1 + logf(l1);
    }
  }
  __syncthreads();
  const int c16 = Dl / 8;
  for (int i = threadIdx.x; i < T * c16; i += blockDim.x) {
    const int t = i / c16, c = i - t * c16;
    *reinterpret_cast<uint4*>(out + ((b * T + t) * S + s) * D + h0 * HD + 8 * c) =
        *reinterpret_cast<const uint4*>(sq + t * ld + 8 * c);
  }
}

template <int NT>
__global__ void __launch_bounds__(512) rowtile_bwd_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                          const __nv_bfloat16* __restrict__ o,
                                                          const __nv_bfloat16* __restrict__ dout,
                                                          const float* __restrict__ lse, int T, int S, int H,
                                                          int causal, __nv_bfloat16* __restrict__ dqkv, float scale,
                                                          float* __restrict__ colsum) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  constexpr int R = 16 * NT, LDR = R + 8;
  const int D = H * HD;
  const int hpc = blockDim.x / 32, h0 = blockIdx.y * hpc;  // this CTA's heads h0 .. h0 + hpc - 1
  const int Dl = hpc * HD;
  const int ldq = 3 * Dl + 8, ldo = Dl + 8;
  const int64_t bs = blockIdx.x;
  const int64_t b = bs / S, s = bs - b * S;
  __nv_bfloat16* sq = reinterpret_cast<__nv_bfloat16*>(smem_raw);  // [R][q | k | v of the CTA's heads]
  __nv_bfloat16* so = sq + R * ldq;  // dQ staging (each warp its own head's columns)
  __nv_bfloat16* sdo = so + R * ldo;
  __nv_bfloat16* sp_all = sdo + R * ldo;
#pragma unroll
  for (int part = 0; part < 3; ++part)
    stage_rows_n(sq + part * Dl, ldq, R, qkv + part * D + h0 * HD, 3 * D, Dl, b, T, S, s);
  stage_rows_n(sdo, ldo, R, dout + h0 * HD, D, Dl, b, T, S, s);
  cp_async_wait_all();
  __syncthreads();
  const int w = warp_id(), h = h0 + w, L = lane_id();
  __nv_bfloat16* sP = sp_all + w * 2 * R * LDR;
  __nv_bfloat16* sdS = sP + R * LDR;
  const __nv_bfloat16* q = sq + w * HD;
  const __nv_bfloat16* k = sq + Dl + w * HD;
  const __nv_bfloat16* v = sq + 2 * Dl + w * HD;
  const __nv_bfloat16* dog = sdo + w * HD;
  const int r0 = L >> 2, cq = 2 * (L & 3);
  const float* lp = lse + (bs * H + h) * T;
#pragma unroll
  for (int qt = 0; qt < NT; ++qt) {
    const int ra = 16 * qt + r0;
    const float L0 = ra < T ? lp[ra] : 0.f, L1 = ra + 8 < T ? lp[ra + 8] : 0.f;
    float P[NT][2][4], dS[NT][2][4];
#pragma unroll
    for (int kt = 0; kt < NT; ++kt) {
      xyT(P[kt], q + 16 * qt * ldq, ldq, k + 16 * kt * ldq, ldq);
      xyT(dS[kt], dog + 16 * qt * ldo, ldo, v + 16 * kt * ldq, ldq);
    }
    float D0 = 0.f, D1 = 0.f;
#pragma unroll
    for (int kt = 0; kt < NT; ++kt)
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = ra + 8 * (e >> 1), col = 16 * kt + 8 * n + cq + (e & 1);
          const bool ok = row < T && col < T && (!causal || col <= row);
          const float p = ok ? __expf(P[kt][n][e] * scale - (e < 2 ? L0 : L1)) : 0.f;
          P[kt][n][e] = p;
          if (e < 2) D0 += p * dS[kt][n][e]; else D1 += p * dS[kt][n][e];
        }
    // Delta over the whole key row from the fp32 registers (no O read; no bf16-O cancellation)
    D0 = quad_sum(D0);
    D1 = quad_sum(D1);
#pragma unroll
    for (int kt = 0; kt < NT; ++kt)
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int e = 0; e < 4; ++e) dS[kt][n][e] = P[kt][n][e] * (dS[kt][n][e] - (e < 2 ? D0 : D1));
    float oq[HD / 16][8];
    zero_frag(oq);
#pragma unroll
    for (int kt = 0; kt < NT; ++kt) {
      c_to_smem_ld(sP + 16 * qt * LDR + 16 * kt, LDR, P[kt]);
      c_to_smem_ld(sdS + 16 * qt * LDR + 16 * kt, LDR, dS[kt]);
      uint32_t a[4];
      c_to_a(a, dS[kt]);
      av_acc(a, k + 16 * kt * ldq, ldq, oq);  // dQ_qt += dS_(qt,kt) K_kt
    }
    frag_to_smem(oq, so + 16 * qt * ldo, ldo, w * HD, scale, scale);
  }
  __syncwarp();
  // dK_kt = scale * sum_qt dS_(qt,kt)^T Q_qt, dV_kt = sum_qt P_(qt,kt)^T dO_qt; K and V are consumed
#pragma unroll
  for (int kt = 0; kt < NT; ++kt) {
    float gk[HD / 16][8], gv[HD / 16][8];
    zero_frag(gk);
    zero_frag(gv);
#pragma unroll
    for (int qt = 0; qt < NT; ++qt) {
      uint32_t a[4];
      load_a_trans(a, sdS + 16 * qt * LDR + 16 * kt, LDR);
      av_acc(a, q + 16 * qt * ldq, ldq, gk);
      load_a_trans(a, sP + 16 * qt * LDR + 16 * kt, LDR);
      av_acc(a, dog + 16 * qt * ldo, ldo, gv);
    }
    frag_to_smem(gk, sq + 16 * kt * ldq, ldq, Dl + w * HD, scale, scale);
    frag_to_smem(gv, sq + 16 * kt * ldq, ldq, 2 * Dl + w * HD, 1.0f, 1.0f);
  }
  __syncthreads();
  // coalesced write-out of the T rows, the CTA's head columns of each of dq | dk | dv:
  // dQ from the O buffer, dK | dV from the qkv buffer (local column c -> global part * D + h0 * HD)
  const int c16 = 3 * Dl / 8, cq16 = Dl / 8;
  for (int i = threadIdx.x; i < T * c16; i += blockDim.x) {
    const int t = i / c16, c = i - t * c16;
    const int part = c / cq16;
    const __nv_bfloat16* src = part == 0 ? so + t * ldo + 8 * c : sq + t * ldq + 8 * c;
    *reinterpret_cast<uint4*>(dqkv + ((b * T + t) * S + s) * (3 * D) + part * D + h0 * HD + 8 * (c - part * cq16)) =
        *reinterpret_cast<const uint4*>(src);
  }
  if (colsum) {
    float* prow = colsum + bs * (3 * D);
    for (int c2 = threadIdx.x; c2 < 3 * Dl / 2; c2 += blockDim.x) {
      const int part = (2 * c2) / Dl;
      float s0 = 0.f, s1 = 0.f;
      for (int t = 0; t < T; ++t) {
        const __nv_bfloat16* src = part == 0 ? so + t * ldo + 2 * c2 : sq + t * ldq + 2 * c2;
        const float2 f = unpack_bf16(*reinterpret_cast<const uint32_t*>(src));
        s0 += f.x;
        s1 += f.y;
      }
      *reinterpret_cast<float2*>(prow + part * D + h0 * HD + 2 * c2 - part * Dl) = make_float2(s0, s1);
    }
  }
}

constexpr size_t kRowTileSmemMax = 227 * 1024;

template <int NT>
static int launch_rowtile(bool bwd, const void* qkv, const void* o, const void* dout, float* lse, int64_t B, int T,
                          int S, int H, int causal, void* out, cudaStream_t st, float* colsum) {
  constexpr int R = 16 * NT;
  const float scale = 0.125f;
  const int64_t BS = B * S;
  if (BS == 0) return JZ_OK;
  // heads per CTA: the largest divisor of H up to 4, so a frame (slot) spreads over H / hpc CTAs
  // and several CTAs share an SM (fwd 4, bwd 2 at R = 32): loads of one overlap another's math
  int hpc = 1;
  for (int c = 4; c >= 1; --c)
    if (H % c == 0) { hpc = c; break; }
  const int Dl = hpc * HD;
  const int threads = 32 * hpc;
  const dim3 grid((unsigned)BS, (unsigned)(H / hpc));
  if (!bwd) {
    const size_t smem = (size_t)R * (3 * Dl + 8) * 2;
    JZ_CHECK_ARG(smem <= kRowTileSmemMax, "row-tile attention: %d rows x %d heads exceed shared memory", T, H);
    JZ_CUDA_TRY(cudaFuncSetAttribute(rowtile_fwd_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    rowtile_fwd_kernel<NT><<<grid, threads, smem, st>>>(reinterpret_cast<const __nv_bfloat16*>(qkv), T, S, H,
                                                                causal, reinterpret_cast<__nv_bfloat16*>(out), lse,
                                                                scale);
  } else {
    const size_t smem = (size_t)R * (3 * Dl + 8) * 2 + (size_t)2 * R * (Dl + 8) * 2 + (size_t)hpc * 2 * R * (R + 8) * 2;
    JZ_CHECK_ARG(smem <= kRowTileSmemMax, "row-tile attention backward: %d rows x %d heads exceed shared memory", T,
                 H);
    JZ_CUDA_TRY(cudaFuncSetAttribute(rowtile_bwd_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    rowtile_bwd_kernel<NT><<<grid, threads, smem, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(qkv), reinterpret_cast<const __nv_bfloat16*>(o),
        reinterpret_cast<const __nv_bfloat16*>(dout), lse, T, S, H, causal, reinterpret_cast<__nv_bfloat16*>(out),
        scale, colsum);
  }
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

static int dispatch_rowtile(bool bwd, const void* qkv, const void* o, const void* dout, float* lse, int64_t B, int T,
                            int S, int H, int causal, void* out, cudaStream_t st, float* colsum) {
  JZ_CHECK_ARG(H >= 1 && H <= 16, "row-tile attention: heads %d unsupported (<= 16)", H);
  JZ_CHECK_ARG(T >= 1 && T <= 32, "row-tile attention: %d rows unsupported (<= 32)", T);
  if (T <= 16) return launch_rowtile<1>(bwd, qkv, o, dout, lse, B, T, S, H, causal, out, st, colsum);
  return launch_rowtile<2>(bwd, qkv, o, dout, lse, B, T, S, H, causal, out, st, colsum);
}

int temporal_tc_fwd(const void* qkv, int64_t B, int T, int S, int H, void* out, float* lse, cudaStream_t st);
int temporal_tc_bwd(const void* qkv, const void* dout, const float* lse, int64_t B, int T, int S, int H, void* dqkv,
                    float* colsum, cudaStream_t st);
int64_t temporal_tc_colsum_parts(int64_t B, int S, int H);

// T <= 16 runs the tcgen05 kernels (attn_temporal_tc.cu) unless JZ_TEMPORAL_TC=0 selects the
// register-tile (mma.sync) kernels below; 16 < T <= 32 runs the row-tile kernels.
static bool temporal_tc_enabled() {
  static const bool on = [] {
    const char* e = getenv("JZ_TEMPORAL_TC");
    return !(e && e[0] == '0');
  }();
  return on;
}

static int dispatch_temporal(bool bwd, const void* qkv, const void* o, const void* dout, float* lse, int64_t B,
                             int T, int S, int H, void* out, cudaStream_t st, float* colsum = nullptr) {
  JZ_CHECK_ARG(H >= 1 && H <= 16, "temporal attention: heads %d unsupported (<= 16)", H);
  JZ_CHECK_ARG(T >= 1 && T <= 32, "temporal attention: T=%d unsupported (<= 32)", T);
  if (T > 16) return dispatch_rowtile(bwd, qkv, o, dout, lse, B, T, S, H, 1, out, st, colsum);
  if (temporal_tc_enabled() && B * S > 0)
    return bwd ? temporal_tc_bwd(qkv, dout, lse, B, T, S, H, out, colsum, st)
               : temporal_tc_fwd(qkv, B, T, S, H, out, lse, st);
  const float scale = 0.125f;  // 1/sqrt(64)
  const int64_t BS = B * S;
  if (BS == 0) return JZ_OK;
  const int D = H * HD;
  const int threads = 32 * H;
  if (!bwd) {
    const size_t smem = (size_t)16 * (3 * D + 8) * 2;
    JZ_CUDA_TRY(cudaFuncSetAttribute(temporal_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    temporal_fwd_kernel<<<(unsigned)BS, threads, smem, st>>>(reinterpret_cast<const __nv_bfloat16*>(qkv), T, S, H,
                                                             reinterpret_cast<__nv_bfloat16*>(out), lse, scale);
  } else {
    const size_t smem = (size_t)16 * (3 * D + 8) * 2 + (size_t)16 * (D + 8) * 2 + (size_t)H * 2 * 16 * LDP * 2;
    JZ_CUDA_TRY(cudaFuncSetAttribute(temporal_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    temporal_bwd_kernel<<<(unsigned)BS, threads, smem, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(qkv), reinterpret_cast<const __nv_bfloat16*>(o),
        reinterpret_cast<const __nv_bfloat16*>(dout), lse, T, S, H, reinterpret_cast<__nv_bfloat16*>(out), scale,
        colsum);
  }
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

}  // namespace jz

using namespace jz;

extern "C" int jz_attn_temporal_fwd(const void* qkv, int64_t B, int T, int S, int H, int head_dim, void* out,
                                    float* lse, jz_stream_t s) {
  JZ_CHECK_ARG(head_dim == 64, "temporal attention: head_dim %d unsupported (64)", head_dim);
  return dispatch_temporal(false, qkv, nullptr, nullptr, lse, B, T, S, H, out, reinterpret_cast<cudaStream_t>(s));
}

extern "C" int64_t jz_attn_temporal_colsum_parts(int64_t B, int S) { return B * S; }

extern "C" int64_t jz_attn_temporal_colsum_parts_t(int64_t B, int S, int T, int H) {
  if (T <= 16 && temporal_tc_enabled()) return temporal_tc_colsum_parts(B, S, H);  // one partial row per CTA
  return B * S;
}

extern "C" int jz_attn_temporal_bwd(const void* qkv, const void* out, const void* dout, const float* lse,
                                    int64_t B, int T, int S, int H, int head_dim, void* dqkv, float* colsum_part,
                                    jz_stream_t s) {
  JZ_CHECK_ARG(head_dim == 64, "temporal attention: head_dim %d unsupported (64)", head_dim);
  return dispatch_temporal(true, qkv, out, dout, const_cast<float*>(lse), B, T, S, H, dqkv,
                           reinterpret_cast<cudaStream_t>(s), colsum_part);
}

extern "C" int jz_attn_spatial_small_fwd(const void* qkv, int64_t frames, int S, int H, int head_dim, void* out,
                                         float* lse, jz_stream_t s) {
  JZ_CHECK_ARG(head_dim == 64, "small spatial attention: head_dim %d unsupported (64)", head_dim);
  return dispatch_rowtile(false, qkv, nullptr, nullptr, lse, frames, S, 1, H, 0, out,
                          reinterpret_cast<cudaStream_t>(s), nullptr);
}

extern "C" int jz_attn_spatial_small_bwd(const void* qkv, const void* out, const void* dout, const float* lse,
                                         int64_t frames, int S, int H, int head_dim, void* dqkv, float* colsum_part,
                                         jz_stream_t s) {
  JZ_CHECK_ARG(head_dim == 64, "small spatial attention: head_dim %d unsupported (64)", head_dim);
  return dispatch_rowtile(true, qkv, out, dout, const_cast<float*>(lse), frames, S, 1, H, 0, dqkv,
                          reinterpret_cast<cudaStream_t>(s), colsum_part);
}
