// Autoregressive MaskGIT sampling on device (dynamics.py:156-260):
//   K12 KV-cached last-frame forward: single-frame embedding with per-sample
//       conditioning, temporal attention of the new frame over cached per-layer K/V
//       (exact: spatial attention is intra-frame and temporal attention is causal, so
//       frames < t never change while frame t is refined), cache fill/append
//   K11 MaskGIT sampler step (_sample_with_confidence, dynamics.py:198-217, and the
//       known/confidence update + stable top-n_keep of dynamics.py:185-192):
//       temperature softmax over K codes, inverse-CDF draw with the caller's numpy
//       Philox stream continued on device, confidence of the sampled code, then
//       known positions get +inf and the n_keep best (conf desc, position asc) become known.
#include "common.h"
#include "philox.cuh"
#include "ptx.cuh"

namespace jz {

// ---------------------------------------------------------------------------
// single-frame embedding: x[b, s] for frame index t (pos_temporal row pt_row)
//   s = 0 -> (cond[b] Wa + ba) + ps[0] + pt;  s >= 1 -> (known ? E[tok] : mt) + ps[s] + pt
//   (known == NULL: every token known)
// ---------------------------------------------------------------------------
// One warp per row (8 rows per 256-thread CTA, grid-stride): lane owns float4 columns
// 4 lane + 128 i; the token id / known flag are read once per row by the whole warp.
constexpr int kEmbedRowsPerCta = 8;
__global__ void __launch_bounds__(32 * kEmbedRowsPerCta) embed_frame_kernel(
    const int64_t* __restrict__ tokens, const uint8_t* __restrict__ known, const float* __restrict__ cond,
    const float* __restrict__ E, const float* __restrict__ mt, const float* __restrict__ Wa,
    const float* __restrict__ ba, const float* __restrict__ ps, const float* __restrict__ pt_row,
    const int* __restrict__ dev_t, int64_t rows, int N, int D, int dl, int K, float* __restrict__ x) {
  const int S = N + 1;
  if (dev_t) pt_row += (int64_t)(*dev_t) * D;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * kEmbedRowsPerCta;
  for (int64_t row = (int64_t)blockIdx.x * kEmbedRowsPerCta + (threadIdx.x >> 5); row < rows; row += nw) {
    const int s = (int)(row % S);
    const int64_t b = row / S;
    const float* src = nullptr;
    if (s > 0) {
      const int64_t pos = b * N + (s - 1);
      if (known && !known[pos]) {
        src = mt;
      } else {
        int64_t tok = tokens[pos];
        tok = tok < 0 ? 0 : (tok >= K ? K - 1 : tok);
        src = E + tok * D;
      }
    }
    for (int d = 4 * lane; d < D; d += 128) {
      float4 v;
      if (s == 0) {
        float4 acc = make_float4(0, 0, 0, 0);
        for (int i = 0; i < dl; ++i) {
          const float c = cond[b * dl + i];
          const float4 w = *reinterpret_cast<const float4*>(Wa + (int64_t)i * D + d);
          acc.x += c * w.x; acc.y += c * w.y; acc.z += c * w.z; acc.w += c * w.w;
        }
        const float4 bb = *reinterpret_cast<const float4*>(ba + d);
        v = make_float4(acc.x + bb.x, acc.y + bb.y, acc.z + bb.z, acc.w + bb.w);
      } else {
        v = *reinterpret_cast<const float4*>(src + d);
      }
      const float4 p1 = *reinterpret_cast<const float4*>(ps + (int64_t)s * D + d);
      const float4 p2 = *reinterpret_cast<const float4*>(pt_row + d);
      v.x = (v.x + p1.x) + p2.x; v.y = (v.y + p1.y) + p2.y;
      v.z = (v.z + p1.z) + p2.z; v.w = (v.w + p1.w) + p2.w;
      *reinterpret_cast<float4*>(x + row * D + d) = v;
    }
  }
}

// ---------------------------------------------------------------------------
// temporal attention of frame t over cache[:, 0..t-1] + itself.  One warp per (b, s)
// covering every head: lane l owns dims [16l, 16l+16) (head l/4), so a head's score is a
// 16-wide partial dot reduced over 4 lanes.  cache [B, Tmax, S, 2D] bf16 (k | v).
// append: also write the current k, v into cache[:, t].  Requires D == 512 (8 heads x 64).
// ---------------------------------------------------------------------------
template <int DPL>
JZ_DEV void loadv(const __nv_bfloat16* p, float (&f)[DPL]) {
#pragma unroll
  for (int c = 0; c < DPL / 4; ++c) {
    const uint2 a = reinterpret_cast<const uint2*>(p)[c];
    const float2 x = unpack_bf16(a.x), y = unpack_bf16(a.y);
    f[4 * c] = x.x; f[4 * c + 1] = x.y; f[4 * c + 2] = y.x; f[4 * c + 3] = y.y;
  }
}

// raw bf16 pairs (converted at use: half the registers of an fp32 copy)
template <int DPL>
JZ_DEV void loadraw(const __nv_bfloat16* p, uint32_t (&w)[DPL / 2]) {
#pragma unroll
  for (int c = 0; c < DPL / 4; ++c) {
    const uint2 a = reinterpret_cast<const uint2*>(p)[c];
    w[2 * c] = a.x;
    w[2 * c + 1] = a.y;
  }
}

template <int DPL>
JZ_DEV void storev(__nv_bfloat16* p, const float (&f)[DPL], float scale) {
#pragma unroll
  for (int c = 0; c < DPL / 4; ++c)
    reinterpret_cast<uint2*>(p)[c] = make_uint2(pack_bf16(f[4 * c] * scale, f[4 * c + 1] * scale),
                                                pack_bf16(f[4 * c + 2] * scale, f[4 * c + 3] * scale));
}

template <int DPL>
JZ_DEV void copyv(__nv_bfloat16* dst, const __nv_bfloat16* src) {
#pragma unroll
  for (int c = 0; c < DPL / 4; ++c) reinterpret_cast<uint2*>(dst)[c] = reinterpret_cast<const uint2*>(src)[c];
}

// DPL = head dims per lane: D = 32*DPL, a head (64 dims) spans 64/DPL lanes.
// One warp per (b, s) over all heads; keys/values tau < t come from the cache, tau = t is the
// current frame's own k/v.  Single pass with an online softmax over chunks of 4 time steps: each
// chunk issues its 8 K/V row loads (clamped to a valid row, masked afterwards) before any use,
// and every loop is fully unrolled (t <= 15) so scores and accumulators stay in registers.
template <int DPL>
__global__ void temporal_decode_kernel(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ cache,
                                       int64_t B, int t, const int* __restrict__ dev_t, int Tmax, int S, int append,
                                       __nv_bfloat16* __restrict__ out) {
  constexpr int D = 32 * DPL;
  constexpr int HL = 64 / DPL;  // lanes per head
  if (dev_t) t = *dev_t;
  const int64_t bs = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (bs >= B * S) return;
  const int s = (int)(bs % S);
  const int64_t b = bs / S;
  const __nv_bfloat16* row = qkv + bs * 3 * D;
  const int d0 = DPL * lane;
  float q[DPL], kc[DPL], vc[DPL];
  loadv<DPL>(row + d0, q);
  loadv<DPL>(row + D + d0, kc);
  loadv<DPL>(row + 2 * D + d0, vc);
  const __nv_bfloat16* base = cache + ((b * Tmax) * S + s) * 2 * D + d0;
  const int64_t tstride = (int64_t)S * 2 * D;
  float m = -INFINITY, l = 0.f, o[DPL];
#pragma unroll
  for (int i = 0; i < DPL; ++i) o[i] = 0.f;
#pragma unroll
  for (int c0 = 0; c0 < 16; c0 += 4) {
    if (c0 > t) break;  // warp-uniform
    uint32_t kk[4][DPL / 2], vv[4][DPL / 2];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int tau = c0 + j;
      const int tt = tau < t ? tau : 0;  // row 0 always exists when t > 0; unused otherwise
      if (t > 0) {
        loadraw<DPL>(base + tt * tstride, kk[j]);
        loadraw<DPL>(base + tt * tstride + D, vv[j]);
      }
    }
    float sc[4];
    float cm = m;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int tau = c0 + j;
      float a = 0.f;
#pragma unroll
      for (int i = 0; i < DPL / 2; ++i) {
        const float2 kf = unpack_bf16(kk[j][i]);
        a += q[2 * i] * (tau < t ? kf.x : kc[2 * i]) + q[2 * i + 1] * (tau < t ? kf.y : kc[2 * i + 1]);
      }
#pragma unroll
      for (int off = 1; off < HL; off <<= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
      sc[j] = tau <= t ? a * 0.125f : -INFINITY;
      cm = fmaxf(cm, sc[j]);
    }
    const float corr = __expf(m - cm);  // 0 on the first chunk (m = -inf)
    l *= corr;
#pragma unroll
    for (int i = 0; i < DPL; ++i) o[i] *= corr;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int tau = c0 + j;
      const float p = __expf(sc[j] - cm);
      l += p;
#pragma unroll
      for (int i = 0; i < DPL / 2; ++i) {
        const float2 vf = unpack_bf16(vv[j][i]);
        o[2 * i] += p * (tau < t ? vf.x : vc[2 * i]);
        o[2 * i + 1] += p * (tau < t ? vf.y : vc[2 * i + 1]);
      }
    }
    m = cm;
  }
  storev<DPL>(out + bs * D + d0, o, 1.0f / l);
  if (append) {
    __nv_bfloat16* cw = cache + ((b * Tmax + t) * S + s) * 2 * D + d0;
    copyv<DPL>(cw, row + D + d0);
    copyv<DPL>(cw + D, row + 2 * D + d0);
  }
}

// Same attention with 16-byte coalesced row accesses (D = 256 NV): lane l owns the 8-dim vectors
// at dims [256 v + 8 l, +8) for v < NV, i.e. one 64-dim head slice per vector (head 4 v + l / 8),
// reduced over 8 lanes.  Every warp-wide load instruction reads 512 contiguous bytes of a K or V row
// (the DPL kernel's 8-byte lane accesses at a 32-byte stride touched each sector 4 times).
template <int NV>
__global__ void __launch_bounds__(128, 4) temporal_decode_v_kernel(
    const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ cache, int64_t B, int t,
    const int* __restrict__ dev_t, int Tmax, int S, int append, __nv_bfloat16* __restrict__ out) {
  constexpr int D = 256 * NV;
  constexpr int RV = D / 8;  // 16-byte vectors per D-wide row
  if (dev_t) t = *dev_t;
  const int64_t bs = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (bs >= B * S) return;
  const int s = (int)(bs % S);
  const int64_t b = bs / S;
  const uint4* row = reinterpret_cast<const uint4*>(qkv + bs * 3 * D) + lane;
  float q[NV][8];
  uint4 kc[NV], vc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const uint4 w = row[v * 32];
    const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = unpack_bf16(ww[e]);
      q[v][2 * e] = f.x;
      q[v][2 * e + 1] = f.y;
    }
    kc[v] = row[RV + v * 32];
    vc[v] = row[2 * RV + v * 32];
  }
  const uint4* base = reinterpret_cast<const uint4*>(cache + ((b * Tmax) * S + s) * 2 * D) + lane;
  const int64_t tstride = (int64_t)S * 2 * RV;  // uint4 per cached frame
  float m[NV], l[NV], o[NV][8];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    m[v] = -INFINITY;
    l[v] = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) o[v][i] = 0.f;
  }
#pragma unroll
  for (int c0 = 0; c0 < 16; c0 += 4) {
    if (c0 > t) break;  // warp-uniform
    uint4 kk[4][NV], vv[4][NV];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int tau = c0 + j;
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        if (tau < t) {
          kk[j][v] = base[tau * tstride + v * 32];
          vv[j][v] = base[tau * tstride + RV + v * 32];
        } else if (tau == t) {
          kk[j][v] = kc[v];
          vv[j][v] = vc[v];
        } else {
          kk[j][v] = make_uint4(0, 0, 0, 0);
          vv[j][v] = make_uint4(0, 0, 0, 0);
        }
      }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      float sc[4];
      float cm = m[v];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t ww[4] = {kk[j][v].x, kk[j][v].y, kk[j][v].z, kk[j][v].w};
        float a = 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 kf = unpack_bf16(ww[e]);
          a += q[v][2 * e] * kf.x + q[v][2 * e + 1] * kf.y;
        }
        a += __shfl_xor_sync(0xffffffffu, a, 1);
        a += __shfl_xor_sync(0xffffffffu, a, 2);
        a += __shfl_xor_sync(0xffffffffu, a, 4);
        sc[j] = (c0 + j) <= t ? a * 0.125f : -INFINITY;
        cm = fmaxf(cm, sc[j]);
      }
      const float corr = __expf(m[v] - cm);  // 0 on the first chunk (m = -inf)
      l[v] *= corr;
#pragma unroll
      for (int i = 0; i < 8; ++i) o[v][i] *= corr;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float pj = __expf(sc[j] - cm);
        l[v] += pj;
        const uint32_t ww[4] = {vv[j][v].x, vv[j][v].y, vv[j][v].z, vv[j][v].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 vf = unpack_bf16(ww[e]);
          o[v][2 * e] += pj * vf.x;
          o[v][2 * e + 1] += pj * vf.y;
        }
      }
      m[v] = cm;
    }
  }
  uint4* orow = reinterpret_cast<uint4*>(out + bs * D) + lane;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const float r = 1.0f / l[v];
    orow[v * 32] = make_uint4(pack_bf16(o[v][0] * r, o[v][1] * r), pack_bf16(o[v][2] * r, o[v][3] * r),
                              pack_bf16(o[v][4] * r, o[v][5] * r), pack_bf16(o[v][6] * r, o[v][7] * r));
  }
  if (append) {
    uint4* cw = reinterpret_cast<uint4*>(cache + ((b * Tmax + t) * S + s) * 2 * D) + lane;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      cw[v * 32] = kc[v];
      cw[RV + v * 32] = vc[v];
    }
  }
}

// cache[b, t0 + tau, s, :] = (k | v) of qkv rows (b, tau, s) for tau < T
__global__ void kv_fill_kernel(const __nv_bfloat16* __restrict__ qkv, __nv_bfloat16* __restrict__ cache, int64_t B,
                               int T, int t0, int Tmax, int S, int D) {
  const int64_t rows = B * T * S;
  const int c8 = 2 * D / 8;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rows * c8;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / c8;
    const int c = (int)(e - r * c8);
    const int s = (int)(r % S);
    const int64_t bt = r / S;
    const int tau = (int)(bt % T);
    const int64_t b = bt / T;
    const uint4 w = reinterpret_cast<const uint4*>(qkv + r * 3 * D + D)[c];
    reinterpret_cast<uint4*>(cache + (((b * Tmax + t0 + tau) * S + s) * 2 * D))[c] = w;
  }
}

// ---------------------------------------------------------------------------
// K11a: per (b, n) row of K logits: temperature softmax, inverse-CDF sample with
// u = draw (draw_base + b*N + n) of the Philox state, confidence; then the
// known/cur/conf update.  One warp per row; lane owns K/32 consecutive codes.
// ---------------------------------------------------------------------------
// Per-row sampler math on the lane's PER consecutive logits v (scaled in place).
template <int PER>
JZ_DEV void sample_row(float (&v)[PER], int64_t r, int lane, int K, float inv_temp, int greedy,
                       const PhiloxState& st, uint64_t draw_base, int64_t* __restrict__ cur,
                       const uint8_t* __restrict__ known, float* __restrict__ conf) {
  float mx = -INFINITY, amax_v = -INFINITY;
  int amax_i = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const float raw = v[i];
    v[i] = __fmul_rn(raw, inv_temp);
    mx = fmaxf(mx, v[i]);
    if (raw > amax_v) { amax_v = raw; amax_i = lane * PER + i; }
  }
  mx = warp_max(mx);
  float local = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    v[i] = __expf(v[i] - mx);
    local += v[i];
  }
  const float total = warp_sum(local);
  const float inv = 1.0f / total;
  int sampled;
  if (greedy) {
    // argmax with first-index ties across lanes
    float bv = amax_v;
    int bi = amax_i;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    sampled = bi;
  } else {
    const double u = u64_to_double(philox_word(st, draw_base + (uint64_t)r));
    // exclusive prefix of lane sums (probabilities), then the count of cdf < u inside the lane
    float lsum = local * inv;
    float pre = lsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const float y = __shfl_up_sync(0xffffffffu, pre, o);
      if (lane >= o) pre += y;
    }
    float cdf = pre - lsum;
    int cnt = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      cdf += v[i] * inv;
      cnt += ((double)cdf < u) ? 1 : 0;
    }
    cnt = (int)warp_sum((float)cnt);
    sampled = cnt < K - 1 ? cnt : K - 1;
  }
  // confidence = probs[sampled] from the very exponentials the CDF used (no recomputation)
  float mine = 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i)
    if (lane * PER + i == sampled) mine = v[i];
  const float p = __shfl_sync(0xffffffffu, mine, sampled / PER) * inv;
  if (lane == 0) {
    const bool kn = known[r] != 0;
    if (!kn) cur[r] = sampled;
    conf[r] = kn ? INFINITY : p;
  }
}

JZ_DEV void load_sampler_params(const int64_t* __restrict__ dev_params, PhiloxState& st, uint64_t& draw_base) {
  if (dev_params) {
    draw_base = (uint64_t)dev_params[0];
    if (dev_params[12] >= 0) {  // Philox state from device memory
      for (int i = 0; i < 4; ++i) {
        st.ctr[i] = (uint64_t)dev_params[2 + i];
        st.buf[i] = (uint64_t)dev_params[8 + i];
      }
      st.key[0] = (uint64_t)dev_params[6];
      st.key[1] = (uint64_t)dev_params[7];
      st.pos = (int)dev_params[12];
    }
  }
}

// GUARD: K is not a multiple of 32 (small vocabularies, e.g. the reference's one-hot sampler
// test); codes past K are padded with -inf, so they add 0 to the CDF and never win the argmax.
template <int PER, bool GUARD = false>  // codes per lane
__global__ void maskgit_sample_kernel(const float* __restrict__ logits, int64_t rows, int K, float inv_temp,
                                      int greedy, PhiloxState st, uint64_t draw_base,
                                      const int64_t* __restrict__ dev_params, int64_t* __restrict__ cur,
                                      const uint8_t* __restrict__ known, float* __restrict__ conf) {
  load_sampler_params(dev_params, st, draw_base);
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* lr = logits + r * K + lane * PER;
  float v[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) v[i] = (!GUARD || lane * PER + i < K) ? lr[i] : -INFINITY;
  sample_row<PER>(v, r, lane, K, inv_temp, greedy, st, draw_base, cur, known, conf);
}

// Pipelined variant (K = 32 PER, PER % 4 == 0): each warp walks rows r, r + nwarps, ... and
// streams row r + nwarps into its second shared-memory buffer (cp.async, 512 contiguous bytes
// per instruction) while it samples row r.  Buffers hold 16-byte units u at u ^ ((u >> 3) & 7),
// so the lane-contiguous reads (lane l: units l PER/4 ..) are conflict-free.
constexpr int kSampleWarps = 4;
template <int PER>
__global__ void __launch_bounds__(32 * kSampleWarps) maskgit_sample_pipe_kernel(
    const float* __restrict__ logits, int64_t rows, int K, float inv_temp, int greedy, PhiloxState st,
    uint64_t draw_base, const int64_t* __restrict__ dev_params, int64_t* __restrict__ cur,
    const uint8_t* __restrict__ known, float* __restrict__ conf) {
  constexpr int U = 8 * PER;  // 16-byte units per row
  extern __shared__ uint4 sbuf[];
  load_sampler_params(dev_params, st, draw_base);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint4* const buf = sbuf + w * 2 * U;
  const int64_t nw = (int64_t)gridDim.x * kSampleWarps;
  auto issue = [&](int64_t row, uint4* dst) {
    const uint4* src = reinterpret_cast<const uint4*>(logits + row * K);
#pragma unroll
    for (int j = 0; j < PER / 4; ++j) {
      const int u = j * 32 + lane;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + (u ^ ((u >> 3) & 7)))),
                   "l"(src + u) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int64_t r = (int64_t)blockIdx.x * kSampleWarps + w;
  if (r < rows) issue(r, buf);
  for (int b = 0; r < rows; r += nw, b ^= 1) {
    const int64_t rn = r + nw;
    if (rn < rows) {
      issue(rn, buf + (b ^ 1) * U);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncwarp();
    const uint4* cb = buf + b * U;
    float v[PER];
#pragma unroll
    for (int i = 0; i < PER / 4; ++i) {
      const int u = lane * (PER / 4) + i;
      const float4 f = *reinterpret_cast<const float4*>(cb + (u ^ ((u >> 3) & 7)));
      v[4 * i] = f.x; v[4 * i + 1] = f.y; v[4 * i + 2] = f.z; v[4 * i + 3] = f.w;
    }
    __syncwarp();  // the buffer is refilled by the next iteration's prefetch
    sample_row<PER>(v, r, lane, K, inv_temp, greedy, st, draw_base, cur, known, conf);
  }
}

// ---------------------------------------------------------------------------
// K11b: per batch row, the n_keep highest-confidence positions (ties by position) become known.
__global__ void maskgit_select_kernel(const float* __restrict__ conf, int N, int n_keep,
                                      const int64_t* __restrict__ dev_params, uint8_t* __restrict__ known) {
  extern __shared__ float sconf[];
  if (dev_params) n_keep = (int)dev_params[1];
  const int64_t b = blockIdx.x;
  for (int i = threadIdx.x; i < N; i += blockDim.x) sconf[i] = conf[b * N + i];
  __syncthreads();
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const float ci = sconf[i];
    int rank = 0;
    for (int j = 0; j < N; ++j) {
      const float cj = sconf[j];
      rank += (cj > ci || (cj == ci && j < i)) ? 1 : 0;
    }
    known[b * N + i] = rank < n_keep ? 1 : 0;
  }
}

}  // namespace jz

using namespace jz;

extern "C" int jz_dyn_embed_frame(const int64_t* tokens, const uint8_t* known, const float* cond,
                                  const float* token_embed, const float* mask_token, const float* action_w,
                                  const float* action_b, const float* pos_spatial, const float* pos_temporal_row,
                                  const int* dev_t, int64_t B, int N, int D, int dl, int K, float* x,
                                  jz_stream_t s) {
  JZ_CHECK_ARG(D % 4 == 0 && D / 4 <= 1024, "embed_frame: D=%d", D);
  if (B == 0) return JZ_OK;
  const int64_t rows = B * (N + 1);
  int64_t grid = (rows + kEmbedRowsPerCta - 1) / kEmbedRowsPerCta;
  if (grid > (int64_t)num_sms() * 8) grid = (int64_t)num_sms() * 8;
  embed_frame_kernel<<<(unsigned)grid, 32 * kEmbedRowsPerCta, 0, reinterpret_cast<cudaStream_t>(s)>>>(
      tokens, known, cond, token_embed, mask_token, action_w, action_b, pos_spatial, pos_temporal_row, dev_t, rows, N,
      D, dl, K, x);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_attn_temporal_decode(const void* qkv, void* cache, int64_t B, int t, const int* dev_t, int Tmax,
                                       int S, int H, int append, void* out, jz_stream_t s) {
  JZ_CHECK_ARG(t >= 0 && t < Tmax && t <= 16, "temporal decode: frame index %d out of range", t);
  const int D = H * 64;
  JZ_CHECK_ARG(D == 128 || D == 256 || D == 512 || D == 1024, "temporal decode: model dim %d unsupported", D);
  const int64_t warps = B * S;
  if (warps == 0) return JZ_OK;
  auto st = reinterpret_cast<cudaStream_t>(s);
  const unsigned grid = (unsigned)((warps + 3) / 4);
  auto q = reinterpret_cast<const __nv_bfloat16*>(qkv);
  auto c = reinterpret_cast<__nv_bfloat16*>(cache);
  auto o = reinterpret_cast<__nv_bfloat16*>(out);
  const bool al16 = ((uintptr_t)qkv % 16) == 0 && ((uintptr_t)cache % 16) == 0 && ((uintptr_t)out % 16) == 0;
  JZ_CHECK_ARG(((uintptr_t)qkv % 8) == 0 && ((uintptr_t)cache % 8) == 0 && ((uintptr_t)out % 8) == 0,
               "temporal decode: qkv / cache / out must be 8-byte aligned");
  if (!al16) {  // 16-byte vector kernel needs 16-byte aligned rows; the 8-byte lane kernel does not
    switch (D) {
      case 128: temporal_decode_kernel<4><<<grid, 128, 0, st>>>(q, c, B, t, dev_t, Tmax, S, append, o); break;
      case 256: temporal_decode_kernel<8><<<grid, 128, 0, st>>>(q, c, B, t, dev_t, Tmax, S, append, o); break;
      case 512: temporal_decode_kernel<16><<<grid, 128, 0, st>>>(q, c, B, t, dev_t, Tmax, S, append, o); break;
      default: temporal_decode_kernel<32><<<grid, 128, 0, st>>>(q, c, B, t, dev_t, Tmax, S, append, o); break;
    }
    JZ_LAUNCH_CHECK();
    return JZ_OK;
  }
  switch (D) {
    case 128: temporal_decode_kernel<4><<<grid, 128, 0, st>>>(q, c, B, t, dev_t, Tmax, S, append, o); break;
    case 256: temporal_decode_v_kernel<1><<<grid, 128, 0, st>>>(q, c, B, t, dev_t, Tmax, S, append, o); break;
    case 512: temporal_decode_v_kernel<2><<<grid, 128, 0, st>>>(q, c, B, t, dev_t, Tmax, S, append, o); break;
    default: temporal_decode_v_kernel<4><<<grid, 128, 0, st>>>(q, c, B, t, dev_t, Tmax, S, append, o); break;
  }
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_kv_fill(const void* qkv, void* cache, int64_t B, int T, int t0, int Tmax, int S, int D,
                          jz_stream_t s) {
  JZ_CHECK_ARG(t0 + T <= Tmax, "kv_fill: %d + %d frames exceed cache %d", t0, T, Tmax);
  const int64_t n = B * T * S * (2 * D / 8);
  if (n == 0) return JZ_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
  kv_fill_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(
      reinterpret_cast<const __nv_bfloat16*>(qkv), reinterpret_cast<__nv_bfloat16*>(cache), B, T, t0, Tmax, S, D);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_maskgit_step(const float* logits, int64_t B, int N, int K, float temperature,
                               const uint64_t* counter4, const uint64_t* key2, const uint64_t* buffer4, int buffer_pos,
                               uint64_t draw_base, int n_keep, const int64_t* dev_params, int64_t* cur,
                               uint8_t* known, float* conf, jz_stream_t s) {
  JZ_CHECK_ARG(K >= 1 && K <= 2048, "maskgit: vocabulary %d unsupported (<= 2048)", K);
  JZ_CHECK_ARG(n_keep >= 0 && n_keep <= N, "maskgit: n_keep %d", n_keep);
  auto st = reinterpret_cast<cudaStream_t>(s);
  PhiloxState ps;
  for (int i = 0; i < 4; ++i) {
    ps.ctr[i] = counter4 ? counter4[i] : 0;
    ps.buf[i] = buffer4 ? buffer4[i] : 0;
  }
  ps.key[0] = key2 ? key2[0] : 0;
  ps.key[1] = key2 ? key2[1] : 0;
  ps.pos = buffer_pos;
  const int greedy = temperature < 1e-6f;
  const float inv_temp = 1.0f / fmaxf(temperature, 1e-8f);
  const int64_t rows = B * N;
  const unsigned grid = (unsigned)((rows + 7) / 8);
  if (rows == 0) return JZ_OK;
  // pipelined kernel: one resident wave (4 CTAs of 4 warps per SM at 128 registers), each warp
  // walking several rows
  int64_t pgrid = (rows + kSampleWarps - 1) / kSampleWarps;
  if (pgrid > (int64_t)num_sms() * 4) pgrid = (int64_t)num_sms() * 4;
  const size_t psmem = (size_t)kSampleWarps * 2 * K * sizeof(float);
  if (K % 32 != 0) {
    const int per = (K + 31) / 32;
#define MG(P) else if (per <= P) maskgit_sample_kernel<P, true><<<grid, 256, 0, st>>>(logits, rows, K, inv_temp, greedy, ps, draw_base, dev_params, cur, known, conf);
    if (false) {}
    MG(1) MG(2) MG(4) MG(8) MG(16) MG(32) MG(64)
#undef MG
    JZ_LAUNCH_CHECK();
    maskgit_select_kernel<<<(unsigned)B, 256, N * sizeof(float), st>>>(conf, N, n_keep, dev_params, known);
    JZ_LAUNCH_CHECK();
    return JZ_OK;
  }
  switch (K / 32) {
#define MS_(P) maskgit_sample_kernel<P><<<grid, 256, 0, st>>>(logits, rows, K, inv_temp, greedy, ps, draw_base, dev_params, cur, known, conf);
#define MS(P) case P: MS_(P) break;
#define MP(P) case P: if (((uintptr_t)logits % 16) != 0) { MS_(P) } else maskgit_sample_pipe_kernel<P><<<(unsigned)pgrid, 32 * kSampleWarps, psmem, st>>>(logits, rows, K, inv_temp, greedy, ps, draw_base, dev_params, cur, known, conf); break;
    MS(1) MS(2) MP(4) MP(8) MP(16) MP(32) MS(64)
#undef MS
#undef MS_
#undef MP
    default: set_error("maskgit: vocabulary %d unsupported", K); return JZ_EINVAL;
  }
  JZ_LAUNCH_CHECK();
  maskgit_select_kernel<<<(unsigned)B, 256, N * sizeof(float), st>>>(conf, N, n_keep, dev_params, known);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}
