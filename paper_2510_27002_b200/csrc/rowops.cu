// Row-parallel, HBM-bound kernels of the hot path (all deterministic):
//   K2  LayerNorm forward / backward (+ fused dgamma/dbeta/dbias partials)
//       replaces nn.layer_norm (nn.py:35-40) and its autodiff backward
//   colsum / partial reduction  (bias gradients: _unbroadcast sums, autodiff.py:22-32)
//   fp32 -> bf16 casts (weight shadows)
//   K7  masked softmax cross-entropy fwd+bwd (nn.py:56-77, dynamics.py:151-152)
//   K13 AdamW (optim.py:34-62), bit-exact f32 arithmetic (no FMA contraction)
//
// Cross-row reductions never use float atomics: each CTA owns a fixed contiguous
// row range and writes a partial row; jz_reduce_partials sums partials in index
// order, so every gradient is bitwise reproducible run to run.
#include "common.h"
#include "ptx.cuh"

namespace jz {

constexpr int kRowThreads = 256;  // 8 warps, one row per warp at a time

// ---------------------------------------------------------------------------
// LayerNorm forward: one warp per row; lane holds D/32 values (float4 strided by 128)
// ---------------------------------------------------------------------------
template <int V4>  // number of float4 per lane: D = 128 * V4
__global__ void __launch_bounds__(kRowThreads) ln_fwd_kernel(const float* __restrict__ x, int64_t rows,
                                                             const float* __restrict__ g,
                                                             const float* __restrict__ b, float eps,
                                                             __nv_bfloat16* __restrict__ y,
                                                             float* __restrict__ y32,
                                                             float* __restrict__ mean_out,
                                                             float* __restrict__ rstd_out,
                                                             int64_t skip_period) {
  constexpr int D = 128 * V4;
  const int lane = threadIdx.x & 31;
  const int64_t warps_total = (int64_t)gridDim.x * (kRowThreads / 32);
  for (int64_t r = (int64_t)blockIdx.x * (kRowThreads / 32) + (threadIdx.x >> 5); r < rows;
       r += warps_total) {
    const float* xr = x + r * D;
    float4 v[V4];
#pragma unroll
    for (int i = 0; i < V4; ++i) v[i] = *reinterpret_cast<const float4*>(xr + 4 * lane + 128 * i);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < V4; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    const float mu = warp_sum(s) / (float)D;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      float a = v[i].x - mu, bb = v[i].y - mu, c = v[i].z - mu, d = v[i].w - mu;
      q += (a * a + bb * bb) + (c * c + d * d);
    }
    const float var = warp_sum(q) / (float)D;
    const float rs = 1.0f / sqrtf(var + eps);
    if (lane == 0) {
      mean_out[r] = mu;
      rstd_out[r] = rs;
    }
    int64_t orow = r;
    if (skip_period > 0) {
      if (r % skip_period == 0) continue;
      orow = r - r / skip_period - 1;
    }
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const int c = 4 * lane + 128 * i;
      float4 gg = *reinterpret_cast<const float4*>(g + c);
      float4 bb = *reinterpret_cast<const float4*>(b + c);
      float o0 = (v[i].x - mu) * rs * gg.x + bb.x;
      float o1 = (v[i].y - mu) * rs * gg.y + bb.y;
      float o2 = (v[i].z - mu) * rs * gg.z + bb.z;
      float o3 = (v[i].w - mu) * rs * gg.w + bb.w;
      if (y) *reinterpret_cast<uint2*>(y + orow * D + c) = make_uint2(pack_bf16(o0, o1), pack_bf16(o2, o3));
      if (y32) *reinterpret_cast<float4*>(y32 + orow * D + c) = make_float4(o0, o1, o2, o3);
    }
  }
}

// ---------------------------------------------------------------------------
// LayerNorm backward (+ residual accumulate + bf16 copy + per-CTA column partials)
//   dxn  = dy * g
//   dx   = rstd * (dxn - mean(dxn) - xhat * mean(dxn * xhat))
//   out  = (accumulate ? dres : 0) + dx      (f32, in place on dres)
//   part_dg[blk] = sum dy*xhat, part_db[blk] = sum dy, part_dbias[blk] = sum out
// One CTA owns rows [blk*rpb, (blk+1)*rpb); warps stride by 8 inside; warp partials are
// combined in warp order through shared memory.
// ---------------------------------------------------------------------------
// dy row loader: fp32 or bf16 (the dX GEMM's bf16 output halves the bytes of this HBM-bound pass)
JZ_DEV float4 load4(const float* p) { return *reinterpret_cast<const float4*>(p); }
JZ_DEV float4 load4(const __nv_bfloat16* p) {
  const uint2 w = *reinterpret_cast<const uint2*>(p);
  const float2 a = unpack_bf16(w.x), b = unpack_bf16(w.y);
  return make_float4(a.x, a.y, b.x, b.y);
}

template <int V4, typename DyT>
__global__ void __launch_bounds__(kRowThreads, 2) ln_bwd_kernel(
    const float* __restrict__ x, const float* __restrict__ mean, const float* __restrict__ rstd,
    const float* __restrict__ g, const DyT* __restrict__ dy, float* dres, int accumulate,
    __nv_bfloat16* __restrict__ dres_bf16, float* __restrict__ part_dg, float* __restrict__ part_db,
    float* __restrict__ part_dbias, int64_t rows, int64_t rows_per_block, int64_t skip_period) {
  constexpr int D = 128 * V4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  float4 adg[V4], adb[V4], adbias[V4];
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    adg[i] = make_float4(0, 0, 0, 0);
    adb[i] = make_float4(0, 0, 0, 0);
    adbias[i] = make_float4(0, 0, 0, 0);
  }
  for (int64_t r = r0 + warp; r < r1; r += kRowThreads / 32) {
    const float mu = mean[r], rs = rstd[r];
    const float* xr = x + r * D;
    float4 xv[V4], dyv[V4], pv[V4];
    bool has_dy = true;
    int64_t irow = r;
    if (skip_period > 0) {
      if (r % skip_period == 0) has_dy = false;
      irow = r - r / skip_period - 1;
    }
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const int c = 4 * lane + 128 * i;
      xv[i] = *reinterpret_cast<const float4*>(xr + c);
      dyv[i] = has_dy ? load4(dy + irow * D + c) : make_float4(0, 0, 0, 0);
      pv[i] = accumulate ? *reinterpret_cast<const float4*>(dres + r * D + c) : make_float4(0, 0, 0, 0);
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const int c = 4 * lane + 128 * i;
      float4 gg = *reinterpret_cast<const float4*>(g + c);
      float4 xh = make_float4((xv[i].x - mu) * rs, (xv[i].y - mu) * rs, (xv[i].z - mu) * rs,
                              (xv[i].w - mu) * rs);
      float4 dn = make_float4(dyv[i].x * gg.x, dyv[i].y * gg.y, dyv[i].z * gg.z, dyv[i].w * gg.w);
      s1 += (dn.x + dn.y) + (dn.z + dn.w);
      s2 += (dn.x * xh.x + dn.y * xh.y) + (dn.z * xh.z + dn.w * xh.w);
      adg[i].x += dyv[i].x * xh.x; adg[i].y += dyv[i].y * xh.y;
      adg[i].z += dyv[i].z * xh.z; adg[i].w += dyv[i].w * xh.w;
      adb[i].x += dyv[i].x; adb[i].y += dyv[i].y; adb[i].z += dyv[i].z; adb[i].w += dyv[i].w;
      xv[i] = xh;      // keep xhat
      dyv[i] = dn;     // keep dxn
    }
    const float m1 = warp_sum(s1) / (float)D;
    const float m2 = warp_sum(s2) / (float)D;
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const int c = 4 * lane + 128 * i;
      float4 o = make_float4(rs * (dyv[i].x - m1 - xv[i].x * m2), rs * (dyv[i].y - m1 - xv[i].y * m2),
                             rs * (dyv[i].z - m1 - xv[i].z * m2), rs * (dyv[i].w - m1 - xv[i].w * m2));
      float* dr = dres + r * D + c;
      o.x += pv[i].x; o.y += pv[i].y; o.z += pv[i].z; o.w += pv[i].w;
      *reinterpret_cast<float4*>(dr) = o;
      if (dres_bf16) {
        uint2 w = make_uint2(pack_bf16(o.x, o.y), pack_bf16(o.z, o.w));
        *reinterpret_cast<uint2*>(dres_bf16 + r * D + c) = w;
      }
      adbias[i].x += o.x; adbias[i].y += o.y; adbias[i].z += o.z; adbias[i].w += o.w;
    }
  }
  // combine warp partials in fixed order
  __shared__ float sm[kRowThreads / 32][D];
  auto flush = [&](float4 (&acc)[V4], float* out) {
#pragma unroll
    for (int i = 0; i < V4; ++i) *reinterpret_cast<float4*>(&sm[warp][4 * lane + 128 * i]) = acc[i];
    __syncthreads();
    for (int c = threadIdx.x; c < D; c += kRowThreads) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < kRowThreads / 32; ++w) s += sm[w][c];
      out[(int64_t)blockIdx.x * D + c] = s;
    }
    __syncthreads();
  };
  if (part_dg) flush(adg, part_dg);
  if (part_db) flush(adb, part_db);
  if (part_dbias) flush(adbias, part_dbias);
}

// ---------------------------------------------------------------------------
// Column sums of a bf16 matrix (bias gradients), per-CTA partials.
// ---------------------------------------------------------------------------
// Threads form `groups` row-groups of cpt = cols/8 threads (8 columns each); group g takes rows
// r0 + g, r0 + g + groups, ... with 16 independent 16-byte loads in flight, and the groups' sums are
// combined in group order through shared memory (deterministic).  cols/8 > kRowThreads: one group,
// looping over column blocks.
__global__ void __launch_bounds__(kRowThreads) colsum_bf16_kernel(const __nv_bfloat16* __restrict__ x,
                                                                  int64_t rows, int cols, int64_t ld,
                                                                  int64_t rows_per_block,
                                                                  float* __restrict__ part) {
  __shared__ float4 red[kRowThreads][2];
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  const int cpt = cols / 8;
  const int groups = cpt >= kRowThreads ? 1 : kRowThreads / cpt;
  const int g = cpt >= kRowThreads ? 0 : threadIdx.x / cpt;
  const int tcol = cpt >= kRowThreads ? threadIdx.x : threadIdx.x - g * cpt;
  const bool live = g < groups;
  for (int c8 = tcol * 8; c8 < cols; c8 += kRowThreads * 8) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (live) {
      int64_t r = r0 + g;
      for (; r + 15 * groups < r1; r += 16 * groups) {
        uint4 w[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) w[q] = __ldg(reinterpret_cast<const uint4*>(x + (r + q * groups) * ld + c8));
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float2 a = unpack_bf16(w[q].x), b = unpack_bf16(w[q].y), c = unpack_bf16(w[q].z), d = unpack_bf16(w[q].w);
          acc[0] += a.x; acc[1] += a.y; acc[2] += b.x; acc[3] += b.y;
          acc[4] += c.x; acc[5] += c.y; acc[6] += d.x; acc[7] += d.y;
        }
      }
      for (; r < r1; r += groups) {
        uint4 w = __ldg(reinterpret_cast<const uint4*>(x + r * ld + c8));
        float2 a = unpack_bf16(w.x), b = unpack_bf16(w.y), c = unpack_bf16(w.z), d = unpack_bf16(w.w);
        acc[0] += a.x; acc[1] += a.y; acc[2] += b.x; acc[3] += b.y;
        acc[4] += c.x; acc[5] += c.y; acc[6] += d.x; acc[7] += d.y;
      }
    }
    if (groups > 1) {
      red[threadIdx.x][0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
      red[threadIdx.x][1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
      __syncthreads();
      if (g == 0) {
        for (int g2 = 1; g2 < groups; ++g2) {
          const float4 u = red[g2 * cpt + tcol][0], v = red[g2 * cpt + tcol][1];
          acc[0] += u.x; acc[1] += u.y; acc[2] += u.z; acc[3] += u.w;
          acc[4] += v.x; acc[5] += v.y; acc[6] += v.z; acc[7] += v.w;
        }
      }
    }
    if (g == 0) {
      float4* out = reinterpret_cast<float4*>(part + (int64_t)blockIdx.x * cols + c8);
      out[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
      out[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
    if (groups > 1) break;  // cpt < kRowThreads: every column is covered by the first pass
  }
}

// out[c] = sum_p part[p * stride][c]: 8 fixed part-groups x 32 columns per CTA, groups combined in order.
__global__ void __launch_bounds__(256) reduce_partials_kernel(const float* __restrict__ part, int nparts, int64_t D,
                                                             float* __restrict__ out, int accumulate,
                                                             int stride = 1) {
  __shared__ float sm[8][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  for (int64_t c0 = (int64_t)blockIdx.x * 32; c0 < D; c0 += (int64_t)gridDim.x * 32) {
    const int64_t c = c0 + lane;
    float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // 8 loads in flight, fixed order
    if (c < D) {
      int p = grp;
      for (; p + 56 < nparts; p += 64) {
#pragma unroll
        for (int q = 0; q < 8; ++q) s[q] += __ldg(part + (int64_t)(p + 8 * q) * stride * D + c);
      }
      for (int q = 0; p < nparts; p += 8, ++q) s[q] += __ldg(part + (int64_t)p * stride * D + c);
    }
    sm[grp][lane] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
    __syncthreads();
    if (grp == 0 && c < D) {
      float t = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) t += sm[k][lane];
      out[c] = accumulate ? out[c] + t : t;
    }
    __syncthreads();
  }
}

// Up to three independent single-stage reductions in one launch (blockIdx.y = which): the
// LayerNorm backward's gamma / beta / residual-bias partials are reduced concurrently instead of by
// three latency-bound launches.  Same per-column summation order as reduce_partials_kernel.
struct Reduce3 {
  const float* part[3];
  float* out[3];
};
__global__ void __launch_bounds__(256) reduce_partials3_kernel(Reduce3 r, int nparts, int64_t D, int accumulate) {
  const float* part = r.part[blockIdx.y];
  float* out = r.out[blockIdx.y];
  if (out == nullptr) return;
  __shared__ float sm[8][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  for (int64_t c0 = (int64_t)blockIdx.x * 32; c0 < D; c0 += (int64_t)gridDim.x * 32) {
    const int64_t c = c0 + lane;
    float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (c < D) {
      int p = grp;
      for (; p + 56 < nparts; p += 64) {
#pragma unroll
        for (int q = 0; q < 8; ++q) s[q] += __ldg(part + (int64_t)(p + 8 * q) * D + c);
      }
      for (int q = 0; p < nparts; p += 8, ++q) s[q] += __ldg(part + (int64_t)p * D + c);
    }
    sm[grp][lane] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
    __syncthreads();
    if (grp == 0 && c < D) {
      float t = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) t += sm[k][lane];
      out[c] = accumulate ? out[c] + t : t;
    }
    __syncthreads();
  }
}

// Stage 1 for many partial rows: CTA (column block x, chunk y) sums rows [256 y, 256 y + 256) of its
// 32 columns in a fixed order and writes the result into row 256 y (a row only it reads).
constexpr int kChunkRows = 256;
__global__ void __launch_bounds__(256) reduce_chunks_kernel(float* __restrict__ part, int nparts, int64_t D) {
  __shared__ float sm[8][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t c = (int64_t)blockIdx.x * 32 + lane;
  const int p0 = blockIdx.y * kChunkRows, p1 = min(nparts, p0 + kChunkRows);
  float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // 8 loads in flight, fixed order
  if (c < D) {
    int p = p0 + grp;
    for (; p + 56 < p1; p += 64) {
#pragma unroll
      for (int q = 0; q < 8; ++q) s[q] += part[(int64_t)(p + 8 * q) * D + c];
    }
    for (int q = 0; p < p1; p += 8, ++q) s[q] += part[(int64_t)p * D + c];
  }
  sm[grp][lane] = ((s[0] + s[1]) + (s[2] + s[3])) + ((s[4] + s[5]) + (s[6] + s[7]));
  __syncthreads();
  if (grp == 0 && c < D) {
    float t = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += sm[k][lane];
    part[(int64_t)p0 * D + c] = t;
  }
}

// contiguous fp32 -> bf16 (the per-step flat weight shadow): 8 elements per thread per iteration
__global__ void cast_flat8_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, int64_t n8) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 a = reinterpret_cast<const float4*>(src)[2 * i];
    const float4 b = reinterpret_cast<const float4*>(src)[2 * i + 1];
    reinterpret_cast<uint4*>(dst)[i] = make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(b.x, b.y),
                                                  pack_bf16(b.z, b.w));
  }
}

__global__ void cast2d_kernel(const float* __restrict__ src, int64_t lds, __nv_bfloat16* __restrict__ dst,
                              int64_t ldd, int64_t rows, int64_t cols) {
  const int64_t n = rows * cols;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / cols, c = i - r * cols;
    dst[r * ldd + c] = __float2bfloat16_rn(src[r * lds + c]);
  }
}

// ---------------------------------------------------------------------------
// K7 masked softmax cross-entropy, forward AND backward in one pass (the loss is the
// end of the graph, so dlogits = grad_scale * w/sum(w) * (softmax - onehot)).
// One warp per row.  count: device int (sum of weights, from the mask kernel).
// ---------------------------------------------------------------------------
template <int KV>  // K = 32 * 4 * KV
__global__ void __launch_bounds__(kRowThreads) ce_kernel(const float* __restrict__ logits, int64_t rows,
                                                         int K, const int64_t* __restrict__ targets,
                                                         const uint8_t* __restrict__ mask,
                                                         const int* __restrict__ count, float grad_scale,
                                                         __nv_bfloat16* __restrict__ dlogits,
                                                         float* __restrict__ row_loss) {
  const int lane = threadIdx.x & 31;
  const int64_t warps_total = (int64_t)gridDim.x * (kRowThreads / 32);
  const int cnt = *count;
  const float inv = cnt > 0 ? 1.0f / (float)cnt : 0.0f;
  for (int64_t r = (int64_t)blockIdx.x * (kRowThreads / 32) + (threadIdx.x >> 5); r < rows;
       r += warps_total) {
    const float* lr = logits + r * K;
    float4 v[KV];
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < KV; ++i) {
      v[i] = *reinterpret_cast<const float4*>(lr + 4 * lane + 128 * i);
      mx = fmaxf(mx, fmaxf(fmaxf(v[i].x, v[i].y), fmaxf(v[i].z, v[i].w)));
    }
    mx = warp_max(mx);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < KV; ++i) {
      v[i].x = expf(v[i].x - mx); v[i].y = expf(v[i].y - mx);
      v[i].z = expf(v[i].z - mx); v[i].w = expf(v[i].w - mx);
      s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
    s = warp_sum(s);
    const int64_t tgt = targets[r];
    const float w = mask ? (float)mask[r] : 1.0f;
    if (lane == 0) {
      const float lt = lr[tgt] - mx;
      row_loss[r] = w * (logf(s) - lt);
    }
    const float coef = grad_scale * w * inv;
    const float invs = 1.0f / s;
    __nv_bfloat16* dr = dlogits + r * K;
#pragma unroll
    for (int i = 0; i < KV; ++i) {
      const int c = 4 * lane + 128 * i;
      float d0 = v[i].x * invs, d1 = v[i].y * invs, d2 = v[i].z * invs, d3 = v[i].w * invs;
      if (tgt == c) d0 -= 1.f;
      if (tgt == c + 1) d1 -= 1.f;
      if (tgt == c + 2) d2 -= 1.f;
      if (tgt == c + 3) d3 -= 1.f;
      uint2 o = make_uint2(pack_bf16(coef * d0, coef * d1), pack_bf16(coef * d2, coef * d3));
      *reinterpret_cast<uint2*>(dr + c) = o;
    }
  }
}

// loss = sum(row_loss) / count  (single CTA, fixed order, f64 accumulation)
__global__ void ce_finalize_kernel(const float* __restrict__ row_loss, int64_t rows,
                                   const int* __restrict__ count, float* __restrict__ loss) {
  __shared__ double sm[1024];
  // thread t sums rows t, t + blockDim, ... (coalesced, 4 loads in flight), fixed order
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  const int64_t nb = blockDim.x;
  int64_t i = threadIdx.x;
  for (; i + 3 * nb < rows; i += 4 * nb) {
#pragma unroll
    for (int q = 0; q < 4; ++q) s[q] += (double)row_loss[i + q * nb];
  }
  for (int q = 0; i < rows; i += nb, ++q) s[q] += (double)row_loss[i];
  sm[threadIdx.x] = (s[0] + s[1]) + (s[2] + s[3]);
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)blockDim.x; ++i) t += sm[i];
    const int c = *count;
    *loss = c > 0 ? (float)(t / (double)c) : 0.0f;
  }
}

// ---------------------------------------------------------------------------
// K13 AdamW.  Exact numpy/NEP-50 f32 semantics of optim.py:52-62:
//   m = m*b1; m = m + omb1*g; v = v*b2; v = v + omb2*(g*g);
//   mh = m/bc1; vh = v/bc2; p = p - lr*(mh/(sqrt(vh)+eps)); [p = p - lrwd*p]
// ---------------------------------------------------------------------------
__global__ void finite_check_kernel(const float* __restrict__ g, int64_t n, int* flag) {
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(g[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(flag, 1);
}

__global__ void adamw_kernel(float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                             float* __restrict__ v, int64_t n, float lr, float b1, float b2, float omb1,
                             float omb2, float bc1, float bc2, float eps, float lrwd,
                             const int* __restrict__ flag, const float* __restrict__ dev_sc) {
  if (flag && *flag) return;  // non-finite gradient somewhere: leave every param untouched
  if (dev_sc) {  // graph replays: this step's scalars from device memory (layout of jz_adamw_step_dev)
    lr = dev_sc[0]; b1 = dev_sc[1]; b2 = dev_sc[2]; omb1 = dev_sc[3]; omb2 = dev_sc[4];
    bc1 = dev_sc[5]; bc2 = dev_sc[6]; eps = dev_sc[7]; lrwd = dev_sc[8];
  }
  // one element, in the reference's operation order with IEEE round-to-nearest throughout
  auto upd1 = [&](float& pi, float& mi, float& vi, float gi) {
    mi = __fadd_rn(__fmul_rn(mi, b1), __fmul_rn(omb1, gi));
    vi = __fadd_rn(__fmul_rn(vi, b2), __fmul_rn(omb2, __fmul_rn(gi, gi)));
    const float mh = __fdiv_rn(mi, bc1);
    const float vh = __fdiv_rn(vi, bc2);
    const float upd = __fmul_rn(lr, __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), eps)));
    pi = __fsub_rn(pi, upd);
    if (lrwd != 0.f) pi = __fsub_rn(pi, __fmul_rn(lrwd, pi));
  };
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(m) |
                     reinterpret_cast<uintptr_t>(v)) & 15) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  // 16-byte vectors: the four streams at full sector efficiency with 4 elements in flight per thread
  for (int64_t i = tid; i < n4; i += nth) {
    const float4 gv = reinterpret_cast<const float4*>(g)[i];
    float4 mv = reinterpret_cast<float4*>(m)[i], vv = reinterpret_cast<float4*>(v)[i],
           pv = reinterpret_cast<float4*>(p)[i];
    upd1(pv.x, mv.x, vv.x, gv.x);
    upd1(pv.y, mv.y, vv.y, gv.y);
    upd1(pv.z, mv.z, vv.z, gv.z);
    upd1(pv.w, mv.w, vv.w, gv.w);
    reinterpret_cast<float4*>(m)[i] = mv;
    reinterpret_cast<float4*>(v)[i] = vv;
    reinterpret_cast<float4*>(p)[i] = pv;
  }
  for (int64_t i = 4 * n4 + tid; i < n; i += nth) {
    float pi = p[i], mi = m[i], vi = v[i];
    upd1(pi, mi, vi, g[i]);
    m[i] = mi;
    v[i] = vi;
    p[i] = pi;
  }
}

static int grid_for(int64_t n, int threads, int max_per_sm = 8) {
  int64_t b = (n + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * max_per_sm;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace jz

using namespace jz;

extern "C" int jz_layernorm_fwd(const float* x, int64_t rows, int D, const float* gamma, const float* beta,
                                float eps, void* y_bf16, float* y_f32, float* mean, float* rstd, int64_t skip_period,
                                jz_stream_t s) {
  JZ_CHECK_ARG(rows >= 0 && D % 128 == 0 && D >= 128 && D <= 1024,
               "layernorm: model dim %d unsupported on device (multiple of 128, <= 1024)", D);
  if (rows == 0) return JZ_OK;
  const int grid = grid_for(rows, 8, 16);
  auto st = reinterpret_cast<cudaStream_t>(s);
  auto y = reinterpret_cast<__nv_bfloat16*>(y_bf16);
  switch (D / 128) {
    case 1: ln_fwd_kernel<1><<<grid, kRowThreads, 0, st>>>(x, rows, gamma, beta, eps, y, y_f32, mean, rstd, skip_period); break;
    case 2: ln_fwd_kernel<2><<<grid, kRowThreads, 0, st>>>(x, rows, gamma, beta, eps, y, y_f32, mean, rstd, skip_period); break;
    case 3: ln_fwd_kernel<3><<<grid, kRowThreads, 0, st>>>(x, rows, gamma, beta, eps, y, y_f32, mean, rstd, skip_period); break;
    case 4: ln_fwd_kernel<4><<<grid, kRowThreads, 0, st>>>(x, rows, gamma, beta, eps, y, y_f32, mean, rstd, skip_period); break;
    case 6: ln_fwd_kernel<6><<<grid, kRowThreads, 0, st>>>(x, rows, gamma, beta, eps, y, y_f32, mean, rstd, skip_period); break;
    case 8: ln_fwd_kernel<8><<<grid, kRowThreads, 0, st>>>(x, rows, gamma, beta, eps, y, y_f32, mean, rstd, skip_period); break;
    default: set_error("layernorm: D=%d unsupported", D); return JZ_EINVAL;
  }
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_row_partials(int64_t rows) {
  // number of per-CTA partial rows used by the column reductions for `rows` input rows
  int64_t p = (int64_t)num_sms() * 2;
  if (rows < p) p = rows > 0 ? rows : 1;
  return (int)p;
}

template <typename DyT>
static int layernorm_bwd_impl(const float* x, const float* mean, const float* rstd, const float* gamma,
                              const DyT* dy, float* dres, int accumulate, void* dres_bf16,
                              float* part_dgamma, float* part_dbeta, float* part_dbias, int nparts,
                              int64_t rows, int D, int64_t skip_period, jz_stream_t s) {
  JZ_CHECK_ARG(D % 128 == 0 && D >= 128 && D <= 1024, "layernorm_bwd: D=%d unsupported", D);
  JZ_CHECK_ARG(nparts >= 1, "layernorm_bwd: nparts");
  if (rows == 0) return JZ_OK;
  const int64_t rpb = (rows + nparts - 1) / nparts;
  const int grid = (int)((rows + rpb - 1) / rpb);
  auto st = reinterpret_cast<cudaStream_t>(s);
  auto yb = reinterpret_cast<__nv_bfloat16*>(dres_bf16);
#define LNB(V)                                                                                         \
  ln_bwd_kernel<V, DyT><<<grid, kRowThreads, 0, st>>>(x, mean, rstd, gamma, dy, dres, accumulate, yb,  \
                                                 part_dgamma, part_dbeta, part_dbias, rows, rpb, skip_period)
  switch (D / 128) {
    case 1: LNB(1); break;
    case 2: LNB(2); break;
    case 4: LNB(4); break;
    case 8: LNB(8); break;
    default: set_error("layernorm_bwd: D=%d unsupported", D); return JZ_EINVAL;
  }
#undef LNB
  JZ_LAUNCH_CHECK();
  // grid may be < nparts for small inputs: zero the unused partial rows
  if (grid < nparts) {
    const size_t bytes = (size_t)(nparts - grid) * D * sizeof(float);
    if (part_dgamma) JZ_CUDA_TRY(cudaMemsetAsync(part_dgamma + (int64_t)grid * D, 0, bytes, st));
    if (part_dbeta) JZ_CUDA_TRY(cudaMemsetAsync(part_dbeta + (int64_t)grid * D, 0, bytes, st));
    if (part_dbias) JZ_CUDA_TRY(cudaMemsetAsync(part_dbias + (int64_t)grid * D, 0, bytes, st));
  }
  return JZ_OK;
}

extern "C" int jz_layernorm_bwd(const float* x, const float* mean, const float* rstd, const float* gamma,
                                const float* dy, float* dres, int accumulate, void* dres_bf16,
                                float* part_dgamma, float* part_dbeta, float* part_dbias, int nparts,
                                int64_t rows, int D, int64_t skip_period, jz_stream_t s) {
  return layernorm_bwd_impl(x, mean, rstd, gamma, dy, dres, accumulate, dres_bf16, part_dgamma, part_dbeta,
                            part_dbias, nparts, rows, D, skip_period, s);
}

extern "C" int jz_layernorm_bwd_bf16dy(const float* x, const float* mean, const float* rstd, const float* gamma,
                                       const void* dy, float* dres, int accumulate, void* dres_bf16,
                                       float* part_dgamma, float* part_dbeta, float* part_dbias, int nparts,
                                       int64_t rows, int D, int64_t skip_period, jz_stream_t s) {
  return layernorm_bwd_impl(x, mean, rstd, gamma, reinterpret_cast<const __nv_bfloat16*>(dy), dres, accumulate,
                            dres_bf16, part_dgamma, part_dbeta, part_dbias, nparts, rows, D, skip_period, s);
}

extern "C" int jz_colsum_bf16(const void* x, int64_t rows, int cols, int64_t ld, float* part, int nparts,
                              jz_stream_t s) {
  JZ_CHECK_ARG(cols % 8 == 0 && ld % 8 == 0, "colsum: cols/ld must be multiples of 8");
  JZ_CHECK_ARG(nparts >= 1, "colsum: nparts");
  auto st = reinterpret_cast<cudaStream_t>(s);
  if (rows == 0) {
    JZ_CUDA_TRY(cudaMemsetAsync(part, 0, (size_t)nparts * cols * sizeof(float), st));
    return JZ_OK;
  }
  const int64_t rpb = (rows + nparts - 1) / nparts;
  const int grid = (int)((rows + rpb - 1) / rpb);
  colsum_bf16_kernel<<<grid, kRowThreads, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(x), rows, cols, ld,
                                                   rpb, part);
  JZ_LAUNCH_CHECK();
  if (grid < nparts)
    JZ_CUDA_TRY(cudaMemsetAsync(part + (int64_t)grid * cols, 0, (size_t)(nparts - grid) * cols * 4, st));
  return JZ_OK;
}

extern "C" int jz_reduce_partials(const float* part, int nparts, int64_t D, float* out, int accumulate,
                                  jz_stream_t s) {
  if (D == 0) return JZ_OK;
  auto st = reinterpret_cast<cudaStream_t>(s);
  int stride = 1;
  if (nparts > 2 * kChunkRows) {
    // two deterministic stages; the partial buffer is scratch (its chunk-leading rows are overwritten)
    const int chunks = (nparts + kChunkRows - 1) / kChunkRows;
    reduce_chunks_kernel<<<dim3((unsigned)((D + 31) / 32), (unsigned)chunks), 256, 0, st>>>(
        const_cast<float*>(part), nparts, D);
    JZ_LAUNCH_CHECK();
    nparts = chunks;
    stride = kChunkRows;
  }
  int64_t blocks = (D + 31) / 32;
  if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
  reduce_partials_kernel<<<(unsigned)blocks, 256, 0, st>>>(part, nparts, D, out, accumulate, stride);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_reduce_partials3(const float* part0, const float* part1, const float* part2, int nparts, int64_t D,
                                   float* out0, float* out1, float* out2, int accumulate, jz_stream_t s) {
  if (D == 0 || (!out0 && !out1 && !out2)) return JZ_OK;
  auto st = reinterpret_cast<cudaStream_t>(s);
  if (nparts > 2 * kChunkRows) {  // large partial counts: the two-stage path, one output at a time
    const float* ps[3] = {part0, part1, part2};
    float* os[3] = {out0, out1, out2};
    for (int i = 0; i < 3; ++i)
      if (os[i]) {
        const int rc = jz_reduce_partials(ps[i], nparts, D, os[i], accumulate, s);
        if (rc) return rc;
      }
    return JZ_OK;
  }
  Reduce3 r;
  r.part[0] = part0; r.part[1] = part1; r.part[2] = part2;
  r.out[0] = out0; r.out[1] = out1; r.out[2] = out2;
  int64_t blocks = (D + 31) / 32;
  if (blocks > (int64_t)num_sms() * 8) blocks = (int64_t)num_sms() * 8;
  reduce_partials3_kernel<<<dim3((unsigned)blocks, 3), 256, 0, st>>>(r, nparts, D, accumulate);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_cast_f32_bf16_2d(const float* src, int64_t lds, void* dst, int64_t ldd, int64_t rows,
                                   int64_t cols, jz_stream_t s) {
  if (rows * cols == 0) return JZ_OK;
  const int64_t n = rows * cols;
  const bool flat = (rows == 1 || (lds == cols && ldd == cols)) && n % 8 == 0 && ((uintptr_t)src % 16) == 0 &&
                    ((uintptr_t)dst % 16) == 0;
  if (flat) {
    cast_flat8_kernel<<<grid_for(n / 8, 256), 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(
        src, reinterpret_cast<__nv_bfloat16*>(dst), n / 8);
    JZ_LAUNCH_CHECK();
    return JZ_OK;
  }
  cast2d_kernel<<<grid_for(rows * cols, 256), 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(
      src, lds, reinterpret_cast<__nv_bfloat16*>(dst), ldd, rows, cols);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_ce_fwd_bwd(const float* logits, int64_t rows, int K, const int64_t* targets,
                             const uint8_t* mask, const int* count, float grad_scale, void* dlogits,
                             float* row_loss, float* loss, jz_stream_t s) {
  JZ_CHECK_ARG(K % 128 == 0 && K >= 128 && K <= 4096, "cross-entropy: K=%d unsupported on device", K);
  auto st = reinterpret_cast<cudaStream_t>(s);
  if (rows > 0) {
    const int grid = grid_for(rows, 8, 16);
    auto dl = reinterpret_cast<__nv_bfloat16*>(dlogits);
    switch (K / 128) {
      case 1: ce_kernel<1><<<grid, kRowThreads, 0, st>>>(logits, rows, K, targets, mask, count, grad_scale, dl, row_loss); break;
      case 2: ce_kernel<2><<<grid, kRowThreads, 0, st>>>(logits, rows, K, targets, mask, count, grad_scale, dl, row_loss); break;
      case 4: ce_kernel<4><<<grid, kRowThreads, 0, st>>>(logits, rows, K, targets, mask, count, grad_scale, dl, row_loss); break;
      case 8: ce_kernel<8><<<grid, kRowThreads, 0, st>>>(logits, rows, K, targets, mask, count, grad_scale, dl, row_loss); break;
      case 16: ce_kernel<16><<<grid, kRowThreads, 0, st>>>(logits, rows, K, targets, mask, count, grad_scale, dl, row_loss); break;
      case 32: ce_kernel<32><<<grid, kRowThreads, 0, st>>>(logits, rows, K, targets, mask, count, grad_scale, dl, row_loss); break;
      default: set_error("cross-entropy: K=%d unsupported", K); return JZ_EINVAL;
    }
    JZ_LAUNCH_CHECK();
  }
  ce_finalize_kernel<<<1, 1024, 0, st>>>(row_loss, rows, count, loss);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_finite_check(const float* g, int64_t n, int* flag, jz_stream_t s) {
  if (n == 0) return JZ_OK;
  finite_check_kernel<<<grid_for(n, 256), 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(g, n, flag);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_adamw_step(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1,
                             float b2, float omb1, float omb2, float bc1, float bc2, float eps, float lrwd,
                             const int* flag, jz_stream_t s) {
  if (n == 0) return JZ_OK;
  adamw_kernel<<<grid_for(n, 256), 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(
      p, g, m, v, n, lr, b1, b2, omb1, omb2, bc1, bc2, eps, lrwd, flag, nullptr);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_adamw_step_dev(float* p, const float* g, float* m, float* v, int64_t n, const float* dev_scalars,
                                 const int* flag, jz_stream_t s) {
  JZ_CHECK_ARG(dev_scalars != nullptr, "adamw: null device scalars");
  if (n == 0) return JZ_OK;
  adamw_kernel<<<grid_for(n, 256), 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(
      p, g, m, v, n, 0.f, 0.f, 0.f, 0.f, 0.f, 1.f, 1.f, 0.f, 0.f, flag, dev_scalars);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}
