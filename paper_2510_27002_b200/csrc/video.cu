// Pixel/latent-side kernels of the tokenizer and latent action model (all HBM-bound):
//   K9  frames_to_unit + patchify        (tokenizer.py:49-51, nn.py:113-121)
//       unpatchify + unit_to_frames     (nn.py:124-131, tokenizer.py:54-55; round half-even)
//   token assembly: (+ prepended action token) + spatial + temporal positions, fwd/bwd
//       (tokenizer.py:113-119, lam.py:86-90, lam.py:108-113)
//   K10 mean-pool over patches           (lam.py:92-93)
//   K15 recon MSE fwd/bwd                (nn.py:50-53, tokenizer.py:139, lam.py:125)
//   small fp32 linear (CUDA cores) for the 32-wide latent projections whose outputs feed
//       argmins (lam.py:94, lam.py:109) — too small for tensor-core tiles
#include <mutex>

#include "common.h"
#include "ptx.cuh"

namespace jz {

static int grid_of(int64_t n, int threads, int per_sm = 8) {
  int64_t b = (n + threads - 1) / threads;
  int64_t cap = (int64_t)num_sms() * per_sm;
  return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

// out[(bt*N + n)][(ph*P + pw)*C + c] = unit(frames[bt][gh*P+ph][gw*P+pw][c]),  n = gh*GW + gw
__global__ void patchify_kernel(const void* __restrict__ frames, int is_u8, int64_t BT, int H, int W, int C, int P,
                                __nv_bfloat16* __restrict__ out, float* __restrict__ out32) {
  const int GW = W / P, N = (H / P) * GW, PD = P * P * C;
  const int64_t total = BT * N * PD;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / PD;
    const int col = (int)(e - row * PD);
    const int64_t bt = row / N;
    const int n = (int)(row - bt * N);
    const int gh = n / GW, gw = n - gh * GW;
    const int ph = col / (P * C), rem = col - ph * P * C, pw = rem / C, c = rem - pw * C;
    const int64_t src = ((bt * H + gh * P + ph) * W + gw * P + pw) * C + c;
    float v;
    if (is_u8)
      v = (float)reinterpret_cast<const uint8_t*>(frames)[src] / 127.5f - 1.0f;
    else
      v = reinterpret_cast<const float*>(frames)[src];
    if (out) out[e] = __float2bfloat16_rn(v);
    if (out32) out32[e] = v;
  }
}

__global__ void unpatchify_kernel(const float* __restrict__ patches, int64_t BT, int H, int W, int C, int P,
                                  float* __restrict__ unit, uint8_t* __restrict__ u8) {
  const int GW = W / P, N = (H / P) * GW, PD = P * P * C;
  const int64_t total = BT * H * W * C;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t bt = e / ((int64_t)H * W * C);
    int64_t r = e - bt * H * W * C;
    const int y = (int)(r / (W * C));
    r -= (int64_t)y * W * C;
    const int x = (int)(r / C), c = (int)(r - x * C);
    const int n = (y / P) * GW + x / P;
    const int col = ((y % P) * P + (x % P)) * C + c;
    const float v = patches[(bt * N + n) * PD + col];
    if (unit) unit[e] = v;
    if (u8) {
      float f = (v + 1.0f) * 127.5f;
      f = fminf(fmaxf(f, 0.0f), 255.0f);
      u8[e] = (uint8_t)rintf(f);
    }
  }
}

// x[(b,t,s)] = ((e + ps[s]) + pt[t]);  prepend: s = 0 takes act[b,t], s >= 1 takes emb[b,t,s-1]
__global__ void assemble_fwd_kernel(const float* __restrict__ emb, const float* __restrict__ act,
                                    const float* __restrict__ ps, const float* __restrict__ pt, int T, int N, int D,
                                    int prepend, float* __restrict__ x) {
  const int S = N + prepend;
  const int64_t row = blockIdx.x;
  const int s = (int)(row % S);
  const int64_t bt = row / S;
  const int t = (int)(bt % T);
  const float* src = (prepend && s == 0) ? act + bt * D : emb + (bt * N + (s - prepend)) * D;
  for (int d = threadIdx.x * 4; d < D; d += blockDim.x * 4) {
    float4 v = *reinterpret_cast<const float4*>(src + d);
    const float4 a = *reinterpret_cast<const float4*>(ps + (int64_t)s * D + d);
    const float4 b = *reinterpret_cast<const float4*>(pt + (int64_t)t * D + d);
    v.x = (v.x + a.x) + b.x; v.y = (v.y + a.y) + b.y; v.z = (v.z + a.z) + b.z; v.w = (v.w + a.w) + b.w;
    *reinterpret_cast<float4*>(x + row * D + d) = v;
  }
}

// d_emb (bf16, compact rows s >= prepend) and d_act (f32, rows s == 0) from dx
__global__ void assemble_split_kernel(const float* __restrict__ dx, int N, int D, int prepend,
                                      __nv_bfloat16* __restrict__ demb, float* __restrict__ dact) {
  const int S = N + prepend;
  const int64_t row = blockIdx.x;
  const int s = (int)(row % S);
  const int64_t bt = row / S;
  for (int d = threadIdx.x * 4; d < D; d += blockDim.x * 4) {
    const float4 v = *reinterpret_cast<const float4*>(dx + row * D + d);
    if (prepend && s == 0) {
      if (dact) *reinterpret_cast<float4*>(dact + bt * D + d) = v;
    } else if (demb) {
      *reinterpret_cast<uint2*>(demb + (bt * N + (s - prepend)) * D + d) =
          make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
    }
  }
}

// positions: dps[s] = sum_{t,b} dx[b,t,s];  part_pt[s][t] = sum_b dx[b,t,s]
__global__ void pos_bwd_kernel(const float* __restrict__ dx, int64_t B, int T, int S, int D, float* __restrict__ dps,
                               float* __restrict__ part_pt) {
  const int s = blockIdx.x;
  for (int d = threadIdx.x * 4; d < D; d += blockDim.x * 4) {
    float4 acc_s = make_float4(0, 0, 0, 0);
    for (int t = 0; t < T; ++t) {
      float4 acc_t = make_float4(0, 0, 0, 0);
      for (int64_t b0 = 0; b0 < B; b0 += 4) {
        float4 g[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          g[q] = (b0 + q < B) ? *reinterpret_cast<const float4*>(dx + (((b0 + q) * T + t) * S + s) * D + d)
                              : make_float4(0, 0, 0, 0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc_t.x += g[q].x; acc_t.y += g[q].y; acc_t.z += g[q].z; acc_t.w += g[q].w;
        }
      }
      *reinterpret_cast<float4*>(part_pt + ((int64_t)s * T + t) * D + d) = acc_t;
      acc_s.x += acc_t.x; acc_s.y += acc_t.y; acc_s.z += acc_t.z; acc_s.w += acc_t.w;
    }
    if (dps) *reinterpret_cast<float4*>(dps + (int64_t)s * D + d) = acc_s;
  }
}

// pooled[bt] = mean_n x[bt*N + n]  (fixed order, 4-way ILP with ordered sums)
__global__ void mean_pool_kernel(const float* __restrict__ x, int N, int D, float* __restrict__ out) {
  const int64_t bt = blockIdx.x;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float s = 0.f;
    const float* p = x + bt * N * D + d;
    int n = 0;
    for (; n + 4 <= N; n += 4) {
      const float a = p[(int64_t)n * D], b = p[(int64_t)(n + 1) * D], c = p[(int64_t)(n + 2) * D],
                  e = p[(int64_t)(n + 3) * D];
      s += a; s += b; s += c; s += e;
    }
    for (; n < N; ++n) s += p[(int64_t)n * D];
    out[bt * D + d] = s / (float)N;
  }
}

// dx[bt*N + n] = dpool[bt] / N  (fp32, optional accumulate)
__global__ void mean_pool_bwd_kernel(const float* __restrict__ dpool, int64_t rows, int N, int D,
                                     float* __restrict__ dx) {
  const int64_t total = rows * D;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / D;
    const int d = (int)(e - r * D);
    dx[e] = dpool[(r / N) * D + d] / (float)N;
  }
}

// MSE: per-CTA partial sums of (pred - target)^2 (f64), grad = scale * 2 (pred - target) / n
__global__ void mse_kernel(const float* __restrict__ pred, const float* __restrict__ target, int64_t n,
                           double* __restrict__ part, float gscale, float* __restrict__ grad32,
                           __nv_bfloat16* __restrict__ grad16) {
  double acc = 0.0;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t a = blockIdx.x * per, b = min(n, a + per);
  for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
    const float d = pred[i] - target[i];
    acc += (double)(d * d);
    const float g = gscale * (2.0f * d);
    if (grad32) grad32[i] = g;
    if (grad16) grad16[i] = __float2bfloat16_rn(g);
  }
  __shared__ double sm[256];
  sm[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)blockDim.x; ++i) t += sm[i];
    part[blockIdx.x] = t;
  }
}

// per-CTA f64 partial sums of x (fixed chunking)
__global__ void sum_kernel(const float* __restrict__ x, int64_t n, double* __restrict__ part) {
  double acc = 0.0;
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t a = blockIdx.x * per, b = min(n, a + per);
  for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) acc += (double)x[i];
  __shared__ double sm[256];
  sm[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)blockDim.x; ++i) t += sm[i];
    part[blockIdx.x] = t;
  }
}

__global__ void sum_parts_kernel(const double* __restrict__ part, int nparts, double scale, float* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < nparts; ++i) t += part[i];
    *out = (float)(t * scale);
  }
}

// y[r][j] = sum_k x[r][k] W[k][j] + b[j]   (fp32, one thread per output, sequential k)
__global__ void linear_f32_kernel(const float* __restrict__ x, int64_t R, int K, const float* __restrict__ W, int N,
                                  const float* __restrict__ b, float* __restrict__ y, int accumulate) {
  const int64_t total = R * N;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / N;
    const int j = (int)(e - r * N);
    float s = 0.f;
    for (int k = 0; k < K; ++k) s += x[r * K + k] * W[(int64_t)k * N + j];
    if (b) s += b[j];
    y[e] = accumulate ? y[e] + s : s;
  }
}

// N = 32 (the latent projections, K up to 512): W lives in shared memory, lane j owns output
// column j, a warp computes 4 rows at a time from broadcast float4 reads of x.  Per output the sum
// runs over k in order, bit-identical to linear_f32_kernel.
constexpr int kLinN32Rows = 4;
// TRANS: W is stored [32][K] (dx = dy W^T of a 32 -> K projection) and staged as its transpose.
template <bool TRANS>
__global__ void __launch_bounds__(256) linear_f32_n32_kernel(const float* __restrict__ x, int64_t R, int K,
                                                             const float* __restrict__ W, const float* __restrict__ b,
                                                             float* __restrict__ y, int accumulate) {
  extern __shared__ float sW[];  // [K][32]
  if (TRANS) {
    for (int e = threadIdx.x; e < K * 32; e += blockDim.x) sW[(e % K) * 32 + e / K] = W[e];
  } else {
    for (int e = threadIdx.x * 4; e < K * 32; e += blockDim.x * 4)
      *reinterpret_cast<float4*>(sW + e) = *reinterpret_cast<const float4*>(W + e);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const float bias = b ? b[lane] : 0.f;
  const int64_t groups = (R + kLinN32Rows - 1) / kLinN32Rows;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t gidx = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); gidx < groups; gidx += nw) {
    const int64_t r0 = gidx * kLinN32Rows;
    const float* xr[kLinN32Rows];
#pragma unroll
    for (int j = 0; j < kLinN32Rows; ++j) xr[j] = x + min(r0 + j, R - 1) * K;
    float acc[kLinN32Rows];
#pragma unroll
    for (int j = 0; j < kLinN32Rows; ++j) acc[j] = 0.f;
#pragma unroll 2
    for (int k = 0; k < K; k += 4) {
      float4 xv[kLinN32Rows];
#pragma unroll
      for (int j = 0; j < kLinN32Rows; ++j) xv[j] = __ldg(reinterpret_cast<const float4*>(xr[j] + k));
      const float w0 = sW[(k + 0) * 32 + lane], w1 = sW[(k + 1) * 32 + lane];
      const float w2 = sW[(k + 2) * 32 + lane], w3 = sW[(k + 3) * 32 + lane];
#pragma unroll
      for (int j = 0; j < kLinN32Rows; ++j) {
        acc[j] = fmaf(xv[j].x, w0, acc[j]);
        acc[j] = fmaf(xv[j].y, w1, acc[j]);
        acc[j] = fmaf(xv[j].z, w2, acc[j]);
        acc[j] = fmaf(xv[j].w, w3, acc[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < kLinN32Rows; ++j) {
      const int64_t r = r0 + j;
      if (r < R) {
        float* dst = y + r * 32 + lane;
        const float v = acc[j] + bias;
        *dst = accumulate ? *dst + v : v;
      }
    }
  }
}

// N = 32 forward, row-per-lane: a warp owns 32 rows (lane = row) and all 32 outputs of each in
// registers.  x is staged per warp through shared memory in 32-column chunks (coalesced 512-byte
// row segments in, padded rows so the per-lane column reads are conflict-free), and W [K][32] is
// read as broadcast float4s: 9 shared loads per 32 FFMA (the warp-per-4-rows kernel above issued 8
// loads per 16).  Per output the sum still runs over k in order with fmaf: bit-identical.
constexpr int kLinV2Warps = 8;
constexpr int kLinV2Kc = 16;             // x columns staged per step
constexpr int kLinV2Pad = kLinV2Kc + 1;  // padded staging rows: conflict-free column reads
constexpr int kLinV2Rows = 64;  // rows per warp: lane owns rows lane and lane + 32
__global__ void __launch_bounds__(32 * kLinV2Warps) linear_f32_n32_rows_kernel(
    const float* __restrict__ x, int64_t R, int K, const float* __restrict__ W, const float* __restrict__ b,
    float* __restrict__ y, int accumulate) {
  extern __shared__ float smem[];
  float* sW = smem;                                  // [K][32]
  float* sx = smem + (int64_t)K * 32;                // [warps][64 rows][kLinV2Pad]
  for (int e = threadIdx.x * 4; e < K * 32; e += blockDim.x * 4)
    *reinterpret_cast<float4*>(sW + e) = *reinterpret_cast<const float4*>(W + e);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* xs = sx + warp * kLinV2Rows * kLinV2Pad;
  const int64_t groups = (R + kLinV2Rows - 1) / kLinV2Rows;
  for (int64_t gidx = (int64_t)blockIdx.x * kLinV2Warps + warp; gidx < groups; gidx += (int64_t)gridDim.x * kLinV2Warps) {
    const int64_t r0 = gidx * kLinV2Rows;
    float a0[32], a1[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) a0[j] = a1[j] = 0.f;
    for (int k0 = 0; k0 < K; k0 += kLinV2Kc) {
      // stage x[r0 .. r0+63][k0 .. k0+15]: each instruction moves 8 rows x 64 bytes
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rr = (lane >> 2) + 8 * i;
        const int64_t row = r0 + rr < R ? r0 + rr : R - 1;
        const float4 v = __ldg(reinterpret_cast<const float4*>(x + row * K + k0) + (lane & 3));
        float* d = xs + rr * kLinV2Pad + 4 * (lane & 3);
        d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
      }
      __syncwarp();
#pragma unroll 2
      for (int kk = 0; kk < kLinV2Kc; ++kk) {
        const float x0 = xs[lane * kLinV2Pad + kk], x1 = xs[(lane + 32) * kLinV2Pad + kk];
        const float4* wr = reinterpret_cast<const float4*>(sW + (k0 + kk) * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 w = wr[q];
          a0[4 * q] = fmaf(x0, w.x, a0[4 * q]);
          a0[4 * q + 1] = fmaf(x0, w.y, a0[4 * q + 1]);
          a0[4 * q + 2] = fmaf(x0, w.z, a0[4 * q + 2]);
          a0[4 * q + 3] = fmaf(x0, w.w, a0[4 * q + 3]);
          a1[4 * q] = fmaf(x1, w.x, a1[4 * q]);
          a1[4 * q + 1] = fmaf(x1, w.y, a1[4 * q + 1]);
          a1[4 * q + 2] = fmaf(x1, w.z, a1[4 * q + 2]);
          a1[4 * q + 3] = fmaf(x1, w.w, a1[4 * q + 3]);
        }
      }
    }
    // out: lane holds rows lane and lane + 32 (32 outputs each): write them as two 16-column halves
    // transposed through the staging tile, so every store instruction covers 64-byte row segments
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
      __syncwarp();
#pragma unroll
      for (int j = 0; j < kLinV2Kc; ++j) {
        const float bj = b ? b[16 * hf + j] : 0.f;
        xs[lane * kLinV2Pad + j] = a0[16 * hf + j] + bj;
        xs[(lane + 32) * kLinV2Pad + j] = a1[16 * hf + j] + bj;
      }
      __syncwarp();
#pragma unroll 4
      for (int i = 0; i < kLinV2Rows / 2; ++i) {  // 2 rows x 16 columns per instruction
        const int rr = 2 * i + (lane >> 4);
        const int64_t r = r0 + rr;
        if (r < R) {
          float* dst = y + r * 32 + 16 * hf + (lane & 15);
          const float v = xs[rr * kLinV2Pad + (lane & 15)];
          *dst = accumulate ? *dst + v : v;
        }
      }
    }
  }
}

// dx = dy W^T for a K -> 32 projection (W [K][32], the latent projections' input gradient): W staged
// transposed in shared memory, one warp per row with lane j holding dy[r][j] (shuffle-broadcast),
// lane l computing columns l + 32 q.  Per output the sum runs over j in order (as linear_f32_dx_kernel).
__global__ void __launch_bounds__(256) linear_f32_dx_in32_kernel(const float* __restrict__ dy, int64_t R, int K,
                                                                const float* __restrict__ W,
                                                                float* __restrict__ dx, int accumulate) {
  extern __shared__ float sWT[];  // [32][K]
  for (int e = threadIdx.x; e < K * 32; e += blockDim.x) sWT[(e % 32) * K + e / 32] = W[e];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < R; r += nw) {
    const float dv = dy[r * 32 + lane];
    for (int q0 = 0; q0 < K; q0 += 32 * 8) {
      float acc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc[u] = 0.f;
#pragma unroll 4
      for (int j = 0; j < 32; ++j) {
        const float dj = __shfl_sync(0xffffffffu, dv, j);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int k = q0 + 32 * u + lane;
          if (k < K) acc[u] = fmaf(dj, sWT[j * K + k], acc[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = q0 + 32 * u + lane;
        if (k < K) {
          float* dst = dx + r * K + k;
          *dst = accumulate ? *dst + acc[u] : acc[u];
        }
      }
    }
  }
}

// dW partials of y = x W (+ b) when one side is 32 wide: CTA c sums the rows [c RC, (c + 1) RC) into
// part[c] = x_c^T dy_c ([K][N]) and, when db is wanted, bpart[c] = column sums of dy_c ([N]).  Threads
// own big-dim indices (t, t + 256, ...) and all 32 small-dim indices; rows are staged 16 at a time.
// jz_reduce_partials then folds the chunks in index order (deterministic).
constexpr int kDwRowsPerCta = 256;
constexpr int kDwStage = 16;
template <int BPT>
__global__ void __launch_bounds__(256) linear_f32_dw_part_kernel(const float* __restrict__ x,
                                                                const float* __restrict__ dy, int64_t R, int K,
                                                                int N, int k_big, float* __restrict__ part,
                                                                float* __restrict__ bpart) {
  extern __shared__ float sm[];
  const int Bg = k_big ? K : N;
  float* sbig = sm;                     // [kDwStage][Bg]
  float* ssm = sm + kDwStage * Bg;      // [kDwStage][32]
  const float* big = k_big ? x : dy;
  const float* small = k_big ? dy : x;
  float acc[BPT][32];
#pragma unroll
  for (int i = 0; i < BPT; ++i)
#pragma unroll
    for (int s = 0; s < 32; ++s) acc[i][s] = 0.f;
  float bsum[BPT];  // column sums of dy: columns t + 256 i
#pragma unroll
  for (int i = 0; i < BPT; ++i) bsum[i] = 0.f;
  const int64_t r0 = (int64_t)blockIdx.x * kDwRowsPerCta;
  const int64_t r1 = min(R, r0 + kDwRowsPerCta);
  for (int64_t rb = r0; rb < r1; rb += kDwStage) {
    const int nr = (int)min((int64_t)kDwStage, r1 - rb);
    __syncthreads();
    for (int e = threadIdx.x; e < nr * Bg; e += blockDim.x) sbig[e] = big[rb * Bg + e];
    for (int e = threadIdx.x; e < nr * 32; e += blockDim.x) ssm[e] = small[rb * 32 + e];
    __syncthreads();
    for (int rr = 0; rr < nr; ++rr) {
      float sv[32];
#pragma unroll
      for (int s = 0; s < 32; s += 4) {
        const float4 f = *reinterpret_cast<const float4*>(ssm + rr * 32 + s);
        sv[s] = f.x; sv[s + 1] = f.y; sv[s + 2] = f.z; sv[s + 3] = f.w;
      }
#pragma unroll
      for (int i = 0; i < BPT; ++i) {
        const int b = threadIdx.x + 256 * i;
        if (b < Bg) {
          const float bv = sbig[rr * Bg + b];
#pragma unroll
          for (int s = 0; s < 32; ++s) acc[i][s] = fmaf(bv, sv[s], acc[i][s]);
        }
      }
      if (bpart != nullptr) {
#pragma unroll
        for (int i = 0; i < BPT; ++i) {
          const int j = threadIdx.x + 256 * i;
          if (j < N) bsum[i] += k_big ? ssm[rr * 32 + j] : sbig[rr * Bg + j];
        }
      }
    }
  }
  float* pc = part + (int64_t)blockIdx.x * K * N;
#pragma unroll
  for (int i = 0; i < BPT; ++i) {
    const int b = threadIdx.x + 256 * i;
    if (b < Bg) {
#pragma unroll
      for (int s = 0; s < 32; ++s) {
        if (k_big) pc[(int64_t)b * N + s] = acc[i][s];
        else pc[(int64_t)s * N + b] = acc[i][s];
      }
    }
  }
  if (bpart != nullptr) {
#pragma unroll
    for (int i = 0; i < BPT; ++i) {
      const int j = threadIdx.x + 256 * i;
      if (j < N) bpart[(int64_t)blockIdx.x * N + j] = bsum[i];
    }
  }
}

// dx[r][k] = sum_j dy[r][j] W[k][j]
__global__ void linear_f32_dx_kernel(const float* __restrict__ dy, int64_t R, int N, const float* __restrict__ W,
                                     int K, float* __restrict__ dx, int accumulate) {
  const int64_t total = R * K;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / K;
    const int k = (int)(e - r * K);
    float s = 0.f;
    for (int j = 0; j < N; ++j) s += dy[r * N + j] * W[(int64_t)k * N + j];
    dx[e] = accumulate ? dx[e] + s : s;
  }
}

// dW[k][j] = sum_r x[r][k] dy[r][j];  db[j] = sum_r dy[r][j]   (one thread per output, fixed order)
__global__ void linear_f32_dw_kernel(const float* __restrict__ x, const float* __restrict__ dy, int64_t R, int K, int N,
                                     float* __restrict__ dW, float* __restrict__ db, int accumulate) {
  const int64_t total = (int64_t)K * N + (db ? N : 0);
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    if (e < (int64_t)K * N) {
      const int k = (int)(e / N), j = (int)(e - (int64_t)k * N);
      float s = 0.f;
      for (int64_t r = 0; r < R; ++r) s += x[r * K + k] * dy[r * N + j];
      dW[e] = accumulate ? dW[e] + s : s;
    } else {
      const int j = (int)(e - (int64_t)K * N);
      float s = 0.f;
      for (int64_t r = 0; r < R; ++r) s += dy[r * N + j];
      db[j] = accumulate ? db[j] + s : s;
    }
  }
}

}  // namespace jz

using namespace jz;

extern "C" int jz_patchify(const void* frames, int is_u8, int64_t BT, int H, int W, int C, int P, void* out_bf16,
                           float* out_f32, jz_stream_t s) {
  JZ_CHECK_ARG(P > 0 && H % P == 0 && W % P == 0, "geometry %dx%d not divisible by patch %d", H, W, P);
  const int64_t total = BT * H * W * C;
  if (total == 0) return JZ_OK;
  patchify_kernel<<<grid_of(total, 256), 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(
      frames, is_u8, BT, H, W, C, P, reinterpret_cast<__nv_bfloat16*>(out_bf16), out_f32);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_unpatchify(const float* patches, int64_t BT, int H, int W, int C, int P, float* unit,
                             uint8_t* frames_u8, jz_stream_t s) {
  JZ_CHECK_ARG(P > 0 && H % P == 0 && W % P == 0, "patch grid does not match target geometry");
  const int64_t total = BT * H * W * C;
  if (total == 0) return JZ_OK;
  unpatchify_kernel<<<grid_of(total, 256), 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(patches, BT, H, W, C, P,
                                                                                         unit, frames_u8);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_assemble_fwd(const float* emb, const float* act, const float* pos_spatial, const float* pos_temporal,
                               int64_t B, int T, int N, int D, int prepend, float* x, jz_stream_t s) {
  JZ_CHECK_ARG(D % 4 == 0, "assemble: D %% 4");
  const int64_t rows = B * T * (N + prepend);
  if (rows == 0) return JZ_OK;
  assemble_fwd_kernel<<<(unsigned)rows, 128, 0, reinterpret_cast<cudaStream_t>(s)>>>(emb, act, pos_spatial,
                                                                                     pos_temporal, T, N, D, prepend, x);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int64_t jz_assemble_bwd_workspace(int64_t B, int T, int N, int D, int prepend) {
  return (int64_t)(N + prepend) * T * D;
}

extern "C" int jz_assemble_bwd(const float* dx, int64_t B, int T, int N, int D, int prepend, void* d_emb_bf16,
                               float* d_act, float* d_pos_spatial, float* d_pos_temporal, float* workspace,
                               jz_stream_t s) {
  JZ_CHECK_ARG(D % 4 == 0, "assemble_bwd: D %% 4");
  auto st = reinterpret_cast<cudaStream_t>(s);
  const int S = N + prepend;
  const int64_t rows = B * T * S;
  if (rows == 0) return JZ_OK;
  if (d_emb_bf16 || d_act) {
    assemble_split_kernel<<<(unsigned)rows, 128, 0, st>>>(dx, N, D, prepend,
                                                          reinterpret_cast<__nv_bfloat16*>(d_emb_bf16), d_act);
    JZ_LAUNCH_CHECK();
  }
  if (d_pos_spatial || d_pos_temporal) {
    pos_bwd_kernel<<<S, 128, 0, st>>>(dx, B, T, S, D, d_pos_spatial, workspace);
    JZ_LAUNCH_CHECK();
    if (d_pos_temporal) {
      int rc = jz_reduce_partials(workspace, S, (int64_t)T * D, d_pos_temporal, 0, s);
      if (rc) return rc;
    }
  }
  return JZ_OK;
}

extern "C" int jz_mean_pool(const float* x, int64_t BT, int N, int D, float* out, jz_stream_t s) {
  if (BT == 0) return JZ_OK;
  mean_pool_kernel<<<(unsigned)BT, 128, 0, reinterpret_cast<cudaStream_t>(s)>>>(x, N, D, out);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_mean_pool_bwd(const float* dpool, int64_t BT, int N, int D, float* dx, jz_stream_t s) {
  const int64_t n = BT * N * D;
  if (n == 0) return JZ_OK;
  mean_pool_bwd_kernel<<<grid_of(n, 256), 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(dpool, BT * N, N, D, dx);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_mse(const float* pred, const float* target, int64_t n, float grad_scale, float* loss, float* grad32,
                      void* grad16, double* workspace, jz_stream_t s) {
  auto st = reinterpret_cast<cudaStream_t>(s);
  const int parts = num_sms() * 2;
  mse_kernel<<<parts, 256, 0, st>>>(pred, target, n, workspace, n > 0 ? grad_scale / (float)n : 0.f, grad32,
                                    reinterpret_cast<__nv_bfloat16*>(grad16));
  JZ_LAUNCH_CHECK();
  sum_parts_kernel<<<1, 32, 0, st>>>(workspace, parts, n > 0 ? 1.0 / (double)n : 0.0, loss);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_sum(const float* x, int64_t n, double scale, float* out, double* workspace, jz_stream_t s) {
  auto st = reinterpret_cast<cudaStream_t>(s);
  const int parts = num_sms() * 2;
  sum_kernel<<<parts, 256, 0, st>>>(x, n, workspace);
  JZ_LAUNCH_CHECK();
  sum_parts_kernel<<<1, 32, 0, st>>>(workspace, parts, scale, out);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_linear_f32(const float* x, int64_t R, int K, const float* W, int N, const float* b, float* y,
                             int accumulate, jz_stream_t s) {
  const int64_t n = R * N;
  if (n == 0) return JZ_OK;
  if (N == 32 && K % 32 == 0 && K <= 1024 && ((uintptr_t)x % 16) == 0 && ((uintptr_t)W % 16) == 0) {
    const size_t smem = (size_t)K * 32 * sizeof(float) + (size_t)kLinV2Warps * kLinV2Rows * kLinV2Pad * sizeof(float);
    static std::once_flag once2;
    static cudaError_t attr_err2 = cudaSuccess;
    std::call_once(once2, [] {
      attr_err2 = cudaFuncSetAttribute(linear_f32_n32_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       1024 * 32 * 4 + kLinV2Warps * kLinV2Rows * kLinV2Pad * 4);
    });
    JZ_CUDA_TRY(attr_err2);
    int64_t grid = (R + kLinV2Rows * kLinV2Warps - 1) / (kLinV2Rows * kLinV2Warps);
    if (grid > (int64_t)num_sms() * 2) grid = (int64_t)num_sms() * 2;  // two CTAs per SM
    linear_f32_n32_rows_kernel<<<(unsigned)grid, 32 * kLinV2Warps, smem, reinterpret_cast<cudaStream_t>(s)>>>(
        x, R, K, W, b, y, accumulate);
  } else if (N == 32 && K % 4 == 0 && K <= 1024 && ((uintptr_t)x % 16) == 0 && ((uintptr_t)W % 16) == 0) {
    const size_t smem = (size_t)K * 32 * sizeof(float);
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
      attr_err = cudaFuncSetAttribute(linear_f32_n32_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 * 32 * 4);
    });
    JZ_CUDA_TRY(attr_err);
    int64_t grid = (R + 8 * kLinN32Rows - 1) / (8 * kLinN32Rows);
    if (grid > (int64_t)num_sms() * 2) grid = (int64_t)num_sms() * 2;
    linear_f32_n32_kernel<false><<<(unsigned)grid, 256, smem, reinterpret_cast<cudaStream_t>(s)>>>(x, R, K, W, b, y, accumulate);
  } else {
    linear_f32_kernel<<<grid_of(n, 256), 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(x, R, K, W, N, b, y, accumulate);
  }
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int64_t jz_linear_f32_bwd_workspace(int64_t R, int K, int N) {
  if (!((K == 32 && N <= 1024) || (N == 32 && K <= 1024))) return 0;
  const int64_t chunks = (R + kDwRowsPerCta - 1) / kDwRowsPerCta;
  return chunks * ((int64_t)K * N + N);
}

extern "C" int jz_reduce_partials(const float* part, int nparts, int64_t D, float* out, int accumulate,
                                  jz_stream_t s);

extern "C" int jz_linear_f32_bwd_ws(const float* x, const float* dy, int64_t R, int K, int N, const float* W,
                                    float* dx, float* dW, float* db, int accumulate, float* workspace,
                                    int64_t workspace_floats, jz_stream_t s) {
  auto st = reinterpret_cast<cudaStream_t>(s);
  const int64_t need = jz_linear_f32_bwd_workspace(R, K, N);
  const bool a16 = ((uintptr_t)x % 16) == 0 && ((uintptr_t)dy % 16) == 0;
  if (need == 0 || workspace == nullptr || workspace_floats < need || R == 0 || !a16)
    return jz_linear_f32_bwd(x, dy, R, K, N, W, dx, dW, db, accumulate, s);
  if (dx) {
    int64_t grid = (R + 7) / 8;
    if (grid > (int64_t)num_sms() * 4) grid = (int64_t)num_sms() * 4;
    const size_t smem = (size_t)K * 32 * sizeof(float);
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [] {
      attr_err = cudaFuncSetAttribute(linear_f32_dx_in32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      1024 * 32 * 4);
      if (attr_err == cudaSuccess)
        attr_err = cudaFuncSetAttribute(linear_f32_n32_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        1024 * 32 * 4);
    });
    JZ_CUDA_TRY(attr_err);
    if (N == 32) {  // dx [R][K] = dy [R][32] W^T
      linear_f32_dx_in32_kernel<<<(unsigned)grid, 256, smem, st>>>(dy, R, K, W, dx, 0);
    } else {        // K == 32: dx [R][32] = dy [R][N] W^T with W [32][N]
      int64_t g2 = (R + 8 * kLinN32Rows - 1) / (8 * kLinN32Rows);
      if (g2 > (int64_t)num_sms() * 2) g2 = (int64_t)num_sms() * 2;
      linear_f32_n32_kernel<true><<<(unsigned)g2, 256, (size_t)N * 32 * sizeof(float), st>>>(dy, R, N, W, nullptr,
                                                                                            dx, 0);
    }
    JZ_LAUNCH_CHECK();
  }
  if (dW) {
    const int chunks = (int)((R + kDwRowsPerCta - 1) / kDwRowsPerCta);
    const int Bg = N == 32 ? K : N;
    const int k_big = N == 32 ? 1 : 0;
    float* part = workspace;
    float* bpart = db ? workspace + (int64_t)chunks * K * N : nullptr;
    const size_t smem = (size_t)kDwStage * (Bg + 32) * sizeof(float);
    if (Bg <= 256)
      linear_f32_dw_part_kernel<1><<<chunks, 256, smem, st>>>(x, dy, R, K, N, k_big, part, bpart);
    else if (Bg <= 512)
      linear_f32_dw_part_kernel<2><<<chunks, 256, smem, st>>>(x, dy, R, K, N, k_big, part, bpart);
    else
      linear_f32_dw_part_kernel<4><<<chunks, 256, smem, st>>>(x, dy, R, K, N, k_big, part, bpart);
    JZ_LAUNCH_CHECK();
    int rc = jz_reduce_partials(part, chunks, (int64_t)K * N, dW, accumulate, s);
    if (rc) return rc;
    if (db) {
      rc = jz_reduce_partials(bpart, chunks, N, db, accumulate, s);
      if (rc) return rc;
    }
  }
  return JZ_OK;
}

extern "C" int jz_linear_f32_bwd(const float* x, const float* dy, int64_t R, int K, int N, const float* W, float* dx,
                                 float* dW, float* db, int accumulate, jz_stream_t s) {
  auto st = reinterpret_cast<cudaStream_t>(s);
  if (dx && R * K > 0) {
    linear_f32_dx_kernel<<<grid_of(R * K, 256), 256, 0, st>>>(dy, R, N, W, K, dx, 0);
    JZ_LAUNCH_CHECK();
  }
  if (dW) {
    const int64_t n = (int64_t)K * N + (db ? N : 0);
    linear_f32_dw_kernel<<<grid_of(n, 128), 128, 0, st>>>(x, dy, R, K, N, dW, db, accumulate);
    JZ_LAUNCH_CHECK();
  }
  return JZ_OK;
}
