// K8: vector quantizer shared by the video tokenizer (K = 1024 codes) and the latent
// action model (K = 6), forward and backward.  Replaces tokenizer.vq_quantize
// (tokenizer.py:58-79) and its autodiff backward.
//
//   d2[k]  = (|z|^2 - (2z).c_k) + |c_k|^2           fp32 on CUDA cores (FFMA), as tokenizer.py:69-71
//   idx    = argmin_k d2[k], lowest index on ties    (np.argmin, tokenizer.py:72)
//   z_q_st = z + (c_idx - z)                         straight-through value (tokenizer.py:78)
//   sq_err = sum (c_idx - z)^2 per row               -> codebook and commitment losses (both mse)
// Distances stay fp32 on CUDA cores: a bf16 tensor-core distance would flip argmins
// (SURVEY §7.4.4).  Backward:
//   dz   = g_zq_st + commit_coef * (z - c_idx)
//   dcb[k] = cb_coef * sum_{rows: idx = k} (c_k - z)   deterministic owner-computes scatter
#include "common.h"
#include "ptx.cuh"

namespace jz {

template <int DZ>
__global__ void __launch_bounds__(256) vq_fwd_kernel(const float* __restrict__ z, int64_t rows,
                                                     const float* __restrict__ cb, int K, int64_t* __restrict__ idx,
                                                     float* __restrict__ zq_st, float* __restrict__ row_sq) {
  constexpr int kVqChunk = DZ >= 64 ? 128 : 256;  // codes staged in shared memory per pass
  __shared__ float sc[kVqChunk][DZ + 1];
  __shared__ float scc[kVqChunk];
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = r < rows;
  float zr[DZ];
  float zz = 0.f;
#pragma unroll
  for (int i = 0; i < DZ; ++i) {
    zr[i] = valid ? z[r * DZ + i] : 0.f;
    zz += zr[i] * zr[i];
  }
  float best = INFINITY;
  int bi = 0;
  for (int k0 = 0; k0 < K; k0 += kVqChunk) {
    const int kn = min(kVqChunk, K - k0);
    __syncthreads();
    for (int e = threadIdx.x; e < kn * DZ; e += blockDim.x) sc[e / DZ][e % DZ] = cb[(int64_t)k0 * DZ + e];
    __syncthreads();
    for (int k = threadIdx.x; k < kn; k += blockDim.x) {
      float cc = 0.f;
#pragma unroll
      for (int i = 0; i < DZ; ++i) cc += sc[k][i] * sc[k][i];
      scc[k] = cc;
    }
    __syncthreads();
    for (int k = 0; k < kn; ++k) {
      float dot = 0.f;
#pragma unroll
      for (int i = 0; i < DZ; ++i) dot += (2.0f * zr[i]) * sc[k][i];
      const float d2 = (zz - dot) + scc[k];
      if (d2 < best) {
        best = d2;
        bi = k0 + k;
      }
    }
  }
  if (!valid) return;
  idx[r] = bi;
  float se = 0.f;
#pragma unroll
  for (int i = 0; i < DZ; ++i) {
    const float q = cb[(int64_t)bi * DZ + i];
    const float diff = q - zr[i];
    se += diff * diff;
    if (zq_st) zq_st[r * DZ + i] = zr[i] + diff;
  }
  if (row_sq) row_sq[r] = se;
}

// DZ % 4 == 0: codes staged unpadded (every lane reads the same code -> broadcast float4 reads) and
// two codes per step as independent FMA chains; each distance keeps the sequential i order of
// vq_fwd_kernel and codes are compared in index order, so the result is bit-identical.
template <int DZ>
__global__ void __launch_bounds__(256) vq_fwd4_kernel(const float* __restrict__ z, int64_t rows,
                                                      const float* __restrict__ cb, int K, int64_t* __restrict__ idx,
                                                      float* __restrict__ zq_st, float* __restrict__ row_sq) {
  constexpr int kChunk = DZ >= 64 ? 128 : 256;
  constexpr int V = DZ / 4;
  __shared__ float4 sc[kChunk * V];
  __shared__ float scc[kChunk];
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool valid = r < rows;
  float zr[DZ], z2[DZ];
  float zz = 0.f;
#pragma unroll
  for (int i = 0; i < DZ; ++i) {
    zr[i] = valid ? z[r * DZ + i] : 0.f;
    zz += zr[i] * zr[i];
    z2[i] = 2.0f * zr[i];
  }
  float best = INFINITY;
  int bi = 0;
  for (int k0 = 0; k0 < K; k0 += kChunk) {
    const int kn = min(kChunk, K - k0);
    __syncthreads();
    for (int e = threadIdx.x; e < kn * V; e += blockDim.x)
      sc[e] = *reinterpret_cast<const float4*>(cb + (int64_t)k0 * DZ + 4 * e);
    __syncthreads();
    for (int k = threadIdx.x; k < kn; k += blockDim.x) {
      float cc = 0.f;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const float4 c4 = sc[k * V + v];
        cc += c4.x * c4.x; cc += c4.y * c4.y; cc += c4.z * c4.z; cc += c4.w * c4.w;
      }
      scc[k] = cc;
    }
    __syncthreads();
    int k = 0;
    for (; k + 1 < kn; k += 2) {
      float d0 = 0.f, d1 = 0.f;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const float4 a = sc[k * V + v], c = sc[(k + 1) * V + v];
        d0 += z2[4 * v] * a.x; d0 += z2[4 * v + 1] * a.y; d0 += z2[4 * v + 2] * a.z; d0 += z2[4 * v + 3] * a.w;
        d1 += z2[4 * v] * c.x; d1 += z2[4 * v + 1] * c.y; d1 += z2[4 * v + 2] * c.z; d1 += z2[4 * v + 3] * c.w;
      }
      const float e0 = (zz - d0) + scc[k], e1 = (zz - d1) + scc[k + 1];
      if (e0 < best) { best = e0; bi = k0 + k; }
      if (e1 < best) { best = e1; bi = k0 + k + 1; }
    }
    if (k < kn) {
      float d0 = 0.f;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const float4 a = sc[k * V + v];
        d0 += z2[4 * v] * a.x; d0 += z2[4 * v + 1] * a.y; d0 += z2[4 * v + 2] * a.z; d0 += z2[4 * v + 3] * a.w;
      }
      const float e0 = (zz - d0) + scc[k];
      if (e0 < best) { best = e0; bi = k0 + k; }
    }
  }
  if (!valid) return;
  idx[r] = bi;
  float se = 0.f;
#pragma unroll
  for (int i = 0; i < DZ; ++i) {
    const float q = cb[(int64_t)bi * DZ + i];
    const float diff = q - zr[i];
    se += diff * diff;
    if (zq_st) zq_st[r * DZ + i] = zr[i] + diff;
  }
  if (row_sq) row_sq[r] = se;
}

// R rows per thread (rows r, r + 256, .. of the CTA's 256 R), CP codes per step: every staged code
// is read from shared memory once for R rows, so the broadcast loads no longer bound the FFMA pipe
// (one LDS.128 per 4 R FFMAs instead of four). Each (row, code) distance keeps vq_fwd_kernel's
// sequential i order and codes are compared in index order per row, so the result is
// bit-identical. 2 z_i is kept instead of z_i (z_i = 0.5 * (2 z_i) exactly).
template <int DZ, int R, int CP, int kChunk>
__global__ void __launch_bounds__(256, R >= 4 ? 1 : 2) vq_fwd4r_kernel(const float* __restrict__ z, int64_t rows,
                                                                       const float* __restrict__ cb, int K,
                                                                       int64_t* __restrict__ idx,
                                                                       float* __restrict__ zq_st,
                                                                       float* __restrict__ row_sq) {
  constexpr int V = DZ / 4;
  extern __shared__ float4 vq_smem[];  // kChunk codes (float4 x V each), then kChunk squared norms
  float4* sc = vq_smem;
  float* scc = reinterpret_cast<float*>(vq_smem + kChunk * V);
  const int64_t rb = (int64_t)blockIdx.x * (256 * R) + threadIdx.x;
  float z2[R][DZ];
  float zz[R];
#pragma unroll
  for (int h = 0; h < R; ++h) {
    const int64_t r = rb + 256 * h;
    zz[h] = 0.f;
#pragma unroll
    for (int i = 0; i < DZ; ++i) {
      const float x = r < rows ? z[r * DZ + i] : 0.f;
      zz[h] += x * x;
      z2[h][i] = 2.0f * x;
    }
  }
  float best[R];
  int bi[R];
#pragma unroll
  for (int h = 0; h < R; ++h) {
    best[h] = INFINITY;
    bi[h] = 0;
  }
  for (int k0 = 0; k0 < K; k0 += kChunk) {
    const int kn = min(kChunk, K - k0);
    __syncthreads();
    for (int e = threadIdx.x; e < kn * V; e += blockDim.x)
      sc[e] = *reinterpret_cast<const float4*>(cb + (int64_t)k0 * DZ + 4 * e);
    __syncthreads();
    for (int k = threadIdx.x; k < kn; k += blockDim.x) {
      float cc = 0.f;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const float4 c4 = sc[k * V + v];
        cc += c4.x * c4.x; cc += c4.y * c4.y; cc += c4.z * c4.z; cc += c4.w * c4.w;
      }
      scc[k] = cc;
    }
    __syncthreads();
    int k = 0;
    for (; k + CP <= kn; k += CP) {
      float d[CP][R];  // codes k .. k + CP - 1 x rows
#pragma unroll
      for (int c = 0; c < CP; ++c)
#pragma unroll
        for (int h = 0; h < R; ++h) d[c][h] = 0.f;
#pragma unroll
      for (int v = 0; v < V; ++v) {
#pragma unroll
        for (int c = 0; c < CP; ++c) {
          const float4 p = sc[(k + c) * V + v];
#pragma unroll
          for (int h = 0; h < R; ++h) {
            d[c][h] += z2[h][4 * v] * p.x; d[c][h] += z2[h][4 * v + 1] * p.y;
            d[c][h] += z2[h][4 * v + 2] * p.z; d[c][h] += z2[h][4 * v + 3] * p.w;
          }
        }
      }
#pragma unroll
      for (int c = 0; c < CP; ++c) {
        const float cc = scc[k + c];
#pragma unroll
        for (int h = 0; h < R; ++h) {
          const float e = (zz[h] - d[c][h]) + cc;
          if (e < best[h]) { best[h] = e; bi[h] = k0 + k + c; }
        }
      }
    }
    for (; k < kn; ++k) {
      float d0[R];
#pragma unroll
      for (int h = 0; h < R; ++h) d0[h] = 0.f;
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const float4 p = sc[k * V + v];
#pragma unroll
        for (int h = 0; h < R; ++h) {
          d0[h] += z2[h][4 * v] * p.x; d0[h] += z2[h][4 * v + 1] * p.y;
          d0[h] += z2[h][4 * v + 2] * p.z; d0[h] += z2[h][4 * v + 3] * p.w;
        }
      }
#pragma unroll
      for (int h = 0; h < R; ++h) {
        const float e0 = (zz[h] - d0[h]) + scc[k];
        if (e0 < best[h]) { best[h] = e0; bi[h] = k0 + k; }
      }
    }
  }
#pragma unroll
  for (int h = 0; h < R; ++h) {
    const int64_t r = rb + 256 * h;
    if (r >= rows) continue;
    idx[r] = bi[h];
    float se = 0.f;
#pragma unroll
    for (int i = 0; i < DZ; ++i) {
      const float zi = 0.5f * z2[h][i];
      const float q = cb[(int64_t)bi[h] * DZ + i];
      const float diff = q - zi;
      se += diff * diff;
      if (zq_st) zq_st[r * DZ + i] = zi + diff;
    }
    if (row_sq) row_sq[r] = se;
  }
}


// dz = g + commit_coef * (z - c_idx)
__global__ void vq_bwd_z_kernel(const float* __restrict__ z, const float* __restrict__ cb,
                                const int64_t* __restrict__ idx, const float* __restrict__ g, int64_t rows, int dz,
                                float commit_coef, float* __restrict__ dzout) {
  const int64_t total = rows * dz;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / dz;
    const int i = (int)(e - r * dz);
    const float q = cb[idx[r] * dz + i];
    dzout[e] = (g ? g[e] : 0.f) + commit_coef * (z[e] - q);
  }
}

// dcb[k] = cb_coef * sum_{r: idx[r]=k} (c_k - z_r); CTA c owns codes k = c, c+G, ...; warp w scans a fixed
// row range in order (lane = latent column, dz <= 64), warps summed in order.
constexpr int kVqOwn = 8;
__global__ void __launch_bounds__(256) vq_bwd_cb_kernel(const float* __restrict__ z, const float* __restrict__ cb,
                                                        const int64_t* __restrict__ idx, int64_t rows, int K, int dz,
                                                        float cb_coef, float* __restrict__ dcb) {
  const int G = gridDim.x, c = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float acc[kVqOwn][2];
  int cnt[kVqOwn];
#pragma unroll
  for (int j = 0; j < kVqOwn; ++j) {
    acc[j][0] = acc[j][1] = 0.f;
    cnt[j] = 0;
  }
  const int64_t per = (rows + 7) / 8;
  const int64_t p0 = warp * per, p1 = min(rows, p0 + per);
  for (int64_t base = p0; base < p1; base += 32) {
    const int64_t r = base + lane;
    const int64_t k = r < p1 ? idx[r] : -1;
    const bool mine = k >= 0 && (k % G) == c;
    unsigned bal = __ballot_sync(0xffffffffu, mine);
    while (bal) {
      const int src = __ffs(bal) - 1;
      bal &= bal - 1;
      const int64_t kk = __shfl_sync(0xffffffffu, k, src);
      const int64_t rr = base + src;
      const int j = (int)(kk / G);
#pragma unroll
      for (int jj = 0; jj < kVqOwn; ++jj)
        if (jj == j) {
          if (lane < dz) acc[jj][0] += -z[rr * dz + lane];
          if (lane + 32 < dz) acc[jj][1] += -z[rr * dz + lane + 32];
          cnt[jj] += 1;
        }
    }
  }
  __shared__ float sm[8][64];
  __shared__ int scnt[8];
  for (int j = 0; j < kVqOwn; ++j) {
    const int k = c + j * G;
    if (k >= K) break;
    sm[warp][lane] = acc[j][0];
    sm[warp][lane + 32] = acc[j][1];
    if (lane == 0) scnt[warp] = cnt[j];
    __syncthreads();
    if (threadIdx.x < dz) {
      float s = 0.f;
      int n = 0;
      for (int w = 0; w < 8; ++w) {
        s += sm[w][threadIdx.x];
        n += scnt[w];
      }
      // sum_r (c_k - z_r) = n * c_k + sum_r (-z_r)
      dcb[(int64_t)k * dz + threadIdx.x] = cb_coef * ((float)n * cb[(int64_t)k * dz + threadIdx.x] + s);
    }
    __syncthreads();
  }
}

}  // namespace jz

using namespace jz;

extern "C" int jz_vq_fwd(const float* z, int64_t rows, int dz, const float* codebook, int K, int64_t* idx,
                         float* zq_st, float* row_sq, jz_stream_t s) {
  JZ_CHECK_ARG(K >= 1, "empty codebook");
  JZ_CHECK_ARG(dz == 8 || dz == 16 || dz == 32 || dz == 64, "vq: latent dim %d unsupported (8/16/32/64)", dz);
  if (rows == 0) return JZ_OK;
  const unsigned grid = (unsigned)((rows + 255) / 256);
  auto st = reinterpret_cast<cudaStream_t>(s);
  switch (dz) {
    case 8: vq_fwd_kernel<8><<<grid, 256, 0, st>>>(z, rows, codebook, K, idx, zq_st, row_sq); break;
    case 16: vq_fwd_kernel<16><<<grid, 256, 0, st>>>(z, rows, codebook, K, idx, zq_st, row_sq); break;
    case 32:
      // several rows per thread while that still gives about a CTA per SM; one row for small batches
      if (((uintptr_t)codebook % 16) == 0 && rows >= (int64_t)num_sms() * 1024 * 7 / 8) {
        vq_fwd4r_kernel<32, 4, 4, 256><<<(unsigned)((rows + 1023) / 1024), 256, 256 * (32 * 4 + 4), st>>>(
            z, rows, codebook, K, idx, zq_st, row_sq);
      } else if (((uintptr_t)codebook % 16) == 0 && rows >= (int64_t)num_sms() * 512)
        vq_fwd4r_kernel<32, 2, 2, 256><<<(unsigned)((rows + 511) / 512), 256, 256 * (32 * 4 + 4), st>>>(
            z, rows, codebook, K, idx, zq_st, row_sq);
      else if (((uintptr_t)codebook % 16) == 0) vq_fwd4_kernel<32><<<grid, 256, 0, st>>>(z, rows, codebook, K, idx, zq_st, row_sq);
      else vq_fwd_kernel<32><<<grid, 256, 0, st>>>(z, rows, codebook, K, idx, zq_st, row_sq);
      break;
    default: vq_fwd_kernel<64><<<grid, 256, 0, st>>>(z, rows, codebook, K, idx, zq_st, row_sq); break;
  }
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_vq_bwd(const float* z, const float* codebook, const int64_t* idx, const float* g_zq_st, int64_t rows,
                         int dz, int K, float commit_coef, float cb_coef, float* dz_out, float* dcodebook,
                         jz_stream_t s) {
  JZ_CHECK_ARG(dz <= 64, "vq_bwd: latent dim %d unsupported", dz);
  auto st = reinterpret_cast<cudaStream_t>(s);
  if (dz_out && rows > 0) {
    const int64_t n = rows * dz;
    int64_t b = (n + 255) / 256;
    if (b > (int64_t)num_sms() * 8) b = (int64_t)num_sms() * 8;
    vq_bwd_z_kernel<<<(unsigned)b, 256, 0, st>>>(z, codebook, idx, g_zq_st, rows, dz, commit_coef, dz_out);
    JZ_LAUNCH_CHECK();
  }
  if (dcodebook) {
    int G = (K + kVqOwn - 1) / kVqOwn;
    if (G < num_sms()) G = K < num_sms() ? K : num_sms();
    JZ_CHECK_ARG((K + G - 1) / G <= kVqOwn, "vq_bwd: codebook too large");
    vq_bwd_cb_kernel<<<G, 256, 0, st>>>(z, codebook, idx, rows, K, dz, cb_coef, dcodebook);
    JZ_LAUNCH_CHECK();
  }
  return JZ_OK;
}
