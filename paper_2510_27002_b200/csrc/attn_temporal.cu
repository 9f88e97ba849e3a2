// K4: causal temporal (inter-frame) attention, forward and backward.
//
// Replaces the temporal sub-layer's attention of st_block (st.py:74-76) =
// multi_head_attention(causal=True) (nn.py:80-110) over the (B, S, T, D) transpose.
// Here nothing is transposed: qkv stays in the (b, t, s) row order the GEMMs
// produce, and one CTA gathers the T rows of one spatial slot (b, s) for all
// heads.  With T = 16 and hd = 64 the arithmetic intensity is ~4 FLOP/B, so the
// kernel is HBM-bound and runs on CUDA cores with 16-byte vectorised I/O
// (SURVEY §2.3 K4); its roofline is HBM bandwidth.
//
// qkv bf16 [M, 3*D] (cols [q | k | v], head h = cols 64h..64h+63 of each),
// out bf16 [M, D], lse f32 [(b*S + s) * H * T + h * T + t].
#include "common.h"
#include "ptx.cuh"

namespace jz {

constexpr int HD = 64;

JZ_DEV void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
JZ_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// 64-element dot / axpy against a bf16 smem row with 16-byte loads
JZ_DEV float dot8x8(const float (&x)[64], const __nv_bfloat16* row) {
  float a = 0.f;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint4 w = reinterpret_cast<const uint4*>(row)[c];
    const float2 f0 = unpack_bf16(w.x), f1 = unpack_bf16(w.y), f2 = unpack_bf16(w.z), f3 = unpack_bf16(w.w);
    a += x[8 * c] * f0.x + x[8 * c + 1] * f0.y + x[8 * c + 2] * f1.x + x[8 * c + 3] * f1.y +
         x[8 * c + 4] * f2.x + x[8 * c + 5] * f2.y + x[8 * c + 6] * f3.x + x[8 * c + 7] * f3.y;
  }
  return a;
}

JZ_DEV void axpy8x8(float (&y)[64], float a, const __nv_bfloat16* row) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint4 w = reinterpret_cast<const uint4*>(row)[c];
    const float2 f0 = unpack_bf16(w.x), f1 = unpack_bf16(w.y), f2 = unpack_bf16(w.z), f3 = unpack_bf16(w.w);
    y[8 * c] += a * f0.x; y[8 * c + 1] += a * f0.y; y[8 * c + 2] += a * f1.x; y[8 * c + 3] += a * f1.y;
    y[8 * c + 4] += a * f2.x; y[8 * c + 5] += a * f2.y; y[8 * c + 6] += a * f3.x; y[8 * c + 7] += a * f3.y;
  }
}

template <int T>
__global__ void __launch_bounds__(256)
    temporal_fwd_kernel(const __nv_bfloat16* __restrict__ qkv, int S, int H, __nv_bfloat16* __restrict__ out,
                        float* __restrict__ lse, float scale) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int D = H * HD;
  const int64_t bs = blockIdx.x;  // b*S + s
  const int64_t b = bs / S, s = bs - b * S;
  __nv_bfloat16* sq = reinterpret_cast<__nv_bfloat16*>(smem_raw);  // [T][3D]
  const int row_u4 = 3 * D / 8;
  for (int i = threadIdx.x; i < T * row_u4; i += blockDim.x) {
    const int t = i / row_u4, c = i - t * row_u4;
    const int64_t row = (b * T + t) * S + s;
    cp_async16(reinterpret_cast<uint4*>(sq + (int64_t)t * 3 * D) + c, reinterpret_cast<const uint4*>(qkv + row * 3 * D) + c);
  }
  cp_async_wait_all();
  __syncthreads();
  const int h = threadIdx.x / T, t = threadIdx.x % T;
  if (h >= H) return;
  const __nv_bfloat16* q = sq + (int64_t)t * 3 * D + h * HD;
  float qf[HD];
#pragma unroll
  for (int d = 0; d < HD; d += 2) {
    float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(q + d));
    qf[d] = f.x; qf[d + 1] = f.y;
  }
  float sc[T];
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < T; ++j) {
    if (j <= t) {
      const __nv_bfloat16* k = sq + (int64_t)j * 3 * D + D + h * HD;
      float a = dot8x8(qf, k);
      sc[j] = a * scale;
      mx = fmaxf(mx, sc[j]);
    } else {
      sc[j] = -INFINITY;
    }
  }
  float sum = 0.f;
#pragma unroll
  for (int j = 0; j < T; ++j) {
    sc[j] = j <= t ? __expf(sc[j] - mx) : 0.f;
    sum += sc[j];
  }
  const float inv = 1.0f / sum;
  float o[HD];
#pragma unroll
  for (int d = 0; d < HD; ++d) o[d] = 0.f;
#pragma unroll
  for (int j = 0; j < T; ++j) {
    if (j <= t) {
      const __nv_bfloat16* v = sq + (int64_t)j * 3 * D + 2 * D + h * HD;
      axpy8x8(o, sc[j] * inv, v);
    }
  }
  const int64_t row = (b * T + t) * S + s;
  uint4* dst = reinterpret_cast<uint4*>(out + row * D + h * HD);
#pragma unroll
  for (int d = 0; d < HD; d += 8)
    dst[d / 8] = make_uint4(pack_bf16(o[d], o[d + 1]), pack_bf16(o[d + 2], o[d + 3]),
                            pack_bf16(o[d + 4], o[d + 5]), pack_bf16(o[d + 6], o[d + 7]));
  lse[(bs * H + h) * T + t] = mx + logf(sum);
}

// Backward.  smem: qkv rows [T][3D], o rows [T][D], do rows [T][D], P and dS [H][T][T].
template <int T>
__global__ void __launch_bounds__(256)
    temporal_bwd_kernel(const __nv_bfloat16* __restrict__ qkv, const __nv_bfloat16* __restrict__ o,
                        const __nv_bfloat16* __restrict__ dout, const float* __restrict__ lse, int S, int H,
                        __nv_bfloat16* __restrict__ dqkv, float scale) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int D = H * HD;
  const int64_t bs = blockIdx.x;
  const int64_t b = bs / S, s = bs - b * S;
  __nv_bfloat16* sq = reinterpret_cast<__nv_bfloat16*>(smem_raw);  // [T][3D]
  __nv_bfloat16* so = sq + (int64_t)T * 3 * D;                     // [T][D]
  __nv_bfloat16* sdo = so + (int64_t)T * D;                        // [T][D]
  float* sp = reinterpret_cast<float*>(sdo + (int64_t)T * D);      // [H][T][T]
  float* sds = sp + H * T * T;                                     // [H][T][T]
  {
    const int row_u4 = 3 * D / 8, row2 = D / 8;
    for (int i = threadIdx.x; i < T * row_u4; i += blockDim.x) {
      const int t = i / row_u4, c = i - t * row_u4;
      const int64_t row = (b * T + t) * S + s;
      cp_async16(reinterpret_cast<uint4*>(sq + (int64_t)t * 3 * D) + c, reinterpret_cast<const uint4*>(qkv + row * 3 * D) + c);
    }
    for (int i = threadIdx.x; i < T * row2; i += blockDim.x) {
      const int t = i / row2, c = i - t * row2;
      const int64_t row = (b * T + t) * S + s;
      cp_async16(reinterpret_cast<uint4*>(so + (int64_t)t * D) + c, reinterpret_cast<const uint4*>(o + row * D) + c);
      cp_async16(reinterpret_cast<uint4*>(sdo + (int64_t)t * D) + c, reinterpret_cast<const uint4*>(dout + row * D) + c);
    }
    cp_async_wait_all();
  }
  __syncthreads();
  const int h = threadIdx.x / T, t = threadIdx.x % T;
  const bool active = h < H;
  if (active) {
    // query role: row t of head h
    float qf[HD], dof[HD];
    float Dt = 0.f;
#pragma unroll
    for (int d = 0; d < HD; d += 2) {
      float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sq + (int64_t)t * 3 * D + h * HD + d));
      float2 g = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(sdo + (int64_t)t * D + h * HD + d));
      float2 w = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(so + (int64_t)t * D + h * HD + d));
      qf[d] = a.x; qf[d + 1] = a.y;
      dof[d] = g.x; dof[d + 1] = g.y;
      Dt += g.x * w.x + g.y * w.y;
    }
    const float L = lse[(bs * H + h) * T + t];
#pragma unroll 1
    for (int j = 0; j < T; ++j) {
      float p = 0.f, ds = 0.f;
      if (j <= t) {
        const __nv_bfloat16* k = sq + (int64_t)j * 3 * D + D + h * HD;
        const __nv_bfloat16* v = sq + (int64_t)j * 3 * D + 2 * D + h * HD;
        const float a = dot8x8(qf, k);
        const float dp = dot8x8(dof, v);
        p = __expf(a * scale - L);
        ds = p * (dp - Dt);
      }
      sp[(h * T + t) * T + j] = p;
      sds[(h * T + t) * T + j] = ds;
    }
    float dq[HD];
#pragma unroll
    for (int d = 0; d < HD; ++d) dq[d] = 0.f;
#pragma unroll 1
    for (int j = 0; j <= t; ++j) axpy8x8(dq, sds[(h * T + t) * T + j], sq + (int64_t)j * 3 * D + D + h * HD);
    const int64_t row = (b * T + t) * S + s;
    uint4* dst = reinterpret_cast<uint4*>(dqkv + row * 3 * D + h * HD);
#pragma unroll
    for (int d = 0; d < HD; d += 8)
      dst[d / 8] = make_uint4(pack_bf16(scale * dq[d], scale * dq[d + 1]), pack_bf16(scale * dq[d + 2], scale * dq[d + 3]),
                              pack_bf16(scale * dq[d + 4], scale * dq[d + 5]), pack_bf16(scale * dq[d + 6], scale * dq[d + 7]));
  }
  __syncthreads();
  if (active) {
    // key role: key j = t of head h
    const int j = t;
    float dk[HD], dv[HD];
#pragma unroll
    for (int d = 0; d < HD; ++d) { dk[d] = 0.f; dv[d] = 0.f; }
    for (int tq = j; tq < T; ++tq) {
      const float p = sp[(h * T + tq) * T + j], ds = sds[(h * T + tq) * T + j];
      axpy8x8(dk, ds, sq + (int64_t)tq * 3 * D + h * HD);
      axpy8x8(dv, p, sdo + (int64_t)tq * D + h * HD);
    }
    const int64_t row = (b * T + j) * S + s;
    uint4* dk_dst = reinterpret_cast<uint4*>(dqkv + row * 3 * D + D + h * HD);
    uint4* dv_dst = reinterpret_cast<uint4*>(dqkv + row * 3 * D + 2 * D + h * HD);
#pragma unroll
    for (int d = 0; d < HD; d += 8) {
      dk_dst[d / 8] = make_uint4(pack_bf16(scale * dk[d], scale * dk[d + 1]), pack_bf16(scale * dk[d + 2], scale * dk[d + 3]),
                                 pack_bf16(scale * dk[d + 4], scale * dk[d + 5]), pack_bf16(scale * dk[d + 6], scale * dk[d + 7]));
      dv_dst[d / 8] = make_uint4(pack_bf16(dv[d], dv[d + 1]), pack_bf16(dv[d + 2], dv[d + 3]),
                                 pack_bf16(dv[d + 4], dv[d + 5]), pack_bf16(dv[d + 6], dv[d + 7]));
    }
  }
}

template <int T>
static int launch_temporal(bool bwd, const void* qkv, const void* o, const void* dout, float* lse, int64_t BS,
                           int S, int H, void* out, float scale, cudaStream_t st) {
  const int D = H * HD;
  const int threads = ((T * H + 31) / 32) * 32 < 128 ? 128 : ((T * H + 31) / 32) * 32;
  if (!bwd) {
    const size_t smem = (size_t)T * 3 * D * 2;
    if (smem > 48 * 1024)
      JZ_CUDA_TRY(cudaFuncSetAttribute(temporal_fwd_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    temporal_fwd_kernel<T><<<(unsigned)BS, threads, smem, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(qkv), S, H, reinterpret_cast<__nv_bfloat16*>(out), lse, scale);
  } else {
    const size_t smem = (size_t)T * 5 * D * 2 + (size_t)2 * H * T * T * 4;
    if (smem > 48 * 1024)
      JZ_CUDA_TRY(cudaFuncSetAttribute(temporal_bwd_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    temporal_bwd_kernel<T><<<(unsigned)BS, threads, smem, st>>>(
        reinterpret_cast<const __nv_bfloat16*>(qkv), reinterpret_cast<const __nv_bfloat16*>(o),
        reinterpret_cast<const __nv_bfloat16*>(dout), lse, S, H, reinterpret_cast<__nv_bfloat16*>(out), scale);
  }
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

static int dispatch_temporal(bool bwd, const void* qkv, const void* o, const void* dout, float* lse, int64_t B,
                             int T, int S, int H, void* out, cudaStream_t st) {
  JZ_CHECK_ARG(H >= 1 && H * T <= 256, "temporal attention: heads*T=%d too large (<= 256)", H * T);
  const float scale = 0.125f;  // 1/sqrt(64)
  const int64_t BS = B * S;
  if (BS == 0) return JZ_OK;
  switch (T) {
#define TC(n) case n: return launch_temporal<n>(bwd, qkv, o, dout, lse, BS, S, H, out, scale, st);
    TC(1) TC(2) TC(3) TC(4) TC(5) TC(6) TC(7) TC(8) TC(9) TC(10) TC(11) TC(12) TC(13) TC(14) TC(15) TC(16)
#undef TC
    default:
      set_error("temporal attention: T=%d unsupported (<= 16)", T);
      return JZ_EINVAL;
  }
}

}  // namespace jz

using namespace jz;

extern "C" int jz_attn_temporal_fwd(const void* qkv, int64_t B, int T, int S, int H, int head_dim, void* out,
                                    float* lse, jz_stream_t s) {
  JZ_CHECK_ARG(head_dim == 64, "temporal attention: head_dim %d unsupported (64)", head_dim);
  return dispatch_temporal(false, qkv, nullptr, nullptr, lse, B, T, S, H, out, reinterpret_cast<cudaStream_t>(s));
}

extern "C" int jz_attn_temporal_bwd(const void* qkv, const void* out, const void* dout, const float* lse,
                                    int64_t B, int T, int S, int H, int head_dim, void* dqkv, jz_stream_t s) {
  JZ_CHECK_ARG(head_dim == 64, "temporal attention: head_dim %d unsupported (64)", head_dim);
  return dispatch_temporal(true, qkv, out, dout, const_cast<float*>(lse), B, T, S, H, dqkv,
                           reinterpret_cast<cudaStream_t>(s));
}
