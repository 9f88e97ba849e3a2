// Cycles per 64-element softmax exponential chunk (FFMA + ex2.approx + bf16x2 pack, as in the
// spatial forward's exp pass) with 1 or 2 warps per SM sub-partition, and the same with a share of
// the exponentials on the FMA pipe (degree-3 polynomial).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/elr tools/exp_loop_rate.cu && /tmp/elr
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  uint32_t p;
  asm("cvt.rn.bf16x2.f32 %0, %2, %1;" : "=r"(p) : "f"(a), "f"(b));
  return p;
}
// 2^x for x <= 0 on the FMA pipe: round-to-nearest split, cubic on f in [-0.5, 0.5]
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -127.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: integer part in the low mantissa bits
  const float fi = t - 12582912.f;
  const float f = x - fi;
  const float p = fmaf(fmaf(fmaf(0.0555041086648216f, f, 0.2402264923172690f), f, 0.6931471805599453f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

template <int NPOLY>  // exponentials per 64 on the FMA pipe
__global__ void loop_kernel(int iters, unsigned long long* cyc, uint32_t* sink) {
  float v[64];
#pragma unroll
  for (int j = 0; j < 64; ++j) v[j] = -0.01f * (threadIdx.x + j);
  uint32_t acc = 0;
  const float c2 = 0.18033688f, mb = 0.5f;
  __syncthreads();
  const unsigned long long c0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t pk[32];
#pragma unroll
    for (int j = 0; j < 64; j += 2) {
      const float x0 = fmaf(v[j], c2, -mb), x1 = fmaf(v[j + 1], c2, -mb);
      const float p0 = (j < NPOLY) ? ex2_poly(x0) : ex2f(x0);
      const float p1 = (j + 1 < NPOLY) ? ex2_poly(x1) : ex2f(x1);
      pk[j / 2] = pack2(p0, p1);
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) acc ^= pk[j];
#pragma unroll
    for (int j = 0; j < 64; ++j) v[j] = __int_as_float(__float_as_int(v[j]) ^ (acc & 1));
  }
  __syncthreads();
  const unsigned long long c1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  const int iters = 1024;
  for (int warps : {4, 8}) {
    for (int np : {0, 8, 16, 24}) {
      if (np == 0) loop_kernel<0><<<148, warps * 32>>>(iters, cyc, sink);
      if (np == 8) loop_kernel<8><<<148, warps * 32>>>(iters, cyc, sink);
      if (np == 16) loop_kernel<16><<<148, warps * 32>>>(iters, cyc, sink);
      if (np == 24) loop_kernel<24><<<148, warps * 32>>>(iters, cyc, sink);
      cudaDeviceSynchronize();
      unsigned long long h;
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("%d warps/SM (%d per SMSP), %2d of 64 exp2 on the FMA pipe: %.0f cycles per 64-element chunk per warp "
             "(MUFU floor %d)\n", warps, warps / 4, np, (double)h / iters, 8 * (64 - np) * (warps / 4));
    }
  }
  return 0;
}
