// Issue rates of the softmax building blocks per SM per cycle: ex2.approx (MUFU), cvt.rn.bf16x2.f32
// (F2FP pack), FFMA, and a degree-3 polynomial exp2 on the FMA pipe.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/xu tools/xu_rate.cu && /tmp/xu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void rate_kernel(int iters, unsigned long long* cyc, float* sink) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 0.001f * (threadIdx.x + k);
  uint32_t u = 0;
  __syncthreads();
  const unsigned long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) {
        float y;
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(a[k]));
        a[k] = y * -0.5f;  // keep it bounded; one FMUL per ex2
      } else if (OP == 1) {
        uint32_t p;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "f"(a[k]), "f"(a[(k + 1) & 7]));
        u ^= p;
        a[k] += 1.0f;
      } else if (OP == 2) {
        a[k] = fmaf(a[k], 0.999f, 0.001f);
      } else {
        // 2^x for x <= 0: split integer/fraction, cubic on the fraction (FMA pipe only)
        float x = fmaxf(a[k], -126.f);
        float fi = floorf(x);
        float f = x - fi;
        float p = fmaf(fmaf(fmaf(0.0555041086648216f, f, 0.2402264923172690f), f, 0.6931471805599453f), f, 1.0f);
        a[k] = __int_as_float(__float_as_int(p) + ((int)fi << 23)) - 1.5f;
      }
    }
  }
  __syncthreads();
  const unsigned long long c1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)u;
}

int main() {
  unsigned long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  const int iters = 2048;
  const char* names[] = {"ex2.approx (+FMUL)", "cvt.rn.bf16x2.f32 (+FADD)", "FFMA", "poly exp2 (FMA pipe)"};
  for (int op = 0; op < 4; ++op) {
    for (int warps : {8, 16, 32}) {
      if (op == 0) rate_kernel<0><<<148, warps * 32>>>(iters, cyc, sink);
      if (op == 1) rate_kernel<1><<<148, warps * 32>>>(iters, cyc, sink);
      if (op == 2) rate_kernel<2><<<148, warps * 32>>>(iters, cyc, sink);
      if (op == 3) rate_kernel<3><<<148, warps * 32>>>(iters, cyc, sink);
      cudaDeviceSynchronize();
      unsigned long long h;
      cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double ops = (double)warps * 32 * iters * 8;
      printf("%-28s warps %2d: %.1f ops/cycle/SM\n", names[op], warps, ops / h);
    }
  }
  return 0;
}
