// FFMA throughput microbenchmark (fp32 FMA pipe peak of this B200): 8 independent FMA chains per
// thread, enough warps to fill every scheduler.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0.001f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.f) out[blockIdx.x] = s;
}
int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* out;
  cudaMalloc(&out, 1 << 20);
  const int iters = 4096, threads = 1024, blocks = sms * 2;
  ffma_kernel<<<blocks, threads>>>(out, 64, 0.999f, 0.001f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  ffma_kernel<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
  printf("{\"ffma_tflops\": %.1f, \"ms\": %.3f, \"sms\": %d}\n", flops / (ms * 1e-3) / 1e12, ms, sms);
  return 0;
}
