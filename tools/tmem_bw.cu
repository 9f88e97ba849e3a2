// TMEM -> register load bandwidth per SM (tcgen05.ld.32x32b.x32 + wait), by warps per CTA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_bw tools/tmem_bw.cu && /tmp/tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int X>
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t* r);

template <>
__device__ __forceinline__ void ld32<32>(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

__global__ void tmem_bw_kernel(int iters, unsigned long long* cycles, float* sink, int cstride, int wrap, int wmask_lo, int wmask_hi) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = base + (((warp & 3) * 32) << 16) + ((cstride * (warp >> 2)) % wrap);
  uint32_t r[32];
  float acc = 0.f;
  __syncthreads();
  const unsigned long long c0 = clock64();
  const bool active = warp >= wmask_lo && warp < wmask_hi;
  for (int i = 0; i < iters && active; ++i) {
    ld32<32>(t, r);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    uint32_t x = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) x ^= r[j];
    acc += __uint_as_float(x);
  }
  __syncthreads();
  const unsigned long long c1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = c1 - c0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

int main() {
  unsigned long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  const int iters = 4096;
  int cfg[][5] = {{4, 32, 512, 0, 4}, {16, 0, 512, 0, 16}, {16, 32, 512, 0, 16}, {20, 32, 512, 0, 20}, {24, 32, 512, 0, 24}, {32, 32, 512, 0, 32},
                  {32, 32, 512, 0, 16}, {32, 32, 512, 16, 32}, {32, 32, 512, 0, 8}, {32, 32, 512, 8, 16},
                  {8, 32, 512, 0, 8}, {32, 32, 512, 0, 4}, {32, 32, 512, 16, 20}};
  for (auto& c : cfg) {
    const int warps = c[0];
    printf("active warps [%2d,%2d) of ", c[3], c[4]);
    tmem_bw_kernel<<<148, warps * 32>>>(iters, cyc, sink, c[1], c[2], c[3], c[4]);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    unsigned long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double bytes = (double)(c[4] - c[3]) * iters * 32 * 32 * 4;
    printf("warps %2d: %.1f bytes/cycle/SM (%.0f cycles per x32 warp-load)\n", warps, bytes / h[0],
           (double)h[0] / iters);
  }
  return 0;
}
