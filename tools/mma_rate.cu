// tcgen05.mma issue-to-completion throughput per SM for the operand shapes of the attention kernels.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2510_27002_b200/csrc -o /tmp/mma tools/mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda.h>

#include "ptx.cuh"

using namespace jz;

// mode: 0 ss K/K N=64, 1 ss K/MN N=64, 2 ss MN/MN N=64, 3 ts A-TMEM / B MN N=64, 4 ss K/K N=256, 5 ss K/K N=128,
//       6 ts A-TMEM / B K N=64, 7 ss K/K N=16
__global__ void __launch_bounds__(128, 1) mma_kernel(int mode, int iters, unsigned long long* cyc, int nacc, int variant) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < 65536 / 4; k += blockDim.x) reinterpret_cast<uint32_t*>(smem)[k] = 0x3c003c00u;
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 1) {
    const uint32_t a4 = smem_u32(smem) >> 4, b4 = smem_u32(smem + 32768) >> 4;
    const uint32_t dhi = (uint32_t)(sdesc_sw128(0, 0, 1024) >> 32);
    auto dsc = [dhi](uint32_t addr4, uint32_t off, uint32_t lbo) -> uint64_t {
      return ((uint64_t)dhi << 32) | (addr4 + (off >> 4) + ((lbo >> 4) << 16));
    };
    const uint32_t N = mode == 4 ? 256 : mode == 5 ? 128 : mode == 7 ? 16 : 64;
    const bool amn = mode == 2, bmn = mode == 1 || mode == 2 || mode == 3;
    const uint32_t idesc = idesc_bf16_f32(128, N, amn, bmn);
    uint64_t ads[4], bds[4];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      ads[ks] = amn ? dsc(a4, ks * 2048, 16384) : dsc(a4, ks * 32, 16);
      bds[ks] = bmn ? dsc(b4, ks * 2048, 8192) : dsc(b4, ks * 32, 16);
    }
    const unsigned long long c0 = clock64();
    if (variant == 1) {
      uint32_t e;
      asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(e));
      if (e) {
        for (int it = 0; it < iters; ++it) {
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            const uint32_t dcol = 256 + (uint32_t)((ks % nacc) * N);
            if (mode == 3 || mode == 6)
              umma_bf16_ts(tmem + dcol, tmem + 8 * ks, bds[ks], idesc, 1);
            else
              umma_bf16_ss(tmem + dcol, ads[ks], bds[ks], idesc, 1);
          }
        }
      }
      __syncwarp();
    } else {
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) {
          const uint32_t dcol = 256 + (uint32_t)((ks % 4) * (mode == 4 ? 0 : N));
          if (mode == 3 || mode == 6)
            umma_bf16_ts_w(tmem + dcol, tmem + 8 * ks, variant == 2 ? bds[ks] : (bmn ? dsc(b4, ks * 2048, 8192) : dsc(b4, ks * 32, 16)), idesc, 1);
          else
            umma_bf16_ss_w(tmem + dcol, variant == 2 ? ads[ks] : (amn ? dsc(a4, ks * 2048, 16384) : dsc(a4, ks * 32, 16)),
                           variant == 2 ? bds[ks] : (bmn ? dsc(b4, ks * 2048, 8192) : dsc(b4, ks * 32, 16)), idesc, 1);
        }
      }
    }
    umma_commit_w(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long c1 = clock64();
    if (lane_id() == 0 && blockIdx.x == 0) *cyc = c1 - c0;
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  const char* names[] = {"ss K/K   N=64 ", "ss K/MN  N=64 ", "ss MN/MN N=64 ", "ts -/MN  N=64 ",
                         "ss K/K   N=256", "ss K/K   N=128", "ts -/K   N=64 ", "ss K/K   N=16 "};
  const int iters = 2000;
  for (int mode = 0; mode < 8; ++mode) {
    for (int nacc : {1, 2, 4}) {
      const int variant = 1;
      if (mode == 4 && nacc > 1) continue;
      if (mode == 5 && nacc > 2) continue;
      const int grid = 148;
      mma_kernel<<<grid, 128, 66 * 1024>>>(mode, iters, d, nacc, variant);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
      unsigned long long h;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      const double n = mode == 4 ? 256 : mode == 5 ? 128 : mode == 7 ? 16 : 64;
      const double per = (double)h / (iters * 4);
      printf("%s single-thread issue, %d accumulators: %.1f cycles per K=16 MMA (ideal %.0f), %.0f flop/cycle\n", names[mode], nacc, per,
             128.0 * n / 256.0, 2.0 * 128 * n * 16 / per);
    }
  }
  return 0;
}
