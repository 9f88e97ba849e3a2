// The spatial backward's per-unit tcgen05 sequence in isolation (no barriers, no other warps):
// 8 blocks of {4 ts S^T, 4 ts dP^T, 4 ts dV, 4 ts dK, (odd blocks) 8 ss dQ}, with / without commits.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2510_27002_b200/csrc -Iinclude -o /tmp/seq tools/mma_seq.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace jz;

__global__ void __launch_bounds__(128, 1) seq_kernel(int units, int commits, int mode, unsigned long long* cyc, int fences) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar[4];
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
  for (int k = threadIdx.x; k < 160 * 1024 / 4; k += blockDim.x) reinterpret_cast<uint32_t*>(smem)[k] = 0x3c003c00u;
  if (warp == 0) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 0) {
    for (int b = 0; b < 4; ++b) mbar_init(&bar[b], 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, tbase, 0);
  if (warp == 1) {
    constexpr int TILE = 16384;
    const uint32_t dhi = (uint32_t)(sdesc_sw128(0, 0, 1024) >> 32);
    auto dsc = [dhi](uint32_t addr4, uint32_t off, uint32_t lbo) -> uint64_t {
      return ((uint64_t)dhi << 32) | (addr4 + (off >> 4) + ((lbo >> 4) << 16));
    };
    const uint32_t aq = smem_u32(smem) >> 4, ado = smem_u32(smem + 2 * TILE) >> 4, ak = smem_u32(smem + 4 * TILE) >> 4,
                   ads = smem_u32(smem + 6 * TILE) >> 4;
    constexpr uint32_t id_s = idesc_bf16_f32(128, 64, false, false);
    constexpr uint32_t id_kv = idesc_bf16_f32(128, 64, false, true);
    constexpr uint32_t id_q = idesc_bf16_f32(128, 64, true, true);
    const unsigned long long c0 = clock64();
    for (int u = 0; u < units; ++u) {
      for (int x = 0; x < 8; ++x) {
        const int c = x & 3, j = x >> 2;
        const uint32_t sS = tmem + ((x & 1) ? 128 : 0), sP = tmem + 64;
        const uint32_t qoff = (c >> 1) * TILE + (c & 1) * 8192;
        if (mode == 0 || mode == 1) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) umma_bf16_ts_w(sS, tmem + 448 + 8 * kk, dsc(aq, qoff + kk * 32, 16), id_s, kk > 0);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) umma_bf16_ts_w(sP, tmem + 480 + 8 * kk, dsc(ado, qoff + kk * 32, 16), id_s, kk > 0);
          if (commits) umma_commit_w(&bar[0]);
          if (fences) tc_fence_after();
        }
        if (mode == 0 || mode == 2) {
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            umma_bf16_ts_w(tmem + 192, sS + 16 * ks, dsc(ado, qoff + ks * 2048, 8192), id_kv, (c > 0 || ks > 0));
            umma_bf16_ts_w(tmem + 256, sS + 16 * ks + 8, dsc(aq, qoff + ks * 2048, 8192), id_kv, (c > 0 || ks > 0));
          }
          if (c & 1) {
            const int t = c >> 1;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
              umma_bf16_ss_w(tmem + 320 + 64 * t, dsc(ads, 2 * t * TILE + ks * 2048, TILE),
                             dsc(ak, j * TILE + ks * 2048, 8192), id_q, (j > 0 || ks > 0));
            if (commits) umma_commit_w(&bar[1]);
          }
          if (commits && c == 3) umma_commit_w(&bar[2]);
          if (fences) tc_fence_after();
        }
      }
    }
    umma_commit_w(&bar[3]);
    mbar_wait(&bar[3], 0);
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
  cudaFuncSetAttribute(seq_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 161 * 1024);
  const int units = 50;
  const char* names[] = {"full sequence", "S^T/dP^T only", "gradients only"};
  for (int mode = 0; mode < 3; ++mode)
    for (int commits = 0; commits < 4; ++commits) {
      seq_kernel<<<148, 128, 161 * 1024>>>(units, commits & 1, mode, d, commits >> 1);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; }
      unsigned long long h;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      const int mmas = mode == 0 ? 8 * 16 + 4 * 8 : mode == 1 ? 64 : 64 + 32;
      printf("%-16s commits %d fences %d: %.0f cycles per unit, %.1f per MMA\n", names[mode], commits & 1, commits >> 1, (double)h / units,
             (double)h / units / mmas);
    }
  return 0;
}
