// Layout check: tcgen05.cp.128x256b of a 128-row x 64-bf16 K-major SW128 smem tile into TMEM, read back
// with tcgen05.ld.32x32b; lane m / column c should hold the bf16 pair (k = 2c, 2c + 1) of row m.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2510_27002_b200/csrc -Iinclude -o /tmp/cpk tools/tcgen05_cp_check.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace jz;

__global__ void cp_kernel(uint32_t* out, int* bad) {
  __shared__ __align__(1024) uint8_t tile[16384];
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // element (m, k) = m * 64 + k as bf16 bits of small ints is awkward; store a tag in the raw 16 bits:
  // tag = (m << 6) | k (fits 13 bits), written at the SW128 position of (m, k)
  for (int e = threadIdx.x; e < 128 * 64; e += blockDim.x) {
    const int m = e >> 6, k = e & 63;
    const int chunk = k >> 3, within = k & 7;
    const uint32_t off = m * 128 + ((chunk ^ (m & 7)) << 4) + within * 2;
    *reinterpret_cast<uint16_t*>(tile + off) = (uint16_t)((m << 6) | k);
  }
  if (warp == 0) tmem_alloc<128>(&tbase);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp == 1) {
    const uint32_t a4 = smem_u32(tile) >> 4;
    const uint32_t dhi = (uint32_t)(sdesc_sw128(0, 0, 1024) >> 32);
    if (lane == 0) {
      for (int kk = 0; kk < 4; ++kk) {
        const uint64_t d = ((uint64_t)dhi << 32) | (a4 + ((kk * 32) >> 4) + ((16 >> 4) << 16));
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + 8 * kk), "l"(d));
      }
      umma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp < 4) {
    uint32_t v[32];
    tmem_ld_32x32b_x32(tmem + ((warp * 32) << 16), v);
    tmem_ld_wait();
    const int m = warp * 32 + lane;
    int nb = 0;
    for (int c = 0; c < 32; ++c) {
      const uint32_t want = (uint32_t)((m << 6) | (2 * c)) | ((uint32_t)((m << 6) | (2 * c + 1)) << 16);
      out[m * 32 + c] = v[c];
      nb += v[c] != want;
    }
    atomicAdd(bad, nb);
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

int main() {
  uint32_t* out;
  int* bad;
  cudaMalloc(&out, 128 * 32 * 4);
  cudaMalloc(&bad, 4);
  cudaMemset(bad, 0, 4);
  cp_kernel<<<1, 128>>>(out, bad);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
  int h;
  cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost);
  uint32_t o[8];
  cudaMemcpy(o, out, 32, cudaMemcpyDeviceToHost);
  printf("mismatching words: %d of 4096; row 0 cols 0..3: %08x %08x %08x %08x\n", h, o[0], o[1], o[2], o[3]);
  uint32_t o1[4];
  cudaMemcpy(o1, out + 9 * 32, 16, cudaMemcpyDeviceToHost);
  printf("row 9 cols 0..3: %08x %08x %08x %08x\n", o1[0], o1[1], o1[2], o1[3]);
  return 0;
}
