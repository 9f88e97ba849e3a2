// Host-side shared plumbing for libjz: status codes, thread-local error text,
// TMA descriptor encoding through the driver entry point (no -lcuda needed).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/jz.h"

namespace jz {

void set_error(const char* fmt, ...);
void count_launch();

#define JZ_CHECK_ARG(cond, ...)        \
  do {                                 \
    if (!(cond)) {                     \
      ::jz::set_error(__VA_ARGS__);    \
      return JZ_EINVAL;                \
    }                                  \
  } while (0)

#define JZ_CUDA_TRY(expr)                                                              \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess) {                                                           \
      ::jz::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return JZ_ECUDA;                                                                 \
    }                                                                                  \
  } while (0)

#define JZ_LAUNCH_CHECK()                                                                      \
  do {                                                                                         \
    ::jz::count_launch();                                                                      \
    cudaError_t _e = cudaGetLastError();                                                       \
    if (_e != cudaSuccess) {                                                                   \
      ::jz::set_error("%s:%d kernel launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return JZ_ECUDA;                                                                         \
    }                                                                                          \
  } while (0)

// 2-D bf16 tensor map: `inner` contiguous elements per row, `outer` rows, row pitch in
// elements; box = box_inner x box_outer with 128-byte swizzle.
int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                      uint64_t pitch_elems, uint32_t box_inner, uint32_t box_outer);
// generic: elem_bytes 2 (bf16) or 4 (f32), 128-byte swizzle
int make_tmap_2d(CUtensorMap* map, const void* base, int elem_bytes, uint64_t inner, uint64_t outer,
                 uint64_t pitch_elems, uint32_t box_inner, uint32_t box_outer, bool swizzle128 = true);

// explicit swizzle span in bytes: 0 (none), 64 or 128
int make_tmap_2d_sw(CUtensorMap* map, const void* base, int elem_bytes, uint64_t inner, uint64_t outer,
                    uint64_t pitch_elems, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes);

// 4-D bf16 tensor map, 128-byte swizzle; strides of dims 1..3 in bytes
int make_tmap_4d_bf16(CUtensorMap* map, const void* base, const uint64_t dims[4], const uint64_t strides_bytes[3],
                      const uint32_t box[4]);

int num_sms();

}  // namespace jz
