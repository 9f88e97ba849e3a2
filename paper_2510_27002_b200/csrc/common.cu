// libjz host plumbing: error text, device check, TMA descriptor encoding.
#include <cudaTypedefs.h>
#include <stdarg.h>
#include <string.h>

#include <atomic>
#include <mutex>

#include "common.h"

#define JZ_STR(x) #x
#define JZ_XSTR(x) JZ_STR(x)

namespace jz {

static thread_local char g_err[1024] = {0};
static std::atomic<unsigned long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode;
}

int make_tmap_2d(CUtensorMap* map, const void* base, int elem_bytes, uint64_t inner, uint64_t outer,
                 uint64_t pitch_elems, uint32_t box_inner, uint32_t box_outer, bool swizzle128) {
  return make_tmap_2d_sw(map, base, elem_bytes, inner, outer, pitch_elems, box_inner, box_outer, swizzle128 ? 128 : 0);
}

int make_tmap_2d_sw(CUtensorMap* map, const void* base, int elem_bytes, uint64_t inner, uint64_t outer,
                    uint64_t pitch_elems, uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
  auto enc = encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return JZ_ECUDA;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {pitch_elems * (uint64_t)elem_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                        : (swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE),
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu pitch=%llu box=%ux%u", (int)r,
              (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)pitch_elems, box_inner,
              box_outer);
    return JZ_ECUDA;
  }
  return JZ_OK;
}

int make_tmap_4d_bf16(CUtensorMap* map, const void* base, const uint64_t dims[4], const uint64_t strides_bytes[3],
                      const uint32_t box[4]) {
  auto enc = encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return JZ_ECUDA;
  }
  cuuint64_t d[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t st[3] = {strides_bytes[0], strides_bytes[1], strides_bytes[2]};
  cuuint32_t bx[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), d, st, bx, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (4d) failed (%d): dims %llu x %llu x %llu x %llu", (int)r,
              (unsigned long long)dims[0], (unsigned long long)dims[1], (unsigned long long)dims[2],
              (unsigned long long)dims[3]);
    return JZ_ECUDA;
  }
  return JZ_OK;
}

int make_tmap_2d_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                      uint64_t pitch_elems, uint32_t box_inner, uint32_t box_outer) {
  return make_tmap_2d(map, base, 2, inner, outer, pitch_elems, box_inner, box_outer);
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n = v > 0 ? v : 148;
  }
  return n;
}

}  // namespace jz

extern "C" const char* jz_last_error(void) { return jz::g_err; }

extern "C" int jz_device_check(int device) {
  int major = 0, minor = 0;
  cudaError_t e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (e != cudaSuccess) {
    jz::set_error("cudaDeviceGetAttribute: %s", cudaGetErrorString(e));
    return JZ_ECUDA;
  }
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  if (major != 10 || minor != 0) {
    jz::set_error("libjz is built for sm_100a only; device %d is sm_%d%d", device, major, minor);
    return JZ_EUNSUPPORTED;
  }
  return JZ_OK;
}

extern "C" const char* jz_build_info(void) {
  return "libjz sm_100a (tcgen05/TMEM/TMA), CUDA " JZ_XSTR(__CUDACC_VER_MAJOR__) "." JZ_XSTR(__CUDACC_VER_MINOR__);
}

extern "C" unsigned long long jz_launch_count(void) { return jz::g_launches.load(std::memory_order_relaxed); }
