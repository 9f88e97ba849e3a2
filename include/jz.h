/*
 * jz.h — C ABI of libjz, the sm_100a (B200) kernels behind the Jasmine/Genie
 * training and sampling hot path.
 *
 * The reference (deskworld, /root/reference/pkg/src/deskworld) is pure numpy and
 * has no FFI of its own: its boundary is the Python module API of
 * deskworld.{nn,st,tokenizer,lam,dynamics,optim,rng}.  Each entry point below
 * names the reference function(s) it replaces (file:line).  The Python mirror in
 * paper_2510_27002_b200/ binds these symbols with ctypes.
 *
 * Conventions
 *  - Every entry point returns 0 (JZ_OK) or a negative JZ_E* status; the
 *    message of the last failure on the calling thread is jz_last_error().
 *  - All pointers are device pointers unless stated; outputs and workspaces are
 *    caller-allocated (libjz never allocates device memory).
 *  - Every call is stream-ordered on the explicit `stream` argument and is
 *    reentrant (no mutable globals besides one-time kernel attribute setup).
 *  - Row-major storage; `ld*` arguments are row pitches in ELEMENTS.
 *  - bf16 buffers are passed as void*; fp32 as float*.
 */
#ifndef JZ_H_
#define JZ_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define JZ_API __attribute__((visibility("default")))

typedef struct CUstream_st* jz_stream_t; /* == cudaStream_t */

enum {
  JZ_OK = 0,
  JZ_EINVAL = -1,       /* shape / config violation  -> ValueError  */
  JZ_EINDEX = -2,       /* id out of range           -> IndexError  */
  JZ_ECUDA = -3,        /* CUDA runtime failure      -> RuntimeError */
  JZ_EUNSUPPORTED = -4, /* not an sm_100 device / unsupported dims */
  JZ_ENONFINITE = -5    /* non-finite gradient (optim.py:48-49) */
};

/* Thread-local text of the last failure. */
JZ_API const char* jz_last_error(void);

/* 0 when `device` is an sm_100 (B200-class) GPU, JZ_EUNSUPPORTED otherwise.
 * Reference: none (the reference is CPU-only). */
JZ_API int jz_device_check(int device);

/* Library build identification (compile-time arch list). */
JZ_API const char* jz_build_info(void);

/* ------------------------------------------------------------------------
 * K1  GEMM  D[M,N] = epilogue( A[M,K] . B[K,N] )   bf16 x bf16 -> fp32 (TMEM)
 * Replaces nn.linear (nn.py:43-47) and the matmul forward/backward of
 * autodiff.Tensor.__matmul__ (autodiff.py:180-193).
 *
 *  A: a_kmajor=1 -> element (m,k) at A[m*lda + k]   (activations X)
 *     a_kmajor=0 -> element (m,k) at A[k*lda + m]   (X^T for weight grads)
 *  B: b_kmajor=1 -> element (k,n) at B[n*ldb + k]   (W^T for input grads)
 *     b_kmajor=0 -> element (k,n) at B[k*ldb + n]   (W (din,dout) as stored)
 *  All bf16.  lda/ldb must be multiples of 8 (16-byte TMA pitch).
 * ---------------------------------------------------------------------- */
enum {
  JZ_EPI_F32 = 0,       /* D f32  = acc (+ bias)                                  */
  JZ_EPI_BF16 = 1,      /* D bf16 = acc (+ bias)                                  */
  JZ_EPI_RESID = 2,     /* D f32  = aux_f32 + acc (+ bias)   (aux may alias D)    */
  JZ_EPI_GELU = 3,      /* D bf16 = gelu(acc + bias); D2 bf16 = acc + bias        */
  JZ_EPI_GELU_BWD = 4,  /* D bf16 = acc * gelu'(aux_bf16)                          */
  JZ_EPI_F32_ACC = 5,   /* D f32 += acc                                           */
  JZ_EPI_BF16_F32 = 6   /* D f32 = acc (+bias); D2 bf16 copy                       */
};

/* Workspace bytes needed for a split-K GEMM (0 when split_k <= 1). */
JZ_API int64_t jz_gemm_workspace_bytes(int64_t M, int64_t N, int split_k);

JZ_API int jz_gemm_bf16(const void* A, int64_t lda, int a_kmajor, const void* B, int64_t ldb,
                 int b_kmajor, void* D, int64_t ldd, int64_t M, int64_t N, int64_t K,
                 int epilogue, const float* bias, const void* aux, int64_t ldaux, void* D2,
                 int64_t ldd2, int split_k, void* workspace, jz_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* JZ_H_ */
