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

/* Number of kernels libjz has launched in this process (all threads). */
JZ_API unsigned long long jz_launch_count(void);

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
  JZ_EPI_GELU = 3,      /* D bf16 = gelu(acc + bias); D2 bf16 = acc + bias (D2 may be NULL) */
  JZ_EPI_GELU_BWD = 4,  /* D bf16 = acc * gelu'(aux_bf16)                          */
  JZ_EPI_F32_ACC = 5,   /* D f32 += acc                                           */
  JZ_EPI_BF16_F32 = 6,  /* D f32 = acc (+bias); D2 bf16 copy                       */
  /* value 7 is reserved (no-store timing probe) */
  JZ_EPI_GELU_DG = 8,   /* D bf16 = gelu(acc + bias); D2 f16 = gelu'(acc + bias) (D2 required):
                           the training forward saves the GELU derivative, not the pre-activation */
  JZ_EPI_MUL_F16 = 9    /* D bf16 = acc * aux_f16 (the backward of JZ_EPI_GELU_DG: aux = its D2) */
};

/* Workspace bytes needed for a split-K GEMM (0 when split_k <= 1). */
JZ_API int64_t jz_gemm_workspace_bytes(int64_t M, int64_t N, int split_k);

JZ_API int jz_gemm_bf16(const void* A, int64_t lda, int a_kmajor, const void* B, int64_t ldb,
                 int b_kmajor, void* D, int64_t ldd, int64_t M, int64_t N, int64_t K,
                 int epilogue, const float* bias, const void* aux, int64_t ldaux, void* D2,
                 int64_t ldd2, int split_k, void* workspace, jz_stream_t stream);

/* Same GEMM (split_k = 1, bf16-output epilogues) that also writes the column sums of its bf16
 * output per 32-row block: colsum_part f32 [jz_gemm_colsum_parts(M)][N].  jz_reduce_partials
 * over those rows gives the bias gradient of the layer that consumes D (autodiff.py:22-32
 * _unbroadcast) without re-reading D.  Needs N % 8 == 0 and N > 64. */
JZ_API int64_t jz_gemm_colsum_parts(int64_t M);
JZ_API int jz_gemm_bf16_colsum(const void* A, int64_t lda, int a_kmajor, const void* B, int64_t ldb,
                               int b_kmajor, void* D, int64_t ldd, int64_t M, int64_t N, int64_t K,
                               int epilogue, const float* bias, const void* aux, int64_t ldaux, void* D2,
                               int64_t ldd2, float* colsum_part, jz_stream_t stream);


/* LayerNorm fused into the K1 GEMM epilogue (nn.layer_norm, nn.py:35-40, and its backward), for
 * N = 512 (one CTA pair computes both 256-column tiles of a 256-row block back to back, so each
 * row's statistics close inside the pair; no separate LayerNorm pass over HBM).
 *
 * jz_gemm_bf16_ln_fwd: the residual projection and the next sub-layer's LayerNorm (st.py:73-79):
 *   D f32 = resid + A.B + bias                       (the residual stream, as JZ_EPI_RESID)
 *   xn bf16 = (D - mean) * rstd * gamma + beta       (two-pass statistics, biased variance, eps)
 *   mean, rstd f32 [M]; skip_period > 0 drops rows r % skip_period == 0 from xn (compacted rows).
 * jz_gemm_bf16_ln_bwd: the input-gradient GEMM of a LayerNorm-fed layer and the LayerNorm backward:
 *   dy = A.B (gradient of xn); dres f32 (+)= LN_bwd(dy; x, mean, rstd, gamma); dres_bf16 copy (may be
 *   NULL); dgamma = sum dy*xhat, dbeta = sum dy, dbias = sum dres (column sums, each may be NULL),
 *   reduced deterministically from `part` f32 [3][nparts][512], nparts = jz_gemm_ln_bwd_parts(M).
 * A must be K-major (activations); b_kmajor as in jz_gemm_bf16. */
JZ_API int jz_gemm_bf16_ln_fwd(const void* A, int64_t lda, int a_kmajor, const void* B, int64_t ldb, int b_kmajor,
                               float* D, int64_t ldd, int64_t M, int64_t N, int64_t K, const float* bias,
                               const float* resid, int64_t ld_resid, const float* gamma, const float* beta,
                               float eps, void* xn_bf16, float* mean, float* rstd, int64_t skip_period,
                               jz_stream_t stream);
JZ_API int64_t jz_gemm_ln_bwd_parts(int64_t M);
JZ_API int jz_gemm_bf16_ln_bwd(const void* A, int64_t lda, int a_kmajor, const void* B, int64_t ldb, int b_kmajor,
                               int64_t M, int64_t N, int64_t K, const float* x, const float* mean,
                               const float* rstd, const float* gamma, float* dres, int accumulate,
                               void* dres_bf16, float* part, int64_t nparts, float* dgamma, float* dbeta,
                               float* dbias, jz_stream_t stream);

/* ------------------------------------------------------------------------
 * Column reductions (bias / LayerNorm-affine gradients; replaces the
 * _unbroadcast sums of autodiff.py:22-32).  Deterministic two-stage scheme:
 * a kernel writes `nparts` per-CTA partial rows, jz_reduce_partials sums them in
 * index order.  jz_row_partials(rows) = the nparts the library uses.
 * ---------------------------------------------------------------------- */
JZ_API int jz_row_partials(int64_t rows);
JZ_API int jz_colsum_bf16(const void* x, int64_t rows, int cols, int64_t ld, float* part, int nparts,
                          jz_stream_t stream);
/* out[c] (+)= sum_p part[p][c] in a fixed order.  With nparts > 512 the reduction runs in two stages
 * and uses `part` as scratch (rows 0, 256, 512, ... are overwritten). */
JZ_API int jz_reduce_partials(const float* part, int nparts, int64_t D, float* out, int accumulate,
                              jz_stream_t stream);
/* Three independent reductions of the same shape in one launch (NULL outputs are skipped); the
 * partial rows of each may live anywhere.  Used for the LayerNorm backward's gamma / beta / bias. */
JZ_API int jz_reduce_partials3(const float* part0, const float* part1, const float* part2, int nparts, int64_t D,
                               float* out0, float* out1, float* out2, int accumulate, jz_stream_t stream);
/* dst_bf16[r*ldd + c] = bf16(src[r*lds + c])  (weight shadows) */
JZ_API int jz_cast_f32_bf16_2d(const float* src, int64_t lds, void* dst, int64_t ldd, int64_t rows,
                               int64_t cols, jz_stream_t stream);

/* ------------------------------------------------------------------------
 * K2  LayerNorm, eps inside the sqrt, biased variance, two-pass (nn.py:35-40).
 * x f32 [rows, D] -> y bf16 and/or y_f32 (either may be NULL); mean/rstd f32 [rows]
 * saved for the backward.
 * skip_period > 0: rows r with r % skip_period == 0 are not written and the
 * output is compacted (drops the prepended action token before to_logits,
 * dynamics.py:135-136).  D multiple of 128, <= 1024.
 * ---------------------------------------------------------------------- */
JZ_API int jz_layernorm_fwd(const float* x, int64_t rows, int D, const float* gamma, const float* beta,
                            float eps, void* y_bf16, float* y_f32, float* mean, float* rstd, int64_t skip_period,
                            jz_stream_t stream);
/* dres[r] = (accumulate ? dres[r] : 0) + LN_bwd(dy[r]); optional bf16 copy of dres;
 * per-CTA partials of dgamma = sum dy*xhat, dbeta = sum dy, dbias = sum dres_out
 * ([nparts, D] each, any may be NULL).  dy is compacted when skip_period > 0. */
JZ_API int jz_layernorm_bwd(const float* x, const float* mean, const float* rstd, const float* gamma,
                            const float* dy, float* dres, int accumulate, void* dres_bf16,
                            float* part_dgamma, float* part_dbeta, float* part_dbias, int nparts,
                            int64_t rows, int D, int64_t skip_period, jz_stream_t stream);
/* Same with dy bf16 (the producing dX GEMM writes bf16: half the bytes of this HBM-bound pass). */
JZ_API int jz_layernorm_bwd_bf16dy(const float* x, const float* mean, const float* rstd, const float* gamma,
                                   const void* dy, float* dres, int accumulate, void* dres_bf16,
                                   float* part_dgamma, float* part_dbeta, float* part_dbias, int nparts,
                                   int64_t rows, int D, int64_t skip_period, jz_stream_t stream);

/* ------------------------------------------------------------------------
 * K7  masked softmax cross-entropy (nn.py:56-77 with weights = mask,
 * dynamics.py:151-152), forward and backward in one pass:
 *   row_loss[r] = mask[r] * (logsumexp(logits[r]) - logits[r, target[r]])
 *   loss        = sum(row_loss) / count            (0 when count == 0)
 *   dlogits     = grad_scale * mask[r]/count * (softmax - onehot)   (bf16)
 * count is a device int (the number of masked positions, from jz_philox_mask).
 * ---------------------------------------------------------------------- */
JZ_API int jz_ce_fwd_bwd(const float* logits, int64_t rows, int K, const int64_t* targets,
                         const uint8_t* mask, const int* count, float grad_scale, void* dlogits,
                         float* row_loss, float* loss, jz_stream_t stream);

/* ------------------------------------------------------------------------
 * K13 AdamW (optim.py:34-62), f32 with numpy/NEP-50 scalar casting and no FMA
 * contraction: bit-identical to the reference on identical inputs.
 *   omb1 = f32(1-b1), omb2 = f32(1-b2), bc1 = f32(1-b1^t), bc2 = f32(1-b2^t),
 *   lrwd = f32(lr*wd).  `flag` (device int, may be NULL): when non-zero the
 *   update is skipped (a non-finite gradient was seen by jz_finite_check).
 * ---------------------------------------------------------------------- */
JZ_API int jz_finite_check(const float* g, int64_t n, int* flag, jz_stream_t stream);
JZ_API int jz_adamw_step(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1,
                         float b2, float omb1, float omb2, float bc1, float bc2, float eps, float lrwd,
                         const int* flag, jz_stream_t stream);
/* Same update with the step's scalars read from device memory (CUDA-graph replays):
 * float dev_scalars[9] = lr, b1, b2, 1-b1, 1-b2, 1-b1^t, 1-b2^t, eps, lr*wd. */
JZ_API int jz_adamw_step_dev(float* p, const float* g, float* m, float* v, int64_t n, const float* dev_scalars,
                             const int* flag, jz_stream_t stream);

/* ------------------------------------------------------------------------
 * K6  Bernoulli MaskGIT masks, bit-exact with dynamics.sample_masks
 * (dynamics.py:52-62) over numpy's Philox4x64-10 stream (rng.py:38-44).
 * The numpy bit-generator state (counter[4], key[2], buffer[4], buffer_pos) is
 * passed in; samples [b0, b0+B_local) of a global batch of B_global are drawn by
 * counter skip-ahead (data-parallel sharding).  mask u8 [B_local, T, N];
 * *count += number of True entries (device int, must be zeroed by the caller).
 * ---------------------------------------------------------------------- */
JZ_API int jz_philox_mask(const uint64_t* counter4, const uint64_t* key2, const uint64_t* buffer4,
                          int buffer_pos, int64_t B_global, int64_t b0, int64_t B_local, int T, int N,
                          double mask_limit, uint8_t* mask, int* count, jz_stream_t stream);
/* Same mask with the stream state read from device memory (CUDA-graph replays of a training
 * step): int64 dev_state[11] = counter[4], key[2], buffer[4], buffer_pos. */
JZ_API int jz_philox_mask_dev(const int64_t* dev_state, int64_t B_global, int64_t b0, int64_t B_local, int T, int N,
                              double mask_limit, uint8_t* mask, int* count, jz_stream_t stream);

/* ------------------------------------------------------------------------
 * K5  dynamics input embedding (dynamics.py:101-133): token embed, mask-token
 * select, latent-action conditioning (prepend: action token at s=0; additive),
 * spatial + temporal positions.  tokens int64 [B,T,N]; mask u8 [B,T,N] or NULL;
 * latents f32 [B,T-1,dl]; x f32 [B,T,S,D] with S = N + prepend.
 * *err is set to 1 when a token id is out of range (the Python layer validates
 * host inputs first and raises IndexError, autodiff.py:353-354).
 * ---------------------------------------------------------------------- */
JZ_API int jz_dyn_embed_fwd(const int64_t* tokens, const uint8_t* mask, const float* latents,
                            const float* token_embed, const float* mask_token, const float* null_action,
                            const float* action_w, const float* action_b, const float* pos_spatial,
                            const float* pos_temporal, int64_t B, int T, int N, int D, int dl, int K,
                            int prepend, float* x, int* err, jz_stream_t stream);
/* Workspace (floats) for jz_dyn_embed_bwd; K = vocabulary (token-table sort buffers). */
/* Small embedding-table backward (autodiff.embedding backward, autodiff.py:344-364):
 * dtable[k] (=|+=) sum_{i: ids[i]==k} dout[i] in increasing i (deterministic, no atomics).
 * dout f32 [n, D]; err (may be NULL) is set to 1 when an id is outside [0, K). */
JZ_API int jz_embedding_table_bwd(const float* dout, const int64_t* ids, int64_t n, int K, int D, float* dtable,
                                  int accumulate, int* err, jz_stream_t stream);
JZ_API int64_t jz_dyn_embed_bwd_workspace(int64_t B, int T, int N, int D, int dl, int prepend, int K);
/* Deterministic backward of jz_dyn_embed_fwd (no float atomics).  d_latents may be NULL. */
JZ_API int jz_dyn_embed_bwd(const float* dx, const int64_t* tokens, const uint8_t* mask,
                            const float* latents, const float* null_action, const float* action_w,
                            int64_t B, int T, int N, int D, int dl, int K, int prepend,
                            float* d_token_embed, float* d_mask_token, float* d_null_action,
                            float* d_action_w, float* d_action_b, float* d_pos_spatial,
                            float* d_pos_temporal, float* d_latents, float* workspace,
                            jz_stream_t stream);

/* ------------------------------------------------------------------------
 * K3  spatial (intra-frame) attention, tcgen05/TMEM + TMA (st.py:73,
 * nn.py:80-110, causal=False).  qkv bf16 [frames*S, 3*H*64] (q|k|v, head h =
 * cols 64h..), out bf16 [frames*S, H*64], out_lo (optional, may be NULL) bf16 the
 * rounding residual O - bf16(O) of the fp32 output (out + out_lo carries O to ~16
 * mantissa bits for the backward's Delta), lse f32 [frames, H, S] (natural-log softmax
 * normaliser).
 * S in {256, 257}, head_dim 64.
 * ---------------------------------------------------------------------- */
JZ_API int jz_attn_spatial_fwd(const void* qkv, int64_t frames, int S, int H, int head_dim, void* out,
                               void* out_lo, float* lse, jz_stream_t stream);
/* dqkv bf16 [frames*S, 3*H*64] (fully overwritten).  out / out_lo are the forward's output
 * and residual: Delta_i = dO_i . (out + out_lo)_i is formed from them (first launch, into
 * per-(frame, head) vector blocks in `workspace`, with lse and the token-256 vectors) so
 * dP - Delta does not cancel against the bf16 rounding of O.  workspace: caller-owned,
 * jz_attn_spatial_bwd_workspace_bytes(frames, S, H) bytes, 16-byte aligned. */
JZ_API int64_t jz_attn_spatial_bwd_workspace_bytes(int64_t frames, int S, int H);
/* colsum_part (nullable): fp32 [jz_attn_spatial_colsum_parts(frames)][3*H*64] partial column sums
 * of dqkv (the QKV bias gradient after jz_reduce_partials), written instead of re-reading dqkv. */
JZ_API int64_t jz_attn_spatial_colsum_parts(int64_t frames);
JZ_API int jz_attn_spatial_bwd(const void* qkv, const void* out, const void* out_lo, const void* dout, const float* lse,
                               int64_t frames, int S, int H, int head_dim, void* dqkv, void* workspace,
                               float* colsum_part, jz_stream_t stream);

/* ------------------------------------------------------------------------
 * K4  causal temporal (inter-frame) attention (st.py:74-76, nn.py:103-105):
 * for every (b, s) the T rows (b, t, s) attend causally over t.  qkv/out as
 * above with rows ordered (b, t, s); lse f32 [B*S, H, T].  T <= 32, head_dim 64
 * (T > 16: two 16-row register tiles; one CTA per (slot, group of up to 4 heads)).
 * ---------------------------------------------------------------------- */
JZ_API int jz_attn_temporal_fwd(const void* qkv, int64_t B, int T, int S, int H, int head_dim, void* out,
                                float* lse, jz_stream_t stream);
/* colsum_part (nullable): fp32 [jz_attn_temporal_colsum_parts(B, S)][3*H*64], as the spatial one. */
JZ_API int64_t jz_attn_temporal_colsum_parts(int64_t B, int S);
/* partial rows the backward writes for these dims (use this one; the two-argument form is the
 * register-tile kernels' count): T <= 16 runs the tcgen05 kernels, one partial row per CTA. */
JZ_API int64_t jz_attn_temporal_colsum_parts_t(int64_t B, int S, int T, int H);
/* out: the forward output; not read (Delta_t = sum_j P_tj dP_tj is formed from the kernel's fp32
 * P and dP registers, which removes the O read and the dP - Delta cancellation against a bf16 O);
 * kept for interface stability, may be NULL. */
JZ_API int jz_attn_temporal_bwd(const void* qkv, const void* out, const void* dout, const float* lse,
                                int64_t B, int T, int S, int H, int head_dim, void* dqkv, float* colsum_part,
                                jz_stream_t stream);

/* ------------------------------------------------------------------------
 * K3s spatial attention of small frames, S <= 32 (st.py:73, nn.py:80-110,
 * causal=False): the reference's patch-16 presets (S = 16/17), the MAE
 * tokenizer (S = 16) and the ST-DiT (S = N + 2, diffusion.py:164-180).
 * Register-tile MMAs, one CTA per frame.  qkv/out/lse in the K3 layouts
 * (lse f32 [frames, H, S]); the backward's `out` is not read (may be NULL), as K4's.
 * colsum_part (nullable): fp32 [frames][3*H*64] partial column sums of dqkv.
 * ---------------------------------------------------------------------- */
JZ_API int jz_attn_spatial_small_fwd(const void* qkv, int64_t frames, int S, int H, int head_dim, void* out,
                                     float* lse, jz_stream_t stream);
JZ_API int jz_attn_spatial_small_bwd(const void* qkv, const void* out, const void* dout, const float* lse,
                                     int64_t frames, int S, int H, int head_dim, void* dqkv, float* colsum_part,
                                     jz_stream_t stream);

/* ------------------------------------------------------------------------
 * K9  frames -> patches and back (tokenizer.py:49-55, nn.py:113-131).
 * frames: uint8 (is_u8=1, unit = x/127.5 - 1) or fp32 unit-range, [BT, H, W, C];
 * patches [BT*N, P*P*C] in (gh, gw) row-major order, inner (ph, pw, c): bf16
 * (GEMM operand) and/or fp32 (recon target).  unpatchify writes fp32 unit frames
 * and/or uint8 frames = rint(clip((u+1)*127.5, 0, 255)) (round half-even).
 * ---------------------------------------------------------------------- */
JZ_API int jz_patchify(const void* frames, int is_u8, int64_t BT, int H, int W, int C, int P, void* out_bf16,
                       float* out_f32, jz_stream_t stream);
JZ_API int jz_unpatchify(const float* patches, int64_t BT, int H, int W, int C, int P, float* unit,
                         uint8_t* frames_u8, jz_stream_t stream);

/* Token assembly: x[b,t,s] = (e + pos_spatial[s]) + pos_temporal[t] where e is the
 * patch embedding emb[b,t,s-prepend] or, when prepend and s == 0, act[b,t]
 * (tokenizer.py:113-119, lam.py:86-90, lam.py:108-113).  Backward splits dx into a
 * compact bf16 d_emb, an fp32 d_act and deterministic position gradients. */
JZ_API int jz_assemble_fwd(const float* emb, const float* act, const float* pos_spatial, const float* pos_temporal,
                           int64_t B, int T, int N, int D, int prepend, float* x, jz_stream_t stream);
JZ_API int64_t jz_assemble_bwd_workspace(int64_t B, int T, int N, int D, int prepend);
JZ_API int jz_assemble_bwd(const float* dx, int64_t B, int T, int N, int D, int prepend, void* d_emb_bf16,
                           float* d_act, float* d_pos_spatial, float* d_pos_temporal, float* workspace,
                           jz_stream_t stream);

/* K10 mean over the N patch rows of each frame (lam.py:92) and its backward. */
JZ_API int jz_mean_pool(const float* x, int64_t BT, int N, int D, float* out, jz_stream_t stream);
JZ_API int jz_mean_pool_bwd(const float* dpool, int64_t BT, int N, int D, float* dx, jz_stream_t stream);

/* K15 loss = mean((pred - target)^2) (nn.py:50-53); grad = grad_scale * 2 (pred - target) / n
 * into grad32 and/or grad16 (either may be NULL).  workspace: 2*num_SMs doubles. */
JZ_API int jz_mse(const float* pred, const float* target, int64_t n, float grad_scale, float* loss, float* grad32,
                  void* grad16, double* workspace, jz_stream_t stream);

/* out = scale * sum(x) (fp64 accumulation, fixed order).  workspace: 2*num_SMs doubles. */
JZ_API int jz_sum(const float* x, int64_t n, double scale, float* out, double* workspace, jz_stream_t stream);

/* fp32 CUDA-core linear for the 32-wide latent projections (lam.py:94, lam.py:109):
 * y = x W + b (W (K, N) as stored by the reference); backward dx = dy W^T,
 * dW = x^T dy, db = sum dy (any output may be NULL; fixed summation order). */
JZ_API int jz_linear_f32(const float* x, int64_t R, int K, const float* W, int N, const float* b, float* y,
                         int accumulate, jz_stream_t stream);
JZ_API int jz_linear_f32_bwd(const float* x, const float* dy, int64_t R, int K, int N, const float* W, float* dx,
                             float* dW, float* db, int accumulate, jz_stream_t stream);
/* Same gradients through parallel kernels when one side of W is 32 wide (the latent projections):
 * dW from per-256-row partials folded in index order by jz_reduce_partials (deterministic), dx from
 * W staged in shared memory.  workspace: jz_linear_f32_bwd_workspace(R, K, N) floats (0: the shape
 * is not covered and the call runs jz_linear_f32_bwd). */
JZ_API int64_t jz_linear_f32_bwd_workspace(int64_t R, int K, int N);
JZ_API int jz_linear_f32_bwd_ws(const float* x, const float* dy, int64_t R, int K, int N, const float* W, float* dx,
                                float* dW, float* db, int accumulate, float* workspace, int64_t workspace_floats,
                                jz_stream_t stream);

/* ------------------------------------------------------------------------
 * K8  vector quantizer (tokenizer.vq_quantize, tokenizer.py:58-79), fp32:
 * d2 = (|z|^2 - (2z).c) + |c|^2, idx = argmin (lowest index on ties),
 * zq_st = z + (c_idx - z), row_sq[r] = sum (c_idx - z)^2 (losses = mean).
 * Backward: dz = g_zq_st + commit_coef (z - c_idx);
 *           dcodebook[k] = cb_coef * sum_{idx=k} (c_k - z)  (deterministic).
 * ---------------------------------------------------------------------- */
JZ_API int jz_vq_fwd(const float* z, int64_t rows, int dz, const float* codebook, int K, int64_t* idx,
                     float* zq_st, float* row_sq, jz_stream_t stream);
JZ_API int jz_vq_bwd(const float* z, const float* codebook, const int64_t* idx, const float* g_zq_st, int64_t rows,
                     int dz, int K, float commit_coef, float cb_coef, float* dz_out, float* dcodebook,
                     jz_stream_t stream);

/* ------------------------------------------------------------------------
 * K12 KV-cached MaskGIT decoding (dynamics.py:156-194 computes the full clip's
 * logits every step; by temporal causality only the last frame changes).
 * jz_dyn_embed_frame: one frame's tokens (B, N) -> x [B*(N+1), D] with the
 *   action token from cond [B, dl]; known[b,n] == 0 selects the mask token
 *   (known == NULL: all known); pos_temporal_row = pos_temporal + t*D, or, when
 *   dev_t != NULL, pos_temporal + (*dev_t)*D (frame index read on device).
 * jz_attn_temporal_decode: temporal attention of the frame (qkv [B*S, 3D]) over
 *   cache [B, Tmax, S, 2D] (k|v, bf16) frames 0..t-1 plus itself; append writes
 *   its k, v into cache[:, t]; dev_t != NULL overrides t from device memory.
 * jz_kv_fill: cache[:, t0 .. t0+T) = k|v of qkv rows (b, tau, s).
 * ---------------------------------------------------------------------- */
JZ_API int jz_dyn_embed_frame(const int64_t* tokens, const uint8_t* known, const float* cond,
                              const float* token_embed, const float* mask_token, const float* action_w,
                              const float* action_b, const float* pos_spatial, const float* pos_temporal_row,
                              const int* dev_t, int64_t B, int N, int D, int dl, int K, float* x,
                              jz_stream_t stream);
JZ_API int jz_attn_temporal_decode(const void* qkv, void* cache, int64_t B, int t, const int* dev_t, int Tmax,
                                   int S, int H, int append, void* out, jz_stream_t stream);
JZ_API int jz_kv_fill(const void* qkv, void* cache, int64_t B, int T, int t0, int Tmax, int S, int D,
                      jz_stream_t stream);

/* K11 one MaskGIT refinement step (dynamics.py:177-192 with _sample_with_confidence,
 * dynamics.py:198-217): for each (b, n): softmax(logits/T), u = draw (draw_base +
 * b*N + n) of the numpy Philox state (counter/key/buffer/pos as in jz_philox_mask),
 * sampled = #(u > cdf) clamped to K-1 (argmax when T < 1e-6, no draw), conf =
 * p[sampled]; cur = known ? cur : sampled; conf = known ? +inf : conf; then the
 * n_keep best (conf desc, position asc) of each row become known.  dev_params (may be
 * NULL): device int64[13] {draw_base, n_keep, counter[4], key[2], buffer[4], buffer_pos}
 * read by the kernels instead of the host values (buffer_pos < 0: keep the host Philox
 * state), so one captured CUDA graph serves every refinement step of every frame.
 * K <= 2048 (any K; K % 32 != 0 runs a padded lane layout). */
JZ_API int jz_maskgit_step(const float* logits, int64_t B, int N, int K, float temperature,
                           const uint64_t* counter4, const uint64_t* key2, const uint64_t* buffer4,
                           int buffer_pos, uint64_t draw_base, int n_keep, const int64_t* dev_params,
                           int64_t* cur, uint8_t* known, float* conf, jz_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* JZ_H_ */
