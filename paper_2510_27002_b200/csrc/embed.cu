// MaskGIT dynamics input side (K5, K6):
//   K6  Philox4x64-10 Bernoulli masks, bit-exact to sample_masks (dynamics.py:52-62)
//   K5  token embed + mask-token select + latent-action conditioning (prepend / additive)
//       + spatial/temporal positions, forward and deterministic backward
//       (dynamics.py:101-133; autodiff.embedding/where/concat backward, autodiff.py:318-364)
#include "common.h"
#include "philox.cuh"
#include "ptx.cuh"

namespace jz {

// ---------------------------------------------------------------------------
// K6: mask[b_local, t, n] = u[Bg + ((b0+b_local)*T + t)*N + n] < p_{b0+b_local},  mask[:,0] = 0
//     p_b = lim + (1 - lim) * u[b]
// ---------------------------------------------------------------------------
__global__ void philox_mask_kernel(PhiloxState st, int64_t B_global, int64_t b0, int64_t B_local, int T,
                                   int N, double lim, uint8_t* __restrict__ mask, int* __restrict__ count) {
  const int64_t total = B_local * T * N;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool m = false;
  if (e < total) {
    const int64_t bl = e / ((int64_t)T * N);
    const int64_t rem = e - bl * T * N;
    const int t = (int)(rem / N);
    const int64_t b = b0 + bl;
    const double pb = lim + (1.0 - lim) * u64_to_double(philox_word(st, (uint64_t)b));
    const double u = u64_to_double(philox_word(st, (uint64_t)(B_global + b * T * N + rem)));
    m = (t != 0) && (u < pb);
    mask[e] = m ? 1 : 0;
  }
  const unsigned bal = __ballot_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0 && bal) atomicAdd(count, __popc(bal));
}

// ---------------------------------------------------------------------------
// K5 forward.  One CTA (D/4 threads) per output row (b, t, s).
//   prepend : s = 0 -> act(b,t) + ps[0] + pt[t];  s >= 1 -> sel(b,t,s-1) + ps[s] + pt[t]
//   additive: s = n -> (sel(b,t,n) + act(b,t)) + ps[n] + pt[t]
//   sel = mask ? mask_token : E[token];  act = cond @ Wa + ba, cond = t ? lat[b,t-1] : null
// ---------------------------------------------------------------------------
__device__ __forceinline__ float4 act_proj4(const float* cond, int dl, const float* __restrict__ Wa,
                                            const float* __restrict__ ba, int D, int d) {
  float4 acc = make_float4(0, 0, 0, 0);
  for (int i = 0; i < dl; ++i) {
    const float c = cond[i];
    float4 w = *reinterpret_cast<const float4*>(Wa + (int64_t)i * D + d);
    acc.x += c * w.x; acc.y += c * w.y; acc.z += c * w.z; acc.w += c * w.w;
  }
  float4 b = *reinterpret_cast<const float4*>(ba + d);
  return make_float4(acc.x + b.x, acc.y + b.y, acc.z + b.z, acc.w + b.w);
}

__global__ void dyn_embed_fwd_kernel(const int64_t* __restrict__ tokens, const uint8_t* __restrict__ mask,
                                     const float* __restrict__ latents, const float* __restrict__ E,
                                     const float* __restrict__ mask_token, const float* __restrict__ null_action,
                                     const float* __restrict__ Wa, const float* __restrict__ ba,
                                     const float* __restrict__ ps, const float* __restrict__ pt, int T, int N,
                                     int D, int dl, int K, int prepend, float* __restrict__ x, int* err) {
  const int S = N + (prepend ? 1 : 0);
  const int64_t row = blockIdx.x;  // (b*T + t)*S + s
  const int s = (int)(row % S);
  const int64_t bt = row / S;
  const int t = (int)(bt % T);
  const int64_t b = bt / T;
  const int d = threadIdx.x * 4;
  if (d >= D) return;
  __shared__ float cond[64];
  const bool need_act = prepend ? (s == 0) : true;
  if (need_act) {
    for (int i = threadIdx.x; i < dl; i += blockDim.x)
      cond[i] = t == 0 ? null_action[i] : latents[(b * (T - 1) + (t - 1)) * dl + i];
    __syncthreads();
  }
  float4 v;
  if (prepend && s == 0) {
    v = act_proj4(cond, dl, Wa, ba, D, d);
  } else {
    const int n = prepend ? s - 1 : s;
    const int64_t pos = bt * N + n;
    if (mask && mask[pos]) {
      v = *reinterpret_cast<const float4*>(mask_token + d);
    } else {
      int64_t tok = tokens[pos];
      if (tok < 0 || tok >= K) {
        if (threadIdx.x == 0) atomicExch(err, 1);
        tok = 0;
      }
      v = *reinterpret_cast<const float4*>(E + tok * D + d);
    }
    if (!prepend) {
      float4 a = act_proj4(cond, dl, Wa, ba, D, d);
      v.x += a.x; v.y += a.y; v.z += a.z; v.w += a.w;
    }
  }
  float4 p1 = *reinterpret_cast<const float4*>(ps + (int64_t)s * D + d);
  float4 p2 = *reinterpret_cast<const float4*>(pt + (int64_t)t * D + d);
  v.x = (v.x + p1.x) + p2.x; v.y = (v.y + p1.y) + p2.y;
  v.z = (v.z + p1.z) + p2.z; v.w = (v.w + p1.w) + p2.w;
  *reinterpret_cast<float4*>(x + row * D + d) = v;
}

// ---------------------------------------------------------------------------
// K5 backward, positions + mask token.  CTA per spatial slot s:
//   dps[s]          = sum_{t,b} dx[b,t,s]
//   part_pt[s][t]   = sum_b dx[b,t,s]                 (-> dpt[t] = sum_s part_pt[s][t])
//   part_mt[s]      = sum_{b,t: mask[b,t,n(s)]} dx[b,t,s]   (-> dmask_token)
// ---------------------------------------------------------------------------
// One CTA per spatial slot s: 4 thread groups split the T frames (each group 128 threads x 4 dims
// over D = 512), 8 row loads in flight per thread; the groups' spatial / mask-token sums are then
// combined in group order through shared memory (deterministic).
constexpr int kPosGroups = 4;
__global__ void __launch_bounds__(128 * kPosGroups) dyn_embed_bwd_pos_kernel(
    const float* __restrict__ dx, const uint8_t* __restrict__ mask, int64_t B, int T, int N, int D, int prepend,
    float* __restrict__ dps, float* __restrict__ part_pt, float* __restrict__ part_mt) {
  __shared__ float4 red_s[kPosGroups - 1][128], red_m[kPosGroups - 1][128];
  const int S = N + (prepend ? 1 : 0);
  const int s = blockIdx.x;
  const int n = prepend ? s - 1 : s;
  const int grp = threadIdx.x >> 7, tid = threadIdx.x & 127;
  for (int d0 = 0; d0 < D; d0 += 512) {
    const int d = d0 + 4 * tid;
    const bool live = d < D;
    float4 acc_s = make_float4(0, 0, 0, 0), acc_m = make_float4(0, 0, 0, 0);
    for (int t = grp; t < T; t += kPosGroups) {
      float4 acc_t = make_float4(0, 0, 0, 0);
      for (int64_t b0 = 0; b0 < B; b0 += 8) {
        float4 g[8];
        bool mk[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int64_t b = b0 + q;
          g[q] = make_float4(0, 0, 0, 0);
          mk[q] = false;
          if (live && b < B) {
            const int64_t row = (b * T + t) * S + s;
            g[q] = __ldg(reinterpret_cast<const float4*>(dx + row * D + d));
            mk[q] = n >= 0 && mask && mask[(b * T + t) * N + n];
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          acc_t.x += g[q].x; acc_t.y += g[q].y; acc_t.z += g[q].z; acc_t.w += g[q].w;
          if (mk[q]) { acc_m.x += g[q].x; acc_m.y += g[q].y; acc_m.z += g[q].z; acc_m.w += g[q].w; }
        }
      }
      if (live) *reinterpret_cast<float4*>(part_pt + ((int64_t)s * T + t) * D + d) = acc_t;
      acc_s.x += acc_t.x; acc_s.y += acc_t.y; acc_s.z += acc_t.z; acc_s.w += acc_t.w;
    }
    if (grp > 0) {
      red_s[grp - 1][tid] = acc_s;
      red_m[grp - 1][tid] = acc_m;
    }
    __syncthreads();
    if (grp == 0 && live) {
#pragma unroll
      for (int g2 = 0; g2 < kPosGroups - 1; ++g2) {
        const float4 a = red_s[g2][tid], m = red_m[g2][tid];
        acc_s.x += a.x; acc_s.y += a.y; acc_s.z += a.z; acc_s.w += a.w;
        acc_m.x += m.x; acc_m.y += m.y; acc_m.z += m.z; acc_m.w += m.w;
      }
      *reinterpret_cast<float4*>(dps + (int64_t)s * D + d) = acc_s;
      *reinterpret_cast<float4*>(part_mt + (int64_t)s * D + d) = acc_m;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K5 backward, token table (deterministic scatter-add, "owner computes"):
// CTA c owns token ids k = c, c+G, c+2G, ... (at most kOwn).  Warp w scans the fixed
// position range [w*P/8, (w+1)*P/8) in order and accumulates unmasked rows into its
// own registers; warps are then summed in warp order.
// ---------------------------------------------------------------------------
constexpr int kOwn = 8;

template <int V4>  // D = 128 * V4
__global__ void __launch_bounds__(256) dyn_embed_bwd_tok_kernel(const float* __restrict__ dx,
                                                                const int64_t* __restrict__ tokens,
                                                                const uint8_t* __restrict__ mask, int64_t P,
                                                                int N, int S, int prepend, int K,
                                                                float* __restrict__ dE) {
  constexpr int D = 128 * V4;
  const int G = gridDim.x;
  const int c = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n_own = (K - c + G - 1) / G;  // ids c + j*G < K
  float4 acc[kOwn][V4];
#pragma unroll
  for (int j = 0; j < kOwn; ++j)
#pragma unroll
    for (int i = 0; i < V4; ++i) acc[j][i] = make_float4(0, 0, 0, 0);
  const int64_t per = (P + 7) / 8;
  const int64_t p0 = warp * per, p1 = min(P, p0 + per);
  for (int64_t base = p0; base < p1; base += 32) {
    const int64_t p = base + lane;
    int64_t tok = -1;
    if (p < p1 && !(mask && mask[p])) tok = tokens[p];
    const bool mine = tok >= 0 && tok < K && (tok % G) == c;
    unsigned bal = __ballot_sync(0xffffffffu, mine);
    while (bal) {
      const int src = __ffs(bal) - 1;
      bal &= bal - 1;
      const int64_t tk = __shfl_sync(0xffffffffu, tok, src);
      const int64_t pp = base + src;
      const int j = (int)(tk / G);
      const int64_t row = prepend ? (pp / N) * S + (pp % N) + 1 : pp;
      const float* g = dx + row * D;
#pragma unroll
      for (int jj = 0; jj < kOwn; ++jj) {
        if (jj == j) {
#pragma unroll
          for (int i = 0; i < V4; ++i) {
            float4 v = *reinterpret_cast<const float4*>(g + 4 * lane + 128 * i);
            acc[jj][i].x += v.x; acc[jj][i].y += v.y; acc[jj][i].z += v.z; acc[jj][i].w += v.w;
          }
        }
      }
    }
  }
  __shared__ float sm[8][D];
  for (int j = 0; j < n_own && j < kOwn; ++j) {
#pragma unroll
    for (int i = 0; i < V4; ++i) *reinterpret_cast<float4*>(&sm[warp][4 * lane + 128 * i]) = acc[j][i];
    __syncthreads();
    for (int d = threadIdx.x; d < D; d += 256) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += sm[w][d];
      dE[(int64_t)(c + j * G) * D + d] = s;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K5 backward, action conditioning.  dact[bt] = prepend ? dx[bt, s=0] : sum_n dx[bt, n]
//   dWa[i][d] = sum_bt cond[bt][i] dact[bt][d];  dba[d] = sum_bt dact[bt][d]
//   dcond[bt][i] = sum_d dact[bt][d] Wa[i][d];   dnull = sum_b dcond[b,0];  dlat[b,t-1] = dcond[b,t]
// ---------------------------------------------------------------------------
__global__ void dyn_dact_additive_kernel(const float* __restrict__ dx, int64_t BT, int N, int D,
                                         float* __restrict__ dact) {
  const int64_t bt = blockIdx.x;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float s = 0.f;
    for (int n = 0; n < N; ++n) s += dx[(bt * N + n) * D + d];
    dact[bt * D + d] = s;
  }
}

// partial[chunk][i][d] (i < dl) and partial_b[chunk][d] over bt in [chunk*per, (chunk+1)*per)
__global__ void dyn_action_w_kernel(const float* __restrict__ dact, int64_t dact_stride, int64_t B, int T,
                                    const float* __restrict__ latents, const float* __restrict__ null_action,
                                    int dl, int D, int64_t per, float* __restrict__ part_w, float* __restrict__ part_b) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  const int chunk = blockIdx.y;
  if (d >= D) return;
  float acc[64];
  for (int i = 0; i < dl; ++i) acc[i] = 0.f;
  float sb = 0.f;
  const int64_t BT = B * T;
  const int64_t bt0 = chunk * per, bt1 = min(BT, bt0 + per);
  for (int64_t bt = bt0; bt < bt1; ++bt) {
    const int64_t b = bt / T;
    const int t = (int)(bt - b * T);
    const float g = dact[bt * dact_stride + d];
    const float* cond = t == 0 ? null_action : latents + (b * (T - 1) + (t - 1)) * dl;
    for (int i = 0; i < dl; ++i) acc[i] += cond[i] * g;
    sb += g;
  }
  for (int i = 0; i < dl; ++i) part_w[((int64_t)chunk * dl + i) * D + d] = acc[i];
  part_b[(int64_t)chunk * D + d] = sb;
}

__global__ void dyn_action_cond_kernel(const float* __restrict__ dact, int64_t dact_stride, int64_t BT,
                                       const float* __restrict__ Wa, int dl, int D, float* __restrict__ dcond) {
  const int64_t bt = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (bt >= BT) return;
  for (int i = lane; i < dl; i += 32) {
    float s = 0.f;
    for (int d = 0; d < D; ++d) s += dact[bt * dact_stride + d] * Wa[(int64_t)i * D + d];
    dcond[bt * dl + i] = s;
  }
}

__global__ void dyn_action_split_kernel(const float* __restrict__ dcond, int64_t B, int T, int dl,
                                        float* __restrict__ dnull, float* __restrict__ dlat) {
  const int i = threadIdx.x;
  if (i < dl) {
    float s = 0.f;
    for (int64_t b = 0; b < B; ++b) s += dcond[(b * T) * dl + i];
    if (dnull) dnull[i] = s;
  }
  if (dlat) {
    const int64_t n = B * (T - 1) * dl;
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
      const int64_t b = e / ((int64_t)(T - 1) * dl);
      const int64_t r = e - b * (T - 1) * dl;
      dlat[e] = dcond[(b * T + 1) * dl + r];
    }
  }
}

}  // namespace jz

using namespace jz;

extern "C" int jz_philox_mask(const uint64_t* counter4, const uint64_t* key2, const uint64_t* buffer4,
                              int buffer_pos, int64_t B_global, int64_t b0, int64_t B_local, int T, int N,
                              double mask_limit, uint8_t* mask, int* count, jz_stream_t s) {
  JZ_CHECK_ARG(buffer_pos >= 0 && buffer_pos <= 4, "philox: buffer_pos");
  JZ_CHECK_ARG(b0 >= 0 && b0 + B_local <= B_global, "philox: shard out of range");
  PhiloxState st;
  for (int i = 0; i < 4; ++i) {
    st.ctr[i] = counter4[i];
    st.buf[i] = buffer4[i];
  }
  st.key[0] = key2[0];
  st.key[1] = key2[1];
  st.pos = buffer_pos;
  const int64_t total = B_local * T * N;
  if (total == 0) return JZ_OK;
  const int threads = 256;
  philox_mask_kernel<<<(unsigned)((total + threads - 1) / threads), threads, 0,
                       reinterpret_cast<cudaStream_t>(s)>>>(st, B_global, b0, B_local, T, N, mask_limit,
                                                            mask, count);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_dyn_embed_fwd(const int64_t* tokens, const uint8_t* mask, const float* latents,
                                const float* token_embed, const float* mask_token, const float* null_action,
                                const float* action_w, const float* action_b, const float* pos_spatial,
                                const float* pos_temporal, int64_t B, int T, int N, int D, int dl, int K,
                                int prepend, float* x, int* err, jz_stream_t s) {
  JZ_CHECK_ARG(D % 4 == 0 && D <= 4096, "embed: D=%d", D);
  JZ_CHECK_ARG(dl >= 1 && dl <= 64, "embed: latent dim %d unsupported (<= 64)", dl);
  const int S = N + (prepend ? 1 : 0);
  const int64_t rows = B * T * S;
  if (rows == 0) return JZ_OK;
  dyn_embed_fwd_kernel<<<(unsigned)rows, D / 4, 0, reinterpret_cast<cudaStream_t>(s)>>>(
      tokens, mask, latents, token_embed, mask_token, null_action, action_w, action_b, pos_spatial,
      pos_temporal, T, N, D, dl, K, prepend, x, err);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

// Workspace floats needed by jz_dyn_embed_bwd.
extern "C" int64_t jz_dyn_embed_bwd_workspace(int64_t B, int T, int N, int D, int dl, int prepend) {
  const int S = N + (prepend ? 1 : 0);
  return (int64_t)S * T * D + (int64_t)S * D + (prepend ? 0 : B * T * D) + B * T * dl + 64ll * (dl + 1) * D;
}

extern "C" int jz_dyn_embed_bwd(const float* dx, const int64_t* tokens, const uint8_t* mask,
                                const float* latents, const float* null_action, const float* action_w,
                                int64_t B, int T, int N, int D, int dl, int K, int prepend, float* d_token_embed,
                                float* d_mask_token, float* d_null_action, float* d_action_w, float* d_action_b,
                                float* d_pos_spatial, float* d_pos_temporal, float* d_latents, float* workspace,
                                jz_stream_t s) {
  JZ_CHECK_ARG(D % 128 == 0 && D <= 1024, "embed_bwd: D=%d unsupported", D);
  JZ_CHECK_ARG(dl >= 1 && dl <= 64, "embed_bwd: latent dim %d unsupported", dl);
  auto st = reinterpret_cast<cudaStream_t>(s);
  const int S = N + (prepend ? 1 : 0);
  float* part_pt = workspace;
  float* part_mt = part_pt + (int64_t)S * T * D;
  float* dact_buf = part_mt + (int64_t)S * D;
  float* dcond = dact_buf + (prepend ? 0 : B * T * D);
  // positions + mask token
  dyn_embed_bwd_pos_kernel<<<S, 128 * kPosGroups, 0, st>>>(dx, mask, B, T, N, D, prepend, d_pos_spatial, part_pt,
                                                           part_mt);
  JZ_LAUNCH_CHECK();
  int rc = jz_reduce_partials(part_pt, S, (int64_t)T * D, d_pos_temporal, 0, s);
  if (rc) return rc;
  rc = jz_reduce_partials(part_mt, S, D, d_mask_token, 0, s);
  if (rc) return rc;
  // token table
  const int G = (K + kOwn - 1) / kOwn < num_sms() ? num_sms() : (K + kOwn - 1) / kOwn;
  JZ_CHECK_ARG((K + G - 1) / G <= kOwn, "embed_bwd: vocabulary %d too large", K);
  const int64_t P = B * T * N;
  switch (D / 128) {
    case 1: dyn_embed_bwd_tok_kernel<1><<<G, 256, 0, st>>>(dx, tokens, mask, P, N, S, prepend, K, d_token_embed); break;
    case 2: dyn_embed_bwd_tok_kernel<2><<<G, 256, 0, st>>>(dx, tokens, mask, P, N, S, prepend, K, d_token_embed); break;
    case 4: dyn_embed_bwd_tok_kernel<4><<<G, 256, 0, st>>>(dx, tokens, mask, P, N, S, prepend, K, d_token_embed); break;
    case 8: dyn_embed_bwd_tok_kernel<8><<<G, 256, 0, st>>>(dx, tokens, mask, P, N, S, prepend, K, d_token_embed); break;
    default: set_error("embed_bwd: D=%d unsupported", D); return JZ_EINVAL;
  }
  JZ_LAUNCH_CHECK();
  if (G < K) {
    // ids >= G*? all covered: ids c + j*G for j < n_own cover [0, K)
  }
  // action conditioning
  const float* dact = dx;
  int64_t dact_stride = (int64_t)S * D;
  if (!prepend) {
    dyn_dact_additive_kernel<<<(unsigned)(B * T), 128, 0, st>>>(dx, B * T, N, D, dact_buf);
    JZ_LAUNCH_CHECK();
    dact = dact_buf;
    dact_stride = D;
  }
  {
    const int chunks = 64;
    const int64_t per = (B * T + chunks - 1) / chunks;
    float* part_w = dcond + B * T * dl;
    float* part_b = part_w + (int64_t)chunks * dl * D;
    dyn_action_w_kernel<<<dim3((D + 127) / 128, chunks), 128, 0, st>>>(dact, dact_stride, B, T, latents, null_action,
                                                                        dl, D, per, part_w, part_b);
    JZ_LAUNCH_CHECK();
    rc = jz_reduce_partials(part_w, chunks, (int64_t)dl * D, d_action_w, 0, s);
    if (rc) return rc;
    rc = jz_reduce_partials(part_b, chunks, D, d_action_b, 0, s);
    if (rc) return rc;
  }
  dyn_action_cond_kernel<<<(unsigned)((B * T + 7) / 8), 256, 0, st>>>(dact, dact_stride, B * T, action_w, dl, D,
                                                                       dcond);
  JZ_LAUNCH_CHECK();
  dyn_action_split_kernel<<<1, 256, 0, st>>>(dcond, B, T, dl, d_null_action, d_latents);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}
