// MaskGIT dynamics input side (K5, K6):
//   K6  Philox4x64-10 Bernoulli masks, bit-exact to sample_masks (dynamics.py:52-62)
//   K5  token embed + mask-token select + latent-action conditioning (prepend / additive)
//       + spatial/temporal positions, forward and deterministic backward
//       (dynamics.py:101-133; autodiff.embedding/where/concat backward, autodiff.py:318-364)
#include <string.h>

#include "common.h"
#include "philox.cuh"
#include "ptx.cuh"

namespace jz {

// ---------------------------------------------------------------------------
// K6: mask[b_local, t, n] = u[Bg + ((b0+b_local)*T + t)*N + n] < p_{b0+b_local},  mask[:,0] = 0
//     p_b = lim + (1 - lim) * u[b]
// ---------------------------------------------------------------------------
__global__ void philox_mask_kernel(PhiloxState st, int64_t B_global, int64_t b0, int64_t B_local, int T,
                                   int N, double lim, uint8_t* __restrict__ mask, int* __restrict__ count,
                                   const int64_t* __restrict__ dev_state) {
  if (dev_state) {  // graph replays: the step's stream state lives in device memory (layout of jz_philox_mask_dev)
    for (int i = 0; i < 4; ++i) {
      st.ctr[i] = (uint64_t)dev_state[i];
      st.buf[i] = (uint64_t)dev_state[6 + i];
    }
    st.key[0] = (uint64_t)dev_state[4];
    st.key[1] = (uint64_t)dev_state[5];
    st.pos = (int)dev_state[10];
  }
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
// K5 forward.  One warp per output row (b, t, s).
//   prepend : s = 0 -> act(b,t) + ps[0] + pt[t];  s >= 1 -> sel(b,t,s-1) + ps[s] + pt[t]
//   additive: s = n -> (sel(b,t,n) + act(b,t)) + ps[n] + pt[t]
//   sel = mask ? mask_token : E[token];  act = cond @ Wa + ba, cond = t ? lat[b,t-1] : null
// ---------------------------------------------------------------------------
// One warp per output row (grid-stride), lane l covering dims 4l + 128i; row -> (b, t, s) index math in
// 32 bits when the row count allows (IDX = uint32_t: the int64 div/mod chain dominated the issue slots).
// The action projection keeps the sequential i-order of cond @ Wa (cond broadcast from lanes by shuffle).
// NC = D/128 chunks per lane when known at compile time (row loads issue before the stores), 0 = generic.
template <int NC, typename IDX>
__global__ void __launch_bounds__(256) dyn_embed_fwd_kernel(
    const int64_t* __restrict__ tokens, const uint8_t* __restrict__ mask, const float* __restrict__ latents,
    const float* __restrict__ E, const float* __restrict__ mask_token, const float* __restrict__ null_action,
    const float* __restrict__ Wa, const float* __restrict__ ba, const float* __restrict__ ps,
    const float* __restrict__ pt, int64_t rows, int T, int N, int D, int dl, int K, int prepend,
    float* __restrict__ x, int* err) {
  const IDX S = (IDX)(N + (prepend ? 1 : 0));
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = w0; row < rows; row += nw) {
    const IDX bt = (IDX)row / S;
    const int s = (int)((IDX)row - bt * S);
    const IDX bq = bt / (IDX)T;
    const int t = (int)(bt - bq * (IDX)T);
    const bool need_act = prepend ? (s == 0) : true;
    float c0 = 0.f, c1 = 0.f;  // cond[lane], cond[32 + lane]
    if (need_act) {
      const float* cp = t == 0 ? null_action : latents + ((int64_t)bq * (T - 1) + (t - 1)) * dl;
      if (lane < dl) c0 = cp[lane];
      if (32 + lane < dl) c1 = cp[32 + lane];
    }
    const float* src = nullptr;  // token / mask-token row (nullptr for the prepended action slot)
    if (!(prepend && s == 0)) {
      const int64_t pos = (int64_t)bt * N + (prepend ? s - 1 : s);
      if (mask && mask[pos]) {
        src = mask_token;
      } else {
        int64_t tok = tokens[pos];
        if (tok < 0 || tok >= K) {
          if (lane == 0) atomicExch(err, 1);
          tok = 0;
        }
        src = E + tok * D;
      }
    }
    const float* psr = ps + (int64_t)s * D;
    const float* ptr_ = pt + (int64_t)t * D;
    float* xr = x + row * D;
    auto chunk = [&](int d, float4 v) {
      if (need_act) {
        float4 acc = make_float4(0, 0, 0, 0);
        for (int i = 0; i < dl; ++i) {
          const float c = __shfl_sync(0xffffffffu, i < 32 ? c0 : c1, i & 31);
          const float4 w = __ldg(reinterpret_cast<const float4*>(Wa + (int64_t)i * D + d));
          acc.x += c * w.x; acc.y += c * w.y; acc.z += c * w.z; acc.w += c * w.w;
        }
        const float4 bb = __ldg(reinterpret_cast<const float4*>(ba + d));
        const float4 a = make_float4(acc.x + bb.x, acc.y + bb.y, acc.z + bb.z, acc.w + bb.w);
        if (prepend) {
          v = a;
        } else {
          v.x += a.x; v.y += a.y; v.z += a.z; v.w += a.w;
        }
      }
      const float4 p1 = __ldg(reinterpret_cast<const float4*>(psr + d));
      const float4 p2 = __ldg(reinterpret_cast<const float4*>(ptr_ + d));
      float4 o;
      o.x = (v.x + p1.x) + p2.x; o.y = (v.y + p1.y) + p2.y;
      o.z = (v.z + p1.z) + p2.z; o.w = (v.w + p1.w) + p2.w;
      *reinterpret_cast<float4*>(xr + d) = o;
    };
    if constexpr (NC > 0) {
      float4 v[NC];
#pragma unroll
      for (int i = 0; i < NC; ++i)
        v[i] = src ? __ldg(reinterpret_cast<const float4*>(src + 4 * lane + 128 * i)) : make_float4(0, 0, 0, 0);
#pragma unroll
      for (int i = 0; i < NC; ++i) chunk(4 * lane + 128 * i, v[i]);
    } else {
      for (int d = 4 * lane; d < D; d += 128)
        chunk(d, src ? __ldg(reinterpret_cast<const float4*>(src + d)) : make_float4(0, 0, 0, 0));
    }
  }
}

// ---------------------------------------------------------------------------
// K5 backward, positions + mask token.  CTA per spatial slot s:
//   dps[s]          = sum_{t,b} dx[b,t,s]
//   part_pt[s][t]   = sum_b dx[b,t,s]                 (-> dpt[t] = sum_s part_pt[s][t])
//   part_mt[s]      = sum_{b,t: mask[b,t,n(s)]} dx[b,t,s]   (-> dmask_token)
// ---------------------------------------------------------------------------
// CTA per (spatial slot s, 128-dim slice): 4 warps split the T frames (warp g takes t = g mod 4, each lane
// 4 dims), 8 row loads in flight per thread; the warps' spatial / mask-token sums are then combined in
// warp order through shared memory (deterministic).  ~S * D/128 small CTAs keep every SM streaming.
constexpr int kPosGroups = 4;
__global__ void __launch_bounds__(32 * kPosGroups, 8) dyn_embed_bwd_pos_kernel(
    const float* __restrict__ dx, const uint8_t* __restrict__ mask, int64_t B, int T, int N, int D, int prepend,
    float* __restrict__ dps, float* __restrict__ part_pt, float* __restrict__ part_mt) {
  __shared__ float4 red_s[kPosGroups - 1][32], red_m[kPosGroups - 1][32];
  const int S = N + (prepend ? 1 : 0);
  const int s = blockIdx.x;
  const int n = prepend ? s - 1 : s;
  const int grp = threadIdx.x >> 5, tid = threadIdx.x & 31;
  const int d = blockIdx.y * 128 + 4 * tid;
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
        if (b < B) {
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
    *reinterpret_cast<float4*>(part_pt + ((int64_t)s * T + t) * D + d) = acc_t;
    acc_s.x += acc_t.x; acc_s.y += acc_t.y; acc_s.z += acc_t.z; acc_s.w += acc_t.w;
  }
  if (grp > 0) {
    red_s[grp - 1][tid] = acc_s;
    red_m[grp - 1][tid] = acc_m;
  }
  __syncthreads();
  if (grp == 0) {
#pragma unroll
    for (int g2 = 0; g2 < kPosGroups - 1; ++g2) {
      const float4 a = red_s[g2][tid], m = red_m[g2][tid];
      acc_s.x += a.x; acc_s.y += a.y; acc_s.z += a.z; acc_s.w += a.w;
      acc_m.x += m.x; acc_m.y += m.y; acc_m.z += m.z; acc_m.w += m.w;
    }
    *reinterpret_cast<float4*>(dps + (int64_t)s * D + d) = acc_s;
    *reinterpret_cast<float4*>(part_mt + (int64_t)s * D + d) = acc_m;
  }
}


// Token-table backward as a deterministic stable counting sort of positions by token id, then one
// warp per token summing its dx rows in position order:
//   tok_hist:    per position block, counts of unmasked tokens (integer: order-independent)
//   tok_scan:    per-token starts + per-(block, token) offsets, in fixed order
//   tok_scatter: stable placement (one warp per block, 32 positions at a time, __match_any_sync rank)
//   tok_accum:   warp k sums the rows of token k (4 rows in flight), writes dE[k]
constexpr int kTokChunk = 512;  // positions per histogram / scatter block

__global__ void __launch_bounds__(256) tok_hist_kernel(const int64_t* __restrict__ tokens,
                                                       const uint8_t* __restrict__ mask, int64_t P, int K,
                                                       int* __restrict__ hist) {
  extern __shared__ int sh[];
  for (int k = threadIdx.x; k < K; k += blockDim.x) sh[k] = 0;
  __syncthreads();
  const int64_t p0 = (int64_t)blockIdx.x * kTokChunk, p1 = min(P, p0 + kTokChunk);
  for (int64_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
    if (mask && mask[p]) continue;
    const int64_t t = tokens[p];
    if (t >= 0 && t < K) atomicAdd(&sh[t], 1);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x) hist[(int64_t)blockIdx.x * K + k] = sh[k];
}

// per token k (one thread each): hist[b][k] <- sum_{b' < b} hist[b'][k]; total[k] = sum_b hist[b][k]
__global__ void __launch_bounds__(256) tok_colscan_kernel(int* __restrict__ hist, int nb, int K, int* __restrict__ total) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= K) return;
  int r = 0;
  int b0 = 0;
  for (; b0 + 8 <= nb; b0 += 8) {  // 8 independent loads in flight, prefix in registers
    int c[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) c[q] = hist[(int64_t)(b0 + q) * K + k];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      hist[(int64_t)(b0 + q) * K + k] = r;
      r += c[q];
    }
  }
  for (; b0 < nb; ++b0) {
    const int c = hist[(int64_t)b0 * K + k];
    hist[(int64_t)b0 * K + k] = r;
    r += c;
  }
  total[k] = r;
}

// one block of 1024 threads: tok_start[k] = sum_{k' < k} total[k'] (K <= 8192), tok_start[K] = total
__global__ void __launch_bounds__(1024) tok_scan_kernel(const int* __restrict__ total, int K, int* __restrict__ tok_start) {
  __shared__ int wsum[32];
  constexpr int kPer = 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int v[kPer];
  int run = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int k = tid * kPer + q;
    v[q] = k < K ? total[k] : 0;
    run += v[q];
  }
  int incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int start = incl - run;
  for (int w = 0; w < warp; ++w) start += wsum[w];
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int k = tid * kPer + q;
    if (k < K) tok_start[k] = start;
    start += v[q];
  }
  if (tid == 1023) tok_start[K] = start;
}

__global__ void __launch_bounds__(32) tok_scatter_kernel(const int64_t* __restrict__ tokens,
                                                         const uint8_t* __restrict__ mask, int64_t P, int K,
                                                         const int* __restrict__ offsets,
                                                         const int* __restrict__ tok_start,
                                                         int32_t* __restrict__ sorted) {
  extern __shared__ int cur[];
  const int lane = threadIdx.x;
  for (int k = lane; k < K; k += 32) cur[k] = tok_start[k] + offsets[(int64_t)blockIdx.x * K + k];
  __syncwarp();
  const int64_t p0 = (int64_t)blockIdx.x * kTokChunk, p1 = min(P, p0 + kTokChunk);
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t base = p0; base < p1; base += 32) {
    const int64_t p = base + lane;
    int t = -1;
    if (p < p1 && !(mask && mask[p])) {
      const int64_t tt = tokens[p];
      if (tt >= 0 && tt < K) t = (int)tt;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, t);
    const int rank = __popc(peers & lt);
    if (t >= 0) sorted[cur[t] + rank] = (int32_t)p;
    __syncwarp();
    if (t >= 0 && rank == 0) cur[t] += __popc(peers);
    __syncwarp();
  }
}

template <int V4>  // D = 128 * V4; one warp per token
__global__ void __launch_bounds__(256) tok_accum_kernel(const float* __restrict__ dx, const int32_t* __restrict__ sorted,
                                                        const int* __restrict__ tok_start, int K, int N, int S,
                                                        int prepend, float* __restrict__ dE) {
  constexpr int D = 128 * V4;
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (k >= K) return;
  const int e0 = tok_start[k], e1 = tok_start[k + 1];
  float4 acc[V4];
#pragma unroll
  for (int i = 0; i < V4; ++i) acc[i] = make_float4(0, 0, 0, 0);
  for (int e = e0; e < e1; e += 4) {
    float4 v[4][V4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (e + q < e1) {
        const int pp = sorted[e + q];
        const int64_t row = prepend ? ((int64_t)pp / N) * S + (pp % N) + 1 : pp;
        const float* g = dx + row * D;
#pragma unroll
        for (int i = 0; i < V4; ++i) v[q][i] = __ldg(reinterpret_cast<const float4*>(g + 4 * lane + 128 * i));
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (e + q < e1) {
#pragma unroll
        for (int i = 0; i < V4; ++i) {
          acc[i].x += v[q][i].x; acc[i].y += v[q][i].y; acc[i].z += v[q][i].z; acc[i].w += v[q][i].w;
        }
      }
  }
#pragma unroll
  for (int i = 0; i < V4; ++i) *reinterpret_cast<float4*>(dE + (int64_t)k * D + 4 * lane + 128 * i) = acc[i];
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
  // one warp per (b, t) row; lanes stride over d (coalesced dact and Wa rows), one warp sum per output
  const int64_t bt = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (bt >= BT) return;
  const float* a = dact + bt * dact_stride;
  for (int i = 0; i < dl; ++i) {
    const float* w = Wa + (int64_t)i * D;
    float s = 0.f;
    for (int d = lane; d < D; d += 32) s += a[d] * w[d];
    s = warp_sum(s);
    if (lane == 0) dcond[bt * dl + i] = s;
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
                                                            mask, count, nullptr);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

extern "C" int jz_philox_mask_dev(const int64_t* dev_state, int64_t B_global, int64_t b0, int64_t B_local, int T,
                                  int N, double mask_limit, uint8_t* mask, int* count, jz_stream_t s) {
  JZ_CHECK_ARG(dev_state != nullptr, "philox: null device state");
  JZ_CHECK_ARG(b0 >= 0 && b0 + B_local <= B_global, "philox: shard out of range");
  const int64_t total = B_local * T * N;
  if (total == 0) return JZ_OK;
  PhiloxState st;
  memset(&st, 0, sizeof(st));
  const int threads = 256;
  philox_mask_kernel<<<(unsigned)((total + threads - 1) / threads), threads, 0,
                       reinterpret_cast<cudaStream_t>(s)>>>(st, B_global, b0, B_local, T, N, mask_limit,
                                                            mask, count, dev_state);
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
  {
    int64_t blocks = (rows + 7) / 8;  // 8 warps, one row each per pass
    if (blocks > (int64_t)num_sms() * 16) blocks = (int64_t)num_sms() * 16;
    auto st = reinterpret_cast<cudaStream_t>(s);
    auto launch = [&](auto kern) {
      kern<<<(unsigned)blocks, 256, 0, st>>>(tokens, mask, latents, token_embed, mask_token, null_action, action_w,
                                             action_b, pos_spatial, pos_temporal, rows, T, N, D, dl, K, prepend, x,
                                             err);
    };
    const bool small = rows < (1ll << 31);  // 32-bit row -> (b, t, s) math
#define EMB_FWD(NC)                                                                                  \
  (small ? launch(dyn_embed_fwd_kernel<NC, uint32_t>) : launch(dyn_embed_fwd_kernel<NC, uint64_t>))
    EMB_FWD(0);  // the runtime chunk loop measured faster than the unrolled NC variants at D = 512
#undef EMB_FWD
    JZ_LAUNCH_CHECK();
  }
  return JZ_OK;
}

// ---------------------------------------------------------------------------
// Small-table embedding backward (autodiff.embedding, autodiff.py:344-364): d_table[k] (+)= sum over
// positions i with ids[i] == k of dout[i], in increasing i order.  One CTA per (row k, 128 dims):
// the owner scans every id, so the sum has a fixed order (no atomics) -- meant for action tables
// (gt_action_embed, a handful of rows, a few hundred ids per step).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) table_bwd_kernel(const float* __restrict__ dout, const int64_t* __restrict__ ids,
                                                        int64_t n, int K, int D, float* __restrict__ dtab,
                                                        int accumulate, int* __restrict__ err) {
  const int k = blockIdx.x;
  const int d = blockIdx.y * 128 + threadIdx.x;
  __shared__ int64_t sid[256];
  float acc = 0.f;
  for (int64_t i0 = 0; i0 < n; i0 += 256) {
    __syncthreads();
    for (int j = threadIdx.x; j < 256; j += 128) {
      const int64_t id = i0 + j < n ? ids[i0 + j] : -1;
      sid[j] = id;
      if (i0 + j < n && (id < 0 || id >= K) && err) atomicExch(err, 1);
    }
    __syncthreads();
    const int m = (n - i0) < 256 ? (int)(n - i0) : 256;
    if (d < D)
      for (int j = 0; j < m; ++j)
        if (sid[j] == k) acc += dout[(i0 + j) * D + d];
  }
  if (d < D) dtab[(int64_t)k * D + d] = accumulate ? dtab[(int64_t)k * D + d] + acc : acc;
}

extern "C" int jz_embedding_table_bwd(const float* dout, const int64_t* ids, int64_t n, int K, int D, float* dtable,
                                      int accumulate, int* err, jz_stream_t s) {
  JZ_CHECK_ARG(n >= 0 && K >= 1 && K <= 65535 && D >= 1, "table_bwd: bad sizes n=%lld K=%d D=%d", (long long)n, K, D);
  auto st = reinterpret_cast<cudaStream_t>(s);
  table_bwd_kernel<<<dim3((unsigned)K, (unsigned)((D + 127) / 128)), 128, 0, st>>>(dout, ids, n, K, D, dtable,
                                                                                    accumulate, err);
  JZ_LAUNCH_CHECK();
  return JZ_OK;
}

// Workspace floats needed by jz_dyn_embed_bwd.
extern "C" int64_t jz_dyn_embed_bwd_workspace(int64_t B, int T, int N, int D, int dl, int prepend, int K) {
  const int S = N + (prepend ? 1 : 0);
  const int64_t P = B * T * N;
  const int64_t nb = (P + kTokChunk - 1) / kTokChunk;
  return (int64_t)S * T * D + (int64_t)S * D + (prepend ? 0 : B * T * D) + B * T * dl + 64ll * (dl + 1) * D +
         nb * K + 2 * K + 1 + P;  // token sort: histograms/offsets, starts, totals, sorted positions (int32)
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
  dyn_embed_bwd_pos_kernel<<<dim3(S, D / 128), 32 * kPosGroups, 0, st>>>(dx, mask, B, T, N, D, prepend, d_pos_spatial, part_pt,
                                                           part_mt);
  JZ_LAUNCH_CHECK();
  int rc = jz_reduce_partials(part_pt, S, (int64_t)T * D, d_pos_temporal, 0, s);
  if (rc) return rc;
  rc = jz_reduce_partials(part_mt, S, D, d_mask_token, 0, s);
  if (rc) return rc;
  // token table: stable counting sort of positions by token, then one warp per token
  {
    JZ_CHECK_ARG(K >= 1 && K <= 8192, "embed_bwd: vocabulary %d unsupported (<= 8192)", K);
    const int64_t P = B * T * N;
    const int nb = (int)((P + kTokChunk - 1) / kTokChunk);
    int* hist = reinterpret_cast<int*>(dcond + B * T * dl + 64ll * (dl + 1) * D);
    int* tok_start = hist + (int64_t)nb * K;
    int* total = tok_start + K + 1;
    int32_t* sorted = total + K;
    if (P > 0) {
      tok_hist_kernel<<<nb, 256, K * sizeof(int), st>>>(tokens, mask, P, K, hist);
      JZ_LAUNCH_CHECK();
      tok_colscan_kernel<<<(K + 63) / 64, 64, 0, st>>>(hist, nb, K, total);
      JZ_LAUNCH_CHECK();
    } else {
      JZ_CUDA_TRY(cudaMemsetAsync(total, 0, K * sizeof(int), st));
    }
    tok_scan_kernel<<<1, 1024, 0, st>>>(total, K, tok_start);
    JZ_LAUNCH_CHECK();
    if (P > 0) {
      tok_scatter_kernel<<<nb, 32, K * sizeof(int), st>>>(tokens, mask, P, K, hist, tok_start, sorted);
      JZ_LAUNCH_CHECK();
    }
    const unsigned gk = (unsigned)((K + 7) / 8);
    switch (D / 128) {
      case 1: tok_accum_kernel<1><<<gk, 256, 0, st>>>(dx, sorted, tok_start, K, N, S, prepend, d_token_embed); break;
      case 2: tok_accum_kernel<2><<<gk, 256, 0, st>>>(dx, sorted, tok_start, K, N, S, prepend, d_token_embed); break;
      case 4: tok_accum_kernel<4><<<gk, 256, 0, st>>>(dx, sorted, tok_start, K, N, S, prepend, d_token_embed); break;
      case 8: tok_accum_kernel<8><<<gk, 256, 0, st>>>(dx, sorted, tok_start, K, N, S, prepend, d_token_embed); break;
      default: set_error("embed_bwd: D=%d unsupported", D); return JZ_EINVAL;
    }
    JZ_LAUNCH_CHECK();
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
