// Blackwell (sm_100a) PTX helpers shared by every kernel in libjz:
// mbarriers, TMA bulk-tensor loads, tcgen05 (TMEM alloc / MMA / commit / ld),
// UMMA shared-memory and instruction descriptors, bf16 packing.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define JZ_DEV __device__ __forceinline__

namespace jz {

// ----------------------------------------------------------------------------
// generic helpers
// ----------------------------------------------------------------------------
JZ_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

JZ_DEV uint32_t warp_id() { return threadIdx.x >> 5; }
JZ_DEV uint32_t lane_id() { return threadIdx.x & 31; }

JZ_DEV uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

JZ_DEV float2 unpack_bf16(uint32_t u) {
  __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&u);
  return __bfloat1622float2(v);
}

// ----------------------------------------------------------------------------
// mbarrier
// ----------------------------------------------------------------------------
JZ_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

JZ_DEV void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

JZ_DEV void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

JZ_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

JZ_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

JZ_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, 10000000;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// Wait with back-off: a failed try_wait puts the thread to sleep for `ns` before polling again, so
// warps that wait long (load producers, epilogue warps) do not take issue slots from the compute
// warps on their scheduler.
JZ_DEV void mbar_wait_sleep(uint64_t* bar, uint32_t parity, uint32_t ns) {
  const uint32_t addr = smem_u32(bar);
  while (true) {
    uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(ns);
  }
}

// ----------------------------------------------------------------------------
// TMA (cp.async.bulk.tensor)
// ----------------------------------------------------------------------------
JZ_DEV void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

JZ_DEV void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

JZ_DEV void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0, int32_t c1,
                        int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

JZ_DEV void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int32_t c0, int32_t c1, int32_t c2,
                        int32_t c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// L2 prefetch of a 2-D tensor-map box (no shared-memory destination, no barrier)
JZ_DEV void tma_prefetch_2d(const CUtensorMap* map, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1)
               : "memory");
}

JZ_DEV void tma_store_4d(const CUtensorMap* map, const void* src, int32_t c0, int32_t c1, int32_t c2, int32_t c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}

// TMA store smem -> global (bulk async group), completion tracked per thread
JZ_DEV void tma_store_2d(const CUtensorMap* map, const void* src, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}
// plain bulk copy global -> own CTA's shared memory (16-byte aligned, size a multiple of 16),
// completing `bytes` of transaction count on `bar`
JZ_DEV void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
JZ_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
JZ_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
JZ_DEV void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
JZ_DEV void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// ----------------------------------------------------------------------------
// tcgen05 / TMEM
// ----------------------------------------------------------------------------
template <uint32_t kCols>
JZ_DEV void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}

template <uint32_t kCols>
JZ_DEV void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}

JZ_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
JZ_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem], kind::f16 (bf16 inputs, fp32 accumulate)
JZ_DEV void umma_bf16_ss(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// D[tmem] (+)= A[tmem] * B[smem]
JZ_DEV void umma_bf16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                         uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// Warp-wide variants: the whole (converged) warp calls them with warp-uniform operands and one
// elected lane issues.  Keeping the issuer loop convergent lets ptxas hold descriptors / TMEM
// addresses in uniform registers instead of wrapping every MMA in an elect/R2UR waterfall loop.
JZ_DEV void umma_bf16_ss_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
JZ_DEV void umma_bf16_ts_w(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// Four K-steps into one accumulator (K-major A and B advanced by `astep` / `bstep` descriptor units
// per step) from one elected lane: the first step overwrites when `acc0` is 0.
JZ_DEV void umma4_bf16_ss_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t astep, uint32_t bstep,
                            uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      ".reg .b64 a1, a2, a3, b1, b2, b3;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %6, 0;\n"
      "add.s64 a1, %1, %3; add.s64 a2, a1, %3; add.s64 a3, a2, %3;\n"
      "add.s64 b1, %2, %4; add.s64 b2, b1, %4; add.s64 b3, b2, %4;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %5, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %5, 1;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "l"((uint64_t)astep), "l"((uint64_t)bstep), "r"(idesc), "r"(acc0));
}

// Two accumulators, four K-steps each, interleaved, both operands from shared memory (descriptors
// advanced by `astep` / `bstep` units per step): D0 += A0 B0, D1 += A1 B1.
JZ_DEV void umma4x2_bf16_ss_w(uint32_t d0, uint64_t a0, uint64_t b0, uint32_t d1, uint64_t a1, uint64_t b1,
                              uint32_t astep, uint32_t bstep, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      ".reg .b64 x1, x2, x3, y1, y2, y3, u1, u2, u3, v1, v2, v3;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %9, 0;\n"
      "add.s64 x1, %1, %6; add.s64 x2, x1, %6; add.s64 x3, x2, %6;\n"
      "add.s64 y1, %4, %6; add.s64 y2, y1, %6; add.s64 y3, y2, %6;\n"
      "add.s64 u1, %2, %7; add.s64 u2, u1, %7; add.s64 u3, u2, %7;\n"
      "add.s64 v1, %5, %7; add.s64 v2, v1, %7; add.s64 v3, v2, %7;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %8, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%3], %4, %5, %8, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], x1, u1, %8, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%3], y1, v1, %8, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], x2, u2, %8, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%3], y2, v2, %8, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], x3, u3, %8, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%3], y3, v3, %8, 1;\n"
      "}\n" ::"r"(d0),
      "l"(a0), "l"(b0), "r"(d1), "l"(a1), "l"(b1), "l"((uint64_t)astep), "l"((uint64_t)bstep), "r"(idesc),
      "r"(acc0));
}

// Four K-steps into one accumulator, A from TMEM (columns advanced by `atstep`), B from shared memory.
// `bstep` is added to the whole 64-bit descriptor, so a step may move the address and LBO fields
// in opposite directions (two's-complement step).
JZ_DEV void umma4_bf16_ts_w(uint32_t tmem_d, uint32_t a0, uint64_t bdesc, uint32_t atstep, uint64_t bstep,
                            uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      ".reg .b32 x1, x2, x3;\n"
      ".reg .b64 u1, u2, u3;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %6, 0;\n"
      "add.u32 x1, %1, %3; add.u32 x2, x1, %3; add.u32 x3, x2, %3;\n"
      "add.s64 u1, %2, %4; add.s64 u2, u1, %4; add.s64 u3, u2, %4;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %5, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x1], u1, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x2], u2, %5, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x3], u3, %5, 1;\n"
      "}\n" ::"r"(tmem_d),
      "r"(a0), "l"(bdesc), "r"(atstep), "l"((uint64_t)bstep), "r"(idesc), "r"(acc0));
}

// Two accumulators, four K-steps each, interleaved, A from TMEM (columns advanced by `atstep`),
// B from shared memory (descriptor advanced by `bstep`): D0 += A0 B0, D1 += A1 B1 step by step.
JZ_DEV void umma4x2_bf16_ts_w(uint32_t d0, uint32_t a0, uint64_t b0, uint32_t d1, uint32_t a1, uint64_t b1,
                              uint32_t atstep, uint32_t bstep, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      ".reg .b32 x1, x2, x3, y1, y2, y3;\n"
      ".reg .b64 u1, u2, u3, v1, v2, v3;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %9, 0;\n"
      "add.u32 x1, %1, %6; add.u32 x2, x1, %6; add.u32 x3, x2, %6;\n"
      "add.u32 y1, %4, %6; add.u32 y2, y1, %6; add.u32 y3, y2, %6;\n"
      "add.s64 u1, %2, %7; add.s64 u2, u1, %7; add.s64 u3, u2, %7;\n"
      "add.s64 v1, %5, %7; add.s64 v2, v1, %7; add.s64 v3, v2, %7;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %8, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%3], [%4], %5, %8, p;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x1], u1, %8, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%3], [y1], v1, %8, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x2], u2, %8, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%3], [y2], v2, %8, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [x3], u3, %8, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%3], [y3], v3, %8, 1;\n"
      "}\n" ::"r"(d0),
      "r"(a0), "l"(b0), "r"(d1), "r"(a1), "l"(b1), "r"(atstep), "l"((uint64_t)bstep), "r"(idesc), "r"(acc0));
}

// smem (matrix descriptor) -> TMEM copy of 128 rows x 256 bits; warp-wide, one elected lane issues
JZ_DEV void tmem_cp_128x256b_w(uint32_t taddr, uint64_t sdesc) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.cp.cta_group::1.128x256b [%0], %1;\n"
      "}\n" ::"r"(taddr),
      "l"(sdesc));
}
JZ_DEV void umma_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// Arrive on an mbarrier once every previously issued tcgen05 op of this thread completed.
JZ_DEV void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// ----------------------------------------------------------------------------
// CTA pair (cluster of 2, cta_group::2): one MMA spans both SMs' tensor cores,
// each CTA holds half of A (its 128 rows) and half of B, and receives its own
// 128-lane slice of the accumulator in its TMEM.
// ----------------------------------------------------------------------------
JZ_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// shared::cta address of this CTA -> shared::cluster address of the same offset in CTA `rank`
JZ_DEV uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

JZ_DEV void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// Relaxed arrivals for "TMEM drained" barriers: the arriving thread's tcgen05.ld already completed
// (tcgen05.wait::ld) and no generic memory has to be published, so no release fence is needed.
// (A release arrive waits on every outstanding memory op of the thread: the epilogue's lane 0 also
// issued the tile's bulk stores, and that wait was a quarter of the GEMM's stall samples.)
JZ_DEV void mbar_arrive_relaxed(uint64_t* bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
JZ_DEV void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

JZ_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// TMA load into this CTA's smem whose completion bytes are signalled on an mbarrier that may
// live in the peer CTA (the pair leader's full barrier).
JZ_DEV void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t mbar_cluster, int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar_cluster), "r"(c0), "r"(c1)
      : "memory");
}

template <uint32_t kCols>
JZ_DEV void tmem_alloc_pair(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}

template <uint32_t kCols>
JZ_DEV void tmem_dealloc_pair(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols));
}

JZ_DEV void umma_bf16_ss_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                              uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// warp-wide (elect-one) variants of the pair MMA / commit, see umma_bf16_ss_w
JZ_DEV void umma_bf16_ss_pair_w(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
JZ_DEV void umma_commit_pair_w(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n"
      ".reg .pred e;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// Commit the pair's MMAs to the mbarrier at the same offset in every CTA of `mask`.
JZ_DEV void umma_commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// 32 lanes x 32 consecutive fp32 columns: thread i of the warp gets row (lane base + i).
JZ_DEV void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

JZ_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 columns loaded and waited for in one asm statement: the compiler cannot schedule a use of the
// destination registers between the load and tcgen05.wait::ld.
JZ_DEV void tmem_ld_32x32b_x32_wait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
}

// 2 x 32 columns (at taddr and taddr + 32), one wait
JZ_DEV void tmem_ld_32x32b_x64_wait(uint32_t taddr, uint32_t (&r)[64]) {
  asm volatile(
      "{\n.reg .b32 t2;\nadd.u32 t2, %64, 32;\n"
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%64];\n"
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [t2];\n"
      "tcgen05.wait::ld.sync.aligned;\n}"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr)
      : "memory");
}

// 32 lanes x 16 consecutive fp32 columns
JZ_DEV void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// 32 lanes x 16 consecutive 32-bit columns (store registers -> TMEM)
JZ_DEV void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

// 32 lanes x 8 consecutive 32-bit columns (store registers -> TMEM)
JZ_DEV void tmem_st_32x32b_x8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

// 32 lanes x one fp32 column
JZ_DEV uint32_t tmem_ld_32x32b_x1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  return r;
}

JZ_DEV void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ----------------------------------------------------------------------------
// UMMA descriptors (see PTX ISA "Matrix Descriptors" for tcgen05)
// ----------------------------------------------------------------------------
// Shared-memory matrix descriptor, 128-byte swizzle, version 1 (sm_100).
//   K-major tiles : rows of 64 bf16 (128 B) along K, 8-row atoms 1024 B apart (SBO).
//   MN-major tiles: 64 bf16 (128 B) along M/N per row, rows along K; 8-row atoms 1024 B apart
//                   along K (SBO), 64-element MN atoms `lbo` bytes apart (LBO).
JZ_DEV uint64_t sdesc_sw128(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor for kind::f16 with bf16 A/B and fp32 D.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(uint32_t M, uint32_t N, bool a_mn_major,
                                                      bool b_mn_major) {
  return (1u << 4)                       // D format: F32
         | (1u << 7)                     // A format: BF16
         | (1u << 10)                    // B format: BF16
         | ((a_mn_major ? 1u : 0u) << 15)  // A major
         | ((b_mn_major ? 1u : 0u) << 16)  // B major
         | ((N >> 3) << 17)              // N >> 3
         | ((M >> 4) << 24);             // M >> 4
}

// ----------------------------------------------------------------------------
// math
// ----------------------------------------------------------------------------
// tanh-approximation GELU, reference deskworld/nn.py:28-32
JZ_DEV float gelu_tanh(float x) {
  const float c = 0.7978845608028654f;  // sqrt(2/pi)
  float inner = (x + 0.044715f * (x * x * x)) * c;
  return 0.5f * (x * (1.0f + tanhf(inner)));
}

JZ_DEV float gelu_tanh_grad(float x) {
  const float c = 0.7978845608028654f;
  float x2 = x * x;
  float inner = (x + 0.044715f * x2 * x) * c;
  float t = tanhf(inner);
  float dinner = c * (1.0f + 3.0f * 0.044715f * x2);
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * dinner;
}

JZ_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

JZ_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace jz
