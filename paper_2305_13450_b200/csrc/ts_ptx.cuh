// ts_ptx.cuh — thin inline-PTX wrappers for sm_100a: mbarrier, TMA, tcgen05/TMEM,
// release/acquire semaphores. Nothing here is policy-specific.
#pragma once
#include <cuda.h>
#include <stdint.h>

namespace ts {
namespace ptx {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint32_t lane_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t sm_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint64_t global_timer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ---- mbarrier ------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

// try_wait with a suspend-time hint: the waiting thread sleeps in hardware until the
// phase completes (or the hint expires) instead of re-issuing the probe.
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity), "r"(0x989680u)
      : "memory");
  return ok != 0;
}

// Non-blocking probe (no suspension): has the phase with `parity` completed?
__device__ __forceinline__ bool mbar_test_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Wait for a barrier whose arrivals publish shared-memory data written by the peer CTA
// (st.shared::cluster + mbarrier.arrive.release.cluster). The probe loop stays at CTA
// scope — a cluster-scope acquire on every probe compiles to an L1 invalidate
// (CCTL.IVALL) per iteration — and one cluster fence after the phase flips makes the
// peer's writes visible.
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  mbar_wait(bar, parity);
  asm volatile("fence.acq_rel.cluster;" ::: "memory");
}

// ---- clusters ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// shared::cluster address of the same shared variable in CTA `rank` of this cluster.
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}

__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}

__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}

// ---- TMA -------------------------------------------------------------------------------
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

// 2-D tiled load global -> shared, completion counted on `bar` (complete_tx::bytes).
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* m, uint64_t* bar,
                                            int c0, int c1, uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(cache_hint)
      : "memory");
}

// CTA-pair variant: each CTA loads into its own shared memory, completion bytes are
// counted on the leader's barrier (`bar_cluster` = mapa(bar, 0)).
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* m,
                                                 uint32_t bar_cluster, int c0, int c1,
                                                 uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c0), "r"(c1), "l"(cache_hint)
      : "memory");
}

// CTA-pair multicast variant: the box lands at the same CTA-relative offset in every CTA
// of `mask`; each destination's bytes are counted on its own pair leader's barrier
// (`bar_cluster` = this CTA's pair-leader barrier: .cta_group::2 resolves the leader per
// destination pair, as CUTLASS's SM100_TMA_2SM_LOAD_MULTICAST does).
__device__ __forceinline__ void tma_load_2d_pair_mc(void* dst, const CUtensorMap* m,
                                                    uint32_t bar_cluster, int c0, int c1,
                                                    uint16_t mask, uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster.L2::cache_hint [%0], [%1, {%4, %5}], [%2], %3, %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "h"(mask), "r"(c0), "r"(c1),
      "l"(cache_hint)
      : "memory");
}

// 4-D im2col load (NHWC): `pixelsPerColumn` consecutive pixels of the map's bounding box
// from (w, h, n), channels [c, c + channelsPerPixel), each pixel shifted by the filter
// tap offsets (ow, oh); out-of-image pixels read as zero.
// 4-D tiled box (halo-staged convolution windows: (C, W, H, N), negative / past-the-edge
// coordinates zero-filled).
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c,
                                            int w, int h, int n, uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n),
      "l"(cache_hint)
      : "memory");
}

__device__ __forceinline__ void tma_load_im2col(void* dst, const CUtensorMap* m, uint64_t* bar,
                                                int c, int w, int h, int n, uint16_t ow,
                                                uint16_t oh, uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8}, %9;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n),
      "h"(ow), "h"(oh), "l"(cache_hint)
      : "memory");
}

__device__ __forceinline__ void tma_load_im2col_pair(void* dst, const CUtensorMap* m,
                                                     uint32_t bar_cluster, int c, int w, int h,
                                                     int n, uint16_t ow, uint16_t oh,
                                                     uint64_t cache_hint) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx"
      "::bytes.L2::cache_hint [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8}, %9;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c), "r"(w), "r"(h), "r"(n),
      "h"(ow), "h"(oh), "l"(cache_hint)
      : "memory");
}

// L2 cache-policy descriptors (createpolicy) for streaming weights vs reused activations.
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Order this thread's generic-proxy view of global memory before its later async-proxy
// (TMA) accesses, and vice versa.
// generic-proxy shared-memory writes -> async proxy (tcgen05.mma / TMA reads of them)
__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ---- semaphores (the paper's wait_till / post) ------------------------
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Polling load: relaxed (no L1 invalidate per probe); pair with fence_acquire_gpu().
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void fence_acq_rel_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

// Release reduction without a returned value (fire and forget: no round trip on the
// posting thread's critical path).
__device__ __forceinline__ void red_add_release_gpu(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int atom_add_release_gpu(int* p, int v) {
  int old;
  asm volatile("atom.add.release.gpu.global.s32 %0, [%1], %2;"
               : "=r"(old)
               : "l"(p), "r"(v)
               : "memory");
  return old;
}

// System scope (peer GPUs over NVLink / P2P): the tensor-parallel all-reduce stage.
__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int ld_relaxed_sys(const int* p) {
  int v;
  asm volatile("ld.relaxed.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void fence_acq_rel_sys() {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

__device__ __forceinline__ int atom_add_release_sys(int* p, int v) {
  int old;
  asm volatile("atom.add.release.sys.global.s32 %0, [%1], %2;"
               : "=r"(old)
               : "l"(p), "r"(v)
               : "memory");
  return old;
}

// 16-byte asynchronous global -> shared copy (LDGSTS, L2 only) and its completion wait:
// many copies in flight per thread without holding registers.
__device__ __forceinline__ void cp_async16(uint32_t dst_smem, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst_smem), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// 128-bit load that bypasses L1 (peer data is read once, after a system-scope acquire).
__device__ __forceinline__ uint4 ld_global_cg_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

// 128-bit global store with an L2 cache-policy hint (createpolicy): split-K partial
// planes are written evict_last so they are still in L2 when the summing slice reads them.
__device__ __forceinline__ void st_global_v4_hint(void* p, uint4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}

// 128-bit L2-only load with a cache-policy hint (evict_first: a partial plane dies here).
__device__ __forceinline__ float4 ld_global_cg_f4_hint(const float* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.cg.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// 256-bit global store (sm_100: STG.256, one full 32-B sector per lane).
__device__ __forceinline__ void st_global_v8(void* p, const uint32_t* v) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}

// ---- tcgen05 / TMEM -------------------------------------------------------------------
template <uint32_t kCols, int CG>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {
  if constexpr (CG == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  } else {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(dst_smem)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
}

template <uint32_t kCols, int CG>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  if constexpr (CG == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
  } else {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols)
                 : "memory");
  }
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16 (fp16/bf16 in, fp32 accumulate).
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// CTA-pair MMA (issued by the leader): A rows split across the pair (128 each), B rows
// split (N/2 each), each CTA's TMEM receives its 128 x N slice of D.
__device__ __forceinline__ void umma_f16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Pair commit: arrive on the barrier at the same offset in both CTAs (mask 0b11).
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

// Pair commit to the barrier at the same offset in every CTA of `mask` (two pairs sharing
// multicast operands: the ring entries of all four CTAs).
__device__ __forceinline__ void umma_commit_pair_mask(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// Four K=16 sub-steps of one 64-wide K-block in a single issue sequence. `adesc`/`bdesc`
// address the first sub-step; each next one starts 32 bytes further inside the 128-B
// swizzle row (descriptor address field += 2). `acc0` = accumulate flag of sub-step 0.
template <int CG>
__device__ __forceinline__ void umma_f16_kblock(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                                uint32_t idesc, uint32_t acc0) {
  if constexpr (CG == 2) {
    asm volatile(
        "{\n\t.reg .pred p, t;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "setp.eq.b32 t, %4, %4;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %5, %6, %3, t;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %7, %8, %3, t;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %9, %10, %3, t;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc0), "l"(adesc + 2), "l"(bdesc + 2),
        "l"(adesc + 4), "l"(bdesc + 4), "l"(adesc + 6), "l"(bdesc + 6)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p, t;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "setp.eq.b32 t, %4, %4;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %5, %6, %3, t;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %7, %8, %3, t;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %9, %10, %3, t;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc0), "l"(adesc + 2), "l"(bdesc + 2),
        "l"(adesc + 4), "l"(bdesc + 4), "l"(adesc + 6), "l"(bdesc + 6)
        : "memory");
  }
}

// One 64-wide K-block into TWO accumulators, interleaved: d0 += A * B0^T and d1 += A * B1^T
// one 16-deep sub-step at a time, so consecutive MMAs never target the same accumulator.
// Back-to-back MMAs into one accumulator serialize on its read-modify-write (measured,
// scripts/mma_rate.cu: 141 cycles per M=128 N=256 MMA against a 128-cycle floor, 91 cycles
// for N<=128); alternating accumulators issue at the floor.
template <int CG>
__device__ __forceinline__ void umma_f16_kblock2(uint32_t d0, uint32_t d1, uint64_t adesc,
                                                 uint64_t b0, uint64_t b1, uint32_t idesc,
                                                 uint32_t acc0) {
  if constexpr (CG == 2) {
    asm volatile(
        "{\n\t.reg .pred p, t;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "setp.eq.b32 t, %6, %6;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %3, %5, p;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%1], %2, %4, %5, p;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %7, %8, %5, t;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%1], %7, %9, %5, t;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %10, %11, %5, t;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%1], %10, %12, %5, t;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %13, %14, %5, t;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%1], %13, %15, %5, t;\n\t}" ::"r"(d0),
        "r"(d1), "l"(adesc), "l"(b0), "l"(b1), "r"(idesc), "r"(acc0), "l"(adesc + 2),
        "l"(b0 + 2), "l"(b1 + 2), "l"(adesc + 4), "l"(b0 + 4), "l"(b1 + 4), "l"(adesc + 6),
        "l"(b0 + 6), "l"(b1 + 6)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p, t;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "setp.eq.b32 t, %6, %6;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %5, p;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %4, %5, p;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %7, %8, %5, t;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], %7, %9, %5, t;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %10, %11, %5, t;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], %10, %12, %5, t;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %13, %14, %5, t;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%1], %13, %15, %5, t;\n\t}" ::"r"(d0),
        "r"(d1), "l"(adesc), "l"(b0), "l"(b1), "r"(idesc), "r"(acc0), "l"(adesc + 2),
        "l"(b0 + 2), "l"(b1 + 2), "l"(adesc + 4), "l"(b0 + 4), "l"(b1 + 4), "l"(adesc + 6),
        "l"(b0 + 6), "l"(b1 + 6)
        : "memory");
  }
}

// Four K=16 sub-steps of one K-block into four (possibly different) accumulators
// d0..d3 with per-sub-step accumulate flags, in one issue sequence (single CTA).
__device__ __forceinline__ void umma_f16_kblock4(uint32_t d0, uint32_t d1, uint32_t d2,
                                                 uint32_t d3, uint64_t adesc, uint64_t bdesc,
                                                 uint32_t idesc, uint32_t accmask) {
  asm volatile(
      "{\n\t.reg .pred p0, p1, p2, p3;\n\t"
      "setp.ne.b32 p0, %8, 0;\n\t"
      "setp.ne.b32 p1, %9, 0;\n\t"
      "setp.ne.b32 p2, %10, 0;\n\t"
      "setp.ne.b32 p3, %11, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %5, %6, p0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%1], %12, %13, %6, p1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%2], %14, %15, %6, p2;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%3], %16, %17, %6, p3;\n\t}" ::"r"(d0),
      "r"(d1), "r"(d2), "r"(d3), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(0),
      "r"(accmask & 1), "r"(accmask & 2), "r"(accmask & 4), "r"(accmask & 8), "l"(adesc + 2),
      "l"(bdesc + 2), "l"(adesc + 4), "l"(bdesc + 4), "l"(adesc + 6), "l"(bdesc + 6)
      : "memory");
}

// Arrive on `bar` once every previously issued tcgen05.mma of this thread completes.
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// 32 lanes x 32 columns of 32-bit: thread i receives TMEM lane (base+i), 32 columns.
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
}

// 32 lanes x 16 columns of 32-bit: thread i receives TMEM lane (base+i), 16 columns.
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor for a K-major tile written by TMA with 128-byte
// swizzle: rows of 64 16-bit elements (128 B), 8-row core groups 1024 B apart.
// Bits: [0,14) addr>>4, [16,30) LBO>>4 (unused for swizzled K-major, 1 by convention),
// [32,46) SBO>>4, [46,48) version = 1 (sm_100), [61,64) layout = 2 (SWIZZLE_128B).
__device__ __forceinline__ uint64_t smem_desc_k_sw128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>(1u) << 16;
  d |= static_cast<uint64_t>(1024u >> 4) << 32;
  d |= static_cast<uint64_t>(1u) << 46;
  d |= static_cast<uint64_t>(2u) << 61;
  return d;
}

// Instruction descriptor for kind::f16, fp32 accumulate, both operands K-major.
//   [4,6) D fmt = 1 (f32), [7,10) A fmt, [10,13) B fmt (0 f16, 1 bf16),
//   [15] A major = 0, [16] B major = 0, [17,23) N>>3, [24,29) M>>4.
// Instruction descriptor for kind::tf32 (A, B tf32 = 2, D f32), both K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(uint32_t m, uint32_t n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

// One 32-deep K block of kind::tf32 MMAs (4 x K = 8, 32 bytes each) accumulating into D:
// the split-K reduction D += P x I over a 32-column group of a partial plane P.
template <int CG>
__device__ __forceinline__ void umma_tf32_kblock(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                                 uint32_t idesc) {
  if constexpr (CG == 2) {
    asm volatile(
        "{\n\t.reg .pred t;\n\t"
        "setp.eq.b32 t, %3, %3;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, t;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %4, %5, %3, t;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %6, %7, %3, t;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %8, %9, %3, t;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "l"(adesc + 2), "l"(bdesc + 2), "l"(adesc + 4),
        "l"(bdesc + 4), "l"(adesc + 6), "l"(bdesc + 6)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred t;\n\t"
        "setp.eq.b32 t, %3, %3;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, t;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %4, %5, %3, t;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %6, %7, %3, t;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %8, %9, %3, t;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "l"(adesc + 2), "l"(bdesc + 2), "l"(adesc + 4),
        "l"(bdesc + 4), "l"(adesc + 6), "l"(bdesc + 6)
        : "memory");
  }
}

__host__ __device__ constexpr uint32_t idesc_f16(uint32_t m, uint32_t n, uint32_t ab_fmt) {
  return (1u << 4) | (ab_fmt << 7) | (ab_fmt << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

}  // namespace ptx
}  // namespace ts
