// ts_chain_kernel.cuh — persistent, warp-specialized tcgen05 GeMM over a chain of
// dependent tile stages, with the paper's tile-level semaphore protocol.
//
// One launch processes every tile of every stage. Work items are the stages' tiles laid
// end to end (stage 0's tiles first); a single global atomic counter hands them out, so
// any producer tile a consumer waits on was claimed earlier by a CTA that is already
// running it — the persistent replacement for the paper's wait kernel
// (engine.py:183-204). Within a stage, the n-th claim computes tile
// order_tile(order, grid, n) (the paper's stage.tile(); policies.py:181).
//
// Per CTA (256 threads, one CTA per SM):
//   warp 0 lane 0 : scheduler + TMA producer. For a consumer tile it issues the weight
//                   (B) tile first, then spins on the policy's semaphore (ld.acquire.gpu)
//                   and issues the dependent A tile ("+R", PAPER.md:534-540;
//                   kstep_duration engine.py:207-217).
//   warp 1        : tcgen05.mma issuer (one lane), fp32 accumulators in TMEM,
//                   double-buffered so the epilogue of tile i overlaps the mainloop of i+1.
//   warp 2        : TMEM allocator.
//   warps 4-7     : epilogue: tcgen05.ld -> GeLU/SwiGLU -> global stores, then one
//                   thread posts (fence + red.release.gpu) to every outgoing dependency
//                   (stage.post; post_target policies.py:128-142).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "tilesync.h"
#include "ts_policy.cuh"
#include "ts_ptx.cuh"

namespace ts {

constexpr int kBM = 128;        // UMMA M (rows of a tile)
constexpr int kBK = 64;         // K elements per smem stage = one 128-B swizzle row
constexpr int kThreads = 256;
constexpr int kTileRing = 4;    // tile-id hand-off ring between scheduler and consumers
constexpr int kEpiThreads = 128;
constexpr uint64_t kWatchdogNs = 4000000000ull;

struct StageParams {
  CUtensorMap tmap_a;  // [m, k] K-major, box {64, 128}, 128-B swizzle
  CUtensorMap tmap_b;  // [n, k] K-major, box {64, BN}, 128-B swizzle
  void* c;
  int m, n, k, ldc;
  int grid_x, grid_y;
  int order, order_stride;
  int epilogue;
  int k_blocks;
  int item_begin, item_end;
  int in_dep;  // dependency feeding operand A, or -1
  int n_out_deps;
  int out_deps[TS_MAX_DEPS];
};

struct DepParams {
  int* sem;
  int policy, param;
  int pgx, pgy, pgz;    // producer grid (reference Stage.grid)
  int kb_per_kstep;     // consumer K-blocks per reference k-step
  int sem_n;
};

struct ChainParams {
  StageParams st[TS_MAX_STAGES];
  DepParams dep[TS_MAX_DEPS];
  int n_stages, n_deps, total_items;
  int item_lo, item_hi;  // this launch claims global items [item_lo, item_hi)
  int* scratch;
  ts_trace_rec* trace;
  int trace_cap;
  int flags;
};

template <int BN>
struct Cfg {
  static constexpr int kStages = (BN == 256) ? 4 : (BN == 128 ? 6 : 8);
  static constexpr int kABytes = kBM * kBK * 2;
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;  // two accumulator buffers
  static constexpr int kBarOffset = kStages * kStageBytes;
  // full, empty per stage; tmem full/empty x2; tile ring full/empty x kTileRing
  static constexpr int kNumBars = 2 * kStages + 4 + 2 * kTileRing;
  static constexpr int kSmemBytes = 1024 + kBarOffset + kNumBars * 8 + 64;
};

__device__ __forceinline__ int stage_of(const ChainParams& p, int g) {
  int s = 0;
#pragma unroll 1
  while (s + 1 < p.n_stages && g >= p.st[s + 1].item_begin) ++s;
  return s;
}

__device__ __forceinline__ void trace_event(const ChainParams& p, uint64_t t, int kind,
                                            int stage, int tb, int k, int dep, int sem,
                                            int value, int x, int y) {
  if (p.trace == nullptr) return;
  int slot = atomicAdd(&p.scratch[2], 1);
  if (slot >= p.trace_cap) return;
  ts_trace_rec r;
  r.t_ns = t;
  r.kind = kind;
  r.stage = stage;
  r.tb = tb;
  r.k = k;
  r.dep = dep;
  r.sem = sem;
  r.value = value;
  r.x = static_cast<int16_t>(x);
  r.y = static_cast<int16_t>(y);
  r.z = 0;
  r.smid = static_cast<int16_t>(ptx::sm_id());
  r.pad = 0;
  p.trace[slot] = r;
}

template <typename T>
struct AbFormat;
template <>
struct AbFormat<__half> {
  static constexpr uint32_t value = 0;
};
template <>
struct AbFormat<__nv_bfloat16> {
  static constexpr uint32_t value = 1;
};

__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
}

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

template <typename T>
__device__ __forceinline__ uint32_t pack2(float a, float b);
template <>
__device__ __forceinline__ uint32_t pack2<__half>(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Spin until sem >= expected (the paper's wait_till, relaxed to >= so
// the semaphores stay monotone as in SemaphoreArray, policies.py:84-99).
__device__ __forceinline__ void sem_wait(const ChainParams& p, const int* sem, int expected) {
  if (ptx::ld_acquire_gpu(sem) >= expected) return;
  const bool watchdog = (p.flags & TS_FLAG_NO_WATCHDOG) == 0;
  uint64_t t0 = ptx::global_timer();
#pragma unroll 1
  while (ptx::ld_acquire_gpu(sem) < expected) {
    __nanosleep(40);
    if (watchdog && ptx::global_timer() - t0 > kWatchdogNs) {
      atomicExch(&p.scratch[3], 1);
      return;
    }
  }
}

template <int BN, typename T>
__global__ void __launch_bounds__(kThreads, 1) chain_kernel(const __grid_constant__ ChainParams p) {
  using C = Cfg<BN>;
  constexpr int S = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;                       // S x [128 x 64]
  uint8_t* sB = smem + S * C::kABytes;      // S x [BN x 64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOffset);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* tmem_full = bars + 2 * S;
  uint64_t* tmem_empty = tmem_full + 2;
  uint64_t* ti_full = tmem_empty + 2;
  uint64_t* ti_empty = ti_full + kTileRing;
  int* ti_item = reinterpret_cast<int*>(ti_empty + kTileRing);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(ti_item + kTileRing);
  int* last_flag = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&tmem_full[i], 1);
      ptx::mbar_init(&tmem_empty[i], kEpiThreads / 32);
    }
    for (int i = 0; i < kTileRing; ++i) {
      ptx::mbar_init(&ti_full[i], 1);
      ptx::mbar_init(&ti_empty[i], 1 + kEpiThreads / 32);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.n_stages; ++s) {
      ptx::tma_prefetch_desc(&p.st[s].tmap_a);
      ptx::tma_prefetch_desc(&p.st[s].tmap_b);
    }
  }
  if (warp == 2) ptx::tmem_alloc<C::kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== scheduler + TMA producer =====================
    if (lane == 0) {
      const bool reorder = (p.flags & TS_FLAG_NO_REORDER) == 0;
      const uint64_t pol_stream = ptx::policy_evict_first();  // weights: read once
      const uint64_t pol_keep = ptx::policy_evict_last();     // activations: reused
      uint32_t pipe = 0;
#pragma unroll 1
      for (int it = 0;; ++it) {
        const int slot = it % kTileRing;
        ptx::mbar_wait(&ti_empty[slot], ((it / kTileRing) & 1) ^ 1);
        int g = p.item_lo + atomicAdd(&p.scratch[0], 1);
        if (g >= p.item_hi) g = -1;
        ti_item[slot] = g;
        ptx::mbar_arrive(&ti_full[slot]);
        if (g < 0) break;
        const int s = stage_of(p, g);
        const StageParams& st = p.st[s];
        const int tb = g - st.item_begin;
        int tx, ty, tz;
        order_tile(st.order, st.order_stride, Grid3{st.grid_x, st.grid_y, 1}, tb, &tx, &ty, &tz);
        trace_event(p, ptx::global_timer(), 0, s, tb, -1, -1, -1, -1, tx, ty);
        const int m0 = tx * kBM;
        const int n0 = ty * BN;
        const int d = st.in_dep;
#pragma unroll 1
        for (int kb = 0; kb < st.k_blocks; ++kb, ++pipe) {
          const int rs = pipe % S;
          ptx::mbar_wait(&empty[rs], ((pipe / S) & 1) ^ 1);
          ptx::mbar_arrive_expect_tx(&full[rs], C::kStageBytes);
          uint8_t* a_dst = sA + rs * C::kABytes;
          uint8_t* b_dst = sB + rs * C::kBBytes;
          if (reorder) ptx::tma_load_2d(b_dst, &st.tmap_b, &full[rs], kb * kBK, n0, pol_stream);
          if (d >= 0) {
            const DepParams& dp = p.dep[d];
            if (kb % dp.kb_per_kstep == 0) {
              const int kstep = kb / dp.kb_per_kstep;
              Wait w = consumer_wait(dp.policy, dp.param, tx, ty, kstep,
                                     Grid3{dp.pgx, dp.pgy, dp.pgz}, dp.pgz);
              if (w.sem >= 0) {
                trace_event(p, ptx::global_timer(), 1, s, tb, kstep, d, w.sem, w.expected, tx, ty);
                sem_wait(p, dp.sem + w.sem, w.expected);
                trace_event(p, ptx::global_timer(), 2, s, tb, kstep, d, w.sem, w.expected, tx, ty);
                ptx::fence_proxy_async_global();
              }
            }
          }
          ptx::tma_load_2d(a_dst, &st.tmap_a, &full[rs], kb * kBK, m0, pol_keep);
          if (!reorder) ptx::tma_load_2d(b_dst, &st.tmap_b, &full[rs], kb * kBK, n0, pol_stream);
        }
      }
    }
  } else if (warp == 1) {
    // ===================== tcgen05.mma issuer =====================
    constexpr uint32_t kIdesc = ptx::idesc_f16(kBM, BN, AbFormat<T>::value);
    uint32_t pipe = 0;
    uint32_t local = 0;
#pragma unroll 1
    for (int it = 0;; ++it) {
      const int slot = it % kTileRing;
      ptx::mbar_wait(&ti_full[slot], (it / kTileRing) & 1);
      const int g = ti_item[slot];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&ti_empty[slot]);
      if (g < 0) break;
      const int kblocks = p.st[stage_of(p, g)].k_blocks;
      const uint32_t acc = local & 1;
      ptx::mbar_wait(&tmem_empty[acc], ((local >> 1) & 1) ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
#pragma unroll 1
      for (int kb = 0; kb < kblocks; ++kb, ++pipe) {
        const int rs = pipe % S;
        ptx::mbar_wait(&full[rs], (pipe / S) & 1);
        ptx::tc_fence_after();
        if (lane == 0) {
          const uint32_t a_addr = ptx::smem_u32(sA + rs * C::kABytes);
          const uint32_t b_addr = ptx::smem_u32(sB + rs * C::kBBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            ptx::umma_f16(d_tmem, ptx::smem_desc_k_sw128(a_addr + k * 32),
                          ptx::smem_desc_k_sw128(b_addr + k * 32), kIdesc, (kb | k) != 0);
          }
          ptx::umma_commit(&empty[rs]);
        }
        __syncwarp();
      }
      if (lane == 0) ptx::umma_commit(&tmem_full[acc]);
      __syncwarp();
      ++local;
    }
  } else if (warp >= 4) {
    // ===================== epilogue =====================
    const int ew = warp - 4;  // == warp % 4: TMEM lanes [32*ew, 32*ew+32)
    uint32_t local = 0;
#pragma unroll 1
    for (int it = 0;; ++it) {
      const int slot = it % kTileRing;
      ptx::mbar_wait(&ti_full[slot], (it / kTileRing) & 1);
      const int g = ti_item[slot];
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&ti_empty[slot]);
      if (g < 0) break;
      const int s = stage_of(p, g);
      const StageParams& st = p.st[s];
      const int tb = g - st.item_begin;
      int tx, ty, tz;
      order_tile(st.order, st.order_stride, Grid3{st.grid_x, st.grid_y, 1}, tb, &tx, &ty, &tz);
      const uint32_t acc = local & 1;
      ptx::mbar_wait(&tmem_full[acc], (local >> 1) & 1);
      ptx::tc_fence_after();
      const int row = tx * kBM + ew * 32 + lane;
      const bool row_ok = row < st.m;
      const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN;
      T* crow = reinterpret_cast<T*>(st.c) + static_cast<size_t>(row) * st.ldc;
      if (st.epilogue == TS_EPI_SWIGLU) {
        T* out = crow + ty * (BN / 2);
#pragma unroll 1
        for (int cc = 0; cc < BN / 64; ++cc) {
          uint32_t gr[32], ur[32];
          ptx::tmem_ld_32x32b_x32(t_lane + cc * 32, gr);
          ptx::tmem_ld_32x32b_x32(t_lane + BN / 2 + cc * 32, ur);
          ptx::tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float g0 = __uint_as_float(gr[2 * j]), g1 = __uint_as_float(gr[2 * j + 1]);
            float u0 = __uint_as_float(ur[2 * j]), u1 = __uint_as_float(ur[2 * j + 1]);
            pk[j] = pack2<T>(silu(g0) * u0, silu(g1) * u1);
          }
          if (row_ok) {
            uint4* dst = reinterpret_cast<uint4*>(out + cc * 32);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          }
        }
      } else {
        T* out = crow + ty * BN;
        const bool gelu = st.epilogue == TS_EPI_GELU;
#pragma unroll 1
        for (int cc = 0; cc < BN / 32; ++cc) {
          uint32_t r[32];
          ptx::tmem_ld_32x32b_x32(t_lane + cc * 32, r);
          ptx::tmem_ld_wait();
          uint32_t pk[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            float v0 = __uint_as_float(r[2 * j]), v1 = __uint_as_float(r[2 * j + 1]);
            if (gelu) {
              v0 = gelu_erf(v0);
              v1 = gelu_erf(v1);
            }
            pk[j] = pack2<T>(v0, v1);
          }
          if (row_ok) {
            uint4* dst = reinterpret_cast<uint4*>(out + cc * 32);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              dst[q] = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
          }
        }
      }
      ptx::tc_fence_before();
      if (lane == 0) ptx::mbar_arrive(&tmem_empty[acc]);
      // stage.post(): every epilogue thread's stores happen-before the release below.
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
      if (threadIdx.x == 128 && st.n_out_deps > 0) {
        const uint64_t t = ptx::global_timer();
        __threadfence();
        ptx::fence_proxy_async_global();
        for (int i = 0; i < st.n_out_deps; ++i) {
          const int d = st.out_deps[i];
          const DepParams& dp = p.dep[d];
          const int idx = post_target(dp.policy, dp.param, tx, ty, Grid3{dp.pgx, dp.pgy, dp.pgz});
          const int old = ptx::atom_add_release_gpu(dp.sem + idx, 1);
          trace_event(p, t, 3, s, tb, -1, d, idx, old + 1, tx, ty);
        }
        trace_event(p, t, 4, s, tb, -1, -1, -1, -1, tx, ty);
      } else if (threadIdx.x == 128) {
        trace_event(p, ptx::global_timer(), 4, s, tb, -1, -1, -1, -1, tx, ty);
      }
      ++local;
    }
  }

  // ---- teardown: free TMEM; the last CTA out restores the zero invariant -------------
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
  if (threadIdx.x == 0) {
    __threadfence();
    const int prev = atomicAdd(&p.scratch[1], 1);
    *last_flag = (prev == static_cast<int>(gridDim.x) - 1);
  }
  __syncthreads();
  if (*last_flag) {
    __threadfence();
    if ((p.flags & TS_FLAG_KEEP_SEMS) == 0) {
      for (int d = 0; d < p.n_deps; ++d)
        for (int i = threadIdx.x; i < p.dep[d].sem_n; i += kThreads) p.dep[d].sem[i] = 0;
    }
    if (threadIdx.x == 0) {
      p.scratch[0] = 0;
      p.scratch[1] = 0;
    }
    __threadfence();
  }
}

}  // namespace ts
