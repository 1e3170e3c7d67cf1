// ts_launch_impl.cuh — definitions of the launch templates declared in ts_launch.h;
// included only by the ts_inst_*.cu translation units.
#pragma once
#include <atomic>

#include "ts_launch.h"

namespace ts_host {

// Per-device launch preparation of one kernel instantiation, done once per device: the
// dynamic shared-memory opt-in (a per-device function attribute) and the number of
// clusters the device can hold at once (a GPC whose SM count is not a multiple of the
// cluster size leaves SMs idle; 0 = unknown).
template <int BN, int CG, typename T, bool SW, bool QD>
int prepare(int* max_clusters) {
  using C = ts::Cfg<BN, CG, SW, QD>;
  constexpr int kCluster = CG * (QD ? 2 : 1);
  constexpr int kMaxDev = 64;
  static std::atomic<int> done[kMaxDev];
  static std::atomic<int> mcs[kMaxDev];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev < 0 || dev >= kMaxDev) return fail(TS_ERR_CUDA, "device ordinal %d unsupported", dev);
  if (done[dev].load(std::memory_order_acquire) == 0) {
    auto kern = ts::chain_kernel<BN, CG, T, SW, QD>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemBytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
    int mc = 0;
    if (kCluster > 1) {
      int sms = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(sms - sms % kCluster, 1, 1);
      cfg.blockDim = dim3(C::kThreads, 1, 1);
      cfg.dynamicSmemBytes = C::kSmemBytes;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = kCluster;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&mc, kern, &cfg) != cudaSuccess) {
        (void)cudaGetLastError();
        mc = 0;
      }
    }
    mcs[dev].store(mc, std::memory_order_relaxed);
    done[dev].store(1, std::memory_order_release);
  }
  *max_clusters = mcs[dev].load(std::memory_order_relaxed);
  return TS_OK;
}

// `units` = work items in flight at once: CTAs (CG=1), CTA pairs (CG=2) or two-pair
// clusters (QD), capped at the co-resident cluster count so every launched cluster runs
// from the start of the persistent kernel.
template <int BN, int CG, typename T, bool SW, bool QD>
int launch_one(const ts::ChainParams& p, int units, cudaStream_t stream) {
  using C = ts::Cfg<BN, CG, SW, QD>;
  constexpr int kCluster = CG * (QD ? 2 : 1);
  int mc = 0;
  int r = prepare<BN, CG, T, SW, QD>(&mc);
  if (r) return r;
  if (mc > 0 && units > mc) units = mc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(units * kCluster, 1, 1);
  cfg.blockDim = dim3(C::kThreads, 1, 1);
  cfg.dynamicSmemBytes = C::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, ts::chain_kernel<BN, CG, T, SW, QD>, p);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(e, "chain_kernel launch");
  return TS_OK;
}

}  // namespace ts_host
