// mma_rate.cu — tcgen05.mma issue-rate microbenchmark (no operand loads): cycles per
// kind::f16 MMA for M = 128 (cta_group::1) / 256 (cta_group::2) and N = 64..256, with one
// or two accumulators alternating, operands resident in shared memory (zeros).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2305_13450_b200/csrc
//        -I../include mma_rate.cu -o mma_rate && ./mma_rate
#include <cstdio>

#include "ts_ptx.cuh"

using namespace ts::ptx;

template <int CG>
__global__ void __launch_bounds__(128, 1) rate_kernel(int n, int iters, int two_acc, int a_twice,
                                                      long long* out, int commit_every) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint64_t cbar[16];
  __shared__ uint32_t tslot;
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 196608 / 16; i += blockDim.x) reinterpret_cast<uint4*>(s)[i] = make_uint4(0, 0, 0, 0);
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 16; ++i) mbar_init(&cbar[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_alloc<512, CG>(&tslot);
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (rank == 0 && threadIdx.x == 0) {
    const uint32_t idesc = idesc_f16(128 * CG, n, 0);
    const uint64_t ad = smem_desc_k_sw128(smem_u32(s));
    const uint64_t bd = smem_desc_k_sw128(smem_u32(s + 65536));
    const uint64_t bd2 = smem_desc_k_sw128(smem_u32(s + 131072));
    const uint64_t ad2 = a_twice ? ad : smem_desc_k_sw128(smem_u32(s + 16384));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (two_acc == 2) {
        // interleaved: consecutive MMAs target different accumulators
        umma_f16_kblock2<CG>(tmem, tmem + 256, ad, bd, bd2, idesc, 1);
      } else {
        umma_f16_kblock<CG>(tmem, ad, bd, idesc, 1);
        if (two_acc) umma_f16_kblock<CG>(tmem + 256, ad2, bd2, idesc, 1);
      }
      if (commit_every && i % commit_every == 0) {
        if constexpr (CG == 2) umma_commit_pair(&cbar[i & 15]); else umma_commit(&cbar[i & 15]);
      }
    }
    if constexpr (CG == 2) umma_commit_pair(&bar); else umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[0] = t1 - t0;
  }
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512, CG>(tmem);
  }
}

template <int CG>
void run(int n, int two_acc, int a_twice, int commit_every = 0) {
  long long* d;
  cudaMalloc(&d, 8);
  const int iters = 2000;
  auto k = rate_kernel<CG>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CG, 1, 1);
  cfg.blockDim = dim3(128, 1, 1);
  cfg.dynamicSmemBytes = 200000;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, n, iters, two_acc, a_twice, d, commit_every);
  cudaLaunchKernelEx(&cfg, k, n, iters, two_acc, a_twice, d, commit_every);
  long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  const int mmas = iters * 4 * (two_acc ? 2 : 1);
  const double floor = 128.0 * CG * n / (256.0 * CG);  // cycles per MMA (guide: max(M,128) N / (256 cg))
  printf("cg%d M=%d N=%3d two_acc=%d a_twice=%d commit/%d: %7.1f cyc/MMA (floor %5.1f) %s\n", CG, 128 * CG,
         n, two_acc, a_twice, commit_every, double(c) / mmas, CG == 2 ? 256.0 * n / 512 : 128.0 * n / 256,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  (void)floor;
  cudaFree(d);
}

int main() {
  for (int n : {64, 128, 192, 256}) run<1>(n, 0, 0);
  for (int n : {128, 192, 256}) run<1>(n, 1, 1);
  for (int n : {128, 192, 256}) run<1>(n, 2, 1);
  for (int n : {64, 128, 192, 256}) run<2>(n, 0, 0);
  for (int n : {128, 192, 256}) run<2>(n, 1, 1);
  for (int n : {64, 128, 192, 256}) run<2>(n, 2, 1);
  for (int n : {128, 192, 256}) run<2>(n, 2, 0);
  for (int n : {192, 256}) run<2>(n, 1, 1, 1);
  for (int n : {192, 256}) run<2>(n, 2, 1, 1);
  for (int n : {192, 256}) run<2>(n, 0, 1, 1);
  for (int n : {192, 256}) run<2>(n, 0, 1, 2);
  return 0;
}
