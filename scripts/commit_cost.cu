// commit_cost.cu — cycles of tcgen05.commit (mbarrier arrive on completion of the thread's
// prior tcgen05 ops) with and without MMAs in flight, and of an empty mbarrier round trip.
#include <cstdio>
#include "ts_ptx.cuh"
using namespace ts::ptx;

__global__ void __launch_bounds__(128, 1) commit_kernel(long long* out, int iters, int with_mma) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 32768 / 16; i += blockDim.x) reinterpret_cast<uint4*>(s)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_shared();
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_alloc<512, 1>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint64_t ad = smem_desc_k_sw128(smem_u32(s)), bd = smem_desc_k_sw128(smem_u32(s + 16384));
    const uint32_t id = idesc_f16(128, 64, 0);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (with_mma) umma_f16_kblock<1>(tmem, ad, bd, id, 1);
      umma_commit(&bar[0]);
    }
    long long t1 = clock64();
    // round trips: commit then wait for its arrival
    for (int i = 0; i < iters; ++i) {
      umma_commit(&bar[1]);
      mbar_wait(&bar[1], i & 1);
    }
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t1;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512, 1>(tmem);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(commit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  for (int mma = 0; mma < 2; ++mma) {
    commit_kernel<<<1, 128, 40000>>>(d, 200, mma);
    commit_kernel<<<1, 128, 40000>>>(d, 200, mma);
    long long h[2];
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("with_mma %d: issue %.1f cycles per (MMA kblock +) commit; commit->arrive round trip %.1f cycles\n",
           mma, double(h[0]) / 200, double(h[1]) / 200);
  }
  return 0;
}
