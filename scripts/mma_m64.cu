// mma_m64.cu — (1) tcgen05.mma kind::f16 issue rate for M x N = 128x64 (the halo conv today),
// 64x256, 64x128, 128x128, 128x256 (cta_group::1, one accumulator, K = 16 per MMA, operands
// resident in shared memory); (2) where an M = 64 accumulator lands in TMEM: A[m][0] = m + 1,
// A[m][1] = 1, B[n][0] = 1, B[n][1] = n / 256 -> D[m][n] = m + 1 + n / 256; every TMEM lane
// of columns 0 and 5 is read back by its warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2305_13450_b200/csrc
//        -I../include mma_m64.cu -o mma_m64 && ./mma_m64
#include <cstdio>
#include <cuda_fp16.h>

#include "ts_ptx.cuh"

using namespace ts::ptx;

__device__ __forceinline__ int swz(int row, int k) {  // element offset, 16-bit, K-major SW128
  return row * 64 + ((((k >> 3) ^ (row & 7))) << 3) + (k & 7);
}

__global__ void __launch_bounds__(128, 1) kern(int m, int n, int iters, long long* cyc, float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  __half* A = reinterpret_cast<__half*>(s);            // up to 128 rows x 64 K
  __half* B = reinterpret_cast<__half*>(s + 32768);    // up to 256 rows x 64 K
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    A[swz(r, k)] = __float2half(k == 0 ? float(r + 1) : (k == 1 ? 1.f : 0.f));
  }
  for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    B[swz(r, k)] = __float2half(k == 0 ? 1.f : (k == 1 ? float(r) / 256.f : 0.f));
  }
  fence_proxy_async_shared();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_alloc<512, 1>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_f16(m, n, 0);
    const uint64_t ad = smem_desc_k_sw128(smem_u32(A));
    const uint64_t bd = smem_desc_k_sw128(smem_u32(B));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) umma_f16_kblock<1>(tmem, ad, bd, idesc, i != 0);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    cyc[0] = clock64() - t0;
  }
  __syncthreads();
  tc_fence_after();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t r[2];
  const uint32_t base = tmem + (static_cast<uint32_t>(w * 32) << 16);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(base + 0));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[1]) : "r"(base + 5));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  out[threadIdx.x * 2] = __uint_as_float(r[0]);
  out[threadIdx.x * 2 + 1] = __uint_as_float(r[1]);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512, 1>(tmem);
  }
}

int main() {
  long long* cyc;
  float* out;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&out, 256 * 4);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 120000);
  const int shapes[][2] = {{128, 64}, {64, 256}, {64, 128}, {128, 128}, {128, 256}, {64, 64}};
  for (auto& sh : shapes) {
    const int iters = 2000;
    kern<<<1, 128, 120000>>>(sh[0], sh[1], iters, cyc, out);
    cudaError_t e = cudaDeviceSynchronize();
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double per = double(c) / (iters * 4);
    printf("M=%3d N=%3d: %6.1f cycles per K=16 MMA, %6.0f MAC/clk  (%s)\n", sh[0], sh[1], per,
           sh[0] * sh[1] * 16 / per, cudaGetErrorString(e));
  }
  // layout of M = 64 (one MMA with accumulate off, then read)
  kern<<<1, 128, 120000>>>(64, 256, 1, cyc, out);
  cudaDeviceSynchronize();
  float h[256];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  printf("M=64 N=256 accumulator, TMEM lane: (col 0, col 5) [expect m+1+n/256 for its row m]\n");
  for (int l = 0; l < 128; ++l) printf("%3d:(%g,%g)%s", l, h[2 * l], h[2 * l + 1], (l % 8 == 7) ? "\n" : " ");
  return 0;
}
