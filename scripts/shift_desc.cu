// shift_desc.cu — does a K-major 128B-swizzled UMMA operand descriptor whose start address
// is an arbitrary multiple of 128 B (a row offset inside the 8-row swizzle atom) read rows
// start + m with the absolute-address swizzle TMA writes? (A shifted views of one staged
// conv window.) A = 136 rows x 16 fp16 (row r, col k = r + k/16), B = 16 x 16 identity;
// D = A[shift .. shift + 128) read back from TMEM.
#include <cstdio>
#include <cuda_fp16.h>

#include "ts_ptx.cuh"

using namespace ts::ptx;

__global__ void __launch_bounds__(128, 1) shift_kernel(float* out, int shift, int base_off) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  __half* A = reinterpret_cast<__half*>(s);          // 144 rows x 64 fp16 (128 B rows), SW128
  __half* B = reinterpret_cast<__half*>(s + 32768);  // 16 rows x 64, SW128
  for (int i = threadIdx.x; i < 144 * 64; i += blockDim.x) {
    const int r = i >> 6, k = i & 63;
    const int off = r * 128 + (((k >> 3) ^ (r & 7)) << 4) + ((k & 7) << 1);
    A[off >> 1] = __float2half(k < 16 ? float(r) + 0.001f * k : 0.f);
  }
  for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) {
    const int n = i >> 6, k = i & 63;
    const int off = n * 128 + (((k >> 3) ^ (n & 7)) << 4) + ((k & 7) << 1);
    B[off >> 1] = __float2half(k == n ? 1.f : 0.f);
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
    uint64_t ad = smem_desc_k_sw128(smem_u32(s) + shift * 128);
    ad |= static_cast<uint64_t>(base_off ? ((shift & 7)) : 0) << 49;
    const uint64_t bd = smem_desc_k_sw128(smem_u32(B));
    // one K16 MMA (only K 0..15 of A / B are nonzero)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(ad), "l"(bd), "r"(idesc_f16(128, 16, 0))
        : "memory");
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[16];
  tmem_ld_32x32b_x16(tmem + (static_cast<uint32_t>(threadIdx.x & 96) << 16), r);
  tmem_ld_wait();
  for (int k = 0; k < 16; ++k) out[threadIdx.x * 16 + k] = __uint_as_float(r[k]);
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512, 1>(tmem);
  }
}


__global__ void __launch_bounds__(128, 1) shift_rate(long long* out, int shift, int n, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(s)[i] = make_uint4(0, 0, 0, 0);
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
    const uint32_t id = idesc_f16(128, n, 0);
    const uint64_t bd = smem_desc_k_sw128(smem_u32(s + 49152));
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int sh = shift < 0 ? (i % 9) * 1 + (i % 3) * 58 : shift;  // conv-like tap shifts
      const uint64_t ad = smem_desc_k_sw128(smem_u32(s) + sh * 128);
      umma_f16_kblock<1>(tmem, ad, bd, id, 1);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    out[0] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512, 1>(tmem);
  }
}

int main() {
  float* d;
  cudaMalloc(&d, 128 * 16 * 4);
  cudaFuncSetAttribute(shift_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 50000);
  for (int base_off = 0; base_off < 2; ++base_off)
    for (int shift : {0, 1, 3, 7, 8, 13}) {
      shift_kernel<<<1, 128, 50000>>>(d, shift, base_off);
      cudaError_t e = cudaDeviceSynchronize();
      float h[128 * 16];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int k = 0; k < 16; ++k) {
          const float want = float(m + shift) + 0.001f * k;
          if (fabsf(h[m * 16 + k] - want) > 0.05f + 0.002f * want) ++bad;
        }
      printf("base_off field %d shift %2d: %s, %4d bad of 2048; D[0][0..2] = %g %g, D[5][0] = %g\n",
             base_off, shift, cudaGetErrorString(e), bad, h[0], h[1], h[5 * 16]);
    }
  long long* c;
  cudaMalloc(&c, 8);
  cudaFuncSetAttribute(shift_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int n : {64, 128})
    for (int shift : {0, 1, 3, 8, -1}) {
      shift_rate<<<1, 128, 70000>>>(c, shift, n, 2000);
      shift_rate<<<1, 128, 70000>>>(c, shift, n, 2000);
      long long h = 0;
      cudaDeviceSynchronize();
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      printf("N=%d shift %2d: %.1f cycles per K16 MMA\n", n, shift, double(h) / (2000 * 4));
    }
  return 0;
}
