// tf32_red.cu — checks the split-K reduction MMA D += P x I (kind::tf32, N = 32, identity
// B operand in 128-B-swizzled K-major smem) for cta_group::1 and ::2: D is zeroed by an
// f16 MMA of zero operands, P (128 rows x 32 fp32 per CTA) is written to smem in the
// swizzled layout, then D is read back from TMEM and compared with P.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2305_13450_b200/csrc
//        -I../include tf32_red.cu -o tf32_red && ./tf32_red
#include <cstdio>

#include "ts_ptx.cuh"

using namespace ts::ptx;

template <int CG>
__global__ void __launch_bounds__(128, 1) red_kernel(float* out, int ident_rows_mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0;
  float* P = reinterpret_cast<float*>(s);            // 128 x 32 fp32, SW128
  float* I = reinterpret_cast<float*>(s + 16384);    // identity rows, SW128
  uint8_t* Z = s + 32768;                            // zeros for the f16 clear (32 KB)
  for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) {
    const int m = i >> 5, k = i & 31;
    P[(m * 128 + (((k >> 2) ^ (m & 7)) << 4) + ((k & 3) << 2)) >> 2] =
        float(rank * 10000 + m * 32 + k) * 0.25f;
  }
  for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) {
    const int n = i >> 5, k = i & 31;
    const int ng = (CG == 2 && ident_rows_mode == 0 ? 16 * int(rank) : 0) + n;
    I[(n * 128 + (((k >> 2) ^ (n & 7)) << 4) + ((k & 3) << 2)) >> 2] = (k == ng) ? 1.f : 0.f;
  }
  for (int i = threadIdx.x; i < 32768 / 16; i += blockDim.x) reinterpret_cast<uint4*>(Z)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async_shared();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x < 32) tmem_alloc<512, CG>(&tslot);
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (rank == 0 && threadIdx.x == 0) {
    // D = 0 (f16 MMA, N = 32, accumulate off)
    const uint32_t id16 = idesc_f16(128 * CG, 32, 0);
    umma_f16_kblock<CG>(tmem, smem_desc_k_sw128(smem_u32(Z)), smem_desc_k_sw128(smem_u32(Z + 16384)), id16, 0);
    // D += P x I
    umma_tf32_kblock<CG>(tmem, smem_desc_k_sw128(smem_u32(P)), smem_desc_k_sw128(smem_u32(I)),
                         idesc_tf32(128 * CG, 32));
    if constexpr (CG == 2) umma_commit_pair(&bar); else umma_commit(&bar);
  }
  if constexpr (CG == 2) {
    // the leader's commit arrives on both CTAs' barriers
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[32];
  tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(threadIdx.x & 96) << 16), r);
  tmem_ld_wait();
  for (int k = 0; k < 32; ++k) out[(rank * 128 + threadIdx.x) * 32 + k] = __uint_as_float(r[k]);
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512, CG>(tmem);
  }
}

template <int CG>
void run(int mode) {
  float* d;
  cudaMalloc(&d, 256 * 32 * 4);
  cudaMemset(d, 0, 256 * 32 * 4);
  auto k = red_kernel<CG>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80000);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CG, 1, 1);
  cfg.blockDim = dim3(128, 1, 1);
  cfg.dynamicSmemBytes = 80000;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, d, mode);
  cudaError_t e = cudaDeviceSynchronize();
  float h[256 * 32];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  int bad = 0;
  double maxerr = 0;
  for (int rk = 0; rk < CG; ++rk)
    for (int m = 0; m < 128; ++m)
      for (int kk = 0; kk < 32; ++kk) {
        const float want = float(rk * 10000 + m * 32 + kk) * 0.25f;
        const float got = h[(rk * 128 + m) * 32 + kk];
        const double err = fabs(got - want) / (fabs(want) + 1);
        if (err > 1e-2) ++bad;
        if (err > maxerr) maxerr = err;
      }
  printf("cg%d mode %d: %s, %d bad of %d, max rel err %.3g; sample D[0][0..4] = %g %g %g %g, D[1][0] = %g\n",
         CG, mode, cudaGetErrorString(e), bad, CG * 128 * 32, maxerr, h[0], h[1], h[2], h[3], h[32]);
  cudaFree(d);
}

int main() {
  run<1>(0);
  run<2>(0);
  run<2>(1);
  return 0;
}
