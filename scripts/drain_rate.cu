// drain_rate.cu — epilogue drain microbenchmark: one CTA per SM (all 148 busy, as in the
// chain kernel) drains a 128-lane x 512-column fp32 TMEM accumulator (the per-CTA half of a
// 256 x 512 CTA-pair tile) through GeLU to fp16 rows of a row-major output, with the chain
// kernel's thread layout (128 + 256 threads, 8 epilogue warps: 4 TMEM lane quarters x 2
// column groups, 168-register cap). Variants:
//   0  x16 TMEM load, wait, GeLU, 256-bit row-per-lane global store   (the kernel today)
//   1  x32 load, wait, 2 x 16 columns
//   2  x16 loads software-pipelined two deep (next load issued before this one is used)
//   3  4 x16 loads, one wait, 64 columns
//   4  x32 loads -> GeLU -> 128B-swizzled shared-memory staging (4 KB / warp, double
//      buffered) -> TMA tensor store of a 32-row x 64-column box (cp.async.bulk.tensor)
//   5  variant 0 without GeLU (conversion only)      6  variant 0 without the stores
//   7  variant 4 with x16 loads pipelined two deep
// Prints cycles per drain (max over the CTA's warps, mean over CTAs) and the kernel time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2305_13450_b200/csrc
//        -I../include drain_rate.cu -o drain_rate -lcuda && ./drain_rate
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>

#include "ts_ptx.cuh"

using namespace ts::ptx;

__device__ __forceinline__ void gelu2(float& a, float& b) {
  const float ua = a * fmaf(0.0356774081f, a * a, 0.7978845608f);
  const float ub = b * fmaf(0.0356774081f, b * b, 0.7978845608f);
  uint32_t h;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(ub), "f"(ua));
  asm("tanh.approx.f16x2 %0, %0;" : "+r"(h));
  const __half2 t = *reinterpret_cast<const __half2*>(&h);
  const float ha = 0.5f * a, hb = 0.5f * b;
  a = fmaf(ha, __low2float(t), ha);
  b = fmaf(hb, __high2float(t), hb);
}

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <bool kGelu>
__device__ __forceinline__ void act16(const uint32_t* r, uint32_t* pk) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    float v0 = __uint_as_float(r[2 * q]), v1 = __uint_as_float(r[2 * q + 1]);
    if (kGelu) gelu2(v0, v1);
    pk[q] = pack_h2(v0, v1);
  }
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* m, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

__global__ void __launch_bounds__(384, 1) drain_kernel(const __grid_constant__ CUtensorMap cmap,
                                                        __half* c, int ldc, int variant, int reps,
                                                        long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ unsigned long long tmax;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) tmax = 0;
  if (warp == 0) tmem_alloc<512, 1>(&tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp >= 4) {
    const int ew = warp & 3, eg = (warp - 4) >> 2;
    const int row = blockIdx.x * 128 + ew * 32 + lane;
    __half* crow = c + static_cast<size_t>(row) * ldc;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(ew * 32) << 16);
    uint8_t* stg = smem + (warp - 4) * 8192;  // 2 x 4 KB per warp
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
      const int lo = eg * 256, hi = lo + 256;
      if (variant == 0 || variant == 5 || variant == 6) {
#pragma unroll 1
        for (int x = lo; x < hi; x += 16) {
          uint32_t r[16], pk[8];
          tmem_ld_32x32b_x16(lane_base + x, r);
          tmem_ld_wait();
          if (variant == 5) act16<false>(r, pk); else act16<true>(r, pk);
          if (variant != 6) st_global_v8(crow + x, pk);
          else if (pk[0] == 0x12345678u) crow[x] = __half();  // keep the math
        }
      } else if (variant == 1) {
#pragma unroll 1
        for (int x = lo; x < hi; x += 32) {
          uint32_t r[32], pk[16];
          tmem_ld_32x32b_x32(lane_base + x, r);
          tmem_ld_wait();
          act16<true>(r, pk);
          act16<true>(r + 16, pk + 8);
          st_global_v8(crow + x, pk);
          st_global_v8(crow + x + 16, pk + 8);
        }
      } else if (variant == 2) {
        uint32_t ra[16], rb[16];
        tmem_ld_32x32b_x16(lane_base + lo, ra);
#pragma unroll 1
        for (int x = lo; x < hi; x += 32) {
          uint32_t pk[8];
          tmem_ld_wait();
          tmem_ld_32x32b_x16(lane_base + x + 16, rb);
          act16<true>(ra, pk);
          st_global_v8(crow + x, pk);
          tmem_ld_wait();
          if (x + 32 < hi) tmem_ld_32x32b_x16(lane_base + x + 32, ra);
          act16<true>(rb, pk);
          st_global_v8(crow + x + 16, pk);
        }
      } else if (variant == 3) {
#pragma unroll 1
        for (int x = lo; x < hi; x += 64) {
          uint32_t r0[16], r1[16], r2[16], r3[16], pk[8];
          tmem_ld_32x32b_x16(lane_base + x, r0);
          tmem_ld_32x32b_x16(lane_base + x + 16, r1);
          tmem_ld_32x32b_x16(lane_base + x + 32, r2);
          tmem_ld_32x32b_x16(lane_base + x + 48, r3);
          tmem_ld_wait();
          act16<true>(r0, pk);
          st_global_v8(crow + x, pk);
          act16<true>(r1, pk);
          st_global_v8(crow + x + 16, pk);
          act16<true>(r2, pk);
          st_global_v8(crow + x + 32, pk);
          act16<true>(r3, pk);
          st_global_v8(crow + x + 48, pk);
        }
      } else {
        // 64-column chunks through 128B-swizzled staging, TMA store of 32 rows x 64 cols
        int buf = 0;
        uint32_t ra[16], rb[16];
        if (variant == 7) tmem_ld_32x32b_x16(lane_base + lo, ra);
#pragma unroll 1
        for (int x = lo; x < hi; x += 64, buf ^= 1) {
          uint8_t* sb = stg + buf * 4096;
          // the store issued from this buffer two chunks ago must have read it
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            uint32_t pk[8];
            if (variant == 7) {
              tmem_ld_wait();
              if (h & 1) {
                if (h < 3 || x + 64 < hi) tmem_ld_32x32b_x16(lane_base + x + 16 * h + 16, ra);
                act16<true>(rb, pk);
              } else {
                tmem_ld_32x32b_x16(lane_base + x + 16 * h + 16, rb);
                act16<true>(ra, pk);
              }
            } else {
              uint32_t r[16];
              tmem_ld_32x32b_x16(lane_base + x + 16 * h, r);
              tmem_ld_wait();
              act16<true>(r, pk);
            }
            // row `lane` of the box: 128 B = 8 granules of 16 B; granule g at g ^ (lane & 7)
#pragma unroll
            for (int g2 = 0; g2 < 2; ++g2) {
              const int g = 2 * h + g2;
              *reinterpret_cast<uint4*>(sb + lane * 128 + ((g ^ (lane & 7)) << 4)) =
                  make_uint4(pk[4 * g2], pk[4 * g2 + 1], pk[4 * g2 + 2], pk[4 * g2 + 3]);
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&cmap, sb, x, blockIdx.x * 128 + ew * 32);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
      }
    }
    long long t = clock64() - t0;
    atomicMax(&tmax, static_cast<unsigned long long>(t));
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = static_cast<long long>(tmax);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512, 1>(tmem);
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int ldc = 6144, rows = sms * 128;
  __half* c;
  cudaMalloc(&c, size_t(rows) * ldc * 2);
  long long* cyc;
  cudaMalloc(&cyc, sms * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap cmap;
  cuuint64_t dims[2] = {(cuuint64_t)ldc, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)ldc * 2};
  cuuint32_t box[2] = {64, 32}, es[2] = {1, 1};
  CUresult er = ((EncodeFn)fn)(&cmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, c, dims, str, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (er != CUDA_SUCCESS) printf("encode failed %d\n", (int)er);
  const int smem = 8 * 8192 + 2048;
  cudaFuncSetAttribute(drain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const char* names[] = {"x16 wait store (today)", "x32 wait", "x16 pipelined x2", "4 x16 one wait",
                         "x16 smem+TMA store", "today, no GeLU", "today, no stores",
                         "x16 pipelined smem+TMA store"};
  const int reps = 20;
  for (int v = 0; v < 8; ++v) {
    for (int w = 0; w < 2; ++w) drain_kernel<<<sms, 384, smem>>>(cmap, c, ldc, v, reps, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    drain_kernel<<<sms, 384, smem>>>(cmap, c, ldc, v, reps, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[256];
    cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < sms; ++i) mean += h[i];
    mean /= sms;
    cudaError_t e = cudaGetLastError();
    printf("variant %d %-30s %8.0f cyc/drain  %7.2f us/drain (kernel)  %s\n", v, names[v], mean / reps,
           ms * 1e3 / reps, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
