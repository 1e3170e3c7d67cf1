// TMA streaming micro-benchmark: per-SM and chip bandwidth of 2-D tiled loads of a
// [rows, K] fp16 weight matrix (box {64, 128}, 128-B swizzle), as the chain kernel's
// producer issues them, for (a) row-major weights (128 rows of 128 B, 24 KB apart) and
// (b) pre-tiled weights where each box is one contiguous 16 KB block.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../include
//      -I../paper_2305_13450_b200/csrc tma_bw.cu -o tma_bw -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#include "ts_ptx.cuh"

using namespace ts::ptx;

template <int S>
__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ CUtensorMap m,
                                                         int tiles, int kblocks, int tiled,
                                                         int rows_blocks, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * 16384);
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint64_t pol = policy_evict_first();
  unsigned long long acc = 0;
  int issued = 0, done = 0;
  // tiles assigned round-robin to CTAs; each tile = 128 rows x kblocks
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    for (int kb = 0; kb < kblocks; ++kb) {
      if (issued - done == S) {  // ring full: consume the oldest stage
        int rs = done % S;
        mbar_wait(&full[rs], (done / S) & 1);
        acc += smem[rs * 16384 + (done & 1023)];
        ++done;
      }
      int rs = issued % S;
      mbar_arrive_expect_tx(&full[rs], 16384);
      if (tiled) {
        // 3-D map: {64, 128, blocks}; block index = t * kblocks + kb
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem + rs * 16384)),
            "l"(reinterpret_cast<uint64_t>(&m)), "r"(smem_u32(&full[rs])), "r"(0), "r"(0),
            "r"(t * kblocks + kb), "l"(pol)
            : "memory");
      } else {
        tma_load_2d(smem + rs * 16384, &m, &full[rs], ((t / rows_blocks) * kblocks + kb) * 64,
                    (t % rows_blocks) * 128, pol);
      }
      ++issued;
    }
  }
  while (done < issued) {
    int rs = done % S;
    mbar_wait(&full[rs], (done / S) & 1);
    acc += smem[rs * 16384 + (done & 1023)];
    ++done;
  }
  if (acc == 0xffffffffull) *sink = acc;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

int main() {
  const int rows = 6144, K = 12288;
  const size_t bytes = size_t(rows) * K * 2;
  void* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  CUtensorMap m2, m3;
  {
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t str[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    enc(&m2, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t nblocks = (cuuint64_t)(rows / 128) * (K / 64);
    cuuint64_t dims[3] = {64, 128, nblocks};
    cuuint64_t str[2] = {128, 16384};
    cuuint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
    enc(&m3, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  int tiles = rows / 128;  // 48 tiles of 128 rows
  int kblocks = K / 64;
  auto run = [&](auto kern, int S, int grid, int split, int tiled) {
    size_t smem = S * 16384 + 1024 + 256;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // split K into `split` units per tile -> tiles*split work units over `grid` CTAs
    int units = tiles * split, kb = kblocks / split;
    for (int w = 0; w < 3; ++w) kern<<<grid, 128, smem>>>(tiled ? m3 : m2, units, kb, tiled, tiles, sink);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int it = 10;
    for (int i = 0; i < it; ++i) kern<<<grid, 128, smem>>>(tiled ? m3 : m2, units, kb, tiled, tiles, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double us = ms * 1e3 / it;
    printf("S=%2d grid=%3d units=%3d tiled=%d: %7.1f us  %6.2f TB/s  per-CTA %5.1f GB/s\n", S, grid,
           units, tiled, us, bytes / us / 1e6, bytes / us / 1e3 / (grid < units ? grid : units));
    fflush(stdout);
  };
  // Note: with split>1 and the tiled map the unit -> block mapping below is only right
  // for split == 1; bytes moved are identical either way.
  for (int tiled = 0; tiled < 2; ++tiled) {
    for (int grid : {48, 96, 144, 148}) {
      int split = grid >= 144 ? 3 : grid / 48;
      run(stream_kernel<4>, 4, grid, split, tiled);
      run(stream_kernel<8>, 8, grid, split, tiled);
      run(stream_kernel<12>, 12, grid, split, tiled);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
