// ts_launch.h — host-side launch entry points of the chain kernel instantiations.
// Each (tile width, CTA group, dtype, layout, cluster) combination is compiled in its own
// translation unit (ts_inst_*.cu) so the kernels build in parallel; ts_abi.cu only sees
// these declarations.
#pragma once
#include <cuda_runtime.h>

#include "ts_chain_kernel.cuh"

namespace ts_host {

// Record a thread-local error message (ts_last_error) and return `code`.
int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int cuda_fail(cudaError_t e, const char* what);

template <int BN, int CG, typename T, bool SW, bool QD>
int prepare(int* max_clusters);

template <int BN, int CG, typename T, bool SW, bool QD>
int launch_one(const ts::ChainParams& p, int units, cudaStream_t stream);

}  // namespace ts_host

// Explicit instantiation of one kernel configuration's launch entry points.
#define TS_INSTANTIATE(BN, CG, T, SW, QD)                                              \
  template int ts_host::prepare<BN, CG, T, SW, QD>(int*);                              \
  template int ts_host::launch_one<BN, CG, T, SW, QD>(const ts::ChainParams&, int,      \
                                                      cudaStream_t);
