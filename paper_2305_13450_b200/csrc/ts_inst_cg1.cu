// Kernel instantiations (see ts_launch.h).
#include "ts_launch_impl.cuh"

TS_INSTANTIATE(64, 1, __half, false, false)
TS_INSTANTIATE(64, 1, __nv_bfloat16, false, false)
TS_INSTANTIATE(128, 1, __half, false, false)
TS_INSTANTIATE(128, 1, __nv_bfloat16, false, false)
