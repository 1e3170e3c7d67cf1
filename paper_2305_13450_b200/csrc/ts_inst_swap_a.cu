// Kernel instantiations (see ts_launch.h).
#include "ts_launch_impl.cuh"

TS_INSTANTIATE(32, 1, __half, true, false)
TS_INSTANTIATE(32, 1, __nv_bfloat16, true, false)
TS_INSTANTIATE(64, 1, __half, true, false)
TS_INSTANTIATE(64, 1, __nv_bfloat16, true, false)
