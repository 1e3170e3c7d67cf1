// Kernel instantiations (see ts_launch.h).
#include "ts_launch_impl.cuh"

TS_INSTANTIATE(128, 1, __half, true, false)
TS_INSTANTIATE(128, 1, __nv_bfloat16, true, false)
TS_INSTANTIATE(256, 1, __half, true, false)
TS_INSTANTIATE(256, 1, __nv_bfloat16, true, false)
