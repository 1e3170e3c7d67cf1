// Kernel instantiations (see ts_launch.h).
#include "ts_launch_impl.cuh"

TS_INSTANTIATE(128, 2, __half, false, false)
TS_INSTANTIATE(128, 2, __nv_bfloat16, false, false)
