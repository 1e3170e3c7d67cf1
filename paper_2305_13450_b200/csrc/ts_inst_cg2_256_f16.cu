// Kernel instantiations (see ts_launch.h).
#include "ts_launch_impl.cuh"

TS_INSTANTIATE(256, 2, __half, false, false)
