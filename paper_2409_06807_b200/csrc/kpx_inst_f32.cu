// f32 instantiations: throughput build of the plan kernels, batch kernels, host helpers; FMA contraction on
#define KPX_REAL float
#define KPX_SUFFIX f32
#define KPX_FORWARD_LATENCY f32lat
#include "kpx_inst.inl"
