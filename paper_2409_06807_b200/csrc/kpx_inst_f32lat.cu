// f32 instantiations, LATENCY build of the plan kernels (one query on the whole GPU): a translation unit of
// its own so that it compiles beside the throughput build
#define KPX_REAL float
#define KPX_SUFFIX f32lat
#define KPX_VARIANT KPX_LATENCY
#define KPX_PLAN_ONLY 1
#include "kpx_inst.inl"
