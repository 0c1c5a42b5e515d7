// f32 instantiations drawing from Philox4x32-10, LATENCY build of the plan kernels
#define KPX_REAL float
#define KPX_SUFFIX f32latp
#define KPX_INST_RNG 1
#define KPX_VARIANT KPX_LATENCY
#define KPX_PLAN_ONLY 1
#include "kpx_inst.inl"
