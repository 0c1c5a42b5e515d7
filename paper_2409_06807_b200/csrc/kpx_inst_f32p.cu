// f32 instantiations drawing from Philox4x32-10 (the "-philox" backends): throughput build + batch kernels
#define KPX_REAL float
#define KPX_SUFFIX f32p
#define KPX_INST_RNG 1
#define KPX_FORWARD_LATENCY f32latp
#include "kpx_inst.inl"
