// f32 instantiations: throughput build, FMA contraction on
#define KPX_REAL float
#define KPX_SUFFIX f32
#include "kpx_inst.inl"
