// f64 instantiations drawing from Philox4x32-10 (built with -fmad=false like the parity unit)
#define KPX_REAL double
#define KPX_SUFFIX f64p
#define KPX_INST_RNG 1
#include "kpx_inst.inl"
