// f64 instantiations: bit-parity build, compiled with -fmad=false (reference builds with -ffp-contract=off, pkg/setup.py:21)
#define KPX_REAL double
#define KPX_SUFFIX f64
#include "kpx_inst.inl"
