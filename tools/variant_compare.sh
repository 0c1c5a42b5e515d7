#!/usr/bin/env bash
# tools/variant_compare.sh <model> <scene> <workloads...> -- <variants...>: float32 error, f32 parity tests and throughput per libkpx variant
model=$1; scene=$2; shift 2; wl=()
while [ "$1" != "--" ]; do wl+=("$1"); shift; done; shift
P=$PWD/paper_2409_06807_b200
for v in "$@"; do
  lib=$P/libkpx_$v.so; [ $v = default ] && lib=$P/libkpx.so
  echo "=== $v"
  KPX_LIB_PATH=$lib python tools/f32_err.py $scene 8 $model 2>&1 | tail -3
  KPX_LIB_PATH=$lib python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "f32" 2>&1 | tail -1
  KPX_LIB_PATH=$lib bash tools/qbench.sh "${wl[@]}"
done
