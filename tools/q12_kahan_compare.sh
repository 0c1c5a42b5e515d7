P=$PWD/paper_2409_06807_b200
for v in default q12k2 q12nk; do
  lib=$P/libkpx_$v.so; [ $v = default ] && lib=$P/libkpx.so
  echo "=== $v"
  KPX_LIB_PATH=$lib python tools/q12_err.py narrow 2>&1 | tail -3
  KPX_LIB_PATH=$lib python tools/q12_err.py forest 2>&1 | tail -2
  KPX_LIB_PATH=$lib python tools/succ1000.py 2>&1 | grep "cuda-f32 "
  KPX_LIB_PATH=$lib bash tools/qbench.sh quad12_narrow quad12_config5
done
