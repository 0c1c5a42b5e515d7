#!/usr/bin/env bash
# compare libkpx build variants: batch throughput (plans/s) and solo latency, di6/forest and quad12/narrow
for v in "$@"; do
  lib="paper_2409_06807_b200/libkpx_${v}.so"; [ "$v" = "default" ] && lib="paper_2409_06807_b200/libkpx.so"
  echo "=== variant $v"
  KPX_LIB_PATH=$PWD/$lib timeout -s KILL 300 python bench.py --steps 2 --no-cpu-baseline --latency-seeds 20 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(' di6_forest plans/s %.0f  ms/step %.1f  median_ms %.3f dev %.3f frac %.3f'%(d['value'],d['ms_per_step'],d['median_time_to_solution_ms'],d['time_to_solution']['median_device_ms'],d['roofline']['frac']))
    elif 'rror' in l: print(l.strip())"
  KPX_LIB_PATH=$PWD/$lib timeout -s KILL 300 python bench.py --steps 2 --no-cpu-baseline --latency-seeds 10 --workload quad12_narrow 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(' quad12_narrow plans/s %.0f  ms/step %.1f  median_ms %.3f dev %.3f frac %.3f succ %.2f'%(d['value'],d['ms_per_step'],d['median_time_to_solution_ms'],d['time_to_solution']['median_device_ms'],d['roofline']['frac'],d['success_rate']))
    elif 'rror' in l: print(l.strip())"
done
