#!/usr/bin/env bash
# quick A/B of libkpx build variants: di6/forest batch throughput + solo latency (20 seeds), no CPU baseline
for v in "$@"; do
  lib="paper_2409_06807_b200/libkpx_${v}.so"; [ "$v" = "default" ] && lib="paper_2409_06807_b200/libkpx.so"
  KPX_LIB_PATH=$PWD/$lib timeout -s KILL 300 python bench.py --steps 2 --no-cpu-baseline --latency-seeds 20 ${QUICK_ARGS} 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('%-10s plans/s %.0f  ms/step %.1f  median_ms %.3f dev %.3f frac %.3f succ %.2f'%('$v',d['value'],d['ms_per_step'],d['median_time_to_solution_ms'],d['time_to_solution']['median_device_ms'],d['roofline']['frac'],d['success_rate']))
    elif 'rror' in l: print(l.strip())"
done
