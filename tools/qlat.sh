#!/usr/bin/env bash
# quick single-query latency (median device / wall ms over 30 seeds) for a list of workloads
for w in "$@"; do
  timeout -s KILL 600 python bench.py --workload $w --steps 1 --queries 64 --no-cpu-baseline --no-kernel-seam --no-configs --latency-seeds 30 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        t=json.loads(l)['time_to_solution']; print('$w solo device %.3f ms wall %.3f ms solved %d/%d'%(t['median_device_ms'],t['median_wall_ms'],t['solved'],t['seeds']))
    elif 'rror' in l: print(l.strip())"
done
