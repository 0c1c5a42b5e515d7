#!/usr/bin/env bash
# quick throughput lines for a list of workloads (no CPU baseline / latency / seam / configs): tools/qbench.sh di6_forest quad12_narrow ...
for w in "$@"; do
  timeout -s KILL 600 python bench.py --workload $w --steps 3 --no-cpu-baseline --no-latency --no-kernel-seam --no-configs ${QB_ARGS} 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$w plans/s %.0f e2e %.0f ms/step %.1f frac %.3f solved %d/%d'%(d['value'],d['e2e']['value'],d['ms_per_step'],d['roofline']['frac'],d['batch']['solved'],d['batch']['queries']))
    elif 'rror' in l: print(l.strip())"
done
