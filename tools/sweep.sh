#!/bin/bash
# Quick timing sweep: tools/sweep.sh TAG "ENV1" "ENV2" ... (each ENV a space-separated VAR=val list)
TAG=$1; shift
mkdir -p gpurun_out
for e in "$@"; do
  echo "== $e" >> gpurun_out/sweep_$TAG.log
  env $e timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('ms_per_step', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4), 'units_ms', round(d['roofline']['kernel_ms'],3), 'tmpl_ms', round(d['roofline']['templates_ms'],3))
    else: print(l.rstrip()[:300])
" >> gpurun_out/sweep_$TAG.log
done
echo done
