#!/bin/bash
# sweep MERF_TUNE="shade_min,trav_steps" of the march kernel on the bench workload (GPU box)
for t in "$@"; do
  v=$(MERF_TUNE=$t python bench.py --steps 6 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e6,1), round(d['roofline']['avg_launch_ms'],3))")
  echo "tune=$t Mrays/s,march_ms= $v"
done
