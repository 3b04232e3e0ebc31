#!/bin/bash
# Re-measure every ablation / NEXT-row number quoted in DESIGN.md with the current kernels
# (one GPU pass; outputs under gpurun_out/abl_*).
set -u
mkdir -p gpurun_out
python tools/sweep_c5.py --out gpurun_out/abl_c5_sweep.jsonl > gpurun_out/abl_c5.log 2>&1
python bench.py --steps 5 --no-cpu-baseline --no-e2e --dense > gpurun_out/abl_dense.json 2>/dev/null
MERF_NO_SKIPTAB=1 python bench.py --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/abl_noskiptab.json 2>/dev/null
python bench.py --steps 10 --no-cpu-baseline --no-e2e --mlp-ffma > gpurun_out/abl_mlpffma.json 2>/dev/null
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --spherical > gpurun_out/abl_spherical.json 2>/dev/null
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --spherical --sph-persistent > gpurun_out/abl_spherical_persistent.json 2>/dev/null
python tools/bench_progressive.py --out gpurun_out/abl_progressive.jsonl > gpurun_out/abl_progressive.log 2>&1
python tools/bench_qat.py --out gpurun_out/abl_qat.jsonl > gpurun_out/abl_qat.log 2>&1
python tools/bench_bake.py > gpurun_out/abl_bake.log 2>&1
for f in gpurun_out/abl_*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']/1e6,1), 'M rays/s', d['config']['workload'], 'samples/ray', round(d['mean_evaluated_samples_per_ray'],1))"; done
tail -n 4 gpurun_out/abl_c5.log gpurun_out/abl_progressive.log gpurun_out/abl_qat.log gpurun_out/abl_bake.log
