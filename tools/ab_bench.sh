#!/bin/bash
# A/B timing of library variants / env toggles on one GPU (kernel-only bench legs).
#   tools/ab_bench.sh "label|ENV=.. ENV2=.." ...    (MERF_LIB=scratch/libX.so selects a variant)
# prints: label  rays/s  march_ms  setup_ms  shade_ms  frac
for spec in "$@"; do
  label="${spec%%|*}"; envs="${spec#*|}"
  [ "$label" = "$spec" ] && envs=""
  out=$(env $envs python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1)
  python - "$label" "$out" <<'PY'
import json, sys
label, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    p = d["roofline"]["pipeline_ms_per_step"]
    print(f"{label:28s} {d['value']/1e6:8.1f} M rays/s  march {p['march']:.3f}  setup {p['setup']:.3f}  "
          f"shade {p['shade']:.3f}  frac {d['roofline']['frac']:.4f}  clocks {d['clocks']['sm_mhz']}")
except Exception as e:
    print(label, "FAILED", line[:300])
PY
done
