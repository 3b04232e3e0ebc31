#!/bin/bash
# Copy the evidence of tools/gpu_profile_round.sh from gpurun_out/ into profiles/ (round tag $1).
set -eu
R=${1:-r01}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
cp gpurun_out/bench.json profiles/${R}_bench.json
cp gpurun_out/launches.csv profiles/${R}_launches.csv
python tools/launch_summary.py gpurun_out/launches.csv "$CMD" > profiles/${R}_launches_summary.txt
cp gpurun_out/march_full.ncu-rep profiles/${R}_march_full.ncu-rep
FULL="ncu --set full --clock-control none --import-source on -k regex:\"march_kernel|shade_mma|setup_kernel\" -s 3 -c 3 python tools/prof_render.py --views 16"
for k in march setup shade_mma; do
  {
    echo "# ${R}: ncu --set full of the $k kernel, one launch = 16 orbit views at 1920x1080"
    echo "# command: $FULL"
    python tools/ncu_summary.py gpurun_out/march_full.ncu-rep "$k"
    echo
    echo "# per source line (tools/ncu_lines.py)"
    python tools/ncu_lines.py gpurun_out/march_full.ncu-rep 60 "$k"
  } > profiles/${R}_${k}_full.txt
done
python tools/traffic_from_ncu.py gpurun_out/march_full.ncu-rep
