#!/bin/bash
# One GPU pass that regenerates the evidence under gpurun_out/ (then tools/collect_profiles.sh
# copies the summaries into profiles/).  Order matters: the ncu capture is taken first and
# stamped into profiles/render_traffic.json (source digest of the built library), so that the
# bench run that follows reads a capture of the kernels it times ("capture": {"current": true}).
#   march_full.ncu-rep  ncu --set full of one setup + march + shade launch (16 views, 1080p)
#   render_traffic.json DRAM / L2 bytes and instructions per march launch from that capture
#   bench.json          python bench.py (default contract run)
#   launches.csv        ncu launch list of a short bench run (per-launch gpu__time_duration)
set -u
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"march_kernel|shade_mma|setup_kernel" -s 3 -c 3 \
    -o gpurun_out/march_full -f python tools/prof_render.py --views 16 > gpurun_out/ncu_full.log 2>&1
python tools/traffic_from_ncu.py gpurun_out/march_full.ncu-rep > gpurun_out/traffic.log 2>&1
cp profiles/render_traffic.json gpurun_out/render_traffic.json
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
cat gpurun_out/bench.json
