#!/bin/bash
# ncu --set full of the config-2 v6 sweep (current build), raw + source exports
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep6 -c 1 -o /tmp/ev_c2 -f python tools/run_one.py --config 2 --sweeps 12 --burn 2 > gpurun_out/ev_c2.log 2>&1
ncu -i /tmp/ev_c2.ncu-rep --page raw --csv > gpurun_out/ev_c2_raw.csv 2>/dev/null
ncu -i /tmp/ev_c2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ev_c2_src.csv 2>/dev/null
