#!/bin/bash
# evidence: ncu --set full of the config-2 v6 sweep (product build), launch list of the bench,
# and the bench line
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py --steps ${BSTEPS:-20} --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep6 -c 1 -o gpurun_out/ev_c2e -f python tools/run_one.py --config 2 --sweeps 12 --burn 2 > gpurun_out/ev_c2e.log 2>&1
ncu -i gpurun_out/ev_c2e.ncu-rep --page raw --csv > gpurun_out/ev_c2e_raw.csv 2>/dev/null
ncu -i gpurun_out/ev_c2e.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ev_c2e_src.csv 2>/dev/null
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2c.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_bench.log 2>&1; echo "ncu bench rc=$?" >> gpurun_out/ncu_bench.log
