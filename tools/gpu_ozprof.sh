#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
MCINV_CONTRACT_OZAKI=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/oz_launches.csv python tools/run_one.py --config 3 --sweeps 34 --burn 2 --outputs full > gpurun_out/oz_launch.log 2>&1
MCINV_CONTRACT_OZAKI=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ozaki_gemm" -c 1 -o /tmp/ozg -f python tools/run_one.py --config 3 --sweeps 34 --burn 2 --outputs full > gpurun_out/ozg.log 2>&1
ncu -i /tmp/ozg.ncu-rep --page raw --csv > gpurun_out/ozg_raw.csv 2>/dev/null
ncu -i /tmp/ozg.ncu-rep --page details --csv > gpurun_out/ozg_details.csv 2>/dev/null
ncu -i /tmp/ozg.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ozg_src.csv 2>/dev/null
