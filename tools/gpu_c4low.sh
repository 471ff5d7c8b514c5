#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 ncu --set full --clock-control none -k regex:"sweep3" -c 1 -o /tmp/c4low -f python tools/run_one.py --config 4 --chains 1024 --sweeps 3 --burn 1 > gpurun_out/c4low.log 2>&1
ncu -i /tmp/c4low.ncu-rep --page raw --csv > gpurun_out/c4low_raw.csv 2>/dev/null
ncu -i /tmp/c4low.ncu-rep --page details --csv > gpurun_out/c4low_details.csv 2>/dev/null
: > gpurun_out/c4low_time.log
for th in 1024 768 512; do
MCINV_THREADS=$th timeout 300 python tools/run_one.py --config 4 --chains 1024 --sweeps 12 --burn 2 --repeat 2 >> gpurun_out/c4low_time.log 2>&1
done
MCINV_C=4 timeout 300 python tools/run_one.py --config 4 --chains 1024 --sweeps 12 --burn 2 --repeat 2 >> gpurun_out/c4low_time.log 2>&1
MCINV_K=1 timeout 300 python tools/run_one.py --config 4 --chains 1024 --sweeps 12 --burn 2 --repeat 2 >> gpurun_out/c4low_time.log 2>&1
