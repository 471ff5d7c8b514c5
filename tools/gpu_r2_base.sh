#!/bin/bash
# round-2 baseline: build, quick timings, one ncu --set full capture of the config-2 sweep kernel
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/r2_base.log
timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 2 >> gpurun_out/r2_base.log 2>&1
timeout 300 python tools/run_one.py --config 4 --chains 1024 --sweeps 20 --burn 2 --repeat 2 >> gpurun_out/r2_base.log 2>&1
nproc >> gpurun_out/r2_base.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep5" -c 1 -o gpurun_out/ncu_r2_c2 -f python tools/run_one.py --config 2 --sweeps 12 --burn 2 > gpurun_out/ncu_r2_c2.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_r2_c2.log
