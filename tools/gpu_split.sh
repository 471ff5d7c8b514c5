#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/split.log
echo "diag+pattern (20 burn + 200 sampling)" >> gpurun_out/split.log
timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 2 >> gpurun_out/split.log 2>&1
echo "diag only" >> gpurun_out/split.log
timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 2 --outputs diag >> gpurun_out/split.log 2>&1
echo "burn-in only (219 burn + 1)" >> gpurun_out/split.log
timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 219 --repeat 2 >> gpurun_out/split.log 2>&1
echo "zero noise" >> gpurun_out/split.log
timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 2 --noise zero >> gpurun_out/split.log 2>&1
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm,power.limit,serial --format=csv >> gpurun_out/split.log
