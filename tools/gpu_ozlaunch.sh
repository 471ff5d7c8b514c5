#!/bin/bash
# per-kernel launch times of one config-3 contraction cycle (slice kernels vs GEMM)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x -k "ozaki or contraction" > gpurun_out/pytest_oz.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_oz.log
MCINV_CONTRACT_OZAKI=1 timeout 300 python tools/run_one.py --config 3 --sweeps 66 --burn 2 --repeat 2 --outputs full > gpurun_out/oz_time.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/oz_launch.csv python tools/run_one.py --config 3 --sweeps 66 --burn 2 --outputs full > gpurun_out/oz_launch.log 2>&1
python tools/launch_summary.py gpurun_out/oz_launch.csv > gpurun_out/oz_launch.txt 2>&1
