#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "v5_trace or config2_production or config5_production or config5_reduced or dirac_parity or geyer or v4_dataflow" > gpurun_out/pytest_dbg1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dbg1.log
: > gpurun_out/c2_stats.log
timeout 300 python tools/c2_stats.py >> gpurun_out/c2_stats.log 2>&1
MCINV_KERNEL=v5 MCINV_C=8 timeout 300 python tools/c2_stats.py >> gpurun_out/c2_stats.log 2>&1
timeout 300 python tools/c2_stats.py 0x5EED1002 >> gpurun_out/c2_stats.log 2>&1
timeout 300 python tools/c2_stats.py 0x5EED2002 >> gpurun_out/c2_stats.log 2>&1
: > gpurun_out/c5_time.log
timeout 300 python tools/run_one.py --config 5 --sweeps 22 --burn 2 --repeat 2 >> gpurun_out/c5_time.log 2>&1
MCINV_KERNEL=v3 timeout 300 python tools/run_one.py --config 5 --sweeps 22 --burn 2 --repeat 2 >> gpurun_out/c5_time.log 2>&1
timeout 300 python tools/run_one.py --config 5 --sweeps 22 --burn 2 --repeat 2 --outputs diag >> gpurun_out/c5_time.log 2>&1
