#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/c4pf.log
for ch in 1024 8192; do for pf in 3 4; do
echo "chains $ch prefetch $pf" >> gpurun_out/c4pf.log
MCINV_PREFETCH=$pf timeout 300 python tools/run_one.py --config 4 --chains $ch --sweeps 12 --burn 2 --repeat 2 >> gpurun_out/c4pf.log 2>&1
done; done
timeout 600 python -m pytest tests -m gpu -q -x -k "config4_production or both_kernels or chains_per_thread" > gpurun_out/pytest_c4pf.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c4pf.log
