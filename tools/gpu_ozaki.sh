#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x -k "ozaki" > gpurun_out/pytest_oz.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_oz.log
: > gpurun_out/oz_time.log
for oz in 0 1; do
MCINV_CONTRACT_OZAKI=$oz timeout 300 python tools/run_one.py --config 3 --sweeps 66 --burn 2 --repeat 2 --outputs full >> gpurun_out/oz_time.log 2>&1
done
