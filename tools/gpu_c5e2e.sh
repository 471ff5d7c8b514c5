#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "v5_trace or config5 or geyer or dirac_parity or v6 or config2_production" > gpurun_out/pytest_c5e2e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c5e2e.log
: > gpurun_out/c5e2e.log
timeout 300 python tools/run_one.py --config 5 --sweeps 22 --burn 2 --repeat 2 >> gpurun_out/c5e2e.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-per-config --no-cpu-baseline >> gpurun_out/c5e2e.log 2>&1
