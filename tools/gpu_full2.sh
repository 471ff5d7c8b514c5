#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/full2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/full2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full2_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/full2_smoke.log
timeout 1500 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/full2_bench.json 2> gpurun_out/full2_bench.err; echo "bench rc=$?" >> gpurun_out/full2_bench.err
