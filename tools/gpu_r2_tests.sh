#!/bin/bash
# round-2 GPU check: build, full GPU suite, smoke, one bench line (per_config included)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -x --durations=25 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_r2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_r2.log
if [ -z "$NO_BENCH" ]; then
timeout 1200 python bench.py --steps ${STEPS:-3} --warmup 3 > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo "bench rc=$?" >> gpurun_out/bench_r2.err
fi
