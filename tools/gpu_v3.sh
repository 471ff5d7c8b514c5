#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for cfg in 2 3 5 4; do
  for th in 512 1024; do
    MCINV_THREADS=$th timeout 120 python tools/run_one.py --config $cfg --sweeps 22 --repeat 2 >> gpurun_out/run_v3.log 2>&1; echo "cfg $cfg th $th rc=$?" >> gpurun_out/run_v3.log
  done
done
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
