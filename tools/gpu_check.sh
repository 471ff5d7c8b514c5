#!/bin/bash
# One gpurun session: build, GPU tests, quick timings of both sweep kernels, bench.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for k in v1 v2; do
  MCINV_KERNEL=$k timeout 120 python tools/run_one.py --config 2 --sweeps 22 --repeat 2 > gpurun_out/run_c2_$k.log 2>&1; echo "rc=$?" >> gpurun_out/run_c2_$k.log
done
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
