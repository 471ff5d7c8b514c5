#!/bin/bash
# repeated dataflow-kernel parity runs (races would show as intermittent failures) and the
# config-5 per-GPU rate at its strong-scaling shard sizes
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/stress.log
for r in 1 2 3; do
timeout 900 python -m pytest tests -m gpu -q -k "v6 or v5_trace or v4_dataflow or long_dependency or irregular or config2_production or config5_production or level2_states" >> gpurun_out/stress.log 2>&1; echo "round $r rc=$?" >> gpurun_out/stress.log
done
: > gpurun_out/c5chains.log
for ch in 2048 4096 8192 16384; do
timeout 600 python tools/run_one.py --config 5 --chains $ch --sweeps 12 --burn 2 --repeat 2 >> gpurun_out/c5chains.log 2>&1
done
nvidia-smi --query-gpu=name,serial --format=csv >> gpurun_out/c5chains.log
