#!/bin/bash
# repeated dataflow-kernel parity runs at the current build (a race in the row counters or the
# list schedule would show as an intermittent mismatch)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/stress_head.log
for r in 1 2 3 4; do
timeout 900 python -m pytest tests -m gpu -q -k "v6 or v5_trace or v4_dataflow or long_dependency or irregular or config2_production or config5_production or level2_states" 2>&1 | tail -1 >> gpurun_out/stress_head.log; echo "round $r rc=${PIPESTATUS[0]}" >> gpurun_out/stress_head.log
done
nvidia-smi --query-gpu=name,clocks.sm --format=csv >> gpurun_out/stress_head.log
