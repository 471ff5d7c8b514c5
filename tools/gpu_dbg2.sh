#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "v5_trace or config2_production or config5_production or contraction or config1_full or config3_reduced or config3_real or all_outputs or both_kernels" > gpurun_out/pytest_dbg2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dbg2.log
timeout 600 python tools/c2_seeds.py 16 > gpurun_out/c2_seeds.log 2>&1
: > gpurun_out/c3_time.log
for t in 1 0; do
MCINV_CONTRACT_TMA=$t timeout 300 python tools/run_one.py --config 3 --sweeps 40 --burn 2 --repeat 2 --outputs full >> gpurun_out/c3_time.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"contract" -c 1 -o gpurun_out/ncu_k3tma -f python tools/run_one.py --config 3 --sweeps 40 --burn 2 --outputs full > gpurun_out/ncu_k3tma.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_k3tma.log
