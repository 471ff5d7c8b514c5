#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q -x -k "v5_trace or config5 or contraction or config1_full or config3_reduced or config3_real or all_outputs or both_kernels or dirac or geyer or z2 or v4_dataflow or config3_production" > gpurun_out/pytest_dbg3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_dbg3.log
: > gpurun_out/c5_time3.log
timeout 300 python tools/run_one.py --config 5 --sweeps 22 --burn 2 --repeat 2 >> gpurun_out/c5_time3.log 2>&1
MCINV_KERNEL=v3 timeout 300 python tools/run_one.py --config 5 --sweeps 22 --burn 2 --repeat 2 >> gpurun_out/c5_time3.log 2>&1
: > gpurun_out/c3_time3.log
for t in 1 0; do
MCINV_CONTRACT_TMA=$t timeout 300 python tools/run_one.py --config 3 --sweeps 66 --burn 2 --repeat 2 --outputs full >> gpurun_out/c3_time3.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"contract" -c 1 -o gpurun_out/ncu_k3tma2 -f python tools/run_one.py --config 3 --sweeps 40 --burn 2 --outputs full > gpurun_out/ncu_k3tma2.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_k3tma2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep5" -c 1 -o gpurun_out/ncu_c5v5 -f python tools/run_one.py --config 5 --sweeps 6 --burn 2 > gpurun_out/ncu_c5v5.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_c5v5.log
