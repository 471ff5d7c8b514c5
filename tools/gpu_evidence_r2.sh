#!/bin/bash
# round-2 evidence: GPU suite, smoke, bench line (driver's K/W), ncu launch list of the bench
# command, ncu --set full of the sweep kernels (configs 2, 4, 5) and the K3 contraction
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/ev_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev_smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo "bench rc=$?" >> gpurun_out/ev_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config > gpurun_out/ev_ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ev_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep6" -c 1 -o gpurun_out/ev_c2 -f python tools/run_one.py --config 2 --sweeps 12 --burn 2 > gpurun_out/ev_c2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep3" -c 1 -o gpurun_out/ev_c4 -f python tools/run_one.py --config 4 --sweeps 3 --burn 1 > gpurun_out/ev_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep5" -c 1 -o gpurun_out/ev_c5 -f python tools/run_one.py --config 5 --sweeps 4 --burn 1 > gpurun_out/ev_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"contract" -c 1 -o gpurun_out/ev_k3 -f python tools/run_one.py --config 3 --sweeps 40 --burn 2 --outputs full > gpurun_out/ev_k3.log 2>&1
