#!/bin/bash
# v6 + wait masks: parity + timings (mask on/off) + ncu
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "v6 or gaussian or geyer or config2_reduced or irregular or long_dependency or z2 or config1_full" > gpurun_out/pytest_v6e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_v6e.log
: > gpurun_out/v6e_time.log
for k in "v6 512 1" "v6 640 1"; do
  set -- $k
  MCINV_WAITMASK=$3 MCINV_KERNEL=$1 MCINV_THREADS=$2 timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 3 >> gpurun_out/v6e_time.log 2>&1; echo "$k rc=$?" >> gpurun_out/v6e_time.log
done
MCINV_KERNEL=v6 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep6" -c 1 -o gpurun_out/ncu_v6e -f python tools/run_one.py --config 2 --sweeps 12 --burn 2 > gpurun_out/ncu_v6e.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_v6e.log
