#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x -k "ozaki" > gpurun_out/pytest_oz.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_oz.log
: > gpurun_out/oz_time.log
for oz in 1; do
MCINV_CONTRACT_OZAKI=$oz timeout 300 python tools/run_one.py --config 3 --sweeps 66 --burn 2 --repeat 2 --outputs full >> gpurun_out/oz_time.log 2>&1
done
MCINV_CONTRACT_OZAKI=1 timeout 600 ncu --set full --clock-control none -k regex:"ozaki_gemm" -c 1 -o /tmp/ozg -f python tools/run_one.py --config 3 --sweeps 34 --burn 2 --outputs full > gpurun_out/ozg.log 2>&1
ncu -i /tmp/ozg.ncu-rep --page raw --csv > gpurun_out/ozg_raw.csv 2>/dev/null
ncu -i /tmp/ozg.ncu-rep --page source --csv > gpurun_out/ozg_src.csv 2>/dev/null
