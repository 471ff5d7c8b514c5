#!/bin/bash
# Ozaki K3: parity (tiled bulk default and tensor-map TMA), timing A/B, one ncu capture of the default
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest tests -m gpu -q -x -k "ozaki or contraction" > gpurun_out/pytest_oz.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_oz.log
MCINV_OZ_BULK=0 timeout 600 python -m pytest tests -m gpu -q -x -k "ozaki" >> gpurun_out/pytest_oz.log 2>&1; echo "pytest (tensor-map) rc=$?" >> gpurun_out/pytest_oz.log
: > gpurun_out/oz_time.log
for b in 1 0; do
echo "MCINV_OZ_BULK=$b" >> gpurun_out/oz_time.log
MCINV_OZ_BULK=$b MCINV_CONTRACT_OZAKI=1 timeout 300 python tools/run_one.py --config 3 --sweeps 66 --burn 2 --repeat 2 --outputs full >> gpurun_out/oz_time.log 2>&1
done
MCINV_CONTRACT_OZAKI=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ozaki_gemm" -c 1 -o /tmp/ozg -f python tools/run_one.py --config 3 --sweeps 34 --burn 2 --outputs full > gpurun_out/ozg.log 2>&1
ncu -i /tmp/ozg.ncu-rep --page raw --csv > gpurun_out/ozg_raw.csv 2>/dev/null
ncu -i /tmp/ozg.ncu-rep --page source --csv > gpurun_out/ozg_src.csv 2>/dev/null
