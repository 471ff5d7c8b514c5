#!/bin/bash
# v5 complex gather unroll (MCINV_V5_KUC): configs 3 and 5 sweep rate, v5 complex parity
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/v5ku.log
for k in 2 3 4; do
  MCINV_NVCC_EXTRA="-DMCINV_V5_KUC=$k" python -c "from paper_cs_0412107_b200 import build; build.build(force=True)" > gpurun_out/build_v5.log 2>&1 || { echo build failed; exit 1; }
  echo "KUC=$k" >> gpurun_out/v5ku.log
  timeout 300 python tools/run_one.py --config 3 --sweeps 102 --burn 2 --repeat 3 --outputs diag 2>&1 | sed 's/, kernel.*//' | tail -2 >> gpurun_out/v5ku.log
  timeout 300 python tools/run_one.py --config 5 --sweeps 22 --burn 2 --repeat 2 2>&1 | sed 's/, kernel.*//' | tail -1 >> gpurun_out/v5ku.log
  if [ $k != 2 ]; then timeout 900 python -m pytest tests -m gpu -q -x -k "v5 or config3_production or config5_production or lattice or complex" 2>&1 | tail -1 >> gpurun_out/v5ku.log; fi
done
