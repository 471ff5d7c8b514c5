#!/bin/bash
# v6 gather unroll at 512 threads (MCINV_V6_KU512): config 2 rate and the v6 parity tests
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/v6ku.log
for ku in 5 6 7; do
  MCINV_NVCC_EXTRA="-DMCINV_V6_KU512=$ku" python -c "from paper_cs_0412107_b200 import build; build.build(force=True)" > gpurun_out/build_ku$ku.log 2>&1 || { echo build failed; exit 1; }
  echo "KU512=$ku" >> gpurun_out/v6ku.log
  timeout 300 python tools/run_one.py --config 2 --sweeps 202 --burn 2 --repeat 3 2>&1 | sed 's/, kernel.*//' >> gpurun_out/v6ku.log
  if [ $ku != 6 ]; then timeout 600 python -m pytest tests -m gpu -q -x -k "v6 or config2 or pedigree or long_dependency or irregular" 2>&1 | tail -1 >> gpurun_out/v6ku.log; fi
done
