#!/bin/bash
# v6 prefetch variants (compile-time): one lane per row, next item one item ahead
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
: > gpurun_out/v6pf.log
for v in "" "-DMCINV_V6_PF_ONE=1" "-DMCINV_V6_PF_NEXT=1" "-DMCINV_V6_PF_ONE=1 -DMCINV_V6_PF_NEXT=1"; do
  MCINV_NVCC_EXTRA="$v" python -c "from paper_cs_0412107_b200 import build; build.build(force=True)" > gpurun_out/build_pf.log 2>&1 || { echo build failed; exit 1; }
  echo "variant [$v]" >> gpurun_out/v6pf.log
  timeout 300 python tools/run_one.py --config 2 --sweeps 202 --burn 2 --repeat 3 2>&1 | sed 's/, kernel.*//' | tail -2 >> gpurun_out/v6pf.log
  if [ -n "$v" ]; then timeout 600 python -m pytest tests -m gpu -q -x -k "v6 or config2_production or long_dependency" 2>&1 | tail -1 >> gpurun_out/v6pf.log; fi
done
