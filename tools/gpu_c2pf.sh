#!/bin/bash
# config 2 with KU = 6: L2 prefetch on (default 3), L1 (1), off (0)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/c2pf.log
for pf in 3 0 1 3; do
  echo "MCINV_PREFETCH=$pf" >> gpurun_out/c2pf.log
  MCINV_PREFETCH=$pf timeout 300 python tools/run_one.py --config 2 --sweeps 202 --burn 2 --repeat 3 2>&1 | sed 's/, kernel.*//' | tail -2 >> gpurun_out/c2pf.log
done
