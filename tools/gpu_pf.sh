#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/pf.log
for pf in 3 1 0; do
echo "prefetch $pf" >> gpurun_out/pf.log
MCINV_PREFETCH=$pf timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 2 >> gpurun_out/pf.log 2>&1
done
for cv in 60 75 90; do
echo "carve $cv" >> gpurun_out/pf.log
MCINV_PREFETCH=1 MCINV_CARVE=$cv timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 2 >> gpurun_out/pf.log 2>&1
done
