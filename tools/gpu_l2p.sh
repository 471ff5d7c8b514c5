#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/l2p.log
for mb in 0 48 64 32; do
echo "persist $mb MB" >> gpurun_out/l2p.log
MCINV_L2_PERSIST=$mb timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 2 >> gpurun_out/l2p.log 2>&1
done
