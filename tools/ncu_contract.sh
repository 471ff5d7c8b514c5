#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
CMD="python tools/run_one.py --config 3 --sweeps ${NSW:-10} --burn 2"
timeout 300 $CMD > gpurun_out/contract_plain.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:contract -c 1 -o gpurun_out/ncu_${TAG:-contract} -f $CMD > gpurun_out/ncu_${TAG:-contract}.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_${TAG:-contract}.log
