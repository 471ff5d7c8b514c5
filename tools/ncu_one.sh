#!/bin/bash
# ncu --set full of one sweep3 launch: NCFG (config), NSW (sweeps), extra env passed through
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep[345]" -c 1 -o gpurun_out/ncu_${TAG:-x} -f python tools/run_one.py --config ${NCFG:-2} --sweeps ${NSW:-4} --burn 1 ${NARGS} > gpurun_out/ncu_${TAG:-x}.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_${TAG:-x}.log
