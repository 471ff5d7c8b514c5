#!/bin/bash
# parameter sweep of the v3 launch shape: SPECS="cfg:C:threads ..." 
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/sweep.log
for spec in $SPECS; do
  IFS=: read cfg C th <<< "$spec"
  env ${C:+MCINV_C=$C} MCINV_THREADS=$th timeout 120 python tools/run_one.py --config $cfg --sweeps ${SWEEPS:-22} --repeat 2 2>&1 | tail -1 | sed "s/^/[$spec] /" >> gpurun_out/sweep.log
done
