#!/bin/bash
# parameter sweep: SPECS="cfg:C:threads:K:kernel ..."
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/sweep.log
for spec in $SPECS; do
  IFS=: read cfg C th K ker <<< "$spec"
  env ${C:+MCINV_C=$C} ${th:+MCINV_THREADS=$th} ${K:+MCINV_K=$K} ${ker:+MCINV_KERNEL=$ker} timeout 120 python tools/run_one.py --config $cfg --sweeps ${SWEEPS:-22} --repeat 2 2>&1 | tail -1 | sed "s/^/[$spec] /" >> gpurun_out/sweep.log
done
