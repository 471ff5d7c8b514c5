#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
: > gpurun_out/chains.log
for spec in $SPECS; do
  IFS=: read cfg ch C <<< "$spec"
  env ${C:+MCINV_C=$C} timeout 120 python tools/run_one.py --config $cfg --sweeps 22 --repeat 2 --chains $ch 2>&1 | tail -1 | sed "s/^/[$spec] /" >> gpurun_out/chains.log
done
