#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
: > gpurun_out/ablate.log
for spec in "gauss:diag,pattern" "zero:diag,pattern" "gauss:diag" "zero:diag" "z2:diag,pattern" "z2:diag"; do
  IFS=: read nz outs <<< "$spec"
  timeout 120 python tools/run_one.py --config ${CFG:-2} --sweeps 22 --repeat 2 --noise $nz --outputs $outs 2>&1 | tail -1 | sed "s/^/[$spec] /" >> gpurun_out/ablate.log
done
