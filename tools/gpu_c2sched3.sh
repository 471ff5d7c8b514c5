#!/bin/bash
# config 2 diag + pattern (the bench outputs): schedule knobs, 3 repeats each, twice interleaved
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/c2sched3.log
run() { echo "$*" >> gpurun_out/c2sched3.log; env "$@" timeout 300 python tools/run_one.py --config 2 --sweeps 402 --burn 2 --repeat 3 2>&1 | sed 's/, kernel.*//' | tail -2 >> gpurun_out/c2sched3.log; }
for rep in 1 2; do
for v in "MCINV_X=base" "MCINV_SLACK_PAD=10" "MCINV_SIMILAR=64" "MCINV_SLACK_PAD=10 MCINV_SIMILAR=64" "MCINV_SLACK=16 MCINV_SIMILAR=64" "MCINV_SLACK_PAD=10 MCINV_SIMILAR=48"; do
  run $v
done
done
