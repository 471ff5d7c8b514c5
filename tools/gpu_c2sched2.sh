#!/bin/bash
# config 2 (v6, KU = 6): slack x similarity window; configs 3 and 5 (v5) under the same knobs
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/c2sched2.log
run() { local cfg=$1 sw=$2; shift 2; echo "config $cfg: $*" >> gpurun_out/c2sched2.log; env "$@" timeout 300 python tools/run_one.py --config $cfg --sweeps $sw --burn 2 --repeat 2 --outputs diag 2>&1 | sed 's/, kernel.*//' >> gpurun_out/c2sched2.log; }
for v in "MCINV_X=base" "MCINV_SIMILAR=64" "MCINV_SIMILAR=128" "MCINV_SLACK_PAD=10" "MCINV_SLACK_PAD=10 MCINV_SIMILAR=64" "MCINV_SLACK_PAD=10 MCINV_SIMILAR=128" "MCINV_SLACK=16 MCINV_SIMILAR=64"; do
  run 2 202 $v
done
for v in "MCINV_X=base" "MCINV_SIMILAR=64" "MCINV_SLACK_PAD=10 MCINV_SIMILAR=64"; do
  run 3 102 $v
  run 5 12 $v
done
