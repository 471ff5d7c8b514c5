#!/bin/bash
# config 2 (v6, KU = 6): list-schedule knobs -- slack, padding bound, similarity window
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/c2sched.log
run() { echo "$*" >> gpurun_out/c2sched.log; env "$@" timeout 300 python tools/run_one.py --config 2 --sweeps 202 --burn 2 --repeat 2 2>&1 | sed 's/, kernel.*//' | tail -1 >> gpurun_out/c2sched.log; }
run MCINV_X=base
run MCINV_SLACK_PAD=2
run MCINV_SLACK_PAD=10
run MCINV_SLACK_PAD=20
run MCINV_SLACK=16
run MCINV_SLACK=24
run MCINV_SLACK=32
run MCINV_SLACK=8
run MCINV_SIMILAR=16
run MCINV_SIMILAR=64
run MCINV_SIMILAR=0
run MCINV_X=base
