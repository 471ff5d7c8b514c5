#!/bin/bash
# config 4 at 1024 chains (the 8-GPU strong-scaling shard): launch-shape sweep of v3 and the dataflow kernels
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=gpurun_out/c4low2.log; : > $L
run() { echo "[$1] config 4 chains ${CH:-1024}" >> $L; env $1 timeout 300 python tools/run_one.py --config 4 --chains ${CH:-1024} --sweeps 12 --burn 2 --repeat 2 >> $L 2>&1; }
run MCINV_THREADS=1024
run MCINV_THREADS=768
run MCINV_THREADS=512
run MCINV_C=4
run MCINV_K=1
run "MCINV_C=4 MCINV_K=1"
run MCINV_KERNEL=v5
run MCINV_KERNEL=v6
