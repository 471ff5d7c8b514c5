#!/bin/bash
# config 2: per-GPU rate vs chains per run and chains per CTA (is a chain-batched run faster?)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/c2batch.log
for cfg in "1024 8" "512 4" "256 2" "512 2" "256 4" "128 2" "2048 8" "2048 16"; do
  set -- $cfg
  echo "chains $1 C $2" >> gpurun_out/c2batch.log
  MCINV_C=$2 timeout 300 python tools/run_one.py --config 2 --chains $1 --sweeps 202 --burn 2 --repeat 2 >> gpurun_out/c2batch.log 2>&1
done
