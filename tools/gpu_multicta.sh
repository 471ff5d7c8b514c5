#!/bin/bash
# v6 with several CTAs per SM: C chains per CTA, threads, shared-memory budget per CTA
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/multicta.log
for k in "8 512 220" "4 256 100" "4 256 105" "2 128 50" "2 256 100" "4 384 150"; do
  set -- $k
  echo "C=$1 threads=$2 smemKB=$3" >> gpurun_out/multicta.log
  MCINV_C=$1 MCINV_THREADS=$2 MCINV_V6_SMEM_KB=$3 MCINV_CARVE=100 timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 2 >> gpurun_out/multicta.log 2>&1
done
