#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/ecap.log
for k in "0 3" "64 3" "64 1" "48 3" "80 3"; do
  set -- $k
  echo "ecap $1 prefetch $2" >> gpurun_out/ecap.log
  if [ "$1" = "0" ]; then E=""; else E="MCINV_BLOCK_ENTRIES=$1"; fi
  env $E MCINV_PREFETCH=$2 timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 2 >> gpurun_out/ecap.log 2>&1
done
