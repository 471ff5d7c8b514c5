#!/bin/bash
# quick perf iteration: build, a few GPU parity tests, timings, optional ncu of one config-2 sweep launch
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest tests -m gpu -x -q -k "kernels or custom or config1 or config3_reduced or config5_reduced or config2_reduced" > gpurun_out/pytest_quick.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_quick.log
: > gpurun_out/run_quick.log
for cfg in ${CFGS:-2 3 5}; do
  for th in ${THS:-1024}; do
    MCINV_THREADS=$th timeout 120 python tools/run_one.py --config $cfg --sweeps ${SWEEPS:-22} --repeat 2 >> gpurun_out/run_quick.log 2>&1; echo "cfg $cfg th $th rc=$?" >> gpurun_out/run_quick.log
  done
done
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --import-source on -k regex:sweep3 -c 1 -o gpurun_out/ncu_sweep3 -f python tools/run_one.py --config ${NCU} --sweeps 4 --burn 1 > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu.log
fi
