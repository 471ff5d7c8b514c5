#!/bin/bash
# Round evidence: full GPU test suite, the bench line, the ncu launch list of the
# bench command, and one `ncu --set full` capture of the sweep kernel (config 2
# launch shape, 12 sweeps). Outputs in gpurun_out/ (summarised into profiles/).
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
BCMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
if [ -z "$NO_NCU" ]; then
  timeout 600 $BCMD > gpurun_out/bench_plain.log 2>&1 &&
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $BCMD > gpurun_out/ncu_launches.log 2>&1
  echo "launches rc=$?" >> gpurun_out/ncu_launches.log
  RCMD="python tools/run_one.py --config ${NCFG:-2} --sweeps 12 --burn 2"
  timeout 300 $RCMD > gpurun_out/run_plain.log 2>&1 &&
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sweep[345]" -c 1 -o gpurun_out/prof_sweep3 -f $RCMD > gpurun_out/ncu_full.log 2>&1
  echo "full rc=$?" >> gpurun_out/ncu_full.log
fi
