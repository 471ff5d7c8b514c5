#!/bin/bash
# round-2 final evidence after the K3 Ozaki rework: GPU suite, smoke, bench line (driver's K/W),
# ncu launch list of the bench command, ncu --set full of the Ozaki GEMM and slicing kernels
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
if [ -z "$SKIP_TESTS" ]; then
timeout 2400 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/ev_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev_smoke.log
fi
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err; echo "bench rc=$?" >> gpurun_out/ev_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-per-config > gpurun_out/ev_ncu_launch.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ev_ncu_launch.log
python tools/launch_summary.py gpurun_out/ev_launches.csv > gpurun_out/ev_launches.txt 2>&1
cap() {  # tag kernel-regex run_one args...
  local tag=$1 rx=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$rx" -c 1 -o /tmp/$tag -f python tools/run_one.py "$@" > gpurun_out/$tag.log 2>&1
  ncu -i /tmp/$tag.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
  ncu -i /tmp/$tag.ncu-rep > gpurun_out/${tag}_details.txt 2>/dev/null
}
#cap ev_k3oz ozaki_gemm --config 3 --sweeps 66 --burn 2 --outputs full
#cap ev_k3sl ozaki_slice --config 3 --sweeps 66 --burn 2 --outputs full
du -sh gpurun_out
