# v5 barrier-free vs sweep-barrier modes: parity tests, then rates on configs 2 / 3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "v4_dataflow or long_dependency or irregular or bit_counters or config2_reduced or config3_reduced or z2 or bench_configs" > gpurun_out/pytest_free.log 2>&1
echo rc=$? >> gpurun_out/pytest_free.log
for mode in free bytes; do
  for cfg in 2 3; do
    echo "mode $mode config $cfg" >> gpurun_out/free.log
    MCINV_V5_MODE=$mode timeout 300 python tools/run_one.py --config $cfg --sweeps 22 --repeat 3 2>&1 | tail -1 >> gpurun_out/free.log
  done
done
