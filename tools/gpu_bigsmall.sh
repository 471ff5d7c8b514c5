python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "bit_counters or bench_configs or config4" > gpurun_out/pytest_bits2.log 2>&1; echo rc=$? >> gpurun_out/pytest_bits2.log
for ch in 1024 2048 4096; do
  for k in 3 5; do
    echo "chains $ch kernel $k" >> gpurun_out/bigsmall.log
    MCINV_KERNEL=$k timeout 300 python tools/run_one.py --config 4 --chains $ch --sweeps 12 --repeat 2 >> gpurun_out/bigsmall.log 2>&1
  done
done
