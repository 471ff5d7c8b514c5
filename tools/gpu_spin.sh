# dataflow wait polling: MCINV_SPIN_NS sweep on configs 2 / 3 (sweep kernel rate)
for ns in 32 0 16 64 128; do
  for cfg in 2 3; do
    echo "spin $ns config $cfg" >> gpurun_out/spin.log
    MCINV_SPIN_NS=$ns timeout 300 python tools/run_one.py --config $cfg --sweeps 22 --repeat 3 2>&1 | tail -1 >> gpurun_out/spin.log
  done
done
