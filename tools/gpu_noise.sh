# sweep rate by noise mode (cost of the in-kernel noise): gauss / z2 / zero
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: > gpurun_out/noise.log
for nz in gauss z2 zero; do for cfg in 2 3; do
  echo "[$nz] config $cfg" >> gpurun_out/noise.log
  timeout 300 python tools/run_one.py --config $cfg --sweeps 220 --repeat 2 --noise $nz 2>&1 | tail -1 >> gpurun_out/noise.log
done; done
