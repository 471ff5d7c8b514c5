# sweep rate by accumulated outputs (cost of the fused accumulation), config 2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
: > gpurun_out/outs.log
for spec in ${SPECS:-"diag,pattern:2"}; do
  IFS=: read o b gs ker <<< "$spec"
  echo "[$spec]" >> gpurun_out/outs.log
  env ${ker:+MCINV_KERNEL=$ker} timeout 300 python tools/run_one.py --config 2 --sweeps 220 --burn $b --outputs $o --repeat 2 ${gs:+--group-size $gs} 2>&1 | tail -1 >> gpurun_out/outs.log
done
