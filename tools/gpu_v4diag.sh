: > gpurun_out/v4diag.log
for v in "MCINV_RECONV=0" "MCINV_RECONV=1"; do for o in diag diag,pattern; do
  echo "[$v $o]" >> gpurun_out/v4diag.log
  env MCINV_KERNEL=v4 $v timeout 300 python tools/run_one.py --config 2 --sweeps 110 --repeat 2 --outputs $o 2>&1 | tail -1 >> gpurun_out/v4diag.log
done; done
