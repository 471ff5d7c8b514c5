for v in "MCINV_X=0" "MCINV_KERNEL=v3"; do
  echo "[$v diag]" >> gpurun_out/env.log
  env $v timeout 300 python tools/run_one.py --config 5 --sweeps 22 --repeat 2 --outputs diag 2>&1 | tail -1 >> gpurun_out/env.log
done
