: > gpurun_out/dirac_c.log
for C in 16 8 4; do
  echo "[C=$C]" >> gpurun_out/dirac_c.log
  MCINV_C=$C timeout 600 python tools/run_one.py --dirac 18 --sweeps 22 --repeat 2 2>&1 | tail -1 >> gpurun_out/dirac_c.log
done
