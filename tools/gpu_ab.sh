# A/B of a compile-time variant: build A (default flags) then B (MCINV_NVCC_EXTRA="$BFLAGS"),
# config rates with 220 sweeps each; optional quick parity tests on B (BTESTS)
: > gpurun_out/ab.log
for side in A B; do
  if [ $side = A ]; then python -c "from paper_cs_0412107_b200 import build; build.build(force=True)" > gpurun_out/build_A.log 2>&1
  else MCINV_NVCC_EXTRA="$BFLAGS" python -c "from paper_cs_0412107_b200 import build; build.build(force=True)" > gpurun_out/build_B.log 2>&1; fi
  for cfg in ${CFGS:-2 3}; do
    echo "[$side] config $cfg" >> gpurun_out/ab.log
    timeout 300 python tools/run_one.py --config $cfg --sweeps 220 --repeat 2 ${RARGS} 2>&1 | tail -1 >> gpurun_out/ab.log
  done
done
if [ -n "$BTESTS" ]; then timeout 600 python -m pytest tests -m gpu -x -q -k "$BTESTS" > gpurun_out/pytest_ab.log 2>&1; echo rc=$? >> gpurun_out/pytest_ab.log; fi
