# rate of configs under env variants: VARIANTS="NAME=VAL,NAME2=VAL2 ..." CFGS="2 3"
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/env.log
for v in $VARIANTS; do
  for cfg in ${CFGS:-2 3}; do
    echo "[$v] config $cfg" >> gpurun_out/env.log
    env $(echo $v | tr ',' ' ') timeout 300 python tools/run_one.py --config $cfg --sweeps ${SWEEPS:-22} --repeat 3 2>&1 | tail -1 >> gpurun_out/env.log
  done
done
