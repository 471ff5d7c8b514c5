#!/bin/bash
# time config 2/3 with each prebuilt library in ab/ (experiments)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out; : > gpurun_out/libs.log
for f in ab/lib*.so; do
  cp $f paper_cs_0412107_b200/libmcinv.so; touch paper_cs_0412107_b200/libmcinv.so
  for cfg in ${CFGS:-2 3}; do timeout 120 python tools/run_one.py --config $cfg --sweeps 22 --repeat 2 2>&1 | tail -1 | sed "s@^@[$f] @" >> gpurun_out/libs.log; done
done
