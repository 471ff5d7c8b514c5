#!/bin/bash
# v6 gather unroll re-tuned after the late-r2 scoreboard fix: ab/libmcinv_ku<k>.so (sweep6.cu with
# -DMCINV_V6_KU512=k, tools/ab_variant.sh) swapped in for the product .so; config-2 rate (202 sweeps)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
SO=paper_cs_0412107_b200/libmcinv.so
cp $SO /tmp/libmcinv_ku6.so
L=gpurun_out/v6ku_post.log; : > $L
for v in ku6 ku4 ku5 ku7 ku8 ku6; do
  if [ $v = ku6 ]; then cp /tmp/libmcinv_ku6.so $SO; else cp ab/libmcinv_$v.so $SO; fi
  echo "[$v]" >> $L
  timeout 300 python tools/run_one.py --config 2 --sweeps 202 --burn 2 --repeat 3 2>&1 | sed 's/, kernel.*//' >> $L
  if [ $v != ku6 ]; then timeout 600 python -m pytest tests -m gpu -q -x -k "v6 or config2_production" 2>&1 | tail -1 >> $L; fi
done
cp /tmp/libmcinv_ku6.so $SO
