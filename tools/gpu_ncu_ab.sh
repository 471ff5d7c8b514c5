#!/bin/bash
# ncu --set full of the config-2 sweep with an ab/ library variant (NCU_VAR), raw csv out
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=paper_cs_0412107_b200/libmcinv.so
cp $L /tmp/libmcinv_prod.so
cp ab/libmcinv_${NCU_VAR:-ofs}.so $L
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep6 -c 1 -o /tmp/nab -f python tools/run_one.py --config 2 --sweeps 12 --burn 2 > gpurun_out/ncu_ab.log 2>&1
ncu -i /tmp/nab.ncu-rep --page raw --csv > gpurun_out/ncu_ab_raw.csv 2>/dev/null
ncu -i /tmp/nab.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_ab_src.csv 2>/dev/null
cp /tmp/nab.ncu-rep gpurun_out/ncu_ab.ncu-rep
cp /tmp/libmcinv_prod.so $L
