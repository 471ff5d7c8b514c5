#!/bin/bash
# ncu --set full of the Ozaki slice kernel and GEMM (config 3, one contraction)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for k in ozaki_slice_tiled; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -c 1 -o /tmp/$k -f python tools/run_one.py --config 3 --sweeps 66 --burn 2 --outputs full > gpurun_out/ncu_$k.log 2>&1
ncu -i /tmp/$k.ncu-rep --page raw --csv > gpurun_out/${k}_raw.csv 2>/dev/null
ncu -i /tmp/$k.ncu-rep --page source --csv > gpurun_out/${k}_src.csv 2>/dev/null
ncu -i /tmp/$k.ncu-rep > gpurun_out/${k}_details.txt 2>/dev/null
done
