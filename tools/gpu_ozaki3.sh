#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/oz_time3.log
echo "KC 64" >> gpurun_out/oz_time3.log
MCINV_CONTRACT_OZAKI=1 timeout 300 python tools/run_one.py --config 3 --sweeps 66 --burn 2 --repeat 2 --outputs full >> gpurun_out/oz_time3.log 2>&1
MCINV_NVCC_EXTRA="-DMCINV_OZ_KC=32" python -m paper_cs_0412107_b200.build --force > gpurun_out/build_kc.log 2>&1 || echo "build B failed" >> gpurun_out/oz_time3.log
echo "KC 32" >> gpurun_out/oz_time3.log
timeout 600 python -m pytest tests -m gpu -q -x -k "ozaki" >> gpurun_out/oz_time3.log 2>&1
MCINV_CONTRACT_OZAKI=1 timeout 300 python tools/run_one.py --config 3 --sweeps 66 --burn 2 --repeat 2 --outputs full >> gpurun_out/oz_time3.log 2>&1
