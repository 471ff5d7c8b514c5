#!/bin/bash
# Ozaki GEMM: parity + timing with the normal build, then thread-0 cycle buckets (MCINV_OZ_PROF build)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
#timeout 600 python -m pytest tests -m gpu -q -x -k "ozaki or contraction" > gpurun_out/pytest_oz.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_oz.log
: > gpurun_out/ozprof.log
MCINV_CONTRACT_OZAKI=1 timeout 300 python tools/run_one.py --config 3 --sweeps 130 --burn 2 --repeat 2 --outputs full >> gpurun_out/ozprof.log 2>&1
MCINV_NVCC_EXTRA=-DMCINV_OZ_PROF python -c "from paper_cs_0412107_b200 import build; build.build(force=True)" > gpurun_out/build2.log 2>&1 || { echo build failed; exit 1; }
MCINV_CONTRACT_OZAKI=1 timeout 300 python tools/run_one.py --config 3 --sweeps 66 --burn 2 --outputs full 2>&1 | grep -v "^$" | tail -3 >> gpurun_out/ozprof.log
