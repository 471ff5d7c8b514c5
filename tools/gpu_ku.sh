#!/bin/bash
# v6 A/B: gather unroll 4 at 513-768 threads (compile-time), config 4 chain-count sweep
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/ku_time.log
MCINV_THREADS=512 timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 2 >> gpurun_out/ku_time.log 2>&1
for ch in 1024 2048 4096; do
timeout 300 python tools/run_one.py --config 4 --chains $ch --sweeps 12 --burn 2 --repeat 2 >> gpurun_out/ku_time.log 2>&1
done
MCINV_KERNEL=v6 timeout 300 python tools/run_one.py --config 4 --chains 2048 --sweeps 12 --burn 2 --repeat 2 >> gpurun_out/ku_time.log 2>&1
MCINV_NVCC_EXTRA="-DMCINV_V6_KU768=4" python -m paper_cs_0412107_b200.build --force > gpurun_out/build_ku.log 2>&1 || echo "build B failed" >> gpurun_out/ku_time.log
grep -A2 "sweep6_kernelILi4ELi768ELi3ELi2ELb0ELb1E" paper_cs_0412107_b200/build.log | grep -E "regis|spill" >> gpurun_out/ku_time.log
for th in 640 768; do
MCINV_THREADS=$th timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 2 >> gpurun_out/ku_time.log 2>&1
done
