#!/bin/bash
# v6 A/B: two gather chunks in flight (compile-time MCINV_V6_CHUNKS=2)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/chunks_time.log
echo "default (1 chunk)" >> gpurun_out/chunks_time.log
timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 2 >> gpurun_out/chunks_time.log 2>&1
MCINV_NVCC_EXTRA="-DMCINV_V6_CHUNKS=2" python -m paper_cs_0412107_b200.build --force > gpurun_out/build_ch.log 2>&1 || echo "build B failed" >> gpurun_out/chunks_time.log
for th in 512 640 768 1024; do
echo "2 chunks, $th threads" >> gpurun_out/chunks_time.log
MCINV_THREADS=$th timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 2 >> gpurun_out/chunks_time.log 2>&1
done
timeout 600 python -m pytest tests -m gpu -q -x -k "v6 or config2_production or long_dependency" > gpurun_out/pytest_chunks.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_chunks.log
