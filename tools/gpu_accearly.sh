#!/bin/bash
# v6 A/B: accumulate before the publication with the gathered partners (compile-time)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/accearly.log
echo "default" >> gpurun_out/accearly.log
timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 2 >> gpurun_out/accearly.log 2>&1
MCINV_NVCC_EXTRA="-DMCINV_V6_ACC_EARLY=1" python -m paper_cs_0412107_b200.build --force > gpurun_out/build_ae.log 2>&1 || echo "build B failed" >> gpurun_out/accearly.log
echo "accumulate early" >> gpurun_out/accearly.log
timeout 120 python tools/run_one.py --config 2 --sweeps 220 --burn 20 --repeat 2 >> gpurun_out/accearly.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "v6 or config2_production or long_dependency or irregular" > gpurun_out/pytest_ae.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ae.log
