#!/bin/bash
# whole GPU suite + smoke, plus the tensor-map K3 variant's parity test
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
MCINV_OZ_BULK=0 timeout 300 python -m pytest tests -m gpu -q -k "ozaki" > gpurun_out/pytest_oz_tmap.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_oz_tmap.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
