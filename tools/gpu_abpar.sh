#!/bin/bash
# parity subset (v6 / config 2 tests) on a library variant (AB_VAR), then the A/B timings
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
L=paper_cs_0412107_b200/libmcinv.so
cp $L /tmp/libmcinv_prod.so
cp ab/libmcinv_${AB_VAR}.so $L
env ${AB_ENV:-X=1} timeout 900 python -m pytest tests -m gpu -q -x -k "${AB_K:-v6 or config2 or irregular or long_dependency}" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_ab.log
cp /tmp/libmcinv_prod.so $L
bash tools/gpu_abl.sh
