cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "v6 or config2 or irregular or long_dependency or gauss" > gpurun_out/pytest_stage.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_stage.log
ABL_LIST="stage:MCINV_V6_STAGE=0 stage stage:MCINV_V6_STAGE=2 stage:MCINV_V6_STAGE=8 stage:MCINV_PREFETCH=11 stage:MCINV_V6_STAGE=0" bash tools/gpu_abl.sh
