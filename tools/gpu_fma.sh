# noise polynomials with explicit fma (MCINV_NOISE_FMA) vs separate mul/add; prefetch modes
python -c "from paper_cs_0412107_b200 import build; build.build(force=True)" > gpurun_out/build.log 2>&1
: > gpurun_out/fma.log
run() { for cfg in 2 3; do echo "[$1 $2] config $cfg" >> gpurun_out/fma.log; env $2 timeout 300 python tools/run_one.py --config $cfg --sweeps 220 --repeat 2 2>&1 | tail -1 >> gpurun_out/fma.log; done; }
run base MCINV_PREFETCH=2
run base MCINV_PREFETCH=3
MCINV_NVCC_EXTRA=-DMCINV_NOISE_FMA python -c "from paper_cs_0412107_b200 import build; build.build(force=True)" >> gpurun_out/build.log 2>&1
run fma MCINV_PREFETCH=2
run fma MCINV_PREFETCH=3
timeout 300 python -m pytest tests -m gpu -x -q -k "gaussian or config2_reduced or v4_dataflow" > gpurun_out/pytest_fma.log 2>&1; echo rc=$? >> gpurun_out/pytest_fma.log
