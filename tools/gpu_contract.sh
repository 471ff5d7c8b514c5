#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "full or config1 or kernels or config3" > gpurun_out/pytest_contract.log 2>&1; echo rc=$? >> gpurun_out/pytest_contract.log
python - > gpurun_out/contract_time.log 2>&1 <<'PY'
import time, torch, sys
sys.path.insert(0, '.')
import workloads as W, paper_cs_0412107_b200 as M
c, q, run = W.config(3)
inv = M.Inverter(c)
inv.set_timing(True)
for rep in range(2):
    inv.run(run.seed, run.chains, 0, 64, ("full",), group_size=32)
    torch.cuda.synchronize()
    st = inv.stats()
    flops = 8.0 * c.n * c.n * run.chains * 64
    print(f"config 3 full: 64 sampling sweeps, contraction {st['contract_ms']:.1f} ms in {st['contract_launches']} launches "
          f"= {flops / (st['contract_ms'] / 1e3) / 1e12:.2f} TFLOP/s (fp64); sweeps {st['sweep_ms']:.1f} ms", flush=True)
PY
