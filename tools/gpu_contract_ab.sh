# contraction (K3) timing on config 3 under MCINV_CONTRACT_WN variants, then the full-output parity tests
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
: > gpurun_out/contract_ab.log
for spec in ${SPECS:-MCINV_CONTRACT_WN=32 MCINV_CONTRACT_WN=16}; do
env $spec python - >> gpurun_out/contract_ab.log 2>&1 <<'PY'
import os, torch, sys
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
    print(f"{os.environ.get('MCINV_CONTRACT_WN', '')} {os.environ.get('MCINV_CONTRACT_3M', '')} config 3 full: contraction {st['contract_ms']:.1f} ms in {st['contract_launches']} launches "
          f"= {flops / (st['contract_ms'] / 1e3) / 1e12:.2f} TFLOP/s (fp64); sweeps {st['sweep_ms']:.1f} ms", flush=True)
PY
done
env ${TESTENV:-MCINV_CONTRACT_WN=16} timeout 900 python -m pytest tests -m gpu -x -q -k "full or config1 or config3 or contraction" > gpurun_out/pytest_contract.log 2>&1; echo rc=$? >> gpurun_out/pytest_contract.log
