import sys, time
sys.path.insert(0, '.')
import torch, numpy as np
import workloads as W, paper_cs_0412107_b200 as M
c, q, run = W.config(2)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    h = M.Inverter(c, device=0)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    h.run(run.seed, run.chains, run.burn_in, run.cycles, run.outputs, group_size=run.group_size)
    t2 = time.perf_counter()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    res = [h.result(o) for o in run.outputs]
    t4 = time.perf_counter()
    h.close(); torch.cuda.synchronize(); t5 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms, run enqueue {1e3*(t2-t1):.1f} ms, run wait {1e3*(t3-t2):.1f} ms, results {1e3*(t4-t3):.1f} ms, close {1e3*(t5-t4):.1f} ms", flush=True)
