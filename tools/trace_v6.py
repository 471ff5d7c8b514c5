"""Diagnostic: run config 2 on a library built with -DMCINV_TRACE=1 (tools/ab_variant.sh) and
dump the per-item clock64 stamps of CTA 0 (sweep6.cu) to a file for offline analysis."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import workloads as W
    import paper_cs_0412107_b200 as M
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace.bin"
    c, q, run = W.config(2)
    inv = M.Inverter(c, q=q)
    inv.run(run.seed, run.chains, 2, 28, run.outputs, group_size=run.group_size)
    torch.cuda.synchronize()
    L = M.load()
    L.mcinv_debug_trace_dump.restype = ctypes.c_int
    n = L.mcinv_debug_trace_dump(out.encode())
    print("items", n, inv.kernel_info())


if __name__ == "__main__":
    main()
