"""Measured FP64 tensor (DMMA) yardsticks on this B200: cuBLAS DGEMM / ZGEMM
(torch.matmul) at a large square size, and ZGEMM at the contraction's shape
(n x n += n x K . K x n, n = 4096, K = 1024). Prints one JSON line; used as the
roofline peak of the K3 contraction."""
import json
import torch


def timed(f, reps=5):
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        a.record()
        f()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 1e3)
    return best


out = {}
n = 8192
x = torch.randn(n, n, dtype=torch.float64, device="cuda")
out["dgemm_8192_tflops"] = 2 * n ** 3 / timed(lambda: x @ x) / 1e12
z = torch.randn(4096, 4096, dtype=torch.complex128, device="cuda")
out["zgemm_4096_tflops"] = 8 * 4096 ** 3 / timed(lambda: z @ z) / 1e12
a = torch.randn(4096, 1024, dtype=torch.complex128, device="cuda")
c = torch.zeros(4096, 4096, dtype=torch.complex128, device="cuda")
out["zgemm_4096x1024_conjT_tflops"] = 8 * 4096 * 4096 * 1024 / timed(lambda: c.add_(a @ a.conj().T)) / 1e12
print(json.dumps(out))
