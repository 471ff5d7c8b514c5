"""B200-native correlated-chains (CC) Monte Carlo matrix inverter.

Thin Python binding of the C ABI in include/mcinv.h (libmcinv.so, built
in-tree for sm_100a by ``paper_cs_0412107_b200.build``). Argument
marshalling only: every step of the method runs in the library's CUDA
kernels. PyTorch provides device memory (the workspace), the CUDA stream and,
in ``dist``, the NCCL process group. There is no CPU fallback: if the
library or a GPU is missing, calls raise.

Method: Garcia-Cortes & Cabrillo, arXiv cs/0412107 -- Eq. (4)/(5) sweeps
 with shared noise, estimators Eq. (1/C) and
Eq. (tr), Algorithm 1 with a fixed burn-in.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libmcinv.so")
_lib = None

DIAG, PATTERN, FULL, TRACE = 1, 2, 4, 8
OUTPUTS = {"diag": DIAG, "pattern": PATTERN, "full": FULL, "trace": TRACE}
NOISE = {"gauss": 0, "zero": 1, "one": 2, "z2": 3}
F64, C128 = 1, 2

__all__ = ["Inverter", "MCInvError", "load", "philox", "gaussian", "OUTPUTS"]


class MCInvError(RuntimeError):
    def __init__(self, code: int, msg: str = "", index: int = -1):
        self.code, self.msg, self.index = code, msg, index
        name = load().mcinv_status_string(code).decode() if _lib is not None else str(code)
        super().__init__(f"mcinv error {code} ({name}): {msg} [index {index}]")


class _RunArgs(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("chain_begin", ctypes.c_int64), ("chains", ctypes.c_int64),
                ("burn_in", ctypes.c_int64), ("cycles", ctypes.c_int64), ("sweep_begin", ctypes.c_int64),
                ("outputs", ctypes.c_uint), ("noise", ctypes.c_int), ("group_size", ctypes.c_int),
                ("resume", ctypes.c_int), ("snapshot_sweeps", ctypes.c_int), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_size_t), ("stream", ctypes.c_void_p), ("trace_series", ctypes.c_int64)]


SYMBOLS = {
    "mcinv_create": (ctypes.c_int, [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "mcinv_set_trace_q": (ctypes.c_int, [ctypes.c_void_p] * 4),
    "mcinv_set_pattern": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]),
    "mcinv_pattern_size": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]),
    "mcinv_workspace_size": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(_RunArgs), ctypes.POINTER(ctypes.c_size_t)]),
    "mcinv_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(_RunArgs)]),
    "mcinv_accumulators": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p),
                                          ctypes.POINTER(ctypes.c_size_t)]),
    "mcinv_result": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint, ctypes.c_int64, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]),
    "mcinv_coupled_burn_in": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_int64, ctypes.c_void_p,
                                             ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double)]),
    "mcinv_run_until": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(_RunArgs), ctypes.c_uint, ctypes.c_double,
                                       ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                                       ctypes.POINTER(ctypes.c_double)]),
    "mcinv_recenter": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_size_t),
                                      ctypes.POINTER(ctypes.c_size_t)]),
    "mcinv_run_status": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]),
    "mcinv_debug_group_sums": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_void_p]),
    "mcinv_geyer": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "mcinv_run_until_geyer": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(_RunArgs), ctypes.c_double,
                                             ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                                             ctypes.POINTER(ctypes.c_double)]),
    "mcinv_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "mcinv_error_detail": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64),
                                          ctypes.POINTER(ctypes.c_char_p)]),
    "mcinv_destroy": (None, [ctypes.c_void_p]),
    "mcinv_kernel_info": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                         ctypes.POINTER(ctypes.c_int64)]),
    "mcinv_launch_config": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                           ctypes.POINTER(ctypes.c_int)]),
    "mcinv_set_timing": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int]),
    "mcinv_stats": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(ctypes.c_int64)]),
    "mcinv_debug_philox": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p,
                                          ctypes.c_void_p]),
    "mcinv_debug_gaussian": (ctypes.c_int, [ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p,
                                            ctypes.c_void_p]),
    "mcinv_debug_levels": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 6 +
                           [ctypes.c_uint, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                            ctypes.c_void_p, ctypes.c_int64]),
    "mcinv_debug_blocks": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64] + [ctypes.c_void_p] * 6 +
                           [ctypes.c_uint, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]),
    "mcinv_debug_get_state": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                             ctypes.c_void_p]),
    "mcinv_debug_set_state": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                             ctypes.c_void_p]),
}


def load():
    """Load the in-tree libmcinv.so; raise if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise RuntimeError(f"{_SO} is not built: run `python -m paper_cs_0412107_b200.build` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(_SO)
        for name, (res, args) in SYMBOLS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(st: int, h=None):
    if st != 0:
        idx = ctypes.c_int64(-1)
        msg = ctypes.c_char_p()
        if h is not None:
            load().mcinv_error_detail(h, ctypes.byref(idx), ctypes.byref(msg))
        raise MCInvError(st, (msg.value or b"").decode(), idx.value)


def _doubles(val, cplx: bool) -> np.ndarray:
    if cplx:
        return np.ascontiguousarray(np.asarray(val, np.complex128)).view(np.float64)
    return np.ascontiguousarray(np.asarray(val, np.float64))


def philox(ctr: np.ndarray, seed: int, device: int = 0) -> np.ndarray:
    """Philox4x32-10 words computed on the GPU for counters ctr[k, 4]."""
    ctr = np.ascontiguousarray(ctr, np.uint32).reshape(-1, 4)
    out = np.zeros_like(ctr)
    _check(load().mcinv_debug_philox(device, seed, ctr.shape[0], ctr.ctypes.data, out.ctypes.data))
    return out


def gaussian(ctr: np.ndarray, seed: int, device: int = 0) -> np.ndarray:
    """Box-Muller noise of Philox(ctr, seed) computed on the GPU."""
    ctr = np.ascontiguousarray(ctr, np.uint32).reshape(-1, 4)
    out = np.zeros(ctr.shape[0], np.float64)
    _check(load().mcinv_debug_gaussian(device, seed, ctr.shape[0], ctr.ctypes.data, out.ctypes.data))
    return out


def debug_levels(csr, outputs=("diag",), q=None, slot_R: int = 0, slot_L: int = 0):
    """Host-only v3 level schedule (no GPU): (lev[n], info dict); with slot_R > 0
    also info["slots"], the v4 slot schedule (row per slot, -1 = padding)."""
    cplx = np.iscomplexobj(csr.val)
    rp = np.ascontiguousarray(csr.row_ptr, np.int64)
    col = np.ascontiguousarray(csr.col, np.int32)
    val = _doubles(csr.val, cplx)
    args = [C128 if cplx else F64, csr.n, rp.ctypes.data, col.ctypes.data, val.ctypes.data]
    keep = [rp, col, val]
    if q is not None:
        qa = [np.ascontiguousarray(q.row_ptr, np.int64), np.ascontiguousarray(q.col, np.int32), _doubles(q.val, cplx)]
        keep += qa
        args += [a.ctypes.data for a in qa]
    else:
        args += [None, None, None]
    bits = 0
    for o in outputs:
        bits |= OUTPUTS[o]
    lev = np.zeros(csr.n, np.int32)
    info = np.zeros(7, np.int64)
    cap = max(slot_R, 1) * csr.n + 64  # one row per group at worst
    slots = np.zeros(cap, np.int32) if slot_R > 0 else None
    _check(load().mcinv_debug_levels(*args, bits, lev.ctypes.data, info.ctypes.data, slot_R, slot_L,
                                     None if slots is None else slots.ctypes.data, cap))
    names = ["levels", "max_items", "fused_pairs", "deferred_pairs", "trace_items", "entries", "nslots"]
    d = dict(zip(names, (int(x) for x in info)))
    if slots is not None:
        d["slots"] = slots[:d["nslots"]].copy()
    return lev, d


def debug_blocks(csr, outputs=("diag",), q=None, R: int = 8, W: int = 16, pad_ku: int = 0, ecap: int = 0,
                 wmask: bool = True):
    """Host-only dataflow schedule as staged in the TMA plan blocks (no GPU): (slot
    rows, wait masks); rows -1 = padding, -2 - i = trace item of row i."""
    cplx = np.iscomplexobj(csr.val)
    rp = np.ascontiguousarray(csr.row_ptr, np.int64)
    col = np.ascontiguousarray(csr.col, np.int32)
    val = _doubles(csr.val, cplx)
    args = [C128 if cplx else F64, csr.n, rp.ctypes.data, col.ctypes.data, val.ctypes.data]
    keep = [rp, col, val]
    if q is not None:
        qa = [np.ascontiguousarray(q.row_ptr, np.int64), np.ascontiguousarray(q.col, np.int32), _doubles(q.val, cplx)]
        keep += qa
        args += [a.ctypes.data for a in qa]
    else:
        args += [None, None, None]
    bits = 0
    for o in outputs:
        bits |= OUTPUTS[o]
    cap = (csr.n + (csr.n if q is not None else 0)) * R + 64
    x = np.zeros(cap, np.int32)
    m = np.zeros(cap, np.uint32)
    ns = ctypes.c_int64()
    _check(load().mcinv_debug_blocks(*args, bits, R, W, pad_ku, ecap, int(wmask), x.ctypes.data, m.ctypes.data, cap,
                                     ctypes.byref(ns)))
    return x[:ns.value].copy(), m[:ns.value].copy()


class Inverter:
    """Context for one matrix C (CSR, real f64 or complex c128).

    ``csr`` needs attributes n, row_ptr (int64), col (int32), val. ``q``
    (same form) enables the trace output; ``pattern`` = (rows, cols) selects
    the elements of the PATTERN output (default: the pattern of C).
    """

    def __init__(self, csr, device: int = 0, q=None, pattern: Optional[tuple] = None):
        import torch  # device memory and streams only
        self._torch = torch
        self.device = device
        self.n = int(csr.n)
        self.cplx = np.iscomplexobj(csr.val)
        self.e = 2 if self.cplx else 1
        L = load()
        h = ctypes.c_void_p()
        rp = np.ascontiguousarray(csr.row_ptr, np.int64)
        col = np.ascontiguousarray(csr.col, np.int32)
        val = _doubles(csr.val, self.cplx)
        st = L.mcinv_create(ctypes.byref(h), device, C128 if self.cplx else F64, self.n, rp.ctypes.data,
                            col.ctypes.data, val.ctypes.data)
        self._h = h
        if st:
            try:
                _check(st, h)
            finally:
                L.mcinv_destroy(h)
                self._h = None
        if q is not None:
            qrp = np.ascontiguousarray(q.row_ptr, np.int64)
            qc = np.ascontiguousarray(q.col, np.int32)
            qv = _doubles(q.val, self.cplx)
            _check(L.mcinv_set_trace_q(h, qrp.ctypes.data, qc.ctypes.data, qv.ctypes.data), h)
        if pattern is not None:
            pr = np.ascontiguousarray(pattern[0], np.int32)
            pc = np.ascontiguousarray(pattern[1], np.int32)
            _check(L.mcinv_set_pattern(h, pr.size, pr.ctypes.data, pc.ctypes.data), h)
        cnt = ctypes.c_int64()
        _check(L.mcinv_pattern_size(h, ctypes.byref(cnt)), h)
        self.pcount = cnt.value
        self._ws = None
        self._args = None

    # ------------------------------------------------------------------ run
    def _make_args(self, seed, chains, burn_in, cycles, outputs, chain_begin, sweep_begin, group_size, noise,
                   resume, snapshot_sweeps, stream, trace_series=0) -> _RunArgs:
        bits = 0
        for o in outputs:
            bits |= OUTPUTS[o]
        return _RunArgs(seed & 0xFFFFFFFFFFFFFFFF, chain_begin, chains, burn_in, cycles, sweep_begin, bits,
                        NOISE[noise], group_size, int(resume), snapshot_sweeps, None, 0, stream, trace_series)

    def workspace_size(self, **kw) -> int:
        a = self._make_args(**self._defaults(kw))
        b = ctypes.c_size_t()
        _check(load().mcinv_workspace_size(self._h, ctypes.byref(a), ctypes.byref(b)), self._h)
        return b.value

    @staticmethod
    def _defaults(kw):
        d = dict(seed=0, chains=32, burn_in=0, cycles=1, outputs=("diag",), chain_begin=0, sweep_begin=0,
                 group_size=32, noise="gauss", resume=False, snapshot_sweeps=0, stream=None)
        d.update(kw)
        return d

    def run(self, seed: int, chains: int, burn_in: int, cycles: int, outputs: Sequence[str] = ("diag",),
            chain_begin: int = 0, sweep_begin: int = 0, group_size: int = 32, noise: str = "gauss",
            resume: bool = False, snapshot_sweeps: int = 0, stream=None, trace_series: int = 0) -> "Inverter":
        """Enqueue one run (Alg. 1, fixed burn-in) on ``stream`` (torch stream or
        None = current). Returns self; read results with ``result``. trace_series > 0
        (with "trace") keeps the per-sweep realized traces for ``geyer``."""
        torch = self._torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        a = self._make_args(seed, chains, burn_in, cycles, tuple(outputs), chain_begin, sweep_begin, group_size,
                            noise, resume, snapshot_sweeps, sp, trace_series)
        b = ctypes.c_size_t()
        _check(load().mcinv_workspace_size(self._h, ctypes.byref(a), ctypes.byref(b)), self._h)
        need = max(int(b.value), 256)
        if self._ws is None or self._ws.numel() < need:
            if resume:
                raise MCInvError(8, "resume needs the previous workspace")
            self._ws = None
            self._ws = torch.empty(need, dtype=torch.uint8, device=f"cuda:{self.device}")
        a.workspace = self._ws.data_ptr()
        a.workspace_bytes = self._ws.numel()
        _check(load().mcinv_run(self._h, ctypes.byref(a)), self._h)
        self._args = a
        self.outputs = tuple(outputs)
        self.chains = chains
        self.cycles = cycles
        self.acc_cycles = (getattr(self, "acc_cycles", 0) + cycles) if resume else cycles
        self.group_size = group_size
        return self

    def coupled_burn_in(self, tol: float, max_sweeps: int = 100000, stream=None):
        """Coupled burn-in of Alg. 1 (mcinv_coupled_burn_in): (sweeps, final max difference).
        Replaces the last-run state (call before run)."""
        torch = self._torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        n = ctypes.c_int64()
        d = ctypes.c_double()
        _check(load().mcinv_coupled_burn_in(self._h, tol, max_sweeps, sp, ctypes.byref(n), ctypes.byref(d)), self._h)
        self._ws = None
        return n.value, d.value

    def run_until(self, seed: int, chains: int, burn_in: int, outputs: Sequence[str], target: str, rel_se: float,
                  check_cycles: int = 100, max_cycles: int = 100000, group_size: int = 32, chain_begin: int = 0,
                  noise: str = "gauss", stream=None):
        """Adaptive stopping (mcinv_run_until): sampling sweeps in blocks of check_cycles until
        the relative SE of output `target` is below rel_se. Returns (cycles run, relative SE)."""
        torch = self._torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        a = self._make_args(seed, chains, burn_in, check_cycles, tuple(outputs), chain_begin, 0, group_size, noise,
                            False, 0, sp)
        b = ctypes.c_size_t()
        _check(load().mcinv_workspace_size(self._h, ctypes.byref(a), ctypes.byref(b)), self._h)
        need = max(int(b.value), 256)
        if self._ws is None or self._ws.numel() < need:
            self._ws = None
            self._ws = torch.empty(need, dtype=torch.uint8, device=f"cuda:{self.device}")
        a.workspace = self._ws.data_ptr()
        a.workspace_bytes = self._ws.numel()
        done = ctypes.c_int64()
        rse = ctypes.c_double()
        _check(load().mcinv_run_until(self._h, ctypes.byref(a), OUTPUTS[target], rel_se, check_cycles, max_cycles,
                                      ctypes.byref(done), ctypes.byref(rse)), self._h)
        self._args = a
        self.outputs = tuple(outputs)
        self.chains = chains
        self.cycles = self.acc_cycles = done.value
        self.group_size = group_size
        return done.value, rse.value

    def geyer(self) -> dict:
        """mcinv_geyer: Geyer's effective length of the trace series; per
        component (re, im): series mean, gamma_0, sigma2, ess; plus the trace estimate
        and its Geyer standard error."""
        out = np.zeros(8)
        _check(load().mcinv_geyer(self._h, out.ctypes.data), self._h)
        m = self.acc_cycles
        comps = []
        for c in range(self.e):
            mean, g0, s2, ess = out[4 * c:4 * c + 4]
            comps.append(dict(mean=mean, gamma0=g0, sigma2=s2, ess=ess,
                              se=np.sqrt(s2 / m) / self.chains if s2 > 0 else 0.0, estimate=mean / self.chains))
        return dict(re=comps[0], im=comps[1] if self.e == 2 else None)

    def run_until_geyer(self, seed: int, chains: int, burn_in: int, outputs: Sequence[str], rel_se: float,
                        check_cycles: int = 100, max_cycles: int = 100000, group_size: int = 32,
                        chain_begin: int = 0, noise: str = "gauss", stream=None):
        """The paper's stopping rule (mcinv_run_until_geyer): blocks of check_cycles
        sampling sweeps until the trace's Geyer relative SE is below rel_se. Returns
        (cycles run, relative SE)."""
        torch = self._torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else stream
        a = self._make_args(seed, chains, burn_in, check_cycles, tuple(outputs), chain_begin, 0, group_size, noise,
                            False, 0, sp, max_cycles)
        b = ctypes.c_size_t()
        _check(load().mcinv_workspace_size(self._h, ctypes.byref(a), ctypes.byref(b)), self._h)
        need = max(int(b.value), 256)
        if self._ws is None or self._ws.numel() < need:
            self._ws = None
            self._ws = torch.empty(need, dtype=torch.uint8, device=f"cuda:{self.device}")
        a.workspace = self._ws.data_ptr()
        a.workspace_bytes = self._ws.numel()
        done = ctypes.c_int64()
        rse = ctypes.c_double()
        _check(load().mcinv_run_until_geyer(self._h, ctypes.byref(a), rel_se, check_cycles, max_cycles,
                                            ctypes.byref(done), ctypes.byref(rse)), self._h)
        self._args = a
        self.outputs = tuple(outputs)
        self.chains = chains
        self.cycles = self.acc_cycles = done.value
        self.group_size = group_size
        return done.value, rse.value

    def accumulators(self):
        """Device moment vector (torch float64 view) for an all-reduce."""
        p = ctypes.c_void_p()
        cnt = ctypes.c_size_t()
        _check(load().mcinv_accumulators(self._h, ctypes.byref(p), ctypes.byref(cnt)), self._h)
        off = p.value - self._ws.data_ptr()
        return self._ws[off:off + 8 * cnt.value].view(self._torch.float64)

    def recenter(self, total_chains: int):
        """mcinv_recenter: after an all-reduce of accumulators(), recompute this rank's M2
        block about the global mean; returns that block (torch view) for the second
        all-reduce."""
        off, cnt = ctypes.c_size_t(), ctypes.c_size_t()
        _check(load().mcinv_recenter(self._h, total_chains, ctypes.byref(off), ctypes.byref(cnt)), self._h)
        acc = self.accumulators()
        return acc[off.value:off.value + cnt.value]

    def run_status(self) -> int:
        """mcinv_run_status: synchronize and raise on divergence / watchdog; returns the
        divergence count (0)."""
        d = ctypes.c_int64()
        _check(load().mcinv_run_status(self._h, ctypes.byref(d)), self._h)
        return d.value

    def group_sums(self, output: str, group_begin: int = 0, groups: Optional[int] = None) -> np.ndarray:
        """Per-group accumulator sums of one output (test instrumentation)."""
        G = self.chains // self.group_size
        groups = G - group_begin if groups is None else groups
        comps = self.count(output) * self.e
        out = np.zeros((groups, comps))
        _check(load().mcinv_debug_group_sums(self._h, OUTPUTS[output], group_begin, groups, out.ctypes.data),
               self._h)
        return out.view(np.complex128) if self.cplx else out

    def count(self, output: str) -> int:
        return {"diag": self.n, "pattern": self.pcount, "full": self.n * self.n, "trace": 1}[output]

    def result(self, output: str, total_chains: Optional[int] = None, on_device: bool = False):
        """(estimate, std_error) of one output: numpy arrays (complex for
        c128), or torch float64 device tensors (interleaved) with on_device."""
        total = self.chains if total_chains is None else total_chains
        comps = self.count(output) * self.e
        L = load()
        if on_device:
            torch = self._torch
            est = torch.empty(comps, dtype=torch.float64, device=f"cuda:{self.device}")
            se = torch.empty(comps, dtype=torch.float64, device=f"cuda:{self.device}")
            _check(L.mcinv_result(self._h, OUTPUTS[output], total, est.data_ptr(), se.data_ptr(), comps, 1), self._h)
            return est, se
        est = np.zeros(comps)
        se = np.zeros(comps)
        _check(L.mcinv_result(self._h, OUTPUTS[output], total, est.ctypes.data, se.ctypes.data, comps, 0), self._h)
        if self.cplx:
            est = est.view(np.complex128)
            se = se.view(np.complex128)
        shape = (self.n, self.n) if output == "full" else ((self.count(output),) if output != "trace" else ())
        return est.reshape(shape), se.reshape(shape)

    def kernel_info(self) -> dict:
        v, c = ctypes.c_int(), ctypes.c_int()
        st = ctypes.c_int64()
        _check(load().mcinv_kernel_info(self._h, ctypes.byref(v), ctypes.byref(c), ctypes.byref(st)), self._h)
        return dict(version=v.value, chains_per_warp=c.value, steps_per_sweep=st.value)

    def launch_config(self) -> dict:
        t, k, b = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(load().mcinv_launch_config(self._h, ctypes.byref(t), ctypes.byref(k), ctypes.byref(b)), self._h)
        return dict(threads=t.value, chains_per_thread=k.value, blocks=b.value)

    def set_timing(self, enable: bool = True):
        _check(load().mcinv_set_timing(self._h, int(enable)), self._h)

    def stats(self) -> dict:
        """Kernel launches and K1/K3 device time since the last call."""
        la, sl, cl = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        sm, cm = ctypes.c_double(), ctypes.c_double()
        _check(load().mcinv_stats(self._h, ctypes.byref(la), ctypes.byref(sm), ctypes.byref(sl), ctypes.byref(cm),
                                  ctypes.byref(cl)), self._h)
        return dict(launches=la.value, sweep_ms=sm.value, sweep_launches=sl.value, contract_ms=cm.value,
                    contract_launches=cl.value)

    def get_state(self, chain_begin: int = 0, chains: Optional[int] = None):
        ch = self.chains - chain_begin if chains is None else chains
        dt = np.complex128 if self.cplx else np.float64
        z = np.zeros((ch, self.n), dt)
        w = np.zeros((ch, self.n), dt)
        _check(load().mcinv_debug_get_state(self._h, chain_begin, ch, z.ctypes.data, w.ctypes.data), self._h)
        return z, w

    def set_state(self, z, w, chain_begin: int = 0):
        dt = np.complex128 if self.cplx else np.float64
        z = np.ascontiguousarray(z, dt)
        w = np.ascontiguousarray(w, dt)
        _check(load().mcinv_debug_set_state(self._h, chain_begin, z.shape[0], z.ctypes.data, w.ctypes.data),
               self._h)

    def close(self):
        if getattr(self, "_h", None):
            load().mcinv_destroy(self._h)
            self._h = None
        self._ws = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
