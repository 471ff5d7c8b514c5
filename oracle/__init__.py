"""Python front end of the C oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg may import this package. The product
path (paper_cs_0412107_b200) never imports it and shares no code with it.

``run`` wraps ``orc_run`` (Eq. 4/5 sweeps, Alg. 1 with fixed burn-in,
PAPER.md:150-182, 377-423) and ``estimate`` turns per-chain sums into the
Eq. (1/C) / Eq. (tr) estimates with a standard error from disjoint chain
groups (reading R15 replaces the paper's Geyer error).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

DIAG, PATTERN, FULL, TRACE = 1, 2, 4, 8
NOISE_GAUSS, NOISE_ZERO, NOISE_ONE, NOISE_Z2 = 0, 1, 2, 3
OUT_BITS = {"diag": DIAG, "pattern": PATTERN, "full": FULL, "trace": TRACE}
ERRORS = {1: "invalid", 2: "zero diagonal", 3: "diagonal domain", 4: "diverged", 5: "no memory"}


class OracleError(RuntimeError):
    def __init__(self, code, detail=None):
        super().__init__(f"oracle error {code} ({ERRORS.get(code, '?')}) {detail or ''}")
        self.code = code
        self.detail = detail


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C99, no fp contraction)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["gcc", "-std=c99", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                               "-Wall", "-o", _SO + ".tmp", src, "-lm"])
        os.replace(_SO + ".tmp", _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        P = ctypes.POINTER
        u32p = P(ctypes.c_uint32)
        L.orc_philox4x32_10.argtypes = [u32p, u32p, u32p]
        L.orc_philox4x32_10.restype = None
        L.orc_gaussian_from_words.argtypes = [u32p]
        L.orc_gaussian_from_words.restype = ctypes.c_double
        L.orc_gaussian_pair_from_words.argtypes = [u32p, P(ctypes.c_double)]
        L.orc_gaussian_pair_from_words.restype = None
        L.orc_gaussian.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]
        L.orc_gaussian.restype = ctypes.c_double
        L.orc_z2.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_uint32]
        L.orc_z2.restype = ctypes.c_double
        L.orc_matrix_build.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_int, P(ctypes.c_void_p), P(ctypes.c_int64)]
        L.orc_matrix_free.argtypes = [ctypes.c_void_p]
        L.orc_set_q.argtypes = [ctypes.c_void_p] * 4
        L.orc_set_pattern.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_geyer.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.orc_geyer.restype = None
        L.orc_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p] + [ctypes.c_void_p] * 9 + \
            [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _lib = L
    return _lib


class _Args(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("chain_begin", ctypes.c_int64), ("chains", ctypes.c_int64),
                ("burn_in", ctypes.c_int64), ("cycles", ctypes.c_int64), ("sweep_begin", ctypes.c_int64),
                ("outputs", ctypes.c_uint), ("noise", ctypes.c_int), ("use_init", ctypes.c_int)]


def _ptr(a):
    return None if a is None else a.ctypes.data


def philox(ctr, key) -> np.ndarray:
    c = (ctypes.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (ctypes.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return np.array(list(o), dtype=np.uint32)


def gaussian_from_words(r) -> float:
    w = (ctypes.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in r])
    return lib().orc_gaussian_from_words(w)


def gaussian_pair_from_words(r):
    w = (ctypes.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in r])
    g = (ctypes.c_double * 2)()
    lib().orc_gaussian_pair_from_words(w, g)
    return g[0], g[1]


def gaussian(seed: int, row: int, sweep: int, chain: int) -> float:
    return lib().orc_gaussian(seed, row, sweep, chain)


def z2(seed: int, row: int, sweep: int, chain: int) -> float:
    return lib().orc_z2(seed, row, sweep, chain)


def _as_doubles(val: np.ndarray, cplx: bool) -> np.ndarray:
    if cplx:
        return np.ascontiguousarray(np.asarray(val, np.complex128)).view(np.float64)
    return np.ascontiguousarray(np.asarray(val, np.float64))


class Matrix:
    """Oracle-side C = L + D + U plus optional Q and pattern."""

    def __init__(self, csr, q=None, pattern: Optional[tuple] = None):
        self.n = csr.n
        self.cplx = csr.dtype == "c128"
        h = ctypes.c_void_p()
        bad = ctypes.c_int64(-1)
        rp = np.ascontiguousarray(csr.row_ptr, np.int64)
        col = np.ascontiguousarray(csr.col, np.int32)
        val = _as_doubles(csr.val, self.cplx)
        st = lib().orc_matrix_build(self.n, rp.ctypes.data, col.ctypes.data, val.ctypes.data,
                                    int(self.cplx), ctypes.byref(h), ctypes.byref(bad))
        if st:
            raise OracleError(st, f"row {bad.value}")
        self.h = h
        self.pcount = 0
        if q is not None:
            qrp = np.ascontiguousarray(q.row_ptr, np.int64)
            qc = np.ascontiguousarray(q.col, np.int32)
            qv = _as_doubles(q.val, self.cplx)
            st = lib().orc_set_q(self.h, qrp.ctypes.data, qc.ctypes.data, qv.ctypes.data)
            if st:
                raise OracleError(st, "Q")
        if pattern is not None:
            pr = np.ascontiguousarray(pattern[0], np.int32)
            pc = np.ascontiguousarray(pattern[1], np.int32)
            st = lib().orc_set_pattern(self.h, pr.size, pr.ctypes.data, pc.ctypes.data)
            if st:
                raise OracleError(st, "pattern")
            self.pcount = pr.size

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.orc_matrix_free(self.h)
            self.h = None

    def run(self, seed: int, chains: int, burn_in: int, cycles: int, outputs: Sequence[str] = (),
            chain_begin: int = 0, sweep_begin: int = 0, noise: int = NOISE_GAUSS,
            z_init=None, w_init=None, snap_sweeps: Sequence[int] = ()):
        """Per-chain sums and states; see oracle.h ``orc_run``."""
        n, ch = self.n, chains
        dt = np.complex128 if self.cplx else np.float64
        bits = 0
        for o in outputs:
            bits |= OUT_BITS[o]
        a = _Args(seed & 0xFFFFFFFFFFFFFFFF, chain_begin, chains, burn_in, cycles, sweep_begin, bits,
                  noise, int(z_init is not None))
        diag = np.zeros((ch, n), dt) if bits & DIAG else None
        pat = np.zeros((ch, self.pcount), dt) if bits & PATTERN else None
        full = np.zeros((ch, n, n), dt) if bits & FULL else None
        trace = np.zeros((ch,), dt) if bits & TRACE else None
        series = np.zeros((max(cycles, 1),), dt) if bits & TRACE else None
        zo = np.zeros((ch, n), dt)
        wo = np.zeros((ch, n), dt)
        snaps = np.asarray(list(snap_sweeps), np.int64)
        zs = np.zeros((snaps.size, ch, n), dt)
        ws = np.zeros((snaps.size, ch, n), dt)
        zi = wi = None
        if z_init is not None:
            zi = np.ascontiguousarray(np.broadcast_to(np.asarray(z_init, dt), (ch, n)))
            wi = np.ascontiguousarray(np.broadcast_to(np.asarray(w_init, dt), (ch, n)))
        fail = np.zeros(2, np.int64)
        st = lib().orc_run(self.h, ctypes.byref(a), _ptr(zi), _ptr(wi), _ptr(diag), _ptr(pat), _ptr(full),
                           _ptr(trace), _ptr(series), zo.ctypes.data, wo.ctypes.data, snaps.size, _ptr(snaps),
                           zs.ctypes.data, ws.ctypes.data, fail.ctypes.data)
        if st:
            raise OracleError(st, f"chain {fail[0]} sweep {fail[1]}")
        return dict(diag=diag, pattern=pat, full=full, trace=trace, z=zo, w=wo, z_snap=zs, w_snap=ws,
                    trace_series=series[:cycles] if series is not None else None)


def estimate(sums: np.ndarray, cycles: int, group_size: int = 1, chain_begin: int = 0):
    """Eq. (1/C) estimate (1/(m (M-N))) sum_c sum_k and its standard
    error from disjoint groups of ``group_size`` consecutive global chain
    indices: SE = sd(group means) / sqrt(G) (reading R15)."""
    m = sums.shape[0]
    assert m % group_size == 0 and chain_begin % group_size == 0
    est = sums.sum(axis=0) / (m * cycles)
    g = sums.reshape((m // group_size, group_size) + sums.shape[1:]).sum(axis=1) / (group_size * cycles)
    G = g.shape[0]
    if G < 2:
        return est, np.full(est.shape, np.nan)
    if np.iscomplexobj(g):
        se = (np.std(g.real, axis=0, ddof=1) + 1j * np.std(g.imag, axis=0, ddof=1)) / np.sqrt(G)
    else:
        se = np.std(g, axis=0, ddof=1) / np.sqrt(G)
    return est, se


def geyer(x) -> dict:
    """Geyer's initial positive sequence estimator (orc_geyer) of a real
    series: mean, gamma_0, sigma2 (= m Var(mean)), effective length, and the
    standard error of the mean sqrt(sigma2 / m) = sqrt(gamma_0 / ESS)."""
    x = np.ascontiguousarray(x, np.float64)
    out = np.zeros(4)
    lib().orc_geyer(x.ctypes.data, x.size, out.ctypes.data)
    return dict(mean=out[0], gamma0=out[1], sigma2=out[2], ess=out[3],
                se=np.sqrt(out[2] / x.size) if out[2] > 0 else 0.0)
