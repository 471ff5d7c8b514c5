"""CPU check of the v2 step planner (plan.cu) without a GPU.

``mcinv_debug_plan`` returns the record tiles the sweep2 kernel consumes. This
test executes them with a numpy model of the kernel's data flow -- the warp
roles A (update), B (gathers), D (accumulation, reading values in place)
advancing under the kernel's mbarrier rules in two extreme interleavings, the
result ring, the gather buffer, the partner records -- and compares the
resulting z, w and accumulators with the oracle. A planner bug
(a row scheduled before a lower neighbour, a stale far read, a wrong ring
slot or item partner) shows up as an O(1) mismatch; rounding differences
(no fma in numpy) stay below 1e-12.
"""
import numpy as np
import pytest

import workloads as W

KCAP, PDIST = 8, 7


def ngbuf(esz):
    return 16 if esz == 8 else 8


def r16(x):
    return (x + 15) & ~15


class Tile:
    """Parse one record tile (layout: plan.h TileLayout)."""

    def __init__(self, buf, off, R, esz):
        ct = np.complex128 if esz == 16 else np.float64
        self.K, self.P, _, self.has_q = (int(v) for v in np.frombuffer(buf, np.int32, 4, off))
        rs = np.frombuffer(buf, np.int32, 4 * R, off + 32)
        self.rows, self.flags, self.dslot, self.pslot = rs[:R], rs[R:2 * R], rs[2 * R:3 * R], rs[3 * R:]
        dsq = off + 32 + r16(16 * R)
        v = np.frombuffer(buf, ct, 3 * R, dsq)
        self.delta, self.sigma, self.qself = v[:R], v[R:2 * R], v[2 * R:]
        meta = dsq + r16(3 * R * esz)
        self.meta = np.frombuffer(buf, np.int32, 2 * self.K * R, meta).reshape(self.K, R, 2)
        coef = meta + r16(8 * self.K * R)
        self.coef = np.frombuffer(buf, ct, 2 * self.K * R, coef).reshape(self.K, R, 2)
        part = coef + r16(2 * esz * self.K * R)
        pb = 16 + 2 * esz
        raw = np.frombuffer(buf, np.uint8, pb * self.P * R, part).reshape(self.P, R, pb)
        ints = raw[:, :, :16].copy().view(np.int32)
        self.voff, self.pzi, self.pzo = ints[:, :, 0], ints[:, :, 1], ints[:, :, 2]
        qq = raw[:, :, 16:].copy().view(ct)
        self.qr, self.qc = qq[:, :, 0], qq[:, :, 1]
        self.size = part + r16(pb * self.P * R) - off


def emulate(M, orc, c, C, outputs, q=None, pattern=None, seed=5, chain0=0, burn_in=2, cycles=3, lazy_d=False):
    """Numpy model of sweep2_kernel's data flow for one CTA (C chains).

    Warp roles progress under the kernel's barrier rules: A(T) after B(T);
    B(U) after A(U-8) and D(U-NGBUF+1); D(T) after A(T), reading values in
    place. ``lazy_d``: earliest producer, maximally lagging D."""
    R = 32 // C
    cplx = np.iscomplexobj(c.val)
    esz = 16 if cplx else 8
    buf, info = M.debug_plan(c, C, outputs, q=q, pattern=pattern)
    buf = buf.tobytes()
    S = info["steps"]
    tiles, off = [], 0
    for t in range(S):
        tl = Tile(buf, off, R, esz)
        tiles.append(tl)
        off += tl.size
    assert off == len(buf)
    n = c.n
    ct = np.complex128
    zb = 2 * esz                 # bytes of one (z, w) pair
    BLK = 32 * zb
    NGBUF = ngbuf(esz)
    NRING = 2 * NGBUF
    nslot = (NRING + NGBUF * KCAP + 1) * BLK // zb
    vz = np.zeros(nslot, ct)     # value area, indexed by byte offset / zb
    vw = np.zeros(nslot, ct)
    st_z = np.zeros((n, C), ct)
    st_w = np.zeros((n, C), ct)
    npat = len(pattern[0]) if pattern is not None else c.nnz
    diag = np.zeros((C, n), ct)
    pat = np.zeros((C, npat), ct)
    trace = np.zeros(C, ct)
    total = (burn_in + cycles) * S

    def ring_base(T, r):
        return ((T % NRING) * BLK + r * C * zb) // zb

    for qq in range(1, PDIST + 1):  # prologue: ring of the 7 steps before T0 = 0
        tl = tiles[(-qq) % S]
        for r in range(R):
            if tl.rows[r] >= 0 and tl.flags[r] & 2:
                b = ring_base(-qq, r)
                vz[b:b + C] = st_z[tl.rows[r]]
                vw[b:b + C] = st_w[tl.rows[r]]

    acc_z = np.zeros((R, C), ct)
    acc_w = np.zeros((R, C), ct)

    def B(U):
        tl = tiles[U % S]
        for k in range(tl.K):
            for r in range(R):
                o, j = tl.meta[k, r]
                if j >= 0:
                    vz[o // zb:o // zb + C] = st_z[j]
                    vw[o // zb:o // zb + C] = st_w[j]

    def A(T):
        tl = tiles[T % S]
        for r in range(R):
            if tl.flags[r] & 1:
                acc_z[r] = 0
                acc_w[r] = 0
            for k in range(tl.K):
                b = tl.meta[k, r, 0] // zb
                a_, b_ = tl.coef[k, r]
                acc_z[r] = acc_z[r] + a_ * vz[b:b + C]
                acc_w[r] = acc_w[r] + b_ * vw[b:b + C]
            if tl.flags[r] & 2:
                i = tl.rows[r]
                phi = np.array([orc.gaussian(seed, int(i), T // S, chain0 + ch) for ch in range(C)])
                d, sg = tl.delta[r], tl.sigma[r]
                zi = -d * acc_z[r] + sg * phi
                wi = -np.conj(d) * acc_w[r] + np.conj(sg) * phi
                st_z[i] = zi
                st_w[i] = wi
                b = ring_base(T, r)
                vz[b:b + C] = zi
                vw[b:b + C] = wi

    def D(T):
        nonlocal trace
        if T // S < burn_in:
            return
        tl = tiles[T % S]
        for r in range(R):
            if not tl.flags[r] & 2:
                continue
            b = ring_base(T, r)
            zi, wi = vz[b:b + C].copy(), vw[b:b + C].copy()
            if tl.dslot[r] >= 0:
                diag[:, tl.dslot[r]] += zi * np.conj(wi)
            if tl.pslot[r] >= 0:
                pat[:, tl.pslot[r]] += zi * np.conj(wi)
            qz = tl.qself[r] * zi
            qw = np.zeros(C, ct)
            for q_ in range(tl.P):
                pb = tl.voff[q_, r] // zb
                pz, pw = vz[pb:pb + C], vw[pb:pb + C]
                if tl.pzi[q_, r] >= 0:
                    pat[:, tl.pzi[q_, r]] += zi * np.conj(pw)
                if tl.pzo[q_, r] >= 0:
                    pat[:, tl.pzo[q_, r]] += pz * np.conj(wi)
                qz = qz + tl.qr[q_, r] * pz
                qw = qw + tl.qc[q_, r] * np.conj(pw)
            trace += qz * np.conj(wi) + zi * qw

    # A(T) needs B(T); B(U) needs A(U-8) and, once sampling, D(U-NGBUF+1);
    # D(T) needs A(T). Mode ``lazy_d``: priority B > A > D (earliest producer,
    # maximally lagging D); otherwise D > A > B (producer just in time).
    Ts = burn_in * S
    a = b = d = -1

    def can_b():
        U = b + 1
        return U < total and U - 8 <= a and (U - NGBUF + 1 < Ts or U - NGBUF + 1 <= d)

    while d < total - 1:
        order = "BAD" if lazy_d else "DAB"
        for role in order:
            if role == "B" and can_b():
                b += 1
                B(b)
                break
            if role == "A" and a + 1 <= b:
                a += 1
                A(a)
                break
            if role == "D" and d + 1 <= a:
                d += 1
                D(d)
                break
        else:
            raise AssertionError("deadlock in the emulated schedule")
    return st_z.T, st_w.T, diag, pat, trace


def _check(M, orc, c, C, outputs, q=None, pattern=None, burn_in=2, cycles=3):
    for lazy in (False, True):
        _check1(M, orc, c, C, outputs, q, pattern, burn_in, cycles, lazy)


def _check1(M, orc, c, C, outputs, q, pattern, burn_in, cycles, lazy):
    zg, wg, dg, pg, tg = emulate(M, orc, c, C, outputs, q=q, pattern=pattern, burn_in=burn_in, cycles=cycles,
                                 lazy_d=lazy)
    pat_o = pattern if pattern is not None else (np.repeat(np.arange(c.n), np.diff(c.row_ptr)).astype(np.int32),
                                                 c.col)
    r = orc.Matrix(c, q=q, pattern=pat_o).run(5, C, burn_in, cycles, outputs)

    def nw(a, b):
        return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)

    assert nw(zg, r["z"]) < 1e-12 and nw(wg, r["w"]) < 1e-12
    if "diag" in outputs:
        assert nw(dg, r["diag"]) < 1e-12
    if "pattern" in outputs:
        assert nw(pg, r["pattern"]) < 1e-12
    if "trace" in outputs:
        assert nw(tg, r["trace"]) < 1e-12


@pytest.mark.parametrize("C", [8, 16, 32])
def test_plan_pedigree(orc, C):
    import paper_cs_0412107_b200 as M
    _check(M, orc, W.pedigree(200, seed=3), C, ("diag", "pattern"))


@pytest.mark.parametrize("C", [8, 32])
def test_plan_lattice_trace(orc, C):
    import paper_cs_0412107_b200 as M
    c = W.lattice(3, 4, 0.1, seed=4)
    q = W.random_q(c.n, 7, 4)
    _check(M, orc, c, C, ("diag", "trace"), q=q)


def test_plan_long_rows_and_custom_pattern(orc):
    """Dense rows (8 segments), a custom pattern with non-neighbour partners."""
    import paper_cs_0412107_b200 as M
    c = W.random_dense(20, seed=6, complex_=True, ratio=0.6)
    rows = np.array([3, 0, 19, 7, 11, 11], np.int32)
    cols = np.array([17, 0, 2, 7, 4, 12], np.int32)
    _check(M, orc, c, 8, ("diag", "pattern"), pattern=(rows, cols))


def test_plan_nonsymmetric_structure(orc):
    import paper_cs_0412107_b200 as M
    a = np.triu(W.random_dense(25, seed=14, ratio=0.5, density=0.4).to_dense())
    a[np.arange(1, 25), np.arange(24)] = -0.1
    _check(M, orc, W.CSR.from_dense(a), 16, ("diag", "pattern"))


def test_plan_wrap_dependencies(orc):
    """2-D periodic lattice: row 0 reads the previous sweep's row n-1 at step
    distance 1 (near ring across the sweep boundary)."""
    import paper_cs_0412107_b200 as M
    _check(M, orc, W.lattice(5, 2, 0.2, seed=2), 8, ("diag",), burn_in=1, cycles=3)


def test_plan_schedule_stats():
    """Row-level parallelism found by the planner on the BASELINE configs."""
    import paper_cs_0412107_b200 as M
    c, _, run = W.config(2)
    _, info = M.debug_plan(c, 8, run.outputs)
    assert info["steps"] < 1.4 * c.n / 4          # ~4 rows per step (pedigree: random parents)
    c3, _, run3 = W.config(3)
    _, info3 = M.debug_plan(c3, 8, ("diag",))
    assert info3["steps"] < 1.1 * c3.n / 4        # lattice anti-diagonals
