"""CPU check of the v2 step planner (plan.cu) without a GPU.

``mcinv_debug_plan`` returns the record tiles the sweep2 kernel consumes. This
test executes them with a numpy model of the kernel's data flow -- the same
prefetch timing (gathers for step T+7 read the HBM state at iteration T),
the 8-step ring of recent results, the gather buffer, the items -- and
compares the resulting z, w and accumulators with the oracle. A planner bug
(a row scheduled before a lower neighbour, a stale far read, a wrong ring
slot or item partner) shows up as an O(1) mismatch; rounding differences
(no fma in numpy) stay below 1e-12.
"""
import numpy as np
import pytest

import workloads as W

KCAP, PDIST, NRING = 8, 7, 8


def r16(x):
    return (x + 15) & ~15


class Tile:
    def __init__(self, buf, off, R, esz):
        self.K, self.I = (int(v) for v in np.frombuffer(buf, np.int32, 2, off))
        self.rows = np.frombuffer(buf, np.int32, R, off + 32)
        self.flags = np.frombuffer(buf, np.int32, R, off + 32 + 4 * R)
        dsig = off + 32 + r16(8 * R)
        ct = np.complex128 if esz == 16 else np.float64
        self.delta = np.frombuffer(buf, ct, R, dsig)
        self.sigma = np.frombuffer(buf, ct, R, dsig + R * esz)
        meta = dsig + r16(2 * R * esz)
        self.meta = np.frombuffer(buf, np.int32, 2 * self.K * R, meta).reshape(self.K, R, 2)
        coef = meta + r16(8 * self.K * R)
        self.coef = np.frombuffer(buf, ct, 2 * self.K * R, coef).reshape(self.K, R, 2)
        items = coef + r16(2 * esz * self.K * R)
        raw = np.frombuffer(buf, np.uint8, 32 * self.I * R, items).reshape(self.I, R, 32)
        self.icode = raw[:, :, 0:4].copy().view(np.int32)[:, :, 0]
        self.islot = raw[:, :, 4:8].copy().view(np.int32)[:, :, 0]
        self.iprow = raw[:, :, 8:12].copy().view(np.int32)[:, :, 0]
        self.ivoff = raw[:, :, 12:16].copy().view(np.int32)[:, :, 0]
        self.iq = raw[:, :, 16:16 + esz].copy().view(ct)[:, :, 0]
        self.size = items + r16(32 * self.I * R) - off


def emulate(M, orc, c, C, outputs, q=None, pattern=None, seed=5, chain0=0, burn_in=2, cycles=3, gs=None):
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
    BLK = R * C  # elements per block (z and w kept as separate arrays)
    zbytes = 2 * esz
    GB = NRING * 32 * zbytes
    ZERO = GB + NRING * KCAP * 32 * zbytes
    # value area modelled as a flat array of (z, w) pairs indexed by byte offset / zbytes
    nslots = (ZERO + 32 * zbytes) // zbytes
    vz = np.zeros(nslots, ct)
    vw = np.zeros(nslots, ct)
    st_z = np.zeros((n, C), ct)
    st_w = np.zeros((n, C), ct)
    gs = gs or C
    chains = np.arange(C)
    diag = np.zeros((C, n), ct)
    npat = len(pattern[0]) if pattern is not None else c.nnz
    pat = np.zeros((C, npat), ct)
    trace = np.zeros(C, ct)
    total = burn_in + cycles

    def gather(T):
        tl = tiles[T % S]
        for k in range(tl.K):
            for r in range(R):
                o, j = tl.meta[k, r]
                if j >= 0:
                    base = o // zbytes
                    vz[base:base + C] = st_z[j]
                    vw[base:base + C] = st_w[j]

    for qq in range(1, PDIST + 1):  # prologue ring
        T = -qq
        tl = tiles[T % S]
        for r in range(R):
            if tl.rows[r] >= 0 and tl.flags[r] & 2:
                base = ((T % NRING) * 32 * zbytes + r * C * zbytes) // zbytes
                vz[base:base + C] = st_z[tl.rows[r]]
                vw[base:base + C] = st_w[tl.rows[r]]
    for T in range(min(PDIST, total * S)):
        gather(T)
    acc_z = np.zeros((R, C), ct)
    acc_w = np.zeros((R, C), ct)
    for T in range(total * S):
        if T + PDIST < total * S:
            gather(T + PDIST)
        tl = tiles[T % S]
        s_loc = T // S
        zi = np.zeros((R, C), ct)
        wi = np.zeros((R, C), ct)
        for r in range(R):
            if tl.flags[r] & 1:
                acc_z[r] = 0
                acc_w[r] = 0
            for k in range(tl.K):
                base = (tl.meta[k, r, 0] + r * 0) // zbytes
                a, b = tl.coef[k, r]
                acc_z[r] = acc_z[r] + a * vz[base:base + C]
                acc_w[r] = acc_w[r] + b * vw[base:base + C]
            if tl.flags[r] & 2:
                i = tl.rows[r]
                phi = np.array([orc.gaussian(seed, int(i), s_loc, chain0 + int(ch)) for ch in chains])
                d, sg = tl.delta[r], tl.sigma[r]
                zi[r] = -d * acc_z[r] + sg * phi
                wi[r] = -np.conj(d) * acc_w[r] + np.conj(sg) * phi
                st_z[i] = zi[r]
                st_w[i] = wi[r]
                base = ((T % NRING) * 32 * zbytes + r * C * zbytes) // zbytes
                vz[base:base + C] = zi[r]
                vw[base:base + C] = wi[r]
        if s_loc >= burn_in:
            for r in range(R):
                if not tl.flags[r] & 2:
                    continue
                qz = np.zeros(C, ct)
                qw = np.zeros(C, ct)
                for qi in range(tl.I):
                    op = tl.icode[qi, r] & 7
                    if op == 0:
                        continue
                    if tl.icode[qi, r] & 8:
                        base = tl.ivoff[qi, r] // zbytes
                        pz, pw = vz[base:base + C], vw[base:base + C]
                    elif tl.iprow[qi, r] >= 0:
                        pz, pw = st_z[tl.iprow[qi, r]], st_w[tl.iprow[qi, r]]
                    slot = tl.islot[qi, r]
                    if op in (1, 4):
                        prod = zi[r] * np.conj(wi[r])
                    elif op == 2:
                        prod = zi[r] * np.conj(pw)
                    elif op == 3:
                        prod = pz * np.conj(wi[r])
                    elif op == 5:
                        qz += tl.iq[qi, r] * pz
                        continue
                    elif op == 6:
                        qz += tl.iq[qi, r] * zi[r]
                        continue
                    elif op == 7:
                        qw += tl.iq[qi, r] * np.conj(pw)
                        continue
                    if op == 1:
                        diag[:, slot] += prod
                    else:
                        pat[:, slot] += prod
                trace += qz * np.conj(wi[r]) + zi[r] * qw
    return st_z.T, st_w.T, diag, pat, trace


def _check(M, orc, c, C, outputs, q=None, pattern=None, burn_in=2, cycles=3):
    zg, wg, dg, pg, tg = emulate(M, orc, c, C, outputs, q=q, pattern=pattern, burn_in=burn_in, cycles=cycles)
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
