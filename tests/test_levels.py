"""CPU tests of the v3 level schedule (paper_cs_0412107_b200/csrc/levels.cu).

The sweep of Eq. (4)/(5) reads new values of lower
neighbours and old values of upper neighbours; running rows level by level,
lev(i) = 1 + max lev(lower neighbours), reproduces exactly those operands
(DESIGN.md "Level schedule"). These tests pin the planner against an
independent pure-Python longest-path computation and check the invariants
the kernel relies on. No GPU needed (mcinv_debug_levels is host-only).
"""
import numpy as np
import pytest

import workloads as W


@pytest.fixture(scope="module")
def mc():
    import paper_cs_0412107_b200 as M
    M.load()
    return M


def neighbours(c):
    """Undirected neighbour sets of the off-diagonal pattern of C and C^T."""
    nb = [set() for _ in range(c.n)]
    for i in range(c.n):
        for e in range(c.row_ptr[i], c.row_ptr[i + 1]):
            j = int(c.col[e])
            if j != i:
                nb[i].add(j)
                nb[j].add(i)
    return nb


def brute_levels(c):
    """Longest path in the DAG j -> i (j < i neighbours), by repeated
    relaxation until a fixed point (Bellman-Ford style; independent of the
    planner's single ascending pass)."""
    nb = neighbours(c)
    lev = [0] * c.n
    changed = True
    while changed:
        changed = False
        for i in range(c.n):
            want = max([lev[j] + 1 for j in nb[i] if j < i], default=0)
            if want != lev[i]:
                lev[i] = want
                changed = True
    return np.array(lev)


@pytest.mark.parametrize("make", [
    lambda: W.pedigree(400, seed=3),
    lambda: W.lattice(6, 2, 0.2, seed=4),
    lambda: W.lattice(3, 4, 0.1, seed=5),
    lambda: W.dense_config1(24, seed=6),
    lambda: W.diagonal(np.arange(1.0, 9.0)),
])
def test_levels_match_longest_path(mc, make):
    c = make()
    lev, info = mc.debug_levels(c)
    ref = brute_levels(c)
    assert np.array_equal(lev, ref)
    assert info["levels"] == (ref.max() + 1)
    # the schedule respects every ordering constraint of the sequential sweep
    nb = neighbours(c)
    for i in range(c.n):
        for j in nb[i]:
            if j < i:
                assert lev[j] < lev[i]


def test_dense_is_fully_sequential(mc):
    """A dense C (config 1) admits no reordering: n levels of one row."""
    c = W.dense_config1(16, seed=7)
    lev, info = mc.debug_levels(c)
    assert np.array_equal(lev, np.arange(16)) and info["levels"] == 16


def test_diagonal_is_one_level(mc):
    """Diagonal C: rows are independent, one level."""
    lev, info = mc.debug_levels(W.diagonal([2.0, 4.0, 1.0]))
    assert info["levels"] == 1 and not lev.any()


def test_lattice_depth_closed_form(mc):
    """Periodic L^d lattice, x0 fastest: the longest increasing neighbour path
    walks each coordinate from 0 to L-1, d(L-1)+1 levels (config 3: 127,
    config 5: 61)."""
    for L, d in ((8, 2), (4, 3), (5, 2)):
        c = W.lattice(L, d, 0.1, seed=8)
        _, info = mc.debug_levels(c)
        assert info["levels"] == d * (L - 1) + 1


def test_pattern_pairs_all_assigned(mc):
    """Default pattern (the pattern of C): every element is fused into an
    update (diagonal or lower-neighbour pair), none deferred."""
    c = W.pedigree(300, seed=9)
    _, info = mc.debug_levels(c, outputs=("pattern",))
    assert info["fused_pairs"] == c.nnz and info["deferred_pairs"] == 0


def test_trace_items(mc):
    """One deferred trace item per non-empty row of Q."""
    c = W.lattice(4, 2, 0.2, seed=10)
    q = W.random_q(c.n, 11, 3)
    _, info = mc.debug_levels(c, outputs=("trace",), q=q)
    assert info["trace_items"] == int(np.sum(np.diff(q.row_ptr) > 0))
    assert info["levels"] == 2 * 3 + 1


@pytest.mark.parametrize("make,R,L", [
    (lambda: W.pedigree(600, seed=13), 4, 32),
    (lambda: W.pedigree(600, seed=13), 1, 8),
    (lambda: W.lattice(8, 2, 0.2, seed=14), 2, 16),
    (lambda: W.lattice(4, 3, 0.2, seed=15), 8, 4),
    (lambda: W.dense_config1(20, seed=16), 32, 1),
])
def test_v4_slot_schedule(mc, make, R, L):
    """The v4 slot schedule (levels.cu schedule_slots) is what the dataflow
    kernel's correctness and deadlock-freedom rest on: every row
    appears exactly once, the slots come in whole warp groups of R, every
    lower neighbour of a row sits in an EARLIER group (never the same one:
    rows of a group run concurrently), and rows are placed at least L groups
    after their lower neighbours whenever the schedule does not pad."""
    c = make()
    _, info = mc.debug_levels(c, slot_R=R, slot_L=L)
    slots = info["slots"]
    assert slots.size % R == 0
    rows = slots[slots >= 0]
    assert np.array_equal(np.sort(rows), np.arange(c.n))
    group = np.empty(c.n, np.int64)
    group[slots[slots >= 0]] = np.nonzero(slots >= 0)[0] // R
    nb = neighbours(c)
    for i in range(c.n):
        for j in nb[i]:
            if j < i:
                assert group[j] < group[i]
    # every group holds at least one row (padding only completes groups)
    assert slots.size <= R * c.n
    assert np.all((slots.reshape(-1, R) >= 0).any(axis=1))


def test_arrow_row_with_many_lower_neighbours(mc):
    """A row with more than 32767 lower neighbours (an arrow matrix: the last
    row and column couple to every earlier row). Its record packs the lower
    count in the upper 16 bits; decoded as unsigned, the planner still places
    every row exactly once and the arrow row after all of them (a signed
    decode would make the count negative: the row never becomes ready)."""
    n = 40001
    rows = np.concatenate([np.arange(n), np.full(n - 1, n - 1), np.arange(n - 1)])
    cols = np.concatenate([np.arange(n), np.arange(n - 1), np.full(n - 1, n - 1)])
    vals = np.concatenate([np.full(n, 4.0), np.full(n - 1, -1e-5), np.full(n - 1, -2e-5)])
    order = np.lexsort((cols, rows))
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    c = W.CSR(n, np.cumsum(rp), cols[order].astype(np.int32), vals[order])
    lev, info = mc.debug_levels(c, slot_R=4, slot_L=8)
    assert info["levels"] == 2 and lev[-1] == 1 and not lev[:-1].any()
    slots = info["slots"]
    placed = slots[slots >= 0]
    assert np.array_equal(np.sort(placed), np.arange(n))
    assert np.nonzero(slots == n - 1)[0][0] // 4 > np.max(np.nonzero((slots >= 0) & (slots < n - 1))[0]) // 4


def _lower_lists(c):
    nb = neighbours(c)
    return [sorted(j for j in nb[i] if j < i) for i in range(c.n)]


@pytest.mark.parametrize("make,R,W", [
    (lambda: W.pedigree(600, seed=13), 8, 16),      # v6 on config 2's recipe (C = 8)
    (lambda: W.pedigree(900, seed=17), 4, 8),
    (lambda: W.lattice(8, 2, 0.2, seed=14), 2, 24),
    (lambda: W.dense_config1(40, seed=16), 8, 16),  # every row depends on all earlier ones
])
def test_v6_wait_masks_cover_every_lower_neighbour(mc, make, R, W):
    """The dataflow kernels' correctness rests on every lower neighbour j of a
    row i being final when i runs. v6 waits only on the
    neighbours in the host's wait mask; the others must be implied. Replay the
    schedule: Guar(i) = the rows certainly complete once i's waits succeed =
    for each waited j: {j} + Guar(j) (completion is transitive through the
    counters' release/acquire), plus the rows of the previous group of the same
    warp and their Guar (program order). Every lower neighbour must be in it."""
    c = make()
    x, m = mc.debug_blocks(c, ("diag", "pattern"), R=R, W=W)
    low = _lower_lists(c)
    assert np.array_equal(np.sort(x[x >= 0]), np.arange(c.n))
    guar = {}
    last_of_warp = {}
    ngroups = x.size // R
    dropped = 0
    for g in range(ngroups):
        rows = [(int(x[g * R + r]), int(m[g * R + r])) for r in range(R) if x[g * R + r] >= 0]
        prev = last_of_warp.get(g % W, [])
        for i, mask in rows:
            G = set()
            for p in prev:
                G |= {p} | guar[p]
            for e, j in enumerate(low[i]):
                if e >= 32 or (mask >> e) & 1:
                    assert j in guar, f"row {i} waits on {j}, not scheduled earlier"
                    G |= {j} | guar[j]
            for e, j in enumerate(low[i]):
                assert j in G, f"row {i}: lower neighbour {j} neither waited for nor implied"
                if e < 32 and not (mask >> e) & 1:
                    dropped += 1
            guar[i] = G
        last_of_warp[g % W] = [i for i, _ in rows]
    assert len(guar) == c.n
    if R == 8 and c.n == 600:
        assert dropped > 0  # the pedigree's linked parents: one wait per row implied


def test_v5_trace_items_are_scheduled_after_their_rows(mc):
    """v5's trace items (conj(w_i) sum_j Q_ij z_j) enter the schedule after
    rows i and j of Q's row i: every trace item's slot group is
    later than the groups of all those rows, and every row and item appears once."""
    c = W.lattice(4, 3, 0.15, seed=81)
    q = W.random_q(c.n, 82, 4)
    R = 2
    x, _ = mc.debug_blocks(c, ("diag", "trace"), q=q, R=R, W=24, wmask=False)
    grp = np.arange(x.size) // R
    row_grp = {int(v): int(gg) for v, gg in zip(x, grp) if v >= 0}
    assert sorted(row_grp) == list(range(c.n))
    items = [(-2 - int(v), int(gg)) for v, gg in zip(x, grp) if v <= -2]
    assert sorted(i for i, _ in items) == list(range(c.n))
    for i, gg in items:
        deps = {i} | set(int(j) for j in q.col[q.row_ptr[i]:q.row_ptr[i + 1]])
        assert all(row_grp[j] < gg for j in deps), i
