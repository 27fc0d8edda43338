"""Budgets above the 16-bit label range (-m gpu).

PAPER.md:20 takes M in R+ and PAPER.md:27 general integer weights; the fast
16-bit layout holds labels up to WCSP_M_MAX = 65533.  Larger budgets (up to
WCSP_M_MAX_WIDE) switch the solve to 32-bit labels with 64-bit stamped
temporary labels on the sweep engine (include/wcsp.h).  With f2 near the top
of the u8 range (200..255) a face-to-face path of a few hundred edges spends
more than 65533, so these budgets bind.  Bar: (status, F1, F2, X, Y) equal to
oracle tier 2 and the work counters equal to tier 5 (the paper's cycle run
sequentially), exactly as for the 16-bit layout.
"""
import numpy as np
import pytest

import oracle
from paper_1511_06441_b200 import instances as I
from paper_1511_06441_b200 import wcsp

pytestmark = pytest.mark.gpu


def heavy(shape, seed, M=I.M_INF):
    """f1 ~ U{1..10} (times), f2 ~ U{200..255} (weights near the u8 top), faces x0 = 0 -> x0 = n0 - 1."""
    f1, _ = I.grid_values(shape, seed, 1, 10)
    _, f2 = I.grid_values(shape, seed + 7919, 200, 255)
    f2[f1 == 0] = 0
    return I.Instance(tuple(shape), f1, f2, I.set_mask(shape, "face0"), I.set_mask(shape, "face1"), M,
                      None, f"heavy{shape}", seed)


def counters(r):
    return (r.cycles, r.edge_updates, r.arrivals, r.triggered, r.phantoms_created, r.lanes_started, r.relabels)


def budgets(inst):
    lo, hi = oracle.f2_min(inst), oracle.f2_lex(inst)
    assert lo > wcsp.M_MAX, (inst.shape, lo)       # every finite budget of interest is wide
    return sorted({lo, lo + 1, (lo + hi) // 2 + 1, hi + 1, hi + 1000, 10 ** 6})


@pytest.mark.parametrize("engine", ["persistent", "stepped", "wheel", "wheel_stepped"])
def test_wide_budgets_vs_oracle(engine):
    for shape, seed in [((400, 24), 1), ((320, 10, 8), 2)]:
        inst = heavy(shape, seed)
        for M in budgets(inst):
            x = inst.with_M(M)
            o = oracle.solve_pruned(x)
            m, mc = oracle.solve_model(x)
            r = wcsp.solve(x, engine=engine)
            assert r.key() == o.key() == m.key(), (shape, M, engine, r, o)
            assert counters(r) == (mc.cycles, mc.work, mc.arrivals, mc.triggered, mc.created, mc.started,
                                   mc.relabels), (shape, M, engine, r, mc)


def test_wide_small_random_and_thresholds():
    """Random small grids with heavy weights, budgets on both sides of the 16-bit
    limit (65533 narrow, 65534 wide), 1-D lines long enough to need them, and
    removed vertices."""
    rng = np.random.default_rng(4242)
    n = 0
    for i in range(60):
        inst = I.random_small(rng, shapes=[(12, 12), (6, 6, 6), (300,), (3, 3, 3, 3)], lo_hi=(180, 255),
                              M_range=(60000, 140000), max_sources=3, max_targets=3, hole_prob=0.1)
        if i % 5 == 0:
            inst = inst.with_M(wcsp.M_MAX + 1)
        if i % 7 == 3:
            pres = (rng.random(inst.N) > 0.1).astype(np.uint8)
            if not (inst.maskA & pres).any() or not (inst.maskB & pres).any():
                continue
            inst = inst.with_sets(present=pres)
        o = oracle.solve_pruned(inst)
        m, mc = oracle.solve_model(inst)
        for engine in ("persistent", "wheel"):
            r = wcsp.solve(inst, engine=engine)
            assert r.key() == o.key() == m.key(), (inst.shape, inst.M, engine, r, o)
            assert counters(r) == (mc.cycles, mc.work, mc.arrivals, mc.triggered, mc.created, mc.started,
                                   mc.relabels)
        n += o.status == oracle.REACHED
    assert n >= 20


def test_handle_switches_between_layouts():
    """One wheel-engine handle: a 16-bit solve, wide solves (its sweep form), then
    16-bit again and the reconstruction of a wide solve — each equal to a fresh
    handle and to the oracle; the reconstructed path re-sums to (F1, F2)."""
    inst = heavy((300, 16), 5)
    lo, hi = oracle.f2_min(inst), oracle.f2_lex(inst)
    narrow = I.config_face((300, 16), 5, 1500)
    with wcsp.Solver(narrow, engine="wheel") as s:
        r0 = s.solve()
        assert r0.key() == oracle.solve_pruned(narrow).key()
        s.load(inst.with_M((lo + hi) // 2))
        for M in ((lo + hi) // 2, hi + 1, lo + 1):
            s.set_targets(M=M)
            r = s.solve()
            assert r.key() == oracle.solve_pruned(inst.with_M(M)).key() == wcsp.solve(inst.with_M(M)).key()
        path, rr = s.reconstruct()
        st, F1, F2 = oracle.validate_path(inst.with_M(lo + 1), path)
        assert st == 0 and (F1, F2) == (rr.F1, rr.F2)
        s.load(narrow)
        assert s.solve().key() == r0.key()


def test_wide_rejected_where_unsupported():
    inst = heavy((64, 8), 3, 100000)
    with pytest.raises(wcsp.WcspError) as e:
        wcsp.solve(inst, engine="wheel", slabs=2)
    assert e.value.status == wcsp.EINVAL
    with wcsp.Solver(inst.with_M(1000), engine="wheel") as s:
        with pytest.raises(wcsp.WcspError) as e:
            s.staircase(100000)
        assert e.value.status == wcsp.EINVAL
