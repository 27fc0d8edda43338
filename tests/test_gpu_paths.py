"""Rarely-taken paths of the CUDA solver, forced and checked against the oracle (-m gpu).

* The device-side overflow path (north_star; PAPER.md:151 the phantom sequence,
  :173 "difficulties with dynamic memory locations"): a structure that fills up
  ends the run with a flag and the size it needed, the host grows exactly that
  structure and re-runs.  Forced with tiny capacities for the sweep engine's
  phantom pool, the wheel's event ring and its run-descriptor table, and the
  slab engines; after the regrow the outputs equal the oracle's and the work
  counters equal tier 5's (the paper's cycle run sequentially), i.e. an
  overflowed attempt leaves nothing behind.
* The cycle budget (SPEC SolverConfig, include/wcsp.h): WCSP_EBUDGET.
* The wheel treat's staging overflow (events past the shared-memory staging go
  to the open ring regions, then a per-block spill buffer, then runs of one):
  a checkerboard source set makes the initial treatment start an edge on every
  lane of half the grid at once.
* The §6 protocol cubes (water on the boundary, B = the
  centre, 50^3 .. 125^3) at M_bind and M = infinity against tier 2.
* The headline configuration (configs[2], C3 256^3 at M_bind) against tier 2
  run in full (tests/golden/tier2_full.json, scripts/make_tier2_golden.py).
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_1511_06441_b200 import instances as I
from paper_1511_06441_b200 import wcsp

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MBIND = json.load(open(os.path.join(GOLDEN, "mbind.json")))


def counters(r):
    return (r.cycles, r.edge_updates, r.arrivals, r.triggered, r.phantoms_created, r.lanes_started, r.relabels)


def tier5(inst):
    m, mc = oracle.solve_model(inst)
    return m, (mc.cycles, mc.work, mc.arrivals, mc.triggered, mc.created, mc.started, mc.relabels)


OVERFLOW_CASES = [I.config_face((40, 40, 40), 0, 220), I.config_face((160, 160), 1, 640),
                  I.config_face((24, 24, 24), 2, I.M_INF)]


@pytest.mark.parametrize("engine", ["persistent", "stepped"])
def test_phantom_pool_overflow_regrows(engine):
    """Sweep engine: a pool of 256 phantom records overflows within a few cycles;
    the retry grows it to the size the device reported and the result is exact."""
    for inst in OVERFLOW_CASES[:2]:
        m, want = tier5(inst)
        r = wcsp.solve(inst, engine=engine, phantom_capacity=256)
        assert r.retries >= 1 and r.phantom_capacity > 256, r
        assert r.key() == m.key() == oracle.solve_pruned(inst).key()
        assert counters(r) == want, (inst.name, r)


@pytest.mark.parametrize("engine", ["wheel", "wheel_stepped"])
def test_event_ring_overflow_regrows(engine):
    """Wheel engine: a 4096-slot event ring (the auto size is millions) overflows in
    the first treat; the run ends with the ring slots it needed, the host grows the
    ring and re-runs (possibly more than once as the front grows)."""
    for inst in OVERFLOW_CASES:
        m, want = tier5(inst)
        r = wcsp.solve(inst, engine=engine, phantom_capacity=4096)
        assert r.retries >= 1 and r.phantom_capacity > 4096, r
        assert r.key() == m.key()
        assert counters(r) == want, (inst.name, r)


@pytest.mark.parametrize("engine", ["wheel", "wheel_stepped"])
def test_run_descriptor_overflow_regrows(engine, monkeypatch):
    """Wheel engine: 2 run descriptors per (bucket, block) (WCSP_DCAP; default 32)
    overflow; the host doubles only the descriptor table until the run fits."""
    monkeypatch.setenv("WCSP_DCAP", "2")
    for inst in OVERFLOW_CASES[:2]:
        m, want = tier5(inst)
        r = wcsp.solve(inst, engine=engine)
        assert r.retries >= 1, r
        assert r.key() == m.key()
        assert counters(r) == want, (inst.name, r)


@pytest.mark.parametrize("halo", ["copy", "peer"])
def test_slab_engine_overflow_regrows(halo, monkeypatch):
    """Slab engines (virtual slabs): ring and descriptor overflows in any slab stop
    every slab; the group grows what overflowed and re-runs.  Outputs equal the
    oracle's; the peer halo's counters also equal tier 5's."""
    for inst in OVERFLOW_CASES[:2]:
        m, want = tier5(inst)
        r = wcsp.solve(inst, engine="wheel", slabs=2, halo=halo, phantom_capacity=4096)
        assert r.retries >= 1 and r.key() == m.key(), (halo, r)
        if halo == "peer":
            assert counters(r) == want
    monkeypatch.setenv("WCSP_DCAP", "2")
    inst = OVERFLOW_CASES[0]
    m, want = tier5(inst)
    r = wcsp.solve(inst, engine="wheel", slabs=3, halo=halo)
    assert r.retries >= 1 and r.key() == m.key(), (halo, r)


def test_nccl_paths_overflow_regrow():
    """The multi-GPU drivers (NCCL copy halo, IPC peer halo) at one rank: the
    overflow need travels through their allreduce and the retry is exact."""
    inst = OVERFLOW_CASES[0]
    m, want = tier5(inst)
    for halo in ("copy", "peer"):
        with wcsp.Solver(inst, engine="wheel", halo=halo, nranks=1, rank=0, nccl_id=wcsp.nccl_unique_id(),
                         phantom_capacity=4096) as s:
            r = s.solve()
        assert r.retries >= 1 and r.key() == m.key(), (halo, r)
        assert counters(r) == want


@pytest.mark.parametrize("engine", ["persistent", "stepped", "wheel", "wheel_stepped"])
def test_cycle_budget(engine):
    """cycle_budget = k stops the run after k cycles with WCSP_EBUDGET; a budget
    the run does not reach changes nothing."""
    inst = I.config_face((32, 32, 32), 3, 200)
    full = wcsp.solve(inst, engine=engine)
    with pytest.raises(wcsp.WcspError) as e:
        wcsp.solve(inst, engine=engine, cycle_budget=5)
    assert e.value.status == wcsp.EBUDGET
    r = wcsp.solve(inst, engine=engine, cycle_budget=full.cycles + 1)
    assert r.key() == full.key() == oracle.solve_pruned(inst).key()


@pytest.mark.parametrize("slabs,halo", [(2, "copy"), (2, "peer")])
def test_cycle_budget_slabs(slabs, halo):
    inst = I.config_face((32, 32, 32), 3, 200)
    with pytest.raises(wcsp.WcspError) as e:
        wcsp.solve(inst, engine="wheel", slabs=slabs, halo=halo, cycle_budget=4)
    assert e.value.status == wcsp.EBUDGET


def checker_instance(shape, seed, M):
    inst = I.grid_instance(shape, seed, 1, 10, "checker", "corner1", M, f"checker{shape}")
    return inst.with_sets(maskA=inst.maskA & (1 - inst.maskB))


@pytest.mark.parametrize("bps", ["3", "4"])
def test_treat_staging_overflow_paths(bps, monkeypatch):
    """A checkerboard A: the initial treatment (t = 0) starts an edge on every lane
    of half the vertices, ~6 events per vertex, several times the block's
    shared-memory staging in one treat round.  The surplus goes to the spill
    buffer and, past it, to runs of one; later dense rounds append to open ring
    regions.  Outputs equal the oracle's and counters tier 5's, in both builds of
    the cycle kernel (3 and 4 resident blocks per SM)."""
    monkeypatch.setenv("WCSP_BLOCKS_PER_SM", bps)
    seen = np.zeros(3, dtype=np.int64)
    for shape, M in [((64, 64, 64), 300), ((64, 64, 64), I.M_INF), ((512, 256), 900)]:
        inst = checker_instance(shape, 11, M)
        m, want = tier5(inst)
        for engine in ("wheel", "wheel_stepped"):
            r = wcsp.solve(inst, engine=engine)
            assert r.key() == m.key() == oracle.solve_pruned(inst).key(), (shape, M, engine, r)
            assert counters(r) == want, (shape, M, engine, r)
            seen += (r.staging_appended, r.staging_spilled, r.staging_singles)
        rp = wcsp.solve(inst, engine="wheel", slabs=2, halo="peer")
        assert rp.key() == m.key() and counters(rp) == want
    assert seen[1] > 0 and seen[2] > 0, seen        # spill buffer and runs of one both exercised


@pytest.mark.parametrize("side", [50, 75, 100, 125])
def test_paper_section6_cubes(side):
    """§6 protocol replica: a side^3 cube, water on
    the whole boundary, B = the centre vertex (reading R18), f1, f2 ~ U{1..10}
    (R19).  Binding M (M_bind from tests/golden/mbind.json) and M = infinity:
    (status, F1, F2, X, Y) equal to tier 2 bit for bit, for the wheel and sweep
    engines; the §6 graph sizes of PAPER.md:374 hold for 100^3 and 125^3."""
    Mb = MBIND[f"P6-{side}/0"]["M_bind"]
    inst = I.grid_instance((side,) * 3, 0, 1, 10, "boundary", "centre", Mb, f"P6-{side}")
    if side == 100:
        assert inst.N == 1_000_000 and inst.n_edges() == 2_970_000
    if side == 125:
        assert inst.N == 1_953_125 and inst.n_edges() == 5_812_500
    for M in (Mb, I.M_INF):
        x = inst.with_M(M)
        o = oracle.solve_pruned(x)
        assert o.status == oracle.REACHED
        for engine in ("wheel", "persistent"):
            r = wcsp.solve(x, engine=engine)
            assert r.key() == o.key(), (side, M, engine, r, o)
        if M == I.M_INF:
            assert r.key() == oracle.solve_lex(x, 2).key()


@pytest.mark.slow
def test_C3_full_size_vs_tier2_golden():
    """configs[2] (C3 256^3, seed 0, M_bind) — the bench configuration — against
    oracle tier 2 (time-ordered label setting, a definition-based solver) run in
    full on the CPU by scripts/make_tier2_golden.py."""
    path = os.path.join(GOLDEN, "tier2_full.json")
    table = json.load(open(path)) if os.path.exists(path) else {}
    if "C3/0" not in table:
        pytest.skip("tests/golden/tier2_full.json has no C3/0 (scripts/make_tier2_golden.py C3)")
    gold = table["C3/0"]
    inst = I.config_face((256, 256, 256), 0, gold["M"])
    r = wcsp.solve(inst, engine="wheel")
    assert list(r.key()) == gold["key"]
    r = wcsp.solve(inst, engine="persistent")
    assert list(r.key()) == gold["key"]
