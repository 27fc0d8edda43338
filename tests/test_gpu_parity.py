"""Parity of the CUDA path (through the C-ABI) with the CPU oracle (-m gpu).

Bar: integer outputs (status, F1, F2, X, Y) bit-exact
with the oracle; the work counters (cycles, edge_updates = sum over cycles of
live edges + phantoms, arrivals, triggered, phantoms created, lanes started,
relabels) bit-exact with oracle tier 5, the paper's cycle run sequentially
(see check()).
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_1511_06441_b200 import instances as I
from paper_1511_06441_b200 import wcsp

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fixtures.json")))
ENGINES = ["persistent", "stepped", "wheel", "wheel_stepped"]


MODEL_MAX_CELLS = 40_000_000     # N * cycles the sequential model (tier 5) runs in seconds


def model_counters(r):
    return (r.cycles, r.edge_updates, r.arrivals, r.triggered, r.phantoms_created, r.lanes_started,
            r.relabels)


def check(inst, engine="persistent", time_mode="jump", counters=True, want=None, **kw):
    """Outputs bit-exact with oracle tier 2; with counters=True also the work
    counters bit-exact with tier 5, the paper's cycle run sequentially
    (cycles, edge_updates = sum over cycles of live edges + phantoms, arrivals,
    triggered, phantoms created, lanes started, relabels)."""
    r = wcsp.solve(inst, engine=engine, time_mode=time_mode, **kw)
    o = oracle.solve_pruned(inst)
    assert r.key() == o.key(), (inst.name, inst.seed, inst.shape, inst.M, r, o)
    if want is not None:
        assert r.key() == want.key()
    if counters:
        m, mc = oracle.solve_model(inst, unit=time_mode == "unit")
        assert m.key() == r.key()
        assert model_counters(r) == (mc.cycles, mc.work, mc.arrivals, mc.triggered, mc.created,
                                     mc.started, mc.relabels), (inst.name, inst.shape, inst.M, r, mc)
    return r, o


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("name", ["fixtureB", "fixtureD"])
def test_mechanism_fixtures(name, engine):
    inst = getattr(I, "fixture_" + name[-1])()
    e = GOLD[name]["expect"]
    with wcsp.Solver(inst, engine=engine, trace_cap=64) as s:
        r = s.solve()
        tr = s.trace()
    assert r.key() == (wcsp.REACHED, e["F1"], e["F2"], e["X"], e["Y"])
    # the narrated events: a phantom is created exactly at t = 13 (PAPER.md:85 / :97)
    ev = [x for x in GOLD[name]["events"] if "phantom_label" in x][0]
    t_created = tr["t"][tr["created"] > 0]
    assert list(t_created) == [ev["t"]]
    assert r.phantoms_created == 1
    # the whole hand trace of the §4 steps (tests/golden 'hand_trace', pinned in test_oracle.py)
    ht = GOLD[name]["hand_trace"]
    got = [[int(t), int(a), int(e), int(p)] for t, a, e, p in
           zip(tr["t"], tr["active_vertices"], tr["live_lanes"], tr["phantoms"])]
    if engine.startswith("wheel"):   # the wheel keeps no active-vertex list (trace slot reused)
        got = [[x[0], h[1], x[2], x[3]] for x, h in zip(got, ht["cycles"])]
    assert got == ht["cycles"]
    hc = ht["counters"]
    assert model_counters(r) == (hc["cycles"], hc["work"], hc["arrivals"], hc["triggered"], hc["created"],
                                 hc["started"], hc["relabels"])
    # every narrated relabel time is a cycle of the run (jump mode visits exactly these times)
    for x in GOLD[name]["events"]:
        assert x["t"] in set(tr["t"].tolist())


@pytest.mark.parametrize("engine", ENGINES)
def test_random_tiny_vs_brute_force(engine):
    rng = np.random.default_rng(101)
    shapes = [(3, 3), (4, 4), (5, 4), (2, 2, 2), (3, 2, 2), (6, 3), (7,)]
    for i in range(150):
        inst = I.random_small(rng, shapes=shapes, M_range=(3, 25), max_sources=2, max_targets=2,
                              hole_prob=0.15 if i % 3 == 0 else 0.0)
        if i % 10 == 9:
            inst = inst.with_M(I.M_INF)
        r, _ = check(inst, engine)
        assert r.key() == oracle.solve_brute(inst).key()


@pytest.mark.parametrize("engine", ENGINES)
def test_random_mid_sizes(engine):
    rng = np.random.default_rng(202 if engine == "persistent" else 203)
    shapes = [(8, 8), (12, 12), (16, 16), (33, 7), (4, 4, 4), (6, 5, 4), (40,), (3, 3, 3, 3), (40, 40), (10, 10, 10)]
    n_inf = 0
    for i in range(300):
        inst = I.random_small(rng, shapes=shapes, M_range=(5, 120), max_sources=4, max_targets=4,
                              hole_prob=0.1 if i % 4 == 0 else 0.0)
        r, _ = check(inst, engine)
        if inst.M * inst.N <= 2_000_000:
            assert r.key() == oracle.solve_dense(inst).key()
        n_inf += r.status == wcsp.INFEASIBLE
    assert n_inf >= 20


def test_unit_equals_jump():
    """Reading R4: advancing by 1 or by the min residual
     gives identical outputs."""
    rng = np.random.default_rng(303)
    for i in range(60):
        inst = I.random_small(rng, shapes=[(10, 10), (5, 5, 5)], M_range=(5, 80))
        rj, _ = check(inst, time_mode="jump")
        ru, _ = check(inst, time_mode="unit")
        assert rj.key() == ru.key()
        if rj.status == wcsp.REACHED:
            assert ru.cycles == rj.F1   # unit mode visits every t = 1..F1


def test_removed_vertices_and_multi_sets():
    rng = np.random.default_rng(404)
    for i in range(60):
        inst = I.random_small(rng, shapes=[(12, 12), (6, 6, 6)], M_range=(10, 90), max_sources=6, max_targets=6)
        pres = (rng.random(inst.N) > 0.15).astype(np.uint8)
        inst = inst.with_sets(present=pres)
        if not (inst.maskA & pres).any() or not (inst.maskB & pres).any():
            continue
        check(inst)


@pytest.mark.parametrize("seed", range(0, 40))
def test_C1_infeasible_and_C1b(seed):
    c = I.config_C1(seed)
    r = wcsp.solve(c)
    assert r.status == wcsp.INFEASIBLE
    check(c)
    check(I.config_C1(seed, 65))


def test_wheel_equals_sweep_counters():
    """The timing wheel is an exact reformulation of Steps 1/3/7:
    same outputs and the same work counters as the residual-countdown sweep."""
    rng = np.random.default_rng(606)
    insts = [I.random_small(rng, shapes=[(12, 12), (6, 6, 6), (30, 9), (3, 4, 3, 3)], M_range=(5, 120),
                            max_sources=5, max_targets=5, hole_prob=0.1) for _ in range(60)]
    insts += [I.config_face((96, 96), 1, 400), I.config_face((24, 24, 24), 2, 150), I.fixture_B(), I.fixture_D(),
              I.speedway_instance(20)]
    for inst in insts:
        rs = wcsp.solve(inst, engine="persistent")
        for e in ("wheel", "wheel_stepped"):
            rw = wcsp.solve(inst, engine=e)
            assert rw.key() == rs.key(), (inst.name, e)
            assert (rw.cycles, rw.edge_updates, rw.arrivals, rw.phantoms_created, rw.relabels, rw.triggered) == \
                   (rs.cycles, rs.edge_updates, rs.arrivals, rs.phantoms_created, rs.relabels, rs.triggered), \
                   (inst.name, e, rw, rs)
    # per-cycle E and P agree too
    inst = I.config_face((64, 64), 3, 260)
    with wcsp.Solver(inst, trace_cap=4096) as s:
        s.solve()
        ts = s.trace()
    with wcsp.Solver(inst, engine="wheel", trace_cap=4096) as s:
        s.solve()
        tw = s.trace()
    for k in ("t", "live_lanes", "phantoms", "triggered", "arrivals", "created", "relabels"):
        assert np.array_equal(ts[k], tw[k]), k


def test_determinism_repeated_runs():
    inst = I.config_face((96, 96), 5, 300)
    rs = [wcsp.solve(inst, engine=e) for e in ENGINES for _ in range(3)]
    for r in rs[1:]:
        assert (r.key(), r.cycles, r.edge_updates, r.phantoms_created, r.relabels, r.triggered, r.arrivals) == \
               (rs[0].key(), rs[0].cycles, rs[0].edge_updates, rs[0].phantoms_created, rs[0].relabels,
                rs[0].triggered, rs[0].arrivals)


def test_reconstruction_valid_and_optimal():
    """Reading R12 (PAPER.md:25 corrected): the recovered path is an A->B path
    with exactly (F1, F2), checked by the oracle's independent path check."""
    rng = np.random.default_rng(505)
    done = 0
    for i in range(80):
        inst = I.random_small(rng, shapes=[(8, 8), (10, 6), (4, 4, 4)], M_range=(10, 70), max_sources=3,
                              max_targets=3)
        if i % 7 == 6:
            inst = inst.with_M(I.M_INF)
        o = oracle.solve_pruned(inst)
        if o.status != oracle.REACHED:
            continue
        with wcsp.Solver(inst) as s:
            path, r = s.reconstruct()
        assert r.key() == o.key()
        st, F1, F2 = oracle.validate_path(inst, path)
        assert st == 0 and F1 == o.F1
        if inst.M != I.M_INF:
            assert F2 == o.F2
        assert path[-1] == o.X and path[-2] == o.Y
        done += 1
    assert done >= 40


def test_M_infinity_first_passage_and_speedway():
    for n in (8, 20, 33):
        for B in ([(0, n)], [(3, n // 2)], [(-n, n), (n, n)]):
            s = I.speedway_instance(n, B=B)
            r = wcsp.solve(s)
            assert r.key() == oracle.solve_lex(s, 2).key()
            x, y = B[0]
            if len(B) == 1:
                assert r.F1 == y + min(y, 2 * abs(x))
            assert r.phantoms_created == 0                  # M = inf never needs phantoms


# --- full BASELINE sizes (configs[1], configs[2]) -------------------------------------------

@pytest.mark.slow
def test_C2_full_size_binding_M():
    """configs[1]: 1024^2, U{1..10}, face -> face, M_bind; oracle tier 2 in full."""
    inst = I.config_face((1024, 1024), 0, I.M_INF)
    inst = inst.with_M(oracle.m_bind(inst))
    r = wcsp.solve(inst)
    o = oracle.solve_pruned(inst)
    assert r.key() == o.key()
    assert r.cycles >= o.cycles and r.edge_updates >= o.work


@pytest.mark.slow
def test_C3_full_size_M_endpoints_and_properties():
    """configs[2]: 256^3, face -> face.  Exact at the two M endpoints and M = inf
    (P3, P4: lexicographic Dijkstra), and at M_bind the sandwich/monotone
    properties (P5) plus one-step reconstruction consistency (P10)."""
    inst = I.config_face((256, 256, 256), 0, I.M_INF)
    lo = oracle.solve_lex(inst, 1)
    hi = oracle.solve_lex(inst, 0)
    with wcsp.Solver(inst.with_M(hi.F2 + 1)) as s:
        assert s.solve().key() == hi.key()
        s.set_targets(M=lo.F2 + 1)
        assert s.solve().key() == lo.key()
        s.set_targets(M=lo.F2)
        assert s.solve().status == wcsp.INFEASIBLE
        s.set_targets(M=I.M_INF)
        assert s.solve().key() == oracle.solve_lex(inst, 2).key()
        Mb = (lo.F2 + hi.F2) // 2 + 1
        s.set_targets(M=Mb)
        rb = s.solve()
        assert rb.status == wcsp.REACHED and rb.F2 < Mb and hi.F1 <= rb.F1 <= lo.F1
        s.set_targets(M=Mb + 25)
        assert s.solve().F1 <= rb.F1


def test_speedway_active_vertex_sequence():
    """§5 Lemma environment, M = infinity, unit time: the sweep
    engine's active-vertex sequence (trace 'active_vertices' at
    the top of cycle T + 1) equals the method's active set at time T computed
    from first-passage times, which tests/test_oracle.py ties to the corrected
    Lemma (reading R15)."""
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from test_oracle import first_passage, speedway_sets
    n = 48
    s = I.speedway_instance(n)
    tau = first_passage(s)
    with wcsp.Solver(s, time_mode="unit", trace_cap=256) as sv:
        r = sv.solve()
        tr = sv.trace()
    assert r.F1 == n
    checked = 0
    for i, t in enumerate(tr["t"]):
        T = int(t) - 1
        if 3 <= T <= 44:
            _, lazy = speedway_sets(n, T, tau, s)
            assert tr["active_vertices"][i] == len(lazy), T
            checked += 1
    assert checked == 42


@pytest.mark.parametrize("engine", ["persistent", "wheel"])
def test_fractal_C4(engine):
    """configs[3] (Theorem-2 fractal): F1 = t = 2^k (SURVEY
    P7); with M = t + 1 the unique feasible path is the y-axis."""
    for k in range(3, 10):
        f = I.fractal_instance(k)
        t = 1 << k
        r = wcsp.solve(f, engine=engine)
        assert r.key() == oracle.solve_lex(f, 2).key() and r.F1 == t
        assert r.phantoms_created == 0
        want = (wcsp.REACHED, t, t, f.index((t, t)), f.index((t, t - 1)))
        r2 = wcsp.solve(f.with_M(t + 1), engine=engine)
        assert r2.key() == want


@pytest.mark.parametrize("slabs", [2, 3, 5])
def test_slab_engine(slabs):
    """the grid cut into slabs along its last axis (ghost planes,
    one exchange of boundary water and labels per cycle, max-combined cycle
    decisions) gives exactly the single-device outputs (reading R24); its work
    counters differ (one-cycle-stale ghost labels weaken the Step-4 pruning)."""
    rng = np.random.default_rng(700 + slabs)
    shapes = [(12, 12), (9, 20), (6, 6, 6), (5, 4, 11), (3, 3, 3, 8), (40,)]
    for i in range(60):
        inst = I.random_small(rng, shapes=shapes, M_range=(5, 120), max_sources=4, max_targets=4,
                              hole_prob=0.1 if i % 3 == 0 else 0.0)
        if i % 7 == 3:
            inst = inst.with_M(I.M_INF)
        if i % 5 == 4:
            inst = inst.with_sets(present=(rng.random(inst.N) > 0.1).astype(np.uint8))
            if not (inst.maskA & inst.present).any() or not (inst.maskB & inst.present).any():
                continue
        if inst.shape[-1] < slabs:
            continue
        o = oracle.solve_pruned(inst)
        r = wcsp.solve(inst, engine="wheel", slabs=slabs)
        assert r.key() == o.key(), (inst.shape, inst.M, slabs, r, o)
    for inst in (I.config_face((64, 64), 1, 300), I.config_face((32, 32, 32), 2, 200), I.fixture_D()):
        if inst.shape[-1] < slabs:
            continue
        r1 = wcsp.solve(inst, engine="wheel")
        rs = wcsp.solve(inst, engine="wheel", slabs=slabs)
        assert rs.key() == r1.key() == oracle.solve_pruned(inst).key()


def test_slab_engine_nccl_single_rank():
    """The multi-GPU transport (NCCL send/recv + allreduce per cycle) on one
    rank: the allreduce path and the distributed driver give the single-device
    outputs and counters."""
    for inst in (I.config_face((48, 48), 3, 220), I.config_face((16, 16, 16), 1, 120), I.fixture_B(),
                 I.speedway_instance(12)):
        r1 = wcsp.solve(inst, engine="wheel")
        with wcsp.Solver(inst, engine="wheel", nranks=1, rank=0, nccl_id=wcsp.nccl_unique_id()) as s:
            rn = s.solve()
        assert rn.key() == r1.key()
        assert (rn.edge_updates, rn.cycles, rn.phantoms_created) == (r1.edge_updates, r1.cycles, r1.phantoms_created)


@pytest.mark.parametrize("engine", ["wheel", "wheel_stepped"])
def test_staircase_every_budget_in_one_run(engine):
    """one run at M_max records the whole F1*(M) staircase; for
    every budget M <= M_max the oracle's optimum is the first step
    with F2 < M (X and Y included), infeasible below the last step."""
    rng = np.random.default_rng(808)
    checked = 0
    for i in range(25):
        inst = I.random_small(rng, shapes=[(8, 8), (10, 7), (5, 4, 3), (12, 12)], M_range=(1, 1),
                              max_sources=3, max_targets=3)
        hi = oracle.solve_lex(inst, 0)
        if hi.status != oracle.REACHED:
            continue
        M_max = hi.F2 + 4
        with wcsp.Solver(inst.with_M(M_max), engine=engine) as s:
            steps, r = s.staircase(M_max)
        assert steps and all(a[0] < b[0] and a[1] > b[1] for a, b in zip(steps, steps[1:]))
        assert steps[0][:2] == (hi.F1, hi.F2)        # the unconstrained (lexicographic) optimum first
        for M in range(1, M_max + 1):
            o = oracle.solve_pruned(inst.with_M(M))
            st = next((x for x in steps if x[1] < M), None)
            want = (oracle.INFEASIBLE,) if st is None else (oracle.REACHED,) + tuple(st)
            assert o.key() == want, (inst.shape, M, steps, o)
            checked += 1
    assert checked > 300


@pytest.mark.parametrize("slabs", [2, 3, 5, 8])
def test_slab_engine_peer_halo(slabs):
    """the slab boundary fused into one persistent kernel over
    peer memory (water crossing a boundary is a system-scope atomicMax into the
    neighbour's state word; the Step-4 test reads the neighbour's label in
    place).  No stale ghost labels, so outputs AND every work counter equal the
    single-device run (and tier 5)."""
    rng = np.random.default_rng(900 + slabs)
    shapes = [(12, 12), (9, 20), (6, 6, 6), (5, 4, 11), (3, 3, 3, 8), (40,), (16, 16, 16)]
    for i in range(50):
        inst = I.random_small(rng, shapes=shapes, M_range=(5, 120), max_sources=4, max_targets=4,
                              hole_prob=0.1 if i % 3 == 0 else 0.0)
        if i % 7 == 3:
            inst = inst.with_M(I.M_INF)
        if i % 5 == 4:
            inst = inst.with_sets(present=(rng.random(inst.N) > 0.1).astype(np.uint8))
            if not (inst.maskA & inst.present).any() or not (inst.maskB & inst.present).any():
                continue
        if inst.shape[-1] < slabs:
            continue
        r1 = wcsp.solve(inst, engine="wheel")
        rp = wcsp.solve(inst, engine="wheel", slabs=slabs, halo="peer")
        assert rp.key() == r1.key() == oracle.solve_pruned(inst).key(), (inst.shape, inst.M, slabs, rp, r1)
        assert model_counters(rp) == model_counters(r1), (inst.shape, inst.M, slabs, rp, r1)
    for inst in (I.config_face((64, 64), 1, 300), I.config_face((32, 32, 32), 2, 200), I.fixture_D(),
                 I.speedway_instance(20), I.config_face((48, 48, 48), 0, 260)):
        if inst.shape[-1] < slabs:
            continue
        r1 = wcsp.solve(inst, engine="wheel")
        rp = wcsp.solve(inst, engine="wheel", slabs=slabs, halo="peer")
        assert rp.key() == r1.key() == oracle.solve_pruned(inst).key()
        assert model_counters(rp) == model_counters(r1)


def test_peer_halo_nccl_single_rank():
    """The multi-GPU form of the peer halo (IPC handle exchange over NCCL, the
    cross-rank barrier, per-rank result reduction) on one rank."""
    for inst in (I.config_face((48, 48), 3, 220), I.config_face((16, 16, 16), 1, 120), I.fixture_B()):
        r1 = wcsp.solve(inst, engine="wheel")
        with wcsp.Solver(inst, engine="wheel", halo="peer", nranks=1, rank=0, nccl_id=wcsp.nccl_unique_id()) as s:
            rn = s.solve()
        assert rn.key() == r1.key()
        assert model_counters(rn) == model_counters(r1)


MODEL_GOLD = os.path.join(os.path.dirname(__file__), "golden", "model_counters.json")


@pytest.mark.slow
@pytest.mark.parametrize("key", ["C3s/0", "C2/0", "C3/0"])
def test_full_size_counters_vs_model(key):
    """BASELINE sizes: the metric's numerator (edge_updates) and every other
    work counter equal oracle tier 5's (the paper's cycle run sequentially on
    the CPU, stored by scripts/make_model_counters.py), for the default engine
    and the sweep engine."""
    gold = json.load(open(MODEL_GOLD))
    if key not in gold:
        pytest.skip(f"{key} not in {MODEL_GOLD}")
    g = gold[key]
    name, seed = key.split("/")
    shape = {"C2": (1024, 1024), "C3": (256, 256, 256), "C3s": (128, 128, 128)}[name]
    inst = I.config_face(shape, int(seed), I.M_INF).with_M(g["M"])
    c = g["counters"]
    want = (c["cycles"], c["work"], c["arrivals"], c["triggered"], c["created"], c["started"], c["relabels"])
    for engine in ("wheel", "persistent"):
        r = wcsp.solve(inst, engine=engine)
        assert list(r.key()) == g["key"]
        assert model_counters(r) == want, (key, engine, r)
    # the peer-halo slab engine (2 and 4 virtual slabs) gives the same counters at full size
    for slabs in (2, 4):
        r = wcsp.solve(inst, engine="wheel", slabs=slabs, halo="peer")
        assert list(r.key()) == g["key"] and model_counters(r) == want, (key, slabs, r)


@pytest.mark.parametrize("halo", ["copy", "peer"])
def test_slab_handle_reuse_across_budgets(halo):
    """A slab handle solved at one budget and re-solved at another gives the
    same outputs and counters as fresh handles (no state of the earlier run —
    e.g. stamped ghost-plane water — leaks into the next)."""
    for inst in (I.config_face((40, 40), 4, I.M_INF), I.config_face((20, 20, 20), 5, I.M_INF)):
        lo, hi = oracle.solve_lex(inst, 1).F2 + 1, oracle.solve_lex(inst, 0).F2 + 1
        Ms = [hi, lo, (lo + hi) // 2, I.M_INF, hi]
        with wcsp.Solver(inst.with_M(Ms[0]), engine="wheel", slabs=3, halo=halo) as s:
            for M in Ms:
                s.set_targets(M=M)
                r = s.solve()
                fresh = wcsp.solve(inst.with_M(M), engine="wheel", slabs=3, halo=halo)
                assert r.key() == fresh.key() == oracle.solve_pruned(inst.with_M(M)).key()
                assert model_counters(r) == model_counters(fresh)


def test_counters_stable_over_repeats():
    """Repeated solves (sparse cycles with per-block triggered lists, dense
    cycles with the bitmap, both engines) give tier 5's counters every time —
    a race between blocks would show up as a run-to-run difference."""
    for inst in (I.config_face((48, 48, 48), 0, 260), I.fractal_instance(7), I.config_face((200, 200), 6, 700)):
        m, mc = oracle.solve_model(inst)
        want = (mc.cycles, mc.work, mc.arrivals, mc.triggered, mc.created, mc.started, mc.relabels)
        for engine in ("wheel", "wheel_stepped", "persistent"):
            with wcsp.Solver(inst, engine=engine) as s:
                for _ in range(6):
                    r = s.solve()
                    assert r.key() == m.key() and model_counters(r) == want, (inst.name, engine, r)


# --- extremes: full u8 weights, the largest budget, long times (texp refresh, stamp wrap), thin grids ---

def test_extreme_weights_and_budgets():
    """f1, f2 over the whole u8 range (1..255: the wheel's 256 buckets, times
    past 2^16 so the lane-expiry refresh runs), M from 1 to WCSP_M_MAX, and
    degenerate shapes (axes of length 1, one-row grids): outputs vs the oracle,
    counters vs tier 5."""
    rng = np.random.default_rng(1717)
    shapes = [(40, 40), (1, 60), (60, 1), (9, 1, 9), (400,), (7, 7, 7), (2, 2, 2, 30), (1, 1, 1, 50)]
    cases = 0
    for i in range(40):
        shape = shapes[i % len(shapes)]
        lo, hi = [(200, 255), (1, 255), (128, 255)][i % 3]
        inst = I.random_small(rng, shapes=[shape], lo_hi=(lo, hi), M_range=(1, wcsp.M_MAX),
                              max_sources=3, max_targets=3)
        if i % 4 == 0:
            inst = inst.with_M(wcsp.M_MAX)
        if i % 4 == 1:
            inst = inst.with_M(I.M_INF)
        if i % 8 == 2:
            inst = inst.with_M(1)
        for engine in ("wheel", "persistent"):
            check(inst, engine)
        cases += 1
    # one long line: F1 > 2^16 time units with f1 = 255 everywhere
    s = I.grid_instance((300,), 3, 255, 255, "corner0", "corner1", I.M_INF, "line255")
    r, _ = check(s, "wheel")
    assert r.F1 == 255 * 299 and r.F1 > (1 << 16)
    assert cases == 40


@pytest.mark.parametrize("engine", ["wheel", "persistent"])
def test_stamp_wrap_long_run(engine):
    """More than 65534 cycles (the 16-bit cycle stamps wrap, PAPER.md:133's
    'temporary label' is reset by the maintenance pass): a 1-D line of
    70000 unit edges in unit time."""
    n = 70000
    s = I.grid_instance((n,), 5, 1, 1, "corner0", "corner1", I.M_INF, "line1")
    r = wcsp.solve(s, engine=engine, time_mode="unit")
    assert r.key() == oracle.solve_lex(s, 2).key()
    assert r.F1 == n - 1 and r.cycles == n - 1


@pytest.mark.slow
@pytest.mark.skipif(os.environ.get("WCSP_TEST_C5") != "1", reason="C5 (1024^3, ~105 GB of HBM, ~6 min): set WCSP_TEST_C5=1")
def test_C5_full_size_one_gpu():
    """configs[4] unsliced on one B200: at both M endpoints the oracle's tier-3
    values (scripts/make_mbind.py, tests/golden/mbind.json) are reproduced exactly;
    at M_bind the run satisfies F2 < M and F1_lex <= F1 <= F1 at F2_min (P5)."""
    table = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "mbind.json")))
    g = table["C5/0"]
    inst = I.config_face((1024, 1024, 1024), 0, g["M_bind"])
    with wcsp.Solver(inst, engine="wheel") as s:
        r = s.solve()
        assert r.status == wcsp.REACHED and r.F2 < g["M_bind"] and g["F1_lex"] <= r.F1 <= g["F1_at_F2min"]
        s.set_targets(M=g["F2_lex"] + 1)
        r_hi = s.solve()
        assert (r_hi.F1, r_hi.F2) == (g["F1_lex"], g["F2_lex"])
        s.set_targets(M=g["F2_min"] + 1)
        r_lo = s.solve()
        assert (r_lo.F1, r_lo.F2) == (g["F1_at_F2min"], g["F2_min"])
        s.set_targets(M=g["F2_min"])
        assert s.solve().status == wcsp.INFEASIBLE


@pytest.mark.parametrize("bps", ["3", "4"])
def test_both_cycle_kernel_builds(bps, monkeypatch):
    """The persistent wheel kernel exists in two builds (4 resident blocks per SM,
    64 registers, taken for 3-D grids >= 1.5 * 2^20 vertices; 3 blocks, 80 registers, otherwise).
    WCSP_BLOCKS_PER_SM forces either; both must give the oracle's outputs and tier 5's counters,
    on random small cases and on face-to-face cubes that span several treat rounds per block."""
    monkeypatch.setenv("WCSP_BLOCKS_PER_SM", bps)
    rng = np.random.default_rng(909)
    for _ in range(40):
        inst = I.random_small(rng, shapes=[(6, 5, 4), (10, 10, 10), (16, 16), (3, 3, 3, 3)], M_range=(5, 120),
                              max_sources=4, max_targets=4, hole_prob=0.1)
        check(inst, "wheel")
    for shape, seed, M in [((40, 40, 40), 1, 200), ((64, 48, 32), 2, 260), ((128, 96), 3, 500)]:
        r, _ = check(I.config_face(shape, seed, M), "wheel")
        for slabs in (2, 4):         # the fused peer-halo kernel comes in the same two builds
            rp = wcsp.solve(I.config_face(shape, seed, M), engine="wheel", slabs=slabs, halo="peer")
            assert rp.key() == r.key() and model_counters(rp) == model_counters(r), (shape, slabs, rp, r)


@pytest.mark.parametrize("lag", ["0", "1"])
def test_hybrid_one_barrier_kernel(lag, monkeypatch):
    """The neighbourhood-synchronised wheel kernels on every single-device persistent wheel
    solve (WCSP_HYBRID=1): lag=0 the one-barrier hybrid (k_wheel_hybrid: neighbourhood waits
    replace the grid barrier after the treat, time advances by 1 after a fire that delivered
    water and jumps otherwise), lag=1 the lagged-decision kernel (k_wheel_lag: time steps by one,
    treat(c) waits only for the neighbourhood's fire(c), decision c is taken one cycle later and a
    terminating one discards the fire that ran past it).  Only non-empty cycles are counted —
    outputs equal the oracle's and every work counter tier 5's, on random grids (holes, several
    sources/targets, M = infinity), sparse-cycle runs (the fractal, listed treats), repeated
    solves (no run-to-run difference), a tiny event ring (the allocation guard and the regrow)
    and both kernel builds."""
    monkeypatch.setenv("WCSP_HYBRID", "1")
    monkeypatch.setenv("WCSP_HYB_LAG", lag)
    rng = np.random.default_rng(4321)
    for i in range(80):
        inst = I.random_small(rng, shapes=[(12, 12), (6, 6, 6), (30, 9), (3, 4, 3, 3), (40,), (16, 16, 16)],
                              M_range=(5, 120), max_sources=4, max_targets=4, hole_prob=0.1 if i % 3 == 0 else 0.0)
        if i % 7 == 3:
            inst = inst.with_M(I.M_INF)
        check(inst, "wheel")
    for k in (5, 8):
        f = I.fractal_instance(k)
        check(f, "wheel")
        check(f.with_M((1 << k) + 1), "wheel")
    for inst in (I.config_face((48, 48, 48), 0, 260), I.config_face((200, 200), 6, 700)):
        m, mc = oracle.solve_model(inst)
        want = (mc.cycles, mc.work, mc.arrivals, mc.triggered, mc.created, mc.started, mc.relabels)
        with wcsp.Solver(inst, engine="wheel") as s:
            for _ in range(4):
                r = s.solve()
                assert r.key() == m.key() and model_counters(r) == want, (inst.name, r)
        r = wcsp.solve(inst, engine="wheel", phantom_capacity=4096)
        assert r.retries >= 1 and r.key() == m.key() and model_counters(r) == want, r
    for bps in ("3", "4"):
        monkeypatch.setenv("WCSP_BLOCKS_PER_SM", bps)
        check(I.config_face((64, 48, 32), 2, 260), "wheel")
