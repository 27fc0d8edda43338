"""Pins for the CPU oracle (oracle/), -m "not gpu".

Each check ties the oracle to something other than itself (SURVEY §8(c)
"What pins each part"):
  * P1  brute-force simple-path enumeration (C tier 4 and an independent
        pure-Python enumerator below) on tiny grids;
  * P2  dense (tier 1) <-> pruned (tier 2) on mid sizes;
  * P3  feasibility boundary: feasible <=> M > F2_min (Dijkstra on f2);
  * P4  the M endpoints reduce to textbook lexicographic Dijkstra;
  * P5  monotonicity of F1*(M) and F2* < M;
  * P6  the §2 mechanism fixtures (tests/golden/fixtures.json);
  * P9  §6 vertex/edge counts;
  * the §5 Lemma proof's first-passage times on the speedway
        (PAPER.md:270-279): tau(x, y) = y + min(y, 2|x|).
"""
import dataclasses
import json
import os

import numpy as np
import pytest

import oracle
from paper_1511_06441_b200 import instances as I

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fixtures.json")))


# ---------------------------------------------------------------------------
# independent pure-Python brute force (tiny graphs): the definition
# ---------------------------------------------------------------------------

def py_neighbours(inst, v):
    st = I.strides(inst.shape)
    out = []
    pres = inst.present
    if pres is not None and not pres[v]:
        return out
    for k, n in enumerate(inst.shape):
        xk = (v // st[k]) % n
        if xk + 1 < n and inst.f1[k, v] > 0:
            out.append((v + st[k], int(inst.f1[k, v]), int(inst.f2[k, v])))
        if xk > 0 and inst.f1[k, v - st[k]] > 0:
            out.append((v - st[k], int(inst.f1[k, v - st[k]]), int(inst.f2[k, v - st[k]])))
    if pres is not None:
        out = [o for o in out if pres[o[0]]]
    return out


def py_brute(inst):
    """Lexicographic min of (F1, F2, X, Y) over all simple A->B paths with F2 < M."""
    best = None
    minf = inst.M == I.M_INF
    A = [v for v in range(inst.N) if inst.maskA[v]]
    B = set(v for v in range(inst.N) if inst.maskB[v])

    def dfs(path, F1, F2):
        nonlocal best
        v = path[-1]
        if len(path) > 1 and v in B:
            cand = (F1, -1 if minf else F2, v, path[-2])
            if best is None or cand < best:
                best = cand
        for u, a, b in py_neighbours(inst, v):
            if u in path:
                continue
            if not minf and F2 + b >= inst.M:
                continue
            dfs(path + [u], F1 + a, F2 + b)

    for a in A:
        dfs([a], 0, 0)
    return (oracle.INFEASIBLE,) if best is None else (oracle.REACHED,) + best


def tiny_instances(count, seed):
    rng = np.random.default_rng(seed)
    shapes = [(3, 3), (4, 3), (4, 4), (5, 4), (2, 2, 2), (3, 2, 2), (6, 3), (2, 2, 3)]
    out = []
    for i in range(count):
        inst = I.random_small(rng, shapes=shapes, M_range=(3, 25), max_sources=2, max_targets=2,
                              hole_prob=0.15 if i % 3 == 0 else 0.0)
        if i % 10 == 9:
            inst = inst.with_M(I.M_INF)
        out.append(inst)
    return out


def test_brute_c_vs_python_enumeration():
    for inst in tiny_instances(60, 11):
        assert oracle.solve_brute(inst).key() == py_brute(inst), inst


def test_dense_and_pruned_vs_brute_force():
    n_inf = 0
    for inst in tiny_instances(400, 12):
        b = oracle.solve_brute(inst).key()
        p = oracle.solve_pruned(inst).key()
        assert p == b, (inst, p, b)
        if inst.M != I.M_INF:
            d = oracle.solve_dense(inst).key()
            assert d == b, (inst, d, b)
        else:
            assert oracle.solve_lex(inst, 2).key() == b
        n_inf += b[0] == oracle.INFEASIBLE
    assert n_inf >= 20   # the suite exercises the infeasible verdict (2°)


def mid_instances(count, seed):
    rng = np.random.default_rng(seed)
    shapes = [(8, 8), (12, 12), (16, 16), (20, 7), (4, 4, 4), (6, 5, 4), (30,)]
    return [I.random_small(rng, shapes=shapes, M_range=(5, 80),
                           hole_prob=0.1 if i % 4 == 0 else 0.0) for i in range(count)]


def test_pruned_vs_dense_mid_sizes():
    n_inf = 0
    for inst in mid_instances(250, 13):
        d = oracle.solve_dense(inst).key()
        assert oracle.solve_pruned(inst).key() == d, inst
        n_inf += d[0] == oracle.INFEASIBLE
    assert 25 <= n_inf <= 225   # >= 10% infeasible, and mostly feasible


def test_feasibility_boundary_and_M_endpoints():
    """P3: feasible <=> M > F2_min.  P4: M = F2_min + 1 -> lex Dijkstra on
    (f2, f1); M >= F2_lex + 1 -> lex Dijkstra on (f1, f2); M = inf -> f1."""
    rng = np.random.default_rng(14)
    for _ in range(120):
        inst = I.random_small(rng, shapes=[(8, 8), (10, 6), (4, 4, 3), (12, 12)], M_range=(1, 1))
        lo = oracle.solve_lex(inst, 1)
        hi = oracle.solve_lex(inst, 0)
        if lo.status != oracle.REACHED:
            continue
        F2min = lo.F2
        assert oracle.solve_dense(inst.with_M(F2min)).status == oracle.INFEASIBLE
        assert oracle.solve_pruned(inst.with_M(F2min)).status == oracle.INFEASIBLE
        r = oracle.solve_dense(inst.with_M(F2min + 1))
        assert r.key() == lo.key()
        assert oracle.solve_pruned(inst.with_M(F2min + 1)).key() == lo.key()
        for M in (hi.F2 + 1, hi.F2 + 7):
            assert oracle.solve_dense(inst.with_M(M)).key() == hi.key()
            assert oracle.solve_pruned(inst.with_M(M)).key() == hi.key()
        assert oracle.solve_pruned(inst.with_M(I.M_INF)).key() == oracle.solve_lex(inst, 2).key()
        assert oracle.solve_lex(inst, 2).F1 == hi.F1


def test_monotone_in_M():
    """P5: F1*(M) non-increasing in M; F2* < M; sandwich between the endpoints."""
    rng = np.random.default_rng(15)
    for _ in range(25):
        inst = I.random_small(rng, shapes=[(9, 9), (5, 4, 3)], M_range=(1, 1))
        lo, hi = oracle.solve_lex(inst, 1), oracle.solve_lex(inst, 0)
        if lo.status != oracle.REACHED:
            continue
        prev = None
        for M in range(lo.F2 + 1, hi.F2 + 3):
            r = oracle.solve_dense(inst.with_M(M))
            assert r.status == oracle.REACHED and r.F2 < M
            assert hi.F1 <= r.F1 <= lo.F1
            if prev is not None:
                assert r.F1 <= prev
            prev = r.F1


@pytest.mark.parametrize("name", ["fixtureB", "fixtureD"])
def test_mechanism_fixture_results(name):
    g = GOLD[name]
    inst = I.edge_instance(tuple(g["shape"]), [(tuple(a), tuple(b), f1, f2) for a, b, f1, f2 in g["edges"]],
                           [tuple(c) for c in g["A"]], [tuple(c) for c in g["B"]], g["M"], name)
    ours = getattr(I, "fixture_" + name[-1])()
    assert np.array_equal(inst.f1, ours.f1) and np.array_equal(inst.f2, ours.f2)
    e = g["expect"]
    want = (oracle.REACHED, e["F1"], e["F2"], e["X"], e["Y"])
    for solve in (oracle.solve_dense, oracle.solve_brute, oracle.solve_pruned):
        assert solve(inst).key() == want
    assert py_brute(inst) == want


def test_speedway_first_passage_closed_form():
    """PAPER.md:270-279 (Lemma proof): on the speedway, water reaches (x, y)
    at tau = y + min(y, 2|x|) (climb the fast y-axis, then walk |x| slow edges;
    or climb a slow column directly)."""
    n = 14
    pts = [(x, y) for x in range(-n, n + 1, 3) for y in range(1, n + 1, 2)]
    for x, y in pts:
        s = I.speedway_instance(n, B=[(x, y)])
        tau = y + min(y, 2 * abs(x))
        assert oracle.solve_lex(s, 2).F1 == tau
        assert oracle.solve_pruned(s).F1 == tau


def test_counts_P374():
    for side, nv, ne in GOLD["counts_P374"]["cubes"]:
        f1, _ = I.grid_values((side, side, side), 0, 1, 10)
        assert f1.shape[1] == nv
        assert int(np.count_nonzero(f1)) == ne


def test_C1_infeasible_and_C1b_feasible():
    """configs[0] (M = 40) is infeasible for every seed (min F2 over
    paths >= 45); M = 65 is feasible for nearly all seeds."""
    feas = 0
    for seed in range(60):
        c = I.config_C1(seed)
        assert oracle.solve_dense(c).status == oracle.INFEASIBLE
        assert oracle.f2_min(c) >= 40
        feas += oracle.solve_dense(I.config_C1(seed, 65)).status == oracle.REACHED
    assert feas >= 55


def test_validate_path():
    inst = I.fixture_B()
    # the optimal path of fixture B: (0,0) -> (0,1) -> (1,1) -> (2,1)
    path = [0, 3, 4, 5]
    assert oracle.validate_path(inst, path) == (0, 26, 3)
    assert oracle.validate_path(inst, [0, 4, 5])[0] == oracle.EINVAL       # not adjacent
    assert oracle.validate_path(inst, [0, 1, 2, 5])[0] == 0               # 42, 7 < 19
    assert oracle.validate_path(inst.with_M(3), path)[0] == oracle.INFEASIBLE   # F2 = M


def test_generator_is_deterministic_and_uniform():
    a1, a2 = I.grid_values((64, 64), 7, 1, 10)
    b1, b2 = I.grid_values((64, 64), 7, 1, 10)
    assert np.array_equal(a1, b1) and np.array_equal(a2, b2)
    vals = a1[a1 > 0]
    counts = np.bincount(vals, minlength=11)[1:]
    assert counts.min() > 0.8 * counts.mean()
    assert np.corrcoef(a1[a1 > 0], a2[a1 > 0])[0, 1] < 0.05   # f1 independent of f2 (R19)


# ---------------------------------------------------------------------------
# §5: speedway Lemma (corrected, SURVEY E1 / reading R15) and the Theorem-2
# fractal's closed form
# ---------------------------------------------------------------------------

def first_passage(inst):
    """tau(v): plain Dijkstra on f1 from A (textbook, independent of oracle/)."""
    import heapq
    st = I.strides(inst.shape)
    dist = np.full(inst.N, 1 << 60, dtype=np.int64)
    pq = []
    for v in np.flatnonzero(inst.maskA):
        dist[v] = 0
        pq.append((0, int(v)))
    heapq.heapify(pq)
    while pq:
        d, v = heapq.heappop(pq)
        if d > dist[v]:
            continue
        for u, a, _ in py_neighbours(inst, v):
            if d + a < dist[u]:
                dist[u] = d + a
                heapq.heappush(pq, (d + a, u))
    return dist


def speedway_sets(n, T, tau, inst):
    """(eager, lazy) active sets at time T from first-passage times: eager =
    reached and some neighbour not yet reached (the Lemma's notion); lazy =
    some edge started at tau(v) toward a later-reached neighbour is still in
    flight after T (the method's active-vertex sequence)."""
    eager, lazy = set(), set()
    for v in range(inst.N):
        if tau[v] > T:
            continue
        x, y = inst.coords(v)
        nb = py_neighbours(inst, v)
        if any(tau[u] > T for u, _, _ in nb):
            eager.add((x - n, y))
        if any(tau[u] > tau[v] and tau[v] + a > T for u, a, _ in nb):
            lazy.add((x - n, y))
    return eager, lazy


def lemma_printed(T, n):
    """The Lemma exactly as printed."""
    m = (T + 1) // 4
    s = {(0, T), (0, T - 1)}
    for k in range(1, m + 1):
        s |= {(-k, T - 2 * k), (k, T - 2 * k)}
    return s | {(z, T // 2) for z in range(-n, n + 1) if abs(z) > m}


def test_speedway_lemma_corrected():
    """The Lemma's active set, checked against first-passage times on the
    lattice (the proof's own argument): the printed form is
    exact for T <= 6 only; the corrected form (R15) is exact for every T; the
    method's (lazy) active sequence adds (±k, 2k) when T = 4k + 1 and
    (±k, 2k + 1) when T = 4k + 2 (an edge still in flight toward a neighbour
    that was reached another way)."""
    n = 40
    s = I.speedway_instance(n)
    tau = first_passage(s)
    printed_fails = []
    for T in range(3, 41):
        eager, lazy = speedway_sets(n, T, tau, s)
        core, h, m = I.speedway_lemma_set(T)
        corrected = set(core) | {(z, h) for z in range(-n, n + 1) if abs(z) > m}
        assert eager == corrected, T
        if lemma_printed(T, n) != eager:
            printed_fails.append(T)
        extra = set()
        for k in range(1, T):
            if T == 4 * k + 1:
                extra |= {(-k, 2 * k), (k, 2 * k)}
            if T == 4 * k + 2:
                extra |= {(-k, 2 * k + 1), (k, 2 * k + 1)}
        assert lazy == eager | extra, T
    assert printed_fails and min(printed_fails) == 7


def test_fractal_closed_form_P7():
    """Theorem-2 environment: F1 to (0, t) is t = 2^k (the
    fast y-axis; any path needs t vertical steps); with f2 = 1 and M = t + 1 the
    only feasible path is the y-axis itself: F2 = t, X = (0, t), Y = (0, t-1)."""
    for k in range(2, 8):
        f = I.fractal_instance(k)
        t = 1 << k
        assert oracle.solve_lex(f, 2).F1 == t
        assert oracle.solve_pruned(f).F1 == t
        want = (oracle.REACHED, t, t, f.index((t, t)), f.index((t, t - 1)))
        assert oracle.solve_pruned(f.with_M(t + 1)).key() == want
        assert oracle.solve_lex(f, 1).key() == want          # M = F2_min + 1 endpoint (P4)
        # omega_k only adds fast edges to omega_{k-1}
        if k > 2:
            prev = I.fractal_fast_edges(k - 1)
            scale = {((2 * a[0], 2 * a[1]), (2 * b[0], 2 * b[1])) for a, b in prev}
            assert len(I.fractal_fast_edges(k)) > len(prev)
            assert all(abs(x) <= t and 0 <= y <= t for e in I.fractal_fast_edges(k) for (x, y) in e)
            assert scale  # (the scaled previous level is a different lattice; only monotonicity in k is asserted)


# ---------------------------------------------------------------------------
# tier 5: the paper's cycle run sequentially (oracle.solve_model)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["fixtureB", "fixtureD"])
def test_model_hand_trace_and_narrated_events(name):
    """The model reproduces, cycle by cycle, the hand trace of the §4 steps on
    the mechanism fixtures (golden 'hand_trace'), and every event the paper
    narrates for that mechanism (relabel times and labels, the
    phantom's time, endpoints and label)."""
    g = GOLD[name]
    inst = getattr(I, "fixture_" + name[-1])()
    r, c, log = oracle.solve_model(inst, events=1000)
    e = g["expect"]
    assert r.key() == (oracle.REACHED, e["F1"], e["F2"], e["X"], e["Y"])
    ht = g["hand_trace"]
    assert [[x["t"], x["v"], x["u"], x["label"]] for x in log if x["kind"] == "cycle"] == ht["cycles"]
    assert dataclasses.asdict(c) == ht["counters"]
    relabels = {(x["t"], x["v"], x["label"]) for x in log if x["kind"] == "relabel"}
    phantoms = {(x["t"], x["v"], x["u"], x["label"]) for x in log if x["kind"] == "phantom"}
    for ev in g["events"]:
        if "phantom_from" in ev:
            assert (ev["t"], inst.index(tuple(ev["phantom_from"])), inst.index(tuple(ev["phantom_to"])),
                    ev["phantom_label"]) in phantoms
        else:
            assert (ev["t"], inst.index(tuple(ev["vertex"])), ev["label"]) in relabels


def test_model_outputs_vs_brute_and_dense():
    """Tier 5's outputs are the optimum (reading R5 tie-break) in
    jump and unit time (reading R4)."""
    for inst in tiny_instances(200, 14):
        b = oracle.solve_brute(inst).key()
        assert oracle.solve_model(inst)[0].key() == b, inst
        assert oracle.solve_model(inst, unit=True)[0].key() == b, inst
    for inst in mid_instances(80, 15):
        assert oracle.solve_model(inst)[0].key() == oracle.solve_pruned(inst).key(), inst


def test_model_unit_vs_jump_counters():
    """Reading R4: advancing by 1 instead of by the minimum
    residual only inserts idle cycles: the same arrivals,
    triggerings, phantoms, starts and relabels; unit mode visits every
    t = 1..F1; the idle cycles only add work."""
    for inst in mid_instances(60, 16):
        rj, cj = oracle.solve_model(inst)
        ru, cu = oracle.solve_model(inst, unit=True)
        assert rj.key() == ru.key()
        same = ("arrivals", "triggered", "created", "started", "relabels")
        assert [getattr(cj, k) for k in same] == [getattr(cu, k) for k in same]
        assert cu.cycles >= cj.cycles and cu.work >= cj.work
        if rj.status == oracle.REACHED:
            assert cu.cycles == rj.F1


def test_model_counter_identities():
    """Every arrival is a started edge or a created phantom;
    every triggered vertex is relabelled or spawns only phantoms (Step 8.1,
    PAPER.md:211); M = inf never creates a phantom (an active vertex's first
    arrival is already its best)."""
    for inst in mid_instances(60, 17):
        r, c = oracle.solve_model(inst)
        assert c.arrivals <= c.started + c.created
        assert c.relabels <= c.triggered
        assert c.work >= c.arrivals
        ri, ci = oracle.solve_model(inst.with_M(I.M_INF))
        assert ci.created == 0


def test_model_speedway_active_sequence():
    """§5 Lemma environment, unit time, M = inf: the model's
    active-vertex count at the top of cycle T + 1 equals the lazy active set at
    T computed from first-passage times (reading R15, test_speedway_lemma_corrected)."""
    n = 48
    s = I.speedway_instance(n)
    tau = first_passage(s)
    r, c, log = oracle.solve_model(s, unit=True, events=10000)
    assert r.F1 == n
    cyc = [x for x in log if x["kind"] == "cycle"]
    assert [x["t"] for x in cyc] == list(range(1, n + 1))
    for x in cyc:
        T = x["t"] - 1
        if T >= 1:
            assert x["v"] == len(speedway_sets(n, T, tau, s)[1]), T
