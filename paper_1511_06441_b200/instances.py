"""Seeded synthetic instances for the weight-constrained shortest path on Z^d.

This module is the ONE piece shared by the CUDA path (bench, tests) and the
CPU oracle (tests, cpu_baseline).  It holds no arithmetic of the method: it
only draws edge values f = (f1, f2) and the sets A, B, exactly as the problem
statement asks for them ("f : E -> Z_+^2"; "two
fixed disjoint subsets A, B"), plus the budget M as a plain input.

Encoding (the C-ABI's, include/wcsp.h):
  * N = prod(shape); vertex index v = x0 + n0*(x1 + n1*(x2 + ...)) (x0 fastest).
  * f1[k][v], f2[k][v] (uint8, shape (d, N)) are the values of the undirected
    edge (v, v + e_k).  f1 == 0 means "edge absent" (subgraph of Z^d,
    PAPER.md:27); entries with x_k = n_k - 1 are always 0.
  * maskA / maskB: uint8 [N] 0/1.
  * M: int >= 1, or M_INF (-1) for the unconstrained first-passage case
    ("The first passage percolation corresponds to the case
    M = infinity").

Value recipe (SURVEY.md §7 step 1, §8(d) "Concrete synthetic inputs"): f1 and
f2 are iid uniform integers on [lo, hi], independent of each other, drawn by a
counter-based hash so any edge's value is a pure function of (seed, v, k, c):
    sm(x)  = splitmix64 finaliser of (x + 0x9E3779B97F4A7C15)
    h      = sm(sm(seed) ^ (8*v + 2*k + c)),  c = 0 for f1, 1 for f2
    value  = lo + ((h >> 32) mod (hi - lo + 1))
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Sequence

import numpy as np

M_INF = -1

_GOLD = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def _sm(x: np.ndarray) -> np.ndarray:
    """splitmix64: finaliser applied to x + golden gamma (vectorised, wraps mod 2^64)."""
    with np.errstate(over="ignore"):
        z = (x + _GOLD).astype(np.uint64)
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        return z ^ (z >> np.uint64(31))


def sm_scalar(x: int) -> int:
    return int(_sm(np.array([x & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0])


@dataclasses.dataclass
class Instance:
    """A problem instance in the C-ABI encoding (see module docstring)."""
    shape: tuple
    f1: np.ndarray            # uint8 (d, N)
    f2: np.ndarray            # uint8 (d, N)
    maskA: np.ndarray         # uint8 (N,)
    maskB: np.ndarray         # uint8 (N,)
    M: int
    present: Optional[np.ndarray] = None   # uint8 (N,) or None (all present)
    name: str = ""
    seed: int = 0

    @property
    def d(self) -> int:
        return len(self.shape)

    @property
    def N(self) -> int:
        return int(np.prod(self.shape, dtype=np.int64))

    def with_M(self, M: int) -> "Instance":
        return dataclasses.replace(self, M=int(M))

    def with_sets(self, maskA=None, maskB=None, present=None) -> "Instance":
        return dataclasses.replace(
            self,
            maskA=self.maskA if maskA is None else maskA,
            maskB=self.maskB if maskB is None else maskB,
            present=self.present if present is None else present)

    def coords(self, v: int) -> tuple:
        out = []
        for n in self.shape:
            out.append(v % n)
            v //= n
        return tuple(out)

    def index(self, coords: Sequence[int]) -> int:
        v, mul = 0, 1
        for x, n in zip(coords, self.shape):
            v += x * mul
            mul *= n
        return v

    def n_edges(self) -> int:
        """Number of present undirected edges (f1 > 0)."""
        return int(np.count_nonzero(self.f1))


def strides(shape) -> list:
    s, out = 1, []
    for n in shape:
        out.append(s)
        s *= n
    return out


def axis_coord(shape, k: int, v: np.ndarray) -> np.ndarray:
    st = strides(shape)
    return (v // st[k]) % shape[k]


def grid_values(shape, seed: int, lo: int, hi: int, chunk: int = 1 << 22):
    """f1, f2 arrays (uint8, (d, N)) of the full grid, iid U{lo..hi} per edge."""
    assert 1 <= lo <= hi <= 255
    d = len(shape)
    N = int(np.prod(shape, dtype=np.int64))
    f1 = np.zeros((d, N), dtype=np.uint8)
    f2 = np.zeros((d, N), dtype=np.uint8)
    s0 = _sm(np.array([seed & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0]
    span = np.uint64(hi - lo + 1)
    for start in range(0, N, chunk):
        v = np.arange(start, min(N, start + chunk), dtype=np.uint64)
        for k in range(d):
            last = axis_coord(shape, k, v.astype(np.int64)) == shape[k] - 1
            for c, dst in ((0, f1), (1, f2)):
                key = np.uint64(8) * v + np.uint64(2 * k + c)
                h = _sm(s0 ^ key)
                val = (np.uint64(lo) + ((h >> np.uint64(32)) % span)).astype(np.uint8)
                val[last] = 0
                dst[k, start:start + len(v)] = val
    return f1, f2


def set_mask(shape, rule) -> np.ndarray:
    """A/B vertex sets.  rule: 'face0' (x0 = 0), 'face1' (x0 = n0-1), 'corner0'
    (v = 0), 'corner1' (v = N-1), 'centre' (floor(n/2) per axis),
    'boundary' (any x_k in {0, n_k-1}, the §6 protocol),
    'checker' (even coordinate sum: every neighbour of a member is a non-member,
    so the initial treatment starts an edge on every lane — a dense-treat stress
    case), or an explicit iterable of vertex indices."""
    N = int(np.prod(shape, dtype=np.int64))
    m = np.zeros(N, dtype=np.uint8)
    if isinstance(rule, str):
        if rule == "corner0":
            m[0] = 1
        elif rule == "corner1":
            m[N - 1] = 1
        elif rule == "centre":
            v, mul = 0, 1
            for n in shape:
                v += (n // 2) * mul
                mul *= n
            m[v] = 1
        elif rule == "checker":
            v = np.arange(N, dtype=np.int64)
            par = np.zeros(N, dtype=np.int64)
            for k in range(len(shape)):
                par += axis_coord(shape, k, v)
            m[par % 2 == 0] = 1
        elif rule in ("face0", "face1", "boundary"):
            v = np.arange(N, dtype=np.int64)
            x0 = axis_coord(shape, 0, v)
            if rule == "face0":
                m[x0 == 0] = 1
            elif rule == "face1":
                m[x0 == shape[0] - 1] = 1
            else:
                b = np.zeros(N, dtype=bool)
                for k in range(len(shape)):
                    xk = axis_coord(shape, k, v)
                    b |= (xk == 0) | (xk == shape[k] - 1)
                m[b] = 1
        else:
            raise ValueError(f"unknown set rule {rule!r}")
    else:
        m[np.asarray(list(rule), dtype=np.int64)] = 1
    return m


def grid_instance(shape, seed: int, lo: int, hi: int, A="face0", B="face1",
                  M: int = M_INF, name: str = "") -> Instance:
    f1, f2 = grid_values(tuple(shape), seed, lo, hi)
    return Instance(tuple(shape), f1, f2, set_mask(shape, A), set_mask(shape, B),
                    int(M), None, name or f"grid{'x'.join(map(str, shape))}", seed)


def edge_instance(shape, edges, A, B, M, name="") -> Instance:
    """Grid subgraph with ONLY the listed edges present.  edges: iterable of
    ((coords_u), (coords_v), f1, f2) with u, v lattice neighbours."""
    shape = tuple(shape)
    d, N = len(shape), int(np.prod(shape))
    f1 = np.zeros((d, N), dtype=np.uint8)
    f2 = np.zeros((d, N), dtype=np.uint8)
    inst = Instance(shape, f1, f2, np.zeros(N, np.uint8), np.zeros(N, np.uint8), M, None, name)
    for cu, cv, a, b in edges:
        diff = [y - x for x, y in zip(cu, cv)]
        assert sorted(map(abs, diff)) == [0] * (d - 1) + [1], (cu, cv)
        k = [i for i, x in enumerate(diff) if x][0]
        lo_c = cu if diff[k] == 1 else cv
        v = inst.index(lo_c)
        f1[k, v], f2[k, v] = a, b
    inst.maskA[[inst.index(c) for c in A]] = 1
    inst.maskB[[inst.index(c) for c in B]] = 1
    return inst


# ---------------------------------------------------------------------------
# Named workloads (BASELINE.json configs)
# ---------------------------------------------------------------------------

def config_C1(seed: int, M: int = 40) -> Instance:
    """configs[0]: 2D 16x16, f1,f2 ~ U{1..5}, A = corner, B = opposite corner,
    M = 40 (infeasible for every seed); C1b uses M = 65."""
    return grid_instance((16, 16), seed, 1, 5, "corner0", "corner1", M,
                         name="C1" if M == 40 else f"C1(M={M})")


def config_face(shape, seed: int, M: int, lo: int = 1, hi: int = 10, name="") -> Instance:
    """configs[1], [2], [4]: U{1..10}, A = face x0=0, B = face x0=n0-1."""
    return grid_instance(shape, seed, lo, hi, "face0", "face1", M, name)


def fixture_B() -> Instance:
    """SURVEY.md §4 'Fixture B, re-sourcing' (3x2 grid) — the §2 events at
    PAPER.md:75 (L=19-5=14), :83 (L=19-2=17), :85 (12 < 17; 17-2=15 > 14,
    time restored to 7), :87 (edge not triggered since 16 <= 18)."""
    E = [((0, 0), (1, 0), 2, 5), ((1, 0), (1, 1), 7, 2), ((0, 0), (0, 1), 3, 1),
         ((0, 1), (1, 1), 3, 1), ((1, 0), (2, 0), 20, 1), ((1, 1), (2, 1), 20, 1),
         ((2, 0), (2, 1), 20, 1)]
    return edge_instance((3, 2), E, [(0, 0)], [(2, 1)], 19, "fixtureB")


def fixture_D() -> Instance:
    """SURVEY.md §4 'Fixture D, phantom' (3x3 grid) — the §2 events at
    PAPER.md:95-97 (L(7)=11, L(11)=6, phantom 11' with label 11-2=9)."""
    E = [((0, 0), (0, 1), 2, 5), ((0, 1), (0, 2), 2, 6), ((0, 2), (1, 2), 2, 2),
         ((0, 0), (1, 0), 4, 4), ((1, 0), (1, 1), 5, 4), ((1, 1), (1, 2), 4, 2),
         ((1, 2), (2, 2), 30, 1)]
    return edge_instance((3, 3), E, [(0, 0)], [(2, 2)], 19, "fixtureD")


def speedway_instance(n: int, M: int = M_INF, B=None) -> Instance:
    """§5 Lemma environment: V_n = [-n, n] x [0, n]
    (PAPER.md:253), water on the whole x-axis (A = {y = 0}), every y-axis
    edge has time 1, every other edge time 2; all weights f2 = 1.
    Array coordinates: x_arr = x + n, y_arr = y.  B defaults to the top of the
    y-axis, (0, n)."""
    shape = (2 * n + 1, n + 1)
    N = shape[0] * shape[1]
    f1 = np.full((2, N), 2, dtype=np.uint8)
    f2 = np.ones((2, N), dtype=np.uint8)
    v = np.arange(N)
    xa, ya = v % shape[0], v // shape[0]
    f1[0, xa == shape[0] - 1] = 0
    f2[0, xa == shape[0] - 1] = 0
    f1[1, ya == shape[1] - 1] = 0
    f2[1, ya == shape[1] - 1] = 0
    f1[1, (xa == n) & (ya < shape[1] - 1)] = 1
    mA = (ya == 0).astype(np.uint8)
    mB = np.zeros(N, np.uint8)
    for (x, y) in (B or [(0, n)]):
        mB[(x + n) + shape[0] * y] = 1
    return Instance(shape, f1, f2, mA, mB, M, None, f"speedway{n}")


def _staircase(p, q):
    """Unit lattice staircase from p to q (|dx| = |dy|), x-step first
    (SPEC.md:406 rasterisation; SURVEY reading R26).  Returns the edges as
    ((x, y), (x', y')) pairs."""
    (x, y), (x1, y1) = p, q
    n = abs(x1 - x)
    assert n == abs(y1 - y), (p, q)
    sx, sy = (1 if x1 > x else -1), (1 if y1 > y else -1)
    out = []
    for _ in range(n):
        out.append(((x, y), (x + sx, y)))
        x += sx
        out.append(((x, y), (x, y + sy)))
        y += sy
    return out


def _vertical(p, q):
    (x, y), (x1, y1) = p, q
    assert x == x1
    lo, hi = min(y, y1), max(y, y1)
    return [((x, yy), (x, yy + 1)) for yy in range(lo, hi)]


def fractal_fast_edges(k: int):
    """Fast (f1 = 1) edges of the Theorem-2 environment omega_k
    on the left half-plane: the y-axis and segment LO (omega_1),
    then k - 1 refinements; refining a triangle (a, b, c) similar to (L, O, T)
    adds the vertical mid(a,b) -> mid(a,c) and the diagonal mid(c,b) -> mid(a,c)
    (the segments L0X and T0X of PAPER.md:303) and recurses into
    (a, mid(a,b), mid(a,c)) and (mid(a,c), mid(c,b), c) (I_2 of PAPER.md:303).
    t = 2^k; L = (-t/2, 0), O = (0, t/2), T = (0, t)."""
    t = 1 << k
    L, O, T = (-t // 2, 0), (0, t // 2), (0, t)
    edges = set(_vertical((0, 0), (0, t)))            # the y-axis
    edges.update(_staircase(L, O))                    # segment LO
    mid = lambda p, q: ((p[0] + q[0]) // 2, (p[1] + q[1]) // 2)
    tris = [(L, O, T)]
    for _ in range(k - 1):
        nxt = []
        for a, b, c in tris:
            mab, mac, mcb = mid(a, b), mid(a, c), mid(c, b)
            edges.update(_vertical(mab, mac))
            edges.update(_staircase(mcb, mac))
            nxt += [(a, mab, mac), (mac, mcb, c)]
        tris = nxt
    return edges


def fractal_instance(k: int, M: int = M_INF, B=None) -> Instance:
    """configs[3]: the paper's fractal active-set construction (Theorem 2,
    PAPER.md:290-349) on V = [-t, t] x [0, t + 1] (PAPER.md:253 with n = t + 1,
    SURVEY §8(d) C4), t = 2^k, water on the whole x-axis, f1 = 1 on omega_k's
    fast edges (mirrored across the y-axis) and 2 elsewhere
    (PAPER.md:255), f2 = 1; B = {(0, t)} by default."""
    t = 1 << k
    shape = (2 * t + 1, t + 2)
    N = shape[0] * shape[1]
    f1 = np.full((2, N), 2, dtype=np.uint8)
    f2 = np.ones((2, N), dtype=np.uint8)
    v = np.arange(N)
    xa, ya = v % shape[0], v // shape[0]
    for kk, last in ((0, xa == shape[0] - 1), (1, ya == shape[1] - 1)):
        f1[kk, last] = 0
        f2[kk, last] = 0
    for (p, q) in fractal_fast_edges(k):
        for sgn in (1, -1):                            # mirror across x = 0
            (x0, y0), (x1, y1) = (sgn * p[0], p[1]), (sgn * q[0], q[1])
            if (x1, y1) < (x0, y0):
                (x0, y0), (x1, y1) = (x1, y1), (x0, y0)
            kk = 0 if y0 == y1 else 1
            f1[kk, (x0 + t) + shape[0] * y0] = 1
    mA = (ya == 0).astype(np.uint8)
    mB = np.zeros(N, np.uint8)
    for (x, y) in (B or [(0, t)]):
        mB[(x + t) + shape[0] * y] = 1
    return Instance(shape, f1, f2, mA, mB, M, None, f"fractal{k}")


def speedway_lemma_set(T: int):
    """The §5 Lemma's active set at time T with the
    correction of SURVEY E1 / reading R15 (exact for every T >= 3 under eager
    retirement): Lemma ∪ {(±k, T - 2k - 1) : 1 <= k <= floor((T - 3) / 4)}.
    Returned as (finite core, height of the flat part, |z| bound of the core):
    the flat part is {(z, floor(T/2)) : |z| > floor((T+1)/4)}."""
    m = (T + 1) // 4
    core = {(0, T), (0, T - 1)}
    for k in range(1, m + 1):
        core |= {(-k, T - 2 * k), (k, T - 2 * k)}
    for k in range(1, (T - 3) // 4 + 1):
        core |= {(-k, T - 2 * k - 1), (k, T - 2 * k - 1)}
    return core, T // 2, m


def random_small(rng: np.random.Generator, shapes=None, lo_hi=None, M_range=(3, 60),
                 max_sources=3, max_targets=3, hole_prob=0.0) -> Instance:
    """Random small instance for property suites: random shape from `shapes`,
    f ~ U{lo..hi}, random disjoint A/B sets, random M, optionally random edge
    holes (subgraph of Z^d)."""
    shapes = shapes or [(5, 5), (6, 6), (8, 8), (12, 12), (4, 4, 4), (6, 5, 4), (7, 3), (3, 2, 2)]
    shape = tuple(shapes[rng.integers(len(shapes))])
    lo, hi = lo_hi or [(1, 3), (1, 5), (1, 10)][rng.integers(3)]
    seed = int(rng.integers(1 << 62))
    f1, f2 = grid_values(shape, seed, lo, hi)
    N = f1.shape[1]
    if hole_prob > 0:
        holes = rng.random(f1.shape) < hole_prob
        f1[holes] = 0
        f2[holes] = 0
    perm = rng.permutation(N)
    na = int(rng.integers(1, max_sources + 1))
    nb = int(rng.integers(1, max_targets + 1))
    mA = np.zeros(N, np.uint8)
    mB = np.zeros(N, np.uint8)
    mA[perm[:na]] = 1
    mB[perm[na:na + nb]] = 1
    M = int(rng.integers(M_range[0], M_range[1] + 1))
    return Instance(shape, f1, f2, mA, mB, M, None, f"rand{shape}", seed)
