"""CPU oracle for the weight-constrained shortest path (ctypes wrapper of
oracle/wcsp_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg may import this package.  The CUDA product
path (paper_1511_06441_b200) never imports it, and it imports nothing from the
CUDA path (instances come from paper_1511_06441_b200.instances, a module
holding no arithmetic of the method).

Tiers (see wcsp_oracle.c): dense (definition on the product graph, PAPER.md
:13-21), pruned (time-ordered label setting on remaining quality),
lex (Dijkstra with lexicographic keys: the M endpoints and M = infinity),
brute (simple-path enumeration), model (the paper's nine-step cycle run
sequentially, also counting its work).  Parity status: all five pinned by
tests/test_oracle.py (brute force, closed forms P3/P4, monotonicity P5,
fixtures B/D, counts P9, hand-traced cycle counts of fixture B).
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "wcsp_oracle.c")

M_INF = -1
REACHED, INFEASIBLE, EINVAL, ELIMIT, ENOMEM = 0, 1, 2, 3, 4


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain C, -O2) in-tree."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "wcsp_oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-o", _SO, _SRC])
    return _SO


class _Problem(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("shape", ctypes.c_int64 * 4),
                ("f1", ctypes.c_void_p), ("f2", ctypes.c_void_p),
                ("maskA", ctypes.c_void_p), ("maskB", ctypes.c_void_p),
                ("present", ctypes.c_void_p), ("M", ctypes.c_int64)]


class _Result(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int64), ("F1", ctypes.c_int64), ("F2", ctypes.c_int64),
                ("X", ctypes.c_int64), ("Y", ctypes.c_int64), ("work", ctypes.c_int64),
                ("cycles", ctypes.c_int64), ("t_reached", ctypes.c_int64)]


class _Counters(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in
                ("cycles", "work", "arrivals", "triggered", "created", "started", "relabels")]


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        for name in ("orc_dense", "orc_brute"):
            getattr(lib, name).argtypes = [ctypes.POINTER(_Problem), ctypes.POINTER(_Result)]
            getattr(lib, name).restype = ctypes.c_int
        lib.orc_pruned.argtypes = [ctypes.POINTER(_Problem), ctypes.c_int64, ctypes.POINTER(_Result)]
        lib.orc_pruned.restype = ctypes.c_int
        lib.orc_lex.argtypes = [ctypes.POINTER(_Problem), ctypes.c_int, ctypes.POINTER(_Result)]
        lib.orc_lex.restype = ctypes.c_int
        lib.orc_model.argtypes = [ctypes.POINTER(_Problem), ctypes.c_int, ctypes.POINTER(_Result),
                                  ctypes.POINTER(_Counters), ctypes.c_void_p, ctypes.c_int64,
                                  ctypes.POINTER(ctypes.c_int64)]
        lib.orc_model.restype = ctypes.c_int
        lib.orc_validate_path.argtypes = [ctypes.POINTER(_Problem), ctypes.POINTER(ctypes.c_int64),
                                          ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                                          ctypes.POINTER(ctypes.c_int64)]
        lib.orc_validate_path.restype = ctypes.c_int
        _lib = lib
    return _lib


@dataclasses.dataclass
class Result:
    status: int
    F1: int = 0
    F2: int = 0
    X: int = -1
    Y: int = -1
    work: int = 0
    cycles: int = 0
    t_reached: int = 0

    def key(self):
        """The outputs compared bit-exactly with the CUDA path."""
        if self.status != REACHED:
            return (self.status,)
        return (self.status, self.F1, self.F2, self.X, self.Y)


def _problem(inst, M: Optional[int] = None):
    keep = []

    def ptr(a):
        if a is None:
            return None
        a = np.ascontiguousarray(a, dtype=np.uint8)
        keep.append(a)
        return a.ctypes.data

    p = _Problem()
    p.d = len(inst.shape)
    for k, n in enumerate(inst.shape):
        p.shape[k] = n
    p.f1, p.f2 = ptr(inst.f1), ptr(inst.f2)
    p.maskA, p.maskB = ptr(inst.maskA), ptr(inst.maskB)
    p.present = ptr(inst.present)
    p.M = inst.M if M is None else M
    return p, keep


def _res(r: _Result) -> Result:
    return Result(int(r.status), int(r.F1), int(r.F2), int(r.X), int(r.Y), int(r.work),
                  int(r.cycles), int(r.t_reached))


def solve_dense(inst) -> Result:
    p, keep = _problem(inst)
    r = _Result()
    _load().orc_dense(ctypes.byref(p), ctypes.byref(r))
    return _res(r)


def solve_pruned(inst, t_limit: int = 0) -> Result:
    p, keep = _problem(inst)
    r = _Result()
    _load().orc_pruned(ctypes.byref(p), int(t_limit), ctypes.byref(r))
    return _res(r)


def solve_lex(inst, mode: int) -> Result:
    """mode 0: keys (f1, f2); 1: (f2, f1); 2: f1 only (M = infinity)."""
    p, keep = _problem(inst)
    r = _Result()
    _load().orc_lex(ctypes.byref(p), int(mode), ctypes.byref(r))
    return _res(r)


def solve_brute(inst) -> Result:
    p, keep = _problem(inst)
    r = _Result()
    _load().orc_brute(ctypes.byref(p), ctypes.byref(r))
    return _res(r)


@dataclasses.dataclass
class Counters:
    """Work of the method's cycle (tier 5): cycles, sum of live edges + phantoms over
    cycles (work, the north_star numerator), arrivals, triggered vertices, phantoms
    created, lanes started, relabels; the initial treatment of A (t = 0) included."""
    cycles: int
    work: int
    arrivals: int
    triggered: int
    created: int
    started: int
    relabels: int


def solve_model(inst, unit: bool = False, events: int = 0):
    """Tier 5: the paper's nine-step cycle run sequentially -> (Result, Counters), plus,
    if events > 0, the first `events` events as a list of dicts {t, kind, v, u, label}:
    "relabel" (v relabelled to label at t), "phantom" (created at t by v toward u,
    label = L* of v), "cycle" (advancing to t: v = active vertices, u = live
    edges, label = live phantoms at the top of the cycle)."""
    p, keep = _problem(inst)
    r = _Result()
    c = _Counters()
    ev = np.zeros((max(events, 1), 5), dtype=np.int64)
    n = ctypes.c_int64(0)
    _load().orc_model(ctypes.byref(p), 1 if unit else 0, ctypes.byref(r), ctypes.byref(c),
                      ev.ctypes.data if events > 0 else None, int(events), ctypes.byref(n))
    out = (_res(r), Counters(*[int(getattr(c, nm)) for nm, _ in _Counters._fields_]))
    if events <= 0:
        return out
    log = [dict(t=int(e[0]), kind=("relabel", "phantom", "cycle")[int(e[1])], v=int(e[2]), u=int(e[3]),
                label=int(e[4])) for e in ev[:min(n.value, events)]]
    return out + (log,)


def solve(inst) -> Result:
    """Best available tier for the instance: dense when N*M is small, else pruned."""
    if inst.M != M_INF and inst.N * inst.M <= 20_000_000:
        return solve_dense(inst)
    return solve_pruned(inst)


def validate_path(inst, path):
    """(status, F1, F2): status 0 iff `path` is an A->B path with F2 < M."""
    p, keep = _problem(inst)
    arr = (ctypes.c_int64 * len(path))(*[int(x) for x in path])
    f1, f2 = ctypes.c_int64(0), ctypes.c_int64(0)
    st = _load().orc_validate_path(ctypes.byref(p), arr, len(path), ctypes.byref(f1), ctypes.byref(f2))
    return int(st), int(f1.value), int(f2.value)


def f2_min(inst) -> Optional[int]:
    """Minimum F2 over A->B paths (Dijkstra on f2), None if B is unreachable."""
    r = solve_lex(inst, 1)
    return r.F2 if r.status == REACHED else None


def f2_lex(inst) -> Optional[int]:
    """F2 of the lexicographically fastest path (Dijkstra on (f1, f2))."""
    r = solve_lex(inst, 0)
    return r.F2 if r.status == REACHED else None


def m_bind(inst) -> int:
    """M_bind = floor((F2_min + F2_lex) / 2) + 1 (SURVEY §8 notation)."""
    return (f2_min(inst) + f2_lex(inst)) // 2 + 1
