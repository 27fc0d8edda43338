"""Thin Python binding of the C-ABI in include/wcsp.h (argument marshalling only).

Every step of the solve runs in libwcsp.so's CUDA kernels; this module only
packs pointers and sizes.  There is no CPU fallback: if libwcsp.so is missing
or no CUDA device is usable the calls raise.

Inputs are either an `instances.Instance` (host numpy arrays -> WCSP_MEM_HOST)
or torch CUDA tensors (WCSP_MEM_DEVICE, read on the solver's stream).
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("WCSP_LIB") or os.path.join(_PKG, "libwcsp.so")   # WCSP_LIB: A/B builds

M_INF = -1
M_MAX = 65533            # 16-bit label layout (the fast default)
M_MAX_WIDE = 2147483646  # larger budgets run on 32-bit labels (include/wcsp.h)
REACHED, INFEASIBLE, EINVAL, EMISMATCH, EBUDGET, ENOMEM, ECUDA, ENCCL, EOVERFLOW = range(9)
MEM_HOST, MEM_DEVICE = 0, 1
JUMP, UNIT = 0, 1
PERSISTENT, STEPPED, WHEEL, WHEEL_STEPPED = 0, 1, 2, 3
ENGINES = {"persistent": PERSISTENT, "stepped": STEPPED, "wheel": WHEEL, "wheel_stepped": WHEEL_STEPPED}
HALO_COPY, HALO_PEER = 0, 1
HALOS = {"copy": HALO_COPY, "peer": HALO_PEER}
_STATUS = {0: "REACHED", 1: "INFEASIBLE", 2: "EINVAL", 3: "EMISMATCH", 4: "EBUDGET", 5: "ENOMEM",
           6: "ECUDA", 7: "ENCCL", 8: "EOVERFLOW"}


class WcspError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"wcsp {_STATUS.get(status, status)}: {msg}")
        self.status = status


class _Problem(ctypes.Structure):
    _fields_ = [("d", ctypes.c_int32), ("shape", ctypes.c_int64 * 4),
                ("f1", ctypes.c_void_p), ("f2", ctypes.c_void_p),
                ("maskA", ctypes.c_void_p), ("maskB", ctypes.c_void_p), ("present", ctypes.c_void_p),
                ("M", ctypes.c_int64), ("mem", ctypes.c_int32)]


class _Options(ctypes.Structure):
    _fields_ = [("time_mode", ctypes.c_int32), ("engine", ctypes.c_int32), ("demote_twin", ctypes.c_int32),
                ("device", ctypes.c_int32), ("cycle_budget", ctypes.c_int64),
                ("phantom_capacity", ctypes.c_int64), ("trace_cap", ctypes.c_int64),
                ("stream", ctypes.c_void_p), ("slabs", ctypes.c_int32), ("halo", ctypes.c_int32),
                ("nranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("nccl_id", ctypes.c_void_p),
                ("local_slab", ctypes.c_int32)]


class _Result(ctypes.Structure):
    _fields_ = [("F1", ctypes.c_int64), ("F2", ctypes.c_int64), ("X", ctypes.c_int64), ("Y", ctypes.c_int64),
                ("x_lane", ctypes.c_int32), ("via_phantom", ctypes.c_int32),
                ("cycles", ctypes.c_int64), ("edge_updates", ctypes.c_int64), ("arrivals", ctypes.c_int64),
                ("triggered", ctypes.c_int64), ("phantoms_created", ctypes.c_int64),
                ("relabels", ctypes.c_int64), ("lanes_started", ctypes.c_int64), ("peak_active", ctypes.c_int64),
                ("peak_phantoms", ctypes.c_int64), ("phantom_capacity", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("device_ms", ctypes.c_double),
                ("cycle_ms", ctypes.c_double), ("retries", ctypes.c_int64), ("staging_appended", ctypes.c_int64),
                ("staging_spilled", ctypes.c_int64), ("staging_singles", ctypes.c_int64)]


TRACE_FIELDS = ["t", "delta", "active_vertices", "live_lanes", "phantoms", "triggered", "arrivals",
                "created", "relabels", "tested", "ns_arrive", "ns_treat", "ns_arrive_spread", "ns_treat_spread"]


class _TraceRec(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in TRACE_FIELDS]


EXPORTS = ["wcsp_create", "wcsp_load", "wcsp_solve", "wcsp_set_targets", "wcsp_reconstruct", "wcsp_trace",
           "wcsp_validate_path", "wcsp_destroy", "wcsp_last_error", "wcsp_version", "wcsp_nccl_unique_id",
           "wcsp_staircase", "wcsp_generate_grid", "wcsp_generate_mask", "wcsp_slab_planes"]
SET_RULES = {"face0": 0, "face1": 1, "boundary": 2, "centre": 3, "corner0": 4, "corner1": 5}

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libwcsp.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `python -m paper_1511_06441_b200.build` "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P, O, R = ctypes.POINTER(_Problem), ctypes.POINTER(_Options), ctypes.POINTER(_Result)
    lib.wcsp_create.argtypes = [P, O, ctypes.POINTER(ctypes.c_void_p)]
    lib.wcsp_load.argtypes = [ctypes.c_void_p, P]
    lib.wcsp_solve.argtypes = [ctypes.c_void_p, R]
    lib.wcsp_set_targets.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                     ctypes.c_int64, ctypes.c_int32]
    lib.wcsp_reconstruct.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_int64,
                                     ctypes.POINTER(ctypes.c_int64), R]
    lib.wcsp_trace.argtypes = [ctypes.c_void_p, ctypes.POINTER(_TraceRec), ctypes.c_int64,
                               ctypes.POINTER(ctypes.c_int64)]
    lib.wcsp_validate_path.argtypes = [P, ctypes.POINTER(ctypes.c_int64), ctypes.c_int64,
                                       ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    for f in ("wcsp_create", "wcsp_load", "wcsp_solve", "wcsp_set_targets", "wcsp_reconstruct", "wcsp_trace",
              "wcsp_validate_path"):
        getattr(lib, f).restype = ctypes.c_int
    lib.wcsp_destroy.argtypes = [ctypes.c_void_p]
    lib.wcsp_destroy.restype = None
    lib.wcsp_last_error.restype = ctypes.c_char_p
    lib.wcsp_version.restype = ctypes.c_char_p
    lib.wcsp_staircase.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                                   ctypes.c_int64, ctypes.POINTER(ctypes.c_int64), R]
    lib.wcsp_staircase.restype = ctypes.c_int
    I64P = ctypes.POINTER(ctypes.c_int64)
    lib.wcsp_generate_grid.argtypes = [ctypes.c_int32, I64P, ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    lib.wcsp_generate_grid.restype = ctypes.c_int
    lib.wcsp_generate_mask.argtypes = [ctypes.c_int32, I64P, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_void_p, ctypes.c_void_p]
    lib.wcsp_generate_mask.restype = ctypes.c_int
    lib.wcsp_slab_planes.argtypes = [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64)]
    lib.wcsp_slab_planes.restype = ctypes.c_int
    lib.wcsp_nccl_unique_id.argtypes = [ctypes.c_char_p]
    lib.wcsp_nccl_unique_id.restype = ctypes.c_int
    _lib = lib
    return lib


def last_error() -> str:
    return load_library().wcsp_last_error().decode()


@dataclasses.dataclass
class Result:
    status: int
    F1: int = -1
    F2: int = -1
    X: int = -1
    Y: int = -1
    x_lane: int = -1
    via_phantom: int = 0
    cycles: int = 0
    edge_updates: int = 0
    arrivals: int = 0
    triggered: int = 0
    phantoms_created: int = 0
    relabels: int = 0
    lanes_started: int = 0
    peak_active: int = 0
    peak_phantoms: int = 0
    phantom_capacity: int = 0
    kernel_launches: int = 0
    device_ms: float = 0.0
    cycle_ms: float = 0.0
    retries: int = 0
    staging_appended: int = 0
    staging_spilled: int = 0
    staging_singles: int = 0

    def key(self):
        """Outputs compared bit-exactly with the oracle: (status, F1, F2, X, Y)."""
        if self.status != REACHED:
            return (self.status,)
        return (self.status, self.F1, self.F2, self.X, self.Y)


def _res(st: int, r: _Result) -> Result:
    out = Result(st)
    for f, _ in _Result._fields_:
        setattr(out, f, getattr(r, f))
    return out


def _ptr(a, keep):
    """(pointer, mem) of a host numpy array or a torch CUDA tensor (uint8)."""
    if a is None:
        return None, None
    if hasattr(a, "data_ptr") and getattr(a, "is_cuda", False):
        assert a.is_contiguous() and a.element_size() == 1
        keep.append(a)
        return a.data_ptr(), MEM_DEVICE
    arr = np.ascontiguousarray(np.asarray(a), dtype=np.uint8)
    keep.append(arr)
    return arr.ctypes.data, MEM_HOST


def _problem(shape, f1, f2, maskA, maskB, present, M):
    keep = []
    p = _Problem()
    p.d = len(shape)
    for k in range(4):
        p.shape[k] = int(shape[k]) if k < len(shape) else 1
    mems = set()
    for name, a in (("f1", f1), ("f2", f2), ("maskA", maskA), ("maskB", maskB), ("present", present)):
        ptr, mem = _ptr(a, keep)
        setattr(p, name, ptr)
        if mem is not None:
            mems.add(mem)
    if len(mems) != 1:
        raise ValueError("inputs must be all host arrays or all CUDA tensors")
    p.mem = mems.pop()
    p.M = int(M)
    return p, keep


class Solver:
    """A problem resident on one B200; `solve()` runs the sweep."""

    def __init__(self, inst=None, *, shape=None, f1=None, f2=None, maskA=None, maskB=None, present=None,
                 M=None, time_mode: str = "jump", engine: str = "persistent", trace_cap: int = 0,
                 phantom_capacity: int = 0, cycle_budget: int = 0, device: int = 0, stream=None,
                 slabs: int = 0, halo: str = "copy", nranks: int = 1, rank: int = 0, nccl_id: bytes = None,
                 local_slab: bool = False):
        lib = load_library()
        self._lib = lib
        self._h = ctypes.c_void_p()
        if inst is not None:
            shape, f1, f2, maskA, maskB, present, M = (inst.shape, inst.f1, inst.f2, inst.maskA, inst.maskB,
                                                       inst.present, inst.M)
        self.shape = tuple(shape)
        self.N = int(np.prod(self.shape))
        o = _Options()
        o.time_mode = {"jump": JUMP, "unit": UNIT}[time_mode]
        o.engine = ENGINES[engine]
        o.demote_twin = 0
        o.device = int(device)
        o.cycle_budget = int(cycle_budget)
        o.phantom_capacity = int(phantom_capacity)
        o.trace_cap = int(trace_cap)
        o.stream = None if stream is None else (stream if isinstance(stream, int) else stream.cuda_stream)
        o.slabs = int(slabs)
        o.halo = HALOS[halo]
        o.nranks = int(nranks)
        o.rank = int(rank)
        o.local_slab = 1 if local_slab else 0
        self._nccl_id = None
        if nccl_id is not None:
            assert len(nccl_id) == 128
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128)
            o.nccl_id = ctypes.cast(self._nccl_id, ctypes.c_void_p)
        self.trace_cap = int(trace_cap)
        p, keep = _problem(self.shape, f1, f2, maskA, maskB, present, M)
        st = lib.wcsp_create(ctypes.byref(p), ctypes.byref(o), ctypes.byref(self._h))
        if st != REACHED:
            self._h = None
            raise WcspError(st, last_error())

    def load(self, inst=None, *, f1=None, f2=None, maskA=None, maskB=None, present=None, M=None):
        if inst is not None:
            f1, f2, maskA, maskB, present, M = inst.f1, inst.f2, inst.maskA, inst.maskB, inst.present, inst.M
        p, keep = _problem(self.shape, f1, f2, maskA, maskB, present, M)
        st = self._lib.wcsp_load(self._h, ctypes.byref(p))
        if st != REACHED:
            raise WcspError(st, last_error())

    def solve(self) -> Result:
        r = _Result()
        st = self._lib.wcsp_solve(self._h, ctypes.byref(r))
        if st not in (REACHED, INFEASIBLE):
            raise WcspError(st, last_error())
        return _res(st, r)

    def set_targets(self, maskB=None, present=None, present_all: bool = False, M: int = None):
        keep = []
        pb, mb = _ptr(maskB, keep)
        pp, mp = _ptr(present, keep)
        mem = mb if mb is not None else (mp if mp is not None else MEM_HOST)
        st = self._lib.wcsp_set_targets(self._h, pb, pp, int(present_all), int(M), mem)
        if st != REACHED:
            raise WcspError(st, last_error())

    def reconstruct(self, cap: Optional[int] = None):
        """(path list A -> ... -> X, Result of the first solve)."""
        cap = cap or self.N
        buf = (ctypes.c_int64 * cap)()
        n = ctypes.c_int64(0)
        r = _Result()
        st = self._lib.wcsp_reconstruct(self._h, buf, cap, ctypes.byref(n), ctypes.byref(r))
        if st != REACHED:
            raise WcspError(st, last_error())
        return [int(buf[i]) for i in range(n.value)], _res(st, r)

    def staircase(self, M_max: int, f2_stop: int = -(1 << 62), cap: int = 1 << 16):
        """Every step (F1, F2, X, Y) of the F1*(M) staircase for budgets M <= M_max, in
        one run (wcsp_staircase): the optimum for budget M is the first step with F2 < M."""
        buf = (ctypes.c_int64 * (4 * cap))()
        n = ctypes.c_int64(0)
        r = _Result()
        st = self._lib.wcsp_staircase(self._h, int(M_max), int(f2_stop), buf, cap, ctypes.byref(n), ctypes.byref(r))
        if st not in (REACHED, INFEASIBLE):
            raise WcspError(st, last_error())
        m = min(n.value, cap)
        return [tuple(int(buf[4 * i + k]) for k in range(4)) for i in range(m)], _res(st, r)

    def trace(self) -> dict:
        """Per-cycle counters of the last solve: dict of numpy int64 arrays."""
        cap = max(1, self.trace_cap)
        buf = (_TraceRec * cap)()
        n = ctypes.c_int64(0)
        st = self._lib.wcsp_trace(self._h, buf, cap, ctypes.byref(n))
        if st != REACHED:
            raise WcspError(st, last_error())
        arr = np.ctypeslib.as_array(ctypes.cast(buf, ctypes.POINTER(ctypes.c_int64)), shape=(cap, len(TRACE_FIELDS)))[: n.value]
        return {f: arr[:, i].copy() for i, f in enumerate(TRACE_FIELDS)}

    def close(self):
        if getattr(self, "_h", None):
            self._lib.wcsp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def solve(inst, **kw) -> Result:
    with Solver(inst, **kw) as s:
        return s.solve()


def validate_path(inst, path):
    """Host-side check through the C-ABI: (status, F1, F2)."""
    lib = load_library()
    p, keep = _problem(inst.shape, inst.f1, inst.f2, inst.maskA, inst.maskB, inst.present, inst.M)
    arr = (ctypes.c_int64 * len(path))(*[int(x) for x in path])
    f1, f2 = ctypes.c_int64(0), ctypes.c_int64(0)
    st = lib.wcsp_validate_path(ctypes.byref(p), arr, len(path), ctypes.byref(f1), ctypes.byref(f2))
    return int(st), int(f1.value), int(f2.value)


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for Solver(nranks > 1, nccl_id=...); share it from one rank."""
    buf = ctypes.create_string_buffer(128)
    st = load_library().wcsp_nccl_unique_id(buf)
    if st != REACHED:
        raise WcspError(st, last_error())
    return buf.raw


def generate_grid(shape, seed: int, lo: int, hi: int, z0: int = 0, z1: int = -1, stream=None):
    """(f1, f2) of planes [z0, z1) of the last axis as torch uint8 CUDA tensors of shape (d, Nl),
    generated on the device by wcsp_generate_grid (same values as instances.grid_values)."""
    import torch
    d = len(shape)
    sh = (ctypes.c_int64 * 4)(*[int(x) for x in shape], *([1] * (4 - d)))
    nL = int(shape[-1])
    z1 = nL if z1 < 0 else z1
    Nl = (z1 - z0) * int(np.prod(shape[:-1], dtype=np.int64))
    f1 = torch.empty((d, Nl), dtype=torch.uint8, device="cuda")
    f2 = torch.empty((d, Nl), dtype=torch.uint8, device="cuda")
    s = stream if stream is not None else torch.cuda.current_stream()
    st = load_library().wcsp_generate_grid(d, sh, int(seed) & ((1 << 64) - 1), int(lo), int(hi), int(z0), int(z1),
                                           f1.data_ptr(), f2.data_ptr(), s.cuda_stream)
    if st != REACHED:
        raise WcspError(st, last_error())
    return f1, f2


def generate_mask(shape, rule: str, z0: int = 0, z1: int = -1, stream=None):
    """Vertex set `rule` (instances.set_mask rules face0/face1/boundary/centre/corner0/corner1) of
    planes [z0, z1), as a torch uint8 CUDA tensor, generated by wcsp_generate_mask."""
    import torch
    d = len(shape)
    sh = (ctypes.c_int64 * 4)(*[int(x) for x in shape], *([1] * (4 - d)))
    nL = int(shape[-1])
    z1 = nL if z1 < 0 else z1
    Nl = (z1 - z0) * int(np.prod(shape[:-1], dtype=np.int64))
    out = torch.empty(Nl, dtype=torch.uint8, device="cuda")
    s = stream if stream is not None else torch.cuda.current_stream()
    st = load_library().wcsp_generate_mask(d, sh, SET_RULES[rule], int(z0), int(z1), out.data_ptr(), s.cuda_stream)
    if st != REACHED:
        raise WcspError(st, last_error())
    return out


def slab_planes(n_last: int, nranks: int, rank: int):
    """(z0, z1, p0, p1): slab `rank` owns planes [z0, z1) of the last axis; with
    Solver(local_slab=True) its arrays cover planes [p0, p1) (ghosts included)."""
    out = (ctypes.c_int64 * 4)()
    st = load_library().wcsp_slab_planes(int(n_last), int(nranks), int(rank), out)
    if st != REACHED:
        raise WcspError(st, last_error())
    return tuple(int(x) for x in out)


def version() -> str:
    return load_library().wcsp_version().decode()
