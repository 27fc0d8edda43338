"""C-ABI library checks that need no GPU (-m "not gpu"): the library builds and
loads, exports every symbol include/wcsp.h declares, its host-only entry point
(wcsp_validate_path) agrees with the oracle, and the compute entry points fail
loudly instead of falling back to the CPU when no device is usable."""
import os
import re

import numpy as np
import pytest

import oracle
from paper_1511_06441_b200 import build, instances as I, wcsp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "wcsp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(wcsp_[a-z_]+)\s*\(", src)))


def test_library_builds_and_exports_every_declared_symbol():
    build.build()
    lib = wcsp.load_library()
    names = header_functions()
    assert set(names) == set(wcsp.EXPORTS), names
    for n in names:
        assert hasattr(lib, n), n
    # the exported dynamic symbols really are plain C names
    import subprocess
    out = subprocess.run(["nm", "-D", "--defined-only", wcsp.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", out, flags=re.M), n


def test_kernels_are_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", wcsp.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_validate_path_host_side_matches_oracle():
    rng = np.random.default_rng(3)
    for _ in range(30):
        inst = I.random_small(rng, shapes=[(5, 5), (4, 3, 2)], M_range=(5, 40))
        # a random walk from A that stops at the first B vertex (or after 12 steps)
        v = int(np.flatnonzero(inst.maskA)[0])
        path = [v]
        for _ in range(12):
            nb = [u for u in range(inst.N) if oracle.validate_path(inst.with_sets(
                maskA=np.eye(1, inst.N, v, dtype=np.uint8)[0], maskB=np.eye(1, inst.N, u, dtype=np.uint8)[0]),
                [v, u])[0] in (0, oracle.INFEASIBLE)]
            if not nb:
                break
            v = int(rng.choice(nb))
            path.append(v)
        got = wcsp.validate_path(inst, path)
        want = oracle.validate_path(inst, path)
        assert got[0] == want[0]
        if got[0] in (0, 1):
            assert got[1:] == want[1:]


def test_compute_entry_points_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(wcsp.WcspError) as e:
        wcsp.solve(I.fixture_B())
    assert e.value.status == wcsp.ECUDA


def test_budget_range_is_validated_before_any_device_work():
    """M beyond the wide-label range (include/wcsp.h WCSP_M_MAX_WIDE) or M < 1 is
    WCSP_EINVAL; a budget above the 16-bit range is NOT an error (PAPER.md:20,
    M in R+) — without a GPU it gets as far as the device (WCSP_ECUDA)."""
    import torch
    for bad in (0, -5, wcsp.M_MAX_WIDE + 1, 1 << 40):
        with pytest.raises(wcsp.WcspError) as e:
            wcsp.solve(I.fixture_B().with_M(bad))
        assert e.value.status == wcsp.EINVAL, bad
    if not torch.cuda.is_available():
        for ok in (wcsp.M_MAX + 1, 10 ** 6, wcsp.M_MAX_WIDE):
            with pytest.raises(wcsp.WcspError) as e:
                wcsp.solve(I.fixture_B().with_M(ok))
            assert e.value.status == wcsp.ECUDA, ok


def test_slab_planes_partition():
    """wcsp_slab_planes (host arithmetic): the slabs tile the last axis
    exactly, each holds its neighbours' boundary planes as ghosts, and bad
    arguments are WCSP_EINVAL."""
    for n, R in [(1024, 8), (256, 3), (7, 7), (100, 4), (5, 1)]:
        cover = []
        for r in range(R):
            z0, z1, p0, p1 = wcsp.slab_planes(n, R, r)
            assert z0 == r * n // R and z1 == (r + 1) * n // R and z1 > z0
            assert p0 == z0 - (r > 0) and p1 == z1 + (r < R - 1)
            cover += list(range(z0, z1))
        assert cover == list(range(n))
    for bad in [(4, 5, 0), (8, 2, 2), (8, 0, 0), (8, 2, -1)]:
        with pytest.raises(wcsp.WcspError) as e:
            wcsp.slab_planes(*bad)
        assert e.value.status == wcsp.EINVAL
