"""The device-side instance generator (wcsp_generate_grid / wcsp_generate_mask,
include/wcsp.h) reproduces the host recipe of paper_1511_06441_b200/instances.py
byte for byte — whole grids and any slab of planes [z0, z1) of the last axis —
so a rank can build only its own slab of a 1024^3 cube in HBM (-m gpu)."""
import numpy as np
import pytest
import torch

import oracle
from paper_1511_06441_b200 import instances as I
from paper_1511_06441_b200 import wcsp

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,seed,lo,hi", [((7,), 3, 1, 5), ((33, 17), 11, 1, 10), ((16, 9, 5), 0, 1, 10),
                                             ((3, 4, 5, 6), 77, 200, 255), ((1, 40, 1), 5, 1, 1),
                                             ((64, 64, 64), 12345678901234, 1, 255)])
def test_grid_values_byte_equal(shape, seed, lo, hi):
    f1h, f2h = I.grid_values(shape, seed, lo, hi)
    f1d, f2d = wcsp.generate_grid(shape, seed, lo, hi)
    torch.cuda.synchronize()
    assert np.array_equal(f1d.cpu().numpy(), f1h) and np.array_equal(f2d.cpu().numpy(), f2h)
    # every slab of planes: the rows of the whole grid's planes [z0, z1)
    nL, plane = shape[-1], int(np.prod(shape[:-1]))
    rng = np.random.default_rng(seed % 1000)
    for _ in range(4):
        z0 = int(rng.integers(0, nL))
        z1 = int(rng.integers(z0, nL + 1))
        a, b = wcsp.generate_grid(shape, seed, lo, hi, z0, z1)
        assert np.array_equal(a.cpu().numpy(), f1h[:, z0 * plane:z1 * plane])
        assert np.array_equal(b.cpu().numpy(), f2h[:, z0 * plane:z1 * plane])


@pytest.mark.parametrize("shape", [(16, 16), (9, 8, 7), (5, 1, 4), (3, 3, 3, 3), (1, 1, 6)])
def test_masks_byte_equal(shape):
    for rule in ("face0", "face1", "boundary", "centre", "corner0", "corner1"):
        want = I.set_mask(shape, rule)
        got = wcsp.generate_mask(shape, rule).cpu().numpy()
        assert np.array_equal(got, want), rule
        nL, plane = shape[-1], int(np.prod(shape[:-1]))
        got = wcsp.generate_mask(shape, rule, 1, nL).cpu().numpy()
        assert np.array_equal(got, want[plane:]), rule


def test_device_generated_problem_solves_like_host():
    """A face-to-face cube generated in HBM and handed to the solver as device
    arrays gives the host instance's outputs and counters (and the oracle's)."""
    inst = I.config_face((40, 40, 40), 9, 230)
    f1, f2 = wcsp.generate_grid(inst.shape, 9, 1, 10)
    A, B = wcsp.generate_mask(inst.shape, "face0"), wcsp.generate_mask(inst.shape, "face1")
    s = torch.cuda.current_stream()
    with wcsp.Solver(shape=inst.shape, f1=f1, f2=f2, maskA=A, maskB=B, M=230, engine="wheel", stream=s) as sv:
        r = sv.solve()
    rh = wcsp.solve(inst, engine="wheel")
    assert r.key() == rh.key() == oracle.solve_pruned(inst).key()
    assert (r.edge_updates, r.arrivals, r.phantoms_created) == (rh.edge_updates, rh.arrivals, rh.phantoms_created)


def test_generator_rejects_bad_arguments():
    for args in (((8, 8), 1, 0, 5), ((8, 8), 1, 5, 4), ((8, 8), 1, 1, 256)):
        with pytest.raises(wcsp.WcspError) as e:
            wcsp.generate_grid(*args)
        assert e.value.status == wcsp.EINVAL
    with pytest.raises(wcsp.WcspError):
        wcsp.generate_grid((8, 8), 1, 1, 5, 3, 9)


@pytest.mark.parametrize("halo", ["copy", "peer"])
def test_local_slab_problem_single_rank(halo):
    """options.local_slab (include/wcsp.h): a rank passes only its own planes —
    here device-generated — validates them and combines the counts over NCCL;
    at one rank the slab is the whole grid, so the outputs and counters equal the
    single-device run's and the oracle's."""
    inst = I.config_face((36, 30, 24), 4, 210)
    z0, z1, p0, p1 = wcsp.slab_planes(inst.shape[-1], 1, 0)
    assert (z0, z1, p0, p1) == (0, 24, 0, 24)
    f1, f2 = wcsp.generate_grid(inst.shape, 4, 1, 10, p0, p1)
    A = wcsp.generate_mask(inst.shape, "face0", p0, p1)
    B = wcsp.generate_mask(inst.shape, "face1", p0, p1)
    torch.cuda.synchronize()
    with wcsp.Solver(shape=inst.shape, f1=f1, f2=f2, maskA=A, maskB=B, M=210, engine="wheel", halo=halo,
                     nranks=1, rank=0, nccl_id=wcsp.nccl_unique_id(), local_slab=True) as s:
        r = s.solve()
    r1 = wcsp.solve(inst, engine="wheel")
    assert r.key() == r1.key() == oracle.solve_pruned(inst).key()
    assert (r.cycles, r.edge_updates, r.arrivals, r.phantoms_created) == \
           (r1.cycles, r1.edge_updates, r1.arrivals, r1.phantoms_created)
    # the combined validation still rejects bad inputs
    bad = A.clone()
    bad[5] = 1
    Bb = B.clone()
    Bb[5] = 1
    with pytest.raises(wcsp.WcspError) as e:
        wcsp.Solver(shape=inst.shape, f1=f1, f2=f2, maskA=bad, maskB=Bb, M=210, engine="wheel", halo=halo,
                    nranks=1, rank=0, nccl_id=wcsp.nccl_unique_id(), local_slab=True)
    assert e.value.status == wcsp.EINVAL
