"""Multi-process host logic of the N > 1 paths, on CPU with gloo (-m "not gpu").

* the NCCL unique id of the multi-GPU slab engine is made on rank 0 and
  shared through torch.distributed; every rank must hold the same 128 bytes;
* bench.py's multi-rank reductions (max of the device times, sum of the work)
  follow the contract: value = all ranks' units / max time.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from bench import share_nccl_id, reduce_timing
    nid = share_nccl_id(rank)
    t, u = reduce_timing(10.0 * (rank + 1), 1000 * (rank + 1), "cpu")
    q.put((rank, nid, t, u))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_nccl_id_shared_and_timing_reduction(world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids = {o[1] for o in out}
    assert len(ids) == 1 and len(next(iter(ids))) == 128
    for _, _, t, u in out:
        assert t == 10.0 * world            # max over ranks
        assert u == sum(1000 * (r + 1) for r in range(world))
