"""CPU: the N>1 host logic (sharding + best-plan combine) over gloo, world size 2."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2407_13126_b200 import shard


def test_shard_ranges_cover_exactly():
    for n in (0, 1, 7, 4096):
        for world in (1, 2, 3, 8):
            got = []
            for r in range(world):
                lo, hi = shard.shard_range(n, r, world)
                got += list(range(lo, hi))
            assert got == list(range(n))


def test_objective_key_is_monotone():
    xs = [0.0, 1e-300, 0.5, 1.0, 12.5, 34303.47, 1e300]
    keys = [shard.objective_key(x) for x in xs]
    assert keys == sorted(keys)
    assert all(shard.key_objective(k) == x for k, x in zip(keys, xs))
    with pytest.raises(ValueError):
        shard.objective_key(-1.0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, objectives, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    best, owner = shard.combine_best(objectives[rank], rank, world)
    out[rank] = (best, owner)
    dist.destroy_process_group()


@pytest.mark.parametrize("objectives,expect", [([10.0, 12.5], (12.5, 1)), ([7.0, 7.0], (7.0, 0)),
                                               ([34303.47, 0.0], (34303.47, 0))])
def test_combine_best_gloo_world2(objectives, expect):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), objectives, out), nprocs=2, join=True)
    assert out[0] == expect and out[1] == expect
