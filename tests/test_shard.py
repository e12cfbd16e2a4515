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


@pytest.mark.gpu
def test_nccl_shard_path_single_rank(golden_dir):
    """The C-ABI NCCL path on one GPU (a real one-rank communicator): all-gather,
    per-shard best, and the sharded batch solve equal the local batch solve."""
    import numpy as np
    from golden_util import bits
    from paper_2407_13126_b200 import planner
    from paper_2407_13126_b200 import scenario as SC
    cases = golden_dir["random"][:6] + [c for c in golden_dir["c1"] if "S24" in c[0]]
    probs = [SC.Problem(SC.load_scenario(path), 0) for _, path, _ in cases]
    with planner.Planner(0) as pl:
        pl.shard_init(1, 0, pl.nccl_unique_id())
        got = pl.shard_allgather([1, -2, 3], 1)
        assert got.tolist() == [[1, -2, 3]]
        assert pl.shard_best(12.5) == (12.5, 0)
        opts, obj, status = pl.solve_batch_sharded(probs)
        ref_opts, ref_obj, ref_status, _, _ = pl.solve_batch(probs)
    assert (status == ref_status).all() and (status == 0).all()
    assert np.array_equal(opts, ref_opts)
    assert [bits(x) for x in obj] == [bits(x) for x in ref_obj]
    for (stem, _, g), o in zip(cases, obj):
        want = g.get("dp", {}).get("obj")
        if want:
            assert bits(o) == want, stem
