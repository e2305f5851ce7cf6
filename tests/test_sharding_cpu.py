"""CPU: multi-GPU host logic -- band planning, pair sharding, trace merging
and the band gather over torch.distributed with the gloo backend
(world_size 2, 127.0.0.1 rendezvous)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1901_09593_b200 import sharding
from paper_1901_09593_b200.matcher import LevelTrace, PipelineTrace


def test_shard_pairs_partition():
    for world in (1, 2, 4, 8):
        got = sorted(i for r in range(world) for i in sharding.shard_pairs(64, world, r))
        assert got == list(range(64))
        assert all(len(sharding.shard_pairs(64, world, r)) == 64 // world for r in range(world))
    with pytest.raises(ValueError):
        sharding.shard_pairs(4, 2, 2)


@pytest.mark.parametrize("h,world,k", [(6144, 8, 5), (6144, 2, 5), (375, 3, 2), (992, 4, 3),
                                       (1984, 8, 4), (100, 1, 0)])
def test_plan_bands_aligned_partition(h, world, k):
    bands = sharding.plan_bands(h, world, k)
    assert len(bands) == world
    assert bands[0][0] == 0 and bands[-1][1] == h
    for (a0, a1), (b0, b1) in zip(bands, bands[1:]):
        assert a1 == b0
    for b0, b1 in bands:
        assert b0 % (1 << k) == 0 and (b1 % (1 << k) == 0 or b1 == h) and b1 > b0
    sizes = [b1 - b0 for b0, b1 in bands[:-1]]
    if sizes:
        assert max(sizes) - min(sizes) <= (1 << k)


def test_plan_bands_rejects_too_many_bands():
    with pytest.raises(ValueError):
        sharding.plan_bands(64, 8, 4)   # only 4 units of 16 rows


def _trace(vals):
    t = PipelineTrace()
    for lv, v in enumerate(vals):
        t.levels.append(LevelTrace(level=lv, height=8, width=8, d_max=4, block=3, trusted=v,
                                   trusted_evals=2 * v, trusted_window_max=v % 5,
                                   full_search_pixels=64 - v, selection_evals=3 * v,
                                   refined=v, refine_evals=5 * v, median_replaced=1))
    return t


def test_merge_traces_sums_and_maxes():
    m = sharding.merge_traces([_trace([1, 2]), _trace([3, 9])])
    assert [lt.trusted for lt in m.levels] == [4, 11]
    assert [lt.refine_evals for lt in m.levels] == [20, 55]
    assert [lt.trusted_window_max for lt in m.levels] == [3, 4]
    assert [lt.median_replaced for lt in m.levels] == [2, 2]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gather_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h, w = 70, 9
    bands = sharding.plan_bands(h, world, 3)
    b0, b1 = bands[rank]
    full = torch.arange(h * w, dtype=torch.int16).reshape(h, w)
    out = sharding.gather_bands(full[b0:b1].clone(), bands, rank, world)
    costs = sharding.gather_bands(full[b0:b1].float() * 0.5, bands, rank, world)
    # both maps in one collective (bench.py's C5 path); bands of unequal height
    d2, c2 = sharding.gather_maps(full[b0:b1].clone(), full[b0:b1].float() * 0.25, bands,
                                  rank, world)
    if rank == 0:
        q.put((bool(torch.equal(out, full)), bool(torch.equal(costs, full.float() * 0.5)),
               bool(torch.equal(d2, full)), bool(torch.equal(c2, full.float() * 0.25))))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_bands_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=10) == (True, True, True, True)
