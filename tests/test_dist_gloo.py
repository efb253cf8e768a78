"""Multi-process host logic on CPU: world_size-2 gloo process group.

Covers what every rank of a multi-GPU run does on the host before and
around the device path: the block rank layout, the CUDA-IPC blob exchange
(fake blobs here), agreement on the deterministic straggler schedule, and
the max-over-ranks timing reduction bench.py reports.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2005_00124_b200.dist import exchange_blobs, gpu_of_rank, max_over_ranks, rank_layout
from paper_2005_00124_b200.straggler import StragglerPolicy


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
    try:
        P = 8
        local = rank_layout(P, world, rank)
        gathered = [None] * world
        dist.all_gather_object(gathered, list(local))
        blobs = exchange_blobs(rank, bytes([rank]) * 72)
        pol = StragglerPolicy(2, 3.2, selection_seed=12)
        vict = [sorted(pol.victims(t, P)) for t in range(20)]
        all_vict = [None] * world
        dist.all_gather_object(all_vict, vict)
        mx = max_over_ranks(float(rank) * 1.5 + 0.25)
        q.put((rank, gathered, {k: v[:1] for k, v in blobs.items()}, all_vict, mx))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_host_logic(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    for rank, gathered, blobs, all_vict, mx in res:
        # block layout partitions the ranks, rank r on GPU r // (P/G)
        assert sorted(r for g in gathered for r in g) == list(range(8))
        for g, ranks in enumerate(gathered):
            assert all(gpu_of_rank(r, 8, world) == g for r in ranks)
        assert blobs == {g: bytes([g]) for g in range(world)}
        assert all(v == all_vict[0] for v in all_vict)  # every rank sees the same victims
        assert mx == (world - 1) * 1.5 + 0.25


def test_rank_layout_validation():
    assert list(rank_layout(8, 4, 3)) == [6, 7]
    with pytest.raises(ValueError):
        rank_layout(8, 3, 0)
    with pytest.raises(ValueError):
        rank_layout(8, 2, 2)
    assert max_over_ranks(3.0) == 3.0  # no process group: identity
