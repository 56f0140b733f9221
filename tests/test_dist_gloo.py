"""Multi-process (world_size 2, gloo on CPU) coverage of the sharded search's
only exchange step: the per-generation all-gather of rank elites."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2111_00655_b200.es_device import exchange_elites


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W = 3
        # rank r's best fitness; rank 1 holds the global best, rank 2.. ties
        vals = [5.0, 2.5, 2.5, 9.0]
        best = torch.tensor([vals[rank]], dtype=torch.float64)
        row = torch.full((1, W), 100 + rank, dtype=torch.int64)
        out_fit = torch.empty(world, dtype=torch.float64)
        out_rows = torch.empty((world, W), dtype=torch.int64)
        elite, val = exchange_elites(best, row, dist.group.WORLD, out_fit, out_rows)
        results[rank] = (elite.tolist(), float(val))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_elite_allgather_picks_global_best(world):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, results)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    # every rank adopts the same elite: the lowest fitness, first rank on ties
    want = ([[101, 101, 101]], 2.5)
    for r in range(world):
        assert results[r] == want
