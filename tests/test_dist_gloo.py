"""Multi-process (world_size 2 and 3, gloo on CPU) coverage of the sharded
search's only exchange step: the per-generation all-gather of one elite
record per rank ([fitness bits, genome row]) and the pick rule the device
applies to the gathered records (lowest fitness, first rank on ties)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import numpy as np

from paper_2111_00655_b200.es_device import gather_records, pick_elite_host


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
        record = torch.empty((1, 1 + W), dtype=torch.int64)
        record[0, 0] = torch.tensor([vals[rank]], dtype=torch.float64).view(torch.int64)[0]
        record[0, 1:] = 100 + rank
        out = torch.empty((world, 1 + W), dtype=torch.int64)
        gather_records(record, dist.group.WORLD, out)
        recs = out.numpy()
        best, val = pick_elite_host(recs)
        results[rank] = ([recs[best, 1:].tolist()], val)
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
