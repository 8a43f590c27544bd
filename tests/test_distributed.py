"""Multi-rank host logic on CPU (gloo, world_size 2): LP-index sharding
reproduces the single-process batch exactly (seeds keyed by global index),
per-rank oracle results concatenate to the full-batch results, and the
bench's MAX-over-ranks timing reduction. No data-path collective exists."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle_py as O
    from paper_1902_04995_b200 import sharding

    sizes = np.array([17, 300, 64, 1024, 5] * 8, np.int32)
    lo, pb = sharding.generate_shard(sizes, 11, rank, world)
    res = O.solve_batch(pb.astype(np.float32))
    local = torch.tensor([float(lo), float(pb.n), float(res["value"].astype(np.float64).sum()),
                          float(res["work_units"].sum())], dtype=torch.float64)
    gathered = [torch.zeros(4, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, local)
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        q.put(([g.tolist() for g in gathered], float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_solve_matches_single_process():
    import sys

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle_py as O
    import paper_1902_04995_b200 as P

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    sizes = np.array([17, 300, 64, 1024, 5] * 8, np.int32)
    full = O.solve_batch(P.PackedBatch.generate(sizes, 11).astype(np.float32))
    cut = [int(g[0]) for g in gathered] + [len(sizes)]
    for r, g in enumerate(gathered):
        lo, hi = cut[r], cut[r + 1]
        assert int(g[1]) == hi - lo
        assert g[2] == float(full["value"][lo:hi].astype(np.float64).sum())
        assert g[3] == float(full["work_units"][lo:hi].sum())
