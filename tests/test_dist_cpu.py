"""CPU tests of the N>1 path with torch.distributed gloo, world_size 2: instance and seed
sharding plus the rank-0 result gather reproduce the single-process result byte for byte.
(The per-shard compute here is the oracle standing in for each rank's GPU; the GPU path itself
is covered by the -m gpu tests.)"""
import os
import socket

import numpy as np
import pytest


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path[:0] = [str(root), str(root / "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from oracle_lib import Oracle
    from paper_2207_11428_b200.dist import gather_to_rank0, shard_csr
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle()
    speeds, offs = orc.gen_mixes(0xACCE91, 5001)
    lo, hi, loc_off, (r0, r1) = shard_csr(offs, rank, world)
    e, p, o = orc.optimize_batch(speeds[r0 * 5: r1 * 5], loc_off)
    ge = gather_to_rank0(e, len(offs) - 1, rank, world)
    go = gather_to_rank0(o, len(offs) - 1, rank, world)
    gp = gather_to_rank0(p[: r1 - r0], int(offs[-1]), rank, world) if world == 1 else None
    if rank == 0:
        q.put((ge, go))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_partition():
    from paper_2207_11428_b200.dist import shard_range
    for n in (0, 1, 7, 100, 1001):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_gloo_world2_sharded_optimize_matches_single(oracle):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ge, go = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    speeds, offs = oracle.gen_mixes(0xACCE91, 5001)
    e, _, o = oracle.optimize_batch(speeds, offs)
    assert np.array_equal(ge, e)
    assert np.array_equal(go.view(np.uint64), o.view(np.uint64))
