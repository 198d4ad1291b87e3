"""Multi-rank runs of the CUDA path: every rank computes its shard of the
instances / trace seeds with the CUDA kernels on its own GPU (ranks share GPU 0 over gloo when
the box has one), and the rank-0 gather equals a single-process run byte for byte. Also the
driver's entry: `bench.py --gpus 2` spawns its own ranks."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from oracle_lib import Oracle
    import paper_2207_11428_b200 as miso
    from paper_2207_11428_b200.dist import gather_to_rank0, shard_csr, shard_range
    dev = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ctx = miso.Context(dev)
    # instances: the rank's contiguous CSR shard through the device search kernel
    speeds, offs = Oracle().gen_mixes(0xACCE91, 20001)
    lo, hi, loc_off, (r0, r1) = shard_csr(offs, rank, world)
    cand, obj = ctx.optimize_batch(torch.from_numpy(speeds[r0 * 5: r1 * 5]).cuda(),
                                   torch.from_numpy(loc_off.astype(np.int32)).cuda())
    torch.cuda.synchronize()
    gc = gather_to_rank0(cand.cpu().numpy(), len(offs) - 1, rank, world)
    go = gather_to_rank0(obj.cpu().numpy(), len(offs) - 1, rank, world)
    # trace seeds: the rank's seeds through the device simulator (miso, noisy predictor)
    s_lo, s_hi = shard_range(10, rank, world)
    traces = miso.generate_traces(range(s_lo, s_hi), 80, lambda_s=30.0)
    res = miso.simulate_batch(ctx, traces, miso.SimOptions(policy="miso", cluster_size=6,
                                                           predictor="noisy"))
    gm = gather_to_rank0(np.ascontiguousarray(res.metrics).view(np.uint8), 10 * res.metrics.itemsize,
                         rank, world)
    if rank == 0:
        q.put((gc, go, gm))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def test_two_ranks_cuda_shards_gather_byte_equal(ctx, oracle):
    import torch
    import torch.multiprocessing as mp
    import paper_2207_11428_b200 as miso
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    port = _free_port()
    procs = [mpc.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gc, go, gm = q.get(timeout=600)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    speeds, offs = oracle.gen_mixes(0xACCE91, 20001)
    cand, obj = ctx.optimize_batch(torch.from_numpy(speeds).cuda(),
                                   torch.from_numpy(offs.astype(np.int32)).cuda())
    assert np.array_equal(gc, cand.cpu().numpy())
    assert np.array_equal(go.view(np.uint64), obj.cpu().numpy().view(np.uint64))
    e, _, o = oracle.optimize_batch(speeds, offs)  # and the gathered decisions are the oracle's
    assert np.array_equal(ctx.decode(gc, offs)[0], e.astype(np.int32))
    traces = miso.generate_traces(range(10), 80, lambda_s=30.0)
    res = miso.simulate_batch(ctx, traces, miso.SimOptions(policy="miso", cluster_size=6,
                                                           predictor="noisy"))
    assert np.array_equal(gm, np.ascontiguousarray(res.metrics).view(np.uint8))


def test_bench_spawns_its_own_ranks():
    """`python bench.py --gpus 2` outside torchrun re-executes itself with 2 ranks (gloo with
    both on GPU 0 here) and rank 0 prints one line with n_gpus 2 and a byte-exact gather."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "5",
                        "--warmup", "3", "--no-cpu-baseline", "--no-secondary"],
                       capture_output=True, text=True, timeout=900, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2
    g = line["result_gather"]
    assert g["instances"] == 2 * 1_000_000 and g["rank0_shard_byte_exact"]
    assert line["value"] > 0 and line["e2e"]["value"] > 0
