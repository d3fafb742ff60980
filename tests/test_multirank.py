"""N > 1 host logic of bench.py on CPU: world_size-2 gloo ranks (the path shards as independent
replicas, so the only cross-rank step is the max-over-ranks device time)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, ws, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    sys.path.insert(0, ROOT)
    import bench
    ms_local = 10.0 + 5.0 * rank          # rank 1 is the slow one
    ms_step, value = bench.job_value(ms_local, ws)
    bench.barrier(ws)
    out[rank] = (ms_step, value)
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world_size_2():
    torch = pytest.importorskip("torch")
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for r in range(2):
        ms_step, value = out[r]
        assert ms_step == 15.0                 # max over ranks, identical on every rank
        assert value == 7.5                    # 2 replicas solved in one step time


def test_single_rank_value_is_local_time():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.job_value(12.5, 1) == (12.5, 12.5)
