"""Host logic of the multi-GPU path on CPU: balanced window shards and the
gloo (world size 2) all-reduce of the per-rank error sums into MSE/MAE."""
import os
import socket

import numpy as np
import pytest

from paper_2404_02445_b200.sharding import shard_windows


@pytest.mark.parametrize("B", [0, 1, 7, 2789, 10444])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shards_partition_the_batch(B, world):
    spans = [shard_windows(B, world, r) for r in range(world)]
    assert spans[0][0] == 0
    for (s0, n0), (s1, _) in zip(spans, spans[1:]):
        assert s0 + n0 == s1
    assert sum(n for _, n in spans) == B
    assert max(n for _, n in spans) - min(n for _, n in spans) <= 1


def test_traffic_split_matches_survey():
    assert [shard_windows(2789, 8, r)[1] for r in range(8)] == [349] * 5 + [348] * 3


def test_bad_requests():
    for args in [(10, 0, 0), (10, 2, 2), (-1, 2, 0)]:
        with pytest.raises(ValueError):
            shard_windows(*args)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2404_02445_b200.sharding import all_reduce_error_sums, shard_windows
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    y = rng.normal(size=(50, 3, 8))
    t = rng.normal(size=(50, 3, 8))
    s, n = shard_windows(50, world, rank)
    d = y[s:s + n] - t[s:s + n]
    sums = torch.tensor([(d * d).sum(), np.abs(d).sum(), d.size], dtype=torch.float64)
    mse, mae = all_reduce_error_sums(sums)
    q.put((rank, mse, mae))
    dist.destroy_process_group()


def test_gloo_error_allreduce_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(0)
    d = rng.normal(size=(50, 3, 8)) - rng.normal(size=(50, 3, 8))
    for _, mse, mae in res:
        assert abs(mse - (d * d).mean()) < 1e-12 and abs(mae - np.abs(d).mean()) < 1e-12
