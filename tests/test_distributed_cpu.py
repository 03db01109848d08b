"""Multi-process host logic of the data-parallel path on CPU: world_size 2 over gloo
(127.0.0.1).  Checks that the reduction of partial n x 73 matrices carried as int64 is the
uint64 sum modulo 2^64 bit for bit (wrap-around included), which is what makes the
sharded GPU result identical for any number of ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _partials(world, n, seed):
    rng = np.random.default_rng(seed)
    parts = [rng.integers(0, 1 << 63, size=(n, 73), dtype=np.uint64) * np.uint64(2) + np.uint64(r)
             for r in range(world)]
    return parts


def _worker(rank, world, port, n, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1911_10616_b200.parallel import reduce_partials
        parts = _partials(world, n, seed)
        t = torch.from_numpy(parts[rank].view(np.int64).copy())
        reduce_partials(t, dst=0)
        if rank == 0:
            q.put(t.numpy().view(np.uint64).copy())
        t2 = torch.from_numpy(parts[rank].view(np.int64).copy())
        reduce_partials(t2, all_ranks=True)
        q.put((rank, t2.numpy().view(np.uint64).copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_reduce_of_partials_is_mod_2_64_sum(world):
    n, seed = 257, 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world + 1)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts = _partials(world, n, seed)
    expect = np.zeros((n, 73), np.uint64)
    with np.errstate(over="ignore"):
        for p_ in parts:
            expect += p_
    reduced = [r for r in results if not isinstance(r, tuple)][0]
    assert np.array_equal(reduced, expect)
    for r in results:
        if isinstance(r, tuple):
            assert np.array_equal(r[1], expect)
