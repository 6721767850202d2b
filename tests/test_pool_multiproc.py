"""CPU multi-process checks of the N > 1 host logic (gloo, world size 2):
the store-backed dynamic image queue partitions the work exactly once, and
the MAX / SUM reductions used for the job-level throughput are right."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2108_10209_b200 import pool

    assert pool.dist_env() == (rank, rank, world)
    store = pool.default_store()
    dist.barrier()
    mine = list(pool.claim(store, "bench/next_image", total))
    got = [None] * world
    dist.all_gather_object(got, mine)
    t_max = pool.max_over_ranks(10.0 + rank)
    n_sum = pool.sum_over_ranks(len(mine))
    busy = pool.gather_over_ranks(10.0 + rank)
    if rank == 0:
        out.put((got, t_max, n_sum, busy, pool.imbalance(busy)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [1, 7, 64])
def test_dynamic_queue_partitions_images(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, t_max, n_sum, busy, imb = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    flat = sorted(i for shard in got for i in shard)
    assert flat == list(range(total))  # every image exactly once
    assert t_max == 11.0 and n_sum == total
    assert busy == [10.0, 11.0] and abs(imb - 11.0 / 10.5) < 1e-12


def test_static_shard_and_single_process_queue():
    from paper_2108_10209_b200 import pool

    assert pool.static_shard(5, 0, 2) == [0, 2, 4] and pool.static_shard(5, 1, 2) == [1, 3]
    assert list(pool.claim(None, "k", 3)) == [0, 1, 2]
    assert pool.max_over_ranks(3.5) == 3.5
