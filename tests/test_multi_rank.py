"""Multi-rank host logic on CPU (gloo, world_size 2): each rank generates its
contiguous element range independently and the union is bitwise the
single-rank input; the max-over-ranks timing reduction picks the slowest rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1310_1191_b200.partition import max_over_ranks, rank_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1310_1191_b200 as pb

    nx, ny, nz = 5, 3, 4
    total = 2 * nx * ny * nz
    first, count = rank_range(total, world, rank)
    geom = pb.generate_box_mesh(nx, ny, nz, 0.2, 42, first=first, count=count, soa=True)
    coef = pb.generate_cdr_coefficients(42, first, count, soa=True)
    # gather the shards (variable sizes) on every rank
    sizes = [None] * world
    dist.all_gather_object(sizes, count)
    shards = [None] * world
    dist.all_gather_object(shards, (first, geom, coef))
    slow = max_over_ranks(1.0 + rank, dist)
    if rank == 0:
        q.put((total, sizes, shards, slow))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_inputs_reassemble_bitwise(world):
    import paper_1310_1191_b200 as pb

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    total, sizes, shards, slow = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum(sizes) == total and max(sizes) - min(sizes) <= 1
    full_g = pb.generate_box_mesh(5, 3, 4, 0.2, 42, soa=True)
    full_c = pb.generate_cdr_coefficients(42, 0, total, soa=True)
    got_g = np.concatenate([s[1] for s in sorted(shards, key=lambda s: s[0])], axis=1)
    got_c = np.concatenate([s[2] for s in sorted(shards, key=lambda s: s[0])], axis=1)
    assert np.array_equal(got_g, full_g)
    assert np.array_equal(got_c, full_c)
    assert slow == float(world)


def test_rank_range_covers_disjointly():
    for n in (0, 1, 7, 1 << 20):
        for world in (1, 2, 3, 8):
            spans = [rank_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0
            for (a, na), (b, _) in zip(spans, spans[1:]):
                assert a + na == b
            assert sum(c for _, c in spans) == n
    with pytest.raises(ValueError):
        rank_range(10, 2, 2)
