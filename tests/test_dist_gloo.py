"""CPU: the multi-GPU host logic (paper_2006_11494_b200/dist.py) over a real
world_size-2 process group on gloo -- the same calls bench.py makes over NCCL."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2006_11494_b200 import dist as tdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        big = (1 << 64) - 5  # sums wrap mod 2^64 exactly like the hash sum
        stats = [
            dict(triangles=10, positive_triangles=6, negative_triangles=4, probes=100, probes_executed=90,
                 table_builds=7, hash_sum=big, hash_xor=0xF0F0),
            dict(triangles=5, positive_triangles=1, negative_triangles=4, probes=50, probes_executed=45,
                 table_builds=3, hash_sum=9, hash_xor=0x0FF0),
        ][rank]
        out = tdist.reduce_stats(stats)
        off, total = tdist.listing_offsets([7, 11][rank])
        mx = tdist.max_over_ranks([1.5, 2.5][rank])
        q.put((rank, out, off, total, mx))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_reduce_stats_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=100) for _ in range(2))
    for p in procs:
        p.join(30)
        assert p.exitcode == 0
    for rank, out, off, total, mx in res:
        assert out["triangles"] == 15
        assert out["positive_triangles"] == 7 and out["negative_triangles"] == 8
        assert out["probes"] == 150 and out["probes_executed"] == 135 and out["table_builds"] == 10
        assert out["hash_sum"] == ((1 << 64) - 5 + 9) % (1 << 64)
        assert out["hash_xor"] == 0xF0F0 ^ 0x0FF0
        assert total == 18 and off == (0 if rank == 0 else 7)
        assert mx == 2.5
