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
        # the C-ABI's host fold (tl_fold_parts) over the gathered per-rank stats agrees
        from paper_2006_11494_b200 import capi

        gathered = [None, None]
        dist.all_gather_object(gathered, dict(stats, list_ms=[3.0, 4.0][rank]))
        folded, offsets = capi.fold_parts(gathered)
        q.put((rank, out, off, total, mx, folded, offsets))
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
    for rank, out, off, total, mx, folded, offsets in res:
        for k in ("triangles", "positive_triangles", "negative_triangles", "probes", "probes_executed",
                  "table_builds", "hash_sum", "hash_xor"):
            assert folded[k] == out[k], k
        assert offsets == [0, 10] and folded["list_ms"] == 4.0
        assert out["triangles"] == 15
        assert out["positive_triangles"] == 7 and out["negative_triangles"] == 8
        assert out["probes"] == 150 and out["probes_executed"] == 135 and out["table_builds"] == 10
        assert out["hash_sum"] == ((1 << 64) - 5 + 9) % (1 << 64)
        assert out["hash_xor"] == 0xF0F0 ^ 0x0FF0
        assert total == 18 and off == (0 if rank == 0 else 7)
        assert mx == 2.5


def test_fold_parts_host_logic():
    """tl_fold_parts (pure host, no device): sums wrap mod 2^64, xor folds,
    offsets are the exclusive scan of the parts' triangle counts, times are
    the slowest part's; an empty fold is all zeros."""
    from paper_2006_11494_b200 import capi

    M = 1 << 64
    parts = [dict(triangles=3, probes=M - 1, hash_sum=M - 2, hash_xor=0b1010, list_ms=1.0, prep_ms=0.5,
                  merge_comparisons=4),
             dict(triangles=0, probes=5, hash_sum=7, hash_xor=0b0110, list_ms=2.5, prep_ms=0.1),
             dict(triangles=9, probes=1, hash_sum=1, hash_xor=0b0001, list_ms=0.5, prep_ms=0.2,
                  merge_comparisons=M - 4)]
    total, offs = capi.fold_parts(parts)
    assert total["triangles"] == 12 and offs == [0, 3, 3]
    assert total["probes"] == (M - 1 + 5 + 1) % M
    assert total["hash_sum"] == (M - 2 + 7 + 1) % M
    assert total["hash_xor"] == 0b1010 ^ 0b0110 ^ 0b0001
    assert total["merge_comparisons"] == 0
    assert total["list_ms"] == 2.5 and total["prep_ms"] == 0.5
    empty, eoffs = capi.fold_parts([])
    assert empty["triangles"] == 0 and eoffs == []


def test_multi_create_validates_before_device_use():
    """The multi-GPU entry points reject bad arguments before touching a device."""
    from paper_2006_11494_b200 import capi

    h = capi.vp()
    devs = (capi.C.c_int * 1)(0)
    rc = capi.lib().tl_multi_create(None, devs, 1, capi.C.byref(h))
    assert rc == capi.TL_EINVAL
    assert capi.lib().tl_multi_count(None, None, None) == capi.TL_EINVAL
