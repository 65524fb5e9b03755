"""Several GPUs from one process (tl_multi_*) and from several processes
(partitioned runs reduced over a process group).

The GPU pool has one device per box, so tl_multi runs with the device list
[0] here: the whole path (replica bookkeeping, one host thread per device,
ncclCommInitAll, the grouped ncclAllReduce / ncclAllGather of the counters,
xors and emission counts, the listing offsets) executes, and its results
must be bit-identical to the single-device calls.  The multi-process path
runs two gloo ranks that share the device (their kernels never wait on each
other) through the same per-part runs and reductions bench.py uses.
"""
import collections
import os
import socket

import numpy as np
import pytest

import oracle as O
from paper_2006_11494_b200 import capi

pytestmark = pytest.mark.gpu

KEYS = ("triangles", "probes", "merge_comparisons", "table_builds", "positive_triangles", "negative_triangles",
        "probes_executed", "hash_sum", "hash_xor")


def multiset(a):
    return collections.Counter(map(tuple, np.asarray(a).reshape(-1, 3).tolist()))


@pytest.mark.parametrize("algo", ["aot", "cf", "cf-hash", "kclist"])
def test_multi_device_list_of_one_equals_single_device(algo):
    pairs = O.gen_rmat(21, 13, 16 << 13)
    do = capi.DeviceGraph.from_pairs(pairs, 1 << 13).orient()
    mg = capi.MultiOriented(do, [0])
    single_h = do.hash(algo=algo)
    multi_h = mg.hash(algo=algo)
    for k in KEYS:
        assert multi_h[k] == single_h[k], (algo, k)
    multi_c = mg.count(algo=algo)
    assert multi_c["triangles"] == single_h["triangles"]
    st, tri = mg.list(algo=algo)
    assert st["triangles"] == single_h["triangles"]
    assert multiset(tri) == multiset(do.list(algo=algo)[1])
    mg.close()


def test_multi_create_rejects_bad_device_lists():
    pairs = O.gen_rmat(3, 10, 16 << 10)
    do = capi.DeviceGraph.from_pairs(pairs, 1 << 10).orient()
    for devs in ([0, 0], [99], [-1]):
        with pytest.raises(capi.TlError) as e:
            capi.MultiOriented(do, devs)
        assert e.value.code == capi.TL_EINVAL
    mg = capi.MultiOriented(do, [0])
    o = capi.run_options(part=1, nparts=2)
    st = capi.TlStats()
    assert capi.lib().tl_multi_count(mg._h, capi.C.byref(o), capi.C.byref(st)) == capi.TL_EINVAL


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2006_11494_b200 import dist as tdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        pairs = O.gen_rmat(31, 14, 16 << 14)
        do = capi.DeviceGraph.from_pairs(pairs, 1 << 14).orient()  # every rank builds the same replica
        part = do.hash(part=rank, nparts=world)
        whole = tdist.reduce_stats(part)
        _, tri = do.list(canonical=False, part=rank, nparts=world)
        off, total = tdist.listing_offsets(len(tri))
        gathered = [None] * world
        dist.all_gather_object(gathered, (off, tri))
        q.put((rank, whole, total, gathered, do.hash(), do.list()[1] if rank == 0 else None))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_two_ranks_partitioned_run_reduces_to_the_whole():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=500) for _ in range(2)), key=lambda r: r[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    ref_list = res[0][5]
    for rank, whole, total, gathered, single, _ in res:
        for k in ("triangles", "probes", "table_builds", "positive_triangles", "negative_triangles",
                  "probes_executed", "hash_sum", "hash_xor"):
            assert whole[k] == single[k], (rank, k)
        assert total == single["triangles"]
        out = np.empty((total, 3), np.uint32)
        for off, tri in gathered:  # each rank's emissions at its gathered offset
            out[off: off + len(tri)] = tri
        assert multiset(out) == multiset(ref_list)
