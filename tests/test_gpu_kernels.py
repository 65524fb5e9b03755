"""GPU: the reference's comparison kernels (cf merge, cf-hash, kclist3;
engine.hpp:164-236) and the degeneracy / random orders on the device path,
through the C-ABI (tl_run_*, tl_degeneracy_order, tl_random_order) and the
Python mirror, against the oracle, the reference library and the reference's
golden values at full config size (tests/golden/kernels.json)."""
import json
import os

import numpy as np
import pytest

import oracle as O
from paper_2006_11494_b200 import capi
from paper_2006_11494_b200 import trilist
from paper_2006_11494_b200.configs import CONFIGS

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KERNELS = ("cf", "cf-hash", "kclist", "aot")
ORDERS = ("degree", "degeneracy", "id", "random:11")
COUNTERS = ("triangles", "probes", "merge_comparisons", "table_builds", "positive_triangles", "negative_triangles")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "kernels.json")


def device_oriented(n, pairs, order):
    g = capi.DeviceGraph.from_pairs(np.ascontiguousarray(pairs, np.uint32), n)
    return g, g.orient(g.make_order(order))


def multiset(a):
    return sorted(map(tuple, np.asarray(a).tolist()))


def test_k3_id_order_every_kernel():  # test_engine.cpp:31-59
    _, og = device_oriented(3, O.as_pairs(O.complete_graph(3)[1]), "id")
    st, raw = og.list(algo="cf")
    assert [st[k] for k in ("triangles", "probes", "merge_comparisons", "table_builds")] == [1, 0, 2, 0]
    assert raw.tolist() == [[0, 1, 2]]
    st = og.count(algo="cf-hash")
    assert (st["triangles"], st["probes"], st["table_builds"]) == (1, 1, 5)
    assert og.count(algo="cf-hash", reuse=True)["table_builds"] == 3
    st = og.count(algo="kclist")
    assert (st["triangles"], st["probes"], st["table_builds"]) == (1, 1, 3)
    assert st["positive_triangles"] == st["negative_triangles"] == 0


@pytest.mark.parametrize("i", range(0, 40, 4))
def test_kernels_and_orders_vs_oracle(i):
    """Counters, hash, raw role-ordered emissions and the canonical set of
    every kernel under every order equal the oracle's (pinned to the
    reference by tests/test_oracle_kernels.py)."""
    n = 5 + i * 7
    pairs = O.gen_gnp(n, [0.02, 0.1, 0.3][i % 3], 1000 + i)
    cg = O.OracleGraph(n, pairs)
    for order in ORDERS:
        g, og = device_oriented(n, pairs, order)
        rank = cg.make_order(order)
        assert np.array_equal(g.make_order(order), rank), order
        co = cg.orient(rank)
        for algo in KERNELS:
            for reuse in ((False, True) if algo == "cf-hash" else (False,)):
                want, raw = co.run(algo, reuse=reuse, collect=True)
                st = og.count(algo=algo, reuse=reuse)
                assert all(st[k] == want[k] for k in COUNTERS), (algo, order, reuse, st, want)
                h = og.hash(algo=algo, reuse=reuse)
                assert (h["hash_sum"], h["hash_xor"]) == (want["hash_sum"], want["hash_xor"])
                _, got = og.list(algo=algo, reuse=reuse)
                assert multiset(got) == multiset(raw), (algo, order)
                _, canon = og.list(algo=algo, canonical=True)
                assert np.array_equal(canon, O.canonical_sorted(raw))


def test_rmat_every_kernel_vs_reference():
    n, pairs = 1 << 14, O.gen_rmat(21, 14, 16 << 14)
    for order in ("degree", "degeneracy"):
        ref = O.RefGraph(n, pairs, order=order)
        g, og = device_oriented(n, pairs, order)
        assert np.array_equal(g.make_order(order), ref.oriented_csr()["rank"])
        for algo in KERNELS:
            for reuse in ((False, True) if algo == "cf-hash" else (False,)):
                want = ref.run(algo, threads=O.hardware_threads(), reuse=reuse, hash=True)
                got = og.hash(algo=algo, reuse=reuse)
                assert all(got[k] == want[k] for k in COUNTERS), (algo, order, reuse)
                assert (got["hash_sum"], got["hash_xor"]) == (want["hash_sum"], want["hash_xor"])


@pytest.mark.parametrize("nparts", [2, 3, 8])
def test_partitions_sum_to_whole_every_kernel(nparts):  # test_parallel.cpp:11-40 (+ the multi-GPU cut)
    n, pairs = 1 << 13, O.gen_rmat(5, 13, 16 << 13)
    for order in ("degree", "degeneracy"):
        _, og = device_oriented(n, pairs, order)
        for algo in KERNELS:
            whole = og.hash(algo=algo)
            parts = [og.hash(algo=algo, part=p, nparts=nparts) for p in range(nparts)]
            for k in COUNTERS + ("hash_sum", "probes_executed"):
                assert sum(p[k] for p in parts) % (1 << 64) == whole[k], (algo, order, k)
            # every part's counters are over one edge set (no per-part wrap-around)
            assert all(p["merge_comparisons"] < (1 << 63) for p in parts), algo
            assert whole["probes_executed"] <= max(whole["probes"], 1) or algo == "cf", algo
            x = 0
            for p in parts:
                x ^= p["hash_xor"]
            assert x == whole["hash_xor"]
            lists = [og.list(algo=algo, part=p, nparts=nparts)[1] for p in range(nparts)]
            assert multiset(np.concatenate(lists)) == multiset(og.list(algo=algo)[1])


def test_python_mirror_every_kernel():  # test_smoke.py:27-43 (every algo x id/degree/degeneracy)
    g = trilist.Graph.from_edges(7, [(u, v) for u in range(7) for v in range(u + 1, 7)])
    expected = trilist.brute_force_triangles(g)
    assert len(expected) == 35
    for algo in trilist.ALGORITHMS:
        for order in ("id", "degree", "degeneracy"):
            og = trilist.orient(g, order=order)
            assert trilist.list_triangles(og, algo=algo) == expected
    g6 = trilist.Graph.from_edges(6, [(u, v) for u in range(6) for v in range(u + 1, 6)])
    og = trilist.orient(g6, order="degree")
    costs = trilist.cost_model(og)
    assert trilist.run(og, algo="kclist")["probes"] == costs["kclist_cost"]
    assert trilist.run(og, algo="aot")["probes"] == costs["aot_cost"]
    assert trilist.run(og, algo="cf-hash")["probes"] == costs["aot_cost"]
    assert trilist.count_triangles(trilist.Graph.from_edges(4, [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)]),
                                   algo="cf") == 4
    report = trilist.verify_equivalence(trilist.Graph.from_edges(5, [(u, v) for u in range(5)
                                                                     for v in range(u + 1, 5)]))
    assert report["pass"] and report["reference_count"] == 10
    assert [r["algorithm"] for r in report["results"]] == ["cf", "cf-hash", "kclist", "aot"]


def test_merge_rejects_shuffled_layout():  # test_engine.cpp:187-193
    pairs = O.gen_gnp(60, 0.1, 2)
    g = trilist.Graph.from_array(60, pairs)
    shuffled = trilist.orient(g, local_order="random:1")
    with pytest.raises(ValueError, match="rank-ascending"):
        trilist.run(shuffled, algo="cf")
    assert trilist.run(trilist.orient(g), algo="cf")["triangles"] == len(trilist.brute_force_triangles(g))


def test_reuse_on_host_layouts_matches_reference():  # engine.hpp:200-206 on degree-desc / random lists
    pairs = O.gen_gnp(150, 0.08, 15)
    g = trilist.Graph.from_array(150, pairs)
    for local in ("rank-asc", "degree-desc", "random:5"):
        ref = O.RefGraph(150, pairs, local=local).run("cf-hash", reuse=True)
        got = trilist.run(trilist.orient(g, local_order=local), algo="cf-hash", cf_hash_reuse_last_table=True)
        assert all(got[k] == ref[k] for k in COUNTERS), local


def test_verify_anchors_on_first_algorithm_and_catches_fault():  # test_engine.cpp:257-288
    pairs = O.gen_gnp(160, 0.07, 23)
    g = trilist.Graph.from_array(160, pairs)
    anchored = trilist.verify_equivalence(g, order="degeneracy", against_oracle=False)
    assert anchored["pass"] and anchored["reference"] == "cf"
    bad = trilist.verify_equivalence(g, skip_negative_phase=True)
    assert not bad["pass"]
    aot = bad["results"][-1]
    assert aot["algorithm"] == "aot" and aot["missing_count"] > 0 and aot["extra_count"] == 0
    assert all(r["pass"] for r in bad["results"][:-1])


def rank_checksum(rank: np.ndarray) -> str:  # as tests/golden/make_golden_kernels.py
    u = np.arange(rank.size, dtype=np.uint64)
    z = (u << np.uint64(32)) | rank.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
        return str(int(np.sum(z, dtype=np.uint64)))


def golden_configs():
    if not os.path.exists(GOLDEN):
        return []
    return sorted(json.load(open(GOLDEN)).keys())


@pytest.mark.slow
@pytest.mark.parametrize("key", golden_configs())
def test_full_config_every_kernel_vs_reference_golden(key):
    """Full-size configs (C1, C2): every kernel's counters and hash under the
    degree and degeneracy orders equal the reference's (tests/golden/kernels.json)."""
    import torch

    gold = json.load(open(GOLDEN))[key]
    cfg = CONFIGS[key]
    d = torch.empty(2 * cfg["npairs"], dtype=torch.int32, device="cuda")
    capi.gen_pairs_device(cfg, d.data_ptr())
    torch.cuda.synchronize()
    g = capi.DeviceGraph.from_device_pairs(d.data_ptr(), cfg["npairs"], cfg["n"])
    del d
    for order in ("degree", "degeneracy"):
        if order not in gold:
            continue
        rank = g.make_order(order)
        assert rank_checksum(rank) == gold[order]["rank_checksum"], order
        og = g.orient(rank)
        assert og.cost_model() == gold[order]["cost_model"]
        for name, want in gold[order]["kernels"].items():
            algo, reuse = name.split("+")[0], name.endswith("+reuse")
            got = og.hash(algo=algo, reuse=reuse)
            assert all(got[k] == want[k] for k in COUNTERS), (key, order, name, got, want)
            assert (got["hash_sum"], got["hash_xor"]) == (want["hash_sum"], want["hash_xor"]), (key, order, name)
        og.close()


def test_partitioned_listing_at_scale():
    """The multi-GPU cut at a size where the task size exceeds its floor
    (C3, 4 parts): every part's listing (buffer sized by a counting pass over
    the same part) succeeds and emits exactly its counted triangles, and the
    parts add up to the reference's total (tests/golden/configs.json)."""
    import torch

    cfg = CONFIGS["c3"]
    d = torch.empty(2 * cfg["npairs"], dtype=torch.int32, device="cuda")
    capi.gen_pairs_device(cfg, d.data_ptr())
    g = capi.DeviceGraph.from_device_pairs(d.data_ptr(), cfg["npairs"], cfg["n"])
    del d
    og = g.orient()
    g.close()
    torch.cuda.empty_cache()
    total, nparts = 0, 4
    for p in range(nparts):
        counted = og.count(part=p, nparts=nparts)["triangles"]
        s = capi.TlStats()
        o = capi.run_options(False, p, nparts)
        capi._check(capi.lib().tl_aot_list(og._h, capi.C.byref(o), None, 0, 0, capi.C.byref(s)))
        listed = s.as_dict()
        assert listed["triangles"] == counted, p
        assert og.hash(part=p, nparts=nparts)["triangles"] == counted, p
        total += counted
    golden = json.load(open(os.path.join(os.path.dirname(GOLDEN), "configs.json")))["c3"]
    assert total == golden["triangles"]
    og.close()


_EXEC_SNIPPET = r"""
import json, sys
sys.path.insert(0, {root!r})
import oracle as O
from paper_2006_11494_b200 import capi
pairs = O.gen_rmat(17, 13, 16 << 13)
do = capi.DeviceGraph.from_pairs(pairs, 1 << 13).orient()
out = {{}}
for algo in ("aot", "cf", "cf-hash", "kclist"):
    for mode in ("count", "hash"):
        run = do.count if mode == "count" else do.hash
        out[f"{{algo}}/{{mode}}"] = run(algo=algo)["probes_executed"]
        out[f"{{algo}}/{{mode}}/skip"] = run(algo=algo, skip_negative=True)["probes_executed"]
print(json.dumps(out))
"""


def test_probes_executed_matches_the_kernels_own_count():
    """probes_executed (computed outside the hot loop by k_executed from the
    early-exit rule) equals the count the kernel itself keeps when built with
    TL_EXEC_COUNT=1 (lib/variants/lib_exec_count.so), for every kernel, mode
    and the fault hook; and the parts of a split sum to the whole."""
    import json
    import subprocess
    import sys

    from paper_2006_11494_b200 import _build

    lib = os.path.join(_build.LIBDIR, "variants", "lib_exec_count.so")
    assert os.path.exists(lib), lib
    code = _EXEC_SNIPPET.format(root=ROOT)
    ref = json.loads(subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True,
                                    env=dict(os.environ, TL_LIB_PATH=lib)).stdout.strip().splitlines()[-1])
    ours = json.loads(subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                                     check=True).stdout.strip().splitlines()[-1])
    assert ours == ref
    assert all(v > 0 for k, v in ours.items() if not k.startswith("cf/"))
