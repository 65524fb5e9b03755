"""GPU: the reference-shaped Python API (paper_2006_11494_b200.trilist, the
mirror of trilist._core) -- restates proj/tests/python/test_smoke.py against
the device path, plus the C++ facade's exception mapping."""
import itertools

import numpy as np
import pytest

import oracle as O
from paper_2006_11494_b200 import trilist

pytestmark = pytest.mark.gpu


def k(n):
    return trilist.Graph.from_edges(n, [(u, v) for u in range(n) for v in range(u + 1, n)])


def test_graph_shape_and_accessors():  # test_smoke.py:13-18
    g = trilist.Graph.from_edges(3, [(0, 1), (1, 2), (0, 2)])
    assert g.num_vertices == 3 and g.num_edges == 3
    assert g.has_edge(0, 2)
    assert g.neighbors(1) == [0, 2]
    assert g.degree(1) == 2
    with pytest.raises(IndexError):  # std::out_of_range (graph.cpp:209)
        g.degree(3)
    assert g.validate()


def test_from_edges_normalises():  # graph.cpp:189-206: self-loops dropped, duplicates collapsed
    g = trilist.Graph.from_edges(2, [(0, 1), (1, 0), (3, 3), (1, 2), (2, 1), (1, 2)])
    assert g.num_vertices == 4 and g.num_edges == 2
    assert g.duplicates_dropped == 3 and g.self_loops_dropped == 1


def test_all_algorithms_match_brute_force():  # test_smoke.py:27-33
    g = k(7)
    expected = trilist.brute_force_triangles(g)
    assert len(expected) == 35
    for algo, order in itertools.product(trilist.ALGORITHMS, ["id", "degree"]):
        og = trilist.orient(g, order=order)
        assert trilist.list_triangles(og, algo=algo) == expected


def test_counter_exactness():  # test_smoke.py:36-43
    g = k(6)
    og = trilist.orient(g, order="degree")
    costs = trilist.cost_model(og)
    assert costs["aot_cost"] <= costs["kclist_cost"] <= costs["cf_cost"]
    assert trilist.run(og, algo="aot")["probes"] == costs["aot_cost"]


def test_parallel_counters_deterministic():  # test_smoke.py:46-57
    edges = [(u, (u * 7 + 3) % 50) for u in range(50)] + [(u, (u * 11 + 5) % 50) for u in range(50)]
    g = trilist.Graph.from_edges(50, [(u, v) for u, v in edges if u != v])
    og = trilist.orient(g, order="degree")
    base = trilist.run(og, algo="aot", threads=1)
    for threads in (2, 4):
        got = trilist.run(og, algo="aot", threads=threads)
        for key in ("triangles", "probes", "table_builds"):
            assert got[key] == base[key]


def test_count_convenience_and_polarity():  # test_smoke.py:60-64
    g = k(4)
    assert trilist.count_triangles(g, algo="aot") == 4
    og = trilist.orient(g, order="id")
    assert trilist.edge_polarity(og, 0, 1) in ("positive", "negative")
    with pytest.raises(ValueError):  # ordering.cpp:272-274: missing edge
        trilist.edge_polarity(og, 1, 0)


def test_verify_equivalence_report():  # test_smoke.py:67-70
    report = trilist.verify_equivalence(k(5))
    assert report["pass"] and report["reference"] == "oracle"
    assert report["reference_count"] == 10
    assert {r["algorithm"] for r in report["results"]} == set(trilist.ALGORITHMS)


def test_verify_catches_fault_injection():  # test_engine.cpp:278-287
    pairs = O.gen_gnp(160, 0.07, 23)
    g = trilist.Graph.from_array(160, pairs)
    bad = trilist.verify_equivalence(g, skip_negative_phase=True)
    r = next(x for x in bad["results"] if x["algorithm"] == "aot")
    assert not bad["pass"] and r["missing_count"] > 0 and r["extra_count"] == 0
    assert 0 < len(r["missing_samples"]) <= 32


def test_argument_errors():
    og = trilist.orient(k(4))
    with pytest.raises(ValueError, match="unknown algorithm"):  # engine.cpp:22-23
        trilist.run(og, algo="cf_merge")
    with pytest.raises(ValueError, match="unknown order"):
        trilist.orient(k(4), order="fancy")
    with pytest.raises(ValueError, match="workers"):  # parallel.hpp:28-29
        trilist.run(og, threads=0)
    with pytest.raises(ValueError, match="chunk"):
        trilist.run(og, chunk=0)


def test_local_order_layouts_keep_counters():  # test_engine.cpp:172-185
    pairs = O.gen_gnp(150, 0.07, 42)
    g = trilist.Graph.from_array(150, pairs)
    base = trilist.run(trilist.orient(g))
    ref = O.RefGraph(150, pairs, local="degree-desc").oriented_csr()
    for local in ("degree-desc", "random:5"):
        og = trilist.orient(g, local_order=local)
        got = trilist.run(og)
        assert all(got[k] == base[k] for k in base if k != "wall_time_s")
        if local == "degree-desc":  # host-visible lists follow the reference's layout
            for u in range(150):
                s, e = ref["out_offsets"][u], ref["out_offsets"][u + 1]
                assert og.out_neighbors(u) == ref["out"][s:e].tolist()


def test_array_fast_paths_match_oracle():
    pairs = O.gen_rmat(9, 13, 16 << 13)
    g = trilist.Graph.from_array(1 << 13, pairs)
    og = trilist.orient(g)
    cpu = O.OracleGraph(1 << 13, pairs).orient()
    st, raw = cpu.aot(collect=True)
    arr = trilist.list_triangles_array(og)
    assert np.array_equal(arr, O.canonical_sorted(raw))
    h = trilist.hash_triangles(og)
    assert (h["triangles"], h["hash_sum"], h["hash_xor"]) == (st["triangles"], st["hash_sum"], st["hash_xor"])
    assert trilist.run(og)["probes"] == st["probes"]
