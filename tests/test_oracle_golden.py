"""CPU: pin the oracle (oracle/trilist_oracle.c, the C restatement) to the
reference's own known answers and to the reference library itself
(oracle/_ref, built from the unmodified /root/reference sources).

Known-answer values restate proj/tests/test_engine.cpp, test_oracle.cpp,
test_ordering.cpp and acceptance.cpp.
"""
import json
import os

import numpy as np
import pytest

import oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
STAT_KEYS = ("triangles", "probes", "table_builds", "positive_triangles", "negative_triangles")


def orient_with(n, edges, rank=None):
    g = O.OracleGraph(n, O.as_pairs(edges))
    return g, g.orient(None if rank is None else np.asarray(rank, np.uint32))


def test_k3_id_order():  # test_engine.cpp:61-73
    g, og = orient_with(*O.complete_graph(3), rank=[0, 1, 2])
    st, raw = og.aot(collect=True)
    assert (st["triangles"], st["probes"], st["table_builds"]) == (1, 1, 3)
    assert st["positive_triangles"] + st["negative_triangles"] == 1
    assert og.cost_model() == {"cf_cost": 6, "kclist_cost": 1, "aot_cost": 1}


def test_k4_and_oracle_fixtures():  # test_engine.cpp:76-85, test_oracle.cpp:11-17
    g, og = orient_with(*O.complete_graph(4), rank=[0, 1, 2, 3])
    assert og.aot()[0]["triangles"] == 4
    assert O.OracleGraph(3, O.as_pairs(O.complete_graph(3)[1])).brute_force().tolist() == [[0, 1, 2]]
    assert len(O.OracleGraph(*O.cycle_graph(5)).brute_force()) == 0
    assert len(O.OracleGraph(*O.star_graph(6)).brute_force()) == 0
    n, e = O.diamond_graph()
    assert O.OracleGraph(n, O.as_pairs(e)).brute_force().tolist() == [[0, 1, 2], [1, 2, 3]]
    assert len(O.OracleGraph(0, O.as_pairs([])).brute_force()) == 0


def test_paired_hubs():  # test_engine.cpp:87-108, test_oracle.cpp:43-48, acceptance.cpp:216-231
    n, e = O.paired_hubs_graph()
    g, og = orient_with(n, e)
    assert g.degree_order().tolist() == list(range(14))  # degree order == id order here
    cm = og.cost_model()
    assert (cm["kclist_cost"], cm["aot_cost"]) == (21, 12)
    st, raw = og.aot(collect=True)
    assert (st["probes"], st["triangles"]) == (12, 6)
    want = [[6, 9, 12], [6, 9, 13], [7, 10, 12], [7, 10, 13], [8, 11, 12], [8, 11, 13]]
    assert O.canonical_sorted(raw).tolist() == want
    assert g.brute_force().tolist() == want
    assert og.max_out_degree() == 3  # test_cli.cpp:200-209


def test_diamond_fault_injection():  # test_engine.cpp:240-255
    n, e = O.diamond_graph()
    g, og = orient_with(n, e, rank=[0, 1, 2, 3])
    st = og.aot()[0]
    assert (st["triangles"], st["positive_triangles"], st["negative_triangles"]) == (2, 1, 1)
    st = og.aot(skip_negative=True)[0]
    assert (st["triangles"], st["negative_triangles"]) == (1, 0)


def test_zero_cases():  # test_engine.cpp:110-134
    n, e = O.star_graph(5)
    for rank in (None, list(range(6))):
        g, og = orient_with(n, e, rank)
        assert og.cost_model()["aot_cost"] == 0
        st = og.aot()[0]
        assert (st["triangles"], st["probes"]) == (0, 0)
    g, og = orient_with(0, [])
    st = og.aot()[0]
    assert (st["triangles"], st["probes"], st["table_builds"]) == (0, 0, 0)


def test_degree_order_known():  # test_ordering.cpp:28-41
    assert O.OracleGraph(*O.star_graph(4)).degree_order().tolist() == [4, 0, 1, 2, 3]
    assert O.OracleGraph(*O.path_graph(3)).degree_order().tolist() == [0, 2, 1]
    assert O.OracleGraph(*O.complete_graph(4)).degree_order().tolist() == [0, 1, 2, 3]


def test_orient_rejects_non_permutation():  # test_ordering.cpp:84-91
    g = O.OracleGraph(*O.path_graph(3))
    with pytest.raises(ValueError):
        g.orient(np.array([0, 0, 1], np.uint32))


def test_complete_graphs_closed_form():  # acceptance.cpp:252-268
    for n in range(3, 26):
        g, og = orient_with(*O.complete_graph(n))
        assert og.aot()[0]["triangles"] == n * (n - 1) * (n - 2) // 6


@pytest.mark.parametrize("seed", [7, 8, 9])
def test_gnp_vs_brute_force(seed):  # test_engine.cpp:136-150
    pairs = O.gen_gnp(200, 0.05, seed)
    g = O.OracleGraph(200, pairs)
    bf = g.brute_force()
    for rank in (None, np.arange(200, dtype=np.uint32), np.random.default_rng(3).permutation(200)):
        og = g.orient(rank)
        st, raw = og.aot(collect=True)
        assert np.array_equal(O.canonical_sorted(raw), bf)
        assert st["probes"] == og.cost_model()["aot_cost"]  # test_engine.cpp:152-170
        assert st["positive_triangles"] + st["negative_triangles"] == st["triangles"]


def test_acceptance_sweep_vs_reference():
    """acceptance.cpp:146-214: 21 fixtures + 200 G(n, p) graphs; the C
    restatement must equal the reference library bit for bit: CSR, degree
    order, orientation, cost model, counters, raw emissions, hash."""
    suite = [O.complete_graph(n) for n in range(3, 11)]
    suite += [O.star_graph(k) for k in (3, 4, 7, 10)] + [O.path_graph(n) for n in (2, 5, 9)]
    suite += [O.cycle_graph(n) for n in (3, 4, 5, 9)] + [O.diamond_graph(), O.paired_hubs_graph()]
    suite = [(n, O.as_pairs(e)) for n, e in suite]
    ps = (0.02, 0.1, 0.3)
    for i in range(200):
        n = 5 + i * 295 // 199
        suite.append((n, O.gen_gnp(n, ps[i % 3], 0xACCE5500 + i)))
    assert len(suite) == 221
    for n, pairs in suite:
        g = O.OracleGraph(n, pairs)
        ref = O.RefGraph(n, pairs)
        off, adj = g.csr()
        roff, radj = ref.graph_csr()
        assert np.array_equal(off, roff) and np.array_equal(adj, radj)
        og = g.orient()
        a, b = og.csr(), ref.oriented_csr()
        for k in a:
            assert np.array_equal(a[k], b[k]), k
        assert og.cost_model() == ref.cost_model()
        st, raw = og.aot(collect=True)
        rst, rraw = ref.collect(threads=2)
        for k in STAT_KEYS:
            assert st[k] == rst[k], k
        key = lambda r: r[np.lexsort((r[:, 2], r[:, 1], r[:, 0]))] if len(r) else r  # noqa: E731
        assert np.array_equal(key(raw), key(rraw))
        h = ref.hash(threads=2)
        assert (st["hash_sum"], st["hash_xor"]) == (h["hash_sum"], h["hash_xor"])
        assert np.array_equal(O.canonical_sorted(raw), ref.brute_force(max_vertices=n))


def test_parallel_determinism_reference():  # test_parallel.cpp:11-40
    pairs = O.gen_gnp(300, 0.05, 0xDE7E3311)
    ref = O.RefGraph(300, pairs)
    base = ref.count(threads=1)
    og = O.OracleGraph(300, pairs).orient()
    st = og.aot()[0]
    for w in (1, 2, 4, 8):
        for chunk in (1, 7, 64, 1000):
            got = ref.count(threads=w, chunk=chunk)
            for k in STAT_KEYS:
                assert got[k] == base[k] == st[k]


def test_golden_c1_list_and_generators():
    g = json.load(open(os.path.join(HERE, "golden", "configs.json")))
    from paper_2006_11494_b200.configs import CONFIGS

    c1 = g["c1"]
    pairs = O.gen_config(CONFIGS["c1"])
    assert O.pairs_checksum(pairs) == c1["pairs_checksum"]
    og = O.OracleGraph(CONFIGS["c1"]["n"], pairs).orient()
    st, raw = og.aot(collect=True)
    for k in STAT_KEYS:
        assert st[k] == c1[k]
    canon = O.canonical_sorted(raw)
    assert np.array_equal(canon, np.load(os.path.join(HERE, "golden", c1["list_file"])))
    assert O.hash_of_triples(canon) == (c1["triangles"], c1["hash_sum"], c1["hash_xor"])
    assert (st["hash_sum"], st["hash_xor"]) == (c1["hash_sum"], c1["hash_xor"])
    for key in ("c2", "c3"):  # generator definitions pinned by the reference-run checksums
        if key in g:
            first = O.gen_config(dict(CONFIGS[key], npairs=8))
            assert first.tolist() == g[key]["first_pairs"], key


def test_triangle_hash_definition():
    # Z(v) = fmix64(v + golden); a triangle adds Z(a) Z(b) Z(c) mod 2^64 to hash_sum and
    # xors Z(a) & Z(b) & Z(c) into hash_xor (symmetric: no canonical order needed)
    M = (1 << 64) - 1
    a, b, c = 3, 17, 99
    za, zb, zc = (O.fmix64((v + 0x9E3779B97F4A7C15) & M) for v in (a, b, c))
    assert O.vertex_word(a) == za
    assert O.triangle_hash(a, b, c) == (za * zb * zc) & M == O.triangle_hash(c, a, b)
    assert O.triangle_hash_xor(a, b, c) == za & zb & zc == O.triangle_hash_xor(b, c, a)
    cnt, hs, hx = O.hash_of_triples(np.array([[a, b, c], [1, 2, 3]], np.uint32))
    assert cnt == 2
    assert hs == (O.triangle_hash(a, b, c) + O.triangle_hash(1, 2, 3)) & M
    assert hx == O.triangle_hash_xor(a, b, c) ^ O.triangle_hash_xor(1, 2, 3)


def test_draw_is_sequential_splitmix64():
    # draw(seed, k) is the k-th output of the reference's splitmix64 (ordering.cpp:13-19)
    state, seed = 42, 42
    for k in range(5):
        state = (state + 0x9E3779B97F4A7C15) & ((1 << 64) - 1)
        assert O.olib().or_draw(seed, k) == O.fmix64(state)
