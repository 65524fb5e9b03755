"""CPU: pin the oracle's restatement of the reference's comparison kernels
(cf merge, cf-hash, kclist3; engine.hpp:164-236), of the degeneracy / random
vertex orders (ordering.cpp:86-120) and of the local orders
(ordering.cpp:229-266) to the reference's known answers and to the reference
library itself (oracle/_ref)."""
import numpy as np
import pytest

import oracle as O

KERNELS = ("cf", "cf-hash", "kclist", "aot")
ORDERS = ("degree", "degeneracy", "id", "random:11")


def oriented(n, edges, order="id"):
    g = O.OracleGraph(n, O.as_pairs(edges))
    return g, g.orient(g.make_order(order))


def test_k3_id_order_every_kernel():  # test_engine.cpp:31-59
    _, og = oriented(*O.complete_graph(3))
    st, raw = og.run("cf", collect=True)
    assert (st["triangles"], st["probes"], st["merge_comparisons"], st["table_builds"]) == (1, 0, 2, 0)
    assert raw.tolist() == [[0, 1, 2]]
    st, _ = og.run("cf-hash")
    assert (st["triangles"], st["probes"], st["table_builds"]) == (1, 1, 5)
    assert og.run("cf-hash", reuse=True)[0]["table_builds"] == 3
    st, _ = og.run("kclist")
    assert (st["triangles"], st["probes"], st["table_builds"]) == (1, 1, 3)


def test_paired_hubs_kclist():  # test_engine.cpp:87-108 (kclist_cost 21 = kclist probes)
    _, og = oriented(*O.paired_hubs_graph(), order="degree")
    assert og.run("kclist")[0]["probes"] == 21
    assert og.run("kclist")[0]["triangles"] == 6


@pytest.mark.parametrize("order", ORDERS)
def test_counter_identities(order):  # test_engine.cpp:152-170
    graphs = [O.paired_hubs_graph(), O.complete_graph(12), (120, O.gen_gnp(120, 0.1, 4)),
              (300, O.gen_gnp(300, 0.02, 5)), O.star_graph(9), O.cycle_graph(17), O.diamond_graph()]
    for n, e in graphs:
        _, og = oriented(n, e, order)
        cm = og.cost_model()
        assert og.run("kclist")[0]["probes"] == cm["kclist_cost"]
        assert og.run("aot")[0]["probes"] == cm["aot_cost"]
        assert og.run("cf-hash")[0]["probes"] == cm["aot_cost"]
        assert og.run("cf")[0]["merge_comparisons"] <= cm["cf_cost"]
        assert cm["aot_cost"] <= cm["kclist_cost"] <= cm["cf_cost"]


def test_phase_counters_only_for_aot():  # test_engine.cpp:195-206
    _, og = oriented(180, O.gen_gnp(180, 0.06, 1), "degree")
    for algo in ("cf", "cf-hash", "kclist"):
        st = og.run(algo)[0]
        assert st["positive_triangles"] == 0 and st["negative_triangles"] == 0


def test_reuse_only_reduces_builds():  # test_engine.cpp:229-238
    _, og = oriented(150, O.gen_gnp(150, 0.08, 15), "degree")
    plain, cached = og.run("cf-hash")[0], og.run("cf-hash", reuse=True)[0]
    assert cached["triangles"] == plain["triangles"] and cached["probes"] == plain["probes"]
    assert cached["table_builds"] <= plain["table_builds"]


def test_degeneracy_and_random_orders_known():  # test_ordering.cpp (permutation, smallest-last)
    n, e = O.star_graph(5)
    g = O.OracleGraph(n, O.as_pairs(e))
    d = g.degeneracy_order()
    # leaves 1..4 go first; then the hub (degree 1, id 0) precedes leaf 5
    assert d.tolist() == [4, 0, 1, 2, 3, 5]
    r = g.random_order(7)
    assert sorted(r.tolist()) == list(range(n))
    assert np.array_equal(r, g.random_order(7)) and not np.array_equal(r, g.random_order(8))


@pytest.mark.parametrize("i", range(0, 40, 3))
def test_kernels_orders_layouts_vs_reference(i):
    """Every kernel x order x local order on acceptance-style gnp graphs: the
    order, the six counters, the hash and the raw emission multiset equal the
    reference library's."""
    n = 5 + i * 7
    pairs = O.gen_gnp(n, [0.02, 0.1, 0.3][i % 3], 1000 + i)
    g = O.OracleGraph(n, pairs)
    for order in ORDERS:
        rank = g.make_order(order)
        for local in ("rank-asc", "degree-desc", "random:5"):
            ref = O.RefGraph(n, pairs, order=order, local=local)
            assert np.array_equal(ref.oriented_csr()["rank"], rank), order
            og = g.orient(rank)
            if local != "rank-asc":
                og.apply_local_order(local)
            for algo in KERNELS:
                if algo == "cf" and local != "rank-asc":
                    continue  # engine.hpp:143-149: cf rejects other layouts
                for reuse in ((False, True) if algo == "cf-hash" else (False,)):
                    st, raw = og.run(algo, reuse=reuse, collect=True)
                    r = ref.run(algo, reuse=reuse, hash=True)
                    assert all(st[k] == r[k] for k in O.STAT_KEYS), (algo, order, local, reuse)
                    assert (st["hash_sum"], st["hash_xor"]) == (r["hash_sum"], r["hash_xor"])
                    _, rraw = ref.collect_algo(algo, reuse=reuse)
                    assert sorted(map(tuple, raw.tolist())) == sorted(map(tuple, rraw.tolist()))


def test_reference_rejects_merge_on_shuffled_layout():  # test_engine.cpp:187-193
    pairs = O.gen_gnp(60, 0.1, 2)
    ref = O.RefGraph(60, pairs, local="random:1")
    with pytest.raises(RuntimeError, match="rank-ascending"):
        ref.run("cf")
