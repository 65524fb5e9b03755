"""GPU: verify_equivalence's comparison on the device (tl_verify: device
canonicalisation, sort, unique and set differences; engine.cpp:82-130),
against the oracle's sets on small graphs and against the reference's golden
counts at C2 full size."""
import numpy as np
import pytest

import oracle as O
from paper_2006_11494_b200 import capi
from paper_2006_11494_b200.configs import CONFIGS

pytestmark = pytest.mark.gpu

ALGOS = ("cf", "cf-hash", "kclist", "aot")


def canon_set(raw):
    return set(map(tuple, O.canonical_sorted(raw).tolist()))


@pytest.mark.parametrize("seed", [23, 24])
def test_verify_against_oracle_and_fault(seed):  # test_engine.cpp:257-288
    n = 160
    pairs = O.gen_gnp(n, 0.07, seed)
    cg = O.OracleGraph(n, pairs)
    bf = cg.brute_force()
    g = capi.DeviceGraph.from_pairs(pairs, n)
    og = g.orient()
    res, ref_count = og.verify(ALGOS, reference=bf[::-1].copy())  # any order in, sorted + unique on device
    assert ref_count == len(bf)
    for r in res:
        assert r["pass"] and r["unique_triangles"] == len(bf) and r["duplicate_emissions"] == 0
        assert r["missing_count"] == r["extra_count"] == 0 and r["missing_samples"] == []
    # anchored on the first algorithm when there is no oracle
    res, ref_count = og.verify(("kclist", "aot"))
    assert ref_count == len(bf) and all(r["pass"] for r in res)
    # the fault hook drops aot's negative phase: the missing set is exactly
    # the negative-phase triangles, samples are its first 32 in sorted order
    res, _ = og.verify(ALGOS, reference=bf, skip_negative=True)
    assert all(r["pass"] for r in res[:3])
    bad = res[3]
    skipped, _ = cg.orient().aot(skip_negative=True, collect=True)[1], None
    missing = sorted(set(map(tuple, bf.tolist())) - canon_set(skipped))
    assert not bad["pass"] and bad["extra_count"] == 0
    assert bad["missing_count"] == len(missing) > 0
    assert bad["missing_samples"] == missing[:32]
    assert bad["stats"]["negative_triangles"] == 0


def test_verify_reports_extra_triangles():
    """A reference missing some triangles: every algorithm reports them as extra."""
    n = 120
    pairs = O.gen_gnp(n, 0.1, 5)
    bf = O.OracleGraph(n, pairs).brute_force()
    og = capi.DeviceGraph.from_pairs(pairs, n).orient()
    res, ref_count = og.verify(("aot", "cf"), reference=bf[5:])
    assert ref_count == len(bf) - 5
    for r in res:
        assert not r["pass"] and r["missing_count"] == 0 and r["extra_count"] == 5
        assert r["extra_samples"] == [tuple(t) for t in bf[:5].tolist()]


@pytest.mark.slow
def test_verify_c2_full_size(golden):
    import torch

    gold = golden["c2"]
    cfg = CONFIGS["c2"]
    d = torch.empty(2 * cfg["npairs"], dtype=torch.int32, device="cuda")
    capi.gen_pairs_device(cfg, d.data_ptr())
    torch.cuda.synchronize()
    g = capi.DeviceGraph.from_device_pairs(d.data_ptr(), cfg["npairs"], cfg["n"])
    del d
    og = g.orient()
    g.close()
    res, ref_count = og.verify(ALGOS)
    assert ref_count == gold["triangles"]
    assert all(r["pass"] and r["unique_triangles"] == gold["triangles"] for r in res)
    res, ref_count = og.verify(("cf", "aot"), skip_negative=True)
    assert res[1]["missing_count"] == gold["negative_triangles"] and res[1]["extra_count"] == 0
    s = res[1]["missing_samples"]
    assert len(s) == 32 and s == sorted(s) and all(a < b < c for a, b, c in s)


def test_verify_hashes_every_kernel(golden):
    """The hash-based cross-check used where sets cannot be materialised."""
    from paper_2006_11494_b200 import trilist

    pairs = O.gen_rmat(3, 12, 16 << 12)
    g = trilist.Graph.from_array(1 << 12, pairs)
    og = trilist.orient(g)
    rep = trilist.verify_hashes(og)
    assert rep["pass"] and rep["reference"] == "cf" and len(rep["results"]) == 4
    st, _ = O.OracleGraph(1 << 12, pairs).orient().aot()
    assert trilist.verify_hashes(og, expected=st)["pass"]
    assert not trilist.verify_hashes(og, expected=dict(st, hash_xor=st["hash_xor"] ^ 1))["pass"]
