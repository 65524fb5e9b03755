"""GPU: edge-list ingestion (load_edge_list*, graph.cpp:40-146/:240-281) parsed
on the device, against the reference loader (oracle/_ref) and the reference's
own known answers (proj/tests/test_graph.cpp)."""
import gzip
import random

import numpy as np
import pytest

import oracle as O
from paper_2006_11494_b200 import capi
from paper_2006_11494_b200 import trilist

pytestmark = pytest.mark.gpu


def test_duplicates_and_self_loops():  # test_graph.cpp:17-26
    g, d = capi.DeviceGraph.from_text("0 0\n0 1\n1 0\n")
    assert (g.n, g.m) == (2, 1)
    assert d == {"lines_read": 3, "edges_parsed": 3, "self_loops_dropped": 1, "duplicates_dropped": 1}


def test_comments_blank_lines_and_n():  # test_graph.cpp:28-34
    g, d = capi.DeviceGraph.from_text("# comment\n% other comment\n\n   \n2 7\n")
    assert (g.n, g.m, d["lines_read"]) == (8, 1, 5)
    assert g.degrees()[0] == 0


def test_empty_input():  # test_graph.cpp:36-41
    g, d = capi.DeviceGraph.from_text("")
    assert (g.n, g.m, d["lines_read"]) == (0, 0, 0)


@pytest.mark.parametrize("text,line,needle", [  # test_graph.cpp:43-58
    ("0 1\nx 2\n", 2, "line 2"),
    ("0 1\n1 -2\n", 2, "negative"),
    ("3\n", 1, "two vertex ids"),
    ("1 2 3\n", 1, "trailing"),
    ("0 1\n0 1\nbroken\n", 3, "malformed vertex id 'broken'"),
    ("4294967295 1\n", 1, "compact"),  # test_graph.cpp:69-74
])
def test_parse_errors_carry_the_line(text, line, needle):
    with pytest.raises(capi.TlParseError) as e:
        capi.DeviceGraph.from_text(text)
    assert e.value.line == line and needle in str(e.value)
    with pytest.raises(trilist.ParseFailure, match=needle):  # module.cpp:50: ValueError subclass
        trilist.load_edge_list_text(text)


def test_one_indexed_and_compact():  # test_graph.cpp:60-85
    g = trilist.load_edge_list_text("1 2\n2 3\n", one_indexed=True)
    assert g.num_vertices == 3 and g.has_edge(0, 1) and g.has_edge(1, 2)
    with pytest.raises(trilist.ParseFailure):
        trilist.load_edge_list_text("0 1\n", one_indexed=True)
    g = trilist.load_edge_list_text("4294967295 1\n", compact_ids=True)
    assert g.num_vertices == 2 and g.has_edge(0, 1)
    g = trilist.load_edge_list_text("50 10\n10 7\n50 7\n", compact_ids=True)  # 50->0, 10->1, 7->2
    assert (g.num_vertices, g.num_edges) == (3, 3)
    assert g.has_edge(0, 1) and g.has_edge(1, 2) and g.has_edge(0, 2)


def random_text(rng, n_lines, n_ids, error_rate=0.0):
    parts = []
    for _ in range(n_lines):
        r = rng.random()
        if r < 0.05:
            parts.append(rng.choice(["# note", "%x", "", "   ", "\t"]))
            continue
        u, v = rng.randrange(n_ids), rng.randrange(n_ids)
        sep = rng.choice([" ", "\t", "  ", " \t "])
        line = f"{rng.choice(['', ' ', chr(9)])}{u}{sep}{v}{rng.choice(['', ' ', chr(13)])}"
        if rng.random() < error_rate:
            line = rng.choice([f"{u}", f"{u} {v} 7", f"-{u} {v}", f"{u}x {v}", f"{u} +{v}",
                               "99999999999999999999999 1"])
        parts.append(line)
    return "\n".join(parts) + rng.choice(["", "\n"])


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("one_indexed,compact", [(False, False), (True, False), (False, True)])
def test_random_texts_match_reference(seed, one_indexed, compact):
    rng = random.Random(seed * 7 + one_indexed * 3 + compact)
    ids = rng.choice([50, 3000, 1 << 20]) if not compact else rng.choice([50, 10 ** 12])
    text = random_text(rng, rng.randrange(1, 4000), ids, error_rate=rng.choice([0.0, 0.0, 0.002]))
    if one_indexed:
        text = text.replace(" 0\n", " 1\n")
    try:
        ref, rdiag = O.RefGraph.from_text(text, one_indexed=one_indexed, compact=compact)
    except O.RefParseError as e:
        with pytest.raises(capi.TlParseError) as got:
            capi.DeviceGraph.from_text(text, one_indexed=one_indexed, compact_ids=compact)
        assert (got.value.line, str(got.value).split("] ", 1)[1]) == (e.line, str(e))
        return
    g, diag = capi.DeviceGraph.from_text(text, one_indexed=one_indexed, compact_ids=compact)
    assert diag == rdiag
    off, adj = g.csr()
    roff, radj = ref.graph_csr()
    assert np.array_equal(off, roff) and np.array_equal(adj, radj)


def test_gzip_file_and_round_trip(tmp_path):  # test_cli.cpp:104-121, test_graph.cpp:112-125
    pairs = O.gen_gnp(60, 0.1, 17)
    ref = O.RefGraph(60, pairs)
    text = ref.write_edge_list()
    p = tmp_path / "g.txt.gz"
    with gzip.open(p, "wb") as f:
        f.write(text)
    g, diag = trilist.load_edge_list(str(p))
    assert diag["duplicates_dropped"] == 0 and diag["self_loops_dropped"] == 0
    assert trilist.write_edge_list(g) == text
    plain = tmp_path / "g.txt"
    plain.write_bytes(text)
    g2, _ = trilist.load_edge_list(str(plain))
    assert g2.num_edges == g.num_edges
    with pytest.raises(RuntimeError, match="cannot open"):
        trilist.load_edge_list(str(tmp_path / "missing.txt"))


def test_loaded_graph_runs_aot():
    text = "\n".join(f"{u} {v}" for u in range(12) for v in range(u + 1, 12))
    g = trilist.load_edge_list_text(text)
    assert trilist.count_triangles(g) == 12 * 11 * 10 // 6
