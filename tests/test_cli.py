"""The `trilist` command line (paper_2006_11494_b200/bin/trilist), restating
the reference's end-to-end CLI tests (proj/tests/test_cli.cpp) and its JSON
schema (trilist_main.cpp:191-357, report.cpp:10-95).  Usage errors, help and
version run on the CPU (no device call happens before argument validation);
everything that loads a graph runs on the GPU."""
import gzip
import json
import os
import subprocess

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2006_11494_b200", "bin", "trilist")


@pytest.fixture(scope="module")
def cli(built):
    from paper_2006_11494_b200 import _build

    _build.build_cli()
    return BIN


def run(cli, *args, stdin=None, env=None):
    e = dict(os.environ)
    e.pop("TRILIST_THREADS", None)
    e.update(env or {})
    p = subprocess.run([cli, *args], input=stdin, capture_output=True, env=e, timeout=600)
    return p.returncode, p.stdout.decode(), p.stderr.decode()


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode() if isinstance(text, str) else text)
    return str(p)


def edge_text(n_edges):
    return "".join(f"{u} {v}\n" for u, v in n_edges)


# ------------------------------------------------------------------ CPU
def test_usage_errors_exit_2(cli, tmp_path):  # test_cli.cpp:123-134
    p = write(tmp_path, "tiny.txt", "0 1\n")
    assert run(cli, "count", p, "--algo", "nope")[0] == 2
    assert run(cli, "count", p, "--order", "fancy")[0] == 2
    assert run(cli, "count", p, "--algo", "cf", "--local-order", "degree-desc")[0] == 2
    assert run(cli, "count")[0] == 2  # missing input
    assert run(cli, "frobnicate", "x")[0] == 2  # unknown subcommand
    assert run(cli, "count", p, "--threads", "0")[0] == 2
    assert run(cli)[0] == 2  # a subcommand is required
    assert run(cli, "count", p, "--chunk", "abc")[0] == 2
    assert run(cli, "verify", p, "--algos", "aot,bogus")[0] == 2
    assert run(cli, "verify", p, "--inject-fault", "other")[0] == 2
    assert run(cli, "bench", p, "--repeats", "0")[0] == 2
    assert run(cli, "stats", p, "--algo", "aot")[0] == 2  # stats takes no --algo
    assert run(cli, "count", p, env={"TRILIST_THREADS": "0"})[0] == 2  # ->envname + Range
    code, out, _ = run(cli, "--help")
    assert code == 0 and "count" in out and "verify" in out
    assert run(cli, "count", "--help")[0] == 0
    assert run(cli, "--version")[1].strip() == "0.1.0"


def test_missing_file_exits_1(cli, tmp_path):  # test_cli.cpp:136-142 (first half)
    code, _, err = run(cli, "count", str(tmp_path / "absent.txt"))
    assert code == 1 and "error:" in err


# ------------------------------------------------------------------ GPU
K4 = "0 1\n0 2\n0 3\n1 2\n1 3\n2 3\n"


@pytest.mark.gpu
def test_count_k3_report(cli, tmp_path):  # test_cli.cpp:85-102
    code, out, err = run(cli, "count", write(tmp_path, "k3.txt", "0 1\n0 2\n1 2\n"), "--algo", "aot")
    assert code == 0, err
    doc = json.loads(out)
    assert doc["schema_version"] == 1 and doc["command"] == "count"
    assert (doc["triangles"], doc["n"], doc["m"]) == (1, 3, 3)
    assert (doc["algorithm"], doc["order"], doc["local_order"]) == ("aot", "degree", "degree-desc")
    assert doc["stats"]["probes"] == 1 and doc["costs"]["aot_cost"] == 1
    assert "list_s" in doc["timings"]
    assert sorted(doc) == sorted(["schema_version", "command", "dataset", "n", "m", "load", "algorithm", "order",
                                  "local_order", "workers", "chunk", "triangles", "stats", "costs", "timings"])
    assert list(doc) == sorted(doc)  # nlohmann objects are ordered maps
    assert sorted(doc["stats"]) == sorted(["triangles", "probes", "merge_comparisons", "table_builds",
                                           "positive_triangles", "negative_triangles", "wall_time_s"])
    assert sorted(doc["load"]) == sorted(["lines_read", "edges_parsed", "self_loops_dropped", "duplicates_dropped"])
    pretty = run(cli, "count", write(tmp_path, "k3b.txt", "0 1\n0 2\n1 2\n"), "--pretty")[1]
    assert pretty.startswith("{\n  \"") and json.loads(pretty)["triangles"] == 1


@pytest.mark.gpu
def test_count_stdin_and_gzip(cli, tmp_path):  # test_cli.cpp:104-121
    code, out, err = run(cli, "count", "-", "--algo", "kclist", stdin=K4.encode())
    assert code == 0, err
    assert json.loads(out)["triangles"] == 4
    gz = tmp_path / "k4.txt.gz"
    with gzip.open(gz, "wb") as f:
        f.write(K4.encode())
    code, out, err = run(cli, "count", str(gz))
    assert code == 0, err
    assert json.loads(out)["triangles"] == 4


@pytest.mark.gpu
def test_parse_failure_exits_1_with_line(cli, tmp_path):  # test_cli.cpp:136-142
    code, _, err = run(cli, "count", write(tmp_path, "bad.txt", "0 1\nnot numbers\n"))
    assert code == 1 and "line 2" in err


@pytest.mark.gpu
def test_list_sorted_and_out(cli, tmp_path):  # test_cli.cpp:144-165, :235-243
    diamond = edge_text(O.diamond_graph()[1])
    code, out, err = run(cli, "list", write(tmp_path, "d.txt", diamond), "--sorted", "--algo", "cf")
    assert code == 0, err
    assert out == "0 1 2\n1 2 3\n"
    dst = tmp_path / "triangles.txt"
    code, out, err = run(cli, "list", write(tmp_path, "k3.txt", "0 1\n0 2\n1 2\n"), "--sorted", "--out", str(dst))
    assert code == 0 and out == "" and dst.read_text() == "0 1 2\n"
    assert run(cli, "list", write(tmp_path, "k3c.txt", "0 1\n"), "--out", str(tmp_path / "no_dir" / "x.txt"))[0] == 1
    code, out, _ = run(cli, "list", write(tmp_path, "one.txt", "1 2\n1 3\n2 3\n"), "--one-indexed", "--sorted")
    assert code == 0 and out == "0 1 2\n"


@pytest.mark.gpu
def test_list_unsorted_is_the_canonical_set(cli, tmp_path):
    pairs = O.gen_gnp(120, 0.1, 9)
    text = edge_text(pairs.tolist())
    want = O.RefGraph(120, pairs).brute_force()
    for algo in ("aot", "kclist", "cf-hash", "cf"):
        code, out, err = run(cli, "list", write(tmp_path, f"g_{algo}.txt", text), "--algo", algo)
        assert code == 0, err
        got = sorted(tuple(map(int, line.split())) for line in out.splitlines())
        assert got == sorted(map(tuple, want.tolist()))


@pytest.mark.gpu
def test_verify_k5_passes(cli, tmp_path):  # test_cli.cpp:167-178
    k5 = edge_text([(u, v) for u in range(5) for v in range(u + 1, 5)])
    code, out, err = run(cli, "verify", write(tmp_path, "k5.txt", k5))
    assert code == 0, err
    doc = json.loads(out)
    assert doc["pass"] is True and doc["oracle_used"] is True and doc["oracle_triangles"] == 10
    assert doc["cross_order_consistent"] is True and len(doc["orders"]) == 3
    for entry in doc["orders"]:
        for res in entry["report"]["results"]:
            assert res["pass"] is True
    assert [e["order"] for e in doc["orders"]] == ["degree", "degeneracy", "id"]
    assert doc["algorithms"] == ["cf", "cf-hash", "kclist", "aot"]


@pytest.mark.gpu
def test_verify_catches_fault_exit_3(cli, tmp_path):  # test_cli.cpp:180-188
    diamond = edge_text(O.diamond_graph()[1])
    code, out, _ = run(cli, "verify", write(tmp_path, "d.txt", diamond), "--inject-fault", "drop-negative-phase")
    assert code == 3
    assert json.loads(out)["pass"] is False


@pytest.mark.gpu
def test_threads_do_not_change_counters(cli, tmp_path):  # test_cli.cpp:190-198
    p = write(tmp_path, "gnp.txt", edge_text(O.gen_gnp(250, 0.05, 50).tolist()))
    seq = json.loads(run(cli, "count", p, "--threads", "1")[1])
    par = json.loads(run(cli, "count", p, "--threads", "4")[1])
    env = json.loads(run(cli, "count", p, env={"TRILIST_THREADS": "3"})[1])
    for d in (par, env):
        assert d["triangles"] == seq["triangles"]
        assert d["stats"]["probes"] == seq["stats"]["probes"]
        assert d["stats"]["table_builds"] == seq["stats"]["table_builds"]
    assert env["workers"] == 3


@pytest.mark.gpu
def test_stats_pinned_fixture_costs(cli, tmp_path):  # test_cli.cpp:200-209
    n, e = O.paired_hubs_graph()
    code, out, err = run(cli, "stats", write(tmp_path, "hubs.txt", edge_text(e)), "--order", "degree")
    assert code == 0, err
    doc = json.loads(out)
    assert doc["costs"]["kclist_cost"] == 21 and doc["costs"]["aot_cost"] == 12
    assert doc["max_out_degree"] == 3


@pytest.mark.gpu
def test_bench_rows_json_and_csv(cli, tmp_path):  # test_cli.cpp:211-233
    p = write(tmp_path, "bench.txt", edge_text(O.gen_gnp(150, 0.08, 3).tolist()))
    code, out, err = run(cli, "bench", p, "--algos", "kclist,aot", "--orders", "degree,degeneracy",
                         "--threads-list", "1,2", "--repeats", "2")
    assert code == 0, err
    doc = json.loads(out)
    assert len(doc["rows"]) == 8
    kclist_probes = None
    for row in doc["rows"]:
        assert row["repeats"] == 2 and len(row["list_times_s"]) == 2
        if row["algorithm"] == "kclist" and row["order"] == "degree":
            kclist_probes = row["stats"]["probes"]
        if row["algorithm"] == "aot" and row["order"] == "degree":
            assert row["stats"]["probes"] <= kclist_probes
        key = "aot_cost" if row["algorithm"] == "aot" else "kclist_cost"
        assert row["stats"]["probes"] == row["costs"][key]
    code, out, err = run(cli, "bench", p, "--algos", "aot", "--csv", "--repeats", "1")
    assert code == 0, err
    assert out.startswith("dataset,n,m,algorithm,")


@pytest.mark.gpu
def test_counters_match_reference_library(cli, tmp_path):
    """Every kernel's count report equals the reference library's RunStats and
    cost model on the same file, under the CLI's per-algorithm default orders
    (degeneracy for kclist, degree otherwise)."""
    pairs = O.gen_gnp(300, 0.06, 77)
    p = write(tmp_path, "g.txt", edge_text(pairs.tolist()))
    for algo in ("aot", "kclist", "cf-hash", "cf"):
        doc = json.loads(run(cli, "count", p, "--algo", algo)[1])
        order = "degeneracy" if algo == "kclist" else "degree"
        ref = O.RefGraph(300, pairs, order=order)
        want = ref.run(algo)
        for k in ("triangles", "probes", "merge_comparisons", "table_builds", "positive_triangles",
                  "negative_triangles"):
            assert doc["stats"][k] == want[k], (algo, k)
        assert doc["costs"] == ref.cost_model()
        assert doc["order"] == order
