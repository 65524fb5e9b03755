"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): every
device kernel of the library on graphs that reach every probe path (warp
bitmap, warp rank bitmap, warp hash, CTA bitmap / rank / hash), every
algorithm and mode, partitions, ingestion and verification, each checked
against the oracle so a silent corruption also fails.

    compute-sanitizer --tool memcheck --error-exitcode 1 python tools/sanitize_run.py [--size small|medium]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np

    import oracle as O
    from paper_2006_11494_b200 import capi

    ap = argparse.ArgumentParser()
    ap.add_argument("--size", default="small", choices=["small", "medium", "large"])
    a = ap.parse_args()
    graphs = [("gnp", 300, O.gen_gnp(300, 0.05, 7)), ("rmat14", 1 << 14, O.gen_rmat(4, 14, 16 << 14))]
    if a.size in ("medium", "large"):
        graphs.append(("rmat17", 1 << 17, O.gen_rmat(11, 17, 16 << 17)))
    if a.size == "large":
        graphs.append(("rmat19", 1 << 19, O.gen_rmat(12, 19, 16 << 19)))
    for name, n, pairs in graphs:
        g = capi.DeviceGraph.from_pairs(pairs, n)
        cg = O.OracleGraph(n, pairs)
        for order in ("degree", "degeneracy"):
            og = g.orient(g.make_order(order))
            co = cg.orient(cg.make_order(order))
            for algo in ("aot", "kclist", "cf-hash", "cf"):
                want, raw = co.run(algo, collect=True)
                for mode in ("count", "hash"):
                    st = og.count(algo=algo) if mode == "count" else og.hash(algo=algo)
                    assert st["triangles"] == want["triangles"], (name, order, algo, mode)
                    if mode == "hash":
                        assert (st["hash_sum"], st["hash_xor"]) == (want["hash_sum"], want["hash_xor"])
                _, got = og.list(algo=algo, canonical=True)
                assert np.array_equal(got, O.canonical_sorted(raw)), (name, order, algo)
                parts = [og.count(algo=algo, part=p, nparts=3)["triangles"] for p in range(3)]
                assert sum(parts) == want["triangles"]
            res, cnt = og.verify(("cf", "aot"), skip_negative=True)
            assert cnt == want["triangles"] and res[0]["pass"]
            og.close()
        print(name, "ok", flush=True)
    text = "".join(f"{u} {v}\n" for u, v in O.gen_gnp(200, 0.05, 3).tolist()) + "# c\n\n7 7\n"
    g, diag = capi.DeviceGraph.from_text(text, compact_ids=True)
    assert diag["self_loops_dropped"] == 1
    print("ingest ok", flush=True)


if __name__ == "__main__":
    main()
