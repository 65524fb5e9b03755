"""Edge-list ingestion throughput: device parser (tl_graph_from_text: H2D of the
text + line split + parse + Graph::from_edges on the device) vs the reference's
load_edge_list_text (oracle/_ref, single-threaded by design, graph.cpp:61-187).

    python tools/bench_ingest.py [--config c2] [--reps 3]

Prints one JSON line.  The text is the reference's write_edge_list output of
the config's graph (one "u v" line per undirected edge)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import oracle as O
    from paper_2006_11494_b200 import capi
    from paper_2006_11494_b200.configs import CONFIGS

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    ref = O.RefGraph(cfg["n"], O.gen_config(cfg))
    text = ref.write_edge_list()
    m = ref.m
    del ref
    gpu = []
    for _ in range(a.reps + 1):
        t0 = time.perf_counter()
        g, diag = capi.DeviceGraph.from_text(text)
        gpu.append(time.perf_counter() - t0)
        assert g.m == m and diag["edges_parsed"] == m
        g.close()
    gpu = gpu[1:]
    t0 = time.perf_counter()
    r, rdiag = O.RefGraph.from_text(text)  # includes degree order + orient (reported separately below)
    t_ref = time.perf_counter() - t0
    assert rdiag == diag
    line = {"config": a.config, "bytes": len(text), "lines": diag["lines_read"], "edges": m,
            "gpu_s_best": min(gpu), "gpu_GBps": len(text) / min(gpu) / 1e9,
            "gpu_edges_per_s": m / min(gpu),
            "reference_s_load_order_orient": t_ref,
            "note": "gpu time = host text -> device graph (H2D included); reference time = load_edge_list_text "
                    "+ degree_order + orient (single-threaded)"}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
