"""The paper's kernel comparison on the device: every
kernel (cf merge, cf-hash, kclist3, aot) under the degree order on one config,
count mode, best of --reps device times (CUDA events around the listing
kernels, like RunStats.wall_time_s).  Prints one JSON line per kernel and a
summary line; reference wall times come from tests/golden/kernels.json when
the config is there (the reference run in the build container, 8 threads).

    python tools/bench_kernels.py [--config c2] [--reps 5] [--orders degree,degeneracy]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2006_11494_b200 import capi
    from paper_2006_11494_b200.configs import CONFIGS

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--orders", default="degree")
    ap.add_argument("--algos", default="aot,kclist,cf-hash,cf")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    gold_path = os.path.join(ROOT, "tests", "golden", "kernels.json")
    gold = json.load(open(gold_path)).get(a.config, {}) if os.path.exists(gold_path) else {}
    d = torch.empty(2 * cfg["npairs"], dtype=torch.int32, device="cuda")
    capi.gen_pairs_device(cfg, d.data_ptr())
    torch.cuda.synchronize()
    g = capi.DeviceGraph.from_device_pairs(d.data_ptr(), cfg["npairs"], cfg["n"])
    del d
    torch.cuda.empty_cache()
    rows = []
    for order in a.orders.split(","):
        og = g.orient(g.make_order(order))
        cost = og.cost_model()
        for algo in a.algos.split(","):
            best, st = None, None
            for _ in range(a.reps):
                st = og.count(algo=algo)
                best = st["list_ms"] if best is None else min(best, st["list_ms"])
            ref = gold.get(order, {}).get("kernels", {}).get(algo)
            row = {"config": a.config, "order": order, "algo": algo, "best_list_ms": round(best, 3),
                   "prep_ms": round(st["prep_ms"], 3), "triangles": st["triangles"], "probes": st["probes"],
                   "merge_comparisons": st["merge_comparisons"], "table_builds": st["table_builds"],
                   "probes_executed": st["probes_executed"], "cost_model": cost,
                   "counters_equal_reference": None if ref is None else all(
                       st[k] == ref[k] for k in ("triangles", "probes", "merge_comparisons", "table_builds",
                                                 "positive_triangles", "negative_triangles")),
                   "reference_wall_s_8threads": None if ref is None else ref["wall_time_s"]}
            if ref is not None:
                row["speedup_vs_reference"] = round(ref["wall_time_s"] * 1e3 / best, 1)
            rows.append(row)
            print(json.dumps(row), flush=True)
        og.close()


if __name__ == "__main__":
    main()
