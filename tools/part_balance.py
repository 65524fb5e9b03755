"""Multi-GPU load balance, measured on one GPU: run every part of an
nparts-way edge partition (the cut bench.py uses under torchrun) one after
another and report each part's kernel time.  Strong-scaling efficiency at N
GPUs is bounded by mean/max of these times.

    python tools/part_balance.py [--config c4] [--nparts 2,4,8] [--reps 2]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2006_11494_b200 import capi
    from paper_2006_11494_b200.configs import CONFIGS

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--nparts", default="2,4,8")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--mode", default="count", choices=["count", "hash"])
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    d = torch.empty(2 * cfg["npairs"], dtype=torch.int32, device="cuda")
    capi.gen_pairs_device(cfg, d.data_ptr())
    torch.cuda.synchronize()
    g = capi.DeviceGraph.from_device_pairs(d.data_ptr(), cfg["npairs"], cfg["n"])
    del d
    torch.cuda.empty_cache()
    og = g.orient()
    g.close()
    run = og.count if a.mode == "count" else og.hash
    whole = min(run()["list_ms"] for _ in range(a.reps))
    for n in map(int, a.nparts.split(",")):
        times, tri, prep_first, prep_cached = [], 0, [], []
        for p in range(n):
            best = None
            for i in range(a.reps):
                st = run(part=p, nparts=n)
                best = st["list_ms"] if best is None else min(best, st["list_ms"])
                (prep_first if i == 0 else prep_cached).append(st["prep_ms"])
            times.append(best)
            tri += st["triangles"]
        print(json.dumps({"config": a.config, "mode": a.mode, "nparts": n, "whole_ms": round(whole, 3),
                          "part_ms": [round(t, 3) for t in times], "max_ms": round(max(times), 3),
                          "mean_ms": round(sum(times) / n, 3), "balance": round(sum(times) / n / max(times), 4),
                          "ideal_speedup": round(whole / max(times), 3), "triangles_sum": tri,
                          "prep_ms_first_call_max": round(max(prep_first), 3),
                          "prep_ms_cached_max": round(max(prep_cached), 3) if prep_cached else None}), flush=True)


if __name__ == "__main__":
    main()
