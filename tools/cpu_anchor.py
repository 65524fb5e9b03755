"""Same-config CPU anchor: the reference's own run_parallel_count on a FULL
config, timed once on a GPU box's host cores and cached (BASELINE.md §2
allows caching the C4/C5 reference results).

    python tools/cpu_anchor.py [--config c4] [--threads 0] [--reps 1] [--out profiles/cpu_anchor_c4.json]

The pairs come from the device generator (bit-identical to the C
restatement's; the pair-list checksum is recorded and compared against the
golden one, so the cached number is tied to this config, seed and generator).
The reference library (oracle/_ref, the unmodified sources) then runs
Graph::from_edges -> degree_order -> orient (single-threaded, as in the
reference) and run_parallel_count(aot, {threads, 64}) with NullSink; the timer
is the reference's RunStats.wall_time_s (parallel.hpp:54, :76), the same
listing-only scope as the GPU's kernel time.  bench.py reports the cached
line as `cpu_baseline` (kind "reference", sample "full c4").
"""
import argparse
import json
import os
import platform
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def main():
    import oracle as O
    from make_golden import device_pairs
    from oracle import pairs_checksum
    from paper_2006_11494_b200.configs import CONFIGS

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--threads", type=int, default=0, help="0 = every host thread")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    threads = a.threads or O.hardware_threads()
    t0 = time.time()
    pairs = device_pairs(cfg)
    t_gen = time.time() - t0
    checksum = pairs_checksum(pairs)
    golden = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json"))).get(a.config, {})
    ref = O.RefGraph(cfg["n"], pairs)
    del pairs
    walls, st = [], None
    for _ in range(a.reps):
        st = ref.count(threads=threads)
        walls.append(st["wall_time_s"])
    wall = min(walls)
    line = {
        "config": a.config, "workload": f"{a.config}: {cfg['name']} (full graph)", "n": ref.n, "m": ref.m,
        "seed": cfg["seed"], "pairs_checksum": checksum,
        "pairs_checksum_matches_golden": golden.get("pairs_checksum") == checksum if golden else None,
        "call": "run_parallel_count(Algorithm::aot, og, {threads, 64}) -- NullSink, RunStats.wall_time_s",
        "threads": threads, "cpu": cpu_model(), "host": platform.node(), "date": time.strftime("%Y-%m-%d"),
        "wall_time_s": wall, "walls_s": walls, "directed_edges_per_s": ref.m / wall,
        "triangles": st["triangles"], "triangles_per_s": st["triangles"] / wall,
        "counters_match_golden": all(st[k] == golden[k] for k in ("triangles", "probes", "positive_triangles",
                                                                  "negative_triangles", "table_builds"))
        if golden else None,
        "preprocess_s": dict(ref.phase_times, generate_on_device=t_gen),
    }
    out = a.out or os.path.join(ROOT, "profiles", f"cpu_anchor_{a.config}.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(line, f, indent=1)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
