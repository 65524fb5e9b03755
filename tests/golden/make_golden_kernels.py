"""Generates tests/golden/kernels.json from the REFERENCE itself: the
comparison kernels (cf merge, cf-hash with and without table reuse, kclist3;
engine.hpp:164-236) and the degeneracy order (ordering.cpp:86-114) on the
BASELINE configs.

Run in the build container (needs /root/reference to build oracle/_ref):

    python tests/golden/make_golden_kernels.py [c1 c2 ...]

Per config and order ("degree", "degeneracy"): a checksum of the reference's
rank array, then for every kernel the six RunStats counters and the
order-independent hash (count, sum, xor) through a per-worker hash sink
(run_parallel), plus the reference's own listing wall time.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from paper_2006_11494_b200.configs import CONFIGS  # noqa: E402


def rank_checksum(rank: np.ndarray) -> str:
    """sum over u of fmix64(u << 32 | rank[u]) mod 2^64, as a decimal string."""
    u = np.arange(rank.size, dtype=np.uint64)
    z = (u << np.uint64(32)) | rank.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
        return str(int(np.sum(z, dtype=np.uint64)))


def golden_for(key: str, threads: int, orders) -> dict:
    cfg = CONFIGS[key]
    pairs = O.gen_config(cfg)
    out = {"config": key, "ref_threads": threads}
    for order in orders:
        t0 = time.time()
        ref = O.RefGraph(cfg["n"], pairs, order=order)
        entry = {"rank_checksum": rank_checksum(ref.oriented_csr()["rank"]), "phase_times_s": ref.phase_times,
                 "cost_model": ref.cost_model(), "kernels": {}}
        for algo, reuse in (("aot", False), ("kclist", False), ("cf-hash", False), ("cf-hash", True), ("cf", False)):
            r = ref.run(algo, threads=threads, reuse=reuse, hash=True)
            name = algo + ("+reuse" if reuse else "")
            entry["kernels"][name] = r
            print(key, order, name, r["triangles"], f"{r['wall_time_s']:.2f}s", flush=True)
        entry["total_s"] = time.time() - t0
        out[order] = entry
    return out


def main(keys):
    threads = O.hardware_threads()
    path = os.path.join(HERE, "kernels.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    for k in keys:
        data[k] = golden_for(k, threads, ("degree", "degeneracy"))
        json.dump(data, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2"])
