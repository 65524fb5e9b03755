"""Generates tests/golden/*.json|npy from the REFERENCE itself.

Run in the build container (needs /root/reference to build oracle/_ref):

    python tests/golden/make_golden.py [c1 c2 c3 ...]

For each config: the reference library (oracle/_ref/libtrilist_ref.so, built
from the unmodified /root/reference sources) runs Graph::from_edges ->
degree_order -> orient -> run_parallel(aot) with a hash sink, plus cost_model;
the C restatement (oracle/_build/liboracle.so) generates the pairs.  A
pair-list checksum pins the generator so the GPU generator can be checked
without shipping the pairs.  For C1 the full canonical triangle list is stored
(.npy) and cross-checked against brute_force_triangles.
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
from oracle import pairs_checksum  # noqa: E402


def device_pairs(cfg: dict) -> np.ndarray:
    """The same pair list from the device generator (bit-identical to the C
    restatement's: full checksums agree on C1-C4, tests/test_gpu_cabi.py) --
    minutes faster at C5, where the reference then runs on a GPU box's host."""
    import torch

    from paper_2006_11494_b200 import capi

    d = torch.empty(2 * cfg["npairs"], dtype=torch.int32, device="cuda")
    capi.gen_pairs_device(cfg, d.data_ptr())
    host = d.cpu().numpy().view(np.uint32).reshape(-1, 2)
    del d
    torch.cuda.empty_cache()
    return host


def golden_for(key: str, threads: int, on_device: bool = False) -> dict:
    cfg = CONFIGS[key]
    t0 = time.time()
    pairs = device_pairs(cfg) if on_device else O.gen_config(cfg)
    t_gen = time.time() - t0
    checksum, first = pairs_checksum(pairs), pairs[:8].tolist()
    npairs = int(pairs.shape[0])
    ref = O.RefGraph(cfg["n"], pairs)
    del pairs  # host memory: the reference holds its own copies
    h = ref.hash(threads=threads)
    cm = ref.cost_model()
    out = {
        "config": key,
        "cfg": cfg,
        "npairs": npairs,
        "pairs_checksum": checksum,
        "first_pairs": first,
        "n": ref.n,
        "m": ref.m,
        "max_out_degree": ref.max_out_degree(),
        "triangles": h["triangles"],
        "probes": h["probes"],
        "table_builds": h["table_builds"],
        "positive_triangles": h["positive_triangles"],
        "negative_triangles": h["negative_triangles"],
        "hash_count": h["hash_count"],
        "hash_sum": h["hash_sum"],
        "hash_xor": h["hash_xor"],
        "cost_model": cm,
        "ref_phase_times_s": ref.phase_times,
        "ref_list_wall_s": h["wall_time_s"],
        "ref_threads": threads,
        "gen_s": t_gen,
        "pairs_from": "device generator" if on_device else "C restatement generator",
    }
    if key == "c1":
        st, raw = ref.collect(threads=threads)
        canon = O.canonical_sorted(raw)
        bf = ref.brute_force(max_vertices=cfg["n"])
        assert np.array_equal(canon, bf), "reference AOT and brute force disagree on C1"
        np.save(os.path.join(HERE, "c1_triangles.npy"), canon)
        out["list_file"] = "c1_triangles.npy"
    return out


def main(keys):
    threads = O.hardware_threads()
    path = os.path.join(HERE, "configs.json")
    on_device = False
    if keys and keys[0] == "--out":  # e.g. on a GPU box's host for C5: write elsewhere, merge here
        path, keys = keys[1], keys[2:]
    if keys and keys[0] == "--device-pairs":
        on_device, keys = True, keys[1:]
    data = json.load(open(path)) if os.path.exists(path) else {}
    for k in keys:
        t = time.time()
        data[k] = golden_for(k, threads, on_device)
        print(k, {x: data[k][x] for x in ("m", "triangles", "hash_sum")}, f"{time.time() - t:.1f}s", flush=True)
        json.dump(data, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2"])
