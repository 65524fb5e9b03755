#!/usr/bin/env python
"""AOT triangle listing benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

Workload: BASELINE.json configs[3] (R-MAT scale 26, edge factor 16) by default
-- the config the metric ("... 1/2/4/8 B200") is quoted on, and it fits one
GPU -- generated on the device from its seed (inputs resident in HBM).  A
step is one AOT counting run over the oriented graph -- the C-ABI call that
replaces run_parallel_count (task construction + intersection kernels + the
stats read-back), on this rank's cost-balanced share of the directed edges.
`value` = directed edges of the whole graph / max-over-ranks step time
(strong scaling: the graph is fixed, ranks split it).  The L2 is flushed (a
256 MiB write) before every timed step.

`e2e` runs the same metric through the C-ABI with HOST buffers: every step
uploads the reference-layout OrientedGraph from pinned host memory
(tl_oriented_from_csr), counts, and reads the stats back.

`--impl reference` times the reference's own CPU implementation (the
unmodified library built from /root/reference into oracle/_ref) on the host's
cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "directed edges/sec and triangles/sec (count & list), % HBM roofline, 1/2/4/8 B200"
UNIT = "directed edges/s"
L2_FLUSH_BYTES = 256 << 20


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    p.add_argument("--no-list", action="store_true", help="skip the listing-mode measurement")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-threads", type=int, default=0, help="reference threads (0 = all host threads)")
    p.add_argument("--no-warm-build", action="store_true", help="construct the graph once (cold) only")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def algorithmic_bytes(n: int, m: int, aot_cost: int, triangles: int = 0) -> dict:
    """offsets read once, the col array streamed to enumerate
    edges, every out-list staged once as a probe side, and the traversed ids
    (Theta(sum min(deg+)), the un-pruned aot_cost); listing adds 12 B/triangle."""
    b_count = 8 * (n + 1) + 4 * m + 4 * m + 4 * aot_cost
    return {"count": b_count, "list": b_count + 12 * triangles}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.file = None

    def start(self):
        try:
            self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.file, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.file.flush()
        self.file.seek(0)
        rows = [r.split(",") for r in self.file.read().strip().splitlines() if r.strip()]
        os.unlink(self.file.name)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in rows:
            r = [x.strip() for x in r]
            if len(r) < 9:
                continue
            try:
                sm.append(float(r[1]))
                mx.append(float(r[2]))
            except ValueError:
                continue
            for name, val in zip(names, r[5:9]):
                if val.lower() in ("active", "1"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- CPU side
def cpu_reference_run(cfg: dict, steps: int, warmup: int, threads: int) -> dict:
    """The reference library (oracle/_ref) on the host cores: preprocessing
    once (untimed, reported), then `steps` timed run_parallel_count calls;
    the timer is the reference's own RunStats.wall_time_s (listing only)."""
    import oracle as O

    t0 = time.perf_counter()
    pairs = O.gen_config(cfg)
    t_gen = time.perf_counter() - t0
    ref = O.RefGraph(cfg["n"], pairs)
    del pairs
    threads = threads or O.hardware_threads()
    for _ in range(warmup):
        ref.count(threads=threads)
    walls, st = [], None
    for _ in range(steps):
        st = ref.count(threads=threads)
        walls.append(st["wall_time_s"])
    return {"m": ref.m, "n": ref.n, "triangles": st["triangles"] if st else 0, "walls": walls, "threads": threads,
            "phases_s": dict(ref.phase_times, generate=t_gen)}


def sample_config(cfg_key: str) -> tuple[dict, str]:
    """Bounded CPU sample of a config: the config itself up to C2's size,
    otherwise the same generator scaled down to ~16M pairs."""
    from paper_2006_11494_b200.configs import CONFIGS, scaled

    c = CONFIGS[cfg_key]
    if c["npairs"] <= (16 << 20):
        return c, f"full {cfg_key} graph ({c['name']})"
    down = 0
    while scaled(cfg_key, down)["npairs"] > (16 << 20):
        down += 1
    s = scaled(cfg_key, down)
    return s, f"{cfg_key} generator scaled down by 2^{down} ({s['name']}, {s['npairs']} pairs)"


def run_reference_arm(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    cfg, sample = sample_config(args.config)
    r = cpu_reference_run(cfg, max(1, args.steps), max(0, args.warmup), args.cpu_threads)
    t = statistics.mean(r["walls"])
    value = r["m"] / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded generator)",
        "config": {"workload": f"{args.config}: {cfg['name']}", "mode": "count", "n": r["n"], "m": r["m"],
                   "triangles": r["triangles"]},
        "triangles_per_s": r["triangles"] / t,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": r["threads"], "kind": "reference",
                         "sample": f"{sample}; run_parallel_count(aot), {r['threads']} threads, "
                                   f"RunStats.wall_time_s"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_phases_s": r["phases_s"],
    }
    print(json.dumps(line), flush=True)
    return 0


def load_cpu_anchor(config: str, m: int):
    """The cached same-config reference measurement (tools/cpu_anchor.py),
    when it exists for this config and graph (same m, generator checksum equal
    to the golden one)."""
    path = os.path.join(ROOT, "profiles", f"cpu_anchor_{config}.json")
    if not os.path.exists(path):
        return None
    a = json.load(open(path))
    if a.get("m") != m or a.get("pairs_checksum_matches_golden") is False:
        return None
    return {"value": a["directed_edges_per_s"], "unit": UNIT, "cores": a["threads"], "kind": "reference",
            "sample": f"full {config} ({a['workload']}): oracle/_ref {a['call']}, {a['wall_time_s']:.1f} s; "
                      f"measured once on a GPU box's host ({a['cpu']}, {a['threads']} threads, {a['date']}) and "
                      f"cached in profiles/cpu_anchor_{config}.json by tools/cpu_anchor.py",
            "triangles_per_s": a["triangles_per_s"], "wall_time_s": a["wall_time_s"],
            "preprocess_s": a.get("preprocess_s"), "cached": True}


# ----------------------------------------------------------------- GPU side
def gpath_ok(config: str) -> bool:
    path = os.path.join(ROOT, "tests", "golden", "configs.json")
    return os.path.exists(path) and config in json.load(open(path))


def run_e2e(args, og, n, m, rank, world, local, dev, sp, flush, barrier, max_ranks):
    import numpy as np
    import torch

    from paper_2006_11494_b200 import capi

    job = os.environ.get("TORCHELASTIC_RUN_ID", str(os.getppid()))
    base = f"/dev/shm/trilist_e2e_{job}"
    names = {"out_offsets": np.uint64, "out": np.uint32, "rank": np.uint32}
    if int(os.environ.get("LOCAL_RANK", "0")) == 0:
        host = og.csr()  # device -> host once: the reference layout a caller would hold
        for k in names:
            host[k].tofile(f"{base}_{k}.bin")
        del host
    og.close()
    torch.cuda.empty_cache()
    barrier()
    cudart = torch.cuda.cudart()
    maps, ptrs, et, launches = {}, {}, [], 0
    try:
        for k, dt in names.items():
            a = np.memmap(f"{base}_{k}.bin", dtype=dt, mode="r+")  # shared tmpfs pages, never written
            maps[k] = a
            rc = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)  # page-lock for DMA
            if int(rc) != 0:
                raise RuntimeError(f"cudaHostRegister failed ({int(rc)})")
            ptrs[k] = a.ctypes.data
        h2d = sum(a.nbytes for a in maps.values())
        d2h = capi.C.sizeof(capi.TlStats)

        def step():
            up = capi.DeviceOriented.from_host_ptrs(n, m, ptrs["out_offsets"], ptrs["out"], ptrs["rank"], local, sp)
            st = up.count(part=rank, nparts=world, stream=sp)
            up.close()
            return st

        for _ in range(max(1, args.warmup // 2)):
            step()
        torch.cuda.synchronize(dev)
        barrier()
        for _ in range(max(3, args.steps // 2)):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            st = step()
            et.append(time.perf_counter() - t0)
            launches += st["kernel_launches"]
        barrier()
    finally:
        for p in ptrs.values():
            cudart.cudaHostUnregister(p)
        maps.clear()
        if int(os.environ.get("LOCAL_RANK", "0")) == 0:
            for k in names:
                try:
                    os.unlink(f"{base}_{k}.bin")
                except OSError:
                    pass
    e_s = max_ranks(statistics.mean(et))
    return {"value": m / e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": e_s * 1e3, "launches": launches,
            "path": "tl_oriented_from_csr (pinned host reference layout, shared by the node's ranks) + "
                    "tl_aot_count + stats read-back"}


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2006_11494_b200 import capi
    from paper_2006_11494_b200 import dist as tdist
    from paper_2006_11494_b200.configs import CONFIGS

    rank, world, local = dist_env()
    # TL_BENCH_BACKEND=gloo: functional check of the N>1 path with fewer GPUs
    # than ranks (ranks share a device; their kernels never wait on each
    # other, the collectives run on the host) -- not a measurement
    backend = os.environ.get("TL_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cfg = CONFIGS[args.config]
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    def barrier():
        if world > 1:
            dist.barrier()

    def max_ranks(x):
        return tdist.max_over_ranks(x) if world > 1 else x

    # ---- inputs resident in HBM: the seeded pair list generated on device
    phases = {}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    d_pairs = torch.empty(2 * cfg["npairs"], dtype=torch.int32, device=dev)
    ev[0].record(stream)
    capi.gen_pairs_device(cfg, d_pairs.data_ptr(), sp)
    ev[1].record(stream)
    torch.cuda.synchronize(dev)
    phases["generate_ms"] = ev[0].elapsed_time(ev[1])

    # ---- preprocessing on device (reported, excluded from value like the
    #      reference excludes load/orient from RunStats.wall_time_s)
    capi.DeviceGraph.from_pairs(np.array([[0, 1], [1, 2]], np.uint32), 3, local).close()  # library/module warm-up
    torch.cuda.synchronize(dev)

    pairs_holder = [d_pairs]
    del d_pairs

    def construct(last: bool):
        t0 = time.perf_counter()
        g = capi.DeviceGraph.from_device_pairs(pairs_holder[0].data_ptr(), cfg["npairs"], cfg["n"], local, sp)
        t1 = time.perf_counter()
        if last:  # the largest configs need the HBM for orient()
            pairs_holder.clear()
            torch.cuda.empty_cache()
        t2 = time.perf_counter()
        o = g.orient()
        t3 = time.perf_counter()
        return g, o, {"from_edges_ms": (t1 - t0) * 1e3, "order_orient_claims_ms": (t3 - t2) * 1e3}

    # construction twice when the HBM allows (not C5): the first call of a
    # fresh process also grows the device memory pool (cold), the second
    # reuses it (warm) -- the steady cost of building a graph
    warm = args.config not in ("c5",) and not args.no_warm_build
    dg, og, cold = construct(last=not warm)
    phases["cold"] = cold
    if warm:
        og.close()
        dg.close()
        torch.cuda.synchronize(dev)
        dg, og, phases["warm"] = construct(last=True)
    phases.update(phases.get("warm", cold))
    n, m = og.n, og.m
    costs = og.cost_model()
    dg.close()
    torch.cuda.empty_cache()

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device=dev)
    peaks = load_peaks()

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize(dev)
        barrier()
        torch.cuda.synchronize(dev)
        times, stats = [], []
        for _ in range(steps):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            st = fn()
            b.record(stream)
            b.synchronize()
            times.append(a.elapsed_time(b))
            stats.append(st)
        torch.cuda.synchronize(dev)
        barrier()
        return times, stats

    # ---- count (the headline)
    clocks = ClockSampler(local)
    clocks.start()
    times, stats = timed(lambda: og.count(part=rank, nparts=world, stream=sp), args.steps, args.warmup)
    clock_info = clocks.stop()
    step_ms = max_ranks(statistics.mean(times))
    kern_ms = max_ranks(statistics.mean(s["list_ms"] for s in stats))
    prep_ms = max_ranks(statistics.mean(s["prep_ms"] for s in stats))
    launches = sum(s["kernel_launches"] for s in stats)
    whole = tdist.reduce_stats(stats[-1]) if world > 1 else stats[-1]
    T = whole["triangles"]
    B = algorithmic_bytes(n, m, costs["aot_cost"], T)
    achieved = (B["count"] / world) / (kern_ms * 1e-3) / 1e9

    # parity of this run against the reference's golden values (when present)
    parity = None
    gpath = os.path.join(ROOT, "tests", "golden", "configs.json")
    if gpath_ok(args.config):
        g = json.load(open(gpath)).get(args.config)
        if g:
            parity = all(whole[k] == g[k] for k in ("triangles", "probes", "positive_triangles",
                                                    "negative_triangles", "table_builds"))

    # ---- listing: triangles emitted into an HBM buffer (12 B each) when the
    #      list fits in a quarter of the free HBM, otherwise emitted into the
    #      order-independent hash (the large configs' "list with hash").
    list_info = None
    if not args.no_list:
        free_b, _ = torch.cuda.mem_get_info(dev)
        materialise = 12 * T / world < free_b / 4
        mode = "list" if materialise else "hash"

        out_buf = None
        if materialise:  # this part's emissions, kept in HBM (tl_run_list_device: one listing pass)
            T_part = stats[-1]["triangles"]
            out_buf = torch.empty(max(3 * T_part, 3), dtype=torch.int32, device=dev)

        def list_step():
            if materialise:
                return og.list_device(out_buf.data_ptr(), out_buf.numel() // 3, part=rank, nparts=world, stream=sp)
            return og.hash(part=rank, nparts=world, stream=sp)

        lt, ls = timed(list_step, max(3, args.steps // 2), max(1, args.warmup // 2))
        out_buf = None  # release the emissions before the e2e upload
        l_step = max_ranks(statistics.mean(lt))
        l_kern = max_ranks(statistics.mean(s["list_ms"] for s in ls))
        launches += sum(s["kernel_launches"] for s in ls)
        hashed = tdist.reduce_stats(ls[-1]) if world > 1 else ls[-1]
        b_list = B["list"] if materialise else B["count"]
        list_info = {"mode": mode, "ms_per_step": l_step, "kernel_ms": l_kern, "triangles_per_s": T / (l_step * 1e-3),
                     "directed_edges_per_s": m / (l_step * 1e-3),
                     "roofline_frac": (b_list / world) / (l_kern * 1e-3) / 1e9 / peaks["hbm_gbs"]}
        if not materialise:
            list_info["hash"] = {"count": hashed["triangles"], "sum": hashed["hash_sum"], "xor": hashed["hash_xor"]}
            if gpath_ok(args.config):
                g = json.load(open(gpath)).get(args.config)
                list_info["hash_matches_reference"] = (hashed["hash_sum"], hashed["hash_xor"]) == (
                    g["hash_sum"], g["hash_xor"])

    # ---- e2e through the C-ABI with host buffers: every step uploads the
    #      reference-layout OrientedGraph from pinned host memory, counts, and
    #      reads the stats back.  The host copy is shared by the ranks of the
    #      node through /dev/shm (one copy, pinned by every rank); the
    #      device-resident graph is released first (the upload rebuilds one).
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, og, n, m, rank, world, local, dev, sp, flush, barrier, max_ranks)
        launches += e2e.pop("launches")
    og.close()
    torch.cuda.empty_cache()

    # ---- CPU baseline: the reference library on this host (rank 0, N=1):
    #      a bounded scaled-down sample timed live, and -- the same-config
    #      anchor -- the full config's reference run measured once on a GPU
    #      box's host and cached (profiles/cpu_anchor_<config>.json,
    #      tools/cpu_anchor.py; BASELINE.md §2 allows caching C4/C5)
    cpu, cpu_live = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            scfg, sample = sample_config(args.config)
            r = cpu_reference_run(scfg, 2, 0, args.cpu_threads)
            t = min(r["walls"])
            scaled = "scaled down" in sample
            cpu_live = {"value": r["m"] / t, "unit": UNIT, "cores": r["threads"], "kind": "reference",
                        "sample": f"{sample} ({'SCALED, ' if scaled else ''}timed in this run); oracle/_ref "
                                  f"run_parallel_count(aot), best of 2, RunStats.wall_time_s",
                        "triangles_per_s": r["triangles"] / t, "preprocess_s": r["phases_s"]}
        except Exception as e:  # the baseline never blocks the GPU number
            cpu_live = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}
    anchor = load_cpu_anchor(args.config, m)
    if rank == 0:
        cpu = anchor or cpu_live

    if rank == 0:
        traffic = None
        tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
        if os.path.exists(tpath):
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        line = {
            "metric": METRIC, "value": m / (step_ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded generator, generated on device)",
            "config": {"workload": f"{args.config}: {cfg['name']} ({cfg['desc']})", "mode": "count",
                       "n": n, "m": m, "triangles": T, "aot_cost": costs["aot_cost"],
                       "parallelism": f"edge-partition x{world} (cost-prefix cut, replicated CSR)",
                       "l2": f"flushed before every timed step ({L2_FLUSH_BYTES >> 20} MiB write)"},
            "triangles_per_s": T / (step_ms * 1e-3),
            "kernel_ms": kern_ms, "prep_ms": prep_ms,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                         "bytes_per_launch": B["count"] // world, "peak_source": peaks["source"],
                         # `achieved` counts ALGORITHMIC bytes (4 B per logical probe), part of
                         # which the windowed traversal never loads or finds in L2, so frac can pass 1; the
                         # DRAM-level figure is the ncu traffic of one launch over this run's kernel time
                         "traffic_gbs": (traffic / world / (kern_ms * 1e-3) / 1e9) if traffic else None,
                         "traffic_frac": (traffic / world / (kern_ms * 1e-3) / 1e9 / peaks["hbm_gbs"]) if traffic else None,
                         "kernel": "k_aot (AOT intersection, both phases), CUDA events on the launch stream"},
            "cpu_baseline": cpu,
            "cpu_baseline_live_sample": cpu_live if anchor else None,
            "e2e": e2e,
            "list": list_info,
            "gpu_launches": launches,
            "clocks": clock_info,
            "parity_vs_reference": parity,
            "preprocess_ms": phases,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` without a launcher: start the N ranks here (one
    process per GPU, torch.distributed.run on 127.0.0.1) and relay their
    output; rank 0 prints the JSON line.  NCCL's init log (NCCL_DEBUG=INFO,
    subsystem INIT) stays visible so every rank's communicator can be counted."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}: refusing to report a mislabelled run",
              file=sys.stderr, flush=True)
        return 2
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
