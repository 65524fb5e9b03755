"""Phase breakdown of the e2e path (bench.py's `e2e`): upload of the
reference-layout OrientedGraph from pinned host memory, device construction
(tl_oriented_from_csr, TL_DEBUG_PREP timeline on stderr), count.

    TL_DEBUG_PREP=1 python tools/e2e_phases.py --config c4
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2006_11494_b200 import capi
    from paper_2006_11494_b200.configs import CONFIGS

    p = argparse.ArgumentParser()
    p.add_argument("--config", default="c2")
    p.add_argument("--reps", type=int, default=3)
    a = p.parse_args()
    cfg = CONFIGS[a.config]
    d = torch.empty(2 * cfg["npairs"], dtype=torch.int32, device="cuda")
    capi.gen_pairs_device(cfg, d.data_ptr())
    g = capi.DeviceGraph.from_device_pairs(d.data_ptr(), cfg["npairs"], cfg["n"])
    del d
    og = g.orient()
    g.close()
    n, m = og.n, og.m
    host = og.csr()
    og.close()
    torch.cuda.empty_cache()
    pin = {k: torch.from_numpy(host[k].view("int64" if host[k].dtype.itemsize == 8 else "int32")).pin_memory()
           for k in ("out_offsets", "out", "rank")}
    nbytes = sum(t.numel() * t.element_size() for t in pin.values())
    dev = torch.empty(pin["out"].numel(), dtype=torch.int32, device="cuda")
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(pin["out"], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"h2d col {dev.numel() * 4 / 1e9:.2f} GB in {dt * 1e3:.1f} ms = {dev.numel() * 4 / dt / 1e9:.1f} GB/s",
          flush=True)
    del dev
    torch.cuda.empty_cache()
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        up = capi.DeviceOriented.from_host_ptrs(n, m, pin["out_offsets"].data_ptr(), pin["out"].data_ptr(),
                                                pin["rank"].data_ptr())
        t1 = time.perf_counter()
        st = up.count()
        t2 = time.perf_counter()
        up.close()
        t3 = time.perf_counter()
        print(f"from_csr {1e3 * (t1 - t0):.1f} ms, count {1e3 * (t2 - t1):.1f} ms (kernel+prep "
              f"{st['list_ms'] + st['prep_ms']:.1f}), free {1e3 * (t3 - t2):.1f} ms, h2d {nbytes / 1e9:.2f} GB",
              flush=True)


if __name__ == "__main__":
    main()
