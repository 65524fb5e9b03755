"""Summarise an ncu capture (+ launch list) into markdown / JSON for profiles/.

    python tools/ncu_summary.py REPORT.ncu-rep LAUNCHES.csv --config c2 --out profiles/NAME.md
        [--traffic profiles/traffic_c2.json]
"""
import argparse
import collections
import csv
import io
import json
import subprocess


def ncu_csv(report, *args):
    out = subprocess.run(["ncu", "-i", report, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def details(report):
    rows = ncu_csv(report, "--page", "details")
    h = rows[0]
    d = {}
    for r in rows[1:]:
        x = dict(zip(h, r))
        d[x.get("Metric Name")] = (x.get("Metric Value"), x.get("Metric Unit"), x.get("Kernel Name"))
    return d


def raw(report):
    rows = ncu_csv(report, "--page", "raw")
    return {k: (u, v) for k, u, v in zip(rows[0], rows[1], rows[2])}


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return 0.0


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ix = {k: i for i, k in enumerate(h)}
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) < len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        t = num(r[ix["Metric Value"]])
        unit = r[ix["Metric Unit"]]
        t_us = t / 1000 if unit in ("ns", "nsecond") else (t * 1000 if unit in ("ms", "msecond") else t)
        name = r[ix["Kernel Name"]].replace("void ", "").replace("tlb::<unnamed>::", "")
        name = name.replace("(tlb::AotMode)", "mode ")
        depth, cut = 0, len(name)
        for i, ch in enumerate(name):  # drop the argument list, keep template arguments
            depth += ch == "<"
            depth -= ch == ">"
            if ch == "(" and depth == 0:
                cut = i
                break
        name = name[:cut]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t_us
    return agg


def top_lines(report, n=12):
    rows = ncu_csv(report, "--page", "source", "--print-source", "cuda,sass")
    h = rows[2]
    ix = {}
    for i, k in enumerate(h):
        ix.setdefault(k, i)
    data = [r for r in rows[3:] if len(r) > 10 and r[0].isdigit() and r[2] == "-"]
    tot_s = sum(num(r[ix["Warp Stall Sampling (All Samples)"]]) for r in data) or 1
    tot_i = sum(num(r[ix["Instructions Executed"]]) for r in data) or 1
    stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    out = []
    for r in sorted(data, key=lambda r: -num(r[ix["Warp Stall Sampling (All Samples)"]]))[:n]:
        st = sorted(((num(r[ix[c]]), c[6:]) for c in stall_cols), reverse=True)[:2]
        out.append((r[0], 100 * num(r[ix["Warp Stall Sampling (All Samples)"]]) / tot_s,
                    100 * num(r[ix["Instructions Executed"]]) / tot_i, st, r[1].strip()[:90]))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("launch_csv", nargs="?")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--out", required=True)
    ap.add_argument("--traffic")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    d = details(a.report)
    rw = raw(a.report)
    kname = next(iter(v[2] for v in d.values() if v[2]), "?")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

    def nbytes(metric):  # each metric carries its own unit
        unit, v = rw.get(metric, ("byte", 0))
        return num(v) * scale.get(unit, 1)

    traffic = nbytes("dram__bytes_read.sum") + nbytes("dram__bytes_write.sum")
    keys = ["Duration", "Elapsed Cycles", "SM Active Cycles", "Executed Ipc Active", "Issue Slots Busy",
            "Issued Instructions", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
            "L1/TEX Hit Rate", "L2 Hit Rate", "L1/TEX Cache Throughput", "L2 Cache Throughput", "DRAM Throughput",
            "Memory Throughput", "No Eligible", "Dynamic Shared Memory Per Block"]
    lines = [f"# ncu summary {a.title}", "", f"kernel: `{kname}` (config {a.config}, 1 launch, "
             "`ncu --set full --clock-control none --import-source on`)", "",
             "| metric | value |", "|---|---|"]
    for k in keys:
        if k in d:
            lines.append(f"| {k} | {d[k][0]} {d[k][1]} |")
    lines.append(f"| dram__bytes_read.sum + dram__bytes_write.sum | {traffic / 1e9:.3f} GB per launch |")
    for key, label in (("lts__t_sector_hit_rate.pct", "L2 sector hit rate (lts__t_sector_hit_rate.pct)"),
                       ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                        "shared-memory wavefronts, % of peak"),
                       ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared-memory load bank conflicts"),
                       ("memory_l1_wavefronts_shared", "shared-memory wavefronts (actual)"),
                       ("memory_l1_wavefronts_shared_ideal", "shared-memory wavefronts (conflict-free ideal)")):
        if key in rw:
            unit, v = rw[key]
            lines.append(f"| {label} | {v} {unit} |")
    agg = launches(a.launch_csv) if a.launch_csv else {}
    tot = sum(t for _, t in agg.values()) or 1
    lines += [] if not agg else ["", "## launch list (cold-cache, serialised: compare shares)", "",
              "| kernel | launches | avg µs | share of listed GPU time |", "|---|---|---|---|"]
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:  # noqa: B007
        lines.append(f"| `{name[:70]}` | {c} | {t / c:.1f} | {100 * t / tot:.1f}% |")
    lines += ["", "## top source lines by stall samples", "", "| line | stall % | inst % | top stalls | source |",
              "|---|---|---|---|---|"]
    for ln, s, i, st, src in top_lines(a.report):
        lines.append(f"| {ln} | {s:.1f} | {i:.1f} | {', '.join(f'{n}:{int(v)}' for v, n in st)} | `{src}` |")
    open(a.out, "w").write("\n".join(lines) + "\n")
    if a.traffic:
        json.dump({"config": a.config, "kernel": kname, "dram_bytes_per_launch": traffic,
                   "source": a.report}, open(a.traffic, "w"), indent=1)
    print("\n".join(lines[:30]))


if __name__ == "__main__":
    main()
