"""Turns ncu outputs brought back in gpurun_out/ into the small text/JSON summaries kept
under profiles/ (the .ncu-rep itself is scratch).

    python tools/summarise_profiles.py launches gpurun_out/launches.csv profiles/r01_launches_bench_cfg5.txt
    python tools/summarise_profiles.py full gpurun_out/prof.ncu-rep profiles/r01_scan_tiles_cfg5
"""
import collections
import csv
import json
import subprocess
import sys

KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "lts__t_bytes.sum", "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum"]
STALLS = "smsp__average_warps_issue_stalled_"


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    H = rows[hdr]
    ki, vi, ui = H.index("Kernel Name"), H.index("Metric Value"), H.index("Metric Unit")
    scale = {"ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    total = sum(v[1] for v in agg.values())
    with open(dst, "w") as f:
        f.write(f"# source: {src} (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised:\n"
                f"# compare SHARES, not absolutes)\n# total {total / 1e6:.3f} ms over {sum(v[0] for v in agg.values())} launches\n")
        f.write(f"{'ms':>12} {'share%':>8} {'launches':>9}  kernel\n")
        for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{v[1] / 1e6:12.3f} {100 * v[1] / total:8.2f} {v[0]:9d}  {k}\n")
    print(open(dst).read())


def full(src, dst):
    raw = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    H, U = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        rec = {"kernel": r[H.index("Kernel Name")].split("(")[0], "grid": r[H.index("Grid Size")],
               "block": r[H.index("Block Size")]}
        for j, h in enumerate(H):
            if h in KEEP or h.startswith(STALLS):
                rec[f"{h} [{U[j]}]"] = r[j]
        out.append(rec)
    json.dump(out, open(dst + "_raw.json", "w"), indent=1)
    scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}

    def in_bytes(rec, name):
        key = next((k for k in rec if k.startswith(name + " [")), None)
        if key is None:
            return 0.0
        return float(rec[key]) * scale[key.split("[")[1].rstrip("]")]

    per_launch = [in_bytes(rec, "dram__bytes_read.sum") + in_bytes(rec, "dram__bytes_write.sum") for rec in out]
    summary = {"source": src, "launches_captured": len(out),
               "dram_bytes_per_launch": sum(per_launch) / max(1, len(per_launch)),
               "dram_bytes_each": per_launch}
    json.dump(summary, open(dst + "_summary.json", "w"), indent=1)
    print(json.dumps(summary))


if __name__ == "__main__" and sys.argv[1] in ("launches", "full"):
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])


def metrics(src, dst, workload):
    """Per-kernel summary of an `ncu --metrics ... --csv` pass over one search: launches, time, DRAM bytes,
    time-weighted pipe utilisations and the dominant stall reason.  Writes <dst>.json and <dst>.txt."""
    rows = list(csv.reader(open(src, errors="replace")))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    H = rows[hdr]
    ci = {name: H.index(name) for name in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "Grid Size")}
    launches = {}
    for r in rows[hdr + 1:]:
        if len(r) <= ci["Metric Value"]:
            continue
        rec = launches.setdefault(r[ci["ID"]], {"kernel": r[ci["Kernel Name"]].split("(")[0].replace("void ", "").replace("unnamed>::", ""),
                                                "grid": r[ci["Grid Size"]]})
        try:
            value = float(r[ci["Metric Value"]].replace(",", ""))
        except ValueError:
            continue
        unit = r[ci["Metric Unit"]]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6, "second": 1e3, "s": 1e3,
                 "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}.get(unit, 1.0)
        rec[r[ci["Metric Name"]]] = value * scale
    agg = collections.OrderedDict()
    for rec in launches.values():
        a = agg.setdefault(rec["kernel"], {"launches": 0, "ms": 0.0, "dram_read": 0.0, "dram_write": 0.0, "weighted": collections.Counter(),
                                           "longest": None})
        ms = rec.get("gpu__time_duration.sum", 0.0)
        a["launches"] += 1
        a["ms"] += ms
        a["dram_read"] += rec.get("dram__bytes_read.sum", 0.0)
        a["dram_write"] += rec.get("dram__bytes_write.sum", 0.0)
        for k, v in rec.items():
            if k.endswith("pct_of_peak_sustained_active") or k.endswith("pct_of_peak_sustained_elapsed") or k.endswith(".ratio") or k.endswith("hit_rate.pct"):
                a["weighted"][k] += v * ms
        if a["longest"] is None or ms > a["longest"]["ms"]:
            a["longest"] = {"ms": ms, "grid": rec["grid"], "dram_bytes": rec.get("dram__bytes_read.sum", 0.0) + rec.get("dram__bytes_write.sum", 0.0),
                            "fma_pipe_pct": rec.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                            "dram_pct": rec.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")}
    total = sum(a["ms"] for a in agg.values())
    out = {"source": src, "workload": workload, "note": "ncu --metrics pass, cold-cache and serialised: compare shares, not absolutes",
           "total_ms": total, "kernels": {}}
    lines = [f"# {src}: per-kernel ncu metrics of one {workload} search (time-weighted averages; cold-cache, serialised)",
             f"{'kernel':44} {'n':>4} {'ms':>8} {'share':>6} {'DRAM GB':>8} {'GB/s':>7} {'dram%':>6} {'fma%':>6} {'fp64%':>6} {'tensor%':>7} {'issue%':>6} {'occ%':>5}  top stall (per issue)"]
    for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
        w = {k: v / a["ms"] for k, v in a["weighted"].items()} if a["ms"] else {}
        stalls = {k.split("issue_stalled_")[1].replace("_per_issue_active.ratio", ""): v for k, v in w.items() if "issue_stalled" in k}
        top = max(stalls.items(), key=lambda kv: kv[1]) if stalls else ("-", 0.0)
        gb = (a["dram_read"] + a["dram_write"]) / 1e9
        k = {"launches": a["launches"], "ms": a["ms"], "share": a["ms"] / total if total else 0.0, "dram_gb": gb,
             "dram_gb_per_s": gb / (a["ms"] * 1e-3) if a["ms"] else 0.0,
             "dram_pct_of_peak": w.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
             "fma_pipe_pct": w.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
             "fp64_pipe_pct": w.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
             "tensor_pipe_pct": w.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
             "l2_hit_rate_pct": w.get("lts__t_sector_hit_rate.pct"),
             "issue_active_pct": w.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
             "warps_active_pct": w.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
             "l1_throughput_pct": w.get("l1tex__throughput.avg.pct_of_peak_sustained_active"),
             "l2_throughput_pct": w.get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
             "stalls_per_issue": dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:4]), "top_stall": top[0], "longest_launch": a["longest"]}
        out["kernels"][name] = k
        f = lambda v: f"{v:6.1f}" if v is not None else "     -"
        lines.append(f"{name[:44]:44} {a['launches']:4d} {a['ms']:8.3f} {100 * k['share']:5.1f}% {gb:8.3f} {k['dram_gb_per_s']:7.0f} "
                     f"{f(k['dram_pct_of_peak'])} {f(k['fma_pipe_pct'])} {f(k['fp64_pipe_pct'])} {f(k['tensor_pipe_pct'])}  {f(k['issue_active_pct'])} "
                     f"{(k['warps_active_pct'] or 0):5.1f}  {top[0]} {top[1]:.2f}")
    json.dump(out, open(dst + ".json", "w"), indent=1)
    open(dst + ".txt", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "metrics":
    metrics(sys.argv[2], sys.argv[3], sys.argv[4])
