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


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
