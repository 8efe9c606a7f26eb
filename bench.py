"""Benchmark of the discord-search hot path (prepare + search) on B200.

    python bench.py --gpus N --steps K --warmup W            # this repo's CUDA engine
    python bench.py --impl reference --gpus N --steps K ...  # the reference's CPU path

One "step" is one complete discord search (preparation stage + top-k search) of one
BASELINE.json workload.  Default workload: cfg5 (i.i.d. noise, m = 1,000,000, n = 256,
the "pruning worst case" that BASELINE.json uses for raw distance throughput).

Metric (BASELINE.json): subsequence-pair distances per second = distance evaluations
started (the reference's own counter, series.hpp:68-74,120) / step time; the end-to-end
top-k time of a step is reported beside it (`topk_time_s`).
  value : series already resident in HBM, prepare_device + search, CUDA events on the
          stream the kernels run on, max over ranks.
  e2e   : the reference-facing call (run_discovery with a HOST series in pinned memory):
          H2D copy + prepare + search + D2H of the result inside the timed region.
  roofline : the dominant kernel of the workload.  On inputs whose search switches to the
          dot-product form (cfg5) that is the tensor-core tile kernel k_scan_tiles_tc: `bound`
          "tensor", peak = MEASURED_PEAKS.json's dense bf16 figure (fp16 runs at the same rate),
          `achieved` = SURVEY.md 8d's 3 FLOP per term, `executed` = the 6 FLOP per term the kernel
          really issues (three fp16 MMAs on hi / lo split rows).  `cuda_core_path` then repeats
          the workload with the dot form on the CUDA cores (dot_form = 1) and carries the FP32
          roofline north_star asks for.  On other inputs (cfg4) the tile kernels are CUDA-core
          kernels and `roofline` is that FP32 line itself: `achieved` counts the floating-point
          operations the kernels EXECUTE — a term in the direct form (x-y)^2 = FADD + FFMA =
          3 FLOP, a term in the dot-product form = one FFMA = 2 FLOP; `algorithmic_tflops` is
          SURVEY.md 8d's figure (3 FLOP for every term).  Its `peak` is NOMINAL: 148 SMs x 128
          lanes x 2 FLOP x the maximum SM clock (MEASURED_PEAKS.json has no FP32 entry); an
          FFMA-only probe kernel measured live is reported beside it (`peak_probe`).
          `useful_frac` counts only the terms of live candidates against existing rows in
          real columns (no dead tile slots, no padding).
  cpu_baseline : the unmodified reference (oracle/_ref; else the C restatement) on the
          box's host cores, on a bounded sample (a prefix of the same series) — and the GPU
          on EXACTLY that sample beside it (`gpu_same_input_topk_time_s`).
  --gpus N without a launcher (no WORLD_SIZE in the environment): bench.py starts the N
          ranks itself, one process per GPU, each with the engine's own NCCL communicator.

The oracle is used here only as the timed CPU baseline, never on the product path.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "subsequence_pair_distances_per_s"
UNIT = "distances/s"
CPU_SAMPLE = {1: 65536, 2: 262144, 3: 300000, 4: 400000, 5: 200000}  # prefix lengths for the CPU arm
ORACLE_SHAPE = {4: (8, 4)}  # the reference rejects 4^16 words (sax.hpp:80); results are shape-independent


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region (B200_PROFILING.md)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.samples, self._stop, self._thread = index, [], threading.Event(), None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([c.strip() for c in out.splitlines()[0].split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._thread.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = [n for i, n in enumerate(names) if any(s[3 + i].lower().startswith("active") for s in self.samples)]
        power = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(self.samples[0][1]),
                "power_w_max": max(power) if power else None, "reasons": reasons, "samples": len(self.samples)}


def workload_inputs(cfg: int):
    from paper_1901_00155_b200 import workloads as W

    w = W.workload(cfg)
    x, _ = W.series(cfg)
    return w, x


def cpu_reference_run(cfg: int, x: np.ndarray, w, threads: int | None = None, sample_m: int | None = None) -> dict:
    """The reference's own CPU path (prepare + phidd search, exclusion-zone wrapper for k > 1)
    on a prefix of the workload's series.  The one place bench.py executes oracle/."""
    import oracle

    chk = oracle.best()
    sample_m = sample_m or min(CPU_SAMPLE[cfg], len(x))
    word_len, alphabet = ORACLE_SHAPE.get(cfg, (w.word_len, w.alphabet))
    threads = threads or os.cpu_count() or 1
    t0 = time.perf_counter()
    if w.k == 1:
        out = chk.run_discovery(x[:sample_m], w.n, word_len, alphabet, engine="phidd", threads=threads, chunk=64)
        calls, prep_s, search_s = out["calls"], out["prep_s"], out["search_s"]
    else:
        out = chk.topk(x[:sample_m], w.n, word_len, alphabet, w.k, threads=threads, chunk=64)
        calls, prep_s, search_s = out["calls"], out["prep_s"], out["search_s"]
    wall = time.perf_counter() - t0
    step_s = prep_s + search_s
    return {"value": calls / step_s, "unit": UNIT, "cores": threads, "kind": chk.kind,
            "sample": f"prefix of {sample_m} samples of cfg{cfg} (n={w.n}, k={w.k}, SAX {word_len}x{alphabet}), "
                      f"engine=phidd chunk=64",
            "calls": calls, "prep_s": prep_s, "search_s": search_s, "wall_s": wall, "topk_time_s": step_s,
            "sample_m": sample_m, "positions": out.get("positions", [out.get("position")])}


def run_reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w, x = workload_inputs(args.workload)
    sample_m = min(CPU_SAMPLE[args.workload], len(x))
    # warm-up: W short runs (thread pool, page faults, code) on a 20,000-sample prefix — a full
    # sample run costs 10+ s and a CPU search keeps no state between runs
    warm_m = min(20000, sample_m)
    for _ in range(args.warmup):
        cpu_reference_run(args.workload, x, w, sample_m=warm_m)
    runs = [cpu_reference_run(args.workload, x, w) for _ in range(max(1, args.steps))]
    step_s = [r["topk_time_s"] for r in runs]
    calls = runs[0]["calls"]
    value = sum(r["calls"] for r in runs) / sum(step_s)
    base = dict(runs[0])
    base["value"] = value
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": len(runs), "warmup": args.warmup, "ms_per_step": 1e3 * sum(step_s) / len(runs),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        # the series the CPU arm really searches: a PREFIX of the workload (the full one takes the
        # reference about an hour); the CUDA arm times this same prefix as well
        # (cpu_baseline.gpu_same_input_topk_time_s on its line)
        "config": {"workload": f"cfg{args.workload}", "m": sample_m, "n": w.n, "k": w.k, "full_m": w.m,
                   "sample": base["sample"], "warmup_sample": f"prefix of {warm_m} samples"},
        "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "topk_time_s": sum(step_s) / len(runs), "calls_per_step": calls, "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def run_cuda_arm(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_1901_00155_b200 import Context, DiscoveryConfig, parallel, run_discovery

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device; the engine has no CPU fallback")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    w, x = workload_inputs(args.workload)
    k = w.k
    host = torch.from_numpy(x).pin_memory()          # e2e arm: pinned host buffer
    x_pinned = host.numpy()
    dev = host.to(f"cuda:{local}", non_blocking=False)  # value arm: resident in HBM
    stream = torch.cuda.current_stream()

    ctx = Context(local)
    ctx.set_stream(stream.cuda_stream)
    for opt in args.opt:
        name, val = opt.split("=")
        ctx.set_option(name, float(val))
    if world > 1:
        parallel.attach_nccl(ctx)  # the engine's own communicator (ncclCommInitRank inside libtsdd_cuda.so)
    comm_nranks = ctx.comm_size()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def device_step():
        ctx.prepare_device(dev.data_ptr(), w.m, w.n, w.word_len, w.alphabet)
        pos, dd = ctx.search(k)
        return pos, dd, ctx.stats()

    def host_step():
        out = run_discovery(x_pinned, DiscoveryConfig(n=w.n, word_len=w.word_len, alphabet=w.alphabet, k=k,
                                                      device=local), context=ctx)
        return [d.position for d in out.discords], [d.distance for d in out.discords], out.stats

    # FP32 peak, measured on this device now (FFMA-only stream; one FFMA = 2 FLOP)
    ffma_ops, _ = ctx.fp32_probe(0)
    mix_ops, _ = ctx.fp32_probe(3)

    for _ in range(args.warmup):
        device_step()
    barrier()
    sampler = ClockSampler(local)
    totals = {"calls": 0, "terms": 0, "scan_terms": 0, "scan_ms": 0.0, "scan_launches": 0, "ws_launches": 0,
              "dot_launches": 0, "dot_terms": 0, "useful_terms": 0, "tc_terms": 0, "tc_ms": 0.0, "tc_launches": 0,
              "launches": 0,
              "prep_ms": 0.0, "search_ms": 0.0, "build_rows_ms": 0.0, "encode_ms": 0.0, "index_ms": 0.0}
    with sampler:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            pos, dd, st = device_step()
            totals["calls"] += st["calls"]
            totals["terms"] += st["terms"]
            totals["scan_terms"] += st["scan_kernel_terms"]
            totals["scan_ms"] += st["scan_kernel_ms"]
            totals["scan_launches"] += st["scan_kernel_launches"]
            totals["ws_launches"] += st["scan_kernel_ws_launches"]
            totals["dot_launches"] += st["scan_kernel_dot_launches"]
            totals["dot_terms"] += st["scan_kernel_dot_terms"]
            totals["useful_terms"] += st["useful_terms"]
            totals["tc_terms"] += st["scan_kernel_tc_terms"]
            totals["tc_ms"] += st["scan_kernel_tc_ms"]
            totals["tc_launches"] += st["scan_kernel_tc_launches"]
            totals["launches"] += st["kernel_launches"]
            for key in ("prep_ms", "search_ms", "build_rows_ms", "encode_ms", "index_ms"):
                totals[key] += st[key]
        ev1.record(stream)
        barrier()
        elapsed_ms = ev0.elapsed_time(ev1)

        # end to end through the reference-facing call, host buffers
        host_step()
        barrier()
        t0 = time.perf_counter()
        e2e_calls = 0
        for _ in range(args.steps):
            pos_h, dd_h, st_h = host_step()
            e2e_calls += st_h["calls"]
        barrier()
        e2e_s = time.perf_counter() - t0
    assert pos_h == pos, (pos_h, pos)

    t = torch.tensor([elapsed_ms, e2e_s], dtype=torch.float64, device=f"cuda:{local}")
    c = torch.tensor([totals["calls"], e2e_calls], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(c, op=dist.ReduceOp.SUM)
    elapsed_ms, e2e_s = float(t[0]), float(t[1])
    all_calls, all_e2e_calls = float(c[0]), float(c[1])

    if rank == 0:
        golden_ok, golden_all = None, {}
        try:
            golden_all = json.load(open(os.path.join(ROOT, "tests", "golden", "workloads.json")))
            rec = golden_all.get(f"cfg{args.workload}")
            if rec:
                golden_ok = pos == rec["oracle"]["positions"]
        except OSError:
            pass
        clocks = sampler.summary()
        sm_max_mhz = clocks.get("sm_max_mhz") or _measured_peak("sm_max_mhz", 1965.0)[0]
        props = torch.cuda.get_device_properties(local)
        # DRAM traffic of the dominant kernel: only from an ncu capture of THIS workload
        traffic, prof = None, {}
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json"))).get(f"cfg{args.workload}", {})
            traffic = prof.get("dram_bytes_per_launch")
        except (OSError, ValueError):
            pass
        N = w.m - w.n + 1
        matrix_bytes = 4.0 * N * ((w.n + 31) // 32 * 32)
        line = {
            "metric": METRIC, "value": all_calls / (elapsed_ms * 1e-3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": f"cfg{args.workload}", "m": w.m, "n": w.n, "word_len": w.word_len,
                       "alphabet": w.alphabet, "k": k, "rows": N,
                       "parallelism": f"candidates sharded over {world} rank(s), per-batch NCCL max-allreduce"
                       if world > 1 else "single GPU",
                       "l2": "inputs larger than L2" if matrix_bytes > 126e6 else
                       "matrix fits L2; every step rebuilds it from the series"},
            "topk_time_s": elapsed_ms * 1e-3 / args.steps,
            "discords": {"positions": pos, "distances": dd, "matches_golden": golden_ok},
            "e2e": {"value": all_e2e_calls / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(x.nbytes),
                    "d2h_bytes_per_step": int(k * 16 + 160), "topk_time_s": e2e_s / args.steps},
            "gpu_launches": int(totals["launches"]),
            "roofline": None,
            "roofline_prep": {"bound": "hbm", "kernel": "k_build_rows", "unit": "GB/s",
                              "achieved": matrix_bytes * args.steps / (totals["build_rows_ms"] * 1e-3) / 1e9
                              if totals["build_rows_ms"] else None,
                              "peak": _measured_peak("hbm_gbs", 6650.0)[0],
                              "peak_source": _measured_peak("hbm_gbs", 6650.0)[1]},
            "stage_ms_per_step": {key: totals[key] / args.steps for key in
                                  ("prep_ms", "encode_ms", "build_rows_ms", "index_ms", "search_ms")},
            "calls_per_step": all_calls / args.steps, "terms_per_step": totals["terms"] / args.steps,
            "clocks": clocks,
            "comm": {"nranks": comm_nranks, "backend": "the engine's own NCCL communicator (tsdd_cuda_comm_init -> "
                     "ncclCommInitRank; nranks from ncclCommCount)" if world > 1 else "none (one rank)"},
        }
        rp = line["roofline_prep"]
        rp["frac"] = rp["achieved"] / rp["peak"] if rp["achieved"] else None
        fp32 = fp32_roofline(totals, elapsed_ms, props.multi_processor_count, sm_max_mhz, ffma_ops, mix_ops)
        if totals["tc_ms"] > 0.5 * totals["scan_ms"]:  # (by TIME inside the tile kernels)
            # the dominant kernel is the tensor-core tile kernel: the tensor roofline is the line's roofline,
            # the CUDA-core tile kernels' FP32 line (the same workload with dot_form = 1) follows below
            line["roofline"] = tensor_roofline(totals, elapsed_ms, traffic, prof)
            line["dtype"] = "f32 (tile products: fp16 hi/lo parts on the tensor cores, float32 accumulation; decision in f64)"
        else:
            fp32.update({"traffic": traffic,
                         "traffic_source": ("ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum of ONE captured "
                                            "launch of this workload (%s; %s ms; %s) — compare with that launch, not "
                                            "with avg_launch_ms" % (prof.get("captured_kernel"), prof.get("captured_launch_ms"),
                                                                    prof.get("source"))) if traffic else
                                           "no ncu capture of this workload's dominant kernel is on file"})
            line["roofline"] = fp32
        if world == 1 and not args.no_secondary and args.workload != 4:
            line["other_workloads"] = {"cfg4": time_other_workload(ctx, 4, local, golden_all)}
        if (world == 1 and not args.no_secondary and not any(o.startswith("dot_form") for o in args.opt)
                and line["roofline"]["bound"] == "tensor"):
            # the SAME workload with the dot-product form on the CUDA cores (dot_form = 1: k_scan_tiles_ws16, the
            # kernel north_star's FP32 roofline is about), with that path's own FP32 roofline
            cc = time_other_workload(ctx, args.workload, local, golden_all, options={"dot_form": 1})
            ctx.set_option("dot_form", 5)
            t1 = cc.pop("totals")
            cc["roofline"] = fp32_roofline(t1, t1["elapsed_ms"], props.multi_processor_count, sm_max_mhz, ffma_ops, mix_ops)
            line["cuda_core_path"] = cc
        if world == 1 and not args.no_cpu_baseline:
            cb = cpu_reference_run(args.workload, x, w)
            line["cpu_baseline"] = {key: cb[key] for key in ("value", "unit", "cores", "kind", "sample",
                                                             "calls", "topk_time_s")}
            # the GPU on EXACTLY the series the CPU arm searched (same prefix, same n / k; the
            # workload's own SAX shape — results do not depend on it): time against time
            same = time_same_input(ctx, x[:cb["sample_m"]], w, local)
            line["cpu_baseline"].update({
                "gpu_same_input_topk_time_s": same["topk_time_s"], "gpu_same_input_e2e_topk_time_s": same["e2e_topk_time_s"],
                "gpu_same_input_positions_match": same["positions"] == cb["positions"],
                "time_ratio_cpu_over_gpu_same_input": cb["topk_time_s"] / same["e2e_topk_time_s"]})
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def fp32_roofline(totals: dict, elapsed_ms: float, sms: int, sm_max_mhz: float, ffma_ops: float, mix_ops: float) -> dict:
    """The CUDA-core tile kernels against the FP32 FMA peak: executed FLOP (3 per direct-form term, 2 per
    dot-form term; tensor-core terms excluded) over the time inside those kernels."""
    scan_s = (totals["scan_ms"] - totals["tc_ms"]) * 1e-3
    cc_terms = totals["scan_terms"] - totals["tc_terms"]
    dot_terms = totals["dot_terms"] - totals["tc_terms"]
    direct_terms = cc_terms - dot_terms
    useful_share = totals["useful_terms"] / max(1, totals["scan_terms"])
    executed_flop = 3.0 * direct_terms + 2.0 * dot_terms
    pipe_ops = 2.0 * direct_terms + 1.0 * dot_terms  # FP32-pipe lane operations
    achieved = executed_flop / scan_s / 1e12 if scan_s > 0 else 0.0
    peak = sms * 128 * 2 * sm_max_mhz * 1e6 / 1e12  # nominal FP32 FMA peak
    peak_probe = 2.0 * ffma_ops / 1e12
    launches = totals["scan_launches"] - totals["tc_launches"]
    return {"bound": "fp32",
            "kernel": "k_scan_tiles_ws16 / k_scan_tiles_ws / k_scan_tiles (the CUDA-core tile kernels: %d launches, "
                      "%d warp-specialised, %d in the dot-product form, which runs on k_scan_tiles_ws16 while a "
                      "batch fills 256-candidate tiles)" % (launches, totals["ws_launches"] - totals["tc_launches"],
                                                            totals["dot_launches"] - totals["tc_launches"]),
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else None,
            "peak_source": "nominal: %d SMs x 128 FP32 lanes x 2 FLOP x %.0f MHz (the maximum SM clock; "
                           "MEASURED_PEAKS.json has no FP32 entry and B200_PROFILING.md states no FP32 "
                           "fallback)" % (sms, sm_max_mhz),
            "peak_probe": peak_probe, "frac_probe": achieved / peak_probe if peak_probe else None,
            "peak_probe_source": "live FFMA-only probe kernel (csrc/probe_kernels.cu: 16 independent "
                                 "FFMA chains per thread, nothing else in the loop) x 2 FLOP",
            "useful_share_of_terms": useful_share, "useful_frac": achieved * useful_share / peak,
            "useful_definition": "terms of (live candidate, existing neighbour row) pairs in columns "
                                 "t < n: no dead or empty candidate slots of a tile, no slots past the "
                                 "last row, no zero padding of the row stride (share over ALL tile kernels)",
            "terms_per_s": cc_terms / scan_s if scan_s else 0.0,
            "dot_form_share_of_terms": dot_terms / max(1, cc_terms),
            "algorithmic_tflops": 3.0 * cc_terms / scan_s / 1e12 if scan_s else 0.0,
            "fma_pipe_util": pipe_ops / scan_s / (peak * 1e12 / 2.0) if scan_s else 0.0,
            "fma_pipe_util_vs_probe": pipe_ops / scan_s / ffma_ops if scan_s else 0.0,
            "sub_fma_mix_probe_lane_ops_per_s": mix_ops, "ffma_probe_lane_ops_per_s": ffma_ops,
            "launches": int(launches), "avg_launch_ms": scan_s * 1e3 / max(1, launches),
            "kernel_share_of_step": scan_s * 1e3 / elapsed_ms}


def tensor_roofline(totals: dict, elapsed_ms: float, traffic, prof: dict) -> dict:
    """k_scan_tiles_tc against the dense 16-bit tensor peak (MEASURED_PEAKS.json: cuBLAS bf16, burst; fp16
    runs at the same rate).  `achieved` counts SURVEY 8(d)'s 3 FLOP per term; the kernel EXECUTES three
    fp16 MMAs = 6 FLOP per term (hi.hi + hi.lo + lo.hi of the split rows): `executed` / `frac_executed`
    say how busy the tensor pipe is."""
    tc_s = totals["tc_ms"] * 1e-3
    peak, src = _measured_peak("bf16_tflops", 2250.0)
    algorithmic = 3.0 * totals["tc_terms"] / tc_s / 1e12
    executed = 6.0 * totals["tc_terms"] / tc_s / 1e12
    return {"bound": "tensor", "kernel": "k_scan_tiles_tc<symmetric, fp16> (csrc/tc_kernels.cu: tcgen05.mma kind::f16, "
                                         "TMEM accumulators, TMA boxes; %d of %d tile-kernel launches, %.1f %% of all terms)"
                                         % (totals["tc_launches"], totals["scan_launches"],
                                            100.0 * totals["tc_terms"] / max(1, totals["scan_terms"])),
            "achieved": algorithmic, "peak": peak, "unit": "TFLOP/s", "frac": algorithmic / peak,
            "peak_source": src + " bf16_tflops (burst: the kernel's launches are timed one by one)",
            "executed": executed, "frac_executed": executed / peak,
            "flop_per_term": {"algorithmic": 3, "executed": 6},
            "terms_per_s": totals["tc_terms"] / tc_s, "launches": int(totals["tc_launches"]),
            "avg_launch_ms": totals["tc_ms"] / max(1, totals["tc_launches"]),
            "kernel_share_of_step": totals["tc_ms"] / elapsed_ms,
            "useful_share_of_terms": totals["useful_terms"] / max(1, totals["scan_terms"]),
            "traffic": traffic,
            "traffic_source": ("ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum of ONE captured launch of this "
                               "workload (%s; %s ms; %s) — compare with that launch, not with avg_launch_ms"
                               % (prof.get("captured_kernel"), prof.get("captured_launch_ms"), prof.get("source")))
            if traffic else "no ncu capture of this workload's dominant kernel is on file"}


def time_same_input(ctx, sample: np.ndarray, w, device: int, repeats: int = 3) -> dict:
    """Device-resident and end-to-end (host series) top-k time of `sample`, median of `repeats`."""
    import torch

    from paper_1901_00155_b200 import DiscoveryConfig, run_discovery

    host = torch.from_numpy(np.ascontiguousarray(sample)).pin_memory()
    dev = host.to(f"cuda:{device}")
    cfg = DiscoveryConfig(n=w.n, word_len=w.word_len, alphabet=w.alphabet, k=w.k, device=device)
    resident, e2e, pos = [], [], None
    for r in range(repeats + 1):  # (the first run allocates)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.prepare_device(dev.data_ptr(), len(sample), w.n, w.word_len, w.alphabet)
        pos, _ = ctx.search(w.k)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        run_discovery(host.numpy(), cfg, context=ctx)
        t2 = time.perf_counter()
        if r:
            resident.append(t1 - t0)
            e2e.append(t2 - t1)
    return {"topk_time_s": statistics.median(resident), "e2e_topk_time_s": statistics.median(e2e), "positions": pos}


def time_other_workload(ctx, cfg: int, device: int, golden: dict, repeats: int = 3, options: dict | None = None) -> dict:
    """A secondary figure on the same line: one more BASELINE.json workload (or the same one under
    other engine options), device-resident, median of `repeats` complete top-k searches
    (preparation + search, CUDA events)."""
    import torch

    w, x = workload_inputs(cfg)
    dev = torch.from_numpy(x).to(f"cuda:{device}")
    stream = torch.cuda.current_stream()
    times, pos, st = [], None, {}
    for name, value in (options or {}).items():
        ctx.set_option(name, value)
    for r in range(repeats + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.prepare_device(dev.data_ptr(), w.m, w.n, w.word_len, w.alphabet)
        pos, _ = ctx.search(w.k)
        e1.record(stream)
        torch.cuda.synchronize()
        if r:
            times.append(e0.elapsed_time(e1) * 1e-3)
        st = ctx.stats()
    rec = golden.get(f"cfg{cfg}")
    out = {"m": w.m, "n": w.n, "k": w.k, "topk_time_s": statistics.median(times), "runs": repeats,
           "prep_ms": st["prep_ms"], "search_ms": st["search_ms"], "calls": st["calls"],
           "matches_golden": (pos == rec["oracle"]["positions"]) if rec else None}
    if options:
        out.update({"options": options, "scan_kernel_ms": st["scan_kernel_ms"],
                    "tensor_core_launches": st["scan_kernel_tc_launches"],
                    "tensor_core_share_of_terms": st["scan_kernel_tc_terms"] / max(1, st["scan_kernel_terms"]),
                    "totals": {"scan_ms": st["scan_kernel_ms"], "tc_ms": st["scan_kernel_tc_ms"],
                               "scan_terms": st["scan_kernel_terms"], "tc_terms": st["scan_kernel_tc_terms"],
                               "dot_terms": st["scan_kernel_dot_terms"], "useful_terms": st["useful_terms"],
                               "scan_launches": st["scan_kernel_launches"], "tc_launches": st["scan_kernel_tc_launches"],
                               "ws_launches": st["scan_kernel_ws_launches"], "dot_launches": st["scan_kernel_dot_launches"],
                               "elapsed_ms": times[-1] * 1e3}})
    return out


def _measured_peak(key: str, fallback: float):
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))[key]), "MEASURED_PEAKS.json"
    except (OSError, KeyError, ValueError):
        return fallback, "fallback (B200_PROFILING.md)"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--opt", action="append", default=[], help="engine tunable name=value")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the cfg4 figure on the cfg5 line")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args.gpus))
    else:
        run_cuda_arm(args)


def spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` without a launcher: start the N ranks here, one process per GPU
    (RANK / LOCAL_RANK / WORLD_SIZE / MASTER_* as torchrun would set them).  Rank 0 prints the line."""
    import torch

    have = torch.cuda.device_count()
    if have < n:
        raise SystemExit(f"bench.py: --gpus {n} needs {n} CUDA devices, this machine has {have}")
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    procs = []
    for rank in range(n):
        env = dict(os.environ, RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE=str(n), LOCAL_WORLD_SIZE=str(n),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, os.path.abspath(__file__), *sys.argv[1:]], env=env))
    codes = [p.wait() for p in procs]
    return max(abs(c) for c in codes)


if __name__ == "__main__":
    main()
