"""Runs BASELINE.json workloads on cuda:0 and prints result, timings and counters.

    python tools/run_workload.py 5 4 --opt batch=16384 --repeat 2
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1901_00155_b200 import Context, workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfgs", nargs="+", type=int)
    ap.add_argument("--opt", action="append", default=[], help="name=value engine tunable")
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--k", type=int, default=0)
    ap.add_argument("--prefix", type=int, default=0, help="use only the first PREFIX samples")
    ap.add_argument("--no-pruning", action="store_true", help="exhaustive scan (DiscoveryOptions::disable_pruning)")
    args = ap.parse_args()
    golden = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "workloads.json")))
    with Context(0) as ctx:
        for o in args.opt:
            name, value = o.split("=")
            ctx.set_option(name, float(value))
        for cfg in args.cfgs:
            w = W.workload(cfg)
            t0 = time.time()
            x, at = W.series(cfg)
            if args.prefix:
                x = x[:args.prefix]
            gen_s = time.time() - t0
            k = args.k or w.k
            for rep in range(args.repeat):
                t0 = time.time()
                ctx.prepare(x, w.n, w.word_len, w.alphabet)
                t1 = time.time()
                pos, dist = ctx.search(k, args.no_pruning)
                t2 = time.time()
                st = ctx.stats()
                want = golden.get(f"cfg{cfg}", {}).get("oracle") if not args.prefix else None
                ok = None if not want else (pos == want["positions"][:k])
                print(json.dumps(dict(cfg=cfg, rep=rep, m=len(x), n=w.n, k=k, positions=pos, distances=dist,
                                      golden_match=ok, gen_s=round(gen_s, 2), prepare_wall_s=round(t1 - t0, 4),
                                      search_wall_s=round(t2 - t1, 4), stats=st,
                                      terms_per_s=st["scan_kernel_terms"] / max(st["scan_kernel_ms"], 1e-9) * 1e3,
                                      planted=at)), flush=True)


if __name__ == "__main__":
    main()
