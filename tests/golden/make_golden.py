"""Generates tests/golden/workloads.json from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref, i.e. /root/reference):

    python tests/golden/make_golden.py [cfg ...]

For every BASELINE.json workload it records the sha256 of the seeded float32
series (paper_1901_00155_b200/workloads.py) and the reference's top-k
discords (oracle.ref().topk: the exclusion-zone wrapper over the reference's
public potential_discord_stage / refine_discord_stage; phidd_discord itself
for k = 1), together with the reference timings on this container's cores.

Workload 4 asks for SAX shape (16, 4) = 2^32 words, which the reference's
2^24 guard rejects (sax.hpp:80, pipeline.cpp:41-42).  Position and distance
do not depend on the SAX shape (every engine is exact), so the reference is
run at (8, 4) for that workload and the shape used is recorded.
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1901_00155_b200 import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "workloads.json")
ORACLE_SHAPE = {4: (8, 4)}  # legal stand-in SAX shapes (gap G2)
CHUNK = 64


def main(cfgs):
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    ref = oracle.ref()
    for cfg in cfgs:
        w = W.workload(cfg)
        x, at = W.series(cfg)
        word_len, alphabet = ORACLE_SHAPE.get(cfg, (w.word_len, w.alphabet))
        t0 = time.time()
        out = ref.topk(x, w.n, word_len, alphabet, w.k, chunk=CHUNK)
        wall = time.time() - t0
        data[w.name] = dict(
            cfg=cfg, m=w.m, n=w.n, word_len=w.word_len, alphabet=w.alphabet, k=w.k, seed=w.seed,
            sha256=W.sha256(x), anomaly_starts_0based=at,
            oracle=dict(kind="reference", sax_shape=[word_len, alphabet], chunk=CHUNK,
                        threads=out["threads"], positions=out["positions"],
                        distances=out["distances"], calls=out["calls"],
                        abandoned=out["abandoned"], prep_s=out["prep_s"],
                        search_s=out["search_s"], wall_s=wall),
        )
        print(w.name, data[w.name]["oracle"], flush=True)
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)
            f.write("\n")


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3, 5, 4])
