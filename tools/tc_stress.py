"""Repeats searches with the tensor-core kernel to flush out rare pipeline stalls:  python tools/tc_stress.py [reps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1901_00155_b200 import Context, workloads as W

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 30
w = W.workload(5); x, _ = W.series(5)
with Context(0) as c:
    for form in (3, 4):
        c.set_option("dot_form", form)
        for r in range(reps):
            t0 = time.time()
            c.prepare(x, w.n, w.word_len, w.alphabet)
            pos, dist = c.search(1)
            st = c.stats()
            print(form, r, pos, "search %.1f ms scan %.1f tc %d wall %.3f" % (st["search_ms"], st["scan_kernel_ms"], st["scan_kernel_tc_launches"], time.time() - t0), flush=True)
