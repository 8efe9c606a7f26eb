"""Time of one exhaustive (no pruning) scan with the tensor-core kernel: python tools/tc_time_profile.py [form]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1901_00155_b200 import Context
form = int(sys.argv[1]) if len(sys.argv) > 1 else 4
x = np.random.default_rng(3).random(80000).astype(np.float32)
with Context(0) as c:
    c.set_option("dot_form", form)
    c.prepare(x, 256, 8, 4)
    for r in range(3):
        c.nn_profile()
        st = c.stats()
        print("form", form, "rep", r, "search %.2f ms scan %.2f ms terms %.3g tc_launches %d  -> %.3g terms/s" % (
            st["search_ms"], st["scan_kernel_ms"], st["scan_kernel_terms"], st["scan_kernel_tc_launches"],
            st["scan_kernel_terms"] / (st["scan_kernel_ms"] * 1e-3)), flush=True)
