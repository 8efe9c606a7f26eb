"""Absolute error of the exhaustive nn profile (no pruning) under the dot-form kernels against the
float64 oracle: CUDA cores (dot_form 2) vs tensor cores (dot_form 4: tf32 parts, 6: fp16 parts).   python tools/tc_error_probe.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_1901_00155_b200 import Context

chk = oracle.best()
rng = np.random.default_rng(1)
for kind, m, n in [("noise", 20000, 64), ("noise", 20000, 65), ("noise", 30000, 256), ("walk", 20000, 128)]:
    x = rng.random(m).astype(np.float32) if kind == "noise" else np.cumsum(rng.standard_normal(m)).astype(np.float32)
    want = chk.nn_profile(x, n)
    with Context(0) as c:
        for form in (0, 2, 4, 6):
            c.set_option("dot_form", form)
            c.prepare(x, n, 4, 4)
            got = c.nn_profile().astype(np.float64)
            st = c.stats()
            err = got - want
            E = (n + 32) * n * 2.0 ** -24
            print(kind, m, n, "dot_form", form, "tc launches", st["scan_kernel_tc_launches"], "max |err| %.3g  mean err %.3g  min err %.3g  (E = %.3g, typical nn^2 %.1f)"
                  % (np.abs(err).max(), err.mean(), err.min(), E, np.median(want)), flush=True)
