#!/usr/bin/env python3
"""Regenerates the SAX breakpoint table `c_breaks` of csrc/prep_kernels.cu.

Cardinality a gets the a-1 quantiles of N(0,1) at k/a (equiprobable bins); the lower half
is computed with scipy's norm.ppf and mirrored onto the upper half, so the table is exactly
symmetric — the same construction, hence the same doubles, as the reference's built-in
table (/root/reference/proj/src/sax.cpp:14-46, tools/gen_breakpoints.py).  Row a-2 of the
output holds the thresholds of cardinality a; `tests/test_host.py` checks that the table
in the kernel source equals this script's output.
"""
from scipy.stats import norm


def breakpoints(cardinality: int) -> list:
    lower = [float(norm.ppf(k / cardinality)) for k in range(1, (cardinality + 1) // 2)]
    middle = [0.0] if cardinality % 2 == 0 else []
    return lower + middle + [-q for q in reversed(lower)]


def main() -> None:
    print("__constant__ double c_breaks[9][9] = {")
    for a in range(2, 11):
        print("    {" + ", ".join(repr(q) if q != 0.0 else "0" for q in breakpoints(a)) + "},")
    print("};")


if __name__ == "__main__":
    main()
