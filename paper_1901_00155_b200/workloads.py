"""The five seeded BASELINE.json workloads (synthetic float32 series).

Thin ctypes binding over ``csrc/series_gen.cpp`` (host-only C++).  The
generator, not this file, fixes the RNG family and the anomaly offsets;
``tests/golden/workloads.json`` pins the sha256 of every series.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_GEN_PATH = os.path.join(_HERE, "_lib", "libtsdd_gen.so")
_gen = None


def _lib():
    global _gen
    if _gen is None:
        if not os.path.exists(_GEN_PATH):
            raise RuntimeError(
                f"{_GEN_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(_GEN_PATH)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        intp = ctypes.POINTER(ctypes.c_int)
        lib.tsdd_workload_info.argtypes = [ctypes.c_int, u64p, u64p, u64p, u64p, intp, u64p, intp, u64p]
        lib.tsdd_workload_info.restype = ctypes.c_int
        lib.tsdd_workload_series.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, u64p]
        lib.tsdd_workload_series.restype = ctypes.c_int
        lib.tsdd_random_walk.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint64]
        lib.tsdd_random_walk.restype = ctypes.c_int
        _gen = lib
    return _gen


@dataclass(frozen=True)
class Workload:
    cfg: int            # 1..5 = BASELINE.json configs[cfg-1]
    m: int              # series length
    n: int              # subsequence (discord) length
    word_len: int       # PAA segments
    alphabet: int       # SAX cardinality
    k: int              # discords asked for
    seed: int
    anomalies: int
    anomaly_len: int

    @property
    def rows(self) -> int:
        return self.m - self.n + 1

    @property
    def name(self) -> str:
        return f"cfg{self.cfg}"


def workload(cfg: int) -> Workload:
    lib = _lib()
    m, n, w, a, seed, alen = (ctypes.c_uint64() for _ in range(6))
    k, an = ctypes.c_int(), ctypes.c_int()
    rc = lib.tsdd_workload_info(cfg, m, n, w, a, k, seed, an, alen)
    if rc != 0:
        raise ValueError(f"no such workload: cfg={cfg} (expected 1..5)")
    return Workload(cfg, m.value, n.value, w.value, a.value, k.value, seed.value, an.value, alen.value)


def series(cfg: int) -> tuple[np.ndarray, list[int]]:
    """float32 series of workload ``cfg`` and the 0-based starts of its planted windows."""
    w = workload(cfg)
    out = np.empty(w.m, dtype=np.float32)
    at = (ctypes.c_uint64 * 8)()
    rc = _lib().tsdd_workload_series(cfg, out.ctypes.data, w.m, at)
    if rc != 0:
        raise RuntimeError(f"tsdd_workload_series({cfg}) failed with code {rc}")
    return out, [int(at[i]) for i in range(w.anomalies)]


def random_walk(seed: int, m: int) -> np.ndarray:
    """Seeded Gaussian random walk, float32 (the SPEC.md:449-455 sweep family)."""
    out = np.empty(m, dtype=np.float32)
    rc = _lib().tsdd_random_walk(seed, out.ctypes.data, m)
    if rc != 0:
        raise RuntimeError(f"tsdd_random_walk failed with code {rc}")
    return out


def sha256(values: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(values).tobytes()).hexdigest()
