"""TEST INFRASTRUCTURE — ctypes access to the two CPU checkers.

* ``ref``    : the unmodified reference (``oracle/_ref/libtsdd_ref_*.so``,
               built by ``oracle/Makefile`` from ``/root/reference/proj``).
* ``port``   : this repo's plain-C restatement (``oracle/tsdd_oracle.c``),
               pinned against ``ref`` and the SPEC examples by
               ``tests/test_oracle_*.py``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_1901_00155_b200``) never does and has no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

u64 = ctypes.c_uint64
u64p = ctypes.POINTER(ctypes.c_uint64)
f64p = ctypes.POINTER(ctypes.c_double)
intp = ctypes.POINTER(ctypes.c_int)
vp = ctypes.c_void_p

ERR_PARAMETER, ERR_VALIDATION, ERR_INFEASIBLE = 2, 3, 4


class OracleError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"[{code}] {message}")
        self.code = code
        self.message = message


def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    flags = set(line.split(":", 1)[1].split())
                    return {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"} <= flags
    except OSError:
        pass
    return False


def _ptr(a):
    return None if a is None else a.ctypes.data


def _f64(values) -> np.ndarray:
    return np.ascontiguousarray(values, dtype=np.float64)


class _Checker:
    """Shared call surface of ref_* (reference shim) and orc_* (restatement)."""

    prefix = ""
    kind = ""

    def __init__(self, path: str):
        self.path = path
        self.lib = ctypes.CDLL(path)
        L, p = self.lib, self.prefix
        self._last_error = getattr(L, p + "last_error")
        self._last_error.restype = ctypes.c_char_p
        self._max_threads = getattr(L, p + "max_threads")
        self._max_threads.restype = ctypes.c_int
        self._run = getattr(L, p + "run_discovery")
        self._run.argtypes = [vp, u64, u64, u64, u64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                              ctypes.c_int, u64p, f64p, u64p, u64p, f64p, f64p]
        self._prepare = getattr(L, p + "prepare")
        self._prepare.argtypes = [vp, u64, u64, u64, u64, vp, vp, vp, vp, vp, vp, u64p, vp]
        self._distance = getattr(L, p + "distance")
        self._distance.argtypes = [vp, vp, u64, ctypes.c_double, u64, f64p, intp]
        self._paa_row = getattr(L, p + "paa_row")
        self._paa_row.argtypes = [vp, u64, vp, u64]
        self._symbol_for = getattr(L, p + "symbol_for")
        self._symbol_for.argtypes = [u64, ctypes.c_double, ctypes.POINTER(ctypes.c_uint32)]
        self._word_hash = getattr(L, p + "word_hash")
        self._word_hash.argtypes = [vp, u64, u64, u64p]
        self._z_normalize = getattr(L, p + "z_normalize")
        self._z_normalize.argtypes = [vp, u64]
        self._topk = getattr(L, p + "topk")
        self._topk.argtypes = [vp, u64, u64, u64, u64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               vp, vp, u64p, u64p, f64p, f64p]
        self._nn_profile = getattr(L, p + "nn_profile")
        self._nn_profile.argtypes = [vp, u64, u64, ctypes.c_int, vp]

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, (self._last_error() or b"").decode())

    def max_threads(self) -> int:
        return int(self._max_threads())

    def run_discovery(self, series, n, word_len=4, alphabet=4, engine="phidd", threads=None,
                      chunk=1, disable_pruning=False) -> dict:
        x = _f64(series)
        eng = {"brute": 0, "hotsax": 1, "phidd": 2}[engine]
        threads = threads or self.max_threads()
        pos, calls, ab = u64(), u64(), u64()
        dist, prep, search = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        self._check(self._run(x.ctypes.data, x.size, n, word_len, alphabet, eng, threads, chunk,
                              int(disable_pruning), pos, dist, calls, ab, prep, search))
        return dict(position=pos.value, distance=dist.value, calls=calls.value,
                    abandoned=ab.value, prep_s=prep.value, search_s=search.value,
                    threads=threads, engine=engine)

    def prepare(self, series, n, word_len, alphabet, want_rows=True) -> dict:
        x = _f64(series)
        N = x.size - n + 1
        if N < 1:
            N = 1
        rows = np.empty((N, n), dtype=np.float64) if want_rows else None
        paa = np.empty((N, word_len), dtype=np.float64)
        sax = np.empty((N, word_len), dtype=np.uint32)
        hashes = np.empty(N, dtype=np.uint64)
        freq = np.empty(N, dtype=np.uint32)
        cand = np.empty(N, dtype=np.uint64)
        ncand = u64()
        buckets = np.empty(N, dtype=np.uint64)
        self._check(self._prepare(x.ctypes.data, x.size, n, word_len, alphabet, _ptr(rows),
                                  paa.ctypes.data, sax.ctypes.data, hashes.ctypes.data,
                                  freq.ctypes.data, cand.ctypes.data, ncand, buckets.ctypes.data))
        return dict(rows=rows, paa=paa, sax=sax, hashes=hashes, freq=freq,
                    candidates=cand[: ncand.value].copy(), bucket_positions=buckets)

    def distance(self, a, b, threshold=float("inf"), block=8):
        a, b = _f64(a), _f64(b)
        val, ab = ctypes.c_double(), ctypes.c_int()
        self._check(self._distance(a.ctypes.data, b.ctypes.data, a.size, threshold, block, val, ab))
        return None if ab.value else val.value

    def paa_row(self, values, w) -> np.ndarray:
        v = _f64(values)
        out = np.empty(w, dtype=np.float64)
        self._check(self._paa_row(v.ctypes.data, v.size, out.ctypes.data, w))
        return out

    def symbol_for(self, alphabet, value) -> int:
        s = ctypes.c_uint32()
        self._check(self._symbol_for(alphabet, float(value), s))
        return int(s.value)

    def word_hash(self, word, alphabet) -> int:
        wv = np.ascontiguousarray(word, dtype=np.uint32)
        h = u64()
        self._check(self._word_hash(wv.ctypes.data, wv.size, alphabet, h))
        return int(h.value)

    def z_normalize(self, values) -> np.ndarray:
        v = _f64(values).copy()
        self._check(self._z_normalize(v.ctypes.data, v.size))
        return v

    def topk(self, series, n, word_len, alphabet, k, threads=None, chunk=1) -> dict:
        x = _f64(series)
        threads = threads or self.max_threads()
        pos = np.zeros(k, dtype=np.uint64)
        dist = np.zeros(k, dtype=np.float64)
        calls, ab = u64(), u64()
        prep, search = ctypes.c_double(), ctypes.c_double()
        self._check(self._topk(x.ctypes.data, x.size, n, word_len, alphabet, k, threads, chunk,
                               pos.ctypes.data, dist.ctypes.data, calls, ab, prep, search))
        return dict(positions=[int(p) for p in pos], distances=[float(d) for d in dist],
                    calls=calls.value, abandoned=ab.value, prep_s=prep.value,
                    search_s=search.value, threads=threads)

    def nn_profile(self, series, n, threads=None) -> np.ndarray:
        x = _f64(series)
        N = x.size - n + 1
        out = np.empty(N, dtype=np.float64)
        self._check(self._nn_profile(x.ctypes.data, x.size, n, threads or self.max_threads(),
                                     out.ctypes.data))
        return out


class Reference(_Checker):
    prefix = "ref_"
    kind = "reference"

    def generate_series(self, m, anomaly="none", anomaly_pos=0, anomaly_len=64, seed=0) -> np.ndarray:
        """The reference's generate_series (src/generate.cpp:19-59)."""
        fn = self.lib.ref_generate_series
        fn.argtypes = [u64, ctypes.c_char_p, u64, u64, u64, vp]
        out = np.empty(max(int(m), 1), dtype=np.float64)
        self._check(fn(int(m), anomaly.encode(), int(anomaly_pos), int(anomaly_len), int(seed), _ptr(out)))
        return out[:int(m)]


class Port(_Checker):
    prefix = "orc_"
    kind = "port"


_ref = None
_port = None


def ref_available() -> bool:
    return os.path.exists(os.path.join(_HERE, "_ref", "libtsdd_ref_v3.so"))


def ref() -> Reference:
    """The unmodified reference (prebuilt in this container, travels as a .so)."""
    global _ref
    if _ref is None:
        name = "libtsdd_ref_v4.so" if _cpu_has_avx512() else "libtsdd_ref_v3.so"
        path = os.path.join(_HERE, "_ref", name)
        if not os.path.exists(path):
            path = os.path.join(_HERE, "_ref", "libtsdd_ref_v3.so")
        if not os.path.exists(path):
            raise FileNotFoundError("oracle/_ref is not built: run `make -C oracle ref` where "
                                    "/root/reference exists")
        _ref = Reference(path)
    return _ref


def port() -> Port:
    """This repo's C restatement (compiled on demand from oracle/tsdd_oracle.c)."""
    global _port
    if _port is None:
        path = os.path.join(_HERE, "_build", "libtsdd_oracle.so")
        src = os.path.join(_HERE, "tsdd_oracle.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            import subprocess
            subprocess.run(["make", "-C", _HERE, "oracle"], check=True, capture_output=True)
        _port = Port(path)
    return _port


def best() -> _Checker:
    """The reference when its .so is present, else the restatement."""
    return ref() if ref_available() else port()
