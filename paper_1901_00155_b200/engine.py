"""Host-side mirror of the reference's discord-search interface over the C ABI.

Same names, argument meaning and error behaviour as the reference's
``tsdd::run_discovery`` / ``DiscoveryConfig`` / ``DiscordResult`` / ``RunOutcome``
(/root/reference/proj/include/tsdd/pipeline.hpp:15-37, discovery.hpp:16-32) and its
exception types (errors.hpp:10-25), bound with ctypes to ``libtsdd_cuda.so``
(include/tsdd_cuda.h).  The reference's own host language is C++; the C++ mirror of
the same interface is ``include/tsdd/*.hpp``.  This Python layer exists for the
tests and ``bench.py``.

There is no CPU path here: every call that computes anything goes to the sm_100a
kernels, and fails loudly when the library or a CUDA device is missing.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TSDD_CUDA_LIB selects another build of the same library (the tests point it at the checked
# build, _lib/libtsdd_cuda_dbg.so: -DTSDD_DEBUG_BOUNDS, in-kernel index checks)
LIB_PATH = os.environ.get("TSDD_CUDA_LIB") or os.path.join(_HERE, "_lib", "libtsdd_cuda.so")

OK, ERR_PARAMETER, ERR_VALIDATION, ERR_INFEASIBLE, ERR_RUNTIME = 0, 2, 3, 4, 5
SEARCH_DISABLE_PRUNING = 1

FETCH = dict(rows=1, mean=2, inv_sigma=3, paa=4, sax=5, hash=6, freq=7, buckets=8, order=9,
             candidates=10, nn_sq=11, nn_exact=12)


class ParameterError(ValueError):
    """Bad configuration or parameters (errors.hpp:10-13; CLI exit code 2)."""


class ValidationError(RuntimeError):
    """Bad input data: empty or non-finite series (errors.hpp:16-19; CLI exit code 3)."""


class InfeasibleInputError(ParameterError):
    """No subsequence has a non-self match (errors.hpp:22-25)."""


class CudaRuntimeError(RuntimeError):
    """CUDA / NCCL failure, or no usable device (there is no CPU fallback)."""


_ERRORS = {ERR_PARAMETER: ParameterError, ERR_VALIDATION: ValidationError,
           ERR_INFEASIBLE: InfeasibleInputError, ERR_RUNTIME: CudaRuntimeError}


class Stats(ctypes.Structure):
    """tsdd_cuda_stats (include/tsdd_cuda.h)."""
    _fields_ = [("rows", ctypes.c_uint64), ("calls", ctypes.c_uint64), ("abandoned", ctypes.c_uint64),
                ("terms", ctypes.c_uint64), ("buckets", ctypes.c_uint64),
                ("min_freq_candidates", ctypes.c_uint64), ("batches", ctypes.c_uint64),
                ("scanned_candidates", ctypes.c_uint64), ("kernel_launches", ctypes.c_uint64),
                ("prep_ms", ctypes.c_double), ("search_ms", ctypes.c_double),
                ("scan_kernel_ms", ctypes.c_double), ("h2d_ms", ctypes.c_double),
                ("scan_kernel_launches", ctypes.c_uint64), ("scan_kernel_terms", ctypes.c_uint64),
                ("encode_ms", ctypes.c_double), ("build_rows_ms", ctypes.c_double),
                ("index_ms", ctypes.c_double), ("tiles", ctypes.c_uint64),
                ("tile_live_candidates", ctypes.c_uint64), ("lb_skipped", ctypes.c_uint64),
                ("scan_kernel_ws_launches", ctypes.c_uint64),
                ("scan_kernel_dot_launches", ctypes.c_uint64),
                ("scan_kernel_dot_terms", ctypes.c_uint64), ("finalists", ctypes.c_uint64),
                ("exact_reruns", ctypes.c_uint64), ("useful_terms", ctypes.c_uint64),
                ("propagated", ctypes.c_uint64), ("scan_kernel_tc_launches", ctypes.c_uint64),
                ("scan_kernel_tc_terms", ctypes.c_uint64), ("scan_kernel_tc_ms", ctypes.c_double),
                ("tail_restarts", ctypes.c_uint64)]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64), ctypes.c_size_t)

# every symbol include/tsdd_cuda.h declares: (restype, argtypes)
_vp, _sz, _int, _dbl = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_double
SYMBOLS = {
    "tsdd_cuda_create": (_int, [ctypes.POINTER(_vp), _int]),
    "tsdd_cuda_destroy": (None, [_vp]),
    "tsdd_cuda_last_error": (ctypes.c_char_p, [_vp]),
    "tsdd_cuda_set_stream": (_int, [_vp, _vp]),
    "tsdd_cuda_set_option": (_int, [_vp, ctypes.c_char_p, _dbl]),
    "tsdd_cuda_check_config_f32": (_int, [_vp, _sz, _sz, _sz, _sz, ctypes.c_char_p, _sz]),
    "tsdd_cuda_check_config_f64": (_int, [_vp, _sz, _sz, _sz, _sz, ctypes.c_char_p, _sz]),
    "tsdd_cuda_prepare_f32": (_int, [_vp, _vp, _sz, _sz, _sz, _sz]),
    "tsdd_cuda_prepare_f64": (_int, [_vp, _vp, _sz, _sz, _sz, _sz]),
    "tsdd_cuda_prepare_device_f32": (_int, [_vp, _vp, _sz, _sz, _sz, _sz]),
    "tsdd_cuda_reindex": (_int, [_vp, _sz, _sz]),
    "tsdd_cuda_fetch_rows": (_int, [_vp, _sz, _sz, _vp]),
    "tsdd_cuda_search": (_int, [_vp, _int, ctypes.c_uint, _vp, _vp]),
    "tsdd_cuda_get_stats": (_int, [_vp, ctypes.POINTER(Stats)]),
    "tsdd_cuda_row_stride": (_sz, [_vp]),
    "tsdd_cuda_fetch": (_int, [_vp, _int, _vp, _sz]),
    "tsdd_cuda_comm_unique_id": (_int, [ctypes.c_char_p]),
    "tsdd_cuda_comm_init": (_int, [_vp, ctypes.c_char_p, _int, _int]),
    "tsdd_cuda_comm_size": (_int, [_vp, ctypes.POINTER(_int)]),
    "tsdd_cuda_group_create": (_int, [ctypes.POINTER(_vp), _int]),
    "tsdd_cuda_set_exchange": (_int, [_vp, EXCHANGE_FN, _vp, _int, _int]),
    "tsdd_cuda_fp32_probe": (_int, [_vp, _int, ctypes.POINTER(_dbl), ctypes.POINTER(_dbl)]),
    "tsdd_cuda_nn_profile": (_int, [_vp, _vp]),
}

_lib = None


def load_library() -> ctypes.CDLL:
    """Loads libtsdd_cuda.so and binds every declared symbol; raises when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise CudaRuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1901_00155_b200.build` "
                "(the engine has no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (restype, argtypes) in SYMBOLS.items():
            fn = getattr(lib, name)
            fn.restype = restype
            fn.argtypes = argtypes
        _lib = lib
    return _lib


def _raise(code: int, message: str):
    raise _ERRORS.get(code, CudaRuntimeError)(message)


def _as_series(series) -> np.ndarray:
    """float32 stays float32 (the workloads' native precision); everything else is float64
    (the reference's TimeSeries, series.hpp:15)."""
    a = np.asarray(series)
    if a.dtype != np.float32:
        a = a.astype(np.float64, copy=False)
    return np.ascontiguousarray(a.reshape(-1))


# ------------------------------------------------------------------ reference-shaped types
@dataclass
class DiscoveryConfig:
    """pipeline.hpp:15-24.  ``threads`` / ``chunk`` / ``vec_width`` keep the reference's
    validation (>= 1) and have no other effect on the device; ``k`` and ``device`` are new."""
    n: int = 0
    word_len: int = 4
    alphabet: int = 4
    vec_width: int = 8
    engine: str = "cuda"
    threads: int = 1
    chunk: int = 1
    disable_pruning: bool = False
    k: int = 1
    device: int = 0


@dataclass
class DiscordResult:
    """discovery.hpp:20-26: 1-based position, Euclidean distance (sqrt taken once)."""
    position: int = 0
    distance: float = 0.0
    calls: int = 0
    abandoned: int = 0
    engine: str = "cuda"


@dataclass
class RunOutcome:
    """pipeline.hpp:26-31, plus the top-k list and the device counters."""
    result: DiscordResult = field(default_factory=DiscordResult)
    m: int = 0
    prep_time_s: float = 0.0
    search_time_s: float = 0.0
    discords: list = field(default_factory=list)   # k DiscordResult, best first
    stats: dict = field(default_factory=dict)


def check_config(series, config: DiscoveryConfig) -> None:
    """check_config (pipeline.cpp:21-49): every parameter validated before any work, in the
    reference's order.  Pure host logic inside the library; needs no device."""
    lib = load_library()
    x = _as_series(series)
    msg = ctypes.create_string_buffer(512)
    for name in ("n", "word_len", "alphabet", "k"):
        if int(getattr(config, name)) < 0:
            raise ParameterError(f"{name} must not be negative")
    fn = lib.tsdd_cuda_check_config_f32 if x.dtype == np.float32 else lib.tsdd_cuda_check_config_f64
    rc = fn(x.ctypes.data, x.size, int(config.n), int(config.word_len), int(config.alphabet), msg, 512)
    text = msg.value.decode()
    # the reference's order: series, n, word_len, [vec_width, threads, chunk], alphabet,
    # dictionary, feasibility — the bracketed three exist only on the host side
    if rc == ERR_VALIDATION or (rc == ERR_PARAMETER and text.startswith(("n=", "word_len="))):
        _raise(rc, text)
    if config.vec_width < 1:
        raise ParameterError("vec_width must be >= 1")
    if config.threads < 1:
        raise ParameterError(f"threads must be >= 1, got {config.threads}")
    if config.chunk < 1:
        raise ParameterError(f"chunk must be >= 1, got {config.chunk}")
    if config.k < 1:
        raise ParameterError(f"k must be >= 1, got {config.k}")
    if rc != OK:
        _raise(rc, text)


class Context:
    """One engine instance bound to one GPU (tsdd_cuda_ctx).  One call at a time."""

    def __init__(self, device: int = 0):
        self._lib = load_library()
        self._h = ctypes.c_void_p()
        rc = self._lib.tsdd_cuda_create(ctypes.byref(self._h), int(device))
        if rc != OK:
            _raise(rc, self._lib.tsdd_cuda_last_error(None).decode())
        self.device = device
        self._keepalive = None
        self._shape = None

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            self._lib.tsdd_cuda_destroy(self._h)
            self._h = ctypes.c_void_p()

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def _check(self, rc: int):
        if rc != OK:
            _raise(rc, self._lib.tsdd_cuda_last_error(self._h).decode())

    def set_stream(self, cuda_stream: int | None):
        """Run on the caller's stream (``torch.cuda.current_stream().cuda_stream``); None = own."""
        self._check(self._lib.tsdd_cuda_set_stream(self._h, cuda_stream))

    def set_option(self, name: str, value: float):
        self._check(self._lib.tsdd_cuda_set_option(self._h, name.encode(), float(value)))

    def prepare(self, series, n: int, word_len: int, alphabet: int):
        x = _as_series(series)
        fn = self._lib.tsdd_cuda_prepare_f32 if x.dtype == np.float32 else self._lib.tsdd_cuda_prepare_f64
        self._check(fn(self._h, x.ctypes.data, x.size, n, word_len, alphabet))
        self._shape = (x.size, n, word_len, alphabet)

    def prepare_device(self, d_series_ptr: int, m: int, n: int, word_len: int, alphabet: int):
        """float32 series already in device memory (e.g. ``torch_tensor.data_ptr()``)."""
        self._check(self._lib.tsdd_cuda_prepare_device_f32(self._h, d_series_ptr, m, n, word_len, alphabet))
        self._shape = (m, n, word_len, alphabet)

    def reindex(self, word_len: int, alphabet: int):
        """Window encoding + DiscordIndexes::build again for another SAX shape; the matrix stays."""
        self._check(self._lib.tsdd_cuda_reindex(self._h, word_len, alphabet))
        m, n, _, _ = self._shape
        self._shape = (m, n, word_len, alphabet)

    def fetch_rows(self, first: int, count: int) -> np.ndarray:
        out = np.empty((count, self.row_stride()), dtype=np.float32)
        self._check(self._lib.tsdd_cuda_fetch_rows(self._h, first, count, out.ctypes.data))
        return out

    def search(self, k: int = 1, disable_pruning: bool = False):
        pos = np.zeros(max(k, 1), dtype=np.uint64)
        dist = np.zeros(max(k, 1), dtype=np.float64)
        flags = SEARCH_DISABLE_PRUNING if disable_pruning else 0
        self._check(self._lib.tsdd_cuda_search(self._h, k, flags, pos.ctypes.data, dist.ctypes.data))
        return [int(p) for p in pos], [float(d) for d in dist]

    def stats(self) -> dict:
        s = Stats()
        self._check(self._lib.tsdd_cuda_get_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def row_stride(self) -> int:
        return int(self._lib.tsdd_cuda_row_stride(self._h))

    def fetch(self, what: str) -> np.ndarray:
        m, n, w, _ = self._shape
        N = m - n + 1
        st = self.stats()
        shapes = {
            "rows": ((N, self.row_stride()), np.float32), "mean": ((N,), np.float64),
            "inv_sigma": ((N,), np.float64), "paa": ((N, w), np.float64), "sax": ((N, w), np.uint32),
            "hash": ((N,), np.uint64), "freq": ((N,), np.uint32), "buckets": ((N,), np.uint64),
            "order": ((N,), np.uint64), "candidates": ((st["min_freq_candidates"],), np.uint64),
            "nn_sq": ((N,), np.float32), "nn_exact": ((N,), np.uint8),
        }
        shape, dtype = shapes[what]
        out = np.empty(shape, dtype=dtype)
        self._check(self._lib.tsdd_cuda_fetch(self._h, FETCH[what], out.ctypes.data, out.nbytes))
        return out

    def nn_profile(self) -> np.ndarray:
        m, n, _, _ = self._shape
        out = np.empty(m - n + 1, dtype=np.float32)
        self._check(self._lib.tsdd_cuda_nn_profile(self._h, out.ctypes.data))
        return out

    def fp32_probe(self, which: int) -> tuple[float, float]:
        ops, ms = ctypes.c_double(), ctypes.c_double()
        self._check(self._lib.tsdd_cuda_fp32_probe(self._h, which, ctypes.byref(ops), ctypes.byref(ms)))
        return ops.value, ms.value

    # ---- several ranks
    def set_exchange(self, fn, world: int, rank: int):
        """``fn(keys: np.ndarray[uint64]) -> None`` must max-reduce ``keys`` in place over all ranks."""
        if fn is None:
            self._check(self._lib.tsdd_cuda_set_exchange(self._h, EXCHANGE_FN(), None, world, rank))
            self._keepalive = None
            return

        def trampoline(_user, keys, count):
            try:
                view = np.ctypeslib.as_array(keys, shape=(count,))
                fn(view)
                return 0
            except Exception:  # noqa: BLE001 - must not unwind through C
                import traceback
                traceback.print_exc()
                return 1

        cb = EXCHANGE_FN(trampoline)
        self._check(self._lib.tsdd_cuda_set_exchange(self._h, cb, None, world, rank))
        self._keepalive = cb

    def comm_init(self, unique_id: bytes, world: int, rank: int):
        self._check(self._lib.tsdd_cuda_comm_init(self._h, unique_id, world, rank))

    def comm_size(self) -> int:
        n = ctypes.c_int()
        self._check(self._lib.tsdd_cuda_comm_size(self._h, ctypes.byref(n)))
        return n.value


def group_create(contexts) -> None:
    """Links contexts of this process into ranks 0 .. len-1 that exchange over device memory
    (tsdd_cuda_group_create); each must then be driven by its own host thread."""
    handles = (ctypes.c_void_p * len(contexts))(*[c._h.value for c in contexts])
    rc = load_library().tsdd_cuda_group_create(handles, len(contexts))
    if rc != OK:
        _raise(rc, load_library().tsdd_cuda_last_error(contexts[0]._h).decode())


def comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = load_library().tsdd_cuda_comm_unique_id(buf)
    if rc != OK:
        _raise(rc, load_library().tsdd_cuda_last_error(None).decode())
    return buf.raw


def run_discovery(series, config: DiscoveryConfig, context: Context | None = None) -> RunOutcome:
    """tsdd::run_discovery (pipeline.cpp:53-93) on the GPU: validate everything, timed
    preparation, timed search.  ``series`` is host memory (the reference-facing call)."""
    if config.engine != "cuda":
        raise ParameterError(f"unknown engine '{config.engine}' (this library implements 'cuda')")
    check_config(series, config)
    ctx = context or Context(config.device)
    try:
        x = _as_series(series)
        ctx.prepare(x, config.n, config.word_len, config.alphabet)
        positions, distances = ctx.search(config.k, config.disable_pruning)
        st = ctx.stats()
    finally:
        if context is None:
            ctx.close()
    discords = [DiscordResult(p, d, st["calls"], st["abandoned"], "cuda") for p, d in zip(positions, distances)]
    return RunOutcome(result=discords[0], m=int(x.size), prep_time_s=(st["prep_ms"] + st["h2d_ms"]) * 1e-3,
                      search_time_s=st["search_ms"] * 1e-3, discords=discords, stats=st)
