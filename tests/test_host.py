"""Host-side checks that need no GPU: the C ABI loads and exports what include/tsdd_cuda.h
declares, check_config behaves like the reference's, the product never imports the
oracle, the seeded workloads are the pinned ones, and the multi-rank exchange works
over gloo with two processes."""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

import oracle
import paper_1901_00155_b200 as pkg
from paper_1901_00155_b200 import engine, parallel, workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


# ------------------------------------------------------------------ the boundary
def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "tsdd_cuda.h")).read()
    header = re.sub(r"/\*.*?\*/", "", header, flags=re.S)
    declared = set(re.findall(r"\b(tsdd_cuda_\w+)\s*\(", header))
    assert len(declared) >= 18
    assert declared == set(engine.SYMBOLS), declared ^ set(engine.SYMBOLS)
    lib = pkg.load_library()
    for name in declared:
        assert getattr(lib, name) is not None
    out = subprocess.run(["nm", "-D", "--defined-only", engine.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (tsdd_cuda_\w+)", out))
    assert declared <= exported


def test_library_has_sm100a_code_and_blackwell_instructions():
    sass = subprocess.run(["cuobjdump", "-sass", engine.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in sass
    assert "FFMA2" in sass and "FADD2" in sass  # packed f32x2 arithmetic (sm_100+)
    assert "LDGSTS" in sass                      # cp.async staging of the tiles (k_scan_tiles)
    # the warp-specialised tile kernel: bulk async copies onto mbarriers, register rebalancing
    assert "UBLKCP" in sass and "SYNCS" in sass and "USETMAXREG" in sass
    assert "UTMALDG" in sass                     # ... and its tiles as tensor-map (TMA) boxes


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device failure mode")
def test_create_fails_loudly_without_a_device():
    with pytest.raises(pkg.CudaRuntimeError, match="no CPU fallback"):
        pkg.Context(0)
    with pytest.raises(pkg.CudaRuntimeError):
        pkg.run_discovery(W.random_walk(1, 500), pkg.DiscoveryConfig(n=16))


def test_product_never_touches_the_oracle():
    pkg_dir = os.path.join(ROOT, "paper_1901_00155_b200")
    for base, _, files in os.walk(pkg_dir):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".hpp", ".cpp", ".h")):
                text = open(os.path.join(base, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", text, flags=re.M), f
                assert "tsdd_oracle" not in text and "libtsdd_ref" not in text, f


# ------------------------------------------------------------------ check_config vs the reference
BAD = [
    ("empty", lambda: np.zeros(0), dict(n=4), oracle.ERR_VALIDATION),
    ("nan", lambda: np.array([1.0, np.nan] + [0.0] * 62), dict(n=8), oracle.ERR_VALIDATION),
    ("inf", lambda: np.array([np.inf] + [0.0] * 63), dict(n=8), oracle.ERR_VALIDATION),
    ("n_zero", lambda: np.arange(64.0), dict(n=0), oracle.ERR_PARAMETER),
    ("n_gt_m", lambda: np.arange(64.0), dict(n=65), oracle.ERR_PARAMETER),
    ("w_zero", lambda: np.arange(64.0), dict(n=8, word_len=0), oracle.ERR_PARAMETER),
    ("w_gt_n", lambda: np.arange(64.0), dict(n=8, word_len=9), oracle.ERR_PARAMETER),
    ("alphabet_1", lambda: np.arange(64.0), dict(n=8, alphabet=1), oracle.ERR_PARAMETER),
    ("alphabet_11", lambda: np.arange(64.0), dict(n=8, alphabet=11), oracle.ERR_PARAMETER),
    ("infeasible", lambda: np.arange(20.0), dict(n=16, word_len=2), oracle.ERR_INFEASIBLE),
    ("n_eq_m", lambda: np.arange(20.0), dict(n=20, word_len=2), oracle.ERR_INFEASIBLE),
    ("threads_0", lambda: np.arange(64.0), dict(n=8, threads=0), oracle.ERR_PARAMETER),
    ("chunk_0", lambda: np.arange(64.0), dict(n=8, chunk=0), oracle.ERR_PARAMETER),
]
_CLASS = {oracle.ERR_VALIDATION: pkg.ValidationError, oracle.ERR_PARAMETER: pkg.ParameterError,
          oracle.ERR_INFEASIBLE: pkg.InfeasibleInputError}


@pytest.mark.parametrize("name,make,kw,code", BAD, ids=[b[0] for b in BAD])
def test_check_config_matches_reference_errors(name, make, kw, code):
    x = make()
    cfg = pkg.DiscoveryConfig(**kw)
    with pytest.raises(_CLASS[code]) as mine:
        pkg.check_config(x, cfg)
    if code == oracle.ERR_INFEASIBLE:
        assert isinstance(mine.value, pkg.ParameterError)  # errors.hpp:22: Infeasible is-a Parameter
    if name in ("threads_0", "chunk_0", "empty"):
        return  # the oracle shims take these through other paths
    with pytest.raises(oracle.OracleError) as ref:
        oracle.best().run_discovery(x, kw["n"], kw.get("word_len", 4), kw.get("alphabet", 4), threads=1)
    assert ref.value.code == code
    assert str(mine.value) == ref.value.message  # same text as the reference's exception


def test_check_config_error_order_is_the_references():
    # series is validated before any parameter (pipeline.cpp:22), n before word_len, feasibility last
    bad = np.arange(20.0)
    bad[3] = np.nan
    with pytest.raises(pkg.ValidationError, match="index 4"):
        pkg.check_config(bad, pkg.DiscoveryConfig(n=0, word_len=0, alphabet=99))
    with pytest.raises(pkg.ParameterError, match="^n="):
        pkg.check_config(np.arange(20.0), pkg.DiscoveryConfig(n=0, word_len=0, alphabet=99))
    with pytest.raises(pkg.ParameterError, match="alphabet"):
        pkg.check_config(np.arange(20.0), pkg.DiscoveryConfig(n=16, word_len=2, alphabet=99))
    pkg.check_config(np.arange(64.0), pkg.DiscoveryConfig(n=8, word_len=8, alphabet=10))


def test_dictionary_guard_is_2_pow_32():
    x = W.random_walk(1, 4096)
    pkg.check_config(x, pkg.DiscoveryConfig(n=64, word_len=16, alphabet=4))   # 4^16 = 2^32: accepted
    with pytest.raises(pkg.ParameterError, match="2\\^32"):
        pkg.check_config(x, pkg.DiscoveryConfig(n=64, word_len=17, alphabet=4))
    with pytest.raises(pkg.ParameterError):
        pkg.check_config(x, pkg.DiscoveryConfig(n=64, word_len=10, alphabet=10))  # 10^10 > 2^32
    with pytest.raises(pkg.ParameterError, match="engine"):
        pkg.run_discovery(x, pkg.DiscoveryConfig(n=64, engine="phidd"))


# ------------------------------------------------------------------ workloads
def test_workloads_are_the_pinned_series(golden):
    for key, rec in golden.items():
        w = W.workload(rec["cfg"])
        assert (w.m, w.n, w.word_len, w.alphabet, w.k) == (rec["m"], rec["n"], rec["word_len"],
                                                          rec["alphabet"], rec["k"])
        if w.m <= 1_000_000:
            x, at = W.series(rec["cfg"])
            assert W.sha256(x) == rec["sha256"] and at == rec["anomaly_starts_0based"]


def test_workload_table_matches_baseline_json():
    shapes = {1: (65536, 128, 4, 4, 1), 2: (262144, 256, 8, 4, 4), 3: (1000000, 512, 8, 6, 3),
              4: (4000000, 1024, 16, 4, 5), 5: (1000000, 256, 8, 4, 1)}
    for cfg, want in shapes.items():
        w = W.workload(cfg)
        assert (w.m, w.n, w.word_len, w.alphabet, w.k) == want


# ------------------------------------------------------------------ packed keys / sharding
def test_packed_key_order_is_the_reference_merge_rule():
    # greater distance wins; equal distance -> smaller position (discovery.cpp:158-165, 328-340)
    assert parallel.pack_best(2.0, 10) > parallel.pack_best(1.5, 3)
    assert parallel.pack_best(2.0, 3) > parallel.pack_best(2.0, 10)
    assert parallel.unpack_best(parallel.pack_best(7.25, 1234)) == (7.25, 1234)
    rng = np.random.default_rng(0)
    d = rng.random(1000).astype(np.float32) * 100
    rows = rng.integers(0, 4_000_000, 1000)
    keys = [parallel.pack_best(float(a), int(b)) for a, b in zip(d, rows)]
    best = max(range(1000), key=lambda i: (d[i], -rows[i]))
    assert keys.index(max(keys)) == best
    assert all(k < 2 ** 63 for k in keys)
    assert sorted(parallel.owner_of(e, 4) for e in range(8)) == [0, 0, 1, 1, 2, 2, 3, 3]


_GLOO_WORKER = r"""
import os, sys
sys.path.insert(0, {root!r})
import numpy as np
import torch.distributed as dist
from paper_1901_00155_b200 import parallel

dist.init_process_group("gloo", init_method="tcp://127.0.0.1:{port}", rank=int(sys.argv[1]), world_size=2)
rank = dist.get_rank()
ex = parallel.TorchExchange()

# a toy version of the engine's outer loop: each rank owns every other entry of a shared
# order, raises its local best batch by batch, and exchanges (best, more-work) after each
rng = np.random.default_rng(5)
nn = (rng.random(1000) * 50).astype(np.float32)          # same on both ranks
order = rng.permutation(1000)
mine = [int(r) for e, r in enumerate(order) if parallel.owner_of(e, 2) == rank]
if rank == 1:
    mine = mine[:200]                                       # uneven work: rank 1 runs dry first
best, cursor, rounds = 0, 0, 0
while True:
    batch = mine[cursor:cursor + 64]
    cursor += len(batch)
    for r in batch:
        best = max(best, parallel.pack_best(float(nn[r]), r))
    keys = np.array([best, 1 if cursor < len(mine) else 0], dtype=np.uint64)
    ex(keys)
    best, more = int(keys[0]), int(keys[1])
    rounds += 1
    if not more:
        break
seen = [int(r) for e, r in enumerate(order) if e % 2 == 0 or (e % 2 == 1 and e < 400)]
want = max(parallel.pack_best(float(nn[r]), r) for r in seen)
assert best == want, (best, want)
assert rounds == ex.calls == 8, rounds                      # ceil(500/64): both ranks leave together
d2, row = parallel.unpack_best(best)
print("rank", rank, "ok", d2, row, rounds, flush=True)
dist.destroy_process_group()
"""


def test_exchange_over_gloo_with_two_ranks(tmp_path):
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = tmp_path / "worker.py"
    script.write_text(_GLOO_WORKER.format(root=ROOT, port=port))
    procs = [subprocess.Popen([sys.executable, str(script), str(r)], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = [p.communicate(timeout=180)[0] for p in procs]
    for r, (p, out) in enumerate(zip(procs, outs)):
        assert p.returncode == 0, out
        assert f"rank {r} ok" in out
    assert outs[0].split("ok")[1].split()[:2] == outs[1].split("ok")[1].split()[:2]


# ------------------------------------------------------------------ C++ host layer and CLI (tools/tsdd_cuda.cpp)
CLI = os.path.join(ROOT, "paper_1901_00155_b200", "_lib", "tsdd_cuda")


def _cli(*args):
    return subprocess.run([CLI, *[str(a) for a in args]], capture_output=True, text=True)


@pytest.mark.parametrize("args,code,text", [
    (["--n", "16", "--word-len", "2"], 2, "no subsequence has a non-self match: N=5 <= n=16 (need m >= 2n)"),
    (["--n", "0", "--word-len", "2"], 2, "n=0 must satisfy 1 <= n <= m=20"),
    (["--n", "4", "--word-len", "9"], 2, "word_len=9 must satisfy 1 <= word_len <= n=4"),
    (["--n", "4", "--word-len", "2", "--alphabet", "11"], 2, "alphabet"),
    (["--n", "4", "--threads", "0"], 2, "threads must be >= 1, got 0"),
    (["--n", "4", "--engine", "phidd"], 2, "unknown engine"),
    (["--n", "4", "--bogus", "1"], 2, "unknown option '--bogus'"),
    (["--word-len", "2"], 2, "--n is required"),
])
def test_cli_maps_errors_to_reference_exit_codes(tmp_path, args, code, text):  # tools/tsdd.cpp:212-223
    path = tmp_path / "a.f64le"
    np.arange(20.0).tofile(path)
    p = _cli("find", "--input", path, "--format", "f64le", *args)
    assert p.returncode == code and text in p.stderr, p.stderr


def test_cli_series_readers_follow_the_reference(tmp_path):  # src/io.cpp:23-91
    csv = tmp_path / "s.csv"
    csv.write_text("value\n 1.5\n\n2.5\t\r\n3\n")
    p = _cli("find", "--input", csv, "--n", "2", "--word-len", "2")  # header and blanks skipped; m = 3 < 2n
    assert p.returncode == 2 and "N=2 <= n=2" in p.stderr and "series: 3 values, min 1.5, max 3" in p.stderr
    csv.write_text("1\n2\nabc\n")
    p = _cli("find", "--input", csv, "--n", "1")
    assert p.returncode == 3 and f"cannot parse 'abc' at {csv}:3" in p.stderr
    csv.write_text("1\ninf\n")
    p = _cli("find", "--input", csv, "--n", "1")
    assert p.returncode == 3 and f"non-finite value at {csv}:2" in p.stderr
    csv.write_text("header only\n")
    p = _cli("find", "--input", csv, "--n", "1")
    assert p.returncode == 3 and "no values found" in p.stderr
    raw = tmp_path / "s.f64le"
    raw.write_bytes(b"\0" * 20)
    p = _cli("find", "--input", raw, "--format", "f64le", "--n", "1")
    assert p.returncode == 3 and "is not a multiple of 8 (truncated at byte offset 16)" in p.stderr
    x = np.arange(20.0)
    x[6] = np.inf
    x.tofile(raw)
    p = _cli("find", "--input", raw, "--format", "f64le", "--n", "4")
    assert p.returncode == 3 and "non-finite value at index 7" in p.stderr
    p = _cli("find", "--input", tmp_path / "nope", "--n", "4")
    assert p.returncode == 3 and "cannot open" in p.stderr
    p = _cli("find", "--input", raw, "--format", "parquet", "--n", "4")
    assert p.returncode == 2 and "unknown series format 'parquet'" in p.stderr
    p = _cli("bench", "--input", raw, "--format", "f64le", "--n", "4", "--gpus", "2,4")
    assert p.returncode == 2 and "must include 1" in p.stderr


def test_cli_generate_writes_the_pinned_workloads(tmp_path, golden):
    out = tmp_path / "cfg1.f32le"
    p = _cli("generate", "--workload", 1, "--output", out)
    assert p.returncode == 0, p.stderr
    x = np.fromfile(out, dtype=np.float32)
    assert W.sha256(x) == golden["cfg1"]["sha256"]
    out64 = tmp_path / "cfg1.f64le"
    assert _cli("generate", "--workload", 1, "--output", out64, "--format", "f64le").returncode == 0
    np.testing.assert_array_equal(np.fromfile(out64, dtype=np.float64), x.astype(np.float64))
    assert _cli("generate", "--workload", 9, "--output", out).returncode == 2


@pytest.mark.parametrize("flags,kw", [
    (["--m", 500, "--seed", 7], dict(m=500, seed=7)),
    (["--m", 2000, "--anomaly", "spike", "--anomaly-pos", 1200, "--seed", 3],
     dict(m=2000, anomaly="spike", anomaly_pos=1200, seed=3)),
    (["--m", 3000, "--anomaly", "shape", "--anomaly-pos", 901, "--anomaly-len", 100],
     dict(m=3000, anomaly="shape", anomaly_pos=901, anomaly_len=100)),
    (["--m", 64, "--anomaly", "shape", "--anomaly-pos", 1, "--anomaly-len", 64, "--seed", 11],
     dict(m=64, anomaly="shape", anomaly_pos=1, anomaly_len=64, seed=11)),
])
def test_cli_generate_with_the_reference_flags(tmp_path, flags, kw):  # tools/tsdd.cpp:140-153, src/generate.cpp:19-59
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    want = oracle.ref().generate_series(**kw)
    raw = tmp_path / "g.f64le"
    p = _cli("generate", *flags, "--output", raw, "--format", "f64le")
    assert p.returncode == 0, p.stderr
    assert f"series: {kw['m']} values" in p.stderr  # print_series_summary, like the reference's tool
    got = np.fromfile(raw, dtype=np.float64)
    np.testing.assert_array_equal(got, want)  # bit-identical to the reference's generator
    csv = tmp_path / "g.csv"
    assert _cli("generate", *flags, "--output", csv).returncode == 0  # default format: csv, "%.17g" per line
    np.testing.assert_array_equal(np.loadtxt(csv, dtype=np.float64, ndmin=1), want)


@pytest.mark.parametrize("flags,kw", [
    (["--m", 0], dict(m=0)),
    (["--m", 100, "--anomaly", "spike"], dict(m=100, anomaly="spike")),
    (["--m", 100, "--anomaly", "spike", "--anomaly-pos", 101], dict(m=100, anomaly="spike", anomaly_pos=101)),
    (["--m", 100, "--anomaly", "shape", "--anomaly-pos", 50, "--anomaly-len", 52],
     dict(m=100, anomaly="shape", anomaly_pos=50, anomaly_len=52)),
    (["--m", 100, "--anomaly", "shape", "--anomaly-pos", 50, "--anomaly-len", 1],
     dict(m=100, anomaly="shape", anomaly_pos=50, anomaly_len=1)),
    (["--m", 100, "--anomaly", "wave"], dict(m=100, anomaly="wave")),
])
def test_cli_generate_rejects_what_the_reference_rejects(tmp_path, flags, kw):
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    with pytest.raises(oracle.OracleError) as ref:
        oracle.ref().generate_series(**kw)
    p = _cli("generate", *flags, "--output", tmp_path / "x.csv")
    assert ref.value.code == 2 and p.returncode == 2
    assert ref.value.message in p.stderr, (ref.value.message, p.stderr)


def test_breakpoint_generator_reproduces_the_device_table():
    """tools/gen_sax_breakpoints.py (scipy norm.ppf, lower half mirrored) prints exactly the
    c_breaks table of csrc/prep_kernels.cu — the values of the reference's sax.cpp:14-46."""
    import re

    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_sax_breakpoints.py")], capture_output=True,
                       text=True)
    assert p.returncode == 0, p.stderr
    src = open(os.path.join(ROOT, "paper_1901_00155_b200", "csrc", "prep_kernels.cu")).read()
    table = src[src.index("c_breaks[9][9] = {"):]
    table = table[:table.index("};")]
    number = r"-?\d+(?:\.\d+)?(?:e-?\d+)?"
    have = [float(v) for v in re.findall(number, table[table.index("{", 20):])]
    want = [float(v) for v in re.findall(number, p.stdout[p.stdout.index("{"):])]
    assert have == want and len(want) == sum(range(1, 10))
    chk = oracle.best()
    for a in range(2, 11):  # and symbol_for agrees with the table on both sides of every breakpoint
        row = want[sum(range(1, a - 1)):sum(range(1, a))]
        for j, beta in enumerate(row):
            assert chk.symbol_for(a, beta) == j + 2 and chk.symbol_for(a, np.nextafter(beta, -np.inf)) == j + 1


# ------------------------------------------------------------------ bench.py contract (reference arm runs on CPU)
def test_bench_reference_arm_prints_the_contract_line():
    import json

    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "1",
                        "--gpus", "1", "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["metric"] == "subsequence_pair_distances_per_s"
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["cpu_baseline"]["cores"] >= 1
    assert line["config"]["workload"] == "cfg1" and line["vs_baseline"] is None


def test_bench_starts_its_own_ranks_and_refuses_without_the_devices():
    """`python bench.py --gpus N` with no launcher starts N ranks itself (spawn_ranks); on a
    machine with fewer CUDA devices it says so instead of running one rank and printing n_gpus 1."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "64", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert p.returncode != 0 and "--gpus 64 needs 64 CUDA devices" in p.stderr, p.stderr
    assert p.stdout.strip() == ""


def test_bench_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "1",
                        "--gpus", "2", "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env,
                       timeout=120)
    assert p.returncode == 0 and p.stdout.strip() == ""


# ------------------------------------------------------------------ the patched reference
TSDD_PATCHED = os.path.join(ROOT, "oracle", "_ref", "tsdd_patched")
REFERENCE = "/root/reference/proj"


def test_patched_reference_builds_against_the_engine_header(tmp_path):
    """tools/patch_reference.py applies INTEGRATION.md's four edits to a COPY of the reference;
    the copy compiles with TSDD_CUDA_WITH_REFERENCE_HEADERS (the reference's own types under
    include/tsdd/cuda_engine.hpp) and links against libtsdd_cuda.so.  Without a GPU the CPU
    engines of that binary still answer like the oracle, and `cuda` fails loudly."""
    if not os.path.isdir(REFERENCE):
        pytest.skip("the reference tree is not on this machine; oracle/_ref/tsdd_patched travels prebuilt")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "patch_reference.py"), REFERENCE,
                        str(tmp_path / "proj")], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    patched = open(tmp_path / "proj" / "src" / "pipeline.cpp").read()
    assert "TSDD_CUDA_WITH_REFERENCE_HEADERS" in patched and "tsdd::cuda::run_discovery(series, config)" in patched
    assert "cuda" in open(tmp_path / "proj" / "include" / "tsdd" / "discovery.hpp").read()
    assert "cuda" not in open(os.path.join(REFERENCE, "include", "tsdd", "discovery.hpp")).read()  # untouched
    p = subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "_ref/tsdd_patched"], capture_output=True, text=True)
    assert p.returncode == 0, p.stdout + p.stderr
    x = W.random_walk(3, 3000).astype(np.float64)
    x[1500:1564] += 3.0 * np.sin(np.arange(64))
    path = tmp_path / "s.f64le"
    x.tofile(path)
    p = subprocess.run([TSDD_PATCHED, str(path), "phidd", "64", "4", "4", "2"], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    import json
    got = json.loads(p.stdout)
    want = oracle.best().run_discovery(x, 64, 4, 4, threads=2)
    assert got["engine"] == "phidd" and got["pos"] == want["position"] and got["dist"] == want["distance"]
    import torch
    if not torch.cuda.is_available():
        p = subprocess.run([TSDD_PATCHED, str(path), "cuda", "64", "4", "4"], capture_output=True, text=True)
        assert p.returncode == 1 and "no CUDA device" in p.stderr, p.stderr  # no CPU fallback behind `cuda`


def test_checked_build_carries_the_bounds_checks():
    """The -DTSDD_DEBUG_BOUNDS build holds the in-kernel checks (their report string is in the
    binary), the release build compiles them out; both export the same C ABI."""
    lib = os.path.join(ROOT, "paper_1901_00155_b200", "_lib")
    marker = b"TSDD_DEBUG_BOUNDS: "
    assert marker in open(os.path.join(lib, "libtsdd_cuda_dbg.so"), "rb").read()
    assert marker not in open(os.path.join(lib, "libtsdd_cuda.so"), "rb").read()
    import ctypes
    dbg = ctypes.CDLL(os.path.join(lib, "libtsdd_cuda_dbg.so"))
    for name in pkg.engine.SYMBOLS:
        assert hasattr(dbg, name), name
