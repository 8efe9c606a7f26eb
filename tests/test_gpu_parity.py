"""Parity of the CUDA path against the CPU oracle, through the C ABI (libtsdd_cuda.so).

Bars (BASELINE.json north_star): discord positions identical, distances within 1e-4
relative (float32 kernels vs. the float64 reference); every integer array of the
preparation stage (symbols, hashes, frequencies, candidate set, buckets) identical.
The oracle is the unmodified reference when oracle/_ref is present, else the pinned C
restatement (tests/test_oracle_pin.py).
"""
import json
import os
import threading

import numpy as np
import pytest

import oracle
from paper_1901_00155_b200 import (Context, DiscoveryConfig, InfeasibleInputError, run_discovery,
                                   workloads as W)

pytestmark = pytest.mark.gpu
_ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

DIST_RTOL = 1e-4  # north_star: "discord distances must agree to 1e-4 relative"


@pytest.fixture(scope="module")
def ctx():
    c = Context(0)
    yield c
    c.close()


@pytest.fixture(scope="module")
def chk():
    return oracle.best()


def topk_from_profile(profile_sq, n, k):
    """Top-k discords from a float64 nn profile under the brute-force tie rule (greatest distance,
    then smallest position, discovery.cpp:158-165) and the exclusion zone of SURVEY.md 8c."""
    allowed = np.isfinite(profile_sq)
    pos, dist = [], []
    for _ in range(k):
        if not allowed.any() or profile_sq[allowed].max() <= 0.0:
            pos.append(1), dist.append(0.0)
            continue
        top = profile_sq[allowed].max()
        at = int(np.flatnonzero(allowed & (profile_sq == top))[0])
        pos.append(at + 1), dist.append(float(np.sqrt(top)))
        allowed[max(0, at - n + 1):at + n] = False
    return pos, dist


def assert_discords_match(chk, x, n, pos, dist, want):
    """Positions identical, distances within DIST_RTOL.  The one legitimate difference is an
    EXACT tie on the nn distance (e.g. two mutual nearest neighbours, or many rows whose
    nearest neighbour is the same all-zero row): the reference's own choice then depends on
    its candidate order or on float64 rounding noise (SURVEY.md gap G5), this engine takes
    the smallest position.  After such a tie the exclusion zones differ from the reference
    wrapper's, so the REST of the list is checked against the top-k that the reference's
    brute-force nn profile gives under this engine's documented tie rule."""
    for r, (p, d, wp, wd) in enumerate(zip(pos, dist, want["positions"], want["distances"])):
        if p != wp:
            profile_sq = chk.nn_profile(x, n)
            profile = np.sqrt(profile_sq)
            a, b = profile[p - 1], profile[wp - 1]
            assert a == pytest.approx(b, rel=1e-9, abs=1e-9), (r, p, wp, a, b)
            own_pos, own_dist = topk_from_profile(profile_sq, n, len(pos))
            for q in range(r, len(pos)):
                if pos[q] != own_pos[q]:  # only another exact tie (down to rounding noise) may differ
                    assert profile[pos[q] - 1] == pytest.approx(profile[own_pos[q] - 1], rel=1e-9, abs=1e-9), \
                        (q, pos, own_pos)
                    break
                assert dist[q] == pytest.approx(own_dist[q], rel=DIST_RTOL, abs=1e-6), (q, pos, dist, own_dist)
            return
        assert d == pytest.approx(wd, rel=DIST_RTOL, abs=1e-6), (r, p, d, wd)


def planted_walk(seed, m, n):
    x = W.random_walk(seed, m)
    at = m // 3
    x[at:at + n] += np.float32(2.5) * np.sin(np.arange(n, dtype=np.float32) * 0.7)
    return x


# ------------------------------------------------------------------ preparation stage
@pytest.mark.parametrize("m,n,w,a", [(3000, 64, 4, 4), (2500, 50, 3, 5), (4000, 128, 8, 6),
                                     (1500, 33, 7, 10), (5000, 96, 16, 2), (700, 8, 8, 2)])
def test_preparation_arrays_match_the_reference(ctx, chk, m, n, w, a):
    x = W.random_walk(100 + n, m)
    ctx.prepare(x, n, w, a)
    ref = chk.prepare(x, n, w, a)
    N = m - n + 1
    rows = ctx.fetch("rows")
    assert rows.shape == (N, ctx.row_stride()) and ctx.row_stride() % 32 == 0
    # float32 rounding of the float64 rows; padding columns are exactly zero (series.cpp:64-72)
    np.testing.assert_allclose(rows[:, :n], ref["rows"], rtol=0, atol=2e-6)
    assert not rows[:, n:].any()
    np.testing.assert_allclose(ctx.fetch("paa"), ref["paa"], rtol=0, atol=1e-9)
    sax = ctx.fetch("sax")
    flips = sax != ref["sax"]
    assert not flips.any(), f"{flips.sum()} SAX symbols differ"
    np.testing.assert_array_equal(ctx.fetch("hash"), ref["hashes"])
    np.testing.assert_array_equal(ctx.fetch("freq"), ref["freq"])
    np.testing.assert_array_equal(ctx.fetch("candidates"), ref["candidates"])
    np.testing.assert_array_equal(ctx.fetch("buckets"), ref["bucket_positions"])
    # rarity order: a permutation, ascending frequency, ties by position (SURVEY gap G4)
    order = ctx.fetch("order").astype(np.int64) - 1
    assert sorted(order) == list(range(N))
    f = ref["freq"][order].astype(np.int64)
    assert np.all(np.diff(f) >= 0)
    assert np.all(np.diff(order)[np.diff(f) == 0] > 0)
    st = ctx.stats()
    assert st["rows"] == N and st["buckets"] == len(np.unique(ref["hashes"]))
    assert st["min_freq_candidates"] == len(ref["candidates"])


@pytest.mark.parametrize("scale", [1.0, 1e9, 0.0], ids=["tolerance", "everything-close", "exact-only"])
@pytest.mark.parametrize("kind", ["walk", "offset", "steps"])
def test_aligned_encode_keeps_every_symbol(ctx, chk, kind, scale):
    """k_window_encode4<aligned> takes a segment's sum from prefix sums and encodes a window the reference's
    way only where a segment lies within its tolerance of a breakpoint: hashes and frequencies must stay
    those of the reference with the tolerance as it is, inflated (every window takes the exact path) and
    with the form switched off — on a walk, under an offset 1e4 times the spread, on quantised steps."""
    rng = np.random.default_rng(77)
    m, n, w, a = 6000, 128, 8, 6
    if kind == "walk":
        x = np.cumsum(rng.standard_normal(m)).astype(np.float32)
    elif kind == "offset":
        x = (1e4 + rng.standard_normal(m)).astype(np.float32)
    else:
        x = np.round(np.cumsum(rng.standard_normal(m)) / 4).astype(np.float32)  # many exactly equal segment means
    ctx.set_option("encode_tol_scale", scale)
    try:
        ctx.prepare(x, n, w, a)
        got_hash, got_freq = ctx.fetch("hash"), ctx.fetch("freq")
    finally:
        ctx.set_option("encode_tol_scale", 1.0)
    ref = chk.prepare(x, n, w, a)
    np.testing.assert_array_equal(got_hash, ref["hashes"])
    np.testing.assert_array_equal(got_freq, ref["freq"])


def test_flat_windows_become_zero_rows(ctx, chk):
    x = W.random_walk(5, 2000)
    x[500:700] = np.float32(1.25)  # constant stretch: sigma < 1e-12 -> all-zero rows (series.cpp:30-33)
    ctx.prepare(x, 64, 4, 4)
    ref = chk.prepare(x, 64, 4, 4)
    rows = ctx.fetch("rows")[:, :64]
    zero_ref = ~ref["rows"].any(axis=1)
    assert zero_ref.sum() >= 100
    np.testing.assert_array_equal(~rows.any(axis=1), zero_ref)
    np.testing.assert_array_equal(ctx.fetch("hash"), ref["hashes"])


def test_float64_series_is_accepted(ctx, chk):
    x = W.random_walk(21, 3000).astype(np.float64) * 1.000000123  # not float32-representable
    ctx.prepare(x, 64, 4, 4)
    ref = chk.prepare(x, 64, 4, 4)
    np.testing.assert_array_equal(ctx.fetch("hash"), ref["hashes"])
    pos, dist = ctx.search(1)
    want = chk.run_discovery(x, 64, 4, 4, engine="brute")
    assert pos[0] == want["position"] and dist[0] == pytest.approx(want["distance"], rel=DIST_RTOL)


# ------------------------------------------------------------------ search stage
@pytest.mark.parametrize("n", [32, 64, 128])
@pytest.mark.parametrize("seed", range(8))
def test_top1_matches_brute_force_oracle(ctx, chk, seed, n):  # SPEC.md:449-451 sweep family
    x = W.random_walk(1000 + seed, 2000)
    ctx.prepare(x, n, 4, 4)
    pos, dist = ctx.search(1)
    want = chk.run_discovery(x, n, 4, 4, engine="brute")
    assert pos[0] == want["position"]
    assert dist[0] == pytest.approx(want["distance"], rel=DIST_RTOL)
    st = ctx.stats()
    assert st["scan_kernel_launches"] > 0 and st["terms"] > 0 and st["calls"] >= st["abandoned"]


@pytest.mark.parametrize("n,w,a", [(50, 3, 5), (100, 7, 3), (200, 10, 4)])
def test_ragged_shapes(ctx, chk, n, w, a):  # n not a multiple of 32, w does not divide n
    x = planted_walk(77 + n, 6000, n)
    ctx.prepare(x, n, w, a)
    pos, dist = ctx.search(1)
    want = chk.run_discovery(x, n, w, a, engine="phidd")
    assert pos[0] == want["position"]
    assert dist[0] == pytest.approx(want["distance"], rel=DIST_RTOL)


def test_disable_pruning_does_not_change_the_result(ctx, chk):
    x = planted_walk(3, 5000, 64)
    ctx.prepare(x, 64, 4, 4)
    pruned = ctx.search(3)
    calls_pruned = ctx.stats()["calls"]
    full = ctx.search(3, disable_pruning=True)
    st = ctx.stats()
    assert pruned[0] == full[0]
    np.testing.assert_allclose(pruned[1], full[1], rtol=1e-6)
    # without pruning every ordered non-self pair is started exactly once
    N, n = 5000 - 64 + 1, 64
    assert st["calls"] == N * N - N * (2 * n - 1) + n * (n - 1)
    assert st["abandoned"] == 0 and calls_pruned < st["calls"]


@pytest.mark.parametrize("m,n,k", [(8000, 64, 4), (12000, 128, 5)])
def test_topk_matches_exclusion_zone_oracle(ctx, chk, m, n, k):
    x = planted_walk(9, m, n)
    x[m // 2:m // 2 + n] = W.random_walk(99, n) * np.float32(0.2) + x[m // 2]
    ctx.prepare(x, n, 4, 4)
    pos, dist = ctx.search(k)
    want = chk.topk(x, n, 4, 4, k)
    assert pos == want["positions"]
    np.testing.assert_allclose(dist, want["distances"], rtol=DIST_RTOL)
    for i in range(k):
        for j in range(i):
            assert abs(pos[i] - pos[j]) >= n


def test_nn_profile_matches_oracle(ctx, chk):
    x = W.random_walk(31, 3000)
    ctx.prepare(x, 64, 4, 4)
    got = np.sqrt(ctx.nn_profile().astype(np.float64))
    want = np.sqrt(chk.nn_profile(x, 64))  # the oracle's profile is squared (series.hpp:150-164)
    np.testing.assert_allclose(got, want, rtol=DIST_RTOL)
    assert ctx.fetch("nn_exact").all()


def test_search_is_repeatable_and_independent_of_tunables(ctx):
    x = planted_walk(12, 20000, 128)
    ctx.prepare(x, 128, 4, 4)
    base = ctx.search(3)
    for name, value in [("batch", 300), ("rounds", 1), ("rounds", 12), ("bucket_mates", 0),
                        ("symmetric", 0), ("packed", 0), ("first_batch", 4096), ("wide_tile", 1), ("kernel", 2), ("kernel", 1),
                        ("window_rounds", 0), ("rotate", 0), ("growth", 3.0), ("first_range", 128),
                        ("lower_bound", 0), ("margin_delta", 1e-3), ("batch_growth", 2), ("dot_form", 2),
                        ("dot_form", 0), ("seed_rows", 0), ("tensor_map", 0), ("dot_window_rounds", 0), ("dot_growth", 2.0),
                        ("dot_tile16", 0),
                        ("window_rounds", 4)]:
        ctx.set_option(name, value)
        again = ctx.search(3)
        assert again[0] == base[0], name
        np.testing.assert_allclose(again[1], base[1], rtol=1e-6, err_msg=name)
    for name, value in [("batch", 65536), ("rounds", 64), ("bucket_mates", 8), ("symmetric", 1),
                        ("packed", 1), ("first_batch", 128), ("wide_tile", 0), ("kernel", 0),
                        ("window_rounds", 2), ("rotate", 1), ("growth", 2.0), ("first_range", 8192),
                        ("lower_bound", 1), ("margin_delta", -1), ("batch_growth", 12), ("dot_form", 5),
                        ("seed_rows", 4096), ("tensor_map", 1), ("dot_window_rounds", 8), ("dot_growth", 1.3),
                        ("dot_tile16", 1)]:
        ctx.set_option(name, value)


def test_degenerate_series(ctx):
    ctx.prepare(np.full(600, 3.0, dtype=np.float32), 16, 4, 4)
    pos, dist = ctx.search(2)
    assert pos == [1, 1] or pos[0] == 1
    assert dist[0] == 0.0
    with pytest.raises(InfeasibleInputError):
        ctx.prepare(np.arange(20, dtype=np.float32), 16, 2, 4)
    # smallest feasible input: N = n + 1, only rows 0 and N-1 have a non-self match
    x = W.random_walk(2, 2 * 16)
    ctx.prepare(x, 16, 4, 4)
    pos, dist = ctx.search(1)
    want = oracle.best().run_discovery(x, 16, 4, 4, engine="brute")
    assert pos[0] == want["position"] and dist[0] == pytest.approx(want["distance"], rel=DIST_RTOL)


def test_run_discovery_mirror(chk):
    x = planted_walk(4, 10000, 100)
    out = run_discovery(x, DiscoveryConfig(n=100, word_len=5, alphabet=4, k=2))
    want = chk.topk(x, 100, 5, 4, 2)
    assert [d.position for d in out.discords] == want["positions"]
    assert out.result.position == want["positions"][0]
    assert out.result.distance == pytest.approx(want["distances"][0], rel=DIST_RTOL)
    assert out.m == 10000 and out.prep_time_s > 0 and out.search_time_s > 0


# ------------------------------------------------------------------ BASELINE.json workloads
@pytest.mark.parametrize("cfg", [1, 2, 3, 5, 4])
def test_baseline_workload_matches_golden(golden, cfg):
    key = f"cfg{cfg}"
    if key not in golden:
        pytest.skip(f"no golden record for workload {cfg} yet")
    w = W.workload(cfg)
    x, _ = W.series(cfg)
    assert W.sha256(x) == golden[key]["sha256"]
    out = run_discovery(x, DiscoveryConfig(n=w.n, word_len=w.word_len, alphabet=w.alphabet, k=w.k))
    want = golden[key]["oracle"]
    assert [d.position for d in out.discords] == want["positions"]
    np.testing.assert_allclose([d.distance for d in out.discords], want["distances"], rtol=DIST_RTOL)


# ------------------------------------------------------------------ several ranks on one GPU
class _ThreadExchange:
    """Max-reduce between `world` host threads (the kernels never wait on each other)."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self.calls = 0

    def hook(self, rank):
        def fn(keys):
            self.slots[rank] = keys.copy()
            self.barrier.wait(timeout=120)
            merged = np.maximum.reduce([s for s in self.slots])
            self.barrier.wait(timeout=120)
            keys[:] = merged
            if rank == 0:
                self.calls += 1
        return fn


@pytest.mark.parametrize("share", [1, 0])
@pytest.mark.parametrize("world", [2, 3])
def test_rank_count_does_not_change_the_result(chk, world, share):  # the analogue of SPEC.md:349
    x = planted_walk(15, 16000, 64)
    want = chk.topk(x, 64, 4, 4, 3)
    ex = _ThreadExchange(world)
    results, errors = [None] * world, []

    def run(rank):
        try:
            with Context(0) as c:
                c.set_option("batch", 512)
                c.set_option("share_bounds", share)
                c.set_exchange(ex.hook(rank), world, rank)
                c.prepare(x, 64, 4, 4)
                results[rank] = c.search(3)
        except Exception as e:  # noqa: BLE001
            errors.append(e)
            ex.barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    for r in range(world):
        assert results[r][0] == want["positions"], (r, results[r])
        np.testing.assert_allclose(results[r][1], want["distances"], rtol=DIST_RTOL)
    assert ex.calls > 0


@pytest.mark.parametrize("dot", [1, 2])
def test_ranks_agree_on_the_dot_product_form(chk, dot):
    """Noise, two ranks: the switch to the dot-product form (and the wider discard band that
    goes with it) travels in the per-batch exchange, so both ranks take it together."""
    x = np.random.default_rng(11).random(30000).astype(np.float32)
    want = chk.topk(x, 96, 6, 4, 2)
    world, ex = 2, _ThreadExchange(2)
    results, used, errors = [None] * world, [0] * world, []

    def run(rank):
        try:
            with Context(0) as c:
                c.set_option("batch", 4096)
                c.set_option("dot_form", dot)
                c.set_exchange(ex.hook(rank), world, rank)
                c.prepare(x, 96, 6, 4)
                results[rank] = c.search(2)
                used[rank] = c.stats()["scan_kernel_dot_launches"]
        except Exception as e:  # noqa: BLE001
            errors.append(e)
            ex.barrier.abort()

    threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not errors, errors
    for r in range(world):
        assert_discords_match(chk, x, 96, results[r][0], results[r][1], want)
        assert used[r] > 0


def test_sharing_bounds_between_ranks_saves_work():
    """With "share_bounds" every rank sees what the others' scans learnt about a row; the ranks
    together then scan fewer candidates than when each keeps its bounds to itself."""
    x = W.series(1)[0][:40000]
    scanned = {}
    for share in (0, 1):
        world, ex, out = 2, _ThreadExchange(2), [None, None]

        def run(rank, share=share, ex=ex, out=out):
            with Context(0) as c:
                c.set_option("batch", 1024)
                c.set_option("share_bounds", share)
                c.set_exchange(ex.hook(rank), world, rank)
                c.prepare(x, 128, 4, 4)
                res = c.search(1)
                out[rank] = (res, c.stats()["scanned_candidates"], c.stats()["calls"])

        threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=300)
        assert out[0] is not None and out[1] is not None and out[0][0] == out[1][0]
        scanned[share] = (out[0][0], out[0][1] + out[1][1], out[0][2] + out[1][2])
    assert scanned[0][0] == scanned[1][0]              # same discord either way
    assert scanned[1][2] <= scanned[0][2]              # and fewer pair distances with sharing


def _run_group(world, x, n, w, a, k, options=(), devices=None):
    """`world` contexts of this process as the ranks of one group (tsdd_cuda_group_create), one
    host thread each; returns per rank (positions, distances, stats)."""
    from paper_1901_00155_b200.engine import group_create

    ctxs = [Context((devices or [0] * world)[r]) for r in range(world)]
    out, errors = [None] * world, []
    try:
        for c in ctxs:
            for name, value in options:
                c.set_option(name, value)
        group_create(ctxs)

        def run(rank):
            try:
                c = ctxs[rank]
                c.prepare(x, n, w, a)
                pos, dist = c.search(k)
                out[rank] = (pos, dist, c.stats(), c.fetch("hash"), c.fetch("mean"), c.fetch("inv_sigma"))
            except Exception as e:  # noqa: BLE001
                errors.append(e)

        threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=300)
    finally:
        for c in ctxs:
            c.close()
    assert not errors, errors
    return out


@pytest.mark.parametrize("shard", [1, 0])
@pytest.mark.parametrize("world", [2, 3, 5])
def test_group_of_ranks_in_one_process(chk, world, shard):
    """The in-process multi-GPU mode: bounds min-reduced on the device from the peers' memory,
    window statistics / hashes computed in per-rank slices and gathered (option shard_prep)."""
    x = planted_walk(15, 16000, 64)
    want = chk.topk(x, 64, 4, 4, 3)
    ref = chk.prepare(x, 64, 4, 4, want_rows=False)
    out = _run_group(world, x, 64, 4, 4, 3, options=[("batch", 512), ("shard_prep", shard)])
    with Context(0) as single:
        single.prepare(x, 64, 4, 4)
        mean1, inv1 = single.fetch("mean"), single.fetch("inv_sigma")
    for r in range(world):
        pos, dist, st, hashes, mean, inv = out[r]
        assert pos == want["positions"], (r, pos)
        np.testing.assert_allclose(dist, want["distances"], rtol=DIST_RTOL)
        np.testing.assert_array_equal(hashes, ref["hashes"])   # every rank holds every slice
        np.testing.assert_array_equal(mean, mean1)             # bit-identical to the unsharded preparation
        np.testing.assert_array_equal(inv, inv1)
    assert sum(o[2]["scanned_candidates"] for o in out) > 0


def test_group_shares_bounds_on_the_device():
    """Two ranks of a group scan fewer pair distances together than with share_bounds off."""
    x = W.series(1)[0][:40000]
    calls = {}
    for share in (0, 1):
        out = _run_group(2, x, 128, 4, 4, 1, options=[("batch", 1024), ("share_bounds", share)])
        assert out[0][0] == out[1][0]
        calls[share] = (out[0][0], out[0][2]["calls"] + out[1][2]["calls"])
    assert calls[0][0] == calls[1][0] and calls[1][1] <= calls[0][1], calls


def test_group_failure_on_one_rank_releases_the_others():
    from paper_1901_00155_b200 import ParameterError
    from paper_1901_00155_b200.engine import CudaRuntimeError, group_create

    x = planted_walk(4, 6000, 64)
    ctxs = [Context(0), Context(0)]
    seen = [None, None]
    try:
        group_create(ctxs)

        def run(rank):
            try:
                ctxs[rank].prepare(x, 64, 4, 4)
                if rank == 1:
                    ctxs[rank].search(0)   # k = 0: ParameterError on this rank only
                else:
                    ctxs[rank].search(1)
            except Exception as e:  # noqa: BLE001
                seen[rank] = e

        threads = [threading.Thread(target=run, args=(r,)) for r in range(2)]
        for t in threads:
            t.start()
        for t in threads:
            t.join(timeout=120)
            assert not t.is_alive(), "a rank is stuck in the group's barrier"
    finally:
        for c in ctxs:
            c.close()
    assert isinstance(seen[1], ParameterError)
    assert isinstance(seen[0], CudaRuntimeError) and "another rank" in str(seen[0])


_NCCL_WORKER = r"""
import json, os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.environ["TSDD_ROOT"])
from paper_1901_00155_b200 import Context, parallel, workloads as W
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")           # carries only the 128-byte NCCL id
x = W.series(1)[0][:30000]
with Context(rank) as c:
    parallel.attach_nccl(c)               # the ENGINE's communicator: ncclCommInitRank in libtsdd_cuda.so
    c.prepare(x, 128, 4, 4)
    pos, dd = c.search(2)
    st = c.stats()
    print(json.dumps({"rank": rank, "nranks": c.comm_size(), "pos": pos, "dist": dd,
                      "scanned": st["scanned_candidates"], "calls": st["calls"],
                      "hash_sum": int(c.fetch("hash").sum())}), flush=True)
dist.destroy_process_group()
"""


def test_engine_nccl_communicator_across_processes(chk, tmp_path):
    """One process per GPU, the engine's own NCCL communicator: per-batch ncclAllReduce(max) of the
    keys, ncclAllReduce(min) of the N bounds, ncclAllGather of the sharded window statistics.
    Needs two GPUs (NCCL refuses two ranks on one device)."""
    import subprocess
    import sys

    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs: NCCL does not allow two ranks on one device")
    world = 2
    script = tmp_path / "worker.py"
    script.write_text(_NCCL_WORKER)
    procs = []
    for rank in range(world):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT="29631", TSDD_ROOT=_ROOT)
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (so, se) in zip(procs, outs):
        assert p.returncode == 0, se[-2000:]
    lines = [json.loads(so.strip().splitlines()[-1]) for so, _ in outs]
    x = W.series(1)[0][:30000]
    want = chk.topk(x, 128, 4, 4, 2)
    for line in lines:
        assert line["nranks"] == world and line["pos"] == want["positions"]
        np.testing.assert_allclose(line["dist"], want["distances"], rtol=DIST_RTOL)
    assert lines[0]["hash_sum"] == lines[1]["hash_sum"]
    assert all(line["scanned"] > 0 for line in lines)


_GLOO_WORKER = r"""
import json, os, sys
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.environ["TSDD_ROOT"])
from paper_1901_00155_b200 import Context, parallel, workloads as W
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
x = W.series(1)[0][:30000]
with Context(0) as c:                      # both processes on GPU 0; only the HOSTS meet (gloo all_reduce)
    ex = parallel.attach_torch(c)
    c.prepare(x, 128, 4, 4)
    pos, dd = c.search(2)
    st = c.stats()
    print(json.dumps({"rank": rank, "pos": pos, "dist": dd, "scanned": st["scanned_candidates"],
                      "exchanges": ex.calls}), flush=True)
dist.destroy_process_group()
"""


def test_engine_in_two_processes_with_a_torch_distributed_exchange(chk, tmp_path):
    """One process per rank, torch.distributed (gloo) as the exchange hook: the multi-process
    path of parallel.attach_torch with the real engine.  Both ranks share GPU 0 — their kernels
    never wait on one another, only the host processes meet in the all_reduce."""
    import subprocess
    import sys

    world = 2
    script = tmp_path / "worker.py"
    script.write_text(_GLOO_WORKER)
    procs = []
    for rank in range(world):
        env = dict(os.environ, RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT="29641", TSDD_ROOT=_ROOT)
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=600) for p in procs]
    for p, (so, se) in zip(procs, outs):
        assert p.returncode == 0, se[-2000:]
    lines = [json.loads(so.strip().splitlines()[-1]) for so, _ in outs]
    x = W.series(1)[0][:30000]
    want = chk.topk(x, 128, 4, 4, 2)
    for line in lines:
        assert line["pos"] == want["positions"] and line["exchanges"] > 0
        np.testing.assert_allclose(line["dist"], want["distances"], rtol=DIST_RTOL)
    assert sum(line["scanned"] for line in lines) > 0


def test_nccl_exchange_with_one_rank(chk):
    """The engine's own NCCL path (dlopen, communicator, ncclAllReduce(max, uint64) per batch)."""
    import torch  # noqa: F401  (puts the bundled libnccl.so.2 on the loader's list)

    from paper_1901_00155_b200.engine import comm_unique_id

    x = planted_walk(16, 8000, 64)
    want = chk.run_discovery(x, 64, 4, 4, engine="phidd")
    with Context(0) as c:
        c.comm_init(comm_unique_id(), 1, 0)
        c.prepare(x, 64, 4, 4)
        pos, dist = c.search(1)
    assert pos[0] == want["position"] and dist[0] == pytest.approx(want["distance"], rel=DIST_RTOL)


def _cli(*args, env=None):
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "paper_1901_00155_b200", "_lib", "tsdd_cuda")
    full_env = dict(os.environ, **(env or {}))
    return subprocess.run([exe, *[str(a) for a in args]], capture_output=True, text=True, env=full_env)


def test_cli_find_end_to_end(chk, tmp_path):
    """include/tsdd/cuda_engine.hpp through tools/tsdd_cuda.cpp (the `tsdd find` analogue)."""
    import json

    x = planted_walk(8, 9000, 96)
    want = chk.topk(x, 96, 6, 5, 3)
    path = tmp_path / "series.f32le"
    x.tofile(path)
    p = _cli("find", "--input", path, "--format", "f32le", "--n", 96, "--word-len", 6, "--alphabet", 5, "--k", 3)
    assert p.returncode == 0, p.stderr
    got = json.loads(p.stdout)
    assert [d["pos"] for d in got["discords"]] == want["positions"] and got["pos"] == want["positions"][0]
    np.testing.assert_allclose([d["dist"] for d in got["discords"]], want["distances"], rtol=DIST_RTOL)
    assert got["engine"] == "cuda" and got["m"] == 9000 and got["calls"] > 0
    # csv series and csv result (tools/tsdd.cpp:96-108: same columns)
    csv = tmp_path / "series.csv"
    csv.write_text("t\n" + "\n".join(repr(float(v)) for v in x) + "\n")
    p = _cli("find", "--input", csv, "--n", 96, "--word-len", 6, "--alphabet", 5, "--output", "csv")
    assert p.returncode == 0, p.stderr
    header, row = p.stdout.strip().splitlines()
    assert header == "engine,m,n,word_len,alphabet,threads,pos,dist,calls,prep_time_s,search_time_s"
    cells = row.split(",")
    assert cells[0] == "cuda" and int(cells[6]) == want["positions"][0]
    assert float(cells[7]) == pytest.approx(want["distances"][0], rel=DIST_RTOL)


def test_cli_several_ranks_in_one_process(chk, tmp_path):
    """--gpus: one host thread and one context per rank, in-process max-exchange
    (here every rank on device 0; the kernels never wait on one another)."""
    import json

    x = planted_walk(15, 16000, 64)
    want = chk.topk(x, 64, 4, 4, 3)
    path = tmp_path / "series.f32le"
    x.tofile(path)
    p = _cli("find", "--input", path, "--format", "f32le", "--n", 64, "--k", 3, "--gpus", "0,0,0")
    assert p.returncode == 0, p.stderr
    got = json.loads(p.stdout)
    assert got["gpus"] == 3 and [d["pos"] for d in got["discords"]] == want["positions"]
    np.testing.assert_allclose([d["dist"] for d in got["discords"]], want["distances"], rtol=DIST_RTOL)


def test_cli_bench_sweep(chk, tmp_path):  # run_bench / write_bench_csv, src/bench.cpp:21-87
    x = planted_walk(21, 12000, 64)
    path = tmp_path / "series.f32le"
    x.tofile(path)
    p = _cli("bench", "--input", path, "--format", "f32le", "--n", "32,64", "--gpus", "1,2", "--repeats", 2,
             env={"TSDD_CUDA_SAME_DEVICE": "1"})
    assert p.returncode == 0, p.stderr
    lines = p.stdout.strip().splitlines()
    assert lines[0] == ("engine,m,n,threads,wall_time_s,calls,pos,dist,speedup,efficiency,"
                        "gpus,prep_time_s,search_time_s,terms,fma_pipe_util")
    rows = [dict(zip(lines[0].split(","), ln.split(","))) for ln in lines[1:]]
    assert [(int(r["n"]), int(r["gpus"])) for r in rows] == [(32, 1), (32, 2), (64, 1), (64, 2)]
    for r in rows:
        want = chk.run_discovery(x, int(r["n"]), 4, 4, engine="phidd")
        assert int(r["pos"]) == want["position"] and float(r["dist"]) == pytest.approx(want["distance"], rel=DIST_RTOL)
        if int(r["gpus"]) == 1:
            assert float(r["speedup"]) == 1.0 and float(r["efficiency"]) == 1.0
        assert float(r["efficiency"]) == pytest.approx(float(r["speedup"]) / int(r["gpus"]), rel=1e-5)
        assert int(r["terms"]) > 0 and 0.0 < float(r["fma_pipe_util"]) < 1.0


# ------------------------------------------------------------------ randomised small cases (edge shapes)
def _fuzz_series(rng, kind, m):
    if kind == "walk":
        return np.cumsum(rng.standard_normal(m)).astype(np.float32)
    if kind == "noise":
        return rng.random(m).astype(np.float32)
    if kind == "periodic":
        t = np.arange(m)
        return (np.sin(2 * np.pi * t / 37.0) + 0.05 * rng.standard_normal(m)).astype(np.float32)
    if kind == "flat_parts":
        x = np.cumsum(rng.standard_normal(m)).astype(np.float32)
        a = int(rng.integers(0, m // 2))
        x[a:a + m // 5] = x[a]
        return x
    if kind == "repeats":  # exact repetitions: many nearest-neighbour distances are exactly 0
        base = rng.standard_normal(61).astype(np.float32)
        x = np.tile(base, m // 61 + 1)[:m].copy()
        x[m // 2] += np.float32(4.0)
        return x
    raise ValueError(kind)


FUZZ = [(seed, kind, n) for seed, (kind, n) in enumerate(
    [(k, n) for k in ("walk", "noise", "periodic", "flat_parts", "repeats")
     for n in (2, 3, 8, 17, 33, 63, 64, 65, 127, 129, 200)])]


@pytest.mark.parametrize("seed,kind,n", FUZZ, ids=[f"{k}-n{n}" for _, k, n in FUZZ])
def test_randomised_small_cases_match_the_oracle(ctx, chk, seed, kind, n):
    rng = np.random.default_rng(1000 + seed)
    m = int(rng.integers(2 * n + 1, 2 * n + 1500))
    w = int(rng.integers(1, min(n, 12) + 1))
    a = int(rng.integers(2, 11))
    while a ** w > 2 ** 24:  # keep the reference's dictionary guard happy (sax.hpp:80)
        w -= 1
    k = int(rng.integers(1, 4))
    x = _fuzz_series(rng, kind, m)
    ctx.prepare(x, n, w, a)
    pos, dist = ctx.search(k)
    want = chk.topk(x, n, w, a, k)
    assert_discords_match(chk, x, n, pos, dist, want)


_DOT_LAUNCHES = []


@pytest.mark.parametrize("seed,kind,n", FUZZ, ids=[f"{k}-n{n}" for _, k, n in FUZZ])
def test_dot_product_form_matches_the_oracle(ctx, chk, seed, kind, n):
    """The warp-specialised kernel's one-FFMA-per-term form, forced on from the first launch
    (the engine itself waits until the best-so-far dwarfs the form's absolute error): the
    wider discard band and the float64 decision must still give the reference's answer."""
    rng = np.random.default_rng(7000 + seed)
    m = int(rng.integers(2 * n + 200, 2 * n + 3000))
    w = int(rng.integers(1, min(n, 8) + 1))
    a = int(rng.integers(2, 7))
    k = int(rng.integers(1, 4))
    x = _fuzz_series(rng, kind, m)
    ctx.set_option("dot_form", 2)
    ctx.set_option("lower_bound", 0)  # (covering scans on the warp-specialised kernel as well)
    try:
        ctx.prepare(x, n, w, a)
        pos, dist = ctx.search(k)
        _DOT_LAUNCHES.append(ctx.stats()["scan_kernel_dot_launches"])
    finally:
        ctx.set_option("dot_form", 5)
        ctx.set_option("lower_bound", 1)
    want = chk.topk(x, n, w, a, k)
    assert_discords_match(chk, x, n, pos, dist, want)


@pytest.mark.parametrize("seed,kind,n", FUZZ[::3], ids=[f"{k}-n{n}" for _, k, n in FUZZ[::3]])
def test_dot_product_form_on_256_candidate_tiles(ctx, chk, seed, kind, n):
    """k_scan_tiles_ws16 (16 x 8 pairs per thread, candidate rows pairwise interleaved): batches
    large enough to fill 256-candidate tiles from the first launch on, dot form forced."""
    rng = np.random.default_rng(11000 + seed)
    m = int(rng.integers(2 * n + 5000, 2 * n + 9000))
    w = int(rng.integers(1, min(n, 8) + 1))
    a = int(rng.integers(2, 7))
    k = int(rng.integers(1, 4))
    x = _fuzz_series(rng, kind, m)
    for name, value in [("dot_form", 2), ("lower_bound", 0), ("first_batch", 4096)]:
        ctx.set_option(name, value)
    try:
        ctx.prepare(x, n, w, a)
        pos, dist = ctx.search(k)
        st = ctx.stats()
        used = st["scan_kernel_dot_launches"]
        ctx.set_option("dot_tile16", 0)
        again = ctx.search(k)
    finally:
        for name, value in [("dot_form", 5), ("lower_bound", 1), ("first_batch", 128), ("dot_tile16", 1)]:
            ctx.set_option(name, value)
    want = chk.topk(x, n, w, a, k)
    assert_discords_match(chk, x, n, pos, dist, want)
    # (on exact repetitions the bucket mates settle all rows but the few around the perturbed sample:
    # a search that never has 192 candidates to scan does not reach the 256-candidate kernel)
    assert again[0] == pos and (used > 0 or st["scanned_candidates"] <= 192)
    np.testing.assert_allclose(again[1], dist, rtol=1e-9)


@pytest.mark.parametrize("form", [0, 1, 2], ids=["float64", "float32", "runs"])
@pytest.mark.parametrize("kind", ["walk", "periodic", "repeats"])
def test_every_form_of_the_bucket_mates(ctx, chk, kind, form):
    """k_bucket_mates (float64), k_bucket_mates_f32 (float32, inflated) and k_bucket_mates_runs (chains along
    runs of consecutive rows: full sums at the heads, one-product deltas and a segmented prefix sum for the
    rest) publish upper bounds only: whichever runs, the search returns the reference's answer."""
    rng = np.random.default_rng(991)
    m, n, w, a, k = 9000, 96, 4, 3, 2
    if kind == "walk":
        x = planted_walk(17, m, n)
    elif kind == "periodic":
        x = (np.sin(2 * np.pi * np.arange(m) / 61.0) + 0.05 * rng.standard_normal(m)).astype(np.float32)
        x[4000:4050] += np.float32(0.8)
    else:
        x = _fuzz_series(rng, "repeats", m)
    ctx.set_option("mates_form", form)
    try:
        ctx.prepare(x, n, w, a)
        pos, dist = ctx.search(k)
    finally:
        ctx.set_option("mates_form", -1)
    assert_discords_match(chk, x, n, pos, dist, chk.topk(x, n, w, a, k))


@pytest.mark.parametrize("convert", [1, 0], ids=["converting", "split-copies"])
@pytest.mark.parametrize("kind", ["walk", "periodic", "low-noise"])
def test_tails_of_covering_scans_on_the_tensor_cores(ctx, chk, kind, convert):
    """The later ranges of a covering scan move to the tensor cores (engine.cu: tail_now; forced here at the
    first chance, with the lower-bound filter in the kernel's metadata warp), the first batch on trust.  On the
    low-noise series the first batch's best-so-far does NOT dwarf the error band: the search has to notice,
    start over without the tails, and still return the reference's answer.  Both feeds of the kernel: the
    neighbours' fp16 parts made inside it from the float32 matrix (the default), and split copies of the matrix."""
    rng = np.random.default_rng(4242)
    m, n, w, a, k = 40000, 64, 4, 4, 2
    if kind == "walk":
        x = planted_walk(31, m, n)
    elif kind == "periodic":
        x = (np.sin(2 * np.pi * np.arange(m) / 50.0) + 0.3 * rng.standard_normal(m)).astype(np.float32)
        x[17000:17064] += np.float32(1.5)
    else:
        x = (np.sin(2 * np.pi * np.arange(m) / 50.0) + 1e-4 * rng.standard_normal(m)).astype(np.float32)
    for name, value in [("tc_tail_force", 1), ("first_batch", 128), ("tc_convert", convert)]:
        ctx.set_option(name, value)
    try:
        ctx.prepare(x, n, w, a)
        pos, dist = ctx.search(k)
        st = ctx.stats()
    finally:
        ctx.set_option("tc_tail_force", 0)
        ctx.set_option("tc_convert", 1)
    want = chk.topk(x, n, w, a, k)
    assert_discords_match(chk, x, n, pos, dist, want)
    if kind == "low-noise":
        assert st["tail_restarts"] == 1 or st["scan_kernel_tc_launches"] == 0
    else:
        assert st["scan_kernel_tc_launches"] > 0 and st["tail_restarts"] == 0


@pytest.mark.parametrize("form", [4, 6], ids=["tf32", "fp16"])
@pytest.mark.parametrize("seed,kind,n", FUZZ[::3], ids=[f"{k}-n{n}" for _, k, n in FUZZ[::3]])
def test_dot_product_form_on_the_tensor_cores(ctx, chk, seed, kind, n, form):
    """k_scan_tiles_tc (dot_form = 4: tcgen05.mma kind::tf32 on rows split into two tf32 parts; 6:
    kind::f16 on two fp16 parts; accumulators in tensor memory; csrc/tc_kernels.cu), forced from the first launch on batches
    that fill 128-candidate tiles: the wider band and the float64 decision must still give the
    reference's answer, and the answer of the CUDA-core dot form."""
    rng = np.random.default_rng(13000 + seed)
    m = int(rng.integers(2 * n + 5000, 2 * n + 9000))
    w = int(rng.integers(1, min(n, 8) + 1))
    a = int(rng.integers(2, 7))
    k = int(rng.integers(1, 4))
    x = _fuzz_series(rng, kind, m)
    for name, value in [("dot_form", form), ("lower_bound", 0), ("first_batch", 4096)]:
        ctx.set_option(name, value)
    try:
        ctx.prepare(x, n, w, a)
        pos, dist = ctx.search(k)
        st = ctx.stats()
        ctx.set_option("dot_form", 2)
        again = ctx.search(k)
    finally:
        for name, value in [("dot_form", 5), ("lower_bound", 1), ("first_batch", 128)]:
            ctx.set_option(name, value)
    want = chk.topk(x, n, w, a, k)
    assert_discords_match(chk, x, n, pos, dist, want)
    assert st["scan_kernel_tc_launches"] > 0 and 0 < st["scan_kernel_tc_terms"] <= st["scan_kernel_dot_terms"]
    assert_discords_match(chk, x, n, again[0], again[1], want)
    if n >= 8:  # (tiny n: exact ties everywhere, and which of the tied rows gets scanned to the end depends on the path)
        assert again[0] == pos
        np.testing.assert_allclose(again[1], dist, rtol=1e-9)  # both decided in float64


def _hard_series(kind, m, rng):
    if kind == "spikes":      # a few huge outliers: windows whose energy sits in one sample
        x = rng.standard_normal(m).astype(np.float32)
        x[rng.integers(0, m, 12)] += np.float32(1e4)
        return x
    if kind == "offset":      # small noise on a large offset: mean^2 / variance ~ 1e10
        return (np.float32(1e4) + np.float32(0.1) * rng.standard_normal(m)).astype(np.float32)
    if kind == "steps":       # piecewise constant with noise: many near-flat windows
        x = np.repeat(rng.integers(-3, 4, m // 500 + 1), 500)[:m].astype(np.float32)
        return x + np.float32(1e-3) * rng.standard_normal(m).astype(np.float32)
    if kind == "ramp":        # strong trend
        return (np.arange(m, dtype=np.float32) * np.float32(0.01) + rng.standard_normal(m).astype(np.float32))
    raise ValueError(kind)


@pytest.mark.parametrize("dot", [1, 2])
@pytest.mark.parametrize("kind", ["spikes", "offset", "steps", "ramp"])
def test_awkward_value_distributions(ctx, chk, kind, dot):
    """Inputs that stress the float32 matrix and the dot-product form's absolute error band."""
    rng = np.random.default_rng({"spikes": 31, "offset": 32, "steps": 33, "ramp": 34}[kind])
    x = _hard_series(kind, 12000, rng)
    for name, value in [("dot_form", dot), ("first_batch", 1024 if dot == 2 else 128)]:
        ctx.set_option(name, value)
    try:
        ctx.prepare(x, 96, 6, 4)
        pos, dist = ctx.search(3)
    finally:
        ctx.set_option("dot_form", 5)
        ctx.set_option("first_batch", 128)
    want = chk.topk(x, 96, 6, 4, 3)
    assert_discords_match(chk, x, 96, pos, dist, want)


def test_dot_product_form_cases_did_run_the_dot_kernel():
    # batches that have shrunk to <= 64 live candidates use the 64-candidate tile kernel instead
    assert len(_DOT_LAUNCHES) == len(FUZZ) and sum(1 for v in _DOT_LAUNCHES if v > 0) >= len(FUZZ) * 3 // 4, _DOT_LAUNCHES


def test_dot_product_form_is_chosen_where_tiles_are_never_abandoned(ctx, chk):
    """i.i.d. noise (BASELINE.json workload 5 in small): no tile is ever abandoned, so after
    two batches the search switches to the dot-product form; on a random walk with a planted
    anomaly the tiles are abandoned early and it stays with the direct form."""
    x = np.random.default_rng(5).random(40000).astype(np.float32)
    ctx.prepare(x, 128, 8, 4)
    pos, dist = ctx.search(2)
    st = ctx.stats()
    assert st["scan_kernel_dot_launches"] > 0 and 0 < st["scan_kernel_dot_terms"] <= st["scan_kernel_terms"]
    want = chk.topk(x, 128, 8, 4, 2)
    assert_discords_match(chk, x, 128, pos, dist, want)
    ctx.set_option("dot_form", 0)
    try:
        again = ctx.search(2)
        assert ctx.stats()["scan_kernel_dot_launches"] == 0
    finally:
        ctx.set_option("dot_form", 5)
    assert again[0] == pos
    np.testing.assert_allclose(again[1], dist, rtol=1e-9)  # both decided in float64

    y = planted_walk(3, 40000, 128)
    ctx.prepare(y, 128, 4, 4)
    ctx.search(1)
    st = ctx.stats()  # (the only dot-form launches there may be are tails of covering scans on the tensor cores)
    assert st["scan_kernel_dot_launches"] == st["scan_kernel_tc_launches"]
    ctx.set_option("tc_tail", 0)
    try:
        ctx.search(1)
        assert ctx.stats()["scan_kernel_dot_launches"] == 0
    finally:
        ctx.set_option("tc_tail", 1)


@pytest.mark.parametrize("seed,kind,n", FUZZ[::2], ids=[f"{k}-n{n}" for _, k, n in FUZZ[::2]])
def test_filter_on_the_producer_warpgroup_matches_the_oracle(ctx, chk, seed, kind, n):
    """"filter_in_ws": covering scans with the lower-bound filter on the warp-specialised kernel
    (tensor-map loads, the filter on the four producer warps) instead of k_scan_tiles."""
    rng = np.random.default_rng(9000 + seed)
    m = int(rng.integers(2 * n + 400, 2 * n + 4000))
    w = int(rng.integers(1, min(n, 8) + 1))
    a = int(rng.integers(2, 7))
    k = int(rng.integers(1, 4))
    x = _fuzz_series(rng, kind, m)
    ctx.set_option("filter_in_ws", 1)
    try:
        ctx.prepare(x, n, w, a)
        pos, dist = ctx.search(k)
    finally:
        ctx.set_option("filter_in_ws", 0)
    want = chk.topk(x, n, w, a, k)
    assert_discords_match(chk, x, n, pos, dist, want)


def test_filter_on_the_producer_warpgroup_rules_tiles_out(ctx, chk):
    x, _ = W.series(2)
    x = x[:120000]
    ctx.prepare(x, 256, 8, 4)
    base = ctx.search(3)
    ctx.set_option("filter_in_ws", 1)
    try:
        got = ctx.search(3)
        st = ctx.stats()
    finally:
        ctx.set_option("filter_in_ws", 0)
    assert got[0] == base[0]
    np.testing.assert_allclose(got[1], base[1], rtol=1e-9)
    assert st["lb_skipped"] > 0 and st["scan_kernel_ws_launches"] > 0


def test_seeded_best_so_far_saves_work_and_keeps_the_result(ctx, chk):
    """The first pass starts from the greatest lower bound of a nearest-neighbour distance among
    the rarest rows (segment-mean boxes) instead of zero: fewer pair distances, same discords."""
    x, _ = W.series(2)
    x = x[:120000]
    ctx.prepare(x, 256, 8, 4)
    # (pair distances are compared without the tensor-core tails, which start every pair of the tiles they visit)
    ctx.set_option("tc_tail", 0)
    ctx.set_option("seed_rows", 0)
    try:
        plain = ctx.search(3)
        plain_calls = ctx.stats()["calls"]
        ctx.set_option("seed_rows", 4096)
        seeded = ctx.search(3)
        seeded_calls = ctx.stats()["calls"]
    finally:
        ctx.set_option("seed_rows", 4096)
        ctx.set_option("tc_tail", 1)
    with_tails = ctx.search(3)
    assert with_tails[0] == seeded[0]
    np.testing.assert_allclose(with_tails[1], seeded[1], rtol=1e-9)
    assert seeded[0] == plain[0]
    np.testing.assert_allclose(seeded[1], plain[1], rtol=1e-9)
    assert seeded_calls < plain_calls
    want = chk.topk(x, 256, 8, 4, 3)
    assert_discords_match(chk, x, 256, seeded[0], seeded[1], want)


def test_smallest_feasible_and_k_beyond_the_series(ctx, chk):
    for n in (1, 2, 16, 100):
        x = W.random_walk(40 + n, 2 * n)  # m = 2n: N = n + 1, only the two end rows have a non-self match
        ctx.prepare(x, n, 1, 2)
        pos, dist = ctx.search(3)         # more discords than rows that can hold one
        want = chk.topk(x, n, 1, 2, 3)
        assert_discords_match(chk, x, n, pos, dist, want)


def test_long_subsequences(ctx, chk):
    x = planted_walk(5, 24000, 4096)
    ctx.prepare(x, 4096, 16, 4)
    pos, dist = ctx.search(2)
    want = chk.topk(x, 4096, 8, 4, 2)  # the reference's guard rejects 4^16 words; results do not depend on it
    assert pos == want["positions"]
    np.testing.assert_allclose(dist, want["distances"], rtol=DIST_RTOL)


# ------------------------------------------------------------------ the edges of the float32 search
def _low_noise_periodic(seed, m, noise):
    rng = np.random.default_rng(seed)
    t = np.arange(m)
    return (np.sin(2 * np.pi * t / 64.0) + noise * rng.standard_normal(m)).astype(np.float32)


@pytest.mark.parametrize("dot", [1, 2])
@pytest.mark.parametrize("seed,noise", [(0, 1e-4), (1, 1e-4), (2, 3e-5), (3, 1e-3)])
def test_low_noise_periodic_series(ctx, chk, seed, noise, dot):
    """Clean periodic data: nearest-neighbour distances d^2 ~ 1e-5 .. 1e-3, where the float32
    QUANTISATION of the z-normalised rows (d sqrt(n) 2^-22: relative size ~ 1 / d) exceeds the
    relative discard band.  The sqrt(best) term of the band (common.cuh: dead_bound) and the
    float64 decision must still give the reference's positions."""
    x = _low_noise_periodic(seed, 9000, noise)
    ctx.set_option("dot_form", dot)
    try:
        ctx.prepare(x, 256, 8, 4)
        pos, dist = ctx.search(2)
    finally:
        ctx.set_option("dot_form", 5)
    want = chk.topk(x, 256, 8, 4, 2)
    assert pos == want["positions"], (pos, want["positions"], dist, want["distances"])
    np.testing.assert_allclose(dist, want["distances"], rtol=DIST_RTOL)


def test_many_near_tied_finalists_are_all_settled(ctx, chk):
    """More finalists than the first collection has room for: the pass collects again and
    settles ALL of them in float64 (it used to keep the float32 winner).  The discard band is
    widened artificially (margin_delta) so that hundreds of exact rows fall inside it."""
    x = planted_walk(11, 30000, 128)
    ctx.prepare(x, 128, 4, 4)
    base_pos, base_dist = ctx.search(3)
    ctx.set_option("margin_delta", 0.45)
    ctx.set_option("finalist_cap", 2)
    try:
        pos, dist = ctx.search(3)
        st = ctx.stats()
    finally:
        ctx.set_option("margin_delta", -1)
        ctx.set_option("finalist_cap", 64)
    assert st["finalists"] > 64, st["finalists"]
    want = chk.topk(x, 128, 4, 4, 3)
    assert pos == base_pos == want["positions"]
    np.testing.assert_allclose(dist, want["distances"], rtol=DIST_RTOL)
    np.testing.assert_allclose(dist, base_dist, rtol=1e-12)  # both decided in float64


def test_finalists_follow_the_band_after_a_switch_to_the_dot_form(ctx, chk):
    """The search switches to the dot-product form MID-search (noise: no tile is abandoned); the
    discard band then widens by the form's absolute error.  The finalists must be collected with
    that wider band, not with the one the search started with.  Series: noise u followed by its
    mirror image 1 - u, perturbed by 1e-6 — every row has a mirror row whose nn distance differs
    by ~1e-5 .. 1e-4 (squared): far inside the dot form's absolute band (0.0024 at n = 128), and,
    with the relative parts of the band switched off, outside everything else."""
    n = 128
    rng = np.random.default_rng(5)
    u = rng.random(20000).astype(np.float32)
    v = (np.float32(1.0) - u + (1e-6 * rng.standard_normal(20000)).astype(np.float32)).astype(np.float32)
    x = np.concatenate([u, v])
    ctx.set_option("margin_delta", 0)
    ctx.set_option("margin_q", 0)
    try:
        ctx.prepare(x, n, 8, 4)
        pos, dist = ctx.search(2)
        st = ctx.stats()
    finally:
        ctx.set_option("margin_delta", -1)
        ctx.set_option("margin_q", -1)
    assert st["scan_kernel_dot_launches"] > 0 and st["scan_kernel_launches"] > st["scan_kernel_dot_launches"]
    profile = chk.nn_profile(x, n)
    own_pos, own_dist = topk_from_profile(profile, n, 2)
    assert pos == own_pos, (pos, own_pos)
    np.testing.assert_allclose(dist, own_dist, rtol=1e-12)
    # the second discord and its mirror row are a near-tie: both must have been finalists
    second = own_pos[1] - 1
    mirror = second + 20000 if second < 20000 else second - 20000
    gap = abs(profile[second] - profile[mirror])
    assert 0 < gap < 1e-3, gap
    assert st["finalists"] >= 3, st["finalists"]


def test_device_series_is_validated_on_the_device(ctx):
    """validate_series (series.cpp:10-19) for tsdd_cuda_prepare_device_f32: the samples never pass
    through the host, so the finite check runs in k_widen_series."""
    import torch

    from paper_1901_00155_b200 import ValidationError

    x = W.random_walk(1, 5000)
    x[1234] = np.float32("nan")
    x[4000] = np.float32("inf")
    d = torch.from_numpy(x).cuda()
    with pytest.raises(ValidationError, match=r"non-finite value at index 1235$"):
        ctx.prepare_device(d.data_ptr(), len(x), 64, 4, 4)
    with pytest.raises(Exception, match="prepared"):
        ctx.search(1)
    x[1234] = 0.0
    x[4000] = 0.0
    d = torch.from_numpy(x).cuda()
    ctx.prepare_device(d.data_ptr(), len(x), 64, 4, 4)
    ctx.search(1)


# ------------------------------------------------------------------ the reference-shaped C++ boundary
import subprocess  # noqa: E402

MIRROR_CHECK = os.path.join(_ROOT, "paper_1901_00155_b200", "_lib", "mirror_check")
TSDD_PATCHED = os.path.join(_ROOT, "oracle", "_ref", "tsdd_patched")


@pytest.mark.parametrize("m,n,w,a,k", [(3000, 64, 4, 4, 1), (2500, 50, 3, 5, 2), (5000, 128, 6, 3, 3)])
def test_cpp_mirrors_of_the_reference_types(chk, tmp_path, m, n, w, a, k):
    """tsdd::cuda::SubsequenceMatrix::build -> DiscordIndexes::build -> phidd_discord
    (include/tsdd/cuda_engine.hpp), chained as pipeline.cpp:60-87 chains the reference's:
    every accessor the mirrors expose against the reference's own arrays."""
    x = planted_walk(m + n, m, n).astype(np.float64)
    path = tmp_path / "s.f64le"
    x.tofile(path)
    rows_wanted = [0, 1, m - n, (m - n) // 2]
    p = subprocess.run([MIRROR_CHECK, str(path), str(n), str(w), str(a), str(k), ",".join(map(str, rows_wanted))],
                       capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    got = json.loads(p.stdout)
    ref = chk.prepare(x, n, w, a)
    N = m - n + 1
    assert got["rows"] == N and got["n"] == n and got["stride"] == (n + 63) // 64 * 64
    assert got["pad"] == got["stride"] - n and got["vec_width"] == 8
    np.testing.assert_array_equal(np.array(got["hashes"], dtype=np.uint64), ref["hashes"])
    np.testing.assert_array_equal(np.array(got["freq"], dtype=np.uint32), ref["freq"])
    np.testing.assert_array_equal(np.array(got["candidates"], dtype=np.uint64), ref["candidates"])
    assert got["bucket_count"] == a ** w and got["total_positions"] == N
    # WordIndex::bucket(h) (index.hpp:29): ascending 1-based positions of every occupied word
    want_buckets = {}
    for pos in ref["bucket_positions"]:
        want_buckets.setdefault(int(ref["hashes"][int(pos) - 1]), []).append(int(pos))
    assert {int(h): v for h, v in got["buckets"].items()} == want_buckets
    for r in rows_wanted:  # SubsequenceMatrix::row(i) (series.hpp:53), float32 on the device
        row = np.array(got["row_values"][str(r)])
        np.testing.assert_allclose(row[:n], ref["rows"][r], rtol=0, atol=2e-6)
        assert not row[n:].any()
    want = chk.topk(x, n, w, a, k)
    assert got["positions"] == want["positions"] and got["pos"] == want["positions"][0]
    np.testing.assert_allclose(got["distances"], want["distances"], rtol=DIST_RTOL)
    assert got["calls"] > 0 and got["abandoned"] <= got["calls"]


def test_cpp_mirrors_keep_the_reference_error_contract(tmp_path):
    """series.cpp:46-56 (validation, then n, then vec_width), discovery.cpp:22-29,114-121."""
    path = tmp_path / "s.f64le"
    np.arange(20.0).tofile(path)
    p = subprocess.run([MIRROR_CHECK, str(path), "16", "2", "4"], capture_output=True, text=True)
    assert p.returncode == 4 and "N=5 <= n=16 (need series length m >= 2n)" in p.stderr, p.stderr
    p = subprocess.run([MIRROR_CHECK, str(path), "21", "2", "4"], capture_output=True, text=True)
    assert p.returncode == 2 and "subsequence length n=21 must satisfy 1 <= n <= m=20" in p.stderr, p.stderr
    p = subprocess.run([MIRROR_CHECK, str(path), "4", "5", "4"], capture_output=True, text=True)
    assert p.returncode == 2 and "word_len=5 must satisfy 1 <= word_len <= n=4" in p.stderr, p.stderr
    p = subprocess.run([MIRROR_CHECK, str(path), "4", "2", "11"], capture_output=True, text=True)
    assert p.returncode == 2 and "outside the built-in range 2..10" in p.stderr, p.stderr
    bad = np.arange(20.0)
    bad[4] = np.nan
    bad.tofile(path)
    p = subprocess.run([MIRROR_CHECK, str(path), "4", "2", "4"], capture_output=True, text=True)
    assert p.returncode == 3 and "non-finite value at index 5" in p.stderr, p.stderr


def test_patched_reference_runs_the_cuda_engine(golden, chk, tmp_path):
    """oracle/_ref/tsdd_patched = the reference's own sources with INTEGRATION.md's patch
    (tools/patch_reference.py), compiled with TSDD_CUDA_WITH_REFERENCE_HEADERS and linked against
    libtsdd_cuda.so.  `cuda` enters through the reference's tsdd::run_discovery and must return
    what its own CPU engine returns from the same binary — and the golden cfg1 result."""
    if not os.path.exists(TSDD_PATCHED):
        pytest.skip("oracle/_ref/tsdd_patched is built where /root/reference exists")
    x, _ = W.series(1)
    w = W.workload(1)
    path = tmp_path / "cfg1.f64le"
    x.astype(np.float64).tofile(path)

    def run(engine, *extra):
        p = subprocess.run([TSDD_PATCHED, str(path), engine, str(w.n), str(w.word_len), str(w.alphabet), *extra],
                           capture_output=True, text=True)
        assert p.returncode == 0, p.stderr
        return json.loads(p.stdout)

    cuda = run("cuda")
    cpu = run("phidd", str(os.cpu_count() or 1))
    rec = golden["cfg1"]["oracle"]
    assert cuda["engine"] == "cuda" and cpu["engine"] == "phidd"
    assert cuda["pos"] == cpu["pos"] == rec["positions"][0]
    assert cuda["dist"] == pytest.approx(cpu["dist"], rel=DIST_RTOL)
    assert cuda["dist"] == pytest.approx(rec["distances"][0], rel=DIST_RTOL)
    assert cuda["m"] == w.m and cuda["calls"] > 0 and cuda["search_time_s"] > 0
    # the reference's error contract through the patched entry point (tools/tsdd.cpp:212-223)
    p = subprocess.run([TSDD_PATCHED, str(path), "cuda", str(w.m), "4", "4"], capture_output=True, text=True)
    assert p.returncode == 2 and "no subsequence has a non-self match" in p.stderr, p.stderr
    p = subprocess.run([TSDD_PATCHED, str(path), "gpu", "128", "4", "4"], capture_output=True, text=True)
    assert p.returncode == 2 and "unknown engine 'gpu'" in p.stderr, p.stderr


# ------------------------------------------------------------------ soak, and the checked build
@pytest.mark.parametrize("case", range(12))
def test_soak_random_series_shapes_and_options(ctx, chk, case):
    """tools/soak.py, reduced: random kind / length / n / SAX shape / k AND random engine options
    (dot form, first batch, filter, filter on the producer warpgroup, time topology) against the
    reference's exclusion-zone top-k."""
    rng = np.random.default_rng(90000 + case)
    kind = rng.choice(["noise", "walk", "sine"])
    m = int(rng.integers(15000, 40000))
    n = int(rng.choice([24, 50, 64, 100, 128, 200, 256, 300]))
    w, a, k = int(rng.integers(2, 9)), int(rng.integers(2, 7)), int(rng.integers(1, 4))
    if kind == "noise":
        x = rng.random(m).astype(np.float32)
    elif kind == "walk":
        x = np.cumsum(rng.standard_normal(m)).astype(np.float32)
    else:
        x = (np.sin(2 * np.pi * np.arange(m) / rng.integers(20, 200)) + 0.3 * rng.standard_normal(m)).astype(np.float32)
    opts = {"dot_form": int(rng.choice([1, 2, 3, 4, 5, 6])), "first_batch": int(rng.choice([128, 4096])),
            "lower_bound": int(rng.choice([0, 1])), "filter_in_ws": int(rng.choice([0, 1])),
            "propagate": int(rng.choice([0, 2, 8])), "propagate_every": int(rng.choice([0, 1, 2]))}
    defaults = {"dot_form": 5, "first_batch": 128, "lower_bound": 1, "filter_in_ws": 0, "propagate": 8,
                "propagate_every": 2}
    try:
        for name, value in opts.items():
            ctx.set_option(name, value)
        ctx.prepare(x, n, w, a)
        pos, dist = ctx.search(k)
    finally:
        for name, value in defaults.items():
            ctx.set_option(name, value)
    want = chk.topk(x, n, w, a, k)
    assert_discords_match(chk, x, n, pos, dist, want)


def test_checked_build_runs_the_edge_shapes():
    """libtsdd_cuda_dbg.so (-DTSDD_DEBUG_BOUNDS: every data-dependent global-memory index is
    checked inside the kernels and traps on a violation) through the randomised edge-shape tests,
    the dot-product form, the 256-candidate tiles, the filter on the producer warpgroup, the rank
    group and the soak — in place of compute-sanitizer, which this GPU pool does not offer."""
    import subprocess
    import sys

    dbg = os.path.join(_ROOT, "paper_1901_00155_b200", "_lib", "libtsdd_cuda_dbg.so")
    assert os.path.exists(dbg), "build it with python -m paper_1901_00155_b200.build"
    expr = ("randomised_small_cases or dot_product_form_matches or 256_candidate or filter_on_the_producer_warpgroup_matches"
            " or group_of_ranks or soak_random or smallest_feasible or long_subsequences or topk_matches or on_the_tensor_cores")
    p = subprocess.run([sys.executable, "-m", "pytest", os.path.join(_ROOT, "tests", "test_gpu_parity.py"), "-x", "-q",
                        "-m", "gpu", "-k", expr, "-p", "no:cacheprovider"],
                       env=dict(os.environ, TSDD_CUDA_LIB=dbg), capture_output=True, text=True, timeout=1500)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-2000:]
    assert "TSDD_DEBUG_BOUNDS" not in p.stdout + p.stderr
