"""Pins the CPU oracle (oracle/tsdd_oracle.c, the "port") before anything trusts it.

Three anchors:
  1. the SPEC.md known-answer examples (the reference ships no tests; these
     are its only pinned values),
  2. the unmodified reference itself (oracle/_ref, compiled from
     /root/reference/proj) on seeded random inputs, array by array,
  3. tests/golden/workloads.json — reference outputs on the BASELINE.json series.

Integer outputs (symbols, hashes, frequencies, candidates, buckets,
positions) must be identical; float64 distances agree to 1e-12 relative and
z-normalised rows to 1e-10 absolute: the reference build contracts a*b+c into
FMAs where the port (compiled with -ffp-contract=off so that it is the same
on every host) does not, and the cancellation in sum_sq/n - mu^2
(series.cpp:29) amplifies that last-bit difference on random-walk levels.
"""
import math

import numpy as np
import pytest

import oracle
from paper_1901_00155_b200 import workloads as W

port = oracle.port()
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")

CHECKERS = [pytest.param(oracle.port, id="port")] + (
    [pytest.param(oracle.ref, id="reference")] if oracle.ref_available() else [])


# ---------------------------------------------------------------- SPEC known answers
@pytest.mark.parametrize("get", CHECKERS)
class TestSpecExamples:
    def test_znorm_examples(self, get):
        c = get()
        np.testing.assert_allclose(c.z_normalize([1, 2, 3]), [-1.224744871, 0, 1.224744871], atol=1e-8)
        assert np.all(c.z_normalize([5, 5, 5, 5]) == 0)
        z = c.z_normalize(W.random_walk(11, 1000))
        assert abs(z.mean()) < 1e-12 and abs(z.std() - 1) < 1e-12

    def test_matrix_shape_and_rows(self, get):
        c = get()
        p = c.prepare(np.arange(10.0), 4, 2, 4)
        assert p["rows"].shape == (7, 4)
        p = c.prepare(np.array([0.0, 1, 2, 3, 4, 5, 6, 7]), 3, 1, 2)
        np.testing.assert_allclose(p["rows"][0], [-1.224744871, 0, 1.224744871], atol=1e-8)

    def test_distance_examples(self, get):
        c = get()
        assert c.distance([0, 0, 0, 0], [3, 4, 0, 0]) == 25.0
        x = W.random_walk(3, 257).astype(np.float64)
        assert c.distance(x, x) == 0.0
        y = W.random_walk(4, 257).astype(np.float64)
        d = c.distance(x, y)
        assert d == pytest.approx(float(((x - y) ** 2).sum()), rel=1e-9)
        assert c.distance(x, y) == c.distance(y, x)
        # early-abandon soundness: abandoned <=> true distance strictly above the threshold
        assert c.distance(x, y, threshold=d) == d
        assert c.distance(x, y, threshold=np.nextafter(d, 0)) is None
        # padding neutrality
        assert c.distance(np.append(x, [0] * 7), np.append(y, [0] * 7)) == pytest.approx(d, rel=1e-15)

    def test_paa_examples(self, get):
        c = get()
        np.testing.assert_array_equal(c.paa_row([1, 1, 1, 1, 2, 2, 2, 2], 2), [1, 2])
        v = W.random_walk(5, 128).astype(np.float64)
        np.testing.assert_allclose(c.paa_row(v, 4), v.reshape(4, 32).mean(axis=1), atol=1e-12)
        # w does not divide n: fractional overlap keeps the global mean
        v = np.arange(10.0)
        assert c.paa_row(v, 3).mean() == pytest.approx(v.mean(), rel=1e-14)

    def test_sax_examples(self, get):
        c = get()
        assert c.symbol_for(4, 0.0) == 3  # a value on a breakpoint goes to the upper bin
        for a in range(2, 11):
            assert c.symbol_for(a, -10.0) == 1 and c.symbol_for(a, 10.0) == a
        assert [c.symbol_for(4, v) for v in (-1, -0.1, 0.1, 1)] == [1, 2, 3, 4]

    def test_hash_examples(self, get):
        c = get()
        assert c.word_hash([1, 1, 1, 1], 4) == 1 and c.word_hash([4, 4, 4, 4], 4) == 256
        seen = {c.word_hash([a, b, cc, d], 4) for a in range(1, 5) for b in range(1, 5)
                for cc in range(1, 5) for d in range(1, 5)}
        assert seen == set(range(1, 257))

    def test_index_cross_consistency(self, get):
        c = get()
        p = c.prepare(W.random_walk(9, 1500), 32, 3, 4)
        freq, hashes, buckets = p["freq"], p["hashes"], p["bucket_positions"]
        assert len(buckets) == len(freq) and sorted(buckets) == list(range(1, len(freq) + 1))
        assert list(p["candidates"]) == [i + 1 for i in range(len(freq)) if freq[i] == freq.min()]
        # buckets are listed in ascending hash order, ascending positions inside
        hb = hashes[buckets.astype(np.int64) - 1]
        assert np.all(np.diff(hb.astype(np.int64)) >= 0)
        same = np.diff(hb.astype(np.int64)) == 0
        assert np.all(np.diff(buckets.astype(np.int64))[same] > 0)
        # freq[i] = size of row i's bucket
        sizes = {h: int((hashes == h).sum()) for h in np.unique(hashes)}
        assert all(freq[i] == sizes[hashes[i]] for i in range(len(freq)))

    def test_degenerate_and_errors(self, get):
        c = get()
        r = c.run_discovery(np.full(64, 3.0), 8, 2, 4, threads=2)
        assert (r["position"], r["distance"]) == (1, 0.0)
        with pytest.raises(oracle.OracleError) as e:
            c.run_discovery(np.arange(20.0), 16, 2, 4, threads=1)
        assert e.value.code == oracle.ERR_INFEASIBLE
        with pytest.raises(oracle.OracleError) as e:
            c.run_discovery(np.arange(20.0), 20, 2, 4, threads=1)  # n = m
        assert e.value.code == oracle.ERR_INFEASIBLE
        with pytest.raises(oracle.OracleError) as e:
            c.run_discovery(np.arange(64.0), 8, 2, 11, threads=1)
        assert e.value.code == oracle.ERR_PARAMETER
        with pytest.raises(oracle.OracleError) as e:
            c.run_discovery(np.arange(64.0), 8, 13, 4, threads=1)  # 4^13 > 2^24
        assert e.value.code == oracle.ERR_PARAMETER
        bad = np.arange(64.0)
        bad[5] = np.nan
        with pytest.raises(oracle.OracleError) as e:
            c.run_discovery(bad, 8, 2, 4, threads=1)
        assert e.value.code == oracle.ERR_VALIDATION and "index 6" in e.value.message

    def test_engines_agree_and_threads_do_not_matter(self, get):
        c = get()
        x = W.random_walk(21, 2000)
        base = c.run_discovery(x, 64, 4, 4, engine="brute", threads=4)
        # closed-form brute call count
        N, n = 2000 - 64 + 1, 64
        assert base["calls"] == sum(max(0, i - n + 1) + max(0, N - i - n) for i in range(N))
        for eng in ("hotsax", "phidd"):
            for th in (1, 3):
                r = c.run_discovery(x, 64, 4, 4, engine=eng, threads=th)
                assert r["position"] == base["position"]
                assert r["distance"] == pytest.approx(base["distance"], rel=1e-12)
        r = c.run_discovery(x, 64, 4, 4, engine="phidd", threads=2, disable_pruning=True)
        assert r["position"] == base["position"] and r["abandoned"] == 0


# ---------------------------------------------------------------- port == reference
@needs_ref
@pytest.mark.parametrize("seed,m,n,w,a", [(1, 2000, 32, 4, 4), (2, 2000, 64, 8, 3), (3, 1500, 50, 7, 6),
                                          (4, 3000, 128, 4, 10), (5, 1200, 100, 3, 5)])
def test_port_matches_reference_arrays(seed, m, n, w, a):
    x = W.random_walk(seed, m)
    R, P = oracle.ref().prepare(x, n, w, a), port.prepare(x, n, w, a)
    np.testing.assert_allclose(P["rows"], R["rows"], rtol=0, atol=1e-10)
    np.testing.assert_allclose(P["paa"], R["paa"], rtol=0, atol=1e-10)
    for key in ("sax", "hashes", "freq", "candidates", "bucket_positions"):
        np.testing.assert_array_equal(P[key], R[key], err_msg=key)


@needs_ref
@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("n", [32, 64, 128])
def test_port_matches_reference_search(seed, n):  # SPEC.md:449-452 sweep, reduced
    x = W.random_walk(100 + seed, 2000)
    r = oracle.ref().run_discovery(x, n, 4, 4, engine="phidd", threads=4)
    p = port.run_discovery(x, n, 4, 4, engine="phidd", threads=4)
    assert p["position"] == r["position"]
    assert p["distance"] == pytest.approx(r["distance"], rel=1e-12)


@needs_ref
def test_port_matches_reference_topk_and_profile():
    x = W.random_walk(77, 4000)
    n, k = 48, 5
    r = oracle.ref().topk(x, n, 4, 4, k, threads=4)
    p = port.topk(x, n, 4, 4, k, threads=4)
    assert p["positions"] == r["positions"]
    np.testing.assert_allclose(p["distances"], r["distances"], rtol=1e-12)
    # both equal the exclusion-zone arg-max over the exhaustive nn profile
    nn = port.nn_profile(x, n, threads=4)
    np.testing.assert_allclose(nn, oracle.ref().nn_profile(x, n, threads=4), rtol=1e-12)
    prof = np.where(np.isfinite(nn), nn, -1.0)
    for r_pos, r_dist in zip(p["positions"], p["distances"]):
        i = int(np.argmax(prof))
        assert i + 1 == r_pos and math.sqrt(prof[i]) == pytest.approx(r_dist, rel=1e-12)
        prof[max(0, i - n + 1): i + n] = -1.0


@needs_ref
def test_planted_spike_is_found():  # SPEC.md:453-455, reduced length
    x = W.random_walk(5, 20000).astype(np.float64)
    x[12345] += 100.0
    for c in (oracle.ref(), port):
        r = c.run_discovery(x, 128, 4, 4, engine="phidd", threads=4, chunk=64)
        assert 12345 - 128 < r["position"] - 1 <= 12345


# ---------------------------------------------------------------- golden fixtures
def test_workload_series_are_the_pinned_ones(golden):
    for name, g in golden.items():
        x, at = W.series(g["cfg"])
        assert W.sha256(x) == g["sha256"], name
        assert at == g["anomaly_starts_0based"], name
        w = W.workload(g["cfg"])
        assert (w.m, w.n, w.word_len, w.alphabet, w.k) == (g["m"], g["n"], g["word_len"], g["alphabet"], g["k"])


@pytest.mark.parametrize("cfg", [1, 2])
def test_port_reproduces_golden(golden, cfg):
    g = golden[f"cfg{cfg}"]
    x, _ = W.series(cfg)
    p = port.topk(x, g["n"], g["word_len"], g["alphabet"], g["k"], threads=port.max_threads(), chunk=64)
    assert p["positions"] == g["oracle"]["positions"]
    np.testing.assert_allclose(p["distances"], g["oracle"]["distances"], rtol=1e-12)
