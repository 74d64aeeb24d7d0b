"""Pins for the oracle's partition planner: Eq. 1 + largest remainder.

Golden values: tests/golden/eq1_weights.txt, apportion.txt, paper_worked_example.txt
(each line cites the PAPER/SPEC passage).  Brute force: an exact-rational Hamilton
apportionment written with fractions.Fraction (independent of the oracle's integer
quantisation) on random inputs.
"""
import os
from fractions import Fraction

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _lines(name):
    with open(os.path.join(GOLD, name)) as f:
        return [ln.strip() for ln in f if ln.strip() and not ln.startswith("#")]


def test_eq1_golden(orc):
    for ln in _lines("eq1_weights.txt"):
        times, weights, _cite = [s.strip() for s in ln.split(";")]
        t = [float(v) for v in times.split()]
        exp = [float(Fraction(v)) for v in weights.split()]
        np.testing.assert_allclose(orc.eq1_weights(t), exp, rtol=1e-15)


def test_eq1_invariants(orc):
    g = np.random.default_rng(1)
    for _ in range(200):
        t = g.uniform(0.01, 100, g.integers(1, 9))
        w = orc.eq1_weights(t)
        assert abs(w.sum() - 1) < 1e-12
        assert np.max(np.abs(w * t - w[0] * t[0])) < 1e-9 * t[0]
        np.testing.assert_allclose(orc.eq1_weights(t * 3.7), w, rtol=1e-12)
    with pytest.raises(orc.OracleError):
        orc.eq1_weights([1.0, 0.0])


def test_paper_worked_example(orc):
    """10 s and 20 s devices -> 2/3, 1/3 -> ~6.67 s, 1.5x."""
    vals = {ln.split()[0]: ln.split()[1:] for ln in _lines("paper_worked_example.txt")}
    t = [float(v) for v in vals["times"]]
    w = orc.eq1_weights(t)
    perf = [max(t) / ti for ti in t]
    assert perf == [float(v) for v in vals["perf_values"]]
    np.testing.assert_allclose(w, [float(Fraction(v)) for v in vals["weights"]], rtol=1e-15)
    par = max(wi * ti for wi, ti in zip(w, t))
    assert par == pytest.approx(float(vals["parallel_time"][0]), rel=1e-9)
    assert min(t) / par == pytest.approx(float(vals["speedup"][0]), rel=1e-12)


def test_apportion_golden(orc):
    for ln in _lines("apportion.txt"):
        times, numk, counts, begins, _cite = [s.strip() for s in ln.split(";")]
        kb, kc, kw = orc.plan([float(v) for v in times.split()], int(numk))
        assert kc.tolist() == [int(v) for v in counts.split()]
        assert kb.tolist() == [int(v) for v in begins.split()]
        assert all(w % 8 == 0 and c <= w < c + 8 for c, w in zip(kc, kw))


def _hamilton_exact(q, num_k):
    """Largest remainder with exact rationals over the quantised throughputs."""
    tot = sum(q)
    quota = [Fraction(num_k * qi, tot) for qi in q]
    cnt = [int(x) for x in quota]
    rem = [x - int(x) for x in quota]
    order = sorted(range(len(q)), key=lambda i: (-rem[i], i))
    for i in order[: num_k - sum(cnt)]:
        cnt[i] += 1
    return cnt


def test_apportion_brute_force(orc):
    g = np.random.default_rng(2)
    for _ in range(500):
        n = int(g.integers(1, 9))
        t = g.uniform(0.5, 5.0, n)
        num_k = int(g.integers(0, 3000))
        kb, kc, kw = orc.plan(t, num_k)
        q = [round(2 ** 20 * (max(t) / ti)) for ti in t]
        assert kc.tolist() == _hamilton_exact(q, num_k)
        assert kc.sum() == num_k
        assert kb.tolist() == [0] + np.cumsum(kc)[:-1].tolist()
        w = orc.eq1_weights(t)
        assert np.all(np.abs(kc - w * num_k) < 1 + 1e-6)                   # quota rule S:L174


def test_paper_net_partitions(orc):
    """Even and uneven maps used by the BASELINE configs (SURVEY §8 notation, App. A.5)."""
    kb, kc, kw = orc.plan([1.0] * 8, 500)
    assert kc.tolist() == [63, 63, 63, 63, 62, 62, 62, 62] and kw.tolist() == [64] * 8
    kb, kc, kw = orc.plan([1.0] * 8, 1500)
    assert kc.tolist() == [188] * 4 + [187] * 4
    t = [1.0, 1.0, 1.05, 1.05, 1.10, 1.10, 1.20, 1.20]
    assert orc.plan(t, 500)[1].tolist() == [68, 68, 64, 64, 62, 62, 56, 56]
    assert orc.plan(t, 1500)[1].tolist() == [203, 203, 193, 193, 185, 185, 169, 169]
    kb, kc, kw = orc.plan([1.0, 1.0, 1.0], 2)        # zero-kernel ranks are legal
    assert kc.tolist() == [1, 1, 0]
