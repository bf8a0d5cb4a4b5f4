"""Pins for oracle/orderstats.py and for the early-stop behaviour of oracle/engine.py.

Lemma 1 is checked against exact rationals (tests/golden/lemma1.json,
SPEC S:332-352), its closed-form corners, monotonicity ("increasing w.r.t. N")
and Monte Carlo.  The ENGINE's early stop (the decode time depends only on
the M-th completed branch) is pinned by running it on every script of i.i.d. lengths
and comparing the average stop step with E[X_(M)] (tests/golden/early_stop_expectations.json,
brute-forced independently of oracle/).
"""
import itertools
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import orderstats as os_
from oracle.engine import Engine, EngineConfig, ScriptedSource
from synth import Request, Script

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def frac(p):
    return Fraction(p[0], p[1])


def test_lemma1_golden_values():
    g = json.load(open(os.path.join(GOLD, "lemma1.json")))
    for c in g["cdf"]:
        assert os_.cdf_order_stat(c["M"], c["N"], frac(c["F"])) == frac(c["value"]), c
    for c in g["gap"]:
        assert os_.monotonicity_gap(c["M"], c["N"], frac(c["F"])) == frac(c["value"]), c


def test_lemma1_corners_and_grid():
    # corners 1-(1-F)^N and F^N exactly; monotone in F, M, N on the grid
    Fs = [Fraction(k, 10) for k in range(11)]
    for N in range(1, 17):
        for F in Fs:
            assert os_.cdf_order_stat(1, N, F) == 1 - (1 - F) ** N
            assert os_.cdf_order_stat(N, N, F) == F ** N
        for M in range(1, N + 1):
            vals = [os_.cdf_order_stat(M, N, F) for F in Fs]
            assert all(0 <= v <= 1 for v in vals)
            assert all(a <= b for a, b in zip(vals, vals[1:]))          # non-decreasing in F
            for F in Fs:
                v = os_.cdf_order_stat(M, N, F)
                if M < N:
                    assert os_.cdf_order_stat(M + 1, N, F) <= v          # non-increasing in M
                assert os_.cdf_order_stat(M, N + 1, F) >= v              # non-decreasing in N


def test_lemma1_float_matches_exact():
    for N in range(1, 21):
        for M in range(1, N + 1):
            for k in range(0, 11):
                ex = os_.cdf_order_stat(M, N, Fraction(k, 10))
                fl = os_.cdf_order_stat(M, N, k / 10)
                assert abs(float(ex) - fl) < 1e-12


def test_lemma1_monte_carlo():
    rng = np.random.default_rng(123)
    trials = 100_000
    for M, N, x in [(2, 3, 0.5), (1, 4, 0.2), (4, 8, 0.5), (3, 5, 0.3)]:
        u = np.sort(rng.random((trials, N)), axis=1)
        emp = np.mean(u[:, M - 1] <= x)
        p = os_.cdf_order_stat(M, N, x)
        se = np.sqrt(p * (1 - p) / trials)
        assert abs(emp - p) <= 3 * se + 1e-12, (M, N, x, emp, p)


def test_expected_order_stat_golden():
    g = json.load(open(os.path.join(GOLD, "early_stop_expectations.json")))
    for c in g["cases"]:
        k = int(c["dist"].split("..")[1].rstrip("}"))
        pmf = [Fraction(0)] + [Fraction(1, k)] * k
        assert os_.expected_order_stat(c["M"], c["N"], pmf) == frac(c["E"]), c


def _run_scripted(lengths, M, T, cap, scores=None, alpha=-1.0, beta=0, finals=None, bs=16, nb=4096):
    N = len(lengths)
    nbnd = max(1, -(-cap // T))
    sc = np.zeros((N, nbnd), np.float32) if scores is None else np.asarray(scores, np.float32)
    fin = np.ones(N, np.float32) if finals is None else np.asarray(finals, np.float32)
    script = Script(np.asarray(lengths, np.int32), sc, fin, np.zeros(N, np.int32))
    eng = Engine(EngineConfig(block_size=bs, num_blocks=nb, T=T, cap=cap, eos_id=1),
                 ScriptedSource(1))
    eng.admit(Request(0, np.array([5, 6, 7], np.int32), N, M, alpha, beta, script))
    eng.step(10_000)
    res = eng.collect()
    assert len(res) == 1
    return eng, res[0]


@pytest.mark.parametrize("M,expect", [(1, Fraction(177, 128)), (2, Fraction(269, 128)),
                                      (4, Fraction(463, 128))])
def test_engine_early_stop_matches_lemma1(M, expect):
    """T = 1 (control every step): the finalize step is X_(M) per instance, so the
    mean over all 4^4 scripts equals E[X_(M)] from Lemma 1 exactly."""
    N, k = 4, 4
    pmf = [Fraction(0)] + [Fraction(1, k)] * k
    assert os_.expected_order_stat(M, N, pmf) == expect
    total = 0
    tokens = 0
    for lens in itertools.product(range(1, k + 1), repeat=N):
        eng, r = _run_scripted(list(lens), M, T=1, cap=8)
        stop = r["window_final"] + 1            # one step per window, all rows start at window 0
        assert stop == sorted(lens)[M - 1]
        total += stop
        tokens += eng.branch_tokens
    n = k ** N
    assert Fraction(total, n) == expect
    # tokens per request = sum_{j<M} E[X_(j)] + (N-M+1) E[X_(M)]
    Ej = [os_.expected_order_stat(j, N, pmf) for j in range(1, M + 1)]
    assert Fraction(tokens, n) == sum(Ej[:-1], Fraction(0)) + (N - M + 1) * Ej[-1]


def test_engine_early_stop_with_boundaries():
    """T > 1: control only at boundaries (R8) and a window ends early once no row is
    live (R31): stop = min(ceil(X_(M)/T) T, X_(N)) per instance."""
    N, M, T, k = 4, 2, 3, 6
    for lens in itertools.product(range(1, k + 1), repeat=N):
        eng, r = _run_scripted(list(lens), M, T=T, cap=6)
        xs = sorted(lens)
        expect = min(-(-xs[M - 1] // T) * T, xs[-1])
        assert eng.steps == expect, (lens, eng.steps, expect)
        assert r["num_completed"] >= M
        assert r["num_completed"] == sum(1 for x in lens if x <= expect)
        assert r["num_early_stopped"] == N - r["num_completed"]


def _run_es(lens, M, T, cap):
    """Like _run_scripted, with es_every_step (reading R43)."""
    N = len(lens)
    sc = Script(np.asarray(lens, np.int32), np.zeros((N, 1), np.float32), np.zeros(N, np.float32),
                np.zeros(N, np.int32))
    eng = Engine(EngineConfig(block_size=16, num_blocks=4096, T=T, cap=cap, eos_id=1, es_every_step=True),
                 ScriptedSource(1))
    eng.admit(Request(0, np.array([5, 6], np.int32), N, M, -1.0, 0, sc))
    eng.step(1000)
    res = eng.collect()
    assert len(res) == 1
    return eng, res[0]


@pytest.mark.parametrize("T", [1, 3, 4, 16])
@pytest.mark.parametrize("M,expect", [(1, Fraction(177, 128)), (2, Fraction(269, 128)),
                                      (4, Fraction(463, 128))])
def test_es_every_step_stop_is_order_statistic(M, expect, T):
    """Reading R43 (es_every_step): whatever T, the unfinished branches stop at X_(M), the
    M-th smallest of the N lengths -- per instance exactly -- so over all 4^4
    scripts the mean stop step is E[X_(M)] of Lemma 1, and the decoded tokens are
    sum_{j<M} E[X_(j)] + (N-M+1) E[X_(M)]."""
    N, k = 4, 4
    pmf = [Fraction(0)] + [Fraction(1, k)] * k
    total = tokens = 0
    for lens in itertools.product(range(1, k + 1), repeat=N):
        eng, r = _run_es(list(lens), M, T=T, cap=8)
        xm = sorted(lens)[M - 1]
        for b in range(N):
            if lens[b] <= xm:
                assert r["branch_state"][b] == 2 and r["branch_len"][b] == lens[b]
            else:
                assert r["branch_state"][b] == 5 and r["branch_len"][b] == xm, (lens, b, r["branch_len"])
        assert r["num_completed"] == sum(1 for x in lens if x <= xm)
        total += xm
        tokens += eng.branch_tokens
    n = k ** N
    assert Fraction(total, n) == expect
    Ej = [os_.expected_order_stat(j, N, pmf) for j in range(1, M + 1)]
    assert Fraction(tokens, n) == sum(Ej[:-1], Fraction(0)) + (N - M + 1) * Ej[-1]


def test_es_every_step_trace_B():
    """SURVEY §8(c) trace B under es_every_step: b1 completes at 10, b3 at 25 -> M = 2 is
    reached at step 25, so b0 and b2 stop at l = 25; the request finalizes at the boundary
    of window 1 (step 32) with completions {b1, b3} (vote over those two)."""
    from tests_traces import trace_B_request
    eng = Engine(EngineConfig(block_size=16, num_blocks=17, T=16, cap=64, eos_id=1, es_every_step=True),
                 ScriptedSource(1))
    eng.admit(trace_B_request())
    eng.step(100)
    r = eng.collect()[0]
    assert r["window_final"] == 1
    assert r["branch_state"] == [5, 2, 5, 2]
    assert r["branch_len"] == [25, 10, 25, 25]
    assert (r["num_completed"], r["num_early_stopped"]) == (2, 2)
    assert eng.steps == 25                     # window 1 ends early: nothing live after step 25
    assert sorted(eng.free) == list(range(17))
