"""Lemma 1: the CDF of the M-th order statistic.

    F_{X(M)}(x; N) = sum_{i=M}^{N} C(N, i) F(x)^i (1 - F(x))^(N - i)

P:149 ("the probability of requiring L decoding steps") is read as the
probability of requiring AT MOST L steps (reading R13).

Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

from fractions import Fraction
from math import comb
from typing import Sequence, Union

Number = Union[float, Fraction]


def cdf_order_stat(M: int, N: int, F: Number) -> Number:
    """Lemma 1, written out term by term (exact if F is a Fraction)."""
    if not (1 <= M <= N):
        raise ValueError("need 1 <= M <= N")
    if F < 0 or F > 1:
        raise ValueError("F must lie in [0, 1]")
    total = Fraction(0) if isinstance(F, Fraction) else 0.0
    for i in range(M, N + 1):
        total += comb(N, i) * F ** i * (1 - F) ** (N - i)
    return total


def monotonicity_gap(M: int, N: int, F: Number) -> Number:
    """F_{X(M)}(x; N+1) - F_{X(M)}(x; N) >= 0: 'increasing w.r.t. N'."""
    return cdf_order_stat(M, N + 1, F) - cdf_order_stat(M, N, F)


def discrete_cdf(pmf: Sequence[Fraction]):
    """CDF F(L) = P(X <= L) of a length distribution on {0, 1, ..., len(pmf)-1}."""
    def F(L: int) -> Fraction:
        if L < 0:
            return Fraction(0)
        return sum(pmf[: min(L, len(pmf) - 1) + 1], Fraction(0))
    return F


def expected_order_stat(M: int, N: int, pmf: Sequence[Fraction]) -> Fraction:
    """E[X_(M)] = sum_{L >= 0} (1 - F_{X(M)}(L; N)) for a non-negative integer X."""
    F = discrete_cdf(pmf)
    top = len(pmf) - 1
    return sum((1 - cdf_order_stat(M, N, F(L)) for L in range(0, top + 1)), Fraction(0))
