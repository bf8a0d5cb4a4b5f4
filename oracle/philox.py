"""Philox4x32-10 and the Gumbel-max sampler (R24-R25).

The paper says only that branches are produced by stochastic sampling
and fixes no generator.  Reading R25: a counter-based generator keyed by
(request, branch, step) so a branch's tokens do not depend on scheduling.

Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11): 10 rounds of
    (hi0, lo0) = mulhilo(0xD2511F53, c0);  (hi1, lo1) = mulhilo(0xCD9E8D57, c2)
    c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
with the key bumped by (0x9E3779B9, 0xBB67AE85) between rounds.

Sampler: for vocab entry v at decode step s of branch b of request rid,
    counter = (v >> 2, s, rid & 0xffffffff, b),  key = (seed_lo, seed_hi)
    w = philox(counter, key)[v & 3]
    u = ((w >> 8) + 0.5) * 2^-24          in (0, 1)
    G = -ln(-ln u)
    y = argmax_v (logit_v / tau + G_v), ties -> lowest v;  tau = 0 -> argmax logit.

Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def philox4x32_10(ctr, key):
    """Vectorised over numpy arrays of counters: ctr is a tuple of 4 uint arrays (or ints)."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & MASK for c in ctr)
    k0 = np.uint64(key[0] & MASK)
    k1 = np.uint64(key[1] & MASK)
    for r in range(10):
        if r > 0:
            k0 = np.uint64((int(k0) + W0) & MASK)
            k1 = np.uint64((int(k1) + W1) & MASK)
        p0 = np.uint64(M0) * c0
        p1 = np.uint64(M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(MASK)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(MASK)
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0), lo1, (hi0 ^ c3 ^ k1), lo0
    return tuple(x.astype(np.uint32) for x in (c0, c1, c2, c3))


def sampler_words(vocab: int, step: int, request_id: int, branch: int, seed: int) -> np.ndarray:
    """The 32-bit Philox word used for every vocab entry v (O4)."""
    v = np.arange(vocab, dtype=np.uint64)
    ctr = (v >> np.uint64(2), np.full_like(v, step), np.full_like(v, request_id & MASK),
           np.full_like(v, branch))
    words = np.stack(philox4x32_10(ctr, (seed & MASK, (seed >> 32) & MASK)), axis=0)  # [4, V]
    return words[(v & np.uint64(3)).astype(np.int64), np.arange(vocab)]


def gumbel_noise(vocab: int, step: int, request_id: int, branch: int, seed: int) -> np.ndarray:
    w = sampler_words(vocab, step, request_id, branch, seed).astype(np.float64)
    u = (np.floor(w / 256.0) + 0.5) * 2.0 ** -24
    return -np.log(-np.log(u))


def sample(logits: np.ndarray, step: int, request_id: int, branch: int, seed: int,
           tau: float, eos_id: int = -1, forced_len: int = 0) -> int:
    """One token y_s (O4).  Scripted mode: EOS is excluded unless s == forced_len,
    at which step y_s = eos."""
    if forced_len > 0 and step == forced_len:
        return int(eos_id)
    x = np.asarray(logits, dtype=np.float64)
    if tau > 0:
        x = x / tau + gumbel_noise(len(x), step, request_id, branch, seed)
    else:
        x = x.copy()
    if forced_len > 0 and 0 <= eos_id < len(x):
        x[eos_id] = -np.inf
    return int(np.argmax(x))        # numpy argmax returns the lowest index among ties
