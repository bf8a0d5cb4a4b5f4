"""Pins for oracle/philox.py: Random123 known-answer vectors and Gumbel-max statistics."""
import numpy as np

from oracle import philox


def test_philox_kat():
    # Random123 kat_vectors, philox4x32 R=10 (SURVEY §8(c) sampler pin)
    cases = [
        ((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
        ((0xffffffff,) * 4, (0xffffffff, 0xffffffff), (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
        ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
         (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1)),
    ]
    for ctr, key, out in cases:
        got = tuple(int(x) for x in philox.philox4x32_10(ctr, key))
        assert got == out


def test_sampler_word_indexing():
    # word for v is lane v&3 of philox((v>>2, s, rid, b))
    w = philox.sampler_words(10, 3, 77, 2, 0x1234_5678_9ABC)
    for v in range(10):
        ref = philox.philox4x32_10((v >> 2, 3, 77, 2), (0x56789ABC, 0x1234))[v & 3]
        assert int(w[v]) == int(ref)


def test_gumbel_max_matches_softmax():
    """Gumbel-max draws follow softmax(logits / tau): chi-square over 40k draws."""
    logits = np.array([0.3, -1.0, 2.0, 0.0, 1.2, -0.5, 0.9, 0.1])
    tau = 0.8
    p = np.exp(logits / tau)
    p /= p.sum()
    n = 40_000
    counts = np.zeros(len(logits))
    for s in range(1, n + 1):
        counts[philox.sample(logits, s, 5, 1, 42, tau)] += 1
    chi2 = np.sum((counts - n * p) ** 2 / (n * p))
    assert chi2 < 29.9, chi2        # df = 7, p ~ 1e-4


def test_argmax_and_ties_and_forced_eos():
    x = np.array([1.0, 3.0, 3.0, 0.0])
    assert philox.sample(x, 1, 0, 0, 0, 0.0) == 1                     # tau = 0: argmax, lowest tie
    # scripted mode: EOS never sampled before forced_len, exactly at forced_len
    x = np.array([0.0, 50.0, 0.0, 0.0])                               # eos = 1 would win
    assert philox.sample(x, 3, 0, 0, 0, 1.0, eos_id=1, forced_len=5) != 1
    assert philox.sample(x, 5, 0, 0, 0, 1.0, eos_id=1, forced_len=5) == 1


def test_uniform_open_interval():
    w = np.array([0, 0xFFFFFFFF], dtype=np.float64)
    u = (np.floor(w / 256.0) + 0.5) * 2.0 ** -24
    assert 0 < u[0] < u[1] < 1
