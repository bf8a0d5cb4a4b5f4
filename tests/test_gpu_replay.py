"""PP2 in model mode: the GPU's own bf16 token and score streams replayed through the oracle.

With record_trace the engine reports, per window row, the tokens it sampled in the window
and the reward the boundary used (PRM head on the GPU's hidden state), plus a 64-bit FNV-1a
hash of the control state after every boundary (include/sart.h, sart_trace_fetch).  The
oracle's Algorithm 1 engine (oracle/engine.py) replays exactly those streams
(ReplaySource: its model is not used) and must reproduce every boundary's state hash and
every finalized record bit for bit -- SURVEY §8(c) PP2, here on free-running bf16 C1-shape
requests (natural EOS, PRM-head pruning), not on scripts.
"""
import numpy as np
import pytest

from gpu_common import compare_results, fnv_state_hash, gpu_engine, oracle_engine
from oracle.engine import ReplaySource
from synth import SHAPES, Request, gen_prompt, gen_weights

pytestmark = pytest.mark.gpu
EOS = 1


def streams(rows):
    tokens, running, final = {}, {}, {}
    for r in rows:
        key = (r["request_id"], r["branch"])
        t = tokens.setdefault(key, [])
        assert len(t) == r["ell_start"], (key, len(t), r["ell_start"])
        t.extend(r["tokens"])
        if r["running"]:
            running.setdefault(key, []).append(np.float32(r["score"]))
        else:
            final[key] = np.float32(r["score"])
    return tokens, running, final


@pytest.mark.parametrize("es", [False, True])
def test_model_mode_bf16_replay(es):
    """C1 shape (tiny, N=4, M=2, cap 64, T=16, alpha 0.5, beta 2), bf16, free-running: >= 100
    windows of GPU streams replayed bit-exactly (and with es_every_step, reading R43)."""
    shape = SHAPES["tiny"]
    weights = gen_weights(shape, "bf16", std=0.08)
    weights["lm_head"][EOS] = weights["lm_head"][EOS] * 4.0     # exact in bf16: EOS within the cap
    T, cap, bs, nb, B = 16, 64, 16, 512, 4
    g = gpu_engine(shape, "bf16", weights, block_size=bs, num_blocks=nb, max_rows=B, max_requests=16, max_prompt=64,
                   T=T, cap=cap, eos_id=EOS, temperature=1.0, sampler_seed=99, record_trace=True,
                   es_every_step=es)
    reqs = [Request(rid, gen_prompt(rid, shape.vocab, EOS, 4, 40), 4, 2, float(np.float32(0.5)), 2, None)
            for rid in range(110)]
    for r in reqs:
        g.admit(r)
    windows = 0
    while True:
        st = g.step(1)
        if st["windows"] == windows:
            break
        windows = st["windows"]
    gres = g.collect()
    rows, hashes = g.trace_fetch()
    g.close()
    assert len(gres) == len(reqs) and windows >= 100 and len(hashes) == windows
    tokens, running, final = streams(rows)
    o = oracle_engine(bs, nb, T, cap, B=B, source=ReplaySource(tokens, running, final), es=es)
    for r in reqs:
        o.admit(r)
    for w in range(windows):
        o.step(1)
        assert fnv_state_hash(o.snapshot()) == hashes[w], f"first diverging boundary: {w}"
    ores = o.collect()
    compare_results(gres, ores, {r.request_id: r.N for r in reqs})
    for a, b in zip(gres, ores):
        assert a["tokens"] == b["tokens"]
    n_pruned = sum(r["num_pruned"] for r in gres)
    n_eos = sum(1 for r in gres for s in r["branch_state"][:4] if s == 2)
    print(f"replayed {windows} windows, {len(rows)} row-windows, pruned {n_pruned}, EOS completions {n_eos}")
    assert n_pruned > 0 and n_eos > 0
