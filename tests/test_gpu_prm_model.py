"""Row f2: the separate PRM decoder on the GPU vs the fp64 oracle.

At every boundary the GPU's PRM model reads each row's suffix entries decoded in the window
through its own paged KV cache (prefix prefilled once per request, same block ids as the
policy) and scores the last one.  The oracle scores the same branch with ONE uncached causal
forward over prompt + y_1 .. y_{l-1} (reading R42, oracle/model.py prm_model_score), so the
test checks the incremental paged cache, the virtual [prefix ; suffix] key space of the
tensor-core kernel, the chunking of the pass and the last-entry gather all at once.

Inputs: teacher-forced token streams (PP1) with EOS planted mid-window for some branches;
prompt lengths cover an empty prefix (P = 1), P-1 a multiple of the block size and ragged
prefixes; SART_PRM_CHUNK forces the multi-chunk paths (the pass packs every row's new
entries back to back, so rows straddle chunk boundaries and long rows span several chunks).  Tolerance: abs 2e-2 on the score for bf16, 1e-5 for fp32 (north_star).
"""
import os

import numpy as np
import pytest

from gpu_common import compare_results, gpu_engine
from oracle.engine import Engine as OEngine, EngineConfig, ModelSource
from oracle.model import Model
from synth import SHAPES, Request, gen_prompt, gen_weights, pack_blob
from paper_2505_13326_b200 import DBG_PRM_SCORES, DBG_ROWIDS

pytestmark = pytest.mark.gpu

EOS = 1
TOL = {"bf16": 2e-2, "fp32": 1e-5}


def make_inputs(pol, N, cap, prompt_lens, eos_steps):
    rng = np.random.default_rng(5)
    prompts = [gen_prompt(100 + i, pol.vocab, EOS, L, L) for i, L in enumerate(prompt_lens)]
    forced = {}
    for rid in range(len(prompts)):
        f = rng.integers(2, pol.vocab, size=(N, cap)).astype(np.int32)
        for b in range(N):
            k = eos_steps(rid, b)
            if k:
                f[b, k - 1] = EOS                # y_k = EOS: the branch completes at step k
        forced[rid] = f
    return prompts, forced


def engine(pol, prm, dtype, wp, wm, T, cap, chunk, prompts, **kw):
    if chunk:
        os.environ["SART_PRM_CHUNK"] = str(chunk)
    try:
        return gpu_engine(pol, dtype, wp, block_size=16, num_blocks=1024, max_rows=64, max_requests=16,
                          max_prompt=max(len(p) for p in prompts) + 1, T=T, cap=cap, eos_id=EOS, temperature=1.0,
                          sampler_seed=3, enable_forced_tokens=True, prm_shape=prm,
                          prm_host_weights=pack_blob(prm, wm, dtype), **kw)
    finally:
        os.environ.pop("SART_PRM_CHUNK", None)


CASES = [
    # policy, PRM, dtype, T, cap, SART_PRM_CHUNK
    ("tiny", "prm-tiny", "bf16", 16, 40, None),
    ("tiny", "prm-tiny", "fp32", 16, 40, None),
    ("small", "prm-small", "bf16", 16, 40, None),
    ("small", "prm-small", "fp32", 16, 40, None),
    ("tiny", "prm-tiny", "bf16", 16, 40, 100),     # packed chunks of 100 entries: rows straddle chunks
    ("tiny", "prm-tiny", "fp32", 16, 40, 100),
    ("small", "prm-small", "bf16", 80, 200, 64),   # a row's window entries over two chunks
]


@pytest.mark.parametrize("pol_name,prm_name,dtype,T,cap,chunk", CASES)
def test_prm_model_scores_every_boundary(pol_name, prm_name, dtype, T, cap, chunk):
    pol, prm = SHAPES[pol_name], SHAPES[prm_name]
    std = 0.02 if dtype == "bf16" else 0.05
    wp = gen_weights(pol, dtype, std=std)
    wm = gen_weights(prm, dtype, std=std, root_seed=0x77)
    N = 4
    prompt_lens = [1, 17, 30]
    eos = {(0, 1): 5, (1, 2): T + 3, (2, 0): 2 * T, (2, 3): 1}
    prompts, forced = make_inputs(pol, N, cap, prompt_lens, lambda r, b: eos.get((r, b)))
    g = engine(pol, prm, dtype, wp, wm, T, cap, chunk, prompts)
    for rid, p in enumerate(prompts):
        g.admit(Request(rid, p, N, N, -1.0, 0, None), forced_tokens=forced[rid])
    m = Model(prm, wm)
    worst, seen, w = 0.0, 0, 0
    done = []
    while len(done) < len(prompts):
        g.step(1)
        w += 1
        ids = g.debug_fetch(DBG_ROWIDS)
        sc = g.debug_fetch(DBG_PRM_SCORES)
        for i, k in enumerate(ids):
            rid, b = int(k) >> 8, int(k) & 0xFF
            e = eos.get((rid, b)) or cap
            ell = min(w * T, e, cap)
            seq = [int(t) for t in prompts[rid]] + [int(t) for t in forced[rid][b, : ell - 1]]
            ref = m.prm_model_score(seq)
            worst = max(worst, abs(float(sc[i]) - ref))
            seen += 1
        done += g.collect()
        assert w < 50
    g.close()
    print(f"f2 {pol_name}/{prm_name} {dtype} T={T} chunk={chunk}: {seen} row scores, worst abs err {worst:.2e}")
    assert seen >= len(prompts) * N * (cap // T)
    assert worst <= TOL[dtype], worst


def test_prm_model_control_matches_oracle_engine_fp32():
    """End to end with pruning (alpha = 0.5, beta = 2, M = 2): the GPU's decisions, records
    and scores equal the oracle engine driven by the same teacher-forced tokens and the
    oracle's PRM model (fp32, scores within 1e-5; decisions bit-exact)."""
    pol, prm = SHAPES["tiny"], SHAPES["prm-tiny"]
    wp = gen_weights(pol, "fp32", std=0.05)
    wm = gen_weights(prm, "fp32", std=0.08, root_seed=0x78)    # scores spread over (0, 0.9)
    N, T, cap = 6, 8, 48
    prompts, forced = make_inputs(pol, N, cap, [9, 16, 25, 33],
                                  lambda r, b: (7 + 11 * ((r * N + b) % 5)) if (r + b) % 3 == 0 else None)
    g = engine(pol, prm, "fp32", wp, wm, T, cap, None, prompts)
    cfg = EngineConfig(block_size=16, num_blocks=1024, max_rows=64, T=T, cap=cap, eos_id=EOS, temperature=1.0,
                       sampler_seed=3)
    o = OEngine(cfg, ModelSource(Model(pol, wp), cfg, prm_model=Model(prm, wm), forced_tokens=forced))
    for rid, p in enumerate(prompts):
        req = Request(rid, p, N, 2, float(np.float32(0.05)), 2, None)
        g.admit(req, forced_tokens=forced[rid])
        o.admit(req)
    g.step(100)
    o.step(100)
    gres, ores = g.collect(), o.collect()
    g.close()
    assert len(gres) == len(prompts)
    assert sum(r["num_pruned"] for r in ores) > 0, "workload must exercise pruning"
    compare_results(gres, ores, {rid: N for rid in range(len(prompts))}, score_tol=1e-5)


def test_prm_model_production_tiles_1p5b_shape():
    """The f2 pass with production tile shapes: a 1.5B-shape policy and a 1.5B-shape PRM (hd 128,
    GQA 12/2 -> six q heads per prefill CTA, 4-stage ring), 2 layers each, 64 rows, prompts of
    64-200 tokens in 64-token blocks (multi-page prefixes, ragged tails); 8 sampled rows are
    checked at both boundaries against the uncached oracle forward (bf16, abs 2e-2)."""
    pol = SHAPES["1.5B"].with_layers(2)
    prm = SHAPES["1.5B"].with_layers(2)
    wp = gen_weights(pol, "bf16", std=0.02)
    wm = gen_weights(prm, "bf16", std=0.02, root_seed=0x79)
    N, n_req, T, cap = 4, 16, 16, 32
    prompts = [gen_prompt(300 + i, pol.vocab, EOS, 64, 200) for i in range(n_req)]
    rng = np.random.default_rng(8)
    forced = {rid: rng.integers(2, pol.vocab, size=(N, cap)).astype(np.int32) for rid in range(n_req)}
    g = gpu_engine(pol, "bf16", wp, block_size=64, num_blocks=2048, max_rows=64, max_requests=32, max_prompt=201, T=T,
                   cap=cap, eos_id=EOS, temperature=1.0, sampler_seed=3, enable_forced_tokens=True, prm_shape=prm,
                   prm_host_weights=pack_blob(prm, wm, "bf16"))
    for rid in range(n_req):
        g.admit(Request(rid, prompts[rid], N, N, -1.0, 0, None), forced_tokens=forced[rid])
    m = Model(prm, wm)
    sampled = {(0, 0), (3, 3), (7, 1), (9, 2), (11, 0), (13, 3), (14, 2), (15, 1)}
    worst, seen = 0.0, 0
    for w in (1, 2):
        g.step(1)
        ids = g.debug_fetch(DBG_ROWIDS)
        sc = g.debug_fetch(DBG_PRM_SCORES)
        assert len(ids) == n_req * N
        for i, k in enumerate(ids):
            key = (int(k) >> 8, int(k) & 0xFF)
            if key not in sampled:
                continue
            rid, b = key
            seq = [int(t) for t in prompts[rid]] + [int(t) for t in forced[rid][b, : w * T - 1]]
            worst = max(worst, abs(float(sc[i]) - m.prm_model_score(seq)))
            seen += 1
    g.close()
    print(f"f2 1.5B-shape tiles: {seen} sampled row scores, worst abs err {worst:.2e}")
    assert seen == 2 * len(sampled)
    assert worst <= 2e-2, worst
