"""Parity at BASELINE.json's full C2 size, in the launch configuration bench.py times.

C2 (configs[1]): the full 1.5B shape (28 layers, d=1536, GQA 12/2, hd 128, F 8960, V 151936)
in bf16 with host-generated weights, 64 requests x N=8 branches = B = 512 rows resident at
once, prompts U[64, 1024], 64-token blocks, the KV pool sized from free HBM, CUDA-graph
windows -- the same M = 512 GEMM tilings / split-K choices, attention item lists and
sampler grid that bench.py times.  Every branch is teacher-forced (PP1), so
both sides see the same token sequences.

The oracle cannot decode 512 branches of a 1.5B model in fp64 in seconds, so outputs are
SAMPLED: three requests (shortest prompt, longest prompt, one in the middle) x two
branches.  For each sampled row the oracle computes, one by one, the logits at the last
step of each window, the PRM-head score at the boundary and the attention output of
layers {0, 14, 27}; the row-relative error (reading R30) must be <= 2e-2 (bf16,
north_star) for every one of them, logits included -- no allowance.  A second, diagnostic
reference (tests/bf16_emulation.py: fp64 with bf16 rounding at the points any bf16 decode
must round) measures the intrinsic bf16 drift on the same rows; the GPU's mean logits error
must not exceed 1.2x the emulation's (the CUDA path adds no error beyond bf16 storage; two
bf16 paths decorrelate through 28 layers, so a per-row GPU-vs-emulation bound is not a
meaningful check: DESIGN.md R41, profiles/r2_bf16_sensitivity.txt).  For every row (all
512) properties that hold at any size are checked: the logits are finite, and the row order
/ step counts match the teacher-forced schedule.
"""
import numpy as np
import pytest

from bf16_emulation import Bf16Emulation
from gpu_common import gpu_engine, rel_err_rows
from oracle.model import Model
from synth import SHAPES, Request, gen_prompt, gen_weights
from paper_2505_13326_b200 import DBG_ATTN, DBG_LOGITS, DBG_ROWIDS, DBG_SCORES

pytestmark = pytest.mark.gpu

EOS = 1
TOL = 2e-2


def test_c2_full_size_sampled_rows():
    shape = SHAPES["1.5B"]
    N, n_req, T, windows, bs = 8, 64, 8, 2, 64
    steps = T * windows
    layers = [0, shape.n_layers // 2, shape.n_layers - 1]
    weights = gen_weights(shape, "bf16", std=0.02)
    rng = np.random.default_rng(2026)
    prompts = [gen_prompt(rid, shape.vocab, EOS, 64, 1024) for rid in range(n_req)]
    forced = {rid: rng.integers(2, shape.vocab, size=(N, steps)).astype(np.int32) for rid in range(n_req)}
    g = gpu_engine(shape, "bf16", weights, block_size=bs, num_blocks=0, max_rows=n_req * N, max_requests=256,
                   max_prompt=1025, T=T, cap=steps, eos_id=EOS, temperature=1.0, sampler_seed=7,
                   enable_forced_tokens=True, debug_capture=True)
    for rid in range(n_req):
        g.admit(Request(rid, prompts[rid], N, N, -1.0, 0, None), forced_tokens=forced[rid])

    lens = np.array([len(p) for p in prompts])
    order = np.argsort(lens, kind="stable")
    sampled_req = [int(order[0]), int(order[len(order) // 2]), int(order[-1])]
    sampled = [(rid, b) for rid in sampled_req for b in (0, N - 1)]

    gpu = {}
    for w in range(windows):
        st = g.step(1)
        ids = g.debug_fetch(DBG_ROWIDS)
        assert len(ids) == n_req * N, (w, len(ids))          # all 512 rows resident (B = 512)
        lg = g.debug_fetch(DBG_LOGITS)
        assert np.all(np.isfinite(lg)), w
        sc = g.debug_fetch(DBG_SCORES)
        at = {l: g.debug_fetch(DBG_ATTN, l) for l in layers}
        pos = {(int(k) >> 8, int(k) & 0xFF): i for i, k in enumerate(ids)}
        assert sorted(pos) == [(r, b) for r in range(n_req) for b in range(N)]
        for key in sampled:
            i = pos[key]
            gpu[(key, (w + 1) * T)] = dict(logits=lg[i].copy(), prm=float(sc[i]),
                                           attn={l: at[l][i].copy() for l in layers})
        del lg, at
    res = g.collect()
    assert len(res) == n_req
    for r in res:
        assert r["num_completed"] == N and all(x == steps for x in r["branch_len"][:N])
    g.close()

    # ---- oracle: the sampled rows, one by one (batched per step), fp64
    model = Model(shape, weights)
    prefixes = {rid: model.prefill(prompts[rid]) for rid in sampled_req}
    suffix = {key: [{"k": [], "v": []} for _ in range(shape.n_layers)] for key in sampled}
    emu = Bf16Emulation(shape, weights)      # diagnostic: intrinsic bf16 drift at this depth
    e_pre = {rid: emu.prefill(prompts[rid]) for rid in sampled_req}
    e_suf = {key: [[] for _ in range(shape.n_layers)] for key in sampled}
    errs = []
    for s in range(1, steps + 1):
        toks = np.array([prompts[rid][-1] if s == 1 else forced[rid][b, s - 2] for rid, b in sampled])
        posn = np.array([len(prompts[rid]) - 2 + s for rid, _ in sampled])
        dbg = {} if s % T == 0 else None
        z, ref = model.decode(toks, posn, [prefixes[rid] for rid, _ in sampled], [suffix[k] for k in sampled],
                              debug=dbg)
        eref = emu.decode(toks, posn, [e_pre[rid] for rid, _ in sampled], [e_suf[k] for k in sampled])
        if s % T:
            continue
        prm = model.prm_score(z)
        for j, key in enumerate(sampled):
            gv = gpu[(key, s)]
            errs.append(dict(row=key, step=s, logits=rel_err_rows(gv["logits"], ref[j])[0],
                             logits_vs_emu=rel_err_rows(gv["logits"], eref[j])[0],
                             emu_vs_oracle=rel_err_rows(eref[j], ref[j])[0],
                             prm=abs(gv["prm"] - float(prm[j])),
                             attn={l: rel_err_rows(gv["attn"][l], dbg["o"][l][j])[0] for l in layers}))
    for e in errs:
        print("C2 full-size", e)
    print("prompt lengths", [len(prompts[r]) for r in sampled_req])
    worst_attn = max(max(e["attn"].values()) for e in errs)
    assert worst_attn <= TOL, worst_attn
    assert max(e["prm"] for e in errs) <= TOL
    bad = [e for e in errs if e["logits"] > TOL]
    assert not bad, bad
    g_mean = float(np.mean([e["logits"] for e in errs]))
    e_mean = float(np.mean([e["emu_vs_oracle"] for e in errs]))
    print(f"logits row error vs fp64 oracle: GPU mean {g_mean:.4f} max {max(e['logits'] for e in errs):.4f}; "
          f"bf16 emulation mean {e_mean:.4f} max {max(e['emu_vs_oracle'] for e in errs):.4f}")
    assert g_mean <= 1.2 * e_mean, (g_mean, e_mean)
