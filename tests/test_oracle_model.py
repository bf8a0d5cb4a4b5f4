"""Pins for oracle/model.py.

* attention == torch.nn.functional.scaled_dot_product_attention in fp64 (library routine);
  single key -> v; identical keys -> mean(V).
* cascade identity: attention over [prefix ; suffix] equals the LSE merge of the two
  partial attentions (the identity the GPU's cascade kernel relies on).
* RoPE: preserves norms; q(p).k(p') depends only on p - p'.
* Whole decoder (prefill + several decode steps) == an independent torch-fp64 module
  of the same architecture written below (RoPE as complex rotation, SDPA attention).
* PRM head: softmax(...)[1] == sigmoid(l1 - l0).
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as Fnn

from oracle import model as om
from synth import SHAPES, gen_weights, gen_prompt


def test_attention_matches_sdpa():
    rng = np.random.default_rng(0)
    for T in [1, 2, 7, 65]:
        q = rng.standard_normal(64)
        K = rng.standard_normal((T, 64))
        V = rng.standard_normal((T, 64))
        ref = Fnn.scaled_dot_product_attention(torch.tensor(q)[None, None, None], torch.tensor(K)[None, None],
                                               torch.tensor(V)[None, None])[0, 0, 0].numpy()
        assert np.allclose(om.attention(q, K, V), ref, rtol=0, atol=1e-12)


def test_attention_special_cases():
    rng = np.random.default_rng(1)
    q = rng.standard_normal(32)
    v = rng.standard_normal((1, 32))
    assert np.allclose(om.attention(q, rng.standard_normal((1, 32)), v), v[0], atol=0)
    k = np.tile(rng.standard_normal(32), (5, 1))
    V = rng.standard_normal((5, 32))
    assert np.allclose(om.attention(q, k, V), V.mean(axis=0), atol=1e-14)


def test_cascade_lse_merge_identity():
    rng = np.random.default_rng(2)
    hd = 128
    for split in [0, 1, 17, 63, 64]:
        T = 64
        q = rng.standard_normal(hd)
        K = rng.standard_normal((T, hd)) * 2
        V = rng.standard_normal((T, hd))

        def part(Ks, Vs):
            if len(Ks) == 0:
                return np.zeros(hd), -np.inf
            e = Ks @ q / np.sqrt(hd)
            lse = np.log(np.sum(np.exp(e - e.max()))) + e.max()
            return np.exp(e - lse) @ Vs, lse

        oa, la = part(K[:split], V[:split])
        ob, lb = part(K[split:], V[split:])
        m = max(la, lb)
        wa, wb = np.exp(la - m), np.exp(lb - m)
        merged = (wa * oa + wb * ob) / (wa + wb)
        assert np.allclose(merged, om.attention(q, K, V), atol=1e-12)


def test_rope_invariants():
    rng = np.random.default_rng(3)
    q = rng.standard_normal(128)
    k = rng.standard_normal(128)
    for p in [0, 1, 5, 1000, 123456]:
        assert np.isclose(np.linalg.norm(om.rope(q, p, 1e6)), np.linalg.norm(q), rtol=1e-13)
    d = [om.rope(q, p + 7, 1e6) @ om.rope(k, p, 1e6) for p in [0, 3, 100, 5000]]
    assert np.allclose(d, d[0], rtol=1e-10)
    assert np.allclose(om.rope(q, 0, 1e6), q, atol=0)


# ------------------------------------------------------------------ independent torch decoder
class TorchRef:
    """Same architecture, written with torch ops (fp64): linear, complex RoPE, SDPA."""

    def __init__(self, shape, w):
        self.s = shape
        self.w = {k: torch.tensor(v, dtype=torch.float64) for k, v in w.items()}

    def rms(self, x, g):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + self.s.rms_eps) * g

    def rope(self, x, pos):            # x [T, H, hd]; pairs (i, i+hd/2) as complex numbers
        hd = x.shape[-1]
        fr = 1.0 / (self.s.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.float64) / hd))
        ang = pos[:, None].to(torch.float64) * fr[None, :]
        rot = torch.polar(torch.ones_like(ang), ang)[:, None, :]
        c = torch.complex(x[..., : hd // 2], x[..., hd // 2:]) * rot
        return torch.cat([c.real, c.imag], dim=-1)

    def forward(self, toks):
        """Full causal forward over a token sequence; returns logits of every position."""
        s, w = self.s, self.w
        T = len(toks)
        h = w["embed"][torch.tensor(toks)]
        pos = torch.arange(T)
        g = s.n_heads // s.n_kv_heads
        for l in range(s.n_layers):
            a = self.rms(h, w[f"l{l}.attn_norm"])
            y = Fnn.linear(a, w[f"l{l}.wqkv"], w[f"l{l}.bqkv"])
            q, k, v = torch.split(y, [s.n_heads * s.head_dim, s.n_kv_heads * s.head_dim,
                                      s.n_kv_heads * s.head_dim], dim=-1)
            q = self.rope(q.view(T, s.n_heads, s.head_dim), pos)
            k = self.rope(k.view(T, s.n_kv_heads, s.head_dim), pos)
            v = v.view(T, s.n_kv_heads, s.head_dim)
            k, v = k.repeat_interleave(g, dim=1), v.repeat_interleave(g, dim=1)
            o = Fnn.scaled_dot_product_attention(q.transpose(0, 1), k.transpose(0, 1), v.transpose(0, 1),
                                                 is_causal=True).transpose(0, 1).reshape(T, -1)
            h = h + Fnn.linear(o, w[f"l{l}.wo"])
            m = self.rms(h, w[f"l{l}.mlp_norm"])
            h = h + Fnn.linear(Fnn.silu(Fnn.linear(m, w[f"l{l}.wgate"])) * Fnn.linear(m, w[f"l{l}.wup"]),
                               w[f"l{l}.wdown"])
        z = self.rms(h, w["final_norm"])
        return z, Fnn.linear(z, w["lm_head"])


@pytest.mark.parametrize("shape_name,P", [("tiny", 9), ("small", 5), ("tiny", 1)])
def test_decoder_matches_independent_torch(shape_name, P):
    shape = SHAPES[shape_name]
    w = gen_weights(shape, "fp32", std=0.08)
    m = om.Model(shape, w)
    ref = TorchRef(shape, w)
    prompt = gen_prompt(3, shape.vocab, 1, P, P)
    gen = [int(x) for x in np.random.default_rng(4).integers(2, shape.vocab, 6)]
    seq = list(prompt) + gen
    zr, lr = ref.forward(seq)
    prefix = m.prefill(prompt)
    suffix = [{"k": [], "v": []} for _ in range(shape.n_layers)]
    for s in range(1, len(gen) + 1):
        tok = prompt[-1] if s == 1 else gen[s - 2]
        z, logits = m.decode(np.array([tok]), np.array([P - 2 + s]), [prefix], [suffix])
        pos = P - 2 + s
        assert np.allclose(logits[0], lr[pos].numpy(), rtol=0, atol=1e-9 * np.abs(lr[pos].numpy()).max())
        assert np.allclose(z[0], zr[pos].numpy(), atol=1e-10)


def test_prm_head_closed_form():
    shape = SHAPES["tiny"]
    w = gen_weights(shape, "fp32", std=0.08)
    m = om.Model(shape, w)
    z = np.random.default_rng(5).standard_normal((3, shape.d_model))
    hdn = np.maximum(z @ w["prm_w1"].T.astype(np.float64) + w["prm_b1"], 0)
    lg = hdn @ w["prm_w2"].T.astype(np.float64) + w["prm_b2"]
    assert np.allclose(m.prm_score(z), 1.0 / (1.0 + np.exp(-(lg[:, 1] - lg[:, 0]))), atol=1e-14)


def test_causal_attention_equals_per_position_attention():
    rng = np.random.default_rng(9)
    n, hd = 37, 64
    Q, K, V = rng.standard_normal((n, hd)), rng.standard_normal((n, hd)) * 2, rng.standard_normal((n, hd))
    ref = np.stack([om.attention(Q[t], K[: t + 1], V[: t + 1]) for t in range(n)])
    assert np.allclose(om.causal_attention(Q, K, V), ref, atol=1e-12)


# ------------------------------------------------------------------ separate PRM model (row f2)
@pytest.mark.parametrize("shape_name,n", [("prm-tiny", 23), ("prm-small", 9), ("tiny", 1)])
def test_forward_matches_independent_torch(shape_name, n):
    """Model.forward (no cache) == the independent torch module's z at every position."""
    shape = SHAPES[shape_name]
    w = gen_weights(shape, "fp32", std=0.08, root_seed=77)
    seq = gen_prompt(11, shape.vocab, 1, n, n)
    z = om.Model(shape, w).forward(seq)
    zr, _ = TorchRef(shape, w).forward([int(t) for t in seq])
    assert z.shape == (n, shape.d_model)
    assert np.allclose(z, zr.numpy(), rtol=0, atol=1e-10)


def test_prm_model_score_closed_form_and_cache_identity():
    """prm_model_score(seq) = sigmoid(l1 - l0) of the head on the torch module's last z, and
    equals the head on the z the cached path (prefill + decode steps) produces for the same
    last token (a KV cache reproduces the full causal forward exactly)."""
    shape = SHAPES["prm-tiny"]
    w = gen_weights(shape, "fp32", std=0.08, root_seed=78)
    m = om.Model(shape, w)
    prompt = gen_prompt(12, shape.vocab, 1, 7, 7)
    gen = [int(x) for x in np.random.default_rng(6).integers(2, shape.vocab, 5)]
    seq = [int(t) for t in prompt] + gen
    zr, _ = TorchRef(shape, w).forward(seq)
    zl = zr[-1].numpy()
    hdn = np.maximum(zl @ w["prm_w1"].T.astype(np.float64) + w["prm_b1"], 0)
    lg = hdn @ w["prm_w2"].T.astype(np.float64) + w["prm_b2"]
    assert abs(m.prm_model_score(seq) - 1.0 / (1.0 + np.exp(-(lg[1] - lg[0])))) < 1e-12
    pre = m.prefill(prompt)
    suf = [{"k": [], "v": []} for _ in range(shape.n_layers)]
    P = len(prompt)
    for s in range(1, len(gen) + 1):          # decode inputs: prompt[P-1], gen[0..]
        tok = prompt[-1] if s == 1 else gen[s - 2]
        z, _ = m.decode(np.array([tok]), np.array([P - 2 + s]), [pre], [suf])
    # the last decode step consumed gen[-2] at position P+len(gen)-2 == seq[:-1]'s last token
    assert abs(float(m.prm_score(z)[0]) - m.prm_model_score(seq[:-1])) < 1e-12
