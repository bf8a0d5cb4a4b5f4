"""Diagnostic second reference for the full-depth bf16 parity test (test infrastructure).

The fp64 oracle (oracle/model.py) is THE reference.  At full depth (28 layers) the bf16
path's intrinsic rounding -- activations rounded to bf16 wherever they become a tensor-core
operand or a KV-cache entry -- accumulates in the residual stream, so the logits of a
correct bf16 implementation drift from the fp64 result by an amount that depends on depth,
not on the implementation.  This module measures that intrinsic drift: it is the same
textbook decoder step as the oracle, in fp64, with bf16
round-to-nearest-even applied at the points where ANY bf16 decode path must round:

  a = bf16(RMSNorm(h) g1)            (GEMM operand)
  q, k, v = bf16(rope(a W^T + b))    (attention operand / KV cache entry)
  o = bf16(attention)                (GEMM operand)
  m = bf16(RMSNorm(h) g2);  act = bf16(SiLU(m Wg^T) (m Wu^T))   (GEMM operands)
  z = bf16(RMSNorm(h) gf)            (LM-head operand)

The residual stream h, accumulations, softmax and logits stay fp64.  It is written from
the decoder definition, not from the CUDA code; it shares nothing with the CUDA path.
"""
import numpy as np

from synth import bf16_round


def _r(x):
    return bf16_round(np.asarray(x, np.float32)).astype(np.float64)


def _rmsnorm(x, g, eps):
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * g


def _rope(x, pos, theta):
    hd = x.shape[-1]
    half = hd // 2
    inv = theta ** (-2.0 * np.arange(half) / hd)
    ang = np.asarray(pos, np.float64)[:, None, None] * inv
    c, s = np.cos(ang), np.sin(ang)
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


class Bf16Emulation:
    def __init__(self, shape, weights):
        self.s = shape
        self.w = {k: np.asarray(v, np.float64) for k, v in weights.items()}

    def _qkv(self, l, h, pos):
        s, w = self.s, self.w
        a = _r(_rmsnorm(h, w[f"l{l}.attn_norm"], s.rms_eps))
        y = a @ w[f"l{l}.wqkv"].T + w[f"l{l}.bqkv"]
        qd, kd = s.n_heads * s.head_dim, s.n_kv_heads * s.head_dim
        q = y[:, :qd].reshape(-1, s.n_heads, s.head_dim)
        k = y[:, qd:qd + kd].reshape(-1, s.n_kv_heads, s.head_dim)
        v = y[:, qd + kd:].reshape(-1, s.n_kv_heads, s.head_dim)
        return _r(_rope(q, pos, s.rope_theta)), _r(_rope(k, pos, s.rope_theta)), _r(v)

    def _post(self, l, h, o):
        s, w = self.s, self.w
        h = h + _r(o.reshape(len(h), -1)) @ w[f"l{l}.wo"].T
        m = _r(_rmsnorm(h, w[f"l{l}.mlp_norm"], s.rms_eps))
        g = m @ w[f"l{l}.wgate"].T
        act = _r(g / (1.0 + np.exp(-g)) * (m @ w[f"l{l}.wup"].T))
        return h + act @ w[f"l{l}.wdown"].T

    def prefill(self, prompt):
        s = self.s
        toks = np.asarray(prompt[:-1], np.int64)
        n = len(toks)
        h = self.w["embed"][toks]
        g = s.n_heads // s.n_kv_heads
        out = []
        for l in range(s.n_layers):
            q, k, v = self._qkv(l, h, np.arange(n))
            o = np.zeros((n, s.n_heads, s.head_dim))
            mask = np.tril(np.ones((n, n), bool))
            for i in range(s.n_heads):
                e = np.where(mask, q[:, i] @ k[:, i // g].T / np.sqrt(s.head_dim), -np.inf)
                p = np.exp(e - e.max(1, keepdims=True))
                o[:, i] = (_r(p) @ v[:, i // g]) / p.sum(1, keepdims=True)
            out.append((k, v))
            h = self._post(l, h, o)
        return out

    def decode(self, tokens, positions, prefixes, suffixes):
        """suffixes[r]: per-layer list of (k, v) appended in place."""
        s = self.s
        g = s.n_heads // s.n_kv_heads
        h = self.w["embed"][np.asarray(tokens, np.int64)]
        for l in range(s.n_layers):
            q, k, v = self._qkv(l, h, positions)
            o = np.zeros((len(h), s.n_heads, s.head_dim))
            for r in range(len(h)):
                suffixes[r][l].append((k[r], v[r]))
                K = np.concatenate([prefixes[r][l][0], np.stack([x[0] for x in suffixes[r][l]])])
                V = np.concatenate([prefixes[r][l][1], np.stack([x[1] for x in suffixes[r][l]])])
                for i in range(s.n_heads):
                    e = K[:, i // g] @ q[r, i] / np.sqrt(s.head_dim)
                    p = np.exp(e - e.max())
                    o[r, i] = (_r(p) @ V[:, i // g]) / p.sum()
            h = self._post(l, h, o)
        z = _r(_rmsnorm(h, self.w["final_norm"], s.rms_eps))
        return z @ self.w["lm_head"].T
