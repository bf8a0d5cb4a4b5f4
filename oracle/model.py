"""Textbook pre-norm decoder, prefix/suffix attention and PRM head in fp64.

Where the method reaches a plain result, this file writes the plain result:

* Attention (prefix KV shared across branches) is ordinary
  softmax attention of the query over the CONCATENATION [prefix ; suffix].
  Cascade splitting and paging are only a faster route to the same number,
  so they do not appear here.
* A decode step ("the decoding phase ... with each step generating only
  one token") is one textbook pre-norm decoder step:

    per layer:
      a = RMSNorm(h) * g1                         (eps = rms_eps)
      [q, k, v] = a W_qkv^T + b_qkv
      q, k <- RoPE rotate-half at position p, inv_freq_i = theta^(-2i/hd)
      k, v appended to the branch suffix
      o_i = sum_t softmax_t(q_i . k_t / sqrt(hd)) v_t   (kv head = i // g)
      h += o W_o^T
      m = RMSNorm(h) * g2;  h += (SiLU(m W_g^T) * (m W_u^T)) W_d^T
    z = RMSNorm(h) * g_f;  logits = z W_lm^T

* Prefill (Alg. 1 L15 "Perform prefilling", "the same as vanilla LLM
  inference"): causal attention over prompt[0 : P-1], which becomes the shared
  prefix; the last prompt token is every branch's first decode input
  (reading R22).
* PRM head (reading R14/R15, stands in for Qwen2.5-Math-PRM-7B):
    score = softmax(ReLU(z W1^T + b1) W2^T + b2)[1]   in [0, 1] (alpha = 0.5)
  "parity unpinned" as a model of the paper's PRM; its arithmetic is pinned
  by tests/test_oracle_model.py.
* Separate PRM model ("a PRM ... evaluates the
  quality of each intermediate step", "evaluated ... every T steps",
  P:320 Qwen2.5-Math-PRM-7B): a second decoder of its own shape with the same
  head.  Its score of a branch is the head applied to the final-norm hidden
  state of the LAST token of the sequence it has read, computed here by one
  full causal forward over that sequence (no cache):
    prm_model_score(seq) = prm_score(forward(seq)[-1])
  Which tokens it reads is reading R42: prompt + y_1 .. y_{l-1}
  for a branch with l generated tokens.

All arithmetic is fp64; weights are the synth arrays (bf16-representable
values) upcast to fp64.  Test infrastructure only (see oracle/__init__.py).
"""
from __future__ import annotations

from typing import Dict, List, Optional

import numpy as np


def rmsnorm(x: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * np.asarray(g, np.float64)


def rope(x: np.ndarray, pos: float, theta: float) -> np.ndarray:
    """Rotate-half RoPE of the last axis (hd) at integer position ``pos``."""
    hd = x.shape[-1]
    half = hd // 2
    i = np.arange(half, dtype=np.float64)
    inv_freq = theta ** (-2.0 * i / hd)
    ang = pos * inv_freq
    c, s = np.cos(ang), np.sin(ang)
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def attention(q: np.ndarray, K: np.ndarray, V: np.ndarray) -> np.ndarray:
    """o = sum_t softmax_t(q . k_t / sqrt(hd)) v_t  for one query vector."""
    hd = q.shape[-1]
    e = (K @ q) / np.sqrt(hd)
    e = e - np.max(e)
    p = np.exp(e)
    p = p / np.sum(p)
    return p @ V


def causal_attention(Q: np.ndarray, K: np.ndarray, V: np.ndarray) -> np.ndarray:
    """Row t attends to keys 0..t: the same softmax as attention(), written as a masked
    matrix (o_t = sum_{j<=t} softmax_j(q_t . k_j / sqrt(hd)) v_j)."""
    n, hd = Q.shape
    E = (Q @ K.T) / np.sqrt(hd)
    E = np.where(np.tril(np.ones((n, n), dtype=bool)), E, -np.inf)
    E = E - E.max(axis=1, keepdims=True)
    Pm = np.exp(E)
    Pm = Pm / Pm.sum(axis=1, keepdims=True)
    return Pm @ V


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


class Model:
    """Weights + the three entry points the engine needs: prefill, decode, prm."""

    def __init__(self, shape, weights: Dict[str, np.ndarray]):
        self.s = shape
        self.w = weights

    def W(self, name: str) -> np.ndarray:
        return self.w[name]

    # -------------------------------------------------------------- layers
    def _qkv(self, l: int, h: np.ndarray, positions: np.ndarray):
        s = self.s
        a = rmsnorm(h, self.W(f"l{l}.attn_norm"), s.rms_eps)
        y = a @ self.W(f"l{l}.wqkv").T.astype(np.float64) + self.W(f"l{l}.bqkv").astype(np.float64)
        qd, kd = s.n_heads * s.head_dim, s.n_kv_heads * s.head_dim
        q = y[:, :qd].reshape(-1, s.n_heads, s.head_dim)
        k = y[:, qd:qd + kd].reshape(-1, s.n_kv_heads, s.head_dim)
        v = y[:, qd + kd:].reshape(-1, s.n_kv_heads, s.head_dim)
        q = np.stack([rope(q[r], positions[r], s.rope_theta) for r in range(len(positions))])
        k = np.stack([rope(k[r], positions[r], s.rope_theta) for r in range(len(positions))])
        return q, k, v

    def _post_attn(self, l: int, h: np.ndarray, o: np.ndarray) -> np.ndarray:
        s = self.s
        h = h + o.reshape(len(h), -1) @ self.W(f"l{l}.wo").T.astype(np.float64)
        m = rmsnorm(h, self.W(f"l{l}.mlp_norm"), s.rms_eps)
        gate = m @ self.W(f"l{l}.wgate").T.astype(np.float64)
        up = m @ self.W(f"l{l}.wup").T.astype(np.float64)
        return h + (silu(gate) * up) @ self.W(f"l{l}.wdown").T.astype(np.float64)

    def final(self, h: np.ndarray):
        z = rmsnorm(h, self.W("final_norm"), self.s.rms_eps)
        logits = z @ self.W("lm_head").T.astype(np.float64)
        return z, logits

    # -------------------------------------------------------------- prefill
    def prefill(self, prompt: np.ndarray) -> List[Dict[str, np.ndarray]]:
        """KV of prompt[0 : P-1] (positions 0..P-2), causal; returns per-layer {'k','v'}
        of shape [P-1, kvh, hd].  P = 1 gives an empty prefix."""
        s = self.s
        P = len(prompt)
        toks = np.asarray(prompt[: P - 1], dtype=np.int64)
        n = len(toks)
        out = []
        if n == 0:
            z = np.zeros((0, s.n_kv_heads, s.head_dim))
            return [{"k": z, "v": z} for _ in range(s.n_layers)]
        h = self.W("embed")[toks].astype(np.float64)
        pos = np.arange(n, dtype=np.float64)
        g = s.n_heads // s.n_kv_heads
        for l in range(s.n_layers):
            q, k, v = self._qkv(l, h, pos)
            o = np.zeros((n, s.n_heads, s.head_dim))
            for i in range(s.n_heads):
                o[:, i] = causal_attention(q[:, i], k[:, i // g], v[:, i // g])
            out.append({"k": k, "v": v})
            h = self._post_attn(l, h, o)
        return out

    # -------------------------------------------------------------- full forward
    def forward(self, tokens) -> np.ndarray:
        """Causal forward of a whole token sequence at positions 0..n-1 without a cache
        (the definition a KV cache reproduces); returns the final-norm hidden states z [n, d]."""
        s = self.s
        toks = np.asarray(tokens, dtype=np.int64)
        n = len(toks)
        h = self.W("embed")[toks].astype(np.float64)
        pos = np.arange(n, dtype=np.float64)
        g = s.n_heads // s.n_kv_heads
        for l in range(s.n_layers):
            q, k, v = self._qkv(l, h, pos)
            o = np.zeros((n, s.n_heads, s.head_dim))
            for i in range(s.n_heads):
                o[:, i] = causal_attention(q[:, i], k[:, i // g], v[:, i // g])
            h = self._post_attn(l, h, o)
        return rmsnorm(h, self.W("final_norm"), s.rms_eps)

    def prm_model_score(self, tokens) -> float:
        """Separate-PRM-model score of a sequence (row f2): head on z of its last token."""
        return float(self.prm_score(self.forward(tokens)[-1])[0])

    # -------------------------------------------------------------- decode
    def decode(self, tokens: np.ndarray, positions: np.ndarray, prefix_kv: List, suffix_kv: List,
               debug: Optional[dict] = None):
        """One decode step for a batch of branches.

        tokens[r], positions[r]: input token and its position (P-2+s).
        prefix_kv[r]: the request's prefill output (shared, read-only).
        suffix_kv[r]: per-layer {'k': list, 'v': list} of the branch; this
        step's k, v are appended (suffix entry s-1).
        Returns (z [n, d], logits [n, V]).
        """
        s = self.s
        n = len(tokens)
        g = s.n_heads // s.n_kv_heads
        h = self.W("embed")[np.asarray(tokens, dtype=np.int64)].astype(np.float64)
        for l in range(s.n_layers):
            q, k, v = self._qkv(l, h, np.asarray(positions, dtype=np.float64))
            o = np.zeros((n, s.n_heads, s.head_dim))
            for r in range(n):
                suf = suffix_kv[r][l]
                suf["k"].append(k[r])
                suf["v"].append(v[r])
                Ks = np.concatenate([prefix_kv[r][l]["k"], np.stack(suf["k"])], axis=0)
                Vs = np.concatenate([prefix_kv[r][l]["v"], np.stack(suf["v"])], axis=0)
                for i in range(s.n_heads):
                    o[r, i] = attention(q[r, i], Ks[:, i // g], Vs[:, i // g])
            if debug is not None:
                debug.setdefault("q", []).append(q)
                debug.setdefault("k", []).append(k)
                debug.setdefault("v", []).append(v)
                debug.setdefault("o", []).append(o.reshape(n, -1))
            h = self._post_attn(l, h, o)
        return self.final(h)

    # -------------------------------------------------------------- PRM head
    def prm_score(self, z: np.ndarray) -> np.ndarray:
        """softmax(ReLU(z W1^T + b1) W2^T + b2)[1] per row."""
        z = np.atleast_2d(np.asarray(z, dtype=np.float64))
        hdn = np.maximum(z @ self.W("prm_w1").T.astype(np.float64) + self.W("prm_b1"), 0.0)
        lg = hdn @ self.W("prm_w2").T.astype(np.float64) + self.W("prm_b2")
        e = np.exp(lg - lg.max(axis=1, keepdims=True))
        return e[:, 1] / e.sum(axis=1)
