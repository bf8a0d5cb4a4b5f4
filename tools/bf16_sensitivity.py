"""Which bf16 rounding points drive the full-depth logits drift?  (diagnostic tool)

The textbook decoder step in fp64 with bf16 round-to-nearest-even applied
only at a chosen set of points, on the C2 shape (1.5B, 28 layers), teacher-forced; prints the
row-relative logits error (reading R30) against the all-fp64 result for each set.  Points:
  a    RMSNorm output feeding QKV          q    rotated q (attention operand)
  kv   rotated k and v (the KV cache)      p    softmax probabilities (PV operand)
  o    attention output (O-proj operand)   m    RMSNorm output feeding gate/up
  act  SwiGLU output (down operand)        z    final-norm state (LM-head operand)
Usage: python tools/bf16_sensitivity.py [steps] [variant,variant,...]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import SHAPES, bf16_round, gen_prompt, gen_weights  # noqa: E402

ALL = ("a", "q", "kv", "p", "o", "m", "act", "z")


def rnd(x, on):
    return bf16_round(np.asarray(x, np.float32)).astype(np.float64) if on else x


def rmsnorm(x, g, eps):
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * g


def rope(x, pos, theta):
    hd = x.shape[-1]
    half = hd // 2
    inv = theta ** (-2.0 * np.arange(half) / hd)
    ang = np.asarray(pos, np.float64)[:, None, None] * inv
    c, s = np.cos(ang), np.sin(ang)
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


class Dec:
    def __init__(self, shape, w, pts):
        self.s, self.w, self.r = shape, w, {k: (k in pts) for k in ALL}

    def qkv(self, l, h, pos):
        s, w, r = self.s, self.w, self.r
        a = rnd(rmsnorm(h, w[f"l{l}.attn_norm"], s.rms_eps), r["a"])
        y = a @ w[f"l{l}.wqkv"].T + w[f"l{l}.bqkv"]
        qd, kd = s.n_heads * s.head_dim, s.n_kv_heads * s.head_dim
        q = y[:, :qd].reshape(-1, s.n_heads, s.head_dim)
        k = y[:, qd:qd + kd].reshape(-1, s.n_kv_heads, s.head_dim)
        v = y[:, qd + kd:].reshape(-1, s.n_kv_heads, s.head_dim)
        return (rnd(rope(q, pos, s.rope_theta), r["q"]), rnd(rope(k, pos, s.rope_theta), r["kv"]), rnd(v, r["kv"]))

    def post(self, l, h, o):
        s, w, r = self.s, self.w, self.r
        h = h + rnd(o.reshape(len(h), -1), r["o"]) @ w[f"l{l}.wo"].T
        m = rnd(rmsnorm(h, w[f"l{l}.mlp_norm"], s.rms_eps), r["m"])
        g = m @ w[f"l{l}.wgate"].T
        act = rnd(g / (1.0 + np.exp(-g)) * (m @ w[f"l{l}.wup"].T), r["act"])
        return h + act @ w[f"l{l}.wdown"].T

    def attn(self, qv, K, V):
        e = K @ qv / np.sqrt(self.s.head_dim)
        p = np.exp(e - e.max())
        return (rnd(p, self.r["p"]) @ V) / p.sum()

    def prefill(self, prompt):
        s = self.s
        toks = np.asarray(prompt[:-1], np.int64)
        n = len(toks)
        h = self.w["embed"][toks]
        g = s.n_heads // s.n_kv_heads
        out = []
        for l in range(s.n_layers):
            q, k, v = self.qkv(l, h, np.arange(n))
            o = np.zeros((n, s.n_heads, s.head_dim))
            for t in range(n):
                for i in range(s.n_heads):
                    o[t, i] = self.attn(q[t, i], k[: t + 1, i // g], v[: t + 1, i // g])
            out.append((k, v))
            h = self.post(l, h, o)
        return out

    def decode(self, toks, pos, pre, suf):
        s = self.s
        g = s.n_heads // s.n_kv_heads
        h = self.w["embed"][np.asarray(toks, np.int64)]
        for l in range(s.n_layers):
            q, k, v = self.qkv(l, h, pos)
            o = np.zeros((len(h), s.n_heads, s.head_dim))
            for r in range(len(h)):
                suf[r][l].append((k[r], v[r]))
                K = np.concatenate([pre[l][0], np.stack([x[0] for x in suf[r][l]])])
                V = np.concatenate([pre[l][1], np.stack([x[1] for x in suf[r][l]])])
                for i in range(s.n_heads):
                    o[r, i] = self.attn(q[r, i], K[:, i // g], V[:, i // g])
            h = self.post(l, h, o)
        z = rnd(rmsnorm(h, self.w["final_norm"], s.rms_eps), self.r["z"])
        return z @ self.w["lm_head"].T


def run(shape, w, pts, prompt, forced, steps):
    d = Dec(shape, w, pts)
    pre = d.prefill(prompt)
    rows = forced.shape[0]
    suf = [[[] for _ in range(shape.n_layers)] for _ in range(rows)]
    for s in range(1, steps + 1):
        toks = [prompt[-1] if s == 1 else forced[b, s - 2] for b in range(rows)]
        lg = d.decode(toks, np.full(rows, len(prompt) - 2 + s), pre, suf)
    return lg


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    shape = SHAPES["1.5B"]
    w = {k: v.astype(np.float64) for k, v in gen_weights(shape, "bf16", std=0.02).items()}
    if os.environ.get("RESID_SCALE"):      # GPT-2 style residual-projection init: W_o, W_down / sqrt(2L)
        f = 1.0 / np.sqrt(2.0 * shape.n_layers)
        for k in list(w):
            if k.endswith(".wo") or k.endswith(".wdown"):
                w[k] = bf16_round((w[k] * f).astype(np.float32)).astype(np.float64)
    prompt = gen_prompt(3, shape.vocab, 1, 64, 1024)[:72]
    forced = np.random.default_rng(2026).integers(2, shape.vocab, size=(2, steps)).astype(np.int32)
    t = time.time()
    ref = run(shape, w, (), prompt, forced, steps)
    print(f"fp64 reference {time.time() - t:.0f}s", flush=True)
    variants = sys.argv[2].split(",") if len(sys.argv) > 2 else \
        ["all", "kv", "kv+p", "kv+q", "kv+a+m", "kv+o", "kv+act", "kv+z", "all-p", "all-q", "all-a-m", "all-o",
         "all-act"]
    for v in variants:
        if v.startswith("all"):
            pts = set(ALL) - set(x for x in v.split("-")[1:])
        else:
            pts = set(v.split("+"))
        lg = run(shape, w, pts, prompt, forced, steps)
        err = np.max(np.abs(lg - ref), axis=1) / np.max(np.abs(ref), axis=1)
        print(f"{v:12s} rel err per row {np.array2string(err, precision=4)}", flush=True)


if __name__ == "__main__":
    main()
