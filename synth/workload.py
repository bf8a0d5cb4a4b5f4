"""Seeded synthetic workload generators (inputs only; no SART arithmetic).

Recipe:

* Every stream is NumPy PCG64 seeded with
  ``SeedSequence([root_seed, crc32(label), request_id])``,
  root seed 0x5A27 unless a test says otherwise.
* Model shapes: the attention dims named in BASELINE.json configs; FFN width,
  vocab and RoPE theta are the public Qwen2.5 shapes (SURVEY §8 shape table).
* Weights: N(0, std^2) drawn in fp32 then rounded to bf16 (round-to-nearest-
  even) for the bf16 mode; RMSNorm gains 1 + N(0, 0.1^2); biases N(0, std^2).
  The same arrays feed the oracle (upcast to fp64) and the GPU (as a blob).
* Prompts: uniform token ids in [0, V) excluding EOS.
* Branch lengths: lognormal, median cap/2, sigma_log 0.5, clamped to
  [max(1, cap/32), cap], or uniform on an integer range.
* Labels: p_correct ~ Beta(4, 2) per request; label 0 w.p. p_correct else
  uniform in {1..4}, independent of length.
* Rewards: final ~ N(0.8, 0.1) if correct else N(0.4, 0.15), clipped to [0,1];
  the value at the k-th boundary (l = (k+1)T) is final + N(0, 0.15 (1 - l/len))
  clipped.
* Arrivals: exponential gaps (Poisson process).
"""
from __future__ import annotations

import dataclasses
import zlib
from typing import Dict, List, Optional

import numpy as np

ROOT_SEED = 0x5A27

__all__ = [
    "ROOT_SEED", "ModelShape", "SHAPES", "stream", "bf16_round", "bf16_bits",
    "bits_to_f32", "weight_names", "weight_shapes", "gen_weights", "pack_blob",
    "gen_prompt", "gen_script", "gen_requests", "gen_arrivals", "Request",
    "Script",
]


@dataclasses.dataclass(frozen=True)
class ModelShape:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    d_ff: int
    vocab: int
    rope_theta: float = 1.0e6
    rms_eps: float = 1.0e-6

    @property
    def qkv_dim(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    def with_layers(self, n_layers: int) -> "ModelShape":
        return dataclasses.replace(self, name=f"{self.name}-L{n_layers}", n_layers=n_layers)


SHAPES: Dict[str, ModelShape] = {
    # BASELINE.json configs[0]: 2 layers, d=256, 4 heads, vocab 512
    "tiny": ModelShape("tiny", 2, 256, 4, 4, 64, 1024, 512),
    # test-only GQA shape (g=4, hd=128) small enough for the fp64 oracle
    "small": ModelShape("small", 2, 512, 8, 2, 128, 1024, 2048),
    # BASELINE.json configs[1]: 28 layers, d=1536, GQA 12/2, hd 128
    "1.5B": ModelShape("1.5B", 28, 1536, 12, 2, 128, 8960, 151936),
    # BASELINE.json configs[2,3]: 28 layers, d=3584, GQA 28/4
    "7B": ModelShape("7B", 28, 3584, 28, 4, 128, 18944, 152064),
    # BASELINE.json configs[4]: 48 layers, d=5120, GQA 40/8
    "14B": ModelShape("14B", 48, 5120, 40, 8, 128, 13824, 152064),
    # The paper's second model (DeepSeek-R1-Distill-Llama-70B = the Llama-3.3-70B shape:
    # 80 layers, d=8192, GQA 64/8, hd 128, F 28672, V 128256, RoPE theta 5e5).  141 GB of bf16
    # weights: it runs on ONE B200 (TP = 1) with ~30 GB left for the KV pool.
    "70B": ModelShape("70B", 80, 8192, 64, 8, 128, 28672, 128256, rope_theta=5.0e5, rms_eps=1.0e-5),
    # Separate PRM decoders (NEXT row f2).  The PRM reads the policy's tokens, so its vocab is
    # the policy's.  prm-tiny / prm-small pair with tiny / small in tests; PRM-7B is the
    # Qwen2.5-Math-PRM-7B shape (= Qwen2.5-7B) over the 1.5B policy's vocab.
    "prm-tiny": ModelShape("prm-tiny", 3, 384, 6, 2, 64, 768, 512),
    "prm-small": ModelShape("prm-small", 2, 384, 3, 1, 128, 1024, 2048),
    "PRM-7B": ModelShape("PRM-7B", 28, 3584, 28, 4, 128, 18944, 151936),
}


def stream(label: str, request_id: int = 0, root_seed: int = ROOT_SEED) -> np.random.Generator:
    """Named, splittable stream."""
    ss = np.random.SeedSequence([int(root_seed) & 0xFFFFFFFF, zlib.crc32(label.encode()),
                                 int(request_id) & 0xFFFFFFFF, (int(request_id) >> 32) & 0xFFFFFFFF])
    return np.random.Generator(np.random.PCG64(ss))


# ---------------------------------------------------------------- bf16 helpers
def bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit pattern (uint16), round-to-nearest-even (input prep)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return r.astype(np.uint16)


def bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 value, returned as fp32."""
    return bits_to_f32(bf16_bits(x))


# ---------------------------------------------------------------- weights
def weight_names(shape: ModelShape) -> List[str]:
    names = ["embed"]
    for l in range(shape.n_layers):
        names += [f"l{l}.attn_norm", f"l{l}.wqkv", f"l{l}.bqkv", f"l{l}.wo",
                  f"l{l}.mlp_norm", f"l{l}.wgate", f"l{l}.wup", f"l{l}.wdown"]
    names += ["final_norm", "lm_head", "prm_w1", "prm_b1", "prm_w2", "prm_b2"]
    return names


def weight_shapes(shape: ModelShape) -> Dict[str, tuple]:
    d, F, V, qh, hd = shape.d_model, shape.d_ff, shape.vocab, shape.n_heads, shape.head_dim
    out = {"embed": (V, d)}
    for l in range(shape.n_layers):
        out[f"l{l}.attn_norm"] = (d,)
        out[f"l{l}.wqkv"] = (shape.qkv_dim, d)     # nn.Linear layout [out, in]
        out[f"l{l}.bqkv"] = (shape.qkv_dim,)
        out[f"l{l}.wo"] = (d, qh * hd)
        out[f"l{l}.mlp_norm"] = (d,)
        out[f"l{l}.wgate"] = (F, d)
        out[f"l{l}.wup"] = (F, d)
        out[f"l{l}.wdown"] = (d, F)
    out["final_norm"] = (d,)
    out["lm_head"] = (V, d)
    out["prm_w1"] = (d, d)
    out["prm_b1"] = (d,)
    out["prm_w2"] = (2, d)
    out["prm_b2"] = (2,)
    return out


def gen_weights(shape: ModelShape, dtype: str = "bf16", std: float = 0.02,
                root_seed: int = ROOT_SEED) -> Dict[str, np.ndarray]:
    """Random-init weights (fp32 arrays holding bf16-representable values in bf16 mode)."""
    out: Dict[str, np.ndarray] = {}
    shp = weight_shapes(shape)
    for i, name in enumerate(weight_names(shape)):
        g = stream("weights", i, root_seed)
        s = shp[name]
        if name.endswith("norm"):
            a = 1.0 + 0.1 * g.standard_normal(s, dtype=np.float32)
        else:
            a = std * g.standard_normal(s, dtype=np.float32)
        a = a.astype(np.float32)
        if dtype == "bf16":
            a = bf16_round(a)
        out[name] = a
    return out


def pack_blob(shape: ModelShape, weights: Dict[str, np.ndarray], dtype: str = "bf16") -> np.ndarray:
    """Concatenate tensors in ``weight_names`` order, row-major, in the model dtype.

    This is the ``host_weights`` layout documented in include/sart.h.
    Returns a uint16 array (bf16 bits) or a float32 array.
    """
    parts = []
    for name in weight_names(shape):
        a = np.ascontiguousarray(weights[name], dtype=np.float32).ravel()
        parts.append(bf16_bits(a) if dtype == "bf16" else a)
    return np.concatenate(parts)


# ---------------------------------------------------------------- requests
@dataclasses.dataclass
class Script:
    forced_len: np.ndarray      # int32 [N], 1 <= len <= cap
    scores: np.ndarray          # float32 [N, n_bnd]
    final_score: np.ndarray     # float32 [N]
    answer: np.ndarray          # int32 [N]

    @property
    def n_bnd(self) -> int:
        return int(self.scores.shape[1])


@dataclasses.dataclass
class Request:
    request_id: int
    prompt: np.ndarray          # int32 [P]
    N: int
    M: int
    alpha: float                # prune_threshold (float32 value); < 0 disables pruning
    beta: int
    script: Optional[Script] = None
    arrival_ns: int = 0


def gen_prompt(request_id: int, vocab: int, eos_id: int, p_lo: int, p_hi: int,
               root_seed: int = ROOT_SEED) -> np.ndarray:
    g = stream("prompts", request_id, root_seed)
    P = int(g.integers(p_lo, p_hi + 1))
    t = g.integers(0, vocab - 1, size=P)
    t = np.where(t >= eos_id, t + 1, t)   # uniform over [0, V) \ {eos}
    return t.astype(np.int32)


def gen_script(request_id: int, N: int, cap: int, T: int, length: str = "lognormal",
               len_range: Optional[tuple] = None, root_seed: int = ROOT_SEED) -> Script:
    gl = stream("lengths", request_id, root_seed)
    if length == "lognormal":
        lo = max(1, cap // 32)
        x = np.exp(np.log(cap / 2.0) + 0.5 * gl.standard_normal(N))
        forced = np.clip(np.rint(x), lo, cap).astype(np.int32)
    elif length == "uniform":
        lo, hi = len_range if len_range is not None else (1, cap)
        forced = gl.integers(lo, hi + 1, size=N).astype(np.int32)
    else:
        raise ValueError(length)
    gb = stream("labels", request_id, root_seed)
    p_correct = gb.beta(4.0, 2.0)
    correct = gb.random(N) < p_correct
    wrong = gb.integers(1, 5, size=N)
    answer = np.where(correct, 0, wrong).astype(np.int32)
    gs = stream("scores", request_id, root_seed)
    final = np.where(correct, gs.normal(0.8, 0.1, N), gs.normal(0.4, 0.15, N))
    final = np.clip(final, 0.0, 1.0)
    n_bnd = max(1, -(-cap // T))
    t = (np.arange(n_bnd)[None, :] + 1) * T
    sig = 0.15 * np.clip(1.0 - t / forced[:, None], 0.0, None)
    sc = np.clip(final[:, None] + sig * gs.standard_normal((N, n_bnd)), 0.0, 1.0)
    return Script(forced, sc.astype(np.float32), final.astype(np.float32), answer)


def gen_requests(n: int, shape: ModelShape, N: int, M: int, alpha: float, beta: int,
                 cap: int, T: int, eos_id: int, p_range=(64, 1024), scripted: bool = True,
                 length: str = "lognormal", len_range=None, first_id: int = 0,
                 root_seed: int = ROOT_SEED) -> List[Request]:
    reqs = []
    for i in range(n):
        rid = first_id + i
        prompt = gen_prompt(rid, shape.vocab, eos_id, p_range[0], p_range[1], root_seed)
        sc = gen_script(rid, N, cap, T, length, len_range, root_seed) if scripted else None
        reqs.append(Request(rid, prompt, N, M, float(np.float32(alpha)), beta, sc))
    return reqs


def gen_arrivals(n: int, rate_per_s: float, root_seed: int = ROOT_SEED) -> np.ndarray:
    """Arrival times in ns of a Poisson process (exponential gaps)."""
    g = stream("arrivals", 0, root_seed)
    gaps = g.exponential(1.0 / rate_per_s, size=n)
    return (np.cumsum(gaps) * 1e9).astype(np.int64)
