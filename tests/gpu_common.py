"""Helpers shared by the -m gpu parity tests (test infrastructure)."""
import numpy as np

from oracle.engine import Engine as OEngine, EngineConfig, ScriptedSource


def gpu_engine(shape, dtype="bf16", weights=None, **kw):
    from paper_2505_13326_b200 import Engine
    from synth import pack_blob
    blob = pack_blob(shape, weights, dtype) if weights is not None else None
    return Engine(shape, dtype, host_weights=blob, **kw)


def oracle_engine(bs, nb, T, cap, B=1 << 30, eos=1, select=0, source=None, es=False, prefill_chunk=0):
    cfg = EngineConfig(block_size=bs, num_blocks=nb, max_rows=B, T=T, cap=cap, eos_id=eos, select_mode=select,
                       es_every_step=es, prefill_chunk=prefill_chunk)
    return OEngine(cfg, source if source is not None else ScriptedSource(eos))


def norm_oracle_snapshot(s):
    return dict(rows=[tuple(r) for r in s["rows"]], tables=[list(t) for t in s["tables"]], free=list(s["free"]),
                committed=s["committed"],
                meta={k: (v[0], float(np.float32(v[1])), v[2], v[3], v[4], list(v[5])) for k, v in s["meta"].items()})


def norm_gpu_state(s):
    return dict(rows=[tuple(r) for r in s["rows"]], tables=s["tables"], free=s["free"], committed=s["committed"],
                meta={k: (v[0], float(np.float32(v[1])), v[2], v[3], v[4], list(v[5])) for k, v in s["meta"].items()})


def first_diff(a, b):
    for k in a:
        if a[k] != b[k]:
            return k, a[k], b[k]
    return None


RESULT_KEYS = ["request_id", "answer_vote", "vote_count", "chosen_max_reward", "answer_max_reward",
               "num_completed", "num_pruned", "num_early_stopped", "num_discarded_queued", "finalize_reason",
               "phase_at_end", "window_final", "selected_branch"]


def compare_results(gres, ores, N_of, score_tol=0.0):
    assert [r["request_id"] for r in gres] == [r["request_id"] for r in ores]
    for g, o in zip(gres, ores):
        N = N_of[o["request_id"]]
        for k in RESULT_KEYS:
            assert g[k] == o[k], (k, g[k], o[k], o["request_id"])
        assert abs(np.float32(g["threshold_at_end"]) - np.float32(o["threshold_at_end"])) <= score_tol
        assert g["branch_len"][:N] == o["branch_len"][:N]
        assert g["branch_state"][:N] == o["branch_state"][:N]
        gs = np.array(g["branch_score"][:N], np.float32)
        os_ = np.array(o["branch_score"][:N], np.float32)
        assert np.all(np.abs(gs - os_) <= score_tol), (gs, os_)


def rel_err_rows(gpu, ref):
    """max |gpu - ref| / max |ref| per row (SURVEY reading R30)."""
    gpu = np.atleast_2d(np.asarray(gpu, np.float64))
    ref = np.atleast_2d(np.asarray(ref, np.float64))
    return np.max(np.abs(gpu - ref), axis=1) / np.maximum(np.max(np.abs(ref), axis=1), 1e-30)


def fnv_state_hash(snap) -> int:
    """FNV-1a 64 of an oracle snapshot in the byte layout include/sart.h documents for
    sart_trace_fetch (written from that description; shares nothing with the library)."""
    import struct
    h = 1469598103934665603
    buf = bytearray()
    for (rid, b, ell, _nbnd), blocks in zip(snap["rows"], snap["tables"]):
        buf += struct.pack("<qiii", rid, b, ell, len(blocks)) + struct.pack(f"<{len(blocks)}i", *blocks)
    buf += struct.pack("<i", len(snap["free"])) + struct.pack(f"<{len(snap['free'])}i", *snap["free"])
    buf += struct.pack("<q", snap["committed"])
    buf += struct.pack("<i", len(snap["meta"]))
    for rid in sorted(snap["meta"]):
        phase, thr, maxp, nc, np_, pre = snap["meta"][rid]
        buf += struct.pack("<qi", rid, phase) + struct.pack("<f", thr) + struct.pack("<iiii", maxp, nc, np_, len(pre))
        buf += struct.pack(f"<{len(pre)}i", *pre)
    for c in bytes(buf):
        h ^= c
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h
