"""ctypes binding of include/sart.h (argument marshalling only).

Names follow the C-ABI: ``Engine.admit`` -> ``sart_admit``, ``Engine.step`` ->
``sart_step``, ``Engine.collect`` -> ``sart_collect`` ...  No torch types cross the
boundary: device memory, if any, is passed as a plain integer address.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SART_LIB", os.path.join(HERE, "libsart.so"))   # SART_LIB: A/B of build variants

SART_OK, SART_EINVAL, SART_ENOMEM, SART_ECUDA, SART_EFULL, SART_ESTATE, SART_EDUP = 0, -1, -2, -3, -4, -5, -6
SART_BF16, SART_FP32 = 0, 1
SART_ATTN_CASCADE, SART_ATTN_FLAT = 0, 1
(BR_QUEUED, BR_RUNNING, BR_COMPLETED_EOS, BR_COMPLETED_CAP, BR_PRUNED, BR_EARLY_STOPPED,
 BR_DISCARDED) = range(7)
DBG_LOGITS, DBG_TOKENS, DBG_ROWIDS, DBG_SCORES, DBG_ATTN, DBG_Z, DBG_PRM_SCORES = range(7)


class SartError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{msg} ({code})")
        self.code = code


class SartConfig(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
        ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("d_ff", C.c_int32), ("vocab", C.c_int32),
        ("rope_theta", C.c_float), ("rms_eps", C.c_float), ("dtype", C.c_int32),
        ("weight_seed", C.c_uint64), ("weight_std", C.c_float), ("host_weights", C.c_void_p),
        ("block_size", C.c_int32), ("num_blocks", C.c_int64), ("max_rows", C.c_int32),
        ("max_requests", C.c_int32), ("max_prompt", C.c_int32), ("ctl_interval", C.c_int32),
        ("max_new_tokens", C.c_int32), ("eos_id", C.c_int32), ("temperature", C.c_float),
        ("sampler_seed", C.c_uint64), ("select_mode", C.c_int32), ("attn_mode", C.c_int32),
        ("device", C.c_int32), ("stream", C.c_void_p), ("enable_forced_tokens", C.c_int32),
        ("debug_capture", C.c_int32), ("profile", C.c_int32),
        ("prm_n_layers", C.c_int32), ("prm_d_model", C.c_int32), ("prm_n_heads", C.c_int32),
        ("prm_n_kv_heads", C.c_int32), ("prm_head_dim", C.c_int32), ("prm_d_ff", C.c_int32),
        ("prm_weight_seed", C.c_uint64), ("prm_host_weights", C.c_void_p),
        ("kv_pool", C.c_void_p), ("kv_pool_bytes", C.c_size_t), ("es_every_step", C.c_int32),
        ("record_trace", C.c_int32), ("tp_size", C.c_int32), ("tp_rank", C.c_int32),
        ("prefill_chunk", C.c_int32),
    ]


class SartScript(C.Structure):
    _fields_ = [("forced_len", C.POINTER(C.c_int32)), ("scores", C.POINTER(C.c_float)),
                ("final_score", C.POINTER(C.c_float)), ("answer", C.POINTER(C.c_int32)),
                ("n_bnd", C.c_int32), ("forced_tokens", C.POINTER(C.c_int32))]


class SartRequest(C.Structure):
    _fields_ = [("request_id", C.c_int64), ("prompt", C.POINTER(C.c_int32)), ("prompt_len", C.c_int32),
                ("N", C.c_int32), ("M", C.c_int32), ("prune_threshold", C.c_float), ("beta", C.c_int32),
                ("script", C.POINTER(SartScript)), ("arrival_ns", C.c_int64)]


class SartStats(C.Structure):
    _fields_ = [("windows", C.c_int32), ("steps", C.c_int32), ("live_rows", C.c_int32),
                ("queued_branches", C.c_int32), ("queued_requests", C.c_int32),
                ("finalized_total", C.c_int32), ("free_blocks", C.c_int32),
                ("committed_blocks", C.c_int32), ("branch_tokens", C.c_int64)]


class SartResult(C.Structure):
    _fields_ = [("request_id", C.c_int64), ("answer_vote", C.c_int32), ("vote_count", C.c_int32),
                ("chosen_max_reward", C.c_int32), ("answer_max_reward", C.c_int32),
                ("num_completed", C.c_int32), ("num_pruned", C.c_int32), ("num_early_stopped", C.c_int32),
                ("num_discarded_queued", C.c_int32), ("finalize_reason", C.c_int32),
                ("phase_at_end", C.c_int32), ("threshold_at_end", C.c_float),
                ("branch_len", C.c_int32 * 32), ("branch_state", C.c_uint8 * 32),
                ("branch_score", C.c_float * 32), ("t_arrival_ns", C.c_int64), ("t_prefill_ns", C.c_int64),
                ("t_final_ns", C.c_int64), ("window_final", C.c_int32), ("selected_branch", C.c_int32),
                ("tokens_offset", C.c_int64), ("tokens_len", C.c_int32)]


class SartTraceRow(C.Structure):
    _fields_ = [("request_id", C.c_int64), ("branch", C.c_int32), ("window", C.c_int32), ("ell_start", C.c_int32),
                ("n_tokens", C.c_int32), ("running", C.c_int32), ("score", C.c_float), ("tokens_offset", C.c_int64)]


P32 = C.POINTER(C.c_int32)
P64 = C.POINTER(C.c_int64)
PF = C.POINTER(C.c_float)


class SartState(C.Structure):
    _fields_ = [("n_rows", C.c_int32), ("row_request_id", P64), ("row_branch", P32), ("row_ell", P32),
                ("row_nbnd", P32), ("row_table", P32), ("rows_cap", C.c_int32), ("table_cap", C.c_int32),
                ("n_free", C.c_int32), ("free_stack", P32), ("free_cap", C.c_int32), ("committed", C.c_int32),
                ("n_live", C.c_int32), ("live_request_id", P64), ("live_phase", P32),
                ("live_threshold", PF), ("live_max_pruned", P32), ("live_completed", P32),
                ("live_pruned", P32), ("live_prefix", P32), ("live_prefix_n", P32), ("live_cap", C.c_int32),
                ("prefix_cap", C.c_int32)]


class SartProfile(C.Structure):
    _fields_ = [("attn_ms", C.c_double), ("attn_launches", C.c_int64), ("attn_bytes", C.c_double),
                ("kernel_launches", C.c_int64), ("prefill_ms", C.c_double), ("prm_ms", C.c_double),
                ("prm_tokens", C.c_int64), ("prm_passes", C.c_int64), ("h2d_bytes", C.c_int64),
                ("d2h_bytes", C.c_int64), ("first_step_ms_max", C.c_double), ("step_ms_max", C.c_double),
                ("prefix_tc_windows", C.c_int64), ("attn_stream_ms", C.c_double)]


_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libsart.so; raises if it is missing (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not built: run `python -m paper_2505_13326_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(path)
    lib.sart_init.argtypes = [C.POINTER(SartConfig), C.POINTER(C.c_void_p)]
    lib.sart_admit.argtypes = [C.c_void_p, C.POINTER(SartRequest)]
    lib.sart_step.argtypes = [C.c_void_p, C.c_int32, C.POINTER(SartStats)]
    lib.sart_export_counters.argtypes = [C.c_void_p, C.c_void_p]
    lib.sart_collect.argtypes = [C.c_void_p, C.POINTER(SartResult), C.c_int32, P32, P32, C.c_int64]
    lib.sart_destroy.argtypes = [C.c_void_p]
    lib.sart_strerror.argtypes = [C.c_int]
    lib.sart_strerror.restype = C.c_char_p
    lib.sart_last_error.restype = C.c_char_p
    lib.sart_get_state.argtypes = [C.c_void_p, C.POINTER(SartState)]
    lib.sart_debug_fetch.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_size_t, P32]
    lib.sart_get_profile.argtypes = [C.c_void_p, C.POINTER(SartProfile)]
    lib.sart_reset_profile.argtypes = [C.c_void_p]
    lib.sart_set_profile.argtypes = [C.c_void_p, C.c_int32]
    lib.sart_debug_gemm.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_int32, C.c_int32, C.c_int32, C.c_int32]
    lib.sart_debug_prm_plan.argtypes = [P32, P32, C.c_int32, C.c_int32, C.c_int32, P32, C.c_int32, P32, P32, P32,
                                        P32, C.c_int32, P32]
    lib.sart_debug_tp_segments.argtypes = [C.POINTER(SartConfig), C.c_int32, P64, C.c_int32, P32]
    lib.sart_tp_buffer.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.c_void_p]
    lib.sart_tp_connect.argtypes = [C.c_void_p, C.POINTER(C.c_void_p), C.c_void_p]
    lib.sart_trace_fetch.argtypes = [C.c_void_p, C.POINTER(SartTraceRow), C.c_int64, P64, P32, C.c_int64, P64,
                                     C.POINTER(C.c_uint64), C.c_int64, P64]
    for f in ("sart_debug_tp_segments", "sart_tp_buffer", "sart_tp_connect", "sart_trace_fetch", "sart_debug_prm_plan", "sart_init", "sart_admit", "sart_step", "sart_export_counters", "sart_collect", "sart_destroy",
              "sart_get_state", "sart_debug_fetch", "sart_get_profile", "sart_reset_profile", "sart_debug_gemm", "sart_set_profile"):
        getattr(lib, f).restype = C.c_int
    _lib = lib
    return lib


EXPORTED = ["sart_init", "sart_admit", "sart_step", "sart_export_counters", "sart_collect", "sart_destroy",
            "sart_strerror", "sart_last_error", "sart_get_state", "sart_debug_fetch", "sart_get_profile",
            "sart_reset_profile", "sart_debug_gemm", "sart_set_profile", "sart_debug_prm_plan", "sart_trace_fetch",
            "sart_tp_buffer", "sart_tp_connect", "sart_debug_tp_segments"]


def debug_prm_plan(ell_ws, ell, chunk: int, qp: int):
    """sart_debug_prm_plan (host only): returns (segments, qblocks, gathers, chunks) as int
    arrays [k][4] (chunks: tokens, segments, q-blocks, gathers)."""
    lib = load_library()
    ws, el = _i32(ell_ws), _i32(ell)
    n = len(ws)
    cap = 3 * n + 4 * (int(np.sum(el - ws)) // max(1, min(chunk, qp)) + 8) + 64
    out = np.zeros((cap, 4), np.int32)
    ch = np.zeros((int(np.sum(el - ws)) // chunk + n + 2, 4), np.int32)
    ns, nq, ng, nc = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
    _check(lib.sart_debug_prm_plan(ws.ctypes.data_as(P32), el.ctypes.data_as(P32), n, chunk, qp,
                                   out.ctypes.data_as(P32), cap, C.byref(ns), C.byref(nq), C.byref(ng),
                                   ch.ctypes.data_as(P32), len(ch), C.byref(nc)))
    a, b, c = ns.value, nq.value, ng.value
    return out[:a], out[a:a + b], out[a + b:a + b + c], ch[:nc.value]


def debug_tp_segments(shape, tp: int, rank: int, tensor: int):
    """sart_debug_tp_segments (host only): int64 [k][6] {loff, n, cl, cf, c0, goff} records."""
    lib = load_library()
    cfg = SartConfig()
    cfg.n_layers, cfg.d_model, cfg.n_heads = shape.n_layers, shape.d_model, shape.n_heads
    cfg.n_kv_heads, cfg.head_dim, cfg.d_ff, cfg.vocab = shape.n_kv_heads, shape.head_dim, shape.d_ff, shape.vocab
    cfg.tp_size, cfg.tp_rank = tp, rank
    out = np.zeros((8, 6), np.int64)
    n = C.c_int32()
    _check(lib.sart_debug_tp_segments(C.byref(cfg), tensor, out.ctypes.data_as(P64), 8, C.byref(n)))
    return out[: n.value]


def debug_gemm(A_bits: np.ndarray, B_bits: np.ndarray, bias=None, C=None, mode: int = 0, splits: int = 1,
               bn: int = 256, bm: int = 128) -> np.ndarray:
    """sart_debug_gemm: A [M][K], B [N][K] as bf16 bit patterns (uint16).  With splits > 1 the
    result has shape [splits, M, N] (partial products)."""
    lib = load_library()
    A = np.ascontiguousarray(A_bits, np.uint16)
    B = np.ascontiguousarray(B_bits, np.uint16)
    M, K = A.shape
    N = B.shape[0]
    if splits > 1:
        out = np.zeros((splits, M, N), np.float32)
    else:
        out = np.zeros((M, N // 2 if mode == 2 else N), np.float32) if C is None else np.ascontiguousarray(C, np.float32)
    if mode == 1 and C is None:
        raise ValueError("accumulate mode needs C")
    bptr = None
    if bias is not None:
        bias = np.ascontiguousarray(bias, np.float32)
        bptr = bias.ctypes.data
    _check(lib.sart_debug_gemm(M, N, K, A.ctypes.data, B.ctypes.data, bptr, out.ctypes.data, mode, splits, bn, bm))
    return out


def _check(rc: int):
    if rc != SART_OK:
        lib = load_library()
        raise SartError(rc, f"{lib.sart_strerror(rc).decode()}: {lib.sart_last_error().decode()}")


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


class Engine:
    """One sart_ctx on one GPU."""

    def __init__(self, shape, dtype: str = "bf16", *, host_weights: Optional[np.ndarray] = None,
                 weight_seed: int = 0, weight_std: float = 0.02, block_size: int = 64, num_blocks: int = 0,
                 max_rows: int = 0, max_requests: int = 0, max_prompt: int = 0, T: int = 400, cap: int = 4096,
                 eos_id: int = 1, temperature: float = 1.0, sampler_seed: int = 0, select_mode: int = 0,
                 attn_mode: int = SART_ATTN_CASCADE, device: int = 0, stream: int = 0,
                 enable_forced_tokens: bool = False, debug_capture: bool = False, profile: bool = False,
                 prm_shape=None, prm_host_weights: Optional[np.ndarray] = None, prm_weight_seed: int = 0,
                 kv_pool=None, es_every_step: bool = False, record_trace: bool = False, tp=(1, 0),
                 prefill_chunk: int = 0):
        """prm_shape (a synth.ModelShape, vocab = the policy's): the separate PRM decoder of
        row f2; None -> the PRM head on the policy's hidden state.  kv_pool: (device address,
        bytes) of a caller-owned KV pool buffer (e.g. a torch tensor's data_ptr() and nbytes;
        the caller keeps it alive until close()).  tp = (tp_size, tp_rank): tensor parallelism
        (row f4); connect the ranks with tp_buffer() / tp_connect() before the first step."""
        self.lib = load_library()
        self.shape = shape
        self.cap, self.T = cap, T
        cfg = SartConfig()
        cfg.n_layers, cfg.d_model, cfg.n_heads = shape.n_layers, shape.d_model, shape.n_heads
        cfg.n_kv_heads, cfg.head_dim, cfg.d_ff, cfg.vocab = shape.n_kv_heads, shape.head_dim, shape.d_ff, shape.vocab
        cfg.rope_theta, cfg.rms_eps = shape.rope_theta, shape.rms_eps
        cfg.dtype = SART_BF16 if dtype == "bf16" else SART_FP32
        cfg.weight_seed, cfg.weight_std = weight_seed, weight_std
        self._weights = None
        if host_weights is not None:
            self._weights = np.ascontiguousarray(host_weights)
            cfg.host_weights = self._weights.ctypes.data
        cfg.block_size, cfg.num_blocks, cfg.max_rows = block_size, num_blocks, max_rows
        cfg.max_requests, cfg.max_prompt, cfg.ctl_interval = max_requests, max_prompt, T
        cfg.max_new_tokens, cfg.eos_id, cfg.temperature = cap, eos_id, temperature
        cfg.sampler_seed, cfg.select_mode, cfg.attn_mode = sampler_seed, select_mode, attn_mode
        cfg.device, cfg.stream = device, stream or None
        cfg.enable_forced_tokens, cfg.debug_capture = int(enable_forced_tokens), int(debug_capture)
        cfg.profile = int(profile)
        if kv_pool is not None:
            cfg.kv_pool, cfg.kv_pool_bytes = int(kv_pool[0]), int(kv_pool[1])
        cfg.es_every_step, cfg.record_trace = int(es_every_step), int(record_trace)
        cfg.tp_size, cfg.tp_rank = int(tp[0]), int(tp[1])
        cfg.prefill_chunk = int(prefill_chunk)
        self.tp = max(1, int(tp[0]))
        self._prm_weights = None
        if prm_shape is not None:
            if prm_shape.vocab != shape.vocab:
                raise ValueError("the PRM model reads the policy's tokens: vocab must match")
            cfg.prm_n_layers, cfg.prm_d_model, cfg.prm_n_heads = prm_shape.n_layers, prm_shape.d_model, prm_shape.n_heads
            cfg.prm_n_kv_heads, cfg.prm_head_dim, cfg.prm_d_ff = prm_shape.n_kv_heads, prm_shape.head_dim, prm_shape.d_ff
            cfg.prm_weight_seed = prm_weight_seed
            if prm_host_weights is not None:
                self._prm_weights = np.ascontiguousarray(prm_host_weights)
                cfg.prm_host_weights = self._prm_weights.ctypes.data
        h = C.c_void_p()
        _check(self.lib.sart_init(C.byref(cfg), C.byref(h)))
        self._weights = self._prm_weights = None
        self.ctx = h
        self.cfg = cfg

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.sart_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---------------------------------------------------------------- sart_admit
    def admit(self, req, forced_tokens: Optional[np.ndarray] = None, use_script_scores: bool = True,
              use_answers: bool = True, forced_len: bool = True) -> None:
        keep = []
        prompt = _i32(req.prompt)
        keep.append(prompt)
        r = SartRequest()
        r.request_id = req.request_id
        r.prompt = prompt.ctypes.data_as(P32)
        r.prompt_len = len(prompt)
        r.N, r.M = req.N, req.M
        r.prune_threshold = req.alpha
        r.beta = req.beta
        r.arrival_ns = getattr(req, "arrival_ns", 0)
        sc = getattr(req, "script", None)
        if sc is not None or forced_tokens is not None:
            s = SartScript()
            if sc is not None:
                if forced_len and sc.forced_len is not None:
                    fl = _i32(sc.forced_len); keep.append(fl); s.forced_len = fl.ctypes.data_as(P32)
                if use_script_scores:
                    if sc.scores is not None:
                        scores = np.ascontiguousarray(sc.scores, np.float32); keep.append(scores)
                        s.scores = scores.ctypes.data_as(PF)
                        s.n_bnd = scores.shape[1]
                    if sc.final_score is not None:
                        fin = np.ascontiguousarray(sc.final_score, np.float32); keep.append(fin)
                        s.final_score = fin.ctypes.data_as(PF)
                if use_answers and sc.answer is not None:
                    an = _i32(sc.answer); keep.append(an); s.answer = an.ctypes.data_as(P32)
            if forced_tokens is not None:
                ft = _i32(forced_tokens); keep.append(ft); s.forced_tokens = ft.ctypes.data_as(P32)
            keep.append(s)
            r.script = C.pointer(s)
        _check(self.lib.sart_admit(self.ctx, C.byref(r)))

    # ---------------------------------------------------------------- sart_step
    def step(self, max_windows: int = 1) -> Dict[str, int]:
        st = SartStats()
        _check(self.lib.sart_step(self.ctx, max_windows, C.byref(st)))
        return {f: getattr(st, f) for f, _ in SartStats._fields_}

    def export_counters(self, dev_ptr: int) -> None:
        _check(self.lib.sart_export_counters(self.ctx, C.c_void_p(dev_ptr)))

    def counters(self, out):
        """The C1 admission-counter record (sart_export_counters) written into ``out`` -- any
        object exposing ``data_ptr()`` for 16 int32 of device memory on this engine's GPU (a
        ``torch.int32[16]`` for the NCCL all-gather) -- which is returned."""
        self.export_counters(out.data_ptr())
        return out

    # ---------------------------------------------------------------- sart_collect
    def collect(self, cap: int = 4096, tokens_cap: int = 1 << 24) -> List[dict]:
        out: List[dict] = []
        while True:
            res = (SartResult * cap)()
            toks = np.zeros(tokens_cap, np.int32)
            n = C.c_int32()
            rc = self.lib.sart_collect(self.ctx, res, cap, C.byref(n), toks.ctypes.data_as(P32), tokens_cap)
            if rc not in (SART_OK, SART_EFULL):
                _check(rc)
            for i in range(n.value):
                r = res[i]
                N = 32
                d = {f: getattr(r, f) for f, _ in SartResult._fields_
                     if f not in ("branch_len", "branch_state", "branch_score")}
                d["branch_len"] = list(r.branch_len)[:N]
                d["branch_state"] = list(r.branch_state)[:N]
                d["branch_score"] = list(r.branch_score)[:N]
                d["tokens"] = toks[r.tokens_offset:r.tokens_offset + r.tokens_len].tolist()
                out.append(d)
            if rc == SART_OK:
                return out

    # ---------------------------------------------------------------- tensor parallelism
    def tp_buffer(self):
        """sart_tp_buffer: (device address of this rank's receive buffer, 64-byte IPC handle)."""
        p = C.c_void_p()
        h = (C.c_ubyte * 64)()
        _check(self.lib.sart_tp_buffer(self.ctx, C.byref(p), h))
        return p.value, bytes(h)

    def tp_connect(self, ptrs=None, handles=None):
        """sart_tp_connect: every rank's buffer address (ranks of this process) or every
        rank's IPC handle (64 bytes each, rank order; other processes)."""
        if ptrs is not None:
            arr = (C.c_void_p * len(ptrs))(*[C.c_void_p(int(x)) for x in ptrs])
            _check(self.lib.sart_tp_connect(self.ctx, arr, None))
        else:
            blob = b"".join(handles)
            buf = (C.c_ubyte * len(blob)).from_buffer_copy(blob)
            _check(self.lib.sart_tp_connect(self.ctx, None, buf))

    # ---------------------------------------------------------------- PP2 trace
    def trace_fetch(self):
        """sart_trace_fetch: (rows, hashes) recorded since the last call.  rows: dicts with
        request_id, branch, window, ell_start, running, score (fp32) and tokens (this window's)."""
        nr, nt, nh = C.c_int64(), C.c_int64(), C.c_int64()
        rc = self.lib.sart_trace_fetch(self.ctx, None, 0, C.byref(nr), None, 0, C.byref(nt), None, 0, C.byref(nh))
        if rc not in (SART_OK, SART_EFULL):
            _check(rc)
        rows = (SartTraceRow * max(1, nr.value))()
        toks = np.zeros(max(1, nt.value), np.int32)
        hs = np.zeros(max(1, nh.value), np.uint64)
        _check(self.lib.sart_trace_fetch(self.ctx, rows, nr.value, C.byref(nr), toks.ctypes.data_as(P32), nt.value,
                                         C.byref(nt), hs.ctypes.data_as(C.POINTER(C.c_uint64)), nh.value,
                                         C.byref(nh)))
        out = []
        for i in range(nr.value):
            r = rows[i]
            out.append(dict(request_id=r.request_id, branch=r.branch, window=r.window, ell_start=r.ell_start,
                            running=r.running, score=r.score,
                            tokens=toks[r.tokens_offset:r.tokens_offset + r.n_tokens].tolist()))
        return out, [int(h) for h in hs[: nh.value]]

    # ---------------------------------------------------------------- test hooks
    def state(self, rows_cap: int = 4096, table_cap: int = 512, free_cap: int = 1 << 22,
              live_cap: int = 1024, prefix_cap: int = 256) -> dict:
        s = SartState()
        bufs = dict(row_request_id=np.zeros(rows_cap, np.int64), row_branch=np.zeros(rows_cap, np.int32),
                    row_ell=np.zeros(rows_cap, np.int32), row_nbnd=np.zeros(rows_cap, np.int32),
                    row_table=np.zeros(rows_cap * table_cap, np.int32), free_stack=np.zeros(free_cap, np.int32),
                    live_request_id=np.zeros(live_cap, np.int64), live_phase=np.zeros(live_cap, np.int32),
                    live_threshold=np.zeros(live_cap, np.float32), live_max_pruned=np.zeros(live_cap, np.int32),
                    live_completed=np.zeros(live_cap, np.int32), live_pruned=np.zeros(live_cap, np.int32),
                    live_prefix=np.zeros(live_cap * prefix_cap, np.int32), live_prefix_n=np.zeros(live_cap, np.int32))
        for k, v in bufs.items():
            ptype = P64 if v.dtype == np.int64 else (PF if v.dtype == np.float32 else P32)
            setattr(s, k, v.ctypes.data_as(ptype))
        s.rows_cap, s.table_cap, s.free_cap, s.live_cap, s.prefix_cap = rows_cap, table_cap, free_cap, live_cap, prefix_cap
        _check(self.lib.sart_get_state(self.ctx, C.byref(s)))
        n, nl = s.n_rows, s.n_live
        tab = bufs["row_table"][: n * table_cap].reshape(n, table_cap)
        pre = bufs["live_prefix"][: nl * prefix_cap].reshape(nl, prefix_cap)
        return dict(
            rows=[(int(bufs["row_request_id"][i]), int(bufs["row_branch"][i]), int(bufs["row_ell"][i]),
                   int(bufs["row_nbnd"][i])) for i in range(n)],
            tables=[[int(x) for x in tab[i] if x >= 0] for i in range(n)],
            free=bufs["free_stack"][: s.n_free].tolist(), committed=s.committed,
            meta={int(bufs["live_request_id"][i]): (int(bufs["live_phase"][i]), float(bufs["live_threshold"][i]),
                                                    int(bufs["live_max_pruned"][i]), int(bufs["live_completed"][i]),
                                                    int(bufs["live_pruned"][i]),
                                                    [int(x) for x in pre[i][: bufs["live_prefix_n"][i]]])
                  for i in range(nl)})

    def debug_fetch(self, what: int, layer: int = 0) -> np.ndarray:
        sh = self.shape
        n = C.c_int32()
        # query row count first with a tiny fetch
        probe = np.zeros(1 << 16, np.int64)
        _check(self.lib.sart_debug_fetch(self.ctx, DBG_ROWIDS, 0, probe.ctypes.data, probe.nbytes, C.byref(n)))
        rows = n.value
        if what == DBG_ROWIDS:
            return probe[:rows].copy()
        if what == DBG_LOGITS:
            out = np.zeros((rows, sh.vocab), np.float32)
        elif what in (DBG_TOKENS,):
            out = np.zeros(rows, np.int32)
        elif what in (DBG_SCORES, DBG_PRM_SCORES):
            out = np.zeros(rows, np.float32)
        elif what == DBG_ATTN:   # this rank's q heads under tensor parallelism
            out = np.zeros((rows, sh.n_heads // self.tp * sh.head_dim), np.float32)
        elif what == DBG_Z:
            out = np.zeros((rows, sh.d_model), np.float32)
        else:
            raise ValueError(what)
        _check(self.lib.sart_debug_fetch(self.ctx, what, layer, out.ctypes.data, out.nbytes, C.byref(n)))
        return out

    def profile(self) -> dict:
        p = SartProfile()
        _check(self.lib.sart_get_profile(self.ctx, C.byref(p)))
        return {f: getattr(p, f) for f, _ in SartProfile._fields_}

    def reset_profile(self) -> None:
        _check(self.lib.sart_reset_profile(self.ctx))

    def set_profile(self, enable) -> None:
        """False / True (1): events around each attention operator; 2: also between the
        streaming kernel and the merge (attn_stream_ms)."""
        _check(self.lib.sart_set_profile(self.ctx, int(enable)))
