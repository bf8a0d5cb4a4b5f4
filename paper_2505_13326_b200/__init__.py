"""B200-native SART multi-branch decode engine (arXiv 2505.13326).

The product is ``libsart.so`` (CUDA kernels for sm_100a + a C++ host orchestrator)
behind the C-ABI in ``include/sart.h``.  This package is only the thin ctypes binding
with the same names (argument marshalling; every step of the hot path runs in the
library's kernels).  There is no CPU fallback: if the library is missing, importing
the binding raises.
"""
from .sart import (SartError, Engine, SartConfig, load_library, SART_BF16, SART_FP32,  # noqa: F401
                   SART_ATTN_CASCADE, SART_ATTN_FLAT, DBG_LOGITS, DBG_TOKENS, DBG_ROWIDS,
                   DBG_SCORES, DBG_ATTN, DBG_Z, DBG_PRM_SCORES, BR_QUEUED, BR_RUNNING, BR_COMPLETED_EOS,
                   BR_COMPLETED_CAP, BR_PRUNED, BR_EARLY_STOPPED, BR_DISCARDED)
