"""Sweep split-K / tile shape of the tcgen05 GEMM on the C2 decode shapes (M = 512 rows).

    SART_GEMM_BENCH_COPIES=8 SWEEP_TILES=128x128,128x256 python tools/gemm_sweep.py o down
SART_GEMM_BENCH_COPIES cycles over copies of the weights so they stream from HBM as in a step."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SART_GEMM_BENCH_REPS", "200")
from paper_2505_13326_b200.sart import debug_gemm  # noqa: E402

rng = np.random.default_rng(0)
shapes = {"empty1": (128, 128, 64), "empty148": (512, 4736, 64), "o": (512, 1536, 1536), "down": (512, 1536, 8960),
          "qkv": (512, 2048, 1536), "gateup": (512, 17920, 1536)}
only = sys.argv[1:] or list(shapes)
for name, (M, N, K) in shapes.items():
    if name not in only:
        continue
    A = rng.integers(0, 1 << 14, size=(M, K), dtype=np.uint16)
    B = rng.integers(0, 1 << 14, size=(N, K), dtype=np.uint16)
    tiles = os.environ.get("SWEEP_TILES", "128x128,128x256,256x128,256x256")
    for bm, bn in [tuple(int(v) for v in t.split("x")) for t in tiles.split(",")]:
        for S in (1, 2, 3, 4, 6, 8):
            if S > max(1, K // 128):
                continue
            if name == "gateup" and S > 1:
                continue
            print(name, flush=True)
            try:
                debug_gemm(A, B, mode=2 if name == "gateup" and bn == 256 else 0, splits=S, bn=bn, bm=bm)
            except Exception as e:
                print("fail", e)
