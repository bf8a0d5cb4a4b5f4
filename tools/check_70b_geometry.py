import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import dataclasses
from synth import SHAPES, gen_prompt
from test_gpu_parity import run_teacher_forced
sh = dataclasses.replace(SHAPES["70B"].with_layers(1), name="70B-L1-V4096", vocab=4096)
for std in (0.02, 0.01):
    try:
        w = run_teacher_forced(sh, "bf16", [gen_prompt(43, 4096, 1, 70, 70)], N=3, steps=16, bs=64, tol=1.0, std=std, T=8)
        print("non-TP 70B-L1 std", std, w, flush=True)
    except AssertionError as e:
        print("non-TP 70B-L1 std", std, "assert", e, flush=True)
