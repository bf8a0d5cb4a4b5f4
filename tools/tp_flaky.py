"""Debug: repeat the in-process TP=2 group of test_tp2_two_processes_ipc and compare every
repetition with the fp64 oracle and with each other (determinism of the exchange)."""
import os
import sys

os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from tp_ipc_debug import ref_logits  # noqa: E402


def main(reps=4):
    from test_gpu_tp import tp_call, tp_group
    from synth import SHAPES, Request, gen_prompt, gen_weights
    from paper_2505_13326_b200 import DBG_LOGITS, DBG_ROWIDS
    shape = SHAPES["small"]
    weights = gen_weights(shape, "bf16", std=0.02, root_seed=3)
    ft = np.random.default_rng(5).integers(2, shape.vocab, size=(2, 16)).astype(np.int32)
    prompt = gen_prompt(45, shape.vocab, 1, 30, 30)
    ref = ref_logits(shape, weights, prompt, ft, 16)
    outs = []
    for rep in range(reps):
        eng = tp_group(shape, weights, 2, block_size=16, num_blocks=512, max_rows=16, max_requests=4, max_prompt=64,
                       T=8, cap=16, eos_id=1, enable_forced_tokens=True, debug_capture=True)
        for e in eng:
            e.admit(Request(0, prompt, 2, 2, -1.0, 0, None), forced_tokens=ft)
        got = []
        for w in range(2):
            tp_call(eng, lambda e: e.step(1))
            lg = [e.debug_fetch(DBG_LOGITS) for e in eng]
            ids = eng[0].debug_fetch(DBG_ROWIDS)
            errs = []
            for i, k in enumerate(ids):
                r = ref[(int(k) & 0xFF, 8 * (w + 1))]
                errs.append(float(np.max(np.abs(lg[0][i] - r)) / np.max(np.abs(r))))
            print(f"rep {rep} window {w} ranks equal {np.array_equal(lg[0], lg[1])} rel err {errs}", flush=True)
            got.append(lg[0])
        for e in eng:
            e.close()
        outs.append(np.stack(got))
    for rep in range(1, reps):
        print(f"rep {rep} == rep 0: {np.array_equal(outs[rep], outs[0])} max diff {np.max(np.abs(outs[rep] - outs[0])):.3e}")


if __name__ == "__main__":
    main()
