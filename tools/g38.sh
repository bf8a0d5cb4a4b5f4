#!/bin/bash
# LM head + sampler phase 1 fused (GEMM_SAMPLE, SART_FUSED_SAMPLE=1): PP3 parity, control /
# replay with it on, smoke, then the in-graph C2 step A/B (alternating) and a launch list.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SART_FUSED_SAMPLE=1 python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/g38_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/g38_smoke.log
timeout 900 python -m pytest -x -q -s tests/test_gpu_parity.py -k "full_vocab or sampler_matches" > gpurun_out/g38_pp3.log 2>&1; echo pp3 rc=$?; grep -a "PP3\|passed\|failed\|Error" gpurun_out/g38_pp3.log | tail -6
SART_FUSED_SAMPLE=1 timeout 900 python -m pytest -x -q tests/test_gpu_replay.py tests/test_gpu_parity.py -k "replay or sampler_matches or tiny_bf16 or model_mode" > gpurun_out/g38_replay.log 2>&1; echo replay rc=$?; tail -1 gpurun_out/g38_replay.log
for rep in 1 2 3; do for f in 0 1; do
  echo -n "fused=$f "; SART_FUSED_SAMPLE=$f timeout 600 python tools/ablate_c2.py --masks 0 2>&1 | tail -1
done; done
SART_FUSED_SAMPLE=1 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 250000 -c 600 --csv --log-file gpurun_out/g38_launches.csv python tools/prof_c2.py --warm 3 --steps 0 > gpurun_out/g38_launches_run.log 2>&1; echo ncu rc=$?
python tools/launches.py gpurun_out/g38_launches.csv 2>&1 | head -14
