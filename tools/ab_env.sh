#!/bin/bash
# A/B an environment switch on the C2 bench: tools/ab_env.sh VAR "v1 v2 ..." [rounds]
# prints value and ms_per_step per setting, interleaved rounds to average box drift
VAR=$1; VALS=$2; R=${3:-2}
for r in $(seq $R); do for v in $VALS; do
  env $VAR=$v timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$VAR=$v', round(d['value']), round(d['ms_per_step'],1), round(d['roofline']['frac'],3))"
done; done
