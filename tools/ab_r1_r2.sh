#!/bin/bash
# Same-box A/B of the round-1 tree (build_ab/r1 = git archive 1f70874, built in place) against
# the current tree: C2 bench line (device value only) and run_config C3 / C5 / C70.
R=$(pwd)
out=gpurun_out/ab_r1_r2.txt
echo "# tree config branch_tok_s ms_per_step attn_frac" > $out
for i in 1 2; do
  for t in build_ab/r1 .; do
    (cd $R/$t && timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 4 --warmup 3 2>/dev/null | tail -1) | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$t c2', round(d['value']), round(d['ms_per_step'],3), d['roofline']['frac'])" >> $out
  done
done
for c in c3 c5 c70; do
  for t in build_ab/r1 . build_ab/r1 .; do
    (cd $R/$t && timeout 900 python tools/run_config.py --config $c --warmup 2 --windows 2 2>/dev/null | tail -1) | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$t $c', round(d['branch_tokens_per_s']), round(d['ms_per_decode_step'],3), d.get('attn_frac_of_6455'))" >> $out
  done
done
cat $out
