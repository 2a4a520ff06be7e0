#!/bin/bash
# A/B of environment settings on one build, on the GPU box:
#   bash tools/ab_env.sh "2" 3 "SEIS_ORDER=0" "SEIS_ORDER=1"
cfgs=$1; reps=$2; shift 2
for c in $cfgs; do for r in $(seq $reps); do for v in "$@"; do
  st=10; [ $c -ge 2 ] && st=6
  val=$(env $v timeout 300 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('%.0f %.4f %.3f' % (j['value'], j['roofline']['frac'], j['detail']['sweep_kernel_ms_per_step']))")
  echo "config $c [$v] $val"
done; done; done
