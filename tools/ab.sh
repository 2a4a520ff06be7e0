#!/bin/bash
# A/B of alternative builds (tools/build_variant.sh NAME -DFLAG=...), on the GPU box:
#   bash tools/ab.sh "1 2" 2 base variant
# A/B of variant libraries: ab.sh "configs" reps lib1 lib2 ...
cfgs=$1; reps=$2; shift 2
for c in $cfgs; do for r in $(seq $reps); do for v in "$@"; do
  st=10; [ $c -ge 2 ] && st=4
  val=$(SEIS_LIB=paper_1612_00595_b200/_lib/variants/$v.so timeout 300 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('%.0f %.4f' % (j['value'], j['roofline']['frac']))")
  echo "config $c $v $val"
done; done; done
