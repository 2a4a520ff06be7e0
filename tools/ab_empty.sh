#!/bin/bash
# A/B of alternative builds from the empty start (config[1]): ab_empty.sh reps lib1 lib2 ...
reps=$1; shift
for r in $(seq $reps); do for v in "$@"; do
  val=$(SEIS_LIB=paper_1612_00595_b200/_lib/variants/$v.so timeout 300 python bench.py --start empty --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('%.0f %.4f' % (j['value'], j['roofline']['frac']))")
  echo "empty config 1 $v $val"
done; done
