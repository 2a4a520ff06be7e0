#!/bin/bash
# speculation depth sweep (SEIS_SPEC) on configs 1 and 2
for c in 1 2; do for r in 1 2; do for m in 2 3 4; do
  st=10; [ $c -ge 2 ] && st=4
  val=$(SEIS_SPEC=$m timeout 300 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('%.0f %.4f %.3f' % (j['value'], j['roofline']['frac'], j['config']['speculative_discarded_frac']))")
  echo "config $c spec $m $val"
done; done; done
