#!/bin/bash
# A/B of variant libraries with a determinism check (final events / acceptance must agree):
#   bash tools/ab2.sh "2 1" 2 base t1 t2      (base = the in-tree default library)
cfgs=$1; reps=$2; shift 2
for c in $cfgs; do for r in $(seq $reps); do for v in "$@"; do
  st=10; [ $c -ge 2 ] && st=5
  lib=paper_1612_00595_b200/_lib/variants/$v.so; [ $v = base ] && lib=paper_1612_00595_b200/_lib/libseis_b200.so
  val=$(env SEIS_LIB=$lib $SEIS_AB_ENV timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline --no-e2e 2>gpurun_out/ab_err_$v.log | python -c "import json,sys; j=json.loads(sys.stdin.read()); d=j['detail']; print('%.0f frac %.4f kernel_ms %.3f final %d acc %.6f launches %d' % (j['value'], j['roofline']['frac'], d['sweep_kernel_ms_per_step'], d['final_events'], d['acceptance'], j['gpu_launches']))")
  echo "config $c $v $val"
done; done; done
