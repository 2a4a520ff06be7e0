#!/bin/bash
# Evidence for config[4] (bounded k, capacity-limited, no e2e leg) and an ncu
# capture of k_phase from the reference's own start (empty hypothesis):
#   gpurun -- bash tools/evidence_c4_empty.sh
O=gpurun_out
for k in 4 1; do
  timeout 900 python bench.py --config 4 --k $k --capacity 60000 --steps 2 --warmup 3 \
    --no-e2e --no-cpu-baseline > $O/bench_c4_k$k.json 2> $O/bench_c4_k$k.err
  rc=$?; echo "k=$k rc=$rc" >> $O/bench_c4.rc
  [ $rc -eq 0 ] && break
done
timeout 300 python bench.py --start empty --steps 4 --warmup 10 --no-cpu-baseline \
  > $O/bench_c1_empty.json 2> $O/bench_c1_empty.err
# k_phase launch 21 = sweep 11 of the chain from empty (two color phases per sweep)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_phase -s 20 -c 1 \
  -o $O/prof_c1_empty python bench.py --start empty --steps 1 --warmup 10 --no-cpu-baseline \
  > $O/ncu_c1_empty.log 2>&1
ls -la $O
