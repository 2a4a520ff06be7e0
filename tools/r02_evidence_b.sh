#!/bin/bash
# Round-2 evidence, part B (one GPU box): configs [3] (k = 256, chromatic and naive) and [4]
# (k = 64) at their stated parameters, each chromatic line with its e2e leg (their ncu
# captures, at a reduced k, are part of tools/r02_evidence_a.sh)
#   gpurun --timeout 4200 -- bash tools/r02_evidence_b.sh
O=gpurun_out
mkdir -p $O
( time timeout 1500 python bench.py --config 3 --steps 2 --warmup 3 --cpu-seconds 20 > $O/r02_bench_c3.json 2> $O/r02_bench_c3.err ) 2> $O/r02_time_c3.txt
( time timeout 2000 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/r02_bench_c4.json 2> $O/r02_bench_c4.err ) 2> $O/r02_time_c4.txt
( time timeout 900 python bench.py --config 3 --algorithm naive --steps 1 --warmup 3 --no-cpu-baseline > $O/r02_bench_c3_naive.json 2> $O/r02_bench_c3_naive.err ) 2> $O/r02_time_c3n.txt
for f in c3 c4 c3_naive; do echo "== $f"; cut -c1-600 $O/r02_bench_$f.json; tail -3 $O/r02_bench_$f.err; done
cat $O/r02_time_c3.txt $O/r02_time_c4.txt $O/r02_time_c3n.txt
