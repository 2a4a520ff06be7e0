#!/bin/bash
# Round-2 evidence, part C (one GPU box): the config[3] lines (k = 256, chromatic with its e2e
# leg, and naive) on the end-of-round build
#   gpurun --timeout 2400 -- bash tools/r02_evidence_c3.sh
O=gpurun_out
( time timeout 1500 python bench.py --config 3 --steps 2 --warmup 3 --cpu-seconds 20 > $O/r02f_bench_c3.json 2> $O/r02f_bench_c3.err ) 2> $O/r02f_time_c3.txt
( time timeout 600 python bench.py --config 3 --algorithm naive --steps 1 --warmup 3 --no-cpu-baseline > $O/r02f_bench_c3_naive.json 2> $O/r02f_bench_c3_naive.err ) 2> $O/r02f_time_c3n.txt
cut -c1-300 $O/r02f_bench_c3.json; cut -c1-300 $O/r02f_bench_c3_naive.json
