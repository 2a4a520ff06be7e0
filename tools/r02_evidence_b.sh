#!/bin/bash
# Round-2 evidence, part B (one GPU box): configs [3] (k = 256, chromatic and naive) and [4]
# (k = 64) at their stated parameters, each chromatic line with its e2e leg; then the DRAM
# bytes and duration of their k_phase launches under ncu (two metrics passes: a --set full
# capture replays a 50 s launch about 40 times)
#   gpurun --timeout 6000 -- bash tools/r02_evidence_b.sh
O=gpurun_out
mkdir -p $O
( time timeout 1500 python bench.py --config 3 --steps 2 --warmup 3 --cpu-seconds 20 > $O/r02_bench_c3.json 2> $O/r02_bench_c3.err ) 2> $O/r02_time_c3.txt
( time timeout 2000 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/r02_bench_c4.json 2> $O/r02_bench_c4.err ) 2> $O/r02_time_c4.txt
( time timeout 1500 python bench.py --config 3 --algorithm naive --steps 1 --warmup 3 --no-cpu-baseline > $O/r02_bench_c3_naive.json 2> $O/r02_bench_c3_naive.err ) 2> $O/r02_time_c3n.txt
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
timeout 1200 ncu --metrics $M --clock-control none -k regex:k_phase -c 4 --csv --log-file $O/r02_ncu_c3.csv python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c3.log 2>&1
timeout 1200 ncu --metrics $M --clock-control none -k regex:k_phase -c 4 --csv --log-file $O/r02_ncu_c4.csv python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c4.log 2>&1
for f in c3 c4 c3_naive; do echo "== $f"; cut -c1-1500 $O/r02_bench_$f.json; tail -3 $O/r02_bench_$f.err; done
cat $O/r02_time_c3.txt $O/r02_time_c4.txt $O/r02_time_c3n.txt
tail -5 $O/r02_ncu_c3.csv $O/r02_ncu_c4.csv
