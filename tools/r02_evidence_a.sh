#!/bin/bash
# Round-2 evidence, part A (one GPU box): parity tests, smoke, the default bench line
# (config[2]) + reference arm, configs [1] and [0], the launch list and one ncu --set full
# capture of k_phase at config[2]; then ncu captures of configs [3] / [4] at a reduced k
# (the box's ncu wrapper first runs the command without ncu under a 300 s limit, which the
# stated k does not meet: a sweep of config[3] at k = 256 takes 108 s)
#   gpurun --timeout 3300 -- bash tools/r02_evidence_a.sh
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/r02_pytest_gpu.log 2>&1; echo "rc=$?" >> $O/r02_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/r02_smoke.log 2>&1; echo "rc=$?" >> $O/r02_smoke.log
timeout 600 python bench.py > $O/r02_bench_c2.json 2> $O/r02_bench_c2.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > $O/r02_ref_c2.json 2> $O/r02_ref_c2.err
timeout 400 python bench.py --config 1 > $O/r02_bench_c1.json 2> $O/r02_bench_c1.err
timeout 400 python bench.py --config 0 > $O/r02_bench_c0.json 2> $O/r02_bench_c0.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r02_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_phase -s 6 -c 1 -o $O/r02_prof_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c2.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_phase -s 4 -c 1 -o $O/r02_prof_c3 python bench.py --config 3 --k 32 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c3.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_phase -s 4 -c 1 -o $O/r02_prof_c4 python bench.py --config 4 --k 8 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c4.log 2>&1
tail -3 $O/r02_pytest_gpu.log; tail -2 $O/r02_smoke.log; cut -c1-900 $O/r02_bench_c2.json; echo; cut -c1-300 $O/r02_ref_c2.json; echo
tail -2 $O/ncu_c2.log; tail -2 $O/ncu_c3.log; tail -2 $O/ncu_c4.log
ls -la $O | grep -E "ncu-rep|r02_"
