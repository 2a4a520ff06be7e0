#!/bin/bash
# Round-end evidence on the GPU box: parity tests, smoke, bench lines, launch list, ncu captures
#   gpurun -- bash tools/final_evidence.sh
# round-end evidence: bench lines for configs 0-4 + reference arm, launch list, ncu captures
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 300 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
SEIS_PROF=1 timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-e2e > /dev/null 2> $O/prof_c1.txt
timeout 400 python bench.py > $O/bench_c1.json 2> $O/bench_c1.err
timeout 400 python bench.py --config 0 > $O/bench_c0.json 2> $O/bench_c0.err
timeout 600 python bench.py --config 2 --steps 5 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 700 python bench.py --config 3 --k 64 --capacity 160000 --steps 2 --warmup 3 --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
timeout 700 python bench.py --config 4 --k 4 --capacity 60000 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 300 python bench.py --start empty --steps 4 --warmup 10 --no-cpu-baseline > $O/bench_c1_empty.json 2> $O/bench_c1_empty.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_c1.json 2> $O/ref_c1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_phase -s 2 -c 1 -o $O/prof_c1 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_phase -s 2 -c 1 -o $O/prof_c2 python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c2.log 2>&1
ls -la $O
