python -m pytest tests -m gpu -x -q > gpurun_out/r02_gpt3.log 2>&1; tail -3 gpurun_out/r02_gpt3.log
bash tools/ab_env.sh "2 1" 2 "SEIS_ORDER=0" "SEIS_ORDER=1"
ncu --set full --clock-control none --import-source on -k regex:k_phase -s 3 -c 1 -o gpurun_out/r02_c2_a python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_a.log 2>&1
tail -2 gpurun_out/ncu_a.log
