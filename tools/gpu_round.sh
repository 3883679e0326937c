#!/bin/bash
# One GPU call: parity tests, smoke, bench lines, ncu launch list + full capture
# of the dominant kernel.  Usage (under gpurun): bash tools/gpu_round.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi -L > $OUT/gpu_$TAG.txt 2>&1; nproc >> $OUT/gpu_$TAG.txt; lscpu | head -20 >> $OUT/gpu_$TAG.txt
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py smoke > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 600 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err
timeout 600 python bench.py --workload n4096 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/bench4096_$TAG.json 2> $OUT/bench4096_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-subresults > $OUT/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 2 -c 1 -o $OUT/prof_sweep_$TAG -f \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-subresults > $OUT/ncu_full_$TAG.log 2>&1

timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 1 -c 1 -o $OUT/prof_sweep4096_$TAG -f \
  python bench.py --workload n4096 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-subresults > $OUT/ncu_full4096_$TAG.log 2>&1
echo done4096
