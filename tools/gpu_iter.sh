#!/bin/bash
# Iteration call: kernel parity tests, bench lines per kernel, ncu of the default screen.
#   bash tools/gpu_iter.sh TAG "kernel1 kernel2 ..." [full]
TAG=${1:-it}; KERNELS=${2:-"tcgen05"}; OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests/test_tc_gpu.py tests/test_sweep_gpu.py -x -q > $OUT/pytest_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_$TAG.log
for k in $KERNELS; do
  timeout 300 python bench.py --kernel $k --steps 500 --warmup 10 --no-cpu-baseline --no-e2e > $OUT/bench_${TAG}_${k}_n256.json 2>$OUT/bench_${TAG}_${k}_n256.err
  timeout 300 python bench.py --kernel $k --workload n4096 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $OUT/bench_${TAG}_${k}_n4096.json 2>$OUT/bench_${TAG}_${k}_n4096.err
done
if [ "$3" == "full" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 2 -c 1 -o $OUT/prof_sweep_$TAG -f \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1
fi
echo done
