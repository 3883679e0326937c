#!/bin/bash
# Round profile: launch list + full capture of the dominant kernel (n256 and n4096), tagged.
TAG=${1:-r1}; OUT=gpurun_out; mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 2 -c 1 -o $OUT/prof_sweep_$TAG -f \
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 2 -c 1 -o $OUT/prof_sweep_${TAG}_n4096 -f \
  python bench.py --workload n4096 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_full_${TAG}_n4096.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_${TAG}_n4096.csv \
  python bench.py --workload n4096 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_launch_${TAG}_n4096.log 2>&1
# summarize on the box (small markdown + traffic.json) and keep only the n256 report
python tools/ncu_summary.py $TAG --out $OUT/prof_md --traffic-key n256/tcgen05 \
  --note "bench.py default (256 apps, 32,640 pairs x 100 configs @ 400 W); kernel k_sweep_tc3<1,4,2,3>" > /dev/null 2>&1
python tools/ncu_summary.py ${TAG}_n4096 --rep $OUT/prof_sweep_${TAG}_n4096.ncu-rep --launches $OUT/launches_${TAG}_n4096.csv \
  --out $OUT/prof_md --traffic-key n4096/tcgen05 \
  --note "bench.py --workload n4096 (4,096 apps, 8.4M pairs x 100 configs @ 400 W)" > /dev/null 2>&1
rm -f $OUT/prof_sweep_${TAG}_n4096.ncu-rep
