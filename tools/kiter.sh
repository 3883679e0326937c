#!/bin/bash
# Kernel iteration on the GPU box: parity of the screens + bench lines (no e2e / cpu).
#   bash tools/kiter.sh TAG [extra pytest args]
TAG=${1:-it}; OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_tc_gpu.py tests/test_soundness_gpu.py tests/test_sweep_gpu.py -x -q ${@:2} > $OUT/k_$TAG.log 2>&1; echo "rc=$?" >> $OUT/k_$TAG.log
for w in n256 n4096 n1024x5; do
  timeout 300 python bench.py --workload $w --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-subresults > $OUT/k_${TAG}_$w.json 2>$OUT/k_${TAG}_$w.err
done
python - <<PY >> $OUT/k_$TAG.log
import json
for w in ("n256", "n4096", "n1024x5"):
    try:
        d = [json.loads(l) for l in open("$OUT/k_${TAG}_" + w + ".json") if l.startswith("{")][0]
        print(w, "value %.2f G" % (d["value"] / 1e9), "step %.4f ms" % d["ms_per_step"],
              "kernel %.4f ms" % d["roofline"]["kernel_ms"], d["screen"], d["clocks"]["sm_mhz"])
    except Exception as e:
        print(w, "failed", e)
PY
