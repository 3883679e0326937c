#!/bin/bash
# Compare k_sweep_tc3 instances (COSCHED_TC_KIND, 0xV3GS) on the bench workloads.
#   bash tools/kinds.sh TAG KIND [KIND ...]
TAG=$1; shift; OUT=gpurun_out; mkdir -p $OUT
for k in "$@"; do
  for w in n256 n4096; do
    COSCHED_TC_KIND=$k timeout 300 python bench.py --workload $w --steps 200 --warmup 10 --no-cpu-baseline --no-e2e --no-subresults > $OUT/kd_${TAG}_${k}_$w.json 2>$OUT/kd_${TAG}_${k}_$w.err
  done
done
python - "$TAG" "$@" <<'PY' > $OUT/kd_$TAG.log
import json, sys
tag, kinds = sys.argv[1], sys.argv[2:]
for k in kinds:
    for w in ("n256", "n4096"):
        try:
            d = [json.loads(l) for l in open(f"gpurun_out/kd_{tag}_{k}_{w}.json") if l.startswith("{")][0]
            print(k, w, "value %.2f G" % (d["value"] / 1e9), "step %.4f ms" % d["ms_per_step"],
                  "kernel %.4f ms" % d["roofline"]["kernel_ms"], d["screen"]["verify_fail"], d["clocks"]["sm_mhz"])
        except Exception as e:
            print(k, w, "failed", e)
PY
cat $OUT/kd_$TAG.log
