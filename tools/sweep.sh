#!/bin/bash
# Repeat bench.py under a list of environment settings and print one summary
# line each:  tools/sweep.sh "FM_PF_TILES=0" "FM_PF_TILES=1" ...
# (extra bench.py flags via BENCH_ARGS)
mkdir -p gpurun_out
for setting in "$@"; do
  env $setting python bench.py ${BENCH_ARGS:---steps 30 --warmup 3 --no-cpu-baseline} \
    2>gpurun_out/sweep_err.log | python -c '
import json, sys
d = json.loads(sys.stdin.readline())
r = d.get("roofline", {})
print(sys.argv[1], "value", round(d["value"], 1), "ms", round(d["ms_per_step"], 4),
      "kernel_ms", r.get("kernel_ms"), "frac", r.get("frac"), "e2e", d.get("e2e", {}).get("value"))
' "$setting"
done
