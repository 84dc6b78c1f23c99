for b in 8,8,4 4,8,8 8,4,8 16,4,4 4,16,4 4,4,16 16,8,2 2,8,16; do
  python bench.py --steps 30 --warmup 3 --no-cpu-baseline --box $b 2>gpurun_out/box_err_$b.log | python -c '
import json, sys
d = json.loads(sys.stdin.readline()); r = d["roofline"]; t = d["config"]["tiles"]
print(sys.argv[1], "ms", round(d["ms_per_step"], 4), "kernel_ms", round(r["kernel_ms"], 4), "cross", t["cross_entries"], "tiles", t["n_tiles"], "clo", t["closure_cap"])' $b
done
