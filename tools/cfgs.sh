#!/bin/bash
# one summary line per config: ms/step, tile-kernel ms, roofline fractions, launch shape
for c in ${CFGS:-cfg2 cfg2_p1.8 cfg3 cfg4}; do
  timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>gpurun_out/cfg_err_$c.log | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; t=d['config']['tiles']; print('$c', round(d['ms_per_step'],4), round(r['kernel_ms'],4), round(r['frac'],3), round(r['step_frac'],3), t['ctas_per_sm'], t['node_bufs'], t['table_bufs'])"
done
