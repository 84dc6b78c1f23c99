#!/bin/bash
# Round-end measurement batch (one gpurun call): tests, smoke, the default
# bench line, extras, other configs, config-5 shards, reference arm.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/f_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/f_bench.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py --steps 50 --warmup 5 --extras --no-cpu-baseline > gpurun_out/f_extras.log 2>&1; echo "extras rc=$?"
CFGS="cfg1 cfg2 cfg2_p1.8 cfg3" bash tools/cfgs.sh > gpurun_out/f_cfgs.log 2>&1; echo "cfgs rc=$?"
timeout 300 python tools/fd_time.py cfg1 cfg2 cfg3 > gpurun_out/f_fd.log 2>&1
timeout 900 python bench.py --config cfg5 --shard 1/8 --steps 20 --warmup 3 --extras --no-cpu-baseline > gpurun_out/f_cfg5_8.log 2>&1; echo "cfg5/8 rc=$?"
timeout 900 python bench.py --config cfg5 --shard 1/4 --steps 10 --warmup 3 --extras --descent-iters 20 --no-cpu-baseline > gpurun_out/f_cfg5_4.log 2>&1; echo "cfg5/4 rc=$?"
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/f_ref.log 2>&1; echo "ref rc=$?"
