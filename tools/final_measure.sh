#!/bin/bash
# Round-end measurement batch (one gpurun call): tests, smoke, the default
# bench line, extras, other configs, FD, minimizer, config-5 shards, reference
# arm, then the ncu launch list and the full capture of the dominant kernels.
#   gpurun --timeout 3600 -- bash tools/final_measure.sh [tag]
tag=${1:-f}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${tag}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/${tag}_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --steps 50 --warmup 5 --extras --no-cpu-baseline > gpurun_out/${tag}_extras.log 2>&1; echo "extras rc=$?"
CFGS="cfg1 cfg2 cfg2_p1.8 cfg3" bash tools/cfgs.sh > gpurun_out/${tag}_cfgs.log 2>&1; echo "cfgs rc=$?"
timeout 300 python tools/fd_time.py cfg1 cfg2 cfg2_p1.8 cfg3 cfg4 > gpurun_out/${tag}_fd.log 2>&1
timeout 300 python tools/tr_time.py cfg4 10 > gpurun_out/${tag}_tr.log 2>&1
timeout 900 python bench.py --config cfg5 --shard 1/8 --steps 20 --warmup 3 --extras --no-cpu-baseline > gpurun_out/${tag}_cfg5_8.log 2>&1; echo "cfg5/8 rc=$?"
timeout 900 python bench.py --config cfg5 --shard 2/4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_cfg5_4.log 2>&1; echo "cfg5/4 rc=$?"
timeout 1200 python bench.py --config cfg5 --shard 0/2 --steps 10 --warmup 3 --extras --descent-iters 20 --no-cpu-baseline > gpurun_out/${tag}_cfg5_2.log 2>&1; echo "cfg5/2 rc=$?"
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/${tag}_ref.log 2>&1; echo "ref rc=$?"
# ncu: launch list of a short bench run (evaluation kernels only), then the
# full set on the fused kernel + finishing pass and on the FD kernel
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:"k_tile|k_finish|k_energy|k_dot|k_finalize|k_cg|k_descent" -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${tag}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile_exact|k_finish_cross" \
  -s 2 -c 2 -o gpurun_out/${tag}_exact python tools/exact_once.py cfg4 3 > gpurun_out/${tag}_ncu_exact.log 2>&1; echo "ncu exact rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_exact \
  -s 1 -c 1 -o gpurun_out/${tag}_fd python tools/fd_once.py cfg4 2 > gpurun_out/${tag}_ncu_fd.log 2>&1; echo "ncu fd rc=$?"
