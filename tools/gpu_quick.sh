#!/bin/bash
# Quick GPU iteration (one gpurun call): GPU tests, smoke, cfg4/cfg2/cfg3 lines.
#   gpurun --timeout 900 -- bash tools/gpu_quick.sh [tag]
tag=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${tag}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
CFGS="${CFGS:-cfg4 cfg2 cfg2_p1.8 cfg3}" bash tools/cfgs.sh 2>&1 | tee gpurun_out/${tag}_cfgs.log
