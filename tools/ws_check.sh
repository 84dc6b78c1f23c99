#!/bin/bash
# A/B of the warp-specialised fused kernel experiment (fm_eval_ws.cu, compiled
# only into lib/libfemmin_ws.so with -DFM_WS_KERNEL=1 and selected there with
# FM_WS=1) against the product kernel k_tile_exact: gradients compared
# bitwise, both timed; every child under a timeout (a barrier-protocol bug
# would hang the kernel).  Build the variant beforehand (CPU box):
#   python -c "from paper_2109_01158_b200 import build as B; B.build_variant('ws', ['-DFM_WS_KERNEL=1'])"
mkdir -p gpurun_out
for c in ${CFGS:-cfg1 cfg3 cfg4 cfg2}; do
  echo "== $c"
  timeout ${T:-300} python tools/variant_time.py --config $c --n ${N:-50} lib=product lib=ws:FM_WS=1 || echo "rc=$? ($c)"
done
