#!/bin/bash
# --set full of the B=1 router row kernel in the default pipeline
cd "$GRAFT_REPO_ROOT"
P="python tools/profile_decode.py --layers 4 --steps 3 --policy adaptive --budget-frac 0.4 --bias 10000"
timeout 300 $P > gpurun_out/p5_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"router_route_row" -s 6 -c 1 -o gpurun_out/p5_router $P > gpurun_out/p5_ncu_router.log 2>&1
echo "rc=$?" >> gpurun_out/p5_ncu_router.log
